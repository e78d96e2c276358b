// tcgen05 BMU screen (sm_100a): r_ij = c_j + m * (Xh_i . Wh_j) on 5th-gen
// tensor cores, with the per-row candidate window fused into the epilogue so
// the N x K distance matrix never leaves the SM.
//
// Persistent CTAs, one per SM, warp-specialised:
//   warp 0      TMA producer: A = 128 data rows x 64 features, B = 256 nodes x
//               64 features (fp16, SWIZZLE_128B, K-major) into a 4-stage ring
//   warp 1      TMEM owner + single-thread tcgen05.mma.cta_group::1.kind::f16
//               (M=128, N=256, K=16), fp32 accumulators in TMEM, two 256-col
//               accumulator stages (all 512 columns) so the epilogue of tile
//               t overlaps the MMAs of tile t+1
//   warps 2..9  epilogue: tcgen05.ld 32x32b.x32 -> r = fma(acc, m, c_j) ->
//               window candidate set (cand.cuh).  Warp w owns TMEM lane
//               quadrant w % 4 (rows 32(w%4)..+31) and column half (w-2)/4.
// A CTA sweeps all node tiles of one 128-row block before moving on, so each
// row's running minimum / candidate buffer lives in registers + smem for the
// whole sweep and is written out once.
#include <cuda.h>

#include "cand.cuh"

namespace somb {

constexpr int TC_BM = 128;         // rows per CTA tile (UMMA M)
constexpr int TC_BN = 256;         // nodes per tile (UMMA N)
constexpr int TC_BK = 64;          // fp16 features per stage (one 128B swizzle atom)
constexpr int TC_STAGES = 4;
constexpr int TC_UMMA_K = 16;
constexpr int TC_EPI_WARPS = 8;
constexpr int TC_THREADS = 32 * (2 + TC_EPI_WARPS);
constexpr int TC_HALF_CAP = SOMB_CAND_CAP / 2;   // candidates per (row, column half)
constexpr uint32_t TC_A_BYTES = TC_BM * TC_BK * 2;   // 16 KB
constexpr uint32_t TC_B_BYTES = TC_BN * TC_BK * 2;   // 32 KB
constexpr uint32_t TC_STAGE_BYTES = TC_A_BYTES + TC_B_BYTES;
constexpr uint32_t TC_CAND_BYTES = TC_EPI_WARPS * 32 * TC_HALF_CAP * 8;
constexpr uint32_t TC_SMEM = TC_STAGES * TC_STAGE_BYTES + TC_CAND_BYTES + 1024 /*align*/ + 256 /*barriers*/;

// ------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, uint32_t bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
        : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void tc_mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}

// K-major, SWIZZLE_128B smem matrix descriptor: 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);        // start address
    d |= (uint64_t)1 << 16;                        // LBO (ignored for swizzled K-major)
    d |= (uint64_t)(1024 >> 4) << 32;              // SBO = 1024 B
    d |= (uint64_t)1 << 46;                        // descriptor version (sm_100)
    d |= (uint64_t)2 << 61;                        // SWIZZLE_128B
    return d;
}

// kind::f16 instruction descriptor: A,B = f16, D = f32, both K-major, M=128, N=256
constexpr uint32_t TC_IDESC = (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(TC_BN >> 3) << 17) |
                              ((uint32_t)(TC_BM >> 4) << 24);

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// ------------------------------------------------------------------ kernel
__global__ void __launch_bounds__(TC_THREADS, 1)
screen_tc_kernel(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_w,
                 int64_t n, int dp, int kp, const float *__restrict__ c, const float *__restrict__ xnorm,
                 const float *__restrict__ scal, float wcoef, const float *__restrict__ thr0,
                 int *__restrict__ cand, int *__restrict__ ccount, int *__restrict__ flags,
                 float *__restrict__ dump) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *sA = smem;                                     // [stage][16 KB]
    uint8_t *sB = smem + TC_STAGES * TC_A_BYTES;            // [stage][32 KB]
    float *cbv = (float *)(smem + TC_STAGES * TC_STAGE_BYTES);
    int *cbi = (int *)(cbv + TC_EPI_WARPS * 32 * TC_HALF_CAP);
    uint64_t *bars = (uint64_t *)(smem + TC_STAGES * TC_STAGE_BYTES + TC_CAND_BYTES);
    // bars: full[S] empty[S] tfull[2] tempty[2]; then the TMEM base address
    uint32_t *tmem_slot = (uint32_t *)(bars + 2 * TC_STAGES + 4);

    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + TC_STAGES);
    const uint32_t tfull0 = smem_u32(bars + 2 * TC_STAGES), tempty0 = smem_u32(bars + 2 * TC_STAGES + 2);

    if (threadIdx.x == 0) {
        for (int s = 0; s < TC_STAGES; ++s) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(empty0 + 8 * s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tfull0 + 8 * a, 1);
            mbar_init(tempty0 + 8 * a, 32 * TC_EPI_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_x)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_w)) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int num_rb = (int)((n + TC_BM - 1) / TC_BM);
    const int NT = kp / TC_BN;
    const int KB = (dp + TC_BK - 1) / TC_BK;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int rb = blockIdx.x; rb < num_rb; rb += gridDim.x) {
                for (int nt = 0; nt < NT; ++nt) {
                    for (int kb = 0; kb < KB; ++kb) {
                        mbar_wait(empty0 + 8 * stage, phase ^ 1);
                        const uint32_t fb = full0 + 8 * stage;
                        mbar_expect_tx(fb, TC_STAGE_BYTES);
                        tma_load_2d(smem_u32(sA + stage * TC_A_BYTES), &map_x, fb, kb * TC_BK, rb * TC_BM);
                        tma_load_2d(smem_u32(sB + stage * TC_B_BYTES), &map_w, fb, kb * TC_BK, nt * TC_BN);
                        if (++stage == TC_STAGES) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t aphase = 0;
            for (int rb = blockIdx.x; rb < num_rb; rb += gridDim.x) {
                for (int nt = 0; nt < NT; ++nt) {
                    mbar_wait(tempty0 + 8 * acc, aphase ^ 1);
                    tc_fence_after();
                    const uint32_t d_tmem = tmem_base + (uint32_t)(acc * TC_BN);
                    for (int kb = 0; kb < KB; ++kb) {
                        mbar_wait(full0 + 8 * stage, phase);
                        tc_fence_after();
                        const uint32_t a0 = smem_u32(sA + stage * TC_A_BYTES);
                        const uint32_t b0 = smem_u32(sB + stage * TC_B_BYTES);
#pragma unroll
                        for (int k = 0; k < TC_BK / TC_UMMA_K; ++k) {
                            tc_mma_f16(d_tmem, sw128_desc(a0 + 32 * k), sw128_desc(b0 + 32 * k), TC_IDESC,
                                       (kb | k) != 0);
                        }
                        tc_commit(empty0 + 8 * stage);   // frees the smem slot when these MMAs retire
                        if (++stage == TC_STAGES) { stage = 0; phase ^= 1; }
                    }
                    tc_commit(tfull0 + 8 * acc);         // accumulator ready for the epilogue
                    if (++acc == 2) { acc = 0; aphase ^= 1; }
                }
            }
        }
    } else {
        // ---------------------------------------------------------- epilogue
        // Warp group `half` takes the 32-column chunks ch = half, half+2, ...
        // of each 256-node tile (interleaved so that a run of consecutive
        // nodes -- neighbours on the map -- spreads over both groups).
        const int ew = warp - 2;               // 0..7
        const int quad = warp & 3;             // TMEM lane quadrant this warp may access
        const int half = ew >> 2;
        const int et = ew * 32 + lane;         // buffer slot owner id
        const float m = scal[0];
        const float nmax = scal[1];
        const CandBuf cb{smem_u32(cbv + et), smem_u32(cbi + et), 4u * TC_EPI_WARPS * 32};
        int acc = 0;
        uint32_t aphase = 0;
        for (int rb = blockIdx.x; rb < num_rb; rb += gridDim.x) {
            const int64_t row = (int64_t)rb * TC_BM + quad * 32 + lane;
            const bool live = row < n;
            CandRow<TC_HALF_CAP> st;
            cand_init(st, live ? wcoef * xnorm[row] * nmax : 0.0f);
            if (live && thr0) st.thr = thr0[row];
            const bool dumping = dump != nullptr && live;
            for (int nt = 0; nt < NT; ++nt) {
                mbar_wait(tfull0 + 8 * acc, aphase);
                tc_fence_after();
                const uint32_t tbase = tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * TC_BN);
#pragma unroll 1
                for (int ch = half; ch < TC_BN / 32; ch += 2) {
                    float v[32];
                    tmem_ld32(tbase + ch * 32, v);
                    const int jc = nt * TC_BN + ch * 32;
                    const float4 *cp = reinterpret_cast<const float4 *>(c + jc);
                    float lo = INFINITY;
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        float4 cc = __ldg(cp + q);
                        v[4 * q + 0] = fmaf(v[4 * q + 0], m, cc.x);
                        v[4 * q + 1] = fmaf(v[4 * q + 1], m, cc.y);
                        v[4 * q + 2] = fmaf(v[4 * q + 2], m, cc.z);
                        v[4 * q + 3] = fmaf(v[4 * q + 3], m, cc.w);
                        lo = fminf(lo, fminf(fminf(v[4 * q], v[4 * q + 1]), fminf(v[4 * q + 2], v[4 * q + 3])));
                    }
                    if (dumping) {
#pragma unroll
                        for (int q = 0; q < 32; ++q) dump[row * kp + jc + q] = v[q];
                    }
                    if (live && lo <= st.thr) {
                        cand_bound(st, lo);   // the chunk minimum is about to be pushed
#pragma unroll
                        for (int q = 0; q < 32; ++q)
                            if (v[q] <= st.thr) cand_push<TC_HALF_CAP>(st, v[q], jc + q, cb);
                    }
                }
                tc_fence_before();
                mbar_arrive(tempty0 + 8 * acc);
                if (++acc == 2) { acc = 0; aphase ^= 1; }
            }
            if (live) {
                int *out = cand + row * SOMB_CAND_CAP + half * TC_HALF_CAP;
                int cnt = cand_emit<TC_HALF_CAP>(st, cb, out);
                // two halves write disjoint bytes of ccount / flags
                reinterpret_cast<uint8_t *>(ccount + row)[half] = (uint8_t)cnt;
                reinterpret_cast<uint8_t *>(flags + row)[half] = (uint8_t)st.trunc;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
    }
}

// --------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFn)p;
    }
    return fn;
}

static int make_map(CUtensorMap *map, const void *base, uint64_t inner, uint64_t outer, uint32_t box_outer) {
    EncodeTiledFn enc = get_encode();
    SOMB_REQUIRE(enc, SOMB_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {inner * 2};
    cuuint32_t box[2] = {(cuuint32_t)TC_BK, box_outer};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void *>(base), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    SOMB_REQUIRE(r == CUDA_SUCCESS, SOMB_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return SOMB_OK;
}

int launch_screen_tc(const __half *Xh, int64_t n, int dp, const __half *Wh, int kp, const float *c,
                     const float *xnorm, const float *scal, float wcoef, const float *thr0, int *cand,
                     int *ccount, int *flags, float *dump, cudaStream_t st) {
    SOMB_REQUIRE(dp % 8 == 0 && kp % TC_BN == 0, SOMB_E_INPUT, "screen_tc: dp %% 8 and kp %% 256 required");
    CUtensorMap mx, mw;
    int rc = make_map(&mx, Xh, (uint64_t)dp, (uint64_t)n, TC_BM);
    if (rc) return rc;
    rc = make_map(&mw, Wh, (uint64_t)dp, (uint64_t)kp, TC_BN);
    if (rc) return rc;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(screen_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM);
        if (e != cudaSuccess) return cuda_status(e, "screen_tc smem attribute");
        attr_set = true;
    }
    int dev = 0, sms = kSmCount;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaMemsetAsync(ccount, 0, (size_t)n * sizeof(int), st);
    cudaMemsetAsync(flags, 0, (size_t)n * sizeof(int), st);
    int num_rb = (int)((n + TC_BM - 1) / TC_BM);
    int grid = num_rb < sms ? num_rb : sms;
    screen_tc_kernel<<<grid, TC_THREADS, TC_SMEM, st>>>(mx, mw, n, dp, kp, c, xnorm, scal, wcoef, thr0, cand, ccount,
                                                        flags, dump);
    note_launch();
    SOMB_LAUNCH_CHECK("screen_tc");
    return SOMB_OK;
}

}  // namespace somb
