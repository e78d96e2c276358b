// tcgen05 BMU screen (sm_100a): r_ij = c_j + m * (Xh_i . Wh_j) on 5th-gen
// tensor cores, with the per-row candidate window fused into the epilogue so
// the N x K distance matrix never leaves the SM.
//
// Persistent, warp-specialised CTAs; template CG = CTA-group size:
//   CG = 2 (default): CTA pairs (cluster 2x1) run tcgen05.mma.cta_group::2
//     with M = 256 (128 data rows per CTA) x N = 256 nodes.  Each CTA
//     TMA-loads its own 128 rows and HALF (128 nodes) of every codebook tile,
//     so a pair moves 64 KB per 64-feature stage for 4.2M MACs -- one third
//     fewer operand bytes per MAC than CG = 1, which matters because the
//     screen is L2-bandwidth bound (profiles/).  Both CTAs' TMAs complete on
//     the leader's full barrier; the leader's single MMA thread issues the
//     pair MMA and multicasts its commits to both CTAs' empty / tmem-full
//     barriers; both epilogues release the accumulator on the leader's
//     tmem-empty barrier.
//   CG = 1: one CTA per SM, M = 128 x N = 256 (kept for A/B testing).
// Warp roles (per CTA):
//   warp 0      TMA producer (SWIZZLE_128B, K-major fp16 tiles, S-stage ring)
//   warp 1      TMEM owner (512 columns = two 256-column fp32 accumulator
//               stages, so the epilogue of tile t overlaps the MMAs of t+1);
//               lane 0 of the leader issues tcgen05.mma (K = 16 per op)
//   warps 2..9  epilogue: tcgen05.ld 32x32b.x32 -> r = fma(acc, m, c_j) ->
//               window candidate set (cand.cuh).  Warp w owns TMEM lane
//               quadrant w % 4 and the interleaved 32-column chunks
//               (w-2)/4, +2, +4, +6 of each tile.
// A CTA sweeps all node tiles of its rows before moving on, so each row's
// running minimum / candidate buffer lives in registers + smem for the whole
// sweep and is written out once.
#include <cuda.h>

#include <type_traits>

#include "cand.cuh"

namespace somb {

constexpr int TC_BN = 256;         // nodes per tile (UMMA N)
constexpr int TC_BK = 64;          // fp16 features per stage (one 128B swizzle atom)
constexpr int TC_UMMA_K = 16;
constexpr int TC_EPI_WARPS = 8;
constexpr int TC_THREADS = 32 * (2 + TC_EPI_WARPS);
constexpr int TC_ROWS = 128;                      // data rows per CTA (TMEM lanes)

// PASSES = 2: fp16 hi.hi plus the two cross terms hi.lo + lo.hi on the fp8
// (e4m3) tensor path at twice the fp16 rate: per tile, first the fp8 stages
// A8 = [x_hi8 | x_lo8] . B8 = [w_lo8 | w_hi8] (2 dp fp8 features, 128 per
// stage, accumulated from zero so their reduced-precision accumulation is
// relative to the small cross terms), then the fp16 stages on top
// (~2 fp16-pass equivalents instead of 3; error ~0.2 window units).
// PASSES = 1: fp16 operands; PASSES = 3: split operands (hi + lo residual),
// D += hi.hi + hi.lo + lo.hi (~22-bit operand precision, 3x the MMAs) for
// small feature counts where the 1-pass fp16 window holds too many
// near-tied nodes.  A stage holds [A_hi | B_hi | A_lo | B_lo].
// AR = 1: the CTA's data-row (A) operands stay resident in shared memory for
// a whole unit (all node tiles of its 128 rows); only codebook (B) tiles
// stream through the stage ring.  For K-chunk counts <= 4 (d <= 256 1-pass,
// d <= 128 2-pass), where A would otherwise be re-read from L2 per tile.
template <int CG, int PASSES = 1, int HC = SOMB_CAND_CAP / 2, int EPI = TC_EPI_WARPS, int AR = 0>
struct TcCfg {
    static constexpr int EPI_WARPS = EPI;                           // 8 (2 column groups) or 16 (4 groups)
    static constexpr int NGRP = EPI / 4;                            // column groups per row
    static constexpr int THREADS = 32 * (2 + EPI);
    static constexpr int B_ROWS = TC_BN / CG;                      // codebook rows per CTA (smem B tile)
    static constexpr uint32_t A_BYTES = TC_ROWS * TC_BK * 2;       // 16 KB
    static constexpr uint32_t B_BYTES = B_ROWS * TC_BK * 2;        // 32 KB (CG 1) / 16 KB (CG 2)
    static_assert(!AR || PASSES != 3, "A-resident mode: 1- or 2-pass");
    static constexpr uint32_t STAGE_BYTES = AR ? B_BYTES : (PASSES == 3 ? 2 : 1) * (A_BYTES + B_BYTES);
    static constexpr int A_CHUNKS = 4;                                 // resident A: <= 4 K-chunks
    static constexpr uint32_t ARES_BYTES = AR ? A_CHUNKS * A_BYTES : 0;
    // candidates kept per (row, column group): HC (<= SOMB_CAND_CAP / 2) in
    // shared memory; when a group's window holds more, its 3 HC / 4 lowest
    // screened (value, index) pairs are kept (cand.cuh)
    static constexpr int HALF_CAP = HC;
    static_assert(HC <= SOMB_CAND_CAP / 2, "column-group capacity exceeds the candidate list");
    static_assert(HC * NGRP <= SOMB_CAND_CAP, "candidate slots per row exceeded");
    static constexpr uint32_t CAND_BYTES = EPI * 32 * HALF_CAP * 8;
    // c_j of the tiles in flight: a ring of C_SLOTS 256-node slices (one per
    // TMEM accumulator stage), bulk-copied by the producer, read by the
    // epilogue as shared-memory broadcasts instead of L2 loads
    static constexpr int C_SLOTS = 2;
    static constexpr uint32_t C_BYTES = C_SLOTS * TC_BN * 4;
    static constexpr uint32_t BAR_BYTES = 256;
    // the dynamic shared window is 1024-byte aligned (declared __align__(1024),
    // checked at kernel start), so the whole opt-in maximum is usable
    static constexpr uint32_t SMEM_MAX = 232448;
    static constexpr int STAGES_RAW = (int)((SMEM_MAX - ARES_BYTES - CAND_BYTES - C_BYTES - BAR_BYTES) / STAGE_BYTES);
    static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
    static_assert(STAGES >= 2, "pipeline needs two stages");
    static constexpr uint32_t SMEM = ARES_BYTES + STAGES * STAGE_BYTES + CAND_BYTES + C_BYTES + BAR_BYTES;
    // kind::f16 instruction descriptor: A,B = f16, D = f32, K-major, M = 128 CG, N = 256
    static constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(TC_BN >> 3) << 17) | ((uint32_t)((128 * CG) >> 4) << 24);
};

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

__device__ __forceinline__ void mbar_arrive_local(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// arrive on the barrier at the same offset in cluster CTA `cta`.  Default
// (.release.cta) semantics: the arrive only has to order this thread's
// tcgen05.ld reads (tcgen05.fence::before_thread_sync does that), not its
// global stores -- the .release.cluster form compiled to MEMBAR.GPU + ERRBAR
// per tile and warp, 14% of the cfg5 epilogue's stall samples
// (profiles/r2_ncu_screen_cfg5_*.json).
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar, uint32_t cta) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(bar), "r"(cta));
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}

// 1-D bulk copy global -> this CTA's shared memory, completing on `bar`
__device__ __forceinline__ void bulk_load(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

template <int CG>
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, uint32_t bar, int c0, int c1) {
    if constexpr (CG == 1) {
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
            "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
            : "memory");
    } else {
        // the transaction bytes land on the LEADER CTA's barrier (peer bit cleared)
        asm volatile(
            "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
            "l"(reinterpret_cast<uint64_t>(map)), "r"(bar & 0xFEFFFFFFu), "r"(c0), "r"(c1)
            : "memory");
    }
}

// Same with an L2 cache policy (createpolicy): the CTA's own data rows are
// re-read for every node tile of its sweep, so they are loaded evict_last.
template <int CG>
__device__ __forceinline__ void tma_load_2d_hint(uint32_t dst, const CUtensorMap *map, uint32_t bar, int c0, int c1,
                                                 uint64_t pol) {
    if constexpr (CG == 1) {
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst),
            "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1), "l"(pol)
            : "memory");
    } else {
        asm volatile(
            "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst),
            "l"(reinterpret_cast<uint64_t>(map)), "r"(bar & 0xFEFFFFFFu), "r"(c0), "r"(c1), "l"(pol)
            : "memory");
    }
}

// CTA-pair TMA load multicast to the CTAs in `mask` (same smem offset in
// each); the transaction bytes land on each destination pair's leader barrier.
__device__ __forceinline__ void tma_load_2d_mc(uint32_t dst, const CUtensorMap *map, uint32_t bar, int c0, int c1,
                                               uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar & 0xFEFFFFFFu), "r"(c0), "r"(c1), "h"(mask)
        : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

template <int CG>
__device__ __forceinline__ void tc_commit(uint32_t bar, uint16_t mask = 0x3) {
    if constexpr (CG == 1) {
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
    } else {
        // multicast to the CTAs in `mask` (default: both CTAs of the pair), same barrier offset
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
            "h"(mask)
            : "memory");
    }
}

template <int CG>
__device__ __forceinline__ void tc_mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    if constexpr (CG == 1) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
            : "memory");
    } else {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
            : "memory");
    }
}

// kind::f8f6f4 (e4m3 x e4m3, f32 accumulate): K = 32 per op; the instruction
// descriptor bits equal the f16 one (a/b format 0 = E4M3, c format F32)
template <int CG>
__device__ __forceinline__ void tc_mma_f8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    if constexpr (CG == 1) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
            : "memory");
    } else {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
            : "memory");
    }
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

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// 0 = normal; profiling modes (SOMB_SCREEN_PROFILE or knob "screen_profile"):
// 1 = the epilogue releases accumulators without reading them (the TMA +
// tcgen05 feed alone), 2 = TMEM loads only, 3 = loads + window arithmetic
// without the candidate path.
__constant__ int g_profile_mode = 0;
// 1 = load the data-row (A) tiles with an L2 evict_last policy (SOMB_A_EVICT_LAST, default 0: measured no gain at cfg2)
__constant__ int g_a_evict_last = 0;

// ------------------------------------------------------------------ kernel
// MC = 2 (CG = 2 only): clusters of 4 CTAs = 2 pairs on different rows that
// sweep the same node tiles; each CTA TMA-loads half of its pair-half of the
// codebook tile and multicasts it to the same-rank CTA of the other pair, so
// the L2 -> SM codebook traffic halves (the screen is L2-bandwidth bound).
// Both pairs' MMAs must release a stage before it is refilled (empty
// barriers count MC arrivals).
template <int CG, int PASSES, int HC, int MC = 1, int EPI = TC_EPI_WARPS, int AR = 0>
__device__ __forceinline__ void screen_tc_body(const CUtensorMap *map_x, const CUtensorMap *map_w,
                                               const CUtensorMap *map_xl, const CUtensorMap *map_wl, int64_t n,
                                               int dp, int kp, const float *__restrict__ c,
                                               const float *__restrict__ xstat, const float *__restrict__ scal,
                                               float wcoef, const float *__restrict__ thr0, int *__restrict__ cand,
                                               int *__restrict__ ccount, int *__restrict__ flags,
                                               float *__restrict__ dump, unsigned *__restrict__ sync_ctr,
                                               int lag, OvfPool pool, int *__restrict__ ovf_head,
                                               float *__restrict__ ovf_lim) {
    using Cfg = TcCfg<CG, PASSES, HC, EPI, AR>;
    static_assert(!AR || MC == 1, "A-resident mode without codebook multicast");
    constexpr int S = Cfg::STAGES;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    if (smem_u32(smem_raw) & 1023u) __trap();   // SWIZZLE_128B tiles need 1024-byte alignment
    uint8_t *ares = smem_raw;                    // resident A chunks (AR)
    uint8_t *smem = smem_raw + Cfg::ARES_BYTES;  // stage ring
    // stage s: A_hi at smem + s*STAGE_BYTES, B_hi after it, then A_lo, B_lo (3-pass)
    float *cbv = (float *)(smem + S * Cfg::STAGE_BYTES);
    int *cbi = (int *)(cbv + EPI * 32 * Cfg::HALF_CAP);
    float *cring = (float *)(smem + S * Cfg::STAGE_BYTES + Cfg::CAND_BYTES);
    uint64_t *bars = (uint64_t *)(smem + S * Cfg::STAGE_BYTES + Cfg::CAND_BYTES + Cfg::C_BYTES);
    // bars: full[S] empty[S] tfull[2] tempty[2] cfull[C_SLOTS] cempty[C_SLOTS] afull aempty;
    // then the TMEM base address
    constexpr int CS = Cfg::C_SLOTS;
    uint32_t *tmem_slot = (uint32_t *)(bars + 2 * S + 4 + 2 * CS + 2);
    static_assert((2 * S + 4 + 2 * CS + 2) * 8 + 4 <= (int)Cfg::BAR_BYTES, "barrier area");

    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    const uint32_t cl_rank = CG == 2 ? cluster_rank() : 0;
    const uint32_t crank = cl_rank & 1u;            // rank within the CTA pair
    const uint32_t pair = cl_rank >> 1;             // pair within the cluster (MC = 2)
    const bool leader = crank == 0;
    const uint16_t pair_mask = (uint16_t)(0x3u << (2 * pair));
    const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + S);
    const uint32_t tfull0 = smem_u32(bars + 2 * S), tempty0 = smem_u32(bars + 2 * S + 2);
    const uint32_t cfull0 = smem_u32(bars + 2 * S + 4), cempty0 = smem_u32(bars + 2 * S + 4 + CS);
    const uint32_t afull = smem_u32(bars + 2 * S + 4 + 2 * CS), aempty = afull + 8;

    if (threadIdx.x == 0 && blockIdx.x == 0) sync_ctr[3] = Cfg::NGRP;   // candidate-list layout for the re-rank
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(full0 + 8 * s, 1);
            mbar_init(empty0 + 8 * s, MC);   // one MMA-commit arrival per pair sharing the stage
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tfull0 + 8 * a, 1);
            mbar_init(tempty0 + 8 * a, CG * EPI);   // one arrival per epilogue warp of the pair
        }
        for (int a = 0; a < CS; ++a) {
            mbar_init(cfull0 + 8 * a, 1);           // the producer's expect_tx
            mbar_init(cempty0 + 8 * a, EPI);        // one arrival per epilogue warp of this CTA
        }
        mbar_init(afull, 1);                        // resident A loaded (leader's expect_tx)
        mbar_init(aempty, 1);                       // the unit's last MMAs retired (leader's commit)
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map_x)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map_w)) : "memory");
    }
    if (warp == 1) {
        if constexpr (CG == 1) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        }
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (CG == 2) cluster_sync_all();   // peer barriers initialised before any remote arrive
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    // work unit: a block of 128*CG rows; this CTA owns rows [unit*128*CG + 128*crank, +128)
    const int unit_rows = TC_ROWS * CG;
    const int num_units = (int)((n + unit_rows - 1) / unit_rows);
    const int unit0 = blockIdx.x / CG, unit_step = gridDim.x / CG;
    // iterations: with MC = 2 both pairs of a cluster run the same count (the
    // later pair may process a zero-filled dummy unit at the tail)
    const int first_in_cluster = (blockIdx.x / (CG * MC)) * MC;
    const int iters = first_in_cluster < num_units ? (num_units - first_in_cluster + unit_step - 1) / unit_step : 0;
    const int NT = kp / TC_BN;
    const int KB = (dp + TC_BK - 1) / TC_BK;
    const int KB8 = PASSES == 2 ? (2 * dp + 127) / 128 : 0;   // fp8 cross-term stages (128 features each)

    if (warp == 0) {
        if (lane == 0) {
            const uint64_t pol_a = policy_evict_last();
            const bool hint_a = g_a_evict_last != 0;
            int stage = 0;
            uint32_t phase = 0;
            int cslot = 0;
            uint32_t cphase = 0;
            // soft lockstep (lag > 0): a CTA starts its g-th node tile only once
            // all CTAs together have issued P * (g - lag) tiles, so concurrent
            // CTAs sweep the same codebook tiles and share them in L2
            const unsigned P = gridDim.x;
            const int waves = (num_units + unit_step - 1) / unit_step;
            unsigned issued = 0;
            uint32_t arph = 0;
            for (int it = 0; it < (MC == 1 ? (unit0 < num_units ? (num_units - unit0 + unit_step - 1) / unit_step : 0) : iters); ++it) {
                const int u = unit0 + it * unit_step;
                const int row0 = u * unit_rows + TC_ROWS * (int)crank;
                if constexpr (AR) {   // this unit's A chunks, once (after the previous unit's MMAs retired)
                    mbar_wait(aempty, arph ^ 1);
                    if (leader) mbar_expect_tx(afull, CG * (KB8 + KB) * Cfg::A_BYTES);
                    for (int kb = 0; kb < KB8; ++kb)
                        tma_load_2d<CG>(smem_u32(ares + kb * Cfg::A_BYTES), map_xl, afull, kb * 128, row0);
                    for (int kb = 0; kb < KB; ++kb)
                        tma_load_2d<CG>(smem_u32(ares + (KB8 + kb) * Cfg::A_BYTES), map_x, afull, kb * TC_BK, row0);
                    arph ^= 1;
                }
                for (int nt = 0; nt < NT; ++nt) {
                    if (lag > 0 && issued > (unsigned)lag) {
                        const unsigned need = P * (issued - (unsigned)lag);
                        for (int spin = 0; spin < (1 << 20); ++spin) {
                            unsigned cur;
                            asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(sync_ctr) : "memory");
                            if (cur >= need) break;
                            __nanosleep(64);
                        }
                    }
                    const int node0 = nt * TC_BN + Cfg::B_ROWS * (int)crank;
                    // c_j slice of this tile into ring slot `cslot` (once the
                    // epilogue has finished the tile that used it before)
                    auto load_c = [&]() {
                        mbar_wait(cempty0 + 8 * cslot, cphase ^ 1);
                        mbar_expect_tx(cfull0 + 8 * cslot, TC_BN * 4);
                        bulk_load(smem_u32(cring + cslot * TC_BN), c + (size_t)nt * TC_BN, TC_BN * 4, cfull0 + 8 * cslot);
                        if (++cslot == CS) { cslot = 0; cphase ^= 1; }
                    };
                    for (int kb = 0; kb < KB8; ++kb) {   // PASSES == 2: fp8 cross terms first
                        mbar_wait(empty0 + 8 * stage, phase ^ 1);
                        const uint32_t fb = full0 + 8 * stage;
                        if (leader) mbar_expect_tx(fb, CG * Cfg::STAGE_BYTES);
                        uint8_t *st0 = smem + stage * Cfg::STAGE_BYTES;
                        if constexpr (AR) {
                            tma_load_2d<CG>(smem_u32(st0), map_wl, fb, kb * 128, node0);
                        } else if constexpr (MC == 1) {
                            tma_load_2d<CG>(smem_u32(st0), map_xl, fb, kb * 128, row0);
                            tma_load_2d<CG>(smem_u32(st0 + Cfg::A_BYTES), map_wl, fb, kb * 128, node0);
                        } else {
                            tma_load_2d<CG>(smem_u32(st0), map_xl, fb, kb * 128, row0);
                            const uint32_t sub = (uint32_t)pair * (Cfg::B_BYTES / 2);
                            const uint16_t mcm = (uint16_t)((1u << crank) | (1u << (crank + 2)));
                            tma_load_2d_mc(smem_u32(st0 + Cfg::A_BYTES + sub), map_wl, fb, kb * 128,
                                           node0 + (Cfg::B_ROWS / 2) * (int)pair, mcm);
                        }
                        if (++stage == S) { stage = 0; phase ^= 1; }
                    }
                    for (int kb = 0; kb < KB; ++kb) {
                        mbar_wait(empty0 + 8 * stage, phase ^ 1);
                        const uint32_t fb = full0 + 8 * stage;
                        if (leader) mbar_expect_tx(fb, CG * Cfg::STAGE_BYTES);
                        uint8_t *st0 = smem + stage * Cfg::STAGE_BYTES;
                        if constexpr (!AR) {
                            if (hint_a)
                                tma_load_2d_hint<CG>(smem_u32(st0), map_x, fb, kb * TC_BK, row0, pol_a);
                            else
                                tma_load_2d<CG>(smem_u32(st0), map_x, fb, kb * TC_BK, row0);
                        }
                        if constexpr (AR) {
                            tma_load_2d<CG>(smem_u32(st0), map_w, fb, kb * TC_BK, node0);
                        } else if constexpr (MC == 1) {
                            tma_load_2d<CG>(smem_u32(st0 + Cfg::A_BYTES), map_w, fb, kb * TC_BK, node0);
                        } else {   // my sub-box of the pair-half, multicast to the same rank of both pairs
                            const uint32_t sub = (uint32_t)pair * (Cfg::B_BYTES / MC);
                            const uint16_t mcm = (uint16_t)((1u << crank) | (1u << (crank + 2)));
                            tma_load_2d_mc(smem_u32(st0 + Cfg::A_BYTES + sub), map_w, fb, kb * TC_BK,
                                           node0 + (Cfg::B_ROWS / MC) * (int)pair, mcm);
                        }
                        if constexpr (PASSES == 3) {
                            tma_load_2d<CG>(smem_u32(st0 + Cfg::A_BYTES + Cfg::B_BYTES), map_xl, fb, kb * TC_BK, row0);
                            if constexpr (MC == 1) {
                                tma_load_2d<CG>(smem_u32(st0 + 2 * Cfg::A_BYTES + Cfg::B_BYTES), map_wl, fb, kb * TC_BK,
                                                node0);
                            } else {
                                const uint32_t sub = (uint32_t)pair * (Cfg::B_BYTES / MC);
                                const uint16_t mcm = (uint16_t)((1u << crank) | (1u << (crank + 2)));
                                tma_load_2d_mc(smem_u32(st0 + 2 * Cfg::A_BYTES + Cfg::B_BYTES + sub), map_wl, fb,
                                               kb * TC_BK, node0 + (Cfg::B_ROWS / MC) * (int)pair, mcm);
                            }
                        }
                        if (++stage == S) { stage = 0; phase ^= 1; }
                        if (kb == KB - 1) load_c();   // issued with the tile's last stage: the slot is free by then
                    }
                    ++issued;
                    if (lag > 0) atomicAdd(sync_ctr, 1u);
                }
            }
            // CTAs with fewer waves credit their missing tiles so nobody waits on them
            if (lag > 0) {
                const unsigned total = (unsigned)waves * (unsigned)NT;
                if (total > issued) atomicAdd(sync_ctr, total - issued);
            }
        }
    } else if (warp == 1) {
        if (leader && lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t aphase = 0;
            const int my_iters = MC == 1 ? (unit0 < num_units ? (num_units - unit0 + unit_step - 1) / unit_step : 0) : iters;
            uint32_t arph = 0;
            for (int it = 0; it < my_iters; ++it) {
                if constexpr (AR) {   // this unit's resident A chunks have landed (both CTAs)
                    mbar_wait(afull, arph);
                    tc_fence_after();
                    arph ^= 1;
                }
                for (int nt = 0; nt < NT; ++nt) {
                    mbar_wait(tempty0 + 8 * acc, aphase ^ 1);
                    tc_fence_after();
                    const uint32_t d_tmem = tmem_base + (uint32_t)(acc * TC_BN);
                    for (int kb = 0; kb < KB8; ++kb) {   // fp8 cross terms, accumulated from zero
                        mbar_wait(full0 + 8 * stage, phase);
                        tc_fence_after();
                        const uint32_t a0 = AR ? smem_u32(ares + kb * Cfg::A_BYTES) : smem_u32(smem + stage * Cfg::STAGE_BYTES);
                        const uint32_t b0 = AR ? smem_u32(smem + stage * Cfg::STAGE_BYTES) : a0 + Cfg::A_BYTES;
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            tc_mma_f8<CG>(d_tmem, sw128_desc(a0 + 32 * k), sw128_desc(b0 + 32 * k), Cfg::IDESC,
                                          (kb | k) != 0);
                        tc_commit<CG>(empty0 + 8 * stage, MC == 1 ? (uint16_t)0x3 : (uint16_t)0xF);
                        if (++stage == S) { stage = 0; phase ^= 1; }
                    }
                    for (int kb = 0; kb < KB; ++kb) {
                        mbar_wait(full0 + 8 * stage, phase);
                        tc_fence_after();
                        const uint32_t a0 = AR ? smem_u32(ares + (KB8 + kb) * Cfg::A_BYTES)
                                               : smem_u32(smem + stage * Cfg::STAGE_BYTES);
                        const uint32_t b0 = AR ? smem_u32(smem + stage * Cfg::STAGE_BYTES) : a0 + Cfg::A_BYTES;
#pragma unroll
                        for (int k = 0; k < TC_BK / TC_UMMA_K; ++k) {
                            tc_mma_f16<CG>(d_tmem, sw128_desc(a0 + 32 * k), sw128_desc(b0 + 32 * k), Cfg::IDESC,
                                           (KB8 > 0 || (kb | k) != 0) ? 1u : 0u);
                            if constexpr (PASSES == 3) {
                                const uint32_t al = b0 + Cfg::B_BYTES, bl = al + Cfg::A_BYTES;
                                tc_mma_f16<CG>(d_tmem, sw128_desc(a0 + 32 * k), sw128_desc(bl + 32 * k), Cfg::IDESC, 1);
                                tc_mma_f16<CG>(d_tmem, sw128_desc(al + 32 * k), sw128_desc(b0 + 32 * k), Cfg::IDESC, 1);
                            }
                        }
                        tc_commit<CG>(empty0 + 8 * stage, MC == 1 ? (uint16_t)0x3 : (uint16_t)0xF);   // frees the smem slot(s) (of both pairs with MC = 2) when these MMAs retire
                        if (++stage == S) { stage = 0; phase ^= 1; }
                    }
                    tc_commit<CG>(tfull0 + 8 * acc, pair_mask);   // accumulator ready for the pair's epilogues
                    if (++acc == 2) { acc = 0; aphase ^= 1; }
                }
                if constexpr (AR) tc_commit<CG>(aempty, (uint16_t)0x3);   // both CTAs may reload A once these retire
            }
        }
    } else {
        // ---------------------------------------------------------- epilogue
        // Warp group `half` (column group 0..NGRP-1) takes the 32-column
        // chunks ch = half, half+NGRP, ... of each 256-node tile (interleaved
        // so that a run of consecutive nodes -- neighbours on the map --
        // spreads over the groups).  (16 epilogue warps / 4 groups were
        // measured slower at cfg5: register spills at 576 threads.)
        const int ew = warp - 2;               // 0..EPI-1
        const int quad = warp & 3;             // TMEM lane quadrant this warp may access
        const int half = ew >> 2;
        const int et = ew * 32 + lane;         // buffer slot owner id
        constexpr int GS = SOMB_CAND_CAP / Cfg::NGRP;   // candidate slots per group
        const float m = scal[0];
        const CandBuf cb{smem_u32(cbv + et), smem_u32(cbi + et), 4u * EPI * 32};
        int acc = 0;
        uint32_t aphase = 0;
        int cslot = 0;
        uint32_t cphase = 0;
        const int my_iters = MC == 1 ? (unit0 < num_units ? (num_units - unit0 + unit_step - 1) / unit_step : 0) : iters;
        for (int it = 0; it < my_iters; ++it) {
            const int u = unit0 + it * unit_step;
            const int64_t row = (int64_t)u * unit_rows + TC_ROWS * crank + quad * 32 + lane;
            const bool live = row < n;
            CandRow<Cfg::HALF_CAP> st;
            cand_init(st, live ? wcoef * screen_sigma(reinterpret_cast<const float4 *>(xstat)[row], scal) : 0.0f);
            if (live && thr0) st.thr = thr0[row];
            const bool dumping = dump != nullptr && live;
            for (int nt = 0; nt < NT; ++nt) {
                mbar_wait(tfull0 + 8 * acc, aphase);
                tc_fence_after();
                mbar_wait(cfull0 + 8 * cslot, cphase);
                const float *cs = cring + cslot * TC_BN;
                if (g_profile_mode == 1) {   // profiling: release the accumulator untouched
                    __syncwarp();
                    if (lane == 0) {
                        if (CG == 1 || leader) mbar_arrive_local(tempty0 + 8 * acc);
                        else mbar_arrive_cluster(tempty0 + 8 * acc, cl_rank & ~1u);
                        mbar_arrive_local(cempty0 + 8 * cslot);
                    }
                    if (++acc == 2) { acc = 0; aphase ^= 1; }
                    if (++cslot == CS) { cslot = 0; cphase ^= 1; }
                    continue;
                }
                const uint32_t tbase = tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * TC_BN);
                // one 32-column chunk: r = fma(acc, m, c_j), 8-wide group minima,
                // then the window candidate path
                // one 32-column chunk: r = fma(acc, m, c_j) and the 8-wide group
                // minima (arith), then the window candidate path (cands)
                auto arith = [&](float (&v)[32], int ch, float (&gmin)[4]) {
                    const float4 *cp = reinterpret_cast<const float4 *>(cs + ch * 32);
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        float4 cc = cp[q];
                        v[4 * q + 0] = fmaf(v[4 * q + 0], m, cc.x);
                        v[4 * q + 1] = fmaf(v[4 * q + 1], m, cc.y);
                        v[4 * q + 2] = fmaf(v[4 * q + 2], m, cc.z);
                        v[4 * q + 3] = fmaf(v[4 * q + 3], m, cc.w);
                        float l4 = fminf(fminf(v[4 * q], v[4 * q + 1]), fminf(v[4 * q + 2], v[4 * q + 3]));
                        gmin[q >> 1] = (q & 1) ? fminf(gmin[q >> 1], l4) : l4;
                    }
                };
                auto cands = [&](const float (&v)[32], int ch, const float (&gmin)[4]) {
                    const int jc = nt * TC_BN + ch * 32;
                    if (dumping) {
#pragma unroll
                        for (int q = 0; q < 32; ++q) dump[row * kp + jc + q] = v[q];
                    }
                    const float lo = fminf(fminf(gmin[0], gmin[1]), fminf(gmin[2], gmin[3]));
                    if (g_profile_mode == 3) {   // profiling: loads + window arithmetic, no candidate path
                        if (__float_as_uint(lo) == 0x7fc00001u) flags[0] = 1;
                        return;
                    }
                    if (live && lo <= st.thr) {
                        cand_bound(st, lo);   // the chunk minimum is about to be pushed
#pragma unroll
                        for (int g8 = 0; g8 < 4; ++g8) {
                            if (gmin[g8] <= st.thr) {
#pragma unroll
                                for (int q = 8 * g8; q < 8 * g8 + 8; ++q)
                                    if (v[q] <= st.thr) cand_push<Cfg::HALF_CAP>(st, v[q], jc + q, cb, pool);
                            }
                        }
                    }
                };
                auto tmem_only = [&](const float (&v)[32]) {   // profiling mode 2: TMEM loads only
                    float t = v[0];
#pragma unroll
                    for (int q = 1; q < 32; ++q) t = fminf(t, v[q]);
                    if (__float_as_uint(t) == 0x7fc00001u) flags[0] = 1;   // never: keeps the loads
                };
                // Each chunk's TMEM load is waited for at once: keeping the next
                // chunk's load in flight while this one is processed (double-
                // buffered registers) was measured much slower (cfg4 screen
                // 135 -> 226 ms, cfg5 530 -> 626 ms, tools/ab.sh), and so was
                // loading two chunks back to back with one wait and interleaving
                // their arithmetic (cfg4 135 -> 169 ms): longer or overlapping
                // tcgen05.ld traffic holds up the MMAs on the same SM.  (A 16-warp
                // epilogue does not launch: 576 threads exceed the 512 the driver
                // allows this kernel, cudaFuncGetAttributes.)
#pragma unroll 1
                for (int ch = half; ch < TC_BN / 32; ch += Cfg::NGRP) {
                    float v[32], g[4];
                    tmem_ld32(tbase + ch * 32, v);
                    if (g_profile_mode == 2) { tmem_only(v); continue; }
                    arith(v, ch, g);
                    cands(v, ch, g);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (CG == 1 || leader) mbar_arrive_local(tempty0 + 8 * acc);
                    else mbar_arrive_cluster(tempty0 + 8 * acc, cl_rank & ~1u);
                    mbar_arrive_local(cempty0 + 8 * cslot);
                }
                if (++acc == 2) { acc = 0; aphase ^= 1; }
                if (++cslot == CS) { cslot = 0; cphase ^= 1; }
            }
            if (live) {
                int *out = cand + row * SOMB_CAND_CAP + half * GS;
                int cnt = cand_emit<Cfg::HALF_CAP>(st, cb, out);
                // the column groups write disjoint bytes of ccount / flags
                reinterpret_cast<uint8_t *>(ccount + row)[half] = (uint8_t)cnt;
                reinterpret_cast<uint8_t *>(flags + row)[half] = (uint8_t)st.trunc;
                ovf_head[4 * row + half] = st.head;
                ovf_lim[4 * row + half] = st.rmin + st.win;
                if (Cfg::NGRP == 2) ovf_head[4 * row + 2 + half] = -1;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (CG == 2) cluster_sync_all();      // no CTA leaves while its peer's MMAs may target it
    if (warp == 1) {
        tc_fence_after();
        if constexpr (CG == 1)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
        else
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
    }
}

#define SCREEN_TC_ARGS                                                                                              \
    const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_w,                           \
        const __grid_constant__ CUtensorMap map_xl, const __grid_constant__ CUtensorMap map_wl, int64_t n, int dp, int kp, \
        const float *__restrict__ c, const float *__restrict__ xstat, const float *__restrict__ scal, float wcoef,  \
        const float *__restrict__ thr0, int *__restrict__ cand, int *__restrict__ ccount, int *__restrict__ flags,  \
        float *__restrict__ dump, unsigned *__restrict__ sync_ctr, int lag, OvfPool pool, int *__restrict__ ovf_head, \
        float *__restrict__ ovf_lim

template <int P, int HC>
__global__ void __launch_bounds__(TC_THREADS, 1) screen_tc1_kernel(SCREEN_TC_ARGS) {
    screen_tc_body<1, P, HC>(&map_x, &map_w, &map_xl, &map_wl, n, dp, kp, c, xstat, scal, wcoef, thr0, cand, ccount,
                             flags, dump, sync_ctr, lag, pool, ovf_head, ovf_lim);
}

template <int P, int HC>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(TC_THREADS, 1) screen_tc4_kernel(SCREEN_TC_ARGS) {
    screen_tc_body<2, P, HC, 2>(&map_x, &map_w, &map_xl, &map_wl, n, dp, kp, c, xstat, scal, wcoef, thr0, cand, ccount,
                                flags, dump, sync_ctr, lag, pool, ovf_head, ovf_lim);
}

template <int P, int HC>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TC_THREADS, 1) screen_tc2a_kernel(SCREEN_TC_ARGS) {
    screen_tc_body<2, P, HC, 1, TC_EPI_WARPS, 1>(&map_x, &map_w, &map_xl, &map_wl, n, dp, kp, c, xstat, scal, wcoef,
                                                 thr0, cand, ccount, flags, dump, sync_ctr, lag, pool, ovf_head,
                                                 ovf_lim);
}

template <int P, int HC>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TC_THREADS, 1) screen_tc2_kernel(SCREEN_TC_ARGS) {
    screen_tc_body<2, P, HC>(&map_x, &map_w, &map_xl, &map_wl, n, dp, kp, c, xstat, scal, wcoef, thr0, cand, ccount,
                             flags, dump, sync_ctr, lag, pool, ovf_head, ovf_lim);
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

// 2-D K-major map with 128-byte inner boxes: fp16 (64 elements) or, with
// u8 = true, fp8 bytes (128 elements)
static int make_map(CUtensorMap *map, const void *base, uint64_t inner, uint64_t outer, uint32_t box_outer,
                    bool u8 = false) {
    EncodeTiledFn enc = get_encode();
    SOMB_REQUIRE(enc, SOMB_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {inner * (u8 ? 1 : 2)};
    cuuint32_t box[2] = {(cuuint32_t)(u8 ? 128 : TC_BK), box_outer};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(map, u8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2,
                     const_cast<void *>(base), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    SOMB_REQUIRE(r == CUDA_SUCCESS, SOMB_E_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return SOMB_OK;
}

static int g_tc_group = 2;   // SOMB_TC_GROUP=1 selects the single-CTA variant (A/B testing)
static int g_half_cap = 32;  // SOMB_HALF_CAP = 8 | 16 | 32: candidates kept per (row, column group)
static int g_lag = 8;        // SOMB_SCREEN_LAG: soft lockstep of the CTAs' codebook sweeps (0 = off)
static int g_mc = 2;         // SOMB_TC_MULTICAST: 2 = 4-CTA clusters multicasting the codebook tiles (1-pass screen), 1 = off
static int g_ares = 1;       // SOMB_A_RESIDENT / knob "a_resident": data-row operands resident per unit (<= 4 K-chunks;
                             // cfg4 screen 125 -> 107 ms, cfg5 536 -> 510 ms, tools/r2_ar.sh)

template <class KernelT>
static int set_smem(KernelT k, uint32_t bytes, const char *what) {
    cudaError_t r = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    return r == cudaSuccess ? SOMB_OK : cuda_status(r, what);
}

static int screen_tc_init() {
    static bool init = false;
    if (init) return SOMB_OK;
    const char *e = getenv("SOMB_TC_GROUP");
    if (e && atoi(e) == 1) g_tc_group = 1;
    const char *hc = getenv("SOMB_HALF_CAP");
    if (hc) g_half_cap = atoi(hc) <= 8 ? 8 : atoi(hc) <= 16 ? 16 : 32;
    const char *lg = getenv("SOMB_SCREEN_LAG");
    if (lg) g_lag = atoi(lg);
    const char *mc = getenv("SOMB_TC_MULTICAST");
    if (mc) g_mc = atoi(mc) == 2 ? 2 : 1;
    const char *ar = getenv("SOMB_A_RESIDENT");
    if (ar) g_ares = atoi(ar) != 0;
    const char *pm = getenv("SOMB_SCREEN_PROFILE");
    int mode = pm ? atoi(pm) : 0;
    cudaMemcpyToSymbol(g_profile_mode, &mode, sizeof(int));
    const char *ae = getenv("SOMB_A_EVICT_LAST");
    int a_last = ae ? atoi(ae) : 0;
    cudaMemcpyToSymbol(g_a_evict_last, &a_last, sizeof(int));
    int rc = set_smem(screen_tc1_kernel<1, 16>, TcCfg<1, 1, 16>::SMEM, "screen_tc1 smem");
    if (!rc) rc = set_smem(screen_tc1_kernel<3, 16>, TcCfg<1, 3, 16>::SMEM, "screen_tc1x3 smem");
    if (!rc) rc = set_smem(screen_tc2_kernel<1, 8>, TcCfg<2, 1, 8>::SMEM, "screen_tc2 smem");
    if (!rc) rc = set_smem(screen_tc2_kernel<1, 16>, TcCfg<2, 1, 16>::SMEM, "screen_tc2 smem");
    if (!rc) rc = set_smem(screen_tc2_kernel<1, 32>, TcCfg<2, 1, 32>::SMEM, "screen_tc2 smem");
    if (!rc) rc = set_smem(screen_tc2_kernel<3, 8>, TcCfg<2, 3, 8>::SMEM, "screen_tc2x3 smem");
    if (!rc) rc = set_smem(screen_tc2_kernel<3, 16>, TcCfg<2, 3, 16>::SMEM, "screen_tc2x3 smem");
    if (!rc) rc = set_smem(screen_tc2_kernel<3, 32>, TcCfg<2, 3, 32>::SMEM, "screen_tc2x3 smem");
    if (!rc) rc = set_smem(screen_tc2_kernel<2, 32>, TcCfg<2, 2, 32>::SMEM, "screen_tc2x2 smem");
    if (!rc) rc = set_smem(screen_tc2_kernel<2, 16>, TcCfg<2, 2, 16>::SMEM, "screen_tc2x2 smem");
    if (!rc) rc = set_smem(screen_tc2a_kernel<1, 32>, TcCfg<2, 1, 32, TC_EPI_WARPS, 1>::SMEM, "screen_tc2a smem");
    if (!rc) rc = set_smem(screen_tc2a_kernel<2, 32>, TcCfg<2, 2, 32, TC_EPI_WARPS, 1>::SMEM, "screen_tc2a smem");
    if (!rc) rc = set_smem(screen_tc2a_kernel<1, 16>, TcCfg<2, 1, 16, TC_EPI_WARPS, 1>::SMEM, "screen_tc2a smem");
    if (!rc) rc = set_smem(screen_tc2a_kernel<2, 16>, TcCfg<2, 2, 16, TC_EPI_WARPS, 1>::SMEM, "screen_tc2a smem");
    if (!rc) rc = set_smem(screen_tc4_kernel<1, 32>, TcCfg<2, 1, 32>::SMEM, "screen_tc4 smem");
    if (!rc) rc = set_smem(screen_tc4_kernel<2, 32>, TcCfg<2, 2, 32>::SMEM, "screen_tc4x2 smem");
    if (!rc) rc = set_smem(screen_tc4_kernel<3, 32>, TcCfg<2, 3, 32>::SMEM, "screen_tc4x3 smem");
    if (rc) return rc;
    init = true;
    return SOMB_OK;
}

// runtime tuning knobs (somb_set_knob): "screen_lag", "screen_profile", "half_cap", "tc_group"
int screen_tc_set_knob(const char *key, int value) {
    int rc = screen_tc_init();
    if (rc) return rc;
    if (!strcmp(key, "screen_lag")) { g_lag = value; return SOMB_OK; }
    if (!strcmp(key, "half_cap")) { g_half_cap = value <= 8 ? 8 : value <= 16 ? 16 : 32; return SOMB_OK; }
    if (!strcmp(key, "tc_group")) { g_tc_group = value == 1 ? 1 : 2; return SOMB_OK; }
    if (!strcmp(key, "tc_multicast")) { g_mc = value == 2 ? 2 : 1; return SOMB_OK; }
    if (!strcmp(key, "a_resident")) { g_ares = value != 0; return SOMB_OK; }
    if (!strcmp(key, "screen_profile")) {
        cudaError_t r = cudaMemcpyToSymbol(g_profile_mode, &value, sizeof(int));
        return r == cudaSuccess ? SOMB_OK : cuda_status(r, "set screen_profile");
    }
    return SOMB_E_CONFIG;
}

int launch_screen_tc(const __half *Xh, const __half *Xl, int64_t n, int dp, const __half *Wh, const __half *Wl, int kp,
                     const float *c, const float *xstat, const float *scal, float wcoef, const float *thr0, int *cand,
                     int *ccount, int *flags, float *dump, unsigned *ctrs, OvfPool pool, int *ovf_head,
                     float *ovf_lim, int passes, cudaStream_t st) {
    SOMB_REQUIRE(dp % 8 == 0 && kp % TC_BN == 0, SOMB_E_INPUT, "screen_tc: dp %% 8 and kp %% 256 required");
    int rc0 = screen_tc_init();
    if (rc0) return rc0;
    const int cg = g_tc_group;
    // multicast variant: CTA pairs, full capacity, 1-pass (the 3-pass screen is
    // MMA-bound, and 4-CTA cluster packing can leave SMs idle)
    // passes: 1 (fp16), 2 (fp16 + fp8 cross terms; Xl / Wl hold the fp8
    // operands, 2 dp bytes per row), 3 (fp16 hi/lo split)
    SOMB_REQUIRE(passes >= 1 && passes <= 3 && (passes == 1 || (Xl && Wl)), SOMB_E_INPUT,
                 "screen_tc: %d passes need the split operands", passes);
    const bool three = passes == 3, two = passes == 2;
    const int kchunks = (dp + TC_BK - 1) / TC_BK + (two ? (2 * dp + 127) / 128 : 0);
    const bool use_ar = g_ares && cg == 2 && !three && kchunks <= 4;   // A-resident (no codebook multicast)
    const int mcv = cg == 2 && g_half_cap == 32 && passes == 1 && !use_ar ? g_mc : 1;   // (2-pass with multicast measured slower)
    CUtensorMap mx, mw, mxl, mwl;
    int rc = make_map(&mx, Xh, (uint64_t)dp, (uint64_t)n, TC_ROWS);
    if (!rc) rc = make_map(&mw, Wh, (uint64_t)dp, (uint64_t)kp, (uint32_t)(TC_BN / cg / mcv));
    if (two) {
        if (!rc) rc = make_map(&mxl, Xl, (uint64_t)(2 * dp), (uint64_t)n, TC_ROWS, true);
        if (!rc) rc = make_map(&mwl, Wl, (uint64_t)(2 * dp), (uint64_t)kp, (uint32_t)(TC_BN / cg / mcv), true);
    } else {
        if (!rc) rc = make_map(&mxl, three ? Xl : Xh, (uint64_t)dp, (uint64_t)n, TC_ROWS);
        if (!rc) rc = make_map(&mwl, three ? Wl : Wh, (uint64_t)dp, (uint64_t)kp, (uint32_t)(TC_BN / cg / mcv));
    }
    if (rc) return rc;
    int dev = 0, sms = kSmCount;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaMemsetAsync(ccount, 0, (size_t)n * sizeof(int), st);
    cudaMemsetAsync(flags, 0, (size_t)n * sizeof(int), st);
    unsigned *ctr = ctrs;              // [0] lockstep, [1] overflow chunks (pool.ctr)
    const int lag = g_lag;
    cudaMemsetAsync(ctrs, 0, 2 * sizeof(unsigned), st);
    const int units = (int)((n + TC_ROWS * cg - 1) / (TC_ROWS * cg));
    int max_units = sms / cg;
    if (mcv == 2) {   // co-resident 4-CTA clusters (GPC packing can leave SMs idle)
        static int max_clusters = 0;
        if (!max_clusters) {
            cudaLaunchConfig_t lc = {};
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 4;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            lc.gridDim = dim3(4 * (sms / 4));
            lc.blockDim = dim3(TC_THREADS);
            lc.dynamicSmemBytes = TcCfg<2, 1, 32>::SMEM;
            lc.attrs = at;
            lc.numAttrs = 1;
            if (cudaOccupancyMaxActiveClusters(&max_clusters, screen_tc4_kernel<1, 32>, &lc) != cudaSuccess ||
                max_clusters < 1)
                max_clusters = sms / 4;
        }
        max_units = 2 * max_clusters;
    }
    int grid = cg * (units < max_units ? units : max_units);
    if (mcv == 2) grid = 4 * ((grid + 3) / 4);
#define SCREEN_LAUNCH(KERN, CGV, PV, HV)                                                                            \
    KERN<PV, HV><<<grid, TC_THREADS, TcCfg<CGV, PV, HV>::SMEM, st>>>(mx, mw, mxl, mwl, n, dp, kp, c, xstat, scal, wcoef, \
                                                                     thr0, cand, ccount, flags, dump, ctr, lag, pool, \
                                                                     ovf_head, ovf_lim)
#define SCREEN_LAUNCH_AR(PV, HV)                                                                                    \
    screen_tc2a_kernel<PV, HV><<<grid, TC_THREADS, TcCfg<2, PV, HV, TC_EPI_WARPS, 1>::SMEM, st>>>(                    \
        mx, mw, mxl, mwl, n, dp, kp, c, xstat, scal, wcoef, thr0, cand, ccount, flags, dump, ctr, lag, pool, ovf_head, \
        ovf_lim)
    if (use_ar) {
        if (g_half_cap <= 16) {
            if (two) SCREEN_LAUNCH_AR(2, 16); else SCREEN_LAUNCH_AR(1, 16);
        } else {
            if (two) SCREEN_LAUNCH_AR(2, 32); else SCREEN_LAUNCH_AR(1, 32);
        }
    } else if (two) {
        SOMB_REQUIRE(cg == 2, SOMB_E_CONFIG, "screen_tc: the fp8 split screen needs CTA pairs (tc_group 2)");
        if (mcv == 2) SCREEN_LAUNCH(screen_tc4_kernel, 2, 2, 32);
        else if (g_half_cap <= 16) SCREEN_LAUNCH(screen_tc2_kernel, 2, 2, 16);   // smaller lists, one more stage
        else SCREEN_LAUNCH(screen_tc2_kernel, 2, 2, 32);
    } else if (cg == 1) {
        if (three) SCREEN_LAUNCH(screen_tc1_kernel, 1, 3, 16); else SCREEN_LAUNCH(screen_tc1_kernel, 1, 1, 16);
    } else if (mcv == 2) {
        if (three) SCREEN_LAUNCH(screen_tc4_kernel, 2, 3, 32); else SCREEN_LAUNCH(screen_tc4_kernel, 2, 1, 32);
    } else if (three) {
        if (g_half_cap == 8) SCREEN_LAUNCH(screen_tc2_kernel, 2, 3, 8);
        else if (g_half_cap == 16) SCREEN_LAUNCH(screen_tc2_kernel, 2, 3, 16);
        else SCREEN_LAUNCH(screen_tc2_kernel, 2, 3, 32);
    } else {
        if (g_half_cap == 8) SCREEN_LAUNCH(screen_tc2_kernel, 2, 1, 8);
        else if (g_half_cap == 16) SCREEN_LAUNCH(screen_tc2_kernel, 2, 1, 16);
        else SCREEN_LAUNCH(screen_tc2_kernel, 2, 1, 32);
    }
#undef SCREEN_LAUNCH
#undef SCREEN_LAUNCH_AR
    note_launch();
    SOMB_LAUNCH_CHECK("screen_tc");
    return SOMB_OK;
}

}  // namespace somb
