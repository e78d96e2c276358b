// BMU search: screen (tensor-core or SIMT) -> candidates -> exact fp64 re-rank.
//
// Replaces kernels.py:195-205 (_search_chunk_blocked), :182-192 (naive) and
// the qe sum of :407.  The screen ranks r_ij = c_j - 2 x'_i.delta_j on fp16
// operands (prep.cu); the re-rank evaluates the reference formula in fp64
// from the original f32 rows, so the returned BMU is the reference's argmin
// whenever it lies in the screened candidate set.
#include <cuda_fp8.h>

#include "rerank.cuh"

namespace somb {

int launch_screen_tc(const __half *Xh, const __half *Xl, int64_t n, int dp, const __half *Wh,
                     const __half *Wl, int kp, const float *c, const float *xstat, const float *scal,
                     float wcoef, const float *thr0, int *cand, int *ccount, int *flags, float *dump,
                     unsigned *ctrs, OvfPool pool, int *ovf_head, float *ovf_lim, int passes, cudaStream_t st);

// overflow pool: 4 chunks (128 spilled candidates) per row on average on top
// of the 64 shared-memory slots -- near-constant or clustered data keeps
// 100-200 nodes per row inside the window (profiles/r2_window_calib_*.json);
// rows beyond the pool are truncated and repaired by an exact scan
static unsigned ovf_chunks(int64_t n) { return (unsigned)(4 * n > 4096 ? 4 * n : 4096); }
// test knob (somb_set_knob "ovf_chunks"): cap the usable overflow chunks to
// exercise the pool-exhaustion path (0 = the whole pool)
static unsigned g_ovf_limit = 0;
int bmu_set_knob(const char *key, int value) {
    if (!strcmp(key, "ovf_chunks")) { g_ovf_limit = value > 0 ? (unsigned)value : 0u; return SOMB_OK; }
    return SOMB_E_CONFIG;
}

BmuWs bmu_carve(void *ws, int64_t n, size_t *total) {
    BmuWs w;
    char *p = (char *)ws;
    auto take = [&](size_t bytes) { char *r = p; p += align_up(bytes, 256); return r; };
    const unsigned C = ovf_chunks(n);
    w.cand = (int *)take((size_t)n * SOMB_CAND_CAP * sizeof(int));
    w.ccount = (int *)take((size_t)n * sizeof(int));
    w.thr0 = (float *)take((size_t)n * sizeof(float));
    w.ctrs = (unsigned *)take(8 * sizeof(unsigned));
    w.ovf_head = (int *)take((size_t)4 * n * sizeof(int));
    w.ovf_lim = (float *)take((size_t)4 * n * sizeof(float));
    w.pool.next = (int *)take((size_t)C * sizeof(int));
    w.pool.cnt = (int *)take((size_t)C * sizeof(int));
    w.pool.ent = (int2 *)take((size_t)C * kOvfChunk * sizeof(int2));
    w.pool.ctr = w.ctrs + 1;
    w.pool.nchunks = g_ovf_limit && g_ovf_limit < C ? g_ovf_limit : C;   // layout always sized for C
    if (total) *total = (size_t)(p - (char *)ws);
    return w;
}

// Exact repair of truncated rows: a row whose candidate set was cut (the
// overflow pool ran out, cand.cuh) may have lost its true BMU, so its list
// is emptied and the re-rank scans every node for it in fp64 -- the result
// is the reference's argmin (kernels.py:195-205, first-minimum ties 27-28)
// for every row, truncated or not.  flags: bit 0 of any byte = truncated
// (one byte per column group of the tcgen05 screen, one word otherwise);
// ctr counts the repaired rows (ws counter 4, somb_bmu_repaired_rows).
// The row ids are also listed at list[0, *ctr) when a list is given (the
// sparse path re-ranks them with a slab-lockstep exact scan, sparse.cu).
__global__ void repair_truncated_kernel(const int *__restrict__ flags, int *__restrict__ ccount, int64_t n,
                                        unsigned *__restrict__ ctr, int *__restrict__ list) {
    const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= n) return;
    if (flags[row] & 0x01010101) {
        ccount[row] = kScanAll;
        const unsigned i = atomicAdd(ctr, 1u);
        if (list) list[i] = (int)row;
    }
}

int launch_repair_truncated(const int *flags, int *ccount, int64_t n, unsigned *ctrs, cudaStream_t st,
                            int *list) {
    cudaMemsetAsync(ctrs + 4, 0, sizeof(unsigned), st);
    if (n == 0) return SOMB_OK;
    repair_truncated_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(flags, ccount, n, ctrs + 4, list);
    note_launch();
    SOMB_LAUNCH_CHECK("repair_truncated");
    return SOMB_OK;
}


// Seed of each row's acceptance threshold from its previous BMU: the screened
// value of that node (same fp16 operands, fp32 FMA) plus one window and an
// eighth (the extra eighth covers the summation-order difference to the
// tensor-core value of the same node, which is orders of magnitude below the
// window).  Any node the screen will
// keep has r <= r_min + win <= r_prev + win, so seeding never changes the
// final candidate set -- it only skips transient pushes (cand.cuh).
// 3-pass mode (Xl, Wl given): the seed is the fp64 value of the same split
// product, and the slack is 1.5 windows (the tensor-core value differs from
// it by at most the screen error, <= half a window).
__device__ __forceinline__ double e4m3_to_double(uint8_t b) {
    __nv_fp8_e4m3 v;
    v.__x = b;
    return (double)(float)v;
}

// f8 = 1: Xl / Wl hold the fp8 cross operands [x_hi8 | x_lo8], [w_lo8 | w_hi8]
// (2 dp bytes per row, 2-pass screen): the seed is the fp64 value of the same
// hi.hi + cross products, slack 1.5 windows as for the 3-pass screen.
__global__ void screen_seed_kernel(const __half *__restrict__ Xh, const __half *__restrict__ Xl, int64_t n, int dp,
                                   const __half *__restrict__ Wh, const __half *__restrict__ Wl, int K,
                                   const float *__restrict__ c, const float *__restrict__ xstat,
                                   const float *__restrict__ scal, float wcoef, const int *__restrict__ prev,
                                   float *__restrict__ thr0, int f8) {
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (row >= n) return;
    const int j = prev[row];
    float t = FLT_MAX;
    if (j >= 0 && j < K) {
        const __half2 *x = reinterpret_cast<const __half2 *>(Xh + row * (int64_t)dp);
        const __half2 *w = reinterpret_cast<const __half2 *>(Wh + (int64_t)j * dp);
        float win = wcoef * screen_sigma(reinterpret_cast<const float4 *>(xstat)[row], scal);
        float r;
        if (f8) {
            const uint8_t *x8 = reinterpret_cast<const uint8_t *>(Xl) + row * (int64_t)(2 * dp);
            const uint8_t *w8 = reinterpret_cast<const uint8_t *>(Wl) + (int64_t)j * (2 * dp);
            double acc = 0.0;
            for (int k = lane; k < dp; k += 32) {
                acc += (double)__half2float(Xh[row * (int64_t)dp + k]) * (double)__half2float(Wh[(int64_t)j * dp + k]);
                acc += e4m3_to_double(x8[k]) * e4m3_to_double(w8[k]) +
                       e4m3_to_double(x8[dp + k]) * e4m3_to_double(w8[dp + k]);
            }
            acc = warp_sum(acc);
            r = (float)(acc * (double)scal[0] + (double)c[j]);
            if (r < FLT_MAX) r += 1.5f * win;
        } else if (Xl == nullptr) {
            float acc = 0.0f;
            for (int k = lane; k < dp / 2; k += 32) {
                float2 a = __half22float2(x[k]), b = __half22float2(w[k]);
                acc = fmaf(a.x, b.x, acc);
                acc = fmaf(a.y, b.y, acc);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            r = fmaf(acc, scal[0], c[j]);
            if (r < FLT_MAX) r += 1.125f * win;
        } else {
            const __half2 *xl = reinterpret_cast<const __half2 *>(Xl + row * (int64_t)dp);
            const __half2 *wl = reinterpret_cast<const __half2 *>(Wl + (int64_t)j * dp);
            double acc = 0.0;
            for (int k = lane; k < dp / 2; k += 32) {
                float2 a = __half22float2(x[k]), b = __half22float2(w[k]);
                float2 al = __half22float2(xl[k]), bl = __half22float2(wl[k]);
                acc += (double)a.x * b.x + (double)a.x * bl.x + (double)al.x * b.x;
                acc += (double)a.y * b.y + (double)a.y * bl.y + (double)al.y * b.y;
            }
            acc = warp_sum(acc);
            r = (float)(acc * (double)scal[0] + (double)c[j]);
            if (r < FLT_MAX) r += 1.5f * win;
        }
        if (r < FLT_MAX) t = r;
    }
    if (lane == 0) thr0[row] = t;
}

// --------------------------------------------------------- SIMT screen (v0)
// Reference implementation of the screen used by the parity tests to check
// the tcgen05 kernel (same fp16 operands, fp32 FMA accumulation).
constexpr int kSimtRows = 128;
constexpr int kSimtCols = 32;
constexpr int kSimtK = 64;
constexpr int kSimtCap = 32;   // candidates per row of the reference screen (<= SOMB_CAND_CAP)

__global__ void __launch_bounds__(kSimtRows)
screen_simt_kernel(const __half *__restrict__ Xh, int64_t n, int dp, const __half *__restrict__ Wh,
                   int kp, const float *__restrict__ c, const float *__restrict__ xstat,
                   const float *__restrict__ scal, float wcoef, const float *__restrict__ thr0,
                   int *__restrict__ cand, int *__restrict__ ccount, int *__restrict__ flags) {
    __shared__ float wt[kSimtCols][kSimtK + 1];
    __shared__ float bv[kSimtCap * kSimtRows];
    __shared__ int bi[kSimtCap * kSimtRows];
    const int t = threadIdx.x;
    const int64_t row = (int64_t)blockIdx.x * kSimtRows + t;
    const bool live = row < n;
    const float m = scal[0];
    CandRow<kSimtCap> st;
    cand_init(st, live ? wcoef * screen_sigma(reinterpret_cast<const float4 *>(xstat)[row], scal) : 0.0f);
    if (live && thr0) st.thr = thr0[row];
    const CandBuf cb{smem_addr(bv + t), smem_addr(bi + t), 4u * kSimtRows};
    const __half *xr = Xh + (live ? row : 0) * (int64_t)dp;
    for (int j0 = 0; j0 < kp; j0 += kSimtCols) {
        float acc[kSimtCols];
#pragma unroll
        for (int q = 0; q < kSimtCols; ++q) acc[q] = 0.0f;
        for (int k0 = 0; k0 < dp; k0 += kSimtK) {
            __syncthreads();
            for (int e = t; e < kSimtCols * kSimtK; e += kSimtRows) {
                int jj = e / kSimtK, kk = e % kSimtK;
                int k = k0 + kk;
                wt[jj][kk] = k < dp ? __half2float(Wh[(int64_t)(j0 + jj) * dp + k]) : 0.0f;
            }
            __syncthreads();
            float xv[kSimtK];
#pragma unroll
            for (int kk = 0; kk < kSimtK; ++kk) {
                int k = k0 + kk;
                xv[kk] = (live && k < dp) ? __half2float(xr[k]) : 0.0f;
            }
#pragma unroll 4
            for (int q = 0; q < kSimtCols; ++q) {
                float a = acc[q];
#pragma unroll
                for (int kk = 0; kk < kSimtK; ++kk) a = fmaf(xv[kk], wt[q][kk], a);
                acc[q] = a;
            }
        }
        if (live) {
#pragma unroll 1
            for (int q = 0; q < kSimtCols; ++q) {
                float r = fmaf(acc[q], m, c[j0 + q]);
                cand_push<kSimtCap>(st, r, j0 + q, cb);
            }
        }
    }
    if (live) {
        int *out = cand + row * SOMB_CAND_CAP;
        ccount[row] = cand_emit<kSimtCap>(st, cb, out);
        flags[row] = st.trunc;
    }
}

// ----------------------------------------------------------- fp64 re-rank
// One warp per row; `all` = exact scan of every node (screen_impl 2 and the
// empty-candidate safety net).
__global__ void rerank_kernel(const float *__restrict__ X, const double *__restrict__ x2, int64_t n,
                              int d, const float *__restrict__ W, const double *__restrict__ w2,
                              int K, const int *__restrict__ cand, const int *__restrict__ ccount,
                              int dist_mode, int all, int split, const int *__restrict__ order,
                              OvfView ov, int *__restrict__ bmu, double *__restrict__ d2min) {
    const int64_t w = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (w >= n) return;
    const int64_t row = order ? (int64_t)order[w] : w;
    const float *x = X + row * d;
    // candidate list: one segment [0, cc) or, for the two-half tcgen05
    // epilogue, [0, cc & 255) and [CAP/2, CAP/2 + (cc >> 8 & 255))
    int cc = all ? 0 : ccount[row];
    const CandLayout L = cand_layout(cc, split, split && ov.ngp ? (int)*ov.ngp : 2);
    int cnt = L.cnt;
    bool scan_all = all || cand_scan_all(L, ov, row);
    if (scan_all) cnt = K;
    double best = INFINITY;
    int bestj = 0x7fffffff;
    const double xx = x2[row];
    // main list, then (tcgen05 overflow) the spilled chunks of both column groups
    int ovh = -2, ovc = -1;      // current overflow group / chunk
    unsigned ovbal = 0u;
    int2 ove = make_int2(0, -1);
    for (int q = 0;; ++q) {
        int j;
        if (q < cnt) {
            j = scan_all ? q : cand[row * SOMB_CAND_CAP + cand_slot(L, q)];
        } else {
            if (scan_all || ov.head == nullptr) break;
            while (ovbal == 0u) {     // next chunk with in-window entries
                if (ovc >= 0) ovc = ov.next[ovc];
                while (ovc < 0 && ovh < 3) { ++ovh; if (ovh >= 0) ovc = ov.head[4 * row + ovh]; }
                if (ovc < 0) break;
                const int m = ov.cnt[ovc];
                ove = lane < m ? ov.ent[(size_t)ovc * kOvfChunk + lane] : make_int2(0x7f800000, -1);
                ovbal = __ballot_sync(0xffffffffu, lane < m && __int_as_float(ove.x) <= ov.lim[4 * row + ovh]);
            }
            if (ovbal == 0u) break;
            const int src = __ffs(ovbal) - 1;
            ovbal &= ovbal - 1u;
            j = __shfl_sync(0xffffffffu, ove.y, src);
        }
        if ((unsigned)j >= (unsigned)K) continue;
        const float *w = W + (int64_t)j * d;
        double d2;
        if (dist_mode == SOMB_DIST_NAIVE) {
            double s = 0.0;
            for (int k = lane; k < d; k += 32) {
                double df = (double)w[k] - (double)x[k];
                s = __fma_rn(df, df, s);
            }
            d2 = warp_sum(s);
        } else {
            double s = 0.0;
            for (int k = lane; k < d; k += 32) s = __fma_rn((double)x[k], (double)w[k], s);
            s = warp_sum(s);
            // ((-2 dot) + |x|^2) + |w|^2, clamp >= 0 (kernels.py:196-202)
            d2 = __dadd_rn(__dadd_rn(__dmul_rn(-2.0, s), xx), w2[j]);
            d2 = fmax(d2, 0.0);
        }
        if (d2 < best || (d2 == best && j < bestj)) {   // first minimum (lowest index)
            best = d2;
            bestj = j;
        }
    }
    if (lane == 0) {
        bmu[row] = bestj;
        d2min[row] = best;
    }
}

// Vectorised re-rank for d % 4 == 0, d <= 128 * Q: the row lives in
// registers (float4 per lane); candidate indices are fetched once (lane q
// holds candidate q) and broadcast by shuffle; the next candidate's codebook
// row is prefetched while the current one is reduced.  Bound by L2 traffic
// (one 4d-byte codebook row per candidate).
template <int Q>
__device__ __forceinline__ void load_row4(const float *W, int64_t j, int d4, int lane, float4 (&w)[Q]) {
    const float4 *wr = reinterpret_cast<const float4 *>(W + j * (int64_t)(d4 * 4));
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        int e = lane + 32 * q;
        w[q] = e < d4 ? __ldg(wr + e) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

// Four independent fp64 accumulators (one per float4 component) so the DFMA
// chains overlap; summed pairwise at the end (fixed order: deterministic).
template <int Q, int MODE>
__device__ __forceinline__ double dist_part(const float4 (&x)[Q], const float4 (&w)[Q]) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        if (MODE == SOMB_DIST_NAIVE) {
            double a = (double)w[q].x - (double)x[q].x, b = (double)w[q].y - (double)x[q].y;
            double c = (double)w[q].z - (double)x[q].z, e = (double)w[q].w - (double)x[q].w;
            s0 = __fma_rn(a, a, s0); s1 = __fma_rn(b, b, s1); s2 = __fma_rn(c, c, s2); s3 = __fma_rn(e, e, s3);
        } else {
            s0 = __fma_rn((double)x[q].x, (double)w[q].x, s0);
            s1 = __fma_rn((double)x[q].y, (double)w[q].y, s1);
            s2 = __fma_rn((double)x[q].z, (double)w[q].z, s2);
            s3 = __fma_rn((double)x[q].w, (double)w[q].w, s3);
        }
    }
    return __dadd_rn(__dadd_rn(s0, s1), __dadd_rn(s2, s3));
}

template <int Q, int MODE>
__global__ void __launch_bounds__(256, 2)
rerank_vec_kernel(const float *__restrict__ X, const double *__restrict__ x2, int64_t n, int d,
                  const float *__restrict__ W, const double *__restrict__ w2, int K,
                  const int *__restrict__ cand, const int *__restrict__ ccount, int split,
                  const int *__restrict__ order, OvfView ov, int *__restrict__ bmu, double *__restrict__ d2min) {
    const int64_t w = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (w >= n) return;
    const int64_t row = order ? (int64_t)order[w] : w;
    const int d4 = d >> 2;
    float4 xv[Q];
    load_row4<Q>(X, row, d4, lane, xv);
    const int cc = ccount[row];
    const CandLayout L = cand_layout(cc, split, split && ov.ngp ? (int)*ov.ngp : 2);
    int cnt = L.cnt;
    // candidate q lives in lane q % 32, register q / 32 (up to 64 per row)
    auto slot = [&](int q) { return cand_slot(L, q); };
    int myj0 = lane < cnt ? cand[row * SOMB_CAND_CAP + slot(lane)] : -1;
    int myj1 = lane + 32 < cnt ? cand[row * SOMB_CAND_CAP + slot(lane + 32)] : -1;
    auto cand_at = [&](int q) {
        int a = __shfl_sync(0xffffffffu, myj0, q & 31), b = __shfl_sync(0xffffffffu, myj1, q & 31);
        return q < 32 ? a : b;
    };
    const bool all = cand_scan_all(L, ov, row);   // repaired row: exact scan of every node
    if (all) cnt = K;
    const double xx = x2[row];
    double best = INFINITY;
    int bestj = 0x7fffffff;
    int j = all ? 0 : cand_at(0);
    float4 wv[Q];
    load_row4<Q>(W, (unsigned)j < (unsigned)K ? j : 0, d4, lane, wv);
    for (int q = 0; q < cnt; ++q) {
        const int jn = (q + 1 < cnt) ? (all ? q + 1 : cand_at(q + 1)) : j;
        float4 wn[Q];
        load_row4<Q>(W, (unsigned)jn < (unsigned)K ? jn : 0, d4, lane, wn);   // prefetch next
        double s = warp_sum(dist_part<Q, MODE>(xv, wv));
        double v = s;
        if (MODE == SOMB_DIST_BLOCKED)   // ((-2 dot) + |x|^2) + |w|^2, clamp (kernels.py:196-202)
            v = fmax(__dadd_rn(__dadd_rn(__dmul_rn(-2.0, s), xx), w2[(unsigned)j < (unsigned)K ? j : 0]), 0.0);
        if ((unsigned)j < (unsigned)K && (v < best || (v == best && j < bestj))) {
            best = v;
            bestj = j;
        }
        j = jn;
#pragma unroll
        for (int t = 0; t < Q; ++t) wv[t] = wn[t];
    }
    if (ov.head != nullptr && !all) {   // spilled candidates of both column groups
#pragma unroll 1
        for (int h = 0; h < 4; ++h) {
            const float lim = ov.lim[4 * row + h];
#pragma unroll 1
            for (int c = ov.head[4 * row + h]; c >= 0; c = ov.next[c]) {
                const int m = ov.cnt[c];
                const int2 e = lane < m ? ov.ent[(size_t)c * kOvfChunk + lane] : make_int2(0x7f800000, -1);
                unsigned bal = __ballot_sync(0xffffffffu, lane < m && __int_as_float(e.x) <= lim);
                while (bal) {
                    const int src = __ffs(bal) - 1;
                    bal &= bal - 1u;
                    const int jj = __shfl_sync(0xffffffffu, e.y, src);
                    if ((unsigned)jj >= (unsigned)K) continue;
                    load_row4<Q>(W, jj, d4, lane, wv);
                    double sd = warp_sum(dist_part<Q, MODE>(xv, wv));
                    double v = sd;
                    if (MODE == SOMB_DIST_BLOCKED) v = fmax(__dadd_rn(__dadd_rn(__dmul_rn(-2.0, sd), xx), w2[jj]), 0.0);
                    if (v < best || (v == best && jj < bestj)) {
                        best = v;
                        bestj = jj;
                    }
                }
            }
        }
    }
    if (lane == 0) {
        bmu[row] = bestj;
        d2min[row] = best;
    }
}

// Pipelined re-rank: each lane stages ITS OWN float4 slices of the next
// RS candidates' codebook rows in shared memory with cp.async (L2 -> smem,
// no register cost), so a warp keeps RS rows (RS x 4d bytes) in flight
// instead of one -- the plain kernel was bound by memory-level parallelism
// (profiles/).  A lane only ever reads back what it copied itself, so
// cp.async.wait_group alone orders the data (no warp barrier).  Same
// products as rerank_vec_kernel (exact in fp64); eight accumulators instead
// of four (the DFMA dependency chains were the top stall).
constexpr int RS = 4;            // candidate rows in flight per warp
constexpr int RP_WARPS = 4;      // warps per block



// Row operand of the pipelined re-rank: slices q < PQA convert w with F2F,
// the rest with f32_as_f64_scaled (blocked mode keeps those x slices
// pre-scaled by 2^896, exact since |x| < 2^128), splitting the conversions
// over the XU and integer pipes.
template <int Q>
struct PipeSplit { static constexpr int PQA = Q; };
// (a template parameter of the kernel; round 2 measured the split at cfg2,
// ~33 candidates per row: all F2F 26.0 ms, 5 of 8 26.3, 4 27.5, 3 (the
// round-1 choice) 28.6-28.9, 2 30.1, none 34.3 (per-split builds); all F2F
// also took cfg4 8.4 -> 6.7 ms and cfg5 22.4 -> 21.7 ms)

template <int Q, int MODE, int PQ = PipeSplit<Q>::PQA>
__device__ __forceinline__ void row_operand(const float4 (&x)[Q], double (&xd)[Q][4]) {
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const double sc = (MODE != SOMB_DIST_NAIVE && q >= PQ) ? kF64Scale : 1.0;
        xd[q][0] = (double)x[q].x * sc; xd[q][1] = (double)x[q].y * sc;
        xd[q][2] = (double)x[q].z * sc; xd[q][3] = (double)x[q].w * sc;
    }
}

// Eight independent accumulators (component x slice parity); fixed pairwise
// combination order, so the result is deterministic.
template <int Q, int MODE, int PQ = PipeSplit<Q>::PQA>
__device__ __forceinline__ double dist_part_mixed(const double (&x)[Q][4], const float4 (&w)[Q]) {
    double s[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) s[t] = 0.0;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        const float wf[4] = {w[q].x, w[q].y, w[q].z, w[q].w};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            double &acc = s[(q & 1) * 4 + c];
            if (q < PQ) {
                const double wd = (double)wf[c];
                if (MODE == SOMB_DIST_NAIVE) {
                    const double a = wd - x[q][c];
                    acc = __fma_rn(a, a, acc);
                } else {
                    acc = __fma_rn(x[q][c], wd, acc);
                }
            } else {
                const double wb = f32_as_f64_scaled(wf[c]);
                if (MODE == SOMB_DIST_NAIVE) {
                    const double a = __fma_rn(wb, kF64Scale, -x[q][c]);   // == (double)w - x, one rounding
                    acc = __fma_rn(a, a, acc);
                } else {
                    acc = __fma_rn(x[q][c], wb, acc);                    // (x 2^896)(w 2^-896), exact product
                }
            }
        }
    }
    return __dadd_rn(__dadd_rn(__dadd_rn(s[0], s[4]), __dadd_rn(s[1], s[5])),
                     __dadd_rn(__dadd_rn(s[2], s[6]), __dadd_rn(s[3], s[7])));
}

template <int Q, int MODE, int PQ = PipeSplit<Q>::PQA>
__global__ void __launch_bounds__(32 * RP_WARPS, 3)
rerank_pipe_kernel(const float *__restrict__ X, const double *__restrict__ x2, int64_t n, int d,
                   const float *__restrict__ W, const double *__restrict__ w2, int K,
                   const int *__restrict__ cand, const int *__restrict__ ccount, int split,
                   const int *__restrict__ order, OvfView ov, int *__restrict__ bmu, double *__restrict__ d2min) {
    // [warp][stage][q][lane] float4 (dynamic shared memory)
    extern __shared__ float4 ring_raw[];
    auto ring = reinterpret_cast<float4 (*)[RS][Q][32]>(ring_raw);
    const int wib = threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    const int d4 = d >> 2;
    // slices this lane owns (bit q: float4 index lane + 32 q < d4); the ring
    // slots of the others are zeroed once and never written, so reads need
    // no bounds test (x is zero there too)
    unsigned vmask = 0u;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        if (lane + 32 * q < d4) vmask |= 1u << q;
#pragma unroll
        for (int s0 = 0; s0 < RS; ++s0)
            if (lane + 32 * q >= d4) ring[wib][s0][q][lane] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    // persistent warps striding over the (BMU-sorted) rows: no block waits on
    // its slowest row, and concurrently active warps stay on neighbouring rows
#pragma unroll 1
    for (int64_t wi = (int64_t)blockIdx.x * RP_WARPS + wib; wi < n; wi += (int64_t)gridDim.x * RP_WARPS) {
    const int64_t row = order ? (int64_t)order[wi] : wi;
    double xd[Q][4];
    {
        float4 xv[Q];
        load_row4<Q>(X, row, d4, lane, xv);
        row_operand<Q, MODE, PQ>(xv, xd);
    }
    const int cc = ccount[row];
    const CandLayout L = cand_layout(cc, split, split && ov.ngp ? (int)*ov.ngp : 2);
    int cnt = L.cnt;
    auto slot = [&](int q) { return cand_slot(L, q); };
    const int myj0 = lane < cnt ? cand[row * SOMB_CAND_CAP + slot(lane)] : -1;
    const int myj1 = lane + 32 < cnt ? cand[row * SOMB_CAND_CAP + slot(lane + 32)] : -1;
    const bool all = cand_scan_all(L, ov, row);   // repaired row: exact scan of every node
    if (all) cnt = K;
    auto cand_at = [&](int q) {
        if (all) return q;
        int a = __shfl_sync(0xffffffffu, myj0, q & 31), b = __shfl_sync(0xffffffffu, myj1, q & 31);
        return q < 32 ? a : b;
    };
    auto issue = [&](int j, int stg) {
        if ((unsigned)j < (unsigned)K) {
            const float4 *wr = reinterpret_cast<const float4 *>(W + (int64_t)j * d);
#pragma unroll
            for (int q = 0; q < Q; ++q)
                if (vmask >> q & 1u) cp_async16(smem_addr(&ring[wib][stg][q][lane]), wr + lane + 32 * q);
        }
    };
    const double xx = x2[row];
    double best = INFINITY;
    int bestj = 0x7fffffff;
    // lane partials of four candidates -> their exact values, folded into
    // (best, bestj).  A reduce-scatter butterfly: after the xor-16 and xor-8
    // steps lane L carries candidate ((L >> 4) & 1) * 2 + ((L >> 3) & 1), so
    // the four sums take 6 fp64 shuffles on one dependency chain instead of
    // four 5-deep warp_sum chains (the serial shuffle latency was the re-rank's
    // top stall).  The winner is the lowest (value, index) pair, the same
    // total order as the one-at-a-time scan.
    auto consider4 = [&](const double (&p)[4], const int (&jg)[4]) {
        const bool b4 = lane & 16, b3 = lane & 8;
        const double a0 = (b4 ? p[2] : p[0]) + __shfl_xor_sync(0xffffffffu, b4 ? p[0] : p[2], 16);
        const double a1 = (b4 ? p[3] : p[1]) + __shfl_xor_sync(0xffffffffu, b4 ? p[1] : p[3], 16);
        double c = (b3 ? a1 : a0) + __shfl_xor_sync(0xffffffffu, b3 ? a0 : a1, 8);
        c += __shfl_xor_sync(0xffffffffu, c, 4);
        c += __shfl_xor_sync(0xffffffffu, c, 2);
        c += __shfl_xor_sync(0xffffffffu, c, 1);
        const int g = (b4 ? 2 : 0) + (b3 ? 1 : 0);
        const int j = g == 0 ? jg[0] : g == 1 ? jg[1] : g == 2 ? jg[2] : jg[3];
        const bool ok = (unsigned)j < (unsigned)K;
        double v = c;
        if (MODE == SOMB_DIST_BLOCKED)   // ((-2 dot) + |x|^2) + |w|^2, clamp (kernels.py:196-202)
            v = fmax(__dadd_rn(__dadd_rn(__dmul_rn(-2.0, c), xx), w2[ok ? j : 0]), 0.0);
        if (!ok) v = INFINITY;
        int jj = ok ? j : 0x7fffffff;
#pragma unroll
        for (int m = 8; m <= 16; m <<= 1) {
            const double ov2 = __shfl_xor_sync(0xffffffffu, v, m);
            const int oj = __shfl_xor_sync(0xffffffffu, jj, m);
            if (ov2 < v || (ov2 == v && oj < jj)) { v = ov2; jj = oj; }
        }
        if (jj != 0x7fffffff && (v < best || (v == best && jj < bestj))) {
            best = v;
            bestj = jj;
        }
    };
    // one pipelined pass over a candidate list given by get(q), q < m
    auto run = [&](int m, auto get) {
#pragma unroll
        for (int s0 = 0; s0 < RS; ++s0) {
            if (s0 < m) issue(get(s0), s0);
            cp_async_commit();
        }
#pragma unroll 1
        for (int q0 = 0; q0 < m; q0 += 4) {
            double p[4];
            int jg[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int q = q0 + i;
                p[i] = 0.0;
                jg[i] = -1;
                if (q < m) {   // warp-uniform
                    const int stg = q % RS;
                    jg[i] = get(q);
                    const int jn = q + RS < m ? get(q + RS) : -1;
                    cp_async_wait<RS - 1>();
                    float4 wv[Q];
#pragma unroll
                    for (int t = 0; t < Q; ++t) wv[t] = ring[wib][stg][t][lane];
                    if (jn >= 0) issue(jn, stg);
                    cp_async_commit();
                    p[i] = dist_part_mixed<Q, MODE, PQ>(xd, wv);
                }
            }
            consider4(p, jg);
        }
        cp_async_wait<0>();
    };
    run(cnt, cand_at);
    if (ov.head != nullptr && !all) {   // spilled candidates of both column groups, chunk by chunk
#pragma unroll 1
        for (int h = 0; h < 4; ++h) {
            const float lim = ov.lim[4 * row + h];
#pragma unroll 1
            for (int c = ov.head[4 * row + h]; c >= 0; c = ov.next[c]) {
                const int m = ov.cnt[c];
                const int2 e = lane < m ? ov.ent[(size_t)c * kOvfChunk + lane] : make_int2(0x7f800000, -1);
                const unsigned bal = __ballot_sync(0xffffffffu, lane < m && __int_as_float(e.x) <= lim);
                run(__popc(bal), [&](int q) { return __shfl_sync(0xffffffffu, e.y, __fns(bal, 0, q + 1)); });
            }
        }
    }
    if (lane == 0) {
        bmu[row] = bestj;
        d2min[row] = best;
    }
    }
}

template <int Q>
static void launch_rerank_pipe(cudaStream_t st, const float *X, const double *x2, int64_t n, int d, const float *W,
                               const double *w2, int K, const int *cand, const int *ccount, int mode, int split,
                               const int *order, OvfView ov, int *bmu, double *d2min) {
    int dev = 0, sms = kSmCount;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = sizeof(float4) * RP_WARPS * RS * Q * 32;
    static int per_sm = 0;   // resident blocks per SM (same for both modes)
    if (!per_sm) {
        cudaFuncSetAttribute(rerank_pipe_kernel<Q, SOMB_DIST_NAIVE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(rerank_pipe_kernel<Q, SOMB_DIST_BLOCKED>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rerank_pipe_kernel<Q, SOMB_DIST_BLOCKED>, 32 * RP_WARPS, smem);
        if (per_sm < 1) per_sm = 1;
    }
    const int64_t need = (n + RP_WARPS - 1) / RP_WARPS;
    const unsigned blocks = (unsigned)(need < (int64_t)per_sm * sms ? need : (int64_t)per_sm * sms);
    if (mode == SOMB_DIST_NAIVE)
        rerank_pipe_kernel<Q, SOMB_DIST_NAIVE><<<blocks, 32 * RP_WARPS, smem, st>>>(X, x2, n, d, W, w2, K, cand, ccount,
                                                                                  split, order, ov, bmu, d2min);
    else
        rerank_pipe_kernel<Q, SOMB_DIST_BLOCKED><<<blocks, 32 * RP_WARPS, smem, st>>>(X, x2, n, d, W, w2, K, cand,
                                                                                    ccount, split, order, ov, bmu, d2min);
}

template <int Q>
static void launch_rerank_vec(unsigned blocks, cudaStream_t st, const float *X, const double *x2, int64_t n, int d,
                              const float *W, const double *w2, int K, const int *cand, const int *ccount, int mode,
                              int split, const int *order, OvfView ov, int *bmu, double *d2min) {
    if (mode == SOMB_DIST_NAIVE)
        rerank_vec_kernel<Q, SOMB_DIST_NAIVE><<<blocks, 256, 0, st>>>(X, x2, n, d, W, w2, K, cand, ccount, split, order,
                                                                       ov, bmu, d2min);
    else
        rerank_vec_kernel<Q, SOMB_DIST_BLOCKED><<<blocks, 256, 0, st>>>(X, x2, n, d, W, w2, K, cand, ccount, split, order,
                                                                         ov, bmu, d2min);
}

// --------------------------------------------------------- qe reduction
constexpr int kQeTile = 4096;

__global__ void qe_partial(const double *__restrict__ d2min, int64_t n, double *__restrict__ part) {
    __shared__ double sh[256];
    int64_t base = (int64_t)blockIdx.x * kQeTile;
    double s = 0.0;
    for (int q = 0; q < kQeTile / 256; ++q) {
        int64_t i = base + q * 256 + threadIdx.x;
        if (i < n) s += sqrt(d2min[i]);
    }
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void qe_final(const double *__restrict__ part, int np, double *__restrict__ out) {
    __shared__ double sh[256];
    double s = 0.0;
    for (int i = threadIdx.x; i < np; i += 256) s += part[i];
    sh[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = sh[0];
}

}  // namespace somb

using namespace somb;

extern "C" size_t somb_bmu_ws(int64_t n) {
    size_t total = 0;
    bmu_carve(nullptr, n, &total);
    return total + 256;
}

extern "C" int somb_bmu_screen(const uint16_t *Xh, const uint16_t *Xl, const float *xstat, int64_t n, int32_t dp,
                               const uint16_t *Wh, const uint16_t *Wl, const float *c, int32_t K, int32_t kp,
                               const float *scal, float window_coef, const int32_t *prev_bmu,
                               int32_t screen_impl, int32_t *flags, void *ws, void *stream) {
    SOMB_REQUIRE(dp % 8 == 0 && kp % 256 == 0, SOMB_E_INPUT, "bmu_screen: dp=%d kp=%d", dp, kp);
    SOMB_REQUIRE(screen_impl >= 0 && screen_impl <= 3, SOMB_E_CONFIG, "bad screen_impl %d", screen_impl);
    SOMB_REQUIRE(screen_impl != 3 || (Xl && Wl), SOMB_E_INPUT, "bmu_screen: the fp8 split screen needs Xl / Wl");
    if (n == 0 || screen_impl == 2) return SOMB_OK;
    cudaStream_t st = as_stream(stream);
    BmuWs w = bmu_carve(ws, n);
    int *cand = w.cand, *ccount = w.ccount;
    float *thr0 = nullptr;
    if (prev_bmu) {
        thr0 = w.thr0;
        const bool split = Xl != nullptr && Wl != nullptr && (screen_impl == 0 || screen_impl == 3);
        screen_seed_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(
            (const __half *)Xh, split ? (const __half *)Xl : nullptr, n, dp, (const __half *)Wh,
            split ? (const __half *)Wl : nullptr, K, c, xstat, scal, window_coef, prev_bmu, thr0,
            screen_impl == 3);
        note_launch();
    }
    if (screen_impl == 0 || screen_impl == 3) {
        int rc = launch_screen_tc((const __half *)Xh, (const __half *)Xl, n, dp, (const __half *)Wh,
                                  (const __half *)Wl, kp, c, xstat, scal, window_coef, thr0, cand, ccount, flags,
                                  nullptr, w.ctrs, w.pool, w.ovf_head, w.ovf_lim,
                                  screen_impl == 3 ? 2 : (Xl && Wl ? 3 : 1), st);
        if (rc) return rc;
    } else {
        unsigned blocks = (unsigned)((n + kSimtRows - 1) / kSimtRows);
        screen_simt_kernel<<<blocks, kSimtRows, 0, st>>>((const __half *)Xh, n, dp, (const __half *)Wh, kp, c,
                                                          xstat, scal, window_coef, thr0, cand, ccount, flags);
        note_launch();
        SOMB_LAUNCH_CHECK("screen_simt");
    }
    return launch_repair_truncated(flags, ccount, n, w.ctrs, st, nullptr);
}


static int g_rerank_pipe = -1;   // SOMB_RERANK_PIPE=0 selects the unpipelined kernel (A/B testing)

extern "C" int somb_bmu_rerank(const float *X, const double *x2, int64_t n, int32_t d, const float *W,
                               const double *w2, int32_t K, int32_t dist_mode, int32_t screen_impl,
                               const int32_t *row_order, int32_t *bmu, double *d2min, int32_t *flags, void *ws,
                               void *stream) {
    SOMB_REQUIRE(K > 0 && d > 0, SOMB_E_INPUT, "bmu_rerank: bad shape K=%d d=%d", K, d);
    SOMB_REQUIRE(dist_mode == SOMB_DIST_BLOCKED || dist_mode == SOMB_DIST_NAIVE, SOMB_E_CONFIG,
                 "bmu_rerank: bad dist_mode %d", dist_mode);
    if (n == 0) return SOMB_OK;
    cudaStream_t st = as_stream(stream);
    BmuWs bw = bmu_carve(ws, n);
    int *cand = bw.cand, *ccount = bw.ccount;
    if (g_rerank_pipe < 0) {
        const char *e = getenv("SOMB_RERANK_PIPE");
        g_rerank_pipe = e ? atoi(e) != 0 : 1;
    }
    int all = screen_impl == 2, split = screen_impl == 0 || screen_impl == 3;
    OvfView ov{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    if (split) ov = OvfView{bw.ovf_head, bw.ovf_lim, bw.pool.ent, bw.pool.next, bw.pool.cnt, bw.ctrs + 3};
    if (all) cudaMemsetAsync(flags, 0, (size_t)n * sizeof(int), st);
    const int wpb = 8;
    const unsigned blocks = (unsigned)((n + wpb - 1) / wpb);
    if (!all && d % 4 == 0 && d <= 1024 && g_rerank_pipe) {
        if (d <= 128)
            launch_rerank_pipe<1>(st, X, x2, n, d, W, w2, K, cand, ccount, dist_mode, split, row_order, ov, bmu, d2min);
        else if (d <= 256)
            launch_rerank_pipe<2>(st, X, x2, n, d, W, w2, K, cand, ccount, dist_mode, split, row_order, ov, bmu, d2min);
        else if (d <= 512)
            launch_rerank_pipe<4>(st, X, x2, n, d, W, w2, K, cand, ccount, dist_mode, split, row_order, ov, bmu, d2min);
        else
            launch_rerank_pipe<8>(st, X, x2, n, d, W, w2, K, cand, ccount, dist_mode, split, row_order, ov, bmu, d2min);
    } else if (!all && d % 4 == 0 && d <= 1024) {
        if (d <= 128)
            launch_rerank_vec<1>(blocks, st, X, x2, n, d, W, w2, K, cand, ccount, dist_mode, split, row_order, ov, bmu, d2min);
        else if (d <= 256)
            launch_rerank_vec<2>(blocks, st, X, x2, n, d, W, w2, K, cand, ccount, dist_mode, split, row_order, ov, bmu, d2min);
        else if (d <= 512)
            launch_rerank_vec<4>(blocks, st, X, x2, n, d, W, w2, K, cand, ccount, dist_mode, split, row_order, ov, bmu, d2min);
        else
            launch_rerank_vec<8>(blocks, st, X, x2, n, d, W, w2, K, cand, ccount, dist_mode, split, row_order, ov, bmu, d2min);
    } else {
        rerank_kernel<<<blocks, 32 * wpb, 0, st>>>(X, x2, n, d, W, w2, K, cand, ccount, dist_mode, all, split,
                                                   row_order, ov, bmu, d2min);
    }
    note_launch();
    SOMB_LAUNCH_CHECK("rerank");
    return SOMB_OK;
}

extern "C" int somb_bmu_dense(const uint16_t *Xh, const float *X, const float *xstat, const double *x2,
                              int64_t n, int32_t d, int32_t dp, const uint16_t *Wh, const float *W,
                              const float *c, const double *w2, int32_t K, int32_t kp,
                              const float *scal, float window_coef, int32_t dist_mode,
                              int32_t screen_impl, int32_t *bmu, double *d2min, int32_t *flags,
                              void *ws, void *stream) {
    SOMB_REQUIRE(K > 0 && d > 0 && dp >= d && kp >= K, SOMB_E_INPUT,
                 "bmu_dense: bad shape K=%d d=%d dp=%d kp=%d", K, d, dp, kp);
    int rc = somb_bmu_screen(Xh, nullptr, xstat, n, dp, Wh, nullptr, c, K, kp, scal, window_coef, nullptr,
                             screen_impl, flags, ws, stream);
    if (rc) return rc;
    return somb_bmu_rerank(X, x2, n, d, W, w2, K, dist_mode, screen_impl, nullptr, bmu, d2min, flags, ws, stream);
}

extern "C" int64_t somb_bmu_repaired_rows(const void *ws, int64_t n, void *stream) {
    // rows of the last screen whose truncated candidate set was replaced by
    // an exact full scan (host read: synchronises the stream)
    BmuWs w = bmu_carve(const_cast<void *>(ws), n);
    unsigned v = 0;
    cudaStream_t st = as_stream(stream);
    if (cudaMemcpyAsync(&v, w.ctrs + 4, sizeof(unsigned), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return -1;
    return (int64_t)v;
}

extern "C" int somb_qe_sum(const double *d2min, int64_t n, double *out, void *ws, void *stream) {
    cudaStream_t st = as_stream(stream);
    int np = (int)((n + kQeTile - 1) / kQeTile);
    if (np == 0) {
        cudaMemsetAsync(out, 0, sizeof(double), st);
        return SOMB_OK;
    }
    double *part = (double *)ws;   // >= np doubles (callers pass somb_bmu_ws-sized ws)
    qe_partial<<<np, 256, 0, st>>>(d2min, n, part);
    note_launch();
    qe_final<<<1, 256, 0, st>>>(part, np, out);
    note_launch();
    SOMB_LAUNCH_CHECK("qe_sum");
    return SOMB_OK;
}

// Debug/calibration: screened values r_j of rows [0, min(n, 128)) for all kp
// nodes from the tcgen05 kernel (dump [128][kp] f32); candidates are
// computed as usual.  Used to measure the real screen error.
extern "C" int somb_debug_screen_dump(const uint16_t *Xh, const uint16_t *Xl, const float *xstat, int64_t n,
                                      int32_t dp, const uint16_t *Wh, const uint16_t *Wl, const float *c, int32_t kp,
                                      const float *scal, float window_coef, int32_t passes, float *dump, void *ws,
                                      void *stream) {
    int64_t m = n < 128 ? n : 128;
    BmuWs w = bmu_carve(ws, n);
    int *flags = (int *)w.thr0;
    return launch_screen_tc((const __half *)Xh, (const __half *)Xl, m, dp, (const __half *)Wh, (const __half *)Wl, kp,
                            c, xstat, scal, window_coef, nullptr, w.cand, w.ccount, flags, dump, w.ctrs, w.pool,
                            w.ovf_head, w.ovf_lim, passes, as_stream(stream));
}


// Full BMU search in one call: previous-BMU seed + screen + exact re-rank.
extern "C" int somb_bmu_search(const uint16_t *Xh, const uint16_t *Xl, const float *X, const float *xstat,
                               const double *x2, int64_t n, int32_t d, int32_t dp, const uint16_t *Wh,
                               const uint16_t *Wl, const float *W, const float *c, const double *w2, int32_t K,
                               int32_t kp, const float *scal, float window_coef, const int32_t *prev_bmu,
                               const int32_t *row_order, int32_t dist_mode, int32_t screen_impl, int32_t *bmu,
                               double *d2min, int32_t *flags, void *ws, void *stream) {
    SOMB_REQUIRE(K > 0 && d > 0 && dp >= d && dp % 8 == 0 && kp >= K && kp % 256 == 0, SOMB_E_INPUT,
                 "bmu_search: bad shape K=%d d=%d dp=%d kp=%d", K, d, dp, kp);
    int rc = somb_bmu_screen(Xh, Xl, xstat, n, dp, Wh, Wl, c, K, kp, scal, window_coef, prev_bmu, screen_impl, flags,
                             ws, stream);
    if (rc) return rc;
    return somb_bmu_rerank(X, x2, n, d, W, w2, K, dist_mode, screen_impl, row_order, bmu, d2min, flags, ws, stream);
}
