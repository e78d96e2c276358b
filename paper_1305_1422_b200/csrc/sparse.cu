// Sparse (CSR) BMU search and node sums (kernels.py:208-222, 229-242, 315-321).
//
// Screen: dots_ij = sum_{k in nz(i)} v_k delta_j[k] against the centred
// codebook stored TRANSPOSED (dT[k][j] = w_jk - mu_k, fp32, pitch kp), so each
// nonzero gathers one contiguous node slice; r_ij = c_j - 2 dots_ij with
// c_j = |delta_j|^2 + 2 mu.delta_j (prep with nu = 0).  One warp per row, 8
// nodes per lane per 256-node step, fp32 FMA.  The window is rigorous for
// this arithmetic: |r~ - r| <= 2 (nnz + 2) 2^-24 sum|x||delta| + rounding of
// c, bounded through Cauchy-Schwarz by coef * |x_i| * max_j |delta_j|.
// Candidates are collected warp-cooperatively in ascending node order with
// the same window/cap semantics as the dense screen (cand.cuh), then the exact
// fp64 re-rank evaluates the reference's sparse formula (x2 - 2 dots) + w2.
#include "cand.cuh"
#include "rerank.cuh"

namespace somb {

int launch_repair_truncated(const int *flags, int *ccount, int64_t n, unsigned *ctrs, cudaStream_t st, int *list);

constexpr int SP_WARPS = 8;
constexpr int SP_NNZ_BUF = 256;      // staged (col, val) pairs per warp
constexpr int SP_CAP = 32;           // candidates in shared memory per row before spilling to the pool

// dT[k][j] = fp32(w_jk - mu_k) for j < K, 0 for padding (prepare-time transpose)
__global__ void sp_transpose(const float *__restrict__ W, const float *__restrict__ mu, int K, int d, int kp,
                             float *__restrict__ dT) {
    __shared__ float tile[32][33];
    const int j0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;   // 32 x 8
    for (int r = ty; r < 32; r += 8) {
        int j = j0 + r, k = k0 + tx;
        tile[r][tx] = (j < K && k < d) ? (float)((double)W[(int64_t)j * d + k] - (double)mu[k]) : 0.0f;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        int k = k0 + r, j = j0 + tx;
        if (k < d && j < kp) dT[(int64_t)k * kp + j] = tile[tx][r];
    }
}

// WT[k][j] = w_jk exactly (the repair scan's operand), only when rows were
// repaired (*nlist > 0): written into the caller's dT buffer after the screen
// has used it (the next prepare rebuilds dT)
__global__ void sp_transpose_if(const float *__restrict__ W, int K, int d, int kp, float *__restrict__ WT,
                                const unsigned *__restrict__ nlist) {
    if (*nlist == 0) return;
    __shared__ float tile[32][33];
    const int j0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;   // 32 x 8
    for (int r = ty; r < 32; r += 8) {
        int j = j0 + r, k = k0 + tx;
        tile[r][tx] = (j < K && k < d) ? W[(int64_t)j * d + k] : 0.0f;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        int k = k0 + r, j = j0 + tx;
        if (k < d && j < kp) WT[(int64_t)k * kp + j] = tile[tx][r];
    }
}

__global__ void sp_row_norms(const int64_t *__restrict__ rowptr, const float *__restrict__ val, int64_t n,
                             double *__restrict__ x2, float *__restrict__ xnorm, int *__restrict__ nnz_max) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s = 0.0;
    for (int64_t e = rowptr[i]; e < rowptr[i + 1]; ++e) {   // np.add.at order (kernels.py:315-321)
        double v = (double)val[e];
        s += v * v;
    }
    x2[i] = s;
    xnorm[i] = (float)sqrt(s);
    atomicMax(nnz_max, (int)(rowptr[i + 1] - rowptr[i]));
}

__global__ void __launch_bounds__(32 * SP_WARPS)
sp_screen_kernel(const int64_t *__restrict__ rowptr, const int *__restrict__ col, const float *__restrict__ val,
                 int64_t n, const float *__restrict__ dT, int kp, const float *__restrict__ c,
                 const float *__restrict__ xnorm, const float *__restrict__ scal, float wcoef,
                 int *__restrict__ cand, int *__restrict__ ccount, int *__restrict__ flags, OvfPool pool,
                 int *__restrict__ ovf_head, float *__restrict__ ovf_lim) {
    __shared__ int s_col[SP_WARPS][SP_NNZ_BUF];
    __shared__ float s_val[SP_WARPS][SP_NNZ_BUF];
    __shared__ float s_bv[SP_WARPS][SP_CAP];
    __shared__ int s_bi[SP_WARPS][SP_CAP];
    const int w = threadIdx.x / 32, lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * SP_WARPS + w;
    if (row >= n) return;
    const int64_t e0 = rowptr[row], e1 = rowptr[row + 1];
    const int nnz = (int)(e1 - e0);
    const float nmax = scal[1];
    CandRow<SP_CAP> st;   // meaningful in lane 0 only
    cand_init(st, wcoef * (float)(nnz + 2) * xnorm[row] * nmax + ldexpf(scal[4], -21));
    const CandBuf cb{smem_addr(&s_bv[w][0]), smem_addr(&s_bi[w][0]), 4u};
    float thr = st.thr;
    for (int j0 = 0; j0 < kp; j0 += 256) {
        const int jl = j0 + lane * 8;
        const float4 *cp = reinterpret_cast<const float4 *>(c + jl);
        const float4 c0 = __ldg(cp), c1 = __ldg(cp + 1);
        // a chunk of masked nodes (padding, or rows bit-identical to node 0:
        // c = +inf, prep.cu) can never hold the BMU -- skip its gather
        const bool fin = fminf(fminf(fminf(c0.x, c0.y), fminf(c0.z, c0.w)),
                               fminf(fminf(c1.x, c1.y), fminf(c1.z, c1.w))) < INFINITY;
        if (!__any_sync(0xffffffffu, fin)) continue;
        float acc[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = 0.0f;
        for (int b0 = 0; b0 < nnz; b0 += SP_NNZ_BUF) {
            const int m = min(SP_NNZ_BUF, nnz - b0);
            __syncwarp();
            for (int t = lane; t < m; t += 32) {
                s_col[w][t] = col[e0 + b0 + t];
                s_val[w][t] = val[e0 + b0 + t];
            }
            __syncwarp();
            for (int t = 0; t < m; ++t) {
                const float v = s_val[w][t];
                const float4 *p = reinterpret_cast<const float4 *>(dT + (int64_t)s_col[w][t] * kp + jl);
                float4 a = __ldg(p), b = __ldg(p + 1);
                acc[0] = fmaf(v, a.x, acc[0]); acc[1] = fmaf(v, a.y, acc[1]);
                acc[2] = fmaf(v, a.z, acc[2]); acc[3] = fmaf(v, a.w, acc[3]);
                acc[4] = fmaf(v, b.x, acc[4]); acc[5] = fmaf(v, b.y, acc[5]);
                acc[6] = fmaf(v, b.z, acc[6]); acc[7] = fmaf(v, b.w, acc[7]);
            }
        }
        float r[8] = {fmaf(-2.0f, acc[0], c0.x), fmaf(-2.0f, acc[1], c0.y), fmaf(-2.0f, acc[2], c0.z),
                      fmaf(-2.0f, acc[3], c0.w), fmaf(-2.0f, acc[4], c1.x), fmaf(-2.0f, acc[5], c1.y),
                      fmaf(-2.0f, acc[6], c1.z), fmaf(-2.0f, acc[7], c1.w)};
        float lo = fminf(fminf(fminf(r[0], r[1]), fminf(r[2], r[3])), fminf(fminf(r[4], r[5]), fminf(r[6], r[7])));
        unsigned hit = __ballot_sync(0xffffffffu, lo <= thr);
        if (hit) {
            // visit the hit lanes in ascending node order; lane 0 owns the row state
            while (hit) {
                const int src = __ffs(hit) - 1;
                hit &= hit - 1;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    float vq = __shfl_sync(0xffffffffu, r[q], src);
                    if (lane == 0 && vq <= st.thr) cand_push<SP_CAP>(st, vq, j0 + src * 8 + q, cb, pool);
                }
            }
            thr = __shfl_sync(0xffffffffu, st.thr, 0);
        }
    }
    if (lane == 0) {
        ccount[row] = cand_emit<SP_CAP>(st, cb, cand + row * SOMB_CAND_CAP);
        flags[row] = st.trunc;
        ovf_head[4 * row] = st.head;          // one column group: slots 1..3 stay empty
        ovf_lim[4 * row] = st.rmin + st.win;
    }
}

// ------------------------------------------------- lockstep sparse screen
// The gather above is DRAM-bound: every row sweeps the whole transposed
// codebook (2 GB at cfg3), so concurrently running rows touch it at random
// and L2 hits are ~5% (profiles/).  Here the node loop is OUTSIDE: all
// warps sweep one 128-node slab of dT (K-chunk, 25.6 MB at cfg3) over their
// rows before moving to the next, a global counter keeping them within LAG
// slabs of each other, so the slab is served from L2.  Each row's window
// state and candidate buffer persist in global memory between slabs; the
// row's nonzeros are re-staged per slab (2 KB, 1/64 of the gathered bytes).
// Semantics (window, visiting order, spill, emit) equal sp_screen_kernel.
constexpr int SPL_CH = 128;          // nodes per slab (4 per lane)

struct SpRowState {
    float rmin, thr, capbelow, win;
    int cnt, trunc, head, pad;
};

__device__ __forceinline__ void sp_state_load(CandRow<SP_CAP> &st, const SpRowState &g) {
    st.rmin = g.rmin; st.thr = g.thr; st.capbelow = g.capbelow; st.win = g.win;
    st.cnt = g.cnt; st.trunc = g.trunc; st.head = g.head;
}
__device__ __forceinline__ void sp_state_store(const CandRow<SP_CAP> &st, SpRowState &g) {
    g.rmin = st.rmin; g.thr = st.thr; g.capbelow = st.capbelow; g.win = st.win;
    g.cnt = st.cnt; g.trunc = st.trunc; g.head = st.head;
}

__global__ void __launch_bounds__(32 * SP_WARPS)
sp_screen_ls_kernel(const int64_t *__restrict__ rowptr, const int *__restrict__ col, const float *__restrict__ val,
                    int64_t n, const float *__restrict__ dT, int kp, const float *__restrict__ c,
                    const float *__restrict__ xnorm, const float *__restrict__ scal, float wcoef,
                    int *__restrict__ cand, int *__restrict__ ccount, int *__restrict__ flags, OvfPool pool,
                    int *__restrict__ ovf_head, float *__restrict__ ovf_lim, SpRowState *__restrict__ rs,
                    float *__restrict__ gbv, int *__restrict__ gbi, unsigned *__restrict__ done_ctr, int lag) {
    __shared__ int s_col[SP_WARPS][SP_NNZ_BUF];
    __shared__ float s_val[SP_WARPS][SP_NNZ_BUF];
    const int w = threadIdx.x / 32, lane = threadIdx.x & 31;
    const int64_t gw = (int64_t)blockIdx.x * SP_WARPS + w, GW = (int64_t)gridDim.x * SP_WARPS;
    const float nmax = scal[1];
    if (lane == 0) {
        for (int64_t row = gw; row < n; row += GW) {
            CandRow<SP_CAP> st;
            const int nnz = (int)(rowptr[row + 1] - rowptr[row]);
            cand_init(st, wcoef * (float)(nnz + 2) * xnorm[row] * nmax + ldexpf(scal[4], -21));
            sp_state_store(st, rs[row]);
        }
    }
    const int NC = kp / SPL_CH;
    for (int ci = 0; ci < NC; ++ci) {
        if (lane == 0 && ci > lag) {   // soft lockstep over the slabs (lag slabs ahead at most)
            const unsigned need = (unsigned)GW * (unsigned)(ci - lag);
            for (int spin = 0; spin < (1 << 22); ++spin) {
                unsigned cur;
                asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(done_ctr) : "memory");
                if (cur >= need) break;
                __nanosleep(128);
            }
        }
        __syncwarp();
        const int j0 = ci * SPL_CH;
        const int jl = j0 + lane * 4;
        const float4 c4 = __ldg(reinterpret_cast<const float4 *>(c + jl));
        const bool fin = fminf(fminf(c4.x, c4.y), fminf(c4.z, c4.w)) < INFINITY;
        if (__any_sync(0xffffffffu, fin)) {   // a slab of masked nodes cannot hold a BMU
#pragma unroll 1
            for (int64_t row = gw; row < n; row += GW) {
                CandRow<SP_CAP> st;
                if (lane == 0) sp_state_load(st, rs[row]);
                float thr = __shfl_sync(0xffffffffu, lane == 0 ? st.thr : 0.0f, 0);
                const int64_t e0 = rowptr[row], e1 = rowptr[row + 1];
                const int nnz = (int)(e1 - e0);
                float acc[4] = {0.f, 0.f, 0.f, 0.f};
                for (int b0 = 0; b0 < nnz; b0 += SP_NNZ_BUF) {
                    const int m = min(SP_NNZ_BUF, nnz - b0);
                    __syncwarp();
                    for (int t = lane; t < m; t += 32) {
                        s_col[w][t] = col[e0 + b0 + t];
                        s_val[w][t] = val[e0 + b0 + t];
                    }
                    __syncwarp();
#pragma unroll 16
                    for (int t = 0; t < m; ++t) {
                        const float v = s_val[w][t];
                        const float4 a = __ldg(reinterpret_cast<const float4 *>(dT + (int64_t)s_col[w][t] * kp + jl));
                        acc[0] = fmaf(v, a.x, acc[0]); acc[1] = fmaf(v, a.y, acc[1]);
                        acc[2] = fmaf(v, a.z, acc[2]); acc[3] = fmaf(v, a.w, acc[3]);
                    }
                }
                float r[4] = {fmaf(-2.0f, acc[0], c4.x), fmaf(-2.0f, acc[1], c4.y), fmaf(-2.0f, acc[2], c4.z),
                              fmaf(-2.0f, acc[3], c4.w)};
                const float lo = fminf(fminf(r[0], r[1]), fminf(r[2], r[3]));
                unsigned hit = __ballot_sync(0xffffffffu, lo <= thr);
                if (hit) {
                    const CandBufG cb{gbv + row * SP_CAP, gbi + row * SP_CAP};
                    while (hit) {   // ascending node order; lane 0 owns the row state
                        const int src = __ffs(hit) - 1;
                        hit &= hit - 1;
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const float vq = __shfl_sync(0xffffffffu, r[q], src);
                            if (lane == 0 && vq <= st.thr) cand_push<SP_CAP>(st, vq, j0 + src * 4 + q, cb, pool);
                        }
                    }
                    if (lane == 0) sp_state_store(st, rs[row]);
                }
            }
        }
        __syncwarp();
        if (lane == 0) {
            __threadfence();
            atomicAdd(done_ctr, 1u);
        }
    }
    if (lane == 0) {
        for (int64_t row = gw; row < n; row += GW) {
            CandRow<SP_CAP> st;
            sp_state_load(st, rs[row]);
            const CandBufG cb{gbv + row * SP_CAP, gbi + row * SP_CAP};
            ccount[row] = cand_emit<SP_CAP>(st, cb, cand + row * SOMB_CAND_CAP);
            flags[row] = st.trunc;
            ovf_head[4 * row] = st.head;
            ovf_lim[4 * row] = st.rmin + st.win;
        }
    }
}

// Exact fp64 re-rank with the reference's sparse formula:
// d2 = (x2 - 2 sum_t v_t w_j[col_t]) + w2_j, clamp >= 0 (kernels.py:216-219).
__global__ void sp_rerank_kernel(const int64_t *__restrict__ rowptr, const int *__restrict__ col,
                                 const float *__restrict__ val, int64_t n, int d, const float *__restrict__ W,
                                 const double *__restrict__ w2, int K, const double *__restrict__ x2,
                                 const int *__restrict__ cand, const int *__restrict__ ccount, int all,
                                 OvfPool pool, const int *__restrict__ ovf_head, const float *__restrict__ ovf_lim,
                                 int *__restrict__ bmu, double *__restrict__ d2min) {
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (row >= n) return;
    const int64_t e0 = rowptr[row], e1 = rowptr[row + 1];
    int cnt = all == 1 ? 0 : ccount[row];
    if (all == 2 && cnt < 0) return;   // repaired row: somb_bmu_sparse_repair's lockstep scan takes it
    // repaired row (kScanAll), or no candidate anywhere: exact scan of every node
    const bool scan = all == 1 || cnt < 0 || (cnt == 0 && ovf_head[4 * row] < 0);
    if (scan) cnt = K;
    double best = INFINITY;
    int bestj = 0x7fffffff;
    const double xx = x2[row];
    auto eval = [&](int j) {
        if ((unsigned)j >= (unsigned)K) return;
        const float *wr = W + (int64_t)j * d;
        double s = 0.0;
        for (int64_t e = e0 + lane; e < e1; e += 32) s = __fma_rn((double)val[e], (double)wr[col[e]], s);
        s = warp_sum(s);
        double v = fmax(__dadd_rn(__dsub_rn(xx, __dmul_rn(2.0, s)), w2[j]), 0.0);
        if (v < best || (v == best && j < bestj)) {
            best = v;
            bestj = j;
        }
    };
    for (int q = 0; q < cnt; ++q) eval(scan ? q : cand[row * SOMB_CAND_CAP + q]);
    if (!scan) {   // spilled candidates (the screen's overflow chunks within the final window)
        const float lim = ovf_lim[4 * row];
        for (int c = ovf_head[4 * row]; c >= 0; c = pool.next[c]) {
            const int m = pool.cnt[c];
            const int2 e = lane < m ? pool.ent[(size_t)c * kOvfChunk + lane] : make_int2(0x7f800000, -1);
            unsigned bal = __ballot_sync(0xffffffffu, lane < m && __int_as_float(e.x) <= lim);
            while (bal) {
                const int src = __ffs(bal) - 1;
                bal &= bal - 1u;
                eval(__shfl_sync(0xffffffffu, e.y, src));
            }
        }
    }
    if (lane == 0) {
        bmu[row] = bestj;
        d2min[row] = best;
    }
}

// Exact scan of the repaired rows (truncated candidate sets), slab-lockstep
// like the screen: all warps sweep the same 128-node slab of the transposed
// ORIGINAL codebook WT[k][j] = w_jk (exact copy, pitch kp) before the next,
// so the slab stays in L2; per (row, node) the reference's sparse formula
// (x2 - 2 sum_t v_t w_j[col_t]) + w2_j, clamped >= 0 (kernels.py:216-219),
// with fp32 products accumulated exactly in fp64; first minimum (lowest
// index) over nodes.  A row's running best lives in its own (unused)
// candidate slots.  The per-row full scan gathered 250 scattered codebook
// values per node and took 4 s in cfg3's degenerate epoch 1.
__global__ void __launch_bounds__(32 * SP_WARPS)
sp_exact_ls_kernel(const int64_t *__restrict__ rowptr, const int *__restrict__ col, const float *__restrict__ val,
                   const int *__restrict__ list, const unsigned *__restrict__ nlist, const float *__restrict__ WT,
                   int kp, int K, const double *__restrict__ w2, const double *__restrict__ x2,
                   int *__restrict__ cand, int *__restrict__ bmu, double *__restrict__ d2min,
                   unsigned *__restrict__ done_ctr) {
    // values staged as fp64 once per warp (v and v 2^896): the per-lane F2F of
    // every gathered codebook value was the limiter (XU pipe 74% busy, ncu)
    __shared__ int s_col[SP_WARPS][SP_NNZ_BUF];
    __shared__ double s_vd[SP_WARPS][SP_NNZ_BUF];
    __shared__ double s_vs[SP_WARPS][SP_NNZ_BUF];
    const int w = threadIdx.x / 32, lane = threadIdx.x & 31;
    const int64_t gw = (int64_t)blockIdx.x * SP_WARPS + w, GW = (int64_t)gridDim.x * SP_WARPS;
    const int64_t m = (int64_t)*nlist;
    if (m == 0) return;
    auto best_of = [&](int64_t row) { return reinterpret_cast<double *>(cand + row * SOMB_CAND_CAP); };
    if (lane == 0)
        for (int64_t i = gw; i < m; i += GW) {
            const int64_t row = list[i];
            *best_of(row) = INFINITY;
            cand[row * SOMB_CAND_CAP + 2] = 0x7fffffff;
        }
    const int NC = kp / SPL_CH;
    for (int ci = 0; ci < NC; ++ci) {
        if (lane == 0 && ci > 0) {   // slab barrier
            const unsigned need = (unsigned)GW * (unsigned)ci;
            for (int spin = 0; spin < (1 << 22); ++spin) {
                unsigned cur;
                asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(done_ctr) : "memory");
                if (cur >= need) break;
                __nanosleep(128);
            }
        }
        __syncwarp();
        const int jl = ci * SPL_CH + lane * 4;
#pragma unroll 1
        for (int64_t i = gw; i < m; i += GW) {
            const int64_t row = list[i];
            const int64_t e0 = rowptr[row], e1 = rowptr[row + 1];
            const int nnz = (int)(e1 - e0);
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            for (int b0 = 0; b0 < nnz; b0 += SP_NNZ_BUF) {
                const int mm = min(SP_NNZ_BUF, nnz - b0);
                __syncwarp();
                for (int t = lane; t < mm; t += 32) {
                    s_col[w][t] = col[e0 + b0 + t];
                    const double v = (double)val[e0 + b0 + t];
                    s_vd[w][t] = v;
                    s_vs[w][t] = v * kF64Scale;   // exact: |v| < 2^128
                }
                __syncwarp();
                // two components convert on F2F (XU pipe), two by the exact
                // integer re-exponenting against v 2^896 (ALU pipes): every
                // product is the exact v a either way, so the sums are
                // bit-identical to the all-F2F form
#pragma unroll 8
                for (int t = 0; t < mm; ++t) {
                    const double v = s_vd[w][t], vs = s_vs[w][t];
                    const float4 a = __ldg(reinterpret_cast<const float4 *>(WT + (int64_t)s_col[w][t] * kp + jl));
                    acc[0] = __fma_rn(v, (double)a.x, acc[0]); acc[1] = __fma_rn(v, (double)a.y, acc[1]);
                    acc[2] = __fma_rn(vs, f32_as_f64_scaled(a.z), acc[2]);
                    acc[3] = __fma_rn(vs, f32_as_f64_scaled(a.w), acc[3]);
                }
            }
            const double xx = x2[row];
            double bv = INFINITY;
            int bj = 0x7fffffff;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int j = jl + q;
                if (j < K) {
                    const double v = fmax(__dadd_rn(__dsub_rn(xx, __dmul_rn(2.0, acc[q])), w2[j]), 0.0);
                    if (v < bv) { bv = v; bj = j; }   // ascending j: strict < keeps the first minimum
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
                if (ov < bv || (ov == bv && oj < bj)) { bv = ov; bj = oj; }
            }
            if (lane == 0 && bj != 0x7fffffff) {
                double *bp = best_of(row);
                int *jp = cand + row * SOMB_CAND_CAP + 2;
                if (bv < *bp) { *bp = bv; *jp = bj; }   // slabs in ascending node order: earlier wins ties
            }
        }
        __syncwarp();
        if (lane == 0) {
            __threadfence();
            atomicAdd(done_ctr, 1u);
        }
    }
    if (lane == 0)
        for (int64_t i = gw; i < m; i += GW) {
            const int64_t row = list[i];
            bmu[row] = cand[row * SOMB_CAND_CAP + 2];
            d2min[row] = *best_of(row);
        }
}

int node_bucket_sort(const int *bmu, int64_t n, int K, void *ws, const int **perm, const int **off, double *cnt,
                     cudaStream_t st);
void node_seg_plan(void *ws, int64_t n, int d, int K, int seg, int **nseg, int **segoff, int **msegoff, double **P,
                   size_t *P_doubles, cudaStream_t st);

// Large nodes (the reference's degenerate sparse fixed point maps every row
// to node 0) are summed in fixed segments of SP_SEG sorted rows, one block
// per segment, into partial rows folded in segment order (sp_seg_fold) --
// the dense path's scheme (nodesum.cu) with a sparse scatter.
constexpr int SP_SEG = 2048;

__global__ void sp_seg_sum_kernel(const int64_t *__restrict__ rowptr, const int *__restrict__ col,
                                  const float *__restrict__ val, int d, const int *__restrict__ perm,
                                  const int *__restrict__ off, const int *__restrict__ segoff,
                                  const int *__restrict__ msegoff, const int *__restrict__ nseg, int K, int dc,
                                  double *__restrict__ S, double *__restrict__ P) {
    const int s = blockIdx.x;
    if (s >= segoff[K]) return;
    int lo = 0, hi = K;   // b = the node owning global segment s
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (segoff[mid] <= s) lo = mid; else hi = mid - 1;
    }
    int b = lo;
    while (b + 1 <= K && segoff[b + 1] <= s) ++b;
    const int sub = s - segoff[b];
    const int r0 = off[b] + sub * SP_SEG, r1 = min(off[b + 1], r0 + SP_SEG);
    double *prow = nseg[b] > 1 ? P + (int64_t)(msegoff[b] + sub) * d : nullptr;
    for (int t = r0; t < r1; ++t) {
        const int i = perm[t];
        for (int64_t e = rowptr[i] + threadIdx.x; e < rowptr[i + 1]; e += blockDim.x) {
            if (prow) prow[col[e]] += (double)val[e];
            else S[s_index(b, col[e], dc, K)] += (double)val[e];
        }
        __syncthreads();
    }
}

__global__ void sp_seg_fold(const double *__restrict__ P, const int *__restrict__ msegoff,
                            const int *__restrict__ nseg, int d, int K, int dc, double *__restrict__ S) {
    const int b = blockIdx.y;
    const int ns = nseg[b];
    if (ns <= 1) return;
    const double *p = P + (int64_t)msegoff[b] * d;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < d; k += gridDim.x * blockDim.x) {
        double a = 0.0;
        for (int q = 0; q < ns; ++q) a += p[(int64_t)q * d + k];
        S[s_index(b, k, dc, K)] = a;
    }
}

}  // namespace somb

using namespace somb;

extern "C" int somb_sparse_row_stats(const int64_t *rowptr, const float *val, int64_t n, double *x2, float *xnorm,
                                     int32_t *nnz_max, void *stream) {
    cudaStream_t st = as_stream(stream);
    cudaMemsetAsync(nnz_max, 0, sizeof(int), st);
    if (n == 0) return SOMB_OK;
    sp_row_norms<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(rowptr, val, n, x2, xnorm, nnz_max);
    note_launch();
    SOMB_LAUNCH_CHECK("sparse_row_stats");
    return SOMB_OK;
}

extern "C" int somb_sparse_codebook_T(const float *W, const float *mu, int32_t K, int32_t d, int32_t kp, float *dT,
                                      void *stream) {
    SOMB_REQUIRE(kp % 256 == 0 && kp >= K, SOMB_E_INPUT, "sparse_codebook_T: kp must be a multiple of 256");
    dim3 g((kp + 31) / 32, (d + 31) / 32);
    sp_transpose<<<g, dim3(32, 8), 0, as_stream(stream)>>>(W, mu, K, d, kp, dT);
    note_launch();
    SOMB_LAUNCH_CHECK("sparse_codebook_T");
    return SOMB_OK;
}

extern "C" int somb_bmu_sparse(const int64_t *rowptr, const int32_t *col, const float *val, int64_t n, int32_t d,
                               const float *dT, const float *W, const float *c, const double *w2, int32_t K,
                               int32_t kp, const float *scal, const double *x2, const float *xnorm, float window_coef,
                               int32_t exact, int32_t *bmu, double *d2min, int32_t *flags, void *ws, void *stream) {
    SOMB_REQUIRE(K > 0 && d > 0 && kp % 256 == 0, SOMB_E_INPUT, "bmu_sparse: bad shape");
    if (n == 0) return SOMB_OK;
    cudaStream_t st = as_stream(stream);
    BmuWs w = bmu_carve(ws, n);
    int *cand = w.cand, *ccount = w.ccount;
    SOMB_REQUIRE(exact >= 0 && exact <= 2, SOMB_E_CONFIG, "bmu_sparse: exact must be 0, 1 or 2");
    if (exact != 1) {
        cudaMemsetAsync(w.ctrs, 0, 4 * sizeof(unsigned), st);
        static int ls = -1, lag = 0;   // SOMB_SPARSE_LOCKSTEP=0: row-at-a-time gather; SOMB_SPARSE_LAG (0 = slab barrier, measured best)
        if (ls < 0) {
            const char *e = getenv("SOMB_SPARSE_LOCKSTEP");
            ls = e ? atoi(e) != 0 : 1;
            const char *l = getenv("SOMB_SPARSE_LAG");
            if (l) lag = atoi(l);
        }
        if (ls && kp % SPL_CH == 0) {
            size_t base = 0;
            bmu_carve(nullptr, n, &base);
            char *p = (char *)ws + base;
            SpRowState *rs = (SpRowState *)p;
            p += align_up((size_t)n * sizeof(SpRowState), 256);
            float *gbv = (float *)p;
            p += align_up((size_t)n * SP_CAP * sizeof(float), 256);
            int *gbi = (int *)p;
            int dev = 0, sms = kSmCount, per_sm = 1;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sp_screen_ls_kernel, 32 * SP_WARPS, 0);
            if (per_sm < 1) per_sm = 1;
            const int64_t need = (n + SP_WARPS - 1) / SP_WARPS;
            const unsigned grid = (unsigned)(need < (int64_t)per_sm * sms ? need : (int64_t)per_sm * sms);
            sp_screen_ls_kernel<<<grid, 32 * SP_WARPS, 0, st>>>(rowptr, col, val, n, dT, kp, c, xnorm, scal,
                                                               window_coef, cand, ccount, flags, w.pool, w.ovf_head,
                                                               w.ovf_lim, rs, gbv, gbi, w.ctrs + 2, lag);
        } else {
            sp_screen_kernel<<<(unsigned)((n + SP_WARPS - 1) / SP_WARPS), 32 * SP_WARPS, 0, st>>>(
                rowptr, col, val, n, dT, kp, c, xnorm, scal, window_coef, cand, ccount, flags, w.pool, w.ovf_head,
                w.ovf_lim);
        }
        note_launch();
        // truncated rows -> exact full scan (listed in the thr0 area for somb_bmu_sparse_repair)
        int rc = launch_repair_truncated(flags, ccount, n, w.ctrs, st, reinterpret_cast<int *>(w.thr0));
        if (rc) return rc;
    } else {
        cudaMemsetAsync(flags, 0, (size_t)n * sizeof(int), st);
    }
    sp_rerank_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(rowptr, col, val, n, d, W, w2, K, x2, cand, ccount,
                                                              exact, w.pool, w.ovf_head, w.ovf_lim, bmu, d2min);
    note_launch();
    SOMB_LAUNCH_CHECK("bmu_sparse");
    return SOMB_OK;
}

extern "C" int somb_bmu_sparse_repair(const int64_t *rowptr, const int32_t *col, const float *val, int64_t n,
                                      int32_t d, const float *W, int32_t K, int32_t kp, const double *w2,
                                      const double *x2, float *WT, int32_t *bmu, double *d2min, void *ws,
                                      void *stream) {
    SOMB_REQUIRE(K > 0 && d > 0 && kp % SPL_CH == 0 && kp >= K && W && WT, SOMB_E_INPUT,
                 "bmu_sparse_repair: bad shape");
    if (n == 0) return SOMB_OK;
    cudaStream_t st = as_stream(stream);
    BmuWs w = bmu_carve(ws, n);
    sp_transpose_if<<<dim3((kp + 31) / 32, (d + 31) / 32), dim3(32, 8), 0, st>>>(W, K, d, kp, WT, w.ctrs + 4);
    note_launch();
    cudaMemsetAsync(w.ctrs + 6, 0, sizeof(unsigned), st);
    int dev = 0, sms = kSmCount, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sp_exact_ls_kernel, 32 * SP_WARPS, 0);
    if (per_sm < 1) per_sm = 1;
    // a persistent grid that is always co-resident (the slab barrier waits for every warp)
    sp_exact_ls_kernel<<<(unsigned)(per_sm * sms), 32 * SP_WARPS, 0, st>>>(
        rowptr, col, val, reinterpret_cast<const int *>(w.thr0), w.ctrs + 4, WT, kp, K, w2, x2, w.cand, bmu, d2min,
        w.ctrs + 6);
    note_launch();
    SOMB_LAUNCH_CHECK("bmu_sparse_repair");
    return SOMB_OK;
}

extern "C" int somb_node_sums_sparse(const int64_t *rowptr, const int32_t *col, const float *val, int64_t n,
                                     int32_t d, const int32_t *bmu, int32_t K, double *S, double *cnt,
                                     int32_t *row_order, void *ws, void *stream) {
    return somb_node_sums_sparse_cols(rowptr, col, val, n, d, bmu, K, d, S, cnt, row_order, ws, stream);
}

extern "C" int somb_node_sums_sparse_cols(const int64_t *rowptr, const int32_t *col, const float *val, int64_t n,
                                          int32_t d, const int32_t *bmu, int32_t K, int32_t dc, double *S,
                                          double *cnt, int32_t *row_order, void *ws, void *stream) {
    SOMB_REQUIRE(K > 0 && d > 0 && n < (1ll << 31), SOMB_E_INPUT, "node_sums_sparse: bad shape");
    SOMB_REQUIRE(dc > 0 && dc <= d, SOMB_E_INPUT, "node_sums_sparse: column block %d outside [1, d=%d]", dc, d);
    cudaStream_t st = as_stream(stream);
    cudaMemsetAsync(S, 0, s_blocks_size(d, dc, K) * sizeof(double), st);
    const int *perm = nullptr, *off = nullptr;
    int rc = node_bucket_sort(bmu, n, K, ws, &perm, &off, cnt, st);
    if (rc) return rc;
    if (n == 0) return SOMB_OK;
    if (row_order) cudaMemcpyAsync(row_order, perm, (size_t)n * sizeof(int), cudaMemcpyDeviceToDevice, st);
    int *nseg, *segoff, *msegoff;
    double *P;
    size_t P_doubles;
    node_seg_plan(ws, n, d, K, SP_SEG, &nseg, &segoff, &msegoff, &P, &P_doubles, st);
    const size_t need = ((size_t)(n + SP_SEG - 1) / SP_SEG * 2 + 2) * (size_t)d;
    cudaMemsetAsync(P, 0, (need < P_doubles ? need : P_doubles) * sizeof(double), st);
    const unsigned maxseg = (unsigned)(K + (n + SP_SEG - 1) / SP_SEG);
    sp_seg_sum_kernel<<<maxseg, 256, 0, st>>>(rowptr, col, val, d, perm, off, segoff, msegoff, nseg, K, dc, S, P);
    note_launch();
    sp_seg_fold<<<dim3((d + 255) / 256 < 64 ? (d + 255) / 256 : 64, K), 256, 0, st>>>(P, msegoff, nseg, d, K, dc, S);
    note_launch();
    SOMB_LAUNCH_CHECK("node_sums_sparse");
    return SOMB_OK;
}

extern "C" size_t somb_bmu_sparse_ws(int64_t n) {
    size_t base = 0;
    bmu_carve(nullptr, n, &base);
    return base + align_up((size_t)n * sizeof(SpRowState), 256) + 2 * align_up((size_t)n * SP_CAP * 4, 256) + 256;
}
