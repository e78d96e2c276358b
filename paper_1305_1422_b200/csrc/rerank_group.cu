// Grouped exact fp64 re-rank.
//
// The per-row re-rank (bmu.cu rerank_pipe_kernel) reads one 4d-byte codebook
// row from L2 per candidate: ~30 candidates per row at cfg2 is ~120 GB of L2
// reads per epoch, and it ran at ~5 TB/s of scattered L2 traffic.  Rows are
// visited in previous-BMU order (the node-sum sort), so consecutive rows have
// nearly the same candidate nodes.  Here a CTA takes GR_ROWS consecutive rows,
// builds the UNION of their candidate nodes in shared memory (a small hash
// table), and streams the union's codebook rows and the group's data rows
// through shared memory in GR_F-feature chunks (cp.async, double-buffered):
// each codebook row is read from L2 once per group instead of once per
// (row, candidate) pair.  A warp owns GR_RPW rows; lane l evaluates candidates
// l, l + 32, ... of a row, each as a fixed-order fp64 dot (two accumulators:
// even / odd float4 slices), so the result is deterministic; the row's winner
// is the lowest (value, index) pair -- the reference's first minimum
// (kernels.py:27-28) of its blocked formula ((-2 x.w) + |x|^2) + |w|^2,
// clamped >= 0 (kernels.py:196-202), or the naive sum of squares
// (kernels.py:182-192, the final pass of train.py:287-291).
//
// Rows whose candidates do not fit (more than GR_C, or a union larger than
// GR_U) and repaired rows (exact scan of every node) are appended to a
// device-side row list that the per-row kernels re-rank afterwards (one slow
// row must not hold 15 warps at the group barrier).
#include "rerank.cuh"

namespace somb {

constexpr int GR_ROWS = 16;                   // rows per group (consecutive in the visiting order)
constexpr int GR_WARPS = 16;
constexpr int GR_THREADS = 32 * GR_WARPS;
constexpr int GR_RPW = GR_ROWS / GR_WARPS;    // rows per warp
constexpr int GR_F = 32;                      // features per chunk
constexpr int GR_FP = GR_F + 4;               // slice pitch in floats (144 B: float4 rows of a quarter-warp hit distinct banks)
constexpr int GR_NBUF = 4;                    // chunks in flight (cp.async ring): each chunk waits ~one L2 round trip
constexpr int GR_U = 256;                     // union capacity (cfg2: union of 16 rows 100-210 mean, p99 <= 324)
constexpr int GR_C = 128;                     // candidates per row evaluated from shared memory
constexpr int GR_P = GR_C / 32;               // lane passes per row
constexpr int GR_HASH = 1024;

struct GrSmem {
    float wb[GR_NBUF][GR_U][GR_FP];           // union codebook slices (ring)
    float xf[GR_NBUF][GR_ROWS][GR_F];         // data-row slices as loaded
    double xd[GR_WARPS][GR_RPW][GR_F];        // ... converted by the row's warp (odd float4 slices pre-scaled, blocked)
    int hkey[GR_HASH];
    int hval[GR_HASH];
    int uid[GR_U];                            // union slot -> node
    unsigned short cs[GR_ROWS][GR_C];         // row's candidates as union slots
    int rcnt[GR_ROWS];                        // candidates of the row, -1 = per-row kernel, 0 = no row
    long long rid[GR_ROWS];
    int nu;
};

// union slot of node j (inserting it); >= GR_U when the union is full
__device__ __forceinline__ int gr_insert(GrSmem &S, int j) {
    unsigned h = ((unsigned)j * 2654435761u) >> 22;   // 10 bits
    for (int probe = 0; probe < GR_HASH; ++probe) {
        const int old = atomicCAS(&S.hkey[h], -1, j);
        if (old == -1) {
            const int s = atomicAdd(&S.nu, 1);
            if (s < GR_U) S.uid[s] = j;
            atomicExch(&S.hval[h], s);
            return s;
        }
        if (old == j) {
            int s;
            while ((s = atomicAdd(&S.hval[h], 0)) < 0) {
            }
            return s;
        }
        h = (h + 1) & (GR_HASH - 1);
    }
    return GR_U;
}

// Warp-collective: the candidate nodes of `row` (screened list + in-window
// spilled entries) into the union; returns their count, or -1 when the row
// must take the global-memory path.
__device__ int gr_collect(GrSmem &S, int r, int64_t row, int K, const int *__restrict__ cand,
                          const int *__restrict__ ccount, int split, const OvfView &ov, int lane) {
    const int cc = ccount[row];
    const CandLayout L = cand_layout(cc, split, split && ov.ngp ? (int)*ov.ngp : 2);
    const int cnt = L.cnt;
    if (cnt < 0) return -1;   // repaired row: exact scan of every node
    int T = 0;
    bool bad = false;
    auto append = [&](bool valid, int j) {
        const int s = valid ? gr_insert(S, j) : 0;
        const unsigned bal = __ballot_sync(0xffffffffu, valid);
        const int pos = T + __popc(bal & ((1u << lane) - 1u));
        if (valid) {
            if (pos < GR_C && s < GR_U) S.cs[r][pos] = (unsigned short)s;
            else bad = true;
        }
        T += __popc(bal);
    };
    for (int q0 = 0; q0 < cnt; q0 += 32) {
        const int q = q0 + lane;
        const int j = q < cnt ? cand[row * SOMB_CAND_CAP + cand_slot(L, q)] : -1;
        append(q < cnt && (unsigned)j < (unsigned)K, j);
    }
    if (ov.head != nullptr) {
        for (int h = 0; h < 4; ++h) {
            const float lim = ov.lim[4 * row + h];
            for (int c = ov.head[4 * row + h]; c >= 0; c = ov.next[c]) {
                const int m = ov.cnt[c];
                const int2 e = lane < m ? ov.ent[(size_t)c * kOvfChunk + lane] : make_int2(0x7f800000, -1);
                append(lane < m && __int_as_float(e.x) <= lim && (unsigned)e.y < (unsigned)K, e.y);
            }
        }
    }
    bad = __any_sync(0xffffffffu, bad);
    return bad || T == 0 ? -1 : T;   // (no candidate at all: the global path scans every node)
}

template <int MODE>
__device__ __forceinline__ double gr_value(double dot, double xx, const double *__restrict__ w2, int j) {
    if (MODE == SOMB_DIST_NAIVE) return dot;
    return fmax(__dadd_rn(__dadd_rn(__dmul_rn(-2.0, dot), xx), w2[j]), 0.0);
}

// lowest (value, index) over the warp; every lane gets the winner
__device__ __forceinline__ void gr_warp_min(double &v, int &j) {
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) {
        const double ov2 = __shfl_xor_sync(0xffffffffu, v, m);
        const int oj = __shfl_xor_sync(0xffffffffu, j, m);
        if (ov2 < v || (ov2 == v && oj < j)) { v = ov2; j = oj; }
    }
}

template <int MODE>
__global__ void __launch_bounds__(GR_THREADS, 1)
rerank_group_kernel(const float *__restrict__ X, const double *__restrict__ x2, int64_t n, int d,
                    const float *__restrict__ W, const double *__restrict__ w2, int K,
                    const int *__restrict__ cand, const int *__restrict__ ccount, int split,
                    const int *__restrict__ order, OvfView ov, int *__restrict__ bmu, double *__restrict__ d2min,
                    int *__restrict__ left, unsigned *__restrict__ nleft) {
    extern __shared__ __align__(16) uint8_t gr_raw[];
    GrSmem &S = *reinterpret_cast<GrSmem *>(gr_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t ngroups = (n + GR_ROWS - 1) / GR_ROWS;
    const int nchunks = (d + GR_F - 1) / GR_F;
#pragma unroll 1
    for (int64_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
        // ---------------------------------------------------------- union
        for (int i = tid; i < GR_HASH; i += GR_THREADS) {
            S.hkey[i] = -1;
            S.hval[i] = -1;
        }
        if (tid == 0) S.nu = 0;
        __syncthreads();
#pragma unroll
        for (int q = 0; q < GR_RPW; ++q) {
            const int r = warp * GR_RPW + q;
            const int64_t wi = g * GR_ROWS + r;
            const int64_t row = wi < n ? (order ? (int64_t)order[wi] : wi) : -1;
            const int T = row >= 0 ? gr_collect(S, r, row, K, cand, ccount, split, ov, lane) : 0;
            if (lane == 0) {
                S.rcnt[r] = T;
                S.rid[r] = row;
            }
        }
        __syncthreads();
        const int nu = S.nu < GR_U ? S.nu : GR_U;
        // ------------------------------------------------ chunked fp64 dots
        auto issue = [&](int c) {
            if (c < nchunks) {
                const int buf = c % GR_NBUF;
                const int k0 = c * GR_F;
                const int q4 = (d - k0 < GR_F ? d - k0 : GR_F) >> 2;
                for (int e = tid; e < nu * q4; e += GR_THREADS) {
                    const int s = e / q4, q = e - s * q4;
                    cp_async16(smem_addr(&S.wb[buf][s][4 * q]), W + (int64_t)S.uid[s] * d + k0 + 4 * q);
                }
                for (int e = tid; e < GR_ROWS * q4; e += GR_THREADS) {
                    const int r = e / q4, q = e - r * q4;
                    if (S.rcnt[r] > 0) cp_async16(smem_addr(&S.xf[buf][r][4 * q]), X + S.rid[r] * d + k0 + 4 * q);
                }
            }
            cp_async_commit();   // (empty groups keep the wait_group count uniform)
        };
        double acc[GR_RPW][GR_P][2];
#pragma unroll
        for (int q = 0; q < GR_RPW; ++q)
#pragma unroll
            for (int p = 0; p < GR_P; ++p) acc[q][p][0] = acc[q][p][1] = 0.0;
#pragma unroll
        for (int c = 0; c < GR_NBUF - 1; ++c) issue(c);
#pragma unroll 1
        for (int c = 0; c < nchunks; ++c) {
            const int buf = c % GR_NBUF;
            cp_async_wait<GR_NBUF - 2>();
            __syncthreads();   // chunk c landed everywhere; chunk c - 1 fully consumed (its slot is refilled next)
            issue(c + GR_NBUF - 1);
            const int kl = d - c * GR_F < GR_F ? d - c * GR_F : GR_F;
            const int kq = kl >> 2;
#pragma unroll
            for (int q = 0; q < GR_RPW; ++q) {
                const int r = warp * GR_RPW + q;
                const int T = S.rcnt[r];
                if (T <= 0) continue;   // warp-uniform
                // the row's slice to fp64, one feature per lane (this warp's own buffer)
                if (lane < kl) {
                    const double sc = (MODE != SOMB_DIST_NAIVE && ((lane >> 2) & 1)) ? kF64Scale : 1.0;
                    S.xd[warp][q][lane] = (double)S.xf[buf][r][lane] * sc;
                }
                __syncwarp();
#pragma unroll
                for (int p = 0; p < GR_P; ++p) {
                    if (p * 32 >= T) break;   // warp-uniform
                    const int idx = p * 32 + lane;
                    if (idx < T) {
                        const float4 *wp = reinterpret_cast<const float4 *>(S.wb[buf][S.cs[r][idx]]);
                        const double2 *xp = reinterpret_cast<const double2 *>(S.xd[warp][q]);
                        double a0 = acc[q][p][0], a1 = acc[q][p][1];
                        // even float4 slices: F2F conversions (XU pipe); odd: exact
                        // integer re-exponenting against pre-scaled x (ALU pipe)
                        auto step_f2f = [&](int k4, double &a) {
                            const float4 w = wp[k4];
                            const double2 xa = xp[2 * k4], xb = xp[2 * k4 + 1];
                            if (MODE == SOMB_DIST_NAIVE) {
                                double t;
                                t = (double)w.x - xa.x; a = __fma_rn(t, t, a);
                                t = (double)w.y - xa.y; a = __fma_rn(t, t, a);
                                t = (double)w.z - xb.x; a = __fma_rn(t, t, a);
                                t = (double)w.w - xb.y; a = __fma_rn(t, t, a);
                            } else {
                                a = __fma_rn(xa.x, (double)w.x, a);
                                a = __fma_rn(xa.y, (double)w.y, a);
                                a = __fma_rn(xb.x, (double)w.z, a);
                                a = __fma_rn(xb.y, (double)w.w, a);
                            }
                        };
                        auto step_int = [&](int k4, double &a) {
                            const float4 w = wp[k4];
                            const double2 xa = xp[2 * k4], xb = xp[2 * k4 + 1];
                            const double b0 = f32_as_f64_scaled(w.x), b1 = f32_as_f64_scaled(w.y);
                            const double b2 = f32_as_f64_scaled(w.z), b3 = f32_as_f64_scaled(w.w);
                            if (MODE == SOMB_DIST_NAIVE) {
                                double t;
                                t = __fma_rn(b0, kF64Scale, -xa.x); a = __fma_rn(t, t, a);
                                t = __fma_rn(b1, kF64Scale, -xa.y); a = __fma_rn(t, t, a);
                                t = __fma_rn(b2, kF64Scale, -xb.x); a = __fma_rn(t, t, a);
                                t = __fma_rn(b3, kF64Scale, -xb.y); a = __fma_rn(t, t, a);
                            } else {
                                a = __fma_rn(xa.x, b0, a);
                                a = __fma_rn(xa.y, b1, a);
                                a = __fma_rn(xb.x, b2, a);
                                a = __fma_rn(xb.y, b3, a);
                            }
                        };
                        int k4 = 0;
#pragma unroll 2
                        for (; k4 + 1 < kq; k4 += 2) {
                            step_f2f(k4, a0);
                            step_int(k4 + 1, a1);
                        }
                        if (k4 < kq) step_f2f(k4, a0);
                        acc[q][p][0] = a0;
                        acc[q][p][1] = a1;
                    }
                }
                __syncwarp();   // the next row / chunk overwrites this warp's xd
            }
        }
        cp_async_wait<0>();
        // ------------------------------------------------------ winners
#pragma unroll
        for (int q = 0; q < GR_RPW; ++q) {
            const int r = warp * GR_RPW + q;
            const int T = S.rcnt[r];
            const int64_t row = S.rid[r];
            if (T > 0) {
                const double xx = x2[row];
                double best = INFINITY;
                int bestj = 0x7fffffff;
#pragma unroll
                for (int p = 0; p < GR_P; ++p) {
                    const int idx = p * 32 + lane;
                    if (idx < T) {
                        const int j = S.uid[S.cs[r][idx]];
                        const double v = gr_value<MODE>(__dadd_rn(acc[q][p][0], acc[q][p][1]), xx, w2, j);
                        if (v < best || (v == best && j < bestj)) { best = v; bestj = j; }
                    }
                }
                gr_warp_min(best, bestj);
                if (lane == 0) {
                    bmu[row] = bestj;
                    d2min[row] = best;
                }
            } else if (T < 0 && lane == 0) {
                left[atomicAdd(nleft, 1u)] = (int)row;   // the per-row kernel takes it (bmu.cu)
            }
        }
        __syncthreads();   // the next group rebuilds the shared tables
    }
}

size_t rerank_group_smem() { return sizeof(GrSmem); }

int launch_rerank_group(cudaStream_t st, const float *X, const double *x2, int64_t n, int d, const float *W,
                        const double *w2, int K, const int *cand, const int *ccount, int mode, int split,
                        const int *order, OvfView ov, int *bmu, double *d2min, int *left, unsigned *nleft) {
    SOMB_REQUIRE(d % 4 == 0, SOMB_E_INPUT, "rerank_group: d %% 4 required (d=%d)", d);
    static bool init = false;
    const int smem = (int)sizeof(GrSmem);
    if (!init) {
        cudaError_t r1 = cudaFuncSetAttribute(rerank_group_kernel<SOMB_DIST_NAIVE>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaError_t r2 = cudaFuncSetAttribute(rerank_group_kernel<SOMB_DIST_BLOCKED>,
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (r1 != cudaSuccess) return cuda_status(r1, "rerank_group smem");
        if (r2 != cudaSuccess) return cuda_status(r2, "rerank_group smem");
        init = true;
    }
    int dev = 0, sms = kSmCount;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t groups = (n + GR_ROWS - 1) / GR_ROWS;
    const unsigned blocks = (unsigned)(groups < sms ? groups : sms);
    if (mode == SOMB_DIST_NAIVE)
        rerank_group_kernel<SOMB_DIST_NAIVE><<<blocks, GR_THREADS, smem, st>>>(X, x2, n, d, W, w2, K, cand, ccount,
                                                                             split, order, ov, bmu, d2min, left, nleft);
    else
        rerank_group_kernel<SOMB_DIST_BLOCKED><<<blocks, GR_THREADS, smem, st>>>(X, x2, n, d, W, w2, K, cand, ccount,
                                                                               split, order, ov, bmu, d2min, left,
                                                                               nleft);
    note_launch();
    SOMB_LAUNCH_CHECK("rerank_group");
    return SOMB_OK;
}

}  // namespace somb
