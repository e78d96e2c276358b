// Batch update, part 1: BMU histogram + per-node data sums (fp64).
//
// S_b = sum over rows i with bmu_i = b of x_i, cnt_b = |{i}|.  With the
// neighbourhood convolution (hood.cu) num = H S and den = H cnt, which is the
// reference accumulate (kernels.py:225-226, h^T x per 256-row chunk) regrouped
// by BMU.  Rows are grouped with a stable LSD radix sort of the BMU keys so
// each node's rows are summed in ascending row order (deterministic, equal to
// np.add.at order for nodes with <= 256 rows); larger nodes are summed in
// fixed 256-row segments folded in segment order.  HBM-bound: one read of X.
#include "common.cuh"

namespace somb {

constexpr int kSortTile = 4096;
constexpr int kSortThreads = 256;
constexpr int kSeg = 256;

// ------------------------------------------------ single-block exclusive scan
// out[i] = sum_{k<i} in[i]; out[len] = total (out has len+1 entries).
__global__ void __launch_bounds__(1024) exclusive_scan_kernel(const int *__restrict__ in, int len,
                                                              int *__restrict__ out) {
    __shared__ int warp_tot[32];
    __shared__ int carry_sh;
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    if (t == 0) carry_sh = 0;
    __syncthreads();
    for (int base = 0; base < len; base += 4096) {
        int v[4];
        int s = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            int i = base + t * 4 + q;
            v[q] = i < len ? in[i] : 0;
            s += v[q];
        }
        int incl = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) warp_tot[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            int w = warp_tot[lane];
            int wi = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int y = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= o) wi += y;
            }
            warp_tot[lane] = wi - w;   // exclusive warp offsets
        }
        __syncthreads();
        int run = carry_sh + warp_tot[wid] + incl - s;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            int i = base + t * 4 + q;
            if (i < len) out[i] = run;
            run += v[q];
        }
        __syncthreads();
        if (t == 1023) carry_sh = run;
        __syncthreads();
    }
    if (t == 0) out[len] = carry_sh;
}

// -------------------------------------------------------------- radix sort
__global__ void radix_hist(const int *__restrict__ keys, int64_t n, int shift, int ntiles,
                           int *__restrict__ hist) {
    __shared__ int h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    int64_t base = (int64_t)blockIdx.x * kSortTile;
    for (int q = threadIdx.x; q < kSortTile; q += kSortThreads) {
        int64_t i = base + q;
        if (i < n) atomicAdd(&h[(keys[i] >> shift) & 255], 1);
    }
    __syncthreads();
    hist[threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(kSortThreads)
radix_scatter(const int *__restrict__ kin, const int *__restrict__ vin, int64_t n, int shift,
              int ntiles, const int *__restrict__ goff, int *__restrict__ kout,
              int *__restrict__ vout, int iota_vals) {
    __shared__ int wcnt[kSortThreads / 32][256];
    __shared__ int run[256];
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    run[t] = goff[t * ntiles + blockIdx.x];
    const unsigned lt = (1u << lane) - 1u;
    int64_t base = (int64_t)blockIdx.x * kSortTile;
    for (int q = 0; q < kSortTile / kSortThreads; ++q) {
#pragma unroll
        for (int w = 0; w < kSortThreads / 32; ++w) wcnt[w][t] = 0;
        __syncthreads();
        int64_t i = base + q * kSortThreads + t;
        bool valid = i < n;
        int key = valid ? kin[i] : 0;
        int val = valid ? (iota_vals ? (int)i : vin[i]) : 0;
        int dig = valid ? (key >> shift) & 255 : 256;
        unsigned peers = __match_any_sync(0xffffffffu, dig);
        int lrank = __popc(peers & lt);
        if (valid && lrank == 0) wcnt[wid][dig] = __popc(peers);
        __syncthreads();
        {
            int r = run[t];
#pragma unroll
            for (int w = 0; w < kSortThreads / 32; ++w) {
                int cnum = wcnt[w][t];
                wcnt[w][t] = r;
                r += cnum;
            }
            run[t] = r;
        }
        __syncthreads();
        if (valid) {
            int pos = wcnt[wid][dig] + lrank;
            kout[pos] = key;
            vout[pos] = val;
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------- bucketing
__global__ void bucket_count(const int *__restrict__ bmu, int64_t n, int *__restrict__ cnt) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) atomicAdd(&cnt[bmu[i]], 1);
}

__global__ void seg_plan(const int *__restrict__ cnt, int K, int *__restrict__ nseg,
                         int *__restrict__ mseg, double *__restrict__ cnt_out, int seg = kSeg) {
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= K) return;
    int c = cnt[b];
    int s = (c + seg - 1) / seg;
    nseg[b] = s;
    mseg[b] = s > 1 ? s : 0;
    if (cnt_out) cnt_out[b] = (double)c;
}

// One block per 256-row segment of one node: fixed-order fp64 sum.  S is
// written column-block-major (s_index, common.cuh): [ceil(d/dc)][K][dc].
template <int R>
__global__ void __launch_bounds__(128)
seg_sum(const float *__restrict__ X, int d, const int *__restrict__ perm, const int *__restrict__ off,
        const int *__restrict__ seg_off, const int *__restrict__ mseg_off, const int *__restrict__ nseg,
        int K, int dc, double *__restrict__ S, double *__restrict__ P) {
    const int s = blockIdx.x;
    const int total = seg_off[K];
    if (s >= total) return;
    // b = upper_bound(seg_off[0..K], s) - 1
    int lo = 0, hi = K;
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (seg_off[mid] <= s) lo = mid; else hi = mid - 1;
    }
    int b = lo;
    while (b + 1 <= K && seg_off[b + 1] <= s) ++b;   // skip empty buckets sharing the offset
    const int sub = s - seg_off[b];
    const int r0 = off[b] + sub * kSeg;
    const int r1 = min(off[b + 1], r0 + kSeg);
    double *prow = nseg[b] > 1 ? P + (int64_t)(mseg_off[b] + sub) * d : nullptr;
    for (int k0 = 0; k0 < d; k0 += 128 * R) {
        double acc[R];
#pragma unroll
        for (int q = 0; q < R; ++q) acc[q] = 0.0;
        // rows in fixed ascending order; four rows' loads in flight at a time
        int r = r0;
        for (; r + 4 <= r1; r += 4) {
            const float *x0 = X + (int64_t)perm[r] * d, *x1 = X + (int64_t)perm[r + 1] * d;
            const float *x2 = X + (int64_t)perm[r + 2] * d, *x3 = X + (int64_t)perm[r + 3] * d;
#pragma unroll
            for (int q = 0; q < R; ++q) {
                int k = k0 + q * 128 + threadIdx.x;
                if (k < d) {
                    const float a = __ldg(x0 + k), b = __ldg(x1 + k), cc = __ldg(x2 + k), e = __ldg(x3 + k);
                    acc[q] += (double)a;
                    acc[q] += (double)b;
                    acc[q] += (double)cc;
                    acc[q] += (double)e;
                }
            }
        }
        for (; r < r1; ++r) {
            const float *x = X + (int64_t)perm[r] * d;
#pragma unroll
            for (int q = 0; q < R; ++q) {
                int k = k0 + q * 128 + threadIdx.x;
                if (k < d) acc[q] += (double)x[k];
            }
        }
#pragma unroll
        for (int q = 0; q < R; ++q) {
            int k = k0 + q * 128 + threadIdx.x;
            if (k < d) {
                if (prow) prow[k] = acc[q];
                else S[s_index(b, k, dc, K)] = acc[q];
            }
        }
    }
}

__global__ void seg_fold(const double *__restrict__ P, const int *__restrict__ mseg_off,
                         const int *__restrict__ nseg, int d, int K, int dc, double *__restrict__ S) {
    const int b = blockIdx.x;
    const int ns = nseg[b];
    if (ns <= 1) return;
    const double *p = P + (int64_t)mseg_off[b] * d;
    for (int k = threadIdx.x; k < d; k += blockDim.x) {
        double a = 0.0;
        for (int s = 0; s < ns; ++s) a += p[(int64_t)s * d + k];
        S[s_index(b, k, dc, K)] = a;
    }
}

struct NodeSumWs {
    int *kA, *kB, *vA, *vB, *hist, *hsc, *cnt, *off, *nseg, *segoff, *mseg, *msegoff;
    double *P;
};

static NodeSumWs carve(void *ws, int64_t n, int d, int K) {
    NodeSumWs w;
    char *p = (char *)ws;
    auto take = [&](size_t bytes) { char *r = p; p += align_up(bytes, 256); return r; };
    int ntiles = (int)((n + kSortTile - 1) / kSortTile);
    w.kA = (int *)take(n * 4); w.kB = (int *)take(n * 4);
    w.vA = (int *)take(n * 4); w.vB = (int *)take(n * 4);
    w.hist = (int *)take((size_t)256 * ntiles * 4 + 4);
    w.hsc = (int *)take((size_t)256 * ntiles * 4 + 4);
    w.cnt = (int *)take((size_t)(K + 1) * 4);
    w.off = (int *)take((size_t)(K + 1) * 4);
    w.nseg = (int *)take((size_t)(K + 1) * 4);
    w.segoff = (int *)take((size_t)(K + 1) * 4);
    w.mseg = (int *)take((size_t)(K + 1) * 4);
    w.msegoff = (int *)take((size_t)(K + 1) * 4);
    w.P = (double *)take(((size_t)2 * ((n + kSeg - 1) / kSeg) + 2) * d * sizeof(double));
    return w;
}

}  // namespace somb

using namespace somb;

extern "C" size_t somb_node_sums_ws(int64_t n, int32_t d, int32_t K) {
    int ntiles = (int)((n + kSortTile - 1) / kSortTile);
    size_t b = 4 * align_up(n * 4, 256) + 2 * align_up((size_t)256 * ntiles * 4 + 4, 256) +
               6 * align_up((size_t)(K + 1) * 4, 256) +
               align_up(((size_t)2 * ((n + kSeg - 1) / kSeg) + 2) * d * sizeof(double), 256);
    return b + 256;
}

namespace somb {
// Stable grouping of rows by BMU: perm = rows sorted by (bmu, row), off =
// bucket offsets (K + 1), cnt = bucket sizes as fp64.  Shared by the dense and
// sparse node sums.  ws is carved like somb_node_sums_ws.
int node_bucket_sort(const int *bmu, int64_t n, int K, void *ws, const int **perm_out, const int **off_out,
                     double *cnt, cudaStream_t st) {
    NodeSumWs w = carve(ws, n, 1, K);
    cudaMemsetAsync(w.cnt, 0, (size_t)(K + 1) * sizeof(int), st);
    *off_out = w.off;
    if (n == 0) {
        cudaMemsetAsync(cnt, 0, (size_t)K * sizeof(double), st);
        cudaMemsetAsync(w.off, 0, (size_t)(K + 1) * sizeof(int), st);
        *perm_out = w.vA;
        SOMB_LAUNCH_CHECK("node_bucket_sort(empty)");
        return SOMB_OK;
    }
    int bits = 0;
    while ((1 << bits) < K) ++bits;
    int passes = (bits + 7) / 8;
    int ntiles = (int)((n + kSortTile - 1) / kSortTile);
    const int *kin = bmu;
    const int *vin = nullptr;
    int *kout = w.kA, *vout = w.vA;
    if (passes == 0) passes = 1;   // K == 1: one identity pass (all digits 0)
    for (int p = 0; p < passes; ++p) {
        radix_hist<<<ntiles, kSortThreads, 0, st>>>(kin, n, 8 * p, ntiles, w.hist);
        note_launch();
        exclusive_scan_kernel<<<1, 1024, 0, st>>>(w.hist, 256 * ntiles, w.hsc);
        note_launch();
        radix_scatter<<<ntiles, kSortThreads, 0, st>>>(kin, vin, n, 8 * p, ntiles, w.hsc, kout, vout, p == 0);
        note_launch();
        kin = kout;
        vin = vout;
        kout = (kout == w.kA) ? w.kB : w.kA;
        vout = (vout == w.vA) ? w.vB : w.vA;
    }
    *perm_out = vin;
    bucket_count<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(bmu, n, w.cnt);
    note_launch();
    exclusive_scan_kernel<<<1, 1024, 0, st>>>(w.cnt, K, w.off);
    note_launch();
    seg_plan<<<(K + 255) / 256, 256, 0, st>>>(w.cnt, K, w.nseg, w.mseg, cnt);
    note_launch();
    SOMB_LAUNCH_CHECK("node_bucket_sort");
    return SOMB_OK;
}
}  // namespace somb

extern "C" int somb_node_sums_dense(const float *X, int64_t n, int32_t d, const int32_t *bmu, int32_t K,
                                    double *S, double *cnt, int32_t *row_order, void *ws, void *stream) {
    return somb_node_sums_dense_cols(X, n, d, bmu, K, d, S, cnt, row_order, ws, stream);
}

extern "C" int somb_node_sums_dense_cols(const float *X, int64_t n, int32_t d, const int32_t *bmu, int32_t K,
                                         int32_t dc, double *S, double *cnt, int32_t *row_order, void *ws,
                                         void *stream) {
    SOMB_REQUIRE(K > 0 && d > 0 && n >= 0 && n < (1ll << 31), SOMB_E_INPUT,
                 "node_sums: bad shape n=%lld d=%d K=%d", (long long)n, d, K);
    SOMB_REQUIRE(dc > 0 && dc <= d, SOMB_E_INPUT, "node_sums: column block %d outside [1, d=%d]", dc, d);
    cudaStream_t st = as_stream(stream);
    NodeSumWs w = carve(ws, n, d, K);
    cudaMemsetAsync(S, 0, s_blocks_size(d, dc, K) * sizeof(double), st);
    const int *perm = nullptr, *off = nullptr;
    int rc = node_bucket_sort(bmu, n, K, ws, &perm, &off, cnt, st);
    if (rc || n == 0) return rc;
    if (row_order) cudaMemcpyAsync(row_order, perm, (size_t)n * sizeof(int), cudaMemcpyDeviceToDevice, st);
    exclusive_scan_kernel<<<1, 1024, 0, st>>>(w.nseg, K, w.segoff);
    note_launch();
    exclusive_scan_kernel<<<1, 1024, 0, st>>>(w.mseg, K, w.msegoff);
    note_launch();
    unsigned maxseg = (unsigned)(K + (n + kSeg - 1) / kSeg);
    if (d <= 128)
        seg_sum<1><<<maxseg, 128, 0, st>>>(X, d, perm, off, w.segoff, w.msegoff, w.nseg, K, dc, S, w.P);
    else if (d <= 512)
        seg_sum<4><<<maxseg, 128, 0, st>>>(X, d, perm, off, w.segoff, w.msegoff, w.nseg, K, dc, S, w.P);
    else
        seg_sum<8><<<maxseg, 128, 0, st>>>(X, d, perm, off, w.segoff, w.msegoff, w.nseg, K, dc, S, w.P);
    note_launch();
    seg_fold<<<K, 128, 0, st>>>(w.P, w.msegoff, w.nseg, d, K, dc, S);
    note_launch();
    SOMB_LAUNCH_CHECK("node_sums");
    return SOMB_OK;
}

namespace somb {
// Segment plan of the sorted rows for per-node sums in fixed-size row
// segments (the sparse path; the dense path plans inside
// somb_node_sums_dense): nseg/segoff per node, msegoff = partial-slot
// offsets of multi-segment nodes.  ws is carved like somb_node_sums_ws.
void node_seg_plan(void *ws, int64_t n, int d, int K, int seg, int **nseg, int **segoff, int **msegoff,
                   double **P, size_t *P_doubles, cudaStream_t st) {
    NodeSumWs w = carve(ws, n, d, K);
    seg_plan<<<(K + 255) / 256, 256, 0, st>>>(w.cnt, K, w.nseg, w.mseg, nullptr, seg);
    note_launch();
    exclusive_scan_kernel<<<1, 1024, 0, st>>>(w.nseg, K, w.segoff);
    note_launch();
    exclusive_scan_kernel<<<1, 1024, 0, st>>>(w.mseg, K, w.msegoff);
    note_launch();
    *nseg = w.nseg;
    *segoff = w.segoff;
    *msegoff = w.msegoff;
    *P = w.P;
    *P_doubles = ((size_t)2 * ((n + kSeg - 1) / kSeg) + 2) * d;
}

int exclusive_scan(const int *in, int len, int *out, cudaStream_t st) {
    exclusive_scan_kernel<<<1, 1024, 0, st>>>(in, len, out);
    note_launch();
    SOMB_LAUNCH_CHECK("exclusive_scan");
    return SOMB_OK;
}
}  // namespace somb
