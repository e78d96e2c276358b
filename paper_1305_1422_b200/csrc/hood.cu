// Batch update, part 2: neighbourhood convolution over the grid + blend.
//
// h(b, j) depends only on the (wrapped) grid offset between nodes b and j,
// so one small per-epoch table htab[dy][dx] (rect: nx x ny; hex: 2nx x ny in
// half-column units) holds every influence value, computed exactly like the
// reference: d = hypot(dx, dy) (kernels.py:112/127; the host may pass numpy's
// own hypot table for bit parity), h = exp(d / -radius) (kernels.py:128-129),
// h < cutoff -> 0 (kernels.py:146-147).  Extensions: bubble (h = [d <= r]),
// compact support (h = 0 for d > r), hexagonal offset-row lattice.
//
//   den_j = sum_b h(b, j) cnt_b            (fp64, ascending b)
//   num_j = sum_b h(b, j) S_b              (fp64 DFMA tiles)
//   W_j  <- f32((1 - a) W_j + a num_j / den_j)  if den_j > 0   (kernels.py:438-450)
// Only nodes with cnt_b > 0 contribute (S_b = 0 otherwise), so b runs over
// the compacted list of occupied nodes.
#include "common.cuh"

namespace somb {

__global__ void hood_table_kernel(MapDev m, int tw, const double *__restrict__ dist, int nbh,
                                  int compact, double radius, double cutoff,
                                  double *__restrict__ htab) {
    int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= tw * m.ny) return;
    int dxu = e % tw, dy = e / tw;
    double d;
    if (dist) {
        d = dist[e];
    } else if (!m.hex) {
        d = sqrt((double)dxu * dxu + (double)dy * dy);
    } else {
        d = sqrt(0.25 * (double)dxu * dxu + 0.75 * (double)dy * dy);
    }
    double h;
    if (nbh == SOMB_NBH_BUBBLE) {
        h = d <= radius ? 1.0 : 0.0;
    } else {
        h = exp(d / -radius);
        if (compact && d > radius) h = 0.0;
    }
    if (cutoff > 0.0 && h < cutoff) h = 0.0;
    htab[e] = h;
}

// wrapped offset index into htab for nodes a, b
__device__ __forceinline__ int hood_index(const MapDev &m, int tw, int ca, int ra, int cb, int rb) {
    int dy = abs(ra - rb);
    if (m.toroid) dy = min(dy, m.ny - dy);
    int dx;
    if (!m.hex) {
        dx = abs(ca - cb);
        if (m.toroid) dx = min(dx, m.nx - dx);
    } else {
        dx = abs((2 * ca + (ra & 1)) - (2 * cb + (rb & 1)));
        if (m.toroid) dx = min(dx, 2 * m.nx - dx);
    }
    return dy * tw + dx;
}

// occupied-node compaction (ascending b): occ[0..nocc)
__global__ void occ_flags(const double *__restrict__ cnt, int K, int *__restrict__ flag) {
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < K) flag[b] = cnt[b] > 0.0 ? 1 : 0;
}
__global__ void occ_scatter(const int *__restrict__ flag, const int *__restrict__ pos, int K,
                            int *__restrict__ occ) {
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < K && flag[b]) occ[pos[b]] = b;
}

__global__ void __launch_bounds__(256)
hood_den_kernel(MapDev m, int tw, const double *__restrict__ htab, const double *__restrict__ cnt,
                const int *__restrict__ occ, const int *__restrict__ nocc_p, int j0, int j1,
                double *__restrict__ den) {
    __shared__ int sb[256];
    __shared__ double sc[256];
    const int j = j0 + blockIdx.x * 256 + threadIdx.x;
    const int nocc = *nocc_p;
    const int cj = j % m.nx, rj = j / m.nx;
    double acc = 0.0;
    for (int t0 = 0; t0 < nocc; t0 += 256) {
        __syncthreads();
        int q = t0 + threadIdx.x;
        if (q < nocc) {
            int b = occ[q];
            sb[threadIdx.x] = b;
            sc[threadIdx.x] = cnt[b];
        }
        __syncthreads();
        int lim = min(256, nocc - t0);
        if (j < j1) {
            for (int u = 0; u < lim; ++u) {
                int b = sb[u];
                double h = htab[hood_index(m, tw, cj, rj, b % m.nx, b / m.nx)];
                acc = __fma_rn(h, sc[u], acc);
            }
        }
    }
    if (j < j1) den[j] = acc;
}

// num tile = H[j-tile, occ] * S[occ, k-tile]; fused blend epilogue.
constexpr int kHM = 64, kHN = 64, kHK = 16;

__global__ void __launch_bounds__(256)
hood_conv_blend(MapDev m, int tw, const double *__restrict__ htab, const double *__restrict__ S, int d,
                const int *__restrict__ occ, const int *__restrict__ nocc_p, int j0, int j1,
                const double *__restrict__ den, double alpha, double one_minus_alpha,
                const float *__restrict__ Wold, float *__restrict__ Wnew, double *__restrict__ num_out) {
    __shared__ double sh_h[kHK][kHM + 1];
    __shared__ double sh_s[kHK][kHN];
    __shared__ int sh_b[kHK];
    const int t = threadIdx.x, tx = t % 16, ty = t / 16;
    const int jb = j0 + blockIdx.y * kHM;
    const int kb = blockIdx.x * kHN;
    const int nocc = *nocc_p;
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    // this thread's H-tile loader slots: 4 of the 64x16 entries
    for (int t0 = 0; t0 < nocc; t0 += kHK) {
        __syncthreads();
        if (t < kHK) sh_b[t] = (t0 + t < nocc) ? occ[t0 + t] : -1;
        __syncthreads();
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            int e = t + 256 * q;             // 0..1023
            int kk = e / kHM, jj = e % kHM;  // H[kk][jj]
            int b = sh_b[kk];
            int j = jb + jj;
            double h = 0.0;
            if (b >= 0 && j < j1)
                h = htab[hood_index(m, tw, j % m.nx, j / m.nx, b % m.nx, b / m.nx)];
            sh_h[kk][jj] = h;
            int kk2 = e / kHN, dd = e % kHN;  // S[kk2][dd]
            int b2 = sh_b[kk2];
            int k = kb + dd;
            sh_s[kk2][dd] = (b2 >= 0 && k < d) ? S[(int64_t)b2 * d + k] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < kHK; ++kk) {
            double hv[4], sv[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) hv[a] = sh_h[kk][ty + 16 * a];
#pragma unroll
            for (int b = 0; b < 4; ++b) sv[b] = sh_s[kk][tx + 16 * b];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b] = __fma_rn(hv[a], sv[b], acc[a][b]);
        }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        int j = jb + ty + 16 * a;
        if (j >= j1) continue;
        double dj = den[j];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            int k = kb + tx + 16 * b;
            if (k >= d) continue;
            int64_t o = (int64_t)j * d + k;
            double num = acc[a][b];
            if (num_out) num_out[o] = num;
            float w = Wold[o];
            if (dj > 0.0) {
                double upd = __ddiv_rn(num, dj);
                double v = __dadd_rn(__dmul_rn(one_minus_alpha, (double)w), __dmul_rn(alpha, upd));
                w = __double2float_rn(v);
            }
            Wnew[o] = w;
        }
    }
}

int exclusive_scan(const int *in, int len, int *out, cudaStream_t st);
size_t spec_ws_bytes(const somb_map *m, int d);
int spec_update(const somb_map *m, const double *htab, const double *S, const double *cnt, int d, double *den,
                int den_mode, double tau, double scale, const float *Wold, int j0, int j1, float *Wnew,
                double *num_out, void *ws, cudaStream_t st);

}  // namespace somb

using namespace somb;

static int table_width(const somb_map *m) { return m->grid == SOMB_GRID_HEX ? 2 * m->n_columns : m->n_columns; }

static size_t direct_ws(const somb_map *map, int32_t K) {
    return 3 * align_up((size_t)(K + 1) * sizeof(int), 256) + align_up((size_t)K * sizeof(double), 256) +
           align_up((size_t)table_width(map) * map->n_rows * sizeof(double), 256) + 256;
}

extern "C" size_t somb_hood_ws(const somb_map *map, int32_t K, int32_t d) {
    return direct_ws(map, K) + spec_ws_bytes(map, d);
}

static bool use_spectral(const somb_map *m, const somb_hood *h) {
    if (h->method == SOMB_CONV_DIRECT) return false;
    if (h->method == SOMB_CONV_SPECTRAL) return true;
    return (int64_t)m->n_columns * m->n_rows >= 2048;
}

static int check_map(const somb_map *m) {
    SOMB_REQUIRE(m && m->n_columns >= 1 && m->n_rows >= 1, SOMB_E_CONFIG, "map dimensions must be >= 1");
    SOMB_REQUIRE(m->grid == SOMB_GRID_RECT || m->grid == SOMB_GRID_HEX, SOMB_E_CONFIG, "bad grid %d", m->grid);
    SOMB_REQUIRE(m->topology == SOMB_PLANAR || m->topology == SOMB_TOROID, SOMB_E_CONFIG, "bad topology");
    SOMB_REQUIRE(!(m->grid == SOMB_GRID_HEX && m->topology == SOMB_TOROID && (m->n_rows & 1)),
                 SOMB_E_CONFIG, "hexagonal toroid needs an even number of rows, got %d", m->n_rows);
    return SOMB_OK;
}

extern "C" int somb_hood_update(const double *S, const double *cnt, int32_t d, const somb_map *map,
                                const somb_hood *hood, double scale, const double *dist_table,
                                const float *W_old, int32_t node_begin, int32_t node_end, float *W_new,
                                double *num_out, double *den_out, void *ws, void *stream) {
    int rc = check_map(map);
    if (rc) return rc;
    SOMB_REQUIRE(hood && hood->radius > 0.0 && hood->cutoff >= 0.0, SOMB_E_CONFIG,
                 "hood: radius must be > 0 and cutoff >= 0");
    const int K = map->n_columns * map->n_rows;
    SOMB_REQUIRE(d > 0 && 0 <= node_begin && node_begin <= node_end && node_end <= K, SOMB_E_INPUT,
                 "hood: bad node range [%d, %d) for K=%d", node_begin, node_end, K);
    cudaStream_t st = as_stream(stream);
    MapDev m{map->n_columns, map->n_rows, map->grid == SOMB_GRID_HEX, map->topology == SOMB_TOROID};
    const int tw = table_width(map);
    char *p = (char *)ws;
    auto take = [&](size_t bytes) { char *r = p; p += align_up(bytes, 256); return r; };
    int *flag = (int *)take((size_t)(K + 1) * sizeof(int));
    int *pos = (int *)take((size_t)(K + 1) * sizeof(int));
    int *occ = (int *)take((size_t)(K + 1) * sizeof(int));
    double *den = (double *)take((size_t)K * sizeof(double));
    double *htab = (double *)take((size_t)tw * map->n_rows * sizeof(double));
    if (den_out) den = den_out;
    hood_table_kernel<<<(tw * m.ny + 255) / 256, 256, 0, st>>>(m, tw, dist_table, hood->neighborhood,
                                                               hood->compact, hood->radius, hood->cutoff, htab);
    note_launch();
    occ_flags<<<(K + 255) / 256, 256, 0, st>>>(cnt, K, flag);
    note_launch();
    rc = exclusive_scan(flag, K, pos, st);
    if (rc) return rc;
    occ_scatter<<<(K + 255) / 256, 256, 0, st>>>(flag, pos, K, occ);
    note_launch();
    const int *nocc = pos + K;
    const int nn = node_end - node_begin;
    if (nn == 0) return SOMB_OK;
    const bool spectral = use_spectral(map, hood);
    const bool spec_den = spectral && hood->cutoff > 0.0;
    if (!spec_den) {
        hood_den_kernel<<<(nn + 255) / 256, 256, 0, st>>>(m, tw, htab, cnt, occ, nocc, node_begin, node_end, den);
        note_launch();
    }
    if (spectral) {
        char *sws = (char *)ws + direct_ws(map, K);
        return spec_update(map, htab, S, cnt, d, den, spec_den ? 1 : 0, 0.5 * hood->cutoff, scale, W_old, node_begin,
                           node_end, W_new, num_out, sws, st);
    }
    dim3 g((d + kHN - 1) / kHN, (nn + kHM - 1) / kHM);
    hood_conv_blend<<<g, 256, 0, st>>>(m, tw, htab, S, d, occ, nocc, node_begin, node_end, den, scale,
                                       1.0 - scale, W_old, W_new, num_out);
    note_launch();
    SOMB_LAUNCH_CHECK("hood_update");
    return SOMB_OK;
}

namespace somb {
// Standalone blend (kernels.py:438-450) for the reference-compatible
// Accumulators path: same arithmetic as the fused epilogue above.
__global__ void blend_kernel(const float *__restrict__ Wold, const double *__restrict__ num,
                             const double *__restrict__ den, int K, int d, double alpha,
                             double one_minus_alpha, float *__restrict__ Wnew) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (int64_t)K * d) return;
    int j = (int)(e / d);
    float w = Wold[e];
    double dj = den[j];
    if (dj > 0.0) {
        double upd = __ddiv_rn(num[e], dj);
        w = __double2float_rn(__dadd_rn(__dmul_rn(one_minus_alpha, (double)w), __dmul_rn(alpha, upd)));
    }
    Wnew[e] = w;
}
}  // namespace somb

extern "C" int somb_blend(const float *W_old, const double *num, const double *den, int32_t K, int32_t d,
                          double scale, float *W_new, void *stream) {
    SOMB_REQUIRE(K > 0 && d > 0, SOMB_E_INPUT, "blend: bad shape K=%d d=%d", K, d);
    int64_t tot = (int64_t)K * d;
    somb::blend_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, somb::as_stream(stream)>>>(
        W_old, num, den, K, d, scale, 1.0 - scale, W_new);
    note_launch();
    SOMB_LAUNCH_CHECK("blend");
    return SOMB_OK;
}
