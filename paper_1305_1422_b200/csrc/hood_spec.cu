// Spectral neighbourhood convolution (fp64): num = H S without the O(K^2 D)
// direct sum.
//
// h(b, j) depends on the row offset dy (and, on the hex lattice, on the half
// column shift between odd and even rows) and on the column offset t =
// c_j - c_b only.  For every pair of map rows (y_out, y_in) the x-direction
// is therefore a 1-D convolution with a kernel k_{key}[t], key = (dy,
// shift).  A length-L DFT along x diagonalises it:
//   S^[y][f]     = sum_c S[y][c] w^{-fc}                      (fwd, real->complex)
//   N^[y_o][f]   = sum_{y_i} k^_{key(y_o,y_i)}[f] S^[y_i][f]   (complex GEMM per f)
//   num[y_o][c]  = 1/L sum_f wt_f Re(N^[y_o][f] w^{fc})       (inv, fused blend)
// with L = nx on toroids (circular = the reference's min-wrap, kernels.py:
// 109-111) and L = 2 nx on planar maps (zero padding => linear convolution,
// no wrap).  Only the F = L/2 + 1 non-redundant frequencies of the real
// input are carried.  Every step runs in fp64 through one tiled DFMA GEMM
// template with functional operand loaders; the influence values are the same
// htab entries the direct path uses (hood.cu).  den = H cnt rides along as
// one extra channel; its exact zero pattern (the den > 0 blend mask) is
// restored by thresholding at hmin / 2, valid whenever cutoff > 0 (every
// nonzero influence is then >= cutoff); with cutoff = 0 the direct fp64 den
// is used instead.
// Cost ~ F ny^2 D + 4 K F D complex MACs instead of K^2 D.
#include "common.cuh"

namespace somb {

struct SpecGeom {
    int nx, ny, L, F, hex, toroid, tw;
};

// ------------------------------------------------------- generic DFMA GEMM
// C(b)[M x N] = A(b)[M x K] * B(b)[K x N]; loaders return A(b, m, k) /
// B(b, k, n) (0 outside), the epilogue consumes (b, m, n, value).
constexpr int GM = 64, GN = 64, GK = 16;

template <class AL, class BL, class EP>
__global__ void __launch_bounds__(256) dgemm_fn(int M, int N, int Kd, AL al, BL bl, EP ep) {
    __shared__ double sa[GK][GM + 1];
    __shared__ double sb[GK][GN];
    const int t = threadIdx.x, tx = t % 16, ty = t / 16;
    const int b = blockIdx.z;
    const int m0 = blockIdx.y * GM, n0 = blockIdx.x * GN;
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (int k0 = 0; k0 < Kd; k0 += GK) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            int e = t + 256 * q;              // 0..1023
            int kk = e / GM, mm = e % GM;     // A tile: 16 x 64 (k-major in smem)
            int m = m0 + mm, k = k0 + kk;
            sa[kk][mm] = (m < M && k < Kd) ? al(b, m, k) : 0.0;
            int kb = e / GN, nn = e % GN;     // B tile: 16 x 64
            int n = n0 + nn, k2 = k0 + kb;
            sb[kb][nn] = (n < N && k2 < Kd) ? bl(b, k2, n) : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < GK; ++kk) {
            double av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = sa[kk][ty + 16 * i];
#pragma unroll
            for (int j = 0; j < 4; ++j) bv[j] = sb[kk][tx + 16 * j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = __fma_rn(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        int m = m0 + ty + 16 * i;
        if (m >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            int n = n0 + tx + 16 * j;
            if (n < N) ep(b, m, n, acc[i][j]);
        }
    }
}

// FP64 tensor-core variant: mma.sync.m8n8k4.f64 (DMMA).  Block tile 64 x 64
// x 8, four warps of 32 x 32 (4 x 4 m8n8 fragments); next k-tile prefetched
// into registers while the current one is multiplied.  Same loader /
// epilogue interface as dgemm_fn.  The GEMMs here are latency-bound (short
// K, DMMA dependency chains): the 8-deep k-tile keeps registers at 128, so
// four blocks (16 warps) fit per SM -- 14% faster at cfg3 than 16-deep tiles
// at three blocks, 35% faster than 32-deep at two.  DMMA peak measured on
// the B200: 37 TF/s.
constexpr int TM = 64, TN = 64, TK = 8, TPAD = 8;

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

template <class AL, class BL, class EP>
__global__ void __launch_bounds__(128, 4) dgemm_mma_fn(int M, int N, int Kd, AL al, BL bl, EP ep) {
    __shared__ double sa[TK][TM + TPAD];   // A tile stored k-major: sa[k][m]
    __shared__ double sb[TK][TN + TPAD];   // B tile: sb[k][n]
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
    // row tiles vary fastest in the launch order, so the blocks sharing a B
    // column panel run together and read it from L2 once (the panel order
    // re-read B from DRAM once per row tile: 25 GB at cfg3's Mid step)
    const int b = blockIdx.z;
    const int m0 = blockIdx.x * TM, n0 = blockIdx.y * TN;
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    constexpr int QE = TM * TK / 128;   // A (and B) tile elements per thread
    double ra[QE], rb[QE];
    auto fetch = [&](int k0) {
#pragma unroll
        for (int q = 0; q < QE; ++q) {
            int e = t + 128 * q;            // 0..1023
            int kk = e / TM, mm = e % TM;
            int m = m0 + mm, k = k0 + kk;
            ra[q] = (m < M && k < Kd) ? al(b, m, k) : 0.0;
            int kb = e / TN, nn = e % TN;
            int n = n0 + nn, k2 = k0 + kb;
            rb[q] = (n < N && k2 < Kd) ? bl(b, k2, n) : 0.0;
        }
    };
    fetch(0);
    for (int k0 = 0; k0 < Kd; k0 += TK) {
        __syncthreads();
#pragma unroll
        for (int q = 0; q < QE; ++q) {
            int e = t + 128 * q;
            sa[e / TM][e % TM] = ra[q];
            sb[e / TN][e % TN] = rb[q];
        }
        __syncthreads();
        if (k0 + TK < Kd) fetch(k0 + TK);
#pragma unroll
        for (int ks = 0; ks < TK; ks += 4) {
            double af[4], bf[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) af[i] = sa[ks + (lane & 3)][wm + 8 * i + (lane >> 2)];
#pragma unroll
            for (int j = 0; j < 4; ++j) bf[j] = sb[ks + (lane & 3)][wn + 8 * j + (lane >> 2)];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma884(acc[i][j], af[i], bf[j]);
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        int m = m0 + wm + 8 * i + (lane >> 2);
        if (m >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                int n = n0 + wn + 8 * j + 2 * (lane & 3) + h;
                if (n < N) ep(b, m, n, acc[i][j][h]);
            }
        }
    }
}

static int g_dgemm_impl = -1;   // SOMB_DGEMM=dfma selects the DFMA tiles (A/B testing)

template <class AL, class BL, class EP>
static void dgemm_launch(int batch, int M, int N, int Kd, AL al, BL bl, EP ep, cudaStream_t st) {
    if (g_dgemm_impl < 0) {
        const char *e = getenv("SOMB_DGEMM");
        g_dgemm_impl = (e && strcmp(e, "dfma") == 0) ? 0 : 1;
    }
    if (g_dgemm_impl == 1) {
        dim3 g((M + TM - 1) / TM, (N + TN - 1) / TN, batch);
        dgemm_mma_fn<<<g, 128, 0, st>>>(M, N, Kd, al, bl, ep);
    } else {
        dim3 g((N + GN - 1) / GN, (M + GM - 1) / GM, batch);
        dgemm_fn<<<g, 256, 0, st>>>(M, N, Kd, al, bl, ep);
    }
    note_launch();
}

// ------------------------------------------------------------------ tables
// twiddles: cs[q] = cos(2 pi q / L), sn[q] = sin(2 pi q / L), q in [0, L)
__global__ void spec_twiddle(int L, double *cs, double *sn) {
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= L) return;
    double s, c;
    sincospi(2.0 * (double)q / (double)L, &s, &c);
    cs[q] = c;
    sn[q] = s;
}

__device__ __forceinline__ int spec_nkeys_dev(const SpecGeom &g) {
    int ndy = g.toroid ? g.ny / 2 + 1 : g.ny;
    return g.hex ? 3 * ndy : ndy;
}

// key of a row pair: dy (wrapped on toroids) and, on hex, the half-column
// shift sh = (y_out & 1) - (y_in & 1) in {-1, 0, 1}
__device__ __forceinline__ int spec_key(const SpecGeom &g, int yo, int yi) {
    int dy = abs(yo - yi);
    if (g.toroid) dy = min(dy, g.ny - dy);
    if (!g.hex) return dy;
    int sh = (yo & 1) - (yi & 1);
    return dy * 3 + (sh + 1);
}

// Dense DFT operands, built once per update so the GEMM loaders are plain
// loads: Phi [2F][nx] (cos rows, then -sin rows; forward, real -> complex)
// and Psi [nx][2F] (inverse with the real-signal weights w_f / L).
__global__ void spec_dft_mats(SpecGeom g, const double *__restrict__ cs, const double *__restrict__ sn,
                              double *__restrict__ phi, double *__restrict__ psi) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t tot = (int64_t)2 * g.F * g.nx;
    if (e >= tot) return;
    const int r = (int)(e / g.nx), c = (int)(e % g.nx);
    const int plane = r >= g.F, f = r - plane * g.F;
    const int q = (int)(((int64_t)f * c) % g.L);
    phi[e] = plane ? -sn[q] : cs[q];
    const double w = (f == 0 || 2 * f == g.L) ? 1.0 : 2.0;
    psi[(int64_t)c * 2 * g.F + r] = w * (plane ? -sn[q] : cs[q]) / (double)g.L;
}

// ktT [f][key][2]: the kernel spectra regrouped per frequency (MidA locality)
__global__ void spec_ktab_T(int nkeys, int F, const double *__restrict__ ktab, double *__restrict__ ktT) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nkeys * F) return;
    const int key = e / F, f = e % F;
    ktT[((int64_t)f * nkeys + key) * 2 + 0] = ktab[((int64_t)key * 2 + 0) * F + f];
    ktT[((int64_t)f * nkeys + key) * 2 + 1] = ktab[((int64_t)key * 2 + 1) * F + f];
}

// k^[key][f] = sum_t k[t] w^{-f t}; ktab layout [key][2][F] (re, im)
__global__ void spec_kernel_table(SpecGeom g, const double *__restrict__ htab, const double *__restrict__ cs,
                                  const double *__restrict__ sn, double *__restrict__ ktab) {
    extern __shared__ double kt[];   // L values of k[t]
    const int key = blockIdx.x;
    const int dy = g.hex ? key / 3 : key;
    const int sh = g.hex ? key % 3 - 1 : 0;
    for (int t = threadIdx.x; t < g.L; t += blockDim.x) {
        // signed column offset t_s = c_out - c_in
        int ts = t;
        double v = 0.0;
        bool valid = true;
        if (!g.toroid) {
            ts = t < g.nx ? t : t - g.L;              // L = 2 nx
            if (ts <= -g.nx || ts >= g.nx) valid = false;
        }
        if (valid) {
            int idx;
            if (!g.hex) {
                int dx = abs(ts);
                if (g.toroid) dx = min(dx % g.nx, g.nx - dx % g.nx);
                idx = dy * g.tw + dx;
            } else {
                int dx2 = abs(2 * ts + sh);
                if (g.toroid) {
                    dx2 %= 2 * g.nx;
                    dx2 = min(dx2, 2 * g.nx - dx2);
                }
                idx = dy * g.tw + dx2;
            }
            v = htab[idx];
        }
        kt[t] = v;
    }
    __syncthreads();
    for (int f = threadIdx.x; f < g.F; f += blockDim.x) {
        double re = 0.0, im = 0.0;
        int q = 0;                                     // (f * t) mod L, incremental
        for (int t = 0; t < g.L; ++t) {
            double v = kt[t];
            re = __fma_rn(v, cs[q], re);
            im = __fma_rn(-v, sn[q], im);
            q += f;
            if (q >= g.L) q -= g.L;
        }
        ktab[((int64_t)key * 2 + 0) * g.F + f] = re;
        ktab[((int64_t)key * 2 + 1) * g.F + f] = im;
    }
}

// ----------------------------------------------------------- GEMM operands
// fwd: A = Phi [2F x nx] (cos rows then -sin rows), B = S_y [nx x D]
struct FwdA {
    const double *phi; int nx;
    __device__ double operator()(int, int r, int c) const { return phi[(int64_t)r * nx + c]; }
};
// column d == D carries the BMU counts, so den = H cnt rides the same DFTs
struct FwdB {
    SpecGeom g; const double *S; const double *cnt; int D;
    __device__ double operator()(int y, int c, int d) const {
        if (c >= g.nx) return 0.0;
        return d < D ? S[((int64_t)y * g.nx + c) * D + d] : cnt[y * g.nx + c];
    }
};
// Shat layout [plane][f][y][d]
struct FwdEp {
    SpecGeom g; double *Sh; int D;
    __device__ void operator()(int y, int r, int d, double v) const {
        int plane = r >= g.F, f = r - plane * g.F;
        Sh[(((int64_t)plane * g.F + f) * g.ny + y) * D + d] = v;
    }
};
// mid: per f, [Nr; Ni] = [[Kr, -Ki], [Ki, Kr]] [Sr; Si], rows y_out in [y0, y0+nyo)
struct MidA {
    SpecGeom g; const double *ktT; int nkeys, y0, nyo;
    __device__ double operator()(int f, int r, int k) const {
        int pr = r >= nyo, pk = k >= g.ny;
        int yo = y0 + r - pr * nyo, yi = k - pk * g.ny;
        int key = spec_key(g, yo, yi);
        const double2 kk = *reinterpret_cast<const double2 *>(ktT + ((int64_t)f * nkeys + key) * 2);
        double kr = kk.x, ki = kk.y;
        if (!pr) return pk ? -ki : kr;
        return pk ? kr : ki;
    }
};
// the same operand materialised once per update as a dense [f][2 nyo][2 ny]
// array (values bit-identical to MidA), when it fits the workspace budget:
// the GEMM's A loads become plain loads instead of per-element key math
struct MidAm {
    const double *A; int M2, K2;
    __device__ double operator()(int f, int r, int k) const { return A[((int64_t)f * M2 + r) * K2 + k]; }
};
__global__ void spec_mid_mat(MidA a, int F, int M2, int K2, double *__restrict__ out) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t per = (int64_t)M2 * K2;
    if (e >= (int64_t)F * per) return;
    const int f = (int)(e / per), rk = (int)(e % per);
    out[e] = a(f, rk / K2, rk % K2);
}

struct MidB {
    SpecGeom g; const double *Sh; int D;
    __device__ double operator()(int f, int k, int d) const {
        int pk = k >= g.ny, yi = k - pk * g.ny;
        return Sh[(((int64_t)pk * g.F + f) * g.ny + yi) * D + d];
    }
};
// Nhat layout [plane][f][y_local][d]
struct MidEp {
    SpecGeom g; double *Nh; int nyo, D;
    __device__ void operator()(int f, int r, int d, double v) const {
        int pr = r >= nyo, yl = r - pr * nyo;
        Nh[(((int64_t)pr * g.F + f) * nyo + yl) * D + d] = v;
    }
};
// den_j (spec_den_kernel) keeps the exact zero pattern: every nonzero
// influence is >= hmin (cutoff, or 1 for bubble), so a true den_j is 0 or
// >= hmin, while the DFT rounding is orders of magnitude below hmin / 2.
// inv: num_y [nx x D] = Psi [nx x 2F] * [Nr_y; Ni_y]
struct InvA {
    const double *psi; int F2;
    __device__ double operator()(int, int c, int q2) const { return psi[(int64_t)c * F2 + q2]; }
};
struct InvB {
    SpecGeom g; const double *Nh; int nyo, Dp1;
    __device__ double operator()(int yl, int q2, int d) const {
        int plane = q2 >= g.F, f = q2 - plane * g.F;
        return Nh[(((int64_t)plane * g.F + f) * nyo + yl) * Dp1 + d];
    }
};
struct InvEp {
    SpecGeom g; int y0, j0, j1, D;
    const double *den; double alpha, oma;
    const float *Wold; float *Wnew; double *num_out;
    __device__ void operator()(int yl, int c, int d, double num) const {
        if (c >= g.nx) return;
        int j = (y0 + yl) * g.nx + c;
        if (j < j0 || j >= j1) return;
        int64_t o = (int64_t)j * D + d;
        if (num_out) num_out[o] = num;
        float w = Wold[o];
        double dj = den[j];
        if (dj > 0.0) {
            double upd = __ddiv_rn(num, dj);
            w = __double2float_rn(__dadd_rn(__dmul_rn(oma, (double)w), __dmul_rn(alpha, upd)));
        }
        Wnew[o] = w;
    }
};

// den channel of the inverse DFT (N = 1: a GEMV, one thread per output;
// running it through the 64-wide GEMM tile wasted 63/64 of the MMAs).
__global__ void spec_den_kernel(SpecGeom g, const double *__restrict__ psi, const double *__restrict__ Nh, int nyo,
                                int Dp1, int y0, int j0, int j1, double tau, double *__restrict__ den) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nyo * g.nx) return;
    const int yl = e / g.nx, c = e % g.nx;
    const int j = (y0 + yl) * g.nx + c;
    if (j < j0 || j >= j1) return;
    const int F2 = 2 * g.F;
    double v = 0.0;
    for (int q2 = 0; q2 < F2; ++q2) {
        const int plane = q2 >= g.F, f = q2 - plane * g.F;
        v = __fma_rn(psi[(int64_t)c * F2 + q2], Nh[(((int64_t)plane * g.F + f) * nyo + yl) * Dp1 + (Dp1 - 1)], v);
    }
    den[j] = v < tau ? 0.0 : v;
}

static SpecGeom spec_geom(const somb_map *m) {
    SpecGeom g;
    g.nx = m->n_columns;
    g.ny = m->n_rows;
    g.hex = m->grid == SOMB_GRID_HEX;
    g.toroid = m->topology == SOMB_TOROID;
    g.L = g.toroid ? g.nx : 2 * g.nx;
    g.F = g.L / 2 + 1;
    g.tw = g.hex ? 2 * g.nx : g.nx;
    return g;
}

static int spec_nkeys(const SpecGeom &g) {
    int ndy = g.toroid ? g.ny / 2 + 1 : g.ny;
    return g.hex ? 3 * ndy : ndy;
}

// materialised mid operand (MidAm) for all map rows, if within budget
static size_t spec_mid_mat_bytes(const SpecGeom &g) {
    const size_t b = (size_t)g.F * (2 * (size_t)g.ny) * (2 * (size_t)g.ny) * 8;
    return b <= ((size_t)256 << 20) ? b : 0;
}

size_t spec_ws_bytes(const somb_map *m, int d) {
    SpecGeom g = spec_geom(m);
    size_t b = 2 * align_up((size_t)g.L * 8, 256);
    b += 2 * align_up((size_t)spec_nkeys(g) * 2 * g.F * 8, 256);   // ktab + per-frequency copy
    b += 2 * align_up((size_t)2 * g.F * g.nx * 8, 256);             // Phi, Psi
    b += align_up((size_t)2 * g.F * g.ny * (d + 1) * 8, 256);      // Shat (+ count channel)
    b += align_up((size_t)2 * g.F * g.ny * (d + 1) * 8, 256);      // Nhat (worst case: all rows)
    b += align_up(spec_mid_mat_bytes(g), 256);                      // MidAm (0 when over budget)
    return b;
}

// den_mode: 0 = den given (direct, exact), 1 = compute den spectrally into `den`
// with the zero threshold tau = hmin / 2.
int spec_update(const somb_map *m, const double *htab, const double *S, const double *cnt, int d, double *den,
                int den_mode, double tau, double scale, const float *Wold, int j0, int j1, float *Wnew,
                double *num_out, void *ws, cudaStream_t st) {
    SpecGeom g = spec_geom(m);
    char *p = (char *)ws;
    auto take = [&](size_t bytes) { char *r = p; p += align_up(bytes, 256); return r; };
    double *cs = (double *)take((size_t)g.L * 8);
    double *sn = (double *)take((size_t)g.L * 8);
    const int nkeys = spec_nkeys(g);
    double *ktab = (double *)take((size_t)nkeys * 2 * g.F * 8);
    double *ktT = (double *)take((size_t)nkeys * 2 * g.F * 8);
    double *phi = (double *)take((size_t)2 * g.F * g.nx * 8);
    double *psi = (double *)take((size_t)2 * g.F * g.nx * 8);
    const int Dp1 = d + 1;
    double *Sh = (double *)take((size_t)2 * g.F * g.ny * Dp1 * 8);
    const int y0 = j0 / g.nx, y1 = (j1 + g.nx - 1) / g.nx, nyo = y1 - y0;
    double *Nh = (double *)take((size_t)2 * g.F * nyo * Dp1 * 8);
    double *Am = spec_mid_mat_bytes(g) ? (double *)take(spec_mid_mat_bytes(g)) : nullptr;
    spec_twiddle<<<(g.L + 255) / 256, 256, 0, st>>>(g.L, cs, sn);
    note_launch();
    spec_kernel_table<<<nkeys, 256, (size_t)g.L * 8, st>>>(g, htab, cs, sn, ktab);
    note_launch();
    spec_ktab_T<<<(nkeys * g.F + 255) / 256, 256, 0, st>>>(nkeys, g.F, ktab, ktT);
    note_launch();
    spec_dft_mats<<<(unsigned)(((int64_t)2 * g.F * g.nx + 255) / 256), 256, 0, st>>>(g, cs, sn, phi, psi);
    note_launch();
    const int nc = den_mode ? Dp1 : d;     // channels carried through the DFTs
    dgemm_launch(g.ny, 2 * g.F, nc, g.nx, FwdA{phi, g.nx}, FwdB{g, S, cnt, d}, FwdEp{g, Sh, Dp1}, st);
    if (Am) {
        const int64_t tot = (int64_t)g.F * (2 * nyo) * (2 * g.ny);
        spec_mid_mat<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(MidA{g, ktT, nkeys, y0, nyo}, g.F, 2 * nyo,
                                                                    2 * g.ny, Am);
        note_launch();
        dgemm_launch(g.F, 2 * nyo, nc, 2 * g.ny, MidAm{Am, 2 * nyo, 2 * g.ny}, MidB{g, Sh, Dp1},
                     MidEp{g, Nh, nyo, Dp1}, st);
    } else {
        dgemm_launch(g.F, 2 * nyo, nc, 2 * g.ny, MidA{g, ktT, nkeys, y0, nyo}, MidB{g, Sh, Dp1},
                     MidEp{g, Nh, nyo, Dp1}, st);
    }
    if (den_mode) {
        spec_den_kernel<<<(nyo * g.nx + 255) / 256, 256, 0, st>>>(g, psi, Nh, nyo, Dp1, y0, j0, j1, tau, den);
        note_launch();
    }
    dgemm_launch(nyo, g.nx, d, 2 * g.F, InvA{psi, 2 * g.F}, InvB{g, Nh, nyo, Dp1},
                 InvEp{g, y0, j0, j1, d, den, scale, 1.0 - scale, Wold, Wnew, num_out}, st);
    SOMB_LAUNCH_CHECK("spectral hood update");
    return SOMB_OK;
}

}  // namespace somb
