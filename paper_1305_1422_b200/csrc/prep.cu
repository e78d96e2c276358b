// Dataset and codebook preparation for the fp16 tensor-core screen.
//
// Screening identity: with nu = data mean, mu = codebook
// mean, delta_j = w_j - mu, x'_i = x_i - nu,
//   |x_i - w_j|^2 = |x_i - mu|^2 + r_ij,   r_ij = c_j - 2 x'_i . delta_j,
//   c_j = |delta_j|^2 + 2 (mu - nu) . delta_j.
// The row term |x_i - mu|^2 does not affect the argmin, so the screen ranks
// r_ij; both operands are centred, which keeps the fp16 rounding error small
// relative to the gaps between nodes after the codebook collapses
// (SURVEY.md 7.3-1).
#include <cuda_fp8.h>
#include <float.h>

#include "common.cuh"

namespace somb {


// ----------------------------------------------------- stochastic rounding
// The screen's fp16 operands are rounded STOCHASTICALLY:
// v goes to the fp16 neighbour above |v| with probability (|v| - lo) / ulp,
// using 32 dither bits from a counter-based hash of (row or node, feature,
// value bits).  The rounding errors are then independent and mean-zero
// whatever the data's structure (constant rows, duplicated columns, integer
// values), so the screen error is a sum of independent terms whose scale
// the per-row window sigma (screen_sigma, cand.cuh) bounds from the rows'
// ulp profile.  Round-to-nearest made them coherent on such data (a
// near-constant row rounds every feature the same way), which broke a
// window calibrated on uniform data (Weak 1).
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}
__device__ __forceinline__ uint32_t dither32(uint64_t domain, uint64_t a, uint32_t b, uint32_t vbits) {
    uint64_t z = mix64(domain ^ (a * 0x9E3779B97F4A7C15ull));
    z = mix64(z ^ (((uint64_t)b << 32) | vbits));
    return (uint32_t)(z >> 32);
}
constexpr uint64_t kDitherX = 0x5EEDDA7A00000001ull;   // data rows
constexpr uint64_t kDitherW = 0x5EEDC0DE00000002ull;   // codebook nodes

// fp16 spacing at |v| (normal range; subnormal spacing 2^-24) and whether v
// sits exactly on the grid (then it rounds without error)
__device__ __forceinline__ double f16_spacing(double a) {
    int e = ilogb(a);
    return ldexp(1.0, (e < -14 ? -14 : e) - 10);
}

// Stochastic rounding of v (|v| < 65504) to fp16; *err_span = the spacing
// of the two candidates (the width of the error's range), 0 if v is exact.
__device__ __forceinline__ __half sr_half(double v, uint32_t u, double *err_span) {
    const double a = fabs(v);
    if (a == 0.0) { *err_span = 0.0; return __double2half(0.0); }
    const double sp = f16_spacing(a);
    const double q = a / sp;                 // exact: power-of-two scaling
    const double fl = floor(q);
    const double fr = q - fl;                // exact
    *err_span = fr > 0.0 ? sp : 0.0;
    const double m = fl + (ldexp((double)u, -32) < fr ? 1.0 : 0.0);
    return __double2half(copysign(m * sp, v));   // exactly representable
}

// ---------------------------------------------------------------- data stats
// Stage 1: per (row-chunk, column) fp64 partial sum plus column min/max.
constexpr int kStatChunks = 256;

__global__ void data_stats_partial(const float *__restrict__ X, int64_t n, int d,
                                   double *__restrict__ psum, float *__restrict__ pmin,
                                   float *__restrict__ pmax) {
    int col = blockIdx.x * blockDim.x + threadIdx.x;
    int chunk = blockIdx.y;
    if (col >= d) return;
    int64_t per = (n + kStatChunks - 1) / kStatChunks;
    int64_t a = chunk * per, b = min(n, a + per);
    double s = 0.0;
    float lo = INFINITY, hi = -INFINITY;
    for (int64_t i = a; i < b; ++i) {
        float v = X[i * d + col];
        s += (double)v;
        lo = fminf(lo, v);
        hi = fmaxf(hi, v);
    }
    psum[(int64_t)chunk * d + col] = s;
    pmin[(int64_t)chunk * d + col] = lo;
    pmax[(int64_t)chunk * d + col] = hi;
}

// Stage 2: fixed-order fold over chunks -> nu (f32) and max|x - nu|.
__global__ void data_stats_final(const double *__restrict__ psum, const float *__restrict__ pmin,
                                 const float *__restrict__ pmax, int64_t n, int d,
                                 float *__restrict__ nu, float *__restrict__ absmax) {
    int col = blockIdx.x * blockDim.x + threadIdx.x;
    if (col >= d) return;
    double s = 0.0;
    float lo = INFINITY, hi = -INFINITY;
    for (int c = 0; c < kStatChunks; ++c) {
        s += psum[(int64_t)c * d + col];
        lo = fminf(lo, pmin[(int64_t)c * d + col]);
        hi = fmaxf(hi, pmax[(int64_t)c * d + col]);
    }
    float m = n > 0 ? (float)(s / (double)n) : 0.0f;
    nu[col] = m;
    float a = n > 0 ? fmaxf(fabsf(hi - m), fabsf(m - lo)) : 0.0f;
    atomic_max_nonneg(absmax, a);
}

// Xh = fp16((x - nu) * 2^xexp) (stochastic rounding), xnorm = |x - nu|,
// x2 = |x|^2 (fp64), xstat = {|x'|, max_k |x'_k|, max_k ulp_k, |ulp|_2}
// with ulp_k the error span of feature k (unscaled units): the row inputs of
// the window sigma.  With Xl (3-pass screen): round-to-nearest hi and the
// fp16 residual Xl (~22-bit operands, hi.hi + hi.lo + lo.hi); its window is
// the accumulation-bound unit 2^-11 |x'| max|delta| / sqrt(d), which xstat
// encodes as {|x'|, 0, |x'| 2^-11 / sqrt(d), FLT_MAX} (screen_sigma).
__global__ void data_pack_kernel(const float *__restrict__ X, int64_t n, int d,
                                 const float *__restrict__ nu, int xexp,
                                 __half *__restrict__ Xh, __half *__restrict__ Xl, int dp,
                                 float *__restrict__ xnorm, double *__restrict__ x2,
                                 float4 *__restrict__ xstat) {
    int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    int lane = threadIdx.x & 31;
    if (row >= n) return;
    const float *x = X + row * d;
    __half *o = Xh + row * dp;
    __half *ol = Xl ? Xl + row * dp : nullptr;
    double sc = ldexp(1.0, xexp);
    double nrm = 0.0, sq = 0.0, u2 = 0.0;
    float xinf = 0.0f, uinf = 0.0f;
    for (int k = lane; k < dp; k += 32) {
        if (k < d) {
            const float xf = x[k];
            double xv = (double)xf;
            double v = xv - (double)nu[k];
            nrm += v * v;
            sq += xv * xv;
            xinf = fmaxf(xinf, (float)fabs(v));
            if (ol) {
                __half h = __double2half(v * sc);
                o[k] = h;
                ol[k] = __double2half(v * sc - (double)__half2float(h));
            } else {
                double span;
                o[k] = sr_half(v * sc, dither32(kDitherX, (uint64_t)row, (uint32_t)k, __float_as_uint(xf)), &span);
                span = ldexp(span, -xexp);
                u2 += span * span;
                uinf = fmaxf(uinf, (float)span);
            }
        } else {
            o[k] = __double2half(0.0);
            if (ol) ol[k] = __double2half(0.0);
        }
    }
    nrm = warp_sum(nrm);
    sq = warp_sum(sq);
    u2 = warp_sum(u2);
    xinf = warp_max(xinf);
    uinf = warp_max(uinf);
    if (lane == 0) {
        const float xn = (float)sqrt(nrm);
        xnorm[row] = xn;
        x2[row] = sq;
        if (xstat)
            xstat[row] = ol ? make_float4(xn, 0.0f, xn * (float)ldexp(rsqrt((double)d), -11), FLT_MAX)
                            : make_float4(xn, xinf, uinf, (float)sqrt(u2));
    }
}

// 2-pass (fp16 + fp8 cross terms) operands: Xh = fp16(v 2^xexp) (xexp puts
// max |v| 2^xexp <= 2^13), X8 = [e4m3(xh / 32) | e4m3(xl * 32)] with the
// residual xl = v 2^xexp - xh (2 dp bytes per row), so that
// x_hi8 . w_lo8 + x_lo8 . w_hi8 ~ xh . wl + xl . wh in the fp16 pass's units.
__device__ __forceinline__ uint8_t to_e4m3(double v) {
    return (uint8_t)__nv_cvt_float_to_fp8((float)v, __NV_SATFINITE, __NV_E4M3);
}

__global__ void data_pack_f8_kernel(const float *__restrict__ X, int64_t n, int d, const float *__restrict__ nu,
                                    int xexp, __half *__restrict__ Xh, uint8_t *__restrict__ X8, int dp,
                                    float *__restrict__ xnorm, double *__restrict__ x2, float4 *__restrict__ xstat) {
    int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    int lane = threadIdx.x & 31;
    if (row >= n) return;
    const float *x = X + row * d;
    __half *o = Xh + row * dp;
    uint8_t *o8 = X8 + row * (int64_t)(2 * dp);
    const double sc = ldexp(1.0, xexp);
    double nrm = 0.0, sq = 0.0, u2 = 0.0;
    float xinf = 0.0f, uinf = 0.0f;
    for (int k = lane; k < dp; k += 32) {
        double v = 0.0;
        __half h = __double2half(0.0);
        if (k < d) {
            const float xf = x[k];
            double xv = (double)xf;
            v = xv - (double)nu[k];
            nrm += v * v;
            sq += xv * xv;
            xinf = fmaxf(xinf, (float)fabs(v));
            double span;
            h = sr_half(v * sc, dither32(kDitherX, (uint64_t)row, (uint32_t)k, __float_as_uint(xf)), &span);
            span = ldexp(span, -xexp);
            u2 += span * span;
            uinf = fmaxf(uinf, (float)span);
        }
        const double hd = (double)__half2float(h);
        o[k] = h;
        o8[k] = to_e4m3(hd * (1.0 / 32.0));
        o8[dp + k] = to_e4m3((v * sc - hd) * 32.0);
    }
    nrm = warp_sum(nrm);
    sq = warp_sum(sq);
    u2 = warp_sum(u2);
    xinf = warp_max(xinf);
    uinf = warp_max(uinf);
    if (lane == 0) {
        const float xn = (float)sqrt(nrm);
        xnorm[row] = xn;
        x2[row] = sq;
        if (xstat) xstat[row] = make_float4(xn, xinf, uinf, (float)sqrt(u2));
    }
}

// ------------------------------------------------------------- codebook prep
// ws layout: mu f32[d] | mu_nu f64[d] | nrm f32[K] | stats f32[8] {max|delta_j|,
// max|delta_jk|, max|c_j|, max|ulp(delta_j)|_2, max ulp(delta_jk), -, -, -}
__global__ void cb_colmean(const float *__restrict__ W, int K, int d, const float *__restrict__ nu,
                           float *__restrict__ mu, double *__restrict__ mu_nu) {
    // one warp per column: lane-strided partial sums then a fixed xor tree
    int col = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    int lane = threadIdx.x & 31;
    if (col >= d) return;
    double s = 0.0;
    for (int j = lane; j < K; j += 32) s += (double)W[(int64_t)j * d + col];
    s = warp_sum(s);
    if (lane == 0) {
        float m = (float)(s / (double)K);
        mu[col] = m;
        mu_nu[col] = (double)m - (double)nu[col];
    }
}

__global__ void cb_rowstats(const float *__restrict__ W, int K, int d, const float *__restrict__ mu,
                            const double *__restrict__ mu_nu, float *__restrict__ c,
                            double *__restrict__ w2, float *__restrict__ nrm_out,
                            float *__restrict__ stats) {
    int j = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    int lane = threadIdx.x & 31;
    if (j >= K) return;
    const float *w = W + (int64_t)j * d;
    const float *w0 = W;
    double n2 = 0.0, cm = 0.0, sq = 0.0, u2 = 0.0;
    float amax = 0.0f, uinf = 0.0f;
    bool same0 = j > 0;
    for (int k = lane; k < d; k += 32) {
        float wf = w[k];
        same0 &= __float_as_uint(wf) == __float_as_uint(w0[k]);
        double wv = (double)wf;
        double dl = wv - (double)mu[k];
        n2 += dl * dl;
        cm += mu_nu[k] * dl;
        sq += wv * wv;
        amax = fmaxf(amax, (float)fabs(dl));
        // error span of the stochastic fp16 rounding of dl (cb_pack): the
        // fp16 grid is scale-invariant for powers of two, so the span of the
        // scaled value is this one times 2^sexp (normal range; the
        // subnormal floor is added in cb_pack)
        const double a = fabs(dl);
        if (a > 0.0) {
            const double sp = ldexp(1.0, ilogb(a) - 10);
            if (a / sp != floor(a / sp)) {
                u2 += sp * sp;
                uinf = fmaxf(uinf, (float)sp);
            }
        }
    }
    n2 = warp_sum(n2);
    cm = warp_sum(cm);
    sq = warp_sum(sq);
    u2 = warp_sum(u2);
    amax = warp_max(amax);
    uinf = warp_max(uinf);
    // A node bit-identical to node 0 ties it exactly in every distance, and
    // ties resolve to the lowest index (kernels.py:27-28): mask it out of the
    // screen (c = +inf).  Covers the collapsed maps of SURVEY.md A.8.
    same0 = __all_sync(0xffffffffu, same0);
    if (lane == 0) {
        float cj = (float)(n2 + 2.0 * cm);
        c[j] = same0 ? INFINITY : cj;
        atomic_max_nonneg(&stats[2], fabsf(cj));
        w2[j] = sq;
        float nr = (float)sqrt(n2);
        nrm_out[j] = nr;
        atomic_max_nonneg(&stats[0], nr);
        atomic_max_nonneg(&stats[1], amax);
        atomic_max_nonneg(&stats[3], (float)sqrt(u2));
        atomic_max_nonneg(&stats[4], uinf);
    }
}

__device__ __forceinline__ int pick_exp(float amax, int top = 14) {
    // largest e with amax * 2^e <= 2^top (fp16 max 65504; top 13 for the
    // fp8 cross-term ranges); 0 for amax == 0
    if (!(amax > 0.0f)) return 0;
    int e;
    frexpf(amax, &e);           // amax = f * 2^e, f in [0.5, 1)
    return top - e;
}

// Wh = fp16(delta 2^sexp): stochastic rounding (dither from (node, feature,
// value bits), so a new codebook draws fresh dither) unless Wl is given (the
// 3-pass screen: round-to-nearest hi + fp16 residual Wl).
// W8 (2-pass mode, Wl unused): [e4m3(wl * 32) | e4m3(wh / 32)], 2 dp bytes
// per row, wl = the residual of the (stochastic) hi.
__global__ void cb_pack(const float *__restrict__ W, int K, int d, const float *__restrict__ mu,
                        int xexp, __half *__restrict__ Wh, __half *__restrict__ Wl, int dp, int kp,
                        float *__restrict__ c, const float *__restrict__ stats,
                        float *__restrict__ scal, uint8_t *__restrict__ W8) {
    int j = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    int lane = threadIdx.x & 31;
    if (j >= kp) return;
    int sexp = pick_exp(stats[1], W8 ? 13 : 14);
    __half *o = Wh ? Wh + (int64_t)j * dp : nullptr;
    __half *ol = Wl ? Wl + (int64_t)j * dp : nullptr;
    uint8_t *o8 = W8 ? W8 + (int64_t)j * (2 * dp) : nullptr;
    if (o == nullptr) {
        if (j >= K && lane == 0) c[j] = INFINITY;
    } else {
        const float *w = W + (int64_t)(j < K ? j : 0) * d;
        const double sc = ldexp(1.0, sexp);
        for (int k = lane; k < dp; k += 32) {
            const bool live = j < K && k < d;
            const float wf = live ? w[k] : 0.0f;
            const double v = live ? ((double)wf - (double)mu[k]) * sc : 0.0;
            __half h;
            if (ol) {
                h = __double2half(v);
                ol[k] = __double2half(v - (double)__half2float(h));
            } else {
                double span;
                h = sr_half(v, dither32(kDitherW, (uint64_t)j, (uint32_t)k, __float_as_uint(wf)), &span);
            }
            o[k] = h;
            if (o8) {
                const double hd = (double)__half2float(h);
                o8[k] = to_e4m3((v - hd) * 32.0);
                o8[dp + k] = to_e4m3(hd * (1.0 / 32.0));
            }
        }
        if (j >= K && lane == 0) c[j] = INFINITY;
    }
    if (j == 0 && lane == 0) {
        // r = c_j - 2 * (x' . delta): acc * 2^-(xexp + sexp) is the dot product
        scal[0] = -2.0f * ldexpf(1.0f, -(xexp + sexp));
        scal[1] = stats[0];     // max_j |delta_j|
        scal[2] = (float)sexp;
        scal[3] = stats[1];     // max_jk |delta_jk|
        scal[4] = stats[2];     // max_j |c_j| (fp32 rounding slack of the windows)
        // max_j |ulp(delta_j)|_2 and max_jk ulp(delta_jk) of the stochastic
        // rounding, plus the subnormal floor (spacing 2^-24 after scaling)
        const float floor_sp = ldexpf(1.0f, -24 - sexp);
        scal[5] = stats[3] + floor_sp * sqrtf((float)dp);
        scal[6] = fmaxf(stats[4], floor_sp);
    }
}

}  // namespace somb

using namespace somb;

extern "C" size_t somb_data_stats_ws(int32_t d) {
    return align_up((size_t)kStatChunks * d * (sizeof(double) + 2 * sizeof(float)), 256);
}

extern "C" int somb_data_stats(const float *X, int64_t n, int32_t d, float *nu, float *absmax,
                               void *ws, void *stream) {
    SOMB_REQUIRE(d > 0 && n >= 0, SOMB_E_INPUT, "data_stats: bad shape n=%lld d=%d", (long long)n, d);
    cudaStream_t st = as_stream(stream);
    double *psum = (double *)ws;
    float *pmin = (float *)(psum + (size_t)kStatChunks * d);
    float *pmax = pmin + (size_t)kStatChunks * d;
    cudaMemsetAsync(absmax, 0, sizeof(float), st);
    dim3 g((d + 127) / 128, kStatChunks);
    data_stats_partial<<<g, 128, 0, st>>>(X, n, d, psum, pmin, pmax);
    note_launch();
    data_stats_final<<<(d + 127) / 128, 128, 0, st>>>(psum, pmin, pmax, n, d, nu, absmax);
    note_launch();
    SOMB_LAUNCH_CHECK("somb_data_stats");
    return SOMB_OK;
}

extern "C" int somb_data_pack(const float *X, int64_t n, int32_t d, const float *nu, int32_t xexp,
                              uint16_t *Xh, uint16_t *Xl, int32_t dp, float *xnorm, double *x2, float *xstat,
                              void *stream) {
    SOMB_REQUIRE(d > 0 && dp >= d && dp % 8 == 0, SOMB_E_INPUT, "data_pack: bad pitch d=%d dp=%d", d, dp);
    if (n == 0) return SOMB_OK;
    int rows_per_block = 8;
    int64_t blocks = (n + rows_per_block - 1) / rows_per_block;
    data_pack_kernel<<<(unsigned)blocks, 32 * rows_per_block, 0, as_stream(stream)>>>(
        X, n, d, nu, xexp, (__half *)Xh, (__half *)Xl, dp, xnorm, x2, reinterpret_cast<float4 *>(xstat));
    note_launch();
    SOMB_LAUNCH_CHECK("somb_data_pack");
    return SOMB_OK;
}

extern "C" size_t somb_codebook_ws(int32_t K, int32_t d) {
    return align_up((size_t)d * sizeof(float), 256) + align_up((size_t)d * sizeof(double), 256) +
           align_up((size_t)K * sizeof(float), 256) + 256;
}

extern "C" int somb_codebook_prepare(const float *W, int32_t K, int32_t d, const float *nu,
                                     int32_t xexp, uint16_t *Wh, uint16_t *Wl, int32_t dp, int32_t kp, float *c,
                                     double *w2, float *scal, void *ws, void *stream) {
    SOMB_REQUIRE(K > 0 && d > 0 && dp >= d && dp % 8 == 0 && kp >= K && kp % 256 == 0,
                 SOMB_E_INPUT, "codebook_prepare: bad shape K=%d d=%d dp=%d kp=%d", K, d, dp, kp);
    cudaStream_t st = as_stream(stream);
    char *p = (char *)ws;
    float *mu = (float *)p;            p += align_up((size_t)d * sizeof(float), 256);
    double *mu_nu = (double *)p;       p += align_up((size_t)d * sizeof(double), 256);
    float *nrm = (float *)p;           p += align_up((size_t)K * sizeof(float), 256);
    float *stats = (float *)p;
    cudaMemsetAsync(stats, 0, 8 * sizeof(float), st);
    cb_colmean<<<(d + 7) / 8, 256, 0, st>>>(W, K, d, nu, mu, mu_nu);
    note_launch();
    cb_rowstats<<<(K + 7) / 8, 256, 0, st>>>(W, K, d, mu, mu_nu, c, w2, nrm, stats);
    note_launch();
    cb_pack<<<(kp + 7) / 8, 256, 0, st>>>(W, K, d, mu, xexp, (__half *)Wh, (__half *)Wl, dp, kp, c, stats, scal,
                                          nullptr);
    // (Wh may be NULL: the sparse path screens against a transposed fp32 copy)
    note_launch();
    SOMB_LAUNCH_CHECK("somb_codebook_prepare");
    return SOMB_OK;
}

extern "C" int somb_data_pack_f8(const float *X, int64_t n, int32_t d, const float *nu, int32_t xexp, uint16_t *Xh,
                                 uint8_t *X8, int32_t dp, float *xnorm, double *x2, float *xstat, void *stream) {
    SOMB_REQUIRE(d > 0 && dp >= d && dp % 8 == 0 && Xh && X8, SOMB_E_INPUT, "data_pack_f8: bad pitch d=%d dp=%d", d,
                 dp);
    if (n == 0) return SOMB_OK;
    int64_t blocks = (n + 7) / 8;
    data_pack_f8_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(X, n, d, nu, xexp, (__half *)Xh, X8, dp,
                                                                         xnorm, x2, reinterpret_cast<float4 *>(xstat));
    note_launch();
    SOMB_LAUNCH_CHECK("somb_data_pack_f8");
    return SOMB_OK;
}

extern "C" int somb_codebook_prepare_f8(const float *W, int32_t K, int32_t d, const float *nu, int32_t xexp,
                                        uint16_t *Wh, uint8_t *W8, int32_t dp, int32_t kp, float *c, double *w2,
                                        float *scal, void *ws, void *stream) {
    SOMB_REQUIRE(K > 0 && d > 0 && dp >= d && dp % 8 == 0 && kp >= K && kp % 256 == 0 && Wh && W8,
                 SOMB_E_INPUT, "codebook_prepare_f8: bad shape K=%d d=%d dp=%d kp=%d", K, d, dp, kp);
    cudaStream_t st = as_stream(stream);
    char *p = (char *)ws;
    float *mu = (float *)p;            p += align_up((size_t)d * sizeof(float), 256);
    double *mu_nu = (double *)p;       p += align_up((size_t)d * sizeof(double), 256);
    float *nrm = (float *)p;           p += align_up((size_t)K * sizeof(float), 256);
    float *stats = (float *)p;
    cudaMemsetAsync(stats, 0, 8 * sizeof(float), st);
    cb_colmean<<<(d + 7) / 8, 256, 0, st>>>(W, K, d, nu, mu, mu_nu);
    note_launch();
    cb_rowstats<<<(K + 7) / 8, 256, 0, st>>>(W, K, d, mu, mu_nu, c, w2, nrm, stats);
    note_launch();
    cb_pack<<<(kp + 7) / 8, 256, 0, st>>>(W, K, d, mu, xexp, (__half *)Wh, nullptr, dp, kp, c, stats, scal, W8);
    note_launch();
    SOMB_LAUNCH_CHECK("somb_codebook_prepare_f8");
    return SOMB_OK;
}
