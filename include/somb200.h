/*
 * somb200 -- C ABI of the B200-native batch-SOM epoch hot path.
 *
 * Every entry point takes DEVICE pointers, enqueues its work on `stream`
 * (a cudaStream_t passed as void*), never allocates, never synchronises the
 * host, and returns SOMB_OK or a SOMB_E_* status (message: somb_last_error()).
 * Status -> reference exception family (errors.py): SOMB_E_CONFIG ->
 * InvalidConfig (exit 1), SOMB_E_INPUT -> InputError/DimensionMismatch
 * (exit 2), SOMB_E_CUDA / SOMB_E_ARCH -> SomkitError (exit 3).
 *
 * The reference (somkit, pure Python + numpy/OpenBLAS) has no FFI of its
 * own; each function below cites the reference routine it replaces
 * (paths relative to /root/reference/pkg/src/somkit/).  INTEGRATION.md shows
 * the ctypes binding a somkit maintainer would add.
 *
 * Layouts (HBM): X f32 [n][d] row-major; CSR (int64 offsets, int32 sorted
 * cols, f32 vals); codebook W f32 [K][d], K = n_columns*n_rows, flat
 * row-major node order (kernels.py:89-96); fp16 screening copies use a row
 * pitch dp = round_up(d, 8) and K padded to kp = round_up(K, 256).
 */
#ifndef SOMB200_H
#define SOMB200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SOMB_API __attribute__((visibility("default")))
#else
#define SOMB_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define SOMB_OK 0
#define SOMB_E_CONFIG 1
#define SOMB_E_INPUT 2
#define SOMB_E_CUDA 3
#define SOMB_E_ARCH 4

#define SOMB_GRID_RECT 0      /* grid.py lattice (reference)            */
#define SOMB_GRID_HEX 1       /* extension: offset-row hexagonal         */
#define SOMB_PLANAR 0         /* grid.py:15-17                           */
#define SOMB_TOROID 1
#define SOMB_NBH_GAUSSIAN 0   /* exp(-d/r), train.py:138-144             */
#define SOMB_NBH_BUBBLE 1     /* extension: 1 if d <= r                  */
#define SOMB_DIST_BLOCKED 1   /* d2 = -2x.w + |x|^2 + |w|^2 (kernels.py:195-205) */
#define SOMB_DIST_NAIVE 0     /* d2 = sum (w - x)^2       (kernels.py:182-192) */

typedef struct somb_map {
    int32_t n_columns, n_rows;  /* x extent, y extent                    */
    int32_t grid;               /* SOMB_GRID_*                           */
    int32_t topology;           /* SOMB_PLANAR / SOMB_TOROID             */
} somb_map;

typedef struct somb_hood {
    int32_t neighborhood;       /* SOMB_NBH_*                            */
    int32_t compact;            /* 1: h = 0 beyond radius (extension)    */
    double radius;              /* epoch radius (train.py:209-217)       */
    double cutoff;              /* h < cutoff -> 0 (kernels.py:146-147)  */
    int32_t method;             /* SOMB_CONV_*: 0 auto, 1 direct, 2 spectral */
    int32_t reserved;
} somb_hood;

#define SOMB_CONV_AUTO 0
#define SOMB_CONV_DIRECT 1      /* fp64 sum over occupied nodes, O(K^2 D)   */
#define SOMB_CONV_SPECTRAL 2    /* fp64 DFT along x + per-frequency GEMM    */

/* Screening parameters of the tensor-core BMU search. */
#define SOMB_CAND_CAP 64        /* candidates kept per row (2 x 32 column groups) */

SOMB_API const char *somb_version(void);
SOMB_API const char *somb_last_error(void);
/* Tuning / profiling knobs of the tcgen05 screen, settable at run time
 * (defaults shown; the same names upper-cased with a SOMB_ prefix are read
 * from the environment once): "screen_lag" 8 (soft lockstep lag in node
 * tiles, 0 = off), "half_cap" 32 (candidates per row and column group kept
 * in shared memory before spilling), "tc_group" 2 (CTA-pair MMA; 1 = single
 * CTA), "tc_multicast" 2 (1-pass screen in 4-CTA clusters whose two pairs
 * share each codebook tile by TMA multicast; 1 = pairs only), "screen_profile" 0 (1 = skip the epilogue: times the TMA + MMA feed
 * alone; results are invalid), "ovf_chunks" 0 (> 0 caps the usable
 * overflow-pool chunks -- a test hook for the pool-exhaustion path, where a
 * full row keeps its lowest screened candidates and is flagged truncated).
 * Returns SOMB_E_CONFIG for unknown keys. */
SOMB_API int somb_set_knob(const char *key, int32_t value);
/* 0 if device `dev` is sm_100 (B200) and the library's kernels load. */
SOMB_API int somb_device_check(int dev);

/* ---- dense dataset, once per dataset ---------------------------------
 * nu = per-feature mean of X (fp64 fixed-order sum, rounded to f32), the
 * data-side centring of the screen.  Replaces: nothing (the reference
 * screens in fp64 directly); enables kernels.py:195-205 on fp16 tensor
 * cores.  ws: >= somb_data_stats_ws(d) bytes. */
SOMB_API size_t somb_data_stats_ws(int32_t d);
SOMB_API int somb_data_stats(const float *X, int64_t n, int32_t d, float *nu,
                    float *absmax /* [1] max|x - nu| */, void *ws, void *stream);
/* Xh[i][k] = fp16((x_ik - nu_k) * 2^xexp) (pitch dp, zero pad), rounded
 * stochastically (dither hashed from (i, k, value bits)); Xl (may be NULL)
 * = fp16 residual of a round-to-nearest hi (enables the 3-pass screen);
 * xnorm[i] = |x_i - nu|_2 (f32); x2[i] = |x_i|^2 in fp64 (kernels.py:198);
 * xstat[i] (f32 x 4) = {|x'_i|, max_k |x'_ik|, max_k ulp_ik, |ulp_i|_2}, the
 * row terms of the screening window sigma_i (ulp_ik = the span of the
 * stochastic rounding of feature k, unscaled). */
SOMB_API int somb_data_pack(const float *X, int64_t n, int32_t d, const float *nu,
                   int32_t xexp, uint16_t *Xh, uint16_t *Xl, int32_t dp, float *xnorm,
                   double *x2, float *xstat, void *stream);

/* ---- codebook, once per epoch ----------------------------------------
 * mu = mean_j W_j; delta_j = W_j - mu (exact in fp64); Wh = fp16(delta *
 * 2^s) with s picked on device from max|delta|; c_j = |delta_j|^2 +
 * 2 (mu - nu).delta_j (f32, +inf on padding and duplicate rows);
 * w2_j = |w_j|^2 fp64 (kernels.py:389-390); scal[0..3] = {m, nmax, ...}
 * device scalars consumed by somb_bmu_dense.  ws >= somb_codebook_ws(K, d). */
SOMB_API size_t somb_codebook_ws(int32_t K, int32_t d);
SOMB_API int somb_codebook_prepare(const float *W, int32_t K, int32_t d, const float *nu,
                          int32_t xexp, uint16_t *Wh, uint16_t *Wl, int32_t dp, int32_t kp,
                          float *c, double *w2, float *scal, void *ws,
                          void *stream);

/* ---- codebook initialisation (train.py:164-166) ----------------------
 * out[i] = numpy.random.default_rng(seed).random(count, dtype=float32)[i],
 * bit for bit: PCG64 with the 128-bit state/increment numpy derives from
 * the seed (numpy.random.PCG64(seed).state), XSL-RR output, float i from the
 * 32-bit half i%2 of 64-bit output i/2, (u >> 8) * 2^-24. */
SOMB_API int somb_uniform_f32(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                              int64_t count, float *out, void *stream);

/* 2-pass split screen operands (screen_impl 3): the fp16 hi copy plus the
 * fp8 (e4m3) cross-term operands, 2 dp bytes per row -- X8 = [e4m3(xh / 32)
 * | e4m3(xl * 32)], W8 = [e4m3(wl * 32) | e4m3(wh / 32)] with xl, wl the
 * fp16 residuals; scaling puts max|hi| <= 2^13 (xexp = 13 - exponent of
 * max|x - nu|).  The tensor-core screen computes hi.hi (kind::f16) +
 * x_hi8.w_lo8 + x_lo8.w_hi8 (kind::f8f6f4, twice the fp16 rate). */
SOMB_API int somb_data_pack_f8(const float *X, int64_t n, int32_t d, const float *nu, int32_t xexp,
                               uint16_t *Xh, uint8_t *X8, int32_t dp, float *xnorm, double *x2, float *xstat,
                               void *stream);
SOMB_API int somb_codebook_prepare_f8(const float *W, int32_t K, int32_t d, const float *nu, int32_t xexp,
                                      uint16_t *Wh, uint8_t *W8, int32_t dp, int32_t kp, float *c,
                                      double *w2, float *scal, void *ws, void *stream);

/* ---- BMU search (kernels.py:195-205 / 182-192, :407) -----------------
 * fp16 tensor-core screen (tcgen05, TMEM accumulators, TMA-staged tiles)
 * keeping per row every node within the screening window (<= CAP, the
 * lowest screened values when truncated), then an exact fp64 re-rank of
 * the candidates with the reference formula `dist_mode`, first-minimum
 * ties.  Output bmu int32[n], d2min fp64[n] (clamped >= 0), flags int32[n]
 * (bit0 = window truncated).  ws >= somb_bmu_ws(n).  screen_impl: 0 =
 * tcgen05 (sm_100a), 1 = SIMT reference screen (tests), 2 = none (exact
 * scan), 3 = tcgen05 2-pass split (Xl / Wl = the fp8 operands of
 * somb_data_pack_f8 / somb_codebook_prepare_f8). */
SOMB_API int somb_bmu_dense(const uint16_t *Xh, const float *X, const float *xstat,
                   const double *x2, int64_t n, int32_t d, int32_t dp,
                   const uint16_t *Wh, const float *W, const float *c,
                   const double *w2, int32_t K, int32_t kp, const float *scal,
                   float window_coef, int32_t dist_mode, int32_t screen_impl,
                   int32_t *bmu, double *d2min, int32_t *flags, void *ws,
                   void *stream);

/* The two phases of somb_bmu_dense, separately (per-kernel timing):
 * screen -> ws candidate lists; re-rank -> bmu / d2min. */
SOMB_API size_t somb_bmu_ws(int64_t n);
/* prev_bmu (may be NULL): each row's BMU from the previous search; seeds the
 * screening threshold (does not change the result, only the work). */
/* Xl / Wl (both non-NULL): 3-pass split screen hi.hi + hi.lo + lo.hi. */
SOMB_API int somb_bmu_screen(const uint16_t *Xh, const uint16_t *Xl, const float *xstat, int64_t n,
                             int32_t dp, const uint16_t *Wh, const uint16_t *Wl, const float *c,
                             int32_t K, int32_t kp, const float *scal,
                             float window_coef, const int32_t *prev_bmu,
                             int32_t screen_impl, int32_t *flags, void *ws,
                             void *stream);
/* Rows of the last somb_bmu_screen / somb_bmu_sparse whose candidate set
 * was truncated (overflow pool exhausted) and therefore re-ranked by an
 * exact scan of every node instead (the result stays the reference's
 * argmin).  Reads a device counter in ws: synchronises `stream`; -1 on a
 * CUDA error. */
SOMB_API int64_t somb_bmu_repaired_rows(const void *ws, int64_t n, void *stream);
/* Calibration: tcgen05 screened values of rows [0, min(n,128)) x kp nodes. */
SOMB_API int somb_debug_screen_dump(const uint16_t *Xh, const uint16_t *Xl, const float *xstat,
                                    int64_t n, int32_t dp, const uint16_t *Wh, const uint16_t *Wl,
                                    const float *c, int32_t kp, const float *scal,
                                    float window_coef, int32_t passes, float *dump, void *ws,
                                    void *stream);
/* row_order (may be NULL): a permutation of [0, n) giving the order in
 * which rows are re-ranked -- the rows sorted by their previous BMU
 * (somb_node_sums_* row_order), so concurrently re-ranked rows share
 * candidate codebook rows in L2.  Results do not depend on it. */
SOMB_API int somb_bmu_rerank(const float *X, const double *x2, int64_t n,
                             int32_t d, const float *W, const double *w2,
                             int32_t K, int32_t dist_mode, int32_t screen_impl,
                             const int32_t *row_order, int32_t *bmu, double *d2min,
                             int32_t *flags, void *ws, void *stream);

/* The whole BMU search in one call: somb_bmu_screen (seeded from
 * prev_bmu, may be NULL) + somb_bmu_rerank (visiting rows in row_order,
 * may be NULL).  ws >= somb_bmu_ws(n). */
SOMB_API int somb_bmu_search(const uint16_t *Xh, const uint16_t *Xl, const float *X, const float *xstat,
                             const double *x2, int64_t n, int32_t d, int32_t dp, const uint16_t *Wh,
                             const uint16_t *Wl, const float *W, const float *c, const double *w2,
                             int32_t K, int32_t kp, const float *scal, float window_coef,
                             const int32_t *prev_bmu, const int32_t *row_order, int32_t dist_mode,
                             int32_t screen_impl, int32_t *bmu, double *d2min, int32_t *flags,
                             void *ws, void *stream);

/* qe_sum = sum_i sqrt(d2min_i) in fixed order (kernels.py:407, 427). */
SOMB_API int somb_qe_sum(const double *d2min, int64_t n, double *out, void *ws,
                void *stream);

/* ---- batch update: node sums (BMU histogram + per-node data sums) ----
 * S_b = sum_{i: bmu_i = b} x_i in ascending i (fp64), cnt_b = |{i}|;
 * a stable device radix sort groups the rows.  Together with
 * somb_hood_update this replaces the accumulate of kernels.py:225-226
 * (num = H S, den = H cnt).  ws >= somb_node_sums_ws(n, K). */
SOMB_API size_t somb_node_sums_ws(int64_t n, int32_t d, int32_t K);
/* row_order (may be NULL): receives the rows stably sorted by BMU. */
SOMB_API int somb_node_sums_dense(const float *X, int64_t n, int32_t d,
                         const int32_t *bmu, int32_t K, double *S, double *cnt,
                         int32_t *row_order, void *ws, void *stream);
/* The same sums written column-block-major: S is [ceil(d/dc)][K][dc] fp64,
 * S[(k / dc)][b][k % dc] = S_bk (padding columns of the last block are 0),
 * 1 <= dc <= d.  With dc = ceil(d/P) rank r's feature-column block is one
 * contiguous [K][dc] slab: the multi-rank exchange reduce-scatters S in place
 * (replaces the MPI_Reduce of the numerators, distributed.py:492-514). */
SOMB_API int somb_node_sums_dense_cols(const float *X, int64_t n, int32_t d,
                                      const int32_t *bmu, int32_t K, int32_t dc, double *S,
                                      double *cnt, int32_t *row_order, void *ws, void *stream);

/* ---- batch update: neighbourhood convolution + blend ------------------
 * h(b, j) from grid offsets (kernels.py:99-150; hex/bubble/compact are
 * extensions), den_j = sum_b h cnt_b, num_j = sum_b h S_b (fp64), then for
 * nodes [node_begin, node_end): W_new_j = f32((1-scale) W_j + scale num_j /
 * den_j) if den_j > 0 else W_j bit-exact (kernels.py:438-450).
 * num_out / den_out (K x d / K, may be NULL) expose the accumulators for the
 * reference-compatible search_accumulate debug path.
 * dist_table (may be NULL): grid distance per wrapped offset [dy][dx]
 * (rect: n_rows x n_columns) -- the host passes numpy's hypot table so d is
 * bit-identical to kernels.py:112; NULL computes sqrt(dx^2 + dy^2).
 * ws >= somb_hood_ws(map, K). */
SOMB_API size_t somb_hood_ws(const somb_map *map, int32_t K, int32_t d);
SOMB_API int somb_hood_update(const double *S, const double *cnt, int32_t d,
                     const somb_map *map, const somb_hood *hood, double scale,
                     const double *dist_table,
                     const float *W_old, int32_t node_begin, int32_t node_end,
                     float *W_new, double *num_out, double *den_out, void *ws,
                     void *stream);

/* Standalone blend of given accumulators (kernels.py:438-450), same
 * arithmetic as the fused epilogue of somb_hood_update. */
SOMB_API int somb_blend(const float *W_old, const double *num, const double *den,
               int32_t K, int32_t d, double scale, float *W_new, void *stream);

/* ---- sparse (CSR) rows: kernels.py:208-222, 229-242, 315-321 ---------
 * Row stats: x2[i] = sum v^2 (fp64, nnz order), xnorm = sqrt(x2), nnz_max. */
SOMB_API int somb_sparse_row_stats(const int64_t *rowptr, const float *val, int64_t n,
                                   double *x2, float *xnorm, int32_t *nnz_max, void *stream);
/* dT[k][j] = fp32(w_jk - mu_k) (pitch kp, zero padding); mu = the codebook
 * mean written by somb_codebook_prepare into the first d floats of its ws. */
SOMB_API int somb_sparse_codebook_T(const float *W, const float *mu, int32_t K, int32_t d,
                                    int32_t kp, float *dT, void *stream);
/* fp32 gather screen over dT + exact fp64 sparse re-rank (exact = 1: scan
 * every node, no screen; exact = 2: screen, and leave the rows whose
 * candidate set was truncated to somb_bmu_sparse_repair).  ws >= somb_bmu_ws(n). */
SOMB_API int somb_bmu_sparse(const int64_t *rowptr, const int32_t *col, const float *val,
                             int64_t n, int32_t d, const float *dT, const float *W,
                             const float *c, const double *w2, int32_t K, int32_t kp,
                             const float *scal, const double *x2, const float *xnorm,
                             float window_coef, int32_t exact, int32_t *bmu,
                             double *d2min, int32_t *flags, void *ws, void *stream);
/* After somb_bmu_sparse(exact = 2) on the same ws: the exact BMU of every
 * row whose candidate set was truncated, by a slab-lockstep fp64 scan of all
 * nodes over the ORIGINAL codebook transposed into `WT` (d x kp f32 scratch,
 * e.g. the screen's dT buffer once the screen is done; written only when a
 * row was repaired); the reference's sparse formula (kernels.py:216-219),
 * first-minimum ties (kernels.py:27-28). */
SOMB_API int somb_bmu_sparse_repair(const int64_t *rowptr, const int32_t *col, const float *val,
                                    int64_t n, int32_t d, const float *W, int32_t K, int32_t kp,
                                    const double *w2, const double *x2, float *WT, int32_t *bmu,
                                    double *d2min, void *ws, void *stream);
/* S (K x d, fp64, dense) / cnt from CSR rows; ws >= somb_node_sums_ws(n, d, K).
 * Nodes with more than 2048 rows are summed in 2048-row segments folded in
 * segment order (the dense path's scheme), else in ascending row order. */
/* Workspace of somb_bmu_sparse (the lockstep screen keeps each row's window
 * state and candidate buffer between codebook slabs). */
SOMB_API size_t somb_bmu_sparse_ws(int64_t n);
SOMB_API int somb_node_sums_sparse(const int64_t *rowptr, const int32_t *col,
                                   const float *val, int64_t n, int32_t d,
                                   const int32_t *bmu, int32_t K, double *S,
                                   double *cnt, int32_t *row_order, void *ws, void *stream);
/* Column-block-major S as somb_node_sums_dense_cols. */
SOMB_API int somb_node_sums_sparse_cols(const int64_t *rowptr, const int32_t *col,
                                       const float *val, int64_t n, int32_t d,
                                       const int32_t *bmu, int32_t K, int32_t dc, double *S,
                                       double *cnt, int32_t *row_order, void *ws, void *stream);

/* Number of kernels this library has launched (process lifetime). */
SOMB_API unsigned long long somb_launch_count(void);

/* Diagnostics: L2 read-bandwidth probe -- `reps` passes of float4 loads over
 * buf[0, n) (n floats, L2-resident size), enqueued on `stream`; out holds one
 * float per block (4 x SM count).  Times the achievable L2 read rate that
 * bench.py uses as the roofline of the L2-bound kernels (no reference
 * counterpart). */
SOMB_API int somb_l2_probe(const float *buf, int64_t n, int32_t reps, float *out, void *stream);

/* ---- artifact text (fileio.py:322-359), host code, no GPU needed --------
 * The reference's Python formatting f"{float(v):.6g}", space-separated,
 * one row per line; BMU lines "i row col".  Formats into `out` (capacity
 * `cap` bytes) on `threads` host threads and returns the byte count, or
 * -(bytes needed) if `cap` is too small. */
SOMB_API int64_t somb_format_f32_rows(const float *v, int64_t rows, int64_t cols, char *out, int64_t cap,
                                      int32_t threads);
SOMB_API int64_t somb_format_bmus(const int32_t *bm, int64_t n, char *out, int64_t cap, int32_t threads);
/* Dense text ingest (fileio.py:150-229), host code: scan (data rows, columns
 * of the first data row, '%' header lines, first width-mismatch line), then
 * parse into row-major f32 on `threads` threads (tokens as double, rounded
 * to f32).  The parse returns 0 or the line number of the first row needing
 * the reference-exact error path. */
SOMB_API int64_t somb_scan_dense_text(const char *buf, int64_t len, int64_t *cols, int64_t *n_headers,
                                      int64_t *bad_line);
SOMB_API int64_t somb_parse_dense_text(const char *buf, int64_t len, int64_t rows, int64_t cols, float *out,
                                       int32_t threads);

/* ---- U-matrix (umatrix.py:26-45; hex adjacency = extension) ---------- */
SOMB_API int somb_umatrix(const float *W, int32_t d, const somb_map *map, float *U,
                 void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SOMB200_H */
