// Per-row screening-window candidate set.
//
// A thread owns one data row and visits nodes j in ascending order with
// screened values r_j.  It keeps every j with r_j <= rmin + win (rmin =
// running minimum, win = the row's screening window).  If more than CAP
// nodes fall inside the window, the full buffer is spilled to a global
// overflow pool (when one is given and has room), so the set stays complete.
// Otherwise the set is cut to the 3 CAP/4 smallest
// (r, j) pairs in lexicographic order and a cap (capv) is installed: later
// nodes are accepted only with r < capv (their j is larger than every held
// index, so (r, j) < (capv, capi) <=> r < capv).  The final set is thus
// "all nodes within the window, or, when truncated, the smallest screened
// pairs", deterministic for a fixed visiting order, and always holds the
// lowest indices among exact screened ties.  Exact fp64 re-ranking of this
// set (rerank kernel) picks the BMU with first-minimum ties
// (kernels.py:27-28, 203).
//
// The acceptance threshold `thr` may additionally be lowered by any value
// the sweep is guaranteed to meet (cand_bound): a chunk's minimum before its
// elements are pushed, or a seed from the row's previous BMU.  That only
// removes transient entries that the final filter would drop anyway.
//
// Buffers live in shared memory and are addressed with 32-bit shared-window
// addresses (slot e of a thread at base + e * stride bytes).
#pragma once
#include <float.h>

#include "common.cuh"

namespace somb {

__device__ __forceinline__ float lds_f32(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ int lds_s32(uint32_t a) {
    int v;
    asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_f32(uint32_t a, float v) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void sts_s32(uint32_t a, int v) {
    asm volatile("st.shared.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

struct CandBuf {
    uint32_t v, i;      // shared addresses of this thread's slot 0 (values, indices)
    uint32_t stride;    // bytes between slots
};
__device__ __forceinline__ float cb_ldv(const CandBuf &b, int e) { return lds_f32(b.v + e * b.stride); }
__device__ __forceinline__ int cb_ldi(const CandBuf &b, int e) { return lds_s32(b.i + e * b.stride); }
__device__ __forceinline__ void cb_st(const CandBuf &b, int e, float v, int j) {
    sts_f32(b.v + e * b.stride, v);
    sts_s32(b.i + e * b.stride, j);
}

// Overflow pool (optional): when a buffer is full of in-window entries it is
// spilled as one chunk (<= 32 entries) into a global pool and the row keeps
// collecting, so the candidate set stays complete; each (row, group) keeps a
// linked list of its chunks.  Only when the pool is exhausted does the set
// fall back to truncation.  The re-rank filters spilled entries with the
// group's final window limit.
constexpr int kOvfChunk = 32;
struct OvfPool {
    int2 *ent;          // [nchunks][kOvfChunk] (value bits, node)
    int *next;          // [nchunks] next chunk of the same list, -1 = end
    int *cnt;           // [nchunks] entries used
    unsigned *ctr;      // chunks allocated so far
    unsigned nchunks;   // 0 = no pool (truncate when full)
};

// BMU workspace (bmu.cu): cand [n][CAP] int | ccount [n] int | thr0 [n]
// float | counters | overflow: head [2n] int, lim [2n] float, next [C],
// cnt [C], entries [C][32] int2 with C = max(4096, 4 n) chunks.
struct BmuWs {
    int *cand, *ccount;
    float *thr0;
    unsigned *ctrs;     // [0] screen lockstep, [1] overflow chunks allocated
    int *ovf_head;
    float *ovf_lim;
    OvfPool pool;
};
BmuWs bmu_carve(void *ws, int64_t n, size_t *total = nullptr);

// The same buffer in global memory (one row's slots contiguous): lets a
// row's candidate state persist across kernel phases (sparse lockstep screen).
struct CandBufG {
    float *v;
    int *i;
};
__device__ __forceinline__ float cb_ldv(const CandBufG &b, int e) { return b.v[e]; }
__device__ __forceinline__ int cb_ldi(const CandBufG &b, int e) { return b.i[e]; }
__device__ __forceinline__ void cb_st(const CandBufG &b, int e, float v, int j) {
    b.v[e] = v;
    b.i[e] = j;
}

// Per-row scale sigma_i of the dense screen's error.  The
// fp16 operands are rounded stochastically (prep.cu), so the error of
// x~_i . delta~_j is a sum over features of independent mean-zero terms,
// sum_k e_ik delta_jk + x'_ik f_jk (+ e f), with |e_ik| < ulp_ik and
// |f_jk| < ulp(delta_jk).  Its Hoeffding scale
// sqrt(sum_k ulp_ik^2 delta_jk^2 + x'_ik^2 ulp(delta_jk)^2) is bounded per
// row, for every node j, by two Hoelder forms per term:
//   x side: min(max_k ulp_ik * max_j|delta_j|, |ulp_i|_2 * max_jk|delta_jk|)
//   delta side: min(max_k|x'_ik| * max_j|ulp(delta_j)|_2, |x'_i| * max ulp(delta))
// plus a 2^-20 slack for the fp32 rounding of c_j and of r~ (|r| <= |c| +
// 2 |x'| |delta|).  xs = xstat[row] = {|x'|, max|x'_k|, max ulp_k, |ulp|_2}
// (somb_data_pack); scal[1] = max_j|delta_j|, scal[3] = max_jk|delta_jk|,
// scal[4] = max|c_j|, scal[5] = max_j|ulp(delta_j)|_2, scal[6] = max ulp
// (somb_codebook_prepare).  The screening window of a row is
// window_coef * sigma_i (1-pass: 5, 2-pass fp8 cross terms: 0.5; engine.py).
__device__ __forceinline__ float screen_sigma(float4 xs, const float *__restrict__ scal) {
    const float sx = fminf(xs.z * scal[1], xs.w * scal[3]);
    const float sd = fminf(xs.y * scal[5], xs.x * scal[6]);
    return sqrtf(sx * sx + sd * sd) + ldexpf(scal[4] + 2.0f * xs.x * scal[1], -20);
}

template <int CAP>
struct CandRow {
    float rmin, thr, capbelow, win;
    int cnt;
    int trunc;          // bit 0: truncated (pool exhausted), bit 1: spilled
    int head;           // overflow chunk list, -1 = none
};

template <int CAP>
__device__ __forceinline__ void cand_init(CandRow<CAP> &s, float win) {
    // finite start: screened values of padding / masked nodes are +inf and
    // must never enter the set
    s.rmin = FLT_MAX;
    s.thr = FLT_MAX;
    s.capbelow = FLT_MAX;
    s.win = win;
    s.cnt = 0;
    s.trunc = 0;
    s.head = -1;
}

template <int CAP>
__device__ __forceinline__ void cand_bound(CandRow<CAP> &s, float r_seen) {
    s.thr = fminf(s.thr, r_seen + s.win);
}

// (by value in, by value out: a reference would take the address of the
// caller's CandRow and pin the whole row state to local memory for the
// entire screen sweep -- an LDL of st.thr per chunk)
template <int CAP, class Buf>
__device__ __noinline__ CandRow<CAP> cand_make_room(CandRow<CAP> s, Buf b, OvfPool pool) {
    const float lim = s.rmin + s.win;
    int m = 0;
    for (int e = 0; e < s.cnt; ++e) {
        float v = cb_ldv(b, e);
        int ix = cb_ldi(b, e);
        if (v <= lim) {
            cb_st(b, m, v, ix);
            ++m;
        }
    }
    s.cnt = m;
    if (m < CAP) return s;
    // Full inside the window: spill the buffer into the overflow pool ...
    if (CAP <= kOvfChunk && pool.nchunks) {   // (buffers larger than a chunk never spill)
        const unsigned c = atomicAdd(pool.ctr, 1u);
        if (c < pool.nchunks) {
            int2 *dst = pool.ent + (size_t)c * kOvfChunk;
            for (int e = 0; e < (CAP < kOvfChunk ? CAP : kOvfChunk); ++e) dst[e] = make_int2(__float_as_int(cb_ldv(b, e)), cb_ldi(b, e));
            pool.cnt[c] = CAP;
            pool.next[c] = s.head;
            s.head = (int)c;
            s.cnt = 0;
            s.trunc |= 2;
            return s;
        }
    }
    // ... or, without room there, keep the 3 CAP / 4 smallest (value, index) pairs.
    static_assert(CAP <= 64, "keep mask is 64 bits");
    constexpr int H = 3 * CAP / 4;
    float capv = -INFINITY;
    unsigned long long keep = 0ull;
    for (int e = 0; e < CAP; ++e) {
        float v = cb_ldv(b, e);
        int ix = cb_ldi(b, e);
        int rank = 0;
        for (int f = 0; f < CAP; ++f) {
            float u = cb_ldv(b, f);
            int iu = cb_ldi(b, f);
            rank += (u < v) || (u == v && iu < ix);
        }
        if (rank < H) {
            keep |= 1ull << e;
            capv = fmaxf(capv, v);
        }
    }
    m = 0;
    for (int e = 0; e < CAP; ++e) {
        if (keep >> e & 1ull) {
            cb_st(b, m, cb_ldv(b, e), cb_ldi(b, e));
            ++m;
        }
    }
    s.cnt = m;
    s.trunc |= 1;
    s.capbelow = fminf(s.capbelow, nextafterf(capv, -INFINITY));
    s.thr = fminf(s.thr, s.capbelow);
    return s;
}

template <int CAP, class Buf>
__device__ __forceinline__ void cand_push(CandRow<CAP> &s, float r, int j, const Buf &b,
                                          const OvfPool &pool = OvfPool{nullptr, nullptr, nullptr, nullptr, 0u}) {
    if (r <= s.thr) {
        if (r < s.rmin) {
            s.rmin = r;
            s.thr = fminf(s.thr, r + s.win);
        }
        if (s.cnt == CAP) s = cand_make_room<CAP>(s, b, pool);
        if (r <= s.thr) {
            cb_st(b, s.cnt, r, j);
            ++s.cnt;
        }
    }
}

// Final filter: write { held j : r_j <= rmin + win } in index order.
template <int CAP, class Buf>
__device__ __forceinline__ int cand_emit(const CandRow<CAP> &s, const Buf &b, int *out) {
    const float lim = s.rmin + s.win;
    int m = 0;
    for (int e = 0; e < s.cnt; ++e)
        if (cb_ldv(b, e) <= lim) out[m++] = cb_ldi(b, e);
    return m;
}

}  // namespace somb
