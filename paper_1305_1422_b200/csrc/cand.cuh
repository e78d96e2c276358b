// Per-row screening-window candidate set.
//
// A thread owns one data row and visits nodes j in ascending order with
// screened values r_j.  It keeps every j with r_j <= rmin + win (rmin =
// running minimum, win = the row's screening window).  If more than CAP
// nodes fall inside the window, the set is cut to the CAP/2 smallest
// (r, j) pairs in lexicographic order and a cap (capv) is installed: later
// nodes are accepted only with r < capv (their j is larger than every held
// index, so (r, j) < (capv, capi) <=> r < capv).  The final set is thus
// "all nodes within the window, or, when truncated, the smallest screened
// pairs", deterministic for a fixed visiting order, and always holds the
// lowest indices among exact screened ties.  Exact fp64 re-ranking of this
// set (rerank kernel) picks the BMU with first-minimum ties
// (kernels.py:27-28, 203).
#pragma once
#include <float.h>

#include "common.cuh"

namespace somb {

template <int CAP>
struct CandRow {
    float rmin, thr, capbelow, win;
    int cnt;
    int trunc;
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
}

// Slot e of the thread's buffer lives at [e * stride] (stride = #threads
// sharing the buffer array: conflict-free when lanes touch the same slot).
template <int CAP>
__device__ __noinline__ void cand_make_room(CandRow<CAP> &s, float *bv, int *bi, int stride) {
    const float lim = s.rmin + s.win;
    int m = 0;
    for (int e = 0; e < s.cnt; ++e) {
        float v = bv[e * stride];
        int ix = bi[e * stride];
        if (v <= lim) {
            bv[m * stride] = v;
            bi[m * stride] = ix;
            ++m;
        }
    }
    s.cnt = m;
    if (m < CAP) return;
    // Full inside the window: keep the CAP/2 smallest (value, index) pairs.
    static_assert(CAP <= 64, "keep mask is 64 bits");
    constexpr int H = CAP / 2;
    float capv = -INFINITY;
    unsigned long long keep = 0ull;
    for (int e = 0; e < CAP; ++e) {
        float v = bv[e * stride];
        int ix = bi[e * stride];
        int rank = 0;
        for (int f = 0; f < CAP; ++f) {
            float u = bv[f * stride];
            int iu = bi[f * stride];
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
            bv[m * stride] = bv[e * stride];
            bi[m * stride] = bi[e * stride];
            ++m;
        }
    }
    s.cnt = m;
    s.trunc = 1;
    s.capbelow = fminf(s.capbelow, nextafterf(capv, -INFINITY));
    s.thr = fminf(s.rmin + s.win, s.capbelow);
}

template <int CAP>
__device__ __forceinline__ void cand_push(CandRow<CAP> &s, float r, int j, float *bv, int *bi,
                                          int stride) {
    if (r <= s.thr) {
        if (r < s.rmin) {
            s.rmin = r;
            s.thr = fminf(r + s.win, s.capbelow);
        }
        if (s.cnt == CAP) cand_make_room<CAP>(s, bv, bi, stride);
        if (r <= s.thr) {
            bv[s.cnt * stride] = r;
            bi[s.cnt * stride] = j;
            ++s.cnt;
        }
    }
}

// Final filter: write { held j : r_j <= rmin + win } in index order.
template <int CAP>
__device__ __forceinline__ int cand_emit(const CandRow<CAP> &s, const float *bv, const int *bi,
                                         int stride, int *out) {
    const float lim = s.rmin + s.win;
    int m = 0;
    for (int e = 0; e < s.cnt; ++e)
        if (bv[e * stride] <= lim) out[m++] = bi[e * stride];
    return m;
}

}  // namespace somb
