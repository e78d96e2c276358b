// Shared pieces of the exact fp64 re-rank kernels (bmu.cu):
// the candidate-list layout written by the screens, the overflow-pool view,
// cp.async helpers and the XU-free fp32 -> fp64 conversion.
#pragma once
#include "cand.cuh"

namespace somb {

// Spilled candidates of one row (tcgen05 screen overflow lists), read by the re-rank.
struct OvfView {
    const int *head;    // [4n] per (row, column group), nullptr = no overflow lists
    const float *lim;   // [4n] final window limit of each column group
    const int2 *ent;
    const int *next, *cnt;
    const unsigned *ngp;   // column groups of the tcgen05 lists (written by the screen)
};

// Candidate list of a row: one segment (SIMT screen) or NG column-group
// segments (tcgen05 screen: count byte g, slots [g * 64 / NG, ...)).
struct CandLayout {
    int c[4];
    int ng, gs, cnt;
};
// ccount sentinel written by the truncation repair (bmu.cu): the row's
// candidate set was cut, so the re-rank scans every node.  An EMPTY list is
// different: all of the row's candidates may sit in spilled overflow chunks.
constexpr int kScanAll = -1;

__device__ __forceinline__ CandLayout cand_layout(int cc, int split, int ng) {
    CandLayout L;
    if (cc == kScanAll) {
        L.ng = 1; L.gs = SOMB_CAND_CAP; L.c[0] = L.c[1] = L.c[2] = L.c[3] = 0; L.cnt = -1;
        return L;
    }
    if (!split) {
        L.ng = 1; L.gs = SOMB_CAND_CAP; L.c[0] = cc; L.c[1] = L.c[2] = L.c[3] = 0; L.cnt = cc;
        return L;
    }
    L.ng = ng; L.gs = SOMB_CAND_CAP / ng; L.cnt = 0;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        L.c[g] = g < ng ? (cc >> (8 * g)) & 255 : 0;
        L.cnt += L.c[g];
    }
    return L;
}
// does the row have spilled overflow chunks (tcgen05 lists)?
__device__ __forceinline__ bool row_has_ovf(const OvfView &ov, int64_t row) {
    if (ov.head == nullptr) return false;
    const int4 h = *reinterpret_cast<const int4 *>(ov.head + 4 * row);
    return h.x >= 0 || h.y >= 0 || h.z >= 0 || h.w >= 0;
}

// exact scan of every node: repaired rows, or (defensively) a row with no
// candidate at all
__device__ __forceinline__ bool cand_scan_all(const CandLayout &L, const OvfView &ov, int64_t row) {
    return L.cnt < 0 || (L.cnt == 0 && !row_has_ovf(ov, row));
}

__device__ __forceinline__ int cand_slot(const CandLayout &L, int q) {
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        if (q < L.c[g]) return g * L.gs + q;
        q -= L.c[g];
    }
    return 0;
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// fp32 -> fp64 without the XU pipe: the fp32 bit pattern re-read as an fp64
// with the same exponent field is exactly w * 2^-896 (normal, subnormal and
// zero alike); the 2^896 goes into the other operand, so every product and
// difference below is bit-identical to the (double)w form.  3 ALU ops + 1
// shift instead of one F2F.F64.F32, which issues at 1/8 warp-rate (it was the
// busiest pipe of the re-rank; profiles/).  Inf / NaN codebook entries are not
// preserved (they are finite garbage here, as anywhere after such an update).
__device__ __forceinline__ double f32_as_f64_scaled(float v) {
    const unsigned u = __float_as_uint(v);
    return __hiloint2double((int)(((u & 0x7FFFFFFFu) >> 3) | (u & 0x80000000u)), (int)(u << 29));
}
constexpr double kF64Scale = 0x1p896;

}  // namespace somb
