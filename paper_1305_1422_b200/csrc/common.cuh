// Shared helpers for the somb200 kernels (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "../../include/somb200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "somb200 targets sm_100a only"
#endif

namespace somb {

void set_error(const char *fmt, ...);
void note_launch();   // kernel-launch counter (somb_launch_count)

static inline int cuda_status(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return SOMB_OK;
    set_error("%s: %s", what, cudaGetErrorString(e));
    return SOMB_E_CUDA;
}

#define SOMB_LAUNCH_CHECK(what)                                           \
    do {                                                                  \
        cudaError_t _e = cudaGetLastError();                              \
        if (_e != cudaSuccess) return ::somb::cuda_status(_e, what);      \
    } while (0)

#define SOMB_REQUIRE(cond, code, ...)                                     \
    do {                                                                  \
        if (!(cond)) { ::somb::set_error(__VA_ARGS__); return code; }     \
    } while (0)

static inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }
static inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

constexpr int kSmCount = 148;

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// float max via int compare (valid for non-negative floats)
__device__ __forceinline__ void atomic_max_nonneg(float *addr, float v) {
    atomicMax(reinterpret_cast<int *>(addr), __float_as_int(v));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Node sums S in column-block-major layout [ceil(d/dc)][K][dc] (dc = d: the
// plain row-major [K][d]): each rank's feature-column block of S is
// contiguous, so the multi-rank reduce-scatter reads S in place.
__host__ __device__ __forceinline__ int64_t s_index(int b, int k, int dc, int K) {
    const int blk = k / dc;
    return ((int64_t)blk * K + b) * dc + (k - blk * dc);
}
inline size_t s_blocks_size(int d, int dc, int K) { return (size_t)((d + dc - 1) / dc) * K * dc; }

// ---------------------------------------------------------------- grid
// Node j sits at (col, row) = (j % nx, j / nx) (kernels.py:89-96).
// Squared grid distance between two nodes, exact in fp64:
//  rect: dx^2 + dy^2 with per-axis toroid min-wrap (kernels.py:107-112);
//  hex (extension): x = col + (row & 1)/2, y = row * sqrt(3)/2, so
//  d^2 = dx^2 + 0.75 dr^2 with per-axis min-wrap on the (nx, ny sqrt3/2)
//  period lattice (even ny).
struct MapDev {
    int nx, ny, hex, toroid;
};

__device__ __forceinline__ double grid_d2(const MapDev &m, int a, int b) {
    int ca = a % m.nx, ra = a / m.nx, cb = b % m.nx, rb = b / m.nx;
    if (!m.hex) {
        int dx = abs(ca - cb), dy = abs(ra - rb);
        if (m.toroid) { dx = min(dx, m.nx - dx); dy = min(dy, m.ny - dy); }
        return (double)dx * dx + (double)dy * dy;
    }
    int dx2 = abs((2 * ca + (ra & 1)) - (2 * cb + (rb & 1)));   // 2*dx
    int dr = abs(ra - rb);
    if (m.toroid) { dx2 = min(dx2, 2 * m.nx - dx2); dr = min(dr, m.ny - dr); }
    return 0.25 * (double)dx2 * dx2 + 0.75 * (double)dr * dr;
}

}  // namespace somb
