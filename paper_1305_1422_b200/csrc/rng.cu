// numpy-compatible codebook initialisation on the device.
//
// The reference initialises the codebook with
// numpy.random.default_rng(seed).random((K, D), dtype=float32)
// (train.py:164-166): PCG64 (128-bit LCG, XSL-RR output), float i built from
// 32-bit half i%2 of 64-bit output i/2 (low half first) as
// (u >> 8) * 2^-24.  Generating 40M of them on the host costs ~0.25 s of the
// cfg2 end-to-end run; here every thread jumps the LCG to its own block of
// outputs (O(log n) advance) and writes the identical floats straight into
// the codebook buffer.
#include "common.cuh"

namespace somb {

struct U128 {
    uint64_t lo, hi;
};

__device__ __forceinline__ U128 mul128(U128 a, U128 b) {
    U128 r;
    r.lo = a.lo * b.lo;
    r.hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
    return r;
}

__device__ __forceinline__ U128 add128(U128 a, U128 b) {
    U128 r;
    r.lo = a.lo + b.lo;
    r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
    return r;
}

// PCG64 default multiplier (numpy pcg64.h PCG_DEFAULT_MULTIPLIER_128)
__device__ __constant__ U128 kPcgMult = {0x4385DF649FCCF645ull, 0x2360ED051FC65DA4ull};

// state after `delta` LCG steps (pcg_advance_lcg_128)
__device__ U128 pcg_advance(U128 state, uint64_t delta, U128 inc) {
    U128 acc_mult = {1ull, 0ull}, acc_plus = {0ull, 0ull};
    U128 cur_mult = kPcgMult, cur_plus = inc;
    while (delta) {
        if (delta & 1ull) {
            acc_mult = mul128(acc_mult, cur_mult);
            acc_plus = add128(mul128(acc_plus, cur_mult), cur_plus);
        }
        cur_plus = mul128(add128(cur_mult, U128{1ull, 0ull}), cur_plus);
        cur_mult = mul128(cur_mult, cur_mult);
        delta >>= 1;
    }
    return add128(mul128(acc_mult, state), acc_plus);
}

__device__ __forceinline__ uint64_t pcg_xsl_rr(U128 s) {
    const uint64_t v = s.hi ^ s.lo;
    const unsigned r = (unsigned)(s.hi >> 58);
    return (v >> r) | (v << ((64u - r) & 63u));
}

constexpr int kRngOuts = 8;   // 64-bit outputs (16 floats) per thread

__global__ void pcg64_uniform_f32(U128 s0, U128 inc, int64_t count, float *__restrict__ out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t k0 = t * kRngOuts;                  // first 64-bit output of this thread
    if (2 * k0 >= count) return;
    U128 s = pcg_advance(s0, (uint64_t)k0, inc);      // state before output k0
#pragma unroll
    for (int q = 0; q < kRngOuts; ++q) {
        s = add128(mul128(s, kPcgMult), inc);
        const uint64_t o = pcg_xsl_rr(s);
        const int64_t i = 2 * (k0 + q);
        if (i < count) out[i] = (float)((uint32_t)o >> 8) * (1.0f / 16777216.0f);
        if (i + 1 < count) out[i + 1] = (float)((uint32_t)(o >> 32) >> 8) * (1.0f / 16777216.0f);
    }
}

}  // namespace somb

using namespace somb;

extern "C" int somb_uniform_f32(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                                int64_t count, float *out, void *stream) {
    SOMB_REQUIRE(count >= 0, SOMB_E_INPUT, "uniform_f32: negative count");
    if (count == 0) return SOMB_OK;
    const int64_t outs = (count + 1) / 2;
    const int64_t threads = (outs + kRngOuts - 1) / kRngOuts;
    pcg64_uniform_f32<<<(unsigned)((threads + 255) / 256), 256, 0, as_stream(stream)>>>(
        U128{state_lo, state_hi}, U128{inc_lo, inc_hi}, count, out);
    note_launch();
    SOMB_LAUNCH_CHECK("uniform_f32");
    return SOMB_OK;
}
