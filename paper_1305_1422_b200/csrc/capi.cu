// Library-level entry points: version, last error, device check.
#include <stdarg.h>

#include <atomic>

#include "common.cuh"

namespace somb {
static thread_local char g_err[512] = "";
void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}
static std::atomic<unsigned long long> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
__global__ void probe_kernel(int *out) { *out = 1000; }
}  // namespace somb

extern "C" const char *somb_version(void) { return "somb200 0.1.0 sm_100a"; }
extern "C" const char *somb_last_error(void) { return somb::g_err; }

extern "C" int somb_device_check(int dev) {
    cudaDeviceProp prop;
    cudaError_t e = cudaGetDeviceProperties(&prop, dev);
    if (e != cudaSuccess) return somb::cuda_status(e, "cudaGetDeviceProperties");
    if (prop.major != 10 || prop.minor != 0) {
        somb::set_error("somb200 is built for sm_100a (B200); device %d is sm_%d%d (%s)", dev, prop.major,
                        prop.minor, prop.name);
        return SOMB_E_ARCH;
    }
    cudaFuncAttributes fa;
    e = cudaFuncGetAttributes(&fa, somb::probe_kernel);
    if (e != cudaSuccess) return somb::cuda_status(e, "kernel image load");
    return SOMB_OK;
}

extern "C" unsigned long long somb_launch_count(void) { return somb::g_launches.load(); }

namespace somb {
int screen_tc_set_knob(const char *key, int value);
int bmu_set_knob(const char *key, int value);
}
extern "C" int somb_set_knob(const char *key, int32_t value) {
    SOMB_REQUIRE(key != nullptr, SOMB_E_CONFIG, "set_knob: null key");
    int rc = somb::bmu_set_knob(key, value);
    if (rc == SOMB_E_CONFIG) rc = somb::screen_tc_set_knob(key, value);
    if (rc == SOMB_E_CONFIG) somb::set_error("set_knob: unknown key %s", key);
    return rc;
}

// ------------------------------------------------------------ diagnostics
// L2 read-bandwidth probe: `reps` grid-stride passes of float4 loads over a
// buffer small enough to stay L2-resident (the denominator of the L2-bound
// kernels' rooflines, bench.py; no driver-written L2 peak exists).  One
// partial sum per thread block keeps the loads live.
namespace somb {
__global__ void __launch_bounds__(512) l2_probe_kernel(const float4 *__restrict__ buf, int64_t n4, int reps,
                                                       float *__restrict__ out) {
    float acc = 0.0f;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; ++r) {
        // rotate the start so consecutive passes do not hit the same lines first
        const int64_t off = ((int64_t)r * 7919 * blockDim.x) % n4;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
            int64_t j = i + off;
            if (j >= n4) j -= n4;
            const float4 v = __ldcg(buf + j);
            acc += (v.x + v.y) + (v.z + v.w);
        }
    }
    if (acc == 1.2345e-30f) out[blockIdx.x] = acc;   // never taken: keeps the loads
}
}  // namespace somb

extern "C" int somb_l2_probe(const float *buf, int64_t n, int32_t reps, float *out, void *stream) {
    SOMB_REQUIRE(buf && n >= 4 && reps > 0, SOMB_E_INPUT, "l2_probe: bad arguments");
    int dev = 0, sms = somb::kSmCount;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    somb::l2_probe_kernel<<<4 * sms, 512, 0, somb::as_stream(stream)>>>(reinterpret_cast<const float4 *>(buf), n / 4,
                                                                          reps, out);
    somb::note_launch();
    SOMB_LAUNCH_CHECK("l2_probe");
    return SOMB_OK;
}
