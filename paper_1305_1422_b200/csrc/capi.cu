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
