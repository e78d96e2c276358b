// tcgen05 screen -- placeholder until the tensor-core kernel lands.
#include "common.cuh"
namespace somb {
int launch_screen_tc(const __half *, int64_t, int, const __half *, int, const float *, const float *,
                     const float *, float, int *, int *, int *, cudaStream_t) {
    set_error("tcgen05 screen not built yet; use screen_impl=1");
    return SOMB_E_ARCH;
}
}  // namespace somb
