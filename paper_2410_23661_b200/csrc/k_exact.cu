// K3 exact verifier (placeholder until the enumerating kernels land).
#include <cuda_runtime.h>

#include "launch.hpp"

namespace picker {

cudaError_t launch_exact(const Tables&, const DevBatch&, uint64_t, uint8_t*, unsigned long long*,
                         uint64_t, int, cudaStream_t, int*, std::string& err) {
  err = "exact verifier not built in this version";
  return cudaErrorNotSupported;
}

}  // namespace picker
