// NVRTC-specialised validation kernels (placeholder until the JIT lands).
#include <cuda_runtime.h>

#include "launch.hpp"
#include "loader.hpp"

namespace picker {

struct JitModule {};

JitModule* jit_build(const std::vector<IrKernel>&, const Options&, std::string& err) {
  err = "specialised path not built in this version";
  return nullptr;
}

void jit_destroy(JitModule* m) { delete m; }

cudaError_t launch_jit(JitModule*, const Tables&, const DevBatch&, uint64_t, uint8_t*, uint32_t*,
                       unsigned long long*, int, cudaStream_t, int*) {
  return cudaErrorNotSupported;
}

cudaError_t launch_exact(const Tables&, const DevBatch&, uint64_t, uint8_t*, unsigned long long*,
                         uint64_t, int, cudaStream_t, int*, std::string& err) {
  err = "exact verifier not built in this version";
  return cudaErrorNotSupported;
}

}  // namespace picker
