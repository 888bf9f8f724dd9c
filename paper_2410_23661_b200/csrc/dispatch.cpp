// Path selection and the validate dispatcher.
#include <cuda_runtime.h>

#include "launch.hpp"
#include "loader.hpp"

namespace picker {

cudaError_t launch_generic(const Tables& T, const DevBatch& B, uint64_t n, uint8_t* flags,
                           uint32_t* bits, unsigned long long* counts, int num_sms,
                           cudaStream_t s);
cudaError_t launch_jit(JitModule* m, const Tables& T, const DevBatch& B, uint64_t n,
                       uint8_t* flags, uint32_t* bits, unsigned long long* counts, int num_sms,
                       cudaStream_t s, int* launches);

void select_paths(std::vector<IrKernel>& ks, const Options& opt) {
  for (auto& k : ks) {
    if (k.shortcut) {
      k.path = PATH_SHORTCUT;
      continue;
    }
    size_t nr = 0, nw = 0;
    for (auto& d : k.desc) (d.kind == KIND_R ? nr : nw)++;
    size_t nvars = 0;
    for (auto& d : k.desc) nvars += d.vars.size();
    const bool fits_generic =
        nr <= (size_t)kGenMaxDesc && nw <= (size_t)kGenMaxDesc && nvars <= (size_t)kGenMaxVar;
    if (!fits_generic)
      throw LoadError{PICKER_EFORMAT, "kernel " + std::to_string(k.id) +
                                          ": more than 64 read/write descriptors or variables "
                                          "(wide path not built in this version)"};
    (void)opt;
    k.path = PATH_GENERIC;
  }
}

bool any_jit(const std::vector<IrKernel>& ks) {
  for (auto& k : ks)
    if (k.path == PATH_JIT) return true;
  return false;
}

cudaError_t launch_validate(const Tables& T, JitModule* jit, const Options& opt, const DevBatch& b,
                            uint64_t n, uint8_t* flags, uint32_t* bits,
                            unsigned long long* counts, int num_sms, cudaStream_t s,
                            int* launches) {
  (void)opt;
  if (n == 0) return cudaSuccess;
  if (jit) return launch_jit(jit, T, b, n, flags, bits, counts, num_sms, s, launches);
  *launches += 1;
  return launch_generic(T, b, n, flags, bits, counts, num_sms, s);
}

}  // namespace picker
