// Path selection and the validate dispatcher.
#include <cuda_runtime.h>

#include "launch.hpp"
#include "loader.hpp"

namespace picker {

cudaError_t launch_generic(const Tables& T, const DevBatch& B, uint64_t n, uint8_t* flags,
                           uint32_t* bits, unsigned long long* counts, int num_sms,
                           cudaStream_t s);
cudaError_t launch_bucket_generic(const BucketParams& P, const DevBatch& B, uint64_t n,
                                  uint8_t* flags, uint32_t* bits, unsigned long long* counts,
                                  int num_sms, cudaStream_t s);
cudaError_t launch_stride(const BucketParams& P, const DevBatch& B, uint64_t n, uint8_t* flags, uint32_t* bits,
                          unsigned long long* counts, bool bucket, int num_sms, cudaStream_t s);
cudaError_t launch_jit(JitModule* m, const BucketParams& P, const DevBatch& B, uint64_t n,
                       uint8_t* flags, uint32_t* bits, unsigned long long* counts, int num_sms,
                       cudaStream_t s);

// Largest read x write pair count the specialised path emits as straight-line code.
constexpr int64_t kJitMaxPairs = 4096;

void select_paths(std::vector<IrKernel>& ks, const Options& opt) {
  for (auto& k : ks) {
    if (k.shortcut) {
      k.path = PATH_SHORTCUT;
      continue;
    }
    if (k.never_evaluates) {
      // empty pre/glob box: every record stops at a check before any address,
      // which the table-driven evaluator decides (no specialised code is emitted)
      k.path = PATH_GENERIC;
      continue;
    }
    size_t nr = 0, nw = 0, nvars = 0;
    for (auto& d : k.desc) {
      (d.kind == KIND_R ? nr : nw)++;
      nvars += d.vars.size();
    }
    (void)nvars;
    const int64_t pairs = (int64_t)(nr * nw);
    // many read x write pairs (cuDNN-like kernels with 16+ pointer arguments):
    // the warp-cooperative sort + sweep path (K2, desc_eval.cuh)
    const bool wide = opt.force_path == 3 || pairs > opt.wide_pairs || pairs > kJitMaxPairs;
    if (wide && opt.force_path != 1 && opt.force_path != 2) {
      k.path = PATH_WIDE;
    } else if (opt.jit && opt.force_path != 1 && pairs <= kJitMaxPairs) {
      k.path = PATH_JIT;
    } else {
      k.path = PATH_GENERIC;  // eval_generic also handles kernels beyond its register arrays
    }
  }
}

// The specialised module is built when some kernel is specialised or wide
// (wide kernels run warp-cooperatively inside the module's schedules).
bool any_jit(const std::vector<IrKernel>& ks) {
  for (auto& k : ks)
    if (k.path == PATH_JIT || k.path == PATH_WIDE) return true;
  return false;
}

cudaError_t launch_validate(const BucketParams& P0, JitModule* jit, const Options& opt,
                            const DevBatch& b, uint64_t n, uint8_t* flags, uint32_t* bits,
                            unsigned long long* counts, int num_sms, cudaStream_t s,
                            int* launches) {
  if (n == 0) return cudaSuccess;
  BucketParams P = P0;
  // P.count_slot set: the launch writes counts (flush_counts).  The paths
  // whose kernels only accumulate get the counts zeroed here instead.
  auto accumulate = [&]() -> cudaError_t {
    if (!counts || !P.count_slot) return cudaSuccess;
    P.count_slot = nullptr;
    return cudaMemsetAsync(counts, 0, PICKER_NUM_COUNTS * sizeof(uint64_t), s);
  };
  if (use_wide_kernel(opt)) {  // every evaluating kernel is wide: K2 on its own
    *launches += 1;
    return launch_wide(P, b, n, flags, bits, counts, num_sms, s);
  }
  *launches += jit && opt.stride == jit_is_stride(jit) ? jit_launch_count(jit, n) : 1;
  // stride mode: the specialised module if it was built stride-aware (option
  // set before picker_load_summaries), else the table-driven evaluator
  if (opt.stride && !jit_is_stride(jit)) {
    cudaError_t e = accumulate();
    return e != cudaSuccess ? e : launch_stride(P, b, n, flags, bits, counts, opt.bucket, num_sms, s);
  }
  if (!opt.stride && jit_is_stride(jit)) jit = nullptr;  // stride-aware module, plain verdicts wanted
  if (jit) return launch_jit(jit, P, b, n, flags, bits, counts, num_sms, s);
  if (opt.bucket && bucket_smem_bytes(P.nbins + 2) <= kMaxSmem)
    return launch_bucket_generic(P, b, n, flags, bits, counts, num_sms, s);
  cudaError_t e = accumulate();
  return e != cudaSuccess ? e : launch_generic(P.T, b, n, flags, bits, counts, num_sms, s);
}

}  // namespace picker
