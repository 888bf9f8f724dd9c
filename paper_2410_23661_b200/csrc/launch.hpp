// Host-side launch interfaces of the device paths.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/picker.h"
#include "tables.hpp"

namespace picker {

struct IrKernel;

struct Options {
  bool jit = false;
  int64_t wide_pairs = 1024;  // |R|*|W| above which the wide path is used
  int force_path = 0;         // 0 auto, 1 generic, 2 jit, 3 wide
  int tile = 4096;            // records per CTA super-tile (specialised path)
};

// Records [0, n) at rec; argument slots valid at indices [args_lo, args_hi) of args.
struct DevBatch {
  const picker_rec_t* rec;
  const int64_t* args;
  uint64_t args_lo, args_hi;
};

struct JitModule;

// Assign a path to every kernel (shortcut / generic / jit / wide).
void select_paths(std::vector<IrKernel>& ks, const Options& opt);
bool any_jit(const std::vector<IrKernel>& ks);
JitModule* jit_build(const std::vector<IrKernel>& ks, const Options& opt, std::string& err);
void jit_destroy(JitModule* m);

cudaError_t launch_validate(const Tables& T, JitModule* jit, const Options& opt, const DevBatch& b,
                            uint64_t n, uint8_t* flags, uint32_t* bits,
                            unsigned long long* counts, int num_sms, cudaStream_t s,
                            int* launches);

cudaError_t launch_exact(const Tables& T, const DevBatch& b, uint64_t n, uint8_t* out,
                         unsigned long long* counts, uint64_t max_points, int num_sms,
                         cudaStream_t s, int* launches, std::string& err);

}  // namespace picker
