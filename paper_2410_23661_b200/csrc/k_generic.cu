// K1-generic: table-driven validation, one thread per launch record.
//
// This is the straightforward device rendering of the paper's optimized
// validator (§5): per instance, check the preconditions and global
// condition (Fig. 3 lines 1-2; l.976-979, l.749-752), evaluate each range
// descriptor at the extreme values of its variables (l.950-951) with
// path-condition tightening (l.1023-1026) and induction/fresh ranges
// (l.1063, l.990-992), then test every active read extent against every
// active write extent (l.658-666).  It reads the flattened tables of
// tables.hpp directly.  The specialised path (k_jit / jit.cpp) compiles the
// same semantics per kernel; this path is the fallback and the cross-check.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/picker.h"
#include "eval_generic.cuh"
#include "k_bucket.cuh"
#include "launch.hpp"

namespace picker {

__global__ void __launch_bounds__(256) k_validate_generic(Tables T, DevBatch B, uint64_t n,
                                                          uint8_t* __restrict__ flags,
                                                          uint32_t* __restrict__ bits,
                                                          unsigned long long* __restrict__ counts) {
  __shared__ unsigned int hist[PICKER_NUM_COUNTS];
  if (threadIdx.x < PICKER_NUM_COUNTS) hist[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x; i0 < n; i0 += stride) {
    const uint64_t i = i0 + threadIdx.x;
    const bool valid = i < n;
    uint8_t code = 0;
    if (valid) {
      const picker_rec_t r = load_rec(B.rec + i);
      code = eval_generic(T, r, B.args + r.arg_off, B.args_lo, B.args_hi);
    }
    emit(i, valid, code, flags, bits, hist);
  }
  __syncthreads();
  if (counts && threadIdx.x < PICKER_NUM_COUNTS && hist[threadIdx.x])
    atomicAdd(counts + threadIdx.x, (unsigned long long)hist[threadIdx.x]);
}

template __global__ void k_validate_bucket<GenericDispatch>(const __grid_constant__ BucketParams,
                                                            const __grid_constant__ DevBatch, uint64_t,
                                                            uint8_t*, uint32_t*, unsigned long long*);
template __global__ void k_validate_pipe<GenericDispatch>(const __grid_constant__ BucketParams,
                                                          const __grid_constant__ DevBatch, uint64_t,
                                                          uint8_t*, uint32_t*, unsigned long long*);

// Table-driven evaluation through the staged + bucketed kernel (key = kernel).
// Returns cudaErrorInvalidValue when the per-key arrays do not fit in shared
// memory (the caller then uses the unbucketed kernel).
cudaError_t launch_bucket_generic(const BucketParams& P0, const DevBatch& B, uint64_t n,
                                  uint8_t* flags, uint32_t* bits, unsigned long long* counts,
                                  int num_sms, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  BucketParams P = P0;  // kb_of / kb_unknown: key = bin (set at load time)
  P.nkeys = P.nbins + 2;  // kernels, unknown ids, wide kernels (P.wide_key = nbins + 1)
  const bool pipe = P.nkeys <= kPipeKeys;
  const size_t smem = pipe ? pipe_smem_bytes_for(kTile, PICKER_ARGS_PER_REC) : bucket_smem_bytes(P.nkeys);
  if (smem > kMaxSmem) return cudaErrorInvalidValue;
  static size_t configured[64][2] = {};  // per device
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) dev = -1;
  if (dev < 0 || smem > configured[dev][pipe]) {
    cudaError_t e = cudaFuncSetAttribute(pipe ? k_validate_pipe<GenericDispatch> : k_validate_bucket<GenericDispatch>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (dev >= 0) configured[dev][pipe] = smem;
  }
  const uint64_t ntiles = (n + kTile - 1) / kTile;
  const uint64_t cap = (uint64_t)num_sms * kCtasPerSm;
  const uint64_t grid = ntiles < cap ? ntiles : cap;
  if (pipe)
    k_validate_pipe<GenericDispatch><<<(unsigned)grid, kThreads, smem, s>>>(P, B, n, flags, bits, counts);
  else
    k_validate_bucket<GenericDispatch><<<(unsigned)grid, kThreads, smem, s>>>(P, B, n, flags, bits, counts);
  return cudaGetLastError();
}

cudaError_t launch_generic(const Tables& T, const DevBatch& B, uint64_t n, uint8_t* flags,
                           uint32_t* bits,
                           unsigned long long* counts, int num_sms, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  uint64_t blocks = (n + 255) / 256;
  uint64_t cap = (uint64_t)num_sms * 8;
  if (blocks > cap) blocks = cap;
  k_validate_generic<<<(unsigned)blocks, 256, 0, s>>>(T, B, n, flags, bits, counts);
  return cudaGetLastError();
}

}  // namespace picker
