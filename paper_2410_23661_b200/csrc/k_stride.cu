// Row f4: the stride-aware variant of K1 (picker_set_option "stride" = 1).
// The staged + bucketed kernels of k_bucket.cuh with eval_stride as the
// per-record evaluator (grouped by kernel: the table reads are warp-uniform).
// Wide kernels are evaluated by eval_stride too (wide_key = none).
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/picker.h"
#include "eval_stride.cuh"
#include "k_bucket.cuh"
#include "launch.hpp"

namespace picker {

struct StrideDispatch {
  static __device__ __forceinline__ uint8_t eval(uint32_t key, uint32_t bin, uint32_t kn, bool local,
                                                 const BucketParams& P, const picker_rec_t& r, const int64_t* a,
                                                 const DevBatch& B) {
    (void)key, (void)kn, (void)local;
    if (bin >= P.nbins) return V_ERR_KERNEL;
    return eval_stride(P.T, r, a, B.args_lo, B.args_hi);
  }
};

template __global__ void k_validate_bucket<StrideDispatch>(const __grid_constant__ BucketParams,
                                                           const __grid_constant__ DevBatch, uint64_t, uint8_t*,
                                                           uint32_t*, unsigned long long*);
template __global__ void k_validate_pipe<StrideDispatch>(const __grid_constant__ BucketParams,
                                                         const __grid_constant__ DevBatch, uint64_t, uint8_t*,
                                                         uint32_t*, unsigned long long*);

__global__ void __launch_bounds__(256) k_validate_stride_flat(Tables T, DevBatch B, uint64_t n,
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
      code = eval_stride(T, r, B.args + r.arg_off, B.args_lo, B.args_hi);
    }
    emit(i, valid, code, flags, bits, hist);
  }
  __syncthreads();
  if (counts && threadIdx.x < PICKER_NUM_COUNTS && hist[threadIdx.x])
    atomicAdd(counts + threadIdx.x, (unsigned long long)hist[threadIdx.x]);
}

cudaError_t launch_stride(const BucketParams& P0, const DevBatch& B, uint64_t n, uint8_t* flags, uint32_t* bits,
                          unsigned long long* counts, bool bucket, int num_sms, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  BucketParams P = P0;  // key = bin (table path), no K2 interception
  P.nkeys = P.nbins + 2;
  P.wide_key = 0xFFFFFFFFu;
  const bool pipe = P.nkeys <= kPipeKeys;
  const size_t smem = pipe ? pipe_smem_bytes_for(kTile, PICKER_ARGS_PER_REC) : bucket_smem_bytes(P.nkeys);
  if (bucket && smem <= kMaxSmem) {
    static size_t configured[64][2] = {};  // per device
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) dev = -1;
    if (dev < 0 || smem > configured[dev][pipe]) {
      cudaError_t e = cudaFuncSetAttribute(pipe ? k_validate_pipe<StrideDispatch> : k_validate_bucket<StrideDispatch>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      if (dev >= 0) configured[dev][pipe] = smem;
    }
    const uint64_t ntiles = (n + kTile - 1) / kTile;
    const uint64_t cap = (uint64_t)num_sms * kCtasPerSm;
    const uint64_t grid = ntiles < cap ? ntiles : cap;
    if (pipe)
      k_validate_pipe<StrideDispatch><<<(unsigned)grid, kThreads, smem, s>>>(P, B, n, flags, bits, counts);
    else
      k_validate_bucket<StrideDispatch><<<(unsigned)grid, kThreads, smem, s>>>(P, B, n, flags, bits, counts);
    return cudaGetLastError();
  }
  uint64_t blocks = (n + 255) / 256;
  const uint64_t cap = (uint64_t)num_sms * 8;
  if (blocks > cap) blocks = cap;
  k_validate_stride_flat<<<(unsigned)blocks, 256, 0, s>>>(P.T, B, n, flags, bits, counts);
  return cudaGetLastError();
}

}  // namespace picker
