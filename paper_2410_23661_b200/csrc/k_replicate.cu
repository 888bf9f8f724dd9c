// K6: device-side replication of a launch-record stream (SURVEY §8F C5, §8
// row e: "Generate the shards on device (K6) to avoid PCIe").  Copy c of the
// base trace is the same instances relocated: every pointer argument moves by
// (first + c) * delta, which keeps each verdict (translation invariance,
// SURVEY §8E G9).  Input generation for the multi-GPU stream, not part of the
// validation path; HBM-bound copies with 16-byte accesses.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/picker.h"
#include "launch.hpp"

namespace picker {

__global__ void __launch_bounds__(256) k_replicate_rec(const picker_rec_t* __restrict__ base, uint64_t n,
                                                       uint64_t copies, uint64_t args_len,
                                                       picker_rec_t* __restrict__ out) {
  const uint64_t total = n * copies;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t c = i / n, j = i - c * n;
    const uint4* src = reinterpret_cast<const uint4*>(base + j);
    uint4 a = __ldg(src), b = __ldg(src + 1);
    const uint64_t off = ((uint64_t)b.w << 32 | b.z) + c * args_len;  // arg_off (bytes 24-31)
    b.z = (uint32_t)off, b.w = (uint32_t)(off >> 32);
    uint4* dst = reinterpret_cast<uint4*>(out + i);
    dst[0] = a, dst[1] = b;
  }
}

__global__ void __launch_bounds__(256) k_replicate_args(const int64_t* __restrict__ args, uint64_t args_len,
                                                        const uint8_t* __restrict__ ptr_mask, uint64_t copies,
                                                        uint64_t first, int64_t delta, int64_t* __restrict__ out) {
  const uint64_t total = args_len * copies;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t c = i / args_len, j = i - c * args_len;
    const int64_t v = __ldg(args + j);
    out[i] = ptr_mask[j] ? v + (int64_t)(first + c) * delta : v;
  }
}

cudaError_t launch_replicate(const picker_rec_t* rec, uint64_t n, const int64_t* args, uint64_t args_len,
                             const uint8_t* ptr_mask, uint64_t copies, uint64_t first, int64_t delta,
                             picker_rec_t* rec_out, int64_t* args_out, int num_sms, cudaStream_t s) {
  if (n == 0 || copies == 0) return cudaSuccess;
  const uint64_t cap = (uint64_t)num_sms * 8;
  const uint64_t gr = (n * copies + 255) / 256, ga = (args_len * copies + 255) / 256;
  k_replicate_rec<<<(unsigned)(gr < cap ? gr : cap), 256, 0, s>>>(rec, n, copies, args_len, rec_out);
  if (args_len)
    k_replicate_args<<<(unsigned)(ga < cap ? ga : cap), 256, 0, s>>>(args, args_len, ptr_mask, copies, first, delta,
                                                                     args_out);
  return cudaGetLastError();
}

}  // namespace picker
