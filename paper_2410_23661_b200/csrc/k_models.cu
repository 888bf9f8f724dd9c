// Row f3: consumer models on the verdicts (§7.5 l.1612-1690), the
// standalone pass: one pass over the records and their codes (from
// picker_validate_batch).  The per-record arithmetic is in models.cuh; the
// fused variant (validation and models in one pass over the records) is
// k_validate_pipe compiled with PICKER_MODELS (picker_validate_models).
// Oracle: oracle/picker_oracle.py oracle_input_bytes / oracle_models.
#include <cuda_runtime.h>

#include "launch.hpp"
#include "models.cuh"

namespace picker {

constexpr int kModelThreads = 256, kModelFast = 8;  // read extents per thread in shared memory

// input bytes of one record; false: unknown (reading Q25).  Most records have
// <= kModelFast reads: their extents sort in the thread's shared-memory column
// (stride = threads, conflict-free); more take local arrays.
static __device__ bool input_bytes(const Tables& T, const picker_rec_t& r, const DevBatch& B, uint64_t& bytes,
                                   int64_t* s_lo, int64_t* s_hi) {
  const uint32_t kid = r.kernel_id;
  if (kid >= T.nkernel_slots) return false;
  const DKernel K = T.kernels[kid];
  if (K.shortcut == V_ERR_KERNEL) return false;
  if (!args_in_range(r, K.nparams, B.args_lo, B.args_hi)) return false;
  if (K.shortcut && K.shortcut != V_IDEM_KERNEL) return false;  // kernel-level NI: no verified summary
  const RecVals X(r, B.args + r.arg_off, K.i32mask);
  if (!model_checks(T, K, X)) return false;
  bool of = false;
  if (model_read_union(T, K, X, bytes, s_lo + threadIdx.x, s_hi + threadIdx.x, kModelThreads, kModelFast, of))
    return true;
  return of ? model_read_union_big(T, K, X, bytes) : false;
}

__global__ void __launch_bounds__(kModelThreads) k_models(Tables T, DevBatch B, uint64_t n,
                                                          const uint8_t* __restrict__ codes,
                                                          const uint64_t* __restrict__ ctx_bytes, uint64_t kill_ns,
                                                          ModelDiv save_bpu, ModelAcc* __restrict__ acc) {
  __shared__ int64_t s_elo[kModelFast * kModelThreads], s_ehi[kModelFast * kModelThreads];
  __shared__ uint32_t s_hw[PICKER_MODEL_HIST], s_hi[PICKER_MODEL_HIST];
  for (int i = threadIdx.x; i < PICKER_MODEL_HIST; i += blockDim.x) s_hw[i] = s_hi[i] = 0;
  __syncthreads();
  ModelSums ms{};
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const picker_rec_t r = load_rec(B.rec + i);
    uint64_t b = 0;
    const bool known = input_bytes(T, r, B, b, s_elo, s_ehi);
    model_add(ms, s_hw, s_hi, codes[i], known, b, ctx_bytes ? ctx_bytes[i] : 0, kill_ns, save_bpu);
  }
  __syncthreads();
  model_flush(ms, s_hw, s_hi, acc);
}

cudaError_t model_acc_begin(void** acc_buf, cudaStream_t s) {
  if (!*acc_buf) {  // owned by the caller's context (allocated once)
    cudaError_t e = cudaMalloc(acc_buf, sizeof(ModelAcc));
    if (e != cudaSuccess) {
      *acc_buf = nullptr;
      return e;
    }
  }
  return cudaMemsetAsync(*acc_buf, 0, sizeof(ModelAcc), s);
}

cudaError_t model_acc_end(void* acc_buf, uint64_t n, picker_model_out_t* out, cudaStream_t s) {
  ModelAcc h;
  cudaError_t e = cudaMemcpyAsync(&h, acc_buf, sizeof(ModelAcc), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return e;
  out->n = n;
  out->n_idem = h.n_idem;
  out->ckpt_bytes_all = h.ckpt_all;
  out->ckpt_bytes_ni = h.ckpt_ni;
  out->unknown_input = h.unknown;
  out->preempt_ns_without = h.pre_without;
  out->preempt_ns_with = h.pre_with;
  for (int i = 0; i < PICKER_MODEL_HIST; ++i) out->hist_without[i] = h.hist_without[i], out->hist_with[i] = h.hist_with[i];
  return cudaSuccess;
}

cudaError_t launch_models(const Tables& T, const DevBatch& b, uint64_t n, const uint8_t* codes,
                          const uint64_t* ctx_bytes, uint64_t kill_ns, uint64_t save_bpu, picker_model_out_t* out,
                          void** acc_buf, int num_sms, cudaStream_t s) {
  cudaError_t e = model_acc_begin(acc_buf, s);
  if (e == cudaSuccess && n) {
    const uint64_t blocks = std::min<uint64_t>((n + kModelThreads - 1) / kModelThreads, (uint64_t)num_sms * 3);
    k_models<<<(unsigned)blocks, kModelThreads, 0, s>>>(T, b, n, codes, ctx_bytes, kill_ns,
                                                        ModelDiv::of(save_bpu), (ModelAcc*)*acc_buf);
    e = cudaGetLastError();
  }
  return e == cudaSuccess ? model_acc_end(*acc_buf, n, out, s) : e;
}

}  // namespace picker
