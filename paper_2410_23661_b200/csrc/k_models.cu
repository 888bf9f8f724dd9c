// Row f3: consumer models fused on the verdicts (§7.5 l.1612-1690).
//
// One pass over the records and their codes (from picker_validate_batch):
//   - Asymmetric Resilience (l.1618-1640): "AR checkpoints the input buffer of
//     every GPU kernel instance ... For idempotent instances, AR avoids the
//     memory checkpointing."  Input bytes of an instance = length of the union
//     of its active non-opaque read extents (the K1 extents, re-evaluated from
//     the tables); unknown (0, counted) when not computable -- reading Q25.
//   - Chimera (l.1666-1690): preempting an idempotent instance kills it
//     (kill_ns); otherwise its context is saved, ctx_bytes * 1000 /
//     save_bytes_per_us ns.  Sums and 1-us histograms, integer-exact.
// Oracle: oracle/picker_oracle.py oracle_input_bytes / oracle_models.
#include <cuda_runtime.h>

#include "desc_eval.cuh"
#include "launch.hpp"

namespace picker {

constexpr int kModelMaxReads = 128;  // reading Q25 (oracle MODEL_MAX_READS)

struct ModelAcc {
  unsigned long long n_idem, ckpt_all, ckpt_ni, unknown, pre_without, pre_with;
  unsigned long long hist_without[PICKER_MODEL_HIST], hist_with[PICKER_MODEL_HIST];
};

constexpr int kModelThreads = 256, kModelFast = 8;  // read extents per thread in shared memory

// input bytes of one record; false: unknown.  `lo` / `hi` hold up to `cap`
// extents (the thread's shared-memory rows, or its local arrays).
static __device__ bool input_bytes_in(const Tables& T, const picker_rec_t& r, const DevBatch& B, uint64_t& bytes,
                                      int64_t* lo, int64_t* hi, int stride, int cap, bool& overflow) {
  overflow = false;
  const uint32_t kid = r.kernel_id;
  if (kid >= T.nkernel_slots) return false;
  const DKernel K = T.kernels[kid];
  if (K.shortcut == V_ERR_KERNEL) return false;
  if (!args_in_range(r, K.nparams, B.args_lo, B.args_hi)) return false;
  if (K.shortcut && K.shortcut != V_IDEM_KERNEL) return false;  // kernel-level NI: no verified summary
  const RecVals X(r, B.args + r.arg_off, K.i32mask);
  if (!launch_limits_ok(X)) return false;
  for (int c = 0; c < K.npre + K.nglob; ++c) {
    const DCheck ch = T.checks[K.check + c];
    const int64_t v = X.get(ch.op);
    if (v < ch.lo || v > ch.hi) return false;
  }
  int m = 0;
  for (int d = 0; d < K.ndesc; ++d) {
    const DDesc D = T.descs[K.desc + d];
    if (D.kind != KIND_R) continue;
    int64_t lb = 0, ub = 0;
    if (!desc_active_extent(T, K, D, X, lb, ub)) continue;  // each variable's bounds once
    if (D.opaque || m == kModelMaxReads) return false;
    if (m == cap) {
      overflow = true;
      return false;
    }
    int j = m++;  // insertion by lb
    while (j > 0 && lo[(j - 1) * stride] > lb) {
      lo[j * stride] = lo[(j - 1) * stride];
      hi[j * stride] = hi[(j - 1) * stride];
      --j;
    }
    lo[j * stride] = lb;
    hi[j * stride] = ub;
  }
  uint64_t total = 0;
  for (int i = 0; i < m;) {  // merge touching / overlapping extents
    int64_t a = lo[i * stride], b = hi[i * stride];
    int j = i + 1;
    while (j < m && lo[j * stride] <= b + 1) {
      b = max(b, hi[j * stride]);
      ++j;
    }
    total += (uint64_t)(b - a) + 1;
    i = j;
  }
  bytes = total;
  return true;
}

// Most records have <= kModelFast reads: their extents sort in the thread's
// shared-memory column (stride = threads, conflict-free); more take local arrays.
static __device__ __noinline__ bool input_bytes_big(const Tables& T, const picker_rec_t& r, const DevBatch& B,
                                                    uint64_t& bytes) {
  int64_t lo[kModelMaxReads], hi[kModelMaxReads];
  bool of;
  return input_bytes_in(T, r, B, bytes, lo, hi, 1, kModelMaxReads, of);
}

static __device__ bool input_bytes(const Tables& T, const picker_rec_t& r, const DevBatch& B, uint64_t& bytes,
                                   int64_t* s_lo, int64_t* s_hi) {
  bool of = false;
  if (input_bytes_in(T, r, B, bytes, s_lo + threadIdx.x, s_hi + threadIdx.x, kModelThreads, kModelFast, of)) return true;
  return of ? input_bytes_big(T, r, B, bytes) : false;
}

__global__ void __launch_bounds__(kModelThreads) k_models(Tables T, DevBatch B, uint64_t n,
                                                          const uint8_t* __restrict__ codes,
                                                          const uint64_t* __restrict__ ctx_bytes, uint64_t kill_ns,
                                                          uint64_t save_bpu, ModelAcc* __restrict__ acc) {
  __shared__ int64_t s_elo[kModelFast * kModelThreads], s_ehi[kModelFast * kModelThreads];
  __shared__ unsigned long long s_sum[6];
  __shared__ unsigned int s_hw[PICKER_MODEL_HIST], s_hi[PICKER_MODEL_HIST];
  for (int i = threadIdx.x; i < PICKER_MODEL_HIST; i += blockDim.x) s_hw[i] = s_hi[i] = 0;
  if (threadIdx.x < 6) s_sum[threadIdx.x] = 0;
  __syncthreads();
  unsigned long long n_idem = 0, all = 0, ni = 0, unk = 0, pw = 0, pi = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const picker_rec_t r = load_rec(B.rec + i);
    uint64_t b = 0;
    if (!input_bytes(T, r, B, b, s_elo, s_ehi)) {
      b = 0;
      ++unk;
    }
    const bool idem = codes[i] <= V_IDEM_KERNEL;
    all += b;
    if (!idem) ni += b;
    n_idem += idem;
    const uint64_t save = (ctx_bytes ? ctx_bytes[i] : 0) * 1000ull / save_bpu;
    const uint64_t lat = idem ? kill_ns : save;
    pw += save;
    pi += lat;
    atomicAdd(&s_hw[min(save / 1000, (uint64_t)PICKER_MODEL_HIST - 1)], 1u);
    atomicAdd(&s_hi[min(lat / 1000, (uint64_t)PICKER_MODEL_HIST - 1)], 1u);
  }
  atomicAdd(&s_sum[0], n_idem);
  atomicAdd(&s_sum[1], all);
  atomicAdd(&s_sum[2], ni);
  atomicAdd(&s_sum[3], unk);
  atomicAdd(&s_sum[4], pw);
  atomicAdd(&s_sum[5], pi);
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(&acc->n_idem, s_sum[0]);
    atomicAdd(&acc->ckpt_all, s_sum[1]);
    atomicAdd(&acc->ckpt_ni, s_sum[2]);
    atomicAdd(&acc->unknown, s_sum[3]);
    atomicAdd(&acc->pre_without, s_sum[4]);
    atomicAdd(&acc->pre_with, s_sum[5]);
  }
  for (int i = threadIdx.x; i < PICKER_MODEL_HIST; i += blockDim.x) {
    if (s_hw[i]) atomicAdd(&acc->hist_without[i], (unsigned long long)s_hw[i]);
    if (s_hi[i]) atomicAdd(&acc->hist_with[i], (unsigned long long)s_hi[i]);
  }
}

cudaError_t launch_models(const Tables& T, const DevBatch& b, uint64_t n, const uint8_t* codes,
                          const uint64_t* ctx_bytes, uint64_t kill_ns, uint64_t save_bpu, picker_model_out_t* out,
                          void** acc_buf, int num_sms, cudaStream_t s) {
  // the accumulator is owned by the caller's context (allocated once)
  if (!*acc_buf) {
    cudaError_t e = cudaMalloc(acc_buf, sizeof(ModelAcc));
    if (e != cudaSuccess) {
      *acc_buf = nullptr;
      return e;
    }
  }
  ModelAcc* acc = (ModelAcc*)*acc_buf;
  cudaError_t e = cudaMemsetAsync(acc, 0, sizeof(ModelAcc), s);
  if (e == cudaSuccess && n) {
    const uint64_t blocks = std::min<uint64_t>((n + kModelThreads - 1) / kModelThreads, (uint64_t)num_sms * 3);
    k_models<<<(unsigned)blocks, kModelThreads, 0, s>>>(T, b, n, codes, ctx_bytes, kill_ns, save_bpu, acc);
    e = cudaGetLastError();
  }
  ModelAcc h;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, acc, sizeof(ModelAcc), cudaMemcpyDeviceToHost, s);
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

}  // namespace picker
