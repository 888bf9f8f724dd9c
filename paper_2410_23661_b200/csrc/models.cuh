// Row f3 per-record model arithmetic (§7.5 l.1612-1690), shared by
// the standalone pass (k_models.cu) and the fused one (k_validate_pipe with
// PICKER_MODELS, picker_validate_models):
//   - Asymmetric Resilience (l.1618-1640): "AR checkpoints the input buffer of
//     every GPU kernel instance ... For idempotent instances, AR avoids the
//     memory checkpointing."  Input bytes of an instance = length of the union
//     of its active non-opaque read extents; unknown (0, counted) when not
//     computable -- reading Q25;
//   - Chimera (l.1666-1690): preempting an idempotent instance kills it
//     (kill_ns); otherwise its context is saved, ctx_bytes * 1000 /
//     save_bytes_per_us ns.  Sums and 1-us histograms, integer-exact.
// Oracle: oracle/picker_oracle.py oracle_input_bytes / oracle_models.
#pragma once

#include "desc_eval.cuh"

namespace picker {

constexpr int kModelMaxReads = 128;  // reading Q25 (oracle MODEL_MAX_READS)
// input bytes from a specialised shape (models module): unknown / not computed
// there (more than 12 reads: the table path below)
constexpr uint64_t kInbUnknown = ~0ull, kInbTable = ~0ull - 1;

// The read extents of one record in lb order (insertion into lo / hi, `stride`
// apart, at most `cap`), then the length of their union.  false: unknown (an
// active opaque read, more than kModelMaxReads reads, or more than `cap`:
// `overflow`).  The launch limits and checks must already hold.
static __device__ __forceinline__ bool model_read_union(const Tables& T, const DKernel& K, const RecVals& X,
                                                        uint64_t& bytes, int64_t* lo, int64_t* hi, int stride,
                                                        int cap, bool& overflow) {
  overflow = false;
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

// launch limits, preconditions and the global condition of a record (the
// checks the input bytes need; K1's verdict implies them except for code 1)
static __device__ __forceinline__ bool model_checks(const Tables& T, const DKernel& K, const RecVals& X) {
  if (!launch_limits_ok(X)) return false;
  for (int c = 0; c < K.npre + K.nglob; ++c) {
    const DCheck ch = T.checks[K.check + c];
    const int64_t v = X.get(ch.op);
    if (v < ch.lo || v > ch.hi) return false;
  }
  return true;
}

// More than 8 reads: local arrays of kModelMaxReads (out of line).
static __device__ __noinline__ bool model_read_union_big(const Tables& T, const DKernel& K, const RecVals& X,
                                                         uint64_t& bytes) {
  int64_t lo[kModelMaxReads], hi[kModelMaxReads];
  bool of;
  return model_read_union(T, K, X, bytes, lo, hi, 1, kModelMaxReads, of);
}

// Input bytes of a record whose verdict `code` K1 computed (args `a`: its
// argument slots, staged or global); false: unknown (reading Q25).
static __device__ __noinline__ bool model_input_bytes_coded(const Tables& T, const picker_rec_t& r,
                                                            const int64_t* a, uint32_t code, uint64_t& bytes) {
  // unknown kernel / arity (0xFF / 0xFE), kernel-level NONIDEM (2-6), failed
  // launch limits / preconditions (7) or global condition (8)
  if (code >= V_NI_SO && code != V_NI_OPAQUE && code != V_NI_OVERLAP) return false;
  const DKernel K = T.kernels[r.kernel_id];
  const RecVals X(r, a, K.i32mask);
  if (code == V_IDEM_KERNEL && !model_checks(T, K, X)) return false;  // checks not evaluated by K1
  int64_t lo[8], hi[8];
  bool of = false;
  if (model_read_union(T, K, X, bytes, lo, hi, 1, 8, of)) return true;
  return of ? model_read_union_big(T, K, X, bytes) : false;
}

// Row f1 on K1's extents (picker_validate_sequence with an extents module):
// the specialised shapes put every active non-opaque extent of a record into
// its `cap` arena slots (reads from the front, writes from the back) and the
// activity / opaque flags into fl (1 act_r, 2 act_w, 4 opq_r, 8 opq_w).
struct XOut {
  int64_t* ext;  // 2 x cap int64 (lb, ub) per record
  uint32_t cap, nr, nw, fl;
};
__device__ __forceinline__ void xo_put(XOut& x, bool write, int64_t lb, int64_t ub) {
  const uint32_t k = write ? x.cap - 1 - x.nw++ : x.nr++;
  x.ext[2 * k] = lb, x.ext[2 * k + 1] = ub;
}
// xinfo word of a record: nr | nw << 11 | fl << 22 (cap <= 2047)
__device__ __forceinline__ uint32_t xo_info(const XOut& x) { return x.nr | x.nw << 11 | x.fl << 22; }

// Per-thread sums of the models and their addition to the global accumulator.
struct ModelSums {
  unsigned long long n_idem, all, ni, unk, pw, pi;
};
// x / d with the invariant divisor's multiplier (ModelDiv, tables.hpp)
__device__ __forceinline__ uint64_t model_div(uint64_t x, const ModelDiv& d) {
  const uint64_t t = __umul64hi(d.m, x);
  return (t + ((x - t) >> d.sh1)) >> d.sh2;
}
// one histogram bin += 1 per lane, aggregated over the active lanes with the same bin
__device__ __forceinline__ void hist_inc(uint32_t* hist, uint32_t bin) {
  const unsigned peers = __match_any_sync(__activemask(), bin);
  if ((threadIdx.x & 31) == (uint32_t)(__ffs(peers) - 1)) atomicAdd(&hist[bin], (uint32_t)__popc(peers));
}
__device__ __forceinline__ void model_add(ModelSums& s, uint32_t* hist_without, uint32_t* hist_with, uint32_t code,
                                          bool known, uint64_t bytes, uint64_t ctx_bytes, uint64_t kill_ns,
                                          const ModelDiv& save_bpu) {
  const bool idem = code <= V_IDEM_KERNEL;
  if (!known) ++s.unk, bytes = 0;
  s.all += bytes;
  if (!idem) s.ni += bytes;
  s.n_idem += idem;
  const uint64_t save = model_div(ctx_bytes * 1000ull, save_bpu);
  const uint64_t lat = idem ? kill_ns : save;
  s.pw += save;
  s.pi += lat;
  hist_inc(hist_without, (uint32_t)min(save / 1000, (uint64_t)PICKER_MODEL_HIST - 1));
  hist_inc(hist_with, (uint32_t)min(lat / 1000, (uint64_t)PICKER_MODEL_HIST - 1));
}
// Every thread of the CTA: the CTA's sums (warp reductions + shared atomics)
// and histograms into acc.
__device__ __forceinline__ void model_flush(const ModelSums& s, const uint32_t* hist_without,
                                            const uint32_t* hist_with, ModelAcc* acc) {
  __shared__ unsigned long long s_sum[6];
  if (threadIdx.x < 6) s_sum[threadIdx.x] = 0;
  __syncthreads();
  unsigned long long v[6] = {s.n_idem, s.all, s.ni, s.unk, s.pw, s.pi};
#pragma unroll
  for (int q = 0; q < 6; ++q) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], d);
    if ((threadIdx.x & 31) == 0 && v[q]) atomicAdd(&s_sum[q], v[q]);
  }
  __syncthreads();
  if (threadIdx.x < 6 && s_sum[threadIdx.x]) {
    unsigned long long* dst[6] = {&acc->n_idem, &acc->ckpt_all, &acc->ckpt_ni,
                                  &acc->unknown, &acc->pre_without, &acc->pre_with};
    atomicAdd(dst[threadIdx.x], s_sum[threadIdx.x]);
  }
  for (int i = threadIdx.x; i < PICKER_MODEL_HIST; i += blockDim.x) {
    if (hist_without[i]) atomicAdd(&acc->hist_without[i], (unsigned long long)hist_without[i]);
    if (hist_with[i]) atomicAdd(&acc->hist_with[i], (unsigned long long)hist_with[i]);
  }
}

}  // namespace picker
