// Multi-kernel idempotency:
// "validate the idempotency of a list of sequentially executed GPU kernel
// instances with two steps.  First, Picker predicts the read and write
// addresses of each GPU kernel instance.  Second, Picker sorts the instances by
// their launch order, and then checks the clobber anti-dependency across the
// instances ... [or, for] concurrently executed GPU kernel instances, ... the
// overlap of read and write addresses among all concurrent instances."
//
// The stream is cut into consecutive windows of `window` launches (launch
// order = record order).  S1 (one thread per record) evaluates each record's
// prefix and extents into scratch; S2 (one CTA per window) decides the window:
// the first decisive record code, then the opaque rule, then the overlap of a
// read of instance i with a write of instance j (sequential: i <= j;
// concurrent: any i, j) -- reading Q23 in DESIGN.md, identical to
// oracle.picker_oracle.oracle_sequence.
#include <cuda_runtime.h>

#include <string>

#include "desc_eval.cuh"
#include "launch.hpp"

namespace picker {

constexpr uint8_t kEvaluable = 0x80;
constexpr int kSeqMaxDesc = 64;  // extents kept per record

struct SeqRec {
  uint8_t status;  // decisive verdict, or kEvaluable
  uint8_t flags;   // 1 act_r, 2 act_w, 4 opq_r, 8 opq_w
  uint8_t n;       // active non-opaque extents
  uint8_t pad[5];
  uint64_t wmask;  // bit k: extent k is a write
};

__global__ void k_seq_extents(Tables T, DevBatch B, uint64_t n, SeqRec* __restrict__ sr,
                              int64_t* __restrict__ ext /* [n][kSeqMaxDesc][2] */) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const picker_rec_t r = load_rec(B.rec + i);
    SeqRec s{};
    s.status = kEvaluable;
    const uint32_t kid = r.kernel_id;
    do {
      if (kid >= T.nkernel_slots || T.kernels[kid].shortcut == V_ERR_KERNEL) {
        s.status = V_ERR_KERNEL;
        break;
      }
      const DKernel K = T.kernels[kid];
      if (!args_in_range(r, K.nparams, B.args_lo, B.args_hi)) {
        s.status = V_ERR_ARITY;
        break;
      }
      if (K.shortcut && K.shortcut != V_IDEM_KERNEL) {  // kernel-level NI
        s.status = K.shortcut;
        break;
      }
      const RecVals X(r, B.args + r.arg_off, K.i32mask);
      if (!launch_limits_ok(X)) {
        s.status = V_NI_PRECOND;
        break;
      }
      bool fail = false;
      for (int c = 0; c < K.npre + K.nglob && !fail; ++c) {
        const DCheck ch = T.checks[K.check + c];
        const int64_t v = X.get(ch.op);
        if (v < ch.lo || v > ch.hi) {
          s.status = c < K.npre ? V_NI_PRECOND : V_NI_GLOBAL;
          fail = true;
        }
      }
      if (fail) break;
      for (int d = 0; d < K.ndesc; ++d) {
        const DDesc D = T.descs[K.desc + d];
        if (!desc_active(T, K, D, X)) continue;
        s.flags |= D.kind == KIND_R ? 1 : 2;
        if (D.opaque) {
          s.flags |= D.kind == KIND_R ? 4 : 8;
          continue;
        }
        int64_t lb, ub;
        desc_extent(T, K, D, X, lb, ub);
        ext[(i * kSeqMaxDesc + s.n) * 2] = lb;
        ext[(i * kSeqMaxDesc + s.n) * 2 + 1] = ub;
        if (D.kind == KIND_W) s.wmask |= 1ull << s.n;
        ++s.n;
      }
    } while (false);
    sr[i] = s;
  }
}

__global__ void __launch_bounds__(256) k_seq_windows(const SeqRec* __restrict__ sr, const int64_t* __restrict__ ext,
                                                     uint64_t n, uint32_t window, uint32_t mode,
                                                     uint8_t* __restrict__ out) {
  __shared__ uint8_t s_code;
  __shared__ int s_hit;
  const uint64_t w0 = (uint64_t)blockIdx.x * window;
  const uint32_t m = (uint32_t)min((uint64_t)window, n - w0);
  if (threadIdx.x == 0) {
    uint8_t code = kEvaluable;
    for (uint32_t i = 0; i < m && code == kEvaluable; ++i)
      if (sr[w0 + i].status != kEvaluable) code = sr[w0 + i].status;
    if (code == kEvaluable) {  // opaque rule: reads of instance i against writes of j
      bool pre_opq_r = false, pre_act_r = false;  // over instances <= j (sequential)
      bool opq_r = false, act_r = false, opq_w = false, act_w = false;  // whole window
      for (uint32_t j = 0; j < m; ++j) {
        const uint8_t f = sr[w0 + j].flags;
        pre_opq_r |= (f & 4) != 0;
        pre_act_r |= (f & 1) != 0;
        act_r |= (f & 1) != 0, act_w |= (f & 2) != 0, opq_r |= (f & 4) != 0, opq_w |= (f & 8) != 0;
        if (mode == 0 && ((pre_opq_r && (f & 2)) || (pre_act_r && (f & 8)))) code = V_NI_OPAQUE;
      }
      if (mode == 1 && ((opq_r && act_w) || (act_r && opq_w))) code = V_NI_OPAQUE;
    }
    s_code = code;
    s_hit = 0;
  }
  __syncthreads();
  if (s_code != kEvaluable) {
    if (threadIdx.x == 0) out[blockIdx.x] = s_code;
    return;
  }
  // overlap: instance pairs (i reads, j writes) over the threads
  const uint32_t pairs = m * m;
  for (uint32_t p = threadIdx.x; p < pairs; p += blockDim.x) {
    const uint32_t i = p / m, j = p % m;
    if (mode == 0 && i > j) continue;
    const SeqRec a = sr[w0 + i], b = sr[w0 + j];
    for (uint32_t x = 0; x < a.n; ++x) {
      if ((a.wmask >> x) & 1) continue;
      const int64_t rl = ext[((w0 + i) * kSeqMaxDesc + x) * 2], ru = ext[((w0 + i) * kSeqMaxDesc + x) * 2 + 1];
      for (uint32_t y = 0; y < b.n; ++y) {
        if (!((b.wmask >> y) & 1)) continue;
        const int64_t wl = ext[((w0 + j) * kSeqMaxDesc + y) * 2], wu = ext[((w0 + j) * kSeqMaxDesc + y) * 2 + 1];
        if (rl <= wu && wl <= ru) s_hit = 1;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s_hit ? V_NI_OVERLAP : V_IDEM_CHECKED;
}

cudaError_t launch_sequence(const Tables& T, const DevBatch& b, uint64_t n, uint32_t window, uint32_t mode,
                            uint8_t* out, int num_sms, cudaStream_t s, std::string& err) {
  if (n == 0) return cudaSuccess;
  SeqRec* sr = nullptr;
  int64_t* ext = nullptr;
  cudaError_t e = cudaMallocAsync(&sr, n * sizeof(SeqRec), s);
  if (e == cudaSuccess) e = cudaMallocAsync(&ext, n * kSeqMaxDesc * 2 * sizeof(int64_t), s);
  if (e != cudaSuccess) {
    err = "scratch allocation";
    if (sr) cudaFreeAsync(sr, s);
    return e;
  }
  const uint64_t blocks = std::min<uint64_t>((n + 255) / 256, (uint64_t)num_sms * 8);
  k_seq_extents<<<(unsigned)blocks, 256, 0, s>>>(T, b, n, sr, ext);
  const uint64_t nwin = (n + window - 1) / window;
  k_seq_windows<<<(unsigned)nwin, 256, 0, s>>>(sr, ext, n, window, mode, out);
  e = cudaGetLastError();
  cudaFreeAsync(sr, s);
  cudaFreeAsync(ext, s);
  return e;
}

}  // namespace picker
