// K3: exact (enumerating) verifier -- the paper's strawman validator.
//
// "For each symbolic address, the validator iterates through all block and
// thread IDs to calculate the concrete address accessed by each GPU thread
// ... Finally, the validator determines the idempotency of the instance by
// checking the overlap between the read and write addresses" (PAPER.md
// l.721-730, Fig. 3).  Here the read/write test is done on touched BYTES, so
// the verdict has no range overestimation (the RO false negatives of
// l.1170-1185): comparing it with the range-based verdict measures that
// conservatism, and checks that the range model never misses an overlap.
//
// Two kernels:
//   X1 (one thread per record): the shared prefix (kernel class, launch limits,
//      preconditions, global condition, opaque rule), the point count (cap ->
//      code 11), the range extents.  No pairwise extent intersection => exact 0
//      (exact sets are subsets of the extents).  Otherwise the record is pending
//      with the hull of the pairwise intersections as its window (> 2^31 bytes
//      -> code 11, reading Q22).
//   X2 (one CTA per pending record): a bitmap over the window in a global
//      arena; every point of every active write descriptor sets the bits of its
//      bytes (atomicOr); every point of every active read descriptor tests them.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "desc_eval.cuh"
#include "eval_generic.cuh"
#include "launch.hpp"

namespace picker {

constexpr uint32_t kPending = 0x100;
constexpr uint64_t kExactWindowCap = 1ULL << 31;  // bytes (oracle: EXACT_WINDOW_CAP)
constexpr int kExactThreads = 256;

__device__ __forceinline__ uint64_t sat_mul(uint64_t a, uint64_t b, uint64_t lim) {
  if (a == 0 || b == 0) return 0;
  return a > lim / b ? lim : min(a * b, lim);
}

// X1: final code, or kPending with the window [wlo, whi] to enumerate.
__device__ uint32_t exact_prefix(const Tables& T, const picker_rec_t r, const int64_t* a, uint64_t alo,
                                 uint64_t ahi, uint64_t cap, int64_t& wlo, int64_t& whi) {
  const uint32_t kid = r.kernel_id;
  if (kid >= T.nkernel_slots) return V_ERR_KERNEL;
  const DKernel K = T.kernels[kid];
  if (K.shortcut == V_ERR_KERNEL) return V_ERR_KERNEL;
  if (!args_in_range(r, K.nparams, alo, ahi)) return V_ERR_ARITY;
  if (K.shortcut) return K.shortcut;
  RecVals X(r, a, K.i32mask);
  if (!launch_limits_ok(X)) return V_NI_PRECOND;
  for (int c = 0; c < K.npre + K.nglob; ++c) {
    const DCheck ch = T.checks[K.check + c];
    const int64_t v = X.get(ch.op);
    if (v < ch.lo || v > ch.hi) return c < K.npre ? V_NI_PRECOND : V_NI_GLOBAL;
  }
  bool opq_r = false, opq_w = false, act_r = false, act_w = false;
  uint64_t points = 0;
  const uint64_t lim = cap + 1;
  for (int di = 0; di < K.ndesc; ++di) {
    const DDesc D = T.descs[K.desc + di];
    if (!desc_active(T, K, D, X)) continue;
    (D.kind == KIND_R ? act_r : act_w) = true;
    if (D.opaque) {
      (D.kind == KIND_R ? opq_r : opq_w) = true;
      continue;
    }
    uint64_t p = 1;
    for (int v = 0; v < D.nvar; ++v) {
      if (T.vardef[D.var + v].op != 0) continue;  // derived fresh variable
      int64_t lo, hi;
      slot_bounds(T, K, X, T.varlist[D.var + v], lo, hi);
      p = sat_mul(p, (uint64_t)(hi - lo) + 1, lim);
    }
    points = min(points + p, lim);
  }
  if ((opq_r && act_w) || (opq_w && act_r)) return V_NI_OPAQUE;
  if (points > cap) return V_EXACT_SKIPPED;
  bool any = false;
  for (int i = 0; i < K.ndesc; ++i) {
    const DDesc Ri = T.descs[K.desc + i];
    if (Ri.kind != KIND_R || Ri.opaque || !desc_active(T, K, Ri, X)) continue;
    int64_t rl, ru;
    desc_extent(T, K, Ri, X, rl, ru);
    for (int j = 0; j < K.ndesc; ++j) {
      const DDesc Wj = T.descs[K.desc + j];
      if (Wj.kind != KIND_W || Wj.opaque || !desc_active(T, K, Wj, X)) continue;
      int64_t wl, wu;
      desc_extent(T, K, Wj, X, wl, wu);
      if (rl <= wu && wl <= ru) {
        const int64_t lo = max64(rl, wl), hi = min64(ru, wu);
        wlo = any ? min64(wlo, lo) : lo;
        whi = any ? max64(whi, hi) : hi;
        any = true;
      }
    }
  }
  if (!any) return V_IDEM_CHECKED;
  if ((uint64_t)(whi - wlo) + 1 > kExactWindowCap) return V_EXACT_SKIPPED;
  return kPending;
}

__global__ void k_exact_prefix(Tables T, DevBatch B, uint64_t n, uint64_t cap, uint8_t* __restrict__ out,
                               uint32_t* __restrict__ status, int64_t* __restrict__ win) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const picker_rec_t r = load_rec(B.rec + i);
    int64_t wlo = 0, whi = -1;
    const uint32_t st = exact_prefix(T, r, B.args + r.arg_off, B.args_lo, B.args_hi, cap, wlo, whi);
    status[i] = st;
    win[2 * i] = wlo;
    win[2 * i + 1] = whi;
    out[i] = st == kPending ? 0 : (uint8_t)st;
  }
}

// X2: one CTA per pending record.  Pass 0 marks the window bytes written,
// pass 1 tests the bytes read.
__global__ void __launch_bounds__(kExactThreads) k_exact_enum(Tables T, DevBatch B, const uint32_t* __restrict__ pend,
                                                              const int64_t* __restrict__ win,
                                                              const uint64_t* __restrict__ woff,
                                                              uint32_t* __restrict__ arena, uint8_t* __restrict__ out) {
  __shared__ int64_t s_lo[16], s_sz[16], s_coef[64], s_base;
  __shared__ uint32_t s_div[64];
  __shared__ uint8_t s_lvar[64], s_op[16], s_src[16];
  __shared__ int64_t s_arg[16];
  __shared__ uint64_t s_npts;
  __shared__ int s_on, s_found, s_nv, s_nt;
  const uint64_t i = pend[blockIdx.x];
  const picker_rec_t r = load_rec(B.rec + i);
  const DKernel K = T.kernels[r.kernel_id];
  const RecVals X(r, B.args + r.arg_off, K.i32mask);
  const int64_t wlo = win[2 * i], whi = win[2 * i + 1];
  const uint64_t L = (uint64_t)(whi - wlo) + 1, nwords = (L + 31) / 32;
  uint32_t* bm = arena + woff[blockIdx.x];
  for (uint64_t w = threadIdx.x; w < nwords; w += blockDim.x) bm[w] = 0;
  if (threadIdx.x == 0) s_found = 0;
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass) {
    const uint8_t kind = pass == 0 ? KIND_W : KIND_R;
    for (int di = 0; di < K.ndesc; ++di) {
      const DDesc D = T.descs[K.desc + di];
      if (D.kind != kind || D.opaque) continue;
      if (threadIdx.x == 0) {
        s_on = desc_active(T, K, D, X);
        uint64_t np = 1;
        for (int v = 0; v < D.nvar; ++v) {
          int64_t lo, hi;
          slot_bounds(T, K, X, T.varlist[D.var + v], lo, hi);
          const DVarDef vd = T.vardef[D.var + v];
          s_lo[v] = lo;
          s_sz[v] = hi - lo + 1;
          s_op[v] = vd.op;
          s_src[v] = vd.src;
          s_arg[v] = vd.arg;
          if (vd.op == 0) np *= (uint64_t)(hi - lo + 1);  // bounded by the point cap (X1)
        }
        s_npts = np;
        s_nv = D.nvar;
        s_nt = D.nterm;
        s_base = D.base == OPD_NONE ? 0 : X.get(D.base);
        for (int t = 0; t < D.nterm; ++t) {
          const DTerm tm = T.terms[D.term + t];
          s_coef[t] = prod_val(T, K, X, tm.prod);
          s_div[t] = tm.div;
          s_lvar[t] = T.term_lvar[D.term + t];
        }
      }
      __syncthreads();
      if (s_on) {
        const volatile int* found = &s_found;
        for (uint64_t p = threadIdx.x; p < s_npts && !(pass == 1 && *found); p += blockDim.x) {
          int64_t x[16];
          uint64_t q = p;
          for (int v = 0; v < s_nv; ++v)
            if (s_op[v] == 0) {
              const uint64_t sz = (uint64_t)s_sz[v];
              x[v] = s_lo[v] + (int64_t)(q % sz);
              q /= sz;
            }
          for (int v = 0; v < s_nv; ++v)
            if (s_op[v] != 0) {
              const int64_t src = x[s_src[v]], m = s_arg[v];
              if (s_op[v] == DEF_OP_MOD) {
                int64_t md = src % m;
                x[v] = md < 0 ? md + m : md;  // floor modulo (Python %)
              } else {
                x[v] = src & m;
              }
            }
          int64_t addr = s_base;
          for (int t = 0; t < s_nt; ++t)
            addr = add64(addr, s_lvar[t] == 0xFF ? s_coef[t] : mul64(s_coef[t], floordiv64(x[s_lvar[t]], s_div[t])));
          const int64_t b0 = max64(addr, wlo), b1 = min64(add64(addr, (int64_t)D.width - 1), whi);
          for (int64_t b = b0; b <= b1; ++b) {
            const uint64_t off = (uint64_t)(b - wlo);
            if (pass == 0) {
              atomicOr(bm + (off >> 5), 1u << (off & 31));
            } else if ((bm[off >> 5] >> (off & 31)) & 1u) {
              s_found = 1;
              break;
            }
          }
        }
      }
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) out[i] = s_found ? V_NI_OVERLAP : V_IDEM_CHECKED;
}

__global__ void k_histogram(const uint8_t* __restrict__ codes, uint64_t n, unsigned long long* counts) {
  __shared__ unsigned int h[PICKER_NUM_COUNTS];
  if (threadIdx.x < PICKER_NUM_COUNTS) h[threadIdx.x] = 0;
  __syncthreads();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(h + count_bin(codes[i]), 1u);
  __syncthreads();
  if (threadIdx.x < PICKER_NUM_COUNTS && h[threadIdx.x]) atomicAdd(counts + threadIdx.x, (unsigned long long)h[threadIdx.x]);
}

cudaError_t launch_exact(const Tables& T, const DevBatch& b, uint64_t n, uint8_t* out,
                         unsigned long long* counts, uint64_t cap, int num_sms, cudaStream_t s, int* launches,
                         std::string& err) {
  *launches = 0;
  if (n == 0) return cudaSuccess;
  uint32_t* status = nullptr;
  int64_t* win = nullptr;
  cudaError_t e = cudaMallocAsync(&status, n * sizeof(uint32_t), s);
  if (e == cudaSuccess) e = cudaMallocAsync(&win, 2 * n * sizeof(int64_t), s);
  if (e != cudaSuccess) {
    err = "scratch allocation";
    return e;
  }
  const uint64_t blocks = std::min<uint64_t>((n + 255) / 256, (uint64_t)num_sms * 8);
  k_exact_prefix<<<(unsigned)blocks, 256, 0, s>>>(T, b, n, cap, out, status, win);
  ++*launches;
  std::vector<uint32_t> st(n);
  std::vector<int64_t> w(2 * n);
  e = cudaMemcpyAsync(st.data(), status, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(w.data(), win, 2 * n * sizeof(int64_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    err = "X1 / D2H";
    return e;
  }
  // batches of pending records whose bitmaps fit the arena
  const uint64_t arena_words = 1ULL << 26;  // 256 MB
  uint32_t* arena = nullptr;
  std::vector<uint32_t> pend;
  std::vector<uint64_t> off;
  uint64_t used = 0;
  uint32_t* d_pend = nullptr;
  uint64_t* d_off = nullptr;
  auto flush = [&]() -> cudaError_t {
    if (pend.empty()) return cudaSuccess;
    cudaError_t ee = cudaSuccess;
    if (!arena) ee = cudaMallocAsync(&arena, arena_words * 4, s);
    if (!d_pend && ee == cudaSuccess) ee = cudaMallocAsync(&d_pend, n * sizeof(uint32_t), s);
    if (!d_off && ee == cudaSuccess) ee = cudaMallocAsync(&d_off, n * sizeof(uint64_t), s);
    if (ee == cudaSuccess)
      ee = cudaMemcpyAsync(d_pend, pend.data(), pend.size() * 4, cudaMemcpyHostToDevice, s);
    if (ee == cudaSuccess)
      ee = cudaMemcpyAsync(d_off, off.data(), off.size() * 8, cudaMemcpyHostToDevice, s);
    if (ee != cudaSuccess) return ee;
    k_exact_enum<<<(unsigned)pend.size(), kExactThreads, 0, s>>>(T, b, d_pend, win, d_off, arena, out);
    ++*launches;
    ee = cudaStreamSynchronize(s);  // pend/off host vectors are reused
    pend.clear();
    off.clear();
    used = 0;
    return ee;
  };
  for (uint64_t i = 0; i < n && e == cudaSuccess; ++i) {
    if (st[i] != kPending) continue;
    const uint64_t words = ((uint64_t)(w[2 * i + 1] - w[2 * i]) + 1 + 31) / 32;
    if (used + words > arena_words) e = flush();
    pend.push_back((uint32_t)i);
    off.push_back(used);
    used += (words + 31) & ~31ULL;
  }
  if (e == cudaSuccess) e = flush();
  if (e == cudaSuccess && counts) {
    k_histogram<<<(unsigned)std::min<uint64_t>((n + 255) / 256, (uint64_t)num_sms * 4), 256, 0, s>>>(out, n, counts);
    ++*launches;
  }
  cudaFreeAsync(status, s);
  cudaFreeAsync(win, s);
  if (arena) cudaFreeAsync(arena, s);
  if (d_pend) cudaFreeAsync(d_pend, s);
  if (d_off) cudaFreeAsync(d_off, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess && err.empty()) err = "X2";
  return e == cudaSuccess ? cudaGetLastError() : e;
}

}  // namespace picker
