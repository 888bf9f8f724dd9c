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
// Kernels (all on `stream`, no host round trip):
//   X1 (one thread per record): the shared prefix (kernel class, launch limits,
//      preconditions, global condition, opaque rule), the point count (cap ->
//      code 11), the range extents.  No pairwise extent intersection => exact 0
//      (exact sets are subsets of the extents).  Otherwise the record is pending:
//      its window is the hull of the pairwise intersections (only bytes there
//      can be shared), and it is appended to one of two device lists by the
//      size of its byte-set table (an atomic counter: on-device compaction).
//   X2 (persistent; a CTA claims pending records): the written bytes of the
//      window go into an open-addressing hash table in the CTA's slice of a
//      global arena -- one entry per touched 64-byte block (key = block index,
//      value = 64-bit byte mask; atomicCAS on the key, atomicOr on the mask) --
//      then every read point tests its blocks' masks.  The table is sized from
//      the write points (<= 2 entries per block), so its size is bounded by the
//      point cap, not by the window: no window limit (reading Q22).  Windows of
//      up to 256 KB use a bitmap in shared memory instead (one bit per byte, 64-bit
//      atomicOr per touched block).  Records
//      whose table exceeds a slice of the small pass go to the big pass, whose
//      slices hold the largest table the point cap allows.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "desc_eval.cuh"
#include "eval_generic.cuh"
#include "launch.hpp"

namespace picker {

constexpr uint32_t kPending = 0x100;
constexpr int kExactThreads = 256;
constexpr unsigned long long kEmptyKey = ~0ULL;
constexpr uint64_t kSmemBlocks = 4096;  // shared-memory bitmap: windows up to 256 KB

__device__ __forceinline__ uint64_t sat_mul(uint64_t a, uint64_t b, uint64_t lim) {
  if (a == 0 || b == 0) return 0;
  return a > lim / b ? lim : min(a * b, lim);
}

// 64-byte blocks one point of `width` bytes can touch
__device__ __forceinline__ uint64_t blocks_per_point(uint32_t width) { return (width + 63) / 64 + 1; }

// X1: final code, or kPending with the window [wlo, whi] and the number of
// hash-table blocks the window's written bytes can occupy.
__device__ uint32_t exact_prefix(const Tables& T, const picker_rec_t r, const int64_t* a, uint64_t alo,
                                 uint64_t ahi, uint64_t cap, int64_t& wlo, int64_t& whi, uint64_t& wblocks) {
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
  uint64_t points = 0, wpb = 0;  // wpb: write points x blocks per point
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
    if (D.kind == KIND_W) wpb += p * blocks_per_point(D.width);  // p <= cap + 1 (cap checked below)
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
  const uint64_t wspan = ((uint64_t)(whi - wlo) >> 6) + 2;  // blocks of the window
  wblocks = min(wpb, wspan);
  return kPending;
}

// log2 of the table entries for b blocks: load factor <= 1/2, >= 64 entries
__host__ __device__ __forceinline__ uint32_t table_log2(uint64_t b) {
  uint32_t l = 6;
  while ((1ULL << l) < 2 * b) ++l;
  return l;
}

struct ExactLists {
  uint32_t* pend[2];    // pending record indices: small pass, big pass
  uint32_t* count;      // [0], [1]: list lengths; [2], [3]: claim counters
};

__global__ void k_exact_prefix(Tables T, DevBatch B, uint64_t n, uint64_t cap, uint32_t small_log2,
                               uint8_t* __restrict__ out, int64_t* __restrict__ win, uint8_t* __restrict__ tlog,
                               ExactLists L) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const picker_rec_t r = load_rec(B.rec + i);
    int64_t wlo = 0, whi = -1;
    uint64_t wb = 0;
    const uint32_t st = exact_prefix(T, r, B.args + r.arg_off, B.args_lo, B.args_hi, cap, wlo, whi, wb);
    out[i] = st == kPending ? 0 : (uint8_t)st;
    if (st != kPending) continue;
    win[2 * i] = wlo;
    win[2 * i + 1] = whi;
    const uint32_t tl = table_log2(wb);
    tlog[i] = (uint8_t)tl;
    const int big = tl > small_log2;
    L.pend[big][atomicAdd(L.count + big, 1u)] = (uint32_t)i;
  }
}

// X2: CTAs claim records of list `which`; each has a slice of 2^slice_log2
// table entries (keys, then masks).
__global__ void __launch_bounds__(kExactThreads) k_exact_enum(Tables T, DevBatch B, ExactLists L, int which,
                                                              const int64_t* __restrict__ win,
                                                              const uint8_t* __restrict__ tlog,
                                                              unsigned long long* __restrict__ arena,
                                                              uint32_t slice_log2, uint8_t* __restrict__ out) {
  __shared__ int64_t s_lo[16], s_sz[16], s_coef[64], s_base;
  __shared__ uint32_t s_div[64];
  __shared__ uint8_t s_lvar[64], s_op[16], s_src[16];
  __shared__ int64_t s_arg[16];
  __shared__ uint64_t s_npts;
  __shared__ int s_on, s_found, s_nv, s_nt;
  __shared__ uint32_t s_claim;
  __shared__ unsigned long long s_bits[kSmemBlocks];
  unsigned long long* keys = arena + ((uint64_t)blockIdx.x << (slice_log2 + 1));
  unsigned long long* masks = keys + (1ULL << slice_log2);
  const uint32_t npend = L.count[which];
  for (;;) {
    if (threadIdx.x == 0) s_claim = atomicAdd(L.count + 2 + which, 1u);
    __syncthreads();
    const uint32_t c = s_claim;
    if (c >= npend) return;
    const uint64_t i = L.pend[which][c];
    const picker_rec_t r = load_rec(B.rec + i);
    const DKernel K = T.kernels[r.kernel_id];
    const RecVals X(r, B.args + r.arg_off, K.i32mask);
    const int64_t wlo = win[2 * i], whi = win[2 * i + 1];
    const uint32_t tl = tlog[i];
    const uint64_t tmask = (1ULL << tl) - 1;
    // small windows: a bitmap of the window's 64-byte blocks in shared memory
    // (one bit per byte); larger ones: the hash table in the CTA's slice
    const uint64_t wblocks = ((uint64_t)(whi - wlo) >> 6) + 1;
    const bool in_smem = wblocks <= kSmemBlocks;
    if (in_smem)
      for (uint64_t e = threadIdx.x; e < wblocks; e += blockDim.x) s_bits[e] = 0;
    else
      for (uint64_t e = threadIdx.x; e <= tmask; e += blockDim.x) keys[e] = kEmptyKey, masks[e] = 0;
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
          // early exit once any thread found a shared byte (atomic reads and
          // writes of the flag: no shared-memory race)
          for (uint64_t p = threadIdx.x; p < s_npts && !(pass == 1 && atomicOr(&s_found, 0)); p += blockDim.x) {
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
            // bytes [b0, b1] of the window, as offsets from wlo
            const int64_t b0 = max64(addr, wlo), b1 = min64(add64(addr, (int64_t)D.width - 1), whi);
            if (b0 > b1) continue;
            const uint64_t o0 = (uint64_t)(b0 - wlo), o1 = (uint64_t)(b1 - wlo);
            for (uint64_t blk = o0 >> 6; blk <= (o1 >> 6); ++blk) {
              const uint32_t s0 = blk == (o0 >> 6) ? (uint32_t)(o0 & 63) : 0;
              const uint32_t s1 = blk == (o1 >> 6) ? (uint32_t)(o1 & 63) : 63;
              const unsigned long long m = (~0ULL >> (63 - s1)) & (~0ULL << s0);
              if (in_smem) {
                if (pass == 0) {
                  atomicOr(s_bits + blk, m);
                } else if (s_bits[blk] & m) {
                  atomicExch(&s_found, 1);
                  break;
                }
                continue;
              }
              uint64_t h = (blk * 0x9E3779B97F4A7C15ULL) >> (64 - tl);
              if (pass == 0) {
                for (;;) {
                  const unsigned long long k = atomicCAS(keys + h, kEmptyKey, (unsigned long long)blk);
                  if (k == kEmptyKey || k == blk) {
                    atomicOr(masks + h, m);
                    break;
                  }
                  h = (h + 1) & tmask;
                }
              } else {
                bool hit = false;
                for (;;) {
                  const unsigned long long k = keys[h];
                  if (k == kEmptyKey) break;
                  if (k == blk) {
                    hit = (masks[h] & m) != 0;
                    break;
                  }
                  h = (h + 1) & tmask;
                }
                if (hit) {
                  atomicExch(&s_found, 1);
                  break;
                }
              }
            }
          }
        }
        __syncthreads();
      }
    }
    if (threadIdx.x == 0) out[i] = s_found ? V_NI_OVERLAP : V_IDEM_CHECKED;
    __syncthreads();  // s_claim, the slice and s_found are reused
  }
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
                         unsigned long long* counts, uint64_t cap, uint32_t max_width, void** arena,
                         size_t* arena_bytes, int num_sms, cudaStream_t s, int* launches, std::string& err) {
  *launches = 0;
  if (n == 0) return cudaSuccess;
  if (n >= (1ULL << 32)) {
    err = "more than 2^32 - 1 records";
    return cudaErrorInvalidValue;
  }
  // the largest table a record can need: every write point within the cap,
  // each touching blocks_per_point(max width) blocks
  const uint64_t bpp = (max_width + 63) / 64 + 1;
  if (cap > (1ULL << 40) / bpp) {
    err = "max_points too large for the byte-set tables";
    return cudaErrorInvalidValue;
  }
  const uint32_t big_log2 = table_log2(std::max<uint64_t>(cap * bpp, 1));
  const size_t big_bytes = (size_t)16 << big_log2;
  const size_t want = std::max<size_t>(big_bytes, (size_t)512 << 20);
  if (*arena_bytes < want) {
    if (*arena) cudaFree(*arena);
    *arena = nullptr;
    *arena_bytes = 0;
    cudaError_t e = cudaMalloc(arena, want);
    if (e != cudaSuccess) {
      err = "byte-set arena (" + std::to_string(want >> 20) + " MB)";
      return e;
    }
    *arena_bytes = want;
  }
  const uint64_t entries = *arena_bytes / 16;
  const uint32_t grid_small = (uint32_t)num_sms * 2;
  uint32_t small_log2 = 6;
  while ((2ULL << small_log2) * grid_small <= entries) ++small_log2;
  small_log2 = std::min(small_log2, big_log2);
  const uint32_t grid_big = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(entries >> big_log2, num_sms));

  // scratch: windows, table sizes, two pending lists, 4 counters
  int64_t* win = nullptr;
  uint8_t* tl = nullptr;
  uint32_t* lists = nullptr;
  cudaError_t e = cudaMallocAsync(&win, 2 * n * sizeof(int64_t), s);
  if (e == cudaSuccess) e = cudaMallocAsync(&tl, n, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&lists, (2 * n + 4) * sizeof(uint32_t), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(lists + 2 * n, 0, 4 * sizeof(uint32_t), s);
  if (e != cudaSuccess) {
    err = "scratch allocation";
    return e;
  }
  ExactLists L{{lists, lists + n}, lists + 2 * n};
  const uint64_t blocks = std::min<uint64_t>((n + 255) / 256, (uint64_t)num_sms * 8);
  k_exact_prefix<<<(unsigned)blocks, 256, 0, s>>>(T, b, n, cap, small_log2, out, win, tl, L);
  k_exact_enum<<<grid_small, kExactThreads, 0, s>>>(T, b, L, 0, win, tl, (unsigned long long*)*arena, small_log2,
                                                    out);
  k_exact_enum<<<grid_big, kExactThreads, 0, s>>>(T, b, L, 1, win, tl, (unsigned long long*)*arena, big_log2, out);
  *launches = 3;
  if (counts) {
    k_histogram<<<(unsigned)std::min<uint64_t>((n + 255) / 256, (uint64_t)num_sms * 4), 256, 0, s>>>(out, n, counts);
    ++*launches;
  }
  cudaFreeAsync(win, s);
  cudaFreeAsync(tl, s);
  cudaFreeAsync(lists, s);
  e = cudaGetLastError();
  if (e != cudaSuccess) err = "exact kernels";
  return e;
}

}  // namespace picker
