// Multi-kernel idempotency:
// "validate the idempotency of a list of sequentially executed GPU kernel
// instances with two steps.  First, Picker predicts the read and write
// addresses of each GPU kernel instance.  Second, Picker sorts the instances by
// their launch order, and then checks the clobber anti-dependency across the
// instances ... [or, for] concurrently executed GPU kernel instances, ... the
// overlap of read and write addresses among all concurrent instances."
//
// The stream is cut into consecutive windows of `window` launches (launch
// order = record order); one CTA decides one window at a time (persistent),
// reading DESIGN.md Q23 (identical to oracle.picker_oracle.oracle_sequence):
//   1. threads over the window's records: each record's decisive code (the
//      first one in launch order decides), its activity / opaque flags, and its
//      active non-opaque extents appended to the CTA's read and write lists;
//   2. the opaque rule (sequential: an opaque read of i with a write of j >= i,
//      or a read of i with an opaque write of j >= i; concurrent: any i, j);
//   3. the overlap, as sort + sweep passes over the extents.  Concurrent: one
//      pass, any read against any write.  Sequential ("a read of i and a write
//      of j with i <= j"): divide and conquer over launch order -- a pass per
//      level l of a binary split of the window checks the reads of every left
//      half against the writes of the matching right half (instance bit l = 0
//      vs 1, same higher bits), plus one pass within each instance.  Each pass
//      tags the extents with a node id, sorts the writes by (node, lb) (bitonic,
//      CTA-wide), takes the prefix maxima of ub within each node (the sweep
//      line's running maximum), and probes every read by binary search in its
//      node: some write of the node overlaps the read iff, at the last write
//      with lb <= read.ub, the running maximum ub >= read.lb (closed intervals).
// No per-record limit on descriptors; the lists live in a per-CTA slice of a
// global scratch (window x max descriptors x 48 bytes, L1/L2-resident).
#include <cuda_runtime.h>

#include <string>

#include "desc_eval.cuh"
#include "launch.hpp"

namespace picker {

constexpr int kSeqThreads = 512;
constexpr uint8_t kEvaluable = 0x80;

struct SeqIv {  // one extent: [lb, ub] of instance `inst` of the window
  int64_t lb, ub;
  uint32_t inst, node;
};

__device__ __forceinline__ bool seq_less(const SeqIv& a, const SeqIv& b) {
  return a.node < b.node || (a.node == b.node && a.lb < b.lb);
}

// K1's verdicts and extents of the batch (row f1 reusing K1),
// or all null: the window kernel evaluates the records from the tables.
struct SeqK1 {
  const uint8_t* codes;   // K1 verdict per record
  const uint32_t* xinfo;  // nr | nw << 11 | flags << 22 (models.cuh XOut)
  const int64_t* xarena;  // xcap (lb, ub) slots per record: reads first, writes from the back
  uint32_t xcap;
};

// The threads deciding one window: a CTA (any window size) or one warp (windows
// of <= 32 launches, several windows per CTA), with their shared state.
template <int F>
struct SeqShared {
  uint32_t first, nr, nw, ns, hit;
  uint8_t code;
  uint8_t flags[F];  // per instance: 1 act_r, 2 act_w, 4 opq_r, 8 opq_w
};
struct SeqCta {
  SeqShared<1024>* sh;
  int tid, size;
  __device__ __forceinline__ void sync() const { __syncthreads(); }
};
struct SeqWarp {
  SeqShared<32>* sh;
  int tid, size;
  __device__ __forceinline__ void sync() const { __syncwarp(); }
};

// One window: returns its code (uniform over the group g).
template <class Grp>
__device__ uint8_t seq_window(const Tables& T, const DevBatch& B, uint64_t w0, uint32_t m, uint32_t mode, SeqIv* Rl,
                              SeqIv* Wl, SeqIv* S, int64_t* PM, uint32_t cap, const SeqK1& K1, const Grp& g) {
  auto& sh = *g.sh;
  const int tid = g.tid;
  if (tid == 0) sh.first = 0xFFFFFFFFu, sh.nr = 0, sh.nw = 0, sh.hit = 0;
  g.sync();
  // 1. records of the window
  for (uint32_t i = tid; i < m; i += (uint32_t)g.size) {
    uint8_t status = kEvaluable, fl = 0;
    if (K1.codes) {
      // K1 decided the record: a code before any address decides (0xFF, 0xFE,
      // 2-8); 0 / 9 / 10: its extents and flags are in the arena; 1 (a
      // kernel-level idempotent kernel, whose checks K1 does not evaluate):
      // the tables below
      const uint32_t c = K1.codes[w0 + i];
      if (c >= V_NI_SO && c != V_NI_OPAQUE && c != V_NI_OVERLAP) {
        status = (uint8_t)c;
      } else if (c != V_IDEM_KERNEL) {
        const uint32_t info = K1.xinfo[w0 + i];
        const uint32_t nr = info & 0x7FFu, nw = (info >> 11) & 0x7FFu;
        fl = (uint8_t)(info >> 22);
        const int64_t* x = K1.xarena + (w0 + i) * 2 * K1.xcap;
        const uint32_t pr = nr ? atomicAdd(&sh.nr, nr) : 0u, pw = nw ? atomicAdd(&sh.nw, nw) : 0u;
        for (uint32_t q = 0; q < nr; ++q)
          if (pr + q < cap) Rl[pr + q] = SeqIv{x[2 * q], x[2 * q + 1], i, 0};
        for (uint32_t q = 0; q < nw; ++q) {
          const uint32_t k = K1.xcap - 1 - q;
          if (pw + q < cap) Wl[pw + q] = SeqIv{x[2 * k], x[2 * k + 1], i, 0};
        }
        sh.flags[i] = fl;
        continue;
      }
    }
    const picker_rec_t r = load_rec(B.rec + w0 + i);
    const uint32_t kid = r.kernel_id;
    if (status == kEvaluable) do {
      if (kid >= T.nkernel_slots || T.kernels[kid].shortcut == V_ERR_KERNEL) {
        status = V_ERR_KERNEL;
        break;
      }
      const DKernel K = T.kernels[kid];
      if (!args_in_range(r, K.nparams, B.args_lo, B.args_hi)) {
        status = V_ERR_ARITY;
        break;
      }
      if (K.shortcut && K.shortcut != V_IDEM_KERNEL) {  // kernel-level NI
        status = K.shortcut;
        break;
      }
      const RecVals X(r, B.args + r.arg_off, K.i32mask);
      if (!launch_limits_ok(X)) {
        status = V_NI_PRECOND;
        break;
      }
      for (int c = 0; c < K.npre + K.nglob && status == kEvaluable; ++c) {
        const DCheck ch = T.checks[K.check + c];
        const int64_t v = X.get(ch.op);
        if (v < ch.lo || v > ch.hi) status = c < K.npre ? V_NI_PRECOND : V_NI_GLOBAL;
      }
      if (status != kEvaluable) break;
      // kernel-level idempotent instances take part with their writes (Q23)
      for (int d = 0; d < K.ndesc; ++d) {
        const DDesc D = T.descs[K.desc + d];
        int64_t lb = 0, ub = 0;
        if (!desc_active_extent(T, K, D, X, lb, ub)) continue;
        fl |= D.kind == KIND_R ? 1 : 2;
        if (D.opaque) {
          fl |= D.kind == KIND_R ? 4 : 8;
          continue;
        }
        const uint32_t pos = atomicAdd(D.kind == KIND_R ? &sh.nr : &sh.nw, 1u);
        if (pos < cap) (D.kind == KIND_R ? Rl : Wl)[pos] = SeqIv{lb, ub, i, 0};
      }
    } while (false);
    sh.flags[i] = fl;
    if (status != kEvaluable) atomicMin(&sh.first, (i << 8) | status);
  }
  g.sync();
  // the first decisive record (launch order) decides the window
  if (sh.first != 0xFFFFFFFFu) return (uint8_t)(sh.first & 0xFF);
  // 2. opaque rule
  if (tid == 0) {
    uint8_t code = kEvaluable;
    bool pre_opq_r = false, pre_act_r = false, opq_r = false, act_r = false, opq_w = false, act_w = false;
    for (uint32_t j = 0; j < m; ++j) {
      const uint8_t f = sh.flags[j];
      pre_opq_r |= (f & 4) != 0, pre_act_r |= (f & 1) != 0;
      act_r |= (f & 1) != 0, act_w |= (f & 2) != 0, opq_r |= (f & 4) != 0, opq_w |= (f & 8) != 0;
      if (mode == 0 && ((pre_opq_r && (f & 2)) || (pre_act_r && (f & 8)))) code = V_NI_OPAQUE;
    }
    if (mode == 1 && ((opq_r && act_w) || (act_r && opq_w))) code = V_NI_OPAQUE;
    sh.code = code;
  }
  g.sync();
  if (sh.code != kEvaluable) return sh.code;
  // 3. overlap passes
  const uint32_t nr = sh.nr, nw = sh.nw;
  if (nr == 0 || nw == 0) return V_IDEM_CHECKED;
  if ((uint64_t)nr * nw <= 256ull * (uint32_t)g.size) {
    // few extents (C2 windows of 32: ~70 x 40): every (read, write) pair, the
    // predicate the passes below decide -- a read of i and a write of j share a
    // byte, sequential i <= j, concurrent any i, j -- without their sorts and
    // barriers
    bool hit = false;
    for (uint32_t x = tid; x < nr && !hit; x += (uint32_t)g.size) {
      const SeqIv r = Rl[x];
      for (uint32_t y = 0; y < nw; ++y) {
        const SeqIv w = Wl[y];  // the same element for every thread: one broadcast
        if ((mode == 1 || r.inst <= w.inst) && r.lb <= w.ub && w.lb <= r.ub) {
          hit = true;
          break;
        }
      }
    }
    if (hit) sh.hit = 1;
    g.sync();
    return sh.hit ? V_NI_OVERLAP : V_IDEM_CHECKED;
  }
  uint32_t levels = 0;
  while ((1u << levels) < m) ++levels;
  // pass p: mode 1 -> one pass (node 0); mode 0 -> p = levels .. 0: p == levels is
  // the within-instance pass (node = inst), p < levels the cross pass of level p
  const int first_pass = mode == 1 ? -1 : (int)levels;
  for (int p = first_pass; p >= (mode == 1 ? -1 : 0); --p) {
    auto wnode = [&](uint32_t inst, bool& in) -> uint32_t {
      if (p < 0) return in = true, 0u;
      if (p == (int)levels) return in = true, inst;
      in = (inst >> p) & 1;  // right half of its level-p node
      return inst >> (p + 1);
    };
    auto rnode = [&](uint32_t inst, bool& in) -> uint32_t {
      if (p < 0) return in = true, 0u;
      if (p == (int)levels) return in = true, inst;
      in = !((inst >> p) & 1);  // left half
      return inst >> (p + 1);
    };
    if (tid == 0) sh.ns = 0;
    g.sync();
    for (uint32_t x = tid; x < nw; x += (uint32_t)g.size) {
      SeqIv w = Wl[x];
      bool in;
      w.node = wnode(w.inst, in);
      if (in) S[atomicAdd(&sh.ns, 1u)] = w;
    }
    g.sync();
    const uint32_t ns = sh.ns;
    if (ns == 0) continue;
    uint32_t n2 = 32;
    while (n2 < ns) n2 <<= 1;
    for (uint32_t x = ns + tid; x < n2; x += (uint32_t)g.size)
      S[x] = SeqIv{9223372036854775807LL, (-9223372036854775807LL - 1), 0, 0xFFFFFFFFu};  // sorts last
    g.sync();
    for (uint32_t k = 2; k <= n2; k <<= 1)  // bitonic sort by (node, lb)
      for (uint32_t j = k >> 1; j > 0; j >>= 1) {
        for (uint32_t q = tid; q < n2 / 2; q += (uint32_t)g.size) {
          const uint32_t i = ((q & ~(j - 1)) << 1) | (q & (j - 1)), o = i | j;
          const SeqIv a = S[i], b = S[o];
          if (((i & k) == 0) ? seq_less(b, a) : seq_less(a, b)) S[i] = b, S[o] = a;
        }
        g.sync();
      }
    if (tid < 32) {  // prefix maxima of ub within each node segment (one warp, carried)
      const int lane = tid;
      int64_t carry = (-9223372036854775807LL - 1);
      uint32_t carry_node = 0xFFFFFFFFu;
      for (uint32_t h = 0; h < ns; h += 32) {
        const uint32_t x = h + lane;
        const SeqIv e = x < ns ? S[x] : SeqIv{0, (-9223372036854775807LL - 1), 0, 0xFFFFFFFEu};
        int64_t v = e.ub;
        // segmented inclusive max: only elements of the same node contribute
        for (int d = 1; d < 32; d <<= 1) {
          const int64_t o = __shfl_up_sync(0xffffffffu, v, d);
          const uint32_t on = __shfl_up_sync(0xffffffffu, e.node, d);
          if (lane >= d && on == e.node) v = max64(v, o);
        }
        if (e.node == carry_node) v = max64(v, carry);
        if (x < ns) PM[x] = v;
        carry = __shfl_sync(0xffffffffu, v, 31);
        carry_node = __shfl_sync(0xffffffffu, e.node, 31);
      }
    }
    g.sync();
    for (uint32_t x = tid; x < nr && !sh.hit; x += (uint32_t)g.size) {
      const SeqIv r = Rl[x];
      bool in;
      const uint32_t node = rnode(r.inst, in);
      if (!in) continue;
      // last index whose (node, lb) <= (node, r.ub)
      int lo = -1;
      for (uint32_t step = n2 >> 1; step > 0; step >>= 1) {
        const SeqIv& c = S[lo + (int)step];
        if (c.node < node || (c.node == node && c.lb <= r.ub)) lo += (int)step;
      }
      if (lo + 1 < (int)n2) {
        const SeqIv& c = S[lo + 1];
        if (c.node < node || (c.node == node && c.lb <= r.ub)) ++lo;
      }
      if (lo >= 0 && S[lo].node == node && PM[lo] >= r.lb) sh.hit = 1;
    }
    g.sync();
    if (sh.hit) return V_NI_OVERLAP;
  }
  return V_IDEM_CHECKED;
}

__global__ void __launch_bounds__(kSeqThreads) k_seq_windows(Tables T, DevBatch B, uint64_t n, uint32_t window,
                                                              uint32_t mode, uint8_t* __restrict__ scratch,
                                                              uint64_t slice, uint32_t cap, uint8_t* __restrict__ out,
                                                              const SeqK1 K1) {
  // per-CTA slice: reads [cap], writes [cap], sort buffer [2 cap], prefix maxima [2 cap]
  __shared__ SeqShared<1024> sh;
  const SeqCta grp{&sh, (int)threadIdx.x, (int)blockDim.x};
  SeqIv* Rl = reinterpret_cast<SeqIv*>(scratch + blockIdx.x * slice);
  SeqIv* Wl = Rl + cap;
  SeqIv* S = Wl + cap;
  int64_t* PM = reinterpret_cast<int64_t*>(S + 2 * (uint64_t)cap);
  const uint64_t nwin = (n + window - 1) / window;
  for (uint64_t w = blockIdx.x; w < nwin; w += gridDim.x) {
    const uint64_t w0 = w * window;
    const uint32_t m = (uint32_t)min((uint64_t)window, n - w0);
    const uint8_t code = seq_window(T, B, w0, m, mode, Rl, Wl, S, PM, cap, K1, grp);
    if (threadIdx.x == 0) out[w] = code;
    __syncthreads();  // the slice and the shared state are reused by the next window
  }
}

// Windows of <= 32 launches: one warp per window, 8 windows per CTA at a time
// (a CTA per window of 32 threads was capped at 32 warps per SM by the CTA
// limit); each warp has its own scratch slice and shared state.
constexpr int kSeqWarps = 8;
__global__ void __launch_bounds__(kSeqWarps * 32) k_seq_windows_w(Tables T, DevBatch B, uint64_t n, uint32_t window,
                                                                 uint32_t mode, uint8_t* __restrict__ scratch,
                                                                 uint64_t slice, uint32_t cap,
                                                                 uint8_t* __restrict__ out, const SeqK1 K1) {
  __shared__ SeqShared<32> sh[kSeqWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t gw = (uint64_t)blockIdx.x * kSeqWarps + warp, nwarps = (uint64_t)gridDim.x * kSeqWarps;
  const SeqWarp grp{&sh[warp], lane, 32};
  SeqIv* Rl = reinterpret_cast<SeqIv*>(scratch + gw * slice);
  SeqIv* Wl = Rl + cap;
  SeqIv* S = Wl + cap;
  int64_t* PM = reinterpret_cast<int64_t*>(S + 2 * (uint64_t)cap);
  const uint64_t nwin = (n + window - 1) / window;
  for (uint64_t w = gw; w < nwin; w += nwarps) {
    const uint64_t w0 = w * window;
    const uint32_t m = (uint32_t)min((uint64_t)window, n - w0);
    const uint8_t code = seq_window(T, B, w0, m, mode, Rl, Wl, S, PM, cap, K1, grp);
    if (lane == 0) out[w] = code;
    __syncwarp();  // the slice and the shared state are reused by the next window
  }
}

cudaError_t launch_sequence(const Tables& T, const DevBatch& b, uint64_t n, uint32_t window, uint32_t mode,
                            uint32_t max_desc, uint8_t* out, void** scratch_buf, size_t* scratch_bytes, int num_sms,
                            cudaStream_t s, std::string& err, const uint8_t* k1_codes, const uint32_t* k1_xinfo,
                            const int64_t* k1_xarena, uint32_t k1_xcap) {
  if (n == 0) return cudaSuccess;
  // extents per window <= window x max descriptors per kernel
  const uint32_t cap = std::max<uint32_t>(32, window * std::max<uint32_t>(max_desc, 1));
  const uint64_t slice = (uint64_t)cap * (4 * sizeof(SeqIv) + 2 * sizeof(int64_t));
  const uint64_t nwin = (n + window - 1) / window;
  // a thread per record of a window (32..512 threads per CTA), as many CTAs as
  // fill the SMs (2048 threads each), within ~1 GB of scratch
  // (windows of <= 32 launches: a warp per window, kSeqWarps windows per CTA)
  const bool per_warp = window <= 32;
  const uint32_t threads = per_warp ? kSeqWarps * 32 : std::min<uint32_t>(kSeqThreads, (window + 31) / 32 * 32);
  const uint64_t units_per_cta = per_warp ? kSeqWarps : 1;
  uint64_t grid = std::min<uint64_t>((nwin + units_per_cta - 1) / units_per_cta, (uint64_t)num_sms * (2048 / threads));
  grid = std::max<uint64_t>(1, std::min<uint64_t>(grid, (1ULL << 30) / (slice * units_per_cta)));
  const uint64_t slices = grid * units_per_cta;
  // the slices are owned by the caller's context, grown on demand (a per-call
  // stream-ordered allocation made the timing depend on the pool's state)
  if (*scratch_bytes < slices * slice) {
    cudaError_t e = cudaStreamSynchronize(s);  // a previous call may still use the old buffer
    if (e == cudaSuccess && *scratch_buf) e = cudaFree(*scratch_buf);
    *scratch_buf = nullptr;
    *scratch_bytes = 0;
    if (e == cudaSuccess) e = cudaMalloc(scratch_buf, slices * slice);
    if (e != cudaSuccess) {
      *scratch_buf = nullptr;
      err = "scratch allocation";
      return e;
    }
    *scratch_bytes = slices * slice;
  }
  const SeqK1 K1{k1_codes, k1_xinfo, k1_xarena, k1_xcap};
  if (per_warp)
    k_seq_windows_w<<<(unsigned)grid, threads, 0, s>>>(T, b, n, window, mode, (uint8_t*)*scratch_buf, slice, cap,
                                                       out, K1);
  else
    k_seq_windows<<<(unsigned)grid, threads, 0, s>>>(T, b, n, window, mode, (uint8_t*)*scratch_buf, slice, cap, out,
                                                     K1);
  return cudaGetLastError();
}

}  // namespace picker
