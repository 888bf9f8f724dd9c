// Row f1's window logic (Q23), shared by the standalone window
// kernels (k_seq.cu) and the extents module's pipelined kernel, which decides
// each tile's windows from the extents its shapes put in shared memory.
#pragma once

#include "desc_eval.cuh"

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
  uint64_t base;          // record index of element 0 of the arrays (a tile in shared memory)
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
      const uint64_t ki = w0 + i - K1.base;
      const uint32_t c = K1.codes[ki];
      if (c >= V_NI_SO && c != V_NI_OPAQUE && c != V_NI_OVERLAP) {
        status = (uint8_t)c;
      } else if (c != V_IDEM_KERNEL) {
        const uint32_t info = K1.xinfo[ki];
        const uint32_t nr = info & 0x7FFu, nw = (info >> 11) & 0x7FFu;
        fl = (uint8_t)(info >> 22);
        const int64_t* x = K1.xarena + ki * 2 * K1.xcap;
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

// A window of <= 32 launches decided by one warp: lane i is launch w0 + i,
// with its slot of xcap (lb, ub) pairs (reads from the front, writes from the
// back) and info word.  Extents module (xinfo set): the slots are the tile's in
// shared memory, filled by K1's shapes.  Lazy (xinfo null, `undecided` set):
// the slots are the warp's scratch, filled from the tables only when no
// decisive record decides the window.  Same decisions as seq_window (Q23): the
// first decisive code; records K1 did not evaluate (1, kernel-level
// idempotent) are evaluated from the tables into their own slot (they take
// part with their writes; their checks may decide); the opaque rule on ballots
// (sequential: an opaque read of i and a write of j >= i is the lowest set bit
// of one ballot at or below the highest of the other); then every (read of i,
// write of j) pair, i <= j sequential, any i, j concurrent -- the writes of j
// broadcast, each lane's reads against them.
__device__ __forceinline__ void seq_lane_tables(const Tables& T, const DevBatch& B, uint64_t rec, int64_t* x,
                                                uint32_t xcap, uint32_t& status, uint32_t& info) {
  const picker_rec_t r = load_rec(B.rec + rec);
  const uint32_t kid = r.kernel_id;
  do {
    if (kid >= T.nkernel_slots || T.kernels[kid].shortcut == V_ERR_KERNEL) {
      status = V_ERR_KERNEL;
      break;
    }
    const DKernel K = T.kernels[kid];
    if (!args_in_range(r, K.nparams, B.args_lo, B.args_hi)) {
      status = V_ERR_ARITY;
      break;
    }
    if (K.shortcut && K.shortcut != V_IDEM_KERNEL) {
      status = K.shortcut;
      break;
    }
    const RecVals X(r, B.args + r.arg_off, K.i32mask);
    if (!launch_limits_ok(X)) {
      status = V_NI_PRECOND;
      break;
    }
    for (int q = 0; q < K.npre + K.nglob && status == kEvaluable; ++q) {
      const DCheck ch = T.checks[K.check + q];
      const int64_t v = X.get(ch.op);
      if (v < ch.lo || v > ch.hi) status = q < K.npre ? V_NI_PRECOND : V_NI_GLOBAL;
    }
    if (status != kEvaluable) break;
    uint32_t nr = 0, nw = 0, fl = 0;
    for (int d = 0; d < K.ndesc; ++d) {
      const DDesc D = T.descs[K.desc + d];
      int64_t lb = 0, ub = 0;
      if (!desc_active_extent(T, K, D, X, lb, ub)) continue;
      fl |= D.kind == KIND_R ? 1u : 2u;
      if (D.opaque) {
        fl |= D.kind == KIND_R ? 4u : 8u;
        continue;
      }
      const uint32_t k = D.kind == KIND_R ? nr++ : xcap - 1 - nw++;
      x[2 * k] = lb, x[2 * k + 1] = ub;
    }
    info = nr | nw << 11 | fl << 22;
  } while (false);
}

__device__ __forceinline__ uint8_t seq_window_lanes(const Tables& T, const DevBatch& B, uint64_t w0, uint32_t m,
                                                    uint32_t mode, const uint8_t* codes, const uint32_t* xinfo,
                                                    int64_t* xext, uint32_t xcap, int lane, bool* undecided) {
  constexpr unsigned kAll = 0xffffffffu;
  const bool in = (uint32_t)lane < m;
  uint32_t status = kEvaluable, info = 0, c = 0;
  int64_t* x = xext + (size_t)lane * 2 * xcap;
  if (in) {
    c = codes[lane];
    if (c >= V_NI_SO && c != V_NI_OPAQUE && c != V_NI_OVERLAP) status = c;
    else if (c != V_IDEM_KERNEL && xinfo) info = xinfo[lane];
  }
  // records before the first decisive one that K1 did not evaluate (1): their
  // checks may decide earlier, and they take part with their writes -- only
  // those are evaluated from the tables (all of them in an undecided window)
  const uint32_t first0 = __reduce_min_sync(kAll, (in && status != kEvaluable) ? ((uint32_t)lane << 8 | status) : kAll);
  if (in && c == V_IDEM_KERNEL && (uint32_t)lane < (first0 >> 8)) seq_lane_tables(T, B, w0 + lane, x, xcap, status, info);
  const uint32_t first = __reduce_min_sync(kAll, (in && status != kEvaluable) ? ((uint32_t)lane << 8 | status) : kAll);
  if (first != kAll) return (uint8_t)(first & 0xFF);
  if (!xinfo) {  // lazy: the records K1 passed to the address check (0, 9, 10), from the tables
    *undecided = true;
    if (in && c != V_IDEM_KERNEL) seq_lane_tables(T, B, w0 + lane, x, xcap, status, info);
  }
  const uint32_t fl = info >> 22;
  const unsigned br = __ballot_sync(kAll, fl & 1), bw = __ballot_sync(kAll, fl & 2);
  const unsigned bor = __ballot_sync(kAll, fl & 4), bow = __ballot_sync(kAll, fl & 8);
  if (mode == 0) {
    if ((bor && bw && __ffs(bor) - 1 <= 31 - __clz(bw)) || (br && bow && __ffs(br) - 1 <= 31 - __clz(bow)))
      return V_NI_OPAQUE;
  } else if ((bor && bw) || (br && bow)) {
    return V_NI_OPAQUE;
  }
  const uint32_t nr = info & 0x7FFu, nw = (info >> 11) & 0x7FFu;
  if (!__any_sync(kAll, nr != 0) || !__any_sync(kAll, nw != 0)) return V_IDEM_CHECKED;
  __syncwarp();  // the slots written above, visible to the warp
  // the lane's first reads in registers
  int64_t rl[4], ru[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    rl[q] = (uint32_t)q < nr ? x[2 * q] : 1, ru[q] = (uint32_t)q < nr ? x[2 * q + 1] : 0;  // empty when absent
  }
  bool hit = false;
  for (uint32_t j = 0; j < m; ++j) {
    const uint32_t nwj = __shfl_sync(kAll, nw, j);
    const bool mine = nr != 0 && (mode == 1 || (uint32_t)lane <= j);
    const int64_t* xj = xext + (size_t)j * 2 * xcap;
    for (uint32_t k = 0; k < nwj; ++k) {
      const longlong2 w = *reinterpret_cast<const longlong2*>(xj + 2 * (xcap - 1 - k));  // broadcast
      if (mine) {
#pragma unroll
        for (int q = 0; q < 4; ++q) hit |= rl[q] <= w.y && w.x <= ru[q];
        for (uint32_t q = 4; q < nr; ++q) hit |= x[2 * q] <= w.y && w.x <= x[2 * q + 1];
      }
    }
    if ((j & 3) == 3 || j + 1 == m)
      if (__any_sync(kAll, hit)) return V_NI_OVERLAP;
  }
  return V_IDEM_CHECKED;
}

}  // namespace picker
