// Table-driven per-descriptor helpers (shared by the exact verifier and the
// wide path) and K2: the warp-cooperative wide evaluator.
#pragma once

#include "device_common.cuh"

namespace picker {

static __device__ __forceinline__ int64_t prod_val(const Tables& T, const DKernel& K, const RecVals& X,
                                                   uint16_t j) {
  const DProd p = T.prods[K.prod + j];
  return mul64(mul64(p.k, X.get(p.a)), X.get(p.b));
}

// [lo, hi] of variable slot s: structural bounds tightened by the declared
// bound expressions.
static __device__ __forceinline__ void slot_bounds(const Tables& T, const DKernel& K, const RecVals& X,
                                                   uint16_t s, int64_t& lo, int64_t& hi) {
  const DVar v = T.vars[K.var + s];
  lo = (-9223372036854775807LL - 1);
  hi = 9223372036854775807LL;
  if (v.skind != SK_NONE) {
    const int64_t g = X.get(OPD_GX + v.axis), b = X.get(OPD_BX + v.axis);
    lo = 0;
    hi = (v.skind == SK_TID ? b : v.skind == SK_BID ? g : g * b) - 1;
  }
  auto B = [&](const DBexpr& e) {
    int64_t x = e.k0;
    if (e.p0 != kNone16) x = add64(x, prod_val(T, K, X, e.p0));
    if (e.p1 != kNone16) x = add64(x, prod_val(T, K, X, e.p1));
    return x;
  };
  for (int j = 0; j < v.nlo; ++j) lo = max64(lo, B(T.bexprs[v.bex + j]));
  for (int j = 0; j < v.nhi; ++j) hi = min64(hi, B(T.bexprs[v.bex + v.nlo + j]));
}

// guard holds and no variable range is empty
static __device__ __forceinline__ bool desc_active(const Tables& T, const DKernel& K, const DDesc& D,
                                                   const RecVals& X) {
  for (int g = 0; g < D.nguard; ++g) {
    const DGuard G = T.guards[D.guard + g];
    if (!cmp64(X.get(G.a), G.cmp, G.b == OPD_NONE ? G.bconst : X.get(G.b))) return false;
  }
  for (int v = 0; v < D.nvar; ++v) {
    int64_t lo, hi;
    slot_bounds(T, K, X, T.varlist[D.var + v], lo, hi);
    if (lo > hi) return false;
  }
  return true;
}

// byte extent [lb, ub] of a non-opaque descriptor
static __device__ void desc_extent(const Tables& T, const DKernel& K, const DDesc& D, const RecVals& X,
                                   int64_t& lb, int64_t& ub) {
  lb = D.base == OPD_NONE ? 0 : X.get(D.base);
  ub = lb;
  for (int t = 0; t < D.nterm; ++t) {
    const DTerm tm = T.terms[D.term + t];
    const int64_t c = prod_val(T, K, X, tm.prod);
    if (tm.var == kNone16) {
      lb = add64(lb, c), ub = add64(ub, c);
      continue;
    }
    int64_t lo, hi;
    slot_bounds(T, K, X, tm.var, lo, hi);
    const int64_t a = mul64(c, floordiv64(lo, tm.div)), b = mul64(c, floordiv64(hi, tm.div));
    lb = add64(lb, min64(a, b));
    ub = add64(ub, max64(a, b));
  }
  ub = add64(ub, (int64_t)D.width - 1);
}

// ---------------------------------------------------------------------------
// K2: one warp evaluates one instance with many read/write sites (SURVEY §2.5:
// cuDNN-like / multi-tensor kernels with 16+ pointer arguments).  Lanes
// compute descriptor extents in parallel; the read/write test is a sweep-line
// over the extents sorted by lower bound: an extent overlaps an extent of the
// other kind iff, in lb order, the running maximum ub of the other kind seen
// so far reaches its lb (closed byte intervals; equal lbs overlap in any
// order).  Kernels with <= 64 descriptors sort 2 x 32 extents in registers (a
// warp bitonic network); larger ones (<= kWideMax) write one element per
// descriptor into the warp's scratch (global memory, L1/L2-resident), sort it
// there with the same network (lanes over compare-exchange pairs, __syncwarp
// between stages) and sweep it 32 elements at a time with carried maxima.
// The verdict equals the pairwise definition -- checked
// against the oracle (tests: wide families, wide path forced).
// ---------------------------------------------------------------------------
struct Ext {
  int64_t lb, ub;
  uint32_t kind;  // 0 read, 1 write, 2 none (padding)
};
// scratch element: 32 bytes, two 16-byte halves
struct __align__(16) WideElem {
  int64_t lb, ub;
  uint32_t kind, pad0;
  uint64_t pad1;
};
static_assert(sizeof(WideElem) == kWideElemBytes, "scratch element layout");


static __device__ __forceinline__ Ext shfl_ext(const Ext& e, int src) {
  Ext o;
  o.lb = __shfl_sync(0xffffffffu, e.lb, src);
  o.ub = __shfl_sync(0xffffffffu, e.ub, src);
  o.kind = __shfl_sync(0xffffffffu, e.kind, src);
  return o;
}
static __device__ __forceinline__ Ext shfl_xor_ext(const Ext& e, int m) {
  Ext o;
  o.lb = __shfl_xor_sync(0xffffffffu, e.lb, m);
  o.ub = __shfl_xor_sync(0xffffffffu, e.ub, m);
  o.kind = __shfl_xor_sync(0xffffffffu, e.kind, m);
  return o;
}
static __device__ __forceinline__ bool ext_less(const Ext& a, const Ext& b) {
  // padding sorts last; order among equal lbs is irrelevant to the sweep
  return a.kind != 2 && (b.kind == 2 || a.lb < b.lb);
}

// Bitonic sort of 64 elements held as (e0 = element lane, e1 = element 32 + lane).
static __device__ __forceinline__ void warp_sort64(Ext& e0, Ext& e1, int lane) {
  for (int k = 2; k <= 64; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j == 32) {  // partner is the other register of the same lane
        const bool up = true;  // k == 64 here: the whole sequence ascends
        if (ext_less(e1, e0) == up) {
          Ext t = e0;
          e0 = e1;
          e1 = t;
        }
        continue;
      }
      // element indices i = lane (+32); partner i ^ j lives in lane ^ j, same register
      for (int h = 0; h < 2; ++h) {
        Ext& e = h ? e1 : e0;
        const int i = lane + 32 * h;
        const Ext p = shfl_xor_ext(e, j);
        const bool ascending = ((i & k) == 0);
        const bool lower = (i & j) == 0;
        // the lower index keeps the smaller (ascending) / larger (descending) element
        const bool p_smaller = ext_less(p, e);
        const bool take = lower ? (ascending ? p_smaller : ext_less(e, p)) : (ascending ? ext_less(e, p) : p_smaller);
        if (take) e = p;
      }
    }
  }
}

static __device__ __forceinline__ int64_t warp_incl_max(int64_t v, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int64_t o = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v = max64(v, o);
  }
  return v;
}

// Overlap test over the sorted 64 elements: exclusive prefix max of ub per kind.
static __device__ __forceinline__ bool sweep64(const Ext& e0, const Ext& e1, int lane) {
  const int64_t NEG = (-9223372036854775807LL - 1);
  bool hit = false;
  int64_t carry_r = NEG, carry_w = NEG;
  for (int h = 0; h < 2; ++h) {
    const Ext& e = h ? e1 : e0;
    const int64_t vr = e.kind == 0 ? e.ub : NEG, vw = e.kind == 1 ? e.ub : NEG;
    const int64_t ir = max64(warp_incl_max(vr, lane), carry_r), iw = max64(warp_incl_max(vw, lane), carry_w);
    int64_t xr = __shfl_up_sync(0xffffffffu, ir, 1), xw = __shfl_up_sync(0xffffffffu, iw, 1);
    if (lane == 0) xr = carry_r, xw = carry_w;
    if (e.kind == 0 && xw >= e.lb) hit = true;  // a write before it reaches its first byte
    if (e.kind == 1 && xr >= e.lb) hit = true;
    carry_r = __shfl_sync(0xffffffffu, ir, 31);
    carry_w = __shfl_sync(0xffffffffu, iw, 31);
  }
  return __any_sync(0xffffffffu, hit);
}

// Activity and (non-opaque) extent of one descriptor, each variable's bounds
// evaluated once (desc_active + desc_extent re-evaluate them per term).
constexpr int kWideVars = 8;
static __device__ bool desc_active_extent(const Tables& T, const DKernel& K, const DDesc& D, const RecVals& X,
                                          int64_t& lb, int64_t& ub) {
  for (int g = 0; g < D.nguard; ++g) {
    const DGuard G = T.guards[D.guard + g];
    if (!cmp64(X.get(G.a), G.cmp, G.b == OPD_NONE ? G.bconst : X.get(G.b))) return false;
  }
  if (D.nvar > kWideVars) {
    if (!desc_active(T, K, D, X)) return false;
    if (!D.opaque) desc_extent(T, K, D, X, lb, ub);
    return true;
  }
  int64_t vlo[kWideVars], vhi[kWideVars];
  for (int v = 0; v < D.nvar; ++v) {
    slot_bounds(T, K, X, T.varlist[D.var + v], vlo[v], vhi[v]);
    if (vlo[v] > vhi[v]) return false;
  }
  if (D.opaque) return true;
  lb = D.base == OPD_NONE ? 0 : X.get(D.base);
  ub = lb;
  for (int t = 0; t < D.nterm; ++t) {
    const DTerm tm = T.terms[D.term + t];
    const int64_t c = prod_val(T, K, X, tm.prod);
    if (tm.var == kNone16) {
      lb = add64(lb, c), ub = add64(ub, c);
      continue;
    }
    const int lv = T.term_lvar[D.term + t];
    const int64_t x0 = mul64(c, floordiv64(vlo[lv], tm.div)), x1 = mul64(c, floordiv64(vhi[lv], tm.div));
    lb = add64(lb, min64(x0, x1));
    ub = add64(ub, max64(x0, x1));
  }
  ub = add64(ub, (int64_t)D.width - 1);
  return true;
}

// Scratch layout of the > 64-descriptor path (16-byte intervals):
//   S[0, ns2)   the smaller kind's extents, sorted by lb (ns2 = pow2 >= 32;
//               padding lb = INT64_MAX), then their exclusive-of-nothing
//   M[0, ns2)   prefix maxima of ub in that order (int64),
//   L[0, nl)    the other kind's extents.
// An extent x of the larger kind overlaps some sorted extent iff, for the
// last sorted index i with lb_i <= x.ub, max(ub_0..ub_i) >= x.lb (closed
// intervals) -- the sweep line's running maximum, read by binary search.
struct Iv64 {
  int64_t lb, ub;
};

// Bitonic sort of S[0, n2) by lb, ascending (n2 a power of two >= 32).
static __device__ void iv_sort(Iv64* S, uint32_t n2, int lane) {
  for (uint32_t k = 2; k <= n2; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t p = lane; p < n2 / 2; p += 32) {  // pair p: index with bit j cleared, partner | j
        const uint32_t i = ((p & ~(j - 1)) << 1) | (p & (j - 1)), q = i | j;
        const Iv64 a = S[i], b = S[q];
        const bool swap = ((i & k) == 0) ? b.lb < a.lb : a.lb < b.lb;
        if (swap) S[i] = b, S[q] = a;
      }
      __syncwarp();
    }
  }
}

// Does any of the nl extents L overlap one of the sorted extents S (prefix
// maxima M)?  Lanes over L, binary search in S.
static __device__ bool iv_probe(const Iv64* S, const int64_t* M, uint32_t n2, const Iv64* L, uint32_t nl,
                                int lane) {
  bool hit = false;
  for (uint32_t x = lane; x < nl; x += 32) {
    const Iv64 e = L[x];
    // last index i with S[i].lb <= e.ub (padding sorts last with lb = INT64_MAX)
    int lo = -1;
    for (uint32_t step = n2 >> 1; step > 0; step >>= 1)
      if (S[lo + (int)step].lb <= e.ub) lo += (int)step;
    if (lo + 1 < (int)n2 && S[lo + 1].lb <= e.ub) ++lo;
    if (lo >= 0 && M[lo] >= e.lb) hit = true;
  }
  return __any_sync(0xffffffffu, hit);
}

// Prefix maxima of ub over the sorted S (32 at a time, carried).
static __device__ void iv_prefix_max(const Iv64* S, int64_t* M, uint32_t n2, int lane) {
  int64_t carry = (-9223372036854775807LL - 1);
  for (uint32_t h = 0; h < n2; h += 32) {
    const int64_t v = max64(warp_incl_max(S[h + lane].ub, lane), carry);
    M[h + lane] = v;
    carry = __shfl_sync(0xffffffffu, v, 31);
  }
  __syncwarp();
}

// Verdict of one record, computed by the whole warp (all lanes return it).
// `scratch`: this warp's `cap` elements (shared or global memory; nullptr:
// pairwise for > 64 descriptors).
static __device__ uint8_t eval_wide_warp(const Tables& T, const picker_rec_t& r, const int64_t* a,
                                         uint64_t alo, uint64_t ahi, int lane, WideElem* scratch,
                                         uint32_t cap = kWideMax) {
  // prefix (Fig. 3 order); the preconditions / global condition are split over
  // the lanes: the first failing check in order decides (pre before glob)
  const uint32_t kid = r.kernel_id;
  if (kid >= T.nkernel_slots) return V_ERR_KERNEL;
  const DKernel K = T.kernels[kid];
  if (K.shortcut == V_ERR_KERNEL) return V_ERR_KERNEL;
  if (!args_in_range(r, K.nparams, alo, ahi)) return V_ERR_ARITY;
  if (K.shortcut) return K.shortcut;
  const RecVals X(r, a, K.i32mask);
  if (!launch_limits_ok(X)) return V_NI_PRECOND;
  int first_fail = 0x7FFFFFFF;
  for (int c = lane; c < K.npre + K.nglob; c += 32) {
    const DCheck ch = T.checks[K.check + c];
    const int64_t v = X.get(ch.op);
    if (v < ch.lo || v > ch.hi) {
      first_fail = c;
      break;
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) first_fail = min(first_fail, __shfl_xor_sync(0xffffffffu, first_fail, d));
  if (first_fail != 0x7FFFFFFF) return first_fail < K.npre ? V_NI_PRECOND : V_NI_GLOBAL;
  // per-lane descriptors d = lane, lane + 32, ...: activity, opaque flags,
  // extents (registers for <= 64 descriptors, else element d of the scratch)
  const bool in_regs = K.ndesc <= 64;
  // > 64 descriptors: the smaller kind sorted in the scratch (+ prefix
  // maxima), the larger kind probed against it; bytes needed: 16 per extent +
  // 24 per padded sorted slot
  const uint32_t cap_bytes = cap * (uint32_t)sizeof(WideElem);
  const uint32_t ns_max = min((uint32_t)K.nr, (uint32_t)K.nw);
  const uint32_t n2 = max(32u, 1u << (32 - __clz(max(ns_max, 1u) - 1)));
  const bool in_scratch = !in_regs && scratch != nullptr &&
                          (uint64_t)n2 * 24 + (uint64_t)(K.nr + K.nw) * 16 <= cap_bytes;
  const bool sort_w = K.nw <= K.nr;  // the sorted side (per kernel: warp-uniform)
  Iv64* S = reinterpret_cast<Iv64*>(scratch);
  int64_t* M = reinterpret_cast<int64_t*>(S + n2);
  Iv64* L = reinterpret_cast<Iv64*>(M + n2);
  bool act_r = false, act_w = false, opq_r = false, opq_w = false;
  Ext e[2];
  e[0].kind = e[1].kind = 2;
  e[0].lb = e[0].ub = e[1].lb = e[1].ub = 0;
  uint32_t ns = 0, nl = 0;  // compacted counts (warp-uniform)
#pragma unroll 2
  for (int d0 = 0, k = 0; d0 < K.ndesc; d0 += 32, ++k) {
    const int d = d0 + lane;
    bool have = false, is_r = false;
    int64_t lb = 0, ub = 0;
    if (d < K.ndesc) {
      const DDesc D = T.descs[K.desc + d];
      if (desc_active_extent(T, K, D, X, lb, ub)) {
        (D.kind == KIND_R ? act_r : act_w) = true;
        if (D.opaque)
          (D.kind == KIND_R ? opq_r : opq_w) = true;
        else
          have = true, is_r = D.kind == KIND_R;
      }
    }
    if (in_scratch) {  // compact into the sorted side / the probed side
      const bool to_s = have && (is_r != sort_w);
      const unsigned ms = __ballot_sync(0xffffffffu, to_s), ml = __ballot_sync(0xffffffffu, have && !to_s);
      const unsigned lt = (1u << lane) - 1u;
      if (to_s) S[ns + __popc(ms & lt)] = Iv64{lb, ub};
      if (have && !to_s) L[nl + __popc(ml & lt)] = Iv64{lb, ub};
      ns += __popc(ms), nl += __popc(ml);
    } else if (k < 2 && have) {
      e[k].lb = lb, e[k].ub = ub, e[k].kind = is_r ? 0u : 1u;
    }
  }
  act_r = __any_sync(0xffffffffu, act_r);
  act_w = __any_sync(0xffffffffu, act_w);
  opq_r = __any_sync(0xffffffffu, opq_r);
  opq_w = __any_sync(0xffffffffu, opq_w);
  if ((opq_r && act_w) || (opq_w && act_r)) return V_NI_OPAQUE;
  if (in_regs) {
    // element index of e[0] is lane, of e[1] is 32 + lane
    warp_sort64(e[0], e[1], lane);
    return sweep64(e[0], e[1], lane) ? V_NI_OVERLAP : V_IDEM_CHECKED;
  }
  if (in_scratch) {
    if (ns == 0 || nl == 0) {
      __syncwarp();
      return V_IDEM_CHECKED;
    }
    const uint32_t m2 = max(32u, 1u << (32 - __clz(ns - 1)));  // <= n2
    for (uint32_t x = ns + lane; x < m2; x += 32)
      S[x] = Iv64{9223372036854775807LL, (-9223372036854775807LL - 1)};  // padding sorts last, never reaches
    __syncwarp();
    iv_sort(S, m2, lane);
    iv_prefix_max(S, M, m2, lane);
    const bool hit = iv_probe(S, M, m2, L, nl, lane);
    __syncwarp();  // the scratch is reused by the warp's next record
    return hit ? V_NI_OVERLAP : V_IDEM_CHECKED;
  }
  // beyond the scratch: lanes over all (read, write) descriptor pairs
  const int nd = K.ndesc;
  bool hit = false;
  for (int p = lane; p < nd * nd && !__any_sync(__activemask(), hit); p += 32) {
    const int i = p / nd, j = p % nd;
    const DDesc Di = T.descs[K.desc + i], Dj = T.descs[K.desc + j];
    if (Di.kind != KIND_R || Dj.kind != KIND_W || Di.opaque || Dj.opaque) continue;
    if (!desc_active(T, K, Di, X) || !desc_active(T, K, Dj, X)) continue;
    int64_t rl, ru, wl, wu;
    desc_extent(T, K, Di, X, rl, ru);
    desc_extent(T, K, Dj, X, wl, wu);
    if (rl <= wu && wl <= ru) hit = true;
  }
  return __any_sync(0xffffffffu, hit) ? V_NI_OVERLAP : V_IDEM_CHECKED;
}

}  // namespace picker
