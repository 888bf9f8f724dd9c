// K2 as its own persistent kernel: summaries whose evaluating kernels are all
// wide (many pointer arguments: multi-tensor-apply optimizers, foreach ops,
// multi-tensor norms -- SURVEY §8 row a8, BASELINE configs[3]).
//
// One warp evaluates one instance (north_star: "one warp evaluates one
// instance"), the R/W test is a sort + sweep over its extents (PAPER.md
// l.658-666: NI iff an active read extent and an active write extent share a
// byte, regardless of order).  Per warp, in shared memory:
//   - two argument buffers: while record i is evaluated, record i+1's argument
//     span (<= 247 slots) streams in with 16-byte cp.async (lanes over the
//     chunks) and record i+2's header is loaded; every operand of a record is
//     then one shared load: the buffer holds the 6 launch dimensions, 1 and 0
//     in the 8 slots before the arguments, so operand code `op` is ops[op];
//   - the record's products (lanes over them: k * X[a] * X[b], P:1088-1090
//     "common expression extraction") and variable ranges (lanes over the
//     kernel's variable slots: structural bounds tightened by the declared
//     bounds, induction P:1063, fresh P:990-992), each computed
//     once per record instead of once per descriptor;
//   - the extents (lanes over descriptors, one 32-byte DWDesc load each;
//     P:933-951 LB/UB at the variables' extreme values), compacted by kind;
//   - the sort + sweep: the smaller kind in chunks of 64, each chunk sorted by
//     lb in registers (warp bitonic network; skipped when the chunk is already
//     in order), its prefix maxima of ub (the sweep line's running maximum)
//     written to shared memory, every extent of the other kind probed by binary
//     search: x overlaps some chunk element iff, at the last element with
//     lb <= x.ub, the running maximum ub >= x.lb (closed byte intervals).
// Warps take 32-record chunks of the batch (static stride) and emit their codes,
// idempotent bit word and histogram themselves: no sort of records, no CTA
// barrier in the loop.  Kernels beyond the workspace (more than kWExt
// descriptors, kWProd products or kWVar variable slots) take the round-1
// warp evaluator (eval_wide_warp, global scratch).
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/picker.h"
#include "k_bucket.cuh"
#include "launch.hpp"

namespace picker {

constexpr int kWideWarps = 8, kWideCtas = 2;
constexpr int kWProd = 192, kWVar = 64, kWExt = 320;
constexpr int kWArgBuf = 64 + 2048 + 16;  // 8 operand slots + a 16-byte-rounded span of <= 248 slots
constexpr int64_t kI64Min = (-9223372036854775807LL - 1), kI64Max = 9223372036854775807LL;

struct __align__(16) WideWarpSmem {
  unsigned char args[2][kWArgBuf];
  int64_t pv[kWProd];
  int64_t vlo[kWVar], vhi[kWVar];
  Iv64 ext[kWExt];  // reads from the front, writes from the back
  union {
    struct {
      int64_t lo[kWideSigs], hi[kWideSigs];  // summed term offsets per signature
      uint8_t act[kWideSigs];                // activity per signature
    } s;
    Iv64 chunk[64];  // after the descriptors: one sorted chunk (lb, prefix max of ub)
  } sg;
};
static_assert(sizeof(WideWarpSmem) % 16 == 0, "warp workspace alignment");
constexpr size_t kWideSmem = sizeof(WideWarpSmem) * kWideWarps;

// --- warp sort of 64 keys (lb) with their element index as payload (k0, x0 =
// element lane, k1, x1 = element 32 + lane); branch-free compare-exchange, the
// ub of an element is read back through its index after the sort.  Equal keys
// are never exchanged (both partners compare strictly), so no element is lost.
// take the partner's element iff keys differ and (partner < own) == keep_small
__device__ __forceinline__ void cx64(int64_t& k, uint32_t& x, int j, uint32_t keep_small) {
  const int64_t pk = __shfl_xor_sync(0xffffffffu, k, j);
  const uint32_t px = __shfl_xor_sync(0xffffffffu, x, j);
  asm("{\n\t.reg .pred lt, ne, ks, t;\n\t"
      "setp.lt.s64 lt, %2, %0;\n\t"
      "setp.ne.s64 ne, %2, %0;\n\t"
      "setp.ne.u32 ks, %4, 0;\n\t"
      "xor.pred t, lt, ks;\n\t"
      "not.pred t, t;\n\t"
      "and.pred t, t, ne;\n\t"
      "selp.b64 %0, %2, %0, t;\n\t"
      "selp.b32 %1, %3, %1, t;\n\t}"
      : "+l"(k), "+r"(x)
      : "l"(pk), "r"(px), "r"(keep_small));
}
struct Sort64 {
  int64_t k0, k1;
  uint32_t x0, x1;
};
// Out of line: the caller branches around it when the chunk is in order (an
// inlined copy was if-converted into straight-line code that always ran).
__device__ __noinline__ Sort64 warp_sort64_key(Sort64 s, int lane) {
#pragma unroll
  for (int k = 2; k <= 64; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j == 32) {  // k == 64: the other register of the same lane, ascending
        const bool sw = s.k1 < s.k0;
        const int64_t tk = s.k0;
        const uint32_t tx = s.x0;
        s.k0 = sw ? s.k1 : s.k0, s.x0 = sw ? s.x1 : s.x0;
        s.k1 = sw ? tk : s.k1, s.x1 = sw ? tx : s.x1;
        continue;
      }
      // ascending block: the lower index keeps the smaller key
      const uint32_t lower = (lane & j) == 0;
      cx64(s.k0, s.x0, j, ((lane & k) == 0) == lower);
      cx64(s.k1, s.x1, j, (((lane + 32) & k) == 0) == lower);
    }
  }
  return s;
}

// Is the 64-element chunk (k0 | k1) already in key order?
__device__ __forceinline__ bool chunk_sorted(int64_t k0, int64_t k1, int lane) {
  const int64_t n0 = __shfl_down_sync(0xffffffffu, k0, 1), n1 = __shfl_down_sync(0xffffffffu, k1, 1);
  const int64_t f1 = __shfl_sync(0xffffffffu, k1, 0);
  const bool ok = (lane < 31 ? k0 <= n0 : k0 <= f1) && (lane < 31 ? k1 <= n1 : true);
  return __all_sync(0xffffffffu, ok);
}

// Any of the nl extents L overlapping the sorted chunk C (lb, prefix max ub)?
// Padding elements sort last (lb = INT64_MAX, ub = INT64_MIN) and never raise
// the prefix maximum, so the search may run over all 64 entries.
__device__ __forceinline__ bool probe_chunk(const Iv64* C, const Iv64* L, int nl, int lane) {
  bool hit = false;
  for (int x = lane; x < nl; x += 32) {
    const Iv64 e = L[x];
    int pos = -1;
#pragma unroll
    for (int s = 32; s > 0; s >>= 1)
      if (C[pos + s].lb <= e.ub) pos += s;
    if (pos >= 0 && C[pos].ub >= e.lb) hit = true;
  }
  return __any_sync(0xffffffffu, hit);
}

// Verdict of one record (warp-uniform) from its staged operands `ops`
// (ops[op] = value of operand code op, i32 parameters already sign-extended).
__device__ __forceinline__ uint8_t eval_wide_ws(const Tables& T, const DKernel& K, const int64_t* ops, WideWarpSmem& W,
                                int lane) {
  // preconditions and global condition, split over the lanes: the first
  // failing check in order decides (pre before glob)
  // (no early exit: the loop unrolls and its table loads overlap)
  int first_fail = 0x7FFFFFFF;
  const int nchk = K.npre + K.nglob;
#pragma unroll 4
  for (int c = nchk - 1 - lane; c >= 0; c -= 32) {  // descending: the last failure seen is the first
    const DCheck ch = T.checks[K.check + c];
    const int64_t v = ops[ch.op];
    if (v < ch.lo || v > ch.hi) first_fail = c;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) first_fail = min(first_fail, __shfl_xor_sync(0xffffffffu, first_fail, d));
  if (first_fail != 0x7FFFFFFF) return first_fail < K.npre ? V_NI_PRECOND : V_NI_GLOBAL;

  // products, then variable ranges
  for (int j = lane; j < K.nprod; j += 32) {
    const DProd p = T.prods[K.prod + j];
    W.pv[j] = mul64(mul64(p.k, ops[p.a]), ops[p.b]);
  }
  __syncwarp();
  auto bex = [&](const DBexpr& e) {
    int64_t x = e.k0;
    if (e.p0 != kNone16) x = add64(x, W.pv[e.p0]);
    if (e.p1 != kNone16) x = add64(x, W.pv[e.p1]);
    return x;
  };
  for (int s = lane; s < K.nvar; s += 32) {
    const DVar v = T.vars[K.var + s];
    int64_t lo = kI64Min, hi = kI64Max;
    if (v.skind != SK_NONE) {
      const int64_t g = ops[OPD_GX + v.axis], b = ops[OPD_BX + v.axis];
      lo = 0;
      hi = (v.skind == SK_TID ? b : v.skind == SK_BID ? g : g * b) - 1;
    }
    for (int j = 0; j < v.nlo; ++j) lo = max64(lo, bex(T.bexprs[v.bex + j]));
    for (int j = 0; j < v.nhi; ++j) hi = min64(hi, bex(T.bexprs[v.bex + v.nlo + j]));
    W.vlo[s] = lo, W.vhi[s] = hi;
  }
  __syncwarp();

  // extents, compacted by kind
  auto term = [&](uint16_t prod, uint16_t var, uint32_t div, int64_t& lb, int64_t& ub) {
    const int64_t c = W.pv[prod];
    if (var == kNone16) {
      lb = add64(lb, c), ub = add64(ub, c);
      return;
    }
    const int64_t x0 = mul64(c, floordiv64(W.vlo[var], div)), x1 = mul64(c, floordiv64(W.vhi[var], div));
    lb = add64(lb, min64(x0, x1));
    ub = add64(ub, max64(x0, x1));
  };
  // signatures (activity + summed term offsets shared by descriptors): lanes over them
  for (int g = lane; g < K.nsig; g += 32) {
    const uint4* sp = reinterpret_cast<const uint4*>(T.wsigs + K.desc + g);
    const uint4 s0 = __ldg(sp), s1 = __ldg(sp + 1);
    const uint32_t vs0 = s0.x & 0xFFFFu, vs1 = s0.x >> 16;
    bool on = true;
    if (vs0 != kNone16) on = W.vlo[vs0] <= W.vhi[vs0];
    if (vs1 != kNone16) on = on && W.vlo[vs1] <= W.vhi[vs1];
    int64_t lo = 0, hi = 0;
    const uint32_t tp0 = s0.y & 0xFFFFu, tp1 = s0.y >> 16, tv0 = s0.z & 0xFFFFu, tv1 = s0.z >> 16;
    if (tp0 != kNone16) term((uint16_t)tp0, (uint16_t)tv0, s0.w, lo, hi);
    if (tp1 != kNone16) term((uint16_t)tp1, (uint16_t)tv1, s1.x, lo, hi);
    W.sg.s.act[g] = on;
    W.sg.s.lo[g] = lo, W.sg.s.hi[g] = hi;
  }
  __syncwarp();

  bool act_r = false, act_w = false, opq_r = false, opq_w = false;
  int nr = 0, nw = 0;
  const unsigned lt = (1u << lane) - 1u;
  // one descriptor per lane and round (one 16-byte load, issued a round ahead)
  const uint4* wd = reinterpret_cast<const uint4*>(T.wdescs + K.desc);
  uint4 q = make_uint4(0, 0, 0, 0);
  if (lane < K.ndesc) q = __ldg(wd + lane);
  for (int d0 = 0; d0 < K.ndesc; d0 += 32) {
    const int d = d0 + lane;
    const uint4 w = q;
    if (d + 32 < K.ndesc) q = __ldg(wd + d + 32);
    bool have = false, is_r = false;
    int64_t lb = 0, ub = 0;
    if (d < K.ndesc) {
      // DWDesc: kind, opaque, base, mode | a, b | wm1
      const uint32_t kind = w.x & 0xFFu, opaque = (w.x >> 8) & 0xFFu, base = (w.x >> 16) & 0xFFu, mode = w.x >> 24;
      const uint32_t ia = w.y & 0xFFFFu, ib = w.y >> 16;
      bool on = true;
      if (mode == WD_SIG) {
        on = W.sg.s.act[ia];
        const int64_t b0 = ops[base];  // ops[OPD_NONE] = 0
        lb = add64(b0, W.sg.s.lo[ia]);
        ub = add64(add64(b0, W.sg.s.hi[ia]), (int64_t)w.z);
      } else if (mode == WD_CONST) {
        int64_t c = ops[base];
        if (ia != kNone16) c = add64(c, W.pv[ia]);
        if (ib != kNone16) c = add64(c, W.pv[ib]);
        lb = c, ub = add64(c, (int64_t)w.z);
      } else {  // guards, > 2 variables or > 2 terms: the full tables
        const DDesc D = T.descs[K.desc + d];
        for (int g = 0; g < D.nguard && on; ++g) {
          const DGuard G = T.guards[D.guard + g];
          on = cmp64(ops[G.a], G.cmp, G.b == OPD_NONE ? G.bconst : ops[G.b]);
        }
        for (int v = 0; v < D.nvar && on; ++v) {
          const uint16_t s = T.varlist[D.var + v];
          on = W.vlo[s] <= W.vhi[s];
        }
        if (on && !D.opaque) {
          lb = ops[D.base];
          ub = lb;
          for (int t = 0; t < D.nterm; ++t) {
            const DTerm tm = T.terms[D.term + t];
            term(tm.prod, tm.var, tm.div, lb, ub);
          }
          ub = add64(ub, (int64_t)D.width - 1);
        }
      }
      if (on) {
        (kind == KIND_R ? act_r : act_w) = true;
        if (opaque)
          (kind == KIND_R ? opq_r : opq_w) = true;
        else
          have = true, is_r = kind == KIND_R;
      }
    }
    const unsigned mr = __ballot_sync(0xffffffffu, have && is_r), mw = __ballot_sync(0xffffffffu, have && !is_r);
    if (have && is_r) W.ext[nr + __popc(mr & lt)] = Iv64{lb, ub};
    if (have && !is_r) W.ext[kWExt - 1 - (nw + __popc(mw & lt))] = Iv64{lb, ub};
    nr += __popc(mr), nw += __popc(mw);
  }
  act_r = __any_sync(0xffffffffu, act_r);
  act_w = __any_sync(0xffffffffu, act_w);
  opq_r = __any_sync(0xffffffffu, opq_r);
  opq_w = __any_sync(0xffffffffu, opq_w);
  // opaque rule: an opaque access of one kind with any active
  // access of the other kind
  if ((opq_r && act_w) || (opq_w && act_r)) return V_NI_OPAQUE;
  if (nr == 0 || nw == 0) return V_IDEM_CHECKED;
  __syncwarp();

  // sort + sweep: the smaller kind in chunks of 64 against the other kind
  const bool sort_r = nr < nw;
  // element e of the sorted side in descriptor order (writes were compacted
  // from the back: e-th write at ext[kWExt - 1 - e]), so summaries whose
  // accesses are already in address order skip the sort
  const Iv64* S = sort_r ? W.ext : W.ext + (kWExt - 1);
  const int sdir = sort_r ? 1 : -1;
  const Iv64* L = sort_r ? W.ext + (kWExt - nw) : W.ext;
  const int ns = sort_r ? nr : nw, nl = sort_r ? nw : nr;
  for (int h = 0; h < ns; h += 64) {
    // padding: key INT64_MAX (sorts last), ub INT64_MIN (never raises the maximum)
    const int m = min(64, ns - h);
    int64_t k0 = lane < m ? S[sdir * (h + lane)].lb : kI64Max;
    int64_t k1 = 32 + lane < m ? S[sdir * (h + 32 + lane)].lb : kI64Max;
    uint32_t x0 = lane, x1 = 32 + lane;
    if (!chunk_sorted(k0, k1, lane)) {
      const Sort64 s = warp_sort64_key(Sort64{k0, k1, x0, x1}, lane);
      k0 = s.k0, k1 = s.k1, x0 = s.x0, x1 = s.x1;
    }
    const int64_t u0 = (int)x0 < m ? S[sdir * (h + (int)x0)].ub : kI64Min;
    const int64_t u1 = (int)x1 < m ? S[sdir * (h + (int)x1)].ub : kI64Min;
    const Iv64 e0{k0, u0}, e1{k1, u1};
    const int64_t m0 = warp_incl_max(e0.ub, lane);
    const int64_t m1 = max64(warp_incl_max(e1.ub, lane), __shfl_sync(0xffffffffu, m0, 31));
    __syncwarp();  // the previous chunk's probes are done
    W.sg.chunk[lane] = Iv64{e0.lb, m0};
    W.sg.chunk[32 + lane] = Iv64{e1.lb, m1};
    __syncwarp();
    if (probe_chunk(W.sg.chunk, L, nl, lane)) return V_NI_OVERLAP;
  }
  return V_IDEM_CHECKED;
}

// Kernels beyond the workspace: the round-1 warp evaluator, out of line (its
// code stays out of the hot loop's instruction stream).
__device__ __noinline__ uint8_t wide_fallback(const Tables& T, const picker_rec_t r, const int64_t* a, uint64_t alo,
                                              uint64_t ahi, int lane, WideElem* scratch) {
  return eval_wide_warp(T, r, a, alo, ahi, lane, scratch);
}

// Start the copy of a record's argument span into `buf` (lanes over 16-byte
// chunks; 8-byte copies when the rounded span would leave the pool).  Records
// with a span outside the pool or longer than the buffer are not staged: they
// fail the arity check before any operand is read.  Returns the 8-byte shift
// of the first argument inside the span (0 or 1).
__device__ __forceinline__ uint32_t stage_span(const DevBatch& B, uint64_t arg_off, uint32_t nargs,
                                               unsigned char* buf, int lane) {
  const bool in_pool = arg_off >= B.args_lo && arg_off <= B.args_hi && (uint64_t)nargs <= B.args_hi - arg_off;
  if (!in_pool || nargs > (uint32_t)kMaxParams + 1) return 0;
  const uintptr_t a0 = (uintptr_t)(B.args + arg_off), a1 = a0 + 8ull * nargs;
  const uintptr_t c0 = a0 & ~(uintptr_t)15, c1 = (a1 + 15) & ~(uintptr_t)15;
  const uintptr_t p0 = (uintptr_t)(B.args + B.args_lo), p1 = (uintptr_t)(B.args + B.args_hi);
  const uint32_t dst = smem_u32(buf + 64);
  if (c0 >= p0 && c1 <= p1) {
    for (uintptr_t c = c0 + 16 * lane; c < c1; c += 16 * 32)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + (uint32_t)(c - c0)), "l"(c) : "memory");
  } else {
    for (uintptr_t c = a0 + 8 * lane; c < a1; c += 8 * 32)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst + (uint32_t)(c - c0)), "l"(c) : "memory");
  }
  return (uint32_t)(a0 - c0) >> 3;
}

__device__ __forceinline__ picker_rec_t rec_from_u4(const uint4 a, const uint4 b) {
  picker_rec_t r;
  r.kernel_id = a.x;
  r.nargs = a.y;
  r.grid_x = a.z;
  r.grid_y = (uint16_t)(a.w & 0xFFFF);
  r.grid_z = (uint16_t)(a.w >> 16);
  r.block_x = (uint16_t)(b.x & 0xFFFF);
  r.block_y = (uint16_t)(b.x >> 16);
  r.block_z = (uint16_t)(b.y & 0xFFFF);
  r.reserved = (uint16_t)(b.y >> 16);
  r.arg_off = ((uint64_t)b.w << 32) | b.z;
  return r;
}

__global__ void __launch_bounds__(kWideWarps * 32, kWideCtas)
    k_validate_wide(const __grid_constant__ BucketParams P, const __grid_constant__ DevBatch B, uint64_t n,
                    uint8_t* __restrict__ flags, uint32_t* __restrict__ bits,
                    unsigned long long* __restrict__ counts) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint32_t s_hist[PICKER_NUM_COUNTS];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  WideWarpSmem& W = reinterpret_cast<WideWarpSmem*>(smem)[warp];
  if (tid < PICKER_NUM_COUNTS) s_hist[tid] = 0;
  __syncthreads();
  const Tables& T = P.T;
  const uint64_t nch = (n + 31) / 32;
  const uint64_t stride = (uint64_t)gridDim.x * kWideWarps;
  const uint64_t c_first = (uint64_t)blockIdx.x * kWideWarps + warp;
  // the records of this warp, in order: chunks c_first, c_first + stride, ...
  auto next_of = [&](uint64_t i) -> uint64_t {  // n: none
    if (i >= n) return n;
    if ((i & 31) != 31 && i + 1 < n) return i + 1;
    const uint64_t c = (i >> 5) + stride;
    return c < nch ? c * 32 : n;
  };
  auto load_hdr = [&](uint64_t i, uint4& a, uint4& b) {
    if (i < n) {
      const uint4* q = reinterpret_cast<const uint4*>(B.rec + i);
      a = __ldg(q), b = __ldg(q + 1);
    } else {
      a = b = make_uint4(0, 0, 0, 0);
    }
  };
  uint64_t i = c_first < nch ? c_first * 32 : n;
  uint4 ha, hb, h1a, h1b, h2a, h2b;
  load_hdr(i, ha, hb);
  uint64_t i1 = next_of(i);
  load_hdr(i1, h1a, h1b);
  uint32_t shift = 0, buf = 0;
  if (i < n) shift = stage_span(B, ((uint64_t)hb.w << 32) | hb.z, ha.y, W.args[0], lane);
  asm volatile("cp.async.commit_group;" ::: "memory");
  uint32_t code_mine = 0;
  while (i < n) {
    // record i+2's header and record i+1's arguments are in flight while i runs
    const uint64_t i2 = next_of(i1);
    load_hdr(i2, h2a, h2b);
    uint32_t shift1 = 0;
    if (i1 < n) shift1 = stage_span(B, ((uint64_t)h1b.w << 32) | h1b.z, h1a.y, W.args[buf ^ 1], lane);
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 1;" ::: "memory");
    __syncwarp();
    const picker_rec_t r = rec_from_u4(ha, hb);
    int64_t* ops = reinterpret_cast<int64_t*>(W.args[buf] + 8 * shift);
    uint8_t code;
    const uint32_t kid = r.kernel_id;
    if (kid >= T.nkernel_slots) {
      code = V_ERR_KERNEL;
    } else {
      const DKernel K = T.kernels[kid];
      if (K.shortcut == V_ERR_KERNEL) {
        code = V_ERR_KERNEL;
      } else if (!args_in_range(r, K.nparams, B.args_lo, B.args_hi)) {
        code = V_ERR_ARITY;
      } else if (K.shortcut) {
        code = K.shortcut;
      } else if (!launch_limits_rec(r)) {
        code = V_NI_PRECOND;
      } else if (K.ndesc > kWExt || K.nprod > kWProd || K.nvar > kWVar || K.nsig > kWideSigs) {
        code = wide_fallback(T, r, B.args + r.arg_off, B.args_lo, B.args_hi, lane, wide_scratch(P, warp));
      } else {
        // operand slots 0..7: launch dimensions, 1, 0; i32 parameters sign-extended
        if (lane < 8) {
          const int64_t v = lane == 0 ? (int64_t)r.grid_x : lane == 1 ? r.grid_y : lane == 2 ? r.grid_z
                          : lane == 3 ? r.block_x : lane == 4 ? r.block_y : lane == 5 ? r.block_z
                          : lane == 6 ? 1 : 0;
          ops[lane] = v;
        }
        const uint32_t mw = lane < 6 ? __ldg(&T.kernels[kid].i32mask[lane]) : 0u;
        if (__any_sync(0xffffffffu, mw != 0)) {
          for (int p0 = 0; p0 < (int)K.nparams; p0 += 32) {
            const uint32_t word = __shfl_sync(0xffffffffu, mw, p0 >> 5);
            const int p = p0 + lane;
            if (p < (int)K.nparams && ((word >> lane) & 1u))
              ops[OPD_ARG0 + p] = (int64_t)(int32_t)(uint32_t)ops[OPD_ARG0 + p];
          }
        }
        __syncwarp();
        code = eval_wide_ws(T, K, ops, W, lane);
      }
    }
    if ((uint64_t)lane == (i & 31)) code_mine = code;
    const uint64_t inext = i1;
    // emit the chunk after its last record
    if (inext >= n || (inext >> 5) != (i >> 5)) {
      const uint64_t c0 = i & ~(uint64_t)31;
      const uint32_t m = (uint32_t)min((uint64_t)32, n - c0);
      const bool valid = (uint32_t)lane < m;
      if (valid) flags[c0 + lane] = (uint8_t)code_mine;
      const unsigned idem = __ballot_sync(0xffffffffu, valid && code_mine <= V_IDEM_KERNEL);
      if (bits != nullptr && lane == 0) bits[c0 >> 5] = idem;
      const int hbin = valid ? count_bin((uint8_t)code_mine) : 16;
      const unsigned same = __match_any_sync(0xffffffffu, hbin);
      if (valid && (__ffs(same) - 1) == lane) atomicAdd(s_hist + hbin, (uint32_t)__popc(same));
      code_mine = 0;
    }
    __syncwarp();  // buffer `buf` is restaged two records from now
    i = i1, ha = h1a, hb = h1b;
    i1 = i2, h1a = h2a, h1b = h2b;
    shift = shift1;
    buf ^= 1;
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  flush_counts(s_hist, counts, P.count_slot);
}

cudaError_t launch_wide(const BucketParams& P, const DevBatch& B, uint64_t n, uint8_t* flags, uint32_t* bits,
                        unsigned long long* counts, int num_sms, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  static bool configured[64] = {};  // the attribute is per device
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev >= 64 || !configured[dev]) {
    e = cudaFuncSetAttribute(k_validate_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kWideSmem);
    if (e != cudaSuccess) return e;
    if (dev < 64) configured[dev] = true;
  }
  const uint64_t nch = (n + 31) / 32;
  const uint64_t ctas_needed = (nch + kWideWarps - 1) / kWideWarps;
  const uint64_t cap = (uint64_t)num_sms * kWideCtas;
  const uint64_t grid = ctas_needed < cap ? ctas_needed : cap;
  k_validate_wide<<<(unsigned)grid, kWideWarps * 32, kWideSmem, s>>>(P, B, n, flags, bits, counts);
  return cudaGetLastError();
}

int wide_warps_per_sm() { return kWideWarps * kWideCtas; }

}  // namespace picker
