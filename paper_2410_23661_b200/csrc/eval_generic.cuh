// The table-driven evaluation of one launch record (K1-generic).
//
// The straightforward device rendering of the paper's optimized validator
// (§5): per instance, check the preconditions and global condition
// (Fig. 3 lines 1-2; l.976-979, l.749-752), evaluate each range descriptor at
// the extreme values of its variables (l.950-951) with path-condition
// tightening (l.1023-1026) and induction/fresh ranges (l.1063, l.990-992),
// then test every active read extent against every active write extent
// (l.658-666).  Reads the flattened tables of tables.hpp.  Included by the
// static kernels and by the NVRTC module (as the fallback of its dispatch).
#pragma once

#include "desc_eval.cuh"
#include "device_common.cuh"

namespace picker {

// Kernels beyond the register arrays below: recompute extents per pair instead
// of storing them (same verdict, slower; only reached on the table path).
static __device__ __noinline__ uint8_t eval_nostore(const Tables& T, const DKernel& K, const RecVals& X) {
  bool act_r = false, act_w = false, opq_r = false, opq_w = false;
  for (int d = 0; d < K.ndesc; ++d) {
    const DDesc D = T.descs[K.desc + d];
    if (!desc_active(T, K, D, X)) continue;
    (D.kind == KIND_R ? act_r : act_w) = true;
    if (D.opaque) (D.kind == KIND_R ? opq_r : opq_w) = true;
  }
  if ((opq_r && act_w) || (opq_w && act_r)) return V_NI_OPAQUE;
  for (int i = 0; i < K.ndesc; ++i) {
    const DDesc Di = T.descs[K.desc + i];
    if (Di.kind != KIND_R || Di.opaque || !desc_active(T, K, Di, X)) continue;
    int64_t rl, ru;
    desc_extent(T, K, Di, X, rl, ru);
    for (int j = 0; j < K.ndesc; ++j) {
      const DDesc Dj = T.descs[K.desc + j];
      if (Dj.kind != KIND_W || Dj.opaque || !desc_active(T, K, Dj, X)) continue;
      int64_t wl, wu;
      desc_extent(T, K, Dj, X, wl, wu);
      if (rl <= wu && wl <= ru) return V_NI_OVERLAP;
    }
  }
  return V_IDEM_CHECKED;
}

// `rec_args` = the record's argument slots (args + r.arg_off, or its staged
// shared-memory copy); [args_lo, args_hi) is the valid slot range of the pool.
static __device__ __noinline__ uint8_t eval_generic(const Tables& T, const picker_rec_t r,
                                             const int64_t* rec_args, uint64_t args_lo,
                                             uint64_t args_hi) {
  const uint32_t kid = r.kernel_id;
  if (kid >= T.nkernel_slots) return V_ERR_KERNEL;
  const DKernel K = T.kernels[kid];
  if (K.shortcut == V_ERR_KERNEL) return V_ERR_KERNEL;
  if (!args_in_range(r, K.nparams, args_lo, args_hi)) return V_ERR_ARITY;
  if (K.shortcut) return K.shortcut;

  RecVals X(r, rec_args, K.i32mask);
  if (!launch_limits_ok(X)) return V_NI_PRECOND;
  for (int c = 0; c < K.npre + K.nglob; ++c) {
    const DCheck ch = T.checks[K.check + c];
    const int64_t v = X.get(ch.op);
    if (v < ch.lo || v > ch.hi) return c < K.npre ? V_NI_PRECOND : V_NI_GLOBAL;
  }
  if (K.nr > kGenMaxDesc || K.nw > kGenMaxDesc || K.nvar > kGenMaxVar) return eval_nostore(T, K, X);

  auto P = [&](uint16_t j) -> int64_t {
    const DProd p = T.prods[K.prod + j];
    return mul64(mul64(p.k, X.get(p.a)), X.get(p.b));
  };
  auto B = [&](const DBexpr& b) -> int64_t {
    int64_t v = b.k0;
    if (b.p0 != kNone16) v = add64(v, P(b.p0));
    if (b.p1 != kNone16) v = add64(v, P(b.p1));
    return v;
  };

  int64_t vlo[kGenMaxVar], vhi[kGenMaxVar];
  for (int s = 0; s < K.nvar; ++s) {
    const DVar v = T.vars[K.var + s];
    int64_t lo = (-9223372036854775807LL - 1), hi = 9223372036854775807LL;
    if (v.skind != SK_NONE) {
      const int64_t g = X.get(OPD_GX + v.axis), b = X.get(OPD_BX + v.axis);
      lo = 0;
      hi = (v.skind == SK_TID ? b : v.skind == SK_BID ? g : g * b) - 1;
    }
    for (int j = 0; j < v.nlo; ++j) lo = max64(lo, B(T.bexprs[v.bex + j]));
    for (int j = 0; j < v.nhi; ++j) hi = min64(hi, B(T.bexprs[v.bex + v.nlo + j]));
    vlo[s] = lo;
    vhi[s] = hi;
  }

  int64_t rlb[kGenMaxDesc], rub[kGenMaxDesc], wlb[kGenMaxDesc], wub[kGenMaxDesc];
  int nr = 0, nw = 0;
  bool opq_r = false, opq_w = false, act_r = false, act_w = false;
  for (int di = 0; di < K.ndesc; ++di) {
    const DDesc D = T.descs[K.desc + di];
    bool on = true;
    for (int g = 0; g < D.nguard && on; ++g) {
      const DGuard G = T.guards[D.guard + g];
      on = cmp64(X.get(G.a), G.cmp, G.b == OPD_NONE ? G.bconst : X.get(G.b));
    }
    for (int v = 0; v < D.nvar && on; ++v) {
      const uint16_t s = T.varlist[D.var + v];
      on = vlo[s] <= vhi[s];  // empty range: the site never executes
    }
    if (!on) continue;
    if (D.kind == KIND_R) act_r = true; else act_w = true;
    if (D.opaque) {
      if (D.kind == KIND_R) opq_r = true; else opq_w = true;
      continue;
    }
    int64_t lb = D.base == OPD_NONE ? 0 : X.get(D.base), ub = lb;
    for (int t = 0; t < D.nterm; ++t) {
      const DTerm tm = T.terms[D.term + t];
      const int64_t c = P(tm.prod);
      if (tm.var == kNone16) {
        lb = add64(lb, c);
        ub = add64(ub, c);
      } else {
        const int64_t a = mul64(c, floordiv64(vlo[tm.var], tm.div));
        const int64_t b = mul64(c, floordiv64(vhi[tm.var], tm.div));
        lb = add64(lb, min64(a, b));
        ub = add64(ub, max64(a, b));
      }
    }
    ub = add64(ub, (int64_t)D.width - 1);
    if (D.kind == KIND_R) { rlb[nr] = lb; rub[nr] = ub; ++nr; }
    else { wlb[nw] = lb; wub[nw] = ub; ++nw; }
  }
  if ((opq_r && act_w) || (opq_w && act_r)) return V_NI_OPAQUE;
  for (int i = 0; i < nr; ++i)
    for (int j = 0; j < nw; ++j)
      if (rlb[i] <= wub[j] && wlb[j] <= rub[i]) return V_NI_OVERLAP;
  return V_IDEM_CHECKED;
}

}  // namespace picker
