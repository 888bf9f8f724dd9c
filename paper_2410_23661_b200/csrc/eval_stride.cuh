// Row f4: stride-aware ranges (reading Q24).
//
// The range model's RO false negatives (reads {1,3,5}
// and writes {0,2,4} have overlapping ranges [1,5] and [0,4]) come from
// non-consecutive address sets.  Every address of a descriptor is congruent to
// its lower bound modulo g, the gcd of the coefficients of its varying term
// groups (the terms on one variable with one divisor add up to C * phi(x); a
// group whose phi is constant on the box is a constant).  A read/write pair
// whose byte intervals intersect shares a byte only if some b - a in
// (lb_w - lb_r) + gcd(g_r, g_w) * Z falls in [-(w_w - 1), w_r - 1].  Both tests
// are necessary conditions for an overlap, so the verdict stays sound; it
// refines NI_OVERLAP -> IDEM_CHECKED on strided sets.  lb is an address the
// descriptor attains (corner of the box, by sign-definiteness), so its residue
// is the descriptor's.  Oracle: oracle/picker_oracle.py congruence / may_collide.
#pragma once

#include "desc_eval.cuh"
#include "device_common.cuh"

namespace picker {

static __device__ __noinline__ uint64_t gcd64(uint64_t a, uint64_t b) {
  if (a == 0) return b;
  if (b == 0) return a;
  const int sh = __ffsll((long long)(a | b)) - 1;
  a >>= __ffsll((long long)a) - 1;
  do {
    b >>= __ffsll((long long)b) - 1;
    if (a > b) {
      const uint64_t t = a;
      a = b;
      b = t;
    }
    b -= a;
  } while (b != 0);
  return a << sh;
}

// gcd64 with the common cases inline (a zero, or two powers of two: element
// strides), so that the shapes make no call -- a call spills the caller's live
// registers around it
static __device__ __forceinline__ uint64_t gcd64f(uint64_t a, uint64_t b) {
  if (a == 0) return b;
  if (b == 0) return a;
  if (((a & (a - 1)) | (b & (b - 1))) == 0) return a < b ? a : b;
  return gcd64(a, b);
}

static __device__ __forceinline__ uint64_t uabs64(int64_t x) {
  return x < 0 ? (uint64_t)0 - (uint64_t)x : (uint64_t)x;
}

// x mod m in [0, m), m > 0
static __device__ __forceinline__ uint64_t mod64(int64_t x, uint64_t m) {
  if (x >= 0) return (uint64_t)x % m;
  const uint64_t r = ((uint64_t)0 - (uint64_t)x) % m;  // |x| mod m
  return r == 0 ? 0 : m - r;
}

// g of an active non-opaque descriptor (0: a single address)
static __device__ uint64_t desc_stride(const Tables& T, const DKernel& K, const DDesc& D, const RecVals& X) {
  uint64_t g = 0;
  for (int t = 0; t < D.nterm; ++t) {
    const DTerm tm = T.terms[D.term + t];
    if (tm.var == kNone16) continue;
    bool first = true;  // the group (var, div) is handled at its first term
    for (int u = 0; u < t && first; ++u) {
      const DTerm tu = T.terms[D.term + u];
      first = !(tu.var == tm.var && tu.div == tm.div);
    }
    if (!first) continue;
    int64_t c = 0;
    for (int u = t; u < D.nterm; ++u) {
      const DTerm tu = T.terms[D.term + u];
      if (tu.var == tm.var && tu.div == tm.div) c = add64(c, prod_val(T, K, X, tu.prod));
    }
    int64_t lo, hi;
    slot_bounds(T, K, X, tm.var, lo, hi);
    if (floordiv64(lo, tm.div) == floordiv64(hi, tm.div)) continue;  // constant on the box
    g = gcd64f(g, uabs64(c));
  }
  return g;
}

// can the two congruence classes share a byte (intervals already intersect)?
static __device__ __noinline__ bool may_collide(int64_t lb_r, uint64_t g_r, uint32_t w_r, int64_t lb_w,
                                                   uint64_t g_w, uint32_t w_w) {
  const uint64_t G = gcd64f(g_r, g_w);
  if (G == 0) return true;  // two single addresses: the interval test is exact
  if ((G & (G - 1)) == 0) {  // power of two (element strides): residues by masks, no 64-bit division
    const uint64_t M = G - 1, d = ((uint64_t)lb_w - (uint64_t)lb_r) & M;
    return ((d + (w_w - 1)) & M) <= (uint64_t)w_r + w_w - 2;
  }
  const uint64_t pr = mod64(lb_r, G), pw = mod64(lb_w, G);
  const uint64_t d = pw >= pr ? pw - pr : pw + (G - pr);  // (lb_w - lb_r) mod G
  const uint64_t t = (d + (w_w - 1)) % G;
  return t <= (uint64_t)w_r + w_w - 2;
}

// The stride-aware verdict of one record (table-driven).
static __device__ __noinline__ uint8_t eval_stride(const Tables& T, const picker_rec_t r, const int64_t* rec_args,
                                                   uint64_t args_lo, uint64_t args_hi) {
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
    uint64_t rg = 0;
    bool rg_done = false;  // the stride is computed once an interval test passes
    for (int j = 0; j < K.ndesc; ++j) {
      const DDesc Dj = T.descs[K.desc + j];
      if (Dj.kind != KIND_W || Dj.opaque || !desc_active(T, K, Dj, X)) continue;
      int64_t wl, wu;
      desc_extent(T, K, Dj, X, wl, wu);
      if (!(rl <= wu && wl <= ru)) continue;
      if (!rg_done) rg = desc_stride(T, K, Di, X), rg_done = true;
      if (may_collide(rl, rg, Di.width, wl, desc_stride(T, K, Dj, X), Dj.width)) return V_NI_OVERLAP;
    }
  }
  return V_IDEM_CHECKED;
}

}  // namespace picker
