// Specialised validation functions, compiled at load time with NVRTC.
//
// The paper turns each kernel's symbolic addresses into C, compiles them into
// a shared library and calls the function of the launched kernel (compiled
// execution: "the loop over the symbolic addresses is
// unrolled, and the functions that calculate the ranges are all inlined ...
// common expression extraction").  The B200 analog generates straight-line
// CUDA per kernel *shape*: the structure of a summary (which operands, how
// many checks, descriptors, terms and variables, which sign each term has,
// which read/write pairs exist) becomes code with extents in registers and one
// endpoint per bound; the kernel's integer constants (coefficients, bounds,
// widths) are read from a per-kernel constant table with warp-uniform loads.
// Many kernels share a shape (every TVM dense kernel, every elementwise
// kernel of one arity), so the module stays small enough for the instruction
// caches: specialising per kernel instead made the bucketed kernel
// instruction-fetch bound (ncu: no_instruction stalls, profiles/).
//
// Dispatch (inside k_bucket.cuh, warp-uniform per 32-record group):
//   shape 0: unknown kernel id      shape 1: table-driven evaluator
//   shape 2: kernel-level shortcut  shape 3+s: generated function ks<s>
// Bins are ordered by shape so neighbouring groups run the same code.
// The compiled cubin is cached on disk by source hash ($PICKER_JIT_CACHE,
// default ~/.cache/picker_jit); the cache only saves compile time.
#include <cuda_runtime.h>
#include <nvrtc.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "launch.hpp"
#include "loader.hpp"

namespace picker {

#include "jit_embed.inc"  // kEmbedNames[], kEmbedSrc[], kEmbedCount (build.py)

struct JitModule {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kernel = nullptr;
  cudaKernel_t small_kernel = nullptr;  // k_validate_small: n <= kSmallMax
  bool pipe = false;                    // main kernel is k_validate_pipe (<= kPipeKeysMax keys)
  bool models = false;                  // built with PICKER_MODELS (row f3 fused)
  bool extents = false;                 // built with PICKER_EXTENTS (row f1 on K1's extents)
  uint32_t seq_xcap = 0;                // ... with the tile's extent slots in shared memory
  bool seq_windows = false;             // built with PICKER_SEQ (row f1 from K1's codes)
  size_t smem = 0;
  int64_t* d_consts = nullptr;
  KbEntry* d_kb = nullptr;
  uint32_t kb_unknown = 0;
  uint32_t shortcut_key = 0;  // grouping key of the shortcut kernels and unknown ids
  uint32_t nkeys = 0;
  int nshapes = 0;
  int tile = 0, threads = 0, ctas = 0;
  bool stride = false;  // built with stride-aware shapes (row f4)
  // shape-sorted schedule (k_sorted.cuh): S1 keys, [1 unused], S3 scatter,
  // S4 validate, S5 emit; its scratch grows with the largest batch seen
  cudaKernel_t sk[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  int sort_warps = 0;
  bool sort_ws = false;  // S4 warp-specialised (sk[1], k_validate_sorted_ws)
  size_t sort_smem = 0, sort_ws_smem = 0;
  void* sort_buf = nullptr;
  size_t sort_cap = 0;  // records the scratch holds
};

namespace {

// Grouping keys of the specialised module.  Generated shapes are keys
// SHAPE_FIRST.. (first appearance order) and the shortcut kernels take the key
// after the last shape: warps claim groups in key order, so the cheap shortcut
// groups fill the tail.  (Ordering shapes by decreasing code size was measured
// slower: C4 1.06 -> 0.71 G inst/s, warps enter the largest functions together.)
constexpr uint32_t SHAPE_UNKNOWN = 0, SHAPE_GENERIC = 1, SHAPE_WIDE = 2, SHAPE_FIRST = 3;

std::string lit(int64_t v) {
  if (v == (int64_t)(-9223372036854775807LL - 1)) return "(-9223372036854775807LL - 1)";
  return std::to_string(v) + "LL";
}

std::string opnd(uint8_t o) {
  if (o < 6) return "d" + std::to_string(o);
  if (o == OPD_ONE) return "1LL";
  if (o == OPD_NONE) return "0LL";
  return "x" + std::to_string(o - OPD_ARG0);
}

const char* kCmp[6] = {"<", "<=", ">", ">=", "==", "!="};

void uses(uint8_t o, std::vector<bool>& used) {
  if (o >= OPD_ARG0) used[o - OPD_ARG0] = true;
}

// Emits the body of one kernel's function; integer constants go to `K` and
// appear in the text as __ldg(K + i), so kernels of one shape share the text.
struct Gen {
  std::vector<int64_t>& K;
  std::ostringstream s;
  explicit Gen(std::vector<int64_t>& k) : K(k) {}
  std::string k(int64_t v) {
    K.push_back(v);
    return "__ldg(K + " + std::to_string(K.size() - 1) + ")";
  }
  std::string prod(const IrProd& p) {
    std::string e;
    auto mul = [&](const std::string& x) { e = e.empty() ? x : "mul64(" + e + ", " + x + ")"; };
    if (p.k != 1) mul(k(p.k));
    if (p.a != OPD_ONE) mul(opnd(p.a));
    if (p.b != OPD_ONE) mul(opnd(p.b));
    return e.empty() ? "1LL" : e;
  }
  std::string bexpr(const IrBexpr& b) {
    std::string e = b.k0 ? k(b.k0) : "";
    for (auto& p : b.p) e = e.empty() ? prod(p) : "add64(" + e + ", " + prod(p) + ")";
    return e.empty() ? "0LL" : e;
  }
};

// stride: the stride-aware variant (row f4, eval_stride.cuh): a read/write pair
// whose intervals intersect is an overlap only if may_collide() holds for the
// two descriptors' congruence classes (computed lazily, on intersection).
// Streamed descriptors that differ only in their base argument (same kind,
// activity, term sums and width: e.g. every 16-byte read of a tensor list with
// one shape) are evaluated by a loop over a table of argument indices when a
// class has at least kLoopMin members: many-pointer kernels (C4) otherwise
// emit one straight-line block per descriptor, and a shape of ~4,000 SASS
// instructions does not fit the 32 KB instruction cache.
constexpr size_t kLoopMin = 3;  // class size
size_t g_loop_kernel_min = 6;  // streamed descriptors of the kernel (Options.loop_min, set by jit_plan)
uint64_t fnv1a(const std::string& s);

// models: the module of picker_validate_models -- the reads are the kept side
// and, before the verdict, the length of the union of the active non-opaque
// read extents goes to *inb (row f3, reading Q25; models.cuh).
// extents: the module of picker_validate_sequence on K1's extents (row f1) --
// every active non-opaque extent goes to the record's arena slots and the
// activity / opaque flags to xo.fl (XOut, models.cuh).
std::string gen_body(const IrKernel& k, std::vector<int64_t>& K, bool stride, std::map<std::string, std::string>* defs,
                     bool models = false, bool extents = false) {
  Gen g(K);
  std::ostringstream& s = g.s;
  const int np = (int)k.param_names.size();
  s << "(const picker_rec_t& r, const int64_t* a, const int64_t* __restrict__ K"
    << (models ? ", uint64_t* inb" : "") << (extents ? ", XOut& xo" : "") << ") {\n";
  s << "  const int64_t d0 = r.grid_x, d1 = r.grid_y, d2 = r.grid_z, d3 = r.block_x, d4 = r.block_y,"
       " d5 = r.block_z;\n";
  // (the CUDA launch limits are checked once in the dispatch, before the switch)
  std::vector<bool> used(np, false);
  for (auto* lst : {&k.pre, &k.glob})
    for (auto& c : *lst) uses(c.op, used);
  for (auto& d : k.desc) {
    uses(d.base, used);
    for (auto& gd : d.guard) uses(gd.a, used), uses(gd.b, used);
    for (auto& v : d.vars)
      for (auto* side : {&v.lo, &v.hi})
        for (auto& e : *side)
          for (auto& p : e.p) uses(p.a, used), uses(p.b, used);
    for (auto& t : d.terms) uses(t.c.a, used), uses(t.c.b, used);
  }

  for (int i = 0; i < np; ++i)
    if (used[i]) {
      if (k.param_i32[i])
        s << "  const int64_t x" << i << " = (int64_t)(int32_t)(uint32_t)a[" << i << "];\n";
      else
        s << "  const int64_t x" << i << " = a[" << i << "];\n";
    }
  // lo <= x <= hi; with lo = 0 <= hi (every pointer bound) one unsigned compare
  auto check = [&](const IrCheck& c, const char* code) {
    if (c.op < 6 || (c.op >= OPD_ARG0 && k.param_i32[c.op - OPD_ARG0])) {
      // a launch dimension (in [1, kDimMax], launch limits checked first) or
      // an i32 argument: clamp the bounds to the operand's type range, then one
      // 32-bit compare of x - lo against the span (the range holds <= 2^32
      // values; lo > hi after clamping never reaches a shape: the loader
      // routes such kernels to the table path)
      const int64_t tlo = c.op < 6 ? 1 : -2147483648LL, thi = c.op < 6 ? kDimMax[c.op] : 2147483647LL;
      const int64_t lo = std::max(c.lo, tlo), hi = std::min(c.hi, thi);
      if (lo <= hi) {
        s << "  if ((uint32_t)" << opnd(c.op) << " - (uint32_t)" << g.k(lo) << " > (uint32_t)" << g.k(hi - lo)
          << ") return " << code << ";\n";
        return;
      }
    }
    if (c.lo == 0 && c.hi >= 0)
      s << "  if ((uint64_t)" << opnd(c.op) << " > (uint64_t)" << g.k(c.hi) << ") return " << code << ";\n";
    else
      s << "  if (" << opnd(c.op) << " < " << g.k(c.lo) << " || " << opnd(c.op) << " > " << g.k(c.hi) << ") return "
        << code << ";\n";
  };
  for (auto& c : k.pre) check(c, "V_NI_PRECOND");
  for (auto& c : k.glob) check(c, "V_NI_GLOBAL");
  // variable slots, deduplicated by content (as in flatten())
  struct SlotKey {
    uint8_t skind, axis;
    std::vector<std::pair<int64_t, std::vector<std::tuple<int64_t, int, int>>>> lo, hi;
    bool operator==(const SlotKey& o) const {
      return skind == o.skind && axis == o.axis && lo == o.lo && hi == o.hi;
    }
  };
  auto key_of = [](const IrVar& v) {
    SlotKey kk{v.skind, v.axis, {}, {}};
    for (auto* side : {&v.lo, &v.hi})
      for (auto& e : *side) {
        std::vector<std::tuple<int64_t, int, int>> ps;
        for (auto& p : e.p) ps.emplace_back(p.k, p.a, p.b);
        (side == &v.lo ? kk.lo : kk.hi).emplace_back(e.k0, ps);
      }
    return kk;
  };
  std::vector<SlotKey> keys;
  std::vector<bool> lo0, nonempty;
  auto slot_of = [&](const IrVar& v) -> int {
    SlotKey kk = key_of(v);
    for (size_t i = 0; i < keys.size(); ++i)
      if (keys[i] == kk) return (int)i;
    std::string lo, hi;
    auto add_lo = [&](const std::string& e) { lo = lo.empty() ? e : "max64(" + lo + ", " + e + ")"; };
    auto add_hi = [&](const std::string& e) { hi = hi.empty() ? e : "min64(" + hi + ", " + e + ")"; };
    if (v.skind != SK_NONE) {
      add_lo("0LL");
      std::string gg = "d" + std::to_string(v.axis), b = "d" + std::to_string(3 + v.axis);
      add_hi(v.skind == SK_TID ? b + " - 1" : v.skind == SK_BID ? gg + " - 1" : gg + " * " + b + " - 1");
    }
    for (auto& e : v.lo) add_lo(g.bexpr(e));
    for (auto& e : v.hi) add_hi(g.bexpr(e));
    keys.push_back(kk);
    lo0.push_back(v.skind != SK_NONE && v.lo.empty());
    // [0, dim - 1] with dims >= 1 (launch limits): never empty
    nonempty.push_back(v.skind != SK_NONE && v.lo.empty() && v.hi.empty());
    const size_t i = keys.size() - 1;
    s << "  const int64_t vl" << i << " = " << lo << ", vh" << i << " = " << hi << ";\n";
    return (int)i;
  };
  // Every variable slot first: the streamed descriptors below live in block
  // scopes.  Then the extents of the smaller side (usually the writes) are kept
  // in registers and the other side is streamed through the overlap test, so
  // many-pointer kernels do not keep every extent live (register spills).
  std::vector<std::vector<int>> sids(k.desc.size());
  for (size_t di = 0; di < k.desc.size(); ++di)
    for (auto& v : k.desc[di].vars) sids[di].push_back(slot_of(v));
  size_t nr = 0, nw = 0;
  for (auto& d : k.desc)
    if (!d.opaque) (d.kind == KIND_R ? nr : nw)++;
  const uint8_t kept_kind = models ? KIND_R : nw <= nr ? KIND_W : KIND_R;
  auto on_expr = [&](size_t di) {
    const IrDesc& d = k.desc[di];
    std::string on = "true";
    for (auto& gd : d.guard)
      on += " && (" + opnd(gd.a) + " " + kCmp[gd.cmp] + " " + (gd.b == OPD_NONE ? g.k(gd.bconst) : opnd(gd.b)) + ")";
    for (int x : sids[di])
      if (!nonempty[x]) on += " && (vl" + std::to_string(x) + " <= vh" + std::to_string(x) + ")";
    return on;
  };
  // emits the extent of descriptor di as `const int64_t lb<di>, ub<di>` at indent `ind`
  auto extent = [&](size_t di, const char* ind) {
    const IrDesc& d = k.desc[di];
    // the term sums first and the base last: descriptors with the same terms
    // (e.g. every buffer of one tensor shape) share one offset expression,
    // which the compiler then computes once
    std::string lb = "0LL", ub = lb;
    for (size_t ti = 0; ti < d.terms.size(); ++ti) {
      const IrTerm& t = d.terms[ti];
      std::string c = g.prod(t.c);
      if (t.var < 0) {
        lb = "add64(" + lb + ", " + c + ")";
        ub = "add64(" + ub + ", " + c + ")";
        continue;
      }
      const int x = sids[di][t.var];
      auto phi = [&](const std::string& v) {
        return t.div == 1 ? v : "floordiv64(" + v + ", " + std::to_string(t.div) + "u)";
      };
      const std::string L = "vl" + std::to_string(x), H = "vh" + std::to_string(x);
      const int sign = k.var_sign[di][t.var];
      const std::string mul = t.narrow ? "mulw" : "mul64";
      if (sign > 0) {  // non-decreasing: min at lo, max at hi
        if (!lo0[x]) lb = "add64(" + lb + ", " + mul + "(" + c + ", " + phi(L) + "))";
        ub = "add64(" + ub + ", " + mul + "(" + c + ", " + phi(H) + "))";
      } else if (sign < 0) {
        lb = "add64(" + lb + ", " + mul + "(" + c + ", " + phi(H) + "))";
        if (!lo0[x]) ub = "add64(" + ub + ", " + mul + "(" + c + ", " + phi(L) + "))";
      } else {  // one term of unknown sign: both ends
        const std::string cv = "c" + std::to_string(di) + "_" + std::to_string(ti);
        s << ind << "const int64_t " << cv << " = " << c << ";\n";
        std::string A = mul + "(" + cv + ", " + phi(L) + ")", Bv = mul + "(" + cv + ", " + phi(H) + ")";
        lb = "add64(" + lb + ", min64(" + A + ", " + Bv + "))";
        ub = "add64(" + ub + ", max64(" + A + ", " + Bv + "))";
      }
    }
    if (d.width > 1) ub = "add64(" + ub + ", " + g.k((int64_t)d.width - 1) + ")";
    if (d.base != OPD_NONE) lb = "add64(" + opnd(d.base) + ", " + lb + ")", ub = "add64(" + opnd(d.base) + ", " + ub + ")";
    s << ind << "const int64_t lb" << di << " = " << lb << ", ub" << di << " = " << ub << ";\n";
    if (stride) {  // g = gcd of |sum of coefficients| of the varying (variable, divisor) groups
      std::vector<std::pair<std::pair<int, uint32_t>, std::string>> groups;
      for (const IrTerm& t : d.terms) {
        if (t.var < 0) continue;
        const std::pair<int, uint32_t> key{t.var, (uint32_t)t.div};
        const std::string cc = g.prod(t.c);
        auto it = std::find_if(groups.begin(), groups.end(), [&](auto& e) { return e.first == key; });
        if (it == groups.end()) groups.push_back({key, cc});
        else it->second = "add64(" + it->second + ", " + cc + ")";
      }
      s << ind << "auto G" << di << " = [&]() -> uint64_t {\n" << ind << "  uint64_t gg = 0;\n";
      for (auto& e : groups) {
        const int x = sids[di][e.first.first];
        const uint32_t dv = e.first.second;
        const std::string L = "vl" + std::to_string(x), H = "vh" + std::to_string(x);
        const std::string vary = dv == 1 ? L + " != " + H
                                         : "floordiv64(" + L + ", " + std::to_string(dv) + "u) != floordiv64(" + H +
                                               ", " + std::to_string(dv) + "u)";
        s << ind << "  if (" << vary << ") gg = gcd64f(gg, uabs64(" << e.second << "));\n";
      }
      s << ind << "  return gg;\n" << ind << "};\n";
      s << ind << "const uint32_t W" << di << " = (uint32_t)" << g.k((int64_t)d.width) << ";\n";
    }
  };
  std::vector<int> kept, opq_r, opq_w;
  s << "  bool act_r = false, act_w = false, ov = false;\n";
  for (size_t di = 0; di < k.desc.size(); ++di) {  // opaque sites and the kept side
    const IrDesc& d = k.desc[di];
    if (!d.opaque && d.kind != kept_kind) continue;
    s << "  const bool on" << di << " = " << on_expr(di) << ";\n";
    s << "  act_" << (d.kind == KIND_R ? "r" : "w") << " |= on" << di << ";\n";
    if (d.opaque) {
      (d.kind == KIND_R ? opq_r : opq_w).push_back((int)di);
      if (extents) s << "  if (on" << di << ") xo.fl |= " << (d.kind == KIND_R ? 4 : 8) << "u;\n";
      continue;
    }
    extent(di, "  ");
    if (extents)
      s << "  if (on" << di << ") xo_put(xo, " << (d.kind == KIND_W) << ", lb" << di << ", ub" << di << ");\n";
    kept.push_back((int)di);
  }
  // term sums of a descriptor without its base, constants as literals (the
  // grouping key of the loop classes); false if it cannot join a loop
  auto sums = [&](size_t di, Gen& gg, std::string& lb, std::string& ub) {
    const IrDesc& d = k.desc[di];
    if (stride || d.base < OPD_ARG0 || k.param_i32[d.base - OPD_ARG0]) return false;
    lb = "0LL", ub = lb;
    for (const IrTerm& t : d.terms) {
      const std::string c = gg.prod(t.c);
      if (t.var < 0) {
        lb = "add64(" + lb + ", " + c + ")", ub = "add64(" + ub + ", " + c + ")";
        continue;
      }
      const int x = sids[di][t.var];
      const int sign = k.var_sign[di][t.var];
      if (sign == 0) return false;
      const std::string L = "vl" + std::to_string(x), H = "vh" + std::to_string(x);
      auto phi = [&](const std::string& v) {
        return t.div == 1 ? v : "floordiv64(" + v + ", " + std::to_string(t.div) + "u)";
      };
      const std::string mul = t.narrow ? "mulw" : "mul64";
      const std::string lo_end = sign > 0 ? L : H, hi_end = sign > 0 ? H : L;
      if (!(lo0[x] && sign > 0)) lb = "add64(" + lb + ", " + mul + "(" + c + ", " + phi(lo_end) + "))";
      if (!(lo0[x] && sign < 0)) ub = "add64(" + ub + ", " + mul + "(" + c + ", " + phi(hi_end) + "))";
    }
    return true;  // the width is per member (the index table), not part of the class
  };
  auto literal = [](std::string e, const std::vector<int64_t>& kk) {
    for (size_t p = kk.size(); p-- > 0;) {
      const std::string tok = "__ldg(K + " + std::to_string(p) + ")";
      for (size_t at = e.find(tok); at != std::string::npos; at = e.find(tok, at))
        e.replace(at, tok.size(), "(" + std::to_string(kk[p]) + "LL)");
    }
    return e;
  };
  std::map<std::string, std::vector<int>> cls;  // key -> streamed members
  std::vector<std::string> cls_order;
  for (size_t di = 0; di < k.desc.size(); ++di) {
    const IrDesc& d = k.desc[di];
    if (d.opaque || d.kind == kept_kind || !defs) continue;
    std::vector<int64_t> tk;
    Gen tg(tk);
    std::string lb, ub;
    if (!sums(di, tg, lb, ub)) continue;
    const std::string key = std::to_string(d.kind) + "|" + on_expr(di) + "|" + literal(lb, tk) + "|" + literal(ub, tk);
    if (!cls.count(key)) cls_order.push_back(key);
    cls[key].push_back((int)di);
  }
  std::vector<char> in_loop(k.desc.size(), 0);
  bool any_loop = false;
  size_t nstreamed = 0;
  for (auto& e : cls) nstreamed += e.second.size();
  for (auto& e : cls)
    if (e.second.size() >= kLoopMin && nstreamed >= g_loop_kernel_min) {
      any_loop = true;
      for (int di : e.second) in_loop[di] = 1;
    }
  if (any_loop)  // kept extents with an empty interval when inactive (no on-flag per test)
    for (int j : kept)
      s << "  const int64_t mkl" << j << " = on" << j << " ? lb" << j << " : 9223372036854775807LL, mku" << j
        << " = on" << j << " ? ub" << j << " : (-9223372036854775807LL - 1);\n";
  for (size_t di = 0; di < k.desc.size(); ++di) {  // the streamed side, straight-line
    const IrDesc& d = k.desc[di];
    if (d.opaque || d.kind == kept_kind || in_loop[di]) continue;
    s << "  {\n    const bool on" << di << " = " << on_expr(di) << ";\n";
    s << "    act_" << (d.kind == KIND_R ? "r" : "w") << " |= on" << di << ";\n";
    extent(di, "    ");
    if (extents)
      s << "    if (on" << di << ") xo_put(xo, " << (d.kind == KIND_W) << ", lb" << di << ", ub" << di << ");\n";
    std::string hit = "false";
    for (int j : kept) {
      const std::string I = std::to_string(di), J = std::to_string(j);
      std::string t = "(on" + J + " & (lb" + I + " <= ub" + J + ") & (lb" + J + " <= ub" + I + "))";
      if (stride) t = "(" + t + " && may_collide(lb" + I + ", G" + I + "(), W" + I + ", lb" + J + ", G" + J + "(), W" + J + "))";
      hit += " | " + t;
    }
    // (a hull pre-filter over the kept extents was measured slower on C4:
    // the branch per streamed extent grows the code, which is what bounds it)
    s << "    ov |= on" << di << " & (" << hit << ");\n  }\n";
  }
  for (const std::string& key : cls_order) {  // the streamed side, loop classes
    const std::vector<int>& mem = cls[key];
    if (!in_loop[mem[0]]) continue;
    const int d0 = mem[0];
    std::string idx;
    for (int di : mem)  // argument index | (width - 1) << 8
      idx += (idx.empty() ? "" : ", ") +
             std::to_string((uint32_t)(k.desc[di].base - OPD_ARG0) | ((uint32_t)k.desc[di].width - 1) << 8) + "u";
    char name[32];
    snprintf(name, sizeof(name), "kI%016llx", (unsigned long long)fnv1a(idx));
    (*defs)[name] = "__device__ __constant__ const uint32_t " + std::string(name) + "[" + std::to_string(mem.size()) +
                    "] = {" + idx + "};\n";
    std::string lb, ub;
    sums((size_t)d0, g, lb, ub);
    s << "  {\n    const bool onC = " << on_expr(d0) << ";\n";
    s << "    act_" << (k.desc[d0].kind == KIND_R ? "r" : "w") << " |= onC;\n";
    s << "    if (onC) {\n      const int64_t LOC = " << lb << ", HIC = " << ub << ";\n";
    s << "#pragma unroll 1\n      for (int j = 0; j < " << mem.size() << "; ++j) {\n";
    s << "        const uint32_t ej = " << name << "[j];\n";
    s << "        const int64_t bj = a[ej & 0xFFu];\n";
    s << "        const int64_t lbj = add64(bj, LOC), ubj = add64(add64(bj, HIC), (int64_t)(ej >> 8));\n";
    if (extents) s << "        xo_put(xo, " << (k.desc[d0].kind == KIND_W) << ", lbj, ubj);\n";
    std::string hit = "false";
    for (int j : kept) {
      const std::string J = std::to_string(j);
      hit += " | ((lbj <= mku" + J + ") & (mkl" + J + " <= ubj))";
    }
    s << "        ov |= " << hit << ";\n      }\n    }\n  }\n";
  }
  auto any = [&](const std::vector<int>& a) {
    std::string e = "false";
    for (int i : a) e += " || on" + std::to_string(i);
    return e;
  };
  if (extents) s << "  xo.fl |= (act_r ? 1u : 0u) | (act_w ? 2u : 0u);\n";
  if (models) {
    // union length without sorting: read i contributes its bytes above the
    // highest ub of the reads before it in (lb, index) order (the sweep line)
    if (kept.size() <= 12) {
      s << "  if (inb) {\n    uint64_t un = 0;\n";
      for (int i : kept) {
        const std::string I = std::to_string(i);
        s << "    {\n      int64_t mx = (-9223372036854775807LL - 1);\n";
        for (int j : kept) {
          if (j == i) continue;
          const std::string J = std::to_string(j);
          s << "      if (on" << J << " & (lb" << J << (j < i ? " <= " : " < ") << "lb" << I << ")) mx = max64(mx, ub" << J
            << ");\n";
        }
        s << "      const int64_t st = max64(lb" << I << " - 1, mx);\n";
        s << "      if (on" << I << " & (ub" << I << " > st)) un += (uint64_t)(ub" << I << " - st);\n    }\n";
      }
      s << "    *inb = (" << any(opq_r) << ") ? kInbUnknown : un;\n  }\n";
    } else {
      s << "  if (inb) *inb = kInbTable;\n";
    }
  }
  if (!opq_r.empty() || !opq_w.empty())  // opaque rule before overlap (precedence 9 < 10)
    s << "  if (((" << any(opq_r) << ") && act_w) || ((" << any(opq_w) << ") && act_r)) return V_NI_OPAQUE;\n";
  s << "  return ov ? V_NI_OVERLAP : V_IDEM_CHECKED;\n}\n";
  return s.str();
}

uint64_t fnv1a(const std::string& s) {
  uint64_t h = 1469598103934665603ULL;
  for (unsigned char c : s) h = (h ^ c) * 1099511628211ULL;
  return h;
}

// Module cache directory: $PICKER_JIT_CACHE, else $XDG_CACHE_HOME/picker_jit,
// else $HOME/.cache/picker_jit; empty (no cache) when none is set.  There is no
// shared fallback such as /tmp: a cubin found in the cache is loaded and run,
// so the cache must belong to this user (checked in owned_private()).
std::string cache_dir() {
  if (const char* e = getenv("PICKER_JIT_CACHE"); e && *e) return e;
  if (const char* x = getenv("XDG_CACHE_HOME"); x && *x) return std::string(x) + "/picker_jit";
  if (const char* h = getenv("HOME"); h && *h) return std::string(h) + "/.cache/picker_jit";
  return "";
}

// The path exists, belongs to the calling user and is not writable by group
// or others (a directory or a regular file).
bool owned_private(const std::string& p, bool dir) {
  struct stat st;
  if (lstat(p.c_str(), &st) != 0) return false;
  if (dir ? !S_ISDIR(st.st_mode) : !S_ISREG(st.st_mode)) return false;
  return st.st_uid == getuid() && (st.st_mode & (S_IWGRP | S_IWOTH)) == 0;
}

bool read_file(const std::string& p, std::string& out) {
  if (!owned_private(p, false)) return false;
  std::ifstream f(p, std::ios::binary);
  if (!f) return false;
  std::stringstream ss;
  ss << f.rdbuf();
  out = ss.str();
  return !out.empty();
}

void write_file_atomic(const std::string& dir, const std::string& name, const std::string& data) {
  for (size_t i = 1; i <= dir.size(); ++i)
    if (i == dir.size() || dir[i] == '/') mkdir(dir.substr(0, i).c_str(), 0700);
  if (!owned_private(dir, true)) return;
  std::string tmp = dir + "/" + name + ".tmp" + std::to_string(getpid());
  {
    std::ofstream f(tmp, std::ios::binary);
    if (!f) return;
    f.write(data.data(), (std::streamsize)data.size());
  }
  rename(tmp.c_str(), (dir + "/" + name).c_str());
}

bool nvrtc_compile(const std::string& src, const std::vector<std::string>& defines, std::string& cubin,
                   std::string& lowered, std::string& err) {
  nvrtcProgram prog;
  nvrtcResult r = nvrtcCreateProgram(&prog, src.c_str(), "picker_jit.cu", kEmbedCount, kEmbedSrc, kEmbedNames);
  if (r != NVRTC_SUCCESS) {
    err = nvrtcGetErrorString(r);
    return false;
  }
  const char* name_expr = src.find("k_validate_pipe<JitDispatch>") != std::string::npos
                              ? "picker::k_validate_pipe<picker::JitDispatch>"
                              : "picker::k_validate_bucket<picker::JitDispatch>";
  const char* small_expr = "picker::k_validate_small<picker::JitDispatch>";
  nvrtcAddNameExpression(prog, name_expr);
  nvrtcAddNameExpression(prog, small_expr);
  // the shape-sorted schedule's kernels (k_sorted.cuh), when the module has them
  const bool sorted = src.find("k_validate_sorted<JitDispatch>") != std::string::npos;
  const bool sorted_ws = src.find("k_validate_sorted_ws<JitDispatch>") != std::string::npos;
  const char* sort_exprs[] = {"picker::k_sort_keys", "picker::k_sort_scatter",
                              "picker::k_validate_sorted<picker::JitDispatch>", "picker::k_sort_emit",
                              "picker::k_validate_sorted_ws<picker::JitDispatch>"};
  const int nsort = sorted_ws ? 5 : 4;
  if (sorted)
    for (int q = 0; q < nsort; ++q) nvrtcAddNameExpression(prog, sort_exprs[q]);
  std::vector<const char*> opts = {"--gpu-architecture=sm_100a", "-std=c++17", "-default-device",
                                   "-lineinfo", "-DPICKER_NO_LIBC_HEADERS"};
  for (auto& d : defines) opts.push_back(d.c_str());
  r = nvrtcCompileProgram(prog, (int)opts.size(), opts.data());
  if (r != NVRTC_SUCCESS) {
    size_t n = 0;
    nvrtcGetProgramLogSize(prog, &n);
    std::string log(n, '\0');
    nvrtcGetProgramLog(prog, &log[0]);
    // the errors first (the log starts with the generated code's warnings)
    std::string errs;
    for (size_t a = 0, b; a < log.size(); a = b + 1) {
      b = log.find('\n', a);
      if (b == std::string::npos) b = log.size();
      const std::string ln = log.substr(a, b - a);
      if (ln.find("error") != std::string::npos) errs += ln + "\n";
    }
    err = std::string(nvrtcGetErrorString(r)) + ": " + (errs + log).substr(0, 4000);
    nvrtcDestroyProgram(&prog);
    return false;
  }
  const char* low = nullptr;
  nvrtcGetLoweredName(prog, name_expr, &low);
  lowered = low ? low : "";
  low = nullptr;
  nvrtcGetLoweredName(prog, small_expr, &low);
  lowered += std::string("\n") + (low ? low : "");  // main kernel, small-batch kernel
  if (sorted)
    for (int q = 0; q < nsort; ++q) {  // then the sorted schedule's kernels
      low = nullptr;
      nvrtcGetLoweredName(prog, sort_exprs[q], &low);
      lowered += std::string("\n") + (low ? low : "");
    }
  size_t n = 0;
  nvrtcGetCUBINSize(prog, &n);
  cubin.assign(n, '\0');
  nvrtcGetCUBIN(prog, &cubin[0]);
  nvrtcDestroyProgram(&prog);
  return true;
}

}  // namespace

JitPlan jit_plan(const std::vector<IrKernel>& ks, bool stride, bool sorted, bool sort_ws, int loop_min,
                 bool models, bool extents) {
  g_loop_kernel_min = (size_t)std::max(1, loop_min);
  JitPlan P;
  std::ostringstream src;
  // paths no kernel of this summary takes are left out of the module (code size)
  bool any_wide = false, any_generic = false;
  for (auto& k : ks) any_wide |= k.path == PATH_WIDE, any_generic |= k.path == PATH_GENERIC;
  const bool table_path = any_generic || (stride && any_wide);  // key 1 (and 2 in stride mode)
  src << "// generated by picker jit.cpp\n"
      << (stride || !any_wide ? "#define PICKER_NO_WIDE 1\n" : "")
      << "typedef signed char int8_t; typedef short int16_t; typedef int int32_t; typedef long long int64_t;\n"
         "typedef unsigned char uint8_t; typedef unsigned short uint16_t; typedef unsigned int uint32_t;\n"
         "typedef unsigned long long uint64_t; typedef unsigned long size_t; typedef unsigned long uintptr_t;\n"
         "#include \"eval_generic.cuh\"\n#include \"eval_stride.cuh\"\n#include \"k_bucket.cuh\"\n"
      << (sorted ? "#include \"k_sorted.cuh\"\n" : "")
      << ""
         "namespace picker {\n";
  // pass 1: body text with every constant as a load, grouped into shapes
  std::map<std::string, uint32_t> shape_id;
  std::vector<std::string> shapes;
  std::vector<std::vector<size_t>> members;
  std::vector<std::vector<int64_t>> kconst(ks.size());
  std::vector<int> shape_of(ks.size(), -1);
  std::map<std::string, std::string> idx_defs;  // argument-index tables of the loop classes
  for (size_t i = 0; i < ks.size(); ++i) {
    if (ks[i].path != PATH_JIT) continue;
    std::string body = gen_body(ks[i], kconst[i], stride, &idx_defs, models, extents);
    auto it = shape_id.find(body);
    if (it == shape_id.end()) {
      it = shape_id.emplace(body, (uint32_t)shapes.size()).first;
      shapes.push_back(body);
      members.emplace_back();
    }
    shape_of[i] = (int)it->second;
    members[it->second].push_back(i);
  }
  const uint32_t shape_shortcut = SHAPE_FIRST + (uint32_t)shapes.size();
  // pass 2: a constant position with one value across all kernels of the shape
  // becomes an immediate again; only the varying positions stay in the table.
  // A kernel's varying constants are packed as int32 words (two for a value
  // outside int32, low word first) in 16-byte blocks: the shape reads them
  // with one 128-bit load per 4 words at its start (kv[], registers).
  std::vector<std::vector<int>> slot(shapes.size());  // position -> int32 word, -1: immediate
  std::vector<std::vector<char>> wide(shapes.size());  // position needs two words
  std::vector<int> nwords(shapes.size(), 0);          // per shape, a multiple of 4
  for (size_t s = 0; s < shapes.size(); ++s) {
    const std::vector<int64_t>& k0 = kconst[members[s][0]];
    slot[s].assign(k0.size(), -1);
    wide[s].assign(k0.size(), 0);
    int q = 0;
    for (size_t p = 0; p < k0.size(); ++p) {
      bool uniform = true, fits = true;
      for (size_t i : members[s]) {
        uniform &= kconst[i][p] == k0[p];
        fits &= kconst[i][p] >= INT32_MIN && kconst[i][p] <= INT32_MAX;
      }
      if (uniform) continue;
      wide[s][p] = !fits;
      slot[s][p] = q;
      q += fits ? 1 : 2;
    }
    nwords[s] = (q + 3) & ~3;
    std::string& b = shapes[s];
    for (size_t p = k0.size(); p-- > 0;) {
      const std::string tok = "__ldg(K + " + std::to_string(p) + ")";
      const int w = slot[s][p];
      const std::string rep =
          w < 0 ? "(" + lit(k0[p]) + ")"
          : wide[s][p] ? "((int64_t)kv[" + std::to_string(w + 1) + "] << 32 | (uint32_t)kv[" + std::to_string(w) + "])"
                       : "((int64_t)kv[" + std::to_string(w) + "])";
      for (size_t at = b.find(tok); at != std::string::npos; at = b.find(tok, at + rep.size()))
        b.replace(at, tok.size(), rep);
    }
    if (nwords[s]) {  // the loads go first in the body
      const size_t at = b.find("{\n") + 2;
      b.insert(at, "  int32_t kv[" + std::to_string(nwords[s]) + "];\n#pragma unroll\n  for (int i = 0; i < " +
                       std::to_string(nwords[s] / 4) +
                       "; ++i) {\n    const int4 t = __ldg(reinterpret_cast<const int4*>(K) + i);\n"
                       "    kv[4 * i] = t.x, kv[4 * i + 1] = t.y, kv[4 * i + 2] = t.z, kv[4 * i + 3] = t.w;\n  }\n");
    }
  }
  P.meta.resize(ks.size() + 1);
  for (size_t i = 0; i < ks.size(); ++i) {
    const IrKernel& k = ks[i];
    JitMeta m{SHAPE_GENERIC, (uint32_t)P.consts.size(), (uint32_t)k.param_names.size(), 0};
    if (k.path == PATH_WIDE) {
      m.shape = SHAPE_WIDE;  // evaluated warp-cooperatively by the bucket kernel itself
    } else if (k.path == PATH_SHORTCUT) {
      m.shape = shape_shortcut;  // direct code in the KbEntry (jit_build), no constants
    } else if (k.path == PATH_JIT) {
      const int s = shape_of[i];
      m.shape = SHAPE_FIRST + (uint32_t)s;
      if (P.consts.size() & 1) P.consts.push_back(0);  // 16-byte aligned block
      m.koff = (uint32_t)P.consts.size();
      std::vector<uint32_t> w(nwords[s], 0);
      for (size_t p = 0; p < kconst[i].size(); ++p) {
        if (slot[s][p] < 0) continue;
        w[slot[s][p]] = (uint32_t)(uint64_t)kconst[i][p];
        if (wide[s][p]) w[slot[s][p] + 1] = (uint32_t)((uint64_t)kconst[i][p] >> 32);
      }
      for (size_t j = 0; j < w.size(); j += 2) P.consts.push_back((int64_t)((uint64_t)w[j + 1] << 32 | w[j]));
    }
    P.meta[i] = m;
  }
  P.meta[ks.size()] = JitMeta{SHAPE_UNKNOWN, 0, 0, 0};
  if (P.consts.empty()) P.consts.push_back(0);
  for (auto& m : P.meta) P.key_of.push_back((uint16_t)m.shape);
  for (auto& d : idx_defs) src << d.second;
  for (size_t s = 0; s < shapes.size(); ++s)
    src << "__device__ __forceinline__ uint8_t ks" << s << shapes[s];
  // key = shape (warp-uniform); kn = the lane's kernel: constants offset |
  // nparams << 24 (KbEntry, read in the grouping phase)
  // local: the record's args are in the staged span (inside the pool), so
  // only the arity needs a test
  src << "struct JitDispatch {\n"
         "  static __device__ __forceinline__ uint8_t eval(uint32_t key, uint32_t bin, uint32_t kn, bool local, "
         "const BucketParams& P, const picker_rec_t& r, const int64_t* a, const DevBatch& B"
      << (models ? ", uint64_t* inb = nullptr" : "") << (extents ? ", XOut* xo = nullptr" : "") << ") {\n"
         "    (void)bin;\n"
         "    if (key == 0) return V_ERR_KERNEL;\n"
      << (!table_path ? ""
          : stride    ? "    if (key == 1 || key == 2) return eval_stride(P.T, r, a, B.args_lo, B.args_hi);\n"
                      : "    if (key == 1) return eval_generic(P.T, r, a, B.args_lo, B.args_hi);\n")
      // the pipelined kernel finishes shortcut / unknown records in its key pass
      << (shape_shortcut + 1 <= kPipeKeysMax ? std::string()
                                          : "    if (key == " + std::to_string(shape_shortcut) +
                                                ") return (uint8_t)direct_code(kn, r.nargs, r.arg_off, B.args_lo, "
                                                "B.args_hi);\n")
      // branch-free: a staged record's arguments lie inside the pool
      << "    const bool in_pool = local | ((r.arg_off >= B.args_lo) & (r.arg_off <= B.args_hi) &\n"
         "                                  ((uint64_t)r.nargs <= B.args_hi - r.arg_off));\n"
         "    if ((r.nargs != (kn >> 24)) | !in_pool) return V_ERR_ARITY;\n"
         "    if (!launch_limits_rec(r)) return V_NI_PRECOND;  // every shape's first check\n"
         "    const int64_t* __restrict__ K = P.jit_consts + (kn & 0xFFFFFFu);\n"
         "    switch (key) {\n";
  for (size_t s = 0; s < shapes.size(); ++s)
    src << "      case " << SHAPE_FIRST + s << ": return ks" << s
        << (models ? "(r, a, K, inb);\n" : extents ? "(r, a, K, *xo);\n" : "(r, a, K);\n");
  src << "    }\n    return V_ERR_KERNEL;\n  }\n};\n"
         "template __global__ void " << (shape_shortcut + 1 <= kPipeKeysMax ? "k_validate_pipe" : "k_validate_bucket")
      << "<JitDispatch>(const __grid_constant__ BucketParams, "
         "const __grid_constant__ DevBatch, uint64_t, "
         "uint8_t*, uint32_t*, unsigned long long*);\n"
         "template __global__ void k_validate_small<JitDispatch>(const __grid_constant__ BucketParams, "
         "const __grid_constant__ DevBatch, uint32_t, uint8_t*, uint32_t*, unsigned long long*);\n"
      << (sorted && shape_shortcut + 1 <= kSortKeys
              ? "template __global__ void k_validate_sorted<JitDispatch>(const __grid_constant__ BucketParams, "
                "const __grid_constant__ DevBatch, SortScratch, uint8_t*);\n"
              : "")
      << (sorted && sort_ws && shape_shortcut + 1 <= kSortKeys
              ? "template __global__ void k_validate_sorted_ws<JitDispatch>(const __grid_constant__ BucketParams, "
                "const __grid_constant__ DevBatch, SortScratch, uint8_t*);\n"
              : "")
      << ""
         "}  // namespace picker\n";
  P.src = src.str();
  P.nshapes = (int)shapes.size();
  return P;
}

void order_by_shape(std::vector<IrKernel>& ks) {
  JitPlan P = jit_plan(ks, false);
  std::vector<size_t> idx(ks.size());
  for (size_t i = 0; i < idx.size(); ++i) idx[i] = i;
  std::stable_sort(idx.begin(), idx.end(), [&](size_t a, size_t b) { return P.meta[a].shape < P.meta[b].shape; });
  std::vector<IrKernel> out;
  out.reserve(ks.size());
  for (size_t i : idx) out.push_back(std::move(ks[i]));
  ks.swap(out);
}

std::vector<std::string> geometry_defines(const Options& opt) {
  return {"-DPICKER_TILE=" + std::to_string(opt.tile), "-DPICKER_THREADS=" + std::to_string(opt.threads),
          "-DPICKER_CTAS=" + std::to_string(opt.ctas),
          "-DPICKER_ARGS_PER_REC=" + std::to_string(opt.args_per_rec),
          "-DPICKER_ARG_BUFS=" + std::to_string(opt.arg_bufs),
          opt.models ? "-DPICKER_MODELS=1" : "-DPICKER_NO_MODELS=1",
          opt.extents ? "-DPICKER_EXTENTS=1" : "-DPICKER_NO_EXTENTS=1",
          opt.seq_windows ? "-DPICKER_SEQ=1" : "-DPICKER_NO_SEQ=1",
          "-DPICKER_SORT_WARPS=" + std::to_string(std::max(1, opt.sort_warps)),
          "-DPICKER_SORT_SLOT=" + std::to_string(std::max(16, opt.sort_slot)),
          "-DPICKER_SORT_STAGES=" + std::to_string(std::max(2, opt.sort_warps)),
          "-DPICKER_PIPE_KEYS=" + std::to_string(opt.pipe_keys > 64 ? 128 : 64)};
}

bool jit_compile(const JitPlan& plan, const Options& opt, std::string& cubin, std::string& lowered,
                 bool use_cache, std::string& err) {
  const std::vector<std::string> defs = geometry_defines(opt);
  // the key covers the generated source, the geometry AND the embedded
  // headers (k_bucket.cuh, ...): a library built from changed kernels must not
  // reuse a module compiled from the old ones
  std::string key = plan.src + "|sm_100a|v5";
  for (auto& d : defs) key += "|" + d;
  for (int i = 0; i < kEmbedCount; ++i) key += "|" + std::string(kEmbedNames[i]) + "|" + kEmbedSrc[i];
  const uint64_t h = fnv1a(key);
  char name[64];
  snprintf(name, sizeof(name), "%016llx.cubin", (unsigned long long)h);
  const std::string dir = cache_dir();
  if (dir.empty() || (access(dir.c_str(), F_OK) == 0 && !owned_private(dir, true))) use_cache = false;
  const std::string meta_name = std::string(name) + ".name";
  if (use_cache && read_file(dir + "/" + name, cubin) && read_file(dir + "/" + meta_name, lowered))
    return true;
  if (!nvrtc_compile(plan.src, defs, cubin, lowered, err)) return false;
  if (use_cache) {
    write_file_atomic(dir, name, cubin);
    write_file_atomic(dir, meta_name, lowered);
  }
  return true;
}

// tile = 0 (auto, the default): geometry from the loaded COND kernels' mean
// parameter count.  Few arguments (C2: 3.7, C3: 3.4): 896-record tiles, 448
// threads, 5 staged argument slots per record, one argument buffer, 2 CTAs/SM
// (28 warps; profiles/r01_sweep_geometry.txt has the sweep).
// Many arguments (C4: 33): the argument spans do not fit a staging buffer
// anyway, so the shared memory goes to 2560-record tiles of headers (512
// threads, 1 CTA/SM, 1 staged slot per record, one argument buffer): more
// records per shape per tile fill the warps (C4 1.09 -> 2.01 G inst/s,
// profiles/r01_sweep_geometry.txt).
Options resolve_geometry(const std::vector<IrKernel>& ks, Options opt) {
  double sum = 0;
  int cnt = 0;
  size_t maxargs = 0;
  for (auto& k : ks)
    if (k.path == PATH_JIT || k.path == PATH_WIDE || k.path == PATH_GENERIC)
      sum += k.param_names.size(), ++cnt, maxargs = std::max(maxargs, k.param_names.size());
  const double mean = cnt ? sum / cnt : 4.0;
  // shape-sorted schedule (k_sorted.cuh) for many-argument summaries: one
  // argument slot per lane (the 16-byte-rounded span of up to 62 arguments;
  // longer records read global memory), as many warps as ~200 KB of slots hold
  if (opt.sorted < 0) opt.sorted = mean > 6.0 && !opt.stride;
  if (opt.sorted) {
    const int slot = (int)((std::min<size_t>(std::max<size_t>(maxargs, 1), 62) * 8 + 16 + 15) / 16 * 16);
    if (opt.sort_slot <= 0) opt.sort_slot = slot;
    opt.sort_slot = (opt.sort_slot + 15) / 16 * 16;
    if (opt.sort_ws < 0) opt.sort_ws = 0;  // measured: the warp-specialised S4 is slower (r02_ab_log)
    // plain: one slot per lane; warp-specialised: one stage (32 headers + 32
    // slots) per warp (stages >= consumers + 1)
    if (opt.sort_warps <= 0)
      opt.sort_warps = opt.sort_ws ? std::max(2, std::min(16, (210 * 1024) / (32 * (opt.sort_slot + 32))))
                                   : std::max(1, std::min(16, (200 * 1024) / (32 * opt.sort_slot)));
  }
  if (opt.tile != 0) return opt;
  if (mean <= 6.0) {
    // one argument buffer (the arguments of a tile are fetched while the
    // previous tile is emitted and this one scattered) leaves room for 28
    // warps/SM at 72 registers, no spills: 2 CTAs x 448 threads on 896-record
    // tiles (fuller groups: C2 49.9-50.4 G inst/s) rather than 4 x 224 on 448
    // (C2 47.9-48.1, C3 +1.7 %); profiles/r01_sweep_geometry.txt
    opt.tile = 896, opt.threads = 448, opt.ctas = 2, opt.args_per_rec = 5, opt.arg_bufs = 1;
    // the models module keeps model sums live across the tile loop: 102
    // registers per thread (C2 fused f3 0.953 -> 0.831 ms; r02_ab_log)
    if (opt.models) opt.tile = 640, opt.threads = 320, opt.args_per_rec = 6;
  } else {
    // one argument buffer: its 16 KB go to 2560-record tiles (C4 1.96 -> 2.01 G inst/s)
    opt.tile = 2560, opt.threads = 512, opt.ctas = 1, opt.args_per_rec = 1, opt.arg_bufs = 1;
  }
  return opt;
}

// After planning: few-argument summaries with more than 64 grouping keys (the
// 128-key module; C2-heavy: 70) get one CTA of 28 warps per SM on 1792-record
// tiles: twice the records per key per tile fill the warps' groups, and the
// tile's barrier tail is spread over twice the work (C2-heavy 0.211 -> 0.273 of
// the HBM peak; C2 with 34 keys and C3 are faster on 2 x 896: r02_ab_log).
void geometry_for_keys(Options& opt, bool auto_tile, uint32_t keys) {
  if (!auto_tile || opt.sorted > 0 || keys <= 64 || opt.tile != 896) return;
  opt.tile = 1792, opt.threads = 896, opt.ctas = 1, opt.args_per_rec = 6, opt.arg_bufs = 1;
}

JitModule* jit_build(const std::vector<IrKernel>& ks, const Options& opt_in, std::string& err) {
  Options opt = resolve_geometry(ks, opt_in);
  if (opt.tile < 32 || opt.tile % 32 || opt.tile > 8192 || opt.threads < 32 || opt.threads % 32 ||
      opt.threads > 1024 || opt.ctas < 1 || opt.ctas > 8 || opt.args_per_rec < 1 || opt.arg_bufs < 1 ||
      opt.arg_bufs > 2) {
    err = "invalid tile / threads / ctas / args_per_rec options";
    return nullptr;
  }
  JitPlan plan = jit_plan(ks, opt.stride, opt.sorted > 0, opt.sort_ws > 0, opt.loop_min, opt.models, opt.extents);
  opt.pipe_keys = (int)(SHAPE_FIRST + (uint32_t)plan.nshapes + 1);
  geometry_for_keys(opt, opt_in.tile == 0, (uint32_t)opt.pipe_keys);
  if (SHAPE_FIRST + (uint32_t)plan.nshapes + 1 <= kPipeKeysMax && opt.tile % opt.threads) {
    err = "tile must be a multiple of threads";
    return nullptr;
  }
  std::string cubin, lowered;
  if (!jit_compile(plan, opt, cubin, lowered, true, err)) return nullptr;
  JitModule* m = new JitModule();
  m->nshapes = plan.nshapes;
  m->stride = opt.stride;
  m->tile = opt.tile;
  m->threads = opt.threads;
  m->ctas = opt.ctas;
  m->pipe = plan.src.find("k_validate_pipe<JitDispatch>") != std::string::npos;
  m->models = opt.models;
  m->extents = opt.extents;
  m->seq_xcap = opt.extents ? (uint32_t)opt.seq_xcap : 0u;
  m->seq_windows = opt.seq_windows;
  cudaError_t e = cudaLibraryLoadData(&m->lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
  std::vector<std::string> names;  // main, small, [the sorted schedule's kernels]
  for (size_t a = 0, b; a <= lowered.size(); a = b + 1) {
    b = lowered.find('\n', a);
    if (b == std::string::npos) b = lowered.size();
    names.push_back(lowered.substr(a, b - a));
  }
  if (e == cudaSuccess) e = cudaLibraryGetKernel(&m->kernel, m->lib, names[0].c_str());
  if (e == cudaSuccess && names.size() > 1 && !names[1].empty())
    e = cudaLibraryGetKernel(&m->small_kernel, m->lib, names[1].c_str());
  if (names.size() >= 6) {  // S1 keys, S3 scatter, S4 validate, S5 emit [, S4 warp-specialised]
    for (int q : {0, 2, 3, 4})
      if (e == cudaSuccess) e = cudaLibraryGetKernel(&m->sk[q], m->lib, names[2 + (q ? q - 1 : 0)].c_str());
    if (e == cudaSuccess && names.size() == 7) e = cudaLibraryGetKernel(&m->sk[1], m->lib, names[6].c_str());
  }
  if (e == cudaSuccess && m->sk[3]) {
    m->sort_warps = opt.sort_warps;
    m->sort_ws = opt.sort_ws != 0;
    m->sort_smem = (size_t)opt.sort_warps * 32 * opt.sort_slot;
    m->sort_ws_smem = (size_t)opt.sort_warps * (32 * 32 + 32 * (size_t)opt.sort_slot);  // stages = warps
    e = cudaFuncSetAttribute((const void*)m->sk[3], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)m->sort_smem);
    if (e == cudaSuccess && m->sk[1])
      e = cudaFuncSetAttribute((const void*)m->sk[1], cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)m->sort_ws_smem);
  }
  if (e == cudaSuccess) e = cudaMalloc(&m->d_consts, plan.consts.size() * sizeof(int64_t));
  // kernel id -> (bin | shape << 16); bins are positions in `ks`
  uint32_t maxid = 0;
  for (auto& k : ks) maxid = std::max(maxid, k.id);
  const uint32_t nbins = (uint32_t)ks.size();
  // unknown ids take the shortcut key with the direct code 0xFF (no arity check)
  m->shortcut_key = SHAPE_FIRST + (uint32_t)plan.nshapes;
  m->kb_unknown = nbins | (m->shortcut_key << 16);
  std::vector<KbEntry> kb(ks.empty() ? 1 : (size_t)maxid + 1, KbEntry{m->kb_unknown, V_ERR_KERNEL});
  for (uint32_t i = 0; i < nbins; ++i) {
    const JitMeta& jm = plan.meta[i];
    if (jm.koff >= (1u << 24) || jm.nparams > 255) {
      err = "specialised module: constant table exceeds 2^24 entries";
      jit_destroy(m);
      return nullptr;
    }
    const uint32_t kn = ks[i].path == PATH_SHORTCUT ? (uint32_t)ks[i].shortcut | kDirectArity | (jm.nparams << 24)
                                                    : jm.koff | (jm.nparams << 24);
    kb[ks[i].id] = KbEntry{i | ((uint32_t)plan.key_of[i] << 16), kn};
  }
  if (e == cudaSuccess) e = cudaMalloc(&m->d_kb, kb.size() * sizeof(KbEntry));
  if (e == cudaSuccess)
    e = cudaMemcpy(m->d_kb, kb.data(), kb.size() * sizeof(KbEntry), cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaMemcpy(m->d_consts, plan.consts.data(), plan.consts.size() * sizeof(int64_t),
                   cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    err = std::string("loading the JIT module: ") + cudaGetErrorString(e);
    jit_destroy(m);
    return nullptr;
  }
  m->nkeys = SHAPE_FIRST + (uint32_t)plan.nshapes + 1;
  m->smem = m->nkeys <= kPipeKeysMax ? pipe_smem_bytes_for((uint32_t)opt.tile, (uint32_t)opt.args_per_rec,
                                                        (uint32_t)opt.arg_bufs, opt.models,
                                                        opt.extents ? (uint32_t)opt.seq_xcap : 0u)
                                  : bucket_smem_bytes_for(m->nkeys, (uint32_t)opt.tile, (uint32_t)opt.args_per_rec);
  if (m->smem > kMaxSmem) {
    err = "shared memory of the specialised kernel exceeds 227 KB (lower tile / args_per_rec)";
    jit_destroy(m);
    return nullptr;
  }
  e = cudaFuncSetAttribute((const void*)m->kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)m->smem);
  if (e != cudaSuccess) {
    err = std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e);
    jit_destroy(m);
    return nullptr;
  }
  // the persistent grid is sized by the CTAs that are actually resident
  int resident = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, (const void*)m->kernel, m->threads, m->smem);
  if (e != cudaSuccess || resident < 1) {
    err = std::string("the specialised kernel does not fit on an SM: ") +
          (e != cudaSuccess ? cudaGetErrorString(e) : "0 resident CTAs");
    jit_destroy(m);
    return nullptr;
  }
  m->ctas = std::min(m->ctas, resident);
  return m;
}

bool jit_is_stride(const JitModule* m) { return m && m->stride; }

int jit_warps_per_sm(const JitModule* m) { return m ? m->ctas * m->threads / 32 : 0; }

bool jit_small_path(const JitModule* m, uint64_t n) { return m && m->small_kernel && n <= kSmallMax; }
bool jit_fused_models(const JitModule* m, uint64_t n) {
  return m && m->models && m->pipe && !m->sk[3] && !jit_small_path(m, n);
}
bool jit_extents_ok(const JitModule* m, uint64_t n) {
  return m && m->extents && m->pipe && !m->sk[3] && !jit_small_path(m, n);
}
bool jit_seq_fused(const JitModule* m, uint64_t n, uint32_t window) {
  return jit_extents_ok(m, n) && m->seq_xcap && m->nkeys <= kPipeKeysMax && window <= 32 && m->tile % window == 0;
}
bool jit_seq_lazy(const JitModule* m, uint64_t n, uint32_t window) {
  return m && m->seq_windows && m->pipe && !m->sk[3] && !jit_small_path(m, n) && m->nkeys <= kPipeKeysMax &&
         window <= 32 && m->tile % window == 0;
}
uint64_t jit_pipe_warps(const JitModule* m, uint64_t n, int num_sms) {
  const uint64_t ntiles = (n + m->tile - 1) / m->tile, cap = (uint64_t)num_sms * m->ctas;
  return (ntiles < cap ? ntiles : cap) * (uint64_t)(m->threads / 32);
}

int jit_launch_count(const JitModule* m, uint64_t n) {
  return m && m->sk[3] && n > kSmallMax && n < (1ULL << 32) ? 4 : 1;
}

void jit_destroy(JitModule* m) {
  if (!m) return;
  if (m->sort_buf) cudaFree(m->sort_buf);
  if (m->lib) cudaLibraryUnload(m->lib);
  if (m->d_consts) cudaFree(m->d_consts);
  if (m->d_kb) cudaFree(m->d_kb);
  delete m;
}

cudaError_t launch_jit(JitModule* m, const BucketParams& P0, const DevBatch& B, uint64_t n,
                       uint8_t* flags, uint32_t* bits, unsigned long long* counts, int num_sms,
                       cudaStream_t s) {
  BucketParams P = P0;
  P.jit_consts = m->d_consts;
  P.kb_of = m->d_kb;
  P.kb_unknown = m->kb_unknown;
  P.nkeys = m->nkeys;
  P.wide_key = m->stride ? 0xFFFFFFFFu : SHAPE_WIDE;  // stride mode: wide kernels through eval_stride
  P.direct_key = m->shortcut_key;
  if (jit_small_path(m, n)) {  // one CTA, counts written (no memset needed)
    uint32_t n32 = (uint32_t)n;
    void* argv[] = {(void*)&P, (void*)&B, (void*)&n32, (void*)&flags, (void*)&bits, (void*)&counts};
    return cudaLaunchKernel((const void*)m->small_kernel, dim3(1), dim3(kSmallThreads), argv, 0, s);
  }
  if (m->sk[3] && n < (1ULL << 32)) {  // shape-sorted schedule (k_sorted.cuh)
    SortScratch S{};
    S.nblk = (uint32_t)std::min<uint64_t>({(n + 4095) / 4096, (uint64_t)num_sms * 4, (uint64_t)kSortMaxBlk});
    S.chunk = (uint32_t)(((n + S.nblk - 1) / S.nblk + 31) & ~31ULL);
    const uint32_t max_blk = kSortMaxBlk;
    bool fresh = false;
    if (m->sort_cap < n) {  // keys, permutation, (key, block) counts, per-key tables
      fresh = true;
      if (m->sort_buf) cudaFree(m->sort_buf);
      m->sort_buf = nullptr;
      m->sort_cap = 0;
      const size_t bytes = ((n + 255) & ~255ULL) * 5 + (size_t)kSortKeys * max_blk * 4 + kMetaWords * 4 + 256;
      cudaError_t e = cudaMalloc(&m->sort_buf, bytes);
      if (e != cudaSuccess) return e;
      m->sort_cap = n;
    }
    uint8_t* b = (uint8_t*)m->sort_buf;
    const size_t cap = (m->sort_cap + 255) & ~255ULL;
    S.perm = (uint32_t*)b;
    S.keys = b + cap * 4;
    S.hist = (uint32_t*)(b + cap * 5);
    S.meta = S.hist + (size_t)kSortKeys * max_blk;
    void* a1[] = {(void*)&P, (void*)&B, (void*)&n, (void*)&S, (void*)&flags};
    // key totals, claim counter, S5 ticket: zeroed once here, then by the last
    // CTA of each call's S5 (k_sort_emit)
    cudaError_t e = fresh ? cudaMemsetAsync(S.meta, 0, kMetaWords * 4, s) : cudaSuccess;
    if (e == cudaSuccess) e = cudaLaunchKernel((const void*)m->sk[0], dim3(S.nblk), dim3(kSortBlock), a1, 0, s);
    void* a3[] = {(void*)&n, (void*)&S};
    if (e == cudaSuccess) e = cudaLaunchKernel((const void*)m->sk[2], dim3(S.nblk), dim3(kSortBlock), a3, 0, s);
    void* a4[] = {(void*)&P, (void*)&B, (void*)&S, (void*)&flags};
    if (e == cudaSuccess) {
      const bool ws = m->sort_ws && m->sk[1] && n < (1ULL << 30);
      e = cudaLaunchKernel((const void*)(ws ? m->sk[1] : m->sk[3]), dim3(num_sms), dim3(m->sort_warps * 32), a4,
                           ws ? m->sort_ws_smem : m->sort_smem, s);
    }
    const uint64_t words = (n + 31) / 32;
    const unsigned eb = (unsigned)std::min<uint64_t>((words + 255) / 256, (uint64_t)num_sms * 8);
    const uint8_t* cf = flags;
    CountSlot* slot = P.count_slot;
    void* a5[] = {(void*)&cf, (void*)&n, (void*)&bits, (void*)&counts, (void*)&slot, (void*)&S.meta};
    if (e == cudaSuccess) e = cudaLaunchKernel((const void*)m->sk[4], dim3(eb), dim3(256), a5, 0, s);
    return e;
  }
  const uint64_t ntiles = (n + m->tile - 1) / m->tile;
  const uint64_t cap = (uint64_t)num_sms * m->ctas;
  const uint64_t grid = ntiles < cap ? ntiles : cap;
  void* argv[] = {(void*)&P, (void*)&B, (void*)&n, (void*)&flags, (void*)&bits, (void*)&counts};
  return cudaLaunchKernel((const void*)m->kernel, dim3((unsigned)grid), dim3(m->threads), argv, m->smem, s);
}

}  // namespace picker
