// Summary loader: parse, verify (§6), flatten (§7).
//
// The verifier is what makes the device arithmetic trustworthy: the paper
// assumes preconditions such as "A<2^56, N<2^5, bdim<2^10" so that symbolic
// addresses do not overflow and are monotone, and proves
// monotonicity offline with an SMT solver (l.953-965).  Here every summary is
// checked with interval arithmetic over the precondition (and global
// condition) box: no coefficient, bound, term or partial sum can leave int64,
// and the terms on one variable share a sign, so evaluating each variable at
// its two endpoints gives the exact minimum and maximum (l.950-951).
#include "loader.hpp"

#include <algorithm>
#include <cstring>
#include <map>
#include <set>

#include "../../include/picker.h"
#include "json.hpp"

namespace picker {

namespace {

using i128 = __int128;
constexpr i128 I64MIN = -(((i128)1) << 63);
constexpr i128 I64MAX = (((i128)1) << 63) - 1;

[[noreturn]] void ferr(const std::string& m) { throw LoadError{PICKER_EFORMAT, m}; }
[[noreturn]] void uerr(const std::string& m) { throw LoadError{PICKER_EUNSAFE, m}; }

int64_t as_i64(const Json& j, const std::string& what) {
  i128 v = j.integer();
  if (v < I64MIN || v > I64MAX) ferr(what + ": integer outside int64");
  return (int64_t)v;
}

const char* kDimNames[6] = {"gdim.x", "gdim.y", "gdim.z", "bdim.x", "bdim.y", "bdim.z"};

struct NameMap {
  std::map<std::string, uint8_t> ops;
  explicit NameMap(const std::vector<std::string>& params) {
    for (int d = 0; d < 6; ++d) ops[kDimNames[d]] = (uint8_t)d;
    for (size_t i = 0; i < params.size(); ++i) {
      if (ops.count(params[i])) ferr("duplicate or reserved parameter name '" + params[i] + "'");
      ops[params[i]] = (uint8_t)(OPD_ARG0 + i);
    }
  }
  uint8_t op(const Json& j) const {
    const std::string& s = j.str();
    auto it = ops.find(s);
    if (it == ops.end()) ferr("unknown operand '" + s + "'");
    return it->second;
  }
};

// A factor list (<= 2 operands, integers folded into k) -> canonical product.
IrProd parse_prod(const NameMap& nm, int64_t k, const Json* f) {
  IrProd p{k, OPD_ONE, OPD_ONE};
  if (f) {
    const auto& fs = f->arr();
    if (fs.size() > 2) ferr("at most two factors per product");
    uint8_t o[2] = {OPD_ONE, OPD_ONE};
    int n = 0;
    i128 kk = k;
    for (auto& x : fs) {
      if (x.kind == Json::INT) {
        kk *= x.integer();
        if (kk < I64MIN || kk > I64MAX) ferr("constant factor overflows int64");
      } else {
        o[n++] = nm.op(x);
      }
    }
    p.k = (int64_t)kk;
    p.a = std::min(o[0], o[1]);
    p.b = std::max(o[0], o[1]);
  }
  return p;
}

IrBexpr parse_bexpr(const NameMap& nm, const Json& j) {
  IrBexpr e;
  e.k0 = j.get("k0") ? as_i64(j.at("k0"), "k0") : 0;
  if (const Json* p = j.get("p")) {
    if (p->arr().size() > 2) ferr("at most two products per bound expression");
    for (auto& q : p->arr()) e.p.push_back(parse_prod(nm, as_i64(q.at("k"), "k"), q.get("f")));
  }
  return e;
}

uint8_t parse_cmp(const std::string& s) {
  if (s == "<") return CMP_LT;
  if (s == "<=") return CMP_LE;
  if (s == ">") return CMP_GT;
  if (s == ">=") return CMP_GE;
  if (s == "==") return CMP_EQ;
  if (s == "!=") return CMP_NE;
  ferr("unknown comparison '" + s + "'");
}

bool parse_var_name(const std::string& n, uint8_t& skind, uint8_t& axis) {
  auto ax = [&](const std::string& s) -> int {
    if (s == "x") return 0;
    if (s == "y") return 1;
    if (s == "z") return 2;
    return -1;
  };
  axis = 0;
  for (auto pre : {std::make_pair("tid.", SK_TID), std::make_pair("bid.", SK_BID),
                   std::make_pair("gidx.", SK_GIDX)}) {
    size_t L = strlen(pre.first);
    if (n.compare(0, L, pre.first) == 0) {
      int a = ax(n.substr(L));
      if (a < 0) return false;
      skind = pre.second;
      axis = (uint8_t)a;
      return true;
    }
  }
  if ((n.compare(0, 3, "ind") == 0 || n.compare(0, 2, "fr") == 0)) {
    std::string d = n.substr(n[0] == 'i' ? 3 : 2);
    if (d.empty() || d.size() > 2) return false;
    for (char c : d)
      if (c < '0' || c > '9') return false;
    skind = SK_NONE;
    return true;
  }
  return false;
}

IrKernel parse_kernel(const Json& j) {
  IrKernel k;
  i128 id = j.at("id").integer();
  if (id < 0 || id >= (1 << 20)) ferr("kernel id must be in [0, 2^20)");
  k.id = (uint32_t)id;
  if (const Json* nm = j.get("name")) k.name = nm->kind == Json::STR ? nm->s : "";
  for (auto& p : j.at("params").arr()) {
    k.param_names.push_back(p.at("name").str());
    const std::string& kind = p.at("kind").str();
    if (kind != "ptr" && kind != "i64" && kind != "i32") ferr("unknown param kind '" + kind + "'");
    k.param_i32.push_back(kind == "i32");
  }
  if (k.param_names.size() > 192) ferr("more than 192 parameters");
  NameMap nm(k.param_names);

  const std::string& cls = j.at("class").str();
  if (cls == "COND") {
    k.shortcut = 0;
  } else if (cls == "IDEM") {
    k.shortcut = V_IDEM_KERNEL;
  } else if (cls == "NONIDEM") {
    const std::string& r = j.at("reason").str();
    static const char* reasons[5] = {"SO", "ATOMIC", "IF", "PE", "NA"};
    k.shortcut = 0;
    for (int i = 0; i < 5; ++i)
      if (r == reasons[i]) k.shortcut = (uint8_t)(V_NI_SO + i);
    if (!k.shortcut) ferr("unknown NONIDEM reason '" + r + "'");
  } else {
    ferr("unknown class '" + cls + "'");
  }
  for (const char* key : {"pre", "glob"}) {
    const Json* lst = j.get(key);
    if (!lst) continue;
    for (auto& c : lst->arr()) {
      IrCheck ch{nm.op(c.at("op")), as_i64(c.at("lo"), "lo"), as_i64(c.at("hi"), "hi")};
      (key[0] == 'p' ? k.pre : k.glob).push_back(ch);
    }
  }
  if (k.pre.size() + k.glob.size() > 4096) ferr("too many checks");
  for (auto& dj : j.at("desc").arr()) {
    IrDesc d;
    const std::string& kind = dj.at("kind").str();
    if (kind != "R" && kind != "W") ferr("descriptor kind must be R or W");
    d.kind = kind == "R" ? KIND_R : KIND_W;
    i128 w = dj.at("width").integer();
    if (w < 1 || w > 4096) ferr("width must be in [1, 4096]");
    d.width = (uint32_t)w;
    d.opaque = dj.get("opaque") ? dj.at("opaque").boolean() : false;
    const Json* base = dj.get("base");
    d.base = (base && !base->is_null()) ? nm.op(*base) : OPD_NONE;
    if (const Json* g = dj.get("guard")) {
      for (auto& gj : g->arr()) {
        IrGuard gd;
        gd.a = nm.op(gj.at("a"));
        gd.cmp = parse_cmp(gj.at("cmp").str());
        const Json& b = gj.at("b");
        if (b.kind == Json::INT) {
          gd.b = OPD_NONE;
          gd.bconst = as_i64(b, "guard constant");
        } else {
          gd.b = nm.op(b);
          gd.bconst = 0;
        }
        d.guard.push_back(gd);
      }
    }
    if (d.guard.size() > 32) ferr("too many guard comparisons");
    std::map<std::string, int> vidx;
    if (const Json* vs = dj.get("vars")) {
      if (vs->kind != Json::OBJ) ferr("vars must be an object");
      for (auto& kv : vs->o) {
        IrVar v;
        v.name = kv.first;
        if (!parse_var_name(v.name, v.skind, v.axis)) ferr("unknown variable '" + v.name + "'");
        if (vidx.count(v.name)) ferr("duplicate variable '" + v.name + "'");
        if (const Json* lo = kv.second.get("lo"))
          for (auto& e : lo->arr()) v.lo.push_back(parse_bexpr(nm, e));
        if (const Json* hi = kv.second.get("hi"))
          for (auto& e : hi->arr()) v.hi.push_back(parse_bexpr(nm, e));
        if (v.lo.size() > 8 || v.hi.size() > 8) ferr("at most 8 bound expressions per side");
        if (v.skind == SK_NONE && (v.lo.empty() || v.hi.empty()))
          ferr("variable '" + v.name + "' needs declared lo and hi bounds");
        vidx[v.name] = (int)d.vars.size();
        d.vars.push_back(std::move(v));
      }
      // defs refer to variables of the same descriptor
      size_t i = 0;
      for (auto& kv : vs->o) {
        if (const Json* df = kv.second.get("def")) {
          IrVar& v = d.vars[i];
          auto it = vidx.find(df->at("src").str());
          if (it == vidx.end()) ferr("def source is not a variable of the descriptor");
          v.def_src = it->second;
          if (df->get("mod")) {
            v.def_op = DEF_MOD;
            v.def_arg = as_i64(df->at("mod"), "mod");
            if (v.def_arg < 1) ferr("mod must be >= 1");
          } else if (df->get("and")) {
            v.def_op = DEF_AND;
            v.def_arg = as_i64(df->at("and"), "and");
            if (v.def_arg < 0) ferr("and-mask must be >= 0");
          } else {
            ferr("def needs mod or and");
          }
        }
        ++i;
      }
      for (auto& v : d.vars)
        if (v.def_op != DEF_NONE && d.vars[v.def_src].def_op != DEF_NONE)
          ferr("a def source must not itself be defined");
    }
    if (d.vars.size() > 16) ferr("at most 16 variables per descriptor");
    // gidx.a excludes bid.a / tid.a in the same descriptor
    for (auto& a : d.vars)
      for (auto& b : d.vars)
        if (a.skind == SK_GIDX && (b.skind == SK_TID || b.skind == SK_BID) && a.axis == b.axis)
          ferr("descriptor mixes gidx and bid/tid on one axis");
    if (const Json* ts = dj.get("terms")) {
      for (auto& tj : ts->arr()) {
        IrTerm t;
        t.c = parse_prod(nm, as_i64(tj.at("k"), "k"), tj.get("f"));
        const Json* v = tj.get("var");
        if (!v || v->is_null()) {
          t.var = -1;
        } else {
          auto it = vidx.find(v->str());
          if (it == vidx.end()) ferr("term variable '" + v->str() + "' is not declared");
          t.var = it->second;
        }
        t.div = tj.get("div") ? as_i64(tj.at("div"), "div") : 1;
        if (t.div < 1 || t.div > (1LL << 31)) ferr("div must be in [1, 2^31]");
        d.terms.push_back(t);
      }
    }
    if (d.terms.size() > 64) ferr("at most 64 terms per descriptor");
    k.desc.push_back(std::move(d));
  }
  if (k.desc.size() > 4096) ferr("too many descriptors");
  return k;
}

// ---- interval arithmetic over i128 ----------------------------------------
struct Iv {
  i128 lo, hi;
};
Iv ivc(i128 c) { return {c, c}; }
Iv ivadd(Iv a, Iv b) { return {a.lo + b.lo, a.hi + b.hi}; }
Iv ivmul(Iv a, Iv b) {
  i128 c[4] = {a.lo * b.lo, a.lo * b.hi, a.hi * b.lo, a.hi * b.hi};
  return {*std::min_element(c, c + 4), *std::max_element(c, c + 4)};
}
bool fits(Iv a) { return a.lo >= I64MIN && a.hi <= I64MAX; }
i128 floordiv(i128 x, i128 d) {
  i128 q = x / d;
  if ((x % d != 0) && ((x < 0) != (d < 0))) --q;
  return q;
}

struct Box {
  Iv op[OPD_ARG0 + 192];
  bool bounded[OPD_ARG0 + 192];
};

}  // namespace

std::vector<IrKernel> parse_summaries(const char* text, size_t len) {
  Json root;
  try {
    root = JsonParser(text, len).parse();
  } catch (const JsonError& e) {
    ferr(e.what());
  }
  std::vector<IrKernel> out;
  try {
    if (const Json* v = root.get("version"))
      if (v->integer() != 1) ferr("unsupported summary version");
    std::set<uint32_t> ids;
    for (auto& kj : root.at("kernels").arr()) {
      out.push_back(parse_kernel(kj));
      if (!ids.insert(out.back().id).second) ferr("duplicate kernel id");
      // bins are 16-bit (KbEntry.kb = bin | key << 16); bin 65535 is reserved
      if (out.size() >= 0xFFFF) ferr("more than 65534 kernels in one summary");
    }
  } catch (const JsonError& e) {
    ferr(e.what());
  }
  return out;
}

void verify_kernel(IrKernel& k) {
  const std::string who = "kernel " + std::to_string(k.id) + " (" + k.name + "): ";
  k.var_sign.assign(k.desc.size(), {});
  // IDEM requires a write-only kernel
  if (k.shortcut == V_IDEM_KERNEL)
    for (auto& d : k.desc)
      if (d.kind == KIND_R) uerr(who + "class IDEM but the kernel reads memory");
  // kernel-level NI kernels are never evaluated; IDEM kernels are verified too,
  // because their writes take part in multi-kernel windows (reading Q23)
  if (k.shortcut != 0 && k.shortcut != V_IDEM_KERNEL) {
    k.path = PATH_SHORTCUT;
    return;
  }
  // Operand box: launch limits, i32 ranges, then pre and glob (evaluation only
  // happens when both pass, so their intersection bounds every operand).
  Box box;
  const int nops = OPD_ARG0 + (int)k.param_names.size();
  for (int o = 0; o < nops; ++o) {
    box.bounded[o] = true;
    if (o < 6) {
      box.op[o] = {1, kDimMax[o]};
    } else if (o == OPD_ONE) {
      box.op[o] = ivc(1);
    } else if (o == OPD_NONE) {
      box.op[o] = ivc(0);
    } else if (k.param_i32[o - OPD_ARG0]) {
      box.op[o] = {-(((i128)1) << 31), (((i128)1) << 31) - 1};
    } else {
      box.op[o] = {I64MIN, I64MAX};
      box.bounded[o] = false;
    }
  }
  for (auto* lst : {&k.pre, &k.glob})
    for (auto& c : *lst) {
      Iv& b = box.op[c.op];
      b.lo = std::max(b.lo, (i128)c.lo);
      b.hi = std::min(b.hi, (i128)c.hi);
      box.bounded[c.op] = true;
    }
  for (int o = 0; o < nops; ++o)
    if (box.op[o].lo > box.op[o].hi) {
      k.never_evaluates = true;  // every record fails a check before any address
      k.path = PATH_GENERIC;
      for (size_t di = 0; di < k.desc.size(); ++di) k.var_sign[di].assign(k.desc[di].vars.size(), 0);
      return;
    }
  auto need = [&](uint8_t o) {
    if (o == OPD_ONE) return;
    if (!box.bounded[o])
      uerr(who + "operand '" + k.param_names[o - OPD_ARG0] +
           "' is used in address arithmetic but has no precondition bound (PAPER.md l.976-984)");
  };
  auto prod_iv = [&](const IrProd& p, const std::string& what) {
    need(p.a);
    need(p.b);
    Iv v = ivmul(ivc(p.k), box.op[p.a]);
    if (!fits(v)) uerr(who + what + ": coefficient may overflow int64");
    v = ivmul(v, box.op[p.b]);
    if (!fits(v)) uerr(who + what + ": coefficient may overflow int64");
    return v;
  };
  auto bexpr_iv = [&](const IrBexpr& e) {
    Iv v = ivc(e.k0);
    for (auto& p : e.p) {
      v = ivadd(v, prod_iv(p, "bound"));
      if (!fits(v)) uerr(who + "bound expression may overflow int64");
    }
    return v;
  };
  for (size_t di = 0; di < k.desc.size(); ++di) {
    IrDesc& d = k.desc[di];
    std::vector<Iv> lo(d.vars.size()), hi(d.vars.size());
    for (size_t vi = 0; vi < d.vars.size(); ++vi) {
      IrVar& v = d.vars[vi];
      bool has_lo = false, has_hi = false;
      Iv L{0, 0}, H{0, 0};
      auto lo_in = [&](Iv x) {
        L = has_lo ? Iv{std::max(L.lo, x.lo), std::max(L.hi, x.hi)} : x;
        has_lo = true;
      };
      auto hi_in = [&](Iv x) {
        H = has_hi ? Iv{std::min(H.lo, x.lo), std::min(H.hi, x.hi)} : x;
        has_hi = true;
      };
      if (v.skind != SK_NONE) {
        lo_in(ivc(0));
        Iv g = box.op[OPD_GX + v.axis], b = box.op[OPD_BX + v.axis];
        Iv s = v.skind == SK_TID ? b : v.skind == SK_BID ? g : ivmul(g, b);
        hi_in(ivadd(s, ivc(-1)));
      }
      for (auto& e : v.lo) lo_in(bexpr_iv(e));
      for (auto& e : v.hi) hi_in(bexpr_iv(e));
      lo[vi] = L;
      hi[vi] = H;
      if (v.def_op != DEF_NONE) {
        // the declared range must cover the definition's values
        i128 top = v.def_op == DEF_MOD ? (i128)v.def_arg - 1 : (i128)v.def_arg;
        if (L.hi > 0 || H.lo < top)
          uerr(who + "fresh variable '" + v.name + "' range does not cover its definition");
      }
    }
    if (d.base != OPD_NONE) need(d.base);
    if (d.opaque) {
      k.var_sign[di].assign(d.vars.size(), 0);
      continue;
    }
    // terms: C * floor(x / div) at the variable's endpoints
    i128 mag = 0;
    if (d.base != OPD_NONE)
      mag += std::max(-box.op[d.base].lo, box.op[d.base].hi);
    std::vector<int> pos(d.vars.size(), 0), neg(d.vars.size(), 0), cnt(d.vars.size(), 0);
    for (auto& t : d.terms) {
      Iv c = prod_iv(t.c, "term");
      Iv x = ivc(1);
      if (t.var >= 0) {
        Iv L = lo[t.var], H = hi[t.var];
        x = {std::min(L.lo, H.lo), std::max(L.hi, H.hi)};
        x = {floordiv(x.lo, t.div), floordiv(x.hi, t.div)};
        cnt[t.var]++;
        if (c.lo >= 0) pos[t.var]++;
        if (c.hi <= 0) neg[t.var]++;
      }
      Iv tv = ivmul(c, x);
      if (!fits(tv)) uerr(who + "term may overflow int64");
      // both factors within int32 on every record that reaches the extents:
      // the specialised code multiplies them with one 32x32->64 instruction
      const i128 m31 = ((i128)1) << 31;
      t.narrow = t.var >= 0 && c.lo >= -m31 && c.hi < m31 && x.lo >= -m31 && x.hi < m31;
      mag += std::max(-tv.lo, tv.hi);
    }
    mag += d.width;
    if (mag > I64MAX) uerr(who + "address sum may overflow int64");
    k.var_sign[di].assign(d.vars.size(), 0);
    for (size_t vi = 0; vi < d.vars.size(); ++vi) {
      if (cnt[vi] == 0) continue;
      if (pos[vi] == cnt[vi]) {
        k.var_sign[di][vi] = +1;
      } else if (neg[vi] == cnt[vi]) {
        k.var_sign[di][vi] = -1;
      } else if (cnt[vi] == 1) {
        k.var_sign[di][vi] = 0;  // single term of unknown sign: min/max of both ends
      } else {
        uerr(who + "terms on variable '" + d.vars[vi].name +
             "' are not sign-definite (not provably monotone, PAPER.md l.953-965)");
      }
    }
  }
  k.path = PATH_GENERIC;
}

void flatten(const std::vector<IrKernel>& ks, HostTables& t) {
  uint32_t maxid = 0;
  for (auto& k : ks) maxid = std::max(maxid, k.id);
  t = HostTables{};
  DKernel unknown{};
  unknown.shortcut = V_ERR_KERNEL;
  unknown.path = PATH_SHORTCUT;
  t.kernels.assign(ks.empty() ? 1 : maxid + 1, unknown);
  const uint32_t nb = (uint32_t)ks.size();
  t.kb_unknown = nb | (nb << 16);
  t.kb.assign(t.kernels.size(), KbEntry{t.kb_unknown, 0});
  for (uint32_t i = 0; i < nb; ++i)  // key = bin; every wide kernel shares key nb + 1
    t.kb[ks[i].id] = KbEntry{i | ((ks[i].path == PATH_WIDE ? nb + 1 : i) << 16), 0};
  for (auto& k : ks) {
    DKernel dk{};
    dk.shortcut = k.shortcut;
    dk.nparams = (uint8_t)k.param_names.size();
    dk.path = k.path;
    for (size_t i = 0; i < k.param_i32.size(); ++i)
      if (k.param_i32[i]) dk.i32mask[i / 32] |= 1u << (i % 32);
    dk.check = (uint32_t)t.checks.size();
    dk.npre = (uint16_t)k.pre.size();
    dk.nglob = (uint16_t)k.glob.size();
    for (auto* lst : {&k.pre, &k.glob})
      for (auto& c : *lst) t.checks.push_back(DCheck{c.lo, c.hi, c.op, 0});
    // products (CSE within the kernel)
    dk.prod = (uint32_t)t.prods.size();
    std::vector<IrProd> prods;
    auto prod_id = [&](const IrProd& p) -> uint16_t {
      for (size_t i = 0; i < prods.size(); ++i)
        if (prods[i] == p) return (uint16_t)i;
      prods.push_back(p);
      return (uint16_t)(prods.size() - 1);
    };
    // variable slots (dedup identical (name, bounds) across descriptors)
    dk.var = (uint32_t)t.vars.size();
    struct Slot {
      uint8_t skind, axis;
      std::vector<std::pair<int64_t, std::vector<uint16_t>>> lo, hi;
    };
    std::vector<Slot> slots;
    auto bex_key = [&](const IrBexpr& e) {
      std::vector<uint16_t> ps;
      for (auto& p : e.p) ps.push_back(prod_id(p));
      return std::make_pair(e.k0, ps);
    };
    auto slot_id = [&](const IrVar& v) -> uint16_t {
      Slot s{v.skind, v.axis, {}, {}};
      for (auto& e : v.lo) s.lo.push_back(bex_key(e));
      for (auto& e : v.hi) s.hi.push_back(bex_key(e));
      // induction/fresh variables with equal names and bounds are the same slot
      for (size_t i = 0; i < slots.size(); ++i)
        if (slots[i].skind == s.skind && slots[i].axis == s.axis && slots[i].lo == s.lo &&
            slots[i].hi == s.hi)
          return (uint16_t)i;
      slots.push_back(s);
      return (uint16_t)(slots.size() - 1);
    };
    dk.desc = (uint32_t)t.descs.size();
    dk.ndesc = (uint16_t)k.desc.size();
    std::vector<DWSig> sigs;  // wide-path signatures of this kernel (<= ndesc)
    for (auto& d : k.desc) {
      DDesc dd{};
      dd.kind = d.kind;
      dd.opaque = d.opaque;
      dd.base = d.base;
      dd.width = d.width;
      dd.guard = (uint32_t)t.guards.size();
      dd.nguard = (uint8_t)d.guard.size();
      for (auto& g : d.guard) {
        DGuard dg{};
        dg.bconst = g.bconst;
        dg.a = g.a;
        dg.cmp = g.cmp;
        dg.b = g.b;
        t.guards.push_back(dg);
      }
      dd.var = (uint32_t)t.varlist.size();
      dd.nvar = (uint8_t)d.vars.size();
      std::vector<uint16_t> sid;
      for (auto& v : d.vars) {
        sid.push_back(slot_id(v));
        t.varlist.push_back(sid.back());
        DVarDef vd{};
        vd.op = v.def_op;
        vd.src = (uint8_t)(v.def_src < 0 ? 0 : v.def_src);
        vd.arg = v.def_arg;
        t.vardef.push_back(vd);
      }
      dd.term = (uint32_t)t.terms.size();
      dd.nterm = (uint16_t)(d.opaque ? 0 : d.terms.size());
      if (!d.opaque)
        for (auto& tm : d.terms) {
          t.terms.push_back(DTerm{prod_id(tm.c), tm.var < 0 ? kNone16 : sid[tm.var], (uint32_t)tm.div});
          t.term_lvar.push_back((uint8_t)(tm.var < 0 ? 0xFF : tm.var));
        }
      (d.kind == KIND_R ? dk.nr : dk.nw)++;
      t.descs.push_back(dd);
      // compact form (wide path, tables.hpp): signature, constant or full
      DWDesc w{};
      w.kind = dd.kind;
      w.opaque = dd.opaque;
      w.base = dd.base;
      w.wm1 = dd.width - 1;
      w.a = w.b = kNone16;
      w.mode = WD_FULL;
      if (dd.nguard == 0 && dd.nvar <= 2 && dd.nterm <= 2) {
        DWSig sg{};
        sg.vs[0] = sg.vs[1] = sg.tp[0] = sg.tp[1] = sg.tv[0] = sg.tv[1] = kNone16;
        sg.tdiv[0] = sg.tdiv[1] = 1;
        for (size_t v = 0; v < sid.size(); ++v) sg.vs[v] = sid[v];
        bool any_var = !sid.empty();
        for (uint16_t j = 0; j < dd.nterm; ++j) {
          const DTerm& tm = t.terms[dd.term + j];
          sg.tp[j] = tm.prod, sg.tv[j] = tm.var, sg.tdiv[j] = tm.div;
          any_var |= tm.var != kNone16;
        }
        if (!any_var) {
          w.mode = WD_CONST, w.a = sg.tp[0], w.b = sg.tp[1];
        } else {
          size_t s = 0;
          while (s < sigs.size() && memcmp(&sigs[s], &sg, sizeof(DWSig)) != 0) ++s;
          if (s == sigs.size() && s < (size_t)kWideSigs) sigs.push_back(sg);
          if (s < sigs.size()) w.mode = WD_SIG, w.a = (uint16_t)s;
        }
      }
      t.wdescs.push_back(w);
    }
    dk.nsig = (uint16_t)sigs.size();
    for (size_t i = 0; i < k.desc.size(); ++i) t.wsigs.push_back(i < sigs.size() ? sigs[i] : DWSig{});
    for (auto& s : slots) {
      DVar dv{};
      dv.skind = s.skind;
      dv.axis = s.axis;
      dv.nlo = (uint8_t)s.lo.size();
      dv.nhi = (uint8_t)s.hi.size();
      dv.bex = (uint32_t)t.bexprs.size();
      for (auto* side : {&s.lo, &s.hi})
        for (auto& e : *side) {
          DBexpr b{};
          b.k0 = e.first;
          b.p0 = e.second.size() > 0 ? e.second[0] : kNone16;
          b.p1 = e.second.size() > 1 ? e.second[1] : kNone16;
          t.bexprs.push_back(b);
        }
      t.vars.push_back(dv);
    }
    dk.nvar = (uint16_t)slots.size();
    for (auto& p : prods) t.prods.push_back(DProd{p.k, p.a, p.b, {0}});
    dk.nprod = (uint16_t)prods.size();
    t.kernels[k.id] = dk;
  }
}

}  // namespace picker
