// Summary IR, its verifier and the flattener
// into device tables (tables.hpp).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "tables.hpp"

namespace picker {

struct LoadError {
  int status;  // PICKER_EFORMAT / PICKER_EUNSAFE
  std::string msg;
};

struct IrProd {      // k * X[a] * X[b]
  int64_t k;
  uint8_t a, b;      // operand codes (OPD_ONE when absent); a <= b canonical
  bool operator==(const IrProd& o) const { return k == o.k && a == o.a && b == o.b; }
};

struct IrBexpr {     // k0 + sum p
  int64_t k0;
  std::vector<IrProd> p;
};

enum : uint8_t { DEF_NONE = 0, DEF_MOD = 1, DEF_AND = 2 };

struct IrVar {
  std::string name;
  uint8_t skind, axis;  // SK_*
  std::vector<IrBexpr> lo, hi;
  uint8_t def_op = DEF_NONE;
  int def_src = -1;     // index into the descriptor's vars
  int64_t def_arg = 0;
};

struct IrTerm {
  IrProd c;
  int var;              // index into the descriptor's vars, -1: constant
  int64_t div;          // >= 1
  bool narrow = false;  // verify_kernel: coefficient and floor(x / div) both fit int32
};

struct IrGuard {
  uint8_t a, cmp, b;    // b == OPD_NONE: compare with bconst
  int64_t bconst;
};

struct IrDesc {
  uint8_t kind;         // KIND_R / KIND_W
  uint32_t width;
  bool opaque;
  uint8_t base;         // operand code or OPD_NONE
  std::vector<IrGuard> guard;
  std::vector<IrVar> vars;
  std::vector<IrTerm> terms;
};

struct IrCheck {
  uint8_t op;
  int64_t lo, hi;
};

struct IrKernel {
  uint32_t id;
  std::string name;
  std::vector<std::string> param_names;
  std::vector<uint8_t> param_i32;   // 1 if i32
  uint8_t shortcut;                 // 0 = COND, else verdict code 1..6
  std::vector<IrCheck> pre, glob;
  std::vector<IrDesc> desc;
  // Filled by the verifier:
  bool never_evaluates = false;     // pre/glob box empty: every record fails a check
  std::vector<std::vector<int8_t>> var_sign;  // per desc, per var: +1 / -1 / 0 (no terms)
  uint8_t path = PATH_GENERIC;
};

// Parse the JSON text into kernels.  Throws LoadError.
std::vector<IrKernel> parse_summaries(const char* text, size_t len);

// Verify one kernel (wrap-freedom, sign-definiteness, coverage of fresh
// definitions, class consistency).  Throws LoadError(PICKER_EUNSAFE).
void verify_kernel(IrKernel& k);

// Host images of the device tables.
struct HostTables {
  std::vector<DKernel> kernels;
  std::vector<DCheck> checks;
  std::vector<DProd> prods;
  std::vector<DBexpr> bexprs;
  std::vector<DVar> vars;
  std::vector<DTerm> terms;
  std::vector<DGuard> guards;
  std::vector<DDesc> descs;
  std::vector<uint16_t> varlist;
  std::vector<DVarDef> vardef;
  std::vector<uint8_t> term_lvar;
  std::vector<DWDesc> wdescs;    // parallel to descs
  std::vector<DWSig> wsigs;      // parallel to descs (first nsig of each kernel used)
  std::vector<KbEntry> kb;      // kernel id -> {bin | bin << 16, 0} (table-driven grouping key)
  uint32_t kb_unknown = 0;
};

void flatten(const std::vector<IrKernel>& ks, HostTables& out);

}  // namespace picker
