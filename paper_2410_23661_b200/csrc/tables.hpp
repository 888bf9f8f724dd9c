// Flattened device tables for the summary IR.
//
// The loader (loader.cpp) verifies each kernel summary and flattens it into
// these structure-of-records arrays, uploaded once per picker_load_summaries.
// This is the B200 analog of the paper's compiled execution (PAPER.md
// l.1077-1090): no expression trees on the device, common products shared
// across terms and bounds (the "common expression extraction" of l.1088-1090),
// one variable-bound slot per distinct (variable, bound lists) pair.
#pragma once

#ifndef __CUDACC_RTC__
#include <cstdint>
#endif
#include "../../include/picker.h"

namespace picker {

// Operand codes (u8).  X[op] is the value of an operand for one record.
enum : uint8_t {
  OPD_GX = 0, OPD_GY = 1, OPD_GZ = 2,  // grid dims
  OPD_BX = 3, OPD_BY = 4, OPD_BZ = 5,  // block dims
  OPD_ONE = 6,                         // the constant 1
  OPD_NONE = 7,
  OPD_ARG0 = 8                         // argument i -> OPD_ARG0 + i
};
constexpr int kMaxParams = 247;

// Structural variable kinds (implicit thread-space bounds).
enum : uint8_t { SK_NONE = 0, SK_TID = 1, SK_BID = 2, SK_GIDX = 3 };
enum : uint8_t { CMP_LT = 0, CMP_LE, CMP_GT, CMP_GE, CMP_EQ, CMP_NE };
enum : uint8_t { KIND_R = 0, KIND_W = 1 };

constexpr uint16_t kNone16 = 0xFFFF;

// Verdict codes (mirror include/picker.h).
enum : uint8_t {
  V_IDEM_CHECKED = 0, V_IDEM_KERNEL = 1, V_NI_SO = 2, V_NI_ATOMIC = 3, V_NI_IF = 4,
  V_NI_PE = 5, V_NI_NA = 6, V_NI_PRECOND = 7, V_NI_GLOBAL = 8, V_NI_OPAQUE = 9,
  V_NI_OVERLAP = 10, V_EXACT_SKIPPED = 11, V_ERR_ARITY = 0xFE, V_ERR_KERNEL = 0xFF
};

// Execution paths per kernel.
enum : uint8_t { PATH_SHORTCUT = 0, PATH_GENERIC = 1, PATH_JIT = 2, PATH_WIDE = 3 };

struct DCheck {   // lo <= X[op] <= hi   (24 B)
  int64_t lo, hi;
  uint32_t op, pad;
};

struct DProd {    // value = k * X[a] * X[b]   (16 B)
  int64_t k;
  uint8_t a, b, pad[6];
};

struct DBexpr {   // value = k0 + P[p0] + P[p1]  (p = kNone16: absent)   (16 B)
  int64_t k0;
  uint16_t p0, p1;
  uint32_t pad;
};

struct DVar {     // one variable-bound slot   (8 B)
  uint8_t skind, axis;  // structural bounds (SK_*)
  uint8_t nlo, nhi;     // declared bexprs: lo list at bex, hi list at bex + nlo
  uint32_t bex;
};

struct DTerm {    // contribution C * floor(x / div), C = P[prod]; var = kNone16: constant C   (8 B)
  uint16_t prod, var;
  uint32_t div;
};

struct DGuard {   // X[a] cmp (b == OPD_NONE ? bconst : X[b])   (16 B)
  int64_t bconst;
  uint8_t a, cmp, b, pad[5];
};

struct DDesc {    // one symbolic address (range descriptor)   (24 B)
  uint8_t kind, opaque, base, nguard;  // base = OPD_NONE: address 0
  uint8_t nvar, pad0;
  uint16_t nterm;
  uint32_t guard;  // index into guards[]
  uint32_t var;    // index into varlist[] (u16 var-slot ids of this descriptor)
  uint32_t term;   // index into terms[]
  uint32_t width;
};

struct DKernel {  // 64 B
  uint8_t shortcut;  // 0: evaluate; otherwise the verdict code (1..6, or 0xFF unknown id)
  uint8_t nparams;
  uint8_t path;
  uint8_t pad0;
  uint16_t npre, nglob;   // checks[check .. check+npre) then glob
  uint32_t check;
  uint16_t nprod, nvar;
  uint32_t prod, var;     // prods[prod..], vars[var..]
  uint16_t ndesc, nr, nw, nsig;  // nsig: wide-path signatures (DWSig)
  uint32_t desc;
  uint32_t jit_slot;      // index of the specialised function (PATH_JIT)
  uint32_t i32mask[6];    // bit i: param i is i32 (sign-extend the low 32 bits); params < 192
};
static_assert(sizeof(DKernel) == 64, "DKernel layout");

// The wide path (k_wide.cu) reads each descriptor in one 16-byte load.  A
// descriptor without guards, with <= 2 variables and <= 2 terms is
//   mode WD_SIG:   base + the offsets of a *signature* -- its activity slots
//                  and terms, shared by every descriptor of the kernel with the
//                  same ones (a multi-tensor kernel's T tensors of one size
//                  share one), evaluated once per record;
//   mode WD_CONST: no variable: base + P[a] (+ P[b]), always active;
// any other descriptor (WD_FULL) is read through DDesc / DTerm.
enum : uint8_t { WD_SIG = 0, WD_CONST = 1, WD_FULL = 2 };
constexpr int kWideSigs = 128;  // signatures per kernel (more: WD_FULL)
struct alignas(16) DWDesc {  // 16 B, parallel to descs[]
  uint8_t kind, opaque, base, mode;
  uint16_t a, b;             // WD_SIG: a = signature; WD_CONST: product ids (kNone16: absent)
  uint32_t wm1;              // width - 1
  uint32_t pad;
};
static_assert(sizeof(DWDesc) == 16, "DWDesc layout");
struct alignas(16) DWSig {   // 32 B; the kernel's signatures are at wsigs[K.desc ..)
  uint16_t vs[2];            // variable slots whose ranges must be non-empty (kNone16: none)
  uint16_t tp[2], tv[2];     // term i: product id (kNone16: absent), variable slot (kNone16: constant)
  uint32_t tdiv[2];
  uint32_t pad[3];
};
static_assert(sizeof(DWSig) == 32, "DWSig layout");

enum : uint8_t { DEF_OP_NONE = 0, DEF_OP_MOD = 1, DEF_OP_AND = 2 };

// Exact-verifier extras, parallel to varlist[] / terms[] (picker_exact_check).
struct DVarDef {  // a fresh variable defined from another variable of the descriptor   (16 B)
  uint8_t op;     // 0: free variable (enumerated); 1: src mod arg; 2: src and arg
  uint8_t src;    // index of the source variable within the descriptor
  uint8_t pad[6];
  int64_t arg;
};

// Device-side view of all tables (passed by value to kernels).
struct Tables {
  const DKernel* kernels;
  uint32_t nkernel_slots;  // kernel ids are dense indices < nkernel_slots
  const DCheck* checks;
  const DProd* prods;
  const DBexpr* bexprs;
  const DVar* vars;
  const DTerm* terms;
  const DGuard* guards;
  const DDesc* descs;
  const uint16_t* varlist;
  const DVarDef* vardef;     // [varlist size]
  const uint8_t* term_lvar;  // [terms size]: term's variable as an index into its descriptor's vars
  const DWDesc* wdescs;      // [descs size]: compact form of descs[] (the wide path)
  const DWSig* wsigs;        // [descs size]: kernel k's signatures at [k.desc, k.desc + k.nsig)
};

// Records [0, n) at rec; argument slots valid at indices [args_lo, args_hi) of args.
struct DevBatch {
  const picker_rec_t* rec;
  const int64_t* args;
  uint64_t args_lo, args_hi;
};

// Per-bin entry of the specialised module's plan (jit.cpp, host side): the
// bin's grouping key (shape), where its constants start, its arity.
struct JitMeta {
  uint32_t shape, koff, nparams, pad;
};

// Per kernel id, read once per record when a tile is grouped (k_bucket.cuh):
// kb = bin | key << 16 (key: the grouping key), kn = offset of the kernel's
// constants | nparams << 24 (specialised module; 0 on the table path).  For
// the key BucketParams.direct_key (kernel-level shortcuts and unknown ids of
// the specialised module) kn is a direct code: code | kDirectArity (the arity
// and pool checks apply) | nparams << 24.
struct KbEntry {
  uint32_t kb, kn;
};
constexpr uint32_t kDirectArity = 0x100u;

// Per-launch histogram accumulator (device_common.cuh flush_counts); the
// context owns a ring of kCountSlots, zeroed once, each left zeroed by the
// last CTA of the launch that used it.
struct CountSlot {
  unsigned long long acc[PICKER_NUM_COUNTS];
  unsigned int ticket, pad[3];
};
constexpr int kCountSlots = 64;

// x / d for a call's invariant divisor d (save_bytes_per_us), exact for every
// u64 x (models.cuh model_div): Granlund-Montgomery with l = ceil(log2 d),
// m = floor(2^64 (2^l - d) / d) + 1, t = mulhi(m, x),
// q = (t + ((x - t) >> min(l, 1))) >> max(l - 1, 0).
struct ModelDiv {
  unsigned long long m;
  unsigned int sh1, sh2;
#ifndef __CUDACC_RTC__
  static ModelDiv of(unsigned long long d) {
    unsigned int l = 0;
    while (l < 64 && (1ull << l) < d) ++l;  // ceil(log2 d)
    const unsigned __int128 two64 = (unsigned __int128)1 << 64;
    const unsigned __int128 pl = (unsigned __int128)1 << l;
    ModelDiv v;
    v.m = (unsigned long long)((two64 * (pl - d)) / d + 1);
    v.sh1 = l < 1 ? l : 1;
    v.sh2 = l > 1 ? l - 1 : 0;
    return v;
  }
#endif
};

// Row f3 accumulator (models.cuh): sums and 1-us histograms of one call.
struct ModelAcc {
  unsigned long long n_idem, ckpt_all, ckpt_ni, unknown, pre_without, pre_with;
  unsigned long long hist_without[PICKER_MODEL_HIST], hist_with[PICKER_MODEL_HIST];
};

// Kernel-id -> bucket map for the bucketed kernels (k_bucket.cuh).
struct BucketParams {
  Tables T;
  uint32_t nbins;          // bins 0..nbins-1 are kernels; bin nbins collects unknown ids
  uint32_t nkeys;          // grouping keys 0..nkeys-1
  const struct KbEntry* kb_of;  // [T.nkernel_slots]: per kernel id, see KbEntry
  uint32_t kb_unknown;          // kb of an id that is not loaded
  const int64_t* jit_consts;   // per-kernel constants (specialised module only)
  void* wide_scratch;          // K2: kWideMax 32-byte elements per warp of the grid (desc_eval.cuh)
  uint32_t wide_key;           // grouping key of the wide (K2) kernels; 0xFFFFFFFF: none
  uint32_t direct_key;         // key whose code is final in the key pass (KbEntry.kn = direct
                               // code, see direct_code); 0xFFFFFFFF: none
  CountSlot* count_slot;       // this launch's histogram slot (flush_counts); nullptr: accumulate
  // row f3 fused into the pipelined kernel (module built with PICKER_MODELS)
  const uint64_t* ctx_bytes;   // per record, or nullptr (0)
  const uint8_t* given_codes;  // models on these verdicts (picker_consumer_models), or nullptr: the kernel's own
  unsigned long long kill_ns;
  ModelDiv save_bpu;           // divisor of the context-save latency (save_bytes_per_us)
  ModelAcc* model_acc;
  // row f1 on K1's extents (module built with PICKER_EXTENTS): per record
  // xcap extent slots (2 int64 each) and one info word (models.cuh XOut)
  int64_t* xarena;
  uint32_t* xinfo;
  uint32_t xcap;
  // ... and, with seq_out set, the windows decided inside the pipelined kernel
  // from the tile's extents in shared memory (windows of seq_window <= 32
  // launches, mode 0 sequential / 1 concurrent; tiles are a multiple of it)
  uint8_t* seq_out;
  uint32_t seq_window, seq_mode;
  // PICKER_SEQ: per-warp slot slices (32 x xcap (lb, ub)) for the windows no
  // decisive record decides, and a count of those windows (or null)
  int64_t* seq_scratch;
  uint32_t* seq_undecided;
};

// Staged + bucketed kernel geometry (k_bucket.cuh): records per tile, threads
// per CTA (one CTA per SM), staged argument slots per tile buffer.
// The specialised module is compiled with -DPICKER_TILE/THREADS/CTAS from the
// load options (tuning only); the static library uses the defaults.
#ifndef PICKER_TILE
#define PICKER_TILE 512
#endif
#ifndef PICKER_THREADS
#define PICKER_THREADS 256
#endif
#ifndef PICKER_CTAS
#define PICKER_CTAS 2
#endif
#ifndef PICKER_ARGS_PER_REC
#define PICKER_ARGS_PER_REC 8
#endif
constexpr int kTile = PICKER_TILE;
constexpr int kThreads = PICKER_THREADS;
constexpr int kWarps = kThreads / 32;
constexpr int kCtasPerSm = PICKER_CTAS;
constexpr int kArgCap = PICKER_TILE * PICKER_ARGS_PER_REC;  // staged argument slots per tile
constexpr int kArgBufBytes = kArgCap * 8 + 16;              // + alignment slack
constexpr size_t kMaxSmem = 227 * 1024;
constexpr size_t bucket_smem_bytes_for(uint32_t nkeys, uint32_t tile, uint32_t args_per_rec) {
  // 2 x (headers + args) staging buffers; s_kn (u32), s_key, s_bin, s_perm
  // (u16), s_code (u8) per record; s_cnt, s_off, s_cur (u32) per key; group table
  return (size_t)2 * tile * 32 + (size_t)2 * ((size_t)tile * args_per_rec * 8 + 16) + (size_t)tile * 11 +
         (size_t)nkeys * 12 + ((size_t)tile / 32 + nkeys) * 4 + 128;
}
constexpr size_t bucket_smem_bytes(uint32_t nkeys) {
  return bucket_smem_bytes_for(nkeys, kTile, PICKER_ARGS_PER_REC);
}
// Pipelined variant for at most kPipeKeys grouping keys (k_validate_pipe):
// staging buffers, s_perm (u32 x 2) and two s_code (u8) per record; the per-key
// counters are static shared memory.
// The specialised module is compiled with PICKER_PIPE_KEYS = 64 or 128 (its
// key count); kPipeKeysMax is the host's limit for choosing this kernel.
#ifndef PICKER_PIPE_KEYS
#define PICKER_PIPE_KEYS 64
#endif
constexpr uint32_t kPipeKeys = PICKER_PIPE_KEYS;
constexpr uint32_t kPipeKeysMax = 128;
constexpr int kKPL = (int)(kPipeKeys / 32);  // grouping keys per lane in the scan
// Small-batch kernel of the specialised module (k_validate_small): one CTA.
constexpr uint32_t kSmallMax = 1024, kSmallThreads = 256;
#ifndef PICKER_ARG_BUFS
#define PICKER_ARG_BUFS 2
#endif
constexpr int kArgBufs = PICKER_ARG_BUFS;  // 1 or 2 argument staging buffers (pipelined kernel)
// (models: + the input bytes of two tiles, u64 per record, for the emit;
// xcap > 0: + the tile's extent slots and info words of the extents module)
constexpr size_t pipe_smem_bytes_for(uint32_t tile, uint32_t args_per_rec, uint32_t arg_bufs = 2,
                                     bool models = false, uint32_t xcap = 0) {
  return (size_t)2 * tile * 32 + (size_t)arg_bufs * ((size_t)tile * args_per_rec * 8 + 16) + (size_t)tile * 10 +
         128 + (models ? (size_t)2 * tile * 8 + 8 : 0) + (xcap ? (size_t)tile * (16 * xcap + 4) + 16 : 0);
}

// K2 scratch (desc_eval.cuh): descriptors per kernel sorted in the warp's
// scratch, and the bytes of one element.
constexpr int kWideMax = 1024;
constexpr int kWideElemBytes = 32;

// Shape-sorted schedule (k_sorted.cuh): host-visible layout of its scratch.
constexpr uint32_t kSortKeys = 64;  // grouping keys of a module on the sorted schedule (<= 64)
constexpr uint32_t kSortNoKey = 0xFF;      // final code in S1, not sorted
constexpr int kSortScanThreads = 1024;
constexpr int kSortBlock = 512;  // threads of S1 / S3
constexpr uint32_t kSortMaxBlk = 32 * 24;  // blocks of S1 / S3 (kSortMaxPer per scan lane)
constexpr uint32_t kSortMaxPer = kSortMaxBlk / 32;

// Device scratch of the sorted schedule (owned by the module, jit.cpp).
struct SortScratch {
  uint8_t* keys;   // [n]
  uint32_t* perm;  // [n]: key-sorted position -> record
  uint32_t* hist;  // [kSortKeys * nblk]: offset of (key, block) within the key (S1 atomics)
  uint32_t* meta;  // key totals [kSortKeys] | claim counter (zeroed before S1)
  uint32_t nblk;   // blocks of S1 / S3
  uint32_t chunk;  // records per block (a multiple of 32)
};
constexpr uint32_t kMetaTot = 0, kMetaClaim = kSortKeys, kMetaTicket = kSortKeys + 1,
                   kMetaWords = kSortKeys + 16;  // key totals, claim counter, S5's ticket

// Generic-path limits (a kernel beyond them uses the wide path).
constexpr int kGenMaxDesc = 64;  // per kind
constexpr int kGenMaxVar = 64;

// Launch-limit preconditions (Q21).
constexpr int64_t kDimMax[6] = {2147483647LL, 65535, 65535, 1024, 1024, 64};
constexpr int64_t kBlockMaxThreads = 1024;

}  // namespace picker
