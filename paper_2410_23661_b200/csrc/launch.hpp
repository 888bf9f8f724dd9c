// Host-side launch interfaces of the device paths.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/picker.h"
#include "tables.hpp"

namespace picker {

struct IrKernel;

struct Options {
  bool jit = true;     // NVRTC-specialised functions for every COND kernel
  // table-driven paths: group each tile's records by kernel before evaluating
  // (1), one thread per record (0), or -1: by the summary -- grouped when the
  // mean descriptor count of the COND kernels exceeds 8 (measured: C2/C3
  // kernels are faster ungrouped, 3.7 vs 1.6 G inst/s; C4 grouped, 0.14 vs 0.07)
  int bucket = -1;
  int force_path = 0;  // 0 auto, 1 generic (table-driven), 2 jit, 3 wide, for every COND kernel
  int64_t wide_pairs = 1 << 20;  // read x write pairs above which a kernel takes the wide path
  // geometry of the specialised kernel (tuning; k_bucket.cuh)
  int tile = 0, threads = 256, ctas = 2, args_per_rec = 8;  // tile 0: chosen at load (jit.cpp)
  int arg_bufs = 2;  // argument staging buffers of the pipelined kernel (1: more CTAs per SM)
  bool stride = false;  // stride-aware ranges (row f4): validate through eval_stride (k_stride.cu)
  // shape-sorted schedule (k_sorted.cuh): 1 on, 0 off, -1 by the summary (on
  // for many-argument summaries, the geometry of C4); its warps per CTA and
  // per-record argument slot bytes are resolved with the geometry
  int sorted = -1, sort_warps = 0, sort_slot = 0;
  int pipe_keys = 0;  // grouping keys of the specialised module (set by jit_build)
  int sort_ws = -1;   // sorted schedule: warp-specialised S4 (1), one warp per group (0), -1 auto
  bool models = false;  // module variant with row f3 fused into the pipelined kernel (PICKER_MODELS)
  bool extents = false;  // module variant writing K1's extents for row f1 (PICKER_EXTENTS)
  bool seq_k1 = true;    // picker_validate_sequence on K1's extents when the summary allows it
  // extents module: extent slots per record held in shared memory for the
  // tile (0: the module writes them to the global arena only)
  int seq_xcap = 0;
  // module variant deciding windows in its pipelined kernel from K1's codes,
  // evaluating extents only for windows no decisive record decides (PICKER_SEQ)
  bool seq_windows = false;
  // picker_validate_sequence with that variant: 1 always, 0 never (extents
  // module), -1 by the first call (lazy while <= 1/8 of its windows need extents)
  int seq_lazy = -1;
  // summaries whose evaluating kernels are all wide: the K2 persistent kernel
  // (k_wide.cu; 1 on, 0 off = the module's schedules, -1 auto = on)
  int wide_kernel = -1;
  int loop_min = 6;  // specialised module: loop classes in kernels with >= loop_min streamed descriptors
                     // (measured: C2-heavy 0.186 -> 0.210 of the HBM peak at 6 instead of 12, C2 unchanged)
  bool wide_only = false;  // set at load: every kernel is a shortcut or PATH_WIDE
};

struct JitModule;

// Assign a path to every kernel (shortcut / generic / jit).
void select_paths(std::vector<IrKernel>& ks, const Options& opt);
bool any_jit(const std::vector<IrKernel>& ks);
JitModule* jit_build(const std::vector<IrKernel>& ks, const Options& opt, std::string& err);
void jit_destroy(JitModule* m);
// The generated module of a summary set: source, per-bin (shape, constants).
struct JitPlan {
  std::string src;
  std::vector<JitMeta> meta;   // [kernels + 1], bin order = ks order
  std::vector<int64_t> consts;
  std::vector<uint16_t> key_of;  // [kernels + 1]: grouping key (= shape) of each bin
  int nshapes = 0;
};
JitPlan jit_plan(const std::vector<IrKernel>& ks, bool stride, bool sorted = false, bool sort_ws = false,
                 int loop_min = 6, bool models = false, bool extents = false);
bool jit_is_stride(const JitModule* m);
// Kernel launches one picker_validate_batch of n records makes on the module.
int jit_launch_count(const JitModule* m, uint64_t n);
// Warps per SM of the specialised module's persistent kernel (CTAs x threads / 32).
int jit_warps_per_sm(const JitModule* m);
// The module has the small-batch kernel and n <= kSmallMax (one CTA, counts written).
bool jit_small_path(const JitModule* m, uint64_t n);
// A models module (Options.models) whose launch for n records is the fused
// pipelined kernel (not the small-batch kernel, the bucket kernel or the
// sorted schedule, which carry no model code).
bool jit_fused_models(const JitModule* m, uint64_t n);
// An extents module (Options.extents) whose launch for n records is its pipelined kernel.
// jit_seq_fused: ... that also decides windows of `window` launches itself from
// the tile's extents in shared memory (Options.seq_xcap; window <= 32 dividing
// the tile).
bool jit_seq_fused(const JitModule* m, uint64_t n, uint32_t window);
// A PICKER_SEQ module deciding windows of `window` launches for n records in
// its pipelined kernel; jit_pipe_warps: warps of that kernel's grid.
bool jit_seq_lazy(const JitModule* m, uint64_t n, uint32_t window);
uint64_t jit_pipe_warps(const JitModule* m, uint64_t n, int num_sms);
bool jit_extents_ok(const JitModule* m, uint64_t n);
cudaError_t launch_jit(JitModule* m, const BucketParams& P, const DevBatch& B, uint64_t n, uint8_t* flags,
                       uint32_t* bits, unsigned long long* counts, int num_sms, cudaStream_t s);
// Row f3 accumulator of a context: zero it on `s` / copy it to `out` and sync.
cudaError_t model_acc_begin(void** acc, cudaStream_t s);
cudaError_t model_acc_end(void* acc, uint64_t n, picker_model_out_t* out, cudaStream_t s);
// Fills in the automatic geometry (tile = 0) from the summaries.
Options resolve_geometry(const std::vector<IrKernel>& ks, Options opt);
// ... and adjusts it once the module's grouping-key count is known.
void geometry_for_keys(Options& opt, bool auto_tile, uint32_t keys);
// Stable-sort kernels by generated shape so neighbouring bins share code.
void order_by_shape(std::vector<IrKernel>& ks);
bool jit_compile(const JitPlan& plan, const Options& opt, std::string& cubin, std::string& lowered,
                 bool use_cache, std::string& err);

cudaError_t launch_validate(const BucketParams& P, JitModule* jit, const Options& opt,
                            const DevBatch& b, uint64_t n, uint8_t* flags, uint32_t* bits,
                            unsigned long long* counts, int num_sms, cudaStream_t s,
                            int* launches);

// K2 persistent kernel (k_wide.cu) and its warps per SM.
cudaError_t launch_wide(const BucketParams& P, const DevBatch& B, uint64_t n, uint8_t* flags, uint32_t* bits,
                        unsigned long long* counts, int num_sms, cudaStream_t s);
int wide_warps_per_sm();
inline bool use_wide_kernel(const Options& o) { return o.wide_only && o.wide_kernel != 0 && !o.stride; }

// `scratch` / `scratch_bytes` (f1 window slices) and `acc` (f3 accumulator):
// device buffers owned by the caller's context, grown / allocated here.
cudaError_t launch_sequence(const Tables& T, const DevBatch& b, uint64_t n, uint32_t window, uint32_t mode,
                            uint32_t max_desc, uint8_t* out, void** scratch, size_t* scratch_bytes, int num_sms,
                            cudaStream_t s, std::string& err, const uint8_t* k1_codes = nullptr,
                            const uint32_t* k1_xinfo = nullptr, const int64_t* k1_xarena = nullptr,
                            uint32_t k1_xcap = 0);

cudaError_t launch_models(const Tables& T, const DevBatch& b, uint64_t n, const uint8_t* codes,
                          const uint64_t* ctx_bytes, uint64_t kill_ns, uint64_t save_bpu, picker_model_out_t* out,
                          void** acc, int num_sms, cudaStream_t s);

// Exact verifier (k_exact.cu).  `arena` / `arena_bytes`: the byte-set table
// arena, owned by the caller's context and grown here when max_points needs it.
cudaError_t launch_exact(const Tables& T, const DevBatch& b, uint64_t n, uint8_t* out,
                         unsigned long long* counts, uint64_t max_points, uint32_t max_width,
                         void** arena, size_t* arena_bytes, int num_sms, cudaStream_t s, int* launches,
                         std::string& err);

cudaError_t launch_replicate(const picker_rec_t* rec, uint64_t n, const int64_t* args, uint64_t args_len,
                             const uint8_t* ptr_mask, uint64_t copies, uint64_t first, int64_t delta,
                             picker_rec_t* rec_out, int64_t* args_out, int num_sms, cudaStream_t s);

}  // namespace picker
