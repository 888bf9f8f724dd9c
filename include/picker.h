/*
 * picker.h -- C ABI of the B200-native Picker runtime validator.
 *
 * Picker (arXiv 2410.23661) decides, before a GPU kernel instance runs, whether
 * the instance is idempotent: "an instance is considered non-idempotent if there
 * exists any overlap in the read and write addresses of all potential memory
 * accesses, regardless of the access order ... idempotent if Picker can ensure
 * that each byte of GPU memory is either read-only or write-only"
 * (§4.1).  The addresses come from per-kernel access
 * summaries produced offline (symbolic addresses, path conditions and a global
 * condition, l.690-702) and are evaluated per instance from its launch arguments
 * and grid/block dimensions (Fig. 3, l.717-730), as ranges [LB, UB] per symbolic
 * address (l.920-951) with induction-variable compaction (l.1029-1069).
 *
 * This library runs that validation for whole batches of launch records on a
 * B200 (sm_100a).  Python reaches it through ctypes
 * (paper_2410_23661_b200/_lib.py); nothing here takes a torch type.
 *
 * Conventions for every call:
 *   - Return value: 0 (PICKER_OK) or a negative picker_status; on error a
 *     message is available from picker_last_error(ctx).
 *   - "device pointer" = a CUDA global-memory address on the context's device
 *     (e.g. from torch.empty(..., device="cuda").data_ptr()).  "host pointer" =
 *     ordinary process memory; pinned memory makes the *_host calls faster.
 *   - Calls taking a `stream` (a cudaStream_t; NULL = legacy default stream)
 *     only ENQUEUE work and return: outputs are valid after the stream is
 *     synchronised.  Inputs must stay valid and unmodified until then.
 *   - The caller owns every buffer it passes; the context owns its device
 *     summary tables and scratch until picker_destroy.
 *   - Thread safety: one context per host thread.  Loaded tables are immutable
 *     until the next picker_load_summaries on the same context.
 *   - A context's scratch is shared by its calls and regrown on demand after
 *     synchronising the CALLING stream only: calls of one context on several
 *     streams must be ordered by the caller (events), or use one stream.
 */
#ifndef PICKER_H_
#define PICKER_H_

#ifndef PICKER_NO_LIBC_HEADERS /* defined by the library's NVRTC prelude */
#include <stddef.h>
#include <stdint.h>
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------- */
typedef enum {
  PICKER_OK = 0,
  PICKER_EINVAL = -1,     /* null / misaligned pointer, n > 2^40, bad option  */
  PICKER_EFORMAT = -2,    /* summary text is not valid IR      */
  PICKER_EUNSAFE = -3,    /* summary fails the loader's soundness checks:      */
                          /* an operand without a precondition bound, possible */
                          /* int64 wrap, mixed-sign terms on one variable, a   */
                          /* fresh range not covering its definition (§6)      */
  PICKER_ENOTLOADED = -4, /* no summaries loaded yet                          */
  PICKER_ECUDA = -5,      /* a CUDA runtime / NVRTC call failed               */
  PICKER_ENOMEM = -6      /* device or host allocation failed                 */
} picker_status;

/* ---- verdict codes (one byte per record) -------------------
 * Precedence, first match wins (Fig. 3 order, l.721-730):
 *   0xFF unknown kernel id; 0xFE nargs != param count or args out of range;
 *   1 kernel-level idempotent (write-only kernel, l.769-770, l.1469-1470);
 *   2..6 kernel-level non-idempotent SO/ATOMIC/IF/PE/NA (l.771-773, Table 4);
 *   7 a precondition or a CUDA launch limit fails (l.976-979);
 *   8 the global condition fails (unbounded loops, l.743-752);
 *   9 an active non-parameter (opaque) address meets an active access of the
 *     other kind (l.761-765);
 *   10 an active read extent and an active write extent share a byte (l.658-666);
 *   0 idempotent (checked).
 * picker_exact_check only: 11 = more points than max_points_per_instance.   */
enum {
  PICKER_IDEM_CHECKED = 0,
  PICKER_IDEM_KERNEL = 1,
  PICKER_NI_KERNEL_SO = 2,
  PICKER_NI_KERNEL_ATOMIC = 3,
  PICKER_NI_KERNEL_IF = 4,
  PICKER_NI_KERNEL_PE = 5,
  PICKER_NI_KERNEL_NA = 6,
  PICKER_NI_PRECOND = 7,
  PICKER_NI_GLOBAL = 8,
  PICKER_NI_OPAQUE = 9,
  PICKER_NI_OVERLAP = 10,
  PICKER_EXACT_SKIPPED = 11,
  PICKER_ERR_ARITY = 0xFE,
  PICKER_ERR_KERNEL = 0xFF
};
/* counts_out[c] for c in 0..11; every 0xFE / 0xFF record is counted in [15]. */
#define PICKER_NUM_COUNTS 16

/* ---- launch records: 32 bytes, little-endian --------------
 * An instance = kernel identity + launch arguments + grid/block dims
 * (PAPER.md l.88).  Argument i of record r is args[rec[r].arg_off + i]; i32
 * parameters use the low 32 bits of their slot, sign-extended.              */
typedef struct {
  uint32_t kernel_id;
  uint32_t nargs;
  uint32_t grid_x;
  uint16_t grid_y, grid_z;
  uint16_t block_x, block_y, block_z, reserved;
  uint64_t arg_off;
} picker_rec_t;

/* A batch.  `rec` (16-byte aligned) and `args` (8-byte aligned) point to
 * n records and args_len int64 slots.  In picker_validate_batch /
 * picker_exact_check they are DEVICE pointers; in the *_host calls HOST
 * pointers.  args_packed = 1 promises arg_off[i+1] = arg_off[i] + nargs[i]
 * (lets the kernels stream args contiguously); 0 makes no promise.          */
typedef struct {
  const picker_rec_t* rec;
  const int64_t* args;
  uint64_t args_len;
  uint32_t args_packed;
  uint32_t reserved;
} picker_batch_t;

typedef struct picker_ctx picker_ctx_t;

/* Create a context on CUDA device `device` (>= 0).  *ctx receives the handle. */
int picker_create(picker_ctx_t** ctx, int device);

/* Destroy a context and free its device tables (after its streams are idle). */
void picker_destroy(picker_ctx_t* ctx);

/* Last error message of this context ("" if none).  Valid until the next call
 * on the context.  ctx may be NULL (returns the last create error).          */
const char* picker_last_error(const picker_ctx_t* ctx);

/* Load the per-kernel access summaries: `text` is `len` bytes of UTF-8 JSON in
 * the summary IR (kernels, params, class, pre, glob, desc with
 * guard / vars / terms) -- the analyzer output the validator loads at runtime
 * (PAPER.md l.628-629, l.690-702).  The text is copied; the caller may free it.
 * The loader verifies the summaries and flattens them into
 * device tables (synchronously; not on the per-record clock).  Replaces any
 * previously loaded set.  Returns the number of kernels (>= 0) or an error.  */
int picker_load_summaries(picker_ctx_t* ctx, const char* text, size_t len);

/* Parse and verify summaries without a device (no context needed): the same
 * checks as picker_load_summaries.  Returns the kernel count or an error; the
 * message (NUL-terminated, truncated to msg_len) goes to msg when non-NULL. */
int picker_verify_summaries(const char* text, size_t len, char* msg, size_t msg_len);

/* Generate and compile (NVRTC, sm_100a) the specialised validation module of
 * these summaries without a device -- the load-time compile of
 * picker_load_summaries, exposed for build checks.  Returns the number of
 * distinct specialised functions or an error; msg gets a status line and
 * src_out (both nullable, NUL-terminated, truncated) the generated CUDA source. */
int picker_compile_summaries(const char* text, size_t len, char* msg, size_t msg_len,
                             char* src_out, size_t src_len);

/* Validate n launch records (device pointers) on `stream` (Fig. 3 with the
 * range model of §5.1-5.3).  Outputs (device pointers, caller-owned):
 *   flags_out[n]            one verdict code per record (required);
 *   idem_bits_out[ceil(n/32)] bit (r % 32) of word r/32 = 1 iff record r is
 *                            idempotent (code 0 or 1); NULL to skip;
 *   counts_out[16]          per-code histogram (overwritten, not
 *                            accumulated); NULL to skip.
 * Bad records are not call errors: they get codes 0xFE / 0xFF.
 * The launch writes counts_out itself (no memset launch): its CTAs add into
 * one of the context's 64 histogram slots, the last CTA copies it out and
 * clears it.  So at most 64 calls of one context may be in flight at once
 * (on any streams); more need more contexts.                                 */
int picker_validate_batch(picker_ctx_t* ctx, const picker_batch_t* batch, uint64_t n,
                          uint8_t* flags_out, uint32_t* idem_bits_out,
                          uint64_t* counts_out, void* stream);

/* Same as picker_validate_batch, but batch->rec / batch->args and the outputs
 * are HOST pointers.  The call copies the inputs to the device, validates, and
 * copies the outputs back, pipelined in chunks on `stream` and one internal
 * stream; it returns after the outputs are in host memory (synchronous).     */
int picker_validate_batch_host(picker_ctx_t* ctx, const picker_batch_t* batch, uint64_t n,
                               uint8_t* flags_out, uint32_t* idem_bits_out,
                               uint64_t* counts_out, void* stream);

/* Exact verifier (the paper's strawman, Fig. 3 / l.717-730): identical to
 * picker_validate_batch except that the read/write test enumerates every
 * point (thread, induction and fresh variable) of every active symbolic
 * address and intersects the touched BYTES, so it has no range
 * overestimation (l.1170-1185).  Records with more than
 * max_points_per_instance points (summed over the active symbolic addresses)
 * get code 11; there is no limit on the address span.  exact_out[n] and
 * counts_out[16] are device pointers (counts_out nullable); n < 2^32.
 * Intended for small grids.  Asynchronous on `stream`, like
 * picker_validate_batch.  The context keeps a device arena for the byte-set
 * tables (>= 512 MB, 16 B per table entry, up to 2 entries per 64-byte block
 * a point can write); it grows when max_points needs more (PICKER_ECUDA if
 * that allocation fails).  PICKER_EINVAL when max_points x (blocks per point
 * of the widest descriptor) exceeds 2^40.                                    */
int picker_exact_check(picker_ctx_t* ctx, const picker_batch_t* batch, uint64_t n,
                       uint8_t* exact_out, uint64_t* counts_out,
                       uint64_t max_points_per_instance, void* stream);

/* Device-side replication of a launch-record stream (K6; SURVEY §8F C5 and
 * §8 row e: shards generated on the GPU instead of copied over PCIe).  Writes
 * `copies` copies of the n base records and their argument pool: record
 * c*n + i is base record i with arg_off + c*args_len; slot c*args_len + j is
 * args[j] + (ptr_mask[j] ? (first_copy + c) * delta : 0).  Moving every
 * pointer argument of an instance by the same amount keeps its verdict
 * (translation invariance) as long as the preconditions still
 * hold -- the caller picks delta.  All pointers are DEVICE pointers: batch->rec
 * (n records), batch->args (args_len slots), ptr_mask (args_len bytes),
 * rec_out (n*copies records, 16-byte aligned), args_out (args_len*copies
 * slots).  Asynchronous on `stream`.  PICKER_EINVAL on null / misaligned
 * pointers or more than 2^40 output records.                                   */
int picker_replicate(picker_ctx_t* ctx, const picker_batch_t* batch, uint64_t n, const uint8_t* ptr_mask,
                     uint64_t copies, uint64_t first_copy, int64_t delta, picker_rec_t* rec_out,
                     int64_t* args_out, void* stream);

/* Multi-kernel idempotency: the stream is cut into
 * consecutive windows of `window` launches (1..1024; record order = launch
 * order) and each window is validated as one unit.  mode 0 (sequential list):
 * NI when a write of instance j can clobber a byte read by instance i <= j
 * ("checks the clobber anti-dependency across the instances"); mode 1
 * (concurrent set): NI when any read and any write of the window overlap.  The
 * first record whose own check is decided before any address (0xFF, 0xFE, 2-8;
 * kernel-level idempotent instances take part with their writes) decides the
 * window; then the opaque rule (9); then the overlap (10); else 0.
 * Windows of <= 32 launches dividing the specialised kernel's tile (n > 1,024,
 * specialised kernels only): decided inside K1's pipelined kernel, one warp
 * per window (seq.cuh; option "seq_lazy").  Otherwise: K1's extents to a
 * global arena, then sort + sweep passes over each window's extents
 * (k_seq.cu): concurrent, one pass; sequential, a divide and conquer over
 * launch order.  out[ceil(n/window)] is a device pointer.  PICKER_EINVAL when
 * window x (the most descriptors of a loaded kernel) exceeds 2^24.
 * Asynchronous on `stream` (the context's first call of the in-kernel path
 * synchronises it once, see "seq_lazy").                                       */
int picker_validate_sequence(picker_ctx_t* ctx, const picker_batch_t* batch, uint64_t n,
                             uint32_t window, uint32_t mode, uint8_t* out, void* stream);

/* ---- row f3: consumer models on the verdicts (§7.5) ------------- */
#define PICKER_MODEL_HIST 129 /* 1-us latency buckets; the last holds >= 128 us */
typedef struct {
  uint64_t kill_ns;           /* preemption latency of an idempotent instance:
                               * "less than 1 microsecond" (l.1677-1679) -> 1000 */
  uint64_t save_bytes_per_us; /* context-save bandwidth (> 0), bytes per us     */
} picker_model_params_t;
typedef struct {
  uint64_t n, n_idem;            /* records; records with code 0 or 1           */
  uint64_t ckpt_bytes_all;       /* AR without idempotency: sum of input bytes  */
  uint64_t ckpt_bytes_ni;        /* AR with Picker: over non-idempotent records */
  uint64_t unknown_input;        /* records whose input bytes are unknown (0)   */
  uint64_t preempt_ns_without;   /* Chimera: sum of context-save latencies      */
  uint64_t preempt_ns_with;      /* kill_ns for idempotent records instead      */
  uint64_t hist_without[PICKER_MODEL_HIST], hist_with[PICKER_MODEL_HIST];
} picker_model_out_t;

/* Checkpoint and preemption models of the paper's case studies, evaluated on
 * the device in one pass over the records and their verdict codes:
 *   Asymmetric Resilience (l.1618-1640, "AR checkpoints the input buffer of
 *   every GPU kernel instance ... For idempotent instances, AR avoids the memory
 *   checkpointing"): input bytes of a record = length of the union of its
 *   active non-opaque read extents; unknown (counted as 0, reported) for
 *   unknown kernels, arity errors, kernel-level NONIDEM classes, failed
 *   launch limits / preconditions / global conditions, opaque reads, or more
 *   than 128 read extents (reading Q25).
 *   Chimera (l.1666-1690): latency = kill_ns if the record's code is 0 or 1,
 *   else ctx_bytes[i] * 1000 / save_bytes_per_us ns (ctx_bytes < 2^54).
 * codes: device u8[n] (e.g. picker_validate_batch's flags); ctx_bytes: device
 * u64[n] or NULL (all 0); out: HOST struct.  SYNCHRONOUS on `stream`.
 * Summaries of specialised kernels only, n > 1,024: one launch of the models
 * module's validation kernel (its shapes sum the read-extent unions) with
 * `codes` in place of its own verdicts; otherwise a table-driven pass.       */
int picker_consumer_models(picker_ctx_t* ctx, const picker_batch_t* batch, uint64_t n, const uint8_t* codes,
                           const uint64_t* ctx_bytes, const picker_model_params_t* params,
                           picker_model_out_t* out, void* stream);

/* Validation and the consumer models in ONE pass over the records: the
 * outputs of picker_validate_batch (flags_out required, bits / counts
 * nullable) and of picker_consumer_models on those verdicts, equal to the
 * two calls made in turn.  Each record's input bytes are computed where its
 * verdict is (the pipelined kernel of a specialised module built with the
 * model code on the first call, from the staged arguments); summaries the
 * fused kernel does not take (table path, sorted schedule, K2 kernel,
 * n <= 1024) run the two passes.  ctx_bytes: device u64[n] or NULL; out:
 * HOST struct.  SYNCHRONOUS on `stream`.                                      */
int picker_validate_models(picker_ctx_t* ctx, const picker_batch_t* batch, uint64_t n, uint8_t* flags_out,
                           uint32_t* idem_bits_out, uint64_t* counts_out, const uint64_t* ctx_bytes,
                           const picker_model_params_t* params, picker_model_out_t* out, void* stream);

/* Number of kernels loaded and the path each kernel was compiled to
 * (per-kernel introspection for tests): path_out[i] for kernel id ids_out[i];
 * path 0 = shortcut, 1 = generic table path, 2 = specialised (JIT) path,
 * 3 = wide (sort + sweep) path.  Either array may be NULL; cap bounds both.  */
int picker_kernel_info(picker_ctx_t* ctx, uint32_t* ids_out, uint8_t* path_out, uint32_t cap);

/* Options.  Tuning keys (semantics never depend on them; they take effect at
 * the next picker_load_summaries):
 *   "jit"          0 = table-driven kernels only, 1 = NVRTC-specialised (default 1)
 *   "bucket"       table-driven kernels: 1 = group each tile by kernel, 0 = one
 *                  thread per record, -1 = by the summary (default; grouped when
 *                  COND kernels average more than 8 descriptors)
 *   "wide_pairs"   R*W pair count above which a kernel uses the wide path
 *   "force_path"   0 = automatic, 1 = generic, 2 = jit, 3 = wide
 *   "tile", "threads", "ctas", "args_per_rec", "arg_bufs"   specialised kernel
 *                  geometry (0 tile = chosen from the summaries)
 *   "sorted", "sort_warps", "sort_slot", "sort_ws"   shape-sorted schedule of
 *                  many-argument summaries (-1 / 0 = automatic)
 *   "loop_min"     streamed descriptors from which a specialised shape loops
 *                  over classes of descriptors (default 6)
 *   "wide_kernel"  summaries whose evaluating kernels are all wide: the K2
 *                  persistent kernel (-1 default / 1) or the module's schedules (0)
 *   "seq_k1"       picker_validate_sequence on K1's verdicts and extents (1,
 *                  default, where the summary allows it) or on the tables (0)
 *   "seq_lazy"     windows of <= 32 launches decided from K1's codes, extents
 *                  evaluated only for windows without a decisive record (1),
 *                  always from K1's extents (0), or -1 (default): chosen by the
 *                  context's first call (lazy when <= 1/16 of its windows need
 *                  extents; that call synchronises its stream once)
 * Semantic key (takes effect at the next picker_validate_batch[_host]):
 *   "stride"       1 = stride-aware ranges (reading Q24 of
 *                  DESIGN.md): a read/write pair whose byte intervals intersect
 *                  is an overlap only if their congruence classes (every address
 *                  of a descriptor = its lb mod the gcd of its varying
 *                  coefficients) can share a byte.  Refines code 10 -> 0 on
 *                  strided sets; every other code is
 *                  unchanged.  Default 0 (the paper's range model).
 * Unknown keys: PICKER_EINVAL.                                                */
int picker_set_option(picker_ctx_t* ctx, const char* key, int64_t value);

/* Per-kernel-launch statistics of the last validate call: number of device
 * kernels this library launched (for the bench's gpu_launches).             */
int picker_last_launch_count(const picker_ctx_t* ctx);

#ifdef __cplusplus
}
#endif
#endif /* PICKER_H_ */
