// C ABI (include/picker.h): context, summary loading, batch validation.
#include "../../include/picker.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "launch.hpp"
#include "loader.hpp"

using namespace picker;

struct picker_ctx {
  int device = 0;
  int num_sms = 148;
  std::string err;
  bool loaded = false;
  std::vector<IrKernel> ir;
  HostTables ht;
  void* dev_tables = nullptr;
  size_t dev_tables_bytes = 0;
  BucketParams P{};
  Options opt;
  JitModule* jit = nullptr;
  // host-path staging (two pipelines)
  void* stage[2] = {nullptr, nullptr};
  size_t stage_bytes[2] = {0, 0};
  unsigned long long* dev_counts = nullptr;
  CountSlot* count_slots = nullptr;  // kCountSlots histogram slots (flush_counts), zeroed at allocation
  uint32_t count_seq = 0;            // next slot
  void* seq_scratch = nullptr;       // row f1 window slices (grown on demand)
  size_t seq_scratch_bytes = 0;
  void* model_acc = nullptr;         // row f3 accumulator
  JitModule* jit_models = nullptr;   // the specialised module with row f3 fused (built on first use)
  JitModule* jit_extents = nullptr;  // ... writing K1's extents for row f1 (built on first use)
  void* seq_arena = nullptr;         // row f1: K1's verdicts, extent slots and info words
  JitModule* jit_seq = nullptr;      // ... deciding windows from K1's codes (PICKER_SEQ, first use)
  uint32_t* seq_undecided = nullptr;  // its count of windows that needed extents (first call)
  int seq_lazy_state = -1;           // -1: not calibrated; 0: extents module; 1: PICKER_SEQ module
  size_t seq_arena_bytes = 0;
  cudaStream_t aux = nullptr;
  void* wide_scratch = nullptr;  // K2 sort scratch, kWideMax elements per warp of a grid
  size_t wide_scratch_bytes = 0;
  void* exact_arena = nullptr;  // byte-set tables of the exact verifier
  size_t exact_arena_bytes = 0;
  uint32_t max_width = 1;       // widest descriptor of the loaded summaries
  int last_launches = 0;
  bool bucket_auto = false;  // table-driven grouping when opt.bucket = -1 (launch.hpp)
};

static std::string g_create_err;

namespace {

struct DevGuard {
  int prev = -1;
  bool ok = true;
  explicit DevGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DevGuard() {
    int cur;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

int fail(picker_ctx* c, int status, const std::string& m) {
  if (c) c->err = m;
  return status;
}

int cuda_fail(picker_ctx* c, cudaError_t e, const char* where) {
  return fail(c, PICKER_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

template <class T>
size_t append_bytes(std::vector<uint8_t>& blob, const std::vector<T>& v) {
  size_t off = (blob.size() + 255) & ~(size_t)255;
  blob.resize(off + v.size() * sizeof(T));
  if (!v.empty()) memcpy(blob.data() + off, v.data(), v.size() * sizeof(T));
  return off;
}

int check_batch(picker_ctx* c, const picker_batch_t* b, uint64_t n, const void* out) {
  if (!c) return PICKER_EINVAL;
  if (!b || (!out && n)) return fail(c, PICKER_EINVAL, "null batch or output pointer");
  if (n > (1ULL << 40)) return fail(c, PICKER_EINVAL, "n > 2^40");
  if (n && (!b->rec || ((uintptr_t)b->rec & 15)))
    return fail(c, PICKER_EINVAL, "records must be non-null and 16-byte aligned");
  if (b->args_len && (!b->args || ((uintptr_t)b->args & 7)))
    return fail(c, PICKER_EINVAL, "args must be non-null and 8-byte aligned");
  if (!c->loaded) return fail(c, PICKER_ENOTLOADED, "no summaries loaded");
  return PICKER_OK;
}

// Counts are written by the launch itself (the last CTA through a histogram
// slot, or the small-batch kernel): P.count_slot gets this call's slot;
// launch_validate zeroes counts first only on the paths without slots.
int count_slot(picker_ctx* c, uint64_t* counts, uint64_t n, cudaStream_t s, BucketParams& P) {
  if (counts && n) {
    if (!c->count_slots) {
      cudaError_t e = cudaMalloc(&c->count_slots, kCountSlots * sizeof(CountSlot));
      if (e != cudaSuccess) return fail(c, PICKER_ENOMEM, "cudaMalloc(count slots)");
      e = cudaMemset(c->count_slots, 0, kCountSlots * sizeof(CountSlot));
      if (e != cudaSuccess) return cuda_fail(c, e, "cudaMemset(count slots)");
    }
    P.count_slot = c->count_slots + (c->count_seq++ % kCountSlots);
  } else if (counts) {  // n == 0: nothing launches
    cudaError_t e = cudaMemsetAsync(counts, 0, PICKER_NUM_COUNTS * sizeof(uint64_t), s);
    if (e != cudaSuccess) return cuda_fail(c, e, "cudaMemsetAsync(counts)");
  }
  return PICKER_OK;
}

}  // namespace

extern "C" {

int picker_create(picker_ctx_t** out, int device) {
  if (!out) return PICKER_EINVAL;
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || device < 0 || device >= count) {
    g_create_err = e != cudaSuccess ? std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e)
                                    : "device index out of range";
    return e != cudaSuccess ? PICKER_ECUDA : PICKER_EINVAL;
  }
  picker_ctx* c = new (std::nothrow) picker_ctx();
  if (!c) return PICKER_ENOMEM;
  c->device = device;
  DevGuard g(device);
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  *out = c;
  return PICKER_OK;
}

void picker_destroy(picker_ctx_t* c) {
  if (!c) return;
  {
    DevGuard g(c->device);
    if (c->dev_tables) cudaFree(c->dev_tables);
    if (c->count_slots) cudaFree(c->count_slots);
    if (c->seq_scratch) cudaFree(c->seq_scratch);
    if (c->model_acc) cudaFree(c->model_acc);
    jit_destroy(c->jit_models);
    jit_destroy(c->jit_extents);
    jit_destroy(c->jit_seq);
    if (c->seq_arena) cudaFree(c->seq_arena);
    if (c->seq_undecided) cudaFree(c->seq_undecided);
    for (int i = 0; i < 2; ++i)
      if (c->stage[i]) cudaFree(c->stage[i]);
    if (c->dev_counts) cudaFree(c->dev_counts);
    if (c->aux) cudaStreamDestroy(c->aux);
    if (c->exact_arena) cudaFree(c->exact_arena);
    if (c->wide_scratch) cudaFree(c->wide_scratch);
    jit_destroy(c->jit);
  }
  delete c;
}

const char* picker_last_error(const picker_ctx_t* c) {
  return c ? c->err.c_str() : g_create_err.c_str();
}

int picker_set_option(picker_ctx_t* c, const char* key, int64_t v) {
  if (!c || !key) return PICKER_EINVAL;
  std::string k(key);
  if (k == "jit") c->opt.jit = v != 0;
  else if (k == "bucket") c->opt.bucket = v < 0 ? -1 : (int)(v != 0);
  else if (k == "force_path") c->opt.force_path = (int)v;
  else if (k == "wide_pairs") c->opt.wide_pairs = v;
  else if (k == "tile") c->opt.tile = (int)v;
  else if (k == "threads") c->opt.threads = (int)v;
  else if (k == "ctas") c->opt.ctas = (int)v;
  else if (k == "args_per_rec") c->opt.args_per_rec = (int)v;
  else if (k == "arg_bufs") c->opt.arg_bufs = (int)v;
  else if (k == "stride") c->opt.stride = v != 0;
  else if (k == "sorted") c->opt.sorted = v < 0 ? -1 : (int)(v != 0);
  else if (k == "sort_slot") c->opt.sort_slot = (int)v;    // tuning: average argument bytes per lane
  else if (k == "sort_warps") c->opt.sort_warps = (int)v;  // tuning: warps per CTA of the sorted schedule
  else if (k == "sort_ws") c->opt.sort_ws = v < 0 ? -1 : (int)(v != 0);  // warp-specialised S4
  else if (k == "loop_min") c->opt.loop_min = (int)v;  // tuning: loop classes of the specialised module
  else if (k == "seq_k1") c->opt.seq_k1 = v != 0;  // row f1 on K1's extents (1, default) or the tables (0)
  else if (k == "seq_lazy") c->opt.seq_lazy = v < 0 ? -1 : v != 0, c->seq_lazy_state = -1;
  else if (k == "wide_kernel") c->opt.wide_kernel = v < 0 ? -1 : (int)(v != 0);  // K2 kernel (k_wide.cu)
  else return fail(c, PICKER_EINVAL, "unknown option '" + k + "'");
  return PICKER_OK;
}

int picker_load_summaries(picker_ctx_t* c, const char* text, size_t len) {
  if (!c) return PICKER_EINVAL;
  if (!text && len) return fail(c, PICKER_EINVAL, "null summary text");
  DevGuard g(c->device);
  if (!g.ok) return fail(c, PICKER_ECUDA, "cudaSetDevice failed");
  std::vector<IrKernel> ks;
  HostTables ht;
  try {
    ks = parse_summaries(text, len);
    for (auto& k : ks) verify_kernel(k);
    select_paths(ks, c->opt);
    if (c->opt.jit && any_jit(ks)) order_by_shape(ks);
    flatten(ks, ht);
  } catch (const LoadError& e) {
    return fail(c, e.status, e.msg);
  } catch (const std::exception& e) {
    return fail(c, PICKER_EFORMAT, e.what());
  }
  // one device allocation for all tables
  std::vector<uint8_t> blob;
  size_t o_k = append_bytes(blob, ht.kernels), o_c = append_bytes(blob, ht.checks),
         o_p = append_bytes(blob, ht.prods), o_b = append_bytes(blob, ht.bexprs),
         o_v = append_bytes(blob, ht.vars), o_t = append_bytes(blob, ht.terms),
         o_g = append_bytes(blob, ht.guards), o_d = append_bytes(blob, ht.descs),
         o_l = append_bytes(blob, ht.varlist),
         o_kb = append_bytes(blob, ht.kb), o_vd = append_bytes(blob, ht.vardef),
         o_tl = append_bytes(blob, ht.term_lvar), o_wd = append_bytes(blob, ht.wdescs),
         o_ws = append_bytes(blob, ht.wsigs);
  blob.resize(blob.size() + 256);
  void* dev = nullptr;
  cudaError_t e = cudaMalloc(&dev, blob.size());
  if (e != cudaSuccess) return fail(c, PICKER_ENOMEM, "cudaMalloc(tables) failed");
  e = cudaMemcpy(dev, blob.data(), blob.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(dev);
    return cuda_fail(c, e, "cudaMemcpy(tables)");
  }
  JitModule* jm = nullptr;
  std::string jerr;
  if (c->opt.jit && any_jit(ks)) {
    jm = jit_build(ks, c->opt, jerr);
    if (!jm) {
      cudaFree(dev);
      return fail(c, PICKER_ECUDA, "JIT: " + jerr);
    }
  }
  // K2 scratch for kernels with more than 64 descriptors on the wide path:
  // one slice per warp of the largest persistent grid (or the small kernel)
  size_t scratch_bytes = 0;
  for (auto& k : ks)
    if (k.path == PATH_WIDE && k.desc.size() > 64) {
      const int wps = std::max({kCtasPerSm * kWarps, jit_warps_per_sm(jm), (int)(kSmallThreads / 32),
                                wide_warps_per_sm()});
      scratch_bytes = (size_t)c->num_sms * wps * kWideMax * kWideElemBytes;
      break;
    }
  if (scratch_bytes > c->wide_scratch_bytes) {
    if (c->wide_scratch) cudaFree(c->wide_scratch);
    c->wide_scratch = nullptr;
    c->wide_scratch_bytes = 0;
    if (cudaMalloc(&c->wide_scratch, scratch_bytes) != cudaSuccess) {
      cudaFree(dev);
      jit_destroy(jm);
      return fail(c, PICKER_ENOMEM, "cudaMalloc(wide scratch) failed");
    }
    c->wide_scratch_bytes = scratch_bytes;
  }
  c->P.wide_scratch = scratch_bytes ? c->wide_scratch : nullptr;
  if (c->dev_tables) cudaFree(c->dev_tables);
  jit_destroy(c->jit);
  jit_destroy(c->jit_models);
  c->jit_models = nullptr;
  jit_destroy(c->jit_extents);
  c->jit_extents = nullptr;
  jit_destroy(c->jit_seq);
  c->jit_seq = nullptr;
  c->seq_lazy_state = -1;
  c->jit = jm;
  c->dev_tables = dev;
  c->dev_tables_bytes = blob.size();
  c->max_width = 1;
  for (auto& k : ks)
    for (auto& d : k.desc) c->max_width = std::max<uint32_t>(c->max_width, (uint32_t)d.width);
  uint8_t* b = (uint8_t*)dev;
  c->P.T.kernels = (const DKernel*)(b + o_k);
  c->P.T.nkernel_slots = (uint32_t)ht.kernels.size();
  c->P.T.checks = (const DCheck*)(b + o_c);
  c->P.T.prods = (const DProd*)(b + o_p);
  c->P.T.bexprs = (const DBexpr*)(b + o_b);
  c->P.T.vars = (const DVar*)(b + o_v);
  c->P.T.terms = (const DTerm*)(b + o_t);
  c->P.T.guards = (const DGuard*)(b + o_g);
  c->P.T.descs = (const DDesc*)(b + o_d);
  c->P.T.varlist = (const uint16_t*)(b + o_l);
  c->P.kb_of = (const KbEntry*)(b + o_kb);
  c->P.T.vardef = (const DVarDef*)(b + o_vd);
  c->P.T.term_lvar = (const uint8_t*)(b + o_tl);
  c->P.T.wdescs = (const DWDesc*)(b + o_wd);
  c->P.T.wsigs = (const DWSig*)(b + o_ws);
  c->P.kb_unknown = ht.kb_unknown;
  c->P.nbins = (uint32_t)ks.size();
  c->P.wide_key = c->P.nbins + 1;  // table-driven grouping (the JIT module uses its own)
  c->P.direct_key = 0xFFFFFFFFu;   // the table path evaluates shortcuts in eval_generic
  {
    size_t nd = 0, nc = 0;
    for (auto& k : ks)
      if (k.path != PATH_SHORTCUT) nd += k.desc.size(), ++nc;
    c->bucket_auto = nc && nd > 8 * nc;
    bool any_wide = false, all_wide = true;
    for (auto& k : ks) {
      any_wide |= k.path == PATH_WIDE;
      all_wide &= k.path == PATH_WIDE || k.path == PATH_SHORTCUT;
    }
    c->opt.wide_only = any_wide && all_wide;
  }
  c->ir = std::move(ks);
  c->ht = std::move(ht);
  c->loaded = true;
  c->err.clear();
  return (int)c->ir.size();
}

int picker_verify_summaries(const char* text, size_t len, char* msg, size_t msg_len) {
  auto put = [&](const std::string& m) {
    if (msg && msg_len) {
      size_t k = std::min(m.size(), msg_len - 1);
      memcpy(msg, m.data(), k);
      msg[k] = 0;
    }
  };
  if (!text && len) {
    put("null summary text");
    return PICKER_EINVAL;
  }
  try {
    std::vector<IrKernel> ks = parse_summaries(text, len);
    for (auto& k : ks) verify_kernel(k);
    put("");
    return (int)ks.size();
  } catch (const LoadError& e) {
    put(e.msg);
    return e.status;
  } catch (const std::exception& e) {
    put(e.what());
    return PICKER_EFORMAT;
  }
}

int picker_compile_summaries(const char* text, size_t len, char* msg, size_t msg_len,
                             char* src_out, size_t src_len) {
  auto put = [&](char* dst, size_t cap, const std::string& m) {
    if (dst && cap) {
      size_t k = std::min(m.size(), cap - 1);
      memcpy(dst, m.data(), k);
      dst[k] = 0;
    }
  };
  try {
    std::vector<IrKernel> ks = parse_summaries(text, len);
    for (auto& k : ks) verify_kernel(k);
    Options opt;
    select_paths(ks, opt);
    order_by_shape(ks);
    Options geo = resolve_geometry(ks, opt);
    JitPlan plan = jit_plan(ks, false, geo.sorted > 0, geo.sort_ws > 0, geo.loop_min);
    geo.pipe_keys = 3 + plan.nshapes + 1;  // SHAPE_FIRST + shapes + the shortcut key
    geometry_for_keys(geo, opt.tile == 0, (uint32_t)geo.pipe_keys);
    std::string cubin, lowered, err;
    if (!jit_compile(plan, geo, cubin, lowered, false, err)) {
      put(msg, msg_len, err);
      put(src_out, src_len, plan.src);
      return PICKER_ECUDA;
    }
    if (const char* dump = getenv("PICKER_DUMP_CUBIN")) {  // inspection aid (cuobjdump -sass / -res-usage)
      FILE* f = fopen(dump, "wb");
      if (f) {
        fwrite(cubin.data(), 1, cubin.size(), f);
        fclose(f);
      }
    }
    put(msg, msg_len, "cubin " + std::to_string(cubin.size()) + " bytes, " +
                          std::to_string(plan.consts.size()) + " constants, kernel " + lowered);
    put(src_out, src_len, plan.src);
    return plan.nshapes;
  } catch (const LoadError& e) {
    put(msg, msg_len, e.msg);
    return e.status;
  } catch (const std::exception& e) {
    put(msg, msg_len, e.what());
    return PICKER_EFORMAT;
  }
}

int picker_kernel_info(picker_ctx_t* c, uint32_t* ids, uint8_t* paths, uint32_t cap) {
  if (!c) return PICKER_EINVAL;
  if (!c->loaded) return fail(c, PICKER_ENOTLOADED, "no summaries loaded");
  uint32_t n = 0;
  for (auto& k : c->ir) {
    if (n < cap) {
      if (ids) ids[n] = k.id;
      if (paths) paths[n] = k.path;
    }
    ++n;
  }
  return (int)n;
}

int picker_last_launch_count(const picker_ctx_t* c) { return c ? c->last_launches : 0; }

int picker_validate_batch(picker_ctx_t* c, const picker_batch_t* b, uint64_t n, uint8_t* flags,
                          uint32_t* bits, uint64_t* counts, void* stream) {
  int st = check_batch(c, b, n, flags);
  if (st) return st;
  DevGuard g(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  c->last_launches = 0;
  Options o = c->opt;
  if (o.bucket < 0) o.bucket = c->bucket_auto;
  BucketParams P = c->P;
  st = count_slot(c, counts, n, s, P);
  if (st) return st;
  DevBatch db{b->rec, b->args, 0, b->args_len};
  cudaError_t e = launch_validate(P, c->jit, o, db, n, flags, bits,
                                  (unsigned long long*)counts, c->num_sms, s, &c->last_launches);
  if (e != cudaSuccess) return cuda_fail(c, e, "validate launch");
  return PICKER_OK;
}

int picker_validate_batch_host(picker_ctx_t* c, const picker_batch_t* b, uint64_t n,
                               uint8_t* flags, uint32_t* bits, uint64_t* counts, void* stream) {
  int st = check_batch(c, b, n, flags);
  if (st) return st;
  DevGuard g(c->device);
  cudaError_t e;
  cudaStream_t s[2] = {(cudaStream_t)stream, nullptr};
  if (!c->aux) {
    e = cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking);
    if (e != cudaSuccess) return cuda_fail(c, e, "cudaStreamCreate");
  }
  s[1] = c->aux;
  if (!c->dev_counts) {
    e = cudaMalloc(&c->dev_counts, PICKER_NUM_COUNTS * sizeof(uint64_t));
    if (e != cudaSuccess) return fail(c, PICKER_ENOMEM, "cudaMalloc(counts)");
  }
  c->last_launches = 0;
  // Both pipelines start after anything already queued on the caller's stream.
  cudaEvent_t ev0;
  cudaEventCreateWithFlags(&ev0, cudaEventDisableTiming);
  e = cudaMemsetAsync(c->dev_counts, 0, PICKER_NUM_COUNTS * sizeof(uint64_t), s[0]);
  cudaEventRecord(ev0, s[0]);
  cudaStreamWaitEvent(s[1], ev0, 0);
  cudaEventDestroy(ev0);
  if (e != cudaSuccess) return cuda_fail(c, e, "cudaMemsetAsync");

  const bool packed = b->args_packed != 0;
  // Records per chunk: at most 2^22, balanced over the chunks and a multiple of
  // 32, so that with more than one chunk none is small enough for the
  // small-batch kernel, which writes the counts instead of adding to them.
  const uint64_t nch = (n + (1ULL << 22) - 1) >> 22;
  const uint64_t CH = nch ? (((n + nch - 1) / nch + 31) & ~31ULL) : 32;
  const int64_t* whole_args = nullptr;
  if (!packed && b->args_len) {
    // no contiguity promise: copy the whole pool once into pipeline 1's buffer
    size_t need = b->args_len * 8;
    if (c->stage_bytes[1] < need) {
      if (c->stage[1]) cudaFree(c->stage[1]);
      c->stage[1] = nullptr;
      c->stage_bytes[1] = 0;
      if (cudaMalloc(&c->stage[1], need) != cudaSuccess) return fail(c, PICKER_ENOMEM, "staging");
      c->stage_bytes[1] = need;
    }
    e = cudaMemcpyAsync(c->stage[1], b->args, need, cudaMemcpyHostToDevice, s[0]);
    if (e != cudaSuccess) return cuda_fail(c, e, "H2D args");
    whole_args = (const int64_t*)c->stage[1];
    s[1] = s[0];  // single pipeline
  }
  for (uint64_t c0 = 0, k = 0; c0 < n; c0 += CH, ++k) {
    const uint64_t m = std::min(CH, n - c0);
    const int p = packed ? (int)(k & 1) : 0;
    cudaStream_t ss = s[p];
    uint64_t lo = 0, hi = b->args_len;
    if (packed && b->args_len) {
      lo = std::min<uint64_t>(b->rec[c0].arg_off, b->args_len);
      const picker_rec_t& last = b->rec[c0 + m - 1];
      hi = std::min<uint64_t>(b->args_len, last.arg_off + last.nargs);
      if (hi < lo) hi = lo;
    }
    const size_t rec_b = m * sizeof(picker_rec_t);
    const size_t arg_b = packed ? (hi - lo) * 8 : 0;
    const size_t flag_b = (m + 255) & ~(size_t)255, bits_b = ((m + 31) / 32) * 4;
    const size_t need = rec_b + ((arg_b + 255) & ~(size_t)255) + flag_b + bits_b + 256;
    if (c->stage_bytes[p] < need || (!packed && p == 0 && c->stage[0] == nullptr)) {
      cudaStreamSynchronize(ss);
      if (c->stage[p]) cudaFree(c->stage[p]);
      c->stage[p] = nullptr;
      c->stage_bytes[p] = 0;
      size_t want = std::max(need, (size_t)(CH * 100));
      if (cudaMalloc(&c->stage[p], want) != cudaSuccess) return fail(c, PICKER_ENOMEM, "staging");
      c->stage_bytes[p] = want;
    }
    uint8_t* base = (uint8_t*)c->stage[p];
    picker_rec_t* d_rec = (picker_rec_t*)base;
    int64_t* d_args = (int64_t*)(base + rec_b);
    uint8_t* d_flags = base + rec_b + ((arg_b + 255) & ~(size_t)255);
    uint32_t* d_bits = (uint32_t*)(d_flags + flag_b);
    e = cudaMemcpyAsync(d_rec, b->rec + c0, rec_b, cudaMemcpyHostToDevice, ss);
    if (e == cudaSuccess && arg_b)
      e = cudaMemcpyAsync(d_args, b->args + lo, arg_b, cudaMemcpyHostToDevice, ss);
    if (e != cudaSuccess) return cuda_fail(c, e, "H2D");
    DevBatch db = packed ? DevBatch{d_rec, d_args - lo, lo, hi}
                         : DevBatch{d_rec, whole_args, 0, b->args_len};
    int launches = 0;
    Options o = c->opt;
    if (o.bucket < 0) o.bucket = c->bucket_auto;
    e = launch_validate(c->P, c->jit, o, db, m, d_flags, bits ? d_bits : nullptr,
                        c->dev_counts, c->num_sms, ss, &launches);
    if (e != cudaSuccess) return cuda_fail(c, e, "validate launch");
    c->last_launches += launches;
    e = cudaMemcpyAsync(flags + c0, d_flags, m, cudaMemcpyDeviceToHost, ss);
    if (e == cudaSuccess && bits)
      e = cudaMemcpyAsync(bits + c0 / 32, d_bits, ((m + 31) / 32) * 4, cudaMemcpyDeviceToHost, ss);
    if (e != cudaSuccess) return cuda_fail(c, e, "D2H");
  }
  if (s[1] != s[0]) {
    cudaEvent_t ev;
    cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    cudaEventRecord(ev, s[1]);
    cudaStreamWaitEvent(s[0], ev, 0);
    cudaEventDestroy(ev);
  }
  if (counts) {
    e = cudaMemcpyAsync(counts, c->dev_counts, PICKER_NUM_COUNTS * 8, cudaMemcpyDeviceToHost, s[0]);
    if (e != cudaSuccess) return cuda_fail(c, e, "D2H counts");
  }
  e = cudaStreamSynchronize(s[0]);
  if (e != cudaSuccess) return cuda_fail(c, e, "stream sync");
  return PICKER_OK;
}

int picker_validate_sequence(picker_ctx_t* c, const picker_batch_t* b, uint64_t n, uint32_t window,
                             uint32_t mode, uint8_t* out, void* stream) {
  int st = check_batch(c, b, n, out);
  if (st) return st;
  if (window < 1 || window > 1024 || mode > 1) return fail(c, PICKER_EINVAL, "window must be 1..1024, mode 0/1");
  uint32_t max_desc = 1;
  for (auto& k : c->ir) max_desc = std::max<uint32_t>(max_desc, (uint32_t)k.desc.size());
  if ((uint64_t)window * max_desc > (1u << 24))
    return fail(c, PICKER_EINVAL, "window x descriptors per kernel exceeds 2^24 extents");
  DevGuard g(c->device);
  DevBatch db{b->rec, b->args, 0, b->args_len};
  std::string err;
  cudaStream_t s = (cudaStream_t)stream;
  // Reuse K1's extents: a specialised module built with
  // PICKER_EXTENTS writes each record's verdict and active extents, the window
  // kernel reads them instead of evaluating the tables per record.  Specialised
  // kernels only (no table-path or wide kernel), n > 1024, arena <= 8 GB.
  bool k1 = c->jit && c->opt.seq_k1 && !c->opt.stride && n > kSmallMax && max_desc <= 2047;
  for (auto& k : c->ir) k1 &= k.path != PATH_WIDE && k.path != PATH_GENERIC;
  const size_t slot_b = (size_t)max_desc * 16, need = (size_t)n * (slot_b + 5) + 512;
  k1 &= need <= (8ull << 30);
  // Windows of <= 32 launches from K1's codes (PICKER_SEQ): by Q23 a window
  // with a decisive record is decided by its first one, whatever the
  // addresses, so the extents are evaluated (from the tables, in the same
  // kernel) only for the windows without one.  Calibrated on the first call:
  // kept when at most 1/16 of its windows needed extents, else the extents
  // module below (the same codes either way).  Measured on C2 x686, windows
  // of 32, 20 % of them without a decisive record: lazy 2.25 ms, extents
  // 1.10 ms (the table evaluation of an undecided window's 32 records sits
  // between two tile barriers); K1 alone is 0.25 ms.
  const int lazy = c->opt.seq_lazy >= 0 ? c->opt.seq_lazy : c->seq_lazy_state;
  if (k1 && lazy != 0 && window <= 32) {
    if (!c->jit_seq) {
      Options mo = c->opt;
      mo.seq_windows = true;
      mo.sorted = 0;  // windows are decided in the pipelined kernel
      c->jit_seq = jit_build(c->ir, mo, err);
      if (!c->jit_seq) return fail(c, PICKER_ECUDA, "JIT (sequence): " + err);
    }
    const uint64_t slice = 64ull * max_desc, need_s = jit_pipe_warps(c->jit_seq, n, c->num_sms) * slice * 8;
    if (jit_seq_lazy(c->jit_seq, n, window) && need_s <= (1ull << 30)) {  // slot slices <= 1 GB
      if (c->seq_scratch_bytes < need_s) {
        cudaError_t e = cudaStreamSynchronize(s);  // a previous call may still use the old slices
        if (c->seq_scratch) cudaFree(c->seq_scratch);
        c->seq_scratch = nullptr;
        c->seq_scratch_bytes = 0;
        if (e != cudaSuccess || cudaMalloc(&c->seq_scratch, need_s) != cudaSuccess) {
          c->seq_scratch = nullptr;
          return fail(c, PICKER_ENOMEM, "cudaMalloc(window slots) failed");
        }
        c->seq_scratch_bytes = need_s;
      }
      const bool calibrate = lazy < 0;
      if (calibrate && !c->seq_undecided && cudaMalloc(&c->seq_undecided, 4) != cudaSuccess) {
        c->seq_undecided = nullptr;
        return fail(c, PICKER_ENOMEM, "cudaMalloc(window count) failed");
      }
      BucketParams P = c->P;
      P.xcap = max_desc;
      P.seq_out = out, P.seq_window = window, P.seq_mode = mode;
      P.seq_scratch = (int64_t*)c->seq_scratch;
      P.seq_undecided = calibrate ? c->seq_undecided : nullptr;
      cudaError_t e = calibrate ? cudaMemsetAsync(c->seq_undecided, 0, 4, s) : cudaSuccess;
      if (e == cudaSuccess) e = launch_jit(c->jit_seq, P, db, n, nullptr, nullptr, nullptr, c->num_sms, s);
      if (e == cudaSuccess && calibrate) {
        uint32_t und = 0;
        e = cudaMemcpyAsync(&und, c->seq_undecided, 4, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        const uint64_t nwin = (n + window - 1) / window;
        if (e == cudaSuccess) c->seq_lazy_state = (uint64_t)und * 16 <= nwin ? 1 : 0;
      }
      if (e != cudaSuccess) return cuda_fail(c, e, "sequence (K1 codes)");
      c->last_launches = 1;
      return PICKER_OK;
    }
  }
  if (k1 && !c->jit_extents) {
    Options mo = c->opt;
    mo.extents = true;
    mo.sorted = 0;  // the extents are written by the pipelined kernel
    // windows decided inside the kernel from the tile's extents in shared
    // memory: the first geometry whose shared memory (with 4 KB of static
    // state) fits its CTAs per SM; none: extents through the global arena
    static const int geo[][4] = {{448, 448, 2, 1}, {896, 896, 1, 1}, {224, 224, 4, 1},
                                 {128, 128, 4, 1}};
    auto fits = [&](int tile, int apr, int bufs, int ctas) {
      const size_t sm = pipe_smem_bytes_for((uint32_t)tile, (uint32_t)apr, (uint32_t)bufs, false, max_desc) + 4096;
      return (sm + 1024) * ctas <= 228 * 1024;
    };
    if (mo.tile == 0) {
      for (auto& g : geo)
        if (fits(g[0], 5, g[3], g[2])) {
          mo.tile = g[0], mo.threads = g[1], mo.ctas = g[2], mo.args_per_rec = 5, mo.arg_bufs = g[3];
          mo.seq_xcap = (int)max_desc;
          break;
        }
    } else if (fits(mo.tile, mo.args_per_rec, mo.arg_bufs, 1)) {  // a given geometry (CTAs per SM: what fits)
      mo.seq_xcap = (int)max_desc;
    }
    c->jit_extents = jit_build(c->ir, mo, err);
    if (!c->jit_extents) return fail(c, PICKER_ECUDA, "JIT (extents): " + err);
  }
  if (k1 && jit_seq_fused(c->jit_extents, n, window)) {
    // one launch: verdicts, extents and windows, nothing but the window codes
    // written to global memory
    BucketParams P = c->P;
    P.xarena = nullptr, P.xinfo = nullptr, P.xcap = max_desc;
    P.seq_out = out, P.seq_window = window, P.seq_mode = mode;
    cudaError_t e = launch_jit(c->jit_extents, P, db, n, nullptr, nullptr, nullptr, c->num_sms, s);
    if (e != cudaSuccess) return cuda_fail(c, e, "sequence (K1 fused)");
    c->last_launches = 1;
    return PICKER_OK;
  }
  if (k1 && jit_extents_ok(c->jit_extents, n)) {
    if (c->seq_arena_bytes < need) {
      cudaError_t e = cudaStreamSynchronize(s);  // a previous call may still use the old arena
      if (c->seq_arena) cudaFree(c->seq_arena);
      c->seq_arena = nullptr;
      c->seq_arena_bytes = 0;
      if (e != cudaSuccess || cudaMalloc(&c->seq_arena, need) != cudaSuccess) {
        c->seq_arena = nullptr;
        return fail(c, PICKER_ENOMEM, "cudaMalloc(extent arena) failed");
      }
      c->seq_arena_bytes = need;
    }
    uint8_t* base = (uint8_t*)c->seq_arena;
    int64_t* xarena = (int64_t*)base;
    uint32_t* xinfo = (uint32_t*)(base + (size_t)n * slot_b);
    uint8_t* codes = (uint8_t*)(xinfo + n);
    BucketParams P = c->P;
    P.xarena = xarena, P.xinfo = xinfo, P.xcap = max_desc;
    cudaError_t e = launch_jit(c->jit_extents, P, db, n, codes, nullptr, nullptr, c->num_sms, s);
    if (e == cudaSuccess)
      e = launch_sequence(c->P.T, db, n, window, mode, max_desc, out, &c->seq_scratch, &c->seq_scratch_bytes,
                          c->num_sms, s, err, codes, xinfo, xarena, max_desc);
    if (e != cudaSuccess) return cuda_fail(c, e, ("sequence (K1 extents): " + err).c_str());
    c->last_launches = 2;
    return PICKER_OK;
  }
  cudaError_t e = launch_sequence(c->P.T, db, n, window, mode, max_desc, out, &c->seq_scratch, &c->seq_scratch_bytes,
                                  c->num_sms, s, err);
  if (e != cudaSuccess) return cuda_fail(c, e, ("sequence: " + err).c_str());
  c->last_launches = n ? 1 : 0;
  return PICKER_OK;
}

int picker_consumer_models(picker_ctx_t* c, const picker_batch_t* b, uint64_t n, const uint8_t* codes,
                           const uint64_t* ctx_bytes, const picker_model_params_t* prm, picker_model_out_t* out,
                           void* stream) {
  int st = check_batch(c, b, n, codes);
  if (st) return st;
  if (!prm || !out || prm->save_bytes_per_us == 0)
    return fail(c, PICKER_EINVAL, "params/out must be non-null and save_bytes_per_us > 0");
  DevGuard g(c->device);
  DevBatch db{b->rec, b->args, 0, b->args_len};
  cudaStream_t s = (cudaStream_t)stream;
  // The models module's pipelined kernel on the caller's verdicts: its shapes
  // sum each record's read-extent union (the input bytes do not depend on the
  // verdict), the emit adds the models with codes[i]; its own verdicts are not
  // written.  Same eligibility as picker_validate_models' fused pass.
  bool fused = c->jit && !c->opt.stride && n > kSmallMax;
  for (auto& k : c->ir) fused &= k.path != PATH_WIDE && k.path != PATH_GENERIC;
  if (fused && !c->jit_models) {
    Options mo = c->opt;
    mo.models = true;
    mo.sorted = 0;
    std::string err;
    c->jit_models = jit_build(c->ir, mo, err);
    if (!c->jit_models) return fail(c, PICKER_ECUDA, "JIT (models): " + err);
  }
  if (fused && jit_fused_models(c->jit_models, n)) {
    BucketParams P = c->P;
    P.ctx_bytes = ctx_bytes;
    P.given_codes = codes;
    P.kill_ns = prm->kill_ns;
    P.save_bpu = ModelDiv::of(prm->save_bytes_per_us);
    cudaError_t e = model_acc_begin(&c->model_acc, s);
    P.model_acc = (ModelAcc*)c->model_acc;
    if (e == cudaSuccess) e = launch_jit(c->jit_models, P, db, n, nullptr, nullptr, nullptr, c->num_sms, s);
    if (e == cudaSuccess) e = model_acc_end(c->model_acc, n, out, s);
    if (e != cudaSuccess) return cuda_fail(c, e, "consumer models (fused)");
    c->last_launches = 1;
    return PICKER_OK;
  }
  cudaError_t e = launch_models(c->P.T, db, n, codes, ctx_bytes, prm->kill_ns, prm->save_bytes_per_us, out,
                                &c->model_acc, c->num_sms, s);
  if (e != cudaSuccess) return cuda_fail(c, e, "consumer models");
  c->last_launches = n ? 1 : 0;
  return PICKER_OK;
}

int picker_validate_models(picker_ctx_t* c, const picker_batch_t* b, uint64_t n, uint8_t* flags, uint32_t* bits,
                           uint64_t* counts, const uint64_t* ctx_bytes, const picker_model_params_t* prm,
                           picker_model_out_t* out, void* stream) {
  int st = check_batch(c, b, n, flags);
  if (st) return st;
  if (!prm || !out || prm->save_bytes_per_us == 0)
    return fail(c, PICKER_EINVAL, "params/out must be non-null and save_bytes_per_us > 0");
  DevGuard g(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  // the fused pass: specialised kernels only (no wide kernel: its warp
  // scratch is sized for the main module's geometry), no stride mode
  bool fused = c->jit && !c->opt.stride && n > kSmallMax;
  for (auto& k : c->ir) fused &= k.path != PATH_WIDE && k.path != PATH_GENERIC;
  if (fused && !c->jit_models) {
    Options mo = c->opt;
    mo.models = true;
    mo.sorted = 0;  // the model code is in the pipelined kernel
    std::string err;
    c->jit_models = jit_build(c->ir, mo, err);
    if (!c->jit_models) return fail(c, PICKER_ECUDA, "JIT (models): " + err);
  }
  if (fused && jit_fused_models(c->jit_models, n)) {
    BucketParams P = c->P;
    st = count_slot(c, counts, n, s, P);
    if (st) return st;
    P.ctx_bytes = ctx_bytes;
    P.kill_ns = prm->kill_ns;
    P.save_bpu = ModelDiv::of(prm->save_bytes_per_us);
    cudaError_t e = model_acc_begin(&c->model_acc, s);
    P.model_acc = (ModelAcc*)c->model_acc;
    DevBatch db{b->rec, b->args, 0, b->args_len};
    if (e == cudaSuccess)
      e = launch_jit(c->jit_models, P, db, n, flags, bits, (unsigned long long*)counts, c->num_sms, s);
    if (e == cudaSuccess) e = model_acc_end(c->model_acc, n, out, s);
    if (e != cudaSuccess) return cuda_fail(c, e, "validate + models");
    c->last_launches = 1;
    return PICKER_OK;
  }
  // two passes: the verdicts, then the models on them
  st = picker_validate_batch(c, b, n, flags, bits, counts, stream);
  if (st) return st;
  const int launches = c->last_launches;
  st = picker_consumer_models(c, b, n, flags, ctx_bytes, prm, out, stream);
  c->last_launches += launches;
  return st;
}

int picker_replicate(picker_ctx_t* c, const picker_batch_t* b, uint64_t n, const uint8_t* ptr_mask,
                     uint64_t copies, uint64_t first_copy, int64_t delta, picker_rec_t* rec_out, int64_t* args_out,
                     void* stream) {
  if (!c || !b || (n && (!b->rec || !rec_out)) || (b->args_len && copies && (!b->args || !ptr_mask || !args_out)))
    return fail(c, PICKER_EINVAL, "replicate: null pointer");
  if (((uintptr_t)b->rec | (uintptr_t)rec_out) & 15) return fail(c, PICKER_EINVAL, "replicate: records not 16-B aligned");
  if (copies && n > (1ULL << 40) / copies) return fail(c, PICKER_EINVAL, "replicate: more than 2^40 records");
  DevGuard g(c->device);
  cudaError_t e = launch_replicate(b->rec, n, b->args, b->args_len, ptr_mask, copies, first_copy, delta, rec_out,
                                   args_out, c->num_sms, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(c, e, "replicate");
  c->last_launches = n && copies ? (b->args_len ? 2 : 1) : 0;
  return PICKER_OK;
}

int picker_exact_check(picker_ctx_t* c, const picker_batch_t* b, uint64_t n, uint8_t* out,
                       uint64_t* counts, uint64_t max_points, void* stream) {
  int st = check_batch(c, b, n, out);
  if (st) return st;
  if (n >= (1ULL << 32)) return fail(c, PICKER_EINVAL, "exact check: n must be < 2^32");
  if (max_points > (1ULL << 40) / ((c->max_width + 63) / 64 + 1))
    return fail(c, PICKER_EINVAL, "exact check: max_points too large for the byte-set tables");
  DevGuard g(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (counts) {
    cudaError_t e = cudaMemsetAsync(counts, 0, PICKER_NUM_COUNTS * sizeof(uint64_t), s);
    if (e != cudaSuccess) return cuda_fail(c, e, "cudaMemsetAsync(counts)");
  }
  DevBatch db{b->rec, b->args, 0, b->args_len};
  std::string err;
  cudaError_t e = launch_exact(c->P.T, db, n, out, (unsigned long long*)counts, max_points, c->max_width,
                               &c->exact_arena, &c->exact_arena_bytes, c->num_sms, s, &c->last_launches, err);
  if (e != cudaSuccess) return cuda_fail(c, e, ("exact check: " + err).c_str());
  return PICKER_OK;
}

}  // extern "C"
