// Multi-kernel idempotency:
// "validate the idempotency of a list of sequentially executed GPU kernel
// instances with two steps.  First, Picker predicts the read and write
// addresses of each GPU kernel instance.  Second, Picker sorts the instances by
// their launch order, and then checks the clobber anti-dependency across the
// instances ... [or, for] concurrently executed GPU kernel instances, ... the
// overlap of read and write addresses among all concurrent instances."
//
// The stream is cut into consecutive windows of `window` launches (launch
// order = record order); one CTA decides one window at a time (persistent),
// reading DESIGN.md Q23 (identical to oracle.picker_oracle.oracle_sequence):
//   1. threads over the window's records: each record's decisive code (the
//      first one in launch order decides), its activity / opaque flags, and its
//      active non-opaque extents appended to the CTA's read and write lists;
//   2. the opaque rule (sequential: an opaque read of i with a write of j >= i,
//      or a read of i with an opaque write of j >= i; concurrent: any i, j);
//   3. the overlap, as sort + sweep passes over the extents.  Concurrent: one
//      pass, any read against any write.  Sequential ("a read of i and a write
//      of j with i <= j"): divide and conquer over launch order -- a pass per
//      level l of a binary split of the window checks the reads of every left
//      half against the writes of the matching right half (instance bit l = 0
//      vs 1, same higher bits), plus one pass within each instance.  Each pass
//      tags the extents with a node id, sorts the writes by (node, lb) (bitonic,
//      CTA-wide), takes the prefix maxima of ub within each node (the sweep
//      line's running maximum), and probes every read by binary search in its
//      node: some write of the node overlaps the read iff, at the last write
//      with lb <= read.ub, the running maximum ub >= read.lb (closed intervals).
// No per-record limit on descriptors; the lists live in a per-CTA slice of a
// global scratch (window x max descriptors x 48 bytes, L1/L2-resident).
#include <cuda_runtime.h>

#include <string>

#include "launch.hpp"
#include "seq.cuh"

namespace picker {

__global__ void __launch_bounds__(kSeqThreads) k_seq_windows(Tables T, DevBatch B, uint64_t n, uint32_t window,
                                                              uint32_t mode, uint8_t* __restrict__ scratch,
                                                              uint64_t slice, uint32_t cap, uint8_t* __restrict__ out,
                                                              const SeqK1 K1) {
  // per-CTA slice: reads [cap], writes [cap], sort buffer [2 cap], prefix maxima [2 cap]
  __shared__ SeqShared<1024> sh;
  const SeqCta grp{&sh, (int)threadIdx.x, (int)blockDim.x};
  SeqIv* Rl = reinterpret_cast<SeqIv*>(scratch + blockIdx.x * slice);
  SeqIv* Wl = Rl + cap;
  SeqIv* S = Wl + cap;
  int64_t* PM = reinterpret_cast<int64_t*>(S + 2 * (uint64_t)cap);
  const uint64_t nwin = (n + window - 1) / window;
  for (uint64_t w = blockIdx.x; w < nwin; w += gridDim.x) {
    const uint64_t w0 = w * window;
    const uint32_t m = (uint32_t)min((uint64_t)window, n - w0);
    const uint8_t code = seq_window(T, B, w0, m, mode, Rl, Wl, S, PM, cap, K1, grp);
    if (threadIdx.x == 0) out[w] = code;
    __syncthreads();  // the slice and the shared state are reused by the next window
  }
}

// Windows of <= 32 launches: one warp per window, 8 windows per CTA at a time
// (a CTA per window of 32 threads was capped at 32 warps per SM by the CTA
// limit); each warp has its own scratch slice and shared state.
constexpr int kSeqWarps = 8;
__global__ void __launch_bounds__(kSeqWarps * 32) k_seq_windows_w(Tables T, DevBatch B, uint64_t n, uint32_t window,
                                                                 uint32_t mode, uint8_t* __restrict__ scratch,
                                                                 uint64_t slice, uint32_t cap,
                                                                 uint8_t* __restrict__ out, const SeqK1 K1) {
  __shared__ SeqShared<32> sh[kSeqWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t gw = (uint64_t)blockIdx.x * kSeqWarps + warp, nwarps = (uint64_t)gridDim.x * kSeqWarps;
  const SeqWarp grp{&sh[warp], lane, 32};
  SeqIv* Rl = reinterpret_cast<SeqIv*>(scratch + gw * slice);
  SeqIv* Wl = Rl + cap;
  SeqIv* S = Wl + cap;
  int64_t* PM = reinterpret_cast<int64_t*>(S + 2 * (uint64_t)cap);
  const uint64_t nwin = (n + window - 1) / window;
  for (uint64_t w = gw; w < nwin; w += nwarps) {
    const uint64_t w0 = w * window;
    const uint32_t m = (uint32_t)min((uint64_t)window, n - w0);
    const uint8_t code = seq_window(T, B, w0, m, mode, Rl, Wl, S, PM, cap, K1, grp);
    if (lane == 0) out[w] = code;
    __syncwarp();  // the slice and the shared state are reused by the next window
  }
}

cudaError_t launch_sequence(const Tables& T, const DevBatch& b, uint64_t n, uint32_t window, uint32_t mode,
                            uint32_t max_desc, uint8_t* out, void** scratch_buf, size_t* scratch_bytes, int num_sms,
                            cudaStream_t s, std::string& err, const uint8_t* k1_codes, const uint32_t* k1_xinfo,
                            const int64_t* k1_xarena, uint32_t k1_xcap) {
  if (n == 0) return cudaSuccess;
  // extents per window <= window x max descriptors per kernel
  const uint32_t cap = std::max<uint32_t>(32, window * std::max<uint32_t>(max_desc, 1));
  const uint64_t slice = (uint64_t)cap * (4 * sizeof(SeqIv) + 2 * sizeof(int64_t));
  const uint64_t nwin = (n + window - 1) / window;
  // a thread per record of a window (32..512 threads per CTA), as many CTAs as
  // fill the SMs (2048 threads each), within ~1 GB of scratch
  // (windows of <= 32 launches: a warp per window, kSeqWarps windows per CTA)
  const bool per_warp = window <= 32;
  const uint32_t threads = per_warp ? kSeqWarps * 32 : std::min<uint32_t>(kSeqThreads, (window + 31) / 32 * 32);
  const uint64_t units_per_cta = per_warp ? kSeqWarps : 1;
  uint64_t grid = std::min<uint64_t>((nwin + units_per_cta - 1) / units_per_cta, (uint64_t)num_sms * (2048 / threads));
  grid = std::max<uint64_t>(1, std::min<uint64_t>(grid, (1ULL << 30) / (slice * units_per_cta)));
  const uint64_t slices = grid * units_per_cta;
  // the slices are owned by the caller's context, grown on demand (a per-call
  // stream-ordered allocation made the timing depend on the pool's state)
  if (*scratch_bytes < slices * slice) {
    cudaError_t e = cudaStreamSynchronize(s);  // a previous call may still use the old buffer
    if (e == cudaSuccess && *scratch_buf) e = cudaFree(*scratch_buf);
    *scratch_buf = nullptr;
    *scratch_bytes = 0;
    if (e == cudaSuccess) e = cudaMalloc(scratch_buf, slices * slice);
    if (e != cudaSuccess) {
      *scratch_buf = nullptr;
      err = "scratch allocation";
      return e;
    }
    *scratch_bytes = slices * slice;
  }
  const SeqK1 K1{k1_codes, k1_xinfo, k1_xarena, k1_xcap, 0};
  if (per_warp)
    k_seq_windows_w<<<(unsigned)grid, threads, 0, s>>>(T, b, n, window, mode, (uint8_t*)*scratch_buf, slice, cap,
                                                       out, K1);
  else
    k_seq_windows<<<(unsigned)grid, threads, 0, s>>>(T, b, n, window, mode, (uint8_t*)*scratch_buf, slice, cap, out,
                                                     K1);
  return cudaGetLastError();
}

}  // namespace picker
