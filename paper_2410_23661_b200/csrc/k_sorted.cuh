// K1, shape-sorted schedule: the path for summaries of many-argument kernels
// (C4: cuDNN-like kernels with 16-48 pointer arguments, ~300 bytes per record).
//
// Why a second schedule.  The tiled kernel (k_bucket.cuh) groups records by
// shape inside one tile of shared memory.  With ~300-byte records a tile holds
// a few thousand records, i.e. ~80 per shape for 32 shapes: the 16 warps of an
// SM run ~6 different straight-line shapes of ~20 KB of SASS each at the same
// time, more than the 32 KB L1.5 instruction cache (measured: 21 stalls per
// issue on `no_instruction`, profiles/r02_c4_*).  Evaluating the same records
// in shape order removes those stalls but exposes the uncoalesced per-lane
// argument loads (`lg_throttle`, 11 per issue).  This schedule fixes both:
//   S1 k_sort_keys     thread per record: grouping key of its kernel (shortcut
//                      kernels and unknown ids get their final code here), per
//                      block key counts;
//   S2 k_sort_scan     one CTA: offsets of every (key, block) in key-major order,
//                      per-key record offsets and 32-record group counts;
//   S3 k_sort_scatter  thread per record: record index into key order;
//   S4 k_validate_sorted  persistent; warps claim 32-record groups of ONE key in
//                      global key order (one atomic counter), so at any moment
//                      the whole GPU runs one or two shapes; the group's
//                      argument spans are copied into the warp's shared-memory
//                      slots with coalesced 16-byte cp.async (lanes over the 16-
//                      byte chunks of one record at a time), then each lane
//                      evaluates its record from shared memory;
//   S5 k_sort_emit     thread per 32 records: idempotent bit word and histogram
//                      from the codes.
// Extra traffic over the algorithmic bytes: the headers are read twice (S1,
// S4), plus 1 + 1 (keys) + 4 + 4 (permutation) + 1 (codes re-read) bytes per
// record: ~1.14x on C4.
#pragma once

#include "k_bucket.cuh"

namespace picker {

#ifndef PICKER_SORT_WARPS
#define PICKER_SORT_WARPS 16
#endif
#ifndef PICKER_SORT_SLOT
#define PICKER_SORT_SLOT 432  // bytes of one record's argument slot (multiple of 16)
#endif
constexpr int kSortWarps = PICKER_SORT_WARPS;
constexpr int kSortThreads = kSortWarps * 32;
constexpr uint32_t kSortSlot = PICKER_SORT_SLOT;
__device__ __forceinline__ void kb_lookup(const BucketParams& P, uint32_t kid, uint32_t& kb, uint32_t& kn) {
  kb = P.kb_unknown;
  kn = V_ERR_KERNEL;
  if (kid < P.T.nkernel_slots) {
    const uint2 v = __ldg(reinterpret_cast<const uint2*>(P.kb_of) + kid);
    kb = v.x, kn = v.y;
  }
}

__global__ void __launch_bounds__(256) k_sort_keys(const __grid_constant__ BucketParams P,
                                                   const __grid_constant__ DevBatch B, uint64_t n, SortScratch S,
                                                   uint8_t* __restrict__ flags) {
  __shared__ uint32_t cnt[kSortKeys];
  for (int t = threadIdx.x; t < (int)kSortKeys; t += blockDim.x) cnt[t] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * S.chunk, end = min(n, base + S.chunk);
  for (uint64_t i0 = base; i0 < end; i0 += blockDim.x) {
    const uint64_t i = i0 + threadIdx.x;
    uint32_t key = kSortNoKey;
    if (i < end) {
      const picker_rec_t* rp = B.rec + i;
      uint32_t kb, kn;
      kb_lookup(P, rp->kernel_id, kb, kn);
      key = kb >> 16;
      if (key == P.direct_key || key >= kSortKeys) {  // shortcut / unknown: final now
        flags[i] = (uint8_t)direct_code(kn, rp->nargs, rp->arg_off, B.args_lo, B.args_hi);
        key = kSortNoKey;
      }
      S.keys[i] = (uint8_t)key;
    }
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    if (key != kSortNoKey && (threadIdx.x & 31) == 31 - __clz(peers)) atomicAdd(cnt + key, (uint32_t)__popc(peers));
  }
  __syncthreads();
  for (int t = threadIdx.x; t < (int)kSortKeys; t += blockDim.x) S.hist[t * S.nblk + blockIdx.x] = cnt[t];
}

// One CTA: exclusive scan of hist (key-major), then the per-key tables.  Warp
// w scans keys w and w + 32 over the blocks (coalesced 32-wide chunks with a
// carried sum); one warp scans the 64 key totals; the warps add the offsets.
__global__ void __launch_bounds__(kSortScanThreads) k_sort_scan(SortScratch S) {
  __shared__ uint32_t s_tot[kSortKeys], s_base[kSortKeys];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t k = warp; k < kSortKeys; k += kSortScanThreads / 32) {
    uint32_t* h = S.hist + (size_t)k * S.nblk;
    uint32_t carry = 0;
    for (uint32_t b0 = 0; b0 < S.nblk; b0 += 32) {
      const uint32_t b = b0 + lane;
      const uint32_t c = b < S.nblk ? h[b] : 0u;
      uint32_t v = c;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= d) v += o;
      }
      if (b < S.nblk) h[b] = carry + v - c;  // exclusive within the key
      carry += __shfl_sync(0xffffffffu, v, 31);
    }
    if (lane == 0) s_tot[k] = carry;
  }
  __syncthreads();
  if (warp == 0) {  // exclusive scan of the 64 totals (lane l: keys l and 32 + l)
    const uint32_t t0 = s_tot[lane], t1 = s_tot[lane + 32];
    const uint32_t g0 = (t0 + 31) / 32, g1 = (t1 + 31) / 32;
    uint32_t v0 = t0, v1 = t1, w0 = g0, w1 = g1;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t a = __shfl_up_sync(0xffffffffu, v0, d), b = __shfl_up_sync(0xffffffffu, v1, d);
      const uint32_t c = __shfl_up_sync(0xffffffffu, w0, d), e = __shfl_up_sync(0xffffffffu, w1, d);
      if (lane >= d) v0 += a, v1 += b, w0 += c, w1 += e;
    }
    const uint32_t T0 = __shfl_sync(0xffffffffu, v0, 31), G0 = __shfl_sync(0xffffffffu, w0, 31);
    v1 += T0, w1 += G0;
    s_base[lane] = v0 - t0, s_base[lane + 32] = v1 - t1;
    S.meta[kMetaOff + lane] = v0 - t0, S.meta[kMetaOff + lane + 32] = v1 - t1;
    S.meta[kMetaCnt + lane] = t0, S.meta[kMetaCnt + lane + 32] = t1;
    S.meta[kMetaG + lane] = w0 - g0, S.meta[kMetaG + lane + 32] = w1 - g1;
    if (lane == 31) {
      S.meta[kMetaOff + kSortKeys] = v1;
      S.meta[kMetaG + kSortKeys] = w1;
      S.meta[kMetaClaim] = 0;
    }
  }
  __syncthreads();
  for (uint32_t k = warp; k < kSortKeys; k += kSortScanThreads / 32) {
    uint32_t* h = S.hist + (size_t)k * S.nblk;
    for (uint32_t b = lane; b < S.nblk; b += 32) h[b] += s_base[k];
  }
}

__global__ void __launch_bounds__(256) k_sort_scatter(uint64_t n, SortScratch S) {
  __shared__ uint32_t cur[kSortKeys];
  for (int t = threadIdx.x; t < (int)kSortKeys; t += blockDim.x) cur[t] = S.hist[t * S.nblk + blockIdx.x];
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * S.chunk, end = min(n, base + S.chunk);
  const int lane = threadIdx.x & 31;
  for (uint64_t i0 = base; i0 < end; i0 += blockDim.x) {
    const uint64_t i = i0 + threadIdx.x;
    const uint32_t key = i < end ? S.keys[i] : kSortNoKey;
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    const int leader = 31 - __clz(peers);
    uint32_t b = 0;
    if (key != kSortNoKey && lane == leader) b = atomicAdd(cur + key, (uint32_t)__popc(peers));
    b = __shfl_sync(0xffffffffu, b, leader);
    if (key != kSortNoKey) S.perm[b + __popc(peers & ((1u << lane) - 1u))] = (uint32_t)i;
  }
}

template <class Dispatch>
__global__ void __launch_bounds__(kSortThreads, 1)
    k_validate_sorted(const __grid_constant__ BucketParams P, const __grid_constant__ DevBatch B, SortScratch S,
                      uint8_t* __restrict__ flags) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint32_t s_off[kSortKeys + 1], s_cnt[kSortKeys], s_g[kSortKeys + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int t = tid; t < (int)kMetaClaim; t += kSortThreads) {
    const uint32_t v = S.meta[t];
    if (t < (int)kMetaCnt) s_off[t] = v;
    else if (t < (int)kMetaG) s_cnt[t - kMetaCnt] = v;
    else s_g[t - kMetaG] = v;
  }
  __syncthreads();
  const uint32_t ngroups = s_g[kSortKeys];
  unsigned char* slots = smem + (size_t)warp * 32 * kSortSlot;
  __shared__ __align__(8) uint64_t s_bar[kSortWarps];
  uint64_t* bar = s_bar + warp;
  uint32_t phase = 0;
  if (lane == 0) {
    mbar_init(bar, 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const uintptr_t p0 = (uintptr_t)(B.args + B.args_lo), p1 = (uintptr_t)(B.args + B.args_hi);
  for (;;) {
    uint32_t g = 0;
    if (lane == 0) g = atomicAdd(S.meta + kMetaClaim, 1u);
    g = __shfl_sync(0xffffffffu, g, 0);
    if (g >= ngroups) break;
    // key of group g: the last k with s_g[k] <= g (s_g is non-decreasing)
    uint32_t k = 0;
#pragma unroll
    for (uint32_t step = kSortKeys / 2; step > 0; step >>= 1)
      if (s_g[k + step] <= g) k += step;
    const uint32_t j = g - s_g[k];
    const uint32_t start = s_off[k] + 32u * j, rem = min(32u, s_cnt[k] - 32u * j);
    if (kWidePath && k == P.wide_key) {  // K2: the whole warp on one record at a time
      for (uint32_t q = 0; q < rem; ++q) {
        const uint32_t wi = S.perm[start + q];
        const picker_rec_t r = load_rec(B.rec + wi);
        const uint8_t c = eval_wide_warp(P.T, r, B.args + r.arg_off, B.args_lo, B.args_hi, lane,
                                         wide_scratch(P, warp));
        if (lane == 0) flags[wi] = c;
      }
      continue;
    }
    const bool valid = (uint32_t)lane < rem;
    uint32_t i = 0, kb = 0, kn = 0;
    picker_rec_t r{};
    uint64_t s0 = 0;
    uint32_t nch = 0, shift = 0;
    if (valid) {
      i = S.perm[start + lane];
      r = load_rec(B.rec + i);
      kb_lookup(P, r.kernel_id, kb, kn);
      // stage the argument span when the record is well-formed and it fits
      const uintptr_t a0 = (uintptr_t)(B.args + r.arg_off), a1 = a0 + 8ull * r.nargs;
      const uintptr_t c0 = a0 & ~(uintptr_t)15, c1 = (a1 + 15) & ~(uintptr_t)15;
      const bool in_pool = r.arg_off >= B.args_lo && r.arg_off <= B.args_hi &&
                           (uint64_t)r.nargs <= B.args_hi - r.arg_off;
      if (r.nargs == (kn >> 24) && in_pool && c0 >= p0 && c1 <= p1 && c1 - c0 <= kSortSlot) {
        s0 = c0;
        nch = (uint32_t)((c1 - c0) >> 4);
        shift = (uint32_t)(a0 - c0);
      }
    }
    // each lane stages its record's span with one TMA bulk copy into its slot;
    // the warp's mbarrier completes when all 32 lanes arrived and the bytes landed
    const uint32_t bytes = nch * 16u;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    if (bytes) tma_load_1d(slots + lane * kSortSlot, (const void*)s0, bytes, bar);
    mbar_wait(bar, phase);
    phase ^= 1u;
    if (valid) {
      const bool local = nch != 0;
      const int64_t* a = local ? reinterpret_cast<const int64_t*>(slots + lane * kSortSlot + shift)
                               : B.args + r.arg_off;
      flags[i] = Dispatch::eval(k, kb & 0xFFFFu, kn, local, P, r, a, B);
    }
    __syncwarp();  // the slots are reused by the warp's next group (the next copy is async-proxy)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
}

// S5: one thread per 32 records: the idempotent bit word and the histogram.
__global__ void __launch_bounds__(256) k_sort_emit(const uint8_t* __restrict__ flags, uint64_t n,
                                                   uint32_t* __restrict__ bits, unsigned long long* __restrict__ counts) {
  __shared__ uint32_t s_hist[PICKER_NUM_COUNTS];
  if (threadIdx.x < PICKER_NUM_COUNTS) s_hist[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t nw = (n + 31) / 32;
  for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b0 = 32 * w;
    const int m = (int)min((uint64_t)32, n - b0);
    uint32_t word = 0;
    uint32_t h[PICKER_NUM_COUNTS];
#pragma unroll
    for (int c = 0; c < PICKER_NUM_COUNTS; ++c) h[c] = 0;
    for (int q = 0; q < m; ++q) {
      const uint32_t c = flags[b0 + q];
      word |= (uint32_t)(c <= V_IDEM_KERNEL) << q;
      const int hb = count_bin((uint8_t)c);
#pragma unroll
      for (int x = 0; x < PICKER_NUM_COUNTS; ++x) h[x] += hb == x;
    }
    if (bits) bits[w] = word;
#pragma unroll
    for (int x = 0; x < PICKER_NUM_COUNTS; ++x)
      if (h[x]) atomicAdd(s_hist + x, h[x]);
  }
  __syncthreads();
  if (counts && threadIdx.x < PICKER_NUM_COUNTS && s_hist[threadIdx.x])
    atomicAdd(counts + threadIdx.x, (unsigned long long)s_hist[threadIdx.x]);
}

}  // namespace picker
