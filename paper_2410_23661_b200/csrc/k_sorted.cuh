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
//                      kernels and unknown ids get their final code here); per
//                      block key counts, whose offsets within each key come
//                      from atomic adds on the key totals (no scan pass);
//   S3 k_sort_scatter  thread per record: record index into key order (key
//                      bases from an in-CTA scan of the 64 totals);
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
#ifndef PICKER_SORT_STAGES
#define PICKER_SORT_STAGES 13
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

__global__ void __launch_bounds__(kSortBlock) k_sort_keys(const __grid_constant__ BucketParams P,
                                                   const __grid_constant__ DevBatch B, uint64_t n, SortScratch S,
                                                   uint8_t* __restrict__ flags) {
  __shared__ uint32_t cnt[kSortKeys];
  for (int t = threadIdx.x; t < (int)kSortKeys; t += blockDim.x) cnt[t] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * S.chunk, end = min(n, base + S.chunk);
  constexpr int U = 4;  // records per thread in flight (the kernel-id loads are latency-bound)
  for (uint64_t i0 = base; i0 < end; i0 += U * blockDim.x) {
    uint32_t kid[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = i0 + u * blockDim.x + threadIdx.x;
      kid[u] = __ldg(&B.rec[min(i, end - 1)].kernel_id);  // unconditional: all loads in flight
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = i0 + u * blockDim.x + threadIdx.x;
      uint32_t key = kSortNoKey;
      if (i < end) {
        uint32_t kb, kn;
        kb_lookup(P, kid[u], kb, kn);
        key = kb >> 16;
        if (key == P.direct_key || key >= kSortKeys) {  // shortcut / unknown: final now
          flags[i] = (uint8_t)direct_code(kn, __ldg(&B.rec[i].nargs), __ldg(&B.rec[i].arg_off), B.args_lo, B.args_hi);
          key = kSortNoKey;
        }
        S.keys[i] = (uint8_t)key;
      }
      const unsigned peers = __match_any_sync(0xffffffffu, key);
      if (key != kSortNoKey && (threadIdx.x & 31) == 31 - __clz(peers)) atomicAdd(cnt + key, (uint32_t)__popc(peers));
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < (int)kSortKeys; t += blockDim.x)
    S.hist[t * S.nblk + blockIdx.x] = cnt[t] ? atomicAdd(S.meta + kMetaTot + t, cnt[t]) : 0u;
}

// Per-key tables from the key totals (warp 0 of a CTA): off[k] = first sorted
// position of key k, cnt[k] = its records, gs[k] = its first 32-record group.
__device__ __forceinline__ void key_tables(const SortScratch& S, uint32_t* off, uint32_t* cnt, uint32_t* gs) {
  const int lane = threadIdx.x & 31;
  const uint32_t t0 = S.meta[kMetaTot + lane], t1 = S.meta[kMetaTot + lane + 32];
  const uint32_t g0 = (t0 + 31) / 32, g1 = (t1 + 31) / 32;
  uint32_t v0 = t0, v1 = t1, w0 = g0, w1 = g1;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t a = __shfl_up_sync(0xffffffffu, v0, d), b = __shfl_up_sync(0xffffffffu, v1, d);
    const uint32_t c = __shfl_up_sync(0xffffffffu, w0, d), e = __shfl_up_sync(0xffffffffu, w1, d);
    if (lane >= d) v0 += a, v1 += b, w0 += c, w1 += e;
  }
  v1 += __shfl_sync(0xffffffffu, v0, 31), w1 += __shfl_sync(0xffffffffu, w0, 31);
  off[lane] = v0 - t0, off[lane + 32] = v1 - t1;
  cnt[lane] = t0, cnt[lane + 32] = t1;
  gs[lane] = w0 - g0, gs[lane + 32] = w1 - g1;
  if (lane == 31) off[kSortKeys] = v1, gs[kSortKeys] = w1;
}

__global__ void __launch_bounds__(kSortBlock) k_sort_scatter(uint64_t n, SortScratch S) {
  __shared__ uint32_t cur[kSortKeys], s_off[kSortKeys + 1], s_cnt[kSortKeys], s_g[kSortKeys + 1];
  if (threadIdx.x < 32) key_tables(S, s_off, s_cnt, s_g);
  __syncthreads();
  for (int t = threadIdx.x; t < (int)kSortKeys; t += blockDim.x) cur[t] = s_off[t] + S.hist[t * S.nblk + blockIdx.x];
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * S.chunk, end = min(n, base + S.chunk);
  const int lane = threadIdx.x & 31;
  constexpr int U = 4;
  for (uint64_t i0 = base; i0 < end; i0 += U * blockDim.x) {
    uint32_t kk[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = i0 + u * blockDim.x + threadIdx.x;
      kk[u] = S.keys[min(i, end - 1)];  // unconditional: all loads in flight
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = i0 + u * blockDim.x + threadIdx.x;
      const uint32_t key = i < end ? kk[u] : kSortNoKey;
      const unsigned peers = __match_any_sync(0xffffffffu, key);
      const int leader = 31 - __clz(peers);
      uint32_t b = 0;
      if (key != kSortNoKey && lane == leader) b = atomicAdd(cur + key, (uint32_t)__popc(peers));
      b = __shfl_sync(0xffffffffu, b, leader);
      if (key != kSortNoKey) S.perm[b + __popc(peers & ((1u << lane) - 1u))] = (uint32_t)i;
    }
  }
}

template <class Dispatch>
__global__ void __launch_bounds__(kSortThreads, 1)
    k_validate_sorted(const __grid_constant__ BucketParams P, const __grid_constant__ DevBatch B, SortScratch S,
                      uint8_t* __restrict__ flags) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint32_t s_off[kSortKeys + 1], s_cnt[kSortKeys], s_g[kSortKeys + 1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 32) key_tables(S, s_off, s_cnt, s_g);
  __syncthreads();
  const uint32_t ngroups = s_g[kSortKeys];
  unsigned char* slot = smem + ((size_t)warp * 32 + lane) * kSortSlot;
  const uintptr_t p0 = (uintptr_t)(B.args + B.args_lo), p1 = (uintptr_t)(B.args + B.args_hi);
  // group g -> key, first sorted position, records
  auto group = [&](uint32_t g, uint32_t& k, uint32_t& start, uint32_t& rem) {
    k = 0;
#pragma unroll
    for (uint32_t step = kSortKeys / 2; step > 0; step >>= 1)
      if (s_g[k + step] <= g) k += step;  // the last key whose groups start at or before g
    const uint32_t j = g - s_g[k];
    start = s_off[k] + 32u * j;
    rem = min(32u, s_cnt[k] - 32u * j);
  };
  auto claim = [&]() {
    uint32_t c = 0;
    if (lane == 0) c = atomicAdd(S.meta + kMetaClaim, 1u);
    return c;  // lane 0's value; broadcast where it is consumed
  };
  // software pipeline over a warp's groups: the claim of group g+1 and its
  // permutation entries are loaded while group g is evaluated, and its headers
  // are prefetched into L2 at the end of g, so the claim / permutation / header
  // round trips are off the critical path
  uint32_t g = __shfl_sync(0xffffffffu, claim(), 0);
  uint32_t k = 0, start = 0, rem = 0, pi = 0;
  if (g < ngroups) {
    group(g, k, start, rem);
    pi = (uint32_t)lane < rem ? S.perm[start + lane] : 0u;
  }
  uint32_t gn_lane0 = claim();
  while (g < ngroups) {
    const uint32_t gn = __shfl_sync(0xffffffffu, gn_lane0, 0);
    uint32_t kn_ = 0, startn = 0, remn = 0, pin = 0;
    if (gn < ngroups) {
      group(gn, kn_, startn, remn);
      pin = (uint32_t)lane < remn ? S.perm[startn + lane] : 0u;  // consumed next iteration
    }
    gn_lane0 = claim();
    if (kWidePath && k == P.wide_key) {  // K2: the whole warp on one record at a time
      for (uint32_t q = 0; q < rem; ++q) {
        const uint32_t wi = __shfl_sync(0xffffffffu, pi, q);
        const picker_rec_t r = load_rec(B.rec + wi);
        // the warp's argument slots (unused by K2) hold its sort scratch
        const bool in_smem = P.T.kernels[r.kernel_id < P.T.nkernel_slots ? r.kernel_id : 0].ndesc <= kSortSlot;
        const uint8_t c = eval_wide_warp(P.T, r, B.args + r.arg_off, B.args_lo, B.args_hi, lane,
                                         in_smem ? reinterpret_cast<WideElem*>(smem + (size_t)warp * 32 * kSortSlot)
                                                 : wide_scratch(P, warp),
                                         in_smem ? kSortSlot : (uint32_t)kWideMax);
        if (lane == 0) flags[wi] = c;
      }
    } else if ((uint32_t)lane < rem) {
      const uint32_t i = pi;
      const picker_rec_t r = load_rec(B.rec + i);
      uint32_t kb, kn;
      kb_lookup(P, r.kernel_id, kb, kn);
      // stage the record's argument span (16-byte chunks, cp.async per lane:
      // a bulk copy per lane is serialised by the uniform datapath) when the
      // record is well-formed and the span fits the slot
      const uintptr_t a0 = (uintptr_t)(B.args + r.arg_off), a1 = a0 + 8ull * r.nargs;
      const uintptr_t c0 = a0 & ~(uintptr_t)15, c1 = (a1 + 15) & ~(uintptr_t)15;
      const bool in_pool = r.arg_off >= B.args_lo && r.arg_off <= B.args_hi &&
                           (uint64_t)r.nargs <= B.args_hi - r.arg_off;
      const bool local = r.nargs == (kn >> 24) && in_pool && c0 >= p0 && c1 <= p1 && c1 - c0 <= kSortSlot;
      if (local) {
        for (uintptr_t c = c0; c < c1; c += 16)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(slot + (c - c0))), "l"(c)
                       : "memory");
        asm volatile("cp.async.commit_group;\ncp.async.wait_all;" ::: "memory");
      }
      const int64_t* a = local ? reinterpret_cast<const int64_t*>(slot + (a0 - c0)) : B.args + r.arg_off;
      flags[i] = Dispatch::eval(k, kb & 0xFFFFu, kn, local, P, r, a, B);
    }
    // the next group's headers into L2 while this warp finishes
    if ((uint32_t)lane < remn) asm volatile("prefetch.global.L2 [%0];" ::"l"(B.rec + pin) : "memory");
    g = gn, k = kn_, start = startn, rem = remn, pi = pin;
  }
}

// S4, warp-specialised (PICKER_SORT_WS): warp 0 of each CTA is a producer
// that claims the CTA's groups in order and stages each one -- permutation
// entries, headers and 16-byte-rounded argument spans, all with cp.async --
// into the next stage of a ring in shared memory, completing the stage's
// `full` mbarrier (32 cp.async-tracked arrivals + one arrival that publishes
// the stage's metadata); the other warps are consumers that take stages in
// ring order, evaluate their 32 records from shared memory and release the
// stage (`empty`).  The producer runs up to kSortStages groups ahead, so the
// consumers never wait on a memory round trip of their own; after the last
// group it publishes one DONE stage per consumer.
constexpr uint32_t kSortStages = PICKER_SORT_STAGES;
constexpr uint32_t kStageBytes = 32 * 32 + 32 * kSortSlot;  // headers, argument slots
constexpr uint32_t kGroupDone = 0xFFFFFFFFu;

template <class Dispatch>
__global__ void __launch_bounds__(kSortThreads, 1)
    k_validate_sorted_ws(const __grid_constant__ BucketParams P, const __grid_constant__ DevBatch B, SortScratch S,
                         uint8_t* __restrict__ flags) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint32_t s_off[kSortKeys + 1], s_cnt[kSortKeys], s_g[kSortKeys + 1];
  __shared__ __align__(8) uint64_t s_full[kSortStages], s_empty[kSortStages];
  __shared__ uint32_t s_meta_g[kSortStages];
  __shared__ uint32_t s_meta_i[kSortStages][32];  // record index | local << 31 | shift (8 B) << 28
  __shared__ uint32_t s_take;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 32) key_tables(S, s_off, s_cnt, s_g);
  if (tid == 0) {
    for (uint32_t b = 0; b < kSortStages; ++b) mbar_init(&s_full[b], 33), mbar_init(&s_empty[b], 1);
    s_take = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t ngroups = s_g[kSortKeys];
  auto group = [&](uint32_t g, uint32_t& k, uint32_t& start, uint32_t& rem) {
    k = 0;
#pragma unroll
    for (uint32_t step = kSortKeys / 2; step > 0; step >>= 1)
      if (s_g[k + step] <= g) k += step;
    const uint32_t j = g - s_g[k];
    start = s_off[k] + 32u * j;
    rem = min(32u, s_cnt[k] - 32u * j);
  };
  constexpr uint32_t kConsumers = kSortWarps - 1;
  if (warp == 0) {
    // ---- producer ----
    const uintptr_t p0 = (uintptr_t)(B.args + B.args_lo), p1 = (uintptr_t)(B.args + B.args_hi);
    // the CTA's groups: blockIdx.x + j * gridDim.x (static: increasing, so the
    // DONE stages come last; every CTA walks the shapes in the same order).
    // Lookahead: the permutation entry of j+2 and the header of j+1 are loaded
    // during j, so no load of the producer waits for its own result.
    const uint32_t G = gridDim.x;
    uint32_t g = blockIdx.x;
    uint32_t k = 0, start = 0, rem = 0, pi = 0;
    uint32_t k1 = 0, start1 = 0, rem1 = 0, pi1 = 0;
    picker_rec_t r{};
    if (g < ngroups) {
      group(g, k, start, rem);
      pi = (uint32_t)lane < rem ? S.perm[start + lane] : 0u;
    }
    if (g + G < ngroups) {
      group(g + G, k1, start1, rem1);
      pi1 = (uint32_t)lane < rem1 ? S.perm[start1 + lane] : 0u;
    }
    if (g < ngroups && (uint32_t)lane < rem) r = load_rec(B.rec + pi);
    uint32_t done = 0;
    for (uint32_t t = 0; done < kConsumers; ++t, g += G) {
      const uint32_t b = t % kSortStages, round = t / kSortStages;
      // group j+2's permutation entries, j+1's headers: in flight during j
      uint32_t k2 = 0, start2 = 0, rem2 = 0, pi2 = 0;
      if (g + 2 * G < ngroups) {
        group(g + 2 * G, k2, start2, rem2);
        pi2 = (uint32_t)lane < rem2 ? S.perm[start2 + lane] : 0u;
      }
      picker_rec_t r1{};
      if (g + G < ngroups && (uint32_t)lane < rem1) r1 = load_rec(B.rec + pi1);
      mbar_wait(&s_empty[b], (round & 1) ^ 1);  // released by its consumer of the previous round
      unsigned char* st = smem + (size_t)b * kStageBytes;
      if (g < ngroups) {
        uint32_t info = 0;
        if ((uint32_t)lane < rem) {
          // header into the stage; the argument span when well-formed and small
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n\tcp.async.cg.shared.global [%2], [%3], 16;" ::"r"(
                           smem_u32(st + 32 * lane)),
                       "l"(B.rec + pi), "r"(smem_u32(st + 32 * lane + 16)),
                       "l"(reinterpret_cast<const char*>(B.rec + pi) + 16)
                       : "memory");
          uint32_t kb, kn;
          kb_lookup(P, r.kernel_id, kb, kn);
          const uintptr_t a0 = (uintptr_t)(B.args + r.arg_off), a1 = a0 + 8ull * r.nargs;
          const uintptr_t c0 = a0 & ~(uintptr_t)15, c1 = (a1 + 15) & ~(uintptr_t)15;
          const bool in_pool = r.arg_off >= B.args_lo && r.arg_off <= B.args_hi &&
                               (uint64_t)r.nargs <= B.args_hi - r.arg_off;
          const bool local = !(kWidePath && k == P.wide_key) && r.nargs == (kn >> 24) && in_pool && c0 >= p0 &&
                             c1 <= p1 && c1 - c0 <= kSortSlot;
          if (local) {
            unsigned char* slot = st + 32 * 32 + lane * kSortSlot;
            for (uintptr_t c = c0; c < c1; c += 16)
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(slot + (c - c0))), "l"(c)
                           : "memory");
          }
          info = pi | (local ? 1u << 31 : 0u) | ((uint32_t)(a0 - c0) >> 3) << 30;  // pi < 2^30
        }
        s_meta_i[b][lane] = info;
        if (lane == 0) s_meta_g[b] = g;
      } else {
        if (lane == 0) s_meta_g[b] = kGroupDone;
        ++done;
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&s_full[b])) : "memory");
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&s_full[b])) : "memory");
      k = k1, start = start1, rem = rem1, pi = pi1, r = r1;
      k1 = k2, start1 = start2, rem1 = rem2, pi1 = pi2;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    return;
  }
  // ---- consumers ----
  for (;;) {
    uint32_t t = 0;
    if (lane == 0) t = atomicAdd(&s_take, 1u);
    t = __shfl_sync(0xffffffffu, t, 0);
    const uint32_t b = t % kSortStages, round = t / kSortStages;
    mbar_wait(&s_full[b], round & 1);
    const uint32_t g = s_meta_g[b];
    if (g == kGroupDone) return;
    uint32_t k, start, rem;
    group(g, k, start, rem);
    unsigned char* st = smem + (size_t)b * kStageBytes;
    if (kWidePath && k == P.wide_key) {  // K2: the whole warp on one record at a time, scratch = the slots
      for (uint32_t q = 0; q < rem; ++q) {
        const uint32_t wi = s_meta_i[b][q] & 0x3FFFFFFFu;
        const picker_rec_t r = rec_from_smem(st + 32 * q);
        const bool in_smem = P.T.kernels[r.kernel_id < P.T.nkernel_slots ? r.kernel_id : 0].ndesc <= kSortSlot;
        const uint8_t c = eval_wide_warp(P.T, r, B.args + r.arg_off, B.args_lo, B.args_hi, lane,
                                         in_smem ? reinterpret_cast<WideElem*>(st + 32 * 32) : wide_scratch(P, warp),
                                         in_smem ? kSortSlot : (uint32_t)kWideMax);
        if (lane == 0) flags[wi] = c;
      }
    } else if ((uint32_t)lane < rem) {
      const uint32_t info = s_meta_i[b][lane];
      const uint32_t i = info & 0x3FFFFFFFu;
      const bool local = info >> 31;
      const picker_rec_t r = rec_from_smem(st + 32 * lane);
      uint32_t kb, kn;
      kb_lookup(P, r.kernel_id, kb, kn);
      const int64_t* a = local ? reinterpret_cast<const int64_t*>(st + 32 * 32 + lane * kSortSlot +
                                                                 8 * ((info >> 30) & 1u))
                               : B.args + r.arg_off;
      flags[i] = Dispatch::eval(k, kb & 0xFFFFu, kn, local, P, r, a, B);
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&s_empty[b])) : "memory");
  }
}

// S5: one thread per 32 records: the idempotent bit word and the histogram.
__global__ void __launch_bounds__(256) k_sort_emit(const uint8_t* __restrict__ flags, uint64_t n,
                                                   uint32_t* __restrict__ bits, unsigned long long* __restrict__ counts,
                                                   CountSlot* slot, uint32_t* meta) {
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
  flush_counts(s_hist, counts, slot);
  // the last CTA clears the key totals and claim counter for the next call
  // (S1-S4 are done: they precede S5 on the stream)
  __shared__ uint32_t s_last;
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(meta + kMetaTicket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (s_last)
    for (uint32_t w = threadIdx.x; w < kMetaWords; w += blockDim.x) meta[w] = 0;
}

}  // namespace picker
