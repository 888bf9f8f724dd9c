// K1 staged + bucketed validation kernel.
//
// Persistent CTAs (kCtasPerSm per SM) walk tiles of kTile launch records.
// Each tile's 32-byte headers and its contiguous argument span are copied
// global->shared by the TMA engine (cp.async.bulk, completion on an mbarrier);
// the headers are double-buffered a tile ahead, the arguments double-buffered
// or (kArgBufs == 1, the specialised module's default) fetched into one buffer
// while the previous tile is emitted: every input byte crosses HBM once, in
// bulk, and all per-record gathers hit shared memory.
//
// Inside a tile the records are grouped by `key` before evaluation, so that a
// warp evaluates up to 32 instances that run the SAME code:
//   - specialised module (jit.cpp): key = the kernel's shape, so kernels that
//     share generated code (e.g. every TVM dense kernel) share warps; each lane
//     reads its own kernel's constants;
//   - table-driven path: key = the kernel, so table reads are warp-uniform.
// A launch stream interleaves many kernels (C2: 547), so without grouping 32
// consecutive records would run 32 different control paths.
//
// Per tile:
//   1. key:     key and bin of each record -> smem; per-key counts (smem atomics)
//   2. scan:    exclusive scans of counts and of 32-record group counts; a table
//               of (key, group) work items
//   3. scatter: record index of every slot of the key-sorted order
//   4. eval:    warps take work items round-robin; lane l evaluates the l-th record
//               of the group through Dispatch::eval
//   5. emit:    codes in record order -> flags (u8), ballot-packed idempotent bits,
//               per-code histogram (match_any-aggregated shared atomics)
#pragma once

#include "device_common.cuh"
#include "desc_eval.cuh"
#include "eval_generic.cuh"
#include "models.cuh"
#include "seq.cuh"

namespace picker {

// Row f3 fused into the pipelined kernel (picker_validate_models): every
// record's AR input bytes and Chimera latencies are accumulated where its
// verdict is decided -- the staged arguments are read once for both.
#ifdef PICKER_MODELS
constexpr bool kModels = true;
#else
constexpr bool kModels = false;
#endif
// Row f1 on K1's extents (picker_validate_sequence): the shapes also write each
// record's extents to the arena.
#ifdef PICKER_EXTENTS
constexpr bool kExtents = true;
#else
constexpr bool kExtents = false;
#endif
// ... or from K1's codes alone: the shapes are K1's, a window's extents are
// evaluated (from the tables) only when no decisive record decides it.
#ifdef PICKER_SEQ
constexpr bool kSeqLazy = true;
#else
constexpr bool kSeqLazy = false;
#endif

// A specialised module without wide (K2) kernels is compiled with
// PICKER_NO_WIDE: the warp-cooperative path is then dead code that would sit
// between the hot loop's blocks (instruction-cache locality).
#ifdef PICKER_NO_WIDE
constexpr bool kWidePath = false;
#else
constexpr bool kWidePath = true;
#endif

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)  // suspend-time hint (ns): sleep, do not spin
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// TMA 1-D bulk copy global -> shared (16-byte aligned, size a multiple of 16).
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Thread 0: fetch the argument-span bounds of a tile (its first record's
// arg_off, its last record's arg_off and nargs) into shared memory with
// cp.async, so the load latency (the headers of a tile two steps ahead are not
// in any cache) is not waited for where it is issued; read back by
// bounds_read after cp.async.wait_all.  bnd[2] receives the 4-byte nargs.
__device__ __forceinline__ void bounds_async(const DevBatch& B, uint64_t n, uint64_t tile, uint64_t* bnd) {
  const uint64_t base = tile * kTile;
  if (base >= n) return;
  const uint64_t m = min((uint64_t)kTile, n - base);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(bnd)), "l"(&B.rec[base].arg_off)
               : "memory");
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(bnd + 1)),
               "l"(&B.rec[base + m - 1].arg_off)
               : "memory");
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(bnd + 2)), "l"(&B.rec[base + m - 1].nargs)
               : "memory");
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bounds_read(const uint64_t* bnd, uint64_t& lo, uint64_t& lo_last,
                                            uint64_t& n_last) {
  asm volatile("cp.async.wait_all;" ::: "memory");
  lo = bnd[0], lo_last = bnd[1], n_last = *reinterpret_cast<const uint32_t*>(bnd + 2);
}

struct StageInfo {
  uint64_t lo, hi;  // staged argument slots [lo, hi)
  uint32_t shift;   // byte offset of slot lo inside the staged buffer
  uint32_t staged;  // 1: args of this tile are in shared memory
};

// Thread 0: start the copies of tile `tile` into buffer `buf`.  `lo`, `last_off`
// and `last_n` were loaded earlier (the tile's first arg_off and its last
// record's arg_off / nargs) so their latency is off the critical path.
__device__ __forceinline__ void stage_tile(const DevBatch& B, uint64_t n, uint64_t tile, unsigned char* hdr,
                                           unsigned char* arg, uint64_t* bar, StageInfo* info, uint64_t lo,
                                           uint64_t last_off, uint64_t last_n) {
  const uint64_t base = tile * kTile;
  if (base >= n) return;
  const uint64_t m = min((uint64_t)kTile, n - base);
  const uint32_t hbytes = (uint32_t)(m * sizeof(picker_rec_t));
  // a span longer than the buffer (or running past the pool) is staged up to
  // the buffer's capacity: the records whose arguments lie in the staged
  // prefix read shared memory, the rest global memory (their `local` test)
  const uint64_t hi_all = last_off + last_n;
  const uint64_t hi = min(min(hi_all, lo + (uint64_t)kArgCap), B.args_hi);
  StageInfo si{lo, hi, 0, 0};
  uint32_t abytes = 0;
  const char* src = nullptr;
  if (hi_all >= lo && hi > lo && lo >= B.args_lo) {
    const uintptr_t a0 = (uintptr_t)(B.args + lo), a1 = (uintptr_t)(B.args + hi);
    const uintptr_t s0 = a0 & ~(uintptr_t)15, s1 = (a1 + 15) & ~(uintptr_t)15;
    const uintptr_t p0 = (uintptr_t)(B.args + B.args_lo), p1 = (uintptr_t)(B.args + B.args_hi);
    if (s0 >= p0 && s1 <= p1) {  // the rounded span stays inside the pool
      si.staged = 1;
      si.shift = (uint32_t)(a0 - s0);
      abytes = (uint32_t)(s1 - s0);
      src = (const char*)s0;
    }
  }
  *info = si;
  mbar_arrive_expect_tx(bar, hbytes + abytes);
  tma_load_1d(hdr, B.rec + base, hbytes, bar);
  if (abytes) tma_load_1d(arg, src, abytes, bar);
}

// Split staging for the single argument buffer (kArgBufs == 1): the headers
// of a tile go ahead (double-buffered, sizes known without reading them); its
// arguments are fetched once the previous tile's evaluation has released the
// buffer, with the span read from the headers already in shared memory.
__device__ __forceinline__ void stage_hdr(const DevBatch& B, uint64_t n, uint64_t tile, unsigned char* hdr,
                                          uint64_t* bar) {
  const uint64_t base = tile * kTile;
  if (base >= n) return;
  const uint32_t hbytes = (uint32_t)(min((uint64_t)kTile, n - base) * sizeof(picker_rec_t));
  mbar_arrive_expect_tx(bar, hbytes);
  tma_load_1d(hdr, B.rec + base, hbytes, bar);
}
__device__ __forceinline__ void stage_args(const DevBatch& B, int m, const unsigned char* hdr, unsigned char* arg,
                                           uint64_t* bar, StageInfo* info) {
  const uint64_t lo = *reinterpret_cast<const uint64_t*>(hdr + 24);
  const uint64_t last_off = *reinterpret_cast<const uint64_t*>(hdr + 32 * (m - 1) + 24);
  const uint64_t last_n = *reinterpret_cast<const uint32_t*>(hdr + 32 * (m - 1) + 4);
  // a span longer than the buffer (or running past the pool) is staged up to
  // the buffer's capacity: the records whose arguments lie in the staged
  // prefix read shared memory, the rest global memory (their `local` test)
  const uint64_t hi_all = last_off + last_n;
  const uint64_t hi = min(min(hi_all, lo + (uint64_t)kArgCap), B.args_hi);
  StageInfo si{lo, hi, 0, 0};
  uint32_t abytes = 0;
  const char* src = nullptr;
  if (hi_all >= lo && hi > lo && lo >= B.args_lo) {
    const uintptr_t a0 = (uintptr_t)(B.args + lo), a1 = (uintptr_t)(B.args + hi);
    const uintptr_t s0 = a0 & ~(uintptr_t)15, s1 = (a1 + 15) & ~(uintptr_t)15;
    const uintptr_t p0 = (uintptr_t)(B.args + B.args_lo), p1 = (uintptr_t)(B.args + B.args_hi);
    if (s0 >= p0 && s1 <= p1) {
      si.staged = 1;
      si.shift = (uint32_t)(a0 - s0);
      abytes = (uint32_t)(s1 - s0);
      src = (const char*)s0;
    }
  }
  *info = si;
  mbar_arrive_expect_tx(bar, abytes);  // 0 bytes: the phase completes at once
  if (abytes) tma_load_1d(arg, src, abytes, bar);
}

__device__ __forceinline__ picker_rec_t rec_from_smem(const unsigned char* p) {
  const uint4 a = *reinterpret_cast<const uint4*>(p), b = *reinterpret_cast<const uint4*>(p + 16);
  picker_rec_t r;
  r.kernel_id = a.x;
  r.nargs = a.y;
  r.grid_x = a.z;
  r.grid_y = (uint16_t)(a.w & 0xFFFF);
  r.grid_z = (uint16_t)(a.w >> 16);
  r.block_x = (uint16_t)(b.x & 0xFFFF);
  r.block_y = (uint16_t)(b.x >> 16);
  r.block_z = (uint16_t)(b.y & 0xFFFF);
  r.reserved = (uint16_t)(b.y >> 16);
  r.arg_off = ((uint64_t)b.w << 32) | b.z;
  return r;
}

// The K2 scratch of warp `warp` of this CTA (blockDim.x / 32 warps per CTA).
__device__ __forceinline__ WideElem* wide_scratch(const BucketParams& P, int warp) {
  if (P.wide_scratch == nullptr) return nullptr;
  return reinterpret_cast<WideElem*>(P.wide_scratch) + ((uint64_t)blockIdx.x * (blockDim.x >> 5) + warp) * kWideMax;
}

// Lane 0 claims the next work item; the index is broadcast to the warp.
__device__ __forceinline__ uint32_t warp_claim(uint32_t* counter) {
  uint32_t g = 0;
  if ((threadIdx.x & 31) == 0) g = atomicAdd(counter, 1u);
  return __shfl_sync(0xffffffffu, g, 0);
}

// The bucketed kernel for more than kPipeKeys grouping keys (the table-driven
// path groups by kernel: C2 with the specialised module off has 549 keys).
template <class Dispatch>
__global__ void __launch_bounds__(kThreads, kCtasPerSm)
    k_validate_bucket(const __grid_constant__ BucketParams P, const __grid_constant__ DevBatch B,
                      uint64_t n, uint8_t* __restrict__ flags,
                      uint32_t* __restrict__ bits, unsigned long long* __restrict__ counts) {
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t nk = P.nkeys;
  // staging buffers: headers at smem + buf*kHdrBytes, args at smem + kArgOff + buf*kArgBufBytes
  constexpr uint32_t kHdrBytes = kTile * 32;
  constexpr uint32_t kArgOff = 2 * kHdrBytes;
  uint32_t* s_kn = reinterpret_cast<uint32_t*>(smem + kArgOff + 2 * kArgBufBytes);  // KbEntry.kn
  uint16_t* s_key = reinterpret_cast<uint16_t*>(s_kn + kTile);
  uint16_t* s_bin = s_key + kTile;
  uint16_t* s_perm = s_bin + kTile;  // key-sorted slot -> record
  uint8_t* s_code = reinterpret_cast<uint8_t*>(s_perm + kTile);
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_code + kTile);  // kTile is a multiple of 32
  uint32_t* s_off = s_cnt + nk;
  uint32_t* s_cur = s_off + nk;
  uint32_t* s_grp = s_cur + nk;
  __shared__ uint32_t s_hist[PICKER_NUM_COUNTS];
  __shared__ uint32_t s_wsum[2][kWarps];
  __shared__ uint32_t s_ngrp, s_next;
  __shared__ __align__(8) uint64_t s_bar[2];
  __shared__ StageInfo s_info[2];
  __shared__ __align__(16) uint64_t s_bnd[3];  // thread 0: bounds of the next tile to stage

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t ntiles = (n + kTile - 1) / kTile;
  const uint64_t G = gridDim.x;
  if (tid < PICKER_NUM_COUNTS) s_hist[tid] = 0;
  // arg_off bounds of a tile, loaded ahead of its staging
  auto bounds = [&](uint64_t tile, uint64_t& lo, uint64_t& lo_last, uint64_t& n_last) {
    const uint64_t base = tile * kTile;
    lo = lo_last = n_last = 0;
    if (base < n) {
      const uint64_t m = min((uint64_t)kTile, n - base);
      lo = __ldg(&B.rec[base].arg_off);
      lo_last = __ldg(&B.rec[base + m - 1].arg_off);
      n_last = __ldg(&B.rec[base + m - 1].nargs);
    }
  };
  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    for (int b = 0; b < 2; ++b) {
      uint64_t lo, ll, nl;
      bounds(blockIdx.x + b * G, lo, ll, nl);
      stage_tile(B, n, blockIdx.x + b * G, smem + b * kHdrBytes, smem + kArgOff + b * kArgBufBytes,
                 &s_bar[b], &s_info[b], lo, ll, nl);
    }
  }
  __syncthreads();

  uint32_t it = 0;
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += G, ++it) {
    const uint32_t buf = it & 1, parity = (it >> 1) & 1;
    const uint64_t base = tile * kTile;
    const int m = (int)min((uint64_t)kTile, n - base);
    if (tid == 0) bounds_async(B, n, tile + 2 * G, s_bnd);  // consumed after this tile
    for (uint32_t b = tid; b < nk; b += kThreads) s_cnt[b] = 0;
    mbar_wait(&s_bar[buf], parity);
    const unsigned char* hdr = smem + buf * kHdrBytes;
    const unsigned char* sarg = smem + kArgOff + buf * kArgBufBytes;
    const StageInfo si = s_info[buf];
    __syncthreads();

    // 1. keys and per-key counts
    for (int i = tid; i < m; i += kThreads) {
      const uint32_t kid = *reinterpret_cast<const uint32_t*>(hdr + 32 * i);
      uint32_t kb = P.kb_unknown, kn = 0;
      if (kid < P.T.nkernel_slots) {
        const uint2 v = __ldg(reinterpret_cast<const uint2*>(P.kb_of) + kid);
        kb = v.x, kn = v.y;
      }
      const uint32_t key = kb >> 16;
      s_bin[i] = (uint16_t)(kb & 0xFFFFu);
      s_kn[i] = kn;
      s_key[i] = (uint16_t)key;
      atomicAdd(s_cnt + key, 1u);
    }
    __syncthreads();

    // 2. scans over the CTA: record offsets and 32-record groups per key, and
    //    the (key, group) work list
    {
      const uint32_t per = (nk + kThreads - 1) / kThreads;
      const uint32_t b0 = min(nk, tid * per), b1 = min(nk, b0 + per);
      uint32_t rs = 0, gs = 0;
      for (uint32_t b = b0; b < b1; ++b) {
        const uint32_t c = s_cnt[b];
        rs += c;
        gs += (c + 31) >> 5;
      }
      uint32_t ri = rs, gi = gs;  // inclusive warp scans
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t r2 = __shfl_up_sync(0xffffffffu, ri, d), g2 = __shfl_up_sync(0xffffffffu, gi, d);
        if (lane >= d) ri += r2, gi += g2;
      }
      if (lane == 31) s_wsum[0][warp] = ri, s_wsum[1][warp] = gi;
      __syncthreads();
      uint32_t ro = ri - rs, go = gi - gs;
      for (int w = 0; w < warp; ++w) ro += s_wsum[0][w], go += s_wsum[1][w];
      for (uint32_t b = b0; b < b1; ++b) {
        const uint32_t c = s_cnt[b];
        s_off[b] = ro;
        s_cur[b] = ro;
        const uint32_t ng = (c + 31) >> 5;
        for (uint32_t j = 0; j < ng; ++j) s_grp[go + j] = (b << 8) | j;
        ro += c;
        go += ng;
      }
      if (tid == kThreads - 1) s_ngrp = go, s_next = 0;
    }
    __syncthreads();

    // 3. scatter record indices into key order
    for (int i = tid; i < m; i += kThreads) {
      const uint32_t pos = atomicAdd(s_cur + s_key[i], 1u);
      s_perm[pos] = (uint16_t)i;
    }
    __syncthreads();

    // 4. evaluate one 32-record group of one key per warp (warps claim groups
    //    dynamically: groups of different kernels cost different amounts); the
    //    code goes to shared memory, emitted in record order below
    const uint32_t ngrp = s_ngrp;
    for (uint32_t g = warp_claim(&s_next); g < ngrp; g = warp_claim(&s_next)) {
      const uint32_t e = s_grp[g];
      const uint32_t key = e >> 8, j = e & 255u;
      const uint32_t start = s_off[key] + 32u * j, rem = s_cnt[key] - 32u * j;
      if (kWidePath && key == P.wide_key) {  // K2: the whole warp on one record at a time
        for (uint32_t q = 0; q < min(rem, 32u); ++q) {
          const uint32_t wi = s_perm[start + q];
          const picker_rec_t r = rec_from_smem(hdr + 32 * wi);
          const bool local = si.staged && r.arg_off >= si.lo && r.arg_off <= si.hi &&
                             (uint64_t)r.nargs <= si.hi - r.arg_off;
          const int64_t* a = local ? reinterpret_cast<const int64_t*>(sarg + si.shift + 8 * (r.arg_off - si.lo))
                                   : B.args + r.arg_off;
          const uint8_t c = eval_wide_warp(P.T, r, a, B.args_lo, B.args_hi, lane, wide_scratch(P, warp));
          if (lane == 0) s_code[wi] = c;
        }
        continue;
      }
      if ((uint32_t)lane < rem) {
        const uint32_t li = s_perm[start + lane];
        const picker_rec_t r = rec_from_smem(hdr + 32 * li);
        const bool local = si.staged && r.arg_off >= si.lo && r.arg_off <= si.hi &&
                           (uint64_t)r.nargs <= si.hi - r.arg_off;
        const int64_t* a = local ? reinterpret_cast<const int64_t*>(sarg + si.shift + 8 * (r.arg_off - si.lo))
                                 : B.args + r.arg_off;
        s_code[li] = Dispatch::eval(key, s_bin[li], s_kn[li], local, P, r, a, B);
      }
    }
    __syncthreads();
    // this tile's buffers are free: start the copy of the tile after next
    if (tid == 0) {
      uint64_t nlo, nll, nnl;
      bounds_read(s_bnd, nlo, nll, nnl);
      stage_tile(B, n, tile + 2 * G, smem + buf * kHdrBytes, smem + kArgOff + buf * kArgBufBytes,
                 &s_bar[buf], &s_info[buf], nlo, nll, nnl);
    }

    // 5. emit in record order: u8 codes (coalesced), idempotent bit words
    //    (one ballot per 32 records), histogram (match_any-aggregated)
    for (int i0 = warp * 32; i0 < m; i0 += kThreads) {
      const int i = i0 + lane;
      const bool valid = i < m;
      const uint32_t c = valid ? s_code[i] : 0u;
      const unsigned idem = __ballot_sync(0xffffffffu, valid && c <= V_IDEM_KERNEL);
      if (valid) flags[base + i] = (uint8_t)c;
      if (bits != nullptr && lane == 0) bits[(base + i0) >> 5] = idem;
      const int hb = valid ? count_bin((uint8_t)c) : 16;
      const unsigned same = __match_any_sync(0xffffffffu, hb);
      if (valid && (__ffs(same) - 1) == lane) atomicAdd(s_hist + hb, (uint32_t)__popc(same));
    }
    __syncthreads();  // s_code and the per-key arrays are reused by the next tile
  }
  flush_counts(s_hist, counts, P.count_slot);
}

// Pipelined bucketed kernel for at most kPipeKeys grouping keys (the
// specialised module groups by shape: C2's 547 kernels have 31 shapes).
//
// Same per-tile work as k_validate_bucket, with two barriers per tile instead
// of four and no per-key tables in shared memory:
//   - the key pass of tile t+1 runs right after a warp's last group of tile t,
//     so it fills the tail where warps wait for the slowest group; its results
//     (key, rank within key, bin, kn) stay in registers until the scatter;
//   - every warp scans the <= 64 key counters itself (lane l holds keys l and
//     32 + l) and maps a claimed group index to its key with two ballots;
//   - the scatter writes {record | bin << 16, kn} per sorted slot, so an
//     evaluating lane needs one shared load to find its record and kernel;
//   - shortcut kernels and unknown ids get their final code in the key pass
//     (direct_code) and never enter the sort.
// Per tile t (B = __syncthreads):
//   B_a | [kArgBufs == 1: fetch args(t)] emit(t-1), scan + scatter(t) | B_b |
//   restage (t-1)'s header buffer with t+1, [wait args(t)] eval(t), keys(t+1)
template <class Dispatch>
__global__ void __launch_bounds__(kThreads, kCtasPerSm)
    k_validate_pipe(const __grid_constant__ BucketParams P, const __grid_constant__ DevBatch B, uint64_t n,
                    uint8_t* __restrict__ flags, uint32_t* __restrict__ bits,
                    unsigned long long* __restrict__ counts) {
  static_assert(kTile % kThreads == 0, "tile must be a multiple of the CTA size");
  static_assert(kTile <= 8192, "ranks and record indices are 13-bit");
  constexpr int kPer = kTile / kThreads;
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr uint32_t kHdrBytes = kTile * 32;
  constexpr uint32_t kArgOff = 2 * kHdrBytes;
  uint2* s_perm = reinterpret_cast<uint2*>(smem + kArgOff + kArgBufs * kArgBufBytes);
  // codes per tile parity: keys(t+1) writes direct codes while emit(t-1) is done
  uint8_t* s_code = reinterpret_cast<uint8_t*>(s_perm + kTile);  // [2][kTile]
  __shared__ uint32_t s_cnt[2][kPipeKeys];
  __shared__ uint32_t s_grp[kTile / 32 + kPipeKeys];  // group -> start | rem << 13 | key << 19
  __shared__ uint32_t s_hist[PICKER_NUM_COUNTS];
  __shared__ uint32_t s_next[2];
  __shared__ __align__(8) uint64_t s_bar[2];
  __shared__ __align__(8) uint64_t s_abar;  // kArgBufs == 1: the argument buffer
  __shared__ StageInfo s_info[2];
  __shared__ __align__(16) uint64_t s_bnd[3];  // thread 0: bounds of the next tile to stage
  __shared__ uint32_t s_mh[kModels ? 2 * PICKER_MODEL_HIST : 1];  // model histograms (without, with)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t lt_mask = (1u << lane) - 1u;
  ModelSums ms{};
  if (kModels)
    for (int b = tid; b < 2 * PICKER_MODEL_HIST; b += kThreads) s_mh[b] = 0;
  // models: each record's input bytes (kInbUnknown: unknown) go to s_inb where
  // its verdict is decided; the emit adds the models of 32 records in order
  // (full warps, coalesced context sizes)
  uint64_t* s_inb = reinterpret_cast<uint64_t*>(
      ((uintptr_t)(reinterpret_cast<uint8_t*>(s_perm + kTile) + 2 * kTile) + 7) & ~(uintptr_t)7);  // [2][kTile]
  auto inb_table = [&](uint32_t code, const picker_rec_t& r, const int64_t* a) -> uint64_t {
    uint64_t b = 0;
    return model_input_bytes_coded(P.T, r, a, code, b) ? b : kInbUnknown;
  };
  // extents with P.seq_out (row f1 fused): the tile's extent slots and info
  // words stay in shared memory (same place as s_inb; the two modes are
  // exclusive), and the windows of tile t are decided in the emit slot of
  // t + 1, a warp per window (seq.cuh)
  const bool seq_fused = (kExtents || kSeqLazy) && P.seq_out != nullptr;
  int64_t* s_ext = reinterpret_cast<int64_t*>(
      ((uintptr_t)(reinterpret_cast<uint8_t*>(s_perm + kTile) + 2 * kTile) + 15) & ~(uintptr_t)15);
  uint32_t* s_xinfo = reinterpret_cast<uint32_t*>(s_ext + (size_t)kTile * 2 * P.xcap);
  auto windows = [&](uint64_t tbase, int m, uint32_t cbuf) {
    if constexpr (kExtents || kSeqLazy) {
      if (!seq_fused) return;
      const uint32_t W = P.seq_window, nwin = ((uint32_t)m + W - 1) / W;
      for (uint32_t w = warp; w < nwin; w += kWarps) {
        const uint32_t i0 = w * W;
        bool undecided = false;
        const uint8_t code =
            kSeqLazy ? seq_window_lanes(P.T, B, tbase + i0, min(W, (uint32_t)m - i0), P.seq_mode,
                                        s_code + cbuf * kTile + i0, nullptr,
                                        P.seq_scratch + ((uint64_t)blockIdx.x * kWarps + warp) * 64 * P.xcap, P.xcap,
                                        lane, &undecided)
                     : seq_window_lanes(P.T, B, tbase + i0, min(W, (uint32_t)m - i0), P.seq_mode,
                                        s_code + cbuf * kTile + i0, s_xinfo + i0,
                                        s_ext + (size_t)i0 * 2 * P.xcap, P.xcap, lane, nullptr);
        if (lane == 0) {
          P.seq_out[(tbase + i0) / W] = code;
          if (undecided && P.seq_undecided) atomicAdd(P.seq_undecided, 1u);
        }
      }
    }
  };
  const uint64_t ntiles = (n + kTile - 1) / kTile;
  const uint64_t G = gridDim.x;
  if (tid < PICKER_NUM_COUNTS) s_hist[tid] = 0;
  for (int b = tid; b < 2 * (int)kPipeKeys; b += kThreads) (&s_cnt[0][0])[b] = 0;
  // warp w's first group of a tile is group w (no claim); the counter hands
  // out the rest from kWarps on
  if (tid < 2) s_next[tid] = kWarps;
  auto bounds = [&](uint64_t tile, uint64_t& lo, uint64_t& lo_last, uint64_t& n_last) {
    const uint64_t base = tile * kTile;
    lo = lo_last = n_last = 0;
    if (base < n) {
      const uint64_t m = min((uint64_t)kTile, n - base);
      lo = __ldg(&B.rec[base].arg_off);
      lo_last = __ldg(&B.rec[base + m - 1].arg_off);
      n_last = __ldg(&B.rec[base + m - 1].nargs);
    }
  };
  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    mbar_init(&s_abar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    for (int b = 0; b < 2; ++b) {
      if constexpr (kArgBufs == 1) {
        stage_hdr(B, n, blockIdx.x + b * G, smem + b * kHdrBytes, &s_bar[b]);
      } else {
        uint64_t lo, ll, nl;
        bounds(blockIdx.x + b * G, lo, ll, nl);
        stage_tile(B, n, blockIdx.x + b * G, smem + b * kHdrBytes, smem + kArgOff + b * kArgBufBytes,
                   &s_bar[b], &s_info[b], lo, ll, nl);
      }
    }
  }
  __syncthreads();

  // key pass of one tile: results in registers (key | rank << 8, record | bin << 16, kn)
  uint32_t kr[kPer], rb[kPer], kn[kPer];
  auto keys = [&](uint64_t tile, uint32_t it) {
    const uint32_t buf = it & 1;
    const uint64_t base = tile * kTile;
    const int m = (int)min((uint64_t)kTile, n - base);
    mbar_wait(&s_bar[buf], (it >> 1) & 1);
    const unsigned char* hdr = smem + buf * kHdrBytes;
    // phases over all of the thread's records, so the table loads and the
    // match_any latencies of its records overlap
    uint32_t key[kPer], e[kPer];
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int i = q * kThreads + warp * 32 + lane;
      uint32_t kb = 0xFFu << 16;
      e[q] = V_ERR_KERNEL;
      if (i < m) {
        const uint32_t kid = *reinterpret_cast<const uint32_t*>(hdr + 32 * i);
        kb = P.kb_unknown;
        if (kid < P.T.nkernel_slots) {
          const uint2 v = __ldg(reinterpret_cast<const uint2*>(P.kb_of) + kid);
          kb = v.x, e[q] = v.y;
        }
      }
      key[q] = kb >> 16;
      rb[q] = (uint32_t)i | (kb & 0xFFFFu) << 16;
      // models: the context sizes the emit of this tile reads (an iteration
      // from now, right after a barrier) are fetched into L2 here, so that
      // load does not expose an HBM round trip between two barriers
      if constexpr (kModels)
        if (P.ctx_bytes != nullptr && (lane & 15) == 0 && i < m)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(P.ctx_bytes + base + i));
    }
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int i = q * kThreads + warp * 32 + lane;
      if (key[q] == P.direct_key) {  // shortcut / unknown: final here, not sorted
        const uint2 h = *reinterpret_cast<const uint2*>(hdr + 32 * i + 24);
        const uint32_t dc = direct_code(e[q], *reinterpret_cast<const uint32_t*>(hdr + 32 * i + 4),
                                        (uint64_t)h.y << 32 | h.x, B.args_lo, B.args_hi);
        s_code[buf * kTile + i] = (uint8_t)dc;
        if constexpr (kModels) {  // (the arguments of tile + 1 are not staged yet: global)
          const picker_rec_t r = rec_from_smem(hdr + 32 * i);
          s_inb[buf * kTile + i] = dc == V_IDEM_KERNEL ? inb_table(dc, r, B.args + r.arg_off) : kInbUnknown;
        }
        key[q] = 0xFFu;
      }
    }
    unsigned peers[kPer];
#pragma unroll
    for (int q = 0; q < kPer; ++q) peers[q] = __match_any_sync(0xffffffffu, key[q]);
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int leader = 31 - __clz(peers[q]);  // any lane of the peers does the add
      uint32_t b = 0;
      if (key[q] != 0xFFu && lane == leader) b = atomicAdd(&s_cnt[buf][key[q]], (uint32_t)__popc(peers[q]));
      b = __shfl_sync(0xffffffffu, b, leader);
      kr[q] = key[q] != 0xFFu ? key[q] | (b + __popc(peers[q] & lt_mask)) << 8 : 0xFFu;
      kn[q] = e[q];
    }
  };
  // codes of one tile in record order: u8 flags, idempotent bit words, histogram
  auto emit = [&](uint64_t base, int m, uint32_t buf) {
    for (int i0 = warp * 32; i0 < m; i0 += kThreads) {
      const int i = i0 + lane;
      const bool valid = i < m;
      const uint32_t c = valid ? s_code[buf * kTile + i] : 0u;
      const unsigned idem = __ballot_sync(0xffffffffu, valid && c <= V_IDEM_KERNEL);
      if (valid && flags != nullptr) flags[base + i] = (uint8_t)c;
      if (bits != nullptr && lane == 0) bits[(base + i0) >> 5] = idem;
      const int hb = valid ? count_bin((uint8_t)c) : 16;
      const unsigned same = __match_any_sync(0xffffffffu, hb);
      if (valid && (__ffs(same) - 1) == lane) atomicAdd(s_hist + hb, (uint32_t)__popc(same));
      if constexpr (kModels)
        if (valid) {
          // (the input bytes are the record's own, whatever its verdict; the
          // verdict the models take is the kernel's or the caller's)
          const uint64_t inb = s_inb[buf * kTile + i];
          model_add(ms, s_mh, s_mh + PICKER_MODEL_HIST, P.given_codes ? P.given_codes[base + i] : c,
                    inb != kInbUnknown, inb, P.ctx_bytes ? P.ctx_bytes[base + i] : 0, P.kill_ns, P.save_bpu);
        }
    }
  };

  if ((uint64_t)blockIdx.x < ntiles) keys(blockIdx.x, 0);
  if (kArgBufs == 2 && tid == 0) bounds_async(B, n, blockIdx.x + 2 * G, s_bnd);  // the next tile to stage
  uint32_t it = 0;
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += G, ++it) {
    const uint32_t buf = it & 1;
    const uint64_t base = tile * kTile;
    const int m = (int)min((uint64_t)kTile, n - base);
    __syncthreads();  // B_a: eval(t-1) and keys(t) done
    // single argument buffer: free now; fetch this tile's arguments, which
    // the scan / scatter / emit below overlap
    if (kArgBufs == 1 && tid == 0) stage_args(B, m, smem + buf * kHdrBytes, smem + kArgOff, &s_abar, &s_info[buf]);
    if (it > 0) {  // tiles before the last are full
      emit(base - G * kTile, kTile, buf ^ 1);
      windows(base - G * kTile, kTile, buf ^ 1);
    }
    // counters and claim index of the other parity: last used before B_b of
    // t-1, next used after B_b of t
    for (int b = tid; b < (int)kPipeKeys; b += kThreads) s_cnt[buf ^ 1][b] = 0;  // CTAs of < 64 threads too
    if (tid == 0) s_next[buf ^ 1] = kWarps;
    // scan (every warp, registers): lane l holds keys l, 32 + l, ... as
    // count | groups << 16, inclusive (kKPL keys per lane, chained)
    uint32_t cc[kKPL], vv[kKPL];
#pragma unroll
    for (int h = 0; h < kKPL; ++h) {
      cc[h] = s_cnt[buf][lane + 32 * h];
      vv[h] = cc[h] | ((cc[h] + 31) >> 5) << 16;
    }
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
      for (int h = 0; h < kKPL; ++h) {
        const uint32_t a = __shfl_up_sync(0xffffffffu, vv[h], d);
        if (lane >= d) vv[h] += a;
      }
    }
#pragma unroll
    for (int h = 1; h < kKPL; ++h) vv[h] += __shfl_sync(0xffffffffu, vv[h - 1], 31);
    uint32_t off[kKPL];
#pragma unroll
    for (int h = 0; h < kKPL; ++h) off[h] = (vv[h] & 0xFFFFu) - cc[h];
    const uint32_t ngrp = __shfl_sync(0xffffffffu, vv[kKPL - 1] >> 16, 31);
    // scatter
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const uint32_t key = kr[q] & 0xFFu;
      uint32_t o = 0;
#pragma unroll
      for (int h = 0; h < kKPL; ++h) {
        const uint32_t oh = __shfl_sync(0xffffffffu, off[h], key & 31);
        if ((key >> 5) == (uint32_t)h) o = oh;
      }
      if (key != 0xFFu) s_perm[o + (kr[q] >> 8)] = make_uint2(rb[q], kn[q]);
    }
    // group table: warp w writes groups j = w, w + kWarps, ... of every key
#pragma unroll
    for (int h = 0; h < kKPL; ++h) {
      const uint32_t gs = (vv[h] >> 16) - ((cc[h] + 31) >> 5);
      for (uint32_t j = warp; 32 * j < cc[h]; j += kWarps)
        s_grp[gs + j] = (off[h] + 32 * j) | min(32u, cc[h] - 32 * j) << 13 | (uint32_t)(lane + 32 * h) << 19;
    }
    __syncthreads();  // B_b
    // the previous tile's buffers are free: start the copy of the next tile
    // (after B_b, so this serial thread-0 work is not waited for at a barrier)
    if (it > 0 && tid == 0) {
      if constexpr (kArgBufs == 1) {
        stage_hdr(B, n, tile + G, smem + (buf ^ 1) * kHdrBytes, &s_bar[buf ^ 1]);
      } else {
        uint64_t nlo, nll, nnl;
        bounds_read(s_bnd, nlo, nll, nnl);
        stage_tile(B, n, tile + G, smem + (buf ^ 1) * kHdrBytes, smem + kArgOff + (buf ^ 1) * kArgBufBytes,
                   &s_bar[buf ^ 1], &s_info[buf ^ 1], nlo, nll, nnl);
        bounds_async(B, n, tile + 2 * G, s_bnd);
      }
    }

    const unsigned char* hdr = smem + buf * kHdrBytes;
    const unsigned char* sarg = smem + kArgOff + (kArgBufs == 1 ? 0u : buf * kArgBufBytes);
    if (kArgBufs == 1) mbar_wait(&s_abar, it & 1);
    const StageInfo si = s_info[buf];
    // (claiming one group ahead was measured slower: a warp holding a claimed
    // group lengthens the tail, C4 1.04 -> 0.32 G inst/s)
    for (uint32_t g = (uint32_t)warp; g < ngrp; g = warp_claim(&s_next[buf])) {
      const uint32_t e = s_grp[g];
      const uint32_t key = e >> 19, start = e & 0x1FFFu, rem = (e >> 13) & 63u;
      if (kWidePath && key == P.wide_key) {  // K2: the whole warp on one record at a time
        for (uint32_t q = 0; q < min(rem, 32u); ++q) {
          const uint32_t wi = s_perm[start + q].x & 0xFFFFu;
          const picker_rec_t r = rec_from_smem(hdr + 32 * wi);
          const bool local = si.staged && r.arg_off >= si.lo && r.arg_off <= si.hi &&
                             (uint64_t)r.nargs <= si.hi - r.arg_off;
          const int64_t* a = local ? reinterpret_cast<const int64_t*>(sarg + si.shift + 8 * (r.arg_off - si.lo))
                                   : B.args + r.arg_off;
          const uint8_t cw = eval_wide_warp(P.T, r, a, B.args_lo, B.args_hi, lane, wide_scratch(P, warp));
          if (lane == 0) s_code[buf * kTile + wi] = cw;
          if constexpr (kModels)
            if (lane == 0) s_inb[buf * kTile + wi] = inb_table(cw, r, a);
        }
        continue;
      }
      if ((uint32_t)lane < rem) {
        const uint2 pe = s_perm[start + lane];
        const uint32_t li = pe.x & 0xFFFFu;
        const picker_rec_t r = rec_from_smem(hdr + 32 * li);
        // args inside the staged span [lo, hi) (span < 2^32 slots): one 64-bit
        // subtraction, then 32-bit compares
        const uint64_t rel = r.arg_off - si.lo;
        const bool local = si.staged && (rel >> 32) == 0 && (uint32_t)rel <= (uint32_t)(si.hi - si.lo) &&
                           r.nargs <= (uint32_t)(si.hi - si.lo) - (uint32_t)rel;
        // one call site: a second inlined copy of every shape function (shared
        // vs global pointer) doubles the code and thrashes the instruction
        // cache on large summaries (C4: 1.04 -> 0.32 G inst/s)
        const int64_t* a = local ? reinterpret_cast<const int64_t*>(sarg + si.shift + 8 * (r.arg_off - si.lo))
                                 : B.args + r.arg_off;
        if constexpr (kModels) {  // the shape also returns the input bytes (specialised code)
          uint64_t inb = kInbUnknown;
          const uint8_t code = Dispatch::eval(key, pe.x >> 16, pe.y, local, P, r, a, B, &inb);
          s_code[buf * kTile + li] = code;
          s_inb[buf * kTile + li] = inb == kInbTable ? inb_table(code, r, a) : inb;
        } else if constexpr (kExtents) {
          XOut xo{seq_fused ? s_ext + (size_t)li * 2 * P.xcap : P.xarena + (base + li) * 2 * P.xcap, P.xcap, 0, 0,
                  0};
          const uint8_t code = Dispatch::eval(key, pe.x >> 16, pe.y, local, P, r, a, B, &xo);
          s_code[buf * kTile + li] = code;
          (seq_fused ? s_xinfo[li] : P.xinfo[base + li]) = xo_info(xo);
        } else {
          const uint8_t code = Dispatch::eval(key, pe.x >> 16, pe.y, local, P, r, a, B);
          s_code[buf * kTile + li] = code;
        }
      }
    }
    if (tile + G < ntiles) keys(tile + G, it + 1);
    if (tile + G >= ntiles) {  // last tile of this CTA
      __syncthreads();
      emit(base, m, buf);
      windows(base, m, buf);
    }
  }
  __syncthreads();
  flush_counts(s_hist, counts, P.count_slot);
  if constexpr (kModels) model_flush(ms, s_mh, s_mh + PICKER_MODEL_HIST, P.model_acc);
}

// Small batches (n <= kSmallMax, one CTA): one thread per record straight from
// global memory -- no staging, no sort, no grid-wide atomics.  This is the
// latency path of a launcher that validates a few launches and waits for the
// verdicts (the paper's per-launch use); the counts are written,
// not accumulated, so the caller needs no memset before it.
template <class Dispatch>
__global__ void __launch_bounds__(kSmallThreads)
    k_validate_small(const __grid_constant__ BucketParams P, const __grid_constant__ DevBatch B, uint32_t n,
                     uint8_t* __restrict__ flags, uint32_t* __restrict__ bits,
                     unsigned long long* __restrict__ counts) {
  __shared__ uint32_t s_hist[PICKER_NUM_COUNTS];
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid < PICKER_NUM_COUNTS) s_hist[tid] = 0;
  __syncthreads();
  for (uint32_t i0 = (uint32_t)tid & ~31u; i0 < n; i0 += kSmallThreads) {
    const uint32_t i = i0 + lane;
    const bool valid = i < n;
    uint32_t code = 0, key = 0xFFFFFFFFu, kb = P.kb_unknown, kn = V_ERR_KERNEL;
    picker_rec_t r{};
    if (valid) {
      r = load_rec(B.rec + i);
      if (r.kernel_id < P.T.nkernel_slots) {
        const uint2 v = __ldg(reinterpret_cast<const uint2*>(P.kb_of) + r.kernel_id);
        kb = v.x, kn = v.y;
      }
      key = kb >> 16;
    }
    const bool wide = kWidePath && valid && key == P.wide_key;
    if (kWidePath) {  // K2 records: the whole warp on one record at a time
      for (unsigned wm = __ballot_sync(0xffffffffu, wide); wm; wm &= wm - 1) {
        const uint32_t src = (uint32_t)__ffs(wm) - 1;
        const picker_rec_t rr = load_rec(B.rec + i0 + src);
        const uint8_t cw = eval_wide_warp(P.T, rr, B.args + rr.arg_off, B.args_lo, B.args_hi, lane,
                                          wide_scratch(P, tid >> 5));
        if ((uint32_t)lane == src) code = cw;
      }
    }
    if (valid && key == P.direct_key)  // shortcut / unknown id (not in the pipelined dispatch)
      code = direct_code(kn, r.nargs, r.arg_off, B.args_lo, B.args_hi);
    else if (valid && !wide)
      code = Dispatch::eval(key, kb & 0xFFFFu, kn, false, P, r, B.args + r.arg_off, B);
    const unsigned idem = __ballot_sync(0xffffffffu, valid && code <= V_IDEM_KERNEL);
    if (valid) flags[i] = (uint8_t)code;
    if (bits != nullptr && lane == 0) bits[i0 >> 5] = idem;
    const int hb = valid ? count_bin((uint8_t)code) : 16;
    const unsigned same = __match_any_sync(0xffffffffu, hb);
    if (valid && (__ffs(same) - 1) == lane) atomicAdd(s_hist + hb, (uint32_t)__popc(same));
  }
  __syncthreads();
  if (counts && tid < PICKER_NUM_COUNTS) counts[tid] = s_hist[tid];
}

// Dispatch used by the static library: every bin through the table-driven
// evaluator (grouping by kernel makes its table reads warp-uniform).
struct GenericDispatch {
  static __device__ __forceinline__ uint8_t eval(uint32_t key, uint32_t bin, uint32_t kn, bool local,
                                                 const BucketParams& P, const picker_rec_t& r,
                                                 const int64_t* a, const DevBatch& B) {
    (void)key, (void)kn, (void)local;
    if (bin >= P.nbins) return V_ERR_KERNEL;
    return eval_generic(P.T, r, a, B.args_lo, B.args_hi);
  }
};

}  // namespace picker
