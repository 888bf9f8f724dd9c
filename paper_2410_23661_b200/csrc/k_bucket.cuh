// K1 staged + bucketed validation kernel.
//
// One persistent CTA per SM walks tiles of kTile launch records.  Each tile's
// 32-byte headers and its contiguous argument span are copied global->shared
// by the TMA engine (cp.async.bulk, completion on an mbarrier), double-
// buffered so the copy of the next tile overlaps the evaluation of this one:
// every input byte crosses HBM once, in bulk, and all per-record gathers hit
// shared memory.
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
#include "eval_generic.cuh"

namespace picker {

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
      : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
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
  const uint64_t hi = last_off + last_n;
  StageInfo si{lo, hi, 0, 0};
  uint32_t abytes = 0;
  const char* src = nullptr;
  if (hi > lo && hi - lo <= (uint64_t)kArgCap && lo >= B.args_lo && hi <= B.args_hi) {
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

// ---------------------------------------------------------------------------
// The pipelined kernel.  Warp roles (no CTA-wide barrier in the steady state):
//   warp 0       producer: lane 0 waits until a stage is empty, then issues the
//                TMA bulk copies of the next tile into it (full[s] mbarrier);
//   warps 1, 2   bucketers (tiles alternate): wait full[s], group the tile's
//                records by key (counting sort in shared memory), write the
//                stage's group table, publish ready_tile[s];
//   warps 3..    consumers: claim groups of the oldest ready tile (tile-tagged
//                64-bit counter), evaluate one group of <= 32 records of one key,
//                emit codes / bits / histogram; the consumer that finishes the
//                tile's last group writes its bit words and arrives on empty[s].
// Consumers never wait for stragglers: a warp that finds no group left in a
// tile moves on to the next one.
// ---------------------------------------------------------------------------
constexpr int kMaxStages = 8;

struct StageCtl {
  uint64_t full, empty;        // mbarriers
  uint32_t claim, pad2;        // next group of the tile in `ngrp`
  unsigned long long ngrp;     // (tile << 32) | group count
  unsigned long long ready;    // tile + 1 once bucketed
  uint32_t remaining;          // groups not yet finished
  uint32_t pad;
  StageInfo info;
};

__device__ __forceinline__ void fence_acq_rel_cta() { asm volatile("fence.acq_rel.cta;" ::: "memory"); }
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.cta.shared::cta.u64 [%0], %1;" ::"r"(smem_u32(p)), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.cta.shared::cta.u64 %0, [%1];" : "=l"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t atom_add_acq_rel_u32(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(smem_u32(p)), "r"(v)
               : "memory");
  return old;
}
__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// named barrier of the bucketer warps only (id 1; consumers never take part)
__device__ __forceinline__ void bucket_sync() {
  asm volatile("bar.sync 1, %0;" ::"r"(kBucketThreads) : "memory");
}

template <class Dispatch>
__global__ void __launch_bounds__(kThreads, kCtasPerSm)
    k_validate_bucket(const __grid_constant__ BucketParams P, const __grid_constant__ DevBatch B,
                      uint64_t n, uint8_t* __restrict__ flags, uint32_t* __restrict__ bits,
                      unsigned long long* __restrict__ counts) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ StageCtl ctl[kMaxStages];
  __shared__ uint32_t s_hist[PICKER_NUM_COUNTS];
  const uint32_t nk = P.nkeys;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t ntiles = (n + kTile - 1) / kTile;
  const uint64_t G = gridDim.x;
  // stage s: [headers | args | perm (u32 per record) | groups | bits]
  const size_t sbytes = stage_bytes(nk);  // group table: kTile/32 + nk entries
  auto stage_hdr = [&](int s) { return smem + (size_t)s * sbytes; };
  auto stage_arg = [&](int s) { return smem + (size_t)s * sbytes + kTile * 32; };
  auto stage_perm = [&](int s) {
    return reinterpret_cast<uint32_t*>(smem + (size_t)s * sbytes + kTile * 32 + kArgBufBytes);
  };
  auto stage_bits = [&](int s) { return stage_perm(s) + kTile; };
  auto stage_grp = [&](int s) { return stage_bits(s) + kTile / 32; };

  if (tid < PICKER_NUM_COUNTS) s_hist[tid] = 0;
  if (tid < kStages) {
    StageCtl& c = ctl[tid];
    mbar_init(&c.full, 1);
    mbar_init(&c.empty, 1);
    c.claim = 0;
    c.ngrp = 0;
    c.ready = 0;
    c.remaining = 0;
  }
  for (int s = 0; s < kStages; ++s)
    for (int w = tid; w < kTile / 32; w += kThreads) stage_bits(s)[w] = 0;
  if (tid == 0) {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {
    // ---------------- producer ----------------
    if (lane == 0) {
      // argument-span bounds of a tile (two header fields of its first and last
      // record), loaded one tile ahead so their latency overlaps the empty wait
      auto bounds = [&](uint64_t tile, uint64_t& lo, uint64_t& ll, uint64_t& nl) {
        lo = ll = nl = 0;
        if (tile < ntiles) {
          const uint64_t base = tile * kTile, m = min((uint64_t)kTile, n - base);
          lo = __ldg(&B.rec[base].arg_off);
          ll = __ldg(&B.rec[base + m - 1].arg_off);
          nl = __ldg(&B.rec[base + m - 1].nargs);
        }
      };
      uint64_t lo, ll, nl;
      bounds(blockIdx.x, lo, ll, nl);
      for (uint64_t k = 0;; ++k) {
        const uint64_t tile = blockIdx.x + k * G;
        if (tile >= ntiles) break;
        const int s = (int)(k % kStages);
        const uint64_t clo = lo, cll = ll, cnl = nl;
        bounds(tile + G, lo, ll, nl);
        if (k >= (uint64_t)kStages) {
          mbar_wait(&ctl[s].empty, (uint32_t)((k / kStages - 1) & 1));
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        stage_tile(B, n, tile, stage_hdr(s), stage_arg(s), &ctl[s].full, &ctl[s].info, clo, cll, cnl);
      }
    }
  } else if (warp <= kBucketWarps) {
    // ---------------- bucketers (warps 1..kBucketWarps, one tile at a time) ----------------
    const int bt = tid - 32;  // 0 .. kBucketThreads-1
    uint32_t* sc_kb = reinterpret_cast<uint32_t*>(smem + (size_t)kStages * sbytes);
    uint32_t* cnt = sc_kb + kTile;
    uint32_t* off = cnt + nk;
    __shared__ uint32_t s_ngroups;
    for (uint64_t k = 0;; ++k) {
      const uint64_t tile = blockIdx.x + k * G;
      if (tile >= ntiles) break;
      const int s = (int)(k % kStages);
      const int m = (int)min((uint64_t)kTile, n - tile * kTile);
      for (uint32_t i = bt; i < nk; i += kBucketThreads) cnt[i] = 0;
      mbar_wait(&ctl[s].full, (uint32_t)((k / kStages) & 1));
      bucket_sync();
      const unsigned char* hdr = stage_hdr(s);
      // keys and per-key counts
      for (int i0 = (bt & ~31); i0 < m; i0 += kBucketThreads) {
        const int i = i0 + lane;
        const bool valid = i < m;
        const unsigned mask = __ballot_sync(0xffffffffu, valid);
        if (valid) {
          const uint32_t kid = *reinterpret_cast<const uint32_t*>(hdr + 32 * i);
          const uint32_t kb = kid < P.T.nkernel_slots ? __ldg(P.kb_of + kid) : P.kb_unknown;
          sc_kb[i] = kb;
          const uint32_t key = kb >> 16;
          const unsigned same = __match_any_sync(mask, key);
          if ((__ffs(same) - 1) == lane) atomicAdd(cnt + key, (uint32_t)__popc(same));
        }
      }
      bucket_sync();
      // one warp: exclusive scans of counts and 32-record groups; group table
      uint32_t* grp = stage_grp(s);
      if (warp == 1) {
        const uint32_t per = (nk + 31) / 32;
        const uint32_t b0 = min(nk, lane * per), b1 = min(nk, b0 + per);
        uint32_t rs = 0, gs = 0;
        for (uint32_t q = b0; q < b1; ++q) {
          rs += cnt[q];
          gs += (cnt[q] + 31) >> 5;
        }
        uint32_t ri = rs, gi = gs;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t r2 = __shfl_up_sync(0xffffffffu, ri, d), g2 = __shfl_up_sync(0xffffffffu, gi, d);
          if (lane >= d) ri += r2, gi += g2;
        }
        if (lane == 31) s_ngroups = gi;
        uint32_t ro = ri - rs, go = gi - gs;
        for (uint32_t q = b0; q < b1; ++q) {
          const uint32_t c = cnt[q];
          off[q] = ro;
          for (uint32_t j = 0; 32 * j < c; ++j)
            grp[go++] = (ro + 32 * j) | ((min(32u, c - 32 * j) - 1) << 11) | (q << 16);
          ro += c;
        }
      }
      bucket_sync();
      // scatter record indices (and bins) into key order
      uint32_t* perm = stage_perm(s);
      for (int i0 = (bt & ~31); i0 < m; i0 += kBucketThreads) {
        const int i = i0 + lane;
        const bool valid = i < m;
        const unsigned mask = __ballot_sync(0xffffffffu, valid);
        if (valid) {
          const uint32_t kb = sc_kb[i];
          const uint32_t key = kb >> 16;
          const unsigned same = __match_any_sync(mask, key);
          const int leader = __ffs(same) - 1;
          uint32_t pos0 = 0;
          if (leader == lane) pos0 = atomicAdd(off + key, (uint32_t)__popc(same));
          pos0 = __shfl_sync(same, pos0, leader);
          const uint32_t rank = __popc(same & ((1u << lane) - 1));
          perm[pos0 + rank] = (uint32_t)i | ((kb & 0xFFFFu) << 16);
        }
      }
      bucket_sync();
      if (bt == 0) {
        const uint32_t ngroups = s_ngroups;
        // tag first, then the claim counter: a consumer whose claim hits the reset
        // counter is guaranteed to read the new tag (and skip a tile it does not own)
        ctl[s].remaining = ngroups;
        ctl[s].ngrp = ((unsigned long long)tile << 32) | ngroups;
        fence_acq_rel_cta();
        ctl[s].claim = 0;
        st_release_u64(&ctl[s].ready, tile + 1);
      }
    }
  } else {
    // ---------------- consumers ----------------
    for (uint64_t k = 0;; ++k) {
      const uint64_t tile = blockIdx.x + k * G;
      if (tile >= ntiles) break;
      const int s = (int)(k % kStages);
      if (lane == 0)
        while (ld_acquire_u64(&ctl[s].ready) < tile + 1) __nanosleep(64);
      __syncwarp();
      const uint64_t base = tile * kTile;
      const unsigned char* hdr = stage_hdr(s);
      const unsigned char* sarg = stage_arg(s);
      const uint32_t* perm = stage_perm(s);
      const uint32_t* grp = stage_grp(s);
      uint32_t* sbits = stage_bits(s);
      const StageInfo si = ctl[s].info;
      for (;;) {
        uint32_t g = 0;
        unsigned long long ng = 0;
        if (lane == 0) {
          g = atom_add_acq_rel_u32(&ctl[s].claim, 1u);
          ng = ld_volatile_u64(&ctl[s].ngrp);
        }
        g = __shfl_sync(0xffffffffu, g, 0);
        ng = __shfl_sync(0xffffffffu, ng, 0);
        if ((ng >> 32) != tile || g >= (uint32_t)ng) break;  // no group left / stage reused
        const uint32_t e = grp[g];
        const uint32_t start = e & 0x7FFu, cnt = ((e >> 11) & 31u) + 1, key = e >> 16;
        const bool on = (uint32_t)lane < cnt;
        uint8_t code = 0;
        if (on) {
          const uint32_t pe = perm[start + lane];
          const uint32_t li = pe & 0xFFFFu, bin = pe >> 16;
          const picker_rec_t r = rec_from_smem(hdr + 32 * li);
          const bool local = si.staged && r.arg_off >= si.lo && r.arg_off <= si.hi &&
                             (uint64_t)r.nargs <= si.hi - r.arg_off;
          const int64_t* a = local ? reinterpret_cast<const int64_t*>(sarg + si.shift + 8 * (r.arg_off - si.lo))
                                   : B.args + r.arg_off;
          code = Dispatch::eval(key, bin, P, r, a, B);
          flags[base + li] = code;
          if (code <= V_IDEM_KERNEL) atomicOr(sbits + (li >> 5), 1u << (li & 31));
        }
        const int hb = on ? count_bin(code) : 16;
        const unsigned same = __match_any_sync(0xffffffffu, hb);
        if (on && (__ffs(same) - 1) == lane) atomicAdd(s_hist + hb, (uint32_t)__popc(same));
        __syncwarp();
        uint32_t left = 0;
        if (lane == 0) left = atom_add_acq_rel_u32(&ctl[s].remaining, 0xFFFFFFFFu);  // -1
        left = __shfl_sync(0xffffffffu, left, 0);
        if (left == 1) {  // this warp finished the tile's last group
          const int m = (int)min((uint64_t)kTile, n - base);
          for (int w = lane; w < (m + 31) / 32; w += 32) {
            const uint32_t v = *reinterpret_cast<volatile uint32_t*>(sbits + w);
            if (bits) bits[(base >> 5) + w] = v;
            sbits[w] = 0;
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&ctl[s].empty);
        }
      }
    }
  }
  __syncthreads();
  if (counts && tid < PICKER_NUM_COUNTS && s_hist[tid])
    atomicAdd(counts + tid, (unsigned long long)s_hist[tid]);
}

// Dispatch used by the static library: every bin through the table-driven
// evaluator (grouping by kernel makes its table reads warp-uniform).
struct GenericDispatch {
  static __device__ __forceinline__ uint8_t eval(uint32_t key, uint32_t bin, const BucketParams& P,
                                                 const picker_rec_t& r, const int64_t* a,
                                                 const DevBatch& B) {
    (void)key;
    if (bin >= P.nbins) return V_ERR_KERNEL;
    return eval_generic(P.T, r, a, B.args_lo, B.args_hi);
  }
};

}  // namespace picker
