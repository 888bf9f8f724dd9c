// Device helpers shared by the validation kernels.
#pragma once

#ifndef __CUDACC_RTC__
#include <cuda_runtime.h>

#include <cstdint>
#endif

#include "../../include/picker.h"
#include "tables.hpp"

namespace picker {

// Wrapping 64-bit arithmetic (the loader proves no wrap happens on records
// that pass their checks; unsigned ops keep the other cases defined).
__device__ __forceinline__ int64_t mul64(int64_t a, int64_t b) {
  return (int64_t)((uint64_t)a * (uint64_t)b);
}
// Product of two values the loader proved to fit int32 (IrTerm.narrow): one
// 32x32->64 multiply, exact.
__device__ __forceinline__ int64_t mulw(int64_t a, int64_t b) {
  return (int64_t)(int32_t)a * (int64_t)(int32_t)b;
}
__device__ __forceinline__ int64_t add64(int64_t a, int64_t b) {
  return (int64_t)((uint64_t)a + (uint64_t)b);
}
__device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__device__ __forceinline__ int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }
__device__ __forceinline__ int64_t floordiv64(int64_t x, uint32_t d) {
  if (d == 1) return x;
  int64_t q = x / (int64_t)d;
  if ((q * (int64_t)d != x) && x < 0) --q;
  return q;
}
__device__ __forceinline__ bool cmp64(int64_t a, uint8_t op, int64_t b) {
  switch (op) {
    case CMP_LT: return a < b;
    case CMP_LE: return a <= b;
    case CMP_GT: return a > b;
    case CMP_GE: return a >= b;
    case CMP_EQ: return a == b;
    default: return a != b;
  }
}

__device__ __forceinline__ picker_rec_t load_rec(const picker_rec_t* p) {
  const uint4* q = reinterpret_cast<const uint4*>(p);
  uint4 a = __ldg(q), b = __ldg(q + 1);
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

// Record's args lie inside the pool and match the kernel's arity.
__device__ __forceinline__ bool args_in_range(const picker_rec_t& r, uint32_t nparams,
                                              uint64_t lo, uint64_t hi) {
  return r.nargs == nparams && r.arg_off >= lo && r.arg_off <= hi &&
         (uint64_t)r.nargs <= hi - r.arg_off;
}

// Code of a record whose kernel needs no evaluation (KbEntry.kn direct code):
// unknown ids, kernel-level classes after the arity / pool check.
__device__ __forceinline__ uint32_t direct_code(uint32_t kn, uint32_t nargs, uint64_t arg_off, uint64_t lo,
                                                uint64_t hi) {
  if (!(kn & kDirectArity)) return kn & 0xFFu;
  const bool ok = nargs == (kn >> 24) && arg_off >= lo && arg_off <= hi && (uint64_t)nargs <= hi - arg_off;
  return ok ? (kn & 0xFFu) : (uint32_t)V_ERR_ARITY;
}

// Operand values of one record.  `a` points at the record's own argument
// slots: global memory, or the CTA's shared-memory copy (generic pointer).
struct RecVals {
  int64_t d[6];
  const int64_t* a;
  const uint32_t* m;
  __device__ __forceinline__ RecVals(const picker_rec_t& r, const int64_t* rec_args,
                                     const uint32_t* i32mask)
      : a(rec_args), m(i32mask) {
    d[0] = r.grid_x, d[1] = r.grid_y, d[2] = r.grid_z;
    d[3] = r.block_x, d[4] = r.block_y, d[5] = r.block_z;
  }
  __device__ __forceinline__ int64_t get(uint8_t op) const {
    if (op < 6) return d[op];
    if (op == OPD_ONE) return 1;
    if (op == OPD_NONE) return 0;
    const int i = op - OPD_ARG0;
    int64_t v = a[i];
    if ((m[i >> 5] >> (i & 31)) & 1u) v = (int64_t)(int32_t)(uint32_t)v;
    return v;
  }
};

// CUDA launch limits as implicit preconditions (Q21).
__device__ __forceinline__ bool launch_limits_ok(const RecVals& X) {
  // grid.x <= 2^31-1, grid.y,z <= 65535, block.x,y <= 1024, block.z <= 64
  // (kDimMax); the header fields are unsigned, so only the lower bound and the
  // fields wider than their limit need a test.
  if (X.d[0] < 1 || X.d[0] > 2147483647LL || X.d[1] < 1 || X.d[2] < 1) return false;
  if (X.d[3] < 1 || X.d[3] > 1024 || X.d[4] < 1 || X.d[4] > 1024 || X.d[5] < 1 || X.d[5] > 64)
    return false;
  return X.d[3] * X.d[4] * X.d[5] <= kBlockMaxThreads;
}

// The same limits on the header fields in 32-bit arithmetic (unsigned
// wrap-around turns each two-sided range test into one compare).
// Branch-free (one predicate chain, no early exits); the product can wrap only
// when a factor is already out of range, which sets `bad` on its own.
__device__ __forceinline__ bool launch_limits_rec(const picker_rec_t& r) {
  const uint32_t gx = r.grid_x, gy = r.grid_y, gz = r.grid_z;
  const uint32_t bx = r.block_x, by = r.block_y, bz = r.block_z;
  const bool bad = (gx - 1u > 2147483646u) | (gy == 0u) | (gz == 0u) | (bx - 1u > 1023u) | (by - 1u > 1023u) |
                   (bz - 1u > 63u) | (bx * by * bz > (uint32_t)kBlockMaxThreads);
  return !bad;
}

__device__ __forceinline__ int count_bin(uint8_t code) { return code <= 11 ? code : 15; }

// The CTA's histogram s_hist (final; every thread of the CTA calls this) into
// the caller's counts.  slot == nullptr: atomic adds into counts (the caller
// zeroed them).  Otherwise the CTAs add into the launch's slot and the last
// CTA to finish (ticket) writes counts and leaves the slot zeroed for its
// next launch: no memset launch before the kernel.
__device__ __forceinline__ void flush_counts(const uint32_t* s_hist, unsigned long long* counts, CountSlot* slot) {
  const int tid = threadIdx.x;
  if (counts == nullptr) return;
  if (slot == nullptr) {
    if (tid < PICKER_NUM_COUNTS && s_hist[tid]) atomicAdd(counts + tid, (unsigned long long)s_hist[tid]);
    return;
  }
  __shared__ uint32_t s_last;
  if (tid < PICKER_NUM_COUNTS && s_hist[tid]) atomicAdd(&slot->acc[tid], (unsigned long long)s_hist[tid]);
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(&slot->ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (s_last) {
    __threadfence();
    if (tid < PICKER_NUM_COUNTS) counts[tid] = atomicExch(&slot->acc[tid], 0ull);
    if (tid == 0) atomicExch(&slot->ticket, 0u);
  }
}

// Epilogue: u8 code, ballot-packed idempotent bit, histogram.
// Lane 0 of each warp must hold a record index that is a multiple of 32.
__device__ __forceinline__ void emit(uint64_t i, bool valid, uint8_t code, uint8_t* flags,
                                     uint32_t* bits, unsigned int* hist) {
  const unsigned bal = __ballot_sync(0xffffffffu, valid && code <= V_IDEM_KERNEL);
  if (valid) {
    flags[i] = code;
    atomicAdd(hist + count_bin(code), 1u);
  }
  if (bits && (threadIdx.x & 31) == 0 && valid) bits[i >> 5] = bal;
}

}  // namespace picker
