// Resident validator: the paper's per-launch use ("validates ...
// before launching", under 5 us on the CPU) without a kernel launch per check.
//
// One warp stays resident on the GPU and polls a request mailbox in mapped,
// pinned host memory.  The host writes up to kServeMax launch records and their
// argument slots, then bumps the request sequence number; the warp sees it,
// copies the request into shared memory with one round of parallel 16-byte
// loads over PCIe, evaluates each record with the specialised module's code
// (one lane per record, the same dispatch as the batched kernels), writes the
// codes and then the response sequence number back to host memory.  The host
// spins on that number.  One SM is given up for as long as the validator runs
// (picker_serve_start / picker_serve_stop).
#pragma once

#include "k_bucket.cuh"
#include "serve.hpp"

namespace picker {

template <class Dispatch>
__global__ void __launch_bounds__(32, 1) k_serve(const __grid_constant__ BucketParams P, ServeRequest* req,
                                                 ServeResponse* resp) {
  __shared__ __align__(16) picker_rec_t s_rec[kServeMax];
  __shared__ __align__(16) int64_t s_args[kServeArgs];
  const int lane = threadIdx.x;
  uint32_t seen = req->seq;
  for (;;) {
    uint32_t cur = 0, stop = 0;
    if (lane == 0) {
      do {
        cur = req->seq;
        stop = req->stop;
      } while (cur == seen && !stop);
    }
    cur = __shfl_sync(0xffffffffu, cur, 0);
    stop = __shfl_sync(0xffffffffu, stop, 0);
    if (stop) return;
    seen = cur;
    __threadfence_system();  // acquire: the request body after its sequence number
    const uint32_t n = min(req->n, kServeMax), na = min(req->nargs, kServeArgs);
    // the request into shared memory: 16-byte loads, every lane in flight
    const uint4* src_r = reinterpret_cast<const uint4*>(req->rec);
    uint4* dst_r = reinterpret_cast<uint4*>(s_rec);
    for (uint32_t c = lane; c < 2 * n; c += 32) dst_r[c] = src_r[c];
    const uint4* src_a = reinterpret_cast<const uint4*>(req->args);
    uint4* dst_a = reinterpret_cast<uint4*>(s_args);
    for (uint32_t c = lane; c < (na + 1) / 2; c += 32) dst_a[c] = src_a[c];
    __syncwarp();
    const DevBatch B{s_rec, s_args, 0, na};
    uint8_t code = 0;
    if ((uint32_t)lane < n) {
      const picker_rec_t r = s_rec[lane];
      uint32_t kb = P.kb_unknown, kn = V_ERR_KERNEL;
      if (r.kernel_id < P.T.nkernel_slots) {
        const uint2 v = __ldg(reinterpret_cast<const uint2*>(P.kb_of) + r.kernel_id);
        kb = v.x, kn = v.y;
      }
      const uint32_t key = kb >> 16;
      if (key == P.direct_key)
        code = (uint8_t)direct_code(kn, r.nargs, r.arg_off, 0, na);
      else if (kWidePath && key == P.wide_key)
        code = 0xFD;  // decided below, warp-cooperatively
      else
        code = Dispatch::eval(key, kb & 0xFFFFu, kn, false, P, r, s_args + r.arg_off, B);
    }
    if (kWidePath)  // K2 records: the whole warp on one record at a time (register path only)
      for (unsigned wm = __ballot_sync(0xffffffffu, code == 0xFD && (uint32_t)lane < n); wm; wm &= wm - 1) {
        const uint32_t q = (uint32_t)__ffs(wm) - 1;
        const picker_rec_t rr = s_rec[q];
        const uint8_t cw = eval_wide_warp(P.T, rr, s_args + rr.arg_off, 0, na, lane, nullptr, 0);
        if ((uint32_t)lane == q) code = cw;
      }
    if ((uint32_t)lane < n) resp->codes[lane] = code;
    __threadfence_system();  // release: the codes before the sequence number
    __syncwarp();
    if (lane == 0) resp->seq = cur;
  }
}

}  // namespace picker
