// Host-visible layout of the resident validator's mailboxes (k_serve.cuh).
#pragma once

#ifndef PICKER_NO_LIBC_HEADERS
#include <cstdint>
#endif

#include "../../include/picker.h"

namespace picker {

constexpr uint32_t kServeMax = 32;        // records per request (one lane each)
constexpr uint32_t kServeArgs = 64 * 32;  // argument slots per request

struct alignas(16) ServeRequest {
  volatile uint32_t seq;   // written last by the host
  volatile uint32_t stop;  // 1: the validator exits
  uint32_t n;              // records in this request
  uint32_t nargs;          // argument slots used
  picker_rec_t rec[kServeMax];  // arg_off relative to args[]
  int64_t args[kServeArgs];
};
struct alignas(16) ServeResponse {
  volatile uint32_t seq;  // written last by the GPU
  uint32_t pad[3];
  uint8_t codes[kServeMax];
};

}  // namespace picker
