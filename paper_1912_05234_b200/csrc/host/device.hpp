// device.hpp -- the process-wide device context behind the tloom:: C++ API.
//
// tloom::nn / tloom::net calls are synchronous and thread-safe in the reference (SPEC: pure functions);
// here every call locks the shared tlb_ctx (device TLOOM_B200_DEVICE, default 0; mode TLOOM_B200_MODE
// = exact|fast, default exact) and forwards to the C ABI.
#pragma once

#include <mutex>

#include "tloom_b200.h"

namespace tloom::detail {

struct DeviceLock {
  std::unique_lock<std::mutex> lock;
  tlb_ctx* ctx;
};

// Creates the context on first use; throws tloom::Error if no B200 is available.
DeviceLock device();

// Throws the tloom exception matching a TLB_ERR_* status (with tlb_last_error()).
void check(int status);

}  // namespace tloom::detail
