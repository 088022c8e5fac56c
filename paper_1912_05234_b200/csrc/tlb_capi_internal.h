// tlb_capi_internal.h -- error plumbing shared by the C-ABI translation units.
#pragma once

#include <string>

namespace tlb {

// Records `msg` as the calling thread's last error and returns `code` (tlb_last_error()).
int fail(int code, const std::string& msg);

}  // namespace tlb
