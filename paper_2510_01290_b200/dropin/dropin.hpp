// Shared plumbing of the drop-in adapters: the reference's public C++ API
// (proj/include/thinkv/*.hpp, compiled unchanged against these sources)
// implemented over the library's C ABI (include/thinkv_b200.h, "drop-in"
// section).  Every decision and every value the hot-path functions return
// comes from a CUDA kernel; the C++ objects hold the host-side mirrors the
// API's return types need (BlockPager hands out pointers to host payloads).
#pragma once
#include <string>

#include "thinkv/errors.hpp"
#include "thinkv_b200.h"

namespace thinkv::dropin {

// The device context the adapters run on: $TKV_DEVICE (default 0), created
// on first use and shared by every thread (calls carry their own staging).
tkv_ctx* ctx();

// Status of a tkv_* call -> the reference's exception: OOM and integrity map
// to their kinds, anything else to `fallback` (the kind the reference throws
// for that precondition).
void check(int status, ErrorKind fallback = ErrorKind::kStructural);

}  // namespace thinkv::dropin
