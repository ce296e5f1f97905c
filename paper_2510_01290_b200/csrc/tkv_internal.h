// Definitions shared by the library's host translation units (tkv_host.cpp,
// tkv_dropin.cpp); not part of the C ABI.
#pragma once
#include <string>

struct tkv_ctx {
  int device = 0;
};

// Sets tkv_last_error() of the calling thread.
void tkv_internal_set_error(const std::string& msg);
