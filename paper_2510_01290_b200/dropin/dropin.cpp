#include "dropin.hpp"

#include <cstdlib>
#include <mutex>

namespace thinkv::dropin {

tkv_ctx* ctx() {
  static std::once_flag once;
  static tkv_ctx* c = nullptr;
  std::call_once(once, [] {
    const char* env = std::getenv("TKV_DEVICE");
    const int device = env ? std::atoi(env) : 0;
    check(tkv_init(device, &c), ErrorKind::kConfig);
  });
  return c;
}

void check(int status, ErrorKind fallback) {
  if (status == TKV_OK) return;
  const std::string msg = tkv_last_error();
  switch (status) {
    case TKV_ERR_OOM: throw Error(ErrorKind::kOutOfMemory, msg);
    case TKV_ERR_INTEGRITY: throw Error(ErrorKind::kIntegrity, msg);
    case TKV_ERR_CALIBRATION: throw Error(ErrorKind::kCalibration, msg);
    case TKV_ERR_CONFIG: throw Error(fallback, msg);
    default: throw std::runtime_error("thinkv_b200: " + msg);
  }
}

}  // namespace thinkv::dropin
