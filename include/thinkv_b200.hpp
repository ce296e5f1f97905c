// thinkv_b200.hpp -- C++ host side of the B200 ThinKV decode path.
//
// Header-only RAII layer over the C ABI (thinkv_b200.h) for C++ callers --
// the reference itself is C++20 (proj/include/thinkv/*.hpp).  It mirrors the
// reference's per-step interface and error behaviour:
//
//   reference                                        here
//   -----------------------------------------------  -------------------------------------
//   thinkv::Error{ErrorKind}.exit_code()             thinkv_b200::Error::exit_code()
//     (proj/include/thinkv/errors.hpp:13-49)           (same numbers: 2 config, 4 OOM, 5 integrity)
//   ThinkvMethod(const SimConfig&)  sim.cpp:494-508  DecodeRun(const tkv_run_desc&, device)
//   ThinkvMethod::process(sv)       sim.cpp:748-843  DecodeRun::process(q, k, v, out, stream)
//                                                      DecodeRun::process_layer(l, L, ...) per layer
//   ThinkvMethod::finish()          sim.cpp:871-958  DecodeRun::finish()
//   RunOutput::final_block_tables / final_segments   DecodeRun::dump("tables" | "segments" |
//     / events_jsonl / metrics / step_dumps             "events" | "metrics" | "step_dumps", seq)
//
// Device buffers are caller-owned and must stay valid until the stream
// completes (the C ABI contract).  No exceptions cross the C ABI; this layer
// turns status codes back into exceptions, like the reference's API.
#pragma once

#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "thinkv_b200.h"

namespace thinkv_b200 {

class Error : public std::runtime_error {
 public:
  Error(int code, const std::string& what) : std::runtime_error(what), code_(code) {}
  // thinkv::Error::exit_code() numbering (errors.hpp:31-46).
  int exit_code() const noexcept { return code_; }

 private:
  int code_;
};

inline void check(int rc) {
  if (rc != TKV_OK) throw Error(rc, tkv_last_error());
}

class Context {
 public:
  explicit Context(int device = 0) { check(tkv_init(device, &h_)); }
  ~Context() {
    if (h_) tkv_ctx_destroy(h_);
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  tkv_ctx* get() const noexcept { return h_; }

 private:
  tkv_ctx* h_ = nullptr;
};

class DecodeRun {
 public:
  DecodeRun(Context& ctx, const tkv_run_desc& desc) { check(tkv_run_create(ctx.get(), &desc, &h_)); }
  ~DecodeRun() {
    if (h_) tkv_run_destroy(h_);
  }
  DecodeRun(const DecodeRun&) = delete;
  DecodeRun& operator=(const DecodeRun&) = delete;
  DecodeRun(DecodeRun&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}

  // One decode step for every unit; device pointers, asynchronous on `stream`.
  void process(const void* q, const void* k, const void* v, float* out, void* stream = nullptr) {
    check(tkv_step(h_, q, k, v, out, stream));
  }
  // One layer of a step for a model's decode loop (layers 0 .. num_layers-1 in order).
  void process_layer(int layer, int num_layers, const void* q, const void* k, const void* v, float* out,
                     void* stream = nullptr) {
    check(tkv_step_layer(h_, layer, num_layers, q, k, v, out, stream));
  }
  // Same with host buffers (synchronous).
  void process_host(const void* q, const void* k, const void* v, float* out) {
    check(tkv_step_host(h_, q, k, v, out));
  }
  // Pipelined host-buffer step: buffers stay owned by the run until synchronize().
  void process_host_async(const void* q, const void* k, const void* v, float* out) {
    check(tkv_step_host_async(h_, q, k, v, out));
  }
  void finish() { check(tkv_finish(h_)); }
  void synchronize() { check(tkv_synchronize(h_)); }
  int64_t position() const { return tkv_position(h_); }

  // JSON views in the reference's own formats.
  std::string dump(const char* what, int seq = 0) {
    size_t need = 0;
    check(tkv_dump_json(h_, seq, what, nullptr, 0, &need));
    std::string s(need, '\0');
    check(tkv_dump_json(h_, seq, what, s.data(), s.size(), &need));
    s.resize(need ? need - 1 : 0);
    return s;
  }
  tkv_bytes_t bytes() {
    tkv_bytes_t b{};
    check(tkv_bytes(h_, &b));
    return b;
  }
  tkv_run* get() const noexcept { return h_; }

 private:
  tkv_run* h_ = nullptr;
};

}  // namespace thinkv_b200
