// C ABI of the drop-in batch-1 calls (include/thinkv_b200.h, "drop-in"
// section): the entry points the C++ adapters behind the reference's
// unchanged headers (paper_2510_01290_b200/dropin/) use for every decision
// and every value -- window quantization, payload decoding, slot placement
// and release, K-means medoids, attention and sparsity -- each one kernel
// launch over host arrays copied in and out.
//
// Calls are synchronous and reentrant: each thread owns its device staging
// buffer and runs on its per-thread default stream, so concurrent callers
// (the reference runs independent simulations on worker threads,
// cli.cpp:283-303) never serialise on each other.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/thinkv_b200.h"
#include "tkv_internal.h"
#include "tkv_kernels.h"
#include "tkv_state.h"

namespace {

struct DropinError : std::runtime_error {
  int code;
  DropinError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw DropinError(TKV_ERR_UNEXPECTED, std::string(what) + ": " + cudaGetErrorString(e));
}

// Per-thread device staging: one growable buffer carved into 256-B aligned pieces.
struct Staging {
  uint8_t* base = nullptr;
  size_t cap = 0, used = 0;
  int device = -1;
  ~Staging() {
    if (base) cudaFree(base);
  }
};
thread_local Staging t_stage;

class Call {
 public:
  explicit Call(tkv_ctx* ctx) {
    if (!ctx) throw DropinError(TKV_ERR_CONFIG, "null context");
    cuda_ok(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (t_stage.device != ctx->device && t_stage.base) {
      cudaFree(t_stage.base);
      t_stage.base = nullptr;
      t_stage.cap = 0;
    }
    t_stage.device = ctx->device;
    t_stage.used = 0;
  }
  // Reserve device bytes for this call (before any upload: may reallocate).
  void reserve(size_t bytes) {
    if (bytes <= t_stage.cap) return;
    if (t_stage.base) cuda_ok(cudaFree(t_stage.base), "cudaFree");
    t_stage.base = nullptr;
    const size_t cap = std::max<size_t>(bytes, 1 << 20);
    cuda_ok(cudaMalloc(&t_stage.base, cap), "cudaMalloc");
    t_stage.cap = cap;
  }
  template <typename T>
  T* take(size_t n) {
    const size_t off = (t_stage.used + 255) & ~size_t(255);
    const size_t bytes = std::max<size_t>(n * sizeof(T), 1);
    if (off + bytes > t_stage.cap) throw DropinError(TKV_ERR_UNEXPECTED, "drop-in staging overflow");
    t_stage.used = off + bytes;
    return reinterpret_cast<T*>(t_stage.base + off);
  }
  template <typename T>
  T* up(const T* host, size_t n) {
    T* d = take<T>(n);
    if (n) cuda_ok(cudaMemcpyAsync(d, host, n * sizeof(T), cudaMemcpyHostToDevice, cudaStreamPerThread), "upload");
    return d;
  }
  template <typename T>
  void down(T* host, const T* dev, size_t n) {
    if (n) cuda_ok(cudaMemcpyAsync(host, dev, n * sizeof(T), cudaMemcpyDeviceToHost, cudaStreamPerThread), "download");
  }
  void launched(cudaError_t e, const char* what) { cuda_ok(e, what); }
  void sync() { cuda_ok(cudaStreamSynchronize(cudaStreamPerThread), "synchronize"); }
  static size_t pad(size_t bytes) { return (bytes + 255) & ~size_t(255); }
};

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return TKV_OK;
  } catch (const DropinError& e) {
    tkv_internal_set_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    tkv_internal_set_error(e.what());
    return TKV_ERR_UNEXPECTED;
  }
}

int fmt_of_bits(int bits) {
  switch (bits) {
    case 2: return TKV_FMT_TERNARY;
    case 4: return TKV_FMT_NVFP4;
    case 8: return TKV_FMT_FP8;
  }
  throw DropinError(TKV_ERR_CONFIG, "no quantized storage format for " + std::to_string(bits) + " bits");
}

}  // namespace

extern "C" {

int tkv_dropin_quantize_window(tkv_ctx* ctx, int32_t n, int32_t d, int32_t bits, int32_t group_size,
                               const double* keys, const double* values, uint8_t* key_codes, uint8_t* value_codes,
                               uint8_t* key_scales, uint8_t* value_scales, float* fp8_scales) {
  return guarded([&] {
    if (n < 1 || d < 1 || group_size < 1 || n > group_size) throw DropinError(TKV_ERR_CONFIG, "bad window shape");
    const int fmt = fmt_of_bits(bits);
    const size_t nd = (size_t)n * d, chunks = (size_t)(d + group_size - 1) / group_size;
    Call c(ctx);
    c.reserve(Call::pad(nd * 8) * 2 + Call::pad(nd) * 2 + Call::pad(d) + Call::pad((size_t)n * chunks) + 1024);
    const double* dk = c.up(keys, nd);
    const double* dv = c.up(values, nd);
    uint8_t* kc = c.take<uint8_t>(nd);
    uint8_t* vc = c.take<uint8_t>(nd);
    uint8_t* ksc = c.take<uint8_t>(d);
    uint8_t* vsc = c.take<uint8_t>((size_t)n * chunks);
    float* f8 = c.take<float>(2);
    int* bad = c.take<int>(1);
    cuda_ok(cudaMemsetAsync(bad, 0, sizeof(int), cudaStreamPerThread), "memset");
    c.launched(tkv_launch_window_quant(n, d, fmt, group_size, dk, dv, kc, vc, ksc, vsc, f8, bad, cudaStreamPerThread),
               "window quant kernel");
    int hbad = 0;
    c.down(&hbad, bad, 1);
    c.down(key_codes, kc, nd);
    c.down(value_codes, vc, nd);
    if (fmt == TKV_FMT_FP8) {
      c.down(fp8_scales, f8, 2);
    } else {
      c.down(key_scales, ksc, d);
      c.down(value_scales, vsc, (size_t)n * chunks);
    }
    c.sync();
    if (hbad) throw DropinError(TKV_ERR_CONFIG, "quantize_window: non-finite input");
  });
}

int tkv_dropin_decode(tkv_ctx* ctx, int32_t fmt, int64_t n, const uint8_t* codes, const double* scales, double* out) {
  return guarded([&] {
    if (fmt < TKV_FMT_TERNARY || fmt > TKV_FMT_FP8) throw DropinError(TKV_ERR_CONFIG, "bad code format");
    Call c(ctx);
    c.reserve(Call::pad(n) + 2 * Call::pad(n * 8) + 512);
    const uint8_t* dc = c.up(codes, n);
    const double* ds = c.up(scales, n);
    double* dout = c.take<double>(n);
    c.launched(tkv_launch_decode_codes(fmt, n, dc, ds, dout, cudaStreamPerThread), "decode kernel");
    c.down(out, dout, n);
    c.sync();
  });
}

int tkv_dropin_gqa_attend(tkv_ctx* ctx, int32_t G, int64_t n, int32_t d, double scale, const double* q,
                          const double* keys, const double* values, double* out, double* row) {
  return guarded([&] {
    if (G < 1 || n < 1 || d < 1) throw DropinError(TKV_ERR_CONFIG, "bad attention shape");
    const size_t nd = (size_t)n * d;
    Call c(ctx);
    c.reserve(Call::pad((size_t)G * d * 8) + 2 * Call::pad(nd * 8) + Call::pad(d * 8) + Call::pad(n * 8) + 1024);
    const double* dq = c.up(q, (size_t)G * d);
    const double* dk = c.up(keys, nd);
    const double* dv = c.up(values, nd);
    double* dout = c.take<double>(d);
    double* drow = c.take<double>(n);
    c.launched(tkv_launch_gqa_attend_f64(G, (int)n, d, scale, dq, dk, dv, dout, drow, cudaStreamPerThread),
               "attention kernel");
    c.down(out, dout, d);
    c.down(row, drow, n);
    c.sync();
  });
}

int tkv_dropin_sparsity(tkv_ctx* ctx, const double* scores, const int64_t* offsets, int32_t nrows, double frac,
                        double* out) {
  return guarded([&] {
    if (nrows < 1) throw DropinError(TKV_ERR_CONFIG, "no rows");
    const int64_t total = offsets[nrows];
    for (int r = 0; r < nrows; ++r)
      if (offsets[r + 1] <= offsets[r]) throw DropinError(TKV_ERR_CONFIG, "sparsity of an empty row");
    Call c(ctx);
    c.reserve(Call::pad(total * 8) + Call::pad((nrows + 1) * 8) + Call::pad(nrows * 8) + 512);
    const double* ds = c.up(scores, total);
    const int64_t* doffs = c.up(offsets, (size_t)nrows + 1);
    double* dout = c.take<double>(nrows);
    c.launched(tkv_launch_sparsity_rows(ds, doffs, nrows, frac, dout, cudaStreamPerThread), "sparsity kernel");
    c.down(out, dout, nrows);
    c.sync();
  });
}

int tkv_dropin_kmeans_select(tkv_ctx* ctx, int32_t ninst, int32_t d, const int32_t* m, const int32_t* k,
                             const double* keys, int32_t* medoids) {
  return guarded([&] {
    if (ninst < 1 || d < 1) throw DropinError(TKV_ERR_CONFIG, "kmeans over an empty input");
    std::vector<int64_t> xoff(ninst), ooff(ninst);
    int64_t xs = 0, os = 0;
    for (int i = 0; i < ninst; ++i) {
      if (m[i] < 1 || k[i] < 1) throw DropinError(TKV_ERR_CONFIG, "kmeans over an empty input");
      if (k[i] >= m[i]) throw DropinError(TKV_ERR_CONFIG, "kmeans_select needs k < m (nothing to select otherwise)");
      if (m[i] > 256) throw DropinError(TKV_ERR_CONFIG, "kmeans_select: segments of more than 256 members unsupported");
      xoff[i] = xs;
      ooff[i] = os;
      xs += (int64_t)m[i] * d;
      os += k[i];
    }
    Call c(ctx);
    c.reserve(Call::pad(xs * 8) * 6 + Call::pad(os * 4) + 4 * Call::pad(ninst * 8) + 2048);
    const double* dx = c.up(keys, xs);
    const int32_t* dm = c.up(m, ninst);
    const int32_t* dk = c.up(k, ninst);
    const int64_t* dxo = c.up(xoff.data(), ninst);
    const int64_t* doo = c.up(ooff.data(), ninst);
    double* scratch = c.take<double>(5 * xs);
    int32_t* dout = c.take<int32_t>(os);
    c.launched(tkv_launch_kmeans_select_f64(ninst, dx, dm, dk, dxo, doo, d, scratch, dout, cudaStreamPerThread),
               "kmeans kernel");
    c.down(medoids, dout, os);
    c.sync();
  });
}

int tkv_dropin_pager_place(tkv_ctx* ctx, int32_t P, int32_t bs, int8_t* thought, uint8_t* filled, uint32_t* evict,
                           uint8_t* nstart, int32_t* starts, uint32_t* masks, int32_t* nfree, int32_t band,
                           int32_t seg_start, int32_t n, int32_t* claims, int8_t* reused) {
  return guarded([&] {
    if (P < 1 || bs < 1 || bs > 32 || n < 1) throw DropinError(TKV_ERR_CONFIG, "bad pager shape");
    const size_t ns = (size_t)P * TKV_STARTS_PER_BLOCK(bs), nm = (size_t)P * TKV_MASKS_PER_BLOCK(bs);
    Call c(ctx);
    c.reserve(Call::pad(P) * 3 + Call::pad(P * 4) + Call::pad(ns * 4) + Call::pad(nm * 4) + Call::pad(n * 4) +
              Call::pad(n) + 2048);
    int8_t* dth = c.up(thought, P);
    uint8_t* dfl = c.up(filled, P);
    uint32_t* dev = c.up(evict, P);
    uint8_t* dns = c.up(nstart, P);
    int32_t* dst = c.up(starts, ns);
    uint32_t* dm = c.up(masks, nm);
    int32_t* dnf = c.up(nfree, 1);
    int32_t* dcl = c.take<int32_t>(n);
    int8_t* dre = c.take<int8_t>(n);
    int32_t* drc = c.take<int32_t>(1);
    c.launched(tkv_launch_pager_place(P, bs, dth, dfl, dev, dns, dst, dm, dnf, band, seg_start, n, dcl, dre, drc,
                                      cudaStreamPerThread),
               "placement kernel");
    int32_t rc = 0;
    c.down(&rc, drc, 1);
    c.sync();
    if (rc != 0) throw DropinError(TKV_ERR_OOM, "physical block pool exhausted");
    c.down(thought, dth, P);
    c.down(filled, dfl, P);
    c.down(evict, dev, P);
    c.down(nstart, dns, P);
    c.down(starts, dst, ns);
    c.down(masks, dm, nm);
    c.down(nfree, dnf, 1);
    c.down(claims, dcl, n);
    c.down(reused, dre, n);
    c.sync();
  });
}

int tkv_dropin_pager_evict(tkv_ctx* ctx, int32_t P, int32_t bs, int8_t* thought, uint8_t* filled, uint32_t* evict,
                           uint8_t* nstart, int32_t n, const int32_t* slots, int32_t* freed, int32_t* nfreed) {
  return guarded([&] {
    if (P < 1 || bs < 1 || bs > 32 || n < 0) throw DropinError(TKV_ERR_CONFIG, "bad pager shape");
    Call c(ctx);
    c.reserve(Call::pad(P) * 3 + Call::pad(P * 4) * 2 + Call::pad(n * 4) + 1024);
    int8_t* dth = c.up(thought, P);
    uint8_t* dfl = c.up(filled, P);
    uint32_t* dev = c.up(evict, P);
    uint8_t* dns = c.up(nstart, P);
    const int32_t* dsl = c.up(slots, n);
    int32_t* dfr = c.take<int32_t>(P);
    int32_t* dnf = c.take<int32_t>(1);
    c.launched(tkv_launch_pager_evict(P, bs, dth, dfl, dev, dns, n, dsl, dfr, dnf, cudaStreamPerThread),
               "eviction kernel");
    c.down(nfreed, dnf, 1);
    c.down(thought, dth, P);
    c.down(filled, dfl, P);
    c.down(evict, dev, P);
    c.down(nstart, dns, P);
    c.sync();
    c.down(freed, dfr, *nfreed);
    c.sync();
  });
}

}  // extern "C"
