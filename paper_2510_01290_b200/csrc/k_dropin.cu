// Batch-1 kernels behind the drop-in C++ API: the reference's
// own functions -- quantize_window (proj/src/quant.cpp:486-580),
// gqa_attend (attention.cpp:124-146), sparsity / layer_sparsity_average
// (:148-167) and decode_payload (pager.cpp:89-112) -- over caller-supplied
// fp64 vectors, with the reference's operation order so results carry its
// bits (this file is compiled with --fmad=false; exp is tkv_exp, glibc's).
//
// These are the same computations K1-K3 run on the paged device state; the
// drop-in adapters (paper_2510_01290_b200/dropin/) call them one pager /
// one window / one attention row at a time through tkv_dropin_* in
// include/thinkv_b200.h.
#include <cuda_runtime.h>
#include <math_constants.h>

#include "tkv_codec.cuh"
#include "tkv_exp.cuh"
#include "tkv_kernels.h"

namespace {

constexpr int kThreads = 256;


// quantize_window for n <= group_size tokens of dimension d (bits 2/4/8).
// keys: one group per channel over the n tokens (zero padding never changes
// the absmax, and padded codes are not returned); values: per token, chunks
// of group_size channels; FP8: one f32 scale per side = float(absmax / 448).
__global__ void __launch_bounds__(kThreads) window_quant_kernel(int n, int d, int fmt, int gsz, const double* __restrict__ K,
                                                                const double* __restrict__ V, uint8_t* kc, uint8_t* vc,
                                                                uint8_t* ksc, uint8_t* vsc, float* f8, int* bad) {
  __shared__ double red[2][kThreads / 32];
  bool b = false;
  for (int i = threadIdx.x; i < n * d; i += kThreads)
    if (!isfinite(K[i]) || !isfinite(V[i])) b = true;
  if (fmt == TKV_FMT_FP8) {
    double ak = 0.0, av = 0.0;
    for (int i = threadIdx.x; i < n * d; i += kThreads) {
      ak = fmax(ak, fabs(K[i]));
      av = fmax(av, fabs(V[i]));
    }
    for (int o = 16; o > 0; o >>= 1) {
      ak = fmax(ak, __shfl_xor_sync(0xffffffffu, ak, o));
      av = fmax(av, __shfl_xor_sync(0xffffffffu, av, o));
    }
    if ((threadIdx.x & 31) == 0) {
      red[0][threadIdx.x >> 5] = ak;
      red[1][threadIdx.x >> 5] = av;
    }
    __syncthreads();
    ak = av = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) {
      ak = fmax(ak, red[0][w]);
      av = fmax(av, red[1][w]);
    }
    const float kf = __double2float_rn(__ddiv_rn(ak, 448.0));  // fp8_tensor_scale (quant.cpp:176-178)
    const float vf = __double2float_rn(__ddiv_rn(av, 448.0));
    for (int i = threadIdx.x; i < n * d; i += kThreads) {
      kc[i] = kf > 0.0f ? tkv_e4m3_encode(__ddiv_rn(K[i], (double)kf), &b) : 0;
      vc[i] = vf > 0.0f ? tkv_e4m3_encode(__ddiv_rn(V[i], (double)vf), &b) : 0;
    }
    if (threadIdx.x == 0) {
      f8[0] = kf;
      f8[1] = vf;
    }
  } else {
    for (int ch = threadIdx.x; ch < d; ch += kThreads) {
      double am = 0.0;
      for (int t = 0; t < n; ++t) am = fmax(am, fabs(K[t * d + ch]));
      uint8_t sc;
      if (fmt == TKV_FMT_TERNARY) {  // ternary_group_encode (quant.cpp:141-158)
        sc = tkv_e4m3_encode(am, &b);
        const double delta = tkv_e4m3_decode(sc);
        for (int t = 0; t < n; ++t)
          kc[t * d + ch] = delta > 0.0 ? tkv_ternary_bits((int)fmin(fmax(rint(__ddiv_rn(K[t * d + ch], delta)), -1.0), 1.0)) : 0;
      } else {  // nvfp4_group_encode (quant.cpp:160-174)
        sc = tkv_e4m3_encode(__ddiv_rn(am, 6.0), &b);
        const double s = tkv_e4m3_decode(sc);
        for (int t = 0; t < n; ++t) kc[t * d + ch] = s > 0.0 ? tkv_nvfp4_encode(__ddiv_rn(K[t * d + ch], s)) : 0;
      }
      ksc[ch] = sc;
    }
    const int chunks = (d + gsz - 1) / gsz;
    for (int it = threadIdx.x; it < n * chunks; it += kThreads) {
      const int t = it / chunks, j = it % chunks;
      const int base = j * gsz, len = min(gsz, d - base);
      double am = 0.0;
      for (int q = 0; q < len; ++q) am = fmax(am, fabs(V[t * d + base + q]));
      uint8_t sc;
      if (fmt == TKV_FMT_TERNARY) {
        sc = tkv_e4m3_encode(am, &b);
        const double delta = tkv_e4m3_decode(sc);
        for (int q = 0; q < len; ++q)
          vc[t * d + base + q] =
              delta > 0.0 ? tkv_ternary_bits((int)fmin(fmax(rint(__ddiv_rn(V[t * d + base + q], delta)), -1.0), 1.0)) : 0;
      } else {
        sc = tkv_e4m3_encode(__ddiv_rn(am, 6.0), &b);
        const double s = tkv_e4m3_decode(sc);
        for (int q = 0; q < len; ++q) vc[t * d + base + q] = s > 0.0 ? tkv_nvfp4_encode(__ddiv_rn(V[t * d + base + q], s)) : 0;
      }
      vsc[t * chunks + j] = sc;
    }
  }
  if (b) atomicExch(bad, 1);
}

// gqa_attend (attention.cpp:124-138): G query rows over n keys/values.
//   logit[g][i] = (sum_c q[g][c] * k[i][c], channel order) * scale
//   pooled[i]   = std::max over rows in row order (gqa_aggregate :110-122)
//   s_i = exp(pooled_i - max) / sum (softmax_row :54-67; sum in index order)
//   out[c] = sum_i s_i * v[i][c] in index order (weighted_values :71-78)
// One CTA; the two order-sensitive sums are sequential chains (one thread
// for the denominator, one thread per channel for the output).
__global__ void __launch_bounds__(kThreads) gqa_attend_f64_kernel(int G, int n, int d, double scale,
                                                                  const double* __restrict__ Q,
                                                                  const double* __restrict__ K,
                                                                  const double* __restrict__ V, double* out,
                                                                  double* row) {
  __shared__ double sh_max, sh_sum;
  for (int i = threadIdx.x; i < n; i += kThreads) {
    double pooled = 0.0;
    for (int g = 0; g < G; ++g) {
      double dot = 0.0;
      for (int c = 0; c < d; ++c) dot = __dadd_rn(dot, __dmul_rn(Q[g * d + c], K[(int64_t)i * d + c]));
      const double l = __dmul_rn(dot, scale);
      pooled = g == 0 ? l : (pooled < l ? l : pooled);  // std::max(pooled, l)
    }
    row[i] = pooled;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // *std::max_element: first maximum (value only)
    double m = row[0];
    for (int i = 1; i < n; ++i)
      if (m < row[i]) m = row[i];
    sh_max = m;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += kThreads) row[i] = tkv_exp(__dsub_rn(row[i], sh_max));
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s = __dadd_rn(s, row[i]);
    sh_sum = s;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += kThreads) row[i] = __ddiv_rn(row[i], sh_sum);
  __syncthreads();
  for (int c = threadIdx.x; c < d; c += kThreads) {
    double acc = 0.0;
    for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, __dmul_rn(row[i], V[(int64_t)i * d + c]));
    out[c] = acc;
  }
}

// sparsity (attention.cpp:148-158) of each row: count(s < frac * max) / n,
// strict; one warp per row.
__global__ void sparsity_rows_kernel(const double* __restrict__ S, const int64_t* __restrict__ offs, int nrows,
                                     double frac, double* out) {
  const int r = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (r >= nrows) return;
  const int64_t b = offs[r], e = offs[r + 1];
  double m = -CUDART_INF;
  for (int64_t i = b + lane; i < e; i += 32) m = fmax(m, S[i]);
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  const double thr = __dmul_rn(frac, m);
  long long below = 0;
  for (int64_t i = b + lane; i < e; i += 32) below += S[i] < thr;
  for (int o = 16; o > 0; o >>= 1) below += __shfl_xor_sync(0xffffffffu, below, o);
  if (lane == 0) out[r] = __ddiv_rn((double)below, (double)(e - b));
}

// decode_code (quant.cpp:195-205) elementwise: out[i] = code_value * scale[i].
__global__ void decode_codes_kernel(int fmt, int64_t n, const uint8_t* __restrict__ codes,
                                    const double* __restrict__ scales, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = tkv_decode_code(fmt, codes[i], scales[i]);
}

}  // namespace

cudaError_t tkv_launch_window_quant(int n, int d, int fmt, int group_size, const double* keys, const double* values,
                                    uint8_t* kc, uint8_t* vc, uint8_t* ksc, uint8_t* vsc, float* f8, int* bad,
                                    cudaStream_t stream) {
  window_quant_kernel<<<1, kThreads, 0, stream>>>(n, d, fmt, group_size, keys, values, kc, vc, ksc, vsc, f8, bad);
  return cudaGetLastError();
}

cudaError_t tkv_launch_gqa_attend_f64(int G, int n, int d, double scale, const double* q, const double* k,
                                      const double* v, double* out, double* row, cudaStream_t stream) {
  gqa_attend_f64_kernel<<<1, kThreads, 0, stream>>>(G, n, d, scale, q, k, v, out, row);
  return cudaGetLastError();
}

cudaError_t tkv_launch_sparsity_rows(const double* scores, const int64_t* offs, int nrows, double frac, double* out,
                                     cudaStream_t stream) {
  if (nrows <= 0) return cudaSuccess;
  sparsity_rows_kernel<<<(nrows + 7) / 8, 256, 0, stream>>>(scores, offs, nrows, frac, out);
  return cudaGetLastError();
}

cudaError_t tkv_launch_decode_codes(int fmt, int64_t n, const uint8_t* codes, const double* scales, double* out,
                                    cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const int blocks = (int)((n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024);
  decode_codes_kernel<<<blocks, 256, 0, stream>>>(fmt, n, codes, scales, out);
  return cudaGetLastError();
}
