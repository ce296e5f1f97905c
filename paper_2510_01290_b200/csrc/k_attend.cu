// K1 (SIMT variant): paged mixed-precision decode attention for the shapes
// the tensor-core kernel (k_attend_mma.cu) does not cover -- fp32/fp64
// inputs, head dims other than 64/128, G > 8.
//
// Reference semantics (what one unit computes per step):
//   live view = pager slots in physical (block, slot) order (BlockPager::
//   read_active, proj/src/pager.cpp:261-271) + the fp buffer + the incoming
//   token at full precision (sim.cpp:546-563, 762-765); then gqa_attend
//   (attention.cpp:124-138): logits q.k * 1/sqrt(d), per-head rows or the
//   element-wise max over the G rows (gqa_aggregate, :110-122), softmax,
//   probability-weighted values.
//
// K1 computes the outputs in fp32 with dequantisation fused into the
// QK^T / online-softmax / PV loop: codes are expanded in registers against the
// per-window key scales and per-token value-chunk scales, so no decoded copy
// of the cache is ever materialised.  Dead (soft-evicted) and unfilled slots
// are skipped at slot granularity through a per-CTA compacted live list that
// is grouped by storage format, so every 32-token tile is format-uniform.
//
// The fp64 sparsity statistics (K3a) live in k_score.cu.
#include <cuda_runtime.h>
#include <math_constants.h>

#include "tkv_codec.cuh"
#include "tkv_kernels.h"
#include "tkv_state.h"

namespace {

constexpr int kThreads = 128;
constexpr int kWarps = kThreads / 32;
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ float in_f(const void* p, int dtype, int64_t i) {
  if (dtype == TKV_IN_BF16) return __uint_as_float(((uint32_t) reinterpret_cast<const uint16_t*>(p)[i]) << 16);
  if (dtype == TKV_IN_F32) return reinterpret_cast<const float*>(p)[i];
  return (float)reinterpret_cast<const double*>(p)[i];
}
__device__ __forceinline__ double in_d(const void* p, int dtype, int64_t i) {
  if (dtype == TKV_IN_BF16) return (double)__uint_as_float(((uint32_t) reinterpret_cast<const uint16_t*>(p)[i]) << 16);
  if (dtype == TKV_IN_F32) return (double)reinterpret_cast<const float*>(p)[i];
  return reinterpret_cast<const double*>(p)[i];
}

// Exact fp32 decodes (every value is representable).
__device__ __forceinline__ float e4m3_f(uint32_t c) {
  const uint32_t e = (c >> 3) & 15u, m = c & 7u;
  float v = e == 0 ? (float)m * 0.001953125f : __uint_as_float(((e + 120u) << 23) | (m << 20));
  return (c & 0x80u) ? -v : v;
}
__device__ __forceinline__ float fp4_f(uint32_t c) {
  const uint32_t e = (c >> 1) & 3u, m = c & 1u;
  float v = e == 0 ? 0.5f * (float)m : __uint_as_float(((e + 126u) << 23) | (m << 22));
  return (c & 8u) ? -v : v;
}
__device__ __forceinline__ float tern_f(uint32_t c) {
  c &= 3u;
  return c == 1u ? 1.0f : (c == 3u ? -1.0f : 0.0f);
}

__device__ __forceinline__ float warp_max(float v) {
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Build the per-format compacted list of live slot indices (physical order
// within each format).  Returns counts in cnt[4]; list holds format f's slots
// at [off[f], off[f] + cnt[f]).
__device__ void build_live_list(const TkvState& st, int u, int* list, int* cnt, int* off, int* scan) {
  const TkvDims& dm = st.dm;
  const int P = dm.P, bs = dm.bs;
  const int8_t* th = st.blk_thought + (int64_t)u * P;
  const uint8_t* fl = st.blk_filled + (int64_t)u * P;
  const uint32_t* ev = st.blk_evict + (int64_t)u * P;
  const int per = (P + kThreads - 1) / kThreads;
  const int b0 = threadIdx.x * per, b1 = min(P, b0 + per);
  int c[4] = {0, 0, 0, 0};
  for (int b = b0; b < b1; ++b) {
    const int t = th[b];
    if (t < 0) continue;
    const uint32_t live = ~ev[b] & (fl[b] >= 32 ? 0xffffffffu : ((1u << fl[b]) - 1u));
    c[dm.band_fmt[t]] += __popc(live);
  }
  // exclusive scan over threads, per format (4 x kThreads ints in smem)
  for (int f = 0; f < 4; ++f) scan[f * kThreads + threadIdx.x] = c[f];
  __syncthreads();
  if (threadIdx.x < 4) {
    int run = 0;
    for (int i = 0; i < kThreads; ++i) {
      const int x = scan[threadIdx.x * kThreads + i];
      scan[threadIdx.x * kThreads + i] = run;
      run += x;
    }
    cnt[threadIdx.x] = run;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    off[0] = 0;
    for (int f = 1; f < 4; ++f) off[f] = off[f - 1] + cnt[f - 1];
  }
  __syncthreads();
  int w[4];
  for (int f = 0; f < 4; ++f) w[f] = off[f] + scan[f * kThreads + threadIdx.x];
  for (int b = b0; b < b1; ++b) {
    const int t = th[b];
    if (t < 0) continue;
    uint32_t live = ~ev[b] & (fl[b] >= 32 ? 0xffffffffu : ((1u << fl[b]) - 1u));
    const int f = dm.band_fmt[t];
    while (live) {
      const int s = __ffs(live) - 1;
      live &= live - 1;
      list[w[f]++] = b * bs + s;
    }
  }
  __syncthreads();
}

// Decoded key channel ch of a slot (fp32, exact for 2/4-bit; FP8 scale kept
// out of the code and applied per token).
template <int FMT>
__device__ __forceinline__ float key_chan(const TkvState& st, const uint8_t* kr, const uint8_t* ksc, int ch) {
  if constexpr (FMT == TKV_FMT_TERNARY) return tern_f(kr[ch >> 2] >> (2 * (ch & 3))) * e4m3_f(ksc[ch]);
  else if constexpr (FMT == TKV_FMT_NVFP4) return fp4_f(kr[ch >> 1] >> (4 * (ch & 1))) * e4m3_f(ksc[ch]);
  else if constexpr (FMT == TKV_FMT_FP8) return e4m3_f(kr[ch]);
  else return in_f(kr, st.dm.in_dtype, ch);
}
template <int FMT>
__device__ __forceinline__ float val_chan(const TkvState& st, const uint8_t* vr, const uint8_t* vsc, int ch) {
  if constexpr (FMT == TKV_FMT_TERNARY) return tern_f(vr[ch >> 2] >> (2 * (ch & 3))) * e4m3_f(vsc[ch / st.dm.g]);
  else if constexpr (FMT == TKV_FMT_NVFP4) return fp4_f(vr[ch >> 1] >> (4 * (ch & 1))) * e4m3_f(vsc[ch / st.dm.g]);
  else if constexpr (FMT == TKV_FMT_FP8) return e4m3_f(vr[ch]);
  else return in_f(vr, st.dm.in_dtype, ch);
}

template <int CPL, int GM>
struct WarpState {
  static constexpr int R = GM;  // rows held (G for per-head, 1 used for max-pool)
  float m[R], l[R], acc[R][CPL];
};

template <int CPL, int GM>
__device__ __forceinline__ void softmax_tile(WarpState<CPL, GM>& ws, float (&L)[GM], float (&p)[GM], int R,
                                             bool valid) {
#pragma unroll
  for (int r = 0; r < GM; ++r) {
    if (r >= R) break;
    const float tmax = warp_max(valid ? L[r] : -CUDART_INF_F);
    const float mnew = fmaxf(ws.m[r], tmax);
    const float corr = exp2f(ws.m[r] - mnew);
    p[r] = valid ? exp2f(L[r] - mnew) : 0.0f;
    ws.l[r] = ws.l[r] * corr + warp_sum(p[r]);
#pragma unroll
    for (int i = 0; i < CPL; ++i) ws.acc[r][i] *= corr;
    ws.m[r] = mnew;
  }
}

// One 32-token tile of slots in format FMT.
template <int FMT, int CPL, int GM>
__device__ __forceinline__ void paged_tile(const TkvState& st, int u, const int* list, int n, const float* qs,
                                           WarpState<CPL, GM>& ws) {
  const TkvDims& dm = st.dm;
  const int lane = threadIdx.x & 31;
  const int D = dm.D, G = dm.G, R = dm.maxpool ? 1 : G;
  const bool valid = lane < n;
  const int slot = valid ? list[lane] : 0;
  const int64_t gs = (int64_t)u * dm.NS + slot;
  const uint8_t* kr = st.slot_k + gs * dm.kstride;
  const int win = st.slot_win[gs];
  const uint8_t* ksc = st.win_ks + ((int64_t)u * dm.NW + (win < 0 ? 0 : win)) * D;
  float dot[GM];
#pragma unroll
  for (int g = 0; g < GM; ++g) dot[g] = 0.0f;
  if (valid) {
    for (int ch = 0; ch < D; ++ch) {
      const float kv = key_chan<FMT>(st, kr, ksc, ch);
#pragma unroll
      for (int g = 0; g < GM; ++g)
        if (g < G) dot[g] = fmaf(qs[g * D + ch], kv, dot[g]);
    }
    if constexpr (FMT == TKV_FMT_FP8) {
      const float s = st.win_kf[(int64_t)u * dm.NW + win];
#pragma unroll
      for (int g = 0; g < GM; ++g) dot[g] *= s;
    }
  }
  float L[GM], p[GM];
  if (dm.maxpool) {
    float mx = dot[0];
#pragma unroll
    for (int g = 1; g < GM; ++g)
      if (g < G) mx = fmaxf(mx, dot[g]);
    L[0] = mx;
  } else {
#pragma unroll
    for (int g = 0; g < GM; ++g) L[g] = dot[g];
  }
  softmax_tile<CPL, GM>(ws, L, p, R, valid);
  // PV: lane owns channels [lane*CPL, lane*CPL+CPL).
  for (int j = 0; j < n; ++j) {
    const int sj = __shfl_sync(0xffffffffu, slot, j);
    const int64_t gj = (int64_t)u * dm.NS + sj;
    const uint8_t* vr = st.slot_v + gj * dm.kstride;
    const uint8_t* vsc = st.slot_vs + gj * dm.vchunks;
    float vscale = 1.0f;
    if constexpr (FMT == TKV_FMT_FP8) vscale = st.win_vf[(int64_t)u * dm.NW + st.slot_win[gj]];
    float pj[GM];
#pragma unroll
    for (int r = 0; r < GM; ++r) pj[r] = __shfl_sync(0xffffffffu, p[r], j);
#pragma unroll
    for (int i = 0; i < CPL; ++i) {
      const int ch = lane * CPL + i;
      if (ch < D) {
        const float vv = val_chan<FMT>(st, vr, vsc, ch) * vscale;
#pragma unroll
        for (int r = 0; r < GM; ++r)
          if (r < R) ws.acc[r][i] = fmaf(pj[r], vv, ws.acc[r][i]);
      }
    }
  }
}

// Tail tile: buffered tokens [0, nbuf) and the current token (index nbuf).
template <int CPL, int GM>
__device__ __forceinline__ void input_tile(const TkvState& st, int u, int li, int t0, int n, int nbuf, int buf_half,
                                           const void* kin, const void* vin, const float* qs,
                                           WarpState<CPL, GM>& ws) {
  const TkvDims& dm = st.dm;
  const int lane = threadIdx.x & 31;
  const int D = dm.D, G = dm.G, R = dm.maxpool ? 1 : G;
  const int64_t row = (int64_t)dm.g * D;
  const uint8_t* bk = st.buf + ((int64_t)u * 4 + buf_half * 2 + 0) * row * dm.in_bytes;
  const uint8_t* bv = st.buf + ((int64_t)u * 4 + buf_half * 2 + 1) * row * dm.in_bytes;
  const bool valid = lane < n;
  const int t = t0 + lane;
  float dot[GM];
#pragma unroll
  for (int g = 0; g < GM; ++g) dot[g] = 0.0f;
  if (valid) {
    const void* kp = t < nbuf ? (const void*)(bk + (int64_t)t * D * dm.in_bytes)
                              : (const void*)((const uint8_t*)kin + (int64_t)li * D * dm.in_bytes);
    for (int ch = 0; ch < D; ++ch) {
      const float kv = in_f(kp, dm.in_dtype, ch);
#pragma unroll
      for (int g = 0; g < GM; ++g)
        if (g < G) dot[g] = fmaf(qs[g * D + ch], kv, dot[g]);
    }
  }
  float L[GM], p[GM];
  if (dm.maxpool) {
    float mx = dot[0];
#pragma unroll
    for (int g = 1; g < GM; ++g)
      if (g < G) mx = fmaxf(mx, dot[g]);
    L[0] = mx;
  } else {
#pragma unroll
    for (int g = 0; g < GM; ++g) L[g] = dot[g];
  }
  softmax_tile<CPL, GM>(ws, L, p, R, valid);
  for (int j = 0; j < n; ++j) {
    const int tj = t0 + j;
    const void* vp = tj < nbuf ? (const void*)(bv + (int64_t)tj * D * dm.in_bytes)
                               : (const void*)((const uint8_t*)vin + (int64_t)li * D * dm.in_bytes);
    float pj[GM];
#pragma unroll
    for (int r = 0; r < GM; ++r) pj[r] = __shfl_sync(0xffffffffu, p[r], j);
#pragma unroll
    for (int i = 0; i < CPL; ++i) {
      const int ch = lane * CPL + i;
      if (ch < D) {
        const float vv = in_f(vp, dm.in_dtype, ch);
#pragma unroll
        for (int r = 0; r < GM; ++r)
          if (r < R) ws.acc[r][i] = fmaf(pj[r], vv, ws.acc[r][i]);
      }
    }
  }
}

template <int CPL, int GM>
__global__ void __launch_bounds__(kThreads) attend_kernel(TkvState st, const void* __restrict__ qin,
                                                          const void* __restrict__ kin,
                                                          const void* __restrict__ vin, float* __restrict__ out,
                                                          int buf_half, int nbuf, int put_half, int put_slot) {
  tkv_step_scalars(st, buf_half, nbuf, put_half, put_slot);
  const TkvDims& dm = st.dm;
  const int li = blockIdx.x;             // launch-local index: q/k/v/out rows
  const int u = tkv_unit_of(st, li);     // unit: cache state
  const int D = dm.D, G = dm.G, R = dm.maxpool ? 1 : G;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  extern __shared__ __align__(16) uint8_t dyn[];
  float* qs = reinterpret_cast<float*>(dyn);                     // [G][D]
  float* red = qs + G * D;                                        // [kWarps][2 + D] per row
  int* scan = reinterpret_cast<int*>(red + kWarps * GM * (2 + D)); // [4][kThreads]
  int* list = scan + 4 * kThreads;                                 // [NS]
  __shared__ int cnt[4], off[4];

  const float qscale = dm.scale * kLog2e;  // logits in the log2 domain
  for (int i = threadIdx.x; i < G * D; i += kThreads)
    qs[i] = in_f(qin, dm.in_dtype, (int64_t)li * G * D + i) * qscale;
  build_live_list(st, u, list, cnt, off, scan);  // ends with __syncthreads

  WarpState<CPL, GM> ws;
#pragma unroll
  for (int r = 0; r < GM; ++r) {
    ws.m[r] = -CUDART_INF_F;
    ws.l[r] = 0.0f;
#pragma unroll
    for (int i = 0; i < CPL; ++i) ws.acc[r][i] = 0.0f;
  }
  // Tiles: paged formats first, then the input tail (buffer + current).
  int tiles[5];
  int total = 0;
  for (int f = 0; f < 4; ++f) { tiles[f] = (cnt[f] + 31) / 32; total += tiles[f]; }
  tiles[4] = (nbuf + 1 + 31) / 32;
  total += tiles[4];
  for (int t = warp; t < total; t += kWarps) {
    int f = 0, tt = t;
    while (f < 4 && tt >= tiles[f]) { tt -= tiles[f]; ++f; }
    if (f < 4) {
      const int* lst = list + off[f] + tt * 32;
      const int n = min(32, cnt[f] - tt * 32);
      switch (f) {
        case TKV_FMT_TERNARY: paged_tile<TKV_FMT_TERNARY, CPL, GM>(st, u, lst, n, qs, ws); break;
        case TKV_FMT_NVFP4: paged_tile<TKV_FMT_NVFP4, CPL, GM>(st, u, lst, n, qs, ws); break;
        case TKV_FMT_FP8: paged_tile<TKV_FMT_FP8, CPL, GM>(st, u, lst, n, qs, ws); break;
        default: paged_tile<TKV_FMT_RAW, CPL, GM>(st, u, lst, n, qs, ws); break;
      }
    } else {
      const int n = min(32, nbuf + 1 - tt * 32);
      input_tile<CPL, GM>(st, u, li, tt * 32, n, nbuf, buf_half, kin, vin, qs, ws);
    }
  }
  // Merge the warps' partial softmax states.
  __syncthreads();
  const int stride = 2 + D;
#pragma unroll
  for (int r = 0; r < GM; ++r) {
    if (r >= R) break;
    float* rr = red + (warp * GM + r) * stride;
    if (lane == 0) { rr[0] = ws.m[r]; rr[1] = ws.l[r]; }
#pragma unroll
    for (int i = 0; i < CPL; ++i) {
      const int ch = lane * CPL + i;
      if (ch < D) rr[2 + ch] = ws.acc[r][i];
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < R * D; idx += kThreads) {
    const int r = idx / D, ch = idx % D;
    float M = -CUDART_INF_F;
    for (int w = 0; w < kWarps; ++w) M = fmaxf(M, red[(w * GM + r) * stride]);
    float Lsum = 0.0f, O = 0.0f;
    for (int w = 0; w < kWarps; ++w) {
      const float* rr = red + (w * GM + r) * stride;
      const float f = exp2f(rr[0] - M);
      Lsum += rr[1] * f;
      O += rr[2 + ch] * f;
    }
    out[((int64_t)li * R + r) * D + ch] = O / Lsum;
  }
  // Buffer the incoming token for the next emission (sim.cpp:796-808).
  if (put_slot >= 0) {
    const int64_t row = (int64_t)dm.g * D * dm.in_bytes;
    uint8_t* bk = st.buf + ((int64_t)u * 4 + put_half * 2 + 0) * row + (int64_t)put_slot * D * dm.in_bytes;
    uint8_t* bv = st.buf + ((int64_t)u * 4 + put_half * 2 + 1) * row + (int64_t)put_slot * D * dm.in_bytes;
    const uint8_t* ks = (const uint8_t*)kin + (int64_t)li * D * dm.in_bytes;
    const uint8_t* vs = (const uint8_t*)vin + (int64_t)li * D * dm.in_bytes;
    for (int i = threadIdx.x; i < D * dm.in_bytes; i += kThreads) {
      bk[i] = ks[i];
      bv[i] = vs[i];
    }
  }
}

template <int CPL, int GM>
cudaError_t launch_attend_t(const TkvState& st, const void* q, const void* k, const void* v, float* out,
                            int buf_half, int nbuf, int put_half, int put_slot, cudaStream_t s) {
  const size_t smem = (size_t)st.dm.G * st.dm.D * 4 + (size_t)kWarps * GM * (2 + st.dm.D) * 4 +
                      (size_t)4 * kThreads * 4 + (size_t)st.dm.NS * 4;
  auto kern = attend_kernel<CPL, GM>;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured = true;
  }
  kern<<<tkv_launch_units(st), kThreads, smem, s>>>(st, q, k, v, out, buf_half, nbuf, put_half, put_slot);
  return cudaGetLastError();
}

template <int CPL>
cudaError_t launch_attend_g(const TkvState& st, const void* q, const void* k, const void* v, float* out,
                            int buf_half, int nbuf, int put_half, int put_slot, cudaStream_t s) {
  const int G = st.dm.G;
  if (G <= 1) return launch_attend_t<CPL, 1>(st, q, k, v, out, buf_half, nbuf, put_half, put_slot, s);
  if (G <= 2) return launch_attend_t<CPL, 2>(st, q, k, v, out, buf_half, nbuf, put_half, put_slot, s);
  if (G <= 4) return launch_attend_t<CPL, 4>(st, q, k, v, out, buf_half, nbuf, put_half, put_slot, s);
  if (G <= 8) return launch_attend_t<CPL, 8>(st, q, k, v, out, buf_half, nbuf, put_half, put_slot, s);
  return launch_attend_t<CPL, 16>(st, q, k, v, out, buf_half, nbuf, put_half, put_slot, s);
}

}  // namespace

cudaError_t tkv_launch_attend(const TkvState& st, const void* q, const void* k, const void* v, float* out,
                              int buf_half, int nbuf, int put_half, int put_slot, cudaStream_t s) {
  // Tensor-core kernel for the production shapes (d = 64/128, bf16, G <= 8,
  // quantised bands); the SIMT kernel below covers every other shape/dtype.
  if (tkv_attend_mma_supported(st.dm))
    return tkv_launch_attend_mma(st, q, k, v, out, buf_half, nbuf, put_half, put_slot, s);
  const int D = st.dm.D;
  if (D <= 32) return launch_attend_g<1>(st, q, k, v, out, buf_half, nbuf, put_half, put_slot, s);
  if (D <= 64) return launch_attend_g<2>(st, q, k, v, out, buf_half, nbuf, put_half, put_slot, s);
  if (D <= 128) return launch_attend_g<4>(st, q, k, v, out, buf_half, nbuf, put_half, put_slot, s);
  return launch_attend_g<8>(st, q, k, v, out, buf_half, nbuf, put_half, put_slot, s);
}
