// Gather-compaction comparator: the reference's
// GatherMethod (proj/src/sim.cpp:1117-1206) -- attention-score top-k eviction
// with physical compaction -- on the GPU, so ThinKV's slot reuse can be timed
// against it on the same inputs (BASELINE config 5).
//
// Per unit and step (one CTA per unit):
//   1. append the token's full-precision K/V at row n (cache order = arrival
//      order minus evicted rows) and its id;
//   2. attention over the n+1 rows for every query head (per-head rows, or
//      one max-pooled row), fp32 outputs;
//   3. once n+1 > budget: the head-averaged softmax score of every row --
//      exact fp64 in the reference's order (dot products channel by channel,
//      max-subtracted exp, sequential denominators, division, sequential
//      average over the groups, /groups; attention.cpp:32-67 and
//      sim.cpp:1141-1152) when `exact`, else the fp32 probabilities of step 2
//      -- then the first minimum is evicted (sim.cpp:1160-1163);
//   4. compaction: rows victim+1 .. n shift down by one slot (moved slots =
//      n - victim, the reference's moved_token_slots).
// This file is built with --fmad=false (the exact path).
#include <cuda_runtime.h>
#include <math_constants.h>

#include "tkv_exp.cuh"
#include "tkv_kernels.h"

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxR = 8;    // query heads per unit (G <= 8)
constexpr int kMaxCPL = 4;  // channels per lane (d <= 128)

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

__host__ __device__ inline size_t tkv_gather_smem_main(const TkvGatherState& g, int exact) {
  const size_t base = (size_t)g.G * g.D * 4 + (size_t)((g.G * g.cap + 1) & ~1) * 4;
  return (exact ? base + (size_t)g.G * g.D * 8 + (size_t)2 * g.cap * 8 : base + 8) / 16 * 16 + 16;
}

__device__ __forceinline__ float block_max(float v, float* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float r = red[0];
  for (int w = 1; w < kWarps; ++w) r = fmaxf(r, red[w]);
  return r;
}

// smem: qf [G][D] f32 | lg [G][cap] f32 (logits -> probabilities) | exact
//       mode only: qd [G][D] f64 | sc [cap] f64 (exact scores of one row) |
//       avg [cap] f64
template <int GM>  // query heads rounded up to a power of two (>= G)
__global__ void __launch_bounds__(kThreads) gather_step_kernel(TkvGatherState g, int n, int64_t pos,
                                                               const void* __restrict__ qin,
                                                               const void* __restrict__ kin,
                                                               const void* __restrict__ vin, float* __restrict__ out,
                                                               int exact) {
  const int u = blockIdx.x;
  const int D = g.D, G = g.G, cap = g.cap, eb = g.in_bytes;
  const int R = g.maxpool ? 1 : G;            // softmax rows (groups)
  const int rows = n + 1;
  extern __shared__ __align__(16) uint8_t dyn[];
  float* qf = reinterpret_cast<float*>(dyn);
  float* lg = qf + G * D;
  double* qd = reinterpret_cast<double*>(lg + (((int64_t)G * cap + 1) & ~1ll));
  double* sc = qd + G * D;     // [cap] exact scores of the current group
  double* avg = sc + cap;      // [cap]
  uint8_t* pv_red = dyn + tkv_gather_smem_main(g, exact);  // [kWarps][R][D] f32
  __shared__ float redf[kWarps];
  __shared__ double redd[kWarps];
  __shared__ double sum_s;
  __shared__ int victim_s;
  uint8_t* kc = g.k + (int64_t)u * cap * D * eb;
  uint8_t* vc = g.v + (int64_t)u * cap * D * eb;
  // 1. append
  for (int i = threadIdx.x; i < D * eb; i += kThreads) {
    kc[(int64_t)n * D * eb + i] = reinterpret_cast<const uint8_t*>(kin)[(int64_t)u * D * eb + i];
    vc[(int64_t)n * D * eb + i] = reinterpret_cast<const uint8_t*>(vin)[(int64_t)u * D * eb + i];
  }
  if (threadIdx.x == 0) g.ids[(int64_t)u * cap + n] = (int32_t)pos;
  for (int i = threadIdx.x; i < G * D; i += kThreads) {
    qf[i] = in_f(qin, g.in_dtype, (int64_t)u * G * D + i);
    if (exact) qd[i] = in_d(qin, g.in_dtype, (int64_t)u * G * D + i);
  }
  __syncthreads();
  // 2. fp32 attention: logits per head (warp per row, lanes over channels:
  //    coalesced row reads), row max / softmax, outputs (warps over rows,
  //    lanes over channels, partials merged in warp order)
  const float scale = 1.0f / sqrtf((float)D);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kRU = 4;  // rows per warp iteration: their loads are in flight together
  for (int i0 = warp * kRU; i0 < rows; i0 += kWarps * kRU) {
    float kx[kRU][kMaxCPL];
#pragma unroll
    for (int q = 0; q < kRU; ++q)
#pragma unroll
      for (int j = 0; j < kMaxCPL; ++j) {
        const int c = lane + 32 * j;
        kx[q][j] = (i0 + q < rows && c < D) ? in_f(kc, g.in_dtype, (int64_t)(i0 + q) * D + c) : 0.f;
      }
#pragma unroll
    for (int q = 0; q < kRU; ++q) {
      float dh[GM];
#pragma unroll
      for (int h = 0; h < GM; ++h) dh[h] = 0.f;
#pragma unroll
      for (int j = 0; j < kMaxCPL; ++j) {
        const int c = lane + 32 * j;
        if (c >= D) break;
#pragma unroll
        for (int h = 0; h < GM; ++h) dh[h] = fmaf(qf[h * D + c], kx[q][j], dh[h]);
      }
#pragma unroll
      for (int h = 0; h < GM; ++h)
        for (int o = 16; o > 0; o >>= 1) dh[h] += __shfl_xor_sync(0xffffffffu, dh[h], o);
      const int i = i0 + q;
      if (lane == 0 && i < rows) {
        if (g.maxpool) {  // gqa_aggregate: max over the G heads (row 0)
          float mx = dh[0] * scale;
#pragma unroll
          for (int h = 1; h < GM; ++h)
            if (h < G) mx = fmaxf(mx, dh[h] * scale);
          lg[i] = mx;
        } else {
#pragma unroll
          for (int h = 0; h < GM; ++h)
            if (h < G) lg[(int64_t)h * cap + i] = dh[h] * scale;
        }
      }
    }
  }
  __syncthreads();
  for (int r = 0; r < R; ++r) {
    float* L = lg + (int64_t)r * cap;
    float mx = -CUDART_INF_F;
    for (int i = threadIdx.x; i < rows; i += kThreads) mx = fmaxf(mx, L[i]);
    mx = block_max(mx, redf);
    float s = 0.f;
    for (int i = threadIdx.x; i < rows; i += kThreads) {
      const float e = __expf(L[i] - mx);
      L[i] = e;
      s += e;
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) redf[threadIdx.x >> 5] = s;
    __syncthreads();
    float tot = 0.f;
    for (int w = 0; w < kWarps; ++w) tot += redf[w];
    const float inv = 1.0f / tot;
    for (int i = threadIdx.x; i < rows; i += kThreads) L[i] *= inv;
    __syncthreads();
  }
  {
    constexpr int RM = GM;  // softmax rows held per lane (>= R)
    float acc[RM][kMaxCPL];
#pragma unroll
    for (int r = 0; r < RM; ++r)
#pragma unroll
      for (int j = 0; j < kMaxCPL; ++j) acc[r][j] = 0.f;
    for (int i0 = warp * kRU; i0 < rows; i0 += kWarps * kRU) {
      float vx[kRU][kMaxCPL];
#pragma unroll
      for (int q = 0; q < kRU; ++q)
#pragma unroll
        for (int j = 0; j < kMaxCPL; ++j) {
          const int c = lane + 32 * j;
          vx[q][j] = (i0 + q < rows && c < D) ? in_f(vc, g.in_dtype, (int64_t)(i0 + q) * D + c) : 0.f;
        }
#pragma unroll
      for (int q = 0; q < kRU; ++q) {
        if (i0 + q >= rows) break;
#pragma unroll
        for (int r = 0; r < RM; ++r) {
          if (r >= R) break;
          const float pr = lg[(int64_t)r * cap + i0 + q];
#pragma unroll
          for (int j = 0; j < kMaxCPL; ++j) acc[r][j] = fmaf(pr, vx[q][j], acc[r][j]);
        }
      }
    }
    float* red = reinterpret_cast<float*>(pv_red);  // [kWarps][R][D]
#pragma unroll
    for (int r = 0; r < RM; ++r) {
      if (r >= R) break;
#pragma unroll
      for (int j = 0; j < kMaxCPL; ++j) {
        const int c = lane + 32 * j;
        if (c < D) red[((int64_t)warp * R + r) * D + c] = acc[r][j];
      }
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < R * D; idx += kThreads) {
      float o = 0.f;
      for (int w = 0; w < kWarps; ++w) o += red[(int64_t)w * R * D + idx];
      out[(int64_t)u * R * D + idx] = o;
    }
    __syncthreads();
  }
  if (rows <= g.budget) return;
  // 3. head-averaged scores and the victim
  if (exact) {
    const double dscale = 1.0 / sqrt((double)D);
    for (int i = threadIdx.x; i < rows; i += kThreads) avg[i] = 0.0;
    for (int r = 0; r < R; ++r) {
      // exact logits of softmax row r (per head r, or max-pooled over all heads)
      for (int i = threadIdx.x; i < rows; i += kThreads) {
        double best = 0.0;
        for (int h = (g.maxpool ? 0 : r); h < (g.maxpool ? G : r + 1); ++h) {
          double dot = 0.0;
          for (int c = 0; c < D; ++c)
            dot = __dadd_rn(dot, __dmul_rn(qd[h * D + c], in_d(kc, g.in_dtype, (int64_t)i * D + c)));
          const double l = __dmul_rn(dot, dscale);
          best = h == (g.maxpool ? 0 : r) ? l : fmax(best, l);
        }
        sc[i] = best;
      }
      __syncthreads();
      double mx = -CUDART_INF;
      for (int i = threadIdx.x; i < rows; i += kThreads) mx = fmax(mx, sc[i]);
      for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if ((threadIdx.x & 31) == 0) redd[threadIdx.x >> 5] = mx;
      __syncthreads();
      mx = redd[0];
      for (int w = 1; w < kWarps; ++w) mx = fmax(mx, redd[w]);
      for (int i = threadIdx.x; i < rows; i += kThreads) sc[i] = tkv_exp(__dsub_rn(sc[i], mx));
      __syncthreads();
      if (threadIdx.x == 0) {  // softmax denominator in index order (attention.cpp:59-63)
        double s = 0.0;
        int i = 0;
        for (; i + 8 <= rows; i += 8) {
          double v[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) v[t] = sc[i + t];
#pragma unroll
          for (int t = 0; t < 8; ++t) s = __dadd_rn(s, v[t]);
        }
        for (; i < rows; ++i) s = __dadd_rn(s, sc[i]);
        sum_s = s;
      }
      __syncthreads();
      const double s = sum_s;
      // avg.scores[i] += row.scores[i] in group order (sim.cpp:1148-1150)
      for (int i = threadIdx.x; i < rows; i += kThreads) avg[i] = __dadd_rn(avg[i], __ddiv_rn(sc[i], s));
      __syncthreads();
    }
    for (int i = threadIdx.x; i < rows; i += kThreads) avg[i] = __ddiv_rn(avg[i], (double)R);
  }
  __syncthreads();
  // first minimum (strict <, ascending: sim.cpp:1160-1162)
  {
    double bv = CUDART_INF;
    int bi = 0x7fffffff;
    for (int i = threadIdx.x; i < rows; i += kThreads) {
      double a;
      if (exact) {
        a = avg[i];
      } else {  // fp32 head-averaged probabilities of the attention pass
        float f = 0.f;
        for (int r = 0; r < R; ++r) f += lg[(int64_t)r * cap + i];
        a = (double)f;
      }
      if (a < bv) { bv = a; bi = i; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov < bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    __shared__ double wv[kWarps];
    __shared__ int wi[kWarps];
    if ((threadIdx.x & 31) == 0) { wv[threadIdx.x >> 5] = bv; wi[threadIdx.x >> 5] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double v = wv[0];
      int i = wi[0];
      for (int w = 1; w < kWarps; ++w)
        if (wv[w] < v || (wv[w] == v && wi[w] < i)) { v = wv[w]; i = wi[w]; }
      victim_s = i;
      g.victim[u] = i;
    }
    __syncthreads();
  }
  // 4. compaction: rows victim+1 .. n move down one slot (chunked: a chunk
  //    is read completely before it is written, so the overlap is safe)
  const int vi = victim_s;
  const int64_t rowb = (int64_t)D * eb;
  const int64_t first = (int64_t)vi * rowb, last = (int64_t)n * rowb;  // destination byte range [first, last)
  if (rowb % 16 == 0) {
    constexpr int kU = 8;  // 16-byte words per thread per chunk (32 KB per chunk per array)
    for (int64_t b0 = first; b0 < last; b0 += (int64_t)kThreads * 16 * kU) {
      uint4 kk[kU], vv[kU];
#pragma unroll
      for (int j = 0; j < kU; ++j) {
        const int64_t b = b0 + ((int64_t)j * kThreads + threadIdx.x) * 16;
        if (b < last) {
          kk[j] = *reinterpret_cast<const uint4*>(kc + b + rowb);
          vv[j] = *reinterpret_cast<const uint4*>(vc + b + rowb);
        }
      }
      __syncthreads();
#pragma unroll
      for (int j = 0; j < kU; ++j) {
        const int64_t b = b0 + ((int64_t)j * kThreads + threadIdx.x) * 16;
        if (b < last) {
          *reinterpret_cast<uint4*>(kc + b) = kk[j];
          *reinterpret_cast<uint4*>(vc + b) = vv[j];
        }
      }
      __syncthreads();
    }
  } else {  // small rows: byte granularity
    for (int64_t b0 = first; b0 < last; b0 += kThreads) {
      const int64_t b = b0 + threadIdx.x;
      uint8_t kk = 0, vv = 0;
      const bool act = b < last;
      if (act) { kk = kc[b + rowb]; vv = vc[b + rowb]; }
      __syncthreads();
      if (act) { kc[b] = kk; vc[b] = vv; }
      __syncthreads();
    }
  }
  int32_t* ids = g.ids + (int64_t)u * cap;
  for (int i0 = vi; i0 < n; i0 += kThreads) {
    const int i = i0 + threadIdx.x;
    const int32_t x = i < n ? ids[i + 1] : 0;
    __syncthreads();
    if (i < n) ids[i] = x;
    __syncthreads();
  }
}

}  // namespace

size_t tkv_gather_smem(const TkvGatherState& g, int exact) {
  return tkv_gather_smem_main(g, exact) + (size_t)kWarps * (g.maxpool ? 1 : g.G) * g.D * 4;
}

cudaError_t tkv_launch_gather_step(const TkvGatherState& g, int n, int64_t pos, const void* q, const void* k,
                                   const void* v, float* out, int exact, cudaStream_t s) {
  const size_t smem = tkv_gather_smem(g, exact);
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    kern<<<g.U, kThreads, smem, s>>>(g, n, pos, q, k, v, out, exact);
    return cudaGetLastError();
  };
  if (g.G <= 1) return go(gather_step_kernel<1>);
  if (g.G <= 2) return go(gather_step_kernel<2>);
  if (g.G <= 4) return go(gather_step_kernel<4>);
  return go(gather_step_kernel<8>);
}
