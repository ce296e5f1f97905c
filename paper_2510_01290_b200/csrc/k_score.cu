// K3a: exact fp64 sparsity statistics per unit (layer_sparsity_average,
// proj/src/attention.cpp:148-167, over the rows gqa_attend builds,
// attention.cpp:32-67, 110-138), run on refresh steps only -- the only steps
// whose sparsity is consumed (sim.cpp:704-733).
//
// Bit-exactness: every value is the reference's own double, computed with
// the same operations in the same order (this file is built --fmad=false):
//   * decoded keys are code x E4M3 scale (<= 8 significant bits) -- exact in
//     fp32, so they are formed in fp32 and widened; FP8 keys are code x f32
//     tensor scale, exact in double (<= 28 bits), formed in double;
//   * dot = sum_c q[c] * k[c] sequentially in channel order (dmul, dadd),
//     logit = dot * (1/sqrt(d)) (scaled_logits, attention.cpp:32-45);
//     max-pool rows take the max over the G head logits (gqa_aggregate);
//   * softmax_row (attention.cpp:54-67): m = max, e_i = exp(l_i - m), sum in
//     index order, s_i = e_i / sum;
//   * sparsity: the row maximum of s is fl(1 / sum) exactly (the arg-max
//     logit gives exp(0) = 1 and division by sum is monotone), threshold =
//     frac * that, count s_i < threshold strictly;
//   * layer average: sum of per-row sparsities in row order / rows.
// exp is tkv_exp (tkv_exp.cuh): glibc's exp restated bit for bit, so every e_i,
// the sum and every s_i carry the reference's exact bits.
//
// Layout: one CTA (256 threads) per unit.  The unit's live slots are listed in
// physical (block, slot) order (BlockPager::read_active, pager.cpp:261-271),
// followed by the fp buffer and the incoming token.  Pass p computes the
// logits of up to kRows rows for every key (one key per thread, kChains
// independent dot chains), then each row's softmax statistics.
#include <cuda_runtime.h>
#include <math_constants.h>

#include "tkv_exp.cuh"
#include "tkv_kernels.h"
#include "tkv_state.h"

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kRows = 4;  // softmax rows held in shared memory per pass

__device__ __forceinline__ float e4m3_f(uint32_t c) {
  const uint32_t e = (c >> 3) & 15u, m = c & 7u;
  const float v = e == 0 ? (float)m * 0.001953125f : __uint_as_float(((e + 120u) << 23) | (m << 20));
  return (c & 0x80u) ? -v : v;
}
__device__ __forceinline__ float fp4_f(uint32_t c) {
  const uint32_t e = (c >> 1) & 3u, m = c & 1u;
  const float v = e == 0 ? 0.5f * (float)m : __uint_as_float(((e + 126u) << 23) | (m << 22));
  return (c & 8u) ? -v : v;
}
__device__ __forceinline__ float tern_f(uint32_t c) {
  c &= 3u;
  return c == 1u ? 1.0f : (c == 3u ? -1.0f : 0.0f);
}
__device__ __forceinline__ double raw_d(const uint8_t* p, int dtype, int ch) {
  if (dtype == TKV_IN_BF16) return (double)__uint_as_float(((uint32_t) reinterpret_cast<const uint16_t*>(p)[ch]) << 16);
  if (dtype == TKV_IN_F32) return (double)reinterpret_cast<const float*>(p)[ch];
  return reinterpret_cast<const double*>(p)[ch];
}

// Accumulate the NC dot chains of one key over channels [0, D): dot[j] +=
// q[g0 + j][ch] * k[ch] in channel order.  `dec(ch0, kv[8])` decodes 8
// channels.
template <int NC, bool VEC, typename Dec>
__device__ __forceinline__ void dots(const double* __restrict__ qd, int D, int g0, int ng, Dec dec, double (&dot)[NC]) {
  for (int ch0 = 0; ch0 < D; ch0 += 8) {
    double kv[8];
    dec(ch0, kv);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (!VEC && ch0 + c >= D) break;
#pragma unroll
      for (int j = 0; j < NC; ++j)
        if (j < ng) dot[j] = __dadd_rn(dot[j], __dmul_rn(qd[(g0 + j) * D + ch0 + c], kv[c]));
    }
  }
}

template <int NC, bool VEC>
__global__ void __launch_bounds__(kThreads) score_kernel(TkvState st, const void* __restrict__ qin,
                                                         const void* __restrict__ kin, int buf_half, int nbuf,
                                                         int rp) {
  const TkvDims& dm = st.dm;
  const int li = blockIdx.x;          // launch-local index: q/k rows
  const int u = tkv_unit_of(st, li);  // unit: cache state
  const int D = dm.D, G = dm.G, P = dm.P, bs = dm.bs;
  const int nmax = st.max_live + dm.g + 1;  // live slots + buffer + current token
  extern __shared__ __align__(16) uint8_t dyn[];
  double* lg = reinterpret_cast<double*>(dyn);                 // [rp][nmax]
  double* qd = lg + (int64_t)rp * nmax;                         // [G][D]
  int* list = reinterpret_cast<int*>(qd + (int64_t)G * D);      // [max_live]
  __shared__ int scan[kThreads];
  __shared__ double red[kWarps][kRows];
  __shared__ double rowsum[kRows];
  __shared__ int below[kRows];
  __shared__ int s_nlive;

  // ---- live slots, physical order -----------------------------------------
  const int8_t* th = st.blk_thought + (int64_t)u * P;
  const uint8_t* fl = st.blk_filled + (int64_t)u * P;
  const uint32_t* ev = st.blk_evict + (int64_t)u * P;
  const int per = (P + kThreads - 1) / kThreads;
  const int b0 = threadIdx.x * per, b1 = min(P, b0 + per);
  int c = 0;
  for (int b = b0; b < b1; ++b)
    if (th[b] >= 0) c += __popc(~ev[b] & (fl[b] >= 32 ? 0xffffffffu : ((1u << fl[b]) - 1u)));
  // block-wide exclusive scan (warp shuffles + per-warp totals)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = c;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) scan[warp] = incl;
  for (int i = threadIdx.x; i < G * D; i += kThreads) {
    const int64_t gi = (int64_t)li * G * D + i;
    qd[i] = dm.in_dtype == TKV_IN_BF16
                ? (double)__uint_as_float(((uint32_t) reinterpret_cast<const uint16_t*>(qin)[gi]) << 16)
                : (dm.in_dtype == TKV_IN_F32 ? (double)reinterpret_cast<const float*>(qin)[gi]
                                             : reinterpret_cast<const double*>(qin)[gi]);
  }
  __syncthreads();
  int before = 0, total_live = 0;
  for (int w = 0; w < kWarps; ++w) {
    if (w < warp) before += scan[w];
    total_live += scan[w];
  }
  if (total_live > st.max_live) {  // host bookkeeping disagrees with the block table
    if (threadIdx.x == 0) st.err[u] = TKV_E_INTEGRITY;
    return;
  }
  if (threadIdx.x == kThreads - 1) s_nlive = before + incl;
  {
    int w = before + incl - c;
    for (int b = b0; b < b1; ++b) {
      if (th[b] < 0) continue;
      uint32_t live = ~ev[b] & (fl[b] >= 32 ? 0xffffffffu : ((1u << fl[b]) - 1u));
      while (live) {
        const int sl = __ffs(live) - 1;
        live &= live - 1;
        list[w++] = b * bs + sl;
      }
    }
  }
  __syncthreads();
  const int nlive = s_nlive;
  const int n = nlive + nbuf + 1;
  const bool mp = dm.maxpool != 0;
  const int rows = mp ? 1 : G;
  const double scale = 1.0 / sqrt((double)D);
  const int64_t brow = (int64_t)dm.g * D * dm.in_bytes;
  const uint8_t* bk = st.buf + ((int64_t)u * 4 + buf_half * 2 + 0) * brow;
  const uint8_t* kc = reinterpret_cast<const uint8_t*>(kin) + (int64_t)li * D * dm.in_bytes;
  double total = 0.0;

  for (int r0 = 0; r0 < rows; r0 += rp) {
    const int nr = min(rp, rows - r0);
    // ---- logits of rows r0 .. r0 + nr ------------------------------------------
    // max-pool: one row from all G heads; per-head: heads r0 .. r0 + nr.
    const int g0 = mp ? 0 : r0;
    const int ngc = mp ? G : nr;  // chains per pass (NC >= ngc)
    for (int i = threadIdx.x; i < n; i += kThreads) {
      double dot[NC];
#pragma unroll
      for (int j = 0; j < NC; ++j) dot[j] = 0.0;
      if (i < nlive) {
        const int slot = list[i];
        const int64_t gs = (int64_t)u * dm.NS + slot;
        const int fmt = dm.band_fmt[th[slot / bs]];
        const uint8_t* kr = st.slot_k + gs * dm.kstride;
        const int win = st.slot_win[gs];
        if (fmt == TKV_FMT_NVFP4 || fmt == TKV_FMT_TERNARY) {
          const uint8_t* ks = st.win_ks + ((int64_t)u * dm.NW + win) * D;
          if (!VEC) {
            const bool f4 = fmt == TKV_FMT_NVFP4;
            dots<NC, VEC>(qd, D, g0, ngc, [&](int ch0, double (&kv)[8]) {
#pragma unroll
              for (int t = 0; t < 8; ++t) {
                const int ch = min(ch0 + t, D - 1);
                const float cv = f4 ? fp4_f(kr[ch >> 1] >> (4 * (ch & 1))) : tern_f(kr[ch >> 2] >> (2 * (ch & 3)));
                kv[t] = (double)(cv * e4m3_f(ks[ch]));
              }
            }, dot);
          } else if (fmt == TKV_FMT_NVFP4) {
            dots<NC, VEC>(qd, D, g0, ngc, [&](int ch0, double (&kv)[8]) {
              const uint32_t w = *reinterpret_cast<const uint32_t*>(kr + ch0 / 2);
              const uint2 s = *reinterpret_cast<const uint2*>(ks + ch0);
#pragma unroll
              for (int t = 0; t < 8; ++t)
                kv[t] = (double)(fp4_f(w >> (4 * t)) * e4m3_f(((t < 4 ? s.x : s.y) >> (8 * (t & 3))) & 0xffu));
            }, dot);
          } else {
            dots<NC, VEC>(qd, D, g0, ngc, [&](int ch0, double (&kv)[8]) {
              const uint32_t w = *reinterpret_cast<const uint16_t*>(kr + ch0 / 4);
              const uint2 s = *reinterpret_cast<const uint2*>(ks + ch0);
#pragma unroll
              for (int t = 0; t < 8; ++t)
                kv[t] = (double)(tern_f(w >> (2 * t)) * e4m3_f(((t < 4 ? s.x : s.y) >> (8 * (t & 3))) & 0xffu));
            }, dot);
          }
        } else if (fmt == TKV_FMT_FP8) {
          const double kf = (double)st.win_kf[(int64_t)u * dm.NW + win];
          dots<NC, VEC>(qd, D, g0, ngc, [&](int ch0, double (&kv)[8]) {
            if (VEC) {
              const uint2 w = *reinterpret_cast<const uint2*>(kr + ch0);
#pragma unroll
              for (int t = 0; t < 8; ++t)
                kv[t] = __dmul_rn((double)e4m3_f(((t < 4 ? w.x : w.y) >> (8 * (t & 3))) & 0xffu), kf);
            } else {
#pragma unroll
              for (int t = 0; t < 8; ++t) kv[t] = __dmul_rn((double)e4m3_f(kr[min(ch0 + t, D - 1)]), kf);
            }
          }, dot);
        } else {
          dots<NC, VEC>(qd, D, g0, ngc, [&](int ch0, double (&kv)[8]) {
#pragma unroll
            for (int t = 0; t < 8; ++t) kv[t] = raw_d(kr, dm.in_dtype, min(ch0 + t, D - 1));
          }, dot);
        }
      } else {
        const uint8_t* kr = i < nlive + nbuf ? bk + (int64_t)(i - nlive) * D * dm.in_bytes : kc;
        dots<NC, VEC>(qd, D, g0, ngc, [&](int ch0, double (&kv)[8]) {
#pragma unroll
          for (int t = 0; t < 8; ++t) kv[t] = raw_d(kr, dm.in_dtype, min(ch0 + t, D - 1));
        }, dot);
      }
      if (mp) {
        double best = __dmul_rn(dot[0], scale);
#pragma unroll
        for (int j = 1; j < NC; ++j)
          if (j < G) best = fmax(best, __dmul_rn(dot[j], scale));  // gqa_aggregate
        lg[i] = best;
      } else {
#pragma unroll
        for (int j = 0; j < NC; ++j)
          if (j < nr) lg[(int64_t)j * nmax + i] = __dmul_rn(dot[j], scale);
      }
    }
    __syncthreads();
    // ---- row maxima (exact in any order) ----------------------------------------
    {
      double mx[kRows];
#pragma unroll
      for (int r = 0; r < kRows; ++r) mx[r] = -CUDART_INF;
      for (int i = threadIdx.x; i < n; i += kThreads)
#pragma unroll
        for (int r = 0; r < kRows; ++r)
          if (r < nr) mx[r] = fmax(mx[r], lg[(int64_t)r * nmax + i]);
#pragma unroll
      for (int r = 0; r < kRows; ++r) {
        for (int o = 16; o > 0; o >>= 1) mx[r] = fmax(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], o));
        if (lane == 0) red[warp][r] = mx[r];
      }
    }
    __syncthreads();
    // ---- e_i = exp(l_i - m) in place ---------------------------------------------
    for (int r = 0; r < nr; ++r) {
      double m = red[0][r];
      for (int w = 1; w < kWarps; ++w) m = fmax(m, red[w][r]);
      double* L = lg + (int64_t)r * nmax;
      for (int i = threadIdx.x; i < n; i += kThreads) L[i] = tkv_exp(__dsub_rn(L[i], m));
    }
    __syncthreads();
    // ---- denominators: one lane per row, index order, loads batched ahead -----------
    if (lane == 0 && warp < nr) {
      const double* L = lg + (int64_t)warp * nmax;
      double sum = 0.0;
      int i = 0;
      for (; i + 16 <= n; i += 16) {
        double v[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) v[t] = L[i + t];
#pragma unroll
        for (int t = 0; t < 16; ++t) sum = __dadd_rn(sum, v[t]);
      }
      for (; i < n; ++i) sum = __dadd_rn(sum, L[i]);
      rowsum[warp] = sum;
      below[warp] = 0;
    }
    __syncthreads();
    // ---- counts: s_i = e_i / sum < frac * max_i s_i, max s = fl(1 / sum) -----------
    for (int r = 0; r < nr; ++r) {
      const double sum = rowsum[r];
      const double thr = __dmul_rn(dm.thr_frac, __ddiv_rn(1.0, sum));
      const double* L = lg + (int64_t)r * nmax;
      int cb = 0;
      for (int i = threadIdx.x; i < n; i += kThreads) cb += __ddiv_rn(L[i], sum) < thr ? 1 : 0;
      for (int o = 16; o > 0; o >>= 1) cb += __shfl_xor_sync(0xffffffffu, cb, o);
      if (lane == 0) atomicAdd(&below[r], cb);
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int r = 0; r < nr; ++r) total = __dadd_rn(total, __ddiv_rn((double)below[r], (double)n));
    __syncthreads();
  }
  if (threadIdx.x == 0) st.sparsity[u] = __ddiv_rn(total, (double)rows);
}

template <int NC, bool VEC>
cudaError_t launch_t(const TkvState& st, const void* q, const void* k, int buf_half, int nbuf, size_t smem, int rp,
                     cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(score_kernel<NC, VEC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured = true;
  }
  score_kernel<NC, VEC><<<tkv_launch_units(st), kThreads, smem, s>>>(st, q, k, buf_half, nbuf, rp);
  return cudaGetLastError();
}

template <int NC>
cudaError_t launch_nc(const TkvState& st, const void* q, const void* k, int buf_half, int nbuf, size_t smem, int rp,
                      cudaStream_t s) {
  // 8-channel vector loads need D % 8 == 0 (row and scale-row alignment follows)
  if (st.dm.D % 8 == 0) return launch_t<NC, true>(st, q, k, buf_half, nbuf, smem, rp, s);
  return launch_t<NC, false>(st, q, k, buf_half, nbuf, smem, rp, s);
}

}  // namespace

cudaError_t tkv_launch_score(const TkvState& st, const void* q, const void* k, int buf_half, int nbuf,
                             cudaStream_t s) {
  const TkvDims& dm = st.dm;
  // rows per pass: as many softmax rows as fit next to q and the live list
  const size_t nmax = (size_t)st.max_live + dm.g + 1;
  const size_t fixed = (size_t)dm.G * dm.D * 8 + (size_t)st.max_live * 4;
  int rp = kRows;
  while (rp > 1 && (size_t)rp * nmax * 8 + fixed > 200 * 1024) --rp;
  const size_t smem = (size_t)rp * nmax * 8 + fixed;
  if (smem > 200 * 1024) return cudaErrorInvalidConfiguration;  // > ~24K live slots per unit
  // chains per key and pass: all G heads for max-pool rows, else up to rp heads
  const int nc = dm.maxpool ? dm.G : (dm.G < rp ? dm.G : rp);
  if (nc <= 1) return launch_nc<1>(st, q, k, buf_half, nbuf, smem, rp, s);
  if (nc <= 2) return launch_nc<2>(st, q, k, buf_half, nbuf, smem, rp, s);
  if (nc <= 4) return launch_nc<4>(st, q, k, buf_half, nbuf, smem, rp, s);
  if (nc <= 8) return launch_nc<8>(st, q, k, buf_half, nbuf, smem, rp, s);
  return launch_nc<16>(st, q, k, buf_half, nbuf, smem, rp, s);
}
