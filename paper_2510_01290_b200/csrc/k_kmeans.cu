// K3d v2: bit-exact K-means medoid selection (kmeans_select, proj/src/
// evictor.cpp:55-338) restructured for throughput.
//
// Three kernels per anneal wave:
//   prep     one CTA per (unit, anneal op) "instance": decodes the segment's
//            member keys once (exact: fp32 value x per-point fp64 scale), the
//            exact pairwise distance matrix pd[i][j] = dist2(x_i, x_j)
//            (evictor.cpp:57-64 order: sequential channel sum, no FMA), the
//            mean anchors and the four farthest-first seed sets
//            (evictor.cpp:71-92, 284-314) -- one warp per anchor, reading pd.
//   restart  one CTA per (instance, restart): Lloyd + Hartigan moves + swaps
//            (kmeans_from_seeds, evictor.cpp:94-251) with keys, centroids and
//            an exact point-to-centroid distance cache D2[i][c] in shared
//            memory.  D2 values are the reference's dist2(keys[i], mean_of(c))
//            bit for bit (same operands, same operation order); a move
//            invalidates exactly two columns, which are recomputed, so each
//            Hartigan decision is an O(K) scan of cached values instead of K
//            fresh distance evaluations.  The O(m^2 D) pairwise-swap scan is
//            filtered with the algebraic identity
//              delta = D2[j][a] - D2[i][a] + D2[i][b] - D2[j][b] - (1/na + 1/nb) pd[i][j]
//            plus a margin that dominates the rounding error of both that
//            expression and the reference's channel-wise formula by orders of
//            magnitude; only pairs inside the margin are evaluated with the
//            reference's exact expression, in lexicographic order.  The
//            restart writes its cost (summed in point order) and its medoids.
//   final    one thread per instance: the lowest-cost restart (ties to the
//            earlier one, evictor.cpp:319-325) supplies the retained set.
// The file is compiled with --fmad=false and every order-sensitive value uses
// explicit _rn intrinsics.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdio>
#include <cstdlib>

#include "tkv_codec.cuh"
#include "tkv_kernels.h"
#include "tkv_state.h"

namespace {

constexpr int kMaxM = 256;
constexpr int kSwapWin = 1024;  // pairs per swap-filter window (= candidate list capacity)

__device__ __forceinline__ int find_op(const int32_t* prefix, int nops, int item) {
  int lo = 0, hi = nops - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) / 2;
    if (prefix[mid] <= item) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Scratch geometry of one instance (identical formula on host and device).
struct KmGeo {
  int mmax, kmax, D, W, R;  // R = restart capacity per instance
  __host__ __device__ int64_t x_off() const { return 0; }                                   // f32 [mmax][D]
  __host__ __device__ int64_t xs_off() const { return x_off() + (int64_t)mmax * D * 4; }   // f64 [mmax]
  __host__ __device__ int64_t pd_off() const { return xs_off() + (int64_t)mmax * 8; }      // f64 [mmax][mmax]
  __host__ __device__ int64_t ids_off() const { return pd_off() + (int64_t)mmax * mmax * 8; }  // i32 [mmax]
  __host__ __device__ int64_t seeds_off() const { return ids_off() + (int64_t)mmax * 4; }  // i32 [4][kmax]
  __host__ __device__ int64_t cost_off() const { return (seeds_off() + (int64_t)4 * kmax * 4 + 7) / 8 * 8; }  // f64 [R]
  __host__ __device__ int64_t mask_off() const { return cost_off() + (int64_t)R * 8; }     // u32 [R][W]
  __host__ __device__ int64_t misc_off() const { return mask_off() + (int64_t)R * W * 4; }  // i32 [4]: m, bad
  __host__ __device__ int64_t bytes() const { return (misc_off() + 16 + 255) / 256 * 256; }
};

__device__ int g_kst_small;  // unused
__device__ __forceinline__ void kst(const TkvState& st, int i, unsigned long long v) {
  if (st.kstats && threadIdx.x == 0) atomicAdd(st.kstats + i, v);
}
__device__ __forceinline__ void kstm(const TkvState& st, int m, int i, unsigned long long v) {
  if (st.kstats && threadIdx.x == 0)
    atomicAdd(st.kstats + 32 + 32 * (m <= 8 ? 0 : m <= 16 ? 1 : m <= 32 ? 2 : m <= 64 ? 3 : 4) + i, v);
}

// x / n for a cluster size n >= 1.  For n = 2^k the multiply by the exact
// reciprocal 2^-k is the same correctly rounded real x / 2^k as the
// division, so both produce identical bits; other sizes divide.
// Other sizes up to kInvN: Markstein's correction from the correctly rounded
// reciprocal r = RN(1/n) (c_inv_n, written once per device by the host):
// q0 = RN(x r) lies within one ulp of x/n, the residual x - q0 n is exact in
// one fma, and RN(q0 + residual * r) is the correctly rounded quotient
// (Markstein 1990; Muller et al., Handbook of Floating-Point Arithmetic,
// division by fma) -- the bits of __ddiv_rn(x, n) in 3 fp64 operations
// instead of the division's reciprocal iteration.  A zero quotient keeps the
// sign of x (q0).
constexpr int kInvN = 1024;
__constant__ double c_inv_n[kInvN + 1];
__device__ __forceinline__ double div_n(double x, int n) {
  if ((n & (n - 1)) == 0) return __dmul_rn(x, __longlong_as_double((long long)(1024 - __ffs(n)) << 52));
  if (n > kInvN) return __ddiv_rn(x, (double)n);
  const double r = c_inv_n[n];
  const double q0 = __dmul_rn(x, r);
  const double rem = __fma_rn(-q0, (double)n, x);
  return q0 == 0.0 ? q0 : __fma_rn(rem, r, q0);
}
// Out-of-line form for the warp-per-restart kernel: one copy of the division
// sequence keeps its many concurrent warps inside the instruction cache
// (inlined copies made "no instruction" the dominant stall).
__device__ __noinline__ double div_n_ool(double x, int n) { return div_n(x, n); }

// idx -> (row, channel) for row length D (shift/mask when D is a power of two).
struct RowSplit {
  int D, sh;
  bool p2;
  __device__ explicit RowSplit(int d) : D(d), sh(0), p2((d & (d - 1)) == 0) {
    while ((1 << sh) < d) ++sh;
  }
  __device__ __forceinline__ int row(int idx) const { return p2 ? idx >> sh : idx / D; }
  __device__ __forceinline__ int col(int idx) const { return p2 ? idx & (D - 1) : idx % D; }
};

__device__ __forceinline__ double xget(const float* X, int64_t k) { return (double)X[k]; }
__device__ __forceinline__ double xget(const __half* X, int64_t k) {
  double r;  // one F2F.F64.F16 (exact widening)
  asm("cvt.f64.f16 %0, %1;" : "=d"(r) : "h"(__half_as_ushort(X[k])));
  return r;
}
// Decoded key channel: f32 store, or f16 when every band is a quantised
// format (code x E4M3 scale <= 8 significant bits in [2^-10, 2688], FP8 codes
// in [2^-9, 448]: exact in f16).
template <typename XT>
__device__ __forceinline__ double xval(const XT* X, const double* xs, int i, int ch, int xstride, bool scaled) {
  const double v = xget(X, (int64_t)i * xstride + ch);
  return scaled ? __dmul_rn(v, xs[i]) : v;
}

// ---------------------------------------------------------------------------
// prep
// ---------------------------------------------------------------------------
template <typename XT>
__device__ void decode_point(const TkvState& st, int u, int slot, XT* xrow, double* xs) {
  const TkvDims& dm = st.dm;
  const int64_t gs = (int64_t)u * dm.NS + slot;
  const int fmt = dm.band_fmt[st.blk_thought[(int64_t)u * dm.P + slot / dm.bs]];
  const uint8_t* kr = st.slot_k + gs * dm.kstride;
  const int win = st.slot_win[gs];
  for (int ch = 0; ch < dm.D; ++ch) {
    float v;
    if (fmt == TKV_FMT_RAW) {
      v = dm.in_dtype == TKV_IN_BF16 ? __uint_as_float(((uint32_t) reinterpret_cast<const uint16_t*>(kr)[ch]) << 16)
                                      : reinterpret_cast<const float*>(kr)[ch];
    } else if (fmt == TKV_FMT_FP8) {
      v = (float)tkv_e4m3_decode((uint8_t)kr[ch]);
    } else {
      // code x E4M3 scale: <= 7 significant bits, exact in fp32 (and fp64).
      v = (float)tkv_decode_code(fmt, tkv_get_code(kr, fmt, ch),
                                 tkv_e4m3_decode(st.win_ks[((int64_t)u * dm.NW + win) * dm.D + ch]));
    }
    xrow[ch] = (XT)v;
  }
  *xs = fmt == TKV_FMT_FP8 ? (double)st.win_kf[(int64_t)u * dm.NW + win] : 1.0;
}

template <typename XT>
__global__ void __launch_bounds__(256) km_prep_kernel(TkvState st, const TkvAnnealOp* __restrict__ ops, int nops,
                                                      const int32_t* __restrict__ prefix, int nitems, int item0,
                                                      uint8_t* __restrict__ scratch, KmGeo geo, int scaled_any) {
  const TkvDims& dm = st.dm;
  const int item = item0 + blockIdx.x;
  if (item >= nitems) return;
  const long long t_prep = clock64();
  const int oi = find_op(prefix, nops, item);
  const TkvAnnealOp op = ops[oi];
  const int urel = item - prefix[oi];
  const int u = op.unit0 + urel;
  const int D = dm.D;
  uint8_t* base = scratch + (int64_t)blockIdx.x * geo.bytes();
  kst(st, 0, 1);
  float* X = reinterpret_cast<float*>(base + geo.x_off());
  double* xs = reinterpret_cast<double*>(base + geo.xs_off());
  double* pd = reinterpret_cast<double*>(base + geo.pd_off());
  int32_t* ids = reinterpret_cast<int32_t*>(base + geo.ids_off());
  int32_t* seeds = reinterpret_cast<int32_t*>(base + geo.seeds_off());
  int32_t* misc = reinterpret_cast<int32_t*>(base + geo.misc_off());
  __shared__ int sids[kMaxM], sslot[kMaxM];
  __shared__ int sm_m, sm_bad, sm_found;
  __shared__ double dmean[kMaxM];
  __shared__ int anchors[4];
  const uint32_t* segm = st.seg_mask + ((int64_t)u * dm.NSEG + op.seg) * dm.W;
  if (threadIdx.x == 0) {
    int m = 0;
    for (int b = 0; b < op.span && m < kMaxM; ++b)
      if ((segm[b >> 5] >> (b & 31)) & 1u) sids[m++] = b;
    sm_m = m;
    sm_found = 0;
  }
  __syncthreads();
  if (sm_m == op.m && op.m <= kMaxM) tkv_member_slots(st, u, op.seg_start, op.span, segm, sslot, &sm_found);
  __syncthreads();
  if (threadIdx.x == 0) {
    const int bad = (sm_m != op.m) || sm_found != sm_m || st.err[u] != 0;
    sm_bad = bad;
    misc[0] = sm_m;
    misc[1] = bad;
  }
  __syncthreads();
  if (sm_bad) return;
  const int m = sm_m, K = op.K;
  extern __shared__ __align__(16) uint8_t pdyn[];
  // decoded keys [m][XS] (padded: conflict-free column access); f16 when every
  // band is quantised (exact, see xval), which doubles the CTAs per SM
  XT* sX = reinterpret_cast<XT*>(pdyn);
  const int XS = D + 4 / (int)sizeof(XT);
  __shared__ double sxs[kMaxM];
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    ids[i] = sids[i];
    decode_point(st, u, sslot[i], sX + (int64_t)i * XS, sxs + i);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < m * D; i += blockDim.x) X[i] = (float)sX[(i / D) * XS + i % D];
  for (int i = threadIdx.x; i < m; i += blockDim.x) xs[i] = sxs[i];
  const bool scaled = scaled_any != 0;
  // Exact pairwise distances, upper triangle mirrored ((a-b)^2 == (b-a)^2 in
  // IEEE).  Warp task = 4 rows i x 64 columns j (lane -> j, j + 32), 8
  // independent channel-sequential chains per thread, operands from smem.
  {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int pblocks = (m + 3) / 4, cgroups = (m + 63) / 64;
    for (int task = warp; task < pblocks * cgroups; task += blockDim.x / 32) {
      const int pb = task / cgroups, cg = task % cgroups;
      if (cg * 64 + 63 <= pb * 4) continue;  // entirely on/below the diagonal
      const int j0 = cg * 64 + lane, j1 = j0 + 32;
      const int jj0 = min(j0, m - 1), jj1 = min(j1, m - 1);
      int ip[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) ip[q] = min(pb * 4 + q, m - 1);
      double d[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
      #pragma unroll 2
      for (int ch = 0; ch < D; ++ch) {
        const double a0 = xval(sX, sxs, jj0, ch, XS, scaled), a1 = xval(sX, sxs, jj1, ch, XS, scaled);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double x = xval(sX, sxs, ip[q], ch, XS, scaled);
          const double t0 = __dsub_rn(x, a0), t1 = __dsub_rn(x, a1);
          d[q][0] = __dadd_rn(d[q][0], __dmul_rn(t0, t0));
          d[q][1] = __dadd_rn(d[q][1], __dmul_rn(t1, t1));
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int i = pb * 4 + q;
        if (i >= m) break;
        if (j0 < m && j0 > i) { pd[(int64_t)i * geo.mmax + j0] = d[q][0]; pd[(int64_t)j0 * geo.mmax + i] = d[q][0]; }
        if (j1 < m && j1 > i) { pd[(int64_t)i * geo.mmax + j1] = d[q][1]; pd[(int64_t)j1 * geo.mmax + i] = d[q][1]; }
      }
    }
  }
  for (int i = threadIdx.x; i < m; i += blockDim.x) pd[(int64_t)i * geo.mmax + i] = 0.0;
  __syncthreads();
  kst(st, 1, (unsigned long long)(clock64() - t_prep));
  if (op.nrestart <= 0) return;  // exhaustive seeds: nothing else to prepare
  __syncthreads();
  // anchors: 0, farthest from / nearest to the mean, m/2 (evictor.cpp:296-313)
  __shared__ double mean[256];
  for (int ch = threadIdx.x; ch < D; ch += blockDim.x) {
    double acc = 0.0;
    for (int i = 0; i < m; ++i) acc = __dadd_rn(acc, xval(sX, sxs, i, ch, XS, scaled));
    mean[ch] = __ddiv_rn(acc, (double)m);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    double d = 0.0;
    #pragma unroll 8
    for (int ch = 0; ch < D; ++ch) {
      const double t = __dsub_rn(xval(sX, sxs, i, ch, XS, scaled), mean[ch]);
      d = __dadd_rn(d, __dmul_rn(t, t));
    }
    dmean[i] = d;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int far_idx = 0, near_idx = 0;
    double far_d = -1.0, near_d = CUDART_INF;
    for (int i = 0; i < m; ++i) {
      const double d = dmean[i];
      if (d > far_d) { far_d = d; far_idx = i; }
      if (d < near_d) { near_d = d; near_idx = i; }
    }
    anchors[0] = 0;
    anchors[1] = far_idx;
    anchors[2] = near_idx;
    anchors[3] = m / 2;
  }
  __syncthreads();
  // farthest-first per anchor: one warp each over the precomputed pd.
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < 4) {
    __shared__ double nearest[4][kMaxM];
    __shared__ unsigned char taken[4][kMaxM];
    double* nr = nearest[warp];
    unsigned char* tk = taken[warp];
    int32_t* sd = seeds + warp * geo.kmax;
    for (int i = lane; i < m; i += 32) { nr[i] = CUDART_INF; tk[i] = 0; }
    int last = anchors[warp];
    if (lane == 0) { sd[0] = last; }
    __syncwarp();
    if (lane == 0) tk[last] = 1;
    __syncwarp();
    for (int n = 1; n < K; ++n) {
      double best_d = -1.0;
      int best_i = 0x7fffffff;
      for (int i = lane; i < m; i += 32) {
        const double d = pd[(int64_t)i * geo.mmax + last];
        const double v = d < nr[i] ? d : nr[i];
        nr[i] = v;
        if (!tk[i] && v > best_d) { best_d = v; best_i = i; }
      }
      // first index of the maximum among untaken points
      for (int o = 16; o > 0; o >>= 1) {
        const double od = __shfl_xor_sync(0xffffffffu, best_d, o);
        const int oi2 = __shfl_xor_sync(0xffffffffu, best_i, o);
        if (od > best_d || (od == best_d && oi2 < best_i)) { best_d = od; best_i = oi2; }
      }
      if (best_i == 0x7fffffff) best_i = 0;  // (far initialised to 0, evictor.cpp:80)
      last = best_i;
      if (lane == 0) { sd[n] = last; tk[last] = 1; }
      __syncwarp();
    }
  }
  __syncthreads();
  kst(st, 2, (unsigned long long)(clock64() - t_prep));
}

// ---------------------------------------------------------------------------
// restart
// ---------------------------------------------------------------------------
template <int MAXM>
struct RsSmem {
  static constexpr int CAP = (MAXM == 128 || MAXM == 64) ? 512 : kSwapWin;  // smaller for the multi-CTA classes
  static constexpr int WIN = MAXM * (MAXM - 1) / 2 < CAP ? MAXM * (MAXM - 1) / 2 : CAP;
  int assign[MAXM];
  int sizes[MAXM];
  int order[MAXM];
  int offs[MAXM + 1];
  int cur[MAXM];
  int seeds[MAXM];
  int colsrc[MAXM];   // per centroid column of D2: kColKeep, kColCompute, or a point whose pd column it equals
  int ccols[MAXM];    // compacted kColCompute columns
  int nccols;
  double tabA[MAXM + 1];  // n / (n + 1.0), indexed by cluster size (evictor.cpp:205)
  double tabR[MAXM + 1];  // -n / (n - 1.0) (evictor.cpp:201)
  double mv[MAXM];
  double xs[MAXM];
  double x2[MAXM];    // |x_i|^2 (swap-filter error bound)
  double m2[MAXM];    // |mean_of(c)|^2 (swap-filter error bound)
  int flag, move_i, move_to, pair;
  int ncand[2];  // per swap window, alternating: a window's reset never races the previous window's reads
  int res[32];
  int cand[WIN];
  double cost;
};

constexpr int kColKeep = -2;     // centroid bits unchanged since D2 was filled: column still exact
constexpr int kColCompute = -1;  // recompute the column from the centroid

// D2 columns selected by s.colsrc.  A centroid that IS a point (a seed, or
// the mean of a singleton cluster computed fresh from its member: 0 + x = x,
// x / 1 = x) has dist2(x_i, mu) == pd[i][p] bit for bit -- same operands in
// the same order (t = x_i - x_p, channel-sequential sum) -- so its column is
// copied from the prep kernel's pairwise matrix; unchanged centroids keep
// their column; only the rest are evaluated.
template <int NT, typename SM, typename XT>
__device__ void fill_sel(SM& s, const XT* X, int XS, const double* xs, bool scaled, const double* C, int cstride,
                         double* D2, const double* __restrict__ pd, int pstride, int m, int K, int D,
                         double* stg = nullptr, int stg_rows = 0) {
  if (threadIdx.x < 32) {
    int base = 0;
    for (int c0 = 0; c0 < K; c0 += 32) {
      const int c = c0 + (int)threadIdx.x;
      const bool comp = c < K && s.colsrc[c] == kColCompute;
      const unsigned bal = __ballot_sync(0xffffffffu, comp);
      if (comp) s.ccols[base + __popc(bal & ((1u << threadIdx.x) - 1u))] = c;
      base += __popc(bal);
    }
    if (threadIdx.x == 0) s.nccols = base;
  }
#pragma unroll 4
  for (int t = threadIdx.x; t < m * K; t += NT) {
    const int i = t / K, c = t % K;
    const int src = s.colsrc[c];
    if (src >= 0) D2[(int64_t)i * K + c] = pd[(int64_t)i * pstride + src];
  }
  __syncthreads();
  const int nc = s.nccols;
  if (nc == 0) return;
  if (stg) {
    // means in global memory: stage stg_rows mean rows at a time in shared
    // memory, then (point, column) chains -- consecutive lanes take
    // consecutive points of one column (conflict-free key rows, broadcast mean
    // row), two independent chains per thread.
    for (int c0 = 0; c0 < nc; c0 += stg_rows) {
      const int cn = min(stg_rows, nc - c0);
      for (int t = threadIdx.x; t < cn * D; t += NT) {
        const int j = t / D, ch = t - j * D;
        stg[(int64_t)j * cstride + ch] = C[(int64_t)s.ccols[c0 + j] * cstride + ch];
      }
      __syncthreads();
      const int total = m * cn;
      for (int t = threadIdx.x; t < total; t += 2 * NT) {
        const int t2 = t + NT;
        const bool v1 = t2 < total;
        const int j0 = t / m, i0 = t - j0 * m;
        const int j1 = v1 ? t2 / m : j0, i1 = v1 ? t2 - j1 * m : i0;
        const double* r0 = stg + (int64_t)j0 * cstride;
        const double* r1 = stg + (int64_t)j1 * cstride;
        double d0 = 0.0, d1 = 0.0;
        if (i0 == i1) {  // both chains on one point (m divides NT): widen each key channel once
#pragma unroll 8
          for (int ch = 0; ch < D; ++ch) {
            const double x = xval(X, xs, i0, ch, XS, scaled);
            const double a0 = __dsub_rn(x, r0[ch]), a1 = __dsub_rn(x, r1[ch]);
            d0 = __dadd_rn(d0, __dmul_rn(a0, a0));
            d1 = __dadd_rn(d1, __dmul_rn(a1, a1));
          }
        } else {
#pragma unroll 8
          for (int ch = 0; ch < D; ++ch) {
            const double a0 = __dsub_rn(xval(X, xs, i0, ch, XS, scaled), r0[ch]);
            const double a1 = __dsub_rn(xval(X, xs, i1, ch, XS, scaled), r1[ch]);
            d0 = __dadd_rn(d0, __dmul_rn(a0, a0));
            d1 = __dadd_rn(d1, __dmul_rn(a1, a1));
          }
        }
        D2[(int64_t)i0 * K + s.ccols[c0 + j0]] = d0;
        if (v1) D2[(int64_t)i1 * K + s.ccols[c0 + j1]] = d1;
      }
      __syncthreads();
    }
    return;
  }
  if (nc <= 16) {
    for (int t = threadIdx.x; t < m * nc; t += 2 * NT) {
      const int t2 = t + NT;
      const bool v1 = t2 < m * nc;
      const int i0 = t / nc, c0 = s.ccols[t % nc];
      const int i1 = v1 ? t2 / nc : i0, c1 = v1 ? s.ccols[t2 % nc] : c0;
      const double* r0 = C + (int64_t)c0 * cstride;
      const double* r1 = C + (int64_t)c1 * cstride;
      double d0 = 0.0, d1 = 0.0;
      #pragma unroll 8
      for (int ch = 0; ch < D; ++ch) {
        const double t0 = __dsub_rn(xval(X, xs, i0, ch, XS, scaled), r0[ch]);
        const double t1 = __dsub_rn(xval(X, xs, i1, ch, XS, scaled), r1[ch]);
        d0 = __dadd_rn(d0, __dmul_rn(t0, t0));
        d1 = __dadd_rn(d1, __dmul_rn(t1, t1));
      }
      D2[(int64_t)i0 * K + c0] = d0;
      if (v1) D2[(int64_t)i1 * K + c1] = d1;
    }
    return;
  }
  // warp task = 4 points x 64 compute columns (lane l -> list entries l, l + 32)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pblocks = (m + 3) / 4, cgroups = (nc + 63) / 64;
  for (int task = warp; task < pblocks * cgroups; task += NT / 32) {
    const int pb = task / cgroups, cg = task % cgroups;
    const int j0 = cg * 64 + lane, j1 = j0 + 32;
    const bool v0 = j0 < nc, v1 = j1 < nc;
    const int c0 = s.ccols[v0 ? j0 : 0], c1 = s.ccols[v1 ? j1 : 0];
    const double* r0 = C + (int64_t)c0 * cstride;
    const double* r1 = C + (int64_t)c1 * cstride;
    int ip[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) ip[q] = min(pb * 4 + q, m - 1);
    double d[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
    #pragma unroll 2
    for (int ch = 0; ch < D; ++ch) {
      const double a0 = r0[ch], a1 = r1[ch];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double x = xval(X, xs, ip[q], ch, XS, scaled);
        const double t0 = __dsub_rn(x, a0), t1 = __dsub_rn(x, a1);
        d[q][0] = __dadd_rn(d[q][0], __dmul_rn(t0, t0));
        d[q][1] = __dadd_rn(d[q][1], __dmul_rn(t1, t1));
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = pb * 4 + q;
      if (i >= m) break;
      if (v0) D2[(int64_t)i * K + c0] = d[q][0];
      if (v1) D2[(int64_t)i * K + c1] = d[q][1];
    }
  }
}

// Recompute D2 columns a and b (after a move or swap changed those means).
template <int NT, typename XT>
__device__ void refresh_cols(const XT* X, int XS, const double* xs, bool scaled, const double* ra, const double* rb,
                             double* D2, int m, int K, int D, int a, int b, bool shared_x = false) {
  if (shared_x) {  // one thread per point: the key channel is widened once for both chains
    for (int i = threadIdx.x; i < m; i += NT) {
      double da = 0.0, db = 0.0;
#pragma unroll 8
      for (int ch = 0; ch < D; ++ch) {
        const double x = xval(X, xs, i, ch, XS, scaled);
        const double ta = __dsub_rn(x, ra[ch]), tb = __dsub_rn(x, rb[ch]);
        da = __dadd_rn(da, __dmul_rn(ta, ta));
        db = __dadd_rn(db, __dmul_rn(tb, tb));
      }
      D2[(int64_t)i * K + a] = da;
      D2[(int64_t)i * K + b] = db;
    }
    return;
  }
  for (int t = threadIdx.x; t < 2 * m; t += NT) {
    const int i = t >> 1, c = (t & 1) ? b : a;
    const double* cr = (t & 1) ? rb : ra;
    double d = 0.0;
    #pragma unroll 8
    for (int ch = 0; ch < D; ++ch) {
      const double tt = __dsub_rn(xval(X, xs, i, ch, XS, scaled), cr[ch]);
      d = __dadd_rn(d, __dmul_rn(tt, tt));
    }
    D2[(int64_t)i * K + c] = d;
  }
}

// |mean_of(c)|^2 of one cluster (one warp; any summation order: it only
// scales the swap pre-filter's error bound).
template <typename SM>
__device__ __forceinline__ void mean_norm(SM& s, const double* row, int c, int D, int lane) {
  double acc = 0.0;
  for (int ch = lane; ch < D; ch += 32) acc += row[ch] * row[ch];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) s.m2[c] = acc;
}

// Row i of pair rank p in the lexicographic order of pairs (i < j < m):
// prow(i) = i (2m - i - 1) / 2 <= p < prow(i + 1).  Closed form from the
// quadratic, then corrected with exact integer comparisons.
__device__ __forceinline__ int pair_row(int p, int m) {
  const float b = (float)(2 * m - 1);
  int i = (int)((b - sqrtf(b * b - 8.0f * (float)p)) * 0.5f);
  i = max(0, min(i, m - 2));
  while (i > 0 && i * (2 * m - i - 1) / 2 > p) --i;
  while (i < m - 2 && (i + 1) * (2 * m - i - 2) / 2 <= p) ++i;
  return i;
}

// Member lists per cluster in ascending point order (offs/order).
template <typename SM>
__device__ void members(SM& s, int m, int K) {
  if (threadIdx.x == 0) {
    s.offs[0] = 0;
    for (int c = 0; c < K; ++c) {
      s.offs[c + 1] = s.offs[c] + s.sizes[c];
      s.cur[c] = s.offs[c];
    }
    for (int i = 0; i < m; ++i) s.order[s.cur[s.assign[i]]++] = i;
  }
  __syncthreads();
}

// Parallel member lists (sizes, offs, order ascending within each cluster)
// from s.assign: match_any ranks inside each 32-point warp, per-warp counts
// scanned per cluster, offsets scanned by warp 0.  Needs NT >= m; s.cand is
// the [point-warps][K] count scratch (free outside the swap scan).
template <int NT, typename SM>
__device__ void members_par(SM& s, int m, int K) {
  const int W = (m + 31) / 32;
  int* wc = s.cand;
  if (W * K > (int)(sizeof(s.cand) / sizeof(int))) {  // (not reached for tau <= 128)
    if (threadIdx.x == 0) {
      for (int c = 0; c < K; ++c) s.sizes[c] = 0;
      for (int i = 0; i < m; ++i) ++s.sizes[s.assign[i]];
    }
    __syncthreads();
    members(s, m, K);
    return;
  }
  for (int t = threadIdx.x; t < W * K; t += NT) wc[t] = 0;
  __syncthreads();
  const int i = threadIdx.x, ln = threadIdx.x & 31;
  int a = -1, rank = 0;
  if (i < W * 32) {  // whole warps
    a = i < m ? s.assign[i] : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, a);
    rank = __popc(peers & ((1u << ln) - 1u));
    if (i < m && rank == 0) wc[(i >> 5) * K + a] = __popc(peers);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < K; c += NT) {
    int run = 0;
    for (int w = 0; w < W; ++w) {
      const int x = wc[w * K + c];
      wc[w * K + c] = run;
      run += x;
    }
    s.sizes[c] = run;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    int carry = 0;
    for (int c0 = 0; c0 < K; c0 += 32) {
      const int c = c0 + ln;
      const int x = c < K ? s.sizes[c] : 0;
      int incl = x;
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (ln >= o) incl += y;
      }
      if (c < K) s.offs[c] = carry + incl - x;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (ln == 0) s.offs[K] = carry;
  }
  __syncthreads();
  if (i < m) s.order[s.offs[a] + wc[(i >> 5) * K + a] + rank] = i;
  __syncthreads();
}

// Lloyd assignment: nearest centroid per point, ties to the lowest index
// (evictor.cpp:106-117); up to 8 lanes per point scan interleaved columns.
template <int NT, typename SM>
__device__ void assign_nearest(SM& s, const double* D2, int m, int K) {
  int tpp = 1;
  while (tpp < 8 && tpp * 2 * m <= NT) tpp *= 2;
  const int i = threadIdx.x / tpp, part = threadIdx.x % tpp;
  double bd = CUDART_INF;
  int best = 0x7fffffff;
  if (i < m) {
    const double* row = D2 + (int64_t)i * K;
    for (int c = part; c < K; c += tpp)
      if (best == 0x7fffffff || row[c] < bd) { bd = row[c]; best = c; }
  }
  for (int o = 1; o < tpp; o <<= 1) {
    const double od = __shfl_xor_sync(0xffffffffu, bd, o);
    const int ob = __shfl_xor_sync(0xffffffffu, best, o);
    if (od < bd || (od == bd && ob < best)) { bd = od; best = ob; }
  }
  if (i < m && part == 0) s.assign[i] = best;
}

template <int NT, int MAXM, typename XT>
__global__ void __launch_bounds__(NT, NT == 256 ? (MAXM == 128 ? 2 : 3) : NT == 128 ? (MAXM == 64 ? 5 : 4) : NT == 64 ? 8 : 1)
    km_restart_kernel(TkvState st, const TkvAnnealOp* __restrict__ ops, int nops,
                                                        const int32_t* __restrict__ rprefix, int nruns, int run0,
                                                        const int32_t* __restrict__ item_prefix, int item0,
                                                        uint8_t* __restrict__ scratch, KmGeo geo,
                                                        double* __restrict__ gsums, int scaled_any) {
  const TkvDims& dm = st.dm;
  const int run = run0 + blockIdx.x;
  if (run >= nruns) return;
  // run -> (op, unit, restart): rprefix[op] = first run of op; runs of an op
  // are unit-major: run = rprefix[op] + urel * nrestart_eff + r.
  const int oi = find_op(rprefix, nops, run);
  const TkvAnnealOp op = ops[oi];
  const int nr = op.nrestart > 0 ? op.nrestart : op.ncombos;
  const int local = run - rprefix[oi];
  const int urel = local / nr, r = local % nr;
  const int item = item_prefix[oi] + urel - item0;  // scratch slot of the instance
  uint8_t* base = scratch + (int64_t)item * geo.bytes();
  const int32_t* misc = reinterpret_cast<const int32_t*>(base + geo.misc_off());
  if (misc[1]) return;
  const int m = misc[0], K = op.K, D = dm.D;
  const bool scaled = scaled_any != 0;
  // kMG (the 128-point class at two 256-thread CTAs per SM): the means live in
  // the CTA's global row block; the rows a fill or a refresh needs are staged
  // in shared memory (kStg rows).
  constexpr bool kMG = (NT == 256 && MAXM == 128) || (NT == 128 && MAXM == 64);
  constexpr int kStg = 4;
  extern __shared__ __align__(16) uint8_t dyn[];
  __shared__ RsSmem<MAXM> s;
  double* xs = s.xs;
  // smem: X f32/f16 [m][XS] | means f64 [K][D+1] (not kMG) | D2 f64 [m][K] | staged rows [kStg][D+1] (kMG)
  // (rows padded by one word so column-wise accesses across lanes are conflict-free)
  const int XS = D + 4 / (int)sizeof(XT), MS = D + 1;
  XT* X = reinterpret_cast<XT*>(dyn);
  double* after_x = reinterpret_cast<double*>(dyn + (((int64_t)geo.mmax * XS * sizeof(XT) + 15) / 16 * 16));
  double* gblk = gsums + (int64_t)blockIdx.x * geo.kmax * (kMG ? 2 * D + 1 : D);
  double* Mn = kMG ? gblk + (int64_t)geo.kmax * D : after_x;
  double* D2 = kMG ? after_x : Mn + (int64_t)geo.kmax * MS;
  double* Stg = D2 + (int64_t)geo.mmax * geo.kmax;
  // sums / next: shared memory for small instances, else a global row block per CTA
  double* S = MAXM <= 32 ? D2 + (int64_t)geo.mmax * geo.kmax : gblk;
  const float* gX = reinterpret_cast<const float*>(base + geo.x_off());
  const double* gxs = reinterpret_cast<const double*>(base + geo.xs_off());
  const double* pd = reinterpret_cast<const double*>(base + geo.pd_off());
  const RowSplit rs(D);
  for (int i = threadIdx.x; i < m * D; i += NT) X[rs.row(i) * XS + rs.col(i)] = (XT)gX[i];
  for (int i = threadIdx.x; i < m; i += NT) xs[i] = gxs[i];
  for (int n = threadIdx.x; n <= MAXM; n += NT) {
    const double dn = (double)n;
    s.tabA[n] = __ddiv_rn(dn, __dadd_rn(dn, 1.0));
    s.tabR[n] = __ddiv_rn(-dn, __dsub_rn(dn, 1.0));
  }
  if (threadIdx.x == 0) {
    if (op.nrestart > 0) {
      const int32_t* sd = reinterpret_cast<const int32_t*>(base + geo.seeds_off()) + r * geo.kmax;
      for (int c = 0; c < K; ++c) s.seeds[c] = sd[c];
    } else {
      // r-th K-subset of {0..m-1} in lexicographic order (evictor.cpp:274-283)
      int rank = r, x = 0;
      for (int c = 0; c < K; ++c) {
        while (true) {
          // number of subsets starting with x at position c
          int cnt = 1;  // C(n, k) <= 512 in exact integers (each step divides exactly)
          const int n = m - x - 1, k = K - c - 1;
          for (int t = 0; t < k; ++t) cnt = cnt * (n - t) / (t + 1);
          const int ci = (int)cnt;
          if (rank < ci) break;
          rank -= ci;
          ++x;
        }
        s.seeds[c] = x;
        ++x;
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += NT) {  // |x_i|^2 (bound only: any order)
    double acc = 0.0;
    for (int ch = 0; ch < D; ++ch) {
      const double x = xval(X, xs, i, ch, XS, scaled);
      acc += x * x;
    }
    s.x2[i] = acc;
  }
  const long long t0 = clock64();
  kstm(st, m, 3, 1);
  // ---- Lloyd (evictor.cpp:102-159) ----------------------------------------
  for (int idx = threadIdx.x; idx < K * D; idx += NT) {
    const int c = rs.row(idx), ch = rs.col(idx);
    Mn[(int64_t)c * MS + ch] = xval(X, xs, s.seeds[c], ch, XS, scaled);
  }
  for (int c = threadIdx.x; c < K; c += NT) s.colsrc[c] = s.seeds[c];  // centroids are points
  __syncthreads();
  for (int iter = 0; iter < 50; ++iter) {
    kstm(st, m, 4, 1);
    for (int c = threadIdx.x; c < K; c += NT) s.mv[c] = 0.0;
    const long long tl0 = clock64();
    fill_sel<NT>(s, X, XS, xs, scaled, Mn, MS, D2, pd, geo.mmax, m, K, D, kMG ? Stg : nullptr, kStg);
    __syncthreads();
    const long long tl1 = clock64();
    kstm(st, m, 16, (unsigned long long)(tl1 - tl0));
    assign_nearest<NT>(s, D2, m, K);
    __syncthreads();
    members_par<NT>(s, m, K);
    if (__syncthreads_or(threadIdx.x < K && s.sizes[threadIdx.x] == 0)) {
      if (threadIdx.x == 0) {
      for (int c = 0; c < K; ++c) {  // empty-cluster repair (evictor.cpp:123-141)
        if (s.sizes[c] > 0) continue;
        int donor = 0;
        for (int d2 = 1; d2 < K; ++d2)
          if (s.sizes[d2] > s.sizes[donor]) donor = d2;
        int steal = m;
        double steal_d = -1.0;
        for (int i = 0; i < m; ++i) {
          if (s.assign[i] != donor) continue;
          const double d = D2[(int64_t)i * K + donor];
          if (d > steal_d) { steal = i; steal_d = d; }
        }
        s.assign[steal] = c;
        --s.sizes[donor];
        ++s.sizes[c];
      }
      }
      __syncthreads();
      members_par<NT>(s, m, K);
    }
    const long long tl2 = clock64();
    kstm(st, m, 17, (unsigned long long)(tl2 - tl1));
    if constexpr (MAXM > 32) {  // sums rows in global memory: no read-back chains
    // A cluster whose member set equals the previous iteration's has the same
    // sum (same members, same order) and so the same mean, bit for bit: its
    // next centroid is its current one, movement exactly 0 -- skipped.
    // Changed clusters are flagged in s.ccols (free outside fill_sel); the
    // previous assignment is kept in s.seeds (dead after the first fill).
    for (int c = threadIdx.x; c < K; c += NT) s.ccols[c] = iter == 0;
    __syncthreads();
    if (iter > 0)
      for (int i = threadIdx.x; i < m; i += NT)
        if (s.assign[i] != s.seeds[i]) {
          s.ccols[s.assign[i]] = 1;
          s.ccols[s.seeds[i]] = 1;
        }
    __syncthreads();
    for (int i = threadIdx.x; i < m; i += NT) s.seeds[i] = s.assign[i];
    // next centroids (member sums in point order / size, evictor.cpp:143-152)
    // written in place, and the movement terms (next - old)^2 (evictor.cpp:
    // 153-156) summed per column in any order: only "d == 0" (exact for a sum
    // of non-negative terms) and "sqrt(d) < 1e-6" (decided with a relative
    // margin, else by the channel-order sum from the saved old centroid) are used.
    // Four items per thread at a time, their old centroid values loaded
    // first (independent loads in flight instead of one dependent chain per
    // item); warps whose centroid row is unchanged skip the reduction.
    constexpr int kU = (NT == 256 && MAXM == 128) ? 4 : 1;  // (the 64-point classes spill with more)
    for (int base = 0; base < K * D; base += kU * NT) {
      int cc[kU];
      bool act[kU];
      double old[kU];
#pragma unroll
      for (int k = 0; k < kU; ++k) {
        const int idx = base + k * NT + threadIdx.x;
        const bool valid = idx < K * D;
        cc[k] = valid ? rs.row(idx) : -1;
        act[k] = valid && s.ccols[cc[k]];
        old[k] = act[k] ? Mn[(int64_t)cc[k] * MS + rs.col(idx)] : 0.0;
      }
#pragma unroll
      for (int k = 0; k < kU; ++k) {
        const int idx = base + k * NT + threadIdx.x;
        double t2 = 0.0;
        if (act[k]) {
          const int c = cc[k], ch = rs.col(idx);
          double acc = 0.0;
          for (int q = s.offs[c]; q < s.offs[c + 1]; ++q) acc = __dadd_rn(acc, xval(X, xs, s.order[q], ch, XS, scaled));
          const double nx = div_n(acc, s.sizes[c]);
          const double t = __dsub_rn(nx, old[k]);
          t2 = __dmul_rn(t, t);
          S[idx] = old[k];
          Mn[(int64_t)c * MS + ch] = nx;
        }
        if (!__any_sync(0xffffffffu, act[k])) continue;
        const int c0 = __shfl_sync(0xffffffffu, cc[k], 0);
        if (__all_sync(0xffffffffu, cc[k] == c0)) {
          for (int o = 16; o > 0; o >>= 1) t2 += __shfl_xor_sync(0xffffffffu, t2, o);
          if ((threadIdx.x & 31) == 0 && c0 >= 0) atomicAdd(&s.mv[c0], t2);
        } else if (act[k]) {
          atomicAdd(&s.mv[cc[k]], t2);
        }
      }
    }
    __syncthreads();
    for (int c = threadIdx.x; c < K; c += NT) {
      double d = s.mv[c];
      int code;  // 0: unchanged, 1: moved below the tolerance, 2: moved at or above it
      if (d == 0.0) {
        code = 0;
      } else if (__dsqrt_rn(d * (1.0 + 1e-12)) < 1e-6) {
        code = 1;
      } else if (!(__dsqrt_rn(d * (1.0 - 1e-12)) < 1e-6)) {
        code = 2;
      } else {  // within rounding of the tolerance: the reference's channel-order sum
        d = 0.0;
        for (int ch = 0; ch < D; ++ch) {
          const double t = __dsub_rn(Mn[(int64_t)c * MS + ch], S[(int64_t)c * D + ch]);
          d = __dadd_rn(d, __dmul_rn(t, t));
        }
        code = __dsqrt_rn(d) < 1e-6 ? 1 : 2;
      }
      s.cur[c] = code;
      // next fill: unchanged centroid -> keep; singleton (0 + x) / 1 = x -> pd column
      s.colsrc[c] = code == 0 ? kColKeep : (s.sizes[c] == 1 ? s.order[s.offs[c]] : kColCompute);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int mx = 0;
      for (int c = 0; c < K; ++c) mx = mx < s.cur[c] ? s.cur[c] : mx;
      s.flag = mx < 2;               // movement < 1e-6
      s.cost = mx > 0 ? 1.0 : 0.0;   // movement != 0: the final means differ from the last fill's
    }
    __syncthreads();
    } else {  // shared-memory sums: channel-order movement per centroid
    for (int idx = threadIdx.x; idx < K * D; idx += NT) {
      const int c = rs.row(idx), ch = rs.col(idx);
      double acc = 0.0;
      for (int q = s.offs[c]; q < s.offs[c + 1]; ++q) acc = __dadd_rn(acc, xval(X, xs, s.order[q], ch, XS, scaled));
      S[idx] = div_n(acc, s.sizes[c]);
    }
    __syncthreads();
    for (int c = threadIdx.x; c < K; c += NT) {
      double d = 0.0;
      #pragma unroll 8
      for (int ch = 0; ch < D; ++ch) {
        const double t = __dsub_rn(S[(int64_t)c * D + ch], Mn[(int64_t)c * MS + ch]);
        d = __dadd_rn(d, __dmul_rn(t, t));
      }
      s.mv[c] = __dsqrt_rn(d);
      // next fill: unchanged centroid -> keep; singleton (0 + x) / 1 = x -> pd column
      s.colsrc[c] = d == 0.0 ? kColKeep : (s.sizes[c] == 1 ? s.order[s.offs[c]] : kColCompute);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double movement = 0.0;
      for (int c = 0; c < K; ++c) movement = movement < s.mv[c] ? s.mv[c] : movement;
      s.flag = movement < 1e-6;
      s.cost = movement;  // == 0 exactly: the next centroids equal the ones D2 was filled with
    }
    for (int idx = threadIdx.x; idx < K * D; idx += NT) Mn[rs.row(idx) * MS + rs.col(idx)] = S[idx];
    __syncthreads();
    }
    kstm(st, m, 18, (unsigned long long)(clock64() - tl2));
    if (s.flag) break;
  }
  const long long t1 = clock64();
  kstm(st, m, 5, (unsigned long long)(t1 - t0));
  // ---- Hartigan (evictor.cpp:167-243) --------------------------------------
  members_par<NT>(s, m, K);
  for (int idx = threadIdx.x; idx < K * D; idx += NT) {
    const int c = rs.row(idx), ch = rs.col(idx);
    double acc = 0.0;
    for (int q = s.offs[c]; q < s.offs[c + 1]; ++q) acc = __dadd_rn(acc, xval(X, xs, s.order[q], ch, XS, scaled));
    S[idx] = acc;
    Mn[(int64_t)c * MS + ch] = div_n(acc, s.sizes[c]);
  }
  __syncthreads();
  // Lloyd's last update left colsrc describing the final centroids (= these means)
  if (s.cost != 0.0) fill_sel<NT>(s, X, XS, xs, scaled, Mn, MS, D2, pd, geo.mmax, m, K, D, kMG ? Stg : nullptr, kStg);
  for (int c = threadIdx.x >> 5; c < K; c += NT / 32) mean_norm(s, Mn + (int64_t)c * MS, c, D, threadIdx.x & 31);
  __syncthreads();
  kstm(st, m, 6, (unsigned long long)(clock64() - t1));
  long long tmove = 0, tswap = 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int pass = 0; pass < 100; ++pass) {
    kstm(st, m, 7, 1);
    const long long tp = clock64();
    bool moved = false;  // CTA-uniform
    int start = 0;
    while (true) {
      // Each warp evaluates one of the next NT/32 points against the cached
      // distances; no state changes before the first improving point, so all
      // decisions up to it are exactly the sequential ones (evictor.cpp:196-212).
      {
        const int i = start + warp;
        int mto = -1;
        if (i < m) {
          const int from = s.assign[i];
          if (s.sizes[from] > 1) {
            const double* row = D2 + (int64_t)i * K;
            const double removal = __dmul_rn(s.tabR[s.sizes[from]], row[from]);
            double bd = -1e-12;
            int bt = 0x7fffffff;
            for (int to = lane; to < K; to += 32) {
              if (to == from) continue;
              const double delta = __dadd_rn(removal, __dmul_rn(s.tabA[s.sizes[to]], row[to]));
              if (delta < bd) { bd = delta; bt = to; }
            }
            for (int o = 16; o > 0; o >>= 1) {
              const double od = __shfl_xor_sync(0xffffffffu, bd, o);
              const int ot = __shfl_xor_sync(0xffffffffu, bt, o);
              if (od < bd || (od == bd && ot < bt)) { bd = od; bt = ot; }
            }
            if (bt != 0x7fffffff) mto = bt;
          }
        }
        if (lane == 0) s.res[warp] = mto;
      }
      __syncthreads();
      if (warp == 0) {  // first warp (point order) holding an improving move
        const int r = (lane < NT / 32 && start + lane < m) ? s.res[lane] : -1;
        const unsigned any = __ballot_sync(0xffffffffu, r >= 0);
        if (lane == 0) {
          const int fw = any ? __ffs(any) - 1 : -1;
          s.move_i = fw >= 0 ? start + fw : -1;
          s.move_to = fw >= 0 ? s.res[fw] : -1;
          s.flag = fw >= 0 ? start + fw + 1 : start + NT / 32;
        }
      }
      __syncthreads();
      const int i = s.move_i, to = s.move_to;
      start = s.flag;
      if (i < 0) {
        if (start >= m) break;
        continue;
      }
      const int from = s.assign[i];
      const int nf = s.sizes[from] - 1, nt = s.sizes[to] + 1;
      kstm(st, m, 8, 1);
      moved = true;
      const long long tu0 = clock64();
      __syncthreads();
      if (threadIdx.x == 0) {
        s.sizes[from] = nf;
        s.sizes[to] = nt;
        s.assign[i] = to;
      }
      // apply_move (evictor.cpp:189-196) and mean_of for the two clusters
      for (int ch = threadIdx.x; ch < D; ch += NT) {
        const double x = xval(X, xs, i, ch, XS, scaled);
        const double sf = __dsub_rn(S[(int64_t)from * D + ch], x);
        const double sto = __dadd_rn(S[(int64_t)to * D + ch], x);
        S[(int64_t)from * D + ch] = sf;
        S[(int64_t)to * D + ch] = sto;
        const double mf = div_n(sf, nf), mt = div_n(sto, nt);
        Mn[(int64_t)from * MS + ch] = mf;
        Mn[(int64_t)to * MS + ch] = mt;
        if constexpr (kMG) {
          Stg[ch] = mf;
          Stg[MS + ch] = mt;
        }
      }
      __syncthreads();
      const long long tu1 = clock64();
      {
        const double* ra = kMG ? Stg : Mn + (int64_t)from * MS;
        const double* rb = kMG ? Stg + MS : Mn + (int64_t)to * MS;
        refresh_cols<NT>(X, XS, xs, scaled, ra, rb, D2, m, K, D, from, to, kMG);
        for (int q = threadIdx.x >> 5; q < 2; q += NT / 32) mean_norm(s, q ? rb : ra, q ? to : from, D, threadIdx.x & 31);
      }
      __syncthreads();
      kstm(st, m, 0, (unsigned long long)(tu1 - tu0));          // move update
      kstm(st, m, 2, (unsigned long long)(clock64() - tu1));    // column refresh
    }
    tmove += clock64() - tp;
    if (moved) continue;
    const long long ts = clock64();
    kstm(st, m, 9, 1);
    // ---- pairwise swaps: first improving (i, j) in lexicographic order ------
    if (threadIdx.x == 0) s.pair = 0x7fffffff;
    // Pairs in lexicographic-rank windows of kSwapWin: filter (O(1) per pair
    // from D2 and pd) into a candidate list, evaluate the candidates exactly
    // in parallel, stop at the first window holding an improving pair.
    const int npairs = m * (m - 1) / 2;
    long long tfilt = 0;
    for (int p0 = 0, wi = 0; p0 < npairs; p0 += RsSmem<MAXM>::WIN, wi ^= 1) {
      int& ncand = s.ncand[wi];
      if (threadIdx.x == 0) ncand = 0;
      __syncthreads();
      const long long tf0 = clock64();
      for (int p = p0 + threadIdx.x; p < min(npairs, p0 + RsSmem<MAXM>::WIN); p += NT) {
        const int i = pair_row(p, m), j = i + 1 + (p - i * (2 * m - i - 1) / 2);
        const int a = s.assign[i], b = s.assign[j];
        if (a == b) continue;
        // Two singletons with f16 keys: x_j - x_i is exact in fp64 (f16
        // significands and exponent range), so ma == x_j, mb == x_i and every
        // term of evictor.cpp:222-225 is exactly 0: not an improving swap.
        if (sizeof(XT) == 2 && !scaled && s.sizes[a] == 1 && s.sizes[b] == 1) continue;
        const double na = (double)s.sizes[a], nb = (double)s.sizes[b];
        const double w = 1.0 / na + 1.0 / nb;
        const double dja = D2[(int64_t)j * K + a], dia = D2[(int64_t)i * K + a];
        const double dib = D2[(int64_t)i * K + b], djb = D2[(int64_t)j * K + b];
        const double pij = pd[(int64_t)i * geo.mmax + j];
        const double approx = dja - dia + dib - djb - w * pij;
        // |approx - reference delta| is below (2D + 10) 2^-53 times the operand
        // magnitudes: distances, and per channel x_i^2 + x_j^2 + n (m^2 + mu^2)
        // (evictor.cpp:215-228), <= 14 (|x_i|^2 + |x_j|^2) + 3 (na |mu_a|^2 +
        // nb |mu_b|^2); 1e-12 covers D <= 256 with a >= 17x safety factor.
        const double margin = 1e-12 * (dja + dia + dib + djb + w * pij + 16.0 * (s.x2[i] + s.x2[j]) +
                                       4.0 * (na * s.m2[a] + nb * s.m2[b])) + 1e-12;
        if (approx >= -1e-12 + margin) continue;
        s.cand[atomicAdd(&ncand, 1)] = p;
      }
      __syncthreads();
      tfilt += clock64() - tf0;
      if (ncand == 0) continue;
      kstm(st, m, 10, (unsigned long long)ncand);
      // One warp per candidate: lanes evaluate the per-channel terms (the
      // divisions of different channels are independent), then the terms are
      // accumulated in the reference's channel order through shuffles.
      for (int c = warp; c < ncand; c += NT / 32) {
        const int p = s.cand[c];
        const int i = pair_row(p, m), j = i + 1 + (p - i * (2 * m - i - 1) / 2);
        const int a = s.assign[i], b = s.assign[j];
        const double na = (double)s.sizes[a], nb = (double)s.sizes[b];
        // exact reference expression (evictor.cpp:215-228)
        const double* mua = Mn + (int64_t)a * MS;
        const double* mub = Mn + (int64_t)b * MS;
        // (x / 1.0 == x and 1.0 * x == x exactly, so singleton clusters skip
        // the division and the multiply without changing any bit.)
        const bool ua = na == 1.0, ub = nb == 1.0;
        double TA[8], TB[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int ch = lane + 32 * k;
          TA[k] = TB[k] = 0.0;
          if (ch < D) {
            const double xi = xval(X, xs, i, ch, XS, scaled), xj = xval(X, xs, j, ch, XS, scaled);
            const double dji = __dsub_rn(xj, xi), dij = __dsub_rn(xi, xj);
            const double ma = __dadd_rn(mua[ch], div_n(dji, s.sizes[a]));
            const double mb = __dadd_rn(mub[ch], div_n(dij, s.sizes[b]));
            const double xx = __dsub_rn(__dmul_rn(xj, xj), __dmul_rn(xi, xi));
            const double yy = __dsub_rn(__dmul_rn(xi, xi), __dmul_rn(xj, xj));
            const double ta = __dsub_rn(__dmul_rn(ma, ma), __dmul_rn(mua[ch], mua[ch]));
            const double tb = __dsub_rn(__dmul_rn(mb, mb), __dmul_rn(mub[ch], mub[ch]));
            TA[k] = __dsub_rn(xx, ua ? ta : __dmul_rn(na, ta));
            TB[k] = __dsub_rn(yy, ub ? tb : __dmul_rn(nb, tb));
          }
        }
        // The ordered sum can only fall below -1e-12 if some term is negative
        // and the terms' absolute sum reaches it: a sum of non-negative terms
        // rounds to a non-negative value, and |fl(sum)| <= (1 + 2^-44) sum|t|.
        // Singleton-pair swaps (exact means) have all terms exactly zero.
        bool neg = false;
        double abssum = 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          neg = neg || TA[k] < 0.0 || TB[k] < 0.0;
          abssum += fabs(TA[k]) + fabs(TB[k]);
        }
        for (int o = 16; o > 0; o >>= 1) abssum += __shfl_xor_sync(0xffffffffu, abssum, o);
        if (!__any_sync(0xffffffffu, neg) || abssum < 5e-13) continue;
        if (st.kstats && lane == 0)
          atomicAdd(st.kstats + 32 + 32 * (m <= 8 ? 0 : m <= 16 ? 1 : m <= 32 ? 2 : m <= 64 ? 3 : 4) + 1, 1ull);
        double delta = 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (32 * k >= D) break;
          for (int l = 0; l < 32 && 32 * k + l < D; ++l) {
            delta = __dadd_rn(delta, __shfl_sync(0xffffffffu, TA[k], l));
            delta = __dadd_rn(delta, __shfl_sync(0xffffffffu, TB[k], l));
          }
        }
        if (lane == 0 && delta < -1e-12) atomicMin(&s.pair, p);
      }
      __syncthreads();
      if (s.pair != 0x7fffffff) break;
    }
    __syncthreads();
    const int p = s.pair;
    tswap += clock64() - ts;
    kstm(st, m, 15, (unsigned long long)tfilt);
    if (p == 0x7fffffff) break;
    int i = 0, rem = p;
    while (rem >= m - 1 - i) { rem -= m - 1 - i; ++i; }
    const int j = i + 1 + rem;
    const int a = s.assign[i], b = s.assign[j];
    for (int ch = threadIdx.x; ch < D; ch += NT) {
      const double xi = xval(X, xs, i, ch, XS, scaled), xj = xval(X, xs, j, ch, XS, scaled);
      const double sa = __dadd_rn(__dsub_rn(S[(int64_t)a * D + ch], xi), xj);
      const double sb = __dsub_rn(__dadd_rn(S[(int64_t)b * D + ch], xi), xj);
      S[(int64_t)a * D + ch] = sa;
      S[(int64_t)b * D + ch] = sb;
      const double ma = div_n(sa, s.sizes[a]), mb = div_n(sb, s.sizes[b]);
      Mn[(int64_t)a * MS + ch] = ma;
      Mn[(int64_t)b * MS + ch] = mb;
      if constexpr (kMG) {
        Stg[ch] = ma;
        Stg[MS + ch] = mb;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      s.assign[i] = b;
      s.assign[j] = a;
    }
    {
      const double* ra = kMG ? Stg : Mn + (int64_t)a * MS;
      const double* rb = kMG ? Stg + MS : Mn + (int64_t)b * MS;
      refresh_cols<NT>(X, XS, xs, scaled, ra, rb, D2, m, K, D, a, b, kMG);
      for (int q = threadIdx.x >> 5; q < 2; q += NT / 32) mean_norm(s, q ? rb : ra, q ? b : a, D, threadIdx.x & 31);
    }
    __syncthreads();
  }
  kstm(st, m, 11, (unsigned long long)tmove);
  kstm(st, m, 12, (unsigned long long)tswap);
  kstm(st, m, 13, (unsigned long long)(clock64() - t0));
  kstm(st, m, 14, (unsigned long long)m);
  // ---- cost (point order) and medoids --------------------------------------
  if (threadIdx.x == 0) {
    double c = 0.0;
    for (int i = 0; i < m; ++i) c = __dadd_rn(c, D2[(int64_t)i * K + s.assign[i]]);
    s.cost = c;
  }
  for (int c = threadIdx.x; c < K; c += NT) {
    int bi = m;
    double bd = CUDART_INF;
    for (int i = 0; i < m; ++i) {
      if (s.assign[i] != c) continue;
      const double d = D2[(int64_t)i * K + c];
      if (d < bd) { bd = d; bi = i; }
    }
    s.order[c] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double* cost = reinterpret_cast<double*>(base + geo.cost_off());
    uint32_t* mask = reinterpret_cast<uint32_t*>(base + geo.mask_off()) + (int64_t)r * geo.W;
    const int32_t* ids = reinterpret_cast<const int32_t*>(base + geo.ids_off());
    for (int w = 0; w < geo.W; ++w) mask[w] = 0;
    for (int c = 0; c < K; ++c) {
      const int b = ids[s.order[c]];
      mask[b >> 5] |= 1u << (b & 31);
    }
    cost[r] = s.cost;
  }
}


// ---------------------------------------------------------------------------
// tiny instances (m <= 8, e.g. the 8 -> 4 anneal with all C(8,4) = 70 seed
// subsets): one CTA per instance, one warp per restart (warps loop over the
// restarts), no block barriers after the shared key load.  Lanes = (point,
// centroid) pairs for the distance table, lanes = channels for sums/means,
// and the pairwise swaps (<= 28 pairs) are evaluated one per lane with the
// reference's exact expression (the state cannot change before the first
// improving pair, so the lowest improving pair index is the sequential pick).
// Same operations in the same order as kmeans_from_seeds (evictor.cpp:94-251).
// ---------------------------------------------------------------------------
constexpr int kTinyM = 8;
constexpr int kTinyWarps = 4;

struct TinyState {  // per warp, warp-uniform
  int assign[kTinyM];
  int sizes[kTinyM];
  unsigned members[kTinyM];
  int colsrc[kTinyM];
  int seeds[kTinyM];
  double m2[kTinyM];  // |mean_of(c)|^2 (swap-filter error bound)
};

// |mean_of(c)|^2 of the listed clusters (lanes = channels, any order).
__device__ __forceinline__ void tiny_norms(TinyState& w, const double* Mn, int D, int c0, int c1, int lane) {
  for (int q = 0; q < 2; ++q) {
    const int c = q ? c1 : c0;
    double acc = 0.0;
    for (int ch = lane; ch < D; ch += 32) acc += Mn[c * D + ch] * Mn[c * D + ch];
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) w.m2[c] = acc;
  }
  __syncwarp();
}

template <typename XT>
__device__ __noinline__ double tiny_dist(const XT* X, int XS, const double* xs, bool scaled, int i,
                                            const double* mu, int D) {
  double d = 0.0;
  #pragma unroll 2
  for (int ch = 0; ch < D; ++ch) {
    const double t = __dsub_rn(xval(X, xs, i, ch, XS, scaled), mu[ch]);
    d = __dadd_rn(d, __dmul_rn(t, t));
  }
  return d;
}

// d2 columns per colsrc (pd copy / keep / exact evaluation).
template <typename XT>
__device__ __forceinline__ void tiny_fill(const TinyState& w, const XT* X, int XS, const double* xs, bool scaled,
                                          const double (*pd)[kTinyM], const double* Mn, double* d2, int m, int K,
                                          int D, int lane) {
  for (int p = lane; p < m * K; p += 32) {
    const int i = p / K, c = p % K;
    const int src = w.colsrc[c];
    if (src >= 0) d2[p] = pd[i][src];
    else if (src == kColCompute) d2[p] = tiny_dist(X, XS, xs, scaled, i, Mn + c * D, D);
  }
  __syncwarp();
}

template <typename XT>
__global__ void __launch_bounds__(32 * kTinyWarps) km_tiny_kernel(TkvState st, const TkvAnnealOp* __restrict__ ops,
                                                                  int nops, const int32_t* __restrict__ item_prefix,
                                                                  int nitems, int item0, uint8_t* __restrict__ scratch,
                                                                  KmGeo geo, int scaled_any, int kmax) {
  const TkvDims& dm = st.dm;
  const int item = item0 + blockIdx.x;
  if (item >= nitems) return;
  const int oi = find_op(item_prefix, nops, item);
  const TkvAnnealOp op = ops[oi];
  uint8_t* base = scratch + (int64_t)blockIdx.x * geo.bytes();
  const int32_t* misc = reinterpret_cast<const int32_t*>(base + geo.misc_off());
  if (misc[1]) return;
  const int m = misc[0], K = op.K, D = dm.D;
  const bool scaled = scaled_any != 0;
  const int nr = op.nrestart > 0 ? op.nrestart : op.ncombos;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  extern __shared__ __align__(16) uint8_t dyn[];
  const int XS = D + 4 / (int)sizeof(XT);
  XT* X = reinterpret_cast<XT*>(dyn);
  __shared__ double xs[kTinyM];
  __shared__ double pd[kTinyM][kTinyM];
  __shared__ double tabA[kTinyM + 1], tabR[kTinyM + 1];  // n / (n + 1.0), -n / (n - 1.0) (evictor.cpp:201, 205)
  __shared__ double tx2[kTinyM];  // |x_i|^2 (swap-filter error bound)
  __shared__ TinyState ws[kTinyWarps];
  __shared__ uint32_t fin[512];  // final Lloyd assignment per restart (3 bits per point)
  __shared__ int uniq[512];
  __shared__ int nuniq;
  TinyState& w = ws[warp];
  double* Mn = reinterpret_cast<double*>(dyn + (((int64_t)kTinyM * XS * sizeof(XT) + 15) / 16 * 16)) +
               (int64_t)warp * (2 * kmax * D + kTinyM * kTinyM);
  double* S = Mn + (int64_t)kmax * D;
  double* d2 = S + (int64_t)kmax * D;  // [i * K + c]
  {
    const float* gX = reinterpret_cast<const float*>(base + geo.x_off());
    const double* gxs = reinterpret_cast<const double*>(base + geo.xs_off());
    const double* gpd = reinterpret_cast<const double*>(base + geo.pd_off());
    const RowSplit rs(D);
    for (int i = threadIdx.x; i < m * D; i += blockDim.x) X[rs.row(i) * XS + rs.col(i)] = (XT)gX[i];
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
      xs[i] = gxs[i];
      double acc = 0.0;
      for (int ch = 0; ch < D; ++ch) {
        const double x = scaled_any ? (double)gX[(int64_t)i * D + ch] * gxs[i] : (double)gX[(int64_t)i * D + ch];
        acc += x * x;
      }
      tx2[i] = acc * 1.000001;
    }
    for (int t = threadIdx.x; t < m * m; t += blockDim.x) pd[t / m][t % m] = gpd[(int64_t)(t / m) * geo.mmax + t % m];
    for (int n = threadIdx.x; n <= kTinyM; n += blockDim.x) {
      const double dn = (double)n;
      tabA[n] = __ddiv_rn(dn, __dadd_rn(dn, 1.0));
      tabR[n] = __ddiv_rn(-dn, __dsub_rn(dn, 1.0));
    }
  }
  __syncthreads();
  const RowSplit rsd(D);  // idx -> (centroid, channel) without integer division
  long long tk0 = clock64();
  for (int r = warp; r < nr; r += kTinyWarps) {
    // ---- seeds -------------------------------------------------------------------
    if (lane == 0) {
      if (op.nrestart > 0) {
        const int32_t* sd = reinterpret_cast<const int32_t*>(base + geo.seeds_off()) + r * geo.kmax;
        for (int c = 0; c < K; ++c) w.seeds[c] = sd[c];
      } else {
        // r-th K-subset of {0..m-1} in lexicographic order (evictor.cpp:274-283)
        int rank = r, x = 0;
        for (int c = 0; c < K; ++c) {
          while (true) {
            int cnt = 1;  // C(n, k) <= 512 in exact integers (each step divides exactly)
            const int n = m - x - 1, k = K - c - 1;
            for (int t = 0; t < k; ++t) cnt = cnt * (n - t) / (t + 1);
            const int ci = (int)cnt;
            if (rank < ci) break;
            rank -= ci;
            ++x;
          }
          w.seeds[c] = x;
          ++x;
        }
      }
      for (int c = 0; c < K; ++c) w.colsrc[c] = w.seeds[c];  // centroids are points
    }
    __syncwarp();
    for (int idx = lane; idx < K * D; idx += 32) {
      const int c = rsd.row(idx), ch = rsd.col(idx);
      Mn[idx] = xval(X, xs, w.seeds[c], ch, XS, scaled);
    }
    __syncwarp();
    // ---- Lloyd (evictor.cpp:102-159) ------------------------------------------------
    for (int iter = 0; iter < 50; ++iter) {
      tiny_fill(w, X, XS, xs, scaled, pd, Mn, d2, m, K, D, lane);
      int a = 0;
      if (lane < m) {  // nearest centroid, ties to the lowest index
        double bd = d2[lane * K];
        for (int c = 1; c < K; ++c)
          if (d2[lane * K + c] < bd) { bd = d2[lane * K + c]; a = c; }
        w.assign[lane] = a;
      }
      for (int c = 0; c < K; ++c) {
        const unsigned mb = __ballot_sync(0xffffffffu, lane < m && a == c);
        if (lane == 0) { w.members[c] = mb; w.sizes[c] = __popc(mb); }
      }
      __syncwarp();
      if (lane == 0) {  // empty-cluster repair (evictor.cpp:123-141)
        for (int c = 0; c < K; ++c) {
          if (w.sizes[c] > 0) continue;
          int donor = 0;
          for (int d = 1; d < K; ++d)
            if (w.sizes[d] > w.sizes[donor]) donor = d;
          int steal = m;
          double steal_d = -1.0;
          for (int i = 0; i < m; ++i) {
            if (w.assign[i] != donor) continue;
            const double d = d2[i * K + donor];
            if (d > steal_d) { steal = i; steal_d = d; }
          }
          w.assign[steal] = c;
          w.members[donor] &= ~(1u << steal);
          w.members[c] |= 1u << steal;
          --w.sizes[donor];
          ++w.sizes[c];
        }
      }
      __syncwarp();
      // next centroids: member sums in point order / size (lanes = channels)
      for (int idx = lane; idx < K * D; idx += 32) {
        const int c = rsd.row(idx), ch = rsd.col(idx);
        double acc = 0.0;
        unsigned mm = w.members[c];
        while (mm) {
          const int i = __ffs(mm) - 1;
          mm &= mm - 1;
          acc = __dadd_rn(acc, xval(X, xs, i, ch, XS, scaled));
        }
        S[idx] = div_n_ool(acc, w.sizes[c]);
      }
      __syncwarp();
      // movement per centroid (evictor.cpp:153-156): the terms (next - old)^2
      // summed across lanes in any order decide "== 0" exactly (non-negative
      // terms) and "sqrt < 1e-6" with a relative margin; a sum within the
      // margin is redone in channel order by one lane.  Next fill's columns.
      int code_max = 0;
      for (int c = 0; c < K; ++c) {
        double part = 0.0;
        for (int ch = lane; ch < D; ch += 32) {
          const double t = __dsub_rn(S[c * D + ch], Mn[c * D + ch]);
          part += __dmul_rn(t, t);
        }
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        int code;
        if (part == 0.0) {
          code = 0;
        } else if (__dsqrt_rn(part * (1.0 + 1e-12)) < 1e-6) {
          code = 1;
        } else if (!(__dsqrt_rn(part * (1.0 - 1e-12)) < 1e-6)) {
          code = 2;
        } else {
          double d = 0.0;
          if (lane == 0)
            for (int ch = 0; ch < D; ++ch) {
              const double t = __dsub_rn(S[c * D + ch], Mn[c * D + ch]);
              d = __dadd_rn(d, __dmul_rn(t, t));
            }
          code = __shfl_sync(0xffffffffu, __dsqrt_rn(d) < 1e-6 ? 1 : 2, 0);
        }
        if (lane == 0)
          w.colsrc[c] = code == 0 ? kColKeep : (w.sizes[c] == 1 ? __ffs(w.members[c]) - 1 : kColCompute);
        code_max = code_max > code ? code_max : code;
      }
      for (int idx = lane; idx < K * D; idx += 32) Mn[idx] = S[idx];
      __syncwarp();
      if (code_max < 2) break;  // movement < 1e-6
    }
    // Hartigan's input is the final Lloyd assignment alone (its sums, means and
    // distances are recomputed from it, evictor.cpp:167-187), so restarts that
    // end Lloyd with the same assignment produce identical results: record it
    // and run the refinement once per distinct assignment (phase 2).
    if (lane == 0) {
      uint32_t code = 0;
      for (int i = 0; i < m; ++i) code |= (uint32_t)w.assign[i] << (3 * i);
      fin[r] = code;
    }
    __syncwarp();
  }
  __syncthreads();
  if (st.kstats && lane == 0) { atomicAdd(st.kstats + 32 + 5, (unsigned long long)(clock64() - tk0)); atomicAdd(st.kstats + 32 + 3, (unsigned long long)((nr - warp + kTinyWarps - 1) / kTinyWarps)); }
  // distinct final assignments, first occurrence (lowest restart) first; a
  // later duplicate has the same cost and loses the tie to it (evictor.cpp:319-325)
  if (threadIdx.x == 0) nuniq = 0;
  __syncthreads();
  for (int r = threadIdx.x; r < nr; r += blockDim.x) {
    bool first = true;
    for (int r2 = 0; r2 < r && first; ++r2) first = fin[r2] != fin[r];
    if (first) uniq[atomicAdd(&nuniq, 1)] = r;
    else reinterpret_cast<double*>(base + geo.cost_off())[r] = CUDART_INF;
  }
  __syncthreads();
  const long long tk1 = clock64();
  for (int ui = warp; ui < nuniq; ui += kTinyWarps) {
    const int r = uniq[ui];
    if (lane == 0) {
      for (int c = 0; c < K; ++c) { w.sizes[c] = 0; w.members[c] = 0u; }
      for (int i = 0; i < m; ++i) {
        const int a = (fin[r] >> (3 * i)) & 7;
        w.assign[i] = a;
        w.sizes[a] += 1;
        w.members[a] |= 1u << i;
      }
      // D2 columns: a singleton's mean is its point (pd column), else evaluate
      for (int c = 0; c < K; ++c) w.colsrc[c] = w.sizes[c] == 1 ? __ffs(w.members[c]) - 1 : kColCompute;
    }
    __syncwarp();
    // ---- Hartigan (evictor.cpp:167-243) ---------------------------------------------
    for (int idx = lane; idx < K * D; idx += 32) {
      const int c = rsd.row(idx), ch = rsd.col(idx);
      double acc = 0.0;
      unsigned mm = w.members[c];
      while (mm) {
        const int i = __ffs(mm) - 1;
        mm &= mm - 1;
        acc = __dadd_rn(acc, xval(X, xs, i, ch, XS, scaled));
      }
      S[idx] = acc;
      Mn[idx] = div_n_ool(acc, w.sizes[c]);
    }
    __syncwarp();
    tiny_fill(w, X, XS, xs, scaled, pd, Mn, d2, m, K, D, lane);
    for (int c = 0; c < K; c += 2) tiny_norms(w, Mn, D, c, c + 1 < K ? c + 1 : c, lane);
    for (int pass = 0; pass < 100; ++pass) {
      if (st.kstats && lane == 0) atomicAdd(st.kstats + 32 + 7, 1ull);
      bool moved = false;  // warp-uniform
      for (int i = 0; i < m; ++i) {
        const int from = w.assign[i];
        const int nfrom = w.sizes[from];
        if (nfrom <= 1) continue;
        const double removal = __dmul_rn(tabR[nfrom], d2[i * K + from]);
        double bd = 0.0;
        int bt = 0x7fffffff;
        if (lane < K && lane != from) {
          const double delta = __dadd_rn(removal, __dmul_rn(tabA[w.sizes[lane]], d2[i * K + lane]));
          if (delta < -1e-12) { bd = delta; bt = lane; }
        }
        // best target: the lowest index among the minimal deltas (strict <, ascending)
        for (int o = 16; o > 0; o >>= 1) {
          const double od = __shfl_xor_sync(0xffffffffu, bd, o);
          const int ot = __shfl_xor_sync(0xffffffffu, bt, o);
          if (ot != 0x7fffffff && (bt == 0x7fffffff || od < bd || (od == bd && ot < bt))) { bd = od; bt = ot; }
        }
        if (bt == 0x7fffffff) continue;
        const int to = bt;
        moved = true;
        __syncwarp();
        if (lane == 0) {  // apply_move (evictor.cpp:189-196)
          w.sizes[from] -= 1;
          w.sizes[to] += 1;
          w.members[from] &= ~(1u << i);
          w.members[to] |= 1u << i;
          w.assign[i] = to;
        }
        __syncwarp();
        const int nf = w.sizes[from], nt = w.sizes[to];
        for (int ch = lane; ch < D; ch += 32) {
          const double x = xval(X, xs, i, ch, XS, scaled);
          const double sf = __dsub_rn(S[from * D + ch], x);
          const double sto = __dadd_rn(S[to * D + ch], x);
          S[from * D + ch] = sf;
          S[to * D + ch] = sto;
          Mn[from * D + ch] = div_n_ool(sf, nf);
          Mn[to * D + ch] = div_n_ool(sto, nt);
        }
        __syncwarp();
        tiny_norms(w, Mn, D, from, to, lane);
        for (int p = lane; p < 2 * m; p += 32) {
          const int pi = p >> 1, c = (p & 1) ? to : from;
          d2[pi * K + c] = tiny_dist(X, XS, xs, scaled, pi, Mn + c * D, D);
        }
        __syncwarp();
      }
      if (moved) continue;
      if (st.kstats && lane == 0) atomicAdd(st.kstats + 32 + 9, 1ull);
      // pairwise swaps (evictor.cpp:213-240): pair q = lane in lexicographic order
      int pi = 0, pj = 0;
      bool valid = false;
      for (int i = 0, q = 0; i < m; ++i)
        for (int j = i + 1; j < m; ++j, ++q)
          if (q == lane) { pi = i; pj = j; valid = true; }
      bool improving = false;
      if (valid && w.assign[pi] != w.assign[pj] &&
          !(sizeof(XT) == 2 && !scaled && w.sizes[w.assign[pi]] == 1 && w.sizes[w.assign[pj]] == 1)) {
        const int ai = w.assign[pi], aj = w.assign[pj];
        const int sa = w.sizes[ai], sb = w.sizes[aj];
        const double na = (double)sa, nb = (double)sb;
        // filter: the exact delta equals dja - dia + dib - djb - (1/na + 1/nb) pd[i][j]
        // up to rounding far below the margin (as in km_restart_kernel)
        const double wgt = 1.0 / na + 1.0 / nb;
        const double dja = d2[pj * K + ai], dia = d2[pi * K + ai], dib = d2[pi * K + aj], djb = d2[pj * K + aj];
        const double pij = pd[pi][pj];
        const double approx = dja - dia + dib - djb - wgt * pij;
        // error bound of the identity vs the reference expression (as in km_restart_kernel)
        const double margin = 1e-12 * (dja + dia + dib + djb + wgt * pij + 16.0 * (tx2[pi] + tx2[pj]) +
                                       4.0 * (na * w.m2[ai] + nb * w.m2[aj])) + 1e-12;
        if (approx < -1e-12 + margin) {
          const double* mua = Mn + ai * D;
          const double* mub = Mn + aj * D;
          double delta = 0.0;
          for (int ch = 0; ch < D; ++ch) {
            const double xi = xval(X, xs, pi, ch, XS, scaled), xj = xval(X, xs, pj, ch, XS, scaled);
            const double ma = __dadd_rn(mua[ch], div_n_ool(__dsub_rn(xj, xi), sa));
            const double mb = __dadd_rn(mub[ch], div_n_ool(__dsub_rn(xi, xj), sb));
            delta = __dadd_rn(delta, __dsub_rn(__dsub_rn(__dmul_rn(xj, xj), __dmul_rn(xi, xi)),
                                               __dmul_rn(na, __dsub_rn(__dmul_rn(ma, ma), __dmul_rn(mua[ch], mua[ch])))));
            delta = __dadd_rn(delta, __dsub_rn(__dsub_rn(__dmul_rn(xi, xi), __dmul_rn(xj, xj)),
                                               __dmul_rn(nb, __dsub_rn(__dmul_rn(mb, mb), __dmul_rn(mub[ch], mub[ch])))));
          }
          improving = delta < -1e-12;
        }
      }
      const unsigned imp = __ballot_sync(0xffffffffu, improving);
      if (!imp) break;
      const int q = __ffs(imp) - 1;
      const int si = __shfl_sync(0xffffffffu, pi, q), sj = __shfl_sync(0xffffffffu, pj, q);
      const int a = w.assign[si], b = w.assign[sj];
      __syncwarp();
      if (lane == 0) {  // apply_move(i, a, b); apply_move(j, b, a): sizes unchanged
        w.members[a] = (w.members[a] & ~(1u << si)) | (1u << sj);
        w.members[b] = (w.members[b] & ~(1u << sj)) | (1u << si);
        w.assign[si] = b;
        w.assign[sj] = a;
      }
      __syncwarp();
      const int na_ = w.sizes[a], nb_ = w.sizes[b];
      for (int ch = lane; ch < D; ch += 32) {
        const double xi = xval(X, xs, si, ch, XS, scaled), xj = xval(X, xs, sj, ch, XS, scaled);
        const double sa = __dadd_rn(__dsub_rn(S[a * D + ch], xi), xj);
        const double sb = __dsub_rn(__dadd_rn(S[b * D + ch], xi), xj);
        S[a * D + ch] = sa;
        S[b * D + ch] = sb;
        Mn[a * D + ch] = div_n_ool(sa, na_);
        Mn[b * D + ch] = div_n_ool(sb, nb_);
      }
      __syncwarp();
      tiny_norms(w, Mn, D, a, b, lane);
      for (int p = lane; p < 2 * m; p += 32) {
        const int ii = p >> 1, c = (p & 1) ? b : a;
        d2[ii * K + c] = tiny_dist(X, XS, xs, scaled, ii, Mn + c * D, D);
      }
      __syncwarp();
    }
    // ---- cost (point order) and medoids ---------------------------------------------
    double cst = 0.0;
    for (int i = 0; i < m; ++i) cst = __dadd_rn(cst, d2[i * K + w.assign[i]]);
    int med = m;
    if (lane < K) {  // nearest member, ties to the lowest index
      double bd = CUDART_INF;
      for (int i = 0; i < m; ++i) {
        if (w.assign[i] != lane) continue;
        const double d = d2[i * K + lane];
        if (d < bd) { bd = d; med = i; }
      }
    }
    const int32_t* ids = reinterpret_cast<const int32_t*>(base + geo.ids_off());
    uint32_t* mask = reinterpret_cast<uint32_t*>(base + geo.mask_off()) + (int64_t)r * geo.W;
    for (int wd = lane; wd < geo.W; wd += 32) mask[wd] = 0;
    __syncwarp();
    if (lane < K) atomicOr(mask + (ids[med] >> 5), 1u << (ids[med] & 31));
    if (lane == 0) reinterpret_cast<double*>(base + geo.cost_off())[r] = cst;
    __syncwarp();
    if (st.kstats && lane == 0) atomicAdd(st.kstats + 32 + 8, 1ull);  // distinct refinements
  }
  if (st.kstats && lane == 0) atomicAdd(st.kstats + 32 + 11, (unsigned long long)(clock64() - tk1));
}

// ---------------------------------------------------------------------------
// tiny instances, subset-table form (m <= 8, f16-exact unscaled keys: every
// band quantised, no FP8 window scale).  Every centroid kmeans_from_seeds
// ever forms is the mean of a subset S of the m points: a seed is x_s / 1,
// Lloyd's next[c] is (members summed in index order) / |S|, Hartigan's
// mean_of(c) is (running sum) / |S| (evictor.cpp:94-251).  With f16-exact
// keys every such sum is exact (|x| <= 65504, multiples of 2^-24: at most 43
// significant bits for 8 points), so each is fl(exact subset sum / |S|) --
// the same bits whichever path built it.  Hence dist2(x_i, mean(S)) for all
// 2^m - 1 subsets, each the reference's channel-order chain, is one table
// per instance, built once by all threads; every restart (70 for the
// 8 -> 4 anneal) then runs Lloyd assignments, empty-cluster repair and
// Hartigan moves on table lookups, one warp per restart.  Only the Lloyd
// movement test, the pairwise-swap delta and its filter recompute means, in
// the reference's operation order.
// ---------------------------------------------------------------------------
constexpr int kTabWarps = 8;

struct TabState {  // per warp, warp-uniform
  int assign[kTinyM];
  int sizes[kTinyM];
  unsigned cur[kTinyM];  // subset (point bitmask) whose mean is centroid c
  int seeds[kTinyM];
};

// mean(S) channel ch: the exact subset sum / |S| (div_n: the reference's division bits)
__device__ __forceinline__ double tab_mean(const double* X, int D, unsigned S, int n, int ch) {
  double acc = 0.0;
  while (S) {
    const int i = __ffs(S) - 1;
    S &= S - 1;
    acc = __dadd_rn(acc, X[i * D + ch]);
  }
  return div_n(acc, n);
}

__global__ void __launch_bounds__(32 * kTabWarps) km_table_kernel(TkvState st, const TkvAnnealOp* __restrict__ ops,
                                                                  int nops, const int32_t* __restrict__ item_prefix,
                                                                  int nitems, int item0, uint8_t* __restrict__ scratch,
                                                                  KmGeo geo) {
  const TkvDims& dm = st.dm;
  const int item = item0 + blockIdx.x;
  if (item >= nitems) return;
  const int oi = find_op(item_prefix, nops, item);
  const TkvAnnealOp op = ops[oi];
  uint8_t* base = scratch + (int64_t)blockIdx.x * geo.bytes();
  const int32_t* misc = reinterpret_cast<const int32_t*>(base + geo.misc_off());
  if (misc[1]) return;
  const int m = misc[0], K = op.K, D = dm.D;
  const int nr = op.nrestart > 0 ? op.nrestart : op.ncombos;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nsub = 1 << m;
  extern __shared__ __align__(16) uint8_t dyn[];
  double* X = reinterpret_cast<double*>(dyn);  // [m][D] exact keys
  double* terms = X + kTinyM * D + warp * 2 * D;  // per warp: swap-delta terms [2D]
  __shared__ double T[kTinyM][256];            // dist2(x_i, mean(S))
  __shared__ double M2[256];                   // |mean(S)|^2 (swap-filter error bound only)
  __shared__ double pd[kTinyM][kTinyM];
  __shared__ double tx2[kTinyM];
  __shared__ double tabA[kTinyM + 1], tabR[kTinyM + 1];  // n / (n + 1.0), -n / (n - 1.0) (evictor.cpp:201, 205)
  __shared__ TabState ws[kTabWarps];
  TabState& w = ws[warp];
  {
    const float* gX = reinterpret_cast<const float*>(base + geo.x_off());
    const double* gpd = reinterpret_cast<const double*>(base + geo.pd_off());
    for (int i = threadIdx.x; i < m * D; i += blockDim.x) X[i] = (double)gX[i];
    for (int t = threadIdx.x; t < m * m; t += blockDim.x) pd[t / m][t % m] = gpd[(int64_t)(t / m) * geo.mmax + t % m];
    for (int n = threadIdx.x; n <= kTinyM; n += blockDim.x) {
      const double dn = (double)n;
      tabA[n] = __ddiv_rn(dn, __dadd_rn(dn, 1.0));
      tabR[n] = __ddiv_rn(-dn, __dsub_rn(dn, 1.0));
    }
  }
  __syncthreads();
  const long long tb0 = clock64();
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    double acc = 0.0;
    for (int ch = 0; ch < D; ++ch) acc += X[i * D + ch] * X[i * D + ch];
    tx2[i] = acc * 1.000001;
  }
  // ---- the subset table: one subset per thread, m chains in channel order ----
  for (int S = threadIdx.x + 1; S < nsub; S += blockDim.x) {
    const int n = __popc(S);
    double d[kTinyM];
#pragma unroll
    for (int i = 0; i < kTinyM; ++i) d[i] = 0.0;
    double m2 = 0.0;
    for (int ch = 0; ch < D; ++ch) {
      const double mu = tab_mean(X, D, (unsigned)S, n, ch);
#pragma unroll
      for (int i = 0; i < kTinyM; ++i) {
        if (i < m) {
          const double t = __dsub_rn(X[i * D + ch], mu);
          d[i] = __dadd_rn(d[i], __dmul_rn(t, t));
        }
      }
      m2 += mu * mu;
    }
#pragma unroll
    for (int i = 0; i < kTinyM; ++i)
      if (i < m) T[i][S] = d[i];
    M2[S] = m2;
  }
  __syncthreads();
  if (st.kstats && threadIdx.x == 0) atomicAdd(st.kstats + 32 + 20, (unsigned long long)(clock64() - tb0));
  const int32_t* ids = reinterpret_cast<const int32_t*>(base + geo.ids_off());
  for (int r = warp; r < nr; r += kTabWarps) {
    // ---- seeds: the r-th K-subset in lexicographic order (evictor.cpp:274-283),
    //      or the prep kernel's farthest-first sets
    if (lane == 0) {
      if (op.nrestart > 0) {
        const int32_t* sd = reinterpret_cast<const int32_t*>(base + geo.seeds_off()) + r * geo.kmax;
        for (int c = 0; c < K; ++c) w.seeds[c] = sd[c];
      } else {
        int rank = r, x = 0;
        for (int c = 0; c < K; ++c) {
          while (true) {
            int cnt = 1;
            const int n = m - x - 1, k = K - c - 1;
            for (int t = 0; t < k; ++t) cnt = cnt * (n - t) / (t + 1);
            if (rank < cnt) break;
            rank -= cnt;
            ++x;
          }
          w.seeds[c] = x;
          ++x;
        }
      }
      for (int c = 0; c < K; ++c) w.cur[c] = 1u << w.seeds[c];
    }
    __syncwarp();
    const long long tl0 = clock64();
    // ---- Lloyd (evictor.cpp:102-159) on table lookups ----------------------------
    for (int iter = 0; iter < 50; ++iter) {
      int a = 0;
      if (lane < m) {  // nearest centroid, ties to the lowest index
        double bd = T[lane][w.cur[0]];
        for (int c = 1; c < K; ++c) {
          const double d = T[lane][w.cur[c]];
          if (d < bd) { bd = d; a = c; }
        }
        w.assign[lane] = a;
      }
      unsigned nxt[kTinyM];
      for (int c = 0; c < K; ++c) {
        nxt[c] = __ballot_sync(0xffffffffu, lane < m && a == c);
        if (lane == 0) w.sizes[c] = __popc(nxt[c]);
      }
      __syncwarp();
      if (lane == 0) {  // empty-cluster repair (evictor.cpp:123-141): distances to the current centroids
        for (int c = 0; c < K; ++c) {
          if (w.sizes[c] > 0) continue;
          int donor = 0;
          for (int dd = 1; dd < K; ++dd)
            if (w.sizes[dd] > w.sizes[donor]) donor = dd;
          int steal = m;
          double steal_d = -1.0;
          for (int i = 0; i < m; ++i) {
            if (w.assign[i] != donor) continue;
            const double d = T[i][w.cur[donor]];
            if (d > steal_d) { steal = i; steal_d = d; }
          }
          w.assign[steal] = c;
          nxt[donor] &= ~(1u << steal);
          nxt[c] |= 1u << steal;
          --w.sizes[donor];
          ++w.sizes[c];
        }
        for (int c = 0; c < K; ++c) w.seeds[c] = (int)nxt[c];  // publish the repaired subsets
      }
      __syncwarp();
      for (int c = 0; c < K; ++c) nxt[c] = (unsigned)w.seeds[c];
      // movement (evictor.cpp:153-158): an unchanged subset moves exactly 0;
      // otherwise sum (next - old)^2 across lanes, decide "sqrt < 1e-6" with a
      // relative margin, redo in channel order within the margin.
      int code_max = 0;
      for (int c = 0; c < K; ++c) {
        if (nxt[c] == w.cur[c] || code_max == 2) continue;  // max: one moving centroid decides
        // reverse triangle inequality on the table: |mu' - mu| >= |d(x_i, mu) - d(x_i, mu')|
        double lb = 0.0;
        if (lane < m) lb = fabs(__dsqrt_rn(T[lane][nxt[c]]) - __dsqrt_rn(T[lane][w.cur[c]]));
        for (int o = 16; o > 0; o >>= 1) lb = fmax(lb, __shfl_xor_sync(0xffffffffu, lb, o));
        if (lb > 2e-6) {  // movement >= 1e-6 whatever the rounding of the bound
          code_max = 2;
          continue;
        }
        if (st.kstats && lane == 0) atomicAdd(st.kstats + 32 + 25, 1ull);
        const int nn = __popc(nxt[c]), no = __popc(w.cur[c]);
        double part = 0.0;
        for (int ch = lane; ch < D; ch += 32) {
          const double t = __dsub_rn(tab_mean(X, D, nxt[c], nn, ch), tab_mean(X, D, w.cur[c], no, ch));
          part += __dmul_rn(t, t);
        }
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        int code;
        if (part == 0.0) {
          code = 0;
        } else if (__dsqrt_rn(part * (1.0 + 1e-12)) < 1e-6) {
          code = 1;
        } else if (!(__dsqrt_rn(part * (1.0 - 1e-12)) < 1e-6)) {
          code = 2;
        } else {
          double d = 0.0;
          if (lane == 0)
            for (int ch = 0; ch < D; ++ch) {
              const double t = __dsub_rn(tab_mean(X, D, nxt[c], nn, ch), tab_mean(X, D, w.cur[c], no, ch));
              d = __dadd_rn(d, __dmul_rn(t, t));
            }
          code = __shfl_sync(0xffffffffu, __dsqrt_rn(d) < 1e-6 ? 1 : 2, 0);
        }
        code_max = code_max > code ? code_max : code;
      }
      __syncwarp();
      if (lane == 0)
        for (int c = 0; c < K; ++c) w.cur[c] = nxt[c];
      __syncwarp();
      if (code_max < 2) break;
    }
    const long long th0 = clock64();
    long long tsw = 0;
    // ---- Hartigan single moves + pairwise swaps (evictor.cpp:167-243) ------------
    for (int pass = 0; pass < 100; ++pass) {
      bool moved = false;
      for (int i = 0; i < m; ++i) {
        const int from = w.assign[i];
        const int nfrom = w.sizes[from];
        if (nfrom <= 1) continue;
        const double removal = __dmul_rn(tabR[nfrom], T[i][w.cur[from]]);
        double bd = 0.0;
        int bt = 0x7fffffff;
        if (lane < K && lane != from) {
          const double delta = __dadd_rn(removal, __dmul_rn(tabA[w.sizes[lane]], T[i][w.cur[lane]]));
          if (delta < -1e-12) { bd = delta; bt = lane; }
        }
        for (int o = 16; o > 0; o >>= 1) {  // lowest index among the minimal deltas
          const double od = __shfl_xor_sync(0xffffffffu, bd, o);
          const int ot = __shfl_xor_sync(0xffffffffu, bt, o);
          if (ot != 0x7fffffff && (bt == 0x7fffffff || od < bd || (od == bd && ot < bt))) { bd = od; bt = ot; }
        }
        if (bt == 0x7fffffff) continue;
        moved = true;
        __syncwarp();
        if (lane == 0) {  // apply_move: the two means become other subsets' means
          w.sizes[from] -= 1;
          w.sizes[bt] += 1;
          w.cur[from] &= ~(1u << i);
          w.cur[bt] |= 1u << i;
          w.assign[i] = bt;
        }
        __syncwarp();
      }
      if (moved) continue;
      const long long ts0 = clock64();
      // pairwise swaps: pair q = lane in lexicographic order; the first
      // improving pair is the reference's pick (nothing changes before it)
      int pi = 0, pj = 0;
      bool valid = false;
      for (int i = 0, q = 0; i < m; ++i)
        for (int j = i + 1; j < m; ++j, ++q)
          if (q == lane) { pi = i; pj = j; valid = true; }
      bool cand = false;
      if (valid && w.assign[pi] != w.assign[pj] && !(w.sizes[w.assign[pi]] == 1 && w.sizes[w.assign[pj]] == 1)) {
        // (singleton pairs: the swapped means are the two points, delta exactly 0)
        const int ai = w.assign[pi], aj = w.assign[pj];
        const double na = (double)w.sizes[ai], nb = (double)w.sizes[aj];
        const unsigned Sa = w.cur[ai], Sb = w.cur[aj];
        const double wgt = 1.0 / na + 1.0 / nb;
        const double dja = T[pj][Sa], dia = T[pi][Sa], dib = T[pi][Sb], djb = T[pj][Sb];
        const double pij = pd[pi][pj];
        const double approx = dja - dia + dib - djb - wgt * pij;
        const double margin = 1e-12 * (dja + dia + dib + djb + wgt * pij + 16.0 * (tx2[pi] + tx2[pj]) +
                                       4.0 * (na * M2[Sa] * 1.000001 + nb * M2[Sb] * 1.000001)) + 1e-12;
        cand = approx < -1e-12 + margin;
      }
      // Candidates in lexicographic order, each evaluated exactly by the whole
      // warp: lanes compute the per-channel terms of evictor.cpp:222-225 (the
      // means' divisions are independent across channels), lane 0 adds them in
      // the reference's channel order.  The first improving pair is the pick.
      unsigned cmask = __ballot_sync(0xffffffffu, cand);
      unsigned imp = 0u;
      while (cmask) {
        const int q = __ffs(cmask) - 1;
        cmask &= cmask - 1;
        if (st.kstats && lane == 0) atomicAdd(st.kstats + 32 + 26, 1ull);
        const int ci = __shfl_sync(0xffffffffu, pi, q), cj = __shfl_sync(0xffffffffu, pj, q);
        const int a = w.assign[ci], b = w.assign[cj];
        const int sa = w.sizes[a], sb = w.sizes[b];
        const double na = (double)sa, nb = (double)sb;
        for (int ch = lane; ch < D; ch += 32) {
          const double mua = tab_mean(X, D, w.cur[a], sa, ch), mub = tab_mean(X, D, w.cur[b], sb, ch);
          const double xi = X[ci * D + ch], xj = X[cj * D + ch];
          const double ma = __dadd_rn(mua, div_n(__dsub_rn(xj, xi), sa));
          const double mb = __dadd_rn(mub, div_n(__dsub_rn(xi, xj), sb));
          terms[2 * ch] = __dsub_rn(__dsub_rn(__dmul_rn(xj, xj), __dmul_rn(xi, xi)),
                                    __dmul_rn(na, __dsub_rn(__dmul_rn(ma, ma), __dmul_rn(mua, mua))));
          terms[2 * ch + 1] = __dsub_rn(__dsub_rn(__dmul_rn(xi, xi), __dmul_rn(xj, xj)),
                                        __dmul_rn(nb, __dsub_rn(__dmul_rn(mb, mb), __dmul_rn(mub, mub))));
        }
        __syncwarp();
        int better = 0;
        if (lane == 0) {
          double delta = 0.0;
          for (int t = 0; t < 2 * D; ++t) delta = __dadd_rn(delta, terms[t]);
          better = delta < -1e-12;
        }
        better = __shfl_sync(0xffffffffu, better, 0);
        __syncwarp();
        if (better) {
          imp = 1u << q;
          break;
        }
      }
      tsw += clock64() - ts0;
      if (!imp) break;
      const int q = __ffs(imp) - 1;
      const int si = __shfl_sync(0xffffffffu, pi, q), sj = __shfl_sync(0xffffffffu, pj, q);
      __syncwarp();
      if (lane == 0) {  // apply_move(i, a, b); apply_move(j, b, a): sizes unchanged
        const int a = w.assign[si], b = w.assign[sj];
        w.cur[a] = (w.cur[a] & ~(1u << si)) | (1u << sj);
        w.cur[b] = (w.cur[b] & ~(1u << sj)) | (1u << si);
        w.assign[si] = b;
        w.assign[sj] = a;
      }
      __syncwarp();
    }
    if (st.kstats && lane == 0) {
      atomicAdd(st.kstats + 32 + 21, 1ull);
      atomicAdd(st.kstats + 32 + 22, (unsigned long long)(th0 - tl0));
      atomicAdd(st.kstats + 32 + 23, (unsigned long long)(clock64() - th0 - tsw));
      atomicAdd(st.kstats + 32 + 24, (unsigned long long)tsw);
    }
    // ---- cost (point order) and medoids (nearest member, ties to the lowest index)
    double cst = 0.0;
    for (int i = 0; i < m; ++i) cst = __dadd_rn(cst, T[i][w.cur[w.assign[i]]]);
    int med = m;
    if (lane < K) {
      double bd = CUDART_INF;
      for (int i = 0; i < m; ++i) {
        if (w.assign[i] != lane) continue;
        const double d = T[i][w.cur[lane]];
        if (d < bd) { bd = d; med = i; }
      }
    }
    uint32_t* mask = reinterpret_cast<uint32_t*>(base + geo.mask_off()) + (int64_t)r * geo.W;
    for (int wd = lane; wd < geo.W; wd += 32) mask[wd] = 0;
    __syncwarp();
    if (lane < K) atomicOr(mask + (ids[med] >> 5), 1u << (ids[med] & 31));
    if (lane == 0) reinterpret_cast<double*>(base + geo.cost_off())[r] = cst;
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// final: lowest cost restart -> retained mask, eviction log, segment mask
// ---------------------------------------------------------------------------
__global__ void km_final_kernel(TkvState st, const TkvAnnealOp* __restrict__ ops, int nops,
                                const int32_t* __restrict__ prefix, int nitems, int item0,
                                const uint8_t* __restrict__ scratch, KmGeo geo, uint32_t* __restrict__ log) {
  const TkvDims& dm = st.dm;
  const int li = blockIdx.x * blockDim.x + threadIdx.x;
  const int item = item0 + li;
  if (item >= nitems || li >= (int)gridDim.x * (int)blockDim.x) return;
  const int oi = find_op(prefix, nops, item);
  const TkvAnnealOp op = ops[oi];
  const int urel = item - prefix[oi];
  const int u = op.unit0 + urel;
  const int W = dm.W;
  uint32_t* segm = st.seg_mask + ((int64_t)u * dm.NSEG + op.seg) * W;
  uint32_t* logm = log + op.log_off + (int64_t)urel * W;
  const uint8_t* base = scratch + (int64_t)li * geo.bytes();
  const int32_t* misc = reinterpret_cast<const int32_t*>(base + geo.misc_off());
  if (misc[1]) {
    if (st.err[u] == 0) st.err[u] = TKV_E_INTEGRITY;
    for (int w = 0; w < W; ++w) logm[w] = 0;
    return;
  }
  const int nr = op.nrestart > 0 ? op.nrestart : op.ncombos;
  const double* cost = reinterpret_cast<const double*>(base + geo.cost_off());
  int best = 0;
  for (int r = 1; r < nr; ++r)
    if (cost[r] < cost[best]) best = r;
  const uint32_t* keep = reinterpret_cast<const uint32_t*>(base + geo.mask_off()) + (int64_t)best * W;
  for (int w = 0; w < W; ++w) {
    const uint32_t valid = w * 32 >= op.span ? 0u : (op.span - w * 32 >= 32 ? 0xffffffffu : ((1u << (op.span - w * 32)) - 1u));
    const uint32_t old = segm[w] & valid;
    logm[w] = old & ~keep[w];
    segm[w] = keep[w];
  }
}

}  // namespace

// Host-side planning helpers --------------------------------------------------
int64_t tkv_km_instance_bytes(int mmax, int kmax, int D, int W, int R) {
  KmGeo g{mmax, kmax, D, W, R};
  return g.bytes();
}

size_t tkv_km_restart_smem(int mmax, int kmax, int D, int xbytes, bool means_global) {
  const size_t x = (size_t)(((int64_t)mmax * (D + 4 / xbytes) * xbytes + 15) / 16 * 16);
  if (means_global) return x + (size_t)mmax * kmax * 8 + (size_t)4 * (D + 1) * 8;  // + staged rows
  return x + (size_t)kmax * (D + 1) * 8 + (size_t)mmax * kmax * 8;
}

cudaError_t tkv_launch_kmeans(const TkvState& st, const TkvAnnealOp* ops, int nops, const int32_t* item_prefix,
                              int nitems, const int32_t* run_prefix, int nruns, int item0, int item_count,
                              int run0, int run_count, int mmax, int kmax, int R, uint8_t* scratch, double* gsums,
                              int gsums_ctas, uint32_t* log, int scaled_any, int x16, cudaStream_t stream) {
  {  // RN(1/n) table for div_n, once per device
    static bool done[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64 && !done[dev]) {
      double inv[kInvN + 1];
      inv[0] = 0.0;
      for (int n = 1; n <= kInvN; ++n) inv[n] = 1.0 / (double)n;  // IEEE division: correctly rounded
      const cudaError_t e = cudaMemcpyToSymbol(c_inv_n, inv, sizeof(inv));
      if (e != cudaSuccess) return e;
      done[dev] = true;
    }
  }
  KmGeo geo{mmax, kmax, st.dm.D, st.dm.W, R};
  const size_t psmem = x16 ? (size_t)mmax * (st.dm.D + 2) * 2 : (size_t)mmax * (st.dm.D + 1) * 4;
  if (psmem > 160 * 1024) return cudaErrorInvalidConfiguration;
  cudaError_t e = cudaSuccess;
  auto prep = x16 ? km_prep_kernel<__half> : km_prep_kernel<float>;
  if (psmem > 16 * 1024) {
    e = cudaFuncSetAttribute(prep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem);
    if (e != cudaSuccess) return e;
  }
  // (>= 4 warps: the farthest-first seeds use one warp per anchor)
  prep<<<item_count, mmax > 32 ? 256 : 128, psmem, stream>>>(st, ops, nops, item_prefix, nitems, item0, scratch, geo,
                                                            scaled_any);
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "[kmeans] prep launch failed: items=%d: %s\n", item_count, cudaGetErrorString(e));
    return e;
  }
  if (mmax <= kTinyM && x16 && !scaled_any && getenv("TKV_KM_NO_TINY") == nullptr &&
      getenv("TKV_KM_NO_TABLE") == nullptr) {
    const size_t tsm = (size_t)(kTinyM + kTabWarps * 2) * st.dm.D * 8;
    if (tsm > 16 * 1024) {
      e = cudaFuncSetAttribute(km_table_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm);
      if (e != cudaSuccess) return e;
    }
    km_table_kernel<<<item_count, 32 * kTabWarps, tsm, stream>>>(st, ops, nops, item_prefix, item0 + item_count, item0,
                                                                  scratch, geo);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    km_final_kernel<<<(item_count + 127) / 128, 128, 0, stream>>>(st, ops, nops, item_prefix, item0 + item_count,
                                                                   item0, scratch, geo, log);
    return cudaGetLastError();
  }
  if (mmax <= kTinyM && getenv("TKV_KM_NO_TINY") == nullptr) {
    const int xb = x16 ? 2 : 4;
    const size_t tsm = (size_t)((kTinyM * (st.dm.D + 4 / xb) * xb + 15) / 16 * 16) +
                       (size_t)kTinyWarps * (2 * kmax * st.dm.D + kTinyM * kTinyM) * 8;
    if (tsm > 200 * 1024) return cudaErrorInvalidConfiguration;
    auto kern = x16 ? km_tiny_kernel<__half> : km_tiny_kernel<float>;
    if (tsm > 16 * 1024) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm);
      if (e != cudaSuccess) return e;
    }
    kern<<<item_count, 32 * kTinyWarps, tsm, stream>>>(st, ops, nops, item_prefix, item0 + item_count, item0, scratch,
                                                       geo, scaled_any, kmax);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    km_final_kernel<<<(item_count + 127) / 128, 128, 0, stream>>>(st, ops, nops, item_prefix, item0 + item_count,
                                                                   item0, scratch, geo, log);
    return cudaGetLastError();
  }
  // 64 < m <= 128 with f16 keys: two 256-thread CTAs per SM, means in global memory
  bool mg = x16 && mmax > 64 && mmax <= 128 && getenv("TKV_KM_ONE_CTA") == nullptr;
  if (mg) {  // only worth it at two CTAs per SM
    const size_t dyn = tkv_km_restart_smem(mmax, kmax, st.dm.D, 2, true);
    int nb = 0;
    if (cudaFuncSetAttribute(km_restart_kernel<256, 128, __half>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)dyn) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, km_restart_kernel<256, 128, __half>, 256, dyn) !=
            cudaSuccess)
      cudaGetLastError(), nb = 0;
    mg = nb >= 2;
  }
  // 32 < m <= 64 with f16 keys: six 128-thread CTAs per SM, means in global memory
  bool mg64 = x16 && mmax > 32 && mmax <= 64 && getenv("TKV_KM_ONE_CTA") == nullptr;
  if (mg64) {
    const size_t dyn = tkv_km_restart_smem(mmax, kmax, st.dm.D, 2, true);
    int nb = 0;
    if (cudaFuncSetAttribute(km_restart_kernel<128, 64, __half>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)dyn) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, km_restart_kernel<128, 64, __half>, 128, dyn) !=
            cudaSuccess)
      cudaGetLastError(), nb = 0;
    mg64 = nb >= 5;
  }
  const size_t smem = tkv_km_restart_smem(mmax, kmax, st.dm.D, x16 ? 2 : 4, mg || mg64);
  if (smem > 200 * 1024) return cudaErrorInvalidConfiguration;  // tau x d beyond the smem design point
  // runs are processed in chunks of gsums_ctas CTAs (one global sums buffer each)
  // Small classes keep their sums in shared memory: one launch for all runs.
  // Launches of equal size (no short tail launch): ceil(runs / capacity) of them.
  int chunk = mmax <= 32 ? (run_count > 0 ? run_count : 1) : gsums_ctas;
  if (run_count > chunk) {
    const int nl = (run_count + chunk - 1) / chunk;
    chunk = (run_count + nl - 1) / nl;
  }
  for (int r = 0; r < run_count; r += chunk) {
    const int n = run_count - r < chunk ? run_count - r : chunk;
    // Instance-size variants: static shared arrays and CTA width scale with
    // m, so tiny exhaustive-seed instances (e.g. 8 -> 4, 70 restarts) run as
    // many single-warp CTAs per SM.
    auto go = [&](auto kern, int nt) -> cudaError_t {
      const size_t sm = mmax <= 32 ? smem + (size_t)kmax * st.dm.D * 8 : smem;  // + shared sums rows
      if (sm > 16 * 1024) {  // static + dynamic must opt in beyond 48 KB
        const cudaError_t ee = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (ee != cudaSuccess) return ee;
      }
      kern<<<n, nt, sm, stream>>>(st, ops, nops, run_prefix, run0 + run_count, run0 + r, item_prefix, item0,
                                    scratch, geo, gsums, scaled_any);
      return cudaSuccess;
    };
    if (mg) {
      e = go(km_restart_kernel<256, 128, __half>, 256);
    } else if (mg64) {
      e = go(km_restart_kernel<128, 64, __half>, 128);
    } else if (x16) {
      if (mmax <= 16) e = go(km_restart_kernel<64, 16, __half>, 64);
      else if (mmax <= 32) e = go(km_restart_kernel<128, 32, __half>, 128);
      else if (mmax <= 64) e = go(km_restart_kernel<256, 64, __half>, 256);
      else e = go(km_restart_kernel<512, kMaxM, __half>, 512);
    } else {
      if (mmax <= 16) e = go(km_restart_kernel<64, 16, float>, 64);
      else if (mmax <= 32) e = go(km_restart_kernel<128, 32, float>, 128);
      else if (mmax <= 64) e = go(km_restart_kernel<256, 64, float>, 256);
      else e = go(km_restart_kernel<512, kMaxM, float>, 512);
    }
    if (e != cudaSuccess) return e;
    e = cudaGetLastError();
    if (e != cudaSuccess) {
      fprintf(stderr, "[kmeans] restart launch failed: n=%d smem=%zu mmax=%d kmax=%d R=%d: %s\n", n, smem, mmax, kmax, R,
              cudaGetErrorString(e));
      return e;
    }
  }
  km_final_kernel<<<(item_count + 127) / 128, 128, 0, stream>>>(st, ops, nops, item_prefix, item0 + item_count, item0,
                                                                 scratch, geo, log);
  return cudaGetLastError();
}
