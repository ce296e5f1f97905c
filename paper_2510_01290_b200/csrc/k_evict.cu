// K3d/K3e: thought-budget eviction on device.
//
// K3d (anneal_kernel): one CTA per (unit, anneal op) runs the reference's
// deterministic K-means medoid selection (kmeans_select -> kmeans_cluster ->
// kmeans_from_seeds, proj/src/evictor.cpp:55-338) over the decoded fp64 keys of
// the segment's members.  Every floating-point value is produced by the same
// IEEE operation sequence as the reference build (this file is compiled with
// --fmad=false and uses explicit _rn intrinsics for every accumulation that is
// order-sensitive), so medoid choices -- and therefore eviction decisions --
// are bit-exact.  Parallelism is only taken where the reference's result is
// order-independent: distance evaluations for independent (point, centroid)
// pairs, per-(cluster, channel) sums over members in ascending point order,
// exact max/min reductions with first-index tie breaking, and the
// first-improving pairwise swap found by a lexicographic minimum.
//
// K3e (apply_kernel): BlockPager::apply_eviction_plan (pager.cpp:238-259):
// soft-mask evicted slots, drop window scale references (release_slot_groups,
// :72-87) and return blocks whose live count reaches zero to the free pool
// (free_block, :228-236).  Slots are never moved.
#include <cuda_runtime.h>
#include <math_constants.h>

#include "tkv_codec.cuh"
#include "tkv_kernels.h"
#include "tkv_state.h"

namespace {

constexpr int kThreads = 256;
constexpr int kMaxM = 256;  // segment members (tau <= 256)

__device__ __forceinline__ double dist2(const double* __restrict__ a, const double* __restrict__ b, int D) {
  double d = 0.0;
  for (int i = 0; i < D; ++i) {
    const double t = __dsub_rn(a[i], b[i]);
    d = __dadd_rn(d, __dmul_rn(t, t));
  }
  return d;
}

struct KmSmem {
  int assign[kMaxM];
  int best_assign[kMaxM];
  int order[kMaxM];
  int taken[kMaxM];
  int sizes[kMaxM];
  int offs[kMaxM + 1];
  int seeds[kMaxM];
  int ids[kMaxM];
  int medoid[kMaxM];
  double tmp[kMaxM];
  double cost, best_cost;
  int cur;        // which centroid buffer holds the current centroids
  int flag;       // generic CTA-wide flag
  int best_to;
  int pair;
  int have_best;
};

struct Km {
  int m, K, D;
  double* X;      // [m][D]
  double* cb[2];  // centroid double buffer [K][D]
  double* sums;   // [K][D]
  double* means;  // [K][D]
  double* best;   // [K][D]
  unsigned long long* ks;  // optional counters
};
__device__ __forceinline__ void kstat(const Km& km, int i, unsigned long long v) {
  if (km.ks && threadIdx.x == 0) atomicAdd(km.ks + i, v);
}

// Stable member lists per cluster (ascending point index) from assign/sizes.
__device__ void build_members(KmSmem& s, int m, int K) {
  if (threadIdx.x == 0) {
    s.offs[0] = 0;
    for (int c = 0; c < K; ++c) s.offs[c + 1] = s.offs[c] + s.sizes[c];
    for (int c = 0; c < K; ++c) s.tmp[c] = 0;  // reuse as fill cursor
    for (int i = 0; i < m; ++i) {
      const int a = s.assign[i];
      s.order[s.offs[a] + (int)s.tmp[a]] = i;
      s.tmp[a] += 1.0;
    }
  }
  __syncthreads();
}

__device__ void count_sizes(KmSmem& s, int m, int K) {
  if (threadIdx.x == 0) {
    for (int c = 0; c < K; ++c) s.sizes[c] = 0;
    for (int i = 0; i < m; ++i) ++s.sizes[s.assign[i]];
  }
  __syncthreads();
}

// kmeans_from_seeds (evictor.cpp:94-251).  Leaves assign/sizes in smem, final
// centroids in km.cb[s.cur], cost in s.cost.
__device__ void kmeans_from_seeds(const Km& km, KmSmem& s) {
  const int m = km.m, K = km.K, D = km.D;
  for (int idx = threadIdx.x; idx < K * D; idx += kThreads) {
    const int c = idx / D, ch = idx % D;
    km.cb[0][idx] = km.X[s.seeds[c] * D + ch];
  }
  if (threadIdx.x == 0) s.cur = 0;
  __syncthreads();
  long long c0 = clock64();
  kstat(km, 0, 1);
  for (int iter = 0; iter < 50; ++iter) {
    kstat(km, 1, 1);
    const double* cent = km.cb[s.cur];
    double* next = km.cb[s.cur ^ 1];
    // Assign; ties go to the lowest cluster index.
    for (int i = threadIdx.x; i < m; i += kThreads) {
      int best = 0;
      double bd = dist2(km.X + i * D, cent, D);
      for (int c = 1; c < K; ++c) {
        const double d = dist2(km.X + i * D, cent + c * D, D);
        if (d < bd) { best = c; bd = d; }
      }
      s.assign[i] = best;
    }
    __syncthreads();
    count_sizes(s, m, K);
    // Repair empty clusters: steal the farthest point of the largest cluster.
    if (threadIdx.x == 0) {
      for (int c = 0; c < K; ++c) {
        if (s.sizes[c] > 0) continue;
        int donor = 0;
        for (int d = 1; d < K; ++d)
          if (s.sizes[d] > s.sizes[donor]) donor = d;
        int steal = m;
        double steal_d = -1.0;
        for (int i = 0; i < m; ++i) {
          if (s.assign[i] != donor) continue;
          const double d = dist2(km.X + i * D, cent + donor * D, D);
          if (d > steal_d) { steal = i; steal_d = d; }
        }
        s.assign[steal] = c;
        --s.sizes[donor];
        ++s.sizes[c];
      }
    }
    __syncthreads();
    build_members(s, m, K);
    // Update centroids: per (cluster, channel) ascending-index sums.
    for (int idx = threadIdx.x; idx < K * D; idx += kThreads) {
      const int c = idx / D, ch = idx % D;
      double acc = 0.0;
      for (int k = s.offs[c]; k < s.offs[c + 1]; ++k) acc = __dadd_rn(acc, km.X[s.order[k] * D + ch]);
      next[idx] = __ddiv_rn(acc, (double)s.sizes[c]);
    }
    __syncthreads();
    for (int c = threadIdx.x; c < K; c += kThreads) s.tmp[c] = __dsqrt_rn(dist2(next + c * D, cent + c * D, D));
    __syncthreads();
    if (threadIdx.x == 0) {
      double movement = 0.0;
      for (int c = 0; c < K; ++c) movement = movement < s.tmp[c] ? s.tmp[c] : movement;
      s.cur ^= 1;
      s.flag = movement < 1e-6;
    }
    __syncthreads();
    if (s.flag) break;
  }

  // Hartigan single moves + pairwise swaps (evictor.cpp:179-243).
  long long c1 = clock64();
  kstat(km, 6, (unsigned long long)(c1 - c0));
  count_sizes(s, m, K);
  build_members(s, m, K);
  for (int idx = threadIdx.x; idx < K * D; idx += kThreads) {
    const int c = idx / D, ch = idx % D;
    double acc = 0.0;
    for (int k = s.offs[c]; k < s.offs[c + 1]; ++k) acc = __dadd_rn(acc, km.X[s.order[k] * D + ch]);
    km.sums[idx] = acc;
    km.means[idx] = __ddiv_rn(acc, (double)s.sizes[c]);
  }
  __syncthreads();
  for (int pass = 0; pass < 100; ++pass) {
    kstat(km, 2, 1);
    long long ch0 = clock64();
    bool moved = false;  // CTA-uniform
    for (int i = 0; i < m; ++i) {
      const int from = s.assign[i];
      if (s.sizes[from] <= 1) continue;
      for (int c = threadIdx.x; c < K; c += kThreads) s.tmp[c] = dist2(km.X + i * D, km.means + c * D, D);
      __syncthreads();
      if (threadIdx.x == 0) {
        const double na = (double)s.sizes[from];
        const double removal = __dmul_rn(__ddiv_rn(-na, __dsub_rn(na, 1.0)), s.tmp[from]);
        int best_to = from;
        double best_delta = -1e-12;
        for (int to = 0; to < K; ++to) {
          if (to == from) continue;
          const double nb = (double)s.sizes[to];
          const double delta = __dadd_rn(removal, __dmul_rn(__ddiv_rn(nb, __dadd_rn(nb, 1.0)), s.tmp[to]));
          if (delta < best_delta) { best_delta = delta; best_to = to; }
        }
        s.best_to = best_to;
        if (best_to != from) {
          --s.sizes[from];
          ++s.sizes[best_to];
          s.assign[i] = best_to;
        }
      }
      __syncthreads();
      const int to = s.best_to;
      if (to != from) {
        kstat(km, 3, 1);
        moved = true;
        for (int ch = threadIdx.x; ch < D; ch += kThreads) {
          const double x = km.X[i * D + ch];
          km.sums[from * D + ch] = __dsub_rn(km.sums[from * D + ch], x);
          km.sums[to * D + ch] = __dadd_rn(km.sums[to * D + ch], x);
          km.means[from * D + ch] = __ddiv_rn(km.sums[from * D + ch], (double)s.sizes[from]);
          km.means[to * D + ch] = __ddiv_rn(km.sums[to * D + ch], (double)s.sizes[to]);
        }
      }
      __syncthreads();
    }
    kstat(km, 7, (unsigned long long)(clock64() - ch0));
    if (moved) continue;
    kstat(km, 4, 1);
    long long cs0 = clock64();
    // Pairwise exchanges: the lexicographically first improving (i, j).
    if (threadIdx.x == 0) s.pair = 0x7fffffff;
    __syncthreads();
    const int npairs = m * (m - 1) / 2;
    for (int p = threadIdx.x; p < npairs; p += kThreads) {
      if (p > s.pair) break;
      // unrank p -> (i, j), i < j, row-major over i
      int i = 0, rem = p;
      while (rem >= m - 1 - i) { rem -= m - 1 - i; ++i; }
      const int j = i + 1 + rem;
      const int a = s.assign[i], b = s.assign[j];
      if (a == b) continue;
      const double na = (double)s.sizes[a], nb = (double)s.sizes[b];
      const double* mua = km.means + a * D;
      const double* mub = km.means + b * D;
      const double* xi_ = km.X + i * D;
      const double* xj_ = km.X + j * D;
      double delta = 0.0;
      for (int ch = 0; ch < D; ++ch) {
        const double xi = xi_[ch], xj = xj_[ch];
        const double ma = __dadd_rn(mua[ch], __ddiv_rn(__dsub_rn(xj, xi), na));
        const double mb = __dadd_rn(mub[ch], __ddiv_rn(__dsub_rn(xi, xj), nb));
        const double xx = __dsub_rn(__dmul_rn(xj, xj), __dmul_rn(xi, xi));
        const double yy = __dsub_rn(__dmul_rn(xi, xi), __dmul_rn(xj, xj));
        delta = __dadd_rn(delta, __dsub_rn(xx, __dmul_rn(na, __dsub_rn(__dmul_rn(ma, ma), __dmul_rn(mua[ch], mua[ch])))));
        delta = __dadd_rn(delta, __dsub_rn(yy, __dmul_rn(nb, __dsub_rn(__dmul_rn(mb, mb), __dmul_rn(mub[ch], mub[ch])))));
      }
      if (delta < -1e-12) {
        atomicMin(&s.pair, p);
        break;
      }
    }
    __syncthreads();
    const int p = s.pair;
    kstat(km, 8, (unsigned long long)(clock64() - cs0));
    if (p == 0x7fffffff) break;
    kstat(km, 5, 1);
    int i = 0, rem = p;
    while (rem >= m - 1 - i) { rem -= m - 1 - i; ++i; }
    const int j = i + 1 + rem;
    const int a = s.assign[i], b = s.assign[j];
    for (int ch = threadIdx.x; ch < D; ch += kThreads) {
      const double xi = km.X[i * D + ch], xj = km.X[j * D + ch];
      km.sums[a * D + ch] = __dadd_rn(__dsub_rn(km.sums[a * D + ch], xi), xj);
      km.sums[b * D + ch] = __dsub_rn(__dadd_rn(km.sums[b * D + ch], xi), xj);
      km.means[a * D + ch] = __ddiv_rn(km.sums[a * D + ch], (double)s.sizes[a]);
      km.means[b * D + ch] = __ddiv_rn(km.sums[b * D + ch], (double)s.sizes[b]);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      s.assign[i] = b;
      s.assign[j] = a;
    }
    __syncthreads();
  }
  kstat(km, 9, (unsigned long long)(clock64() - c0));
  // Final centroids = member means; cost summed in point order.
  double* cent = km.cb[s.cur];
  for (int idx = threadIdx.x; idx < K * D; idx += kThreads) cent[idx] = km.means[idx];
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += kThreads) s.tmp[i] = dist2(km.X + i * D, cent + s.assign[i] * D, D);
  __syncthreads();
  if (threadIdx.x == 0) {
    double c = 0.0;
    for (int i = 0; i < m; ++i) c = __dadd_rn(c, s.tmp[i]);
    s.cost = c;
  }
  __syncthreads();
}

// Run one seed set and keep it if it beats the best so far (ties -> earlier).
__device__ void run_seeds(const Km& km, KmSmem& s) {
  kmeans_from_seeds(km, s);
  const bool better = !s.have_best || s.cost < s.best_cost;  // CTA-uniform (smem)
  __syncthreads();
  if (better) {
    const double* cent = km.cb[s.cur];
    for (int idx = threadIdx.x; idx < km.K * km.D; idx += kThreads) km.best[idx] = cent[idx];
    for (int i = threadIdx.x; i < km.m; i += kThreads) s.best_assign[i] = s.assign[i];
    if (threadIdx.x == 0) {
      s.best_cost = s.cost;
      s.have_best = 1;
    }
  }
  __syncthreads();
}

// farthest_first_seeds (evictor.cpp:71-92) into s.seeds.
__device__ void farthest_first(const Km& km, KmSmem& s, int anchor) {
  const int m = km.m, K = km.K, D = km.D;
  for (int i = threadIdx.x; i < m; i += kThreads) {
    s.tmp[i] = CUDART_INF;
    s.taken[i] = 0;
  }
  if (threadIdx.x == 0) {
    s.seeds[0] = anchor;
    s.taken[anchor] = 1;
  }
  __syncthreads();
  for (int n = 1; n < K; ++n) {
    const int last = s.seeds[n - 1];
    for (int i = threadIdx.x; i < m; i += kThreads) {
      const double d = dist2(km.X + i * D, km.X + last * D, D);
      s.tmp[i] = d < s.tmp[i] ? d : s.tmp[i];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int far = 0;
      double far_d = -1.0;
      for (int i = 0; i < m; ++i)
        if (!s.taken[i] && s.tmp[i] > far_d) { far = i; far_d = s.tmp[i]; }
      s.seeds[n] = far;
      s.taken[far] = 1;
    }
    __syncthreads();
  }
}

// kmeans_select's medoid choice (kmeans_cluster, evictor.cpp:255-338) over
// the keys in km.X: seed sets, the restarts (lowest cost wins, ties to the
// earlier), then the member nearest each centroid (ties to the lowest
// index).  Leaves the medoid point index of cluster c in s.medoid[c].
__device__ void select_medoids(const Km& km, KmSmem& s) {
  const int m = km.m, K = km.K, D = km.D;
  // Seed sets (kmeans_cluster, evictor.cpp:255-317).
  double subsets = 1.0;
  for (int i = 0; i < K; ++i) subsets = __dmul_rn(subsets, __ddiv_rn((double)(m - i), (double)(i + 1)));
  kstat(km, 10, 1);
  if (subsets <= 512.0) {
    kstat(km, 11, 1);
    if (threadIdx.x == 0)
      for (int i = 0; i < K; ++i) s.seeds[i] = i;
    __syncthreads();
    while (true) {
      run_seeds(km, s);
      if (threadIdx.x == 0) {
        int j = K;
        while (j > 0 && s.seeds[j - 1] == m - K + j - 1) --j;
        if (j == 0) {
          s.flag = 1;
        } else {
          ++s.seeds[j - 1];
          for (int l = j; l < K; ++l) s.seeds[l] = s.seeds[l - 1] + 1;
          s.flag = 0;
        }
      }
      __syncthreads();
      if (s.flag) break;
    }
  } else {
    // Anchors: index 0, farthest from and nearest to the mean, m/2.
    double* mean = km.best;  // scratch until the first run
    for (int ch = threadIdx.x; ch < D; ch += kThreads) {
      double acc = 0.0;
      for (int i = 0; i < m; ++i) acc = __dadd_rn(acc, km.X[i * D + ch]);
      mean[ch] = __ddiv_rn(acc, (double)m);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < m; i += kThreads) s.tmp[i] = dist2(km.X + i * D, mean, D);
    __syncthreads();
    __shared__ int anchors[4];
    if (threadIdx.x == 0) {
      int far_idx = 0, near_idx = 0;
      double far_d = -1.0, near_d = CUDART_INF;
      for (int i = 0; i < m; ++i) {
        const double d = s.tmp[i];
        if (d > far_d) { far_d = d; far_idx = i; }
        if (d < near_d) { near_d = d; near_idx = i; }
      }
      anchors[0] = 0;
      anchors[1] = far_idx;
      anchors[2] = near_idx;
      anchors[3] = m / 2;
    }
    __syncthreads();
    for (int a = 0; a < 4; ++a) {
      const long long f0 = clock64();
      farthest_first(km, s, anchors[a]);
      kstat(km, 12, (unsigned long long)(clock64() - f0));
      run_seeds(km, s);
    }
  }
  // Medoids: member nearest each centroid, ties to the lowest id.
  for (int c = threadIdx.x; c < K; c += kThreads) {
    int best_i = m;
    double best_d = CUDART_INF;
    for (int i = 0; i < m; ++i) {
      if (s.best_assign[i] != c) continue;
      const double d = dist2(km.X + i * D, km.best + c * D, D);
      if (d < best_d) { best_d = d; best_i = i; }
    }
    s.medoid[c] = best_i;
  }
  __syncthreads();}

__device__ double decode_key(const TkvState& st, int u, int slot, int ch) {
  const TkvDims& dm = st.dm;
  const int64_t gs = (int64_t)u * dm.NS + slot;
  const int fmt = dm.band_fmt[st.blk_thought[(int64_t)u * dm.P + slot / dm.bs]];
  const uint8_t* kr = st.slot_k + gs * dm.kstride;
  if (fmt == TKV_FMT_RAW) {
    if (dm.in_dtype == TKV_IN_BF16) return (double)__uint_as_float(((uint32_t) reinterpret_cast<const uint16_t*>(kr)[ch]) << 16);
    if (dm.in_dtype == TKV_IN_F32) return (double)reinterpret_cast<const float*>(kr)[ch];
    return reinterpret_cast<const double*>(kr)[ch];
  }
  const int win = st.slot_win[gs];
  const uint32_t code = tkv_get_code(kr, fmt, ch);
  if (fmt == TKV_FMT_FP8) return tkv_decode_code(fmt, code, (double)st.win_kf[(int64_t)u * dm.NW + win]);
  return tkv_decode_code(fmt, code, tkv_e4m3_decode(st.win_ks[((int64_t)u * dm.NW + win) * dm.D + ch]));
}

__global__ void __launch_bounds__(kThreads) anneal_kernel(TkvState st, const TkvAnnealOp* __restrict__ ops, int nops,
                                                          const int32_t* __restrict__ prefix, int nitems,
                                                          uint32_t* __restrict__ log, double* __restrict__ scratch,
                                                          int64_t per_cta, int max_m) {
  const TkvDims& dm = st.dm;
  __shared__ KmSmem s;
  __shared__ int opi;
  const int D = dm.D, W = dm.W;
  double* base = scratch + (int64_t)blockIdx.x * per_cta;
  for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
    if (threadIdx.x == 0) {
      int lo = 0, hi = nops - 1;
      while (lo < hi) {  // last op with prefix[op] <= item
        const int mid = (lo + hi + 1) / 2;
        if (prefix[mid] <= item) lo = mid; else hi = mid - 1;
      }
      opi = lo;
    }
    __syncthreads();
    const TkvAnnealOp op = ops[opi];
    const int urel = item - prefix[opi];
    const int u = op.unit0 + urel;
    uint32_t* segm = st.seg_mask + ((int64_t)u * dm.NSEG + op.seg) * W;
    uint32_t* logm = log + op.log_off + (int64_t)urel * W;
    // Members in ascending id order (bit order of the segment mask).
    if (threadIdx.x == 0) {
      int m = 0;
      for (int b = 0; b < op.span && m < kMaxM; ++b)
        if ((segm[b >> 5] >> (b & 31)) & 1u) s.ids[m++] = b;
      s.flag = m;
      s.pair = 0;
    }
    __syncthreads();
    const int m = s.flag;
    bool bad = m != op.m || st.err[u] != 0;
    // member slots (s.taken is free until the seeds are chosen)
    if (!bad) tkv_member_slots(st, u, op.seg_start, op.span, segm, s.taken, &s.pair);
    __syncthreads();
    bad = bad || s.pair != m;
    Km km;
    km.m = m;
    km.K = op.K;
    km.D = D;
    km.X = base;
    km.cb[0] = base + (int64_t)max_m * D;
    km.cb[1] = km.cb[0] + (int64_t)max_m * D;
    km.sums = km.cb[1] + (int64_t)max_m * D;
    km.means = km.sums + (int64_t)max_m * D;
    km.best = km.means + (int64_t)max_m * D;
    km.ks = st.kstats;
    const long long i0 = clock64();
    if (!bad) {
      // Decoded fp64 keys (BlockPager::key_of, pager.cpp:280-287; exact products).
      for (int idx = threadIdx.x; idx < m * D; idx += kThreads) {
        const int i = idx / D, ch = idx % D;
        km.X[idx] = decode_key(st, u, s.taken[i], ch);
      }
      if (threadIdx.x == 0) {
        s.flag = 0;
        s.have_best = 0;
      }
      __syncthreads();
      bad = s.flag != 0;
    }
    __syncthreads();
    if (bad) {
      if (threadIdx.x == 0) {
        if (st.err[u] == 0) st.err[u] = TKV_E_INTEGRITY;
        for (int w = 0; w < W; ++w) logm[w] = 0;
      }
      __syncthreads();
      continue;
    }
    select_medoids(km, s);
    kstat(km, 13, (unsigned long long)(clock64() - i0));
    kstat(km, 14, (unsigned long long)m);
    if (threadIdx.x == 0) {
      uint32_t keep[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int c = 0; c < op.K; ++c) {
        const int b = s.ids[s.medoid[c]];
        keep[b >> 5] |= 1u << (b & 31);
      }
      for (int w = 0; w < W; ++w) {
        const uint32_t old = segm[w] & (w * 32 >= op.span ? 0u : (op.span - w * 32 >= 32 ? 0xffffffffu : ((1u << (op.span - w * 32)) - 1u)));
        logm[w] = old & ~keep[w];
        segm[w] = keep[w];
      }
    }
    __syncthreads();
  }
}

// Drop-in kmeans_select: one CTA per instance over caller-
// supplied fp64 keys (instance i: m[i] <= 256 points of D channels at
// X + xoff[i], K[i] clusters); medoid point indices, one per cluster, to
// out + ooff[i].  Scratch: 5 * m[i] * D doubles at scratch + 5 * xoff[i].
__global__ void __launch_bounds__(kThreads) kmeans_select_f64_kernel(const double* __restrict__ X,
                                                                     const int32_t* __restrict__ ms,
                                                                     const int32_t* __restrict__ ks,
                                                                     const int64_t* __restrict__ xoff,
                                                                     const int64_t* __restrict__ ooff, int D,
                                                                     double* __restrict__ scratch, int32_t* out) {
  __shared__ KmSmem s;
  const int i = blockIdx.x;
  const int m = ms[i], K = ks[i];
  Km km;
  km.m = m;
  km.K = K;
  km.D = D;
  km.X = const_cast<double*>(X) + xoff[i];
  km.cb[0] = scratch + 5 * xoff[i];
  km.cb[1] = km.cb[0] + (int64_t)m * D;
  km.sums = km.cb[1] + (int64_t)m * D;
  km.means = km.sums + (int64_t)m * D;
  km.best = km.means + (int64_t)m * D;
  km.ks = nullptr;
  if (threadIdx.x == 0) s.have_best = 0;
  __syncthreads();
  select_medoids(km, s);
  for (int c = threadIdx.x; c < K; c += kThreads) out[ooff[i] + c] = s.medoid[c];
}

__global__ void __launch_bounds__(32) apply_kernel(TkvState st, const TkvAnnealOp* __restrict__ ops,
                                                   const TkvApplyGroup* __restrict__ groups, int ngroups,
                                                   const int32_t* __restrict__ prefix, int nitems,
                                                   const uint32_t* __restrict__ log) {
  const TkvDims& dm = st.dm;
  const int item = blockIdx.x, lane = threadIdx.x;
  if (item >= nitems) return;
  int gi = 0;
  {
    int lo = 0, hi = ngroups - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) / 2;
      if (prefix[mid] <= item) lo = mid; else hi = mid - 1;
    }
    gi = lo;
  }
  const TkvApplyGroup grp = groups[gi];
  const int urel = item - prefix[gi];
  const int u = grp.unit0 + urel;
  if (st.err[u] != 0) return;  // (uniform: read by every lane before any write)
  __syncwarp();
  const int P = dm.P, bs = dm.bs, W = dm.W;
  int8_t* th = st.blk_thought + (int64_t)u * P;
  uint8_t* fl = st.blk_filled + (int64_t)u * P;
  uint32_t* ev = st.blk_evict + (int64_t)u * P;
  uint8_t* ns = st.blk_nstart + (int64_t)u * P;
  uint32_t touched[64];  // P <= 2048
  for (int i = 0; i < 64; ++i) touched[i] = 0;
  extern __shared__ int rel_slot[];  // [W * 32]: slot of each live id of the op's segment window
  const int32_t* sid = st.slot_id + (int64_t)u * dm.NS;
  bool failed = false;
  for (int oi = grp.op_begin; oi < grp.op_end && !failed; ++oi) {
    const TkvAnnealOp op = ops[oi];
    const uint32_t* lm = log + op.log_off + (int64_t)urel * W;
    // The warp maps the window's live ids to slots (slot_id, skipping evicted
    // slots -- including those of earlier ops of this call); lane 0 then
    // applies the evictions in id order, so window records return to the free
    // stack in the reference's order (release_slot_groups, pager.cpp:72-87).
    __syncwarp();
    for (int r = lane; r < W * 32; r += 32) rel_slot[r] = -1;
    __syncwarp();
    for (int s = lane; s < dm.NS; s += 32) {
      const int rel = sid[s] - op.seg_start;
      const int blk = s / bs, sl = s % bs;
      if (rel >= 0 && rel < op.span && !((ev[blk] >> sl) & 1u) && th[blk] >= 0 && sl < fl[blk]) rel_slot[rel] = s;
    }
    __syncwarp();
    if (lane == 0) {
      for (int w = 0; w < W && !failed; ++w) {
        uint32_t bits = lm[w];
        while (bits) {
          const int b = __ffs(bits) - 1;
          bits &= bits - 1;
          const int slot = rel_slot[w * 32 + b];
          if (slot < 0) {
            st.err[u] = TKV_E_INTEGRITY;
            failed = true;
            break;
          }
          const int blk = slot / bs, sl = slot % bs;
          ev[blk] |= 1u << sl;
          const int64_t gs = (int64_t)u * dm.NS + slot;
          const int win = st.slot_win[gs];
          if (win >= 0) {
            const int64_t wi = (int64_t)u * dm.NW + win;
            if (--st.win_refs[wi] <= 0) {
              st.win_refs[wi] = 0;
              st.win_free[(int64_t)u * dm.NW + st.win_nfree[u]] = win;
              st.win_nfree[u] += 1;
            }
          }
          touched[blk >> 5] |= 1u << (blk & 31);
        }
      }
    }
    failed = __shfl_sync(0xffffffffu, failed, 0);
  }
  if (failed) return;
  if (lane != 0) return;
  for (int w = 0; w < 64; ++w) {
    uint32_t bits = touched[w];
    while (bits) {
      const int b = w * 32 + __ffs(bits) - 1;
      bits &= bits - 1;
      const uint32_t live = ~ev[b] & (fl[b] >= 32 ? 0xffffffffu : ((1u << fl[b]) - 1u));
      if (live == 0) {
        th[b] = -1;
        fl[b] = 0;
        ev[b] = 0;
        ns[b] = 0;
        st.unit_nfree[u] += 1;
      }
    }
  }
}

}  // namespace

cudaError_t tkv_launch_anneal(const TkvState& st, const TkvAnnealOp* ops, int nops, const int32_t* item_prefix,
                              int nitems, uint32_t* log, double* scratch, int scratch_ctas,
                              int64_t scratch_doubles_per_cta, int max_m, cudaStream_t stream) {
  if (nitems <= 0) return cudaSuccess;
  const int grid = nitems < scratch_ctas ? nitems : scratch_ctas;
  anneal_kernel<<<grid, kThreads, 0, stream>>>(st, ops, nops, item_prefix, nitems, log, scratch,
                                               scratch_doubles_per_cta, max_m);
  return cudaGetLastError();
}

cudaError_t tkv_launch_kmeans_select_f64(int ninst, const double* X, const int32_t* m, const int32_t* K,
                                         const int64_t* xoff, const int64_t* ooff, int D, double* scratch,
                                         int32_t* out, cudaStream_t stream) {
  if (ninst <= 0) return cudaSuccess;
  kmeans_select_f64_kernel<<<ninst, kThreads, 0, stream>>>(X, m, K, xoff, ooff, D, scratch, out);
  return cudaGetLastError();
}

cudaError_t tkv_launch_apply(const TkvState& st, const TkvAnnealOp* ops, const TkvApplyGroup* groups,
                             int ngroups, const int32_t* unit_prefix, int nitems, const uint32_t* log,
                             cudaStream_t stream) {
  if (nitems <= 0) return cudaSuccess;
  apply_kernel<<<nitems, 32, (size_t)st.dm.W * 32 * sizeof(int), stream>>>(st, ops, groups, ngroups, unit_prefix,
                                                                          nitems, log);
  return cudaGetLastError();
}
