// K1 (tensor-core variant): paged mixed-precision decode attention for
// head_dim 64/128, bf16 inputs, G <= 8 query heads per KV head.
//
// One CTA (4 warps) per unit.  The live slots (compacted per storage format,
// with their window indices) plus the raw tail (the unit's fp buffer and the
// incoming token, sim.cpp:546-563, 762-765) are cut into 16-token tiles that
// are dealt round-robin to the warps:
//
//   QK^T   mma.m16n8k16 -> f32, A = dequantised K tile (16 tokens x 16
//          channels per k-step), B = q^T (16 channels x 8 heads, heads >= G
//          zero).  The dot product is permutation-invariant, so k-step j of
//          thread (gid, tig) is mapped to physical channels tig*D/4 + 4j..4j+3:
//          every thread's K codes are ONE contiguous 128/64-bit load per row.
//   PV     mma.m16n8k16 with A = V^T (channels x tokens), B = P (tokens x
//          heads) split into hi + lo parts (two mmas) so the probabilities
//          keep ~22 (f16) / ~16 (bf16) bits; thread gid owns the contiguous
//          channels [gid*D/8, (gid+1)*D/8), which is exactly one E4M3
//          value-chunk scale (g = 16) and one 64/32-bit code load per token.
//
// Quantised tiles (NVFP4 / ternary / FP8) run f16 MMAs: codes are expanded in
// registers with the sm_100 converters (F2FP.F16.E2M1 / F2FP.F16.E4M3) and one
// HMUL2 by the E4M3 group scale; every code x scale product is exact in f16
// (<= 8 significant bits, range 2^-10 .. 2688), so QK^T products are exact and
// accumulate in fp32.  FP8 windows keep their fp32 per-window scale out of the
// MMA (applied to the logit / folded into P).  Raw tiles -- 16-bit passthrough
// slots and the tail -- run bf16 MMAs on the stored bf16 words directly (q, K
// and V are exact in bf16).  Online softmax runs in the log2 domain in fp32.
// Loads of tile t+1 are issued before tile t is computed (register double
// buffering).
#include <cuda_runtime.h>
#include <math_constants.h>

#include "tkv_kernels.h"
#include "tkv_state.h"

namespace {

constexpr int kThreads = 128;
constexpr int kWarps = 4;
constexpr float kLog2e = 1.4426950408889634f;
constexpr int kFmtTail = 4;  // pseudo-format: raw bf16 tiles (RAW slots + tail)

__device__ __forceinline__ uint32_t fp4x2_f16x2(uint32_t b) {
  uint32_t r;
  asm("{\n .reg .b8 t;\n cvt.u8.u32 t, %1;\n cvt.rn.f16x2.e2m1x2 %0, t;\n}" : "=r"(r) : "r"(b));
  return r;
}
__device__ __forceinline__ uint32_t e4m3x2_f16x2(uint32_t h) {
  uint32_t r;
  asm("{\n .reg .b16 t;\n cvt.u16.u32 t, %1;\n cvt.rn.f16x2.e4m3x2 %0, t;\n}" : "=r"(r) : "r"(h));
  return r;
}
__device__ __forceinline__ uint32_t hmul2(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
// Two ternary 2-bit codes (sign/magnitude, quant.cpp:219-236) -> f16x2.
__device__ __forceinline__ uint32_t tern2_f16x2(uint32_t nib) {
  const uint32_t c0 = nib & 3u, c1 = (nib >> 2) & 3u;
  const uint32_t h0 = (c0 & 1u) ? (0x3C00u | ((c0 & 2u) << 14)) : 0u;
  const uint32_t h1 = (c1 & 1u) ? (0x3C00u | ((c1 & 2u) << 14)) : 0u;
  return h0 | (h1 << 16);
}
__device__ __forceinline__ uint32_t pack_f16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ float f16lo(uint32_t x) {
  float r;
  asm("{\n .reg .b16 l, h;\n mov.b32 {l, h}, %1;\n cvt.f32.f16 %0, l;\n}" : "=f"(r) : "r"(x));
  return r;
}
__device__ __forceinline__ float f16hi(uint32_t x) {
  float r;
  asm("{\n .reg .b16 l, h;\n mov.b32 {l, h}, %1;\n cvt.f32.f16 %0, h;\n}" : "=f"(r) : "r"(x));
  return r;
}
__device__ __forceinline__ float bf16lo(uint32_t x) { return __uint_as_float(x << 16); }
__device__ __forceinline__ float bf16hi(uint32_t x) { return __uint_as_float(x & 0xffff0000u); }

template <bool BF16>
__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  if constexpr (BF16) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  } else {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
}

template <int N>
struct Words { uint32_t w[N]; };

template <int N>
__device__ __forceinline__ Words<N> ldg_words(const uint8_t* p) {
  Words<N> r;
  if constexpr (N == 1) {
    r.w[0] = __ldg(reinterpret_cast<const uint32_t*>(p));
  } else if constexpr (N == 2) {
    const uint2 x = __ldg(reinterpret_cast<const uint2*>(p));
    r.w[0] = x.x; r.w[1] = x.y;
  } else {
#pragma unroll
    for (int i = 0; i < N / 4; ++i) {
      const uint4 x = __ldg(reinterpret_cast<const uint4*>(p) + i);
      r.w[4 * i] = x.x; r.w[4 * i + 1] = x.y; r.w[4 * i + 2] = x.z; r.w[4 * i + 3] = x.w;
    }
  }
  return r;
}

// Per-format geometry for head dim D.
template <int D, int FMT>
struct Geo {
  static constexpr int KT = D / 16;            // QK k-steps
  static constexpr int CPT = D / 4;            // QK channels per thread (per row)
  static constexpr int MT = D / 16;            // PV m-tiles
  static constexpr int VPT = D / 8;            // PV channels per thread
  static constexpr int BITS = FMT == TKV_FMT_TERNARY ? 2 : (FMT == TKV_FMT_NVFP4 ? 4 : (FMT == TKV_FMT_FP8 ? 8 : 16));
  static constexpr int KBYTES = CPT * BITS / 8;  // per row per thread
  static constexpr int VBYTES = VPT * BITS / 8;  // per token per thread
  static constexpr int KW = KBYTES / 4;
  static constexpr int VW = VBYTES >= 4 ? VBYTES / 4 : 1;
  static constexpr int SW = FMT == kFmtTail ? 1 : CPT / 4;  // key-scale words per row per thread
  static constexpr bool BF16 = FMT == kFmtTail;
};

template <int D, int FMT>
struct Tile {
  using Gm = Geo<D, FMT>;
  Words<Gm::KW> k[2];
  Words<Gm::SW> ks[2];
  Words<Gm::VW> v[4];
  uint32_t vs[4];     // value scale code (grouped) per PV token
  float kf[2];        // fp8 key scale per row
  float vf[4];        // fp8 value scale per PV token
  bool krow_ok[2];
  bool vtok_ok[4];
};

// Row addresses.  Tail entries are encoded as (-1 - t, 0): t < nbuf is buffer
// row t, t == nbuf the incoming token.
struct TailSrc {
  const uint8_t* bk;
  const uint8_t* bv;
  const uint8_t* kc;
  const uint8_t* vc;
  int nbuf;
};

template <int D, int FMT>
__device__ __forceinline__ void load_tile(const TkvState& st, int u, const int2* lst, int n, int t0, int gid,
                                          int tig, const TailSrc& ts, Tile<D, FMT>& T) {
  using Gm = Geo<D, FMT>;
  const TkvDims& dm = st.dm;
  const int64_t ubase = (int64_t)u * dm.NS;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int idx = t0 + gid + 8 * r;
    T.krow_ok[r] = idx < n;
    const int2 e = lst[T.krow_ok[r] ? idx : 0];
    const uint8_t* kr;
    if constexpr (FMT == kFmtTail) {
      if (e.x >= 0) kr = st.slot_k + (ubase + e.x) * dm.kstride;
      else kr = (-1 - e.x) < ts.nbuf ? ts.bk + (int64_t)(-1 - e.x) * D * 2 : ts.kc;
    } else {
      kr = st.slot_k + (ubase + e.x) * dm.kstride;
    }
    T.k[r] = ldg_words<Gm::KW>(kr + tig * Gm::KBYTES);
    if constexpr (FMT == TKV_FMT_FP8) {
      T.kf[r] = __ldg(st.win_kf + (int64_t)u * dm.NW + e.y);
    } else if constexpr (FMT != kFmtTail) {
      const uint8_t* sc = st.win_ks + ((int64_t)u * dm.NW + e.y) * D + tig * Gm::CPT;
      T.ks[r] = ldg_words<Gm::SW>(sc);
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int idx = t0 + tig * 2 + (i & 1) + 8 * (i >> 1);
    T.vtok_ok[i] = idx < n;
    const int2 e = lst[T.vtok_ok[i] ? idx : 0];
    const uint8_t* vr;
    if constexpr (FMT == kFmtTail) {
      if (e.x >= 0) vr = st.slot_v + (ubase + e.x) * dm.kstride;
      else vr = (-1 - e.x) < ts.nbuf ? ts.bv + (int64_t)(-1 - e.x) * D * 2 : ts.vc;
    } else {
      vr = st.slot_v + (ubase + e.x) * dm.kstride;
    }
    vr += gid * Gm::VBYTES;
    if constexpr (Gm::VBYTES >= 4) {
      T.v[i] = ldg_words<Gm::VW>(vr);
    } else {
      T.v[i].w[0] = Gm::VBYTES == 2 ? (uint32_t)__ldg(reinterpret_cast<const unsigned short*>(vr)) : (uint32_t)__ldg(vr);
    }
    if constexpr (FMT == TKV_FMT_FP8) {
      T.vf[i] = __ldg(st.win_vf + (int64_t)u * dm.NW + e.y);
    } else if constexpr (FMT != kFmtTail) {
      T.vs[i] = __ldg(st.slot_vs + (ubase + e.x) * dm.vchunks + (gid * Gm::VPT) / dm.g);
    }
  }
}

template <int D>
struct Acc {
  float o[D / 16][4];
  float m[2], l[2];  // heads tig*2, tig*2+1
};

template <int D, int FMT>
__device__ __forceinline__ void compute_tile(const Tile<D, FMT>& T, const uint32_t (&qb)[D / 16][2],
                                             const uint32_t* qbb, float qscale, int G, bool maxpool, int gid,
                                             int tig, float* ps, Acc<D>& A) {
  using Gm = Geo<D, FMT>;
  // ---- S = K q^T ----------------------------------------------------------
  float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int j = 0; j < Gm::KT; ++j) {
    uint32_t a[4];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      uint32_t lo, hi;
      if constexpr (FMT == TKV_FMT_NVFP4) {
        const uint32_t byte2 = (T.k[r].w[j >> 1] >> ((j & 1) * 16)) & 0xffffu;
        lo = fp4x2_f16x2(byte2 & 0xffu);
        hi = fp4x2_f16x2(byte2 >> 8);
      } else if constexpr (FMT == TKV_FMT_FP8) {
        lo = e4m3x2_f16x2(T.k[r].w[j] & 0xffffu);
        hi = e4m3x2_f16x2(T.k[r].w[j] >> 16);
      } else if constexpr (FMT == TKV_FMT_TERNARY) {
        const uint32_t byte = (T.k[r].w[j >> 2] >> ((j & 3) * 8)) & 0xffu;
        lo = tern2_f16x2(byte & 15u);
        hi = tern2_f16x2(byte >> 4);
      } else {  // raw bf16 words: channels 4j, 4j+1 | 4j+2, 4j+3
        lo = T.k[r].w[2 * j];
        hi = T.k[r].w[2 * j + 1];
      }
      if constexpr (FMT == TKV_FMT_NVFP4 || FMT == TKV_FMT_TERNARY) {
        const uint32_t sw = T.ks[r].w[j];
        lo = hmul2(lo, e4m3x2_f16x2(sw & 0xffffu));
        hi = hmul2(hi, e4m3x2_f16x2(sw >> 16));
      }
      a[r] = lo;       // a0a1 (row gid) / a2a3 (row gid+8), cols tig*2..+1
      a[2 + r] = hi;   // a4a5 / a6a7, cols tig*2+8..+9
    }
    if constexpr (Gm::BF16) {
      mma16816<true>(s, a[0], a[1], a[2], a[3], qbb[j * 2], qbb[j * 2 + 1]);
    } else {
      mma16816<false>(s, a[0], a[1], a[2], a[3], qb[j][0], qb[j][1]);
    }
  }
  // logits (log2 domain); rows: s0,s1 -> token gid, s2,s3 -> token gid+8
  float L[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = i >> 1, h = tig * 2 + (i & 1);
    float x = s[i] * qscale;
    if constexpr (FMT == TKV_FMT_FP8) x *= T.kf[r];
    L[i] = (T.krow_ok[r] && h < G) ? x : -CUDART_INF_F;
  }
  if (maxpool) {
    // one pooled row per token: max over the G heads, kept in column 0
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      float mx = fmaxf(L[2 * r], L[2 * r + 1]);
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      L[2 * r] = tig == 0 ? mx : -CUDART_INF_F;
      L[2 * r + 1] = -CUDART_INF_F;
    }
  }
  // ---- online softmax per head column --------------------------------------
  float p[4];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    float tmax = fmaxf(L[c], L[2 + c]);
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 4));
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 8));
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 16));
    const float mnew = fmaxf(A.m[c], tmax);
    const float corr = mnew == -CUDART_INF_F ? 1.0f : exp2f(A.m[c] - mnew);
    p[c] = mnew == -CUDART_INF_F ? 0.0f : exp2f(L[c] - mnew);
    p[2 + c] = mnew == -CUDART_INF_F ? 0.0f : exp2f(L[2 + c] - mnew);
    float sum = p[c] + p[2 + c];
    sum += __shfl_xor_sync(0xffffffffu, sum, 4);
    sum += __shfl_xor_sync(0xffffffffu, sum, 8);
    sum += __shfl_xor_sync(0xffffffffu, sum, 16);
    A.l[c] = A.l[c] * corr + sum;
    A.m[c] = mnew;
#pragma unroll
    for (int mt = 0; mt < Gm::MT; ++mt) {
      A.o[mt][c] *= corr;
      A.o[mt][2 + c] *= corr;
    }
  }
  // ---- P: C layout (token, head) -> B layout (token = k, head = n) -----------
  ps[gid * 8 + tig * 2] = p[0];
  ps[gid * 8 + tig * 2 + 1] = p[1];
  ps[(gid + 8) * 8 + tig * 2] = p[2];
  ps[(gid + 8) * 8 + tig * 2 + 1] = p[3];
  __syncwarp();
  float pb[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int tok = tig * 2 + (i & 1) + 8 * (i >> 1);
    pb[i] = ps[tok * 8 + gid];
    if constexpr (FMT == TKV_FMT_FP8) pb[i] *= T.vtok_ok[i] ? T.vf[i] : 0.0f;
  }
  __syncwarp();
  uint32_t bh0, bh1, bl0, bl1;
  if constexpr (Gm::BF16) {
    bh0 = pack_bf16x2(pb[0], pb[1]);
    bh1 = pack_bf16x2(pb[2], pb[3]);
    bl0 = pack_bf16x2(pb[0] - bf16lo(bh0), pb[1] - bf16hi(bh0));
    bl1 = pack_bf16x2(pb[2] - bf16lo(bh1), pb[3] - bf16hi(bh1));
  } else {
    bh0 = pack_f16x2(pb[0], pb[1]);
    bh1 = pack_f16x2(pb[2], pb[3]);
    bl0 = pack_f16x2(pb[0] - f16lo(bh0), pb[1] - f16hi(bh0));
    bl1 = pack_f16x2(pb[2] - f16lo(bh1), pb[3] - f16hi(bh1));
  }
  // ---- O^T += V^T P ----------------------------------------------------------
  uint32_t vsc[4];
  if constexpr (FMT == TKV_FMT_NVFP4 || FMT == TKV_FMT_TERNARY) {
#pragma unroll
    for (int i = 0; i < 4; ++i) vsc[i] = e4m3x2_f16x2(T.vs[i] | (T.vs[i] << 8));
  }
#pragma unroll
  for (int mt = 0; mt < Gm::MT; ++mt) {
    uint32_t x[4];  // per PV token: x2 of channels (2mt, 2mt+1) of the thread's range
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t h;
      if constexpr (FMT == TKV_FMT_NVFP4) {
        h = hmul2(fp4x2_f16x2((T.v[i].w[mt >> 2] >> ((mt & 3) * 8)) & 0xffu), vsc[i]);
      } else if constexpr (FMT == TKV_FMT_FP8) {
        h = e4m3x2_f16x2((T.v[i].w[mt >> 1] >> ((mt & 1) * 16)) & 0xffffu);
      } else if constexpr (FMT == TKV_FMT_TERNARY) {
        h = hmul2(tern2_f16x2((T.v[i].w[0] >> (mt * 4)) & 15u), vsc[i]);
      } else {
        h = T.v[i].w[mt];
      }
      x[i] = T.vtok_ok[i] ? h : 0u;
    }
    const uint32_t a0 = __byte_perm(x[0], x[1], 0x5410);  // row gid (ch 2mt), tokens tig*2, tig*2+1
    const uint32_t a1 = __byte_perm(x[0], x[1], 0x7632);  // row gid+8 (ch 2mt+1)
    const uint32_t a2 = __byte_perm(x[2], x[3], 0x5410);  // row gid, tokens +8, +9
    const uint32_t a3 = __byte_perm(x[2], x[3], 0x7632);
    mma16816<Gm::BF16>(A.o[mt], a0, a1, a2, a3, bh0, bh1);
    mma16816<Gm::BF16>(A.o[mt], a0, a1, a2, a3, bl0, bl1);
  }
}

// Tiles of one format with index (global) g = warp + k * kWarps in [g0, g1).
template <int D, int FMT>
__device__ __forceinline__ void run_format(const TkvState& st, int u, const int2* lst, int n, int g0, int warp,
                                           const uint32_t (&qb)[D / 16][2], const uint32_t* qbb, float qscale,
                                           bool maxpool, int gid, int tig, const TailSrc& ts, float* ps, Acc<D>& A) {
  const int tiles = (n + 15) / 16;
  // first tile index of this format handled by this warp
  int t = ((warp - g0) % kWarps + kWarps) % kWarps;
  if (t >= tiles) return;
  if constexpr (FMT == kFmtTail) {  // few tiles, wide rows: no double buffering (registers)
    for (; t < tiles; t += kWarps) {
      Tile<D, FMT> cur;
      load_tile<D, FMT>(st, u, lst, n, t * 16, gid, tig, ts, cur);
      compute_tile<D, FMT>(cur, qb, qbb, qscale, st.dm.G, maxpool, gid, tig, ps, A);
    }
    return;
  }
  Tile<D, FMT> cur, nxt;
  load_tile<D, FMT>(st, u, lst, n, t * 16, gid, tig, ts, cur);
  for (; t < tiles; t += kWarps) {
    const bool more = t + kWarps < tiles;
    if (more) load_tile<D, FMT>(st, u, lst, n, (t + kWarps) * 16, gid, tig, ts, nxt);
    compute_tile<D, FMT>(cur, qb, qbb, qscale, st.dm.G, maxpool, gid, tig, ps, A);
    if (more) cur = nxt;
  }
}

template <int D>
__global__ void __launch_bounds__(kThreads, 3) attend_mma_kernel(TkvState st, const void* __restrict__ qin,
                                                                  const void* __restrict__ kin,
                                                                  const void* __restrict__ vin,
                                                                  float* __restrict__ out, int buf_half, int nbuf,
                                                                  int put_half, int put_slot) {
  const TkvDims& dm = st.dm;
  const int u = blockIdx.x;
  const int G = dm.G, R = dm.maxpool ? 1 : G;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  extern __shared__ __align__(16) uint8_t dyn[];
  float* red = reinterpret_cast<float*>(dyn);                       // [kWarps * 8][2 + D]
  float* ps_all = red + kWarps * 8 * (2 + D);                         // [kWarps][16 * 8]
  uint32_t* qbb_all = reinterpret_cast<uint32_t*>(ps_all + kWarps * 128);  // [32 lanes][D/8] bf16 B frags
  int2* list = reinterpret_cast<int2*>(qbb_all + 32 * (D / 8));        // [NS + g + 1] (slot, window)
  __shared__ int cnt[5], off[5], wsum[kWarps][4];
  const float qscale = dm.scale * kLog2e;

  // q^T B fragments: head gid, channels tig*D/4 + 4j + {0,1} / {2,3}; f16 in
  // registers, the raw bf16 words in shared memory for the bf16 tiles.
  uint32_t qb[D / 16][2];
  {
    const uint16_t* qq = reinterpret_cast<const uint16_t*>(qin) + ((int64_t)u * G + gid) * D + tig * (D / 4);
    uint32_t* qbb = qbb_all + lane * (D / 8);
#pragma unroll
    for (int j = 0; j < D / 16; ++j) {
      uint2 w = make_uint2(0u, 0u);
      if (gid < G) w = *reinterpret_cast<const uint2*>(qq + 4 * j);
      if (warp == 0) { qbb[2 * j] = w.x; qbb[2 * j + 1] = w.y; }
      qb[j][0] = pack_f16x2(bf16lo(w.x), bf16hi(w.x));
      qb[j][1] = pack_f16x2(bf16lo(w.y), bf16hi(w.y));
    }
  }
  // Live-slot list per format with window indices (physical order), then the
  // raw tail appended to the raw list.
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
  int incl[4];  // warp-inclusive scans
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    int x = c[f];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    incl[f] = x;
    if (lane == 31) wsum[warp][f] = x;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int f = 0; f < 4; ++f) {
      off[f] = run;
      int tot = 0;
      for (int w = 0; w < kWarps; ++w) tot += wsum[w][f];
      cnt[f] = tot;
      run += tot;
    }
    cnt[TKV_FMT_RAW] += nbuf + 1;  // tail tokens ride in the raw list
    off[kFmtTail] = 0;
    cnt[kFmtTail] = 0;
  }
  __syncthreads();
  {
    int w[4];
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      int before = 0;
      for (int ww = 0; ww < warp; ++ww) before += wsum[ww][f];
      w[f] = off[f] + before + incl[f] - c[f];
    }
    const int32_t* swin = st.slot_win + (int64_t)u * dm.NS;
    for (int b = b0; b < b1; ++b) {
      const int t = th[b];
      if (t < 0) continue;
      uint32_t live = ~ev[b] & (fl[b] >= 32 ? 0xffffffffu : ((1u << fl[b]) - 1u));
      const int f = dm.band_fmt[t];
      while (live) {
        const int s = __ffs(live) - 1;
        live &= live - 1;
        const int slot = b * bs + s;
        list[w[f]++] = make_int2(slot, max(0, swin[slot]));
      }
    }
    const int rawn = cnt[TKV_FMT_RAW] - (nbuf + 1);
    for (int t = threadIdx.x; t <= nbuf; t += kThreads) list[off[TKV_FMT_RAW] + rawn + t] = make_int2(-1 - t, 0);
  }
  __syncthreads();
  TailSrc ts;
  {
    const int64_t row = (int64_t)dm.g * D * 2;
    ts.bk = st.buf + ((int64_t)u * 4 + buf_half * 2 + 0) * row;
    ts.bv = st.buf + ((int64_t)u * 4 + buf_half * 2 + 1) * row;
    ts.kc = reinterpret_cast<const uint8_t*>(kin) + (int64_t)u * D * 2;
    ts.vc = reinterpret_cast<const uint8_t*>(vin) + (int64_t)u * D * 2;
    ts.nbuf = nbuf;
  }
  Acc<D> A;
#pragma unroll
  for (int mt = 0; mt < D / 16; ++mt)
#pragma unroll
    for (int i = 0; i < 4; ++i) A.o[mt][i] = 0.f;
  A.m[0] = A.m[1] = -CUDART_INF_F;
  A.l[0] = A.l[1] = 0.f;
  float* ps = ps_all + warp * 128;
  const uint32_t* qbb = qbb_all + lane * (D / 8);
  const bool mp = dm.maxpool != 0;
  // Tiles are numbered globally across formats and dealt round-robin.
  int g0 = 0;
  if (cnt[TKV_FMT_NVFP4]) {
    run_format<D, TKV_FMT_NVFP4>(st, u, list + off[TKV_FMT_NVFP4], cnt[TKV_FMT_NVFP4], g0, warp, qb, qbb, qscale, mp,
                                 gid, tig, ts, ps, A);
    g0 += (cnt[TKV_FMT_NVFP4] + 15) / 16;
  }
  if (cnt[TKV_FMT_TERNARY]) {
    run_format<D, TKV_FMT_TERNARY>(st, u, list + off[TKV_FMT_TERNARY], cnt[TKV_FMT_TERNARY], g0, warp, qb, qbb,
                                   qscale, mp, gid, tig, ts, ps, A);
    g0 += (cnt[TKV_FMT_TERNARY] + 15) / 16;
  }
  if (cnt[TKV_FMT_FP8]) {
    run_format<D, TKV_FMT_FP8>(st, u, list + off[TKV_FMT_FP8], cnt[TKV_FMT_FP8], g0, warp, qb, qbb, qscale, mp, gid,
                               tig, ts, ps, A);
    g0 += (cnt[TKV_FMT_FP8] + 15) / 16;
  }
  run_format<D, kFmtTail>(st, u, list + off[TKV_FMT_RAW], cnt[TKV_FMT_RAW], g0, warp, qb, qbb, qscale, mp, gid, tig,
                          ts, ps, A);
  // Per-warp partial state -> smem: red[(warp*8 + h)][0]=m, [1]=l, [2+ch]=acc.
  const int stride = 2 + D;
#pragma unroll
  for (int cc = 0; cc < 2; ++cc) {
    const int h = tig * 2 + cc;
    float* rr = red + (warp * 8 + h) * stride;
    if (gid == 0) { rr[0] = A.m[cc]; rr[1] = A.l[cc]; }
#pragma unroll
    for (int mt = 0; mt < D / 16; ++mt) {
      const int ch0 = gid * (D / 8) + 2 * mt;
      rr[2 + ch0] = A.o[mt][cc];
      rr[2 + ch0 + 1] = A.o[mt][2 + cc];
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < R * D; idx += kThreads) {
    const int r = idx / D, ch = idx % D;
    float M = -CUDART_INF_F;
    for (int w = 0; w < kWarps; ++w) M = fmaxf(M, red[(w * 8 + r) * stride]);
    float Ls = 0.f, O = 0.f;
    for (int w = 0; w < kWarps; ++w) {
      const float* rr = red + (w * 8 + r) * stride;
      if (rr[0] == -CUDART_INF_F) continue;
      const float f = exp2f(rr[0] - M);
      Ls += rr[1] * f;
      O += rr[2 + ch] * f;
    }
    out[((int64_t)u * R + r) * D + ch] = O / Ls;
  }
  if (put_slot >= 0) {  // buffer the incoming token (sim.cpp:796-808)
    const int64_t row = (int64_t)dm.g * D;
    uint16_t* bk = reinterpret_cast<uint16_t*>(st.buf) + ((int64_t)u * 4 + put_half * 2 + 0) * row + (int64_t)put_slot * D;
    uint16_t* bv = reinterpret_cast<uint16_t*>(st.buf) + ((int64_t)u * 4 + put_half * 2 + 1) * row + (int64_t)put_slot * D;
    const uint16_t* ks = reinterpret_cast<const uint16_t*>(kin) + (int64_t)u * D;
    const uint16_t* vs = reinterpret_cast<const uint16_t*>(vin) + (int64_t)u * D;
    for (int i = threadIdx.x; i < D; i += kThreads) {
      bk[i] = ks[i];
      bv[i] = vs[i];
    }
  }
}

}  // namespace

bool tkv_attend_mma_supported(const TkvDims& dm) {
  if (dm.D != 64 && dm.D != 128) return false;
  if (dm.in_dtype != TKV_IN_BF16 || dm.G > 8) return false;
  if (dm.g % (dm.D / 8) != 0) return false;
  return true;
}

cudaError_t tkv_launch_attend_mma(const TkvState& st, const void* q, const void* k, const void* v, float* out,
                                  int buf_half, int nbuf, int put_half, int put_slot, cudaStream_t s) {
  const int D = st.dm.D;
  const size_t smem = (size_t)kWarps * 8 * (2 + D) * 4 + (size_t)kWarps * 128 * 4 + (size_t)32 * (D / 8) * 4 +
                      (size_t)(st.dm.NS + st.dm.g + 1) * 8;
  if (D == 128) {
    static bool cfg = false;
    if (!cfg) { cudaFuncSetAttribute(attend_mma_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); cfg = true; }
    attend_mma_kernel<128><<<st.dm.U, kThreads, smem, s>>>(st, q, k, v, out, buf_half, nbuf, put_half, put_slot);
  } else {
    static bool cfg = false;
    if (!cfg) { cudaFuncSetAttribute(attend_mma_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); cfg = true; }
    attend_mma_kernel<64><<<st.dm.U, kThreads, smem, s>>>(st, q, k, v, out, buf_half, nbuf, put_half, put_slot);
  }
  return cudaGetLastError();
}
