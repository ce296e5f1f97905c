// K1 (tensor-core variant): paged mixed-precision decode attention for
// head_dim 64/128, bf16 inputs, G <= 8 query heads per KV head.
//
// Reference semantics (what one unit computes per step): the live pager slots
// in physical (block, slot) order (BlockPager::read_active, proj/src/
// pager.cpp:261-271), then the fp buffer, then the incoming token at full
// precision (sim.cpp:546-563, 762-765); gqa_attend (attention.cpp:124-138):
// logits q.k / sqrt(d), per-head rows or the max over the G rows
// (gqa_aggregate, :110-122), softmax, probability-weighted values.  The
// output does not depend on the key order, so the kernel is free to group the
// live slots by storage format.
//
// One CTA (4 warps) per unit.  Prologue: scan the unit's block table, build
// per-format live lists (slot, window) in shared memory, each padded to a
// whole 16-token tile with copies of its first entry (padding rows are masked
// to -inf logits, so they contribute exactly zero); the fp buffer and the
// incoming token form the raw "tail" list.  Tiles are numbered across formats
// and dealt round-robin to the warps.  Per tile:
//
//   QK^T   mma.m16n8k16 -> f32, A = dequantised K tile (16 tokens x 16
//          channels per k-step), B = q^T (heads >= G are zero).  k-step j of
//          thread (gid, tig) is mapped to physical channels tig*D/4 + 4j..4j+3
//          (the dot product is order-free), so each thread's K codes and key
//          scales of a row are contiguous vector loads.
//   PV     mma.m16n8k16 with A = V^T (channels x tokens), B = P (tokens x
//          heads) split into hi + lo halves (two mmas) so probabilities keep
//          ~22 (f16) / ~16 (bf16) bits; thread gid owns channels
//          [gid*D/8, (gid+1)*D/8) = one E4M3 value-chunk scale (g = 16).
//
// Dequantisation uses the sm_100 converters F2FP.F16.E2M1 / F2FP.F16.E4M3
// with their byte / half-word operand selectors (PTX mov.b32 unpack), so no
// shift/mask instruction extracts a code.  Ternary codes are spread to e2m1
// nibbles (+-1.0) with a Morton bit spread.  code x E4M3 scale products are
// exact in f16 (<= 8 significant bits, range 2^-10 .. 2688): QK^T products
// are exact, accumulated in fp32.  FP8 windows keep their fp32 per-window
// scale out of the MMA (applied to the logit / folded into P).  Raw tiles
// (16-bit passthrough slots and the tail) run bf16 MMAs on the stored words.
// Online softmax in the log2 domain with lazy rescaling: the running max is
// only raised when a tile exceeds it by more than 2^8, so the accumulators
// are rescaled rarely; O and l always share the same reference max, so the
// result is the same softmax.  Loads of the next tile are issued before the
// current one is computed (two register tiles, ping-pong without copies).
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdlib>

#include "tkv_kernels.h"
#include "tkv_state.h"

namespace {

constexpr int kThreads = 128;
constexpr int kWarps = 4;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescale = 8.0f;  // lazy-rescale threshold (log2 units)
constexpr int kFmtTail = 4;       // pseudo-format: raw bf16 tiles (RAW slots + tail)

// ---- converters (byte / half selectors come free with mov.b32 unpack) -------
__device__ __forceinline__ void e2m1x8(uint32_t w, uint32_t (&r)[4]) {
  asm("{\n .reg .b8 b0, b1, b2, b3;\n mov.b32 {b0, b1, b2, b3}, %4;\n"
      " cvt.rn.f16x2.e2m1x2 %0, b0;\n cvt.rn.f16x2.e2m1x2 %1, b1;\n"
      " cvt.rn.f16x2.e2m1x2 %2, b2;\n cvt.rn.f16x2.e2m1x2 %3, b3;\n}"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(w));
}
__device__ __forceinline__ void e2m1x2_b(uint32_t w, int byte, uint32_t& r) {
  // byte is a compile-time constant after unrolling
  if (byte == 0) asm("{\n .reg .b8 b0, b1, b2, b3;\n mov.b32 {b0, b1, b2, b3}, %1;\n cvt.rn.f16x2.e2m1x2 %0, b0;\n}" : "=r"(r) : "r"(w));
  else if (byte == 1) asm("{\n .reg .b8 b0, b1, b2, b3;\n mov.b32 {b0, b1, b2, b3}, %1;\n cvt.rn.f16x2.e2m1x2 %0, b1;\n}" : "=r"(r) : "r"(w));
  else if (byte == 2) asm("{\n .reg .b8 b0, b1, b2, b3;\n mov.b32 {b0, b1, b2, b3}, %1;\n cvt.rn.f16x2.e2m1x2 %0, b2;\n}" : "=r"(r) : "r"(w));
  else asm("{\n .reg .b8 b0, b1, b2, b3;\n mov.b32 {b0, b1, b2, b3}, %1;\n cvt.rn.f16x2.e2m1x2 %0, b3;\n}" : "=r"(r) : "r"(w));
}
__device__ __forceinline__ void e4m3x4(uint32_t w, uint32_t& lo, uint32_t& hi) {
  asm("{\n .reg .b16 h0, h1;\n mov.b32 {h0, h1}, %2;\n"
      " cvt.rn.f16x2.e4m3x2 %0, h0;\n cvt.rn.f16x2.e4m3x2 %1, h1;\n}"
      : "=r"(lo), "=r"(hi) : "r"(w));
}
__device__ __forceinline__ void e4m3x2_b(uint32_t w, int byte, uint32_t& r) {
  // one E4M3 byte duplicated into both f16 halves: (b, b) -> f16x2
  const uint32_t b = __byte_perm(w, 0u, byte == 0 ? 0x4400 : byte == 1 ? 0x4411 : byte == 2 ? 0x4422 : 0x4433);
  asm("{\n .reg .b16 h0, h1;\n mov.b32 {h0, h1}, %1;\n cvt.rn.f16x2.e4m3x2 %0, h0;\n}" : "=r"(r) : "r"(b));
}
__device__ __forceinline__ uint32_t hmul2(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
// 8 ternary sign/magnitude codes (2 bits each, quant.cpp:219-236) -> 8 e2m1
// nibbles: magnitude bit -> e2m1 bit 1 (1.0), sign bit -> bit 3.
__device__ __forceinline__ uint32_t tern_spread(uint32_t h16) {
  uint32_t x = h16 & 0xffffu;
  x = (x | (x << 8)) & 0x00ff00ffu;
  x = (x | (x << 4)) & 0x0f0f0f0fu;
  x = (x | (x << 2)) & 0x33333333u;
  x = (x | (x << 1)) & 0x55555555u;
  return x << 1;
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
  static constexpr bool SCALED = FMT == TKV_FMT_NVFP4 || FMT == TKV_FMT_TERNARY;
  static constexpr int SW = SCALED ? CPT / 4 : 1;  // key-scale words per row per thread
  static constexpr bool BF16 = FMT == kFmtTail;
};

template <int D, int FMT>
struct Tile {
  using Gm = Geo<D, FMT>;
  Words<Gm::KW> k[2];
  Words<Gm::SW> ks[2];
  Words<Gm::VW> v[4];
  uint32_t vs[4];     // value-chunk scale byte per PV token (grouped formats)
  float kf[2];        // fp8 key scale per row
  float vf[4];        // fp8 value scale per PV token
};

// Per-unit base pointers (computed once per CTA).
struct UnitPtrs {
  const uint8_t* k;   // slot_k of the unit
  const uint8_t* v;
  const uint8_t* vs;  // slot_vs
  const uint8_t* ks;  // win_ks
  const float* kf;
  const float* vf;
  const uint8_t* bk;  // fp buffer keys / values (current half)
  const uint8_t* bv;
  const uint8_t* kc;  // incoming token
  const uint8_t* vc;
  const int32_t* win; // slot -> window (v3)
  int kstride, vchunks, nbuf, vsel;  // vsel: value-chunk index of this thread
  int NS;             // v3: list entries >= NS are tail rows (NS + t)
};

// List entries: (slot, window).  Tail entries are (-1 - t, 0): t < nbuf is
// buffer row t, t == nbuf the incoming token.
template <int D, int FMT>
__device__ __forceinline__ void load_tile(const UnitPtrs& up, const int2* lst, int t0, int gid, int tig,
                                          Tile<D, FMT>& T) {
  using Gm = Geo<D, FMT>;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int2 e = lst[t0 + gid + 8 * r];
    const uint8_t* kr;
    if constexpr (FMT == kFmtTail) {
      if (e.x >= 0) kr = up.k + e.x * up.kstride;
      else kr = (-1 - e.x) < up.nbuf ? up.bk + (-1 - e.x) * (D * 2) : up.kc;
    } else {
      kr = up.k + e.x * up.kstride;
    }
    T.k[r] = ldg_words<Gm::KW>(kr + tig * Gm::KBYTES);
    if constexpr (FMT == TKV_FMT_FP8) T.kf[r] = __ldg(up.kf + e.y);
    if constexpr (Gm::SCALED) T.ks[r] = ldg_words<Gm::SW>(up.ks + e.y * D + tig * Gm::CPT);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int2 e = lst[t0 + tig * 2 + (i & 1) + 8 * (i >> 1)];
    const uint8_t* vr;
    if constexpr (FMT == kFmtTail) {
      if (e.x >= 0) vr = up.v + e.x * up.kstride;
      else vr = (-1 - e.x) < up.nbuf ? up.bv + (-1 - e.x) * (D * 2) : up.vc;
    } else {
      vr = up.v + e.x * up.kstride;
    }
    vr += gid * Gm::VBYTES;
    if constexpr (Gm::VBYTES >= 4) {
      T.v[i] = ldg_words<Gm::VW>(vr);
    } else {
      T.v[i].w[0] = Gm::VBYTES == 2 ? (uint32_t)__ldg(reinterpret_cast<const unsigned short*>(vr)) : (uint32_t)__ldg(vr);
    }
    if constexpr (FMT == TKV_FMT_FP8) T.vf[i] = __ldg(up.vf + e.y);
    if constexpr (Gm::SCALED) T.vs[i] = __ldg(up.vs + e.x * up.vchunks + up.vsel);
  }
}

template <int D>
struct Acc {
  float o[D / 16][4];
  float m[2], l[2];  // heads tig*2, tig*2+1 (log2 domain reference max, denominator)
};

template <int D, int FMT>
__device__ __forceinline__ void compute_tile(const Tile<D, FMT>& T, const uint32_t (&qb)[D / 16][2],
                                             const uint32_t* qbb, float qscale, int G, bool maxpool, int nvalid,
                                             int gid, int tig, float* ps, Acc<D>& A) {
  using Gm = Geo<D, FMT>;
  // ---- S = K q^T ----------------------------------------------------------
  float s[4] = {0.f, 0.f, 0.f, 0.f};
  if constexpr (FMT == TKV_FMT_TERNARY) {
    // 8 codes per 16-bit half -> 8 e2m1 nibbles (one word), 4 k-steps per code word
#pragma unroll
    for (int jw = 0; jw < Gm::KW; ++jw) {
      uint32_t nib[2][2];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        nib[r][0] = tern_spread(T.k[r].w[jw]);
        nib[r][1] = tern_spread(T.k[r].w[jw] >> 16);
      }
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int j = jw * 4 + jj;
        uint32_t a[4];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          uint32_t lo, hi, slo, shi;
          e2m1x2_b(nib[r][jj >> 1], (jj & 1) * 2, lo);
          e2m1x2_b(nib[r][jj >> 1], (jj & 1) * 2 + 1, hi);
          e4m3x4(T.ks[r].w[j], slo, shi);
          a[r] = hmul2(lo, slo);
          a[2 + r] = hmul2(hi, shi);
        }
        mma16816<false>(s, a[0], a[1], a[2], a[3], qb[j][0], qb[j][1]);
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < Gm::KT; ++j) {
      uint32_t a[4];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        uint32_t lo, hi;
        if constexpr (FMT == TKV_FMT_NVFP4) {
          e2m1x2_b(T.k[r].w[j >> 1], (j & 1) * 2, lo);
          e2m1x2_b(T.k[r].w[j >> 1], (j & 1) * 2 + 1, hi);
          uint32_t slo, shi;
          e4m3x4(T.ks[r].w[j], slo, shi);
          lo = hmul2(lo, slo);
          hi = hmul2(hi, shi);
        } else if constexpr (FMT == TKV_FMT_FP8) {
          e4m3x4(T.k[r].w[j], lo, hi);
        } else {  // raw bf16 words: channels 4j, 4j+1 | 4j+2, 4j+3
          lo = T.k[r].w[2 * j];
          hi = T.k[r].w[2 * j + 1];
        }
        a[r] = lo;       // a0a1 (row gid) / a2a3 (row gid+8), cols tig*2..+1
        a[2 + r] = hi;   // a4a5 / a6a7, cols tig*2+8..+9
      }
      if constexpr (Gm::BF16) mma16816<true>(s, a[0], a[1], a[2], a[3], qbb[j * 2], qbb[j * 2 + 1]);
      else mma16816<false>(s, a[0], a[1], a[2], a[3], qb[j][0], qb[j][1]);
    }
  }
  // logits (log2 domain); rows: s0,s1 -> token gid, s2,s3 -> token gid+8
  float L[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = i >> 1, h = tig * 2 + (i & 1);
    float x = s[i] * qscale;
    if constexpr (FMT == TKV_FMT_FP8) x *= T.kf[r];
    L[i] = (gid + 8 * r < nvalid && h < G) ? x : -CUDART_INF_F;
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
  // ---- online softmax per head column (lazy rescale) -------------------------
  float p[4];
  bool grow = false;
  float mnew[2];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    float tmax = fmaxf(L[c], L[2 + c]);
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 4));
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 8));
    tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 16));
    mnew[c] = tmax > A.m[c] + kRescale ? tmax : A.m[c];
    grow = grow || mnew[c] != A.m[c];
  }
  if (__any_sync(0xffffffffu, grow)) {
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const float corr = A.m[c] == -CUDART_INF_F ? 0.0f : exp2f(A.m[c] - mnew[c]);
      if (mnew[c] != A.m[c]) {
        A.l[c] *= corr;
#pragma unroll
        for (int mt = 0; mt < Gm::MT; ++mt) {
          A.o[mt][c] *= corr;
          A.o[mt][2 + c] *= corr;
        }
        A.m[c] = mnew[c];
      }
    }
  }
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const bool live = A.m[c] != -CUDART_INF_F;
    p[c] = live ? exp2f(L[c] - A.m[c]) : 0.0f;
    p[2 + c] = live ? exp2f(L[2 + c] - A.m[c]) : 0.0f;
    float sum = p[c] + p[2 + c];
    sum += __shfl_xor_sync(0xffffffffu, sum, 4);
    sum += __shfl_xor_sync(0xffffffffu, sum, 8);
    sum += __shfl_xor_sync(0xffffffffu, sum, 16);
    A.l[c] += sum;
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
    pb[i] = ps[(tig * 2 + (i & 1) + 8 * (i >> 1)) * 8 + gid];
    if constexpr (FMT == TKV_FMT_FP8) pb[i] *= T.vf[i];
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
  if constexpr (Gm::SCALED) {
#pragma unroll
    for (int i = 0; i < 4; ++i) e4m3x2_b(T.vs[i], 0, vsc[i]);
  }
  uint32_t tsp[4][(Gm::MT + 3) / 4];  // ternary: e2m1 nibbles of each 8-code half-word
  if constexpr (FMT == TKV_FMT_TERNARY) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int h = 0; h < (Gm::MT + 3) / 4; ++h) tsp[i][h] = tern_spread(T.v[i].w[0] >> (16 * h));
  }
#pragma unroll
  for (int mt = 0; mt < Gm::MT; ++mt) {
    uint32_t x[4];  // per PV token: f16x2 / bf16x2 of channels (2mt, 2mt+1) of the thread's range
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if constexpr (FMT == TKV_FMT_NVFP4) {
        uint32_t h;
        e2m1x2_b(T.v[i].w[mt >> 2], mt & 3, h);
        x[i] = hmul2(h, vsc[i]);
      } else if constexpr (FMT == TKV_FMT_FP8) {
        uint32_t lo, hi;
        e4m3x4(T.v[i].w[mt >> 1], lo, hi);
        x[i] = (mt & 1) ? hi : lo;
      } else if constexpr (FMT == TKV_FMT_TERNARY) {
        // codes 2mt, 2mt+1 = byte mt & 3 of the spread of half-word mt >> 2
        uint32_t h;
        e2m1x2_b(tsp[i][mt >> 2], mt & 3, h);
        x[i] = hmul2(h, vsc[i]);
      } else {
        x[i] = T.v[i].w[mt];
      }
    }
    const uint32_t a0 = __byte_perm(x[0], x[1], 0x5410);  // row gid (ch 2mt), tokens tig*2, tig*2+1
    const uint32_t a1 = __byte_perm(x[0], x[1], 0x7632);  // row gid+8 (ch 2mt+1)
    const uint32_t a2 = __byte_perm(x[2], x[3], 0x5410);  // row gid, tokens +8, +9
    const uint32_t a3 = __byte_perm(x[2], x[3], 0x7632);
    mma16816<Gm::BF16>(A.o[mt], a0, a1, a2, a3, bh0, bh1);
    mma16816<Gm::BF16>(A.o[mt], a0, a1, a2, a3, bl0, bl1);
  }
}

// Tiles of one format with global tile index g = warp + k * kWarps in
// [g0, g0 + tiles); the list is padded to whole tiles.
template <int D, int FMT>
__device__ __forceinline__ void run_format(const UnitPtrs& up, const int2* lst, int n, int g0, int warp,
                                           const uint32_t (&qb)[D / 16][2], const uint32_t* qbb, float qscale,
                                           int G, bool maxpool, int gid, int tig, float* ps, Acc<D>& A) {
  const int tiles = (n + 15) / 16;
  int t = ((warp - g0) % kWarps + kWarps) % kWarps;
  if (t >= tiles) return;
  if constexpr (FMT == kFmtTail) {  // few tiles, wide rows: no double buffering (registers)
    for (; t < tiles; t += kWarps) {
      Tile<D, FMT> cur;
      load_tile<D, FMT>(up, lst, t * 16, gid, tig, cur);
      compute_tile<D, FMT>(cur, qb, qbb, qscale, G, maxpool, n - t * 16, gid, tig, ps, A);
    }
    return;
  }
  Tile<D, FMT> ta, tb;
  load_tile<D, FMT>(up, lst, t * 16, gid, tig, ta);
  while (true) {
    if (t + kWarps < tiles) load_tile<D, FMT>(up, lst, (t + kWarps) * 16, gid, tig, tb);
    compute_tile<D, FMT>(ta, qb, qbb, qscale, G, maxpool, n - t * 16, gid, tig, ps, A);
    t += kWarps;
    if (t >= tiles) break;
    if (t + kWarps < tiles) load_tile<D, FMT>(up, lst, (t + kWarps) * 16, gid, tig, ta);
    compute_tile<D, FMT>(tb, qb, qbb, qscale, G, maxpool, n - t * 16, gid, tig, ps, A);
    t += kWarps;
    if (t >= tiles) break;
  }
}

template <int D, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) attend_mma_kernel(TkvState st, const void* __restrict__ qin,
                                                                  const void* __restrict__ kin,
                                                                  const void* __restrict__ vin,
                                                                  float* __restrict__ out, int buf_half, int nbuf,
                                                                  int put_half, int put_slot) {
  tkv_step_scalars(st, buf_half, nbuf, put_half, put_slot);
  const TkvDims& dm = st.dm;
  const int li = blockIdx.x;            // launch-local index: q/k/v/out rows
  const int u = tkv_unit_of(st, li);    // unit: cache state
  const int G = dm.G, R = dm.maxpool ? 1 : G;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  extern __shared__ __align__(16) uint8_t dyn[];
  float* red = reinterpret_cast<float*>(dyn);                       // [kWarps * 8][2 + D]
  float* ps_all = red + kWarps * 8 * (2 + D);                         // [kWarps][16 * 8]
  uint32_t* qbb_all = reinterpret_cast<uint32_t*>(ps_all + kWarps * 128);  // [32 lanes][D/8] bf16 B frags
  int2* list = reinterpret_cast<int2*>(qbb_all + 32 * (D / 8));        // [NS + g + 1 + 4*16] (slot, window)
  int2* binfo = list + (dm.NS + dm.g + 1 + 4 * 16);                    // [P] (live mask, list position)
  __shared__ int cnt[5], off[5], wsum[kWarps][4];
  const float qscale = dm.scale * kLog2e;

  // q^T B fragments: head gid, channels tig*D/4 + 4j + {0,1} / {2,3}; f16 in
  // registers, the raw bf16 words in shared memory for the bf16 tiles.
  uint32_t qb[D / 16][2];
  {
    const uint16_t* qq = reinterpret_cast<const uint16_t*>(qin) + ((int64_t)li * G + gid) * D + tig * (D / 4);
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
  // Live-slot lists per format with window indices (physical order), each
  // padded to a multiple of 16 entries; the raw tail follows the raw list.
  //   pass 1: thread -> contiguous blocks: live masks + per-format counts
  //   scan:   per-format offsets of each thread's first block
  //   pass 2: each thread writes its blocks' live slots (with their windows)
  const int P = dm.P, bs = dm.bs;
  const int8_t* th = st.blk_thought + (int64_t)u * P;
  const uint8_t* fl = st.blk_filled + (int64_t)u * P;
  const uint32_t* ev = st.blk_evict + (int64_t)u * P;
  const int per = (P + kThreads - 1) / kThreads;
  const int b0 = threadIdx.x * per, b1 = min(P, b0 + per);
  int c[4] = {0, 0, 0, 0};
  for (int b = b0; b < b1; ++b) {
    const int t = th[b];
    uint32_t live = 0;
    int f = 0;
    if (t >= 0) {
      live = ~ev[b] & (fl[b] >= 32 ? 0xffffffffu : ((1u << fl[b]) - 1u));
      f = dm.band_fmt[t];
      c[f] += __popc(live);
    }
    binfo[b] = make_int2((int)live, f);
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
      int tot = 0;
      for (int w = 0; w < kWarps; ++w) tot += wsum[w][f];
      if (f == TKV_FMT_RAW) tot += nbuf + 1;  // tail tokens ride in the raw list
      off[f] = run;
      cnt[f] = tot;
      run += (tot + 15) & ~15;  // padded to whole tiles
    }
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
      const int2 bi = binfo[b];
      uint32_t live = (uint32_t)bi.x;
      int pos = 0;
#pragma unroll
      for (int f = 0; f < 4; ++f)
        if (bi.y == f) { pos = w[f]; w[f] += __popc(live); }
      while (live) {
        const int sl = __ffs(live) - 1;
        live &= live - 1;
        list[pos++] = make_int2(b * bs + sl, max(0, __ldg(swin + b * bs + sl)));
      }
    }
    const int rawn = cnt[TKV_FMT_RAW] - (nbuf + 1);
    for (int t = threadIdx.x; t <= nbuf; t += kThreads) list[off[TKV_FMT_RAW] + rawn + t] = make_int2(-1 - t, 0);
  }
  __syncthreads();
  // padding entries: copies of each list's first entry (masked to -inf logits)
  if (threadIdx.x < 4 * 16) {
    const int f = threadIdx.x >> 4, i = threadIdx.x & 15;
    const int n = cnt[f];
    if (n > 0 && n + i < ((n + 15) & ~15)) list[off[f] + n + i] = list[off[f]];
  }
  __syncthreads();
  UnitPtrs up;
  {
    up.kstride = dm.kstride;
    up.vchunks = dm.vchunks;
    up.k = st.slot_k + (int64_t)u * dm.NS * dm.kstride;
    up.v = st.slot_v + (int64_t)u * dm.NS * dm.kstride;
    up.vs = st.slot_vs + (int64_t)u * dm.NS * dm.vchunks;
    up.ks = st.win_ks + (int64_t)u * dm.NW * D;
    up.kf = st.win_kf + (int64_t)u * dm.NW;
    up.vf = st.win_vf + (int64_t)u * dm.NW;
    const int64_t row = (int64_t)dm.g * D * 2;
    up.bk = st.buf + ((int64_t)u * 4 + buf_half * 2 + 0) * row;
    up.bv = st.buf + ((int64_t)u * 4 + buf_half * 2 + 1) * row;
    up.kc = reinterpret_cast<const uint8_t*>(kin) + (int64_t)li * D * 2;
    up.vc = reinterpret_cast<const uint8_t*>(vin) + (int64_t)li * D * 2;
    up.nbuf = nbuf;
    up.vsel = (gid * (D / 8)) / dm.g;
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
    run_format<D, TKV_FMT_NVFP4>(up, list + off[TKV_FMT_NVFP4], cnt[TKV_FMT_NVFP4], g0, warp, qb, qbb, qscale, G,
                                 mp, gid, tig, ps, A);
    g0 += (cnt[TKV_FMT_NVFP4] + 15) / 16;
  }
  if (cnt[TKV_FMT_TERNARY]) {
    run_format<D, TKV_FMT_TERNARY>(up, list + off[TKV_FMT_TERNARY], cnt[TKV_FMT_TERNARY], g0, warp, qb, qbb,
                                   qscale, G, mp, gid, tig, ps, A);
    g0 += (cnt[TKV_FMT_TERNARY] + 15) / 16;
  }
  if (cnt[TKV_FMT_FP8]) {
    run_format<D, TKV_FMT_FP8>(up, list + off[TKV_FMT_FP8], cnt[TKV_FMT_FP8], g0, warp, qb, qbb, qscale, G, mp,
                               gid, tig, ps, A);
    g0 += (cnt[TKV_FMT_FP8] + 15) / 16;
  }
  run_format<D, kFmtTail>(up, list + off[TKV_FMT_RAW], cnt[TKV_FMT_RAW], g0, warp, qb, qbb, qscale, G, mp, gid,
                          tig, ps, A);
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
    out[((int64_t)li * R + r) * D + ch] = O / Ls;
  }
  if (put_slot >= 0) {  // buffer the incoming token (sim.cpp:796-808)
    const int64_t row = (int64_t)dm.g * D;
    uint16_t* bk = reinterpret_cast<uint16_t*>(st.buf) + ((int64_t)u * 4 + put_half * 2 + 0) * row + (int64_t)put_slot * D;
    uint16_t* bv = reinterpret_cast<uint16_t*>(st.buf) + ((int64_t)u * 4 + put_half * 2 + 1) * row + (int64_t)put_slot * D;
    const uint16_t* ks = reinterpret_cast<const uint16_t*>(kin) + (int64_t)li * D;
    const uint16_t* vs = reinterpret_cast<const uint16_t*>(vin) + (int64_t)li * D;
    for (int i = threadIdx.x; i < D; i += kThreads) {
      bk[i] = ks[i];
      bv[i] = vs[i];
    }
  }
}


// ===========================================================================
// v4: one warp per unit.  No block-level barriers: the warp builds its own
// live list (u16 slot ids; tail rows are NS + t), walks every tile of its
// unit, and writes the normalised output itself.  Window indices are not in
// the list: they are fetched two tiles ahead (slot -> window), so the scale
// loads of tile t+1 are issued while tile t computes.
//
// Instruction economy per 16-token tile (the kernel is issue bound):
//   * addresses: per-thread, per-format base pointers are formed once per
//     list; a slot row is one mad.wide.u32 (IMAD.WIDE.U32) of the u16 slot id
//     and the 32-bit stride -- no 64-bit index arithmetic per load;
//   * softmax: the running max moves only when some logit exceeds it by more
//     than 2^8 (lazy rescale), decided by one vote per tile; the max and the
//     denominator are reduced across lanes only on that rare path and once at
//     the end (each lane keeps partial denominators of its own tokens);
//   * PV with R <= 4 output rows: the hi and lo halves of P ride in the
//     MMA's N dimension (columns h = hi, 4 + h = lo), one mma per m-tile
//     instead of two; the halves are added once in the epilogue.
// ===========================================================================
__device__ __forceinline__ const uint8_t* wide_at(const void* base, uint32_t i, uint32_t stride) {
  uint64_t r;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(i), "r"(stride), "l"(reinterpret_cast<uint64_t>(base)));
  return reinterpret_cast<const uint8_t*>(r);
}

// Per-thread base pointers of one format's tiles (loop invariant).
template <int D, int FMT>
struct Bases {
  const uint8_t* k;   // slot_k + tig * KBYTES
  const uint8_t* v;   // slot_v + gid * VBYTES
  const uint8_t* vs;  // slot_vs + vsel
  const uint8_t* ks;  // win_ks + tig * CPT
  __device__ Bases(const UnitPtrs& up, int gid, int tig) {
    using Gm = Geo<D, FMT>;
    k = up.k + tig * Gm::KBYTES;
    v = up.v + gid * Gm::VBYTES;
    vs = up.vs + up.vsel;
    ks = up.ks + tig * Gm::CPT;
  }
};

template <int D, int FMT>
__device__ __forceinline__ void load_wins4(const UnitPtrs& up, const uint16_t* lst, int t0, int gid, int tig,
                                           uint32_t (&wk)[2], uint32_t (&wv)[4]) {
  if constexpr (Geo<D, FMT>::SCALED || FMT == TKV_FMT_FP8) {
#pragma unroll
    for (int r = 0; r < 2; ++r)  // live quantised slots: >= 0
      wk[r] = (uint32_t)__ldg(reinterpret_cast<const int32_t*>(wide_at(up.win, lst[t0 + gid + 8 * r], 4)));
  }
  if constexpr (FMT == TKV_FMT_FP8) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      wv[i] = (uint32_t)__ldg(
          reinterpret_cast<const int32_t*>(wide_at(up.win, lst[t0 + tig * 2 + (i & 1) + 8 * (i >> 1)], 4)));
  }
}

template <int D, int FMT, int KS>
__device__ __forceinline__ void load_tile4(const UnitPtrs& up, const Bases<D, FMT>& B, const uint16_t* lst, int t0,
                                           int gid, int tig, const uint32_t (&wk)[2], const uint32_t (&wv)[4],
                                           Tile<D, FMT>& T) {
  using Gm = Geo<D, FMT>;
  // KS > 0: the slot-row stride is a compile-time constant (and the value
  // chunks per slot D / 16), so each row address is one IMAD.WIDE.U32 with an
  // immediate; a runtime stride makes ptxas split it into a product plus a
  // 64-bit add (three instructions per load address).
  const uint32_t ks = KS > 0 ? (uint32_t)KS : (uint32_t)up.kstride;
  const uint32_t vc = KS > 0 ? (uint32_t)(D / 16) : (uint32_t)up.vchunks;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const uint32_t e = lst[t0 + gid + 8 * r];
    const uint8_t* kr;
    if constexpr (FMT == kFmtTail) {
      if (e < (uint32_t)up.NS) kr = wide_at(B.k, e, ks);
      else kr = (int)e - up.NS < up.nbuf ? up.bk + ((int)e - up.NS) * (D * 2) + tig * Gm::KBYTES
                                         : up.kc + tig * Gm::KBYTES;
    } else {
      kr = wide_at(B.k, e, ks);
    }
    T.k[r] = ldg_words<Gm::KW>(kr);
    if constexpr (FMT == TKV_FMT_FP8) T.kf[r] = __ldg(reinterpret_cast<const float*>(wide_at(up.kf, wk[r], 4)));
    if constexpr (Gm::SCALED) T.ks[r] = ldg_words<Gm::SW>(wide_at(B.ks, wk[r], D));
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t e = lst[t0 + tig * 2 + (i & 1) + 8 * (i >> 1)];
    const uint8_t* vr;
    if constexpr (FMT == kFmtTail) {
      if (e < (uint32_t)up.NS) vr = wide_at(B.v, e, ks);
      else vr = (int)e - up.NS < up.nbuf ? up.bv + ((int)e - up.NS) * (D * 2) + gid * Gm::VBYTES
                                         : up.vc + gid * Gm::VBYTES;
    } else {
      vr = wide_at(B.v, e, ks);
    }
    if constexpr (Gm::VBYTES >= 4) {
      T.v[i] = ldg_words<Gm::VW>(vr);
    } else {
      T.v[i].w[0] = Gm::VBYTES == 2 ? (uint32_t)__ldg(reinterpret_cast<const unsigned short*>(vr)) : (uint32_t)__ldg(vr);
    }
    if constexpr (FMT == TKV_FMT_FP8) T.vf[i] = __ldg(reinterpret_cast<const float*>(wide_at(up.vf, wv[i], 4)));
    if constexpr (Gm::SCALED) T.vs[i] = __ldg(wide_at(B.vs, e, vc));
  }
}

template <int D, int FMT, bool PVN>
__device__ __forceinline__ void compute_tile4(const Tile<D, FMT>& T, const uint32_t (&qb)[D / 16][2],
                                              const uint32_t* qbb, float qscale, bool maxpool, int nvalid,
                                              int gid, int tig, float* ps, Acc<D>& A) {
  using Gm = Geo<D, FMT>;
  // ---- S = K q^T ----------------------------------------------------------
  float s[4] = {0.f, 0.f, 0.f, 0.f};
  if constexpr (FMT == TKV_FMT_TERNARY) {
    // 8 codes per 16-bit half -> 8 e2m1 nibbles (one word), 4 k-steps per code word
#pragma unroll
    for (int jw = 0; jw < Gm::KW; ++jw) {
      uint32_t nib[2][2];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        nib[r][0] = tern_spread(T.k[r].w[jw]);
        nib[r][1] = tern_spread(T.k[r].w[jw] >> 16);
      }
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int j = jw * 4 + jj;
        uint32_t a[4];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          uint32_t lo, hi, slo, shi;
          e2m1x2_b(nib[r][jj >> 1], (jj & 1) * 2, lo);
          e2m1x2_b(nib[r][jj >> 1], (jj & 1) * 2 + 1, hi);
          e4m3x4(T.ks[r].w[j], slo, shi);
          a[r] = hmul2(lo, slo);
          a[2 + r] = hmul2(hi, shi);
        }
        mma16816<false>(s, a[0], a[1], a[2], a[3], qb[j][0], qb[j][1]);
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < Gm::KT; ++j) {
      uint32_t a[4];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        uint32_t lo, hi;
        if constexpr (FMT == TKV_FMT_NVFP4) {
          e2m1x2_b(T.k[r].w[j >> 1], (j & 1) * 2, lo);
          e2m1x2_b(T.k[r].w[j >> 1], (j & 1) * 2 + 1, hi);
          uint32_t slo, shi;
          e4m3x4(T.ks[r].w[j], slo, shi);
          lo = hmul2(lo, slo);
          hi = hmul2(hi, shi);
        } else if constexpr (FMT == TKV_FMT_FP8) {
          e4m3x4(T.k[r].w[j], lo, hi);
        } else {  // raw bf16 words: channels 4j, 4j+1 | 4j+2, 4j+3
          lo = T.k[r].w[2 * j];
          hi = T.k[r].w[2 * j + 1];
        }
        a[r] = lo;
        a[2 + r] = hi;
      }
      if constexpr (Gm::BF16) mma16816<true>(s, a[0], a[1], a[2], a[3], qbb[j * 2], qbb[j * 2 + 1]);
      else mma16816<false>(s, a[0], a[1], a[2], a[3], qb[j][0], qb[j][1]);
    }
  }
  // logits (log2 domain); rows: s0,s1 -> token gid, s2,s3 -> token gid+8.
  // Heads >= G have q = 0: their logits are 0, finite, and never written out.
  float L[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float x = s[i] * qscale;
    if constexpr (FMT == TKV_FMT_FP8) x *= T.kf[i >> 1];
    L[i] = x;
  }
  if (nvalid < 16) {  // the list's last tile: padding rows -> -inf (warp-uniform)
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (gid + 8 * (i >> 1) >= nvalid) L[i] = -CUDART_INF_F;
  }
  if (maxpool) {
    // one pooled row per token: max over the G heads, kept in column 0
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      float mx = fmaxf(L[2 * r], L[2 * r + 1]);
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      L[2 * r] = (PVN ? (tig & 1) == 0 : tig == 0) ? mx : -CUDART_INF_F;  // PVN: column 4 mirrors 0
      L[2 * r + 1] = -CUDART_INF_F;
    }
  }
  // ---- online softmax per head column, lazy rescale --------------------------
  const bool grow = L[0] > A.m[0] + kRescale || L[2] > A.m[0] + kRescale || L[1] > A.m[1] + kRescale ||
                    L[3] > A.m[1] + kRescale;
  if (__any_sync(0xffffffffu, grow)) {  // rare: a new reference max for some column
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      float tmax = fmaxf(L[c], L[2 + c]);
      tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 4));
      tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 8));
      tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, 16));
      if (tmax > A.m[c] + kRescale) {
        const float corr = A.m[c] == -CUDART_INF_F ? 0.0f : exp2f(A.m[c] - tmax);
        A.l[c] *= corr;
#pragma unroll
        for (int mt = 0; mt < Gm::MT; ++mt) {  // (PVN: lo columns mirror their head's max, same corr)
          A.o[mt][c] *= corr;
          A.o[mt][2 + c] *= corr;
        }
        A.m[c] = tmax;
      }
    }
  }
  float p[4];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    // columns that never saw a finite logit (max-pool's unused columns) stay 0
    const bool live = A.m[c] != -CUDART_INF_F;
    p[c] = live ? exp2f(L[c] - A.m[c]) : 0.0f;
    p[2 + c] = live ? exp2f(L[2 + c] - A.m[c]) : 0.0f;
    A.l[c] += p[c] + p[2 + c];  // this lane's tokens only; reduced across lanes at the end
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
    pb[i] = ps[(tig * 2 + (i & 1) + 8 * (i >> 1)) * 8 + (PVN ? (gid & 3) : gid)];
    if constexpr (FMT == TKV_FMT_FP8) pb[i] *= T.vf[i];
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
  if constexpr (PVN) {  // columns 0..3: hi halves of heads 0..3, columns 4..7: lo halves
    if (gid >= 4) { bh0 = bl0; bh1 = bl1; }
  }
  // ---- O^T += V^T P ----------------------------------------------------------
  // Grouped formats (NVFP4, ternary): the code words of a PV token pair are
  // interleaved nibble-wise before conversion -- byte k of lo[p] holds channel
  // 2k of tokens (2p, 2p+1), byte k of hi[p] channel 2k+1 -- so one F2FP yields
  // an A-fragment register directly (no byte_perm transpose per m-tile), and the
  // pair's two value-chunk scales form one f16x2 multiplier.
  constexpr bool kPair = FMT == TKV_FMT_NVFP4 || FMT == TKV_FMT_TERNARY;
  uint32_t vsc[4];
  if constexpr (kPair) {
#pragma unroll
    for (int pp = 0; pp < 2; ++pp) {
      const uint32_t b = __byte_perm(T.vs[2 * pp], T.vs[2 * pp + 1], 0x0040);  // (s_2p, s_2p+1)
      asm("{\n .reg .b16 h0, h1;\n mov.b32 {h0, h1}, %1;\n cvt.rn.f16x2.e4m3x2 %0, h0;\n}" : "=r"(vsc[pp]) : "r"(b));
    }
  }
  constexpr int kVW = FMT == TKV_FMT_TERNARY ? (Gm::MT + 3) / 4 : Gm::VW;  // nibble words per token
  uint32_t vlo[2][kVW], vhi[2][kVW];
  if constexpr (kPair) {
#pragma unroll
    for (int w = 0; w < kVW; ++w)
#pragma unroll
      for (int pp = 0; pp < 2; ++pp) {
        uint32_t wa, wb;
        if constexpr (FMT == TKV_FMT_TERNARY) {
          wa = tern_spread(T.v[2 * pp].w[0] >> (16 * w));
          wb = tern_spread(T.v[2 * pp + 1].w[0] >> (16 * w));
        } else {
          wa = T.v[2 * pp].w[w];
          wb = T.v[2 * pp + 1].w[w];
        }
        vlo[pp][w] = (wa & 0x0f0f0f0fu) | ((wb << 4) & 0xf0f0f0f0u);
        vhi[pp][w] = ((wa >> 4) & 0x0f0f0f0fu) | (wb & 0xf0f0f0f0u);
      }
  }
#pragma unroll
  for (int mt = 0; mt < Gm::MT; ++mt) {
    uint32_t a0, a1, a2, a3;
    if constexpr (kPair) {
      uint32_t c0, c1, c2, c3;
      e2m1x2_b(vlo[0][mt >> 2], mt & 3, c0);  // row gid (ch 2mt), tokens tig*2, tig*2+1
      e2m1x2_b(vhi[0][mt >> 2], mt & 3, c1);  // row gid+8 (ch 2mt+1)
      e2m1x2_b(vlo[1][mt >> 2], mt & 3, c2);  // row gid, tokens +8, +9
      e2m1x2_b(vhi[1][mt >> 2], mt & 3, c3);
      a0 = hmul2(c0, vsc[0]);
      a1 = hmul2(c1, vsc[0]);
      a2 = hmul2(c2, vsc[1]);
      a3 = hmul2(c3, vsc[1]);
    } else {
      uint32_t x[4];  // per PV token: f16x2 / bf16x2 of channels (2mt, 2mt+1) of the thread's range
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if constexpr (FMT == TKV_FMT_FP8) {
          uint32_t lo, hi;
          e4m3x4(T.v[i].w[mt >> 1], lo, hi);
          x[i] = (mt & 1) ? hi : lo;
        } else {
          x[i] = T.v[i].w[mt];
        }
      }
      a0 = __byte_perm(x[0], x[1], 0x5410);  // row gid (ch 2mt), tokens tig*2, tig*2+1
      a1 = __byte_perm(x[0], x[1], 0x7632);  // row gid+8 (ch 2mt+1)
      a2 = __byte_perm(x[2], x[3], 0x5410);  // row gid, tokens +8, +9
      a3 = __byte_perm(x[2], x[3], 0x7632);
    }
    mma16816<Gm::BF16>(A.o[mt], a0, a1, a2, a3, bh0, bh1);
    if constexpr (!PVN) mma16816<Gm::BF16>(A.o[mt], a0, a1, a2, a3, bl0, bl1);
  }
}

template <int D, int FMT, bool PVN, int KS>
__device__ __forceinline__ void run_format4(const UnitPtrs& up, const uint16_t* lst, int n,
                                            const uint32_t (&qb)[D / 16][2], const uint32_t* qbb, float qscale,
                                            bool maxpool, int gid, int tig, float* ps, Acc<D>& A) {
  const int tiles = (n + 15) / 16;
  if (tiles == 0) return;
  const Bases<D, FMT> B(up, gid, tig);
  if constexpr (FMT == kFmtTail) {  // few tiles, wide rows: no double buffering (registers)
    uint32_t wk[2] = {0, 0}, wv[4] = {0, 0, 0, 0};
    for (int t = 0; t < tiles; ++t) {
      Tile<D, FMT> cur;
      load_tile4<D, FMT, KS>(up, B, lst, t * 16, gid, tig, wk, wv, cur);
      compute_tile4<D, FMT, PVN>(cur, qb, qbb, qscale, maxpool, n - t * 16, gid, tig, ps, A);
    }
    return;
  }
  uint32_t wk0[2] = {0, 0}, wv0[4] = {0, 0, 0, 0}, wk1[2] = {0, 0}, wv1[4] = {0, 0, 0, 0};
  Tile<D, FMT> ta, tb;
  load_wins4<D, FMT>(up, lst, 0, gid, tig, wk0, wv0);
  load_tile4<D, FMT, KS>(up, B, lst, 0, gid, tig, wk0, wv0, ta);
  if (tiles > 1) load_wins4<D, FMT>(up, lst, 16, gid, tig, wk1, wv1);
  int t = 0;
  while (true) {
    // ta holds tile t; wk1 the windows of tile t + 1
    if (t + 1 < tiles) {
      load_tile4<D, FMT, KS>(up, B, lst, (t + 1) * 16, gid, tig, wk1, wv1, tb);
      if (t + 2 < tiles) load_wins4<D, FMT>(up, lst, (t + 2) * 16, gid, tig, wk0, wv0);
    }
    compute_tile4<D, FMT, PVN>(ta, qb, qbb, qscale, maxpool, n - t * 16, gid, tig, ps, A);
    if (++t >= tiles) break;
    // tb holds tile t; wk0 the windows of tile t + 1
    if (t + 1 < tiles) {
      load_tile4<D, FMT, KS>(up, B, lst, (t + 1) * 16, gid, tig, wk0, wv0, ta);
      if (t + 2 < tiles) load_wins4<D, FMT>(up, lst, (t + 2) * 16, gid, tig, wk1, wv1);
    }
    compute_tile4<D, FMT, PVN>(tb, qb, qbb, qscale, maxpool, n - t * 16, gid, tig, ps, A);
    if (++t >= tiles) break;
  }
}

// Per-warp shared memory of the v3 kernel.
template <int D>
struct WarpSmem {
  static constexpr int kQbb = 32 * (D / 8);  // u32: bf16 q fragments
  static __host__ __device__ size_t bytes(int live_cap, int g, int P) {
    const size_t lst = ((size_t)(live_cap + g + 1 + 4 * 16) * 2 + 15) / 16 * 16;
    return (size_t)kQbb * 4 + 128 * 4 + (size_t)P * 8 + lst;
  }
};

// PVN: at most 4 output rows per unit (max-pool, or G <= 4): P's hi/lo halves
// share one PV mma (compute_tile4).  Without max-pool the q^T operand's
// columns 4..7 repeat heads 0..3, so the lanes holding the lo columns see their
// head's own logits and track the same running max and denominator.
template <int D, int MINB, bool PVN, int KS>
__global__ void __launch_bounds__(kThreads, MINB) attend_warp_kernel(TkvState st, const void* __restrict__ qin,
                                                                    const void* __restrict__ kin,
                                                                    const void* __restrict__ vin,
                                                                    float* __restrict__ out, int buf_half, int nbuf,
                                                                    int put_half, int put_slot) {
  tkv_step_scalars(st, buf_half, nbuf, put_half, put_slot);
  const TkvDims& dm = st.dm;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int li = blockIdx.x * kWarps + warp;  // launch-local index: q/k/v/out rows
  if (li >= tkv_launch_units(st)) return;
  const int u = tkv_unit_of(st, li);          // unit: cache state
  const int G = dm.G, R = dm.maxpool ? 1 : G;
  const int gid = lane >> 2, tig = lane & 3;
  const int P = dm.P, bs = dm.bs, NS = dm.NS;
  extern __shared__ __align__(16) uint8_t dyn[];
  uint8_t* mine = dyn + (size_t)warp * WarpSmem<D>::bytes(st.max_live, dm.g, P);
  uint32_t* qbb = reinterpret_cast<uint32_t*>(mine) + lane * (D / 8);
  float* ps = reinterpret_cast<float*>(mine + WarpSmem<D>::kQbb * 4);
  int2* binfo = reinterpret_cast<int2*>(mine + WarpSmem<D>::kQbb * 4 + 128 * 4);
  uint16_t* list = reinterpret_cast<uint16_t*>(binfo + P);
  const float qscale = dm.scale * kLog2e;

  uint32_t qb[D / 16][2];
  {
    const int hq = PVN && !dm.maxpool ? (gid & 3) : gid;  // q^T column gid holds head hq
    const uint16_t* qq = reinterpret_cast<const uint16_t*>(qin) + ((int64_t)li * G + hq) * D + tig * (D / 4);
#pragma unroll
    for (int j = 0; j < D / 16; ++j) {
      uint2 w = make_uint2(0u, 0u);
      if (hq < G) w = *reinterpret_cast<const uint2*>(qq + 4 * j);
      qbb[2 * j] = w.x;
      qbb[2 * j + 1] = w.y;
      qb[j][0] = pack_f16x2(bf16lo(w.x), bf16hi(w.x));
      qb[j][1] = pack_f16x2(bf16lo(w.y), bf16hi(w.y));
    }
  }
  // ---- live lists: lane -> contiguous blocks ----------------------------------
  const int8_t* th = st.blk_thought + (int64_t)u * P;
  const uint8_t* fl = st.blk_filled + (int64_t)u * P;
  const uint32_t* ev = st.blk_evict + (int64_t)u * P;
  const int per = (P + 31) / 32;
  const int b0 = lane * per, b1 = min(P, b0 + per);
  int c[4] = {0, 0, 0, 0};
#pragma unroll 4
  for (int b = b0; b < b1; ++b) {
    const int t = th[b];
    const int f = t >= 0 ? dm.band_fmt[t] : 0;
    const uint32_t live = t >= 0 ? ~ev[b] & (fl[b] >= 32 ? 0xffffffffu : ((1u << fl[b]) - 1u)) : 0u;
#pragma unroll
    for (int ff = 0; ff < 4; ++ff) c[ff] += ff == f ? __popc(live) : 0;
    binfo[b] = make_int2((int)live, f);
  }
  int w[4], cnt[4], off[4];
  {
    int run = 0;
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      int x = c[f];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      int tot = __shfl_sync(0xffffffffu, x, 31);
      if (f == TKV_FMT_RAW) tot += nbuf + 1;  // tail rows ride in the raw list
      off[f] = run;
      cnt[f] = tot;
      w[f] = run + x - c[f];
      run += (tot + 15) & ~15;  // padded to whole tiles
    }
    if (run > st.max_live + dm.g + 1 + 4 * 16) {  // host bookkeeping disagrees with the block table
      if (lane == 0) st.err[u] = TKV_E_INTEGRITY;
      return;
    }
  }
  for (int b = b0; b < b1; ++b) {
    const int2 bi = binfo[b];
    uint32_t live = (uint32_t)bi.x;
    int pos = 0;
#pragma unroll
    for (int f = 0; f < 4; ++f)
      if (bi.y == f) { pos = w[f]; w[f] += __popc(live); }
    while (live) {
      const int sl = __ffs(live) - 1;
      live &= live - 1;
      list[pos++] = (uint16_t)(b * bs + sl);
    }
  }
  {
    const int rawn = cnt[TKV_FMT_RAW] - (nbuf + 1);
    for (int t = lane; t <= nbuf; t += 32) list[off[TKV_FMT_RAW] + rawn + t] = (uint16_t)(NS + t);
  }
  __syncwarp();
  // padding entries: copies of each list's first entry (masked to -inf logits)
#pragma unroll
  for (int f = 0; f < 4; ++f) {
    const int n = cnt[f];
    if (lane < 16 && n > 0 && n + lane < ((n + 15) & ~15)) list[off[f] + n + lane] = list[off[f]];
  }
  __syncwarp();
  UnitPtrs up;
  up.kstride = dm.kstride;
  up.vchunks = dm.vchunks;
  up.NS = NS;
  up.k = st.slot_k + (int64_t)u * NS * dm.kstride;
  up.v = st.slot_v + (int64_t)u * NS * dm.kstride;
  up.vs = st.slot_vs + (int64_t)u * NS * dm.vchunks;
  up.win = st.slot_win + (int64_t)u * NS;
  up.ks = st.win_ks + (int64_t)u * dm.NW * D;
  up.kf = st.win_kf + (int64_t)u * dm.NW;
  up.vf = st.win_vf + (int64_t)u * dm.NW;
  {
    const int64_t row = (int64_t)dm.g * D * 2;
    up.bk = st.buf + ((int64_t)u * 4 + buf_half * 2 + 0) * row;
    up.bv = st.buf + ((int64_t)u * 4 + buf_half * 2 + 1) * row;
  }
  up.kc = reinterpret_cast<const uint8_t*>(kin) + (int64_t)li * D * 2;
  up.vc = reinterpret_cast<const uint8_t*>(vin) + (int64_t)li * D * 2;
  up.nbuf = nbuf;
  up.vsel = (gid * (D / 8)) / dm.g;
  Acc<D> A;
#pragma unroll
  for (int mt = 0; mt < D / 16; ++mt)
#pragma unroll
    for (int i = 0; i < 4; ++i) A.o[mt][i] = 0.f;
  A.m[0] = A.m[1] = -CUDART_INF_F;
  A.l[0] = A.l[1] = 0.f;
  const bool mp = dm.maxpool != 0;
  run_format4<D, TKV_FMT_NVFP4, PVN, KS>(up, list + off[TKV_FMT_NVFP4], cnt[TKV_FMT_NVFP4], qb, qbb, qscale, mp, gid, tig,
                                     ps, A);
  run_format4<D, TKV_FMT_TERNARY, PVN, KS>(up, list + off[TKV_FMT_TERNARY], cnt[TKV_FMT_TERNARY], qb, qbb, qscale, mp,
                                       gid, tig, ps, A);
  run_format4<D, TKV_FMT_FP8, PVN, KS>(up, list + off[TKV_FMT_FP8], cnt[TKV_FMT_FP8], qb, qbb, qscale, mp, gid, tig, ps,
                                   A);
  run_format4<D, kFmtTail, PVN, KS>(up, list + off[TKV_FMT_RAW], cnt[TKV_FMT_RAW], qb, qbb, qscale, mp, gid, tig, ps, A);
  // ---- epilogue: heads tig*2 + cc, channels gid*D/8 + 2mt (+1) ------------------
  // denominators: each lane summed its own tokens; reduce over the 8 token lanes
#pragma unroll
  for (int cc = 0; cc < 2; ++cc) {
    float l = A.l[cc];
    l += __shfl_xor_sync(0xffffffffu, l, 4);
    l += __shfl_xor_sync(0xffffffffu, l, 8);
    l += __shfl_xor_sync(0xffffffffu, l, 16);
    A.l[cc] = l;
  }
  if constexpr (PVN) {  // head h = hi column h + lo column 4 + h (lane tig + 2)
#pragma unroll
    for (int mt = 0; mt < D / 16; ++mt)
#pragma unroll
      for (int i = 0; i < 4; ++i) A.o[mt][i] += __shfl_xor_sync(0xffffffffu, A.o[mt][i], 2);
  }
#pragma unroll
  for (int cc = 0; cc < 2; ++cc) {
    const int h = tig * 2 + cc;
    if (h >= R || (PVN && tig >= 2)) continue;
    const float inv = 1.0f / A.l[cc];
    float* o = out + ((int64_t)li * R + h) * D + gid * (D / 8);
#pragma unroll
    for (int mt = 0; mt < D / 16; ++mt)
      *reinterpret_cast<float2*>(o + 2 * mt) = make_float2(A.o[mt][cc] * inv, A.o[mt][2 + cc] * inv);
  }
  if (put_slot >= 0) {  // buffer the incoming token (sim.cpp:796-808)
    const int64_t row = (int64_t)dm.g * D;
    uint16_t* bk = reinterpret_cast<uint16_t*>(st.buf) + ((int64_t)u * 4 + put_half * 2 + 0) * row + (int64_t)put_slot * D;
    uint16_t* bv = reinterpret_cast<uint16_t*>(st.buf) + ((int64_t)u * 4 + put_half * 2 + 1) * row + (int64_t)put_slot * D;
    const uint16_t* ks = reinterpret_cast<const uint16_t*>(kin) + (int64_t)li * D;
    const uint16_t* vs = reinterpret_cast<const uint16_t*>(vin) + (int64_t)li * D;
    for (int i = lane; i < D; i += 32) {
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

template <int D, int MINB>
cudaError_t launch_k1(const TkvState& st, const void* q, const void* k, const void* v, float* out, int buf_half,
                      int nbuf, int put_half, int put_slot, size_t smem, cudaStream_t s) {
  static bool cfg = false;
  if (!cfg) {
    cudaFuncSetAttribute(attend_mma_kernel<D, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cfg = true;
  }
  attend_mma_kernel<D, MINB><<<tkv_launch_units(st), kThreads, smem, s>>>(st, q, k, v, out, buf_half, nbuf, put_half, put_slot);
  return cudaGetLastError();
}

template <int D, int MINB, bool PVN, int KS>
cudaError_t launch_k1_warp(const TkvState& st, const void* q, const void* k, const void* v, float* out, int buf_half,
                           int nbuf, int put_half, int put_slot, cudaStream_t s) {
  const size_t smem = (size_t)kWarps * WarpSmem<D>::bytes(st.max_live, st.dm.g, st.dm.P);
  static bool cfg = false;
  if (!cfg) {
    cudaFuncSetAttribute(attend_warp_kernel<D, MINB, PVN, KS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cfg = true;
  }
  attend_warp_kernel<D, MINB, PVN, KS><<<(tkv_launch_units(st) + kWarps - 1) / kWarps, kThreads, smem, s>>>(
      st, q, k, v, out, buf_half, nbuf, put_half, put_slot);
  return cudaGetLastError();
}

cudaError_t tkv_launch_attend_mma(const TkvState& st, const void* q, const void* k, const void* v, float* out,
                                  int buf_half, int nbuf, int put_half, int put_slot, cudaStream_t s) {
  const int D = st.dm.D;
  // v3 (warp per unit, u16 slot lists) whenever slot ids fit in 16 bits and
  // the per-warp lists fit in shared memory; v2 (CTA per unit) otherwise.
  const bool v3 = st.dm.NS + st.dm.g + 1 + 4 * 16 < 65536 &&
                  (size_t)kWarps * (D == 128 ? WarpSmem<128>::bytes(st.max_live, st.dm.g, st.dm.P)
                                             : WarpSmem<64>::bytes(st.max_live, st.dm.g, st.dm.P)) <= 200 * 1024 &&
                  getenv("TKV_K1_V2") == nullptr;
  if (v3) {
    const bool pvn = st.dm.maxpool || st.dm.G <= 4;
    // 4-bit widest band with 16-channel value groups (BASELINE configs 2-4):
    // slot-row stride D / 2 as an immediate; any other layout: runtime stride.
    const bool imm = st.dm.kstride == D / 2 && st.dm.vchunks == D / 16 && getenv("TKV_K1_RUNTIME_STRIDE") == nullptr;
#define TKV_K1(DD, MB, PV)                                                                                    \
  (imm ? launch_k1_warp<DD, MB, PV, DD / 2>(st, q, k, v, out, buf_half, nbuf, put_half, put_slot, s)         \
       : launch_k1_warp<DD, MB, PV, 0>(st, q, k, v, out, buf_half, nbuf, put_half, put_slot, s))
    if (D == 128) return pvn ? TKV_K1(128, 3, true) : TKV_K1(128, 3, false);
    // d = 64 fits 128 registers without spills: 4 CTAs (16 warps) per SM.
    // Measured at config 3: 3 CTAs/SM 0.287 ms, 4: 0.249 ms, 5 (96 registers,
    // 48 B spilled): 0.308 ms (profiles/r02_c3_k1_minb*.json).
    return pvn ? TKV_K1(64, 4, true) : TKV_K1(64, 4, false);
#undef TKV_K1
  }
  const size_t smem = (size_t)kWarps * 8 * (2 + D) * 4 + (size_t)kWarps * 128 * 4 + (size_t)32 * (D / 8) * 4 +
                      (size_t)(st.dm.NS + st.dm.g + 1 + 4 * 16) * 8 + (size_t)st.dm.P * 8;
  if (D == 128) return launch_k1<128, 3>(st, q, k, v, out, buf_half, nbuf, put_half, put_slot, smem, s);
  return launch_k1<64, 3>(st, q, k, v, out, buf_half, nbuf, put_half, put_slot, smem, s);
}
