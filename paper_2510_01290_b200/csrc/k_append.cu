// K2: quantize-on-append.  One CTA per unit emits the unit's buffered window:
//   phase A  window quantization (quantize_window, proj/src/quant.cpp:486-580)
//            in fp64, bit-exact; keys grouped per channel across the window's
//            tokens, values per token in g-channel chunks, FP8 with one fp32
//            scale per side per window;
//   phase B  ordered slot claim and block-table bookkeeping
//            (BlockPager::append_tokens, proj/src/pager.cpp:114-219): soft-
//            evicted slots of same-thought blocks in physical order, then
//            unfilled tail slots, then the lowest free block ids; the OOM check
//            happens before any mutation (pager.cpp:147-159);
//   phase C  packed code / scale stores into the claimed slots (no compaction:
//            slots never move) and token -> slot index updates.
#include <cuda_runtime.h>

#include "tkv_codec.cuh"
#include "tkv_kernels.h"
#include "tkv_state.h"

namespace {

__device__ __forceinline__ double load_in(const uint8_t* p, int dtype, int64_t idx) {
  if (dtype == TKV_IN_BF16) {
    const uint16_t b = reinterpret_cast<const uint16_t*>(p)[idx];
    return (double)__uint_as_float(((uint32_t)b) << 16);
  }
  if (dtype == TKV_IN_F32) return (double)reinterpret_cast<const float*>(p)[idx];
  return reinterpret_cast<const double*>(p)[idx];
}

__device__ __forceinline__ double block_max(double v, double* red) {
  // max is order-independent, so a tree reduction is exact.
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double r = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) r = fmax(r, red[i]);
  return r;
}

// Division-free encoders for inputs with <= 24 significant bits (bf16/f32).
// The reference rounds q = x / s in double and then picks the nearest grid
// point (NVFP4, ties to the even index, quant.cpp:114-130) or clamps
// rint(q) (ternary, quant.cpp:141-158).  Every decision boundary is a grid
// midpoint M, and s * M (E4M3 scale x midpoint, <= 7 significant bits) is
// exact in fp64.  If x / s != M exactly, x - s*M is a multiple of the
// coarser of the two quanta, >= 2^-26 relative to M, so RN(x / s) lies
// strictly on the same side of M as x / s: comparing |x| with s*M takes the
// same branch, and |x| == s*M is exactly the reference's tie.  fp64 inputs
// keep the division.
__device__ __forceinline__ uint8_t nvfp4_encode_cmp(double x, double s) {
  const double a = fabs(x);
  // midpoints between grid indices k, k+1 of {0, .5, 1, 1.5, 2, 3, 4, 6}; a tie
  // goes to the even index: counted when k + 1 is even
  int i = 0;
  i += a > s * 0.25;
  i += a >= s * 0.75;
  i += a > s * 1.25;
  i += a >= s * 1.75;
  i += a > s * 2.5;
  i += a >= s * 3.5;
  i += a > s * 5.0;
  if (i == 0) return 0;
  return (signbit(x) ? 0x8 : 0x0) | (uint8_t)i;
}
__device__ __forceinline__ uint8_t ternary_encode_cmp(double x, double delta) {
  // clamp(rint(x / delta), -1, 1): |x / delta| <= 0.5 rounds to (signed) 0
  if (!(fabs(x) > delta * 0.5)) return tkv_ternary_bits(0);
  return tkv_ternary_bits(x > 0.0 ? 1 : -1);
}

// BlockPager::append_tokens (pager.cpp:132-164), the claim: n slots for
// thought `band`, in the reference's order -- (1) soft-evicted slots of
// same-thought blocks in physical order, (2) unfilled tail slots of
// same-thought blocks, (3) fresh blocks, lowest free id first
// (allocate_block, pager.cpp:28-47).  The capacity check comes before any
// mutation: TKV_E_OOM with nothing changed.  th_r/fl_r/ev_r are the columns
// the scan reads (a staged copy or the table itself); fresh-block
// allocation writes th/fl/ev/ns and *nfree.  claim[i] = block * bs + slot.
// Shared by K2 (flush_kernel) and the drop-in pager (pager_place_kernel).
__device__ int tkv_claim_slots(const int8_t* th_r, const uint8_t* fl_r, const uint32_t* ev_r, int8_t* th,
                               uint8_t* fl, uint32_t* ev, uint8_t* ns, int32_t* nfree, int P, int bs, int band,
                               int n, int32_t* claim, int8_t* reuse) {
  int claims = 0;
  for (int b = 0; b < P && claims < n; ++b) {
    if (th_r[b] != band) continue;
    uint32_t m = ev_r[b] & (fl_r[b] >= 32 ? 0xffffffffu : ((1u << fl_r[b]) - 1u));
    while (m && claims < n) {
      const int s = __ffs(m) - 1;
      m &= m - 1;
      claim[claims] = b * bs + s;
      reuse[claims] = 1;
      ++claims;
    }
  }
  for (int b = 0; b < P && claims < n; ++b) {
    if (th_r[b] != band) continue;
    for (int s = fl_r[b]; s < bs && claims < n; ++s) {
      claim[claims] = b * bs + s;
      reuse[claims] = 0;
      ++claims;
    }
  }
  const int remaining = n - claims;
  const int fresh = (remaining + bs - 1) / bs;
  if (fresh > *nfree) return TKV_E_OOM;
  for (int b = 0, got = 0; b < P && got < fresh; ++b) {
    if (th_r[b] != -1) continue;
    th[b] = (int8_t)band;
    fl[b] = 0;
    ev[b] = 0;
    ns[b] = 0;
    ++got;
    for (int s = 0; s < bs && claims < n; ++s) {
      claim[claims] = b * bs + s;
      reuse[claims] = 0;
      ++claims;
    }
  }
  *nfree -= fresh;
  return 0;
}

// BlockPager::append_tokens (pager.cpp:166-216), the per-token bookkeeping of
// the claimed slots in placement order: clear the eviction bit and drop the
// slot from older segment masks on reuse (else filled++), append the
// segment's start index and mask when it is new to the block (the first
// segment is implicit), then prune later masks that reuse emptied.
__device__ void tkv_record_placements(uint8_t* fl, uint32_t* ev, uint8_t* ns, int32_t* sstart, uint32_t* smask,
                                      int bs, int32_t seg_start, int n, const int32_t* claim, const int8_t* reuse) {
  for (int i = 0; i < n; ++i) {
    const int b = claim[i] / bs, s = claim[i] % bs;
    const uint32_t bit = 1u << s;
    int32_t* starts = sstart + (int64_t)b * TKV_STARTS_PER_BLOCK(bs);
    uint32_t* masks = smask + (int64_t)b * TKV_MASKS_PER_BLOCK(bs);
    if (reuse[i]) {
      ev[b] &= ~bit;
      for (int k = 0; k + 1 < ns[b]; ++k) masks[k] &= ~bit;
    } else {
      fl[b] += 1;
    }
    int found = -1;
    for (int k = 0; k < ns[b]; ++k)
      if (starts[k] == seg_start) { found = k; break; }
    if (found < 0) {
      starts[ns[b]] = seg_start;
      if (ns[b] > 0) masks[ns[b] - 1] = bit;
      ns[b] += 1;
    } else if (found > 0) {
      masks[found - 1] |= bit;
    }
    for (int k = ns[b] - 2; k >= 0; --k) {
      if (masks[k] != 0) continue;
      for (int j = k; j + 1 < ns[b] - 1; ++j) masks[j] = masks[j + 1];
      for (int j = k + 1; j + 1 < ns[b]; ++j) starts[j] = starts[j + 1];
      ns[b] -= 1;
    }
  }
}

// Claimed blocks staged in shared memory for the placement bookkeeping (a
// 16-token window touches at most 16 blocks; more falls back to global memory).
constexpr int kStageBlocks = 24;

struct FlushSmem {
  int32_t claim[64];
  int8_t reuse[64];
  int32_t nb;                                   // staged blocks
  int32_t sb[kStageBlocks];                     // their ids
  uint8_t fl_t[kStageBlocks], ns_t[kStageBlocks];
  uint32_t ev_t[kStageBlocks];
  int32_t st_t[kStageBlocks][TKV_STARTS_PER_BLOCK(32)];
  uint32_t mk_t[kStageBlocks][TKV_MASKS_PER_BLOCK(32)];
  int32_t win;
  int32_t abort_code;
  int32_t bad;
  float kf, vf;
  double red[32];
};

__global__ void __launch_bounds__(128) flush_kernel(TkvState st, int half, int n, int pos0,
                                                    const TkvFlushCtl* __restrict__ ctl,
                                                    int units_per_group) {
  tkv_flush_scalars(st, half, pos0);
  const TkvDims& dm = st.dm;
  const int u = blockIdx.x;
  if (u >= dm.U) return;
  const int D = dm.D, g = dm.g, bs = dm.bs, P = dm.P;
  const TkvFlushCtl c = ctl[u / units_per_group];
  const int fmt = dm.band_fmt[c.band];
  const int kbytes = dm.band_bytes[c.band];
  extern __shared__ __align__(16) uint8_t dyn[];
  __shared__ FlushSmem sm;
  uint8_t* kc = dyn;                         // [n][D] key codes
  uint8_t* vc = kc + 64 * D;                 // [n][D] value codes
  uint8_t* ksc = vc + 64 * D;                // [D] key scale codes
  uint8_t* vsc = ksc + D;                    // [n][vchunks] value scale codes
  // block-table columns staged for the serial claim (thought, filled, evict mask)
  uint32_t* ev_s = reinterpret_cast<uint32_t*>(dyn + (((int64_t)64 * D * 2 + D + 64 * dm.vchunks + 15) / 16 * 16));
  int8_t* th_s = reinterpret_cast<int8_t*>(ev_s + P);
  uint8_t* fl_s = reinterpret_cast<uint8_t*>(th_s + P);
  const int64_t buf_elems = (int64_t)g * D;
  const uint8_t* bufk = st.buf + ((int64_t)u * 4 + half * 2 + 0) * buf_elems * dm.in_bytes;
  const uint8_t* bufv = st.buf + ((int64_t)u * 4 + half * 2 + 1) * buf_elems * dm.in_bytes;
  if (threadIdx.x == 0) { sm.abort_code = 0; sm.bad = 0; }
  __syncthreads();

  // ---- phase A: quantization -------------------------------------------
  if (fmt != TKV_FMT_RAW) {
    bool bad = false;
    for (int i = threadIdx.x; i < n * D; i += blockDim.x) {
      if (!isfinite(load_in(bufk, dm.in_dtype, i)) || !isfinite(load_in(bufv, dm.in_dtype, i))) bad = true;
    }
    if (bad) atomicExch(&sm.bad, 1);
    if (fmt == TKV_FMT_FP8) {
      double ak = 0.0, av = 0.0;
      for (int i = threadIdx.x; i < n * D; i += blockDim.x) {
        ak = fmax(ak, fabs(load_in(bufk, dm.in_dtype, i)));
        av = fmax(av, fabs(load_in(bufv, dm.in_dtype, i)));
      }
      ak = block_max(ak, sm.red);
      av = block_max(av, sm.red);
      const float kf = __double2float_rn(ak / 448.0);  // fp8_tensor_scale (quant.cpp:176-178)
      const float vf = __double2float_rn(av / 448.0);
      for (int i = threadIdx.x; i < n * D; i += blockDim.x) {
        bool b2 = false;
        kc[i] = kf > 0.0f ? tkv_e4m3_encode(load_in(bufk, dm.in_dtype, i) / (double)kf, &b2) : 0;
        vc[i] = vf > 0.0f ? tkv_e4m3_encode(load_in(bufv, dm.in_dtype, i) / (double)vf, &b2) : 0;
        if (b2) atomicExch(&sm.bad, 1);
      }
      if (threadIdx.x == 0) { sm.kf = kf; sm.vf = vf; }
    } else {
      bool b2 = false;
      const bool narrow = dm.in_dtype != TKV_IN_F64;  // <= 24 significant bits: division-free encoders
      // keys: one group per channel over the window's tokens (zero padding
      // never changes the absmax).
      for (int ch = threadIdx.x; ch < D; ch += blockDim.x) {
        double am = 0.0;
        for (int t = 0; t < n; ++t) am = fmax(am, fabs(load_in(bufk, dm.in_dtype, (int64_t)t * D + ch)));
        uint8_t sc;
        if (fmt == TKV_FMT_TERNARY) {
          sc = tkv_e4m3_encode(am, &b2);                       // quant.cpp:141-158
          const double delta = tkv_e4m3_decode(sc);
          for (int t = 0; t < n; ++t) {
            uint8_t code = 0;
            if (delta > 0.0) {
              const double x = load_in(bufk, dm.in_dtype, (int64_t)t * D + ch);
              if (narrow) {
                code = ternary_encode_cmp(x, delta);
              } else {
                const double r = rint(x / delta);
                code = tkv_ternary_bits((int)fmin(fmax(r, -1.0), 1.0));
              }
            }
            kc[t * D + ch] = code;
          }
        } else {
          sc = tkv_e4m3_encode(am / 6.0, &b2);                 // quant.cpp:160-174
          const double s = tkv_e4m3_decode(sc);
          for (int t = 0; t < n; ++t) {
            const double x = load_in(bufk, dm.in_dtype, (int64_t)t * D + ch);
            kc[t * D + ch] = s > 0.0 ? (narrow ? nvfp4_encode_cmp(x, s) : tkv_nvfp4_encode(x / s)) : 0;
          }
        }
        ksc[ch] = sc;
      }
      // values: per token, chunks of g consecutive channels.
      const int vch = dm.vchunks;
      for (int it = threadIdx.x; it < n * vch; it += blockDim.x) {
        const int t = it / vch, j = it % vch;
        const int base = j * g, len = min(g, D - base);
        double am = 0.0;
        for (int q = 0; q < len; ++q) am = fmax(am, fabs(load_in(bufv, dm.in_dtype, (int64_t)t * D + base + q)));
        uint8_t sc;
        if (fmt == TKV_FMT_TERNARY) {
          sc = tkv_e4m3_encode(am, &b2);
          const double delta = tkv_e4m3_decode(sc);
          for (int q = 0; q < len; ++q) {
            uint8_t code = 0;
            if (delta > 0.0) {
              const double x = load_in(bufv, dm.in_dtype, (int64_t)t * D + base + q);
              if (narrow) {
                code = ternary_encode_cmp(x, delta);
              } else {
                const double r = rint(x / delta);
                code = tkv_ternary_bits((int)fmin(fmax(r, -1.0), 1.0));
              }
            }
            vc[t * D + base + q] = code;
          }
        } else {
          sc = tkv_e4m3_encode(am / 6.0, &b2);
          const double s = tkv_e4m3_decode(sc);
          for (int q = 0; q < len; ++q) {
            const double x = load_in(bufv, dm.in_dtype, (int64_t)t * D + base + q);
            vc[t * D + base + q] = s > 0.0 ? (narrow ? nvfp4_encode_cmp(x, s) : tkv_nvfp4_encode(x / s)) : 0;
          }
        }
        vsc[t * vch + j] = sc;
      }
      if (b2) atomicExch(&sm.bad, 1);
    }
  }
  for (int b = threadIdx.x; b < P; b += blockDim.x) {
    th_s[b] = st.blk_thought[(int64_t)u * P + b];
    fl_s[b] = st.blk_filled[(int64_t)u * P + b];
    ev_s[b] = st.blk_evict[(int64_t)u * P + b];
  }
  __syncthreads();

  // ---- phase B: ordered claim + block-table bookkeeping (one thread) -----
  if (threadIdx.x == 0) {
    int* err = st.err + u;
    if (sm.bad) {
      sm.abort_code = TKV_E_STRUCTURAL;
    } else if (*err != 0) {
      sm.abort_code = *err;  // sticky: a failed unit stops mutating
    }
    int8_t* th = st.blk_thought + (int64_t)u * P;
    uint8_t* fl = st.blk_filled + (int64_t)u * P;
    uint32_t* ev = st.blk_evict + (int64_t)u * P;
    uint8_t* ns = st.blk_nstart + (int64_t)u * P;
    int32_t* sstart = st.blk_start + (int64_t)u * P * TKV_STARTS_PER_BLOCK(bs);
    uint32_t* smask = st.blk_segmask + (int64_t)u * P * TKV_MASKS_PER_BLOCK(bs);
    if (sm.abort_code == 0)
      sm.abort_code = tkv_claim_slots(th_s, fl_s, ev_s, th, fl, ev, ns, st.unit_nfree + u, P, bs, c.band, n,
                                      sm.claim, sm.reuse);
    if (sm.abort_code != 0) {
      *err = sm.abort_code;
    } else {
      int w = -1;
      if (fmt != TKV_FMT_RAW) {
        const int nf = st.win_nfree[u];
        if (nf <= 0) {
          sm.abort_code = TKV_E_INTEGRITY;
          *err = TKV_E_INTEGRITY;
        } else {
          w = st.win_free[(int64_t)u * dm.NW + nf - 1];
          st.win_nfree[u] = nf - 1;
        }
      }
      sm.win = w;
      // distinct claimed blocks, in first-claim order
      int nb = 0;
      for (int i = 0; i < n; ++i) {
        const int b = sm.claim[i] / bs;
        int k = 0;
        while (k < nb && sm.sb[k] != b) ++k;
        if (k == nb) {
          if (nb == kStageBlocks) { nb = -1; break; }
          sm.sb[nb++] = b;
        }
      }
      sm.nb = nb;
      if (nb < 0) tkv_record_placements(fl, ev, ns, sstart, smask, bs, c.seg_start, n, sm.claim, sm.reuse);
    }
  }
  __syncthreads();
  if (sm.abort_code != 0) return;
  // Placement bookkeeping (tkv_record_placements, pager.cpp:166-216) on
  // shared-memory copies of the claimed blocks: the warp stages them, one
  // thread applies the claims in order, the warp writes them back -- the
  // serial part no longer waits on dependent global loads.
  if (sm.nb >= 0) {
    const int nb = sm.nb, SP = TKV_STARTS_PER_BLOCK(bs), MP = TKV_MASKS_PER_BLOCK(bs);
    uint8_t* fl = st.blk_filled + (int64_t)u * P;
    uint32_t* ev = st.blk_evict + (int64_t)u * P;
    uint8_t* ns = st.blk_nstart + (int64_t)u * P;
    int32_t* sstart = st.blk_start + (int64_t)u * P * SP;
    uint32_t* smask = st.blk_segmask + (int64_t)u * P * MP;
    for (int k = threadIdx.x; k < nb; k += blockDim.x) {
      const int b = sm.sb[k];
      sm.fl_t[k] = fl[b];
      sm.ev_t[k] = ev[b];
      sm.ns_t[k] = ns[b];
    }
    for (int t = threadIdx.x; t < nb * SP; t += blockDim.x) sm.st_t[t / SP][t % SP] = sstart[(int64_t)sm.sb[t / SP] * SP + t % SP];
    for (int t = threadIdx.x; t < nb * MP; t += blockDim.x) sm.mk_t[t / MP][t % MP] = smask[(int64_t)sm.sb[t / MP] * MP + t % MP];
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int i = 0; i < n; ++i) {
        const int b = sm.claim[i] / bs, sl = sm.claim[i] % bs;
        int k = 0;
        while (sm.sb[k] != b) ++k;
        const uint32_t bit = 1u << sl;
        int32_t* starts = sm.st_t[k];
        uint32_t* masks = sm.mk_t[k];
        int nsb = sm.ns_t[k];
        if (sm.reuse[i]) {
          sm.ev_t[k] &= ~bit;
          for (int q = 0; q + 1 < nsb; ++q) masks[q] &= ~bit;
        } else {
          sm.fl_t[k] += 1;
        }
        int found = -1;
        for (int q = 0; q < nsb; ++q)
          if (starts[q] == c.seg_start) { found = q; break; }
        if (found < 0) {
          starts[nsb] = c.seg_start;
          if (nsb > 0) masks[nsb - 1] = bit;
          nsb += 1;
        } else if (found > 0) {
          masks[found - 1] |= bit;
        }
        for (int q = nsb - 2; q >= 0; --q) {
          if (masks[q] != 0) continue;
          for (int j = q; j + 1 < nsb - 1; ++j) masks[j] = masks[j + 1];
          for (int j = q + 1; j + 1 < nsb; ++j) starts[j] = starts[j + 1];
          nsb -= 1;
        }
        sm.ns_t[k] = (uint8_t)nsb;
      }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < nb; k += blockDim.x) {
      const int b = sm.sb[k];
      fl[b] = sm.fl_t[k];
      ev[b] = sm.ev_t[k];
      ns[b] = sm.ns_t[k];
    }
    for (int t = threadIdx.x; t < nb * SP; t += blockDim.x) sstart[(int64_t)sm.sb[t / SP] * SP + t % SP] = sm.st_t[t / SP][t % SP];
    for (int t = threadIdx.x; t < nb * MP; t += blockDim.x) smask[(int64_t)sm.sb[t / MP] * MP + t % MP] = sm.mk_t[t / MP][t % MP];
  }

  // ---- phase C: slot payload stores ----------------------------------------
  const int w = sm.win;
  const int vch = dm.vchunks;
  const int ks = dm.kstride;
  for (int i = 0; i < n; ++i) {
    const int64_t slot = (int64_t)u * dm.NS + sm.claim[i];
    uint8_t* kd = st.slot_k + slot * ks;
    uint8_t* vd = st.slot_v + slot * ks;
    if (fmt == TKV_FMT_RAW) {
      const int64_t bytes = (int64_t)D * dm.in_bytes;
      for (int64_t q = threadIdx.x; q < bytes; q += blockDim.x) {
        kd[q] = bufk[(int64_t)i * bytes + q];
        vd[q] = bufv[(int64_t)i * bytes + q];
      }
    } else {
      for (int q = threadIdx.x; q < kbytes; q += blockDim.x) {
        uint32_t kb = 0, vb = 0;
        if (fmt == TKV_FMT_TERNARY) {
          for (int e = 0; e < 4; ++e) {
            const int ch = q * 4 + e;
            if (ch < D) { kb |= (uint32_t)kc[i * D + ch] << (2 * e); vb |= (uint32_t)vc[i * D + ch] << (2 * e); }
          }
        } else if (fmt == TKV_FMT_NVFP4) {
          for (int e = 0; e < 2; ++e) {
            const int ch = q * 2 + e;
            if (ch < D) { kb |= (uint32_t)kc[i * D + ch] << (4 * e); vb |= (uint32_t)vc[i * D + ch] << (4 * e); }
          }
        } else {
          kb = kc[i * D + q];
          vb = vc[i * D + q];
        }
        kd[q] = (uint8_t)kb;
        vd[q] = (uint8_t)vb;
      }
      if (fmt != TKV_FMT_FP8)
        for (int j = threadIdx.x; j < vch; j += blockDim.x) st.slot_vs[slot * vch + j] = vsc[i * vch + j];
    }
    if (threadIdx.x == 0) {
      st.slot_win[slot] = w;
      st.slot_id[slot] = pos0 + i;
    }
  }
  if (w >= 0) {
    const int64_t wi = (int64_t)u * dm.NW + w;
    if (fmt == TKV_FMT_FP8) {
      if (threadIdx.x == 0) { st.win_kf[wi] = sm.kf; st.win_vf[wi] = sm.vf; }
    } else {
      for (int ch = threadIdx.x; ch < D; ch += blockDim.x) st.win_ks[wi * D + ch] = ksc[ch];
    }
    if (threadIdx.x == 0) st.win_refs[wi] = n;
  }
}


// ---- drop-in pager: one BlockPager's table per launch --------
// BlockPager::append_tokens' placement over a caller-supplied table (the
// drop-in adapter's host mirror, uploaded for the call): the same claim and
// bookkeeping K2 runs on the paged state.
__global__ void pager_place_kernel(int P, int bs, int8_t* th, uint8_t* fl, uint32_t* ev, uint8_t* ns, int32_t* sstart,
                                   uint32_t* smask, int32_t* nfree, int band, int32_t seg_start, int n, int32_t* claim,
                                   int8_t* reuse, int32_t* rc) {
  if (threadIdx.x != 0) return;
  const int r = tkv_claim_slots(th, fl, ev, th, fl, ev, ns, nfree, P, bs, band, n, claim, reuse);
  *rc = r;
  if (r == 0) tkv_record_placements(fl, ev, ns, sstart, smask, bs, seg_start, n, claim, reuse);
}

// BlockPager::apply_eviction_plan (pager.cpp:238-259) on the table: mask the
// listed slots, then free every touched block whose live count reached zero,
// in ascending block id (free_block :228-236).  freed[] lists them.
__global__ void pager_evict_kernel(int P, int bs, int8_t* th, uint8_t* fl, uint32_t* ev, uint8_t* ns, int n,
                                   const int32_t* slots, int32_t* freed, int32_t* nfreed) {
  extern __shared__ uint8_t touched[];
  for (int b = threadIdx.x; b < P; b += blockDim.x) touched[b] = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 0; i < n; ++i) {
      const int b = slots[i] / bs, s = slots[i] % bs;
      ev[b] |= 1u << s;
      touched[b] = 1;
    }
    int k = 0;
    for (int b = 0; b < P; ++b) {
      if (!touched[b]) continue;
      const uint32_t filled = fl[b] >= 32 ? 0xffffffffu : ((1u << fl[b]) - 1u);
      if ((~ev[b] & filled) != 0) continue;  // live_in_block > 0
      th[b] = -1;
      fl[b] = 0;
      ev[b] = 0;
      ns[b] = 0;
      freed[k++] = b;
    }
    *nfreed = k;
  }
}

}  // namespace

cudaError_t tkv_launch_pager_place(int P, int bs, int8_t* th, uint8_t* fl, uint32_t* ev, uint8_t* ns, int32_t* sstart,
                                   uint32_t* smask, int32_t* nfree, int band, int32_t seg_start, int n, int32_t* claim,
                                   int8_t* reuse, int32_t* rc, cudaStream_t stream) {
  pager_place_kernel<<<1, 32, 0, stream>>>(P, bs, th, fl, ev, ns, sstart, smask, nfree, band, seg_start, n, claim,
                                           reuse, rc);
  return cudaGetLastError();
}

cudaError_t tkv_launch_pager_evict(int P, int bs, int8_t* th, uint8_t* fl, uint32_t* ev, uint8_t* ns, int n,
                                   const int32_t* slots, int32_t* freed, int32_t* nfreed, cudaStream_t stream) {
  pager_evict_kernel<<<1, 128, P, stream>>>(P, bs, th, fl, ev, ns, n, slots, freed, nfreed);
  return cudaGetLastError();
}

cudaError_t tkv_launch_flush(const TkvState& st, int half, int n, int pos0, const TkvFlushCtl* ctl,
                             int units_per_group, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const size_t smem = ((size_t)64 * st.dm.D * 2 + st.dm.D + (size_t)64 * st.dm.vchunks + 15) / 16 * 16 +
                      (size_t)st.dm.P * 6;  // + staged block-table columns
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(flush_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  flush_kernel<<<st.dm.U, 128, smem, stream>>>(st, half, n, pos0, ctl, units_per_group);
  return cudaGetLastError();
}
