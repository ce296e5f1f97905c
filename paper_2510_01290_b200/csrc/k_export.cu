// Compressed-cache export in the reference wire layout.
//
// Every live pager token of a unit is written as part of a *record*: a
// maximal run of live tokens, in ascending token id, that share one key-scale
// window (one emission, flush_layer sim.cpp:565-650) -- or, for 16-bit
// passthrough, one thought band.  Quantised payloads are written as
// QuantizedGroups serialised exactly as serialize_group (proj/src/
// quant.cpp:274-324) writes them: format tag, g (u16 LE), scale (E4M3 byte,
// or f32 LE for FP8), then 2/4/8-bit codes packed little-endian.
//
//   unit    := u32 nrecords | u32 nlive | u16 head_dim | u16 value_group | record*
//   record  := u8 kind (0 ternary, 1 nvfp4, 2 fp8, 3 raw) | u8 band | u16 n |
//              i64 id[n] | body
//   body    := kind 0/1: d key groups   (channel c: g = n, scale = the window's
//                        channel-c key scale, codes = the n tokens' channel-c codes)
//                        then per token ceil(d/vg) value groups (chunk j: channels
//                        [j*vg, min(d, (j+1)*vg)), scale = the token's chunk scale)
//              kind 2:   one key group and one value group (g = n*d, token-major
//                        codes, f32 window scale)
//              kind 3:   per token d f64 key values then d f64 value values
//
// The token order and the grouping are the reference's own: group ids are
// allocated in flush order (sim.cpp:589-628), so ascending key_group_base is
// ascending token id.  The oracle (oracle_driver.cpp orc_export) builds the
// same bytes from BlockPager::read_active / group_table through the compiled
// thinkv::serialize_group.
//
// Two launches: pass 0 sizes every unit, the host scans the sizes into
// offsets, pass 1 writes.  One warp per unit; live tokens are compacted in id
// order: the block table's live slots, sorted by token id in shared memory.
#include <cuda_runtime.h>

#include "tkv_codec.cuh"
#include "tkv_kernels.h"
#include "tkv_state.h"

namespace {

constexpr int kWarps = 4;

__device__ __forceinline__ int packed_bytes(int fmt, int n) {
  return fmt == TKV_FMT_TERNARY ? (n + 3) / 4 : (fmt == TKV_FMT_NVFP4 ? (n + 1) / 2 : n);
}

__device__ __forceinline__ int slot_kind(const TkvState& st, int u, int slot, int* band) {
  const int b = st.blk_thought[(int64_t)u * st.dm.P + slot / st.dm.bs];
  *band = b;
  return st.dm.band_fmt[b];
}

__device__ __forceinline__ int64_t record_bytes(const TkvDims& dm, int kind, int n) {
  int64_t b = 4 + 8 * (int64_t)n;
  if (kind == TKV_FMT_RAW) return b + (int64_t)n * 2 * dm.D * 8;
  if (kind == TKV_FMT_FP8) return b + 2 * (7 + (int64_t)n * dm.D);
  b += (int64_t)dm.D * (4 + packed_bytes(kind, n));
  int64_t per_tok = 0;
  for (int j = 0; j < dm.vchunks; ++j) per_tok += 4 + packed_bytes(kind, min(dm.g, dm.D - j * dm.g));
  return b + (int64_t)n * per_tok;
}

__device__ __forceinline__ void put16(uint8_t* p, uint32_t v) {
  p[0] = (uint8_t)v;
  p[1] = (uint8_t)(v >> 8);
}
__device__ __forceinline__ void put32(uint8_t* p, uint32_t v) {
  for (int i = 0; i < 4; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
__device__ __forceinline__ void put64(uint8_t* p, uint64_t v) {
  for (int i = 0; i < 8; ++i) p[i] = (uint8_t)(v >> (8 * i));
}

// Raw passthrough element (input dtype) widened exactly to f64.
__device__ __forceinline__ double raw_elem(const TkvDims& dm, const uint8_t* row, int c) {
  if (dm.in_dtype == TKV_IN_BF16) return (double)__uint_as_float(((uint32_t) reinterpret_cast<const uint16_t*>(row)[c]) << 16);
  if (dm.in_dtype == TKV_IN_F32) return (double)reinterpret_cast<const float*>(row)[c];
  return reinterpret_cast<const double*>(row)[c];
}

// Serialised QuantizedGroup of `n` codes taken from code(i): header then
// packed codes (quant.cpp:274-324).  Written by one thread.
template <typename F>
__device__ uint8_t* put_group(uint8_t* p, int fmt, int n, uint32_t scale_code, float scale_f32, F code) {
  p[0] = (uint8_t)fmt;
  put16(p + 1, (uint32_t)n);
  p += 3;
  if (fmt == TKV_FMT_FP8) {
    put32(p, __float_as_uint(scale_f32));
    p += 4;
  } else {
    *p++ = (uint8_t)scale_code;
  }
  if (fmt == TKV_FMT_TERNARY) {
    for (int i = 0; i < n; i += 4) {
      uint32_t b = 0;
      for (int e = 0; e < 4 && i + e < n; ++e) b |= (code(i + e) & 3u) << (2 * e);
      *p++ = (uint8_t)b;
    }
  } else if (fmt == TKV_FMT_NVFP4) {
    for (int i = 0; i < n; i += 2) {
      uint32_t b = code(i) & 15u;
      if (i + 1 < n) b |= (code(i + 1) & 15u) << 4;
      *p++ = (uint8_t)b;
    }
  } else {
    for (int i = 0; i < n; ++i) *p++ = (uint8_t)code(i);
  }
  return p;
}

__global__ void __launch_bounds__(32 * kWarps) export_kernel(TkvState st, int unit0, int nunits, int npos, int pass,
                                                             int64_t* __restrict__ sizes,
                                                             const int64_t* __restrict__ offsets,
                                                             uint8_t* __restrict__ dst) {
  const TkvDims& dm = st.dm;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ui = blockIdx.x * (blockDim.x >> 5) + warp;
  if (ui >= nunits) return;
  const int u = unit0 + ui;
  extern __shared__ int32_t sh[];
  // per warp: slot[NS] then record starts[NS + 1]
  int32_t* lslot = sh + (int64_t)warp * (2 * dm.NS + 2);
  int32_t* rstart = lslot + dm.NS;
  const unsigned below = (1u << lane) - 1u;
  // 1. live tokens in ascending id: the live slots of the block table
  //    (BlockPager::read_active, pager.cpp:261-271) as (id, slot) keys, then a
  //    bitonic sort by id in place (implicit +inf padding to a power of two:
  //    every compare-exchange is ascending, so partners beyond n are no-ops).
  uint64_t* key = reinterpret_cast<uint64_t*>(lslot);  // NS + 1 keys fit in the warp's 2 NS + 2 words
  int n = 0;
  {
    const int8_t* th = st.blk_thought + (int64_t)u * dm.P;
    const uint8_t* fl = st.blk_filled + (int64_t)u * dm.P;
    const uint32_t* ev = st.blk_evict + (int64_t)u * dm.P;
    const int32_t* sid = st.slot_id + (int64_t)u * dm.NS;
    for (int b = 0; b < dm.NS; b += 32) {
      const int s = b + lane;
      bool live = false;
      if (s < dm.NS) {
        const int blk = s / dm.bs, sl = s % dm.bs;
        live = th[blk] >= 0 && sl < fl[blk] && !((ev[blk] >> sl) & 1u);
      }
      const unsigned bal = __ballot_sync(0xffffffffu, live);
      if (live) key[n + __popc(bal & below)] = ((uint64_t)(uint32_t)sid[s] << 32) | (uint32_t)s;
      n += __popc(bal);
    }
  }
  __syncwarp();
  int p2 = 1;
  while (p2 < n) p2 <<= 1;
  for (int k = 2; k <= p2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = lane; t < p2 / 2; t += 32) {
        // pair t of this stage: i < partner, both in one block of size 2j
        const int i = (t / j) * 2 * j + (t % j);
        const int partner = j == (k >> 1) ? (i | (2 * j - 1)) - (i & (2 * j - 1)) : i + j;  // flip, then half-cleaners
        if (partner < n) {
          const uint64_t a = key[i], c = key[partner];
          if (a > c) { key[i] = c; key[partner] = a; }
        }
      }
      __syncwarp();
    }
  }
  // keys -> slots in place: chunk c's slots overwrite keys of chunks <= c / 2, already read
  for (int b = 0; b < n; b += 32) {
    const int i = b + lane;
    const int s = i < n ? (int)(uint32_t)key[i] : 0;
    __syncwarp();
    if (i < n) lslot[i] = s;
    __syncwarp();
  }
  // 2. record starts: kind/band change, or (quantised) a different window
  int nrec = 0;
  for (int b = 0; b < n; b += 32) {
    const int i = b + lane;
    bool start = false;
    if (i < n) {
      int band, pband = -1;
      const int s = lslot[i];
      const int kind = slot_kind(st, u, s, &band);
      if (i == 0) {
        start = true;
      } else {
        const int ps = lslot[i - 1];
        const int pkind = slot_kind(st, u, ps, &pband);
        start = kind != pkind || band != pband ||
                (kind != TKV_FMT_RAW && st.slot_win[(int64_t)u * dm.NS + s] != st.slot_win[(int64_t)u * dm.NS + ps]);
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, start);
    if (start) rstart[nrec + __popc(bal & below)] = i;
    nrec += __popc(bal);
  }
  if (lane == 0) rstart[nrec] = n;
  __syncwarp();
  // 3. size (u16 n per record: runs longer than 65535 tokens cannot occur --
  //    a window holds <= group_size tokens and raw runs are bounded by the pool)
  if (pass == 0) {
    int64_t bytes = 0;
    for (int r = lane; r < nrec; r += 32) {
      int band;
      const int kind = slot_kind(st, u, lslot[rstart[r]], &band);
      bytes += record_bytes(dm, kind, rstart[r + 1] - rstart[r]);
    }
    for (int o = 16; o > 0; o >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
    if (lane == 0) sizes[ui] = 12 + bytes;
    return;
  }
  uint8_t* out = dst + offsets[ui];
  if (lane == 0) {
    put32(out, (uint32_t)nrec);
    put32(out + 4, (uint32_t)n);
    put16(out + 8, (uint32_t)dm.D);
    put16(out + 10, (uint32_t)dm.g);
  }
  int64_t off = 12;
  const uint8_t* kbase = st.slot_k + (int64_t)u * dm.NS * dm.kstride;
  const uint8_t* vbase = st.slot_v + (int64_t)u * dm.NS * dm.kstride;
  for (int r = 0; r < nrec; ++r) {
    const int i0 = rstart[r], cnt = rstart[r + 1] - i0;
    const int32_t* sl = lslot + i0;
    int band;
    const int kind = slot_kind(st, u, sl[0], &band);
    uint8_t* p = out + off;
    if (lane == 0) {
      p[0] = (uint8_t)kind;
      p[1] = (uint8_t)band;
      put16(p + 2, (uint32_t)cnt);
    }
    for (int t = lane; t < cnt; t += 32) put64(p + 4 + 8 * t, (uint64_t)(int64_t)st.slot_id[(int64_t)u * dm.NS + sl[t]]);
    p += 4 + 8 * (int64_t)cnt;
    if (kind == TKV_FMT_RAW) {
      const int D = dm.D;
      for (int e = lane; e < cnt * 2 * D; e += 32) {
        const int t = e / (2 * D), c = e % (2 * D);
        const uint8_t* row = (c < D ? kbase : vbase) + (int64_t)sl[t] * dm.kstride;
        put64(p + 8 * (int64_t)e, (uint64_t)__double_as_longlong(raw_elem(dm, row, c < D ? c : c - D)));
      }
    } else if (kind == TKV_FMT_FP8) {
      const int64_t w = (int64_t)u * dm.NW + st.slot_win[(int64_t)u * dm.NS + sl[0]];
      const int nd = cnt * dm.D;
      if (lane == 0) {
        p[0] = TKV_FMT_FP8;
        put16(p + 1, (uint32_t)nd);
        put32(p + 3, __float_as_uint(st.win_kf[w]));
        uint8_t* q = p + 7 + nd;
        q[0] = TKV_FMT_FP8;
        put16(q + 1, (uint32_t)nd);
        put32(q + 3, __float_as_uint(st.win_vf[w]));
      }
      for (int e = lane; e < nd; e += 32) {
        const int t = e / dm.D, c = e % dm.D;
        p[7 + e] = kbase[(int64_t)sl[t] * dm.kstride + c];
        p[7 + nd + 7 + e] = vbase[(int64_t)sl[t] * dm.kstride + c];
      }
    } else {
      const int64_t w = (int64_t)u * dm.NW + st.slot_win[(int64_t)u * dm.NS + sl[0]];
      const int kg = 4 + packed_bytes(kind, cnt);
      for (int c = lane; c < dm.D; c += 32) {
        put_group(p + (int64_t)c * kg, kind, cnt, st.win_ks[w * dm.D + c], 0.f, [&](int t) {
          return tkv_get_code(kbase + (int64_t)sl[t] * dm.kstride, kind, c);
        });
      }
      p += (int64_t)dm.D * kg;
      int per_tok = 0;
      for (int j = 0; j < dm.vchunks; ++j) per_tok += 4 + packed_bytes(kind, min(dm.g, dm.D - j * dm.g));
      for (int e = lane; e < cnt * dm.vchunks; e += 32) {
        const int t = e / dm.vchunks, j = e % dm.vchunks;
        int jo = 0;
        for (int jj = 0; jj < j; ++jj) jo += 4 + packed_bytes(kind, min(dm.g, dm.D - jj * dm.g));
        const int c0 = j * dm.g, len = min(dm.g, dm.D - c0);
        const uint8_t* row = vbase + (int64_t)sl[t] * dm.kstride;
        put_group(p + (int64_t)t * per_tok + jo, kind, len, st.slot_vs[((int64_t)u * dm.NS + sl[t]) * dm.vchunks + j],
                  0.f, [&](int i) { return tkv_get_code(row, kind, c0 + i); });
      }
    }
    off += record_bytes(dm, kind, cnt);
  }
}

}  // namespace

// Warps (units) per CTA: kWarps, fewer when a large pool's per-warp lists
// would not fit in shared memory.
static int export_warps(const TkvState& st) {
  const size_t per = (2 * (size_t)st.dm.NS + 2) * sizeof(int32_t);
  int w = kWarps;
  while (w > 1 && (size_t)w * per > 200 * 1024) --w;
  return w;
}
size_t tkv_export_smem(const TkvState& st) { return (size_t)export_warps(st) * (2 * st.dm.NS + 2) * sizeof(int32_t); }

cudaError_t tkv_launch_export(const TkvState& st, int unit0, int nunits, int npos, int pass, int64_t* sizes,
                              const int64_t* offsets, uint8_t* dst, cudaStream_t stream) {
  if (nunits <= 0) return cudaSuccess;
  const int w = export_warps(st);
  const size_t smem = tkv_export_smem(st);
  if (smem > 200 * 1024) return cudaErrorInvalidConfiguration;  // NS > ~25K slots per unit
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(export_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  export_kernel<<<(nunits + w - 1) / w, 32 * w, smem, stream>>>(st, unit0, nunits, npos, pass, sizes, offsets, dst);
  return cudaGetLastError();
}
