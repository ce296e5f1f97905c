// Algorithmic-byte accounting of one attention launch, computed on the device
// from the state that launch reads (the roofline numerator).
//
// Rules are the reference's own FragmentationStats (proj/src/pager.cpp:299-325)
// restricted to what K1 must read from HBM:
//   live code bytes   2 * band_bytes per live slot (key + value codes)
//   live scale bytes  ceil(d/g) E4M3 value-chunk scales per live slot, plus
//                     d E4M3 key scales per live window (a window = one
//                     16-token emission; its record is counted once however
//                     many of its tokens are live, refs > 0 in the reference),
//                     or 8 B (two f32 scales) per live FP8 window
//   metadata          6 B per pool block (thought, filled, eviction mask) and
//                     4 B per live slot (slot -> window index)
// The host adds the buffer, current-token, q and out bytes (known per launch).
//
// One CTA per unit: pass 1 walks the block table (a thread per block: live
// slot mask, counts, code and value-scale bytes), pass 2 reads the window
// index of live slots only (coalesced) and marks distinct live windows in a
// shared-memory bitmap (one bit per window id).  Runs when byte accounting is
// enabled (tkv_bytes_accounting), right after the attention launch of a step
// whose pager state changed since the previous accounted launch (an emission,
// an eviction, a layer-by-layer launch): the counts depend only on the block
// table and the slot -> window map, which K1 does not modify, so a launch on
// unchanged state reads exactly the bytes of the previous one.  The kernel
// keeps each unit's latest counts (last[u][5]) and first credits the
// `repeat` unchanged launches since it last ran; the host credits the tail
// (last x pending) when it reads.  Counts accumulate per unit (acc[u][5]);
// the host sums the rows when it reads them.
#include <cuda_runtime.h>

#include "tkv_kernels.h"
#include "tkv_state.h"

namespace {

constexpr int kThreads = 128;

__global__ void __launch_bounds__(kThreads) bytes_kernel(TkvState st, unsigned long long* acc,
                                                         unsigned long long* last, long long repeat) {
  extern __shared__ uint32_t win_bits[];  // [2][nwords] E4M3-scaled | FP8 windows, then live slot masks [P]
  const TkvDims& dm = st.dm;
  const int u = tkv_unit_of(st, blockIdx.x);
  const int nwords = (dm.NW + 31) / 32;
  uint32_t* live_m = win_bits + 2 * nwords;                      // live slot mask per block
  uint8_t* blk_fp8 = reinterpret_cast<uint8_t*>(live_m + dm.P);  // FP8 block flags
  for (int i = threadIdx.x; i < 2 * nwords; i += kThreads) win_bits[i] = 0u;
  unsigned long long live = 0, resident = 0, code = 0, scale = 0, meta = 0;
  // pass 1: one block per thread -- live slot mask, counts, code bytes
  for (int b = threadIdx.x; b < dm.P; b += kThreads) {
    meta += 6;
    const int t = st.blk_thought[(int64_t)u * dm.P + b];
    uint32_t lm = 0;
    if (t >= 0) {
      const int f = st.blk_filled[(int64_t)u * dm.P + b];
      const uint32_t fm = f >= 32 ? 0xffffffffu : ((1u << f) - 1u);
      lm = fm & ~st.blk_evict[(int64_t)u * dm.P + b];
      const int nl = __popc(lm);
      resident += (unsigned)f;
      live += (unsigned)nl;
      meta += 4ull * nl;
      code += 2ull * (unsigned)dm.band_bytes[t] * nl;
      const int fmt = dm.band_fmt[t];
      if (fmt == TKV_FMT_RAW) lm = 0;  // no scales
      else if (fmt != TKV_FMT_FP8) scale += (unsigned long long)dm.vchunks * nl;
    }
    live_m[b] = lm;
    blk_fp8[b] = t >= 0 && dm.band_fmt[t] == TKV_FMT_FP8;
  }
  __syncthreads();
  // pass 2: slot-parallel, coalesced slot -> window reads of live slots only,
  // kUnroll independent loads in flight per thread (the walk is latency bound)
  constexpr int kUnroll = 8;
  const int bs = dm.bs;
  const int32_t* sw = st.slot_win + (int64_t)u * dm.NS;
  for (int s0 = threadIdx.x; s0 < dm.NS; s0 += kThreads * kUnroll) {
    int w[kUnroll];
    int fp8[kUnroll];
#pragma unroll
    for (int j = 0; j < kUnroll; ++j) {
      const int s = s0 + j * kThreads;
      w[j] = -1;
      fp8[j] = 0;
      if (s < dm.NS) {
        const int b = s / bs;
        const uint32_t lm = live_m[b];
        if ((lm >> (s - b * bs)) & 1u) {
          w[j] = __ldg(sw + s);
          fp8[j] = blk_fp8[b];
        }
      }
    }
#pragma unroll
    for (int j = 0; j < kUnroll; ++j)
      if (w[j] >= 0) atomicOr(&win_bits[(fp8[j] ? nwords : 0) + (w[j] >> 5)], 1u << (w[j] & 31));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * nwords; i += kThreads)
    scale += (unsigned long long)__popc(win_bits[i]) * (i < nwords ? (unsigned)dm.D : 8u);
  // block reduce, then one plain add per counter into this unit's own row
  // (no same-address atomics across the grid)
  __shared__ unsigned long long red[kThreads / 32][5];
  unsigned long long v[5] = {live, resident, code, scale, meta};
#pragma unroll
  for (int j = 0; j < 5; ++j) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[j] += __shfl_xor_sync(0xffffffffu, v[j], o);
  }
  if ((threadIdx.x & 31) == 0)
#pragma unroll
    for (int j = 0; j < 5; ++j) red[threadIdx.x >> 5][j] = v[j];
  __syncthreads();
  if (threadIdx.x < 5) {
    unsigned long long t = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) t += red[w][threadIdx.x];
    const int64_t i = (int64_t)u * 5 + threadIdx.x;
    acc[i] += last[i] * (unsigned long long)repeat + t;
    last[i] = t;
  }
}

// acc += last * repeat for every unit (before a launch that covers a unit subset)
__global__ void bytes_repeat_kernel(unsigned long long* acc, const unsigned long long* last, int64_t n,
                                    long long repeat) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    acc[i] += last[i] * (unsigned long long)repeat;
}

}  // namespace

cudaError_t tkv_launch_bytes_repeat(unsigned long long* acc, const unsigned long long* last, int64_t units,
                                    long long repeat, cudaStream_t stream) {
  if (repeat <= 0 || units <= 0) return cudaSuccess;
  bytes_repeat_kernel<<<(int)((units * 5 + 255) / 256), 256, 0, stream>>>(acc, last, units * 5, repeat);
  return cudaGetLastError();
}

cudaError_t tkv_launch_bytes(const TkvState& st, unsigned long long* acc, unsigned long long* last,
                             long long repeat, cudaStream_t stream) {
  const int n = tkv_launch_units(st);
  if (n <= 0) return cudaSuccess;
  const size_t smem = (2 * (size_t)((st.dm.NW + 31) / 32) + st.dm.P) * sizeof(uint32_t) + st.dm.P;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(bytes_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  bytes_kernel<<<n, kThreads, smem, stream>>>(st, acc, last, repeat);
  return cudaGetLastError();
}
