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
// One CTA per unit.  Distinct live windows are counted with a bitmap in
// shared memory (one bit per window id).  Runs when byte accounting is
// enabled (tkv_bytes_accounting), right after the attention launch of a step,
// so every timed K1 launch is matched with its own exact byte count.
#include <cuda_runtime.h>

#include "tkv_kernels.h"
#include "tkv_state.h"

namespace {

constexpr int kThreads = 128;

__global__ void __launch_bounds__(kThreads) bytes_kernel(TkvState st, unsigned long long* acc) {
  extern __shared__ uint32_t win_bits[];  // [2][nwords]: E4M3-scaled windows | FP8 windows
  const TkvDims& dm = st.dm;
  const int u = tkv_unit_of(st, blockIdx.x);
  const int nwords = (dm.NW + 31) / 32;
  for (int i = threadIdx.x; i < 2 * nwords; i += kThreads) win_bits[i] = 0u;
  __syncthreads();
  unsigned long long live = 0, resident = 0, code = 0, scale = 0, meta = 0;
  const int8_t* th = st.blk_thought + (int64_t)u * dm.P;
  const uint8_t* fl = st.blk_filled + (int64_t)u * dm.P;
  const uint32_t* ev = st.blk_evict + (int64_t)u * dm.P;
  const int32_t* sw = st.slot_win + (int64_t)u * dm.NS;
  // slot-granular walk: thread i takes slots i, i + 128, ...
  for (int s = threadIdx.x; s < dm.NS; s += kThreads) {
    const int b = s / dm.bs, sl = s - b * dm.bs;
    if (sl == 0) meta += 6;
    const int t = th[b];
    if (t < 0 || sl >= fl[b]) continue;
    resident += 1;
    if ((ev[b] >> sl) & 1u) continue;
    live += 1;
    meta += 4;
    code += 2ull * (unsigned)dm.band_bytes[t];
    const int fmt = dm.band_fmt[t];
    if (fmt == TKV_FMT_RAW) continue;
    const int w = sw[s];
    if (w < 0) continue;
    if (fmt != TKV_FMT_FP8) scale += (unsigned)dm.vchunks;
    atomicOr(&win_bits[(fmt == TKV_FMT_FP8 ? nwords : 0) + (w >> 5)], 1u << (w & 31));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * nwords; i += kThreads)
    scale += (unsigned long long)__popc(win_bits[i]) * (i < nwords ? (unsigned)dm.D : 8u);
  // warp reduce, then one atomic per warp per counter
  unsigned long long v[5] = {live, resident, code, scale, meta};
#pragma unroll
  for (int j = 0; j < 5; ++j) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[j] += __shfl_xor_sync(0xffffffffu, v[j], o);
  }
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int j = 0; j < 5; ++j)
      if (v[j]) atomicAdd(acc + j, v[j]);
  }
}

}  // namespace

cudaError_t tkv_launch_bytes(const TkvState& st, unsigned long long* acc, cudaStream_t stream) {
  const int n = tkv_launch_units(st);
  if (n <= 0) return cudaSuccess;
  const size_t smem = 2 * (size_t)((st.dm.NW + 31) / 32) * sizeof(uint32_t);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(bytes_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  bytes_kernel<<<n, kThreads, smem, stream>>>(st, acc);
  return cudaGetLastError();
}
