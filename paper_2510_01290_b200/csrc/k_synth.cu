// Device-side synthetic decode inputs (same integer generator as the host
// oracle, synth.h), so benchmark context can be built without host traffic.
#include <cuda_runtime.h>

#include "synth.h"
#include "tkv_kernels.h"

namespace {

__global__ void synth_kernel(tkv_synth_params p, int64_t unit0, int units, int G, int D, int64_t step,
                             uint16_t* q, uint16_t* k, uint16_t* v) {
  const int64_t n_q = (int64_t)units * G * D;
  const int64_t n_kv = (int64_t)units * D;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_q + n_kv;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < n_q) {
      const int64_t u = i / ((int64_t)G * D);
      const int g = (int)((i / D) % G), c = (int)(i % D);
      q[i] = tkv_synth_q(&p, unit0 + u, step, g, c);
    } else {
      const int64_t j = i - n_q;
      const int64_t u = j / D;
      const int c = (int)(j % D);
      k[j] = tkv_synth_k(&p, unit0 + u, step, c);
      v[j] = tkv_synth_v(&p, unit0 + u, step, c);
    }
  }
}

}  // namespace

cudaError_t tkv_launch_synth(uint64_t seed, int units_per_seq, int tau, int sink_tokens, int64_t unit0, int units,
                             int G, int D, int64_t step, uint16_t* q, uint16_t* k, uint16_t* v,
                             cudaStream_t stream) {
  tkv_synth_params p;
  p.seed = seed;
  p.units_per_seq = units_per_seq;
  p.tau = tau;
  p.sink_tokens = sink_tokens;
  p.reserved = 0;
  const int64_t total = (int64_t)units * (G + 1) * D;
  int grid = (int)((total + 255) / 256);
  if (grid > 148 * 16) grid = 148 * 16;
  synth_kernel<<<grid, 256, 0, stream>>>(p, unit0, units, G, D, step, q, k, v);
  return cudaGetLastError();
}

namespace {
__global__ void init_kernel(TkvState st, int P) {
  const TkvDims& dm = st.dm;
  const int64_t total = (int64_t)dm.U * dm.NW;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x)
    st.win_free[i] = (int32_t)(i % dm.NW);
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < dm.U; u += (int64_t)gridDim.x * blockDim.x) {
    st.win_nfree[u] = dm.NW;
    st.unit_nfree[u] = P;
    st.err[u] = 0;
    st.sparsity[u] = 0.0;
  }
}
}  // namespace

cudaError_t tkv_launch_init(const TkvState& st, cudaStream_t stream) {
  init_kernel<<<148 * 4, 256, 0, stream>>>(st, st.dm.P);
  return cudaGetLastError();
}
