// Device evaluation of tkv_exp (tkv_exp.cuh) over an array: the entry point
// tkv_exp_f64 exposes the exp that K3a (k_score.cu) and the gather
// comparator's exact mode (k_gather.cu) use, so tests can hold the device
// build to the C library's exp() bit for bit.
#include <cuda_runtime.h>

#include "tkv_exp.cuh"
#include "tkv_kernels.h"

namespace {

__global__ void exp_kernel(const double* __restrict__ x, double* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = tkv_exp(x[i]);
}

}  // namespace

cudaError_t tkv_launch_exp(const double* x, double* y, int64_t n, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const int blocks = (int)((n + 255) / 256 < 148 * 16 ? (n + 255) / 256 : 148 * 16);
  exp_kernel<<<blocks, 256, 0, stream>>>(x, y, n);
  return cudaGetLastError();
}
