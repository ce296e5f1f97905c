// exp(x) in double, bit-identical to the exp() the reference's CPU build
// calls: attention.cpp:62 (softmax_row) -> glibc >= 2.28 exp, the ARM
// optimized-routines algorithm (sysdeps/ieee754/dbl-64/e_exp.c), in the form
// glibc's x86-64 ifunc selects on CPUs with FMA + AVX2 (__exp_fma: the same C
// source compiled with -mfma, so GCC fused the multiply-adds listed below).
//
//   x = k ln2/128 + r,  exp(x) = 2^(k/128) exp(r)
//   kd  = fma(x, 128/ln2, 0x1.8p52)    ki = bits(kd)    kd -= 0x1.8p52
//   r   = fma(kd, -ln2hi/128, x);  r = fma(kd, -ln2lo/128, r)
//   tmp = fma(r2*r2, fma(r, C5, C4), fma(fma(r, C3, C2), r2, tail + r))
//   exp = fma(scale, tmp, scale),  scale = bits(T[2j+1] + (ki << 45))
// plus the reference's handling of tiny, huge and subnormal-result inputs.
//
// The operation sequence (which products are fused, the association of
// every sum) was read off this image's libm (objdump of __exp_fma);
// tests/test_exp.py checks a host build of this function against the C
// library's exp() bit for bit, and tests/test_gpu_exp.py the device build.
// CUDA's own exp() is within 1 ulp but rounds differently on a fraction of
// inputs, which would flip sparsity counts and gather victims that the
// reference decides with this exp.
#pragma once
#include <stdint.h>
#include <string.h>

#include "tkv_exp_table.h"

#if defined(__CUDACC__)
#define TKV_EXP_HD __host__ __device__
#else
#define TKV_EXP_HD
#include <cmath>
#endif

#if defined(__CUDACC__)
static __device__ const uint64_t tkv_exp_tab_dev[256] = TKV_EXP_TABLE_INIT;
#endif
static const uint64_t tkv_exp_tab_host[256] = TKV_EXP_TABLE_INIT;

namespace tkv_exp_detail {

TKV_EXP_HD inline double as_double(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)u);
#else
  double d;
  memcpy(&d, &u, sizeof d);
  return d;
#endif
}
TKV_EXP_HD inline uint64_t as_u64(double d) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__double_as_longlong(d);
#else
  uint64_t u;
  memcpy(&u, &d, sizeof u);
  return u;
#endif
}
// Explicitly rounded IEEE operations (device: no contraction whatever the flags).
TKV_EXP_HD inline double fma_rn(double a, double b, double c) {
#if defined(__CUDA_ARCH__)
  return __fma_rn(a, b, c);
#else
  return std::fma(a, b, c);
#endif
}
TKV_EXP_HD inline double mul_rn(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dmul_rn(a, b);
#else
  volatile double p = a * b;
  return p;
#endif
}
TKV_EXP_HD inline double add_rn(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dadd_rn(a, b);
#else
  volatile double s = a + b;
  return s;
#endif
}
TKV_EXP_HD inline double sub_rn(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dsub_rn(a, b);
#else
  volatile double s = a - b;
  return s;
#endif
}
TKV_EXP_HD inline uint64_t tab(int i) {
#if defined(__CUDA_ARCH__)
  return tkv_exp_tab_dev[i];
#else
  return tkv_exp_tab_host[i];
#endif
}

constexpr double kInvLn2N = 0x1.71547652b82fep+7;
constexpr double kShift = 0x1.8p52;
constexpr double kNegLn2hiN = -0x1.62e42fefa0000p-8;
constexpr double kNegLn2loN = -0x1.cf79abc9e3b3ap-47;
constexpr double kC2 = 0x1.ffffffffffdbdp-2;
constexpr double kC3 = 0x1.555555555543cp-3;
constexpr double kC4 = 0x1.55555cf172b91p-5;
constexpr double kC5 = 0x1.1111167a4d017p-7;

// Results whose exponent leaves the normal range of scale (|x| >= 512).
TKV_EXP_HD inline double specialcase(double tmp, uint64_t sbits, uint64_t ki) {
  if ((ki & 0x80000000ull) == 0) {
    // k > 0: the exponent of scale may have overflowed by <= 460
    const double scale = as_double(sbits - (1009ull << 52));
    return mul_rn(fma_rn(scale, tmp, scale), 0x1p1009);
  }
  // k < 0: round once to the final precision before scaling into the subnormals
  const double scale = as_double(sbits + (1022ull << 52));
  const double st = mul_rn(scale, tmp);
  double y = add_rn(scale, st);
  if (1.0 > y) {
    const double hi = add_rn(y, 1.0);
    const double lo = add_rn(sub_rn(scale, y), st);
    double v = add_rn(sub_rn(1.0, hi), y);
    v = add_rn(v, lo);
    v = add_rn(v, hi);
    y = sub_rn(v, 1.0);
    if (y == 0.0) y = 0.0;
  }
  return mul_rn(y, 0x1p-1022);
}

}  // namespace tkv_exp_detail

TKV_EXP_HD inline double tkv_exp(double x) {
  using namespace tkv_exp_detail;
  const uint64_t ux = as_u64(x);
  uint32_t abstop = (uint32_t)(ux >> 52) & 0x7ffu;
  if (abstop - 0x3c9u >= 0x3fu) {  // |x| < 2^-54 or |x| >= 512 (or inf/nan)
    if ((int32_t)(abstop - 0x3c9u) < 0) return add_rn(x, 1.0);
    if (abstop >= 0x409u) {
      if (ux == 0xfff0000000000000ull) return 0.0;
      if (abstop >= 0x7ffu) return add_rn(x, 1.0);
      return (ux >> 63) ? 0.0 : as_double(0x7ff0000000000000ull);
    }
    abstop = 0;  // 512 <= |x| < 1024: scale handled in specialcase
  }
  double kd = fma_rn(x, kInvLn2N, kShift);
  const uint64_t ki = as_u64(kd);
  kd = sub_rn(kd, kShift);
  double r = fma_rn(kd, kNegLn2hiN, x);
  r = fma_rn(kd, kNegLn2loN, r);
  const int idx = 2 * (int)(ki & 127u);
  const uint64_t top = ki << 45;
  const double tail = as_double(tab(idx));
  const uint64_t sbits = tab(idx + 1) + top;
  const double p1 = fma_rn(r, kC3, kC2);
  const double a = add_rn(r, tail);
  const double r2 = mul_rn(r, r);
  const double p2 = fma_rn(r, kC5, kC4);
  const double b = fma_rn(p1, r2, a);
  const double r4 = mul_rn(r2, r2);
  const double tmp = fma_rn(r4, p2, b);
  if (abstop == 0) return specialcase(tmp, sbits, ki);
  const double scale = as_double(sbits);
  return fma_rn(scale, tmp, scale);
}
