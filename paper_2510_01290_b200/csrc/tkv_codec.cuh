// Scalar codecs on device, fp64 and bit-exact with the reference
// (proj/src/quant.cpp).  Division, rint (round-half-even, = nearbyint in the
// default rounding mode), frexp and fabs are IEEE-exact in CUDA double
// precision, and this file is compiled with --fmad=false, so every value
// matches the reference's baseline-x86-64 build bit for bit.
#pragma once
#include <stdint.h>

// quant.cpp:67-89 -- saturating E4M3, round-to-nearest-even, NaN -> error.
__device__ __forceinline__ uint8_t tkv_e4m3_encode(double x, bool* bad) {
  if (isnan(x)) { *bad = true; return 0; }
  const uint8_t sign = signbit(x) ? 0x80 : 0x00;
  const double a = fabs(x);
  if (a >= 448.0) return sign | 0x7E;
  if (a < 0.015625) {                      // 2^-6: subnormal range, unit 2^-9
    const double r = rint(a * 512.0);
    if (r >= 8.0) return sign | 0x08;
    return sign | (uint8_t)r;
  }
  int e = 0;
  double fr = frexp(a, &e);
  e -= 1;
  fr *= 2.0;
  double m = rint((fr - 1.0) * 8.0);
  if (m >= 8.0) { e += 1; m = 0.0; }
  if (e > 8 || (e == 8 && m > 6.0)) return sign | 0x7E;
  return sign | (uint8_t)((e + 7) << 3) | (uint8_t)m;
}

// quant.cpp:91-99
__device__ __forceinline__ double tkv_e4m3_decode(uint8_t code) {
  const double sign = (code & 0x80) ? -1.0 : 1.0;
  const int e = (code >> 3) & 0xF;
  const int m = code & 0x7;
  if (e == 15 && m == 7) return __longlong_as_double(0x7ff8000000000000ll);
  const double v = (e == 0) ? m * 0.001953125 : (1.0 + m / 8.0) * ldexp(1.0, e - 7);
  return sign * v;
}

__device__ __forceinline__ double tkv_nvfp4_grid(int i) {
  // {0, 0.5, 1, 1.5, 2, 3, 4, 6} (quant.cpp:106)
  return i < 4 ? 0.5 * i : (i == 4 ? 2.0 : (i == 5 ? 3.0 : (i == 6 ? 4.0 : 6.0)));
}

// quant.cpp:114-130 -- nearest grid point, ties to the even grid index.
__device__ __forceinline__ uint8_t tkv_nvfp4_encode(double x) {
  if (x == 0.0) return 0;
  const uint8_t sign = signbit(x) ? 0x8 : 0x0;
  const double a = fabs(x);
  int best = 0;
  double best_dist = fabs(a - tkv_nvfp4_grid(0));
  for (int i = 1; i < 8; ++i) {
    const double dist = fabs(a - tkv_nvfp4_grid(i));
    if (dist < best_dist || (dist == best_dist && (i & 1) == 0)) {
      best = i;
      best_dist = dist;
    }
  }
  if (best == 0) return 0;
  return sign | (uint8_t)best;
}

// quant.cpp:219-236 -- ternary sign/magnitude 2-bit patterns.
__device__ __forceinline__ uint8_t tkv_ternary_bits(int v) { return v == 0 ? 0 : (v > 0 ? 1 : 3); }
__device__ __forceinline__ int tkv_ternary_value(uint32_t bits) {
  bits &= 3u;
  return bits == 1 ? 1 : (bits == 3 ? -1 : 0);
}

__device__ __forceinline__ double tkv_nvfp4_value(uint32_t code) {
  const double s = (code & 0x8) ? -1.0 : 1.0;
  return s * tkv_nvfp4_grid(code & 7);
}

// decode_code (quant.cpp:195-205) for one stored code; exact in fp64.
__device__ __forceinline__ double tkv_decode_code(int fmt, uint32_t code, double scale) {
  if (fmt == 0) return (double)tkv_ternary_value(code) * scale;
  if (fmt == 1) return tkv_nvfp4_value(code) * scale;
  return tkv_e4m3_decode((uint8_t)code) * scale;
}

// Packed code extraction: ternary 4 codes/byte (2 bits, low first), NVFP4 2
// codes/byte (low nibble first), FP8 one code/byte -- the little-endian bit
// order of the reference wire layout (quant.cpp:281-320).
__device__ __forceinline__ uint32_t tkv_get_code(const uint8_t* row, int fmt, int c) {
  if (fmt == 0) return (row[c >> 2] >> (2 * (c & 3))) & 3u;
  if (fmt == 1) return (row[c >> 1] >> (4 * (c & 1))) & 15u;
  return row[c];
}
