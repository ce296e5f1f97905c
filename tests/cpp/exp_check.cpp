// Host build of tkv_exp (csrc/tkv_exp.cuh) against the C library's exp(),
// bit for bit, over N inputs per range (tests/test_exp.py).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

#include "tkv_exp.cuh"

static uint64_t bits(double d) {
  uint64_t u;
  std::memcpy(&u, &d, sizeof u);
  return u;
}

int main(int argc, char** argv) {
  const long n = argc > 1 ? std::atol(argv[1]) : 1000000;
  std::mt19937_64 rng(12345);
  struct Range { double lo, hi; } ranges[] = {
      {-1.0, 1.0}, {-50.0, 0.0}, {-800.0, 800.0}, {-746.0, -700.0}, {-1100.0, -500.0}, {500.0, 720.0},
      {-1e-15, 1e-15}, {-40.0, 40.0}};
  long bad = 0, total = 0;
  for (const Range& r : ranges) {
    std::uniform_real_distribution<double> U(r.lo, r.hi);
    for (long i = 0; i < n; ++i) {
      const double x = U(rng);
      const double a = tkv_exp(x), b = std::exp(x);
      ++total;
      if (bits(a) != bits(b)) {
        if (bad < 10) std::printf("mismatch x=%a tkv=%a libc=%a\n", x, a, b);
        ++bad;
      }
    }
  }
  // random bit patterns (every exponent, signs, subnormals, inf/nan)
  for (long i = 0; i < n; ++i) {
    uint64_t u = rng();
    double x;
    std::memcpy(&x, &u, sizeof x);
    const double a = tkv_exp(x), b = std::exp(x);
    ++total;
    if (bits(a) != bits(b) && !(std::isnan(a) && std::isnan(b))) {
      if (bad < 10) std::printf("mismatch x=%a tkv=%a libc=%a\n", x, a, b);
      ++bad;
    }
  }
  const double specials[] = {0.0, -0.0, 512.0, -512.0, 709.782712893384, 709.7827128933841, -708.3964185322641,
                             -745.1332191019411, -745.1332191019412, 1024.0, -1024.0, 0x1p-54, -0x1p-54,
                             0x1p-55, INFINITY, -INFINITY};
  for (double x : specials) {
    const double a = tkv_exp(x), b = std::exp(x);
    ++total;
    if (bits(a) != bits(b)) {
      std::printf("mismatch x=%a tkv=%a libc=%a\n", x, a, b);
      ++bad;
    }
  }
  std::printf("checked %ld mismatches %ld\n", total, bad);
  return bad != 0;
}
