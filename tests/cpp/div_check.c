/* Markstein division by a small integer (k_kmeans.cu div_n): for every
 * n in [3, 1024] that is not a power of two and many x (random doubles and
 * sums of few-bit values like the K-means key sums),
 *   r = RN(1/n), q0 = RN(x r), rem = fma(-q0, n, x), q = fma(rem, r, q0)
 * must equal RN(x / n) bit for bit.  Prints "bad <count> of <total>". */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static uint64_t s = 0x9E3779B97F4A7C15ull;
static inline uint64_t rnd(void) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }

int main(int argc, char** argv) {
  const long per = argc > 1 ? atol(argv[1]) : 200000;
  long bad = 0, tot = 0;
  for (int n = 3; n <= 1024; ++n) {
    if ((n & (n - 1)) == 0) continue;
    const double r = 1.0 / (double)n;
    for (long k = 0; k < per; ++k) {
      double x;
      if (k & 1) {
        x = ldexp((double)(int64_t)(rnd() % (1ull << 40)) - (double)(1ull << 39), (int)(rnd() % 40) - 60);
      } else {
        const uint64_t e = 1023 - 40 + (rnd() % 80);
        const uint64_t bits = (rnd() & 0x000FFFFFFFFFFFFFull) | (e << 52) | (rnd() & 0x8000000000000000ull);
        memcpy(&x, &bits, 8);
      }
      const double q0 = x * r;
      const double rem = fma(-q0, (double)n, x);
      const double q = q0 == 0.0 ? q0 : fma(rem, r, q0);
      const double want = x / (double)n;
      ++tot;
      if (memcmp(&q, &want, 8) != 0) ++bad;
    }
  }
  printf("bad %ld of %ld\n", bad, tot);
  return bad != 0;
}
