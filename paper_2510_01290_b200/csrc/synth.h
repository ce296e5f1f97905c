// Deterministic synthetic decode-step inputs, bit-identical on host and device.
//
// Units are (sequence, layer, kv-head) triples flattened as
//   u = (seq * layers + layer) * kv_heads + head
// and every value is produced by integer arithmetic on a counter-based hash,
// converted to float exactly (|x| < 2^24 * 2^-15) and rounded to bf16 with an
// explicit round-to-nearest-even bit trick, so the C oracle and the CUDA
// kernels see the same bf16 bits without sharing any floating-point
// evaluation order.
//
// Distribution (SURVEY.md §8d "Synthetic inputs"):
//   noise      ~ Irwin-Hall(4) over 16-bit uniforms, mean 0, std ~= 1.15
//   k[c]       = noise + 0.5*drift(segment,c) + (pos < 4 ? 4*sink[c] : 0)
//   q[g][c]    = alpha(seq, interval) * noise + sink[c]
//   v[c]       = noise
// where sink[c] is a per-unit +-1 pattern (the attention-sink direction,
// mirroring proj/src/toy_model.cpp:95-101), drift is a per-(unit, tau-interval)
// offset and alpha in {0.5, 1, 2, 4} varies per (sequence, interval) so the
// rows span a range of sparsities.  The hash is splitmix64's finaliser, the
// same mixer as thinkv::Rng::mix (proj/include/thinkv/rng.hpp:56-61).
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define TKV_HD __host__ __device__ __forceinline__
#else
#define TKV_HD static inline
#endif

TKV_HD uint64_t tkv_mix64(uint64_t a, uint64_t b) {
  uint64_t z = a + 0x9E3779B97F4A7C15ull * (b + 1);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Irwin-Hall(4) noise in units of 2^-15: range [-131070, 131070].
TKV_HD int32_t tkv_noise_units(uint64_t h) {
  const int32_t s = (int32_t)(h & 0xFFFF) + (int32_t)((h >> 16) & 0xFFFF) +
                    (int32_t)((h >> 32) & 0xFFFF) + (int32_t)((h >> 48) & 0xFFFF);
  return s - 131070;
}

// Exact integer (units of 2^-15, |v| < 2^24) -> float -> bf16 bits (RNE).
TKV_HD uint16_t tkv_units_to_bf16(int32_t units) {
  float f = (float)units * (1.0f / 32768.0f);  // exact: |units| < 2^24
  union { float f; uint32_t u; } cvt;
  cvt.f = f;
  uint32_t bits = cvt.u;
  bits += 0x7FFFu + ((bits >> 16) & 1u);
  return (uint16_t)(bits >> 16);
}

TKV_HD float tkv_bf16_to_float(uint16_t b) {
  union { uint32_t u; float f; } cvt;
  cvt.u = ((uint32_t)b) << 16;
  return cvt.f;
}

typedef struct tkv_synth_params {
  uint64_t seed;
  int32_t units_per_seq;  // layers * kv_heads
  int32_t tau;            // drift / alpha change every tau steps
  int32_t sink_tokens;    // positions < sink_tokens carry the sink bias
  int32_t reserved;
} tkv_synth_params;

enum { TKV_ROLE_Q = 1, TKV_ROLE_K = 2, TKV_ROLE_V = 3, TKV_ROLE_SINK = 4,
       TKV_ROLE_DRIFT = 5, TKV_ROLE_ALPHA = 6, TKV_ROLE_LABEL = 7 };

// Per-unit sink sign for channel c: +1 or -1 (units of 2^-15 * 32768 = 1.0).
TKV_HD int32_t tkv_sink_units(const tkv_synth_params* p, int64_t unit, int c) {
  const uint64_t h = tkv_mix64(tkv_mix64(p->seed, TKV_ROLE_SINK), (uint64_t)unit);
  const uint64_t hc = tkv_mix64(h, (uint64_t)(c >> 6));
  return ((hc >> (c & 63)) & 1u) ? 32768 : -32768;
}

// alpha(seq, interval) as a left shift of the noise: 0.5, 1, 2, 4.
TKV_HD int tkv_alpha_shift(const tkv_synth_params* p, int64_t seq, int64_t step) {
  const int64_t interval = step / (p->tau > 0 ? p->tau : 1);
  const uint64_t h = tkv_mix64(tkv_mix64(p->seed, TKV_ROLE_ALPHA),
                               tkv_mix64((uint64_t)seq, (uint64_t)interval));
  return (int)(h & 3u) - 1;  // -1 .. 2
}

TKV_HD uint16_t tkv_synth_k(const tkv_synth_params* p, int64_t unit, int64_t step, int c) {
  const uint64_t hu = tkv_mix64(tkv_mix64(p->seed, TKV_ROLE_K), (uint64_t)unit);
  const uint64_t h = tkv_mix64(tkv_mix64(hu, (uint64_t)step), (uint64_t)c);
  int32_t v = tkv_noise_units(h);
  const int64_t interval = step / (p->tau > 0 ? p->tau : 1);
  const uint64_t hd = tkv_mix64(tkv_mix64(tkv_mix64(p->seed, TKV_ROLE_DRIFT), (uint64_t)unit),
                                tkv_mix64((uint64_t)interval, (uint64_t)c));
  v += tkv_noise_units(hd) / 2;
  if (step < p->sink_tokens) v += 4 * tkv_sink_units(p, unit, c);
  return tkv_units_to_bf16(v);
}

TKV_HD uint16_t tkv_synth_v(const tkv_synth_params* p, int64_t unit, int64_t step, int c) {
  const uint64_t hu = tkv_mix64(tkv_mix64(p->seed, TKV_ROLE_V), (uint64_t)unit);
  const uint64_t h = tkv_mix64(tkv_mix64(hu, (uint64_t)step), (uint64_t)c);
  return tkv_units_to_bf16(tkv_noise_units(h));
}

TKV_HD uint16_t tkv_synth_q(const tkv_synth_params* p, int64_t unit, int64_t step, int g, int c) {
  const uint64_t hu = tkv_mix64(tkv_mix64(p->seed, TKV_ROLE_Q), (uint64_t)unit);
  const uint64_t h = tkv_mix64(tkv_mix64(hu, (uint64_t)step), (uint64_t)(g * 4096 + c));
  int32_t n = tkv_noise_units(h);
  const int64_t seq = unit / (p->units_per_seq > 0 ? p->units_per_seq : 1);
  const int sh = tkv_alpha_shift(p, seq, step);
  n = sh < 0 ? n / 2 : n * (1 << sh);
  return tkv_units_to_bf16(n + tkv_sink_units(p, unit, c));
}

// Scripted thought band of refresh interval `interval` of sequence `seq`:
// T (band num_thoughts-1) with probability pT_permille/1000, otherwise the
// remaining bands uniformly (R/E 50/50 for the canonical taxonomy).
TKV_HD int tkv_synth_band(uint64_t seed, int64_t seq, int64_t interval,
                          int num_thoughts, int pT_permille) {
  const uint64_t h = tkv_mix64(tkv_mix64(seed, TKV_ROLE_LABEL),
                               tkv_mix64((uint64_t)seq, (uint64_t)interval));
  if (num_thoughts < 3) return (int)((h >> 20) % (uint64_t)num_thoughts);
  if ((int)(h % 1000u) < pT_permille) return num_thoughts - 1;
  return (int)((h >> 20) % (uint64_t)(num_thoughts - 1));
}
