// thinkv::quantize_window (proj/include/thinkv/quant.hpp:170-172) over the
// device window encoder (tkv_dropin_quantize_window: the fp64 group
// encoders K2 runs at every emission, quant.cpp:141-193 semantics).  The
// argument checks and the 16-bit passthrough (no codes: the tokens are kept
// as given) stay on the host.
#include <vector>

#include "dropin.hpp"
#include "thinkv/quant.hpp"

namespace thinkv {

QuantizedWindow quantize_window(std::span<const KVEntry> tokens, ThoughtLabel label, const PrecisionMap& psi,
                                int group_size) {
  if (tokens.empty()) throw Error(ErrorKind::kStructural, "quantize_window: empty window");
  const int n = static_cast<int>(tokens.size());
  if (n > group_size) throw Error(ErrorKind::kStructural, "quantize_window: window exceeds g");
  const int d = static_cast<int>(tokens.front().key.size());
  for (const KVEntry& t : tokens) {
    if (!(t.thought == label)) throw Error(ErrorKind::kStructural, "quantize_window: mixed thought labels");
    if (static_cast<int>(t.key.size()) != d || static_cast<int>(t.value.size()) != d)
      throw Error(ErrorKind::kStructural, "quantize_window: ragged vectors");
  }
  QuantizedWindow w;
  w.head_dim = d;
  w.group_size = group_size;
  w.pad = group_size - n;
  const int bits = psi.bits_for(label);
  if (bits == 16) {
    w.raw = true;
    for (const KVEntry& t : tokens) {
      w.raw_keys.push_back(t.key);
      w.raw_values.push_back(t.value);
    }
    return w;
  }
  w.format = format_for_bits(bits);
  std::vector<double> K((std::size_t)n * d), V((std::size_t)n * d);
  for (int t = 0; t < n; ++t)
    for (int c = 0; c < d; ++c) {
      K[(std::size_t)t * d + c] = tokens[t].key[c];
      V[(std::size_t)t * d + c] = tokens[t].value[c];
    }
  const int chunks = (d + group_size - 1) / group_size;
  std::vector<std::uint8_t> kc((std::size_t)n * d), vc((std::size_t)n * d), ks(d), vs((std::size_t)n * chunks);
  float f8[2] = {0.0f, 0.0f};
  dropin::check(tkv_dropin_quantize_window(dropin::ctx(), n, d, bits, group_size, K.data(), V.data(), kc.data(),
                                           vc.data(), ks.data(), vs.data(), f8));
  w.key_codes.assign(n, std::vector<std::uint8_t>(d));
  w.value_codes.assign(n, std::vector<std::uint8_t>(d));
  for (int t = 0; t < n; ++t)
    for (int c = 0; c < d; ++c) {
      w.key_codes[t][c] = kc[(std::size_t)t * d + c];
      w.value_codes[t][c] = vc[(std::size_t)t * d + c];
    }
  if (w.format == Format::kFp8E4M3) {
    w.key_scale_f32 = f8[0];
    w.value_scale_f32 = f8[1];
    return w;
  }
  w.key_scale_codes = ks;
  w.value_scale_codes.assign(n, std::vector<std::uint8_t>(chunks));
  for (int t = 0; t < n; ++t)
    for (int j = 0; j < chunks; ++j) w.value_scale_codes[t][j] = vs[(std::size_t)t * chunks + j];
  return w;
}

}  // namespace thinkv
