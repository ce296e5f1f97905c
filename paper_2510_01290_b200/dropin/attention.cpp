// thinkv::gqa_attend / sparsity / layer_sparsity_average
// (proj/include/thinkv/attention.hpp:62-76) over the device kernels: fp64 in
// the reference's operation order with glibc's exp (tkv_exp), so outputs and
// scores carry the reference's bits (attention.cpp:124-167).
#include <vector>

#include "dropin.hpp"
#include "thinkv/attention.hpp"

namespace thinkv {

AttendResult gqa_attend(std::span<const Vec> queries, std::span<const Vec* const> keys,
                        std::span<const Vec* const> values, double scale) {
  if (queries.empty()) throw Error(ErrorKind::kStructural, "gqa_attend: empty query group");
  if (keys.size() != values.size()) throw Error(ErrorKind::kStructural, "key/value count mismatch");
  if (keys.empty()) throw Error(ErrorKind::kStructural, "attention over an empty cache");
  const std::size_t d = queries.front().size();
  for (const Vec& q : queries)
    if (q.size() != d) throw Error(ErrorKind::kStructural, "gqa_aggregate: ragged logit rows");
  for (const Vec* k : keys)
    if (k->size() != d) throw Error(ErrorKind::kStructural, "key/query dimension mismatch");
  const std::size_t vd = values.front()->size();
  for (const Vec* v : values)
    if (v->size() != vd) throw Error(ErrorKind::kStructural, "value dimension mismatch");
  if (vd != d) throw Error(ErrorKind::kStructural, "value/query dimension mismatch");
  const std::size_t n = keys.size();
  std::vector<double> Q(queries.size() * d), K(n * d), V(n * d);
  for (std::size_t g = 0; g < queries.size(); ++g) std::copy(queries[g].begin(), queries[g].end(), Q.begin() + g * d);
  for (std::size_t i = 0; i < n; ++i) {
    std::copy(keys[i]->begin(), keys[i]->end(), K.begin() + i * d);
    std::copy(values[i]->begin(), values[i]->end(), V.begin() + i * d);
  }
  AttendResult r;
  r.output.resize(d);
  r.row.scores.resize(n);
  dropin::check(tkv_dropin_gqa_attend(dropin::ctx(), static_cast<int32_t>(queries.size()), static_cast<int64_t>(n),
                                      static_cast<int32_t>(d), scale, Q.data(), K.data(), V.data(), r.output.data(),
                                      r.row.scores.data()));
  return r;
}

AttendResult gqa_attend(std::span<const Vec> queries, std::span<const Vec> keys, std::span<const Vec> values,
                        double scale) {
  std::vector<const Vec*> kp, vp;
  for (const Vec& k : keys) kp.push_back(&k);
  for (const Vec& v : values) vp.push_back(&v);
  return gqa_attend(queries, std::span<const Vec* const>(kp), std::span<const Vec* const>(vp), scale);
}

namespace {

std::vector<double> row_sparsities(std::span<const AttentionRow> rows, double threshold_fraction) {
  std::vector<double> scores;
  std::vector<int64_t> offs{0};
  for (const AttentionRow& r : rows) {
    if (r.scores.empty()) throw Error(ErrorKind::kStructural, "sparsity of an empty row");
    scores.insert(scores.end(), r.scores.begin(), r.scores.end());
    offs.push_back(static_cast<int64_t>(scores.size()));
  }
  std::vector<double> out(rows.size());
  dropin::check(tkv_dropin_sparsity(dropin::ctx(), scores.data(), offs.data(), static_cast<int32_t>(rows.size()),
                                    threshold_fraction, out.data()));
  return out;
}

}  // namespace

double sparsity(const AttentionRow& row, double threshold_fraction) {
  return row_sparsities(std::span<const AttentionRow>(&row, 1), threshold_fraction)[0];
}

double layer_sparsity_average(std::span<const AttentionRow> rows, double threshold_fraction) {
  if (rows.empty()) throw Error(ErrorKind::kStructural, "layer_sparsity_average: no rows");
  double sum = 0.0;
  for (double s : row_sparsities(rows, threshold_fraction)) sum += s;  // row order, as the reference sums
  return sum / static_cast<double>(rows.size());
}

}  // namespace thinkv
