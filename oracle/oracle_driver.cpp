// Oracle driver (TEST INFRASTRUCTURE ONLY).  See oracle_driver.h.
//
// `SeqOracle` restates the reference's private ThinkvMethod
// (/root/reference/proj/src/sim.cpp:494-958) step for step; each member
// function cites the lines it follows.  All arithmetic goes through the
// compiled reference library, so the only thing restated here is control
// flow and bookkeeping, and that restatement is pinned against
// thinkv::generation_loop itself by orc_toy_compare (tests/test_oracle.py).
#include "oracle_driver.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <numeric>
#include <set>
#include <string>
#include <unordered_set>
#include <vector>

#include "thinkv/attention.hpp"
#include "thinkv/errors.hpp"
#include "thinkv/evictor.hpp"
#include "thinkv/pager.hpp"
#include "thinkv/quant.hpp"
#include "thinkv/rng.hpp"
#include "thinkv/sim.hpp"
#include "thinkv/thought.hpp"
#include "thinkv/toy_model.hpp"

using nlohmann::json;
using namespace thinkv;

namespace {

// One decode step's inputs for every unit of a sequence (sim.cpp:348-356).
struct StepIn {
  std::int64_t pos = 0;
  bool prefill = false;
  std::vector<std::vector<Vec>> queries;  // [unit][head]
  std::vector<Vec> keys, values;          // [unit]
  // Optional shadow references for the fidelity metrics (sim.cpp:770-776).
  bool has_shadow = false;
  std::vector<AttentionRow> full_avg_rows;
  std::vector<Vec> full_outputs;
};

struct Fidelity {  // sim.cpp:467-481
  std::vector<double> recall, error;
  double recall_sum = 0.0;
  std::int64_t recall_count = 0;
};

double l2(const Vec& a, const Vec& b) {
  double d = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    const double t = a[i] - b[i];
    d += t * t;
  }
  return std::sqrt(d);
}

class SeqOracle {
 public:
  explicit SeqOracle(const SimConfig& cfg) : cfg_(cfg), psi_(cfg.effective_psi()) {
    const int n = cfg.model.num_layers;
    const int pool = static_cast<int>(cfg.effective_pool_blocks());
    pagers_.reserve(n);
    for (int u = 0; u < n; ++u) pagers_.emplace_back(static_cast<int>(cfg.block_size), pool);
    segs_.resize(n);
    open_.assign(n, -1);
    buf_.resize(n);
    next_group_.assign(n, 1);
    dump_at_.insert(cfg.dump_positions.begin(), cfg.dump_positions.end());
  }

  // sim.cpp:748-843
  void process(const StepIn& in, std::vector<Vec>* outputs) {
    const int n = cfg_.model.num_layers;
    const int groups = cfg_.model.num_groups();
    const int gs = cfg_.model.gqa_group_size;
    const double scale = 1.0 / std::sqrt(static_cast<double>(cfg_.model.head_dim));
    const bool decode = !in.prefill;

    // (1) attention over pager slots, buffer and the incoming token.
    sparsity_.assign(n, 0.0);
    double err_sum = 0.0, rec_sum = 0.0;
    bool truncated = false;
    for (int u = 0; u < n; ++u) {
      std::vector<const Vec*> ks, vs;
      std::vector<TokenId> ids;
      for (const SlotPayload* p : pagers_[u].read_active()) {  // sim.cpp:546-563
        ks.push_back(&p->key_fp);
        vs.push_back(&p->value_fp);
        ids.push_back(p->id);
      }
      for (const KVEntry& e : buf_[u]) {
        ks.push_back(&e.key);
        vs.push_back(&e.value);
        ids.push_back(e.step);
      }
      ks.push_back(&in.keys[u]);
      vs.push_back(&in.values[u]);
      ids.push_back(in.pos);
      std::vector<AttentionRow> rows;
      Vec cat;
      for (int g = 0; g < groups; ++g) {
        std::span<const Vec> qs(in.queries[u].data() + g * gs, gs);
        AttendResult r = gqa_attend(qs, std::span<const Vec* const>(ks),
                                    std::span<const Vec* const>(vs), scale);
        cat.insert(cat.end(), r.output.begin(), r.output.end());
        rows.push_back(std::move(r.row));
      }
      sparsity_[u] = layer_sparsity_average(rows, cfg_.threshold_fraction);
      if (decode && in.has_shadow) {
        err_sum += l2(cat, in.full_outputs[u]);
        const RecallResult rr = recall_at_10(in.full_avg_rows[u], ids);
        rec_sum += rr.value;
        truncated = rr.truncated;
      }
      if (outputs) (*outputs)[u] = std::move(cat);
    }
    if (decode && in.has_shadow) {
      fid_.error.push_back(err_sum / n);
      if (!truncated) {
        fid_.recall.push_back(rec_sum / n);
        fid_.recall_sum += rec_sum / n;
        fid_.recall_count += 1;
      }
    }

    // (2) refresh boundary (sim.cpp:790-794).
    const std::int64_t bstep = decode ? in.pos - cfg_.prompt_len : in.pos;
    if (refresh_due(bstep, cfg_.tau)) boundary(in.pos, decode);

    // (3) buffer the token under the open segment (sim.cpp:796-808).
    for (int u = 0; u < n; ++u) {
      SegmentRecord& open = segs_[u][open_[u]];
      KVEntry e;
      e.key = in.keys[u];
      e.value = in.values[u];
      e.thought = open.thought;
      e.step = in.pos;
      e.layer = u;
      buf_[u].push_back(std::move(e));
      open.member_ids.push_back(in.pos);
      open.initial_size += 1;
    }
    if (decode)
      generated_by_thought_[thought_name(segs_[0][open_[0]].thought, cfg_.num_thoughts)] += 1;

    // (4) emit at g buffered tokens (sim.cpp:813-817).
    if (static_cast<std::int64_t>(buf_[0].size()) >= cfg_.group_size)
      for (int u = 0; u < n; ++u) flush(u, in.pos);

    // (5) Case-2 budget enforcement per unit (sim.cpp:819-838).
    bool any = false, infeasible = false;
    for (int u = 0; u < n; ++u) {
      if (total_members(segs_[u]) <= cfg_.budget) continue;
      EvictionPlan plan = on_budget_overflow(
          segs_[u], cfg_.budget, [this, u](TokenId id) { return pagers_[u].key_of(id); },
          cfg_.schedule, cfg_.num_thoughts);
      infeasible = infeasible || plan.budget_infeasible;
      any = true;
      apply(u, plan, in.pos);
    }
    if (any) {
      overflow_calls_ += 1;
      if (decode) eviction_steps_ += 1;
      if (infeasible) infeasible_events_ += 1;
    }
    if (dump_at_.count(in.pos))
      step_dumps_[std::to_string(in.pos)] = json{{"block_tables", tables()}, {"segments", segments()}};
  }

  // sim.cpp:871-958 (fidelity metrics only when shadow references were fed).
  json finish(bool with_fidelity) {
    const int n = cfg_.model.num_layers;
    const std::int64_t total = cfg_.prompt_len + cfg_.max_gen_len;
    for (int u = 0; u < n; ++u) flush(u, total);
    bool final_overflow = false;
    for (int u = 0; u < n; ++u) {
      if (open_[u] >= 0) segs_[u][open_[u]].open = false;
      if (total_members(segs_[u]) <= cfg_.budget) continue;
      EvictionPlan plan = on_budget_overflow(
          segs_[u], cfg_.budget, [this, u](TokenId id) { return pagers_[u].key_of(id); },
          cfg_.schedule, cfg_.num_thoughts);
      if (plan.budget_infeasible) infeasible_events_ += 1;
      apply(u, plan, total);
      final_overflow = true;
    }
    if (final_overflow) overflow_calls_ += 1;

    RunMetrics m;
    m.method = "thinkv";
    m.generated_length = cfg_.max_gen_len;
    m.prompt_length = cfg_.prompt_len;
    const int d = cfg_.model.head_dim;
    std::int64_t bits = 0, slots = 0;
    for (int u = 0; u < n; ++u) {
      const FragmentationStats st = pagers_[u].fragmentation_stats();
      bits += st.total_live_code_bits();
      slots += st.live_slots;
    }
    std::int64_t live_prompt = 0, live_gen = 0;
    for (const SlotPayload* p : pagers_[0].read_active()) {
      (p->step < cfg_.prompt_len ? live_prompt : live_gen) += 1;
      m.live_by_thought[thought_name(p->thought, cfg_.num_thoughts)] += 1;
    }
    m.live_tokens_final = live_prompt + live_gen;
    m.live_prompt_final = live_prompt;
    m.live_generated_final = live_gen;
    m.generated_by_thought = generated_by_thought_;
    m.avg_bits_per_token = slots > 0 ? static_cast<double>(bits) / (static_cast<double>(slots) * 2.0 * d) : 16.0;
    m.a = m.avg_bits_per_token / 16.0;
    m.b = cfg_.max_gen_len > 0 ? static_cast<double>(live_gen) / static_cast<double>(cfg_.max_gen_len) : 1.0;
    const double denom = static_cast<double>(n) * static_cast<double>(total) * 2.0 * d * 16.0;
    m.memory_footprint_fraction = static_cast<double>(bits) / denom;
    m.compression_ratio = m.memory_footprint_fraction > 0.0 ? 1.0 / m.memory_footprint_fraction : 0.0;
    m.eviction_call_fraction = static_cast<double>(eviction_steps_) / static_cast<double>(cfg_.max_gen_len);
    if (with_fidelity) {
      m.recall_at_10 = fid_.recall;
      m.attention_output_error = fid_.error;
      m.recall_at_10_mean = fid_.recall_count > 0 ? fid_.recall_sum / fid_.recall_count : 1.0;
      m.attention_output_error_mean =
          fid_.error.empty() ? 0.0
                             : std::accumulate(fid_.error.begin(), fid_.error.end(), 0.0) /
                                   static_cast<double>(fid_.error.size());
    }
    m.eviction_steps = eviction_steps_;
    m.transition_calls = transition_calls_;
    m.overflow_calls = overflow_calls_;
    m.budget_infeasible_events = infeasible_events_;
    m.moved_token_slots = 0;
    for (const auto& pg : pagers_) m.moved_token_slots += pg.moved_slot_count();
    return m.to_json();
  }

  // Compressed-cache export (k_export.cu layout) through the reference's own
  // public pager API and serialize_group (quant.cpp:274-324).
  std::vector<std::uint8_t> export_unit(int u) const {
    const BlockPager& pg = pagers_.at(u);
    std::vector<const SlotPayload*> live = pg.read_active();
    std::sort(live.begin(), live.end(), [](const SlotPayload* a, const SlotPayload* b) { return a->id < b->id; });
    const auto& groups = pg.group_table();
    auto kind = [](const SlotPayload* p) { return p->raw ? 3 : static_cast<int>(p->format); };
    auto same = [&](const SlotPayload* a, const SlotPayload* b) {
      return kind(a) == kind(b) && a->thought.band == b->thought.band &&
             (a->raw || a->key_group_base == b->key_group_base);
    };
    std::vector<std::uint8_t> out(12, 0);
    auto put = [&](std::uint64_t v, int n) {
      for (int i = 0; i < n; ++i) out.push_back(static_cast<std::uint8_t>(v >> (8 * i)));
    };
    auto put_group = [&](const QuantizedGroup& g) {
      const auto b = serialize_group(g);
      out.insert(out.end(), b.begin(), b.end());
    };
    const int d = cfg_.model.head_dim;
    std::uint32_t nrec = 0;
    for (std::size_t i0 = 0; i0 < live.size();) {
      std::size_t i1 = i0 + 1;
      while (i1 < live.size() && same(live[i0], live[i1])) ++i1;
      const SlotPayload* h = live[i0];
      const int n = static_cast<int>(i1 - i0);
      ++nrec;
      put(static_cast<std::uint64_t>(kind(h)), 1);
      put(static_cast<std::uint64_t>(h->thought.band), 1);
      put(static_cast<std::uint64_t>(n), 2);
      for (std::size_t i = i0; i < i1; ++i) put(static_cast<std::uint64_t>(live[i]->id), 8);
      if (h->raw) {
        for (std::size_t i = i0; i < i1; ++i)
          for (const Vec* v : {&live[i]->key_fp, &live[i]->value_fp})
            for (double x : *v) {
              std::uint64_t bits;
              std::memcpy(&bits, &x, 8);
              put(bits, 8);
            }
      } else if (h->format == Format::kFp8E4M3) {
        for (int side = 0; side < 2; ++side) {
          QuantizedGroup g;
          g.format = h->format;
          g.g = static_cast<std::uint16_t>(n * d);
          g.scale_f32 = groups.at(side == 0 ? h->key_group_base : h->value_group_base).scale_f32;
          for (std::size_t i = i0; i < i1; ++i) {
            const auto& c = side == 0 ? live[i]->key_codes : live[i]->value_codes;
            g.codes.insert(g.codes.end(), c.begin(), c.end());
          }
          put_group(g);
        }
      } else {
        for (int c = 0; c < d; ++c) {
          QuantizedGroup g;
          g.format = h->format;
          g.g = static_cast<std::uint16_t>(n);
          g.scale_code = groups.at(h->key_group_base + c).scale_code;
          for (std::size_t i = i0; i < i1; ++i) g.codes.push_back(live[i]->key_codes[c]);
          put_group(g);
        }
        for (std::size_t i = i0; i < i1; ++i) {
          const SlotPayload* p = live[i];
          for (int j = 0; j < p->value_chunks; ++j) {
            const int c0 = j * p->group_size, len = std::min(p->group_size, d - c0);
            QuantizedGroup g;
            g.format = p->format;
            g.g = static_cast<std::uint16_t>(len);
            g.scale_code = groups.at(p->value_group_base + j).scale_code;
            g.codes.assign(p->value_codes.begin() + c0, p->value_codes.begin() + c0 + len);
            put_group(g);
          }
        }
      }
      i0 = i1;
    }
    for (int i = 0; i < 4; ++i) out[i] = static_cast<std::uint8_t>(nrec >> (8 * i));
    for (int i = 0; i < 4; ++i) out[4 + i] = static_cast<std::uint8_t>(live.size() >> (8 * i));
    out[8] = static_cast<std::uint8_t>(d);
    out[9] = static_cast<std::uint8_t>(d >> 8);
    out[10] = static_cast<std::uint8_t>(cfg_.group_size);
    out[11] = static_cast<std::uint8_t>(cfg_.group_size >> 8);
    return out;
  }

  json frag() const {  // BlockPager::fragmentation_stats (pager.cpp:299-325), one object per unit
    json arr = json::array();
    for (const auto& pg : pagers_) {
      const FragmentationStats st = pg.fragmentation_stats();
      arr.push_back(json{{"live_slots", st.live_slots},
                         {"masked_slots", st.masked_slots},
                         {"unfilled_slots", st.unfilled_slots},
                         {"blocks_in_use", st.blocks_in_use},
                         {"free_blocks", st.free_blocks},
                         {"live_code_bits", st.total_live_code_bits()},
                         {"live_code_bits_by_format", st.live_code_bits_by_format},
                         {"live_scale_bytes", st.live_scale_bytes}});
    }
    return arr;
  }
  json tables() const {  // sim.cpp:939-943
    json arr = json::array();
    for (const auto& pg : pagers_) arr.push_back(pg.dump());
    return arr;
  }
  json segments() const {  // sim.cpp:919-937
    json units = json::array();
    for (const auto& list : segs_) {
      json arr = json::array();
      for (const auto& s : list)
        arr.push_back(json{{"id", s.id},
                           {"band", s.thought.band},
                           {"thought", thought_name(s.thought, cfg_.num_thoughts)},
                           {"start", s.start_step},
                           {"anneal_level", s.anneal_level},
                           {"open", s.open},
                           {"initial_size", s.initial_size},
                           {"size", s.size()},
                           {"members", s.member_ids}});
      units.push_back(std::move(arr));
    }
    return units;
  }
  std::string events() const {
    std::string s;
    for (const auto& e : events_) s += e.dump() + "\n";
    return s;
  }
  const json& step_dumps() const { return step_dumps_; }
  const std::vector<double>& sparsity() const { return sparsity_; }

 private:
  // sim.cpp:565-650: quantize the buffered window and place it in the pager.
  void flush(int u, std::int64_t pos) {
    auto& buffer = buf_[u];
    if (buffer.empty()) return;
    SegmentRecord& open = segs_[u][open_[u]];
    const ThoughtLabel label = open.thought;
    const int g = static_cast<int>(cfg_.group_size);
    const int d = cfg_.model.head_dim;
    QuantizedWindow w = quantize_window(buffer, label, psi_, g);
    const int n = static_cast<int>(buffer.size());
    std::vector<SlotPayload> slots(n);
    BlockPager& pager = pagers_[u];
    const TokenId first = buffer.front().step, last = buffer.back().step;
    for (int t = 0; t < n; ++t) {
      slots[t].id = buffer[t].step;
      slots[t].step = buffer[t].step;
      slots[t].thought = label;
    }
    if (w.raw) {
      for (int t = 0; t < n; ++t) {
        slots[t].raw = true;
        slots[t].key_fp = std::move(w.raw_keys[t]);
        slots[t].value_fp = std::move(w.raw_values[t]);
      }
    } else if (w.format == Format::kFp8E4M3) {
      const std::uint64_t kb = next_group_[u]++;
      const std::uint64_t vb = next_group_[u]++;
      pager.install_group(kb, GroupScaleRecord{w.format, true, 0, w.key_scale_f32, 0, first, last});
      pager.install_group(vb, GroupScaleRecord{w.format, true, 0, w.value_scale_f32, 0, first, last});
      for (int t = 0; t < n; ++t) {
        SlotPayload& s = slots[t];
        s.format = w.format;
        s.key_codes = std::move(w.key_codes[t]);
        s.value_codes = std::move(w.value_codes[t]);
        s.key_group_base = kb;
        s.value_group_base = vb;
        s.shared_scale = true;
        s.group_size = g;
      }
    } else {
      const int chunks = w.value_chunks();
      const std::uint64_t kb = next_group_[u];
      next_group_[u] += d;
      for (int c = 0; c < d; ++c)
        pager.install_group(kb + c, GroupScaleRecord{w.format, false, w.key_scale_codes[c], 0.0f, 0, first, last});
      const std::uint64_t vb = next_group_[u];
      next_group_[u] += static_cast<std::uint64_t>(n) * chunks;
      for (int t = 0; t < n; ++t) {
        for (int j = 0; j < chunks; ++j)
          pager.install_group(vb + static_cast<std::uint64_t>(t) * chunks + j,
                              GroupScaleRecord{w.format, false, w.value_scale_codes[t][j], 0.0f, 0,
                                               buffer[t].step, buffer[t].step});
        SlotPayload& s = slots[t];
        s.format = w.format;
        s.key_codes = std::move(w.key_codes[t]);
        s.value_codes = std::move(w.value_codes[t]);
        s.key_group_base = kb;
        s.value_group_base = vb + static_cast<std::uint64_t>(t) * chunks;
        s.value_chunks = chunks;
        s.group_size = g;
      }
    }
    pager.append_tokens(label, std::move(slots), open.start_step);
    events_.push_back(json{{"type", "emit"}, {"step", pos}, {"layer", u},
                           {"format", w.raw ? "RAW16" : format_name(w.format)},
                           {"tokens", n}, {"pad", w.pad}});
    buffer.clear();
  }

  // sim.cpp:652-671
  void apply(int u, const EvictionPlan& plan, std::int64_t pos) {
    if (plan.empty() && !plan.budget_infeasible) return;
    pagers_[u].apply_eviction_plan(plan);
    json segs = json::array();
    for (const auto& s : plan.segments)
      segs.push_back(json{{"segment", s.segment_id}, {"retained", s.retained.size()}, {"evicted", s.evicted}});
    const std::int64_t after = total_members(segs_[u]);
    events_.push_back(json{{"type", "evict"}, {"trigger", trigger_name(plan.trigger)}, {"step", pos},
                           {"layer", u}, {"segments", segs}, {"infeasible", plan.budget_infeasible},
                           {"retained_before", after + plan.evicted_count()}, {"retained_total", after}});
  }

  // sim.cpp:673-746
  void boundary(std::int64_t pos, bool decode) {
    const int n = cfg_.model.num_layers;
    for (int u = 0; u < n; ++u) flush(u, pos);
    bool fired = false;
    for (int u = 0; u < n; ++u) {
      if (open_[u] < 0) continue;
      SegmentRecord& open = segs_[u][open_[u]];
      open.open = false;
      if (decode && is_transition(open.thought, cfg_.num_thoughts)) {
        EvictionPlan plan = on_transition_end(
            segs_[u], open.start_step, [this, u](TokenId id) { return pagers_[u].key_of(id); },
            cfg_.schedule);
        const std::int64_t closing = open.start_step;
        const bool had_predecessors =
            std::any_of(segs_[u].begin(), segs_[u].end(),
                        [&](const SegmentRecord& s) { return s.start_step < closing; });
        apply(u, plan, pos);
        fired = fired || had_predecessors;
      }
      open_[u] = -1;
    }
    if (fired) {
      transition_calls_ += 1;
      eviction_steps_ += 1;
    }
    std::vector<int> bands(n, prefill_thought(cfg_.num_thoughts).band);
    double mean = 0.0;
    if (decode) {
      const std::int64_t dstep = pos - cfg_.prompt_len;
      const std::int64_t interval = dstep / cfg_.tau;
      if (cfg_.scripted.has_value()) {
        std::fill(bands.begin(), bands.end(), cfg_.scripted->band_at(interval));
        for (int u = 0; u < n; ++u) mean += sparsity_[u];
        mean /= static_cast<double>(n);
      } else if (cfg_.per_layer_thought) {
        for (int u = 0; u < n; ++u) bands[u] = classify(sparsity_[u], cfg_.calibration->thresholds).band;
      } else {
        for (int u : cfg_.calibration->layers) mean += sparsity_[u];
        mean /= static_cast<double>(cfg_.calibration->layers.size());
        const int band = classify(mean, cfg_.calibration->thresholds).band;
        std::fill(bands.begin(), bands.end(), band);
      }
      json ev{{"type", "refresh"}, {"step", pos}, {"dstep", dstep}, {"sparsity", mean}};
      if (cfg_.per_layer_thought && !cfg_.scripted.has_value())
        ev["bands"] = bands;
      else
        ev["band"] = bands[0];
      events_.push_back(std::move(ev));
    }
    for (int u = 0; u < n; ++u) {
      SegmentRecord s;
      s.id = next_seg_id_;
      s.thought = ThoughtLabel{bands[u]};
      s.start_step = pos;
      s.open = true;
      segs_[u].push_back(std::move(s));
      open_[u] = static_cast<int>(segs_[u].size()) - 1;
    }
    next_seg_id_ += 1;
  }

  SimConfig cfg_;
  PrecisionMap psi_;
  std::vector<BlockPager> pagers_;
  std::vector<std::vector<SegmentRecord>> segs_;
  std::vector<int> open_;
  std::vector<std::vector<KVEntry>> buf_;
  std::vector<std::uint64_t> next_group_;
  int next_seg_id_ = 0;
  std::vector<double> sparsity_;
  Fidelity fid_;
  std::vector<json> events_;
  std::int64_t eviction_steps_ = 0, transition_calls_ = 0, overflow_calls_ = 0, infeasible_events_ = 0;
  std::map<std::string, std::int64_t> generated_by_thought_;
  std::set<std::int64_t> dump_at_;
  json step_dumps_ = json::object();
};

SimConfig config_for_seq(const orc_desc& d, int seq) {
  SimConfig c;
  c.model.num_layers = d.units_per_seq;
  c.model.head_dim = d.head_dim;
  c.model.num_heads = d.num_q_heads;
  c.model.gqa_group_size = d.gqa_maxpool ? d.num_q_heads : 1;
  c.tau = d.tau;
  c.group_size = d.group_size;
  c.block_size = d.block_size;
  c.budget = d.budget;
  c.schedule.levels.assign(d.levels, d.levels + d.num_levels);
  c.num_thoughts = d.num_thoughts;
  c.psi = PrecisionMap();
  for (int b = 0; b < d.num_thoughts; ++b) c.psi.set(ThoughtLabel{b}, d.psi_bits[b]);
  c.max_gen_len = d.max_gen_len;
  c.prompt_len = d.prompt_len;
  c.pool_blocks = d.pool_blocks;
  c.per_layer_thought = d.per_layer_thought != 0;
  c.threshold_fraction = d.threshold_fraction;
  if (d.scripted) {
    ScriptedTrace t;
    t.interval_bands.assign(d.script_bands + static_cast<std::size_t>(seq) * d.script_len,
                            d.script_bands + static_cast<std::size_t>(seq + 1) * d.script_len);
    c.scripted = t;
  } else {
    CalibrationResult cal;
    cal.num_thoughts = d.num_thoughts;
    cal.thresholds.assign(d.thresholds, d.thresholds + d.num_thresholds);
    cal.layers.assign(d.calib_units, d.calib_units + d.num_calib_units);
    c.calibration = cal;
  }
  if (d.num_dump_positions > 0)
    c.dump_positions.assign(d.dump_positions, d.dump_positions + d.num_dump_positions);
  return c;
}


// GatherMethod restatement (sim.cpp:1117-1206) for external per-unit inputs.
// Arithmetic goes through the compiled reference (gqa_attend); only the
// cache bookkeeping is restated.
struct GatherOracle {
  int units = 0, G = 0, D = 0, groups = 0, gsize = 0;
  std::int64_t budget = 0, pos = 0, moved = 0, eviction_steps = 0;
  std::vector<std::vector<TokenId>> ids;
  std::vector<std::vector<Vec>> keys, values;

  // sim.cpp:1130-1170 for every unit; returns victims (-1 = none).
  void step(bool prefill, const double* q, const double* k, const double* v, double* out, std::int64_t* victims) {
    const double scale = 1.0 / std::sqrt(static_cast<double>(D));
    bool evicted = false;
    for (int l = 0; l < units; ++l) {
      keys[l].push_back(Vec(k + static_cast<std::size_t>(l) * D, k + static_cast<std::size_t>(l + 1) * D));
      values[l].push_back(Vec(v + static_cast<std::size_t>(l) * D, v + static_cast<std::size_t>(l + 1) * D));
      ids[l].push_back(pos);
      std::vector<const Vec*> kp, vp;
      for (const Vec& x : keys[l]) kp.push_back(&x);
      for (const Vec& x : values[l]) vp.push_back(&x);
      std::vector<Vec> qs(G);
      for (int h = 0; h < G; ++h)
        qs[h].assign(q + (static_cast<std::size_t>(l) * G + h) * D, q + (static_cast<std::size_t>(l) * G + h + 1) * D);
      AttentionRow avg;
      avg.scores.assign(kp.size(), 0.0);
      for (int g = 0; g < groups; ++g) {
        std::span<const Vec> qg(qs.data() + g * gsize, gsize);
        AttendResult r = gqa_attend(qg, std::span<const Vec* const>(kp), std::span<const Vec* const>(vp), scale);
        std::copy(r.output.begin(), r.output.end(), out + (static_cast<std::size_t>(l) * groups + g) * D);
        for (std::size_t i = 0; i < avg.scores.size(); ++i) avg.scores[i] += r.row.scores[i];
      }
      for (double& x : avg.scores) x /= static_cast<double>(groups);
      victims[l] = -1;
      if (static_cast<std::int64_t>(ids[l].size()) > budget) {
        std::size_t victim = 0;
        for (std::size_t i = 1; i < avg.scores.size(); ++i)
          if (avg.scores[i] < avg.scores[victim]) victim = i;
        moved += static_cast<std::int64_t>(ids[l].size() - victim - 1);
        ids[l].erase(ids[l].begin() + victim);
        keys[l].erase(keys[l].begin() + victim);
        values[l].erase(values[l].begin() + victim);
        victims[l] = static_cast<std::int64_t>(victim);
        evicted = true;
      }
    }
    if (!prefill && evicted) eviction_steps += 1;
    pos += 1;
  }
};

int error_code_of(const std::exception_ptr& ep, std::string* msg) {
  try {
    std::rethrow_exception(ep);
  } catch (const Error& e) {
    *msg = e.what();
    return e.exit_code();
  } catch (const std::exception& e) {
    *msg = e.what();
    return 1;
  }
  return 1;
}

}  // namespace

struct orc_run {
  orc_desc desc;
  std::vector<std::unique_ptr<SeqOracle>> seqs;
  std::int64_t pos = 0;
  std::string scratch, error;
  json metrics = json::array();
};

extern "C" {

orc_run* orc_create(const orc_desc* desc, char* err, int errlen) {
  try {
    auto run = std::make_unique<orc_run>();
    run->desc = *desc;
    for (int s = 0; s < desc->num_seqs; ++s) {
      SimConfig c = config_for_seq(*desc, s);
      const auto errors = c.validate();
      if (!errors.empty()) throw Error(ErrorKind::kConfig, "invalid oracle config: " + errors.front());
      run->seqs.push_back(std::make_unique<SeqOracle>(c));
    }
    return run.release();
  } catch (const std::exception& e) {
    if (err && errlen > 0) std::snprintf(err, errlen, "%s", e.what());
    return nullptr;
  }
}

void orc_destroy(orc_run* run) { delete run; }
int64_t orc_export(orc_run* run, int seq, int unit, uint8_t* buf, int64_t cap) {
  try {
    const auto b = run->seqs.at(seq)->export_unit(unit);
    if (buf && cap >= static_cast<int64_t>(b.size())) std::memcpy(buf, b.data(), b.size());
    return static_cast<int64_t>(b.size());
  } catch (...) {
    return -error_code_of(std::current_exception(), &run->error);
  }
}


int orc_step(orc_run* run, const double* q, const double* k, const double* v, double* out,
             double* sparsity) {
  const orc_desc& d = run->desc;
  const int U = d.units_per_seq, G = d.num_q_heads, D = d.head_dim;
  const int groups = d.gqa_maxpool ? 1 : G;
  try {
    for (int s = 0; s < d.num_seqs; ++s) {
      StepIn in;
      in.pos = run->pos;
      in.prefill = run->pos < d.prompt_len;
      in.queries.resize(U);
      in.keys.resize(U);
      in.values.resize(U);
      for (int u = 0; u < U; ++u) {
        const std::size_t gu = static_cast<std::size_t>(s) * U + u;
        in.queries[u].resize(G);
        for (int g = 0; g < G; ++g)
          in.queries[u][g].assign(q + (gu * G + g) * D, q + (gu * G + g + 1) * D);
        in.keys[u].assign(k + gu * D, k + (gu + 1) * D);
        in.values[u].assign(v + gu * D, v + (gu + 1) * D);
      }
      std::vector<Vec> outs(U);
      run->seqs[s]->process(in, &outs);
      for (int u = 0; u < U; ++u) {
        const std::size_t gu = static_cast<std::size_t>(s) * U + u;
        if (out) std::copy(outs[u].begin(), outs[u].end(), out + gu * groups * D);
        if (sparsity) sparsity[gu] = run->seqs[s]->sparsity()[u];
      }
    }
    run->pos += 1;
    return 0;
  } catch (...) {
    return error_code_of(std::current_exception(), &run->error);
  }
}

int orc_finish(orc_run* run) {
  try {
    run->metrics = json::array();
    for (auto& s : run->seqs) run->metrics.push_back(s->finish(false));
    return 0;
  } catch (...) {
    return error_code_of(std::current_exception(), &run->error);
  }
}

const char* orc_dump(orc_run* run, int seq, const char* what) {
  const std::string w(what);
  if (w == "error") {
    run->scratch = run->error;
  } else if (w == "tables") {
    run->scratch = run->seqs.at(seq)->tables().dump();
  } else if (w == "segments") {
    run->scratch = run->seqs.at(seq)->segments().dump();
  } else if (w == "frag") {
    run->scratch = run->seqs.at(seq)->frag().dump();
  } else if (w == "events") {
    run->scratch = run->seqs.at(seq)->events();
  } else if (w == "step_dumps") {
    run->scratch = run->seqs.at(seq)->step_dumps().dump();
  } else if (w == "metrics") {
    run->scratch = run->metrics.at(seq).dump();
  } else {
    run->scratch = "";
  }
  return run->scratch.c_str();
}

// ShadowStream restatement (sim.cpp:355-456) feeding SeqOracle, compared
// against the reference's own generation_loop on the same config.
const char* orc_toy_compare(const char* config_json) {
  static thread_local std::string result;
  try {
    const SimConfig cfg = SimConfig::from_json(json::parse(config_json));
    const RunOutput ref = generation_loop(cfg);

    ToyModel model(cfg.model);
    const std::vector<TokenId> prompt = model.sample_prompt(cfg.seed, cfg.prompt_len);
    Rng rng(Rng::mix(cfg.seed, 0xBEEF));
    TokenId next = rng.uniform_int(0, cfg.model.embed_dim - 1);
    const int L = cfg.model.num_layers, groups = cfg.model.num_groups(), gs = cfg.model.gqa_group_size;
    const double scale = 1.0 / std::sqrt(static_cast<double>(cfg.model.head_dim));
    std::vector<std::vector<Vec>> cache_k(L), cache_v(L);
    SeqOracle oracle(cfg);
    const std::int64_t steps = cfg.prompt_len + cfg.max_gen_len;
    for (std::int64_t pos = 0; pos < steps; ++pos) {
      StepIn in;
      in.pos = pos;
      in.prefill = pos < cfg.prompt_len;
      in.has_shadow = true;
      const TokenId tok = in.prefill ? prompt[pos] : next;
      in.queries.resize(L);
      in.keys.resize(L);
      in.values.resize(L);
      in.full_avg_rows.resize(L);
      in.full_outputs.resize(L);
      Vec hidden = model.embed(tok);
      for (int l = 0; l < L; ++l) {
        ToyModel::LayerProjection pr = model.project(l, hidden, pos);
        cache_k[l].push_back(pr.key);
        cache_v[l].push_back(pr.value);
        std::vector<const Vec*> kp, vp;
        for (const Vec& x : cache_k[l]) kp.push_back(&x);
        for (const Vec& x : cache_v[l]) vp.push_back(&x);
        std::vector<Vec> gouts;
        std::vector<AttentionRow> rows;
        for (int g = 0; g < groups; ++g) {
          std::span<const Vec> qs(pr.queries.data() + g * gs, gs);
          AttendResult r = gqa_attend(qs, std::span<const Vec* const>(kp), std::span<const Vec* const>(vp), scale);
          gouts.push_back(std::move(r.output));
          rows.push_back(std::move(r.row));
        }
        AttentionRow avg;
        avg.scores.assign(cache_k[l].size(), 0.0);
        for (const AttentionRow& r : rows)
          for (std::size_t i = 0; i < avg.scores.size(); ++i) avg.scores[i] += r.scores[i];
        for (double& x : avg.scores) x /= static_cast<double>(rows.size());
        in.full_avg_rows[l] = std::move(avg);
        Vec cat;
        for (const Vec& go : gouts) cat.insert(cat.end(), go.begin(), go.end());
        in.full_outputs[l] = cat;
        in.queries[l] = std::move(pr.queries);
        in.keys[l] = cache_k[l].back();
        in.values[l] = cache_v[l].back();
        hidden = model.combine(l, hidden, gouts);
      }
      next = model.readout(hidden);
      oracle.process(in, nullptr);
    }
    json o;
    o["metrics"] = oracle.finish(true);
    o["events"] = oracle.events();
    o["tables"] = oracle.tables();
    o["segments"] = oracle.segments();
    o["step_dumps"] = oracle.step_dumps();
    json r;
    r["metrics"] = ref.metrics.to_json();
    r["events"] = ref.events_jsonl;
    r["tables"] = ref.final_block_tables;
    r["segments"] = ref.final_segments;
    r["step_dumps"] = ref.step_dumps;
    result = json{{"reference", r}, {"oracle", o}}.dump();
  } catch (const std::exception& e) {
    result = json{{"error", e.what()}}.dump();
  }
  return result.c_str();
}

int orc_toy_stream(const char* config_json, double* q, double* k, double* v) {
  try {
    const SimConfig cfg = SimConfig::from_json(json::parse(config_json));
    ToyModel model(cfg.model);
    const std::vector<TokenId> prompt = model.sample_prompt(cfg.seed, cfg.prompt_len);
    Rng rng(Rng::mix(cfg.seed, 0xBEEF));
    TokenId next = rng.uniform_int(0, cfg.model.embed_dim - 1);
    const int L = cfg.model.num_layers, H = cfg.model.num_heads, D = cfg.model.head_dim;
    const int groups = cfg.model.num_groups(), gs = cfg.model.gqa_group_size;
    const double scale = 1.0 / std::sqrt(static_cast<double>(D));
    std::vector<std::vector<Vec>> ck(L), cv(L);
    const std::int64_t steps = cfg.prompt_len + cfg.max_gen_len;
    for (std::int64_t pos = 0; pos < steps; ++pos) {
      const TokenId tok = pos < cfg.prompt_len ? prompt[pos] : next;
      Vec hidden = model.embed(tok);
      for (int l = 0; l < L; ++l) {
        ToyModel::LayerProjection pr = model.project(l, hidden, pos);
        ck[l].push_back(pr.key);
        cv[l].push_back(pr.value);
        for (int h = 0; h < H; ++h)
          std::copy(pr.queries[h].begin(), pr.queries[h].end(), q + ((pos * L + l) * H + h) * D);
        std::copy(pr.key.begin(), pr.key.end(), k + (pos * L + l) * D);
        std::copy(pr.value.begin(), pr.value.end(), v + (pos * L + l) * D);
        std::vector<const Vec*> kp, vp;
        for (const Vec& x : ck[l]) kp.push_back(&x);
        for (const Vec& x : cv[l]) vp.push_back(&x);
        std::vector<Vec> gouts;
        for (int g = 0; g < groups; ++g) {
          std::span<const Vec> qs(pr.queries.data() + g * gs, gs);
          gouts.push_back(gqa_attend(qs, std::span<const Vec* const>(kp), std::span<const Vec* const>(vp), scale).output);
        }
        hidden = model.combine(l, hidden, gouts);
      }
      next = model.readout(hidden);
    }
    return 0;
  } catch (...) {
    return 2;
  }
}


struct orc_gather {
  GatherOracle g;
};

orc_gather* orc_gather_create(int32_t units, int32_t num_q_heads, int32_t gqa_maxpool, int32_t head_dim,
                              int64_t budget) {
  auto* r = new orc_gather();
  r->g.units = units;
  r->g.G = num_q_heads;
  r->g.D = head_dim;
  r->g.gsize = gqa_maxpool ? num_q_heads : 1;
  r->g.groups = num_q_heads / r->g.gsize;
  r->g.budget = budget;
  r->g.ids.resize(units);
  r->g.keys.resize(units);
  r->g.values.resize(units);
  return r;
}

void orc_gather_destroy(orc_gather* g) { delete g; }

int orc_gather_step(orc_gather* g, int32_t prefill, const double* q, const double* k, const double* v, double* out,
                    int64_t* victims) {
  try {
    g->g.step(prefill != 0, q, k, v, out, victims);
    return 0;
  } catch (const Error& e) {
    return e.exit_code();
  } catch (...) {
    return 1;
  }
}

int64_t orc_gather_ids(orc_gather* g, int32_t unit, int64_t* ids, int64_t cap) {
  const auto& v = g->g.ids.at(unit);
  for (int64_t i = 0; i < cap && i < static_cast<int64_t>(v.size()); ++i) ids[i] = v[i];
  return static_cast<int64_t>(v.size());
}

void orc_gather_stats(orc_gather* g, int64_t* moved, int64_t* eviction_steps) {
  *moved = g->g.moved;
  *eviction_steps = g->g.eviction_steps;
}

const char* orc_gather_toy_compare(const char* config_json) {
  static thread_local std::string result;
  try {
    const SimConfig cfg = SimConfig::from_json(json::parse(config_json));
    const RunOutput ref = run_baseline(cfg, "gather_compaction");
    const int L = cfg.model.num_layers, H = cfg.model.num_heads, D = cfg.model.head_dim;
    const std::int64_t steps = cfg.prompt_len + cfg.max_gen_len;
    std::vector<double> q(static_cast<std::size_t>(steps) * L * H * D), k(static_cast<std::size_t>(steps) * L * D),
        v(static_cast<std::size_t>(steps) * L * D);
    if (orc_toy_stream(config_json, q.data(), k.data(), v.data()) != 0) throw std::runtime_error("toy stream failed");
    orc_gather* g = orc_gather_create(L, H, cfg.model.gqa_group_size == H && H > 1 ? 1 : 0, D, cfg.budget);
    if (cfg.model.gqa_group_size != 1 && cfg.model.gqa_group_size != H)
      throw std::runtime_error("gather compare: gqa_group_size must be 1 or num_heads");
    std::vector<double> out(static_cast<std::size_t>(L) * H * D);
    std::vector<int64_t> vict(L);
    for (std::int64_t pos = 0; pos < steps; ++pos)
      orc_gather_step(g, pos < cfg.prompt_len, q.data() + static_cast<std::size_t>(pos) * L * H * D,
                      k.data() + static_cast<std::size_t>(pos) * L * D, v.data() + static_cast<std::size_t>(pos) * L * D,
                      out.data(), vict.data());
    std::int64_t live_gen = 0;
    for (TokenId id : g->g.ids[0])
      if (id >= cfg.prompt_len) ++live_gen;
    json o{{"moved_token_slots", g->g.moved},
           {"eviction_steps", g->g.eviction_steps},
           {"live_tokens_final", static_cast<std::int64_t>(g->g.ids[0].size())},
           {"live_generated_final", live_gen}};
    orc_gather_destroy(g);
    const json rm = ref.metrics.to_json();
    json r{{"moved_token_slots", rm.at("moved_token_slots")},
           {"eviction_steps", rm.at("eviction_steps")},
           {"live_tokens_final", rm.at("live_tokens_final")},
           {"live_generated_final", rm.at("live_generated_final")}};
    result = json{{"reference", r}, {"oracle", o}}.dump();
  } catch (const std::exception& e) {
    result = json{{"error", e.what()}}.dump();
  }
  return result.c_str();
}

void orc_synth_step(const tkv_synth_params* p, int64_t unit0, int32_t units, int32_t G, int32_t d,
                    int64_t step, uint16_t* q, uint16_t* k, uint16_t* v) {
  for (int32_t i = 0; i < units; ++i) {
    const int64_t u = unit0 + i;
    for (int32_t g = 0; g < G; ++g)
      for (int32_t c = 0; c < d; ++c)
        q[(static_cast<std::size_t>(i) * G + g) * d + c] = tkv_synth_q(p, u, step, g, c);
    for (int32_t c = 0; c < d; ++c) {
      k[static_cast<std::size_t>(i) * d + c] = tkv_synth_k(p, u, step, c);
      v[static_cast<std::size_t>(i) * d + c] = tkv_synth_v(p, u, step, c);
    }
  }
}

}  // extern "C"
