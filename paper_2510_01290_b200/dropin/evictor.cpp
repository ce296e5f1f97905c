// thinkv::kmeans_select / on_transition_end / on_budget_overflow
// (proj/include/thinkv/evictor.hpp:83-110) over the device K-means
// (tkv_dropin_kmeans_select: the fp64 medoid selection K3d runs, bit-exact
// with evictor.cpp:55-338).
//
// The triggers are planned the way the device path plans them
// (csrc/tkv_host.cpp): which segment anneals, how often and to what size
// depends only on segment sizes and levels (target = min(size, R_level),
// evictor.cpp:348-367), so the whole sequence of anneals is fixed first and
// the K-means instances then run in waves -- every segment's first anneal in
// one launch, the second anneals (over the first's medoids) in the next --
// instead of one instance at a time.
#include <algorithm>
#include <iterator>
#include <map>
#include <vector>

#include "dropin.hpp"
#include "thinkv/evictor.hpp"

namespace thinkv {

namespace {

struct Instance {
  const std::vector<TokenId>* ids;  // members (ascending) before this anneal
  std::vector<Vec> keys;
  std::int64_t k;
  std::vector<TokenId> medoids;     // result: retained ids, ascending
};

// One launch for every instance (k < m each); fills medoids.
void run_instances(std::vector<Instance*>& insts) {
  if (insts.empty()) return;
  const int d = static_cast<int>(insts.front()->keys.front().size());
  std::vector<int32_t> m, k;
  std::vector<double> keys;
  for (Instance* in : insts) {
    for (const Vec& key : in->keys) {
      if (static_cast<int>(key.size()) != d) throw Error(ErrorKind::kStructural, "kmeans: ragged key vectors");
      keys.insert(keys.end(), key.begin(), key.end());
    }
    m.push_back(static_cast<int32_t>(in->keys.size()));
    k.push_back(static_cast<int32_t>(in->k));
  }
  std::vector<int32_t> med;
  for (int32_t x : k) med.resize(med.size() + x);
  dropin::check(tkv_dropin_kmeans_select(dropin::ctx(), static_cast<int32_t>(insts.size()), d, m.data(), k.data(),
                                         keys.data(), med.data()));
  std::size_t off = 0;
  for (Instance* in : insts) {
    in->medoids.clear();
    for (std::int64_t c = 0; c < in->k; ++c) in->medoids.push_back((*in->ids)[med[off + c]]);
    off += in->k;
    std::sort(in->medoids.begin(), in->medoids.end());
  }
}

// Retention targets of `seg` for its next `times` anneals (levels advance
// each time; a target not below the size evicts nothing), from sizes only.
struct Step {
  SegmentRecord* seg;
  std::int64_t target;  // < size before the anneal, or -1 (no eviction)
};

// Applies the planned anneals: K-means waves, member lists, the plan's
// per-segment entries (merge order: first appearance; evicted ids sorted,
// retained = the final members).
void execute(std::vector<Step>& steps, const KeyLookup& key_of, EvictionPlan& plan) {
  std::map<SegmentRecord*, std::vector<TokenId>> evicted;
  std::vector<SegmentRecord*> order;
  std::map<SegmentRecord*, std::vector<std::int64_t>> chain;  // targets per segment, in anneal order
  for (const Step& s : steps) {
    if (s.target < 0) continue;
    if (!chain.count(s.seg)) order.push_back(s.seg);
    chain[s.seg].push_back(s.target);
  }
  // wave w = the w-th anneal of every segment that has one
  std::map<SegmentRecord*, std::vector<Vec>> keys;  // current members' keys
  for (SegmentRecord* seg : order) {
    std::vector<Vec>& ks = keys[seg];
    for (TokenId id : seg->member_ids) ks.push_back(key_of(id));
  }
  for (std::size_t w = 0;; ++w) {
    std::vector<Instance> insts;
    std::vector<SegmentRecord*> who;
    for (SegmentRecord* seg : order)
      if (chain[seg].size() > w) {
        insts.push_back(Instance{&seg->member_ids, keys[seg], chain[seg][w], {}});
        who.push_back(seg);
      }
    if (insts.empty()) break;
    std::vector<Instance*> ptrs;
    for (Instance& in : insts) ptrs.push_back(&in);
    run_instances(ptrs);
    for (std::size_t i = 0; i < insts.size(); ++i) {
      SegmentRecord* seg = who[i];
      std::vector<TokenId> gone;
      std::set_difference(seg->member_ids.begin(), seg->member_ids.end(), insts[i].medoids.begin(),
                          insts[i].medoids.end(), std::back_inserter(gone));
      std::vector<Vec> kept;
      for (std::size_t j = 0, r = 0; j < seg->member_ids.size(); ++j)
        if (r < insts[i].medoids.size() && seg->member_ids[j] == insts[i].medoids[r]) {
          kept.push_back(keys[seg][j]);
          ++r;
        }
      keys[seg] = std::move(kept);
      seg->member_ids = insts[i].medoids;
      std::vector<TokenId>& ev = evicted[seg];
      ev.insert(ev.end(), gone.begin(), gone.end());
    }
  }
  for (SegmentRecord* seg : order) {
    std::vector<TokenId>& ev = evicted[seg];
    if (ev.empty()) continue;
    std::sort(ev.begin(), ev.end());
    plan.segments.push_back(SegmentEviction{seg->id, seg->member_ids, ev});
  }
}

// anneal_one on sizes (evictor.cpp:348-367): the level always advances.
std::int64_t plan_anneal(SegmentRecord& seg, std::int64_t& size, const RetentionSchedule& schedule) {
  const std::int64_t target = std::min(size, schedule.anneal_size(seg.anneal_level));
  seg.anneal_level += 1;
  if (target >= size) return -1;
  size = target;
  return target;
}

}  // namespace

std::vector<TokenId> kmeans_select(std::span<const TokenId> ids, std::span<const Vec> keys, std::int64_t k) {
  if (k >= static_cast<std::int64_t>(ids.size())) return std::vector<TokenId>(ids.begin(), ids.end());
  if (ids.empty() || k < 1) throw Error(ErrorKind::kStructural, "kmeans over an empty input");
  if (keys.size() != ids.size()) throw Error(ErrorKind::kStructural, "kmeans ids/keys size mismatch");
  const std::vector<TokenId> members(ids.begin(), ids.end());
  Instance in{&members, std::vector<Vec>(keys.begin(), keys.end()), k, {}};
  std::vector<Instance*> one{&in};
  run_instances(one);
  return in.medoids;
}

EvictionPlan on_transition_end(std::vector<SegmentRecord>& segments, std::int64_t closing_start_step,
                               const KeyLookup& key_of, const RetentionSchedule& schedule) {
  EvictionPlan plan;
  plan.trigger = TriggerCase::kTransitionEnd;
  std::vector<Step> steps;
  for (SegmentRecord& seg : segments) {
    if (seg.open || seg.start_step >= closing_start_step) continue;
    std::int64_t size = seg.size();
    steps.push_back(Step{&seg, plan_anneal(seg, size, schedule)});
  }
  execute(steps, key_of, plan);
  return plan;
}

EvictionPlan on_budget_overflow(std::vector<SegmentRecord>& segments, std::int64_t budget, const KeyLookup& key_of,
                                const RetentionSchedule& schedule, int num_thoughts) {
  EvictionPlan plan;
  plan.trigger = TriggerCase::kBudgetOverflow;
  const std::int64_t floor = schedule.floor();
  std::vector<std::int64_t> size(segments.size());
  std::int64_t total = 0;
  for (std::size_t i = 0; i < segments.size(); ++i) total += size[i] = segments[i].size();
  std::vector<Step> steps;
  const std::size_t passes = segments.size() * (schedule.levels.size() + 2) + 1;
  for (std::size_t pass = 0; pass < passes && total > budget; ++pass) {
    // victim: least important thought, then earliest start, among closed
    // segments above the floor
    int v = -1;
    for (int i = 0; i < static_cast<int>(segments.size()); ++i) {
      const SegmentRecord& s = segments[i];
      if (s.open || size[i] <= floor) continue;
      if (v < 0) {
        v = i;
        continue;
      }
      const int ri = thought_importance(s.thought, num_thoughts);
      const int rv = thought_importance(segments[v].thought, num_thoughts);
      if (ri < rv || (ri == rv && s.start_step < segments[v].start_step)) v = i;
    }
    if (v < 0) {
      plan.budget_infeasible = true;
      break;
    }
    const std::int64_t before = size[v];
    steps.push_back(Step{&segments[v], plan_anneal(segments[v], size[v], schedule)});
    total -= before - size[v];
  }
  execute(steps, key_of, plan);
  return plan;
}

}  // namespace thinkv
