// Host control plane + C ABI (include/thinkv_b200.h).
//
// The reference's per-step driver ThinkvMethod (proj/src/sim.cpp:494-958)
// mixes three kinds of work.  Here they are split by where they belong:
//   * schedule arithmetic that depends only on segment *sizes* (refresh
//     boundaries, emission points, transition/overflow victim choice and
//     retention targets -- evictor.cpp:348-433) is identical for every unit of
//     a sequence, because all units share the sequence's thought labels
//     (sim.cpp:717-722) and sizes evolve deterministically
//     (target = min(size, R_level)).  The host runs it once per sequence.
//   * everything that depends on cache *contents* -- codes, scales, slot
//     placement, K-means medoids, soft-eviction masks, block release,
//     attention -- runs on the GPU, one CTA per unit, in stream order.
//   * reporting (events, dumps, metrics) is reconstructed on demand from
//     device state plus the host's op records.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "json.hpp"
#include "../../include/thinkv_b200.h"
#include "synth.h"
#include "tkv_internal.h"
#include "tkv_kernels.h"
#include "tkv_state.h"

using nlohmann::json;

namespace {

thread_local std::string g_last_error;

struct TkvError : std::runtime_error {
  int code;
  TkvError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CUDA_OK(expr)                                                                         \
  do {                                                                                        \
    cudaError_t e_ = (expr);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      throw TkvError(TKV_ERR_UNEXPECTED, std::string("CUDA error: ") + cudaGetErrorString(e_) + \
                                             " at " #expr);                                   \
  } while (0)

int fail(const TkvError& e) {
  g_last_error = e.what();
  return e.code;
}

// Thought taxonomy helpers (proj/src/common.cpp:13-61).
std::string thought_name(int band, int num_thoughts) {
  if (num_thoughts == 3) {
    if (band == 0) return "E";
    if (band == 1) return "R";
    if (band == 2) return "T";
  }
  return "B" + std::to_string(band);
}
int importance(int band, int num_thoughts) {
  if (num_thoughts == 3) return band == 0 ? 1 : (band == 1 ? 2 : 0);
  return num_thoughts - 1 - band;
}
bool is_transition(int band, int num_thoughts) { return num_thoughts >= 3 && band == num_thoughts - 1; }
int prefill_band(int num_thoughts) { return num_thoughts == 3 ? 1 : 0; }
const char* format_name(int fmt) {
  switch (fmt) {
    case TKV_FMT_TERNARY: return "TERNARY2";
    case TKV_FMT_NVFP4: return "NVFP4";
    case TKV_FMT_FP8: return "FP8E4M3";
    default: return "RAW16";
  }
}

struct HSeg {
  int id = 0;
  int band = 0;
  int64_t start = 0;
  int64_t size = 0;
  int level = 0;
  bool open = false;
  int64_t initial = 0;
  int dev = 0;
};

struct EvSeg {
  int seg_id;
  int64_t seg_start;
  int64_t retained;
  std::vector<int64_t> log_offs;  // one per op on this segment in this call
};

struct EventRec {
  int kind = 0;  // 0 emit, 1 evict, 2 refresh
  int64_t step = 0;
  // emit / evict: one JSON line per unit, layers layer0 .. layer0 + nlayers - 1
  int layer0 = 0, nlayers = 1;
  // emit
  int fmt = 0, tokens = 0, pad = 0;
  // evict
  int trigger = 0;  // 0 transition_end, 1 budget_overflow
  bool infeasible = false;
  std::vector<EvSeg> segs;
  int64_t after = 0, evicted = 0;
  // refresh
  int64_t dstep = 0;
  double sparsity = 0.0;
  int band = 0;
  std::vector<int> bands;  // per-layer labels (per_layer_thought, sim.cpp:713-716, :728-730)
};

// Units whose segment sizes evolve together: every unit of a sequence
// (their labels are shared, sim.cpp:717-722), or one unit when labels are
// per layer (per_layer_thought).  The host plans evictions once per group.
struct Group {
  int seq = 0, unit0 = 0, nunits = 0;
  std::vector<HSeg> segs;
  int open = -1;
  int next_seg_id = 0;
  int64_t total = 0;
};

// One reference run (one ThinkvMethod, sim.cpp:494-545): a sequence's units,
// its event log, step counters and dumps.
struct SeqRec {
  int unit0 = 0, nunits = 0;
  int group0 = 0, ngroups = 0;
  std::vector<EventRec> events;
  int64_t eviction_steps = 0, transition_calls = 0, overflow_calls = 0, infeasible_events = 0;
  std::map<std::string, int64_t> gen_by_thought;
  json step_dumps = json::object();
};

// One anneal of one segment of one group (identical across its units).
struct PlanOp {
  int seg_idx;
  int64_t m, K;
};
struct GroupPlan {
  int group;
  int trigger;
  bool infeasible = false;
  std::vector<PlanOp> ops;
};

}  // namespace


struct tkv_run {
  tkv_ctx* ctx = nullptr;
  tkv_run_desc desc{};
  std::vector<int32_t> script;
  std::set<int64_t> dump_at;
  std::vector<int64_t> levels;
  TkvState st{};
  cudaStream_t stream = nullptr;
  std::vector<Group> groups;
  std::vector<SeqRec> seqs;
  int group_units = 1;  // units per planning group (units_per_seq, or 1 per layer)
  int64_t pos = 0;
  int cur_half = 0;
  int buf_len = 0;
  int64_t buf_pos0 = 0;
  int64_t total_steps = 0;
  bool finished = false;
  // device arenas
  uint8_t* d_arena = nullptr;
  size_t arena_cap = 0, arena_used = 0;
  uint8_t* h_pinned[2] = {nullptr, nullptr};
  cudaEvent_t pinned_ev[2]{};
  int phase = 0;
  uint32_t* d_log = nullptr;
  int64_t log_cap = 0, log_used = 0;
  double* d_scratch = nullptr;
  uint8_t* km_scratch = nullptr;   // K-means v2 per-instance scratch (grown on demand)
  int64_t km_scratch_bytes = 0;
  double* km_sums = nullptr;       // per restart-CTA sums rows
  int64_t km_sums_doubles = 0;     // capacity
  double* km_sums_grown = nullptr; // (owned) replacement when a wave needs more row blocks
  int scratch_ctas = 0;
  int64_t scratch_per_cta = 0;
  int max_m = 0;
  TkvFlushCtl* d_ctl = nullptr;
  std::vector<double> last_sparsity;
  double* d_trace = nullptr;  // [max_gen_len][U] sparsity per decode step (record_sparsity_trace)
  int64_t trace_steps = 0;
  std::vector<std::vector<double>> refresh_sparsity;  // per refresh (record mode)
  std::vector<json> metrics;
  // per-kernel timing (tkv_timing_enable / tkv_timing_read)
  struct TimedLaunch {
    int cat;
    cudaEvent_t a, b;
  };
  bool timing = false;
  std::vector<TimedLaunch> timed;
  std::vector<cudaEvent_t> ev_pool;
  double acc_ms[5] = {0, 0, 0, 0, 0};
  int64_t acc_n[5] = {0, 0, 0, 0, 0};
  int64_t launches = 0;
  // host side of the step calls (tkv_timing_t host_ms / host_wait_ms / steps)
  double host_ms = 0.0, host_wait_ms = 0.0;
  int64_t host_steps = 0;
  // device byte accounting (tkv_bytes_accounting)
  bool bytes_on = false;
  unsigned long long* d_bytes_acc = nullptr;   // [U][5] per-unit sums
  unsigned long long* d_bytes_last = nullptr;  // [U][5] counts of the latest accounted launch
  int64_t bytes_launches = 0, bytes_host = 0;  // accounted launches, host-known bytes (buffer, q, out)
  bool bytes_dirty = true;     // pager state changed since the bytes kernel last ran
  int64_t bytes_pending = 0;   // full-step launches on unchanged state since then
  // host-pointer step staging: two slots, copies on their own stream so the
  // transfers of one step overlap the kernels of its neighbours
  void* d_q[2] = {nullptr, nullptr};
  void* d_k[2] = {nullptr, nullptr};
  void* d_v[2] = {nullptr, nullptr};
  float* d_out[2] = {nullptr, nullptr};
  cudaStream_t copy_stream = nullptr;  // uploads
  cudaStream_t d2h_stream = nullptr;   // downloads (separate, so step t's download never delays step t+1's upload)
  cudaEvent_t h2d_done[2]{}, step_done[2]{}, d2h_done[2]{};
  int hslot = 0;
  // layer-by-layer stepping (tkv_step_layer): the open step, next expected layer
  int next_layer = 0;
  int step_layers = 0;
  int64_t open_pos = -1;
  bool open_decode = false, open_refresh = false;
  int open_put_half = 0, open_put_slot = 0;
  // CUDA-graph replay of plain steps (tkv_step_plain / tkv_graph_step_begin):
  // K1 launches recorded under stream capture read {buf_half, nbuf,
  // put_half, put_slot} from d_stepdesc, staged per replayed step through a
  // pinned ring on the caller's stream.
  static constexpr int kDescRing = 64;
  static constexpr int kDescInts = 8;  // K1: buf_half, nbuf, put_half, put_slot; K2: half, pos0
  int32_t* d_stepdesc = nullptr;
  int32_t* h_stepdesc = nullptr;  // pinned [kDescRing][kDescInts]
  TkvFlushCtl* d_ctl_graph = nullptr;  // K2's per-group controls for replayed emission steps
  TkvFlushCtl* h_ctl_ring = nullptr;   // pinned [kDescRing][groups]
  bool replaying = false;              // step_end of a replayed step: host bookkeeping only
  cudaEvent_t desc_ev[kDescRing]{};
  int desc_next = 0;
  int cap_next_layer = 0, cap_layers = 0;
  int cap_kind = 0;            // kind of step being captured (1 plain, 2 emission)
  int64_t cap_launches = 0;    // launches recorded by the capture in progress
  int64_t graph_launches[3] = {0, 0, 0};  // ... by the last completed capture of each kind
  int64_t graph_steps = 0;     // steps advanced by tkv_graph_step_begin
  std::vector<void*> allocations;
};

namespace {

template <typename T>
T* dalloc(tkv_run* r, size_t n, int fill = -2) {
  void* p = nullptr;
  if (n == 0) n = 1;
  CUDA_OK(cudaMalloc(&p, n * sizeof(T)));
  r->allocations.push_back(p);
  if (fill != -2) CUDA_OK(cudaMemsetAsync(p, fill, n * sizeof(T), r->stream));
  return static_cast<T*>(p);
}

int fmt_for_bits(int bits) {
  switch (bits) {
    case 2: return TKV_FMT_TERNARY;
    case 4: return TKV_FMT_NVFP4;
    case 8: return TKV_FMT_FP8;
    case 16: return TKV_FMT_RAW;
  }
  throw TkvError(TKV_ERR_CONFIG, "unsupported precision " + std::to_string(bits) + " bits");
}

int64_t effective_pool(const tkv_run_desc& d) {  // SimConfig::effective_pool_blocks (sim.cpp:65-78)
  if (d.pool_blocks > 0) return d.pool_blocks;
  const int64_t segments = (d.prompt_len + d.max_gen_len + d.tau - 1) / d.tau;
  const int64_t floor = d.num_levels > 0 ? d.levels[d.num_levels - 1] : 1;
  const int64_t closed = std::max<int64_t>(d.budget, segments * floor);
  const int64_t resident = closed + d.tau + d.group_size + d.prompt_len;
  return std::max<int64_t>(1, (2 * resident + d.block_size - 1) / d.block_size);
}

void validate(const tkv_run_desc& d) {
  std::vector<std::string> errs;  // SimConfig::validate (sim.cpp:84-133) + device limits
  if (d.num_seqs < 1 || d.units_per_seq < 1) errs.push_back("num_seqs and units_per_seq must be >= 1");
  if (d.num_q_heads < 1 || d.num_q_heads > TKV_MAX_G) errs.push_back("num_q_heads must lie in [1, 16]");
  if (d.head_dim < 1 || d.head_dim > 256) errs.push_back("head_dim must lie in [1, 256]");
  if (d.num_thoughts < 1 || d.num_thoughts > TKV_MAX_BANDS) errs.push_back("num_thoughts must lie in [1, 8]");
  if (d.tau < 1 || d.tau > 256) errs.push_back("tau must lie in [1, 256]");
  if (d.group_size < 1 || d.group_size > 64) errs.push_back("group_size must lie in [1, 64]");
  if (d.block_size < 1 || d.block_size > 32) errs.push_back("block_size must lie in [1, 32]");
  if (d.max_gen_len < 1) errs.push_back("max_gen_len must be >= 1");
  if (d.prompt_len < 0) errs.push_back("prompt_len must be >= 0");
  if (d.pool_blocks < 0) errs.push_back("pool_blocks must be >= 0");
  if (!(d.threshold_fraction > 0.0) || d.threshold_fraction > 1.0)
    errs.push_back("threshold_fraction must lie in (0, 1]");
  if (d.num_levels < 1 || d.num_levels > 16) {
    errs.push_back("retention schedule must not be empty");
  } else {
    for (int i = 0; i < d.num_levels; ++i) {
      if (d.levels[i] <= 0) errs.push_back("retention levels must be positive");
      if (i > 0 && d.levels[i] >= d.levels[i - 1]) errs.push_back("retention levels must be strictly descending");
    }
    if (errs.empty() && d.budget < d.num_thoughts * d.levels[d.num_levels - 1])
      errs.push_back("budget must be >= num_thoughts * retention floor");
  }
  if (d.scripted) {
    if (d.script_len < 1 || !d.script_bands) errs.push_back("scripted trace has no labels");
    else
      for (int64_t i = 0; i < (int64_t)d.num_seqs * d.script_len; ++i)
        if (d.script_bands[i] < 0 || d.script_bands[i] >= d.num_thoughts) errs.push_back("scripted band out of range");
  } else {
    if (d.num_thresholds != d.num_thoughts - 1) errs.push_back("calibration must carry num_thoughts - 1 thresholds");
    if (d.num_calib_units < 1) errs.push_back("calibration layer subset is empty");
    if (d.num_calib_units > 64) errs.push_back("calibration layer subset holds more than 64 layers");
    for (int i = 0; i < std::min(d.num_calib_units, 64); ++i)
      if (d.calib_units[i] < 0 || d.calib_units[i] >= d.units_per_seq)
        errs.push_back("calibration layer index out of range");
  }
  if (d.input_dtype < 0 || d.input_dtype > 2) errs.push_back("input_dtype must be bf16, f32 or f64");
  if (d.num_dump_positions < 0 || (d.num_dump_positions > 0 && !d.dump_positions))
    errs.push_back("dump positions: negative count or null array");
  if (!errs.empty()) {
    std::string what = "invalid run config:";
    for (const auto& e : errs) what += "\n  - " + e;
    throw TkvError(TKV_ERR_CONFIG, what);
  }
  for (int b = 0; b < d.num_thoughts; ++b) fmt_for_bits(d.psi_bits[b]);
}

// -------------------------------------------------------------------------
// uploads: pinned double buffer (by call phase) -> device arena
// -------------------------------------------------------------------------
void begin_phase(tkv_run* r) {
  r->phase ^= 1;
  if (r->timing) {
    const auto t0 = std::chrono::steady_clock::now();
    CUDA_OK(cudaEventSynchronize(r->pinned_ev[r->phase]));
    r->host_wait_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  } else {
    CUDA_OK(cudaEventSynchronize(r->pinned_ev[r->phase]));
  }
  r->arena_used = 0;
}
// Host time of one public step call, net of the begin_phase wait (timing on).
struct HostClock {
  tkv_run* r;
  double wait0;
  std::chrono::steady_clock::time_point t0;
  explicit HostClock(tkv_run* run) : r(run), wait0(run->host_wait_ms), t0(std::chrono::steady_clock::now()) {}
  ~HostClock() {
    if (!r->timing) return;
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    r->host_ms += ms - (r->host_wait_ms - wait0);
    r->host_steps += 1;
  }
};

void end_phase(tkv_run* r) { CUDA_OK(cudaEventRecord(r->pinned_ev[r->phase], r->stream)); }

template <typename T>
T* upload(tkv_run* r, const T* data, size_t n) {
  const size_t bytes = std::max<size_t>(n * sizeof(T), 1);
  const size_t off = (r->arena_used + 255) & ~size_t(255);
  if (off + bytes > r->arena_cap) throw TkvError(TKV_ERR_UNEXPECTED, "upload arena exhausted");
  std::memcpy(r->h_pinned[r->phase] + off, data, n * sizeof(T));
  CUDA_OK(cudaMemcpyAsync(r->d_arena + off, r->h_pinned[r->phase] + off, bytes, cudaMemcpyHostToDevice, r->stream));
  r->arena_used = off + bytes;
  return reinterpret_cast<T*>(r->d_arena + off);
}

void check_launch(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw TkvError(TKV_ERR_UNEXPECTED, std::string(what) + ": " + cudaGetErrorString(e));
}

enum { CAT_ATTEND = 0, CAT_SCORE = 1, CAT_FLUSH = 2, CAT_ANNEAL = 3, CAT_APPLY = 4 };

cudaEvent_t pool_event(tkv_run* r) {
  if (!r->ev_pool.empty()) {
    cudaEvent_t e = r->ev_pool.back();
    r->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  CUDA_OK(cudaEventCreate(&e));
  return e;
}

void drain_timing(tkv_run* r) {
  CUDA_OK(cudaStreamSynchronize(r->stream));
  for (auto& t : r->timed) {
    float ms = 0.f;
    CUDA_OK(cudaEventElapsedTime(&ms, t.a, t.b));
    r->acc_ms[t.cat] += ms;
    r->acc_n[t.cat] += 1;
    r->ev_pool.push_back(t.a);
    r->ev_pool.push_back(t.b);
  }
  r->timed.clear();
}

// Every kernel launch of the run goes through here (launch count + optional
// CUDA-event timing on the run's stream).
template <typename F>
void launch(tkv_run* r, int cat, const char* what, F&& fn) {
  r->launches += 1;
  if (cat != CAT_ATTEND && cat != CAT_SCORE) r->bytes_dirty = true;  // block table / windows may change
  if (!r->timing) {
    check_launch(fn(), what);
    return;
  }
  if (r->timed.size() >= 4096) drain_timing(r);
  cudaEvent_t a = pool_event(r), b = pool_event(r);
  CUDA_OK(cudaEventRecord(a, r->stream));
  check_launch(fn(), what);
  CUDA_OK(cudaEventRecord(b, r->stream));
  r->timed.push_back({cat, a, b});
}

// -------------------------------------------------------------------------
// schedule arithmetic (sizes only): evictor.cpp:348-433
// -------------------------------------------------------------------------
int64_t anneal_size(const tkv_run* r, int level) {
  return level < (int)r->levels.size() ? r->levels[level] : r->levels.back();
}

// anneal_one on sizes: advances the level, returns an op if tokens leave.
void anneal_one(const tkv_run* r, Group& g, int si, GroupPlan& plan) {
  HSeg& s = g.segs[si];
  const int64_t target = std::min(s.size, anneal_size(r, s.level));
  s.level += 1;
  if (target >= s.size) return;
  plan.ops.push_back(PlanOp{si, s.size, target});
  g.total -= s.size - target;
  s.size = target;
}

GroupPlan plan_transition(const tkv_run* r, Group& g, int gi, int64_t closing_start) {
  GroupPlan p{gi, 0, false, {}};
  for (int si = 0; si < (int)g.segs.size(); ++si) {
    const HSeg& s = g.segs[si];
    if (s.open || s.start >= closing_start) continue;
    anneal_one(r, g, si, p);
  }
  return p;
}

GroupPlan plan_overflow(const tkv_run* r, Group& g, int gi) {
  GroupPlan p{gi, 1, false, {}};
  const int64_t floor = r->levels.back();
  const int64_t budget = r->desc.budget;
  const int nt = r->desc.num_thoughts;
  const size_t max_passes = g.segs.size() * (r->levels.size() + 2) + 1;
  for (size_t pass = 0; g.total > budget && pass < max_passes; ++pass) {
    int victim = -1;
    for (int si = 0; si < (int)g.segs.size(); ++si) {
      const HSeg& s = g.segs[si];
      if (s.open || s.size <= floor) continue;
      if (victim < 0) { victim = si; continue; }
      const int rs = importance(s.band, nt), rv = importance(g.segs[victim].band, nt);
      if (rs < rv || (rs == rv && s.start < g.segs[victim].start)) victim = si;
    }
    if (victim < 0) {
      p.infeasible = true;
      break;
    }
    anneal_one(r, g, victim, p);
  }
  return p;
}

// Launch the K-means anneals (in waves: an op that re-anneals a segment
// already annealed in this call waits for the previous wave) and the apply
// kernel, and record the evict events (sim.cpp:652-671).
void execute_plans(tkv_run* r, std::vector<GroupPlan>& plans, int64_t step) {
  const int W = r->st.dm.W;
  std::vector<std::vector<TkvAnnealOp>> waves;
  std::vector<std::vector<std::pair<int, TkvAnnealOp>>> per_group(plans.size());
  for (size_t pi = 0; pi < plans.size(); ++pi) {
    GroupPlan& p = plans[pi];
    Group& g = r->groups[p.group];
    std::map<int, int> seen;
    for (const PlanOp& o : p.ops) {
      const int wave = seen[o.seg_idx]++;
      const HSeg& s = g.segs[o.seg_idx];
      TkvAnnealOp op{};
      op.unit0 = g.unit0;
      op.nunits = g.nunits;
      op.seg = s.dev;
      op.seg_start = (int32_t)s.start;
      op.span = (int32_t)s.initial;
      op.m = (int32_t)o.m;
      op.K = (int32_t)o.K;
      // seed sets (kmeans_cluster, evictor.cpp:266-314): every K-subset when
      // C(m, K) <= 512 (computed exactly as the reference does), else 4
      // farthest-first restarts.
      double subsets = 1.0;
      for (int64_t i = 0; i < o.K; ++i) subsets *= (double)(o.m - i) / (double)(i + 1);
      op.nrestart = subsets <= 512.0 ? 0 : 4;
      op.ncombos = subsets <= 512.0 ? (int32_t)std::llround(subsets) : 0;
      const int64_t need = (int64_t)g.nunits * W;
      if (r->log_used + need > r->log_cap) throw TkvError(TKV_ERR_UNEXPECTED, "eviction log capacity exceeded");
      op.log_off = (int32_t)r->log_used;
      r->log_used += need;
      if ((int)waves.size() <= wave) waves.resize(wave + 1);
      waves[wave].push_back(op);
      per_group[pi].push_back({o.seg_idx, op});
    }
  }
  const TkvDims& dm = r->st.dm;
  bool f64_raw = false, fp8 = false, raw = false;
  for (int b = 0; b < dm.num_bands; ++b) {
    f64_raw = f64_raw || (dm.band_fmt[b] == TKV_FMT_RAW && dm.in_dtype == TKV_IN_F64);
    fp8 = fp8 || dm.band_fmt[b] == TKV_FMT_FP8;
    raw = raw || dm.band_fmt[b] == TKV_FMT_RAW;
  }
  // Ops of one wave are independent; split each wave by instance-size class
  // so small instances get the small (high-occupancy) restart variant
  // instead of inheriting the shared-memory footprint of the largest op.
  std::vector<std::vector<TkvAnnealOp>> subwaves;
  for (auto& wv : waves) {
    std::vector<TkvAnnealOp> cls[5];
    for (const TkvAnnealOp& op : wv)
      cls[op.m <= 8 ? 0 : op.m <= 16 ? 1 : op.m <= 32 ? 2 : op.m <= 64 ? 3 : 4].push_back(op);
    for (auto& c : cls)
      if (!c.empty()) subwaves.push_back(std::move(c));
  }
  for (auto& wv : subwaves) {
    std::vector<int32_t> prefix(wv.size()), rprefix(wv.size());
    int32_t items = 0, runs = 0;
    int mmax = 1, kmax = 1, R = 1;
    for (size_t i = 0; i < wv.size(); ++i) {
      prefix[i] = items;
      rprefix[i] = runs;
      const int nr = wv[i].nrestart > 0 ? wv[i].nrestart : wv[i].ncombos;
      items += wv[i].nunits;
      runs += wv[i].nunits * nr;
      mmax = std::max(mmax, (int)wv[i].m);
      kmax = std::max(kmax, (int)wv[i].K);
      R = std::max(R, nr);
    }
    TkvAnnealOp* d_ops = upload(r, wv.data(), wv.size());
    int32_t* d_pre = upload(r, prefix.data(), prefix.size());
    if (f64_raw) {  // raw fp64 keys are not representable in the v2 key store
      launch(r, CAT_ANNEAL, "anneal kernel", [&] {
        return tkv_launch_anneal(r->st, d_ops, (int)wv.size(), d_pre, items, r->d_log, r->d_scratch,
                                 r->scratch_ctas, r->scratch_per_cta, r->max_m, r->stream);
      });
      continue;
    }
    int32_t* d_rpre = upload(r, rprefix.data(), rprefix.size());
    const int64_t inst = tkv_km_instance_bytes(mmax, kmax, dm.D, dm.W, R);
    const int64_t want = inst * std::min<int64_t>(items, 16384);
    if (want > r->km_scratch_bytes) {
      CUDA_OK(cudaStreamSynchronize(r->stream));
      if (r->km_scratch) CUDA_OK(cudaFree(r->km_scratch));
      CUDA_OK(cudaMalloc(&r->km_scratch, want));
      r->km_scratch_bytes = want;
    }
    const int per_chunk = (int)std::max<int64_t>(1, r->km_scratch_bytes / inst);
    for (int i0 = 0; i0 < items; i0 += per_chunk) {
      const int cnt = std::min(per_chunk, items - i0);
      // runs of items [i0, i0 + cnt): ops are item-contiguous and runs are
      // (op, unit, restart)-ordered, so they form one contiguous range.
      auto run_of_item = [&](int item) {
        int o = (int)(std::upper_bound(prefix.begin(), prefix.end(), item) - prefix.begin()) - 1;
        const int nr = wv[o].nrestart > 0 ? wv[o].nrestart : wv[o].ncombos;
        return rprefix[o] + (item - prefix[o]) * nr;
      };
      const int run0 = run_of_item(i0);
      const int run1 = i0 + cnt < items ? run_of_item(i0 + cnt) : runs;
      // One restart launch per chunk: the global sums row blocks (one per
      // restart CTA of the m > 32 classes) grow to hold every run, so the
      // wave has a single tail instead of one per sub-launch (<= 16 GB).
      const int64_t block = (int64_t)std::max(1, kmax) * (2 * dm.D + 1);
      if (mmax > 32) {
        const int64_t need = std::min<int64_t>((int64_t)(run1 - run0) * block, (int64_t)2 << 30);
        if (need > r->km_sums_doubles) {
          CUDA_OK(cudaStreamSynchronize(r->stream));
          if (r->km_sums_grown) CUDA_OK(cudaFree(r->km_sums_grown));
          CUDA_OK(cudaMalloc(&r->km_sums_grown, (size_t)need * sizeof(double)));
          r->km_sums = r->km_sums_grown;
          r->km_sums_doubles = need;
        }
      }
      const int gctas = (int)std::max<int64_t>(1, std::min<int64_t>(1 << 30, r->km_sums_doubles / block));
      launch(r, CAT_ANNEAL, "kmeans kernels", [&] {
        return tkv_launch_kmeans(r->st, d_ops, (int)wv.size(), d_pre, items, d_rpre, runs, i0, cnt, run0,
                                 run1 - run0, mmax, kmax, R, r->km_scratch, r->km_sums, gctas, r->d_log,
                                 fp8 ? 1 : 0, raw ? 0 : 1, r->stream);
      });
    }
  }
  std::vector<TkvAnnealOp> aops;
  std::vector<TkvApplyGroup> ag;
  std::vector<int32_t> aprefix;
  int32_t aitems = 0;
  for (size_t pi = 0; pi < plans.size(); ++pi) {
    if (per_group[pi].empty()) continue;
    const Group& g = r->groups[plans[pi].group];
    TkvApplyGroup a{g.unit0, g.nunits, (int32_t)aops.size(), 0};
    for (auto& x : per_group[pi]) aops.push_back(x.second);
    a.op_end = (int32_t)aops.size();
    ag.push_back(a);
    aprefix.push_back(aitems);
    aitems += g.nunits;
  }
  if (!ag.empty()) {
    TkvAnnealOp* d_aops = upload(r, aops.data(), aops.size());
    TkvApplyGroup* d_ag = upload(r, ag.data(), ag.size());
    int32_t* d_apre = upload(r, aprefix.data(), aprefix.size());
    launch(r, CAT_APPLY, "apply kernel", [&] {
      return tkv_launch_apply(r->st, d_aops, d_ag, (int)ag.size(), d_apre, aitems, r->d_log, r->stream);
    });
  }
  // events
  for (size_t pi = 0; pi < plans.size(); ++pi) {
    GroupPlan& p = plans[pi];
    Group& g = r->groups[p.group];
    if (p.ops.empty() && !p.infeasible) continue;
    EventRec ev;
    ev.kind = 1;
    ev.step = step;
    ev.trigger = p.trigger;
    ev.infeasible = p.infeasible;
    for (auto& x : per_group[pi]) {
      const HSeg& s = g.segs[x.first];
      auto it = std::find_if(ev.segs.begin(), ev.segs.end(), [&](const EvSeg& e) { return e.seg_id == s.id; });
      if (it == ev.segs.end()) {
        ev.segs.push_back(EvSeg{s.id, s.start, s.size, {}});
        it = ev.segs.end() - 1;
      }
      it->log_offs.push_back(x.second.log_off);
      it->retained = s.size;
      ev.evicted += x.second.m - x.second.K;
    }
    ev.after = g.total;
    ev.layer0 = g.unit0 - r->seqs[g.seq].unit0;
    ev.nlayers = g.nunits;
    if (r->desc.record_events) r->seqs[g.seq].events.push_back(std::move(ev));
  }
}

// -------------------------------------------------------------------------
// emission (flush_layer, sim.cpp:565-650) for every unit
// -------------------------------------------------------------------------
void flush_ctl(const tkv_run* r, TkvFlushCtl* ctl) {
  for (size_t gi = 0; gi < r->groups.size(); ++gi) {
    const Group& g = r->groups[gi];
    const HSeg& s = g.segs[g.open];
    ctl[gi].band = s.band;
    ctl[gi].seg_start = (int32_t)s.start;
  }
}

void flush_all(tkv_run* r, int64_t step) {
  if (r->buf_len <= 0) return;
  if (!r->replaying) {  // (a replayed emission step's K2 is in the graph)
    std::vector<TkvFlushCtl> ctl(r->groups.size());
    flush_ctl(r, ctl.data());
    TkvFlushCtl* d_ctl = upload(r, ctl.data(), ctl.size());
    launch(r, CAT_FLUSH, "flush kernel", [&] {
      return tkv_launch_flush(r->st, r->cur_half, r->buf_len, (int)r->buf_pos0, d_ctl, r->group_units, r->stream);
    });
  }
  if (r->desc.record_events) {
    for (size_t gi = 0; gi < r->groups.size(); ++gi) {
      Group& g = r->groups[gi];
      EventRec ev;
      ev.kind = 0;
      ev.step = step;
      ev.fmt = r->st.dm.band_fmt[g.segs[g.open].band];
      ev.tokens = r->buf_len;
      ev.pad = r->desc.group_size - r->buf_len;
      ev.layer0 = g.unit0 - r->seqs[g.seq].unit0;
      ev.nlayers = g.nunits;
      r->seqs[g.seq].events.push_back(ev);
    }
  }
  r->cur_half ^= 1;
  r->buf_len = 0;
}

std::vector<double> download_sparsity(tkv_run* r) {
  std::vector<double> sp(r->st.dm.U);
  CUDA_OK(cudaMemcpyAsync(sp.data(), r->st.sparsity, sp.size() * sizeof(double), cudaMemcpyDeviceToHost, r->stream));
  CUDA_OK(cudaStreamSynchronize(r->stream));
  return sp;
}

// boundary (sim.cpp:673-746)
void boundary(tkv_run* r, int64_t pos, bool decode) {
  const tkv_run_desc& d = r->desc;
  flush_all(r, pos);
  std::vector<GroupPlan> plans;
  std::vector<char> fired(r->seqs.size(), 0);
  for (size_t gi = 0; gi < r->groups.size(); ++gi) {
    Group& g = r->groups[gi];
    if (g.open < 0) continue;
    HSeg& open = g.segs[g.open];
    open.open = false;
    if (decode && is_transition(open.band, d.num_thoughts)) {
      const int64_t closing = open.start;
      plans.push_back(plan_transition(r, g, (int)gi, closing));
      bool pred = false;
      for (const HSeg& s : g.segs) pred = pred || s.start < closing;
      fired[g.seq] |= pred;
    }
    g.open = -1;
  }
  if (!plans.empty()) execute_plans(r, plans, pos);
  for (size_t si = 0; si < r->seqs.size(); ++si) {
    if (!fired[si]) continue;
    r->seqs[si].transition_calls += 1;
    r->seqs[si].eviction_steps += 1;
  }
  // labels for the next interval: one per sequence (scripted, or classify of
  // the mean over the calibrated layers), or one per layer (per_layer_thought)
  const bool per_layer = d.per_layer_thought && !d.scripted;
  std::vector<double> sp;
  const bool need_sp = decode && (!d.scripted || d.record_events);
  if (need_sp) sp = download_sparsity(r);
  for (size_t si = 0; si < r->seqs.size(); ++si) {
    SeqRec& q = r->seqs[si];
    std::vector<int> bands(q.ngroups, prefill_band(d.num_thoughts));
    double mean = 0.0;
    if (decode) {
      const int64_t dstep = pos - d.prompt_len;
      const int64_t interval = dstep / d.tau;
      auto classify = [&](double x) {  // thought.cpp:353-359
        int band = 0;
        for (int i = 0; i < d.num_thresholds; ++i)
          if (x > d.thresholds[i]) ++band;
        return band;
      };
      if (d.scripted) {
        const int64_t i = std::min<int64_t>(interval, d.script_len - 1);
        std::fill(bands.begin(), bands.end(), r->script[(size_t)si * d.script_len + i]);
        if (need_sp) {
          for (int u = 0; u < q.nunits; ++u) mean += sp[(size_t)q.unit0 + u];
          mean /= (double)q.nunits;
        }
      } else if (per_layer) {
        for (int gi = 0; gi < q.ngroups; ++gi) bands[gi] = classify(sp[(size_t)r->groups[q.group0 + gi].unit0]);
      } else {
        for (int i = 0; i < d.num_calib_units; ++i) mean += sp[(size_t)q.unit0 + d.calib_units[i]];
        mean /= (double)d.num_calib_units;
        std::fill(bands.begin(), bands.end(), classify(mean));
      }
      if (d.record_events) {
        EventRec ev;
        ev.kind = 2;
        ev.step = pos;
        ev.dstep = dstep;
        ev.sparsity = mean;
        ev.band = bands[0];
        if (per_layer) ev.bands = bands;
        q.events.push_back(ev);
      }
    }
    for (int gi = 0; gi < q.ngroups; ++gi) {
      Group& g = r->groups[q.group0 + gi];
      HSeg s;
      s.id = g.next_seg_id++;
      s.band = bands[gi];
      s.start = pos;
      s.open = true;
      s.dev = (int)g.segs.size();
      if (s.dev >= r->st.dm.NSEG) throw TkvError(TKV_ERR_UNEXPECTED, "segment capacity exceeded");
      g.segs.push_back(s);
      g.open = s.dev;
    }
  }
}

// Case-2 budget enforcement (sim.cpp:819-837 in process, :876-883 in finish).
void overflow_pass(tkv_run* r, int64_t step, bool decode, bool final_pass) {
  std::vector<GroupPlan> plans;
  for (size_t gi = 0; gi < r->groups.size(); ++gi) {
    Group& g = r->groups[gi];
    if (g.total <= r->desc.budget) continue;
    plans.push_back(plan_overflow(r, g, (int)gi));
  }
  if (plans.empty()) return;
  execute_plans(r, plans, step);
  std::vector<char> any(r->seqs.size(), 0), infeasible(r->seqs.size(), 0);
  for (const GroupPlan& p : plans) {
    const Group& g = r->groups[p.group];
    any[g.seq] = 1;
    if (!p.infeasible) continue;
    infeasible[g.seq] = 1;
    // finish() counts one infeasible event per layer whose final plan is
    // infeasible (sim.cpp:879); process() one per step (:835-837)
    if (final_pass) r->seqs[g.seq].infeasible_events += g.nunits;
  }
  for (size_t si = 0; si < r->seqs.size(); ++si) {
    if (!any[si]) continue;
    SeqRec& q = r->seqs[si];
    q.overflow_calls += 1;
    if (final_pass) continue;
    if (decode) q.eviction_steps += 1;
    if (infeasible[si]) q.infeasible_events += 1;
  }
}

// -------------------------------------------------------------------------
// dumps (device -> host) in the reference's JSON shapes
// -------------------------------------------------------------------------
struct UnitSnap {
  std::vector<int8_t> th;
  std::vector<uint8_t> fl, ns;
  std::vector<uint32_t> ev, smask, segm;
  std::vector<int32_t> start, sid, swin, wrefs;
};

template <typename T>
void d2h(tkv_run* r, std::vector<T>& v, const T* src, size_t n) {
  v.resize(n);
  CUDA_OK(cudaMemcpyAsync(v.data(), src, n * sizeof(T), cudaMemcpyDeviceToHost, r->stream));
}

std::vector<UnitSnap> snapshot(tkv_run* r, int u0, int n) {
  const TkvDims& dm = r->st.dm;
  std::vector<UnitSnap> out(n);
  for (int i = 0; i < n; ++i) {
    const int64_t u = u0 + i;
    UnitSnap& s = out[i];
    d2h(r, s.th, r->st.blk_thought + u * dm.P, dm.P);
    d2h(r, s.fl, r->st.blk_filled + u * dm.P, dm.P);
    d2h(r, s.ns, r->st.blk_nstart + u * dm.P, dm.P);
    d2h(r, s.ev, r->st.blk_evict + u * dm.P, dm.P);
    d2h(r, s.smask, r->st.blk_segmask + u * dm.P * TKV_MASKS_PER_BLOCK(dm.bs), (size_t)dm.P * TKV_MASKS_PER_BLOCK(dm.bs));
    d2h(r, s.start, r->st.blk_start + u * dm.P * TKV_STARTS_PER_BLOCK(dm.bs), (size_t)dm.P * TKV_STARTS_PER_BLOCK(dm.bs));
    d2h(r, s.sid, r->st.slot_id + u * dm.NS, dm.NS);
    d2h(r, s.swin, r->st.slot_win + u * dm.NS, dm.NS);
    d2h(r, s.wrefs, r->st.win_refs + u * dm.NW, dm.NW);
    d2h(r, s.segm, r->st.seg_mask + u * dm.NSEG * dm.W, (size_t)dm.NSEG * dm.W);
  }
  CUDA_OK(cudaStreamSynchronize(r->stream));
  return out;
}

std::string mask_string(uint32_t m, int bs) {
  std::string s(bs, '0');
  for (int i = 0; i < bs; ++i)
    if ((m >> i) & 1u) s[i] = '1';
  return s;
}

json table_json(const tkv_run* r, const UnitSnap& s) {  // BlockPager::dump (pager.cpp:327-362)
  const TkvDims& dm = r->st.dm;
  json j;
  j["block_size"] = dm.bs;
  j["pool_blocks"] = dm.P;
  json blocks = json::array();
  std::vector<int> free_ids;
  for (int b = 0; b < dm.P; ++b) {
    if (s.th[b] < 0) {
      free_ids.push_back(b);
      continue;
    }
    json e;
    e["physical_block"] = b;
    e["filled"] = (int)s.fl[b];
    e["thought"] = (int)s.th[b];
    std::vector<int64_t> starts;
    for (int k = 0; k < s.ns[b]; ++k) starts.push_back(s.start[(size_t)b * TKV_STARTS_PER_BLOCK(dm.bs) + k]);
    e["start_indices"] = starts;
    json masks = json::array();
    for (int k = 0; k + 1 < s.ns[b]; ++k) masks.push_back(mask_string(s.smask[(size_t)b * TKV_MASKS_PER_BLOCK(dm.bs) + k], dm.bs));
    e["segment_masks"] = masks;
    e["eviction_mask"] = mask_string(s.ev[b], dm.bs);
    json toks = json::array();
    for (int sl = 0; sl < dm.bs; ++sl) {
      if (sl < s.fl[b]) toks.push_back((int64_t)s.sid[(size_t)b * dm.bs + sl]);
      else toks.push_back(nullptr);
    }
    e["tokens"] = toks;
    blocks.push_back(std::move(e));
  }
  j["blocks"] = std::move(blocks);
  j["free_blocks"] = free_ids;
  return j;
}

std::vector<int64_t> members_of(const tkv_run* r, const UnitSnap& s, const HSeg& seg) {
  std::vector<int64_t> m;
  if (seg.open) {
    for (int64_t i = 0; i < seg.size; ++i) m.push_back(seg.start + i);
    return m;
  }
  const int W = r->st.dm.W;
  for (int64_t b = 0; b < seg.initial; ++b)
    if ((s.segm[(size_t)seg.dev * W + (b >> 5)] >> (b & 31)) & 1u) m.push_back(seg.start + b);
  return m;
}

json segments_json(const tkv_run* r, const SeqRec& q, const std::vector<UnitSnap>& snaps) {  // sim.cpp:919-937
  json units = json::array();
  for (int gi = 0; gi < q.ngroups; ++gi) {
    const Group& g = r->groups[q.group0 + gi];
    for (int i = 0; i < g.nunits; ++i) {
      const UnitSnap& snap = snaps[g.unit0 - q.unit0 + i];
      json arr = json::array();
      for (const HSeg& s : g.segs) {
        const auto mem = members_of(r, snap, s);
        if ((int64_t)mem.size() != s.size)
          throw TkvError(TKV_ERR_INTEGRITY, "device member mask disagrees with the host segment size");
        arr.push_back(json{{"id", s.id},
                           {"band", s.band},
                           {"thought", thought_name(s.band, r->desc.num_thoughts)},
                           {"start", s.start},
                           {"anneal_level", s.level},
                           {"open", s.open},
                           {"initial_size", s.initial},
                           {"size", s.size},
                           {"members", mem}});
      }
      units.push_back(std::move(arr));
    }
  }
  return units;
}

json tables_json(const tkv_run* r, const std::vector<UnitSnap>& snaps) {
  json arr = json::array();
  for (const auto& s : snaps) arr.push_back(table_json(r, s));
  return arr;
}

void check_device_errors(tkv_run* r) {
  CUDA_OK(cudaStreamSynchronize(r->stream));
  if (r->copy_stream) CUDA_OK(cudaStreamSynchronize(r->copy_stream));
  if (r->d2h_stream) CUDA_OK(cudaStreamSynchronize(r->d2h_stream));
  std::vector<int32_t> err(r->st.dm.U);
  CUDA_OK(cudaMemcpy(err.data(), r->st.err, err.size() * sizeof(int32_t), cudaMemcpyDeviceToHost));
  for (size_t u = 0; u < err.size(); ++u) {
    if (err[u] == 0) continue;
    const char* what = err[u] == TKV_ERR_OOM ? "physical block pool exhausted"
                       : err[u] == TKV_ERR_INTEGRITY ? "integrity failure (unknown token id / bookkeeping)"
                       : err[u] == TKV_ERR_CONFIG ? "structural error (non-finite input element)"
                                                  : "device error";
    throw TkvError(err[u], std::string(what) + " in unit " + std::to_string(u));
  }
}

json events_json_lines(tkv_run* r, const SeqRec& g, std::string* out) {
  // evicted ids come from the device log
  std::vector<uint32_t> log;
  if (r->log_used > 0) {
    log.resize(r->log_used);
    CUDA_OK(cudaMemcpy(log.data(), r->d_log, log.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  }
  const int W = r->st.dm.W;
  std::string s;
  for (const EventRec& e : g.events) {
    if (e.kind == 2) {
      json ev{{"type", "refresh"}, {"step", e.step}, {"dstep", e.dstep}, {"sparsity", e.sparsity}};
      if (e.bands.empty()) ev["band"] = e.band;
      else ev["bands"] = e.bands;
      s += ev.dump() + "\n";
      continue;
    }
    for (int i = 0; i < e.nlayers; ++i) {
      if (e.kind == 0) {
        json ev{{"type", "emit"}, {"step", e.step}, {"layer", e.layer0 + i}, {"format", format_name(e.fmt)},
                {"tokens", e.tokens}, {"pad", e.pad}};
        s += ev.dump() + "\n";
        continue;
      }
      json segs = json::array();
      for (const EvSeg& es : e.segs) {
        std::vector<int64_t> ids;
        for (int64_t off : es.log_offs)
          for (int w = 0; w < W; ++w) {
            uint32_t bits = log[(size_t)off + (size_t)i * W + w];
            while (bits) {
              const int b = __builtin_ctz(bits);
              bits &= bits - 1;
              ids.push_back(es.seg_start + w * 32 + b);
            }
          }
        std::sort(ids.begin(), ids.end());
        segs.push_back(json{{"segment", es.seg_id}, {"retained", es.retained}, {"evicted", ids}});
      }
      json ev{{"type", "evict"},
              {"trigger", e.trigger == 0 ? "transition_end" : "budget_overflow"},
              {"step", e.step},
              {"layer", e.layer0 + i},
              {"segments", segs},
              {"infeasible", e.infeasible},
              {"retained_before", e.after + e.evicted},
              {"retained_total", e.after}};
      s += ev.dump() + "\n";
    }
  }
  *out = s;
  return json();
}

// Metrics (ThinkvMethod::finish, sim.cpp:889-957) from device state.
json metrics_json(tkv_run* r, const SeqRec& g, const std::vector<UnitSnap>& snaps) {
  const TkvDims& dm = r->st.dm;
  const tkv_run_desc& d = r->desc;
  int64_t bits = 0, slots = 0;
  for (const UnitSnap& s : snaps) {
    for (int b = 0; b < dm.P; ++b) {
      if (s.th[b] < 0) continue;
      const int fmt = dm.band_fmt[s.th[b]];
      const int64_t per = (int64_t)(fmt == TKV_FMT_RAW ? 16 : (fmt == TKV_FMT_TERNARY ? 2 : (fmt == TKV_FMT_NVFP4 ? 4 : 8))) * dm.D * 2;
      for (int sl = 0; sl < s.fl[b]; ++sl)
        if (!((s.ev[b] >> sl) & 1u)) { bits += per; slots += 1; }
    }
  }
  int64_t live_prompt = 0, live_gen = 0;
  std::map<std::string, int64_t> live_by;
  const UnitSnap& s0 = snaps[0];
  for (int b = 0; b < dm.P; ++b) {
    if (s0.th[b] < 0) continue;
    for (int sl = 0; sl < s0.fl[b]; ++sl) {
      if ((s0.ev[b] >> sl) & 1u) continue;
      const int64_t id = s0.sid[(size_t)b * dm.bs + sl];
      (id < d.prompt_len ? live_prompt : live_gen) += 1;
      live_by[thought_name(s0.th[b], d.num_thoughts)] += 1;
    }
  }
  const int64_t total = d.prompt_len + d.max_gen_len;
  json m;
  m["method"] = "thinkv";
  m["generated_length"] = d.max_gen_len;
  m["prompt_length"] = d.prompt_len;
  m["live_tokens_final"] = live_prompt + live_gen;
  m["live_prompt_final"] = live_prompt;
  m["live_generated_final"] = live_gen;
  m["live_by_thought"] = live_by;
  m["generated_by_thought"] = g.gen_by_thought;
  const double avg = slots > 0 ? (double)bits / ((double)slots * 2.0 * dm.D) : 16.0;
  m["avg_bits_per_token"] = avg;
  m["a"] = avg / 16.0;
  m["b"] = d.max_gen_len > 0 ? (double)live_gen / (double)d.max_gen_len : 1.0;
  const double denom = (double)g.nunits * (double)total * 2.0 * dm.D * 16.0;
  const double mf = (double)bits / denom;
  m["memory_footprint_fraction"] = mf;
  m["compression_ratio"] = mf > 0.0 ? 1.0 / mf : 0.0;
  m["eviction_call_fraction"] = (double)g.eviction_steps / (double)d.max_gen_len;
  m["recall_at_10_mean"] = 1.0;
  m["attention_output_error_mean"] = 0.0;
  m["recall_at_10"] = json::array();
  m["attention_output_error"] = json::array();
  m["eviction_steps"] = g.eviction_steps;
  m["transition_calls"] = g.transition_calls;
  m["overflow_calls"] = g.overflow_calls;
  m["budget_infeasible_events"] = g.infeasible_events;
  m["moved_token_slots"] = 0;
  return m;
}

// the step (ThinkvMethod::process, sim.cpp:748-843), in three parts so a model
// can run the attention layer by layer (tkv_step_layer):
//   step_begin   phase bookkeeping, refresh/put decisions, live-list bound
//   step_attend  K3a (refresh steps) + K1 for all units or one layer's units
//   step_end     boundary, buffering, emission, Case-2 eviction, dumps
struct StepCtx {
  int64_t pos = 0;
  bool decode = false, refresh = false;
  int put_half = 0, put_slot = 0;
};

StepCtx step_begin(tkv_run* r) {
  const tkv_run_desc& d = r->desc;
  if (r->finished) throw TkvError(TKV_ERR_CONFIG, "run already finished");
  if (r->pos >= r->total_steps) throw TkvError(TKV_ERR_CONFIG, "step beyond prompt_len + max_gen_len");
  begin_phase(r);
  if (!d.record_events) r->log_used = 0;
  StepCtx c;
  c.pos = r->pos;
  c.decode = c.pos >= d.prompt_len;
  const int64_t bstep = c.decode ? c.pos - d.prompt_len : c.pos;
  c.refresh = bstep % d.tau == 0;
  const bool flush_first = c.refresh && r->buf_len > 0;
  c.put_half = flush_first ? (r->cur_half ^ 1) : r->cur_half;
  c.put_slot = flush_first ? 0 : r->buf_len;
  // live pager slots per unit = the sequence's segment members minus its buffered tokens
  int64_t mx = 0;
  for (const Group& g : r->groups) mx = std::max(mx, g.total - (int64_t)r->buf_len);
  r->st.max_live = (int32_t)std::min<int64_t>(mx, r->st.dm.NS);
  return c;
}

// lmap_h > 0: the launch covers layer `layer` only (q/k/v/out hold that layer's
// num_seqs x lmap_h units); lmap_h == 0: every unit.
void step_attend(tkv_run* r, const StepCtx& c, const void* q, const void* k, const void* v, float* out,
                 int lmap_h, int layer) {
  r->st.lmap_h = lmap_h;
  r->st.lmap_ups = r->desc.units_per_seq;
  r->st.lmap_off = layer * lmap_h;
  r->st.lmap_count = r->desc.num_seqs * lmap_h;
  // 1. attention (+ exact sparsity on refresh steps, where it is consumed, or
  //    on every decode step when a sparsity trace is recorded)
  //    scripted labels without an event log read no sparsity (boundary(), the
  //    refresh event's mean), so the score kernel is skipped there.
  const bool trace = c.decode && r->desc.record_sparsity_trace;
  const bool consumed = c.refresh && c.decode && (!r->desc.scripted || r->desc.record_events);
  if (consumed || trace)
    launch(r, CAT_SCORE, "score kernel",
           [&] { return tkv_launch_score(r->st, q, k, r->cur_half, r->buf_len, r->stream); });
  launch(r, CAT_ATTEND, "attend kernel", [&] {
    return tkv_launch_attend(r->st, q, k, v, out, r->cur_half, r->buf_len, c.put_half, c.put_slot, r->stream);
  });
  if (r->bytes_on) {
    // the device counts change only with the pager state (k_bytes.cu): a
    // full-step launch on unchanged state repeats the previous counts
    if (lmap_h == 0 && !r->bytes_dirty) {
      r->bytes_pending += 1;
    } else {
      r->launches += 1;
      if (lmap_h != 0 && r->bytes_pending > 0) {
        r->launches += 1;
        check_launch(tkv_launch_bytes_repeat(r->d_bytes_acc, r->d_bytes_last, r->st.dm.U, r->bytes_pending,
                                             r->stream), "bytes repeat kernel");
        r->bytes_pending = 0;
      }
      check_launch(tkv_launch_bytes(r->st, r->d_bytes_acc, r->d_bytes_last, r->bytes_pending, r->stream),
                   "bytes kernel");
      r->bytes_pending = 0;
      r->bytes_dirty = lmap_h != 0;
    }
    const TkvDims& dm = r->st.dm;
    const int64_t n = tkv_launch_units(r->st);
    const int rows = dm.maxpool ? 1 : dm.G;
    r->bytes_host += n * ((int64_t)(r->buf_len + 1) * 2 * dm.D * dm.in_bytes +
                          (int64_t)dm.G * dm.D * dm.in_bytes + (int64_t)rows * dm.D * 4);
    if (lmap_h == 0 || layer == 0) r->bytes_launches += 1;
  }
  r->st.lmap_h = 0;
}

void trace_sparsity(tkv_run* r, const StepCtx& c) {
  if (!(c.decode && r->desc.record_sparsity_trace)) return;
  const int64_t dstep = c.pos - r->desc.prompt_len;
  CUDA_OK(cudaMemcpyAsync(r->d_trace + dstep * r->st.dm.U, r->st.sparsity, (size_t)r->st.dm.U * sizeof(double),
                          cudaMemcpyDeviceToDevice, r->stream));
  r->trace_steps = dstep + 1;
}

void step_end(tkv_run* r, const StepCtx& c) {
  trace_sparsity(r, c);
  const tkv_run_desc& d = r->desc;
  const int64_t pos = c.pos;
  // 2. refresh boundary
  if (c.refresh) boundary(r, pos, c.decode);
  // 3. buffer the token under the open segment
  if (r->buf_len == 0) r->buf_pos0 = pos;
  r->buf_len += 1;
  for (Group& g : r->groups) {
    HSeg& open = g.segs[g.open];
    open.size += 1;
    open.initial += 1;
    g.total += 1;
  }
  if (c.decode)  // generated_by_thought counts layer 0's label (sim.cpp:809-812)
    for (SeqRec& q : r->seqs) {
      const Group& g0 = r->groups[q.group0];
      q.gen_by_thought[thought_name(g0.segs[g0.open].band, d.num_thoughts)] += 1;
    }
  // 4. emission at g tokens
  if (r->buf_len >= d.group_size) flush_all(r, pos);
  // 5. Case-2 budget enforcement
  overflow_pass(r, pos, c.decode, false);
  end_phase(r);
  if (r->dump_at.count(pos)) {
    check_device_errors(r);
    for (SeqRec& q : r->seqs) {
      const auto snaps = snapshot(r, q.unit0, q.nunits);
      q.step_dumps[std::to_string(pos)] = json{{"block_tables", tables_json(r, snaps)},
                                               {"segments", segments_json(r, q, snaps)}};
    }
  }
  r->pos += 1;
}

void do_step(tkv_run* r, const void* q, const void* k, const void* v, float* out) {
  if (r->next_layer != 0) throw TkvError(TKV_ERR_CONFIG, "a layer-by-layer step is open (tkv_step_layer)");
  const StepCtx c = step_begin(r);
  step_attend(r, c, q, k, v, out, 0, 0);
  step_end(r, c);
}

// ---- CUDA-graph replay of plain and emission steps ------------
// Capturable step kinds: 1 = plain (the only device work is K1, which also
// buffers the incoming token), 2 = emission (K1, then K2 flushing the full
// window).  Neither may hold a refresh boundary, a Case-2 anneal, a dump, a
// sparsity trace or byte accounting; decided with the size arithmetic the
// step itself runs (plan_overflow on a copy of each over-budget group; an
// emission moves tokens from the buffer into the pager without changing
// segment sizes).  0 = step eagerly.
int next_step_kind(const tkv_run* r) {
  const tkv_run_desc& d = r->desc;
  if (r->finished || r->pos >= r->total_steps || r->next_layer != 0) return 0;
  const bool decode = r->pos >= d.prompt_len;
  const int64_t bstep = decode ? r->pos - d.prompt_len : r->pos;
  if (bstep % d.tau == 0 || r->buf_len + 1 > d.group_size) return 0;
  if (r->dump_at.count(r->pos) || (decode && d.record_sparsity_trace) || r->bytes_on) return 0;
  for (const Group& g : r->groups) {
    if (g.open < 0) return 0;
    if (g.total + 1 <= d.budget) continue;
    Group c = g;  // the step buffers one token under the open segment, then enforces the budget
    c.segs[c.open].size += 1;
    c.segs[c.open].initial += 1;
    c.total += 1;
    if (!plan_overflow(r, c, 0).ops.empty()) return 0;
  }
  return r->buf_len + 1 == d.group_size ? 2 : 1;
}

bool capturing(cudaStream_t s) {
  if (!s) return false;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CUDA_OK(cudaStreamIsCapturing(s, &cs));
  return cs == cudaStreamCaptureStatusActive;
}

TkvState replay_state(const tkv_run* r) {
  TkvState st = r->st;
  st.step_dev = r->d_stepdesc;
  st.max_live = st.dm.NS;
  return st;
}

// Record one K1 launch on the capturing stream.  The per-step scalars come
// from d_stepdesc at replay time and the live lists are sized for the whole
// pool, so the one launch is valid for every step it is replayed for.
void capture_attend(tkv_run* r, cudaStream_t s, const void* q, const void* k, const void* v, float* out,
                    int lmap_h, int layer) {
  TkvState st = replay_state(r);
  st.lmap_h = lmap_h;
  st.lmap_ups = r->desc.units_per_seq;
  st.lmap_off = layer * lmap_h;
  st.lmap_count = r->desc.num_seqs * lmap_h;
  check_launch(tkv_launch_attend(st, q, k, v, out, 0, 0, 0, -1, s), "attend kernel (capture)");
  r->cap_launches += 1;
}

void capture_layer(tkv_run* r, cudaStream_t s, int layer, int num_layers, const void* q, const void* k,
                   const void* v, float* out) {
  if (layer != r->cap_next_layer || (layer > 0 && num_layers != r->cap_layers))
    throw TkvError(TKV_ERR_CONFIG, "captured layers of a step must be recorded in order 0 .. num_layers-1");
  if (layer == 0) {
    r->cap_kind = next_step_kind(r);
    if (r->cap_kind == 0)
      throw TkvError(TKV_ERR_CONFIG, "the next step cannot be captured (boundary or eviction): step it eagerly");
    r->cap_layers = num_layers;
    r->cap_launches = 0;
  }
  capture_attend(r, s, q, k, v, out, num_layers ? r->desc.units_per_seq / num_layers : 0, layer);
  if (layer == num_layers - 1 || num_layers == 0) {
    if (r->cap_kind == 2) {  // the emission: K2 over the full window, controls staged per replay
      check_launch(tkv_launch_flush(replay_state(r), 0, r->desc.group_size, 0, r->d_ctl_graph, r->group_units, s),
                   "flush kernel (capture)");
      r->cap_launches += 1;
    }
    r->cap_next_layer = 0;
    r->graph_launches[r->cap_kind] = r->cap_launches;
  } else {
    r->cap_next_layer = layer + 1;
  }
}

// Before each replay of a captured step on `s`: stage this step's scalars
// (and, for an emission, K2's per-group controls), stream-ordered on s after
// the previous replay read them, and advance the run's host state exactly as
// the eager step would.
void graph_step_begin(tkv_run* r, cudaStream_t s) {
  const int kind = next_step_kind(r);
  if (kind == 0)
    throw TkvError(TKV_ERR_CONFIG, "the next step cannot be replayed (boundary or eviction): step it eagerly");
  if (r->graph_launches[kind] == 0)
    throw TkvError(TKV_ERR_CONFIG, kind == 1 ? "no captured plain step (record one under stream capture)"
                                             : "no captured emission step (record one under stream capture)");
  const StepCtx c = step_begin(r);
  const int slot = r->desc_next;
  r->desc_next = (slot + 1) % tkv_run::kDescRing;
  CUDA_OK(cudaEventSynchronize(r->desc_ev[slot]));
  int32_t* h = r->h_stepdesc + tkv_run::kDescInts * slot;
  h[0] = r->cur_half;
  h[1] = r->buf_len;
  h[2] = c.put_half;
  h[3] = c.put_slot;
  h[4] = r->cur_half;                             // K2: the buffer half the window fills
  h[5] = (int)(r->buf_len == 0 ? c.pos : r->buf_pos0);  // K2: position of the window's first token
  // order the replay after the run's own stream (eager steps), then stage
  cudaEvent_t ev = pool_event(r);
  CUDA_OK(cudaEventRecord(ev, r->stream));
  CUDA_OK(cudaStreamWaitEvent(s, ev, 0));
  r->ev_pool.push_back(ev);
  CUDA_OK(cudaMemcpyAsync(r->d_stepdesc, h, tkv_run::kDescInts * sizeof(int32_t), cudaMemcpyHostToDevice, s));
  if (kind == 2) {
    TkvFlushCtl* hc = r->h_ctl_ring + (size_t)slot * r->groups.size();
    flush_ctl(r, hc);
    CUDA_OK(cudaMemcpyAsync(r->d_ctl_graph, hc, r->groups.size() * sizeof(TkvFlushCtl), cudaMemcpyHostToDevice, s));
  }
  CUDA_OK(cudaEventRecord(r->desc_ev[slot], s));
  r->launches += r->graph_launches[kind];
  r->replaying = true;
  try {
    step_end(r, c);
  } catch (...) {
    r->replaying = false;
    throw;
  }
  r->replaying = false;
  r->graph_steps += 1;
}

void do_finish(tkv_run* r) {
  if (r->finished) return;
  begin_phase(r);
  if (!r->desc.record_events) r->log_used = 0;
  const int64_t total = r->desc.prompt_len + r->desc.max_gen_len;
  flush_all(r, total);
  for (Group& g : r->groups)
    if (g.open >= 0) g.segs[g.open].open = false;
  overflow_pass(r, total, true, true);
  end_phase(r);
  check_device_errors(r);
  r->metrics.clear();
  for (SeqRec& q : r->seqs) {
    const auto snaps = snapshot(r, q.unit0, q.nunits);
    r->metrics.push_back(metrics_json(r, q, snaps));
  }
  r->finished = true;
}

void create_run(tkv_ctx* ctx, const tkv_run_desc* desc, tkv_run* r) {
  if (!desc) throw TkvError(TKV_ERR_CONFIG, "null run description");
  validate(*desc);
  if (!ctx) throw TkvError(TKV_ERR_CONFIG, "null context");
  r->ctx = ctx;
  r->desc = *desc;
  const tkv_run_desc& d = r->desc;
  if (d.scripted) r->script.assign(d.script_bands, d.script_bands + (size_t)d.num_seqs * d.script_len);
  r->desc.script_bands = nullptr;
  for (int i = 0; i < d.num_dump_positions; ++i) r->dump_at.insert(d.dump_positions[i]);
  r->desc.dump_positions = nullptr;
  r->levels.assign(d.levels, d.levels + d.num_levels);
  r->total_steps = d.prompt_len + d.max_gen_len;
  CUDA_OK(cudaSetDevice(ctx->device));
  // A blocking stream: ordered with the legacy default stream (what PyTorch
  // uses unless told otherwise); other caller streams are joined with events.
  CUDA_OK(cudaStreamCreate(&r->stream));

  TkvDims dm{};
  dm.U = d.num_seqs * d.units_per_seq;
  dm.G = d.num_q_heads;
  dm.D = d.head_dim;
  dm.maxpool = d.gqa_maxpool ? 1 : 0;
  dm.bs = d.block_size;
  const int64_t P = effective_pool(d);
  if (P > 2048) throw TkvError(TKV_ERR_CONFIG, "pool_blocks > 2048 per unit is not supported");
  dm.P = (int32_t)P;
  dm.NS = dm.P * dm.bs;
  dm.NW = dm.NS + 1;
  dm.g = d.group_size;
  dm.vchunks = (dm.D + dm.g - 1) / dm.g;
  dm.in_dtype = d.input_dtype;
  dm.in_bytes = d.input_dtype == TKV_DTYPE_BF16 ? 2 : (d.input_dtype == TKV_DTYPE_F32 ? 4 : 8);
  int kbytes = 1;
  dm.num_bands = d.num_thoughts;
  for (int b = 0; b < d.num_thoughts; ++b) {
    dm.band_fmt[b] = fmt_for_bits(d.psi_bits[b]);
    const int bytes = dm.band_fmt[b] == TKV_FMT_RAW ? dm.D * dm.in_bytes
                                                   : (dm.D * d.psi_bits[b] + 7) / 8;
    dm.band_bytes[b] = bytes;
    kbytes = std::max(kbytes, bytes);
  }
  dm.kstride = (kbytes + 15) / 16 * 16;
  const int64_t T = r->total_steps;
  if (T > (int64_t)1 << 30) throw TkvError(TKV_ERR_CONFIG, "run too long");
  dm.T = (int32_t)T;
  dm.W = (d.tau + 31) / 32;
  dm.NSEG = (int32_t)((T + d.tau - 1) / d.tau + 2);
  dm.scale = (float)(1.0 / std::sqrt((double)dm.D));
  dm.thr_frac = d.threshold_fraction;
  r->st.dm = dm;
  const size_t U = dm.U;
  TkvState& st = r->st;
  st.blk_thought = dalloc<int8_t>(r, U * dm.P, 0xFF);
  st.blk_filled = dalloc<uint8_t>(r, U * dm.P, 0);
  st.blk_evict = dalloc<uint32_t>(r, U * dm.P, 0);
  st.blk_nstart = dalloc<uint8_t>(r, U * dm.P, 0);
  st.blk_start = dalloc<int32_t>(r, U * dm.P * TKV_STARTS_PER_BLOCK(dm.bs), 0);
  st.blk_segmask = dalloc<uint32_t>(r, U * dm.P * TKV_MASKS_PER_BLOCK(dm.bs), 0);
  st.unit_nfree = dalloc<int32_t>(r, U);
  st.slot_k = dalloc<uint8_t>(r, U * dm.NS * dm.kstride, 0);
  st.slot_v = dalloc<uint8_t>(r, U * dm.NS * dm.kstride, 0);
  st.slot_vs = dalloc<uint8_t>(r, U * dm.NS * dm.vchunks, 0);
  st.slot_win = dalloc<int32_t>(r, U * dm.NS, 0xFF);
  st.slot_id = dalloc<int32_t>(r, U * dm.NS, 0xFF);
  st.win_ks = dalloc<uint8_t>(r, U * dm.NW * dm.D, 0);
  st.win_kf = dalloc<float>(r, U * dm.NW, 0);
  st.win_vf = dalloc<float>(r, U * dm.NW, 0);
  st.win_refs = dalloc<int32_t>(r, U * dm.NW, 0);
  st.win_free = dalloc<int32_t>(r, U * dm.NW);
  st.win_nfree = dalloc<int32_t>(r, U);
  st.seg_mask = dalloc<uint32_t>(r, U * dm.NSEG * dm.W, 0xFF);
  st.buf = dalloc<uint8_t>(r, U * 4 * (size_t)dm.g * dm.D * dm.in_bytes, 0);
  st.sparsity = dalloc<double>(r, U);
  if (desc->record_sparsity_trace)
    r->d_trace = dalloc<double>(r, (size_t)desc->max_gen_len * dm.U, 0);
  st.kstats = nullptr;
  st.max_live = st.dm.NS;
  if (getenv("TKV_KSTATS")) st.kstats = dalloc<unsigned long long>(r, 256, 0);
  st.err = dalloc<int32_t>(r, U);
  r->d_bytes_acc = dalloc<unsigned long long>(r, U * 5, 0);
  r->d_bytes_last = dalloc<unsigned long long>(r, U * 5, 0);
  check_launch(tkv_launch_init(st, r->stream), "init kernel");
  // arenas
  r->arena_cap = 8 << 20;
  r->d_arena = dalloc<uint8_t>(r, r->arena_cap);
  r->d_stepdesc = dalloc<int32_t>(r, tkv_run::kDescInts, 0);
  CUDA_OK(cudaMallocHost(&r->h_stepdesc, sizeof(int32_t) * tkv_run::kDescInts * tkv_run::kDescRing));
  for (int i = 0; i < tkv_run::kDescRing; ++i) CUDA_OK(cudaEventCreateWithFlags(&r->desc_ev[i], cudaEventDisableTiming));
  for (int i = 0; i < 2; ++i) {
    CUDA_OK(cudaMallocHost(&r->h_pinned[i], r->arena_cap));
    CUDA_OK(cudaEventCreateWithFlags(&r->pinned_ev[i], cudaEventDisableTiming));
    CUDA_OK(cudaEventRecord(r->pinned_ev[i], r->stream));
  }
  const int64_t per_step_ops = 64;
  const int64_t ops_bound = d.record_events ? (int64_t)dm.NSEG * (d.num_levels + 1) + 16 : per_step_ops;
  r->log_cap = ops_bound * (int64_t)U * dm.W;
  r->d_log = dalloc<uint32_t>(r, r->log_cap, 0);
  r->max_m = std::max<int>(d.tau, 1);
  bool f64_raw = false;
  for (int b = 0; b < d.num_thoughts; ++b)
    f64_raw = f64_raw || (dm.band_fmt[b] == TKV_FMT_RAW && dm.in_dtype == TKV_IN_F64);
  // v1 anneal scratch only for raw fp64 keys; everything else runs K-means v2.
  r->scratch_per_cta = f64_raw ? (int64_t)6 * r->max_m * dm.D : 1;
  r->scratch_ctas = f64_raw ? (int)std::min<int64_t>(148 * 4, std::max<int64_t>(1, U)) : 1;
  r->d_scratch = dalloc<double>(r, (size_t)r->scratch_ctas * r->scratch_per_cta);
  // K-means scratch sized up front for the largest wave the schedule can
  // produce (every unit annealing a tau-token segment to the first level,
  // 4 restarts each), so no timed step pays a synchronising re-allocation;
  // execute_plans still grows either buffer if a wave exceeds it.
  {
    const int kmax = (int)std::min<int64_t>(std::max(1, r->max_m - 1), d.num_levels > 0 ? d.levels[0] : 1);
    const int64_t items = std::min<int64_t>(U, 16384);
    r->km_sums_doubles = std::max<int64_t>((int64_t)2048 * std::max(1, r->max_m - 1),
                                           4 * items * std::max(1, kmax)) * (2 * dm.D + 1);
    r->km_sums_doubles = std::min<int64_t>(r->km_sums_doubles, (int64_t)2 << 30);
    r->km_sums = dalloc<double>(r, (size_t)r->km_sums_doubles);
    if (r->max_m > 8) {
      r->km_scratch_bytes = tkv_km_instance_bytes(r->max_m, kmax, dm.D, dm.W, 4) * items;
      CUDA_OK(cudaMalloc(&r->km_scratch, (size_t)r->km_scratch_bytes));
    }
  }
  // sequences, and their planning groups: the whole sequence, or one unit
  // per group when labels are per layer (sizes then evolve per layer)
  r->group_units = (d.per_layer_thought && !d.scripted) ? 1 : d.units_per_seq;
  for (int s = 0; s < d.num_seqs; ++s) {
    SeqRec q;
    q.unit0 = s * d.units_per_seq;
    q.nunits = d.units_per_seq;
    q.group0 = (int)r->groups.size();
    q.ngroups = d.units_per_seq / r->group_units;
    for (int i = 0; i < q.ngroups; ++i) {
      Group g;
      g.seq = s;
      g.unit0 = q.unit0 + i * r->group_units;
      g.nunits = r->group_units;
      r->groups.push_back(std::move(g));
    }
    r->seqs.push_back(std::move(q));
  }
  r->d_ctl_graph = dalloc<TkvFlushCtl>(r, r->groups.size());
  CUDA_OK(cudaMallocHost(&r->h_ctl_ring, sizeof(TkvFlushCtl) * r->groups.size() * tkv_run::kDescRing));
  CUDA_OK(cudaStreamSynchronize(r->stream));
}

void destroy_run(tkv_run* r) {
  if (r->stream) cudaStreamSynchronize(r->stream);
  if (r->copy_stream) {
    cudaStreamSynchronize(r->copy_stream);
    cudaStreamSynchronize(r->d2h_stream);
    cudaStreamDestroy(r->copy_stream);
    cudaStreamDestroy(r->d2h_stream);
    for (int i = 0; i < 2; ++i) {
      cudaEventDestroy(r->h2d_done[i]);
      cudaEventDestroy(r->step_done[i]);
      cudaEventDestroy(r->d2h_done[i]);
    }
  }
  for (void* p : r->allocations) cudaFree(p);
  if (r->km_scratch) cudaFree(r->km_scratch);
  if (r->km_sums_grown) cudaFree(r->km_sums_grown);
  if (r->h_stepdesc) {
    for (int i = 0; i < tkv_run::kDescRing; ++i) cudaEventSynchronize(r->desc_ev[i]);
    cudaFreeHost(r->h_stepdesc);
  }
  if (r->h_ctl_ring) cudaFreeHost(r->h_ctl_ring);
  for (int i = 0; i < tkv_run::kDescRing; ++i)
    if (r->desc_ev[i]) cudaEventDestroy(r->desc_ev[i]);
  for (auto& t : r->timed) { cudaEventDestroy(t.a); cudaEventDestroy(t.b); }
  for (auto e : r->ev_pool) cudaEventDestroy(e);
  for (int i = 0; i < 2; ++i) {
    if (r->h_pinned[i]) cudaFreeHost(r->h_pinned[i]);
    if (r->pinned_ev[i]) cudaEventDestroy(r->pinned_ev[i]);
  }
  if (r->stream) cudaStreamDestroy(r->stream);
}

int64_t live_bytes_stats(tkv_run* r, tkv_bytes_t* out) {
  const TkvDims& dm = r->st.dm;
  std::memset(out, 0, sizeof(*out));
  const size_t U = dm.U;
  std::vector<int8_t> th;
  std::vector<uint8_t> fl;
  std::vector<uint32_t> ev;
  std::vector<int32_t> swin;
  d2h(r, th, r->st.blk_thought, U * dm.P);
  d2h(r, fl, r->st.blk_filled, U * dm.P);
  d2h(r, ev, r->st.blk_evict, U * dm.P);
  d2h(r, swin, r->st.slot_win, U * dm.NS);
  CUDA_OK(cudaStreamSynchronize(r->stream));
  std::vector<uint8_t> win_seen;
  for (size_t u = 0; u < U; ++u) {
    win_seen.assign(dm.NW, 0);
    for (int b = 0; b < dm.P; ++b) {
      const int t = th[u * dm.P + b];
      out->meta_bytes += 6;  // thought, filled, evict mask
      if (t < 0) continue;
      const int fmt = dm.band_fmt[t];
      for (int s = 0; s < fl[u * dm.P + b]; ++s) {
        out->resident_slots += 1;
        if ((ev[u * dm.P + b] >> s) & 1u) continue;
        out->live_slots += 1;
        out->live_code_bytes += 2 * (int64_t)dm.band_bytes[t];
        out->meta_bytes += 4;  // slot -> window index (the live list K1 builds is in shared memory)
        if (fmt == TKV_FMT_RAW) continue;
        const int w = swin[u * dm.NS + (size_t)b * dm.bs + s];
        if (fmt == TKV_FMT_FP8) {
          if (w >= 0 && !win_seen[w]) { win_seen[w] = 1; out->live_scale_bytes += 8; }
        } else {
          out->live_scale_bytes += dm.vchunks;  // per-token value-chunk scales
          if (w >= 0 && !win_seen[w]) { win_seen[w] = 1; out->live_scale_bytes += dm.D; }
        }
      }
    }
  }
  out->buffer_bytes = (int64_t)U * (r->buf_len + 1) * 2 * dm.D * dm.in_bytes;
  const int rows = dm.maxpool ? 1 : dm.G;
  out->qo_bytes = (int64_t)U * ((int64_t)dm.G * dm.D * dm.in_bytes + (int64_t)rows * dm.D * 4);
  out->algorithmic_bytes = out->live_code_bytes + out->live_scale_bytes + out->buffer_bytes + out->qo_bytes +
                           out->meta_bytes;
  return 0;
}

}  // namespace

void tkv_internal_set_error(const std::string& msg) { g_last_error = msg; }

extern "C" {

const char* tkv_last_error(void) { return g_last_error.c_str(); }
int tkv_abi_version(void) { return TKV_ABI_VERSION; }

int tkv_init(int device, tkv_ctx** out) {
  try {
    int n = 0;
    CUDA_OK(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) throw TkvError(TKV_ERR_CONFIG, "no such CUDA device");
    cudaDeviceProp prop{};
    CUDA_OK(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) throw TkvError(TKV_ERR_CONFIG, "this build targets sm_100a (B200)");
    CUDA_OK(cudaSetDevice(device));
    *out = new tkv_ctx{device};
    return TKV_OK;
  } catch (const TkvError& e) {
    return fail(e);
  }
}

int tkv_ctx_destroy(tkv_ctx* ctx) {
  delete ctx;
  return TKV_OK;
}

int tkv_run_create(tkv_ctx* ctx, const tkv_run_desc* desc, tkv_run** out) {
  auto r = std::make_unique<tkv_run>();
  try {
    create_run(ctx, desc, r.get());
    *out = r.release();
    return TKV_OK;
  } catch (const TkvError& e) {
    destroy_run(r.get());
    return fail(e);
  } catch (const std::exception& e) {
    destroy_run(r.get());
    return fail(TkvError(TKV_ERR_UNEXPECTED, e.what()));
  }
}

int tkv_run_destroy(tkv_run* run) {
  if (!run) return TKV_OK;
  destroy_run(run);
  delete run;
  return TKV_OK;
}

int tkv_step(tkv_run* run, const void* q, const void* k, const void* v, float* out, void* stream) {
  try {
    cudaStream_t user = static_cast<cudaStream_t>(stream);
    if (capturing(user)) {  // record, do not execute (tkv_graph_step_begin replays)
      capture_layer(run, user, 0, 0, q, k, v, out);
      return TKV_OK;
    }
    HostClock hc(run);
    cudaEvent_t ev = nullptr;
    if (user && user != run->stream) {  // order the run's stream after the caller's
      CUDA_OK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      CUDA_OK(cudaEventRecord(ev, user));
      CUDA_OK(cudaStreamWaitEvent(run->stream, ev, 0));
    }
    do_step(run, q, k, v, out);
    if (ev) {
      CUDA_OK(cudaEventRecord(ev, run->stream));
      CUDA_OK(cudaStreamWaitEvent(user, ev, 0));
      CUDA_OK(cudaEventDestroy(ev));
    }
    return TKV_OK;
  } catch (const TkvError& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail(TkvError(TKV_ERR_UNEXPECTED, e.what()));
  }
}

// Host-buffer step: H2D of this step's inputs and D2H of its output run on
// the copy stream through one of two device staging slots; the kernels run
// on the run's stream.  Step t's upload overlaps step t-1's kernels and step
// t-1's download overlaps step t's kernels.
void step_host_async(tkv_run* run, const void* q, const void* k, const void* v, float* out) {
  const TkvDims& dm = run->st.dm;
  const size_t qb = (size_t)dm.U * dm.G * dm.D * dm.in_bytes, kb = (size_t)dm.U * dm.D * dm.in_bytes;
  const size_t ob = (size_t)dm.U * (dm.maxpool ? 1 : dm.G) * dm.D * sizeof(float);
  if (!run->copy_stream) {
    CUDA_OK(cudaStreamCreateWithFlags(&run->copy_stream, cudaStreamNonBlocking));
    CUDA_OK(cudaStreamCreateWithFlags(&run->d2h_stream, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      run->d_q[i] = dalloc<uint8_t>(run, qb);
      run->d_k[i] = dalloc<uint8_t>(run, kb);
      run->d_v[i] = dalloc<uint8_t>(run, kb);
      run->d_out[i] = dalloc<float>(run, ob / sizeof(float));
      CUDA_OK(cudaEventCreateWithFlags(&run->h2d_done[i], cudaEventDisableTiming));
      CUDA_OK(cudaEventCreateWithFlags(&run->step_done[i], cudaEventDisableTiming));
      CUDA_OK(cudaEventCreateWithFlags(&run->d2h_done[i], cudaEventDisableTiming));
      CUDA_OK(cudaEventRecord(run->step_done[i], run->stream));
    }
  }
  const int sl = run->hslot;
  run->hslot ^= 1;
  // the slot's previous step must be done reading its inputs / writing its output
  CUDA_OK(cudaStreamWaitEvent(run->copy_stream, run->step_done[sl], 0));
  CUDA_OK(cudaMemcpyAsync(run->d_q[sl], q, qb, cudaMemcpyHostToDevice, run->copy_stream));
  CUDA_OK(cudaMemcpyAsync(run->d_k[sl], k, kb, cudaMemcpyHostToDevice, run->copy_stream));
  CUDA_OK(cudaMemcpyAsync(run->d_v[sl], v, kb, cudaMemcpyHostToDevice, run->copy_stream));
  CUDA_OK(cudaEventRecord(run->h2d_done[sl], run->copy_stream));
  CUDA_OK(cudaStreamWaitEvent(run->stream, run->h2d_done[sl], 0));
  CUDA_OK(cudaStreamWaitEvent(run->stream, run->d2h_done[sl], 0));  // d_out[sl] drained
  do_step(run, run->d_q[sl], run->d_k[sl], run->d_v[sl], run->d_out[sl]);
  CUDA_OK(cudaEventRecord(run->step_done[sl], run->stream));
  CUDA_OK(cudaStreamWaitEvent(run->d2h_stream, run->step_done[sl], 0));
  CUDA_OK(cudaMemcpyAsync(out, run->d_out[sl], ob, cudaMemcpyDeviceToHost, run->d2h_stream));
  CUDA_OK(cudaEventRecord(run->d2h_done[sl], run->d2h_stream));
}

int tkv_step_layer(tkv_run* run, int layer, int num_layers, const void* q, const void* k, const void* v, float* out,
                   void* stream) {
  try {
    const tkv_run_desc& d = run->desc;
    if (num_layers < 1 || d.units_per_seq % num_layers != 0)
      throw TkvError(TKV_ERR_CONFIG, "num_layers must divide units_per_seq");
    if (capturing(static_cast<cudaStream_t>(stream))) {
      capture_layer(run, static_cast<cudaStream_t>(stream), layer, num_layers, q, k, v, out);
      return TKV_OK;
    }
    HostClock hc(run);
    if (layer != run->next_layer || (layer > 0 && num_layers != run->step_layers))
      throw TkvError(TKV_ERR_CONFIG, "layers of a step must be stepped in order 0 .. num_layers-1");
    cudaStream_t user = static_cast<cudaStream_t>(stream);
    cudaEvent_t ev = nullptr;
    if (user && user != run->stream) {
      CUDA_OK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      CUDA_OK(cudaEventRecord(ev, user));
      CUDA_OK(cudaStreamWaitEvent(run->stream, ev, 0));
    }
    StepCtx c;
    if (layer == 0) {
      c = step_begin(run);
      run->open_pos = c.pos;
      run->open_decode = c.decode;
      run->open_refresh = c.refresh;
      run->open_put_half = c.put_half;
      run->open_put_slot = c.put_slot;
      run->step_layers = num_layers;
    } else {
      c.pos = run->open_pos;
      c.decode = run->open_decode;
      c.refresh = run->open_refresh;
      c.put_half = run->open_put_half;
      c.put_slot = run->open_put_slot;
    }
    step_attend(run, c, q, k, v, out, d.units_per_seq / num_layers, layer);
    if (layer == num_layers - 1) {
      step_end(run, c);
      run->next_layer = 0;
      run->open_pos = -1;
    } else {
      run->next_layer = layer + 1;
    }
    if (ev) {
      CUDA_OK(cudaEventRecord(ev, run->stream));
      CUDA_OK(cudaStreamWaitEvent(user, ev, 0));
      CUDA_OK(cudaEventDestroy(ev));
    }
    return TKV_OK;
  } catch (const TkvError& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail(TkvError(TKV_ERR_UNEXPECTED, e.what()));
  }
}

int tkv_step_host(tkv_run* run, const void* q, const void* k, const void* v, float* out) {
  try {
    step_host_async(run, q, k, v, out);
    CUDA_OK(cudaStreamSynchronize(run->d2h_stream));
    return TKV_OK;
  } catch (const TkvError& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail(TkvError(TKV_ERR_UNEXPECTED, e.what()));
  }
}

int tkv_step_host_async(tkv_run* run, const void* q, const void* k, const void* v, float* out) {
  try {
    HostClock hc(run);
    step_host_async(run, q, k, v, out);
    return TKV_OK;
  } catch (const TkvError& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail(TkvError(TKV_ERR_UNEXPECTED, e.what()));
  }
}

int tkv_step_plain(tkv_run* run) {
  try {
    if (!run) throw TkvError(TKV_ERR_CONFIG, "null run");
    return next_step_kind(run);
  } catch (const TkvError& e) {
    return -fail(e);
  }
}

int tkv_graph_step_begin(tkv_run* run, void* stream) {
  try {
    HostClock hc(run);
    graph_step_begin(run, static_cast<cudaStream_t>(stream));
    return TKV_OK;
  } catch (const TkvError& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail(TkvError(TKV_ERR_UNEXPECTED, e.what()));
  }
}

int tkv_finish(tkv_run* run) {
  try {
    do_finish(run);
    return TKV_OK;
  } catch (const TkvError& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail(TkvError(TKV_ERR_UNEXPECTED, e.what()));
  }
}

int tkv_synchronize(tkv_run* run) {
  try {
    check_device_errors(run);
    return TKV_OK;
  } catch (const TkvError& e) {
    return fail(e);
  }
}

int64_t tkv_position(const tkv_run* run) { return run->pos; }

int tkv_dump_json(tkv_run* run, int seq, const char* what, char* buf, size_t cap, size_t* needed) {
  try {
    if (seq < 0 || seq >= (int)run->seqs.size()) throw TkvError(TKV_ERR_CONFIG, "no such sequence");
    check_device_errors(run);
    const std::string w(what);
    SeqRec& g = run->seqs[seq];
    std::string s;
    if (w == "tables") {
      s = tables_json(run, snapshot(run, g.unit0, g.nunits)).dump();
    } else if (w == "segments") {
      s = segments_json(run, g, snapshot(run, g.unit0, g.nunits)).dump();
    } else if (w == "events") {
      if (!run->desc.record_events) throw TkvError(TKV_ERR_CONFIG, "run was created without record_events");
      events_json_lines(run, g, &s);
    } else if (w == "metrics") {
      if (!run->finished) throw TkvError(TKV_ERR_CONFIG, "metrics are available after tkv_finish");
      s = run->metrics.at(seq).dump();
    } else if (w == "step_dumps") {
      s = g.step_dumps.dump();
    } else if (w == "sparsity_trace") {
      if (!run->desc.record_sparsity_trace)
        throw TkvError(TKV_ERR_CONFIG, "run was created without record_sparsity_trace");
      CUDA_OK(cudaStreamSynchronize(run->stream));
      const int64_t n = run->trace_steps, U = run->st.dm.U;
      std::vector<double> tr((size_t)std::max<int64_t>(n, 1) * U);
      if (n > 0) CUDA_OK(cudaMemcpy(tr.data(), run->d_trace, (size_t)n * U * sizeof(double), cudaMemcpyDeviceToHost));
      json rec = json::object();
      for (int uu = 0; uu < g.nunits; ++uu) {
        std::vector<double> col((size_t)n);
        for (int64_t t = 0; t < n; ++t) col[t] = tr[(size_t)t * U + g.unit0 + uu];
        rec[std::to_string(uu)] = col;
      }
      s = rec.dump() + "\n";
    } else {
      throw TkvError(TKV_ERR_CONFIG, "unknown dump '" + w + "'");
    }
    if (needed) *needed = s.size() + 1;
    if (buf && cap > 0) {
      const size_t n = std::min(cap - 1, s.size());
      std::memcpy(buf, s.data(), n);
      buf[n] = 0;
    }
    return TKV_OK;
  } catch (const TkvError& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail(TkvError(TKV_ERR_UNEXPECTED, e.what()));
  }
}

int tkv_bytes(tkv_run* run, tkv_bytes_t* out) {
  try {
    live_bytes_stats(run, out);
    return TKV_OK;
  } catch (const TkvError& e) {
    return fail(e);
  }
}

int tkv_exp_f64(tkv_ctx* ctx, const double* x, double* y, int64_t n) {
  try {
    if (!ctx || (n > 0 && (!x || !y))) throw TkvError(TKV_ERR_CONFIG, "null argument");
    if (n <= 0) return TKV_OK;
    CUDA_OK(cudaSetDevice(ctx->device));
    double* d = nullptr;
    CUDA_OK(cudaMalloc(&d, 2 * n * sizeof(double)));
    cudaError_t e = cudaMemcpy(d, x, n * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = tkv_launch_exp(d, d + n, n, nullptr);
    if (e == cudaSuccess) e = cudaMemcpy(y, d + n, n * sizeof(double), cudaMemcpyDeviceToHost);
    cudaFree(d);
    CUDA_OK(e);
    return TKV_OK;
  } catch (const TkvError& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail(TkvError(TKV_ERR_UNEXPECTED, e.what()));
  }
}

int tkv_bytes_accounting(tkv_run* run, int enable) {
  try {
    if (!run) throw TkvError(TKV_ERR_CONFIG, "null run");
    CUDA_OK(cudaMemsetAsync(run->d_bytes_acc, 0, (size_t)run->st.dm.U * 5 * sizeof(unsigned long long), run->stream));
    CUDA_OK(cudaMemsetAsync(run->d_bytes_last, 0, (size_t)run->st.dm.U * 5 * sizeof(unsigned long long), run->stream));
    run->bytes_launches = 0;
    run->bytes_host = 0;
    run->bytes_on = enable != 0;
    run->bytes_dirty = true;
    run->bytes_pending = 0;
    return 0;
  } catch (const TkvError& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail(TkvError(TKV_ERR_UNEXPECTED, e.what()));
  }
}

int tkv_bytes_accumulated(tkv_run* run, tkv_bytes_t* sum, int64_t* launches) {
  try {
    if (!run || !sum) throw TkvError(TKV_ERR_CONFIG, "null argument");
    std::vector<unsigned long long> per_unit((size_t)run->st.dm.U * 5), last(per_unit.size());
    CUDA_OK(cudaMemcpyAsync(per_unit.data(), run->d_bytes_acc, per_unit.size() * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, run->stream));
    CUDA_OK(cudaMemcpyAsync(last.data(), run->d_bytes_last, last.size() * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, run->stream));
    CUDA_OK(cudaStreamSynchronize(run->stream));
    unsigned long long acc[5] = {0, 0, 0, 0, 0};
    // + the launches on unchanged state since the bytes kernel last ran
    const unsigned long long rep = (unsigned long long)run->bytes_pending;
    for (size_t i = 0; i < per_unit.size(); ++i) acc[i % 5] += per_unit[i] + last[i] * rep;
    std::memset(sum, 0, sizeof(*sum));
    sum->live_slots = (int64_t)acc[0];
    sum->resident_slots = (int64_t)acc[1];
    sum->live_code_bytes = (int64_t)acc[2];
    sum->live_scale_bytes = (int64_t)acc[3];
    sum->meta_bytes = (int64_t)acc[4];
    const TkvDims& dm = run->st.dm;
    const int rows = dm.maxpool ? 1 : dm.G;
    const int64_t qo = (int64_t)dm.G * dm.D * dm.in_bytes + (int64_t)rows * dm.D * 4;
    // host-known bytes: split back into buffer and q/out parts
    const int64_t unit_launches = run->bytes_launches * (int64_t)dm.U;
    sum->qo_bytes = unit_launches * qo;
    sum->buffer_bytes = run->bytes_host - sum->qo_bytes;
    sum->algorithmic_bytes = sum->live_code_bytes + sum->live_scale_bytes + sum->buffer_bytes + sum->qo_bytes +
                             sum->meta_bytes;
    if (launches) *launches = run->bytes_launches;
    return 0;
  } catch (const TkvError& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail(TkvError(TKV_ERR_UNEXPECTED, e.what()));
  }
}

int tkv_export_cache(tkv_run* run, int64_t unit0, int64_t nunits, void* dst, size_t cap, int64_t* unit_offsets,
                     size_t* needed) {
  int64_t* d_buf = nullptr;
  try {
    check_device_errors(run);
    const int64_t U = run->st.dm.U;
    if (unit0 < 0 || nunits < 0 || unit0 + nunits > U) throw TkvError(TKV_ERR_CONFIG, "unit range out of bounds");
    if (run->open_pos >= 0) throw TkvError(TKV_ERR_CONFIG, "export inside an open layer-by-layer step");
    std::vector<int64_t> offs((size_t)nunits + 1, 0);
    if (nunits > 0) {
      CUDA_OK(cudaMalloc(&d_buf, (size_t)(2 * nunits + 1) * sizeof(int64_t)));
      const int npos = (int)std::min<int64_t>(run->pos, run->st.dm.T);
      launch(run, CAT_APPLY, "export size kernel", [&] {
        return tkv_launch_export(run->st, (int)unit0, (int)nunits, npos, 0, d_buf, nullptr, nullptr, run->stream);
      });
      std::vector<int64_t> sizes((size_t)nunits);
      CUDA_OK(cudaMemcpyAsync(sizes.data(), d_buf, (size_t)nunits * sizeof(int64_t), cudaMemcpyDeviceToHost,
                              run->stream));
      CUDA_OK(cudaStreamSynchronize(run->stream));
      for (int64_t i = 0; i < nunits; ++i) offs[(size_t)i + 1] = offs[(size_t)i] + sizes[(size_t)i];
      if (dst && cap >= (size_t)offs.back()) {
        CUDA_OK(cudaMemcpyAsync(d_buf + nunits, offs.data(), (size_t)(nunits + 1) * sizeof(int64_t),
                                cudaMemcpyHostToDevice, run->stream));
        launch(run, CAT_APPLY, "export write kernel", [&] {
          return tkv_launch_export(run->st, (int)unit0, (int)nunits, npos, 1, nullptr, d_buf + nunits,
                                   static_cast<uint8_t*>(dst), run->stream);
        });
        CUDA_OK(cudaStreamSynchronize(run->stream));
      }
      CUDA_OK(cudaFree(d_buf));
      d_buf = nullptr;
    }
    if (unit_offsets) std::memcpy(unit_offsets, offs.data(), offs.size() * sizeof(int64_t));
    if (needed) *needed = (size_t)offs.back();
    if (dst && cap < (size_t)offs.back()) throw TkvError(TKV_ERR_CONFIG, "export buffer too small");
    return TKV_OK;
  } catch (const TkvError& e) {
    if (d_buf) cudaFree(d_buf);
    return fail(e);
  }
}

int tkv_unit_sparsity(tkv_run* run, double* out, int64_t n) {
  try {
    const auto sp = download_sparsity(run);
    std::memcpy(out, sp.data(), std::min<int64_t>(n, (int64_t)sp.size()) * sizeof(double));
    return TKV_OK;
  } catch (const TkvError& e) {
    return fail(e);
  }
}

int tkv_timing_enable(tkv_run* run, int enable) {
  try {
    if (run->timing) drain_timing(run);
    run->timing = enable != 0;
    for (int i = 0; i < 5; ++i) { run->acc_ms[i] = 0.0; run->acc_n[i] = 0; }
    run->launches = 0;
    run->host_ms = run->host_wait_ms = 0.0;
    run->host_steps = 0;
    return TKV_OK;
  } catch (const TkvError& e) {
    return fail(e);
  }
}

int tkv_timing_read(tkv_run* run, tkv_timing_t* out) {
  try {
    drain_timing(run);
    if (run->st.kstats) {
      unsigned long long k[256];
      CUDA_OK(cudaMemcpy(k, run->st.kstats, sizeof(k), cudaMemcpyDeviceToHost));
      fprintf(stderr, "[kstats] prep=%llu cyc_pd=%llu cyc_prep=%llu\n", k[0], k[1], k[2]);
      static const char* cls[5] = {"m<=8", "m<=16", "m<=32", "m<=64", "m<=128"};
      if (k[32 + 3])
        fprintf(stderr, "[kstats tiny] restarts/warp=%llu cyc_lloyd_phase=%llu refinements=%llu passes=%llu swapscans=%llu "
                "cyc_refine_phase=%llu\n", k[32 + 3], k[32 + 5], k[32 + 8], k[32 + 7], k[32 + 9], k[32 + 11]);
      if (k[32 + 21])
        fprintf(stderr, "[kstats table] cyc_build=%llu restarts=%llu cyc_lloyd=%llu cyc_moves=%llu cyc_swaps=%llu "
                "exact_movement=%llu exact_swaps=%llu\n", k[32 + 20], k[32 + 21], k[32 + 22], k[32 + 23], k[32 + 24],
                k[32 + 25], k[32 + 26]);
      for (int c = 1; c < 5; ++c) {
        const unsigned long long* q = k + 32 + 32 * c;
        if (!q[3]) continue;
        fprintf(stderr, "[kstats %s] restarts=%llu sum_m=%llu lloyd_it=%llu cyc_lloyd=%llu cyc_hinit=%llu passes=%llu "
                "moves=%llu swapscans=%llu cand=%llu ordered_sums=%llu cyc_moves=%llu cyc_swaps=%llu cyc_swapfilter=%llu "
                "cyc_restart=%llu cyc_move_update=%llu cyc_refresh=%llu cyc_lloyd_fill=%llu cyc_lloyd_assign=%llu "
                "cyc_lloyd_update=%llu\n",
                cls[c], q[3], q[14], q[4], q[5], q[6], q[7], q[8], q[9], q[10], q[1], q[11], q[12], q[15], q[13], q[0],
                q[2], q[16], q[17], q[18]);
      }
      CUDA_OK(cudaMemset(run->st.kstats, 0, sizeof(k)));
    }
    out->attend_ms = run->acc_ms[CAT_ATTEND];
    out->score_ms = run->acc_ms[CAT_SCORE];
    out->flush_ms = run->acc_ms[CAT_FLUSH];
    out->anneal_ms = run->acc_ms[CAT_ANNEAL];
    out->apply_ms = run->acc_ms[CAT_APPLY];
    out->attend_launches = run->acc_n[CAT_ATTEND];
    out->score_launches = run->acc_n[CAT_SCORE];
    out->flush_launches = run->acc_n[CAT_FLUSH];
    out->anneal_launches = run->acc_n[CAT_ANNEAL];
    out->apply_launches = run->acc_n[CAT_APPLY];
    out->total_launches = run->launches;
    out->host_ms = run->host_ms;
    out->host_wait_ms = run->host_wait_ms;
    out->steps = run->host_steps;
    return TKV_OK;
  } catch (const TkvError& e) {
    return fail(e);
  }
}

int tkv_synth_inputs(tkv_run* run, uint64_t seed, int64_t unit0, int64_t step, void* q, void* k, void* v,
                     void* stream) {
  try {
    const TkvDims& dm = run->st.dm;
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : run->stream;
    check_launch(tkv_launch_synth(seed, run->desc.units_per_seq, run->desc.tau, 4, unit0, dm.U, dm.G, dm.D, step,
                                  static_cast<uint16_t*>(q), static_cast<uint16_t*>(k), static_cast<uint16_t*>(v), s),
                 "synth kernel");
    return TKV_OK;
  } catch (const TkvError& e) {
    return fail(e);
  }
}

// ---------------------------------------------------------------------------
// gather-compaction comparator (GatherMethod, sim.cpp:1117-1206)
// ---------------------------------------------------------------------------
struct tkv_gather {
  tkv_ctx* ctx = nullptr;
  tkv_gather_desc desc{};
  TkvGatherState st{};
  cudaStream_t stream = nullptr;
  int64_t n = 0;        // rows held by every unit (identical across units)
  int64_t pos = 0;
  int64_t moved = 0, eviction_steps = 0;
  std::vector<int64_t> pending;  // steps whose victims are not yet accounted (decode flag in bit 62)
  int32_t* d_victims_log = nullptr;  // [log_cap][U]
  int64_t log_cap = 0, log_used = 0;
};

namespace {
void gather_drain(tkv_gather* g) {
  CUDA_OK(cudaStreamSynchronize(g->stream));
  if (g->log_used == 0) return;
  const int U = g->st.U;
  std::vector<int32_t> v((size_t)g->log_used * U);
  CUDA_OK(cudaMemcpy(v.data(), g->d_victims_log, v.size() * sizeof(int32_t), cudaMemcpyDeviceToHost));
  for (int64_t s = 0; s < g->log_used; ++s) {
    const int64_t rows = g->pending[s] & ((1ll << 40) - 1);  // rows after the append
    const bool decode = (g->pending[s] >> 62) & 1;
    for (int u = 0; u < U; ++u) g->moved += rows - 1 - v[(size_t)s * U + u];
    if (decode) g->eviction_steps += 1;
  }
  g->log_used = 0;
  g->pending.clear();
}
}  // namespace

int tkv_gather_create(tkv_ctx* ctx, const tkv_gather_desc* d, tkv_gather** out) {
  try {
    if (!ctx || !d || !out) throw TkvError(TKV_ERR_CONFIG, "null argument");
    if (d->num_units < 1 || d->num_q_heads < 1 || d->head_dim < 1 || d->budget < 1)
      throw TkvError(TKV_ERR_CONFIG, "gather: units, heads, head_dim and budget must be positive");
    if (d->input_dtype < 0 || d->input_dtype > 2) throw TkvError(TKV_ERR_CONFIG, "gather: unknown input dtype");
    if (d->num_q_heads > 8 || d->head_dim > 128)
      throw TkvError(TKV_ERR_CONFIG, "gather: supports up to 8 query heads per kv head and head_dim <= 128");
    CUDA_OK(cudaSetDevice(ctx->device));
    auto g = std::make_unique<tkv_gather>();
    g->ctx = ctx;
    g->desc = *d;
    TkvGatherState& st = g->st;
    st.U = d->num_units;
    st.G = d->num_q_heads;
    st.D = d->head_dim;
    st.maxpool = d->gqa_maxpool ? 1 : 0;
    st.budget = d->budget;
    st.cap = (int32_t)(d->budget + 1);
    st.in_dtype = d->input_dtype;
    st.in_bytes = d->input_dtype == TKV_DTYPE_BF16 ? 2 : (d->input_dtype == TKV_DTYPE_F32 ? 4 : 8);
    if (tkv_gather_smem(st, d->exact_scores) > 200 * 1024)
      throw TkvError(TKV_ERR_CONFIG, "gather: budget x heads exceeds shared memory");
    const size_t rows = (size_t)st.U * st.cap;
    CUDA_OK(cudaMalloc(&st.k, rows * st.D * st.in_bytes));
    CUDA_OK(cudaMalloc(&st.v, rows * st.D * st.in_bytes));
    CUDA_OK(cudaMalloc(&st.ids, rows * sizeof(int32_t)));
    CUDA_OK(cudaMalloc(&st.victim, (size_t)st.U * sizeof(int32_t)));
    g->log_cap = 256;
    CUDA_OK(cudaMalloc(&g->d_victims_log, (size_t)g->log_cap * st.U * sizeof(int32_t)));
    CUDA_OK(cudaStreamCreate(&g->stream));
    *out = g.release();
    return TKV_OK;
  } catch (const TkvError& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail(TkvError(TKV_ERR_UNEXPECTED, e.what()));
  }
}

int tkv_gather_destroy(tkv_gather* g) {
  if (!g) return TKV_OK;
  if (g->stream) cudaStreamSynchronize(g->stream);
  cudaFree(g->st.k);
  cudaFree(g->st.v);
  cudaFree(g->st.ids);
  cudaFree(g->st.victim);
  cudaFree(g->d_victims_log);
  if (g->stream) cudaStreamDestroy(g->stream);
  delete g;
  return TKV_OK;
}

int tkv_gather_step(tkv_gather* g, int prefill, const void* q, const void* k, const void* v, float* out,
                    void* stream) {
  try {
    cudaStream_t user = static_cast<cudaStream_t>(stream);
    cudaStream_t s = user ? user : g->stream;
    check_launch(tkv_launch_gather_step(g->st, (int)g->n, g->pos, q, k, v, out, g->desc.exact_scores, s),
                 "gather step kernel");
    const int64_t rows = g->n + 1;
    if (rows > g->st.budget) {  // every unit evicted one row this step
      if (g->log_used == g->log_cap) {
        CUDA_OK(cudaStreamSynchronize(s));
        gather_drain(g);
      }
      CUDA_OK(cudaMemcpyAsync(g->d_victims_log + (size_t)g->log_used * g->st.U, g->st.victim,
                              (size_t)g->st.U * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
      g->pending.push_back(rows | ((int64_t)(prefill ? 0 : 1) << 62));
      g->log_used += 1;
      g->n = rows - 1;
    } else {
      g->n = rows;
    }
    g->pos += 1;
    if (user && user != g->stream) {  // keep later synchronising calls ordered
      cudaEvent_t ev;
      CUDA_OK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      CUDA_OK(cudaEventRecord(ev, user));
      CUDA_OK(cudaStreamWaitEvent(g->stream, ev, 0));
      CUDA_OK(cudaEventDestroy(ev));
    }
    return TKV_OK;
  } catch (const TkvError& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail(TkvError(TKV_ERR_UNEXPECTED, e.what()));
  }
}

int tkv_gather_stats(tkv_gather* g, int64_t* moved, int64_t* eviction_steps) {
  try {
    gather_drain(g);
    if (moved) *moved = g->moved;
    if (eviction_steps) *eviction_steps = g->eviction_steps;
    return TKV_OK;
  } catch (const TkvError& e) {
    return fail(e);
  }
}

int tkv_gather_ids(tkv_gather* g, int unit, int64_t* ids, int64_t cap, int64_t* n) {
  try {
    if (unit < 0 || unit >= g->st.U) throw TkvError(TKV_ERR_CONFIG, "no such unit");
    CUDA_OK(cudaStreamSynchronize(g->stream));
    std::vector<int32_t> v(g->n);
    if (g->n > 0)
      CUDA_OK(cudaMemcpy(v.data(), g->st.ids + (size_t)unit * g->st.cap, v.size() * sizeof(int32_t),
                         cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < cap && i < g->n; ++i) ids[i] = v[i];
    if (n) *n = g->n;
    return TKV_OK;
  } catch (const TkvError& e) {
    return fail(e);
  }
}

}  // extern "C"
