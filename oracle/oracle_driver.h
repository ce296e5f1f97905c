// Oracle driver C API (TEST INFRASTRUCTURE ONLY -- never linked by the product).
//
// The oracle restates the reference's private per-step driver
// `ThinkvMethod` (/root/reference/proj/src/sim.cpp:494-958) so it accepts
// externally supplied per-unit q/k/v instead of the ToyModel stream, and
// performs every arithmetic operation by calling the compiled, unmodified
// reference library (quantize_window, BlockPager, on_transition_end,
// on_budget_overflow, kmeans_select, gqa_attend, layer_sparsity_average,
// classify, refresh_due).  Units are the reference's "layers": one sequence
// with N units is one ThinkvMethod whose model has num_layers = N.
#pragma once
#include <stdint.h>

#include "../paper_2510_01290_b200/csrc/synth.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_desc {
  int32_t num_seqs;
  int32_t units_per_seq;   // reference num_layers per sequence
  int32_t num_q_heads;     // G query heads sharing a unit's single KV head
  int32_t gqa_maxpool;     // 1: gqa_group_size = G (paper GQA max-pool); 0: per-head rows
  int32_t head_dim;
  int32_t tau;
  int32_t group_size;
  int32_t block_size;
  int32_t pool_blocks;     // 0 = SimConfig::effective_pool_blocks()
  int64_t budget;
  int32_t num_levels;
  int64_t levels[16];
  int32_t psi_bits[8];     // bits per band (2/4/8/16)
  int32_t num_thoughts;
  double threshold_fraction;
  int64_t prompt_len;
  int64_t max_gen_len;
  int32_t scripted;        // 1: scripted labels from script_bands
  int32_t script_len;      // intervals per sequence in script_bands
  const int32_t* script_bands;  // [num_seqs][script_len]
  int32_t per_layer_thought;
  int32_t num_thresholds;
  double thresholds[8];
  int32_t num_calib_units;
  int32_t calib_units[64];
  int32_t num_dump_positions;
  const int64_t* dump_positions;
} orc_desc;

typedef struct orc_run orc_run;

// Returns NULL and writes a message into err on invalid configuration.
orc_run* orc_create(const orc_desc* desc, char* err, int errlen);
void orc_destroy(orc_run* run);

// One step for all sequences.  q: [units][G][d], k/v: [units][d] (row-major,
// doubles).  out: [units][groups][d] where groups = G (per-head) or 1
// (max-pool).  sparsity (optional): [units] layer_sparsity_average values.
// Returns 0 or the reference Error::exit_code() (errors.hpp:31-46).
int orc_step(orc_run* run, const double* q, const double* k, const double* v,
             double* out, double* sparsity);
int orc_finish(orc_run* run);

// JSON views (string owned by the run, valid until the next orc_dump call).
// what: "tables" | "segments" | "events" | "metrics" | "step_dumps" | "error"
const char* orc_dump(orc_run* run, int seq, const char* what);

// Compressed-cache export of one unit (layout: paper_2510_01290_b200/csrc/
// k_export.cu) built from BlockPager::read_active / group_table and
// thinkv::serialize_group.  Returns the byte count (copies when cap
// suffices) or -(error code).
int64_t orc_export(orc_run* run, int seq, int unit, uint8_t* buf, int64_t cap);

// Runs thinkv::generation_loop(config_json) and the oracle restatement fed by
// a ShadowStream restatement (sim.cpp:355-456) on the same config; returns
// {"reference": {...}, "oracle": {...}} with metrics/events/tables/segments/
// step_dumps for each.  Used to pin the restatement (tests/test_oracle.py).
const char* orc_toy_compare(const char* config_json);

// The ToyModel input stream of a SimConfig (ShadowStream restatement,
// sim.cpp:383-447): q [steps][layers][heads][d], k/v [steps][layers][d].
// Arrays must be sized by the caller (see oracle.py toy_stream).
int orc_toy_stream(const char* config_json, double* q, double* k, double* v);

// ---- gather-compaction comparator (GatherMethod, sim.cpp:1117-1206) -------
// Restated for external q/k/v per unit (one unit = one reference layer).
// Every step: append the token, gqa_attend per group, head-averaged scores;
// over budget: evict the first minimum and shift later tokens down.
typedef struct orc_gather orc_gather;
orc_gather* orc_gather_create(int32_t units, int32_t num_q_heads, int32_t gqa_maxpool, int32_t head_dim,
                              int64_t budget);
void orc_gather_destroy(orc_gather* g);
// out: [units][groups][d]; victims: [units] evicted index (-1: none).
int orc_gather_step(orc_gather* g, int32_t prefill, const double* q, const double* k, const double* v,
                    double* out, int64_t* victims);
// Token ids (step positions) kept by a unit, in cache order; returns the count.
int64_t orc_gather_ids(orc_gather* g, int32_t unit, int64_t* ids, int64_t cap);
void orc_gather_stats(orc_gather* g, int64_t* moved, int64_t* eviction_steps);
// thinkv::run_baseline(config, "gather_compaction") vs the restatement fed
// the ToyModel stream: {"reference": metrics, "oracle": metrics}.
const char* orc_gather_toy_compare(const char* config_json);

// Synthetic bf16 inputs for `units` units starting at unit index unit0.
void orc_synth_step(const tkv_synth_params* p, int64_t unit0, int32_t units,
                    int32_t G, int32_t d, int64_t step, uint16_t* q,
                    uint16_t* k, uint16_t* v);

#ifdef __cplusplus
}
#endif
