/* thinkv_b200.h -- C ABI of the B200-native ThinKV decode path.
 *
 * The reference (arxiv 2510.01290 desk simulator, /root/reference/proj) has no
 * FFI: its hot path is the private per-step driver ThinkvMethod
 * (proj/src/sim.cpp:494-958) over the public C++ API in proj/include/thinkv/.
 * This header is the drop-in boundary for that path: plain C types, device or
 * host pointers plus sizes, status codes instead of exceptions.  Each entry
 * point names the reference interface it replaces.
 *
 * Status codes mirror thinkv::Error::exit_code() (proj/include/thinkv/errors.hpp:31-46):
 *   0 ok, 1 unexpected, 2 structural/config/parse, 3 calibration,
 *   4 out-of-memory (block pool exhausted), 5 integrity.
 * The message of the last failure on the calling thread is tkv_last_error().
 *
 * Threading: a run is single-threaded (SPEC.md:426 -- one pager per layer
 * needs external mutual exclusion); distinct runs may be driven from distinct
 * threads.  Device work is asynchronous on the run's stream; device-side
 * failures (e.g. pool exhaustion inside the emission kernel) are sticky per
 * unit and reported by the next synchronising call (tkv_synchronize,
 * tkv_finish, tkv_dump_json).
 */
#ifndef THINKV_B200_H
#define THINKV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TKV_ABI_VERSION 2

enum tkv_status {
  TKV_OK = 0,
  TKV_ERR_UNEXPECTED = 1,
  TKV_ERR_CONFIG = 2,
  TKV_ERR_CALIBRATION = 3,
  TKV_ERR_OOM = 4,
  TKV_ERR_INTEGRITY = 5
};

enum tkv_dtype { TKV_DTYPE_BF16 = 0, TKV_DTYPE_F32 = 1, TKV_DTYPE_F64 = 2 };

typedef struct tkv_ctx tkv_ctx;
typedef struct tkv_run tkv_run;

/* Run description: the hot-path fields of thinkv::SimConfig
 * (proj/include/thinkv/sim.hpp:38-68) for num_seqs independent sequences of
 * units_per_seq units each.  A unit is one (layer, kv-head) of a sequence --
 * one reference "layer" (one BlockPager, segment list and buffer).  All units
 * of a sequence share thought labels (sim.cpp:717-722). */
typedef struct tkv_run_desc {
  int32_t num_seqs;
  int32_t units_per_seq;
  int32_t num_q_heads;      /* G query heads sharing a unit's KV head */
  int32_t gqa_maxpool;      /* 1: gqa_group_size = G (one max-pooled row, attention.cpp:110-122); 0: per-head rows */
  int32_t head_dim;
  int32_t tau;              /* refresh interval (thought.cpp:361-365) */
  int32_t group_size;       /* emission window g (<= 64) */
  int32_t block_size;       /* slots per block (<= 32) */
  int32_t pool_blocks;      /* 0 = SimConfig::effective_pool_blocks() (sim.cpp:65-78) */
  int64_t budget;
  int32_t num_levels;
  int64_t levels[16];       /* RetentionSchedule (evictor.hpp:19-27) */
  int32_t psi_bits[8];      /* PrecisionMap bits per band: 2, 4, 8 or 16 */
  int32_t num_thoughts;
  double threshold_fraction;
  int64_t prompt_len;
  int64_t max_gen_len;
  int32_t scripted;         /* 1: ScriptedTrace labels (sim.hpp:24-36) */
  int32_t script_len;
  const int32_t* script_bands;  /* [num_seqs][script_len], copied at create */
  int32_t per_layer_thought;    /* must be 0 in this version */
  int32_t num_thresholds;
  double thresholds[8];     /* CalibrationResult::thresholds */
  int32_t num_calib_units;
  int32_t calib_units[64];  /* CalibrationResult::layers (unit indices within a sequence) */
  int32_t input_dtype;      /* tkv_dtype of q/k/v */
  int32_t record_events;    /* keep the evict/refresh/emit event log for tkv_dump_json("events") */
  int32_t num_dump_positions;
  const int64_t* dump_positions;  /* SimConfig::dump_positions, copied at create */
  int32_t record_sparsity_trace;  /* 1: exact per-unit sparsity on every decode step, exported by
                                     tkv_dump_json(..., "sparsity_trace") in calibration-trace form */
} tkv_run_desc;

typedef struct tkv_bytes_t {
  int64_t live_slots;        /* live (unmasked) pager slots over all units */
  int64_t resident_slots;    /* filled slots incl. soft-evicted */
  int64_t live_code_bytes;   /* K+V code bytes of live slots */
  int64_t live_scale_bytes;  /* live E4M3 key/value group scales + FP8 f32 scales (pager.cpp:321-323) */
  int64_t buffer_bytes;      /* fp buffer + current token K/V bytes */
  int64_t qo_bytes;          /* q read + output written */
  int64_t meta_bytes;        /* block-table metadata read by the attention kernel */
  int64_t algorithmic_bytes; /* sum of the above: the roofline numerator of one attention launch */
} tkv_bytes_t;

const char* tkv_last_error(void);
int tkv_abi_version(void);

int tkv_init(int device, tkv_ctx** out);
int tkv_ctx_destroy(tkv_ctx* ctx);

/* Replaces constructing ThinkvMethod (sim.cpp:494-508) + SimConfig::validate (sim.cpp:84-133). */
int tkv_run_create(tkv_ctx* ctx, const tkv_run_desc* desc, tkv_run** out);
int tkv_run_destroy(tkv_run* run);

/* Replaces ThinkvMethod::process (sim.cpp:748-843) for every unit at once.
 * q: [units][G][d], k/v: [units][d] in input_dtype, DEVICE pointers;
 * out: [units][rows][d] fp32 DEVICE pointer, rows = 1 (max-pool) or G.
 * stream: cudaStream_t (NULL = the run's own stream). */
int tkv_step(tkv_run* run, const void* q, const void* k, const void* v, float* out, void* stream);

/* Layer-by-layer form of tkv_step for a model's decode loop:
 * a step is num_layers calls, layer = 0 .. num_layers-1 in order, each with
 * that layer's inputs: q [num_seqs][H][G][d], k/v [num_seqs][H][d], out
 * [num_seqs][H][rows][d], H = units_per_seq / num_layers kv heads (units are
 * numbered seq, layer, kv-head).  Each call runs that layer's attention (and,
 * on refresh steps, its sparsity statistics); the last call also runs the
 * step's refresh boundary, emission and eviction -- the same state
 * transitions as one tkv_step with all layers' inputs. */
int tkv_step_layer(tkv_run* run, int layer, int num_layers, const void* q, const void* k, const void* v,
                   float* out, void* stream);

/* Same with HOST buffers: copies q/k/v in, steps, copies out back (synchronous). */
int tkv_step_host(tkv_run* run, const void* q, const void* k, const void* v, float* out);

/* Pipelined HOST-buffer step: enqueues the upload, the step and the download
 * and returns.  Uploads/downloads run on a copy stream through two device
 * staging slots, so step t's transfers overlap the kernels of steps t-1/t+1.
 * q/k/v must stay valid and unmodified, and out must not be read, until
 * tkv_synchronize returns (use page-locked host memory for overlap). */
int tkv_step_host_async(tkv_run* run, const void* q, const void* k, const void* v, float* out);

/* CUDA-graph replay of plain and emission steps (the
 * real-model caller).  Two step kinds are capturable: 1 = *plain* (the only
 * device work is the attention, K1, which also buffers the incoming token)
 * and 2 = *emission* (K1, then K2 quantising the full g-token window into
 * reclaimed slots).  Neither may hold a refresh boundary, a Case-2 anneal, a
 * dump, a sparsity trace or byte accounting.  At g = 16, 15 of every 16
 * decode steps are plain and the 16th an emission, except at boundaries.
 *
 * Capture: while `stream` is capturing (cudaStreamBeginCapture), tkv_step /
 * tkv_step_layer RECORD the next step's launches on `stream` (K1 per call,
 * and K2 after the last layer of an emission step) and leave the run
 * unchanged; the recorded launches read the per-step scalars (buffer half,
 * buffered tokens, put slot, window position) and K2's per-sequence controls
 * from device memory, so one graph per kind holding a model decode step
 * (projections, tkv_step_layer for every layer, ...) can be replayed for
 * every step of that kind.
 * Replay: call tkv_graph_step_begin(run, stream) before each
 * cudaGraphLaunch(exec, stream) of the graph of kind tkv_step_plain(run).
 * It fails with TKV_ERR_CONFIG unless that kind is 1 or 2 and was captured,
 * stages the step's scalars (stream-ordered on `stream`) and advances the
 * run's host state by one step exactly as the eager step would.  Other steps
 * run eagerly (tkv_step / tkv_step_layer with the same stream).
 * tkv_step_plain: the next step's kind (1 plain, 2 emission, 0 neither),
 * < 0 on error. */
int tkv_step_plain(tkv_run* run);
int tkv_graph_step_begin(tkv_run* run, void* stream);

/* Replaces ThinkvMethod::finish (sim.cpp:871-958): final partial window,
 * final budget pass, metrics. */
int tkv_finish(tkv_run* run);

/* Waits for the run's stream and reports sticky device-side errors. */
int tkv_synchronize(tkv_run* run);
int64_t tkv_position(const tkv_run* run);

/* JSON views in the reference's own formats: "tables" (BlockPager::dump,
 * pager.cpp:327-362, one per unit), "segments" (sim.cpp:919-937), "events"
 * (JSON lines, sim.cpp:643-648/663-670/724-733), "metrics" (RunMetrics::to_json),
 * "step_dumps", "sparsity_trace" (one SparsityTrace::to_jsonl line,
 * thought.cpp:66-75: {"<unit>": [sparsity per decode step]} -- the record
 * collect_sparsity_record (sim.cpp:1268-1281) feeds offline calibration,
 * here over the compressed cache; needs record_sparsity_trace).  Writes up
 * to cap bytes (NUL-terminated) and the full length to *needed. */
int tkv_dump_json(tkv_run* run, int seq, const char* what, char* buf, size_t cap, size_t* needed);

/* Byte accounting of the attention view for the next step (FragmentationStats,
 * pager.cpp:299-325, extended with buffer/q/out/metadata bytes). */
int tkv_bytes(tkv_run* run, tkv_bytes_t* out);

/* Per-launch byte accounting on the device (k_bytes.cu): while enabled,
 * every attention launch is followed by a kernel that computes, from the
 * state that launch read, the same algorithmic bytes as tkv_bytes; the
 * counts are summed over launches.  Enabling resets the sums.  Reading
 * synchronises; *launches = attention launches accounted. */
int tkv_bytes_accounting(tkv_run* run, int enable);
int tkv_bytes_accumulated(tkv_run* run, tkv_bytes_t* sum, int64_t* launches);

/* y[i] = exp(x[i]) for HOST arrays, evaluated on the device with the exp the
 * fp64 kernels use (K3a sparsity, exact gather scores): glibc's exp
 * (attention.cpp:62 calls it through std::exp) restated bit for bit. */
int tkv_exp_f64(tkv_ctx* ctx, const double* x, double* y, int64_t n);

/* Compressed-cache export: the live pager tokens of units
 * [unit0, unit0 + nunits) as QuantizedGroups in the reference wire layout of
 * serialize_group (proj/src/quant.cpp:274-324, quant.hpp:104-110), one byte
 * stream per unit (layout: k_export.cu header).  dst is DEVICE memory; with
 * dst == NULL only *needed and unit_offsets (host, nunits + 1 entries, may be
 * NULL) are produced.  A non-NULL dst smaller than *needed is a config error
 * (nothing written).  Synchronises the run's stream. */
int tkv_export_cache(tkv_run* run, int64_t unit0, int64_t nunits, void* dst, size_t cap, int64_t* unit_offsets,
                     size_t* needed);

/* Last fp64 per-unit sparsity (layer_sparsity_average) computed on a refresh step.  It is computed only
 * where something consumes it: calibrated labels, an event log (record_events) or a sparsity trace. */
int tkv_unit_sparsity(tkv_run* run, double* out, int64_t n);

/* Per-kernel device time of the run's launches (CUDA events on the run's
 * stream).  Enabling resets the counters; reading synchronises. */
typedef struct tkv_timing_t {
  double attend_ms, score_ms, flush_ms, anneal_ms, apply_ms;
  int64_t attend_launches, score_launches, flush_launches, anneal_launches, apply_launches;
  int64_t total_launches;  /* every kernel launched by the run since enable */
  /* host side of tkv_step / tkv_step_layer / tkv_step_host_async since enable:
   * host_ms = time in the call minus host_wait_ms, the time blocked waiting
   * for the step two calls back (pinned staging reuse); steps = calls */
  double host_ms, host_wait_ms;
  int64_t steps;
} tkv_timing_t;
int tkv_timing_enable(tkv_run* run, int enable);
int tkv_timing_read(tkv_run* run, tkv_timing_t* out);

/* Deterministic synthetic bf16 inputs for step `step` (synth.h) on device.
 * Unit u of the run receives the inputs of global unit unit0 + u, so a
 * sequence-sharded run (rank r: unit0 = r * units) sees exactly the inputs
 * the same sequences get in a 1-GPU run of the whole batch. */
int tkv_synth_inputs(tkv_run* run, uint64_t seed, int64_t unit0, int64_t step, void* q, void* k, void* v,
                     void* stream);

/* ---- drop-in batch-1 calls ------------------------------------------------
 * The kernels behind the reference's own C++ API (the unchanged headers in
 * proj/include/thinkv/, implemented as adapters in paper_2510_01290_b200/
 * dropin/ -- SURVEY §8b).  One call = one kernel launch over HOST arrays
 * (copied in and out; synchronous; reentrant: per-thread staging and
 * stream).  Formats: 0 ternary, 1 NVFP4, 2 FP8 (E4M3). */

/* quantize_window (quant.hpp:170-172, quant.cpp:486-580) for bits 2/4/8:
 * keys/values [n][d] (n <= group_size); key_codes/value_codes [n][d];
 * key_scales [d] and value_scales [n][ceil(d/group_size)] (E4M3 codes) or
 * fp8_scales [2] (key, value f32 window scales) for 8 bits.  Non-finite
 * input: TKV_ERR_CONFIG (the reference's kStructural). */
int tkv_dropin_quantize_window(tkv_ctx* ctx, int32_t n, int32_t d, int32_t bits, int32_t group_size,
                               const double* keys, const double* values, uint8_t* key_codes, uint8_t* value_codes,
                               uint8_t* key_scales, uint8_t* value_scales, float* fp8_scales);
/* decode_code (quant.cpp:195-205) elementwise: out[i] = value(codes[i]) * scales[i]
 * (BlockPager::decode_payload, pager.cpp:89-112). */
int tkv_dropin_decode(tkv_ctx* ctx, int32_t fmt, int64_t n, const uint8_t* codes, const double* scales, double* out);
/* gqa_attend (attention.hpp:62-66, attention.cpp:124-146): q [G][d], keys/values
 * [n][d]; out [d], row [n] (softmax scores).  fp64 in the reference's operation
 * order, glibc's exp: the reference's bits. */
int tkv_dropin_gqa_attend(tkv_ctx* ctx, int32_t G, int64_t n, int32_t d, double scale, const double* q,
                          const double* keys, const double* values, double* out, double* row);
/* sparsity (attention.cpp:148-158) of rows [offsets[r], offsets[r+1]) of scores. */
int tkv_dropin_sparsity(tkv_ctx* ctx, const double* scores, const int64_t* offsets, int32_t nrows, double frac,
                        double* out);
/* kmeans_select (evictor.hpp:98-108, evictor.cpp:255-338) for ninst
 * independent instances in one launch: instance i has m[i] <= 256 points of
 * d channels (keys concatenated, [sum m][d]) and 1 <= k[i] < m[i] clusters;
 * medoids (concatenated, [sum k]) = each cluster's medoid point index. */
int tkv_dropin_kmeans_select(tkv_ctx* ctx, int32_t ninst, int32_t d, const int32_t* m, const int32_t* k,
                             const double* keys, int32_t* medoids);
/* BlockPager::append_tokens' placement (pager.cpp:114-219) over one pager's
 * table -- thought/filled/evict (slot bitmask)/nstart [P], starts [P][bs+2],
 * masks [P][bs+1], nfree: updated in place -- for n tokens of band `band`
 * in segment seg_start: claims [n] = block * bs + slot, reused [n].
 * TKV_ERR_OOM with the table unchanged when the pool is short.  bs <= 32. */
int tkv_dropin_pager_place(tkv_ctx* ctx, int32_t P, int32_t bs, int8_t* thought, uint8_t* filled, uint32_t* evict,
                           uint8_t* nstart, int32_t* starts, uint32_t* masks, int32_t* nfree, int32_t band,
                           int32_t seg_start, int32_t n, int32_t* claims, int8_t* reused);
/* BlockPager::apply_eviction_plan (pager.cpp:238-259) on the table: mask
 * slots [n] (block * bs + slot), free touched blocks left without live
 * slots; freed [<= P] lists them in ascending id, *nfreed their count. */
int tkv_dropin_pager_evict(tkv_ctx* ctx, int32_t P, int32_t bs, int8_t* thought, uint8_t* filled, uint32_t* evict,
                           uint8_t* nstart, int32_t n, const int32_t* slots, int32_t* freed, int32_t* nfreed);

/* ---- gather-compaction comparator ---------------------------------------
 * Replaces the reference's GatherMethod (proj/src/sim.cpp:1117-1206), the
 * R-KV-style baseline of BASELINE config 5: every unit keeps a dense
 * full-precision K/V cache in arrival order; once it holds more than
 * `budget` tokens the row with the lowest head-averaged attention score is
 * evicted and every later row shifts down one slot (moved_token_slots).
 * exact_scores = 1 computes the scores in fp64 in the reference's operation
 * order (bit-exact victims); 0 uses the fp32 probabilities of the attention
 * pass (victims can differ from the reference on near-ties). */
typedef struct tkv_gather tkv_gather;
typedef struct tkv_gather_desc {
  int32_t num_units;
  int32_t num_q_heads;
  int32_t gqa_maxpool;
  int32_t head_dim;
  int64_t budget;
  int32_t input_dtype;   /* tkv_dtype of q/k/v (also the cache element type) */
  int32_t exact_scores;
} tkv_gather_desc;

int tkv_gather_create(tkv_ctx* ctx, const tkv_gather_desc* desc, tkv_gather** out);
int tkv_gather_destroy(tkv_gather* g);
/* GatherMethod::process for every unit: q [units][G][d], k/v [units][d]
 * (device pointers, input dtype); out [units][rows][d] fp32. */
int tkv_gather_step(tkv_gather* g, int prefill, const void* q, const void* k, const void* v, float* out,
                    void* stream);
/* Totals over all units (synchronises): moved_token_slots and eviction steps
 * (steps on which any unit evicted, decode steps only: sim.cpp:1166-1169). */
int tkv_gather_stats(tkv_gather* g, int64_t* moved_token_slots, int64_t* eviction_steps);
/* Token ids kept by one unit in cache order; writes min(n, cap), returns n in *n. */
int tkv_gather_ids(tkv_gather* g, int unit, int64_t* ids, int64_t cap, int64_t* n);

#ifdef __cplusplus
}
#endif
#endif /* THINKV_B200_H */
