// Host-side launchers for the sm_100a kernels (implemented in k_*.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "tkv_state.h"

// K1: paged mixed-precision decode attention over every unit's live slots,
// its fp buffer (first nbuf tokens of half buf_half) and the current token.
// Also stores the current k/v into buffer (put_half, put_slot) when put_slot >= 0.
cudaError_t tkv_launch_attend(const TkvState& st, const void* q, const void* k, const void* v,
                              float* out, int buf_half, int nbuf, int put_half, int put_slot,
                              cudaStream_t stream);

// K1 tensor-core variant (k_attend_mma.cu) and its shape predicate.
bool tkv_attend_mma_supported(const TkvDims& dm);
cudaError_t tkv_launch_attend_mma(const TkvState& st, const void* q, const void* k, const void* v, float* out,
                                  int buf_half, int nbuf, int put_half, int put_slot, cudaStream_t stream);

// Algorithmic-byte accounting of the state an attention launch reads
// (k_bytes.cu): adds live slots, resident slots, live code bytes, live scale
// bytes and metadata bytes of every launched unit to acc[0..5).
cudaError_t tkv_launch_bytes(const TkvState& st, unsigned long long* acc, unsigned long long* last,
                             long long repeat, cudaStream_t stream);
cudaError_t tkv_launch_bytes_repeat(unsigned long long* acc, const unsigned long long* last, int64_t units,
                                    long long repeat, cudaStream_t stream);

// y[i] = tkv_exp(x[i]) (k_math.cu): glibc's exp, bit for bit.
cudaError_t tkv_launch_exp(const double* x, double* y, int64_t n, cudaStream_t stream);

// K3a: fp64 sparsity statistics (layer_sparsity_average) over the same view.
cudaError_t tkv_launch_score(const TkvState& st, const void* q, const void* k, int buf_half,
                             int nbuf, cudaStream_t stream);

// K2: quantize the n buffered tokens of half `half` (token ids pos0..pos0+n-1)
// and place them; ctl is indexed by group = unit / units_per_group.
cudaError_t tkv_launch_flush(const TkvState& st, int half, int n, int pos0, const TkvFlushCtl* ctl,
                             int units_per_group, cudaStream_t stream);

// K3d: K-means medoid anneals.  ops[nops] with item prefix sums over units;
// evicted masks are logged at log + op.log_off + unit_rel * W.
cudaError_t tkv_launch_anneal(const TkvState& st, const TkvAnnealOp* ops, int nops,
                              const int32_t* item_prefix, int nitems, uint32_t* log,
                              double* scratch, int scratch_ctas, int64_t scratch_doubles_per_cta,
                              int max_m, cudaStream_t stream);

// K3d v2 (k_kmeans.cu): prep / restart / final kernels over instances
// [item0, item0 + item_count) whose restarts are [run0, run0 + run_count).
int64_t tkv_km_instance_bytes(int mmax, int kmax, int D, int W, int R);
size_t tkv_km_restart_smem(int mmax, int kmax, int D, int xbytes, bool means_global);
cudaError_t tkv_launch_kmeans(const TkvState& st, const TkvAnnealOp* ops, int nops, const int32_t* item_prefix,
                              int nitems, const int32_t* run_prefix, int nruns, int item0, int item_count,
                              int run0, int run_count, int mmax, int kmax, int R, uint8_t* scratch, double* gsums,
                              int gsums_ctas, uint32_t* log, int scaled_any, int x16, cudaStream_t stream);

// K3e: apply the evictions of ops[0..nops) (soft-mask slots, release window
// references, free empty blocks).  One CTA per unit of the listed groups.
cudaError_t tkv_launch_apply(const TkvState& st, const TkvAnnealOp* ops,
                             const TkvApplyGroup* groups, int ngroups,
                             const int32_t* unit_prefix, int nitems, const uint32_t* log,
                             cudaStream_t stream);

// ---- drop-in batch-1 kernels (k_dropin.cu, k_append.cu, k_evict.cu) ----
// quantize_window over n <= group_size fp64 tokens (fmt = TKV_FMT_TERNARY/NVFP4/FP8):
// kc/vc [n][d], ksc [d], vsc [n][ceil(d/group_size)], f8 [2] (FP8 key/value scales);
// *bad = 1 on a non-finite input (the reference throws kStructural).
cudaError_t tkv_launch_window_quant(int n, int d, int fmt, int group_size, const double* keys, const double* values,
                                    uint8_t* kc, uint8_t* vc, uint8_t* ksc, uint8_t* vsc, float* f8, int* bad,
                                    cudaStream_t stream);
// gqa_attend in fp64 (reference order): out [d], row [n] (the softmax scores).
cudaError_t tkv_launch_gqa_attend_f64(int G, int n, int d, double scale, const double* q, const double* k,
                                      const double* v, double* out, double* row, cudaStream_t stream);
// sparsity of rows [offs[r], offs[r+1]) of scores.
cudaError_t tkv_launch_sparsity_rows(const double* scores, const int64_t* offs, int nrows, double frac, double* out,
                                     cudaStream_t stream);
// decode_code elementwise.
cudaError_t tkv_launch_decode_codes(int fmt, int64_t n, const uint8_t* codes, const double* scales, double* out,
                                    cudaStream_t stream);
// BlockPager placement / eviction over one pager's table (layout as TkvState's
// block table for one unit: th/fl/ev/ns [P], starts [P][bs+2], masks [P][bs+1]).
cudaError_t tkv_launch_pager_place(int P, int bs, int8_t* th, uint8_t* fl, uint32_t* ev, uint8_t* ns, int32_t* sstart,
                                   uint32_t* smask, int32_t* nfree, int band, int32_t seg_start, int n, int32_t* claim,
                                   int8_t* reuse, int32_t* rc, cudaStream_t stream);
cudaError_t tkv_launch_pager_evict(int P, int bs, int8_t* th, uint8_t* fl, uint32_t* ev, uint8_t* ns, int n,
                                   const int32_t* slots, int32_t* freed, int32_t* nfreed, cudaStream_t stream);
// kmeans_select medoid indices of ninst instances (instance i: m[i] <= 256 points
// of D channels at X + xoff[i], 1 <= K[i] < m[i]; out + ooff[i]); scratch >= 5 * total points * D.
cudaError_t tkv_launch_kmeans_select_f64(int ninst, const double* X, const int32_t* m, const int32_t* K,
                                         const int64_t* xoff, const int64_t* ooff, int D, double* scratch,
                                         int32_t* out, cudaStream_t stream);

// Synthetic decode inputs (bf16) generated on device with the same integer
// generator as the host oracle (synth.h).
cudaError_t tkv_launch_synth(uint64_t seed, int units_per_seq, int tau, int sink_tokens, int64_t unit0,
                             int units, int G, int D, int64_t step, uint16_t* q, uint16_t* k,
                             uint16_t* v, cudaStream_t stream);

// One-time state initialisation (window free stacks, free-block counts).
cudaError_t tkv_launch_init(const TkvState& st, cudaStream_t stream);

// Gather-compaction comparator (k_gather.cu): append, attention, head-averaged
// scores (exact fp64 when `exact`), first-minimum eviction and compaction.
size_t tkv_gather_smem(const TkvGatherState& g, int exact);
cudaError_t tkv_launch_gather_step(const TkvGatherState& g, int n, int64_t pos, const void* q, const void* k,
                                   const void* v, float* out, int exact, cudaStream_t stream);

// Compressed-cache export in the reference wire layout (k_export.cu, SURVEY
// §8f-3): pass 0 writes each unit's byte size into sizes[0..nunits), pass 1
// writes the unit streams at offsets[] into dst.  Tokens with id < npos.
size_t tkv_export_smem(const TkvState& st);
cudaError_t tkv_launch_export(const TkvState& st, int unit0, int nunits, int npos, int pass, int64_t* sizes,
                              const int64_t* offsets, uint8_t* dst, cudaStream_t stream);
