// Device-resident cache state for the ThinKV decode path (one struct of raw
// device pointers, passed by value to every kernel).
//
// A *unit* is one (sequence, layer, kv-head) triple -- one reference
// "layer" (proj/src/sim.cpp:496-508 gives every layer its own BlockPager,
// segment list and buffer).  All per-unit arrays are unit-major so a CTA that
// owns a unit touches one contiguous region per array.
//
// HBM layout (SoA; P = pool blocks per unit, bs = block size, NS = P*bs):
//   block table   thought[P] i8, filled[P] u8, evict[P] u32 (slot bitmask),
//                 nstart[P] u8, start[P][bs+2] i32, segmask[P][bs+1] u32
//                 -- BlockTableEntry (pager.hpp:55-62) with the segment masks
//                 stored as bitmasks, one per start index beyond the first.
//                 Masks are disjoint and non-empty after pruning, so a block
//                 holds at most bs masks + the implicit first segment; while a
//                 placement runs (pager.cpp:190-216: append the new segment's
//                 mask, then prune the ones its reuse emptied) there can be one
//                 more of each, hence bs + 2 starts and bs + 1 masks.
//   slots         kcode[NS][kstride] u8, vcode[NS][vstride] u8 (packed 2/4/8-bit
//                 codes, or raw input-dtype values for 16-bit passthrough),
//                 vscale[NS][vchunks] u8 (E4M3 per-token value-chunk scales),
//                 win[NS] i32 (window -> key scales), id[NS] i32 (token id).
//   windows       kscale[NW][d] u8 (per-channel E4M3 key scales, one window =
//                 one 16-token emission), kscale_f32[NW], vscale_f32[NW] (FP8
//                 per-window scales), refs[NW] (live slots referencing it),
//                 free stack[NW] + nfree.
//   segments      segmask[NSEG][W] u32: member bitmask relative to start_step.
//   buffer        buf_k/buf_v[2][g][d] input dtype (double-buffered emission window).
#pragma once
#include <stdint.h>

#define TKV_MAX_BANDS 8
#define TKV_MAX_G 16
#define TKV_STARTS_PER_BLOCK(bs) ((bs) + 2)
#define TKV_MASKS_PER_BLOCK(bs) ((bs) + 1)

enum { TKV_FMT_TERNARY = 0, TKV_FMT_NVFP4 = 1, TKV_FMT_FP8 = 2, TKV_FMT_RAW = 3 };
enum { TKV_IN_BF16 = 0, TKV_IN_F32 = 1, TKV_IN_F64 = 2 };

// Error codes mirror thinkv::Error::exit_code() (proj/include/thinkv/errors.hpp:31-46).
enum { TKV_E_OK = 0, TKV_E_UNEXPECTED = 1, TKV_E_STRUCTURAL = 2, TKV_E_CALIBRATION = 3,
       TKV_E_OOM = 4, TKV_E_INTEGRITY = 5 };

struct TkvDims {
  int32_t U;          // units
  int32_t G;          // query heads per unit
  int32_t D;          // head dim
  int32_t maxpool;    // 1 = one max-pooled softmax row per unit
  int32_t bs;         // block size (<= 32)
  int32_t P;          // pool blocks per unit
  int32_t NS;         // slots per unit = P * bs
  int32_t NW;         // window capacity per unit
  int32_t g;          // quantization group size (emission window length)
  int32_t vchunks;    // ceil(D / g)
  int32_t kstride;    // bytes per slot in kcode/vcode
  int32_t T;          // token-id capacity (prompt_len + max_gen_len)
  int32_t W;          // u32 words per segment member mask = ceil(tau / 32)
  int32_t NSEG;       // segment capacity per unit
  int32_t in_dtype;   // TKV_IN_*
  int32_t in_bytes;   // bytes per input element
  int32_t num_bands;
  int32_t band_fmt[TKV_MAX_BANDS];   // TKV_FMT_* per thought band
  int32_t band_bytes[TKV_MAX_BANDS]; // code bytes per K (or V) vector per band
  float scale;        // 1/sqrt(D)
  double thr_frac;    // sparsity threshold fraction
};

struct TkvState {
  TkvDims dm;
  // block table
  int8_t* blk_thought;
  uint8_t* blk_filled;
  uint32_t* blk_evict;
  uint8_t* blk_nstart;
  int32_t* blk_start;
  uint32_t* blk_segmask;
  int32_t* unit_nfree;    // free blocks per unit
  // slots
  uint8_t* slot_k;
  uint8_t* slot_v;
  uint8_t* slot_vs;
  int32_t* slot_win;
  int32_t* slot_id;
  // windows
  uint8_t* win_ks;
  float* win_kf;
  float* win_vf;
  int32_t* win_refs;
  int32_t* win_free;
  int32_t* win_nfree;
  // segments / buffer
  uint32_t* seg_mask;
  uint8_t* buf;          // [U][2][2 (k,v)][g][D] * in_bytes
  // per-unit outputs of the score kernel and sticky device errors
  double* sparsity;      // [U]
  unsigned long long* kstats;  // optional K-means counters (TKV_KSTATS=1), else null
  int32_t* err;          // [U]
  // Upper bound on live pager slots of any unit at the next attention launch
  // (host-exact: every unit of a sequence holds its segments' total members
  // minus the buffered tokens).  Sizes the per-unit live lists in shared memory.
  int32_t max_live;
  // Launch-local index i -> unit (per-layer stepping, tkv_step_layer): units
  // of one layer are strided in the sequence-major unit order, so a layer
  // launch covers i in [0, num_seqs * lmap_h) and
  // u = (i / lmap_h) * lmap_ups + lmap_off + i % lmap_h.  lmap_h == 0: u = i.
  int32_t lmap_h, lmap_ups, lmap_off, lmap_count;
  // Per-step scalars in device memory (CUDA-graph replay of plain and
  // emission steps, tkv_graph_step_begin): when non-null, K1 reads
  // {buf_half, nbuf, put_half, put_slot} = step_dev[0..3] and K2 its
  // {half, pos0} = step_dev[4..5] instead of their launch parameters, so one
  // captured launch serves every replayed step.  Null on eager launches.
  const int32_t* step_dev;
};

// K2's per-step scalars: launch parameters, or the device copy (graph replay).
__host__ __device__ inline void tkv_flush_scalars(const TkvState& st, int& half, int& pos0) {
#ifdef __CUDA_ARCH__
  if (st.step_dev) {
    half = st.step_dev[4];
    pos0 = st.step_dev[5];
  }
#else
  (void)st; (void)half; (void)pos0;
#endif
}

// K1's per-step scalars: launch parameters, or the device copy (graph replay).
__host__ __device__ inline void tkv_step_scalars(const TkvState& st, int& buf_half, int& nbuf, int& put_half,
                                                 int& put_slot) {
#ifdef __CUDA_ARCH__
  if (st.step_dev) {
    buf_half = st.step_dev[0];
    nbuf = st.step_dev[1];
    put_half = st.step_dev[2];
    put_slot = st.step_dev[3];
  }
#else
  (void)st; (void)buf_half; (void)nbuf; (void)put_half; (void)put_slot;
#endif
}

#ifdef __CUDACC__
// Slots of a closed segment's members (BlockPager::key_of, pager.cpp:280-287)
// without a token-id index: a live slot holds a member iff its token id lies
// in the segment's window [seg_start, seg_start + span) and the id's member
// bit is set.  A token is written to exactly one slot and its member bit is
// cleared when it is evicted, so every member is found exactly once; evicted
// slots are skipped as well.  Block-cooperative: rank_slot[r] = the slot of the
// r-th member in id order; *found (shared, zeroed by the caller) counts them.
__device__ inline void tkv_member_slots(const TkvState& st, int u, int seg_start, int span, const uint32_t* segm,
                                        int* rank_slot, int* found) {
  const TkvDims& dm = st.dm;
  const int32_t* sid = st.slot_id + (int64_t)u * dm.NS;
  const uint32_t* ev = st.blk_evict + (int64_t)u * dm.P;
  for (int s = threadIdx.x; s < dm.NS; s += blockDim.x) {
    const int rel = sid[s] - seg_start;
    if (rel < 0 || rel >= span) continue;
    const uint32_t w = segm[rel >> 5];
    const int blk = s / dm.bs, sl = s % dm.bs;
    if (!((w >> (rel & 31)) & 1u) || ((ev[blk] >> sl) & 1u) || st.blk_thought[(int64_t)u * dm.P + blk] < 0 ||
        sl >= st.blk_filled[(int64_t)u * dm.P + blk])
      continue;
    int rank = __popc(w & ((1u << (rel & 31)) - 1u));
    for (int k = 0; k < (rel >> 5); ++k) rank += __popc(segm[k]);
    rank_slot[rank] = s;
    atomicAdd(found, 1);
  }
}
#endif

__host__ __device__ inline int tkv_unit_of(const TkvState& st, int i) {
  return st.lmap_h ? (i / st.lmap_h) * st.lmap_ups + st.lmap_off + i % st.lmap_h : i;
}
__host__ __device__ inline int tkv_launch_units(const TkvState& st) { return st.lmap_h ? st.lmap_count : st.dm.U; }

// Per-group (sequence) control values for an emission (flush).
struct TkvFlushCtl {
  int32_t band;        // open segment's thought band
  int32_t seg_start;   // open segment's start_step (start index for the block table)
};

// One K-means anneal of one segment, identical for every unit of a group.
struct TkvAnnealOp {
  int32_t unit0, nunits;  // unit range of the group
  int32_t seg;            // device segment index
  int32_t seg_start;      // start_step (bit 0 of the member mask)
  int32_t span;           // initial_size (valid member bits)
  int32_t m;              // members before this anneal
  int32_t K;              // retention target (< m)
  int32_t log_off;        // offset (in u32 words) of this op's evicted-mask log, per unit: + u_rel*W
  int32_t nrestart;       // 4 farthest-first restarts, or 0 when seeds enumerate all K-subsets
  int32_t ncombos;        // C(m, K) when nrestart == 0 (<= 512, evictor.cpp:270-283)
};

// Units of one group whose anneal ops [op_begin, op_end) are applied together
// (one evict event per unit, sim.cpp:652-671).
struct TkvApplyGroup {
  int32_t unit0, nunits;
  int32_t op_begin, op_end;
};

// Gather-compaction comparator state (GatherMethod, sim.cpp:1117-1206): per
// unit a dense full-precision K/V cache in arrival order, compacted on every
// eviction.  cap = budget + 1 rows.
struct TkvGatherState {
  int32_t U, G, D, maxpool, cap, in_dtype, in_bytes;
  int64_t budget;
  uint8_t* k;       // [U][cap][D] input dtype
  uint8_t* v;
  int32_t* ids;     // [U][cap] token ids (positions)
  int32_t* victim;  // [U] last evicted row
};
