// thinkv::BlockPager (proj/include/thinkv/pager.hpp:90-160) over the device
// placement and release kernels.
//
// The class layout is the reference header's; its members are the host
// mirror of one pager.  The decisions -- which slot each token takes (the
// ordered claim of pager.cpp:132-164 with allocation and OOM check), the
// segment start/mask bookkeeping (:166-216), which blocks an eviction frees
// (:238-259) -- and the decoded payload values (:89-112) are computed by
// the library's kernels (tkv_dropin_pager_place / _evict / _decode, the code
// K2/K3e run on the paged state).  Each call uploads the table, launches,
// and applies the kernel's result to the mirror.
#include <algorithm>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "dropin.hpp"
#include "thinkv/pager.hpp"

namespace thinkv {

namespace {

// The device form of one pager's block table (TkvState layout for one unit).
struct DeviceTable {
  int P = 0, bs = 0;
  std::vector<int8_t> thought;
  std::vector<uint8_t> filled, nstart;
  std::vector<uint32_t> evict, masks;
  std::vector<int32_t> starts;
  int32_t nfree = 0;

  int sstride() const { return bs + 2; }
  int mstride() const { return bs + 1; }
};

DeviceTable pack(int bs, int P, const std::map<int, BlockTableEntry>& table, std::size_t nfree) {
  if (bs > 32) throw Error(ErrorKind::kConfig, "device pager: block_size > 32 is not supported");
  DeviceTable t;
  t.P = P;
  t.bs = bs;
  t.thought.assign(P, -1);
  t.filled.assign(P, 0);
  t.nstart.assign(P, 0);
  t.evict.assign(P, 0);
  t.starts.assign((std::size_t)P * t.sstride(), 0);
  t.masks.assign((std::size_t)P * t.mstride(), 0);
  t.nfree = static_cast<int32_t>(nfree);
  for (const auto& [bid, e] : table) {
    t.thought[bid] = static_cast<int8_t>(e.thought.band);
    t.filled[bid] = static_cast<uint8_t>(e.filled);
    uint32_t ev = 0;
    for (int s = 0; s < bs; ++s)
      if (e.eviction_mask[s]) ev |= 1u << s;
    t.evict[bid] = ev;
    if (e.start_indices.size() > static_cast<std::size_t>(bs + 1))
      throw Error(ErrorKind::kIntegrity, "block holds more segment starts than slots");
    t.nstart[bid] = static_cast<uint8_t>(e.start_indices.size());
    for (std::size_t k = 0; k < e.start_indices.size(); ++k) {
      if (e.start_indices[k] != static_cast<int32_t>(e.start_indices[k]))
        throw Error(ErrorKind::kConfig, "device pager: segment start beyond 32 bits");
      t.starts[(std::size_t)bid * t.sstride() + k] = static_cast<int32_t>(e.start_indices[k]);
    }
    for (std::size_t k = 0; k < e.segment_masks.size(); ++k) {
      uint32_t m = 0;
      for (int s = 0; s < bs; ++s)
        if (e.segment_masks[k][s]) m |= 1u << s;
      t.masks[(std::size_t)bid * t.mstride() + k] = m;
    }
  }
  return t;
}

// Device table row of block `bid` -> the mirror's entry.
void unpack_entry(const DeviceTable& t, int bid, BlockTableEntry& e) {
  e.physical_block = bid;
  e.thought = ThoughtLabel{t.thought[bid]};
  e.filled = t.filled[bid];
  e.eviction_mask.assign(t.bs, 0);
  for (int s = 0; s < t.bs; ++s) e.eviction_mask[s] = (t.evict[bid] >> s) & 1u;
  const int ns = t.nstart[bid];
  e.start_indices.assign(ns, 0);
  for (int k = 0; k < ns; ++k) e.start_indices[k] = t.starts[(std::size_t)bid * t.sstride() + k];
  e.segment_masks.assign(ns > 0 ? ns - 1 : 0, std::vector<std::uint8_t>(t.bs, 0));
  for (int k = 0; k + 1 < ns; ++k) {
    const uint32_t m = t.masks[(std::size_t)bid * t.mstride() + k];
    for (int s = 0; s < t.bs; ++s) e.segment_masks[k][s] = (m >> s) & 1u;
  }
}

int format_int(const SlotPayload& p) { return static_cast<int>(p.format); }

}  // namespace

double GroupScaleRecord::value() const { return f32 ? static_cast<double>(scale_f32) : e4m3_decode(scale_code); }

std::int64_t FragmentationStats::total_live_code_bits() const {
  std::int64_t bits = 0;
  for (const auto& kv : live_code_bits_by_format) bits += kv.second;
  return bits;
}

BlockPager::BlockPager(int block_size, int pool_blocks) : block_size_(block_size), pool_blocks_(pool_blocks) {
  if (block_size < 1 || pool_blocks < 1) throw Error(ErrorKind::kConfig, "pager needs block_size >= 1 and a pool");
  blocks_.resize(pool_blocks);
  for (int b = 0; b < pool_blocks; ++b) {
    blocks_[b].slots.resize(block_size);
    blocks_[b].occupied.assign(block_size, 0);
    free_.insert(b);
  }
}

int BlockPager::allocate_block(ThoughtLabel thought) {
  if (free_.empty()) {
    const FragmentationStats st = fragmentation_stats();
    throw Error(ErrorKind::kOutOfMemory, "physical block pool exhausted (" + std::to_string(st.blocks_in_use) + "/" +
                                             std::to_string(pool_blocks_) + " blocks in use, " +
                                             std::to_string(st.live_slots) + " live slots, " +
                                             std::to_string(st.masked_slots) + " masked)");
  }
  const int bid = *free_.begin();
  free_.erase(free_.begin());
  BlockTableEntry e;
  e.physical_block = bid;
  e.thought = thought;
  e.eviction_mask.assign(block_size_, 0);
  table_[bid] = std::move(e);
  return bid;
}

void BlockPager::install_group(std::uint64_t group_id, GroupScaleRecord record) {
  record.refs = 0;
  groups_[group_id] = record;
}

void BlockPager::add_slot_groups(const SlotPayload& p) {
  if (p.raw) return;
  auto ref = [&](std::uint64_t gid) {
    auto it = groups_.find(gid);
    if (it == groups_.end()) throw Error(ErrorKind::kIntegrity, "slot references unknown group " + std::to_string(gid));
    ++it->second.refs;
  };
  if (p.shared_scale) {
    ref(p.key_group_base);
    ref(p.value_group_base);
    return;
  }
  for (int c = 0; c < p.head_dim(); ++c) ref(p.key_group_base + c);
  for (int j = 0; j < p.value_chunks; ++j) ref(p.value_group_base + j);
}

void BlockPager::release_slot_groups(const SlotPayload& p) {
  if (p.raw) return;
  auto unref = [&](std::uint64_t gid) {
    auto it = groups_.find(gid);
    if (it != groups_.end() && --it->second.refs <= 0) groups_.erase(it);
  };
  if (p.shared_scale) {
    unref(p.key_group_base);
    unref(p.value_group_base);
    return;
  }
  for (int c = 0; c < p.head_dim(); ++c) unref(p.key_group_base + c);
  for (int j = 0; j < p.value_chunks; ++j) unref(p.value_group_base + j);
}

// One payload's decode on the device: per-channel scale values from the
// group records, then code x scale in the kernel.
void BlockPager::decode_payload(SlotPayload& p) const {
  if (p.raw) return;
  const int d = p.head_dim();
  std::vector<std::uint8_t> codes(2 * (std::size_t)d);
  std::vector<double> scales(2 * (std::size_t)d);
  for (int c = 0; c < d; ++c) {
    codes[c] = p.key_codes[c];
    codes[d + c] = p.value_codes[c];
    if (p.shared_scale) {
      scales[c] = groups_.at(p.key_group_base).value();
      scales[d + c] = groups_.at(p.value_group_base).value();
    } else {
      const int chunk = std::min(c / std::max(1, p.group_size), std::max(0, p.value_chunks - 1));
      scales[c] = groups_.at(p.key_group_base + c).value();
      scales[d + c] = groups_.at(p.value_group_base + chunk).value();
    }
  }
  std::vector<double> out(2 * (std::size_t)d);
  dropin::check(tkv_dropin_decode(dropin::ctx(), format_int(p), 2 * (int64_t)d, codes.data(), scales.data(), out.data()));
  p.key_fp.assign(out.begin(), out.begin() + d);
  p.value_fp.assign(out.begin() + d, out.end());
}

std::vector<Placement> BlockPager::append_tokens(ThoughtLabel thought, std::vector<SlotPayload> tokens,
                                                 std::int64_t segment_start) {
  if (tokens.empty()) return {};
  for (const SlotPayload& t : tokens)
    if (!(t.thought == thought)) throw Error(ErrorKind::kStructural, "append_tokens: mixed thought labels");
  const int n = static_cast<int>(tokens.size());
  if (segment_start != static_cast<int32_t>(segment_start))
    throw Error(ErrorKind::kConfig, "device pager: segment start beyond 32 bits");

  // 1. placement on the device
  DeviceTable t = pack(block_size_, pool_blocks_, table_, free_.size());
  std::vector<int32_t> claims(n);
  std::vector<int8_t> reused(n);
  const int rc = tkv_dropin_pager_place(dropin::ctx(), t.P, t.bs, t.thought.data(), t.filled.data(), t.evict.data(),
                                        t.nstart.data(), t.starts.data(), t.masks.data(), &t.nfree, thought.band,
                                        static_cast<int32_t>(segment_start), n, claims.data(), reused.data());
  if (rc == TKV_ERR_OOM) {
    const FragmentationStats st = fragmentation_stats();
    throw Error(ErrorKind::kOutOfMemory, "append of " + std::to_string(n) + " tokens: physical block pool exhausted (" +
                                             std::to_string(free_.size()) + " free blocks, " +
                                             std::to_string(st.live_slots) + " live, " +
                                             std::to_string(st.masked_slots) + " masked slots)");
  }
  dropin::check(rc);

  // 2. mirror: newly allocated blocks, then every touched block's entry
  std::vector<char> touched(pool_blocks_, 0);
  for (int i = 0; i < n; ++i) touched[claims[i] / block_size_] = 1;
  for (int b = 0; b < pool_blocks_; ++b) {
    if (!touched[b]) continue;
    if (!table_.count(b)) free_.erase(b);
    unpack_entry(t, b, table_[b]);
  }

  // 3. payloads in placement order; every quantized payload is decoded in
  //    one launch (decode reads group scales only, which placement does not
  //    change, so batching equals the reference's per-token decode)
  std::vector<std::uint8_t> codes;
  std::vector<double> scales;
  std::vector<int> fmt_of;  // per token: format, -1 raw
  for (const SlotPayload& p : tokens) {
    fmt_of.push_back(p.raw ? -1 : format_int(p));
    if (p.raw) continue;
    const int d = p.head_dim();
    for (int c = 0; c < d; ++c) {
      codes.push_back(p.key_codes[c]);
      scales.push_back(groups_.at(p.shared_scale ? p.key_group_base : p.key_group_base + c).value());
    }
    for (int c = 0; c < d; ++c) {
      const int chunk = std::min(c / std::max(1, p.group_size), std::max(0, p.value_chunks - 1));
      codes.push_back(p.value_codes[c]);
      scales.push_back(groups_.at(p.shared_scale ? p.value_group_base : p.value_group_base + chunk).value());
    }
  }
  // one format per append (a window is one band), but decode per run of equal formats regardless
  std::vector<double> decoded(codes.size());
  for (std::size_t i = 0, off = 0; i < tokens.size();) {
    if (fmt_of[i] < 0) { ++i; continue; }
    std::size_t j = i, len = 0;
    while (j < tokens.size() && fmt_of[j] == fmt_of[i]) len += 2 * (std::size_t)tokens[j++].head_dim();
    dropin::check(tkv_dropin_decode(dropin::ctx(), fmt_of[i], (int64_t)len, codes.data() + off, scales.data() + off,
                                    decoded.data() + off));
    off += len;
    i = j;
  }
  std::vector<Placement> out;
  out.reserve(n);
  for (int i = 0, off = 0; i < n; ++i) {
    const int b = claims[i] / block_size_, s = claims[i] % block_size_;
    SlotPayload p = std::move(tokens[i]);
    if (!p.raw) {
      const int d = p.head_dim();
      p.key_fp.assign(decoded.begin() + off, decoded.begin() + off + d);
      p.value_fp.assign(decoded.begin() + off + d, decoded.begin() + off + 2 * d);
      off += 2 * d;
    }
    add_slot_groups(p);
    index_[p.id] = {b, s};
    out.push_back(Placement{p.id, b, s, reused[i] != 0});
    blocks_[b].slots[s] = std::move(p);
    blocks_[b].occupied[s] = 1;
  }
  return out;
}

int BlockPager::live_in_block(const BlockTableEntry& entry) const {
  int n = 0;
  for (int s = 0; s < entry.filled; ++s) n += entry.eviction_mask[s] ? 0 : 1;
  return n;
}

void BlockPager::free_block(int block_id) {
  PhysicalBlock& blk = blocks_[block_id];
  std::fill(blk.slots.begin(), blk.slots.end(), SlotPayload{});
  std::fill(blk.occupied.begin(), blk.occupied.end(), 0);
  table_.erase(block_id);
  free_.insert(block_id);
}

void BlockPager::apply_eviction_plan(const EvictionPlan& plan) {
  // Resolve ids to slots in plan order; the reference stops at the first
  // unknown id with the earlier ones already masked and no block freed.
  std::vector<int32_t> slots;
  std::vector<TokenId> ids;
  for (const SegmentEviction& seg : plan.segments) {
    for (TokenId id : seg.evicted) {
      const auto it = index_.find(id);
      if (it == index_.end()) {
        for (std::size_t i = 0; i < ids.size(); ++i) {
          const int b = slots[i] / block_size_, s = slots[i] % block_size_;
          table_.at(b).eviction_mask[s] = 1;
          release_slot_groups(blocks_[b].slots[s]);
          index_.erase(ids[i]);
        }
        throw Error(ErrorKind::kIntegrity, "eviction plan references unknown token id " + std::to_string(id));
      }
      slots.push_back(it->second.first * block_size_ + it->second.second);
      ids.push_back(id);
      index_.erase(it);  // a repeated id is unknown the second time, as in the reference
    }
  }
  if (slots.empty()) return;
  DeviceTable t = pack(block_size_, pool_blocks_, table_, free_.size());
  std::vector<int32_t> freed(pool_blocks_);
  int32_t nfreed = 0;
  dropin::check(tkv_dropin_pager_evict(dropin::ctx(), t.P, t.bs, t.thought.data(), t.filled.data(), t.evict.data(),
                                       t.nstart.data(), static_cast<int32_t>(slots.size()), slots.data(),
                                       freed.data(), &nfreed),
                ErrorKind::kIntegrity);
  for (int32_t sl : slots) {
    const int b = sl / block_size_, s = sl % block_size_;
    table_.at(b).eviction_mask[s] = 1;
    release_slot_groups(blocks_[b].slots[s]);
  }
  for (int i = 0; i < nfreed; ++i) free_block(freed[i]);
}

std::vector<const SlotPayload*> BlockPager::read_active() const {
  std::vector<const SlotPayload*> live;
  live.reserve(index_.size());
  for (const auto& [bid, e] : table_)
    for (int s = 0; s < e.filled; ++s)
      if (!e.eviction_mask[s]) live.push_back(&blocks_[bid].slots[s]);
  return live;
}

std::vector<TokenId> BlockPager::live_token_ids() const {
  std::vector<TokenId> ids;
  for (const SlotPayload* p : read_active()) ids.push_back(p->id);
  return ids;
}

const Vec& BlockPager::key_of(TokenId id) const {
  const auto it = index_.find(id);
  if (it == index_.end()) throw Error(ErrorKind::kIntegrity, "key_of: token " + std::to_string(id) + " is not live");
  return blocks_[it->second.first].slots[it->second.second].key_fp;
}

const SlotPayload& BlockPager::slot(int block, int slot_idx) const { return blocks_.at(block).slots.at(slot_idx); }

FragmentationStats BlockPager::fragmentation_stats() const {
  FragmentationStats st;
  for (const auto& [bid, e] : table_) {
    ++st.blocks_in_use;
    st.unfilled_slots += block_size_ - e.filled;
    for (int s = 0; s < e.filled; ++s) {
      const SlotPayload& p = blocks_[bid].slots[s];
      const std::string fmt = p.raw ? "RAW16" : format_name(p.format);
      const std::int64_t bits = (std::int64_t)(p.raw ? 16 : format_code_bits(p.format)) * p.head_dim() * 2;
      st.resident_code_bits_by_format[fmt] += bits;
      if (e.eviction_mask[s]) {
        ++st.masked_slots;
      } else {
        ++st.live_slots;
        st.live_code_bits_by_format[fmt] += bits;
      }
    }
  }
  st.free_blocks = static_cast<std::int64_t>(free_.size());
  for (const auto& kv : groups_)
    if (kv.second.refs > 0) st.live_scale_bytes += kv.second.f32 ? 4 : 1;
  return st;
}

nlohmann::json BlockPager::dump() const {
  auto bits = [&](const std::vector<std::uint8_t>& m) {
    std::string out(block_size_, '0');
    for (int i = 0; i < block_size_; ++i) out[i] = m[i] ? '1' : '0';
    return out;
  };
  nlohmann::json blocks = nlohmann::json::array();
  for (const auto& [bid, e] : table_) {
    nlohmann::json masks = nlohmann::json::array(), toks = nlohmann::json::array();
    for (const auto& m : e.segment_masks) masks.push_back(bits(m));
    for (int s = 0; s < block_size_; ++s) {
      if (s < e.filled) toks.push_back(blocks_[bid].slots[s].id);
      else toks.push_back(nullptr);
    }
    nlohmann::json b;
    b["physical_block"] = bid;
    b["filled"] = e.filled;
    b["thought"] = e.thought.band;
    b["start_indices"] = e.start_indices;
    b["segment_masks"] = masks;
    b["eviction_mask"] = bits(e.eviction_mask);
    b["tokens"] = toks;
    blocks.push_back(std::move(b));
  }
  nlohmann::json j;
  j["block_size"] = block_size_;
  j["pool_blocks"] = pool_blocks_;
  j["blocks"] = std::move(blocks);
  j["free_blocks"] = std::vector<int>(free_.begin(), free_.end());
  return j;
}

}  // namespace thinkv
