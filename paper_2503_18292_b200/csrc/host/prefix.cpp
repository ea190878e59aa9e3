// Prefix-cache lookup: per-kind valid prefixes, their mapping onto the global
// sequence axis, the longest common prefix across groups and the pinning of
// the pages that back it.  Semantics follow reference layer_policies.cpp,
// prefix_cache.cpp and kv_allocator.cpp (cited per function).
#include <algorithm>

#include "jenga_host.hpp"

namespace jenga {

// reference range_set.cpp:12-28
void PrefixRangeSet::append_range(uint64_t lo, uint64_t hi) {
  JENGA_CHECK(lo <= hi, "range set: inverted range");
  if (!r_.empty()) {
    JENGA_CHECK(lo > r_.back().second, "range set: appends must be increasing");
    if (lo == r_.back().second + 1) {
      r_.back().second = hi;
      return;
    }
  }
  r_.emplace_back(lo, hi);
}

bool PrefixRangeSet::contains(uint64_t v) const {
  auto it = std::upper_bound(r_.begin(), r_.end(), v,
                             [](uint64_t x, const std::pair<uint64_t, uint64_t>& r) { return x < r.first; });
  if (it == r_.begin()) return false;
  --it;
  return v >= it->first && v <= it->second;
}

// reference range_set.cpp:46-63 (two-pointer sweep)
PrefixRangeSet PrefixRangeSet::intersect(const PrefixRangeSet& a, const PrefixRangeSet& b) {
  PrefixRangeSet out;
  size_t i = 0, j = 0;
  while (i < a.r_.size() && j < b.r_.size()) {
    const uint64_t lo = std::max(a.r_[i].first, b.r_[j].first);
    const uint64_t hi = std::min(a.r_[i].second, b.r_[j].second);
    if (lo <= hi) out.append_range(lo, hi);
    if (a.r_[i].second < b.r_[j].second) ++i;
    else ++j;
  }
  return out;
}

// reference layer_policies.cpp:9-40
std::vector<uint64_t> required_tokens(const LayerGroupSpec& g, uint64_t p, bool* defined) {
  JENGA_CHECK(p >= 1, "required_tokens: prefix length must be >= 1");
  if (defined) *defined = true;
  std::vector<uint64_t> out;
  switch (g.kind) {
    case LayerKind::kFullAttention:
    case LayerKind::kCrossAttention:
      out.reserve(p);
      for (uint64_t i = 1; i <= p; ++i) out.push_back(i);
      break;
    case LayerKind::kSlidingWindow: {
      const uint64_t lo = p > g.window_tokens ? p - g.window_tokens + 1 : 1;
      for (uint64_t i = lo; i <= p; ++i) out.push_back(i);
      break;
    }
    case LayerKind::kMamba:
      if (p % g.checkpoint_interval_tokens == 0) out.push_back(p);
      else if (defined) *defined = false;
      break;
    case LayerKind::kVisionEmbedding:
      break;
  }
  return out;
}

// reference layer_policies.cpp:42-77
PrefixRangeSet possible_prefixes(const LayerGroupSpec& g, const std::vector<bool>& is_hit) {
  const uint64_t n = is_hit.size();
  PrefixRangeSet out;
  switch (g.kind) {
    case LayerKind::kFullAttention:
    case LayerKind::kCrossAttention: {
      uint64_t run = 0;
      while (run < n && is_hit[run]) ++run;
      if (run >= 1) out.append_range(1, run);
      break;
    }
    case LayerKind::kSlidingWindow: {
      // maximal runs of valid p appended whole (same set as appending each p)
      uint64_t run = 0, open = 0;
      for (uint64_t p = 1; p <= n; ++p) {
        run = is_hit[p - 1] ? run + 1 : 0;
        const bool ok = run >= std::min(g.window_tokens, p);
        if (ok && open == 0) open = p;
        if (!ok && open != 0) {
          out.append_range(open, p - 1);
          open = 0;
        }
      }
      if (open != 0) out.append_range(open, n);
      break;
    }
    case LayerKind::kMamba: {
      const uint64_t k = g.checkpoint_interval_tokens;
      for (uint64_t p = k; p <= n; p += k)
        if (is_hit[p - 1]) out.append(p);
      break;
    }
    case LayerKind::kVisionEmbedding:
      if (n >= 1) out.append_range(1, n);
      break;
  }
  return out;
}

// reference prefix_cache.cpp:25-47: global prefix p contains stored ordinals
// 1..c(p); valid when c(p) is 0 or a valid stored prefix.
PrefixRangeSet stored_to_global_prefixes(const PrefixRangeSet& valid, const std::vector<uint64_t>& stored,
                                         uint64_t sequence_length) {
  PrefixRangeSet out;
  if (sequence_length == 0) return out;
  const uint64_t m = stored.size();
  uint64_t prev_hi = 0;
  // counts rise monotonically: walk valid's ranges alongside instead of a binary
  // search per count
  const auto& vr = valid.ranges();
  size_t vi = 0;
  for (uint64_t count = 0; count <= m; ++count) {
    const uint64_t lo = count == 0 ? 1 : stored[count - 1];
    const uint64_t hi = count == m ? sequence_length : stored[count] - 1;
    if (lo > hi) continue;
    while (vi < vr.size() && vr[vi].second < count) ++vi;
    const bool in_valid = vi < vr.size() && count >= vr[vi].first;
    if (count == 0 || in_valid) {
      JENGA_CHECK(lo > prev_hi, "stored positions out of order");
      out.append_range(lo, hi);
      prev_hi = hi;
    }
  }
  return out;
}

// reference prefix_cache.cpp:49-57
uint64_t find_longest_common_prefix(const std::vector<PrefixRangeSet>& per_group) {
  if (per_group.empty()) return 0;
  PrefixRangeSet acc = per_group.front();
  for (size_t i = 1; i < per_group.size(); ++i) acc = PrefixRangeSet::intersect(acc, per_group[i]);
  return acc.max_value();
}

// reference kv_allocator.cpp:241-303
LookupResult KvAllocator::lookup_and_pin(const std::vector<GroupLookupInput>& inputs, uint64_t sequence_length,
                                         uint64_t request) {
  JENGA_CHECK(inputs.size() == num_groups(), "one lookup input per group");
  LookupResult out;
  out.pinned.resize(num_groups());
  if (sequence_length == 0) return out;
  std::vector<PrefixRangeSet> global_sets;
  global_sets.reserve(num_groups());
  for (size_t g = 0; g < num_groups(); ++g) {
    const auto& in = inputs[g];
    const uint64_t m = in.stored_positions.size();
    std::vector<bool> is_hit(m, false);
    uint64_t ordinal = 0;
    for (size_t b = 0; b < in.blocks.size(); ++b) {
      const uint64_t end = in.block_end_ordinal[b];
      JENGA_CHECK(end <= m, "block covers unknown ordinals");
      if (cache_.find(g, in.blocks[b]).has_value())
        for (uint64_t i = ordinal; i < end; ++i) is_hit[i] = true;
      ordinal = end;
    }
    global_sets.push_back(
        stored_to_global_prefixes(possible_prefixes(spec_.groups[g], is_hit), in.stored_positions, sequence_length));
  }
  const uint64_t p = find_longest_common_prefix(global_sets);
  if (p == 0) return out;
  out.hit_length = p;
  for (size_t g = 0; g < num_groups(); ++g) {
    const auto& in = inputs[g];
    const uint64_t m = static_cast<uint64_t>(
        std::upper_bound(in.stored_positions.begin(), in.stored_positions.end(), p) - in.stored_positions.begin());
    if (m == 0) continue;
    // required_tokens(g, m) is one contiguous ordinal range per kind (empty for
    // vision): pin every block that holds one of them, in block order -- the blocks
    // the reference's per-ordinal walk pins, without materialising the ordinals
    const LayerGroupSpec& gs = spec_.groups[g];
    uint64_t ord_lo = 1, ord_hi = m;
    switch (gs.kind) {
      case LayerKind::kFullAttention:
      case LayerKind::kCrossAttention:
        break;
      case LayerKind::kSlidingWindow:
        ord_lo = m > gs.window_tokens ? m - gs.window_tokens + 1 : 1;
        break;
      case LayerKind::kMamba:
        JENGA_CHECK(m % gs.checkpoint_interval_tokens == 0, "common prefix invalid for a group policy");
        ord_lo = m;
        break;
      case LayerKind::kVisionEmbedding:
        ord_lo = 1;
        ord_hi = 0;  // nothing required
        break;
    }
    if (ord_lo > ord_hi) continue;
    const auto& be = in.block_end_ordinal;
    const uint64_t b_lo = static_cast<uint64_t>(std::lower_bound(be.begin(), be.end(), ord_lo) - be.begin());
    const uint64_t b_hi = static_cast<uint64_t>(std::lower_bound(be.begin(), be.end(), ord_hi) - be.begin());
    JENGA_CHECK(b_hi < in.blocks.size(), "required ordinal beyond blocks");
    for (uint64_t b = b_lo; b <= b_hi; ++b) {
      auto page = cache_.find(g, in.blocks[b]);
      JENGA_CHECK(page.has_value(), "hit block vanished before pinning");
      pin(g, *page, request);
      out.pinned[g].emplace_back(b, *page);
    }
  }
  return out;
}

}  // namespace jenga
