// Page-layer address map and per-kind liveness policies.
#include "jenga_host.hpp"

namespace jenga {

// reference memory_layout.cpp:10-20: large = LCM; per group the small page,
// the per-layer slice (bytes/token/layer x tokens/page) and slots per large page.
AddressMap::AddressMap(const ModelSpec& spec) : spec_(spec) {
  spec_.validate();
  large_ = lcm_page_size(spec_);
  for (const auto& g : spec_.groups) {
    const uint64_t s = small_page_size(g);
    small_.push_back(s);
    per_layer_.push_back(checked_mul(g.bytes_per_token_per_layer, g.tokens_per_page,
                                     "per_layer_bytes"));
    slots_.push_back(static_cast<uint32_t>(large_ / s));
  }
}

// reference memory_layout.cpp:22-27
uint64_t AddressMap::global_page_index(size_t g, SmallPageId p) const {
  JENGA_CHECK(g < num_groups(), "group index out of range");
  JENGA_CHECK(p.slot < slots_[g], "slot out of range");
  return uint64_t{p.large.index} * slots_[g] + p.slot;
}

// reference memory_layout.cpp:29-39
ByteRange AddressMap::address_of(size_t g, uint32_t layer, SmallPageId p) const {
  JENGA_CHECK(g < num_groups(), "group index out of range");
  JENGA_CHECK(layer < spec_.groups[g].num_layers, "layer index out of range");
  JENGA_CHECK(p.slot < slots_[g], "slot out of range");
  const uint64_t begin =
      uint64_t{p.large.index} * large_ + uint64_t{p.slot} * small_[g] + uint64_t{layer} * per_layer_[g];
  return ByteRange{begin, begin + per_layer_[g]};
}

// reference memory_layout.cpp:41-47
LayerView AddressMap::layer_view(size_t g, uint32_t layer) const {
  JENGA_CHECK(g < num_groups(), "group index out of range");
  JENGA_CHECK(layer < spec_.groups[g].num_layers, "layer index out of range");
  return LayerView{uint64_t{layer} * per_layer_[g], small_[g], per_layer_[g]};
}

// reference memory_layout.cpp:49-55
ByteRange AddressMap::view_address(size_t g, uint32_t layer, SmallPageId p) const {
  const LayerView v = layer_view(g, layer);
  const uint64_t begin = v.start_offset + global_page_index(g, p) * v.page_stride;
  return ByteRange{begin, begin + v.exec_page_size};
}

// reference layer_policies.cpp:105-120
bool needs_token(const LayerGroupSpec& g, uint64_t i, uint64_t new_tokens,
                 uint64_t consumed_tokens) {
  JENGA_CHECK(i >= 1 && i <= new_tokens, "needs_token: ordinal out of range");
  switch (g.kind) {
    case LayerKind::kFullAttention:
    case LayerKind::kCrossAttention: return true;
    case LayerKind::kSlidingWindow: return i + g.window_tokens > new_tokens;
    case LayerKind::kMamba: return i == new_tokens;
    case LayerKind::kVisionEmbedding: return i > consumed_tokens;
  }
  return true;
}

// reference layer_policies.cpp:79-103
std::pair<uint64_t, uint64_t> accessed_range(const LayerGroupSpec& g, uint64_t prev_tokens,
                                             uint64_t new_tokens) {
  if (new_tokens == 0) return {1, 0};
  switch (g.kind) {
    case LayerKind::kFullAttention:
    case LayerKind::kCrossAttention:
    case LayerKind::kVisionEmbedding: return {1, new_tokens};
    case LayerKind::kSlidingWindow: {
      const uint64_t first_new = prev_tokens + 1;
      const uint64_t lo = first_new > g.window_tokens ? first_new - g.window_tokens + 1 : 1;
      return {lo, new_tokens};
    }
    case LayerKind::kMamba: {
      const uint64_t k = g.checkpoint_interval_tokens;
      const uint64_t ckpt = (new_tokens / k) * k;
      if (ckpt == 0) return {1, 0};
      return {ckpt, ckpt};
    }
  }
  return {1, 0};
}

}  // namespace jenga
