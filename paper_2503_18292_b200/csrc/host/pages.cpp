// Per-request page lists: the producer of every block table.  Semantics are
// those of the reference simulator's GroupRuntime bookkeeping (cited per
// method); scheduling, metrics and preemption policy stay with the caller.
#include <algorithm>

#include "jenga_host.hpp"

namespace jenga {

PageLists::PageLists(KvAllocator* kv, bool prefix_caching)
    : kv_(kv), prefix_caching_(prefix_caching) {
  JENGA_CHECK(kv_ != nullptr, "page lists need an allocator");
  for (size_t g = 0; g < kv_->num_groups(); ++g)  // simulator.cpp:76-78
    draft_flags_.push_back(kv_->group(g).name.rfind("draft.", 0) == 0 ? 1 : 0);
}

void PageLists::add_request(uint64_t id) {
  if (index_.count(id)) throw ConfigError("duplicate request id " + std::to_string(id));
  index_[id] = requests_.size();
  Request r;
  r.id = id;
  reset_groups(r);
  r.restore.assign(kv_->num_groups(), std::nullopt);
  requests_.push_back(std::move(r));
}

void PageLists::reset_groups(Request& r) {
  r.groups.assign(kv_->num_groups(), GroupRuntime{});
  for (GroupRuntime& rt : r.groups) bump(rt);
}

PageLists::Request& PageLists::req(uint64_t id) {
  auto it = index_.find(id);
  JENGA_CHECK(it != index_.end(), "unknown request");
  return requests_[it->second];
}

const PageLists::Request& PageLists::request(uint64_t id) const {
  auto it = index_.find(id);
  JENGA_CHECK(it != index_.end(), "unknown request");
  return requests_[it->second];
}

// reference simulator.cpp:151-158
bool PageLists::group_stores_position(size_t g, const Request& r, uint64_t pos) const {
  const LayerGroupSpec& grp = kv_->group(g);
  const bool image = r.is_image[pos - 1] != 0;
  if (grp.stores_image_tokens()) return image;
  return !image || kv_->spec().decoder_stores_images();
}

// reference simulator.cpp:196-215
void PageLists::append_chain(Request& r, size_t g) {
  if (!prefix_caching_) return;
  GroupRuntime& rt = r.groups[g];
  const LayerGroupSpec& grp = kv_->group(g);
  const uint64_t t = grp.kind == LayerKind::kMamba ? grp.checkpoint_interval_tokens
                                                   : grp.tokens_per_page;
  while ((rt.chain.size() + 1) * t <= rt.stored) {
    BlockContent c;
    c.parent_key = rt.chain.empty() ? block_chain_salt(grp.name) : rt.chain.back().key;
    const uint64_t first = rt.chain.size() * t;
    c.tokens.reserve(t);
    for (uint64_t i = 0; i < t; ++i) c.tokens.push_back(r.tokens[rt.stored_positions[first + i] - 1]);
    c.key = chain_block_key(c.parent_key, c.tokens);
    rt.chain.push_back(std::move(c));
  }
}

// reference simulator.cpp:217-282
bool PageLists::store_position(uint64_t id, size_t g, uint64_t pos, uint64_t now) {
  return store_position(req(id), g, pos, now);
}

// the request already resolved (the per-position loops of append / prefill)
bool PageLists::store_position(Request& r, size_t g, uint64_t pos, uint64_t now) {
  const uint64_t id = r.id;
  JENGA_CHECK(g < r.groups.size(), "group index out of range");
  const LayerGroupSpec& grp = kv_->group(g);
  // draft groups record draft-sequence ordinals (simulator.cpp:603-607)
  JENGA_CHECK(pos >= 1 && (draft_flags_[g] || pos <= r.tokens.size()), "position beyond the sequence");
  GroupRuntime& rt = r.groups[g];
  TypeAllocator& ta = kv_->type_allocator(g);

  if (grp.kind == LayerKind::kMamba) {
    if (!rt.working_page.has_value()) {
      auto res = kv_->allocate(g, id);
      if (!res) return false;
      rt.working_page = res->page;
      ta.set_prefix_length(*rt.working_page, 0);
    }
    rt.stored++;
    rt.stored_positions.push_back(pos);
    append_chain(r, g);
    const uint64_t k = grp.checkpoint_interval_tokens;
    if (prefix_caching_ && rt.stored % k == 0) {
      auto res = kv_->allocate(g, id);
      if (!res) return false;
      ta.set_prefix_length(res->page, pos);
      ta.touch(res->page, now);
      rt.checkpoints = rt.stored / k;
      kv_->free(g, res->page, rt.chain[rt.checkpoints - 1]);
      checkpoint_copies_.push_back(CheckpointCopy{id, static_cast<uint32_t>(g), rt.stored, *rt.working_page,
                                                  res->page, rt.chain[rt.checkpoints - 1]});
    }
    return true;
  }

  rt.stored++;
  rt.stored_positions.push_back(pos);
  const uint64_t t = grp.tokens_per_page;
  const uint64_t bidx = (rt.stored - 1) / t;
  if (bidx >= rt.blocks.size()) {
    auto res = kv_->allocate(g, id);
    if (!res) {
      // Leave the ordinal un-stored so a retry after preemption is clean.
      rt.stored--;
      rt.stored_positions.pop_back();
      return false;
    }
    rt.blocks.push_back(Block{res->page, true});
    rt.live_blocks++;
  } else {
    JENGA_CHECK(rt.blocks[bidx].live, "stored into a dead block");
  }
  rt.held_tokens++;
  append_chain(r, g);
  const uint64_t ordinal_value = grp.stores_image_tokens() ? r.image_ordinal[pos - 1] : pos;
  ta.set_prefix_length(rt.blocks[bidx].page, ordinal_value);

  if (grp.kind == LayerKind::kSlidingWindow && !r.defer_window_free && !r.suppress_window_free) {
    const uint64_t w = grp.window_tokens;
    if (rt.stored > w) {
      const uint64_t exited = rt.stored - w;
      while (rt.freed_blocks * t + t <= exited) free_block(r, g, rt.freed_blocks, true, now);
    }
  }
  return true;
}

// reference simulator.cpp:284-312
void PageLists::free_block(Request& r, size_t g, uint64_t b, bool allow_cache, uint64_t now) {
  GroupRuntime& rt = r.groups[g];
  JENGA_CHECK(b < rt.blocks.size(), "free of unknown block");
  Block& blk = rt.blocks[b];
  JENGA_CHECK(blk.live, "free of a dead block");
  const uint64_t t = kv_->group(g).tokens_per_page;
  const uint64_t covered = std::min(rt.stored, (b + 1) * t) - b * t;
  kv_->type_allocator(g).touch(blk.page, now);
  const bool cacheable = allow_cache && prefix_caching_ && b < rt.chain.size();
  if (cacheable) kv_->free(g, blk.page, rt.chain[b]);
  else kv_->free(g, blk.page, std::nullopt);
  blk.live = false;
  rt.live_blocks--;
  rt.held_tokens -= covered;
  if (kv_->group(g).kind == LayerKind::kVisionEmbedding) rt.consumed_held -= std::min(rt.consumed_held, covered);
  while (rt.freed_blocks < rt.blocks.size() && !rt.blocks[rt.freed_blocks].live) rt.freed_blocks++;
}

// reference simulator.cpp:549-566 (decode_one) / 504-523 (prefill_some):
// one position, every storing group in group order; vision-embedding groups
// are driven separately by the caller (jenga_pages_store).
bool PageLists::append(uint64_t id, uint64_t token, bool is_image, uint64_t image_ordinal,
                       uint64_t now) {
  refresh_mamba_checkpoints(id, now);  // decode_one, simulator.cpp:551
  Request& r = req(id);
  JENGA_CHECK(!r.needs_release, "append after OOM: release (preempt) the request first");
  r.tokens.push_back(token);
  r.is_image.push_back(is_image ? 1 : 0);
  r.image_ordinal.push_back(image_ordinal);
  const uint64_t pos = r.tokens.size();
  for (size_t g = 0; g < kv_->num_groups(); ++g) {
    if (kv_->group(g).kind == LayerKind::kVisionEmbedding) continue;
    if (!group_stores_position(g, r, pos)) continue;
    if (!store_position(r, g, pos, now)) {
      // The reference pops the token on a failed decode (simulator.cpp:557-561).
      Request& rr = req(id);
      rr.tokens.pop_back();
      rr.is_image.pop_back();
      rr.image_ordinal.pop_back();
      rr.needs_release = true;
      return false;
    }
  }
  return true;
}

// reference simulator.cpp:360-389
std::vector<GroupLookupInput> PageLists::build_lookup_inputs(const Request& r) const {
  std::vector<GroupLookupInput> inputs(kv_->num_groups());
  for (size_t g = 0; g < kv_->num_groups(); ++g) {
    GroupLookupInput& in = inputs[g];
    const LayerGroupSpec& grp = kv_->group(g);
    in.stored_positions.reserve(r.prompt_len);
    for (uint64_t pos = 1; pos <= r.prompt_len; ++pos)
      if (group_stores_position(g, r, pos)) in.stored_positions.push_back(pos);
    if (grp.kind == LayerKind::kVisionEmbedding) continue;  // never cached
    const uint64_t t = grp.kind == LayerKind::kMamba ? grp.checkpoint_interval_tokens : grp.tokens_per_page;
    const uint64_t full_blocks = in.stored_positions.size() / t;
    in.blocks.reserve(full_blocks);
    in.block_end_ordinal.reserve(full_blocks);
    for (uint64_t b = 0; b < full_blocks; ++b) {
      BlockContent c;
      c.tokens.reserve(t);
      for (uint64_t i = 0; i < t; ++i) c.tokens.push_back(r.tokens[in.stored_positions[b * t + i] - 1]);
      in.blocks.push_back(std::move(c));
      in.block_end_ordinal.push_back((b + 1) * t);
    }
  }
  // Block-chain keys (chain_block_key: one serially dependent mix per token).
  // Groups holding the same tokens block for block (same block size, same
  // stored positions; e.g. a full and a sliding-window group over a text
  // prompt) differ only in their salt: their chains run interleaved, two
  // independent dependency chains per loop, with each token's mix shared.
  std::vector<bool> done(kv_->num_groups(), false);
  for (size_t g = 0; g < kv_->num_groups(); ++g) {
    if (done[g] || inputs[g].blocks.empty()) continue;
    done[g] = true;
    size_t h = g + 1;
    for (; h < kv_->num_groups(); ++h)
      if (!done[h] && inputs[h].block_end_ordinal == inputs[g].block_end_ordinal &&
          inputs[h].stored_positions == inputs[g].stored_positions)
        break;
    auto& a = inputs[g].blocks;
    uint64_t ka = block_chain_salt(kv_->group(g).name);
    if (h == kv_->num_groups()) {
      for (BlockContent& c : a) {
        c.parent_key = ka;
        c.key = ka = chain_block_key(ka, c.tokens);
      }
      continue;
    }
    done[h] = true;
    auto& b = inputs[h].blocks;
    uint64_t kb = block_chain_salt(kv_->group(h).name);
    for (size_t i = 0; i < a.size(); ++i) {
      a[i].parent_key = ka;
      b[i].parent_key = kb;
      for (const uint64_t tok : a[i].tokens) {
        const uint64_t m = mix64(tok);  // chain_block_key's per-token step: mix64(k ^ mix64(tok))
        ka = mix64(ka ^ m);
        kb = mix64(kb ^ m);
      }
      a[i].key = ka;
      b[i].key = kb;
    }
  }
  return inputs;
}

// reference simulator.cpp:435-452 (admit) + 391-433 (adopt_lookup_result)
uint64_t PageLists::admit(uint64_t id, const std::vector<uint64_t>& tokens, const std::vector<uint8_t>& is_image,
                          const std::vector<uint64_t>& image_ordinals, uint64_t now, bool* oom) {
  if (oom) *oom = false;
  Request& r = req(id);
  JENGA_CHECK(is_image.empty() || is_image.size() == tokens.size(), "is_image length mismatch");
  r.tokens = tokens;
  r.is_image = is_image.empty() ? std::vector<uint8_t>(tokens.size(), 0) : is_image;
  r.image_ordinal = image_ordinals.size() == tokens.size() ? image_ordinals : std::vector<uint64_t>(tokens.size(), 0);
  r.prompt_len = tokens.size();
  r.consumed = 0;
  reset_groups(r);
  r.restore.assign(kv_->num_groups(), std::nullopt);
  r.needs_release = false;
  r.suppress_window_free = false;
  r.draft_len = 0;
  // image spans: maximal runs of image positions of one image (one ordinal);
  // the reference keeps them per trace segment (simulator.cpp:130-137)
  r.images.clear();
  for (uint64_t pos = 1; pos <= r.prompt_len; ++pos) {
    if (!r.is_image[pos - 1]) continue;
    if (!r.images.empty() && r.images.back().end == pos - 1 && r.image_ordinal[pos - 2] == r.image_ordinal[pos - 1])
      r.images.back().end = pos;
    else
      r.images.push_back(ImageSpan{pos, pos});
  }
  const uint64_t hit = prefix_caching_ ? adopt_prefix(r, now) : 0;
  r.consumed = hit;
  // reference simulator.cpp:453-476
  if (vision_mode_ == VisionMode::kAllocateOnDemand) {
    // encode: embeddings of every image the hit does not fully cover
    for (size_t g = 0; g < kv_->num_groups(); ++g) {
      if (kv_->group(g).kind != LayerKind::kVisionEmbedding) continue;
      for (const ImageSpan& img : r.images) {
        if (img.end <= r.consumed) continue;
        for (uint64_t pos = img.begin; pos <= img.end; ++pos) {
          if (!store_position(id, g, pos, now)) {
            req(id).needs_release = true;
            if (oom) *oom = true;
            return hit;
          }
        }
      }
    }
  } else {
    // all prompt KV up front; embeddings overlay the unwritten pages
    r.suppress_window_free = true;
    for (uint64_t pos = r.consumed + 1; pos <= r.prompt_len; ++pos) {
      for (size_t g = 0; g < kv_->num_groups(); ++g) {
        if (kv_->group(g).kind == LayerKind::kVisionEmbedding) continue;
        if (!group_stores_position(g, req(id), pos)) continue;
        if (!store_position(id, g, pos, now)) {
          req(id).needs_release = true;
          if (oom) *oom = true;
          return hit;
        }
      }
    }
  }
  Request& rr = req(id);
  if (rr.consumed >= rr.prompt_len) finish_prefill(rr, now);
  return hit;
}

// reference simulator.cpp:441-448 (lookup) + 391-433 (adopt_lookup_result)
uint64_t PageLists::adopt_prefix(Request& r, uint64_t now) {
  (void)now;
  const uint64_t id = r.id;
  const auto inputs = build_lookup_inputs(r);
  const LookupResult res = kv_->lookup_and_pin(inputs, r.prompt_len, id);
  const uint64_t hit = res.hit_length;
  if (hit == 0) return 0;
  for (size_t g = 0; g < kv_->num_groups(); ++g) {
    GroupRuntime& rt = r.groups[g];
    const GroupLookupInput& in = inputs[g];
    const LayerGroupSpec& grp = kv_->group(g);
    const uint64_t m = static_cast<uint64_t>(
        std::upper_bound(in.stored_positions.begin(), in.stored_positions.end(), hit) - in.stored_positions.begin());
    if (grp.kind == LayerKind::kVisionEmbedding) continue;
    rt.stored = m;
    rt.stored_positions.assign(in.stored_positions.begin(), in.stored_positions.begin() + m);
    if (grp.kind == LayerKind::kMamba) {
      const uint64_t k = grp.checkpoint_interval_tokens;
      JENGA_CHECK(m % k == 0, "mamba hit not on a checkpoint boundary");
      rt.checkpoints = m / k;
      rt.chain.assign(in.blocks.begin(), in.blocks.begin() + rt.checkpoints);
      // The checkpoint page lookup_and_pin pinned: the state to restore.
      if (fix_mamba_restore && !res.pinned[g].empty()) r.restore[g] = res.pinned[g].back().second;
      continue;
    }
    const uint64_t t = grp.tokens_per_page;
    const uint64_t covering = (m + t - 1) / t;
    rt.blocks.assign(covering, Block{});
    rt.chain.assign(in.blocks.begin(), in.blocks.begin() + std::min<uint64_t>(covering, in.blocks.size()));
    for (const auto& [b, page] : res.pinned[g]) {
      JENGA_CHECK(b < covering, "pinned block beyond hit prefix");
      rt.blocks[b] = Block{page, true};
      rt.live_blocks++;
      rt.held_tokens += std::min(m, (b + 1) * t) - b * t;
    }
    while (rt.freed_blocks < rt.blocks.size() && !rt.blocks[rt.freed_blocks].live) rt.freed_blocks++;
  }
  return hit;
}

// reference simulator.cpp:504-547 (text path)
uint64_t PageLists::prefill(uint64_t id, uint64_t budget, uint64_t now, bool* oom) {
  Request& r = req(id);
  if (oom) *oom = false;
  const bool prealloc = vision_mode_ == VisionMode::kFullyAllocatedReuse;
  uint64_t done = 0;
  while (done < budget && r.consumed < r.prompt_len) {
    const uint64_t pos = r.consumed + 1;
    for (size_t g = 0; g < kv_->num_groups(); ++g) {
      if (kv_->group(g).kind == LayerKind::kVisionEmbedding) continue;
      if (prealloc) continue;  // pages already exist
      if (!group_stores_position(g, r, pos)) continue;
      const GroupRuntime& rt = r.groups[g];
      if (!rt.stored_positions.empty() && pos <= rt.stored_positions.back()) continue;  // pinned block
      if (!store_position(r, g, pos, now)) {
        r.needs_release = true;
        if (oom) *oom = true;
        return done;
      }
    }
    r.consumed++;
    done++;
    // consume the vision embeddings of image positions as they prefill
    if (vision_mode_ == VisionMode::kAllocateOnDemand && r.is_image[pos - 1]) {
      for (size_t g = 0; g < kv_->num_groups(); ++g) {
        const LayerGroupSpec& grp = kv_->group(g);
        if (grp.kind != LayerKind::kVisionEmbedding) continue;
        GroupRuntime& rt = r.groups[g];
        rt.consumed_ordinals++;
        rt.consumed_held++;
        const uint64_t t = grp.tokens_per_page;
        while (rt.freed_blocks < rt.blocks.size() && rt.blocks[rt.freed_blocks].live &&
               std::min(rt.stored, (rt.freed_blocks + 1) * t) <= rt.consumed_ordinals)
          free_block(r, g, rt.freed_blocks, /*allow_cache=*/false, now);
      }
    }
  }
  refresh_mamba_checkpoints(id, now);
  if (r.consumed >= r.prompt_len) finish_prefill(r, now);
  return done;
}

// reference simulator.cpp:484-502: the deferred out-of-window frees once the
// prompt is written (a caller-held defer_window_free keeps them pending).
void PageLists::finish_prefill(Request& r, uint64_t now) {
  if (!r.suppress_window_free) return;
  r.suppress_window_free = false;
  if (r.defer_window_free) return;
  apply_window_free(r.id, now);
}

// reference simulator.cpp:568-597
void PageLists::rollback_newest(uint64_t id, size_t g, uint64_t count, uint64_t now) {
  Request& r = req(id);
  JENGA_CHECK(g < r.groups.size(), "group index out of range");
  GroupRuntime& rt = r.groups[g];
  const LayerGroupSpec& grp = kv_->group(g);
  if (grp.kind == LayerKind::kMamba) {
    const uint64_t drop = std::min(count, rt.stored);
    rt.stored -= drop;
    rt.stored_positions.resize(rt.stored);
    return;
  }
  const uint64_t t = grp.tokens_per_page;
  for (uint64_t i = 0; i < count && rt.stored > 0; ++i) {
    const uint64_t bidx = (rt.stored - 1) / t;
    rt.stored--;
    rt.stored_positions.pop_back();
    if (bidx < rt.blocks.size() && rt.blocks[bidx].live) {
      rt.held_tokens--;
      if (rt.stored <= bidx * t) {  // block emptied out: drop the page
        kv_->type_allocator(g).touch(rt.blocks[bidx].page, now);
        kv_->free(g, rt.blocks[bidx].page, std::nullopt);
        rt.blocks[bidx].live = false;
        rt.live_blocks--;
        rt.blocks.pop_back();
        bump(rt);
      }
    }
  }
  while (!rt.chain.empty() && rt.chain.size() * t > rt.stored) rt.chain.pop_back();
}

// reference simulator.cpp:600-640
bool PageLists::speculative_decode(uint64_t id, uint32_t propose_k, uint64_t accepted, const uint64_t* target_tokens,
                                   uint64_t n_target, uint64_t now) {
  JENGA_CHECK(accepted <= propose_k, "accepted more tokens than proposed");
  JENGA_CHECK(n_target <= std::max<uint64_t>(accepted, 1), "more target tokens than max(accepted, 1)");
  {
    Request& r = req(id);
    JENGA_CHECK(!r.needs_release, "decode after OOM: release (preempt) the request first");
  }
  for (uint32_t i = 1; i <= propose_k; ++i) {
    const uint64_t pos = req(id).draft_len + i;
    for (size_t g = 0; g < kv_->num_groups(); ++g) {
      if (!draft_flags_[g]) continue;
      if (!store_position(id, g, pos, now)) {
        req(id).needs_release = true;
        return false;
      }
    }
  }
  for (size_t g = 0; g < kv_->num_groups(); ++g)
    if (draft_flags_[g]) rollback_newest(id, g, propose_k - accepted, now);
  req(id).draft_len += accepted;
  for (uint64_t j = 0; j < n_target; ++j) {
    Request& r = req(id);
    r.tokens.push_back(target_tokens ? target_tokens[j] : 0);
    r.is_image.push_back(0);
    r.image_ordinal.push_back(0);
    const uint64_t pos = r.tokens.size();
    for (size_t g = 0; g < kv_->num_groups(); ++g) {
      if (draft_flags_[g]) continue;
      if (!group_stores_position(g, req(id), pos)) continue;
      if (!store_position(id, g, pos, now)) {
        Request& rr = req(id);
        rr.tokens.pop_back();
        rr.is_image.pop_back();
        rr.image_ordinal.pop_back();
        rr.needs_release = true;
        return false;
      }
    }
  }
  return true;
}

// reference simulator.cpp:347-358
void PageLists::refresh_mamba_checkpoints(uint64_t id, uint64_t now) {
  if (!prefix_caching_) return;
  Request& r = req(id);
  for (size_t g = 0; g < kv_->num_groups(); ++g) {
    if (kv_->group(g).kind != LayerKind::kMamba) continue;
    GroupRuntime& rt = r.groups[g];
    if (rt.checkpoints == 0 || rt.chain.size() < rt.checkpoints) continue;
    auto page = kv_->cache().find(g, rt.chain[rt.checkpoints - 1]);
    if (page.has_value()) kv_->type_allocator(g).touch(*page, now);
  }
}

void PageLists::apply_window_free(uint64_t id, uint64_t now) {
  Request& r = req(id);
  for (size_t g = 0; g < kv_->num_groups(); ++g) {
    const LayerGroupSpec& grp = kv_->group(g);
    if (grp.kind != LayerKind::kSlidingWindow) continue;
    GroupRuntime& rt = r.groups[g];
    if (rt.stored <= grp.window_tokens) continue;
    const uint64_t t = grp.tokens_per_page;
    const uint64_t exited = rt.stored - grp.window_tokens;
    while (rt.freed_blocks * t + t <= exited) free_block(r, g, rt.freed_blocks, true, now);
  }
}

void PageLists::finish_restore(uint64_t id, size_t g, uint64_t now) {
  Request& r = req(id);
  JENGA_CHECK(g < r.restore.size() && r.restore[g].has_value(), "no pending Mamba restore");
  GroupRuntime& rt = r.groups[g];
  JENGA_CHECK(rt.checkpoints >= 1 && rt.chain.size() >= rt.checkpoints, "restore without a checkpoint chain");
  const SmallPageId page = *r.restore[g];
  kv_->type_allocator(g).touch(page, now);
  kv_->free(g, page, rt.chain[rt.checkpoints - 1]);  // back to the cache as the same checkpoint
  r.restore[g].reset();
}

std::vector<PageLists::CheckpointCopy> PageLists::take_checkpoint_copies() {
  std::vector<CheckpointCopy> out;
  for (CheckpointCopy& c : checkpoint_copies_) {
    // still registered under its key <=> not evicted (and so not re-allocated)
    const auto page = kv_->cache().find(c.g, c.key);
    if (page.has_value() && *page == c.checkpoint) out.push_back(std::move(c));
  }
  checkpoint_copies_.clear();
  return out;
}

// reference simulator.cpp:314-327
void PageLists::release(uint64_t id, bool allow_cache, uint64_t now) {
  Request& r = req(id);
  for (size_t g = 0; g < kv_->num_groups(); ++g) {
    if (g < r.restore.size() && r.restore[g].has_value()) finish_restore(id, g, now);
    GroupRuntime& rt = r.groups[g];
    for (uint64_t b = 0; b < rt.blocks.size(); ++b)
      if (rt.blocks[b].live) free_block(r, g, b, allow_cache && prefix_caching_, now);
    if (rt.working_page.has_value()) {
      kv_->type_allocator(g).touch(*rt.working_page, now);
      kv_->free(g, *rt.working_page, std::nullopt);
      rt.working_page.reset();
    }
  }
  reset_groups(r);
  r.needs_release = false;
  r.draft_len = 0;
  r.suppress_window_free = false;
}

}  // namespace jenga
