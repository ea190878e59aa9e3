// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.  An extern "C" shim over the
// UNMODIFIED reference library (compiled from the sources under
// /root/reference/proj/src by oracle/build_oracle.py into oracle/_ref/), so
// tests can check the product against the reference itself:
//   * ModelSpec / AddressMap / LayerPolicy / KvAllocator calls, 1:1;
//   * the reference SimEngine, stepped, with its per-request page lists read
//     back (the shim is compiled with `private` mapped to `public` to read
//     SimEngine::requests_ — the reference code itself is untouched);
//   * a page-list driver (rpl_*) restating SimEngine::store_position
//     (simulator.cpp:217-282) over the reference KvAllocator, used to build
//     the bench workload's page lists with the reference's own allocator.
// Never linked into the product.
#include <algorithm>
#include <array>
#include <cstdint>
#include <cstring>
#include <iosfwd>
#include <map>
#include <memory>
#include <optional>
#include <random>
#include <set>
#include <sstream>
#include <stdexcept>
#include <string>
#include <tuple>
#include <unordered_map>
#include <utility>
#include <vector>

#define private public
#include "jenga/kv_allocator.hpp"
#include "jenga/layer_policies.hpp"
#include "jenga/memory_layout.hpp"
#include "jenga/model_config.hpp"
#include "jenga/simulator.hpp"
#include "jenga/trace.hpp"
#undef private

#define EXPORT extern "C" __attribute__((visibility("default")))

using namespace jenga;

namespace {
thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 1;
  } catch (const InvariantError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

struct Spec {
  ModelSpec spec;
};
}  // namespace

EXPORT const char* ref_last_error() { return g_err.c_str(); }

// ------------------------------------------------------------ spec
EXPORT int ref_spec_from_json(const char* text, void** out) {
  return guarded([&] { *out = new Spec{parse_model_spec_json(text)}; });
}
EXPORT void ref_spec_destroy(void* s) { delete static_cast<Spec*>(s); }
EXPORT int ref_small_page_size(void* s, int g, uint64_t* out) {
  return guarded([&] { *out = small_page_size(static_cast<Spec*>(s)->spec.groups.at(g)); });
}
EXPORT int ref_lcm_page_size(void* s, uint64_t* out) {
  return guarded([&] { *out = compatible_page_size(static_cast<Spec*>(s)->spec, PageSizeStrategy::kLcm); });
}
EXPORT int ref_lcm_blowup_ratio(void* s, double* out) {
  return guarded([&] { *out = lcm_blowup_ratio(static_cast<Spec*>(s)->spec); });
}
EXPORT int ref_needs_token(void* s, int g, uint64_t i, uint64_t n, uint64_t consumed, int* out) {
  return guarded([&] {
    LayerPolicy p(static_cast<Spec*>(s)->spec.groups.at(g));
    *out = p.needs_token(i, n, consumed) ? 1 : 0;
  });
}
EXPORT int ref_accessed_range(void* s, int g, uint64_t prev, uint64_t n, uint64_t* lo, uint64_t* hi) {
  return guarded([&] {
    LayerPolicy p(static_cast<Spec*>(s)->spec.groups.at(g));
    auto r = p.accessed_range(prev, n);
    *lo = r.first;
    *hi = r.second;
  });
}

// ------------------------------------------------------------ address map
EXPORT int ref_addr_create(void* s, void** out) {
  return guarded([&] { *out = new AddressMap(static_cast<Spec*>(s)->spec); });
}
EXPORT void ref_addr_destroy(void* a) { delete static_cast<AddressMap*>(a); }
EXPORT int ref_addr_info(void* a, int g, uint64_t* large, uint64_t* small, uint64_t* per_layer, uint32_t* slots) {
  return guarded([&] {
    auto* m = static_cast<AddressMap*>(a);
    *large = m->large_page_bytes();
    *small = m->small_page_bytes(g);
    *per_layer = m->per_layer_bytes(g);
    *slots = m->slots_per_large(g);
  });
}
EXPORT int ref_addr_global(void* a, int g, uint32_t large, uint32_t slot, uint64_t* out) {
  return guarded([&] { *out = static_cast<AddressMap*>(a)->global_page_index(g, SmallPageId{LargePageId{large}, slot}); });
}
EXPORT int ref_addr_address_of(void* a, int g, uint32_t layer, uint32_t large, uint32_t slot, uint64_t* b,
                               uint64_t* e) {
  return guarded([&] {
    auto r = static_cast<AddressMap*>(a)->address_of(g, layer, SmallPageId{LargePageId{large}, slot});
    *b = r.begin;
    *e = r.end;
  });
}
EXPORT int ref_addr_view_address(void* a, int g, uint32_t layer, uint32_t large, uint32_t slot, uint64_t* b,
                                 uint64_t* e) {
  return guarded([&] {
    auto r = static_cast<AddressMap*>(a)->view_address(g, layer, SmallPageId{LargePageId{large}, slot});
    *b = r.begin;
    *e = r.end;
  });
}
EXPORT int ref_addr_layer_view(void* a, int g, uint32_t layer, uint64_t* start, uint64_t* stride, uint64_t* exec) {
  return guarded([&] {
    auto v = static_cast<AddressMap*>(a)->layer_view(g, layer);
    *start = v.start_offset;
    *stride = v.page_stride;
    *exec = v.exec_page_size;
  });
}
EXPORT int ref_addr_dump(void* a, uint32_t large_pages, char* buf, uint64_t cap, uint64_t* len) {
  return guarded([&] {
    std::ostringstream os;
    static_cast<AddressMap*>(a)->dump(os, large_pages);
    const std::string s = os.str();
    *len = s.size();
    if (buf && cap) {
      const uint64_t n = std::min<uint64_t>(cap - 1, s.size());
      std::memcpy(buf, s.data(), n);
      buf[n] = 0;
    }
  });
}

// ------------------------------------------------------------ allocator
EXPORT int ref_kv_create(void* s, uint64_t budget, void** out) {
  return guarded([&] { *out = new KvAllocator(static_cast<Spec*>(s)->spec, AllocStrategy::kJenga, budget); });
}
EXPORT void ref_kv_destroy(void* kv) { delete static_cast<KvAllocator*>(kv); }
EXPORT int ref_kv_pool_info(void* kv, uint64_t* page_bytes, uint32_t* pages, uint64_t* remainder) {
  return guarded([&] {
    auto& p = static_cast<KvAllocator*>(kv)->pool_of(0);
    *page_bytes = p.large_page_bytes();
    *pages = p.num_pages();
    *remainder = p.reserved_remainder_bytes();
  });
}
EXPORT int ref_kv_allocate(void* kv, int g, uint64_t req, uint32_t* large, uint32_t* slot, int* step) {
  int oom = 0;
  int rc = guarded([&] {
    auto r = static_cast<KvAllocator*>(kv)->allocate(g, req);
    if (!r) {
      oom = 1;
      return;
    }
    *large = r->page.large.index;
    *slot = r->page.slot;
    *step = r->step;
  });
  return rc ? rc : (oom ? 3 : 0);
}
static BlockContent content(uint64_t key, uint64_t parent, const uint64_t* toks, uint64_t n) {
  BlockContent c;
  c.key = key;
  c.parent_key = parent;
  if (n) c.tokens.assign(toks, toks + n);
  return c;
}
EXPORT int ref_kv_free(void* kv, int g, uint32_t large, uint32_t slot, int has, uint64_t key, uint64_t parent,
                       const uint64_t* toks, uint64_t n) {
  return guarded([&] {
    std::optional<BlockContent> c;
    if (has) c = content(key, parent, toks, n);
    static_cast<KvAllocator*>(kv)->free(g, SmallPageId{LargePageId{large}, slot}, c);
  });
}
EXPORT int ref_kv_pin(void* kv, int g, uint32_t large, uint32_t slot, uint64_t req) {
  return guarded([&] { static_cast<KvAllocator*>(kv)->pin(g, SmallPageId{LargePageId{large}, slot}, req); });
}
EXPORT int ref_kv_evict(void* kv, uint32_t* out) {
  return guarded([&] {
    auto r = static_cast<KvAllocator*>(kv)->evict_lru_large_page(0);
    *out = r ? r->index : UINT32_MAX;
  });
}
EXPORT int ref_kv_touch(void* kv, int g, uint32_t large, uint32_t slot, uint64_t step) {
  return guarded([&] {
    static_cast<KvAllocator*>(kv)->type_allocator(g).touch(SmallPageId{LargePageId{large}, slot}, step);
  });
}
EXPORT int ref_kv_set_prefix_length(void* kv, int g, uint32_t large, uint32_t slot, uint64_t len) {
  return guarded([&] {
    static_cast<KvAllocator*>(kv)->type_allocator(g).set_prefix_length(SmallPageId{LargePageId{large}, slot}, len);
  });
}
EXPORT int ref_kv_set_request_aware(void* kv, int on) {
  return guarded([&] { static_cast<KvAllocator*>(kv)->set_request_aware(on != 0); });
}
EXPORT int ref_kv_record(void* kv, int g, uint32_t large, uint32_t slot, int* state, uint64_t* assoc,
                         uint64_t* last, uint64_t* prefix) {
  return guarded([&] {
    const auto& r = static_cast<KvAllocator*>(kv)->type_allocator(g).record(SmallPageId{LargePageId{large}, slot});
    *state = static_cast<int>(r.state);
    *assoc = r.associated_request;
    *last = r.last_access;
    *prefix = r.prefix_length;
  });
}
EXPORT int ref_kv_cache_find(void* kv, int g, uint64_t key, uint64_t parent, const uint64_t* toks, uint64_t n,
                             int* found, uint32_t* large, uint32_t* slot) {
  return guarded([&] {
    auto r = static_cast<KvAllocator*>(kv)->cache().find(g, content(key, parent, toks, n));
    *found = r ? 1 : 0;
    if (r) {
      *large = r->large.index;
      *slot = r->slot;
    }
  });
}
EXPORT int ref_kv_counts(void* kv, int g, uint64_t* used, uint64_t* evictable, uint64_t* empty, uint64_t* owned,
                         uint32_t* pool_free) {
  return guarded([&] {
    auto* k = static_cast<KvAllocator*>(kv);
    const auto& t = k->type_allocator(g);
    *used = t.used_pages();
    *evictable = t.evictable_pages();
    *empty = t.empty_pages();
    *owned = t.owned_units();
    *pool_free = k->pool_of(g).num_free();
  });
}
EXPORT int ref_kv_fragmentation(void* kv, int g, uint64_t* used, uint64_t* evictable, uint64_t* stranded) {
  return guarded([&] {
    auto r = static_cast<KvAllocator*>(kv)->type_allocator(g).fragmentation_report();
    *used = r.used_bytes;
    *evictable = r.evictable_bytes;
    *stranded = r.empty_stranded_bytes;
  });
}
EXPORT int ref_kv_has_associated_empty(void* kv, int g, uint64_t req, int* out) {
  return guarded([&] { *out = static_cast<KvAllocator*>(kv)->type_allocator(g).has_associated_empty(req) ? 1 : 0; });
}
EXPORT int ref_kv_check_invariants(void* kv) {
  return guarded([&] { static_cast<KvAllocator*>(kv)->check_invariants(); });
}

// ------------------------------------------------------------ SimEngine
// Text/image segments per request: seg_is_image / seg_tokens flattened, with
// seg_count[r] segments for request r.
EXPORT int ref_sim_create(void* s, uint64_t budget, uint64_t chunk, int prefix_caching, int n_req,
                          const uint64_t* ids, const uint64_t* arrival, const uint64_t* output_tokens,
                          const int* seg_count, const int* seg_is_image, const uint64_t* seg_tokens,
                          const int* prefix_group, void** out) {
  return guarded([&] {
    EngineConfig cfg;
    cfg.memory_budget = budget;
    cfg.chunked_prefill_size = chunk;
    cfg.prefix_caching = prefix_caching != 0;
    Trace tr;
    int k = 0;
    for (int r = 0; r < n_req; ++r) {
      TraceRequest q;
      q.id = ids[r];
      q.arrival_step = arrival[r];
      q.output_tokens = output_tokens[r];
      if (prefix_group && prefix_group[r] >= 0) q.prefix_group = "article-" + std::to_string(prefix_group[r]);
      for (int i = 0; i < seg_count[r]; ++i, ++k) q.segments.push_back(Segment{seg_is_image[k] != 0, seg_tokens[k]});
      tr.requests.push_back(q);
    }
    *out = new SimEngine(static_cast<Spec*>(s)->spec, cfg, tr);
  });
}
// As ref_sim_create plus the vision mode (0 on_demand, 1 full_reuse) and,
// when draft != NULL, a speculative config (SpeculativeConfig, simulator.hpp:
// 30-34) with the engine seed the acceptance draws derive from.
EXPORT int ref_sim_create_ex(void* s, uint64_t budget, uint64_t chunk, int prefix_caching, int n_req,
                             const uint64_t* ids, const uint64_t* arrival, const uint64_t* output_tokens,
                             const int* seg_count, const int* seg_is_image, const uint64_t* seg_tokens,
                             const int* prefix_group, int vision_mode, void* draft, uint32_t propose_k,
                             double acceptance, uint64_t seed, void** out) {
  return guarded([&] {
    EngineConfig cfg;
    cfg.memory_budget = budget;
    cfg.chunked_prefill_size = chunk;
    cfg.prefix_caching = prefix_caching != 0;
    cfg.vision_mode = vision_mode ? VisionMode::kFullyAllocatedReuse : VisionMode::kAllocateOnDemand;
    cfg.seed = seed;
    if (draft) cfg.speculative = SpeculativeConfig{static_cast<Spec*>(draft)->spec, propose_k, acceptance};
    Trace tr;
    int k = 0;
    for (int r = 0; r < n_req; ++r) {
      TraceRequest q;
      q.id = ids[r];
      q.arrival_step = arrival[r];
      q.output_tokens = output_tokens[r];
      if (prefix_group && prefix_group[r] >= 0) q.prefix_group = "article-" + std::to_string(prefix_group[r]);
      for (int i = 0; i < seg_count[r]; ++i, ++k) q.segments.push_back(Segment{seg_is_image[k] != 0, seg_tokens[k]});
      tr.requests.push_back(q);
    }
    *out = new SimEngine(static_cast<Spec*>(s)->spec, cfg, tr);
  });
}
// The acceptance draws of request `id` (simulator.cpp:109, 44-52 restated:
// per request mt19937_64 seeded mix64(seed, mix64(id, 0x5bec)); each draw
// counts successes of propose_k Bernoulli(acceptance) coins).
EXPORT void ref_spec_accept_draws(uint64_t seed, uint64_t id, uint32_t propose_k, double acceptance, int n,
                                  uint64_t* out) {
  std::mt19937_64 rng;
  rng.seed(mix64(seed, mix64(id, 0x5bec)));
  for (int i = 0; i < n; ++i) {
    std::bernoulli_distribution coin(std::clamp(acceptance, 0.0, 1.0));
    uint64_t successes = 0;
    for (uint32_t j = 0; j < propose_k; ++j)
      if (coin(rng)) ++successes;
    out[i] = successes;
  }
}
// The reference draft_len of a request (speculative runs).
EXPORT int ref_sim_draft_len(void* e, uint64_t id, uint64_t* draft_len) {
  return guarded([&] {
    for (auto& r : static_cast<SimEngine*>(e)->requests_) {
      if (r.meta.id != id) continue;
      *draft_len = r.draft_len;
      return;
    }
    throw InvariantError("unknown request");
  });
}
// The reference multi-article prefix trace (trace.cpp:144-169), flattened:
// per request id, arrival, output, prefix group index, and 2 text segments.
EXPORT int ref_gen_multi_article(uint32_t articles, uint32_t questions, uint64_t article_tokens,
                                 uint64_t question_tokens, uint64_t output_tokens, uint64_t spacing, uint64_t seed,
                                 uint64_t* ids, uint64_t* arrival, uint64_t* out_tokens, int* group,
                                 uint64_t* seg_tokens /* [n][2] */, int cap, int* n) {
  return guarded([&] {
    MultiArticleParams p;
    p.num_articles = articles;
    p.questions_per_article = questions;
    p.article_tokens = article_tokens;
    p.question_tokens = question_tokens;
    p.output_tokens = output_tokens;
    p.round_spacing_steps = spacing;
    const Trace t = gen_multi_article_prefix(p, seed);
    *n = static_cast<int>(t.requests.size());
    for (int i = 0; i < *n && i < cap; ++i) {
      const auto& r = t.requests[i];
      ids[i] = r.id;
      arrival[i] = r.arrival_step;
      out_tokens[i] = r.output_tokens;
      group[i] = std::stoi(r.prefix_group->substr(8));
      seg_tokens[2 * i] = r.segments[0].tokens;
      seg_tokens[2 * i + 1] = r.segments[1].tokens;
    }
  });
}
EXPORT void ref_sim_destroy(void* e) { delete static_cast<SimEngine*>(e); }
EXPORT int ref_sim_step(void* e, uint32_t* decode_batch) {
  return guarded([&] { *decode_batch = static_cast<SimEngine*>(e)->step().decode_batch; });
}
EXPORT int ref_sim_done(void* e) { return static_cast<SimEngine*>(e)->done() ? 1 : 0; }
EXPORT uint64_t ref_sim_now(void* e) { return static_cast<SimEngine*>(e)->current_step(); }
EXPORT void* ref_sim_allocator(void* e) { return &static_cast<SimEngine*>(e)->allocator(); }
// phase: 0 waiting, 1 prefill, 2 decode, 3 done
EXPORT int ref_sim_request(void* e, uint64_t id, int* phase, uint64_t* seq_len, uint64_t* consumed) {
  return guarded([&] {
    for (auto& r : static_cast<SimEngine*>(e)->requests_) {
      if (r.meta.id != id) continue;
      *phase = static_cast<int>(r.phase);
      *seq_len = r.tokens.size();
      *consumed = r.consumed;
      return;
    }
    throw InvariantError("unknown request");
  });
}
EXPORT int ref_sim_tokens(void* e, uint64_t id, uint64_t* tokens, uint8_t* is_image, uint64_t cap, uint64_t* n) {
  return guarded([&] {
    for (auto& r : static_cast<SimEngine*>(e)->requests_) {
      if (r.meta.id != id) continue;
      *n = r.tokens.size();
      for (uint64_t i = 0; i < r.tokens.size() && i < cap; ++i) {
        if (tokens) tokens[i] = r.tokens[i];
        if (is_image) is_image[i] = r.is_image[i];
      }
      return;
    }
    throw InvariantError("unknown request");
  });
}
EXPORT int ref_sim_group_state(void* e, uint64_t id, int g, uint32_t* pages /*[cap][2]*/, uint8_t* live, uint64_t cap,
                               uint64_t* n_blocks, uint64_t* stored, uint64_t* freed, int* has_working,
                               uint32_t* working /*[2]*/) {
  return guarded([&] {
    for (auto& r : static_cast<SimEngine*>(e)->requests_) {
      if (r.meta.id != id) continue;
      if (static_cast<size_t>(g) >= r.groups.size()) {
        *n_blocks = 0;
        *stored = 0;
        *freed = 0;
        *has_working = 0;
        return;
      }
      const auto& rt = r.groups[g];
      *n_blocks = rt.blocks.size();
      *stored = rt.stored;
      *freed = rt.freed_blocks;
      *has_working = rt.working_page.has_value() ? 1 : 0;
      if (rt.working_page) {
        working[0] = rt.working_page->large.index;
        working[1] = rt.working_page->slot;
      }
      for (uint64_t i = 0; i < rt.blocks.size() && i < cap; ++i) {
        if (pages) {
          pages[2 * i] = rt.blocks[i].page.large.index;
          pages[2 * i + 1] = rt.blocks[i].page.slot;
        }
        if (live) live[i] = rt.blocks[i].live ? 1 : 0;
      }
      return;
    }
    throw InvariantError("unknown request");
  });
}

// ------------------------------------------------------------ page-list driver
// Restates SimEngine::store_position (simulator.cpp:217-282) and free_block
// (:284-312) without prefix caching, over the reference KvAllocator.
namespace {
struct RBlock {
  SmallPageId page;
  bool live;
};
struct RGroup {
  uint64_t stored = 0, freed = 0;
  std::vector<RBlock> blocks;
  std::optional<SmallPageId> working;
};
struct RReq {
  std::vector<uint8_t> is_image;
  std::vector<RGroup> groups;
};
struct RPL {
  KvAllocator* kv;
  std::unordered_map<uint64_t, RReq> reqs;
};

bool rpl_store(RPL* pl, uint64_t id, RReq& r, size_t g, uint64_t pos, uint64_t now) {
  const LayerGroupSpec& grp = pl->kv->group(g);
  RGroup& rt = r.groups[g];
  if (grp.kind == LayerKind::kMamba) {
    if (!rt.working) {
      auto res = pl->kv->allocate(g, id);
      if (!res) return false;
      rt.working = res->page;
      pl->kv->type_allocator(g).set_prefix_length(*rt.working, 0);
    }
    rt.stored++;
    return true;
  }
  rt.stored++;
  const uint64_t t = grp.tokens_per_page;
  const uint64_t bidx = (rt.stored - 1) / t;
  if (bidx >= rt.blocks.size()) {
    auto res = pl->kv->allocate(g, id);
    if (!res) {
      rt.stored--;
      return false;
    }
    rt.blocks.push_back(RBlock{res->page, true});
  }
  pl->kv->type_allocator(g).set_prefix_length(rt.blocks[bidx].page, pos);
  if (grp.kind == LayerKind::kSlidingWindow && rt.stored > grp.window_tokens) {
    const uint64_t exited = rt.stored - grp.window_tokens;
    while (rt.freed * t + t <= exited) {
      RBlock& blk = rt.blocks[rt.freed];
      pl->kv->type_allocator(g).touch(blk.page, now);
      pl->kv->free(g, blk.page, std::nullopt);
      blk.live = false;
      while (rt.freed < rt.blocks.size() && !rt.blocks[rt.freed].live) rt.freed++;
    }
  }
  return true;
}
}  // namespace

EXPORT void* rpl_create(void* kv) { return new RPL{static_cast<KvAllocator*>(kv), {}}; }
EXPORT void rpl_destroy(void* pl) { delete static_cast<RPL*>(pl); }
// Appends one position to each request in ids[0..n) in order (one decode
// step for the batch).  Returns 3 on OOM.
EXPORT int rpl_append_batch(void* p, const uint64_t* ids, int n, const uint8_t* is_image, uint64_t now) {
  int oom = 0;
  int rc = guarded([&] {
    auto* pl = static_cast<RPL*>(p);
    for (int i = 0; i < n && !oom; ++i) {
      auto it = pl->reqs.find(ids[i]);
      if (it == pl->reqs.end()) {
        RReq r;
        r.groups.resize(pl->kv->num_groups());
        it = pl->reqs.emplace(ids[i], std::move(r)).first;
      }
      RReq& r = it->second;
      const bool img = is_image ? is_image[i] != 0 : false;
      r.is_image.push_back(img ? 1 : 0);
      const uint64_t pos = r.is_image.size();
      bool decoder_images = true;
      for (size_t g = 0; g < pl->kv->num_groups(); ++g)
        if (pl->kv->group(g).kind == LayerKind::kCrossAttention) decoder_images = false;
      for (size_t g = 0; g < pl->kv->num_groups(); ++g) {
        const LayerGroupSpec& grp = pl->kv->group(g);
        if (grp.kind == LayerKind::kVisionEmbedding) continue;
        const bool stores = grp.stores_image_tokens() ? img : (!img || decoder_images);
        if (!stores) continue;
        if (!rpl_store(pl, ids[i], r, g, pos, now)) {
          oom = 1;
          break;
        }
      }
    }
  });
  return rc ? rc : (oom ? 3 : 0);
}
EXPORT int rpl_group_state(void* p, uint64_t id, int g, uint32_t* pages, uint8_t* live, uint64_t cap,
                           uint64_t* n_blocks, uint64_t* stored, uint64_t* freed) {
  return guarded([&] {
    auto* pl = static_cast<RPL*>(p);
    const RGroup& rt = pl->reqs.at(id).groups.at(g);
    *n_blocks = rt.blocks.size();
    *stored = rt.stored;
    *freed = rt.freed;
    for (uint64_t i = 0; i < rt.blocks.size() && i < cap; ++i) {
      if (pages) {
        pages[2 * i] = rt.blocks[i].page.large.index;
        pages[2 * i + 1] = rt.blocks[i].page.slot;
      }
      if (live) live[i] = rt.blocks[i].live ? 1 : 0;
    }
  });
}
// Block table through the reference AddressMap (memory_layout.cpp:22-27):
// table[r][b] = global_page_index for live blocks, -1 otherwise.
EXPORT int rpl_block_table(void* p, void* addr, int g, const uint64_t* ids, int n, int max_blocks, int32_t* table) {
  return guarded([&] {
    auto* pl = static_cast<RPL*>(p);
    auto* m = static_cast<AddressMap*>(addr);
    for (int i = 0; i < n; ++i) {
      const RGroup& rt = pl->reqs.at(ids[i]).groups.at(g);
      for (int b = 0; b < max_blocks; ++b) {
        int32_t v = -1;
        if (static_cast<size_t>(b) < rt.blocks.size() && rt.blocks[b].live)
          v = static_cast<int32_t>(m->global_page_index(g, rt.blocks[b].page));
        table[static_cast<int64_t>(i) * max_blocks + b] = v;
      }
    }
  });
}
// Reference host path timed end to end for the CPU baseline: for every live
// block of every request, resolve the byte range of every layer through
// AddressMap::view_address (what a worker prepares per layer).
EXPORT int rpl_resolve_views(void* p, void* addr, int g, const uint64_t* ids, int n, uint64_t* checksum) {
  return guarded([&] {
    auto* pl = static_cast<RPL*>(p);
    auto* m = static_cast<AddressMap*>(addr);
    const uint32_t layers = pl->kv->group(g).num_layers;
    uint64_t acc = 0;
    for (int i = 0; i < n; ++i) {
      const RGroup& rt = pl->reqs.at(ids[i]).groups.at(g);
      for (const auto& blk : rt.blocks) {
        if (!blk.live) continue;
        for (uint32_t l = 0; l < layers; ++l) acc += m->view_address(g, l, blk.page).begin;
      }
    }
    *checksum = acc;
  });
}
