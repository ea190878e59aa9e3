// extern "C" boundary for the host half of include/jenga_gpu.h.  Every entry
// catches the C++ exceptions of the reference convention and returns the
// matching status; the message is kept per thread for jenga_last_error().
#include <cstring>
#include <string>

#include "../../../include/jenga_gpu.h"
#include "jenga_host.hpp"

#define JENGA_EXPORT extern "C" __attribute__((visibility("default")))

namespace {
thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return JENGA_OK;
  } catch (const jenga::ConfigError& e) {
    return fail(JENGA_ERR_CONFIG, e.what());
  } catch (const jenga::InvariantError& e) {
    return fail(JENGA_ERR_INVARIANT, e.what());
  } catch (const std::bad_alloc&) {
    return fail(JENGA_ERR_CONFIG, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(JENGA_ERR_INVARIANT, e.what());
  }
}

jenga::SmallPageId to_id(jenga_small_page p) {
  return jenga::SmallPageId{jenga::LargePageId{p.large}, p.slot};
}
jenga_small_page to_c(jenga::SmallPageId p) { return jenga_small_page{p.large.index, p.slot}; }

}  // namespace

// Used by the device half (kernels/*.cu) to report launch failures.
namespace jenga_host_err {
int set(int code, const char* msg) { return fail(code, msg ? msg : ""); }
}  // namespace jenga_host_err

struct jenga_spec {
  jenga::ModelSpec spec;
};
struct jenga_kv {
  std::unique_ptr<jenga::KvAllocator> kv;
};
struct jenga_addr {
  std::unique_ptr<jenga::AddressMap> map;
};
struct jenga_pages {
  std::unique_ptr<jenga::PageLists> pl;
  jenga::KvAllocator* kv;
  std::vector<jenga_checkpoint_copy> pending_copies;  // drained, not yet handed out
};

#define ARG_CHECK(cond) \
  if (!(cond)) return fail(JENGA_ERR_ARG, "invalid argument: " #cond)

JENGA_EXPORT int jenga_abi_version(void) { return JENGA_ABI_VERSION; }
JENGA_EXPORT const char* jenga_last_error(void) { return g_last_error.c_str(); }

// ------------------------------------------------------------ spec
JENGA_EXPORT int jenga_spec_create(const char* name, jenga_spec** out) {
  ARG_CHECK(out != nullptr);
  return guarded([&] {
    auto* s = new jenga_spec;
    s->spec.name = name ? name : "unnamed";
    *out = s;
  });
}

JENGA_EXPORT int jenga_spec_from_json(const char* json_text, jenga_spec** out) {
  ARG_CHECK(out != nullptr && json_text != nullptr);
  return guarded([&] {
    auto spec = jenga::parse_model_spec_json(json_text);
    auto* s = new jenga_spec;
    s->spec = std::move(spec);
    *out = s;
  });
}

JENGA_EXPORT void jenga_spec_destroy(jenga_spec* spec) { delete spec; }

JENGA_EXPORT int jenga_spec_add_group(jenga_spec* spec, const char* name, int kind,
                                      uint32_t num_layers, uint64_t bptl, uint32_t tpp,
                                      uint64_t window, uint64_t ckpt) {
  ARG_CHECK(spec != nullptr && name != nullptr);
  if (kind < 0 || kind > 4) return fail(JENGA_ERR_CONFIG, "unknown layer kind");
  return guarded([&] {
    jenga::LayerGroupSpec g;
    g.name = name;
    g.kind = static_cast<jenga::LayerKind>(kind);
    g.num_layers = num_layers;
    g.bytes_per_token_per_layer = bptl;
    g.tokens_per_page = tpp;
    g.window_tokens = window;
    g.checkpoint_interval_tokens = ckpt;
    spec->spec.groups.push_back(std::move(g));
  });
}

// reference combine_with_draft (simulator.cpp:32-41): the target's groups
// followed by the draft's, renamed "draft.<name>", validated.
JENGA_EXPORT int jenga_spec_combine_with_draft(const jenga_spec* target, const jenga_spec* draft, jenga_spec** out) {
  ARG_CHECK(target != nullptr && draft != nullptr && out != nullptr);
  return guarded([&] {
    auto* s = new jenga_spec;
    s->spec = target->spec;
    s->spec.name = target->spec.name + "+draft";
    for (jenga::LayerGroupSpec g : draft->spec.groups) {
      g.name = "draft." + g.name;
      s->spec.groups.push_back(std::move(g));
    }
    try {
      s->spec.validate();
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

JENGA_EXPORT int jenga_spec_validate(const jenga_spec* spec) {
  ARG_CHECK(spec != nullptr);
  return guarded([&] { spec->spec.validate(); });
}

JENGA_EXPORT int jenga_spec_num_groups(const jenga_spec* spec) {
  return spec ? static_cast<int>(spec->spec.groups.size()) : -1;
}

JENGA_EXPORT int jenga_spec_small_page_size(const jenga_spec* spec, int g, uint64_t* out) {
  ARG_CHECK(spec != nullptr && out != nullptr);
  ARG_CHECK(g >= 0 && static_cast<size_t>(g) < spec->spec.groups.size());
  return guarded([&] { *out = jenga::small_page_size(spec->spec.groups[g]); });
}

JENGA_EXPORT int jenga_spec_lcm_page_size(const jenga_spec* spec, uint64_t* out) {
  ARG_CHECK(spec != nullptr && out != nullptr);
  return guarded([&] { *out = jenga::lcm_page_size(spec->spec); });
}

JENGA_EXPORT int jenga_spec_lcm_blowup_ratio(const jenga_spec* spec, double* out) {
  ARG_CHECK(spec != nullptr && out != nullptr);
  return guarded([&] { *out = jenga::lcm_blowup_ratio(spec->spec); });
}

// ------------------------------------------------------------ address map
JENGA_EXPORT int jenga_addr_create(const jenga_spec* spec, jenga_addr** out) {
  ARG_CHECK(spec != nullptr && out != nullptr);
  return guarded([&] {
    auto m = std::make_unique<jenga::AddressMap>(spec->spec);
    auto* a = new jenga_addr;
    a->map = std::move(m);
    *out = a;
  });
}

JENGA_EXPORT void jenga_addr_destroy(jenga_addr* map) { delete map; }

JENGA_EXPORT uint64_t jenga_addr_large_page_bytes(const jenga_addr* map) {
  return map ? map->map->large_page_bytes() : 0;
}

JENGA_EXPORT int jenga_addr_group_info(const jenga_addr* map, int g, uint64_t* small,
                                       uint64_t* per_layer, uint32_t* slots) {
  ARG_CHECK(map != nullptr);
  if (g < 0 || static_cast<size_t>(g) >= map->map->num_groups())
    return fail(JENGA_ERR_INVARIANT, "group index out of range");
  if (small) *small = map->map->small_page_bytes(g);
  if (per_layer) *per_layer = map->map->per_layer_bytes(g);
  if (slots) *slots = map->map->slots_per_large(g);
  return JENGA_OK;
}

JENGA_EXPORT int jenga_addr_global_page_index(const jenga_addr* map, int g,
                                              jenga_small_page page, uint64_t* out) {
  ARG_CHECK(map != nullptr && out != nullptr && g >= 0);
  return guarded([&] { *out = map->map->global_page_index(g, to_id(page)); });
}

JENGA_EXPORT int jenga_addr_address_of(const jenga_addr* map, int g, uint32_t layer,
                                       jenga_small_page page, jenga_byte_range* out) {
  ARG_CHECK(map != nullptr && out != nullptr && g >= 0);
  return guarded([&] {
    auto r = map->map->address_of(g, layer, to_id(page));
    *out = jenga_byte_range{r.begin, r.end};
  });
}

JENGA_EXPORT int jenga_addr_layer_view(const jenga_addr* map, int g, uint32_t layer,
                                       jenga_layer_view* out) {
  ARG_CHECK(map != nullptr && out != nullptr && g >= 0);
  return guarded([&] {
    auto v = map->map->layer_view(g, layer);
    *out = jenga_layer_view{v.start_offset, v.page_stride, v.exec_page_size};
  });
}

JENGA_EXPORT int jenga_addr_view_address(const jenga_addr* map, int g, uint32_t layer,
                                         jenga_small_page page, jenga_byte_range* out) {
  ARG_CHECK(map != nullptr && out != nullptr && g >= 0);
  return guarded([&] {
    auto r = map->map->view_address(g, layer, to_id(page));
    *out = jenga_byte_range{r.begin, r.end};
  });
}

// ------------------------------------------------------------ allocator
JENGA_EXPORT int jenga_kv_create(const jenga_spec* spec, uint64_t budget, jenga_kv** out) {
  ARG_CHECK(spec != nullptr && out != nullptr);
  return guarded([&] {
    auto kv = std::make_unique<jenga::KvAllocator>(spec->spec, budget);
    auto* k = new jenga_kv;
    k->kv = std::move(kv);
    *out = k;
  });
}

JENGA_EXPORT void jenga_kv_destroy(jenga_kv* kv) { delete kv; }

JENGA_EXPORT int jenga_kv_num_groups(const jenga_kv* kv) {
  return kv ? static_cast<int>(kv->kv->num_groups()) : -1;
}

JENGA_EXPORT int jenga_kv_pool_info(const jenga_kv* kv, uint64_t* large_page_bytes,
                                    uint32_t* num_large_pages, uint64_t* remainder) {
  ARG_CHECK(kv != nullptr);
  const auto& p = kv->kv->pool();
  if (large_page_bytes) *large_page_bytes = p.large_page_bytes();
  if (num_large_pages) *num_large_pages = p.num_pages();
  if (remainder) *remainder = p.reserved_remainder_bytes();
  return JENGA_OK;
}

#define GROUP_CHECK(kvp, g)                                                 \
  if ((g) < 0 || static_cast<size_t>(g) >= (kvp)->kv->num_groups())        \
  return fail(JENGA_ERR_INVARIANT, "group index out of range")

JENGA_EXPORT int jenga_kv_allocate(jenga_kv* kv, int g, uint64_t request,
                                   jenga_small_page* page, int* step) {
  ARG_CHECK(kv != nullptr && page != nullptr);
  GROUP_CHECK(kv, g);
  bool oom = false;
  int rc = guarded([&] {
    auto res = kv->kv->allocate(g, request);
    if (!res) {
      oom = true;
      return;
    }
    *page = to_c(res->page);
    if (step) *step = res->step;
  });
  if (rc == JENGA_OK && oom) return fail(JENGA_ERR_OOM, "out of KV memory");
  return rc;
}

static jenga::BlockContent make_content(uint64_t key, uint64_t parent, const uint64_t* tokens,
                                        size_t n) {
  jenga::BlockContent c;
  c.key = key;
  c.parent_key = parent;
  if (n) c.tokens.assign(tokens, tokens + n);
  return c;
}

JENGA_EXPORT int jenga_kv_free(jenga_kv* kv, int g, jenga_small_page page, int has_content,
                               uint64_t key, uint64_t parent, const uint64_t* tokens,
                               size_t n_tokens) {
  ARG_CHECK(kv != nullptr && (n_tokens == 0 || tokens != nullptr));
  GROUP_CHECK(kv, g);
  return guarded([&] {
    if (has_content)
      kv->kv->free(g, to_id(page), make_content(key, parent, tokens, n_tokens));
    else
      kv->kv->free(g, to_id(page), std::nullopt);
  });
}

JENGA_EXPORT int jenga_kv_pin(jenga_kv* kv, int g, jenga_small_page page, uint64_t request) {
  ARG_CHECK(kv != nullptr);
  GROUP_CHECK(kv, g);
  return guarded([&] { kv->kv->pin(g, to_id(page), request); });
}

JENGA_EXPORT int jenga_kv_evict_lru_large_page(jenga_kv* kv, uint32_t* evicted) {
  ARG_CHECK(kv != nullptr && evicted != nullptr);
  return guarded([&] {
    auto r = kv->kv->evict_lru_large_page();
    *evicted = r ? r->index : UINT32_MAX;
  });
}

JENGA_EXPORT int jenga_kv_touch(jenga_kv* kv, int g, jenga_small_page page, uint64_t step) {
  ARG_CHECK(kv != nullptr);
  GROUP_CHECK(kv, g);
  return guarded([&] { kv->kv->type_allocator(g).touch(to_id(page), step); });
}

JENGA_EXPORT int jenga_kv_set_prefix_length(jenga_kv* kv, int g, jenga_small_page page,
                                            uint64_t len) {
  ARG_CHECK(kv != nullptr);
  GROUP_CHECK(kv, g);
  return guarded([&] { kv->kv->type_allocator(g).set_prefix_length(to_id(page), len); });
}

JENGA_EXPORT int jenga_kv_set_request_aware(jenga_kv* kv, int on) {
  ARG_CHECK(kv != nullptr);
  kv->kv->set_request_aware(on != 0);
  return JENGA_OK;
}

JENGA_EXPORT int jenga_kv_page_record(const jenga_kv* kv, int g, jenga_small_page page,
                                      int* state, uint64_t* assoc, uint64_t* last_access,
                                      uint64_t* prefix_length) {
  ARG_CHECK(kv != nullptr);
  GROUP_CHECK(kv, g);
  return guarded([&] {
    const auto& r = kv->kv->type_allocator(g).record(to_id(page));
    if (state) *state = static_cast<int>(r.state);
    if (assoc) *assoc = r.associated_request;
    if (last_access) *last_access = r.last_access;
    if (prefix_length) *prefix_length = r.prefix_length;
  });
}

JENGA_EXPORT int jenga_kv_cache_find(const jenga_kv* kv, int g, uint64_t key, uint64_t parent,
                                     const uint64_t* tokens, size_t n_tokens, int* found,
                                     jenga_small_page* page) {
  ARG_CHECK(kv != nullptr && found != nullptr && (n_tokens == 0 || tokens != nullptr));
  GROUP_CHECK(kv, g);
  return guarded([&] {
    auto r = kv->kv->cache().find(g, make_content(key, parent, tokens, n_tokens));
    *found = r.has_value() ? 1 : 0;
    if (r && page) *page = to_c(*r);
  });
}

JENGA_EXPORT int jenga_kv_group_counts(const jenga_kv* kv, int g, uint64_t* used,
                                       uint64_t* evictable, uint64_t* empty,
                                       uint64_t* owned_units) {
  ARG_CHECK(kv != nullptr);
  GROUP_CHECK(kv, g);
  const auto& t = kv->kv->type_allocator(g);
  if (used) *used = t.used_pages();
  if (evictable) *evictable = t.evictable_pages();
  if (empty) *empty = t.empty_pages();
  if (owned_units) *owned_units = t.owned_units();
  return JENGA_OK;
}

JENGA_EXPORT int jenga_kv_pool_free_pages(const jenga_kv* kv, uint32_t* num_free) {
  ARG_CHECK(kv != nullptr && num_free != nullptr);
  *num_free = kv->kv->pool().num_free();
  return JENGA_OK;
}

JENGA_EXPORT int jenga_kv_fragmentation(const jenga_kv* kv, int g, uint64_t* used,
                                        uint64_t* evictable, uint64_t* stranded) {
  ARG_CHECK(kv != nullptr);
  GROUP_CHECK(kv, g);
  auto r = kv->kv->type_allocator(g).fragmentation_report();
  if (used) *used = r.used_bytes;
  if (evictable) *evictable = r.evictable_bytes;
  if (stranded) *stranded = r.empty_stranded_bytes;
  return JENGA_OK;
}

JENGA_EXPORT int jenga_kv_alloc_step_counts(const jenga_kv* kv, uint64_t counts[6]) {
  ARG_CHECK(kv != nullptr && counts != nullptr);
  std::memcpy(counts, kv->kv->alloc_step_counts(), 6 * sizeof(uint64_t));
  return JENGA_OK;
}

JENGA_EXPORT int jenga_kv_check_invariants(const jenga_kv* kv) {
  ARG_CHECK(kv != nullptr);
  return guarded([&] { kv->kv->check_invariants(); });
}

// ------------------------------------------------------------ policies
JENGA_EXPORT int jenga_policy_needs_token(const jenga_spec* spec, int g, uint64_t i,
                                          uint64_t new_tokens, uint64_t consumed, int* out) {
  ARG_CHECK(spec != nullptr && out != nullptr);
  ARG_CHECK(g >= 0 && static_cast<size_t>(g) < spec->spec.groups.size());
  return guarded([&] { *out = jenga::needs_token(spec->spec.groups[g], i, new_tokens, consumed); });
}

JENGA_EXPORT int jenga_policy_accessed_range(const jenga_spec* spec, int g, uint64_t prev,
                                             uint64_t new_tokens, uint64_t* lo, uint64_t* hi) {
  ARG_CHECK(spec != nullptr && lo != nullptr && hi != nullptr);
  ARG_CHECK(g >= 0 && static_cast<size_t>(g) < spec->spec.groups.size());
  return guarded([&] {
    auto r = jenga::accessed_range(spec->spec.groups[g], prev, new_tokens);
    *lo = r.first;
    *hi = r.second;
  });
}

// ------------------------------------------------------------ page lists
JENGA_EXPORT int jenga_pages_create(jenga_kv* kv, int prefix_caching, jenga_pages** out) {
  ARG_CHECK(kv != nullptr && out != nullptr);
  return guarded([&] {
    auto* p = new jenga_pages;
    p->pl = std::make_unique<jenga::PageLists>(kv->kv.get(), prefix_caching != 0);
    p->kv = kv->kv.get();
    *out = p;
  });
}

JENGA_EXPORT void jenga_pages_destroy(jenga_pages* pl) { delete pl; }

JENGA_EXPORT int jenga_pages_add_request(jenga_pages* pl, uint64_t request) {
  ARG_CHECK(pl != nullptr);
  return guarded([&] { pl->pl->add_request(request); });
}

JENGA_EXPORT int jenga_pages_append(jenga_pages* pl, uint64_t request, uint64_t token_id,
                                    int is_image, uint64_t image_ordinal, uint64_t now) {
  ARG_CHECK(pl != nullptr);
  bool ok = true;
  int rc = guarded([&] { ok = pl->pl->append(request, token_id, is_image != 0, image_ordinal, now); });
  if (rc == JENGA_OK && !ok) return fail(JENGA_ERR_OOM, "out of KV memory (preempt the request)");
  return rc;
}

JENGA_EXPORT int jenga_pages_append_batch(jenga_pages* pl, const uint64_t* ids, int n,
                                          const uint64_t* token_ids, const uint8_t* is_image, uint64_t now,
                                          int* n_done) {
  ARG_CHECK(pl != nullptr && (n == 0 || ids != nullptr) && n >= 0);
  int done = 0;
  bool ok = true;
  int rc = guarded([&] {
    for (; done < n; ++done) {
      ok = pl->pl->append(ids[done], token_ids ? token_ids[done] : 0, is_image ? is_image[done] != 0 : false, 0,
                          now);
      if (!ok) break;
    }
  });
  if (n_done) *n_done = done;
  if (rc == JENGA_OK && !ok) return fail(JENGA_ERR_OOM, "out of KV memory (preempt the request)");
  return rc;
}

JENGA_EXPORT int jenga_pages_store(jenga_pages* pl, uint64_t request, int g, uint64_t pos,
                                   uint64_t now) {
  ARG_CHECK(pl != nullptr && g >= 0);
  bool ok = true;
  int rc = guarded([&] { ok = pl->pl->store_position(request, g, pos, now); });
  if (rc == JENGA_OK && !ok) return fail(JENGA_ERR_OOM, "out of KV memory (preempt the request)");
  return rc;
}

JENGA_EXPORT int jenga_pages_release(jenga_pages* pl, uint64_t request, int allow_cache,
                                     uint64_t now) {
  ARG_CHECK(pl != nullptr);
  return guarded([&] { pl->pl->release(request, allow_cache != 0, now); });
}

JENGA_EXPORT int jenga_pages_admit(jenga_pages* pl, uint64_t request, const uint64_t* tokens,
                                   const uint8_t* is_image, const uint64_t* image_ordinals, uint64_t n,
                                   uint64_t now, uint64_t* hit) {
  ARG_CHECK(pl != nullptr && (n == 0 || tokens != nullptr));
  bool oom = false;
  const int rc = guarded([&] {
    std::vector<uint64_t> t(tokens, tokens + n);
    std::vector<uint8_t> img = is_image ? std::vector<uint8_t>(is_image, is_image + n) : std::vector<uint8_t>();
    std::vector<uint64_t> ord =
        image_ordinals ? std::vector<uint64_t>(image_ordinals, image_ordinals + n) : std::vector<uint64_t>();
    const uint64_t h = pl->pl->admit(request, t, img, ord, now, &oom);
    if (hit) *hit = h;
  });
  if (rc == JENGA_OK && oom) return fail(JENGA_ERR_OOM, "out of KV memory at admission (preempt the request)");
  return rc;
}

JENGA_EXPORT int jenga_pages_set_vision_mode(jenga_pages* pl, int mode) {
  ARG_CHECK(pl != nullptr && (mode == 0 || mode == 1));
  return guarded([&] { pl->pl->set_vision_mode(static_cast<jenga::PageLists::VisionMode>(mode)); });
}

JENGA_EXPORT int jenga_pages_rollback_newest(jenga_pages* pl, uint64_t request, int g, uint64_t count,
                                             uint64_t now) {
  ARG_CHECK(pl != nullptr && g >= 0);
  return guarded([&] { pl->pl->rollback_newest(request, static_cast<size_t>(g), count, now); });
}

JENGA_EXPORT int jenga_pages_speculative_decode(jenga_pages* pl, uint64_t request, uint32_t propose_k,
                                                uint64_t accepted, const uint64_t* target_tokens,
                                                uint64_t n_target, uint64_t now) {
  ARG_CHECK(pl != nullptr);
  bool ok = true;
  int rc = guarded([&] { ok = pl->pl->speculative_decode(request, propose_k, accepted, target_tokens, n_target, now); });
  if (rc == JENGA_OK && !ok) return fail(JENGA_ERR_OOM, "out of KV memory (preempt the request)");
  return rc;
}

JENGA_EXPORT int jenga_pages_is_draft_group(const jenga_pages* pl, int g, int* is_draft) {
  ARG_CHECK(pl != nullptr && is_draft != nullptr && g >= 0);
  return guarded([&] { *is_draft = pl->pl->is_draft_group(static_cast<size_t>(g)) ? 1 : 0; });
}

JENGA_EXPORT int jenga_pages_prefill(jenga_pages* pl, uint64_t request, uint64_t budget, uint64_t now,
                                     uint64_t* consumed) {
  ARG_CHECK(pl != nullptr);
  bool oom = false;
  int rc = guarded([&] {
    const uint64_t c = pl->pl->prefill(request, budget, now, &oom);
    if (consumed) *consumed = c;
  });
  if (rc == JENGA_OK && oom) return fail(JENGA_ERR_OOM, "out of KV memory during prefill (preempt the request)");
  return rc;
}

JENGA_EXPORT int jenga_pages_restore_pending(const jenga_pages* pl, uint64_t request, int g, int* has,
                                             jenga_small_page* checkpoint) {
  ARG_CHECK(pl != nullptr && has != nullptr && g >= 0);
  return guarded([&] {
    const auto& r = pl->pl->request(request);
    *has = (static_cast<size_t>(g) < r.restore.size() && r.restore[g].has_value()) ? 1 : 0;
    if (*has && checkpoint) *checkpoint = to_c(*r.restore[g]);
  });
}

JENGA_EXPORT int jenga_pages_finish_restore(jenga_pages* pl, uint64_t request, int g, uint64_t now) {
  ARG_CHECK(pl != nullptr && g >= 0);
  return guarded([&] { pl->pl->finish_restore(request, static_cast<size_t>(g), now); });
}

JENGA_EXPORT int jenga_pages_take_checkpoint_copies(jenga_pages* pl, jenga_checkpoint_copy* out, int capacity,
                                                   int* n) {
  ARG_CHECK(pl != nullptr && n != nullptr && capacity >= 0 && (capacity == 0 || out != nullptr));
  return guarded([&] {
    auto& pending = pl->pending_copies;
    auto fresh = pl->pl->take_checkpoint_copies();
    for (auto& c : fresh)
      pending.push_back(jenga_checkpoint_copy{c.request, c.g, 0, c.ordinal, to_c(c.working), to_c(c.checkpoint)});
    const int take = std::min<int>(capacity, static_cast<int>(pending.size()));
    for (int i = 0; i < take; ++i) out[i] = pending[i];
    pending.erase(pending.begin(), pending.begin() + take);
    *n = take;
  });
}

JENGA_EXPORT int jenga_pages_set_fix_mamba_restore(jenga_pages* pl, int on) {
  ARG_CHECK(pl != nullptr);
  pl->pl->fix_mamba_restore = on != 0;
  return JENGA_OK;
}

JENGA_EXPORT int jenga_pages_set_defer_window_free(jenga_pages* pl, uint64_t request, int on) {
  ARG_CHECK(pl != nullptr);
  return guarded([&] { pl->pl->set_defer_window_free(request, on != 0); });
}

JENGA_EXPORT int jenga_pages_apply_window_free(jenga_pages* pl, uint64_t request, uint64_t now) {
  ARG_CHECK(pl != nullptr);
  return guarded([&] { pl->pl->apply_window_free(request, now); });
}

JENGA_EXPORT int jenga_kv_cache_entries(const jenga_kv* kv, int g, uint64_t* n) {
  ARG_CHECK(kv != nullptr && n != nullptr);
  GROUP_CHECK(kv, g);
  return guarded([&] { *n = kv->kv->cache().entries(g); });
}

JENGA_EXPORT int jenga_pages_seq_len(const jenga_pages* pl, uint64_t request, uint64_t* len) {
  ARG_CHECK(pl != nullptr && len != nullptr);
  return guarded([&] { *len = pl->pl->request(request).tokens.size(); });
}

JENGA_EXPORT int jenga_pages_group_state(const jenga_pages* pl, uint64_t request, int g,
                                         uint64_t* stored, uint64_t* num_blocks,
                                         uint64_t* freed_blocks, uint64_t* held_tokens,
                                         int* has_working, jenga_small_page* working) {
  ARG_CHECK(pl != nullptr && g >= 0);
  return guarded([&] {
    const auto& r = pl->pl->request(request);
    JENGA_CHECK(static_cast<size_t>(g) < r.groups.size(), "group index out of range");
    const auto& rt = r.groups[g];
    if (stored) *stored = rt.stored;
    if (num_blocks) *num_blocks = rt.blocks.size();
    if (freed_blocks) *freed_blocks = rt.freed_blocks;
    if (held_tokens) *held_tokens = rt.held_tokens;
    if (has_working) *has_working = rt.working_page.has_value() ? 1 : 0;
    if (working && rt.working_page) *working = to_c(*rt.working_page);
  });
}

JENGA_EXPORT int jenga_pages_blocks(const jenga_pages* pl, uint64_t request, int g,
                                    jenga_small_page* pages, uint8_t* live, uint64_t capacity,
                                    uint64_t* n) {
  ARG_CHECK(pl != nullptr && n != nullptr && g >= 0);
  return guarded([&] {
    const auto& r = pl->pl->request(request);
    JENGA_CHECK(static_cast<size_t>(g) < r.groups.size(), "group index out of range");
    const auto& blocks = r.groups[g].blocks;
    *n = blocks.size();
    for (uint64_t i = 0; i < blocks.size() && i < capacity; ++i) {
      if (pages) pages[i] = to_c(blocks[i].page);
      if (live) live[i] = blocks[i].live ? 1 : 0;
    }
  });
}

JENGA_EXPORT int jenga_pages_pack_csr(const jenga_pages* pl, int g, const uint64_t* requests,
                                      int n_req, int max_blocks, int64_t pages_capacity, int32_t* offsets,
                                      jenga_small_page* pages, int32_t* first_live, int32_t* n_stored) {
  ARG_CHECK(pl != nullptr && requests != nullptr && offsets != nullptr && n_req >= 0 && g >= 0);
  ARG_CHECK(pages == nullptr || pages_capacity >= 0);
  return guarded([&] {
    JENGA_CHECK(static_cast<size_t>(g) < pl->kv->num_groups(), "group index out of range");
    const bool mamba = pl->kv->group(g).kind == jenga::LayerKind::kMamba;
    // Block tables hold int32 AddressMap global indices (large*slots_per_large + slot).
    JENGA_CHECK(uint64_t{pl->kv->pool().num_pages()} * pl->kv->type_allocator(g).geometry().slots_per_large <=
                    uint64_t{INT32_MAX},
                "pool too large for int32 global page indices");
    // Pass 1: count and validate everything before writing a byte, so an
    // undersized caller buffer is rejected instead of overrun.
    int64_t off = 0;
    offsets[0] = 0;
    for (int i = 0; i < n_req; ++i) {
      const auto& r = pl->pl->request(requests[i]);
      JENGA_CHECK(static_cast<size_t>(g) < r.groups.size(), "group index out of range");
      const auto& rt = r.groups[g];
      const int64_t cnt = mamba ? (rt.working_page ? 1 : 0) : static_cast<int64_t>(rt.blocks.size());
      if (max_blocks > 0 && cnt > max_blocks)
        throw jenga::ConfigError("request " + std::to_string(requests[i]) + " holds " + std::to_string(cnt) +
                                 " blocks; the block table is " + std::to_string(max_blocks) + " wide");
      if (!mamba) {
        // the device table marks blocks [0, freed_blocks) dead and every later one
        // live: a hole after the first live block would hand a freed page to a kernel
        for (int64_t b = static_cast<int64_t>(rt.freed_blocks); b < cnt; ++b)
          JENGA_CHECK(rt.blocks[b].live, "dead block after the first live block");
      }
      off += cnt;
      JENGA_CHECK(off <= INT32_MAX, "page list too long for int32 offsets");
      offsets[i + 1] = static_cast<int32_t>(off);
    }
    if (pages != nullptr && off > pages_capacity)
      throw jenga::ConfigError("page lists need " + std::to_string(off) + " entries; the buffer holds " +
                               std::to_string(pages_capacity));
    // Pass 2: write.
    for (int i = 0; i < n_req; ++i) {
      const auto& rt = pl->pl->request(requests[i]).groups[g];
      const int64_t o = offsets[i];
      if (pages) {
        if (mamba) {
          if (rt.working_page) pages[o] = to_c(*rt.working_page);
        } else {
          for (int64_t b = 0, cnt = offsets[i + 1] - o; b < cnt; ++b) pages[o + b] = to_c(rt.blocks[b].page);
        }
      }
      if (first_live) first_live[i] = mamba ? 0 : static_cast<int32_t>(rt.freed_blocks);
      if (n_stored) n_stored[i] = static_cast<int32_t>(rt.stored);
    }
  });
}

// ------------------------------------------------------------------------
// Delta page-list upload.  A decode step changes at most
// two entries of a (request, group) row — the block store_position appended
// (simulator.cpp:248-253) and a sliding-window block it freed (:272-280) — so
// instead of re-packing every list, a host mirror of what the device table
// holds diffs each row against the page lists and emits only the changed
// entries, plus every row's seq_len and newest-token slot.
struct jenga_table_mirror {
  const jenga_pages* pl = nullptr;
  int g = 0;
  int max_batch = 0, max_blocks = 0;
  uint32_t slots_per_large = 1, tpp = 1;
  bool mamba = false;
  struct Row {
    uint64_t request = UINT64_MAX;  // none
    uint64_t epoch = 0;
    int64_t count = 0, first_live = 0;
  };
  std::vector<Row> rows;
  int n_rows = 0;  // rows the last pack described
  std::vector<int32_t> rec;  // staging: (flat index, value) pairs
  // The last packed buffer and its sequence number: the device writes the
  // number back (header word 4) when it applies the buffer, so a pack whose
  // predecessor was never applied (overwritten, or packed before a graph
  // capture and never replayed) knows the device table is not what the
  // mirror says, and rewrites every row over the full width instead.
  const volatile int32_t* last_buf = nullptr;
  int32_t last_seq = 0;
  void invalidate() {
    for (auto& r : rows) r = Row{UINT64_MAX - 1, 0, max_blocks, 0};
    n_rows = max_batch;
  }
};

namespace {
// int32 n_records, n_rows, max_blocks, seq, ack (device-written), 3 x reserved
constexpr size_t kDeltaHeader = 32;
// header | int64 slots[n_rows] | int32 seq_lens[n_rows] (+4 B pad when n_rows is
// odd, so the (int32, int32) records are 8-byte aligned) | records
size_t records_offset(int n_rows) { return kDeltaHeader + static_cast<size_t>(n_rows) * 12 + (n_rows & 1) * 4; }
size_t delta_bytes(int n_rows, size_t n_records) { return records_offset(n_rows) + n_records * 8; }
}  // namespace

JENGA_EXPORT size_t jenga_delta_bytes(int n_rows, int n_records) {
  if (n_rows < 0 || n_records < 0) return 0;
  return delta_bytes(n_rows, static_cast<size_t>(n_records));
}

JENGA_EXPORT size_t jenga_delta_buffer_bytes(int max_batch, int max_blocks) {
  if (max_batch < 0 || max_blocks < 0) return 0;
  // worst case: every row rewritten in full, twice its width (old + new length)
  return delta_bytes(max_batch, 2 * static_cast<size_t>(max_batch) * static_cast<size_t>(max_blocks));
}

JENGA_EXPORT int jenga_table_mirror_create(const jenga_pages* pl, int g, int max_batch, int max_blocks,
                                           jenga_table_mirror** out) {
  ARG_CHECK(pl != nullptr && out != nullptr && g >= 0 && max_batch >= 0 && max_blocks > 0);
  return guarded([&] {
    JENGA_CHECK(static_cast<size_t>(g) < pl->kv->num_groups(), "group index out of range");
    JENGA_CHECK(int64_t{max_batch} * max_blocks <= INT32_MAX, "block table too large for int32 entry indices");
    const auto& geo = pl->kv->type_allocator(g).geometry();
    JENGA_CHECK(uint64_t{pl->kv->pool().num_pages()} * geo.slots_per_large <= uint64_t{INT32_MAX},
                "pool too large for int32 global page indices");
    auto m = std::make_unique<jenga_table_mirror>();
    m->pl = pl;
    m->g = g;
    m->max_batch = max_batch;
    m->max_blocks = max_blocks;
    m->slots_per_large = geo.slots_per_large;
    m->tpp = pl->kv->group(g).tokens_per_page;
    m->mamba = pl->kv->group(g).kind == jenga::LayerKind::kMamba;
    m->rows.assign(max_batch, jenga_table_mirror::Row{});
    *out = m.release();
  });
}

JENGA_EXPORT void jenga_table_mirror_destroy(jenga_table_mirror* m) { delete m; }

JENGA_EXPORT int jenga_table_mirror_reset(jenga_table_mirror* m) {
  ARG_CHECK(m != nullptr);
  // the device table is assumed all -1 again (a freshly filled table)
  for (auto& r : m->rows) r = jenga_table_mirror::Row{};
  m->n_rows = 0;
  m->last_buf = nullptr;
  m->last_seq = 0;
  return JENGA_OK;
}

JENGA_EXPORT int jenga_pages_pack_deltas(jenga_table_mirror* m, const uint64_t* requests, int n_req, void* delta,
                                         size_t capacity_bytes, size_t* used_bytes, int* n_records) {
  ARG_CHECK(m != nullptr && (n_req == 0 || requests != nullptr) && n_req >= 0 && delta != nullptr);
  return guarded([&] {
    if (n_req > m->max_batch)
      throw jenga::ConfigError("batch of " + std::to_string(n_req) + " exceeds the mirror's " +
                               std::to_string(m->max_batch) + " rows");
    const int g = m->g;
    const int64_t W = m->max_blocks;
    if (m->last_buf != nullptr && m->last_buf[4] != m->last_seq) m->invalidate();
    m->rec.clear();
    auto global_of = [&](const jenga::SmallPageId& p) {
      return static_cast<int32_t>(uint64_t{p.large.index} * m->slots_per_large + p.slot);
    };
    struct RowOut {
      int32_t seq;
      int64_t slot;
      jenga_table_mirror::Row next;
    };
    std::vector<RowOut> outs(std::max(n_req, m->n_rows));
    // Pass 1: diff every row into the staging records; the mirror itself is only
    // updated once the caller's buffer is known to be large enough.
    for (int i = 0; i < n_req; ++i) {
      const auto& r = m->pl->pl->request(requests[i]);
      JENGA_CHECK(static_cast<size_t>(g) < r.groups.size(), "group index out of range");
      const auto& rt = r.groups[g];
      const int64_t cnt = m->mamba ? (rt.working_page ? 1 : 0) : static_cast<int64_t>(rt.blocks.size());
      const int64_t fl = m->mamba ? 0 : static_cast<int64_t>(rt.freed_blocks);
      if (cnt > W)
        throw jenga::ConfigError("request " + std::to_string(requests[i]) + " holds " + std::to_string(cnt) +
                                 " blocks; the block table is " + std::to_string(W) + " wide");
      if (!m->mamba)
        for (int64_t b = fl; b < cnt; ++b) JENGA_CHECK(rt.blocks[b].live, "dead block after the first live block");
      auto value = [&](int64_t b) -> int32_t {
        if (b < fl || b >= cnt) return -1;
        return global_of(m->mamba ? *rt.working_page : rt.blocks[b].page);
      };
      const auto& old = m->rows[i];
      const int64_t base = static_cast<int64_t>(i) * W;
      const bool full = old.request != r.id || old.epoch != rt.epoch || cnt < old.count || fl < old.first_live;
      if (full) {
        for (int64_t b = 0, end = std::max(cnt, old.count); b < end; ++b) {
          m->rec.push_back(static_cast<int32_t>(base + b));
          m->rec.push_back(value(b));
        }
      } else {
        for (int64_t b = old.first_live, end = std::min(fl, old.count); b < end; ++b) {  // newly dead
          m->rec.push_back(static_cast<int32_t>(base + b));
          m->rec.push_back(-1);
        }
        for (int64_t b = old.count; b < cnt; ++b) {  // appended
          m->rec.push_back(static_cast<int32_t>(base + b));
          m->rec.push_back(value(b));
        }
      }
      // newest stored ordinal's slot (exactly jenga_build_block_tables' rule)
      int64_t slot = -1;
      const int64_t n = static_cast<int64_t>(rt.stored);
      if (n > 0) {
        const int64_t blk = (n - 1) / m->tpp;
        if (blk < cnt && blk >= fl) slot = int64_t{value(blk)} * m->tpp + (n - 1) % m->tpp;
      }
      JENGA_CHECK(n <= INT32_MAX, "sequence too long for int32 seq_lens");
      outs[i] = RowOut{static_cast<int32_t>(n), slot, jenga_table_mirror::Row{r.id, rt.epoch, cnt, fl}};
    }
    for (int i = n_req; i < m->n_rows; ++i) {  // rows that left the batch: clear them
      const auto& old = m->rows[i];
      for (int64_t b = 0; b < old.count; ++b) {
        m->rec.push_back(static_cast<int32_t>(int64_t{i} * W + b));
        m->rec.push_back(-1);
      }
      outs[i] = RowOut{0, -1, jenga_table_mirror::Row{}};
    }
    const int rows_out = static_cast<int>(outs.size());
    const size_t nrec = m->rec.size() / 2;
    const size_t need = delta_bytes(rows_out, nrec);
    if (used_bytes) *used_bytes = need;
    if (n_records) *n_records = static_cast<int>(nrec);
    if (need > capacity_bytes)
      throw jenga::ConfigError("delta needs " + std::to_string(need) + " bytes; the buffer holds " +
                               std::to_string(capacity_bytes));
    JENGA_CHECK(nrec <= static_cast<size_t>(INT32_MAX), "too many delta records");
    // Pass 2: write the buffer, then commit the mirror.
    auto* w = static_cast<uint8_t*>(delta);
    int64_t* slots = reinterpret_cast<int64_t*>(w + kDeltaHeader);
    int32_t* seqs = reinterpret_cast<int32_t*>(w + kDeltaHeader + 8 * static_cast<size_t>(rows_out));
    int32_t* recs = reinterpret_cast<int32_t*>(w + records_offset(rows_out));
    for (int i = 0; i < rows_out; ++i) {
      slots[i] = outs[i].slot;
      seqs[i] = outs[i].seq;
    }
    if (nrec) std::memcpy(recs, m->rec.data(), nrec * 8);
    int32_t* hdr = reinterpret_cast<int32_t*>(w);
    m->last_seq = m->last_seq == INT32_MAX ? 1 : m->last_seq + 1;
    hdr[0] = static_cast<int32_t>(nrec);
    hdr[1] = rows_out;
    hdr[2] = m->max_blocks;
    hdr[3] = m->last_seq;
    hdr[4] = 0;  // ack: the applying kernel writes seq here
    hdr[5] = hdr[6] = hdr[7] = 0;
    for (int i = 0; i < rows_out; ++i) m->rows[i] = outs[i].next;
    m->n_rows = n_req;
    m->last_buf = reinterpret_cast<const volatile int32_t*>(w);
  });
}
