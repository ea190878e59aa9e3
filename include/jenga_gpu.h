/*
 * jenga_gpu.h — C ABI of the B200-native Jenga KV-cache hot path.
 *
 * This is the drop-in boundary between the reference's host-side allocator /
 * page-table API (the reference headers under proj/include/jenga) and the
 * sm_100a kernels.  Everything here is `extern "C"`, plain pointers and sizes,
 * int status codes, no exceptions and no torch types.  Device launches are
 * asynchronous on a caller-provided cudaStream_t (passed as void*).
 *
 * Two halves:
 *   (1) host API — a C++ re-implementation of the reference's Jenga allocator
 *       (ModelSpec / LargePagePool / TypeAllocator / KvAllocator / AddressMap /
 *       LayerPolicy) plus the per-request page-list runtime that
 *       SimEngine::store_position maintains.  Each entry cites the reference
 *       interface it replaces.
 *   (2) device API — one contiguous HBM arena per GPU, block-table and slot-
 *       mapping construction, reshape_and_cache, paged decode attention
 *       (full / sliding-window / cross), Mamba state gather/scatter and page
 *       copy.
 *
 * Status codes map onto the reference's exception types
 * (reference proj/include/jenga/util.hpp:11-21):
 *   JENGA_ERR_CONFIG    <-> jenga::ConfigError   (config, byte overflow)
 *   JENGA_ERR_INVARIANT <-> jenga::InvariantError (JENGA_CHECK violations)
 *   JENGA_ERR_OOM       <-> std::nullopt from KvAllocator::allocate
 *                           (reference kv_allocator.hpp:77-80)
 * jenga_last_error() returns the message of the last failure on this thread.
 */
#ifndef JENGA_GPU_H_
#define JENGA_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define JENGA_ABI_VERSION 1

enum jenga_status {
  JENGA_OK = 0,
  JENGA_ERR_CONFIG = 1,
  JENGA_ERR_INVARIANT = 2,
  JENGA_ERR_OOM = 3,
  JENGA_ERR_CUDA = 4,
  JENGA_ERR_ARG = 5,
  JENGA_ERR_UNSUPPORTED = 6,
};

/* reference model_config.hpp:15-21 (LayerKind), same numbering. */
enum jenga_layer_kind {
  JENGA_KIND_FULL = 0,
  JENGA_KIND_SLIDING_WINDOW = 1,
  JENGA_KIND_MAMBA = 2,
  JENGA_KIND_CROSS_ATTENTION = 3,
  JENGA_KIND_VISION_EMBEDDING = 4,
};

enum jenga_dtype { JENGA_F32 = 0, JENGA_BF16 = 1, JENGA_F16 = 2 };

/* reference type_allocator.hpp:22-33 (SmallPageId{LargePageId large; u32 slot}). */
typedef struct jenga_small_page {
  uint32_t large;
  uint32_t slot;
} jenga_small_page;

/* reference memory_layout.hpp:14-23 (ByteRange). */
typedef struct jenga_byte_range {
  uint64_t begin;
  uint64_t end;
} jenga_byte_range;

/* reference memory_layout.hpp:25-32 (LayerView) — the kernel contract. */
typedef struct jenga_layer_view {
  uint64_t start_offset;
  uint64_t page_stride;
  uint64_t exec_page_size;
} jenga_layer_view;

typedef struct jenga_spec jenga_spec;       /* ModelSpec */
typedef struct jenga_kv jenga_kv;           /* KvAllocator (Jenga strategy) */
typedef struct jenga_addr jenga_addr;       /* AddressMap */
typedef struct jenga_pages jenga_pages;     /* per-request page lists (SimEngine GroupRuntime) */
typedef struct jenga_arena jenga_arena;     /* one HBM arena per GPU */

int jenga_abi_version(void);
const char* jenga_last_error(void);

/* ------------------------------------------------------------------------
 * ModelSpec — reference model_config.hpp:26-54, model_config.cpp:41-127
 * ---------------------------------------------------------------------- */
int jenga_spec_create(const char* name, jenga_spec** out);
/* Parses the reference's JSON config format (model_config.cpp:196-243). */
int jenga_spec_from_json(const char* json_text, jenga_spec** out);
void jenga_spec_destroy(jenga_spec* spec);
int jenga_spec_add_group(jenga_spec* spec, const char* name, int kind,
                         uint32_t num_layers, uint64_t bytes_per_token_per_layer,
                         uint32_t tokens_per_page, uint64_t window_tokens,
                         uint64_t checkpoint_interval_tokens);
/* reference combine_with_draft (simulator.cpp:32-41): a new spec holding the
 * target's groups then the draft's renamed "draft.<name>" — one LCM pool for
 * both models (speculative decoding). */
int jenga_spec_combine_with_draft(const jenga_spec* target, const jenga_spec* draft, jenga_spec** out);
int jenga_spec_validate(const jenga_spec* spec);
int jenga_spec_num_groups(const jenga_spec* spec);
/* small_page_size(group g) — model_config.cpp:85-89 */
int jenga_spec_small_page_size(const jenga_spec* spec, int g, uint64_t* out);
/* compatible_page_size(spec, kLcm) — model_config.cpp:100-107 */
int jenga_spec_lcm_page_size(const jenga_spec* spec, uint64_t* out);
/* lcm_blowup_ratio — model_config.cpp:129-142 */
int jenga_spec_lcm_blowup_ratio(const jenga_spec* spec, double* out);

/* ------------------------------------------------------------------------
 * AddressMap — reference memory_layout.hpp:34-69, memory_layout.cpp:10-55
 * ---------------------------------------------------------------------- */
int jenga_addr_create(const jenga_spec* spec, jenga_addr** out);
void jenga_addr_destroy(jenga_addr* map);
uint64_t jenga_addr_large_page_bytes(const jenga_addr* map);
int jenga_addr_group_info(const jenga_addr* map, int g, uint64_t* small_page_bytes,
                          uint64_t* per_layer_bytes, uint32_t* slots_per_large);
int jenga_addr_global_page_index(const jenga_addr* map, int g, jenga_small_page page,
                                 uint64_t* out);
int jenga_addr_address_of(const jenga_addr* map, int g, uint32_t layer,
                          jenga_small_page page, jenga_byte_range* out);
int jenga_addr_layer_view(const jenga_addr* map, int g, uint32_t layer,
                          jenga_layer_view* out);
int jenga_addr_view_address(const jenga_addr* map, int g, uint32_t layer,
                            jenga_small_page page, jenga_byte_range* out);

/* ------------------------------------------------------------------------
 * KvAllocator, Jenga strategy — reference kv_allocator.hpp:62-119,
 * kv_allocator.cpp:67-79 (geometry), 154-239 (allocate/free/pin/evict).
 * ---------------------------------------------------------------------- */
int jenga_kv_create(const jenga_spec* spec, uint64_t budget_bytes, jenga_kv** out);
void jenga_kv_destroy(jenga_kv* kv);
int jenga_kv_num_groups(const jenga_kv* kv);
/* EngineGeometry (kv_allocator.hpp:27-35): one LCM pool. */
int jenga_kv_pool_info(const jenga_kv* kv, uint64_t* large_page_bytes,
                       uint32_t* num_large_pages, uint64_t* reserved_remainder);
/* Five-step allocate (kv_allocator.cpp:154-197). JENGA_ERR_OOM = nullopt. */
int jenga_kv_allocate(jenga_kv* kv, int g, uint64_t request, jenga_small_page* page,
                      int* step);
/* free(g, page, cached) (kv_allocator.cpp:199-208). has_content=0 -> nullopt.
 * Content = BlockContent{key, parent_key, tokens} (prefix_cache.hpp:20-29). */
int jenga_kv_free(jenga_kv* kv, int g, jenga_small_page page, int has_content,
                  uint64_t key, uint64_t parent_key, const uint64_t* tokens,
                  size_t n_tokens);
int jenga_kv_pin(jenga_kv* kv, int g, jenga_small_page page, uint64_t request);
/* evict_lru_large_page (kv_allocator.cpp:218-239). *evicted = UINT32_MAX if none. */
int jenga_kv_evict_lru_large_page(jenga_kv* kv, uint32_t* evicted);
int jenga_kv_touch(jenga_kv* kv, int g, jenga_small_page page, uint64_t step);
int jenga_kv_set_prefix_length(jenga_kv* kv, int g, jenga_small_page page, uint64_t len);
int jenga_kv_set_request_aware(jenga_kv* kv, int on);
/* record(id) (type_allocator.hpp:35-42): state 0 Empty, 1 Evictable, 2 Used. */
int jenga_kv_page_record(const jenga_kv* kv, int g, jenga_small_page page, int* state,
                         uint64_t* associated_request, uint64_t* last_access,
                         uint64_t* prefix_length);
/* PrefixCache::find (prefix_cache.cpp:77-87): *found=0 when absent. */
int jenga_kv_cache_find(const jenga_kv* kv, int g, uint64_t key, uint64_t parent_key,
                        const uint64_t* tokens, size_t n_tokens, int* found,
                        jenga_small_page* page);
/* counters: used/evictable/empty small pages, owned units (type_allocator.hpp:133-136) */
int jenga_kv_group_counts(const jenga_kv* kv, int g, uint64_t* used, uint64_t* evictable,
                          uint64_t* empty, uint64_t* owned_units);
int jenga_kv_pool_free_pages(const jenga_kv* kv, uint32_t* num_free);
/* fragmentation_report (type_allocator.cpp:261-281) */
int jenga_kv_fragmentation(const jenga_kv* kv, int g, uint64_t* used_bytes,
                           uint64_t* evictable_bytes, uint64_t* empty_stranded_bytes);
int jenga_kv_alloc_step_counts(const jenga_kv* kv, uint64_t counts[6]);
int jenga_kv_check_invariants(const jenga_kv* kv);

/* ------------------------------------------------------------------------
 * LayerPolicy — reference layer_policies.cpp:79-120
 * ---------------------------------------------------------------------- */
int jenga_policy_needs_token(const jenga_spec* spec, int g, uint64_t i,
                             uint64_t new_tokens, uint64_t consumed_tokens, int* out);
int jenga_policy_accessed_range(const jenga_spec* spec, int g, uint64_t prev_tokens,
                                uint64_t new_tokens, uint64_t* lo, uint64_t* hi);

/* ------------------------------------------------------------------------
 * Per-request page lists — the state SimEngine keeps per (request, group)
 * (reference simulator.hpp:123-139) and updates in store_position
 * (simulator.cpp:217-282), group_stores_position (:151-158),
 * free_block (:284-312), release_all_pages (:314-327).
 * The page-list object borrows the allocator (single owner, not thread-safe,
 * as the reference: SPEC.md:170).
 * ---------------------------------------------------------------------- */
int jenga_pages_create(jenga_kv* kv, int prefix_caching, jenga_pages** out);
void jenga_pages_destroy(jenga_pages* pl);
int jenga_pages_add_request(jenga_pages* pl, uint64_t request);
/* Append one sequence position to every group that stores it (decode_one,
 * simulator.cpp:549-566).  image_ordinal is the eviction ordinal image-storing
 * groups record for an image position (simulator.cpp:160-162, 261-270).
 * OOM returns JENGA_ERR_OOM; the request must then be released (preempted,
 * simulator.cpp:329-338) before it is appended to again. */
int jenga_pages_append(jenga_pages* pl, uint64_t request, uint64_t token_id,
                       int is_image, uint64_t image_ordinal, uint64_t now_step);
/* One decode step for a batch: append one position (token_ids[i], is_image
 * may be NULL = text) to each request ids[i], in the given order.  Stops at
 * the first OOM (JENGA_ERR_OOM, *n_done = requests fully appended). */
int jenga_pages_append_batch(jenga_pages* pl, const uint64_t* ids, int n,
                             const uint64_t* token_ids, const uint8_t* is_image,
                             uint64_t now_step, int* n_done);
/* Append one position to ONE group (prefill / vision paths drive groups
 * separately in the reference). */
int jenga_pages_store(jenga_pages* pl, uint64_t request, int g, uint64_t pos,
                      uint64_t now_step);
int jenga_pages_release(jenga_pages* pl, uint64_t request, int allow_cache,
                        uint64_t now_step);
/* Admission with prefix caching (reference SimEngine::admit + KvAllocator::
 * lookup_and_pin + adopt_lookup_result, simulator.cpp:435-452, 391-433,
 * kv_allocator.cpp:241-303): install the prompt (n tokens; is_image and
 * image_ordinals may be NULL), pin the longest cached prefix and splice its
 * pages into the page lists.  *hit = prompt positions already resident. */
int jenga_pages_admit(jenga_pages* pl, uint64_t request, const uint64_t* tokens,
                      const uint8_t* is_image, const uint64_t* image_ordinals, uint64_t n,
                      uint64_t now_step, uint64_t* hit);
/* Chunked prefill of up to `budget` prompt positions (simulator.cpp:504-547).
 * *consumed = positions stored; JENGA_ERR_OOM when an allocation failed. */
int jenga_pages_prefill(jenga_pages* pl, uint64_t request, uint64_t budget, uint64_t now_step,
                        uint64_t* consumed);
/* Vision-embedding pages (reference EngineConfig::vision_mode, simulator.hpp:
 * 25-41; simulator.cpp:453-476, 504-547): mode 0 = on_demand (admit stores
 * the embeddings of images the prefix hit does not cover; prefill frees them
 * as image positions are consumed), 1 = full_reuse (admit stores all prompt
 * KV up front and defers window frees to the prompt's end; embeddings are
 * parked in the unwritten KV pages, see jenga_token_rows_scatter).  Set
 * before admitting requests. */
int jenga_pages_set_vision_mode(jenga_pages* pl, int mode);
/* Speculative decoding (simulator.cpp:568-640).  Draft groups are those named
 * "draft.*" (jenga_spec_combine_with_draft).  rollback_newest drops the newest
 * `count` stored positions of group g, freeing pages that empty out.
 * speculative_decode: the draft groups store propose_k positions, the
 * propose_k - accepted rejected ones roll back, then the target groups store
 * n_target (<= max(accepted, 1)) tokens.  JENGA_ERR_OOM: release the request. */
int jenga_pages_rollback_newest(jenga_pages* pl, uint64_t request, int g, uint64_t count,
                                uint64_t now_step);
int jenga_pages_speculative_decode(jenga_pages* pl, uint64_t request, uint32_t propose_k,
                                   uint64_t accepted, const uint64_t* target_tokens,
                                   uint64_t n_target, uint64_t now_step);
int jenga_pages_is_draft_group(const jenga_pages* pl, int g, int* is_draft);
/* Mamba restore after a prefix hit: the pinned checkpoint page of group g
 * (*has=0 when none is pending).  The caller copies it into the working page
 * (jenga_page_copy) and then calls jenga_pages_finish_restore, which returns
 * the checkpoint to the cache — the reference instead leaks the pinned page
 * (simulator.cpp:409-414). */
int jenga_pages_restore_pending(const jenga_pages* pl, uint64_t request, int g, int* has,
                                jenga_small_page* checkpoint);
int jenga_pages_finish_restore(jenga_pages* pl, uint64_t request, int g, uint64_t now_step);
int jenga_pages_set_fix_mamba_restore(jenga_pages* pl, int on);
/* Mamba checkpoint snapshots.  store_position allocates a checkpoint page
 * every checkpoint_interval stored positions and frees it straight into the
 * prefix cache (simulator.cpp:231-242); the reference models bytes only.  On
 * the device the working state at that ordinal must be copied into the page
 * (jenga_page_copy working -> checkpoint) before a later prefix hit restores
 * from it.  Each such page is queued; this drains up to `capacity` entries,
 * skipping pages evicted from the cache since (they may already belong to
 * another request).  Call it after the host half of a step and issue the
 * copies before the step's device work can overwrite the pages. */
typedef struct jenga_checkpoint_copy {
  uint64_t request;
  int32_t group;
  int32_t reserved;
  uint64_t ordinal;              /* stored ordinal the state corresponds to */
  jenga_small_page working;      /* source: the request's working page */
  jenga_small_page checkpoint;   /* destination: the cached checkpoint page */
} jenga_checkpoint_copy;
int jenga_pages_take_checkpoint_copies(jenga_pages* pl, jenga_checkpoint_copy* out, int capacity, int* n);
/* Defer sliding-window frees across a prefill chunk (the reference's
 * suppress_window_free, simulator.cpp:466-500): while on, stored positions
 * never free out-of-window blocks; apply performs the pending frees once the
 * chunk's attention has run. */
int jenga_pages_set_defer_window_free(jenga_pages* pl, uint64_t request, int on);
int jenga_pages_apply_window_free(jenga_pages* pl, uint64_t request, uint64_t now_step);
/* PrefixCache::entries (prefix_cache.hpp:71) */
int jenga_kv_cache_entries(const jenga_kv* kv, int g, uint64_t* n);
int jenga_pages_seq_len(const jenga_pages* pl, uint64_t request, uint64_t* len);
/* Per-group state of one request. */
int jenga_pages_group_state(const jenga_pages* pl, uint64_t request, int g,
                            uint64_t* stored, uint64_t* num_blocks,
                            uint64_t* freed_blocks, uint64_t* held_tokens,
                            int* has_working_page, jenga_small_page* working_page);
/* Copy the block list (dead blocks included, flagged live=0). */
int jenga_pages_blocks(const jenga_pages* pl, uint64_t request, int g,
                       jenga_small_page* pages, uint8_t* live, uint64_t capacity,
                       uint64_t* n);
/* Pack the CSR page lists of `n_req` requests for group g, ready for
 * jenga_build_block_tables:
 *   offsets[n_req+1], pages[offsets[n_req]], first_live_block[n_req],
 *   n_stored[n_req] (stored ordinals; for mamba groups 1 page = working).
 * Pass pages=NULL to query offsets only.  Everything is validated before
 * anything is written: a request holding more than max_blocks blocks (the
 * block-table width; <= 0 = unchecked) or a total above pages_capacity
 * (entries of `pages`) fails with JENGA_ERR_CONFIG, a dead block after the
 * first live one (the table encodes dead blocks as a leading prefix) or a
 * pool whose global page indices overflow int32 with JENGA_ERR_INVARIANT. */
int jenga_pages_pack_csr(const jenga_pages* pl, int g, const uint64_t* requests,
                         int n_req, int max_blocks, int64_t pages_capacity, int32_t* offsets,
                         jenga_small_page* pages, int32_t* first_live_block, int32_t* n_stored);

/* ------------------------------------------------------------------------
 * Delta page-list upload (the CSR path above re-packs
 * every list).  A decode step changes at most two entries of a (request,
 * group) row — the block store_position appended (simulator.cpp:248-253) and
 * a sliding-window block it freed (:272-280).  A table mirror remembers what
 * one group's device block table [max_batch][max_blocks] holds; each pack
 * diffs the page lists of requests[0..n_req) (row i = requests[i]) against it
 * and writes only the changed entries, plus every row's seq_len and newest-
 * token slot, into `delta`.  Rows whose list changed in any other way
 * (rollback, prefix adoption, release, a different request) are resent in
 * full; rows beyond n_req that held a request are cleared.  Each packed
 * buffer must be applied to the device table exactly once, in order
 * (jenga_upload_page_list_deltas); reset the mirror after rebuilding the
 * table any other way.  Validation happens before anything is written:
 * JENGA_ERR_CONFIG for a batch or request wider than the mirror or a buffer
 * smaller than *used_bytes (reported either way).
 * ---------------------------------------------------------------------- */
typedef struct jenga_table_mirror jenga_table_mirror;
/* Bytes a delta buffer needs in the worst case (every row rewritten), and
 * the bytes of a delta describing n_rows rows with n_records records (a
 * caller copying only a fixed prefix of the buffer to the device each step
 * sizes it with this and copies the whole used size when a pack needs more). */
size_t jenga_delta_buffer_bytes(int max_batch, int max_blocks);
size_t jenga_delta_bytes(int n_rows, int n_records);
int jenga_table_mirror_create(const jenga_pages* pl, int g, int max_batch, int max_blocks,
                              jenga_table_mirror** out);
void jenga_table_mirror_destroy(jenga_table_mirror* mirror);
/* The device table is all -1 again (e.g. freshly filled). */
int jenga_table_mirror_reset(jenga_table_mirror* mirror);
int jenga_pages_pack_deltas(jenga_table_mirror* mirror, const uint64_t* requests, int n_req,
                            void* delta, size_t capacity_bytes, size_t* used_bytes,
                            int* n_records);

/* ------------------------------------------------------------------------
 * Device API (sm_100a).  One arena per GPU: num_large_pages x large_page_bytes
 * (= LargePagePool sizing, lcm_allocator.cpp:12-18), 4 KiB aligned.
 * All launches are async on `stream` (cudaStream_t). Pointers are device
 * pointers unless stated.
 * ---------------------------------------------------------------------- */
int jenga_arena_create(int device, uint64_t num_large_pages, uint64_t large_page_bytes,
                       jenga_arena** out);
void jenga_arena_destroy(jenga_arena* arena);
void* jenga_arena_base(const jenga_arena* arena);
uint64_t jenga_arena_bytes(const jenga_arena* arena);

/* AddressMap::global_page_index + slot mapping on device
 * (memory_layout.cpp:22-27; slot = global*tpp + (ord-1)%tpp).
 *   offsets[B+1], pages[], first_live_block[B], n_stored[B]  — CSR page lists
 *   block_table[B][max_blocks] (int32, -1 = dead or absent)
 *   slot_mapping[B] (int64): slot of each request's newest stored ordinal
 *   (n_stored[b]) or -1 if n_stored[b]==0; may be NULL.
 *   seq_lens[B] (int32) = n_stored; may be NULL. */
int jenga_build_block_tables(const int32_t* offsets, const jenga_small_page* pages,
                             const int32_t* first_live_block, const int32_t* n_stored,
                             int batch, uint32_t slots_per_large, uint32_t tokens_per_page,
                             int max_blocks, int32_t* block_table, int64_t* slot_mapping,
                             int32_t* seq_lens, void* stream);

/* Apply a delta buffer from jenga_pages_pack_deltas to one group's table:
 * block_table[max_batch][max_blocks] entries, seq_lens[] and slot_mapping[]
 * (the newest stored ordinal's slot; -1 none) of the rows it describes.
 * `delta` is a device copy of the packed host buffer (the caller copies its
 * used bytes; a fixed-size prefix copy plus an extra copy only when a pack
 * outgrows it keeps the step capturable in a CUDA graph).  The launch writes
 * the buffer's sequence number to `ack` — the host buffer's word 4, pinned
 * memory the device stores to — so the next pack knows whether its
 * predecessor reached the device; a pack whose predecessor never did (a
 * buffer packed and overwritten, or packed before a graph capture and not
 * replayed) rewrites every row over the full table width.  ack may be NULL
 * (the next pack then always rewrites everything).  The host buffer must not
 * be rewritten before the copy has read it (record an event). */
int jenga_upload_page_list_deltas(const void* delta, int32_t* ack, int max_batch, int max_blocks,
                                  int32_t* block_table, int32_t* seq_lens,
                                  int64_t* slot_mapping, void* stream);

/* Slot mapping for a run of new tokens (prefill chunk):
 *   token t of request req[t] at 1-based ordinal ord[t] ->
 *   block_table[req][(ord-1)/tpp]*tpp + (ord-1)%tpp. */
int jenga_slot_mapping(const int32_t* block_table, int max_blocks, const int32_t* req,
                       const int32_t* ord, int n_tokens, uint32_t tokens_per_page,
                       int64_t* slot_mapping, void* stream);

/* Intra-slice layout (documented in DESIGN.md): one layer's slice of one small
 * page is [Hkv][K|V][tpp][D] of dtype (head-major: head h's K rows, then its
 * V rows) — exec_page_size = 2*Hkv*D*e*tpp.
 * Scatter K/V[T][Hkv][D] (row stride kv_row_stride elements between tokens)
 * into their slots; slot < 0 skips. */
int jenga_reshape_and_cache(void* arena_base, jenga_layer_view view, int dtype,
                            int num_kv_heads, int head_dim, uint32_t tokens_per_page,
                            const void* key, const void* value, int64_t kv_token_stride,
                            const int64_t* slot_mapping, int n_tokens, void* stream);

/* PDL ordering: decode launches (jenga_paged_decode / _append) use programmatic
 * dependent launch and may stream K/V tiles before their predecessor in the
 * stream has finished.  The library tracks, per stream, whether a kernel that
 * lets its dependents start early and writes arena bytes (jenga_reshape_and_cache,
 * the page / state copies) is still in the PDL chain, and then makes the decode
 * wait before its first load; every library launch on one stream is therefore
 * ordered as issued.  Kernels of your own that write the arena between library
 * launches must not use the programmatic-serialization attribute.
 * jenga_mamba_state_update records a column footprint instead (bytes
 * [start_offset, start_offset + num_layers * exec_page_size) of every page of
 * stride page_stride) and loads its own states early when every pending writer
 * is such a footprint on the same page grid with disjoint columns — per-layer
 * updates in model order overlap one layer's drain with the next one's loads.
 * Like block tables and seq_lens, the page_globals it reads early must come
 * from a launch without the attribute (any torch / plain CUDA launch). 
 *
 * Paged decode attention through the two-level table.
 *   kind: JENGA_KIND_FULL / SLIDING_WINDOW / CROSS_ATTENTION
 *   q[B][Hq][D], out[B][Hq][D] (dtype), block_table[B][max_blocks],
 *   seq_lens[B] = live length n (ordinals 1..n stored; SWA attends (n-W, n]).
 *   workspace: device scratch of jenga_paged_decode_workspace_size() bytes;
 *   the counters region must be zero before the first call (kernels re-zero
 *   it themselves).  softcap <= 0 disables logit soft-capping. */
size_t jenga_paged_decode_workspace_size(int batch, int num_q_heads, int num_kv_heads,
                                         int head_dim, int max_blocks,
                                         uint32_t tokens_per_page);
int jenga_paged_decode(void* arena_base, jenga_layer_view view, int kind, int dtype,
                       uint64_t window, const void* q, void* out, const int32_t* block_table,
                       const int32_t* seq_lens, int batch, int max_blocks, int num_q_heads,
                       int num_kv_heads, int head_dim, uint32_t tokens_per_page,
                       float scale, float softcap, void* workspace, size_t workspace_bytes,
                       void* stream);

/* One decode step of one layer in a single launch: the newest token's key/value
 * rows ([B][Hkv][D], written to slot_mapping[b]; < 0 skips) are appended to the
 * arena and attended together with the stored ordinals — the reshape_and_cache
 * + paged_decode pair of SimEngine::decode_one (simulator.cpp:549-566) fused.
 * seq_lens[b] must already count the new token (it is ordinal seq_lens[b]).
 * Full / sliding-window groups only (cross-attention KV is static in decode).
 * The tensor-core kernel patches the row into its staged K/V tile; other
 * shapes run reshape_and_cache then paged_decode on the same stream. */
int jenga_paged_decode_append(void* arena_base, jenga_layer_view view, int kind, int dtype,
                              uint64_t window, const void* q, const void* key, const void* value,
                              const int64_t* slot_mapping, void* out, const int32_t* block_table,
                              const int32_t* seq_lens, int batch, int max_blocks, int num_q_heads,
                              int num_kv_heads, int head_dim, uint32_t tokens_per_page, float scale,
                              float softcap, void* workspace, size_t workspace_bytes, void* stream);

/* Chunked-prefill paged attention (bf16/fp16, tokens_per_page % 16 == 0):
 * request b's queries are q[cu_q[b] .. cu_q[b+1]) — its newest ordinals
 * (0-based positions seq_lens[b]-C_b .. seq_lens[b]-1), whose K/V were already
 * written with jenga_reshape_and_cache.  Causal (+ window for SWA); cross
 * attention attends all seq_lens[b] image keys.  q/out [total_tokens][Hq][D],
 * 16-byte aligned (q is read by TMA; total_tokens = cu_q[batch]);
 * max_chunk = max C_b.  arena_base must come from jenga_arena_create.  head_dim
 * 128 / 256 run on a persistent grid (one CTA pair per two SMs) that needs no
 * workspace. */
int jenga_paged_prefill(void* arena_base, jenga_layer_view view, int kind, int dtype,
                        uint64_t window, const void* q, void* out, const int32_t* cu_q,
                        int total_tokens, int max_chunk, const int32_t* block_table,
                        const int32_t* seq_lens, int batch, int max_blocks, int num_q_heads,
                        int num_kv_heads, int head_dim, uint32_t tokens_per_page, float scale,
                        float softcap, void* stream);

/* Mamba last-token state (one working page per request, tpp=1):
 * gather dense[B][exec_page_size] <- arena slice; scatter the reverse
 * (simulator.cpp:222-244 keeps the working page). page_globals[b] < 0 skips. */
int jenga_mamba_state_gather(const void* arena_base, jenga_layer_view view,
                             const int64_t* page_globals, int batch, void* dense,
                             void* stream);
int jenga_mamba_state_scatter(void* arena_base, jenga_layer_view view,
                              const int64_t* page_globals, int batch, const void* dense,
                              void* stream);
/* The fused form of gather -> SSM update -> scatter (as jenga_paged_decode_append
 * is of reshape_and_cache + paged_decode): layers [l, l + num_layers) of every
 * request's working page — view = layer l's LayerView; the slices are one
 * contiguous run of num_layers * exec_page_size bytes per page — are read
 * through the page table and written back in place, each fp32 state element
 * multiplied by `decay` (the stand-in for the selective-scan state update,
 * whose math is out of scope; decay = 1 moves the bytes unchanged).  No dense
 * staging buffer: HBM traffic is exactly the state read + write.
 * page_globals[b] < 0 skips.  The state bytes must be fp32 (decay != 1). */
int jenga_mamba_state_update(void* arena_base, jenga_layer_view view, uint32_t num_layers,
                             const int64_t* page_globals, int batch, float decay, void* stream);
/* Token rows <-> pages (vision-embedding pages, simulator.cpp:453-476,
 * 525-542).  Row t (row_bytes, row_stride_bytes apart)
 * of the token at slot_mapping[t] = page_global*tpp + off (negative = skip;
 * gather writes zeros) is cut into piece_bytes pieces; piece p lives in layer
 * p / pieces_per_layer of `view` (layer l at view.start_offset +
 * l*view.exec_page_size), sub-slice q = p % pieces_per_layer:
 *   start + layer*exec_page_size + page*page_stride + (q*tpp + off)*piece_bytes
 * - a vision-embedding group's own pages: pieces_per_layer = 1,
 *   piece_bytes = bytes_per_token_per_layer;
 * - the full_reuse overlay into a KV group's unwritten pages:
 *   pieces_per_layer = 2*Hkv, piece_bytes = D*dtype — exactly the bytes
 *   jenga_reshape_and_cache later writes for the same token.
 * row_bytes <= num_layers*pieces_per_layer*piece_bytes; 16-byte multiples. */
int jenga_token_rows_scatter(void* arena_base, jenga_layer_view view, uint32_t num_layers,
                             uint32_t pieces_per_layer, uint32_t piece_bytes, uint32_t tokens_per_page,
                             const void* rows, uint64_t row_bytes, int64_t row_stride_bytes,
                             const int64_t* slot_mapping, int n_tokens, void* stream);
int jenga_token_rows_gather(const void* arena_base, jenga_layer_view view, uint32_t num_layers,
                            uint32_t pieces_per_layer, uint32_t piece_bytes, uint32_t tokens_per_page,
                            void* rows, uint64_t row_bytes, int64_t row_stride_bytes,
                            const int64_t* slot_mapping, int n_tokens, void* stream);
/* Whole-small-page copy (all layers of a group): checkpoint snapshot / restore
 * (simulator.cpp:231-242). Addresses = global * small_page_bytes. */
int jenga_page_copy(void* arena_base, uint64_t small_page_bytes, const int64_t* src_globals,
                    const int64_t* dst_globals, int n_pages, void* stream);

/* Number of device kernels launched by this library since load (evidence). */
uint64_t jenga_kernel_launch_count(void);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif  /* JENGA_GPU_H_ */
