// B200-native Jenga host runtime: model geometry, the two-level (LCM large
// page -> per-type small page) allocator, the page-layer address map and the
// per-request page lists that feed the device block tables.
//
// The public surface mirrors the reference C++ API (reference
// proj/include/jenga/*.hpp) name for name so that host code written against
// the reference drops in; the internals are our own: bitmap free lists with
// a summary level instead of std::set, flat per-large-page unit tables instead
// of std::map, and owner ids instead of owner strings.  Exported only through
// the C ABI in include/jenga_gpu.h (the .so is built -fvisibility=hidden).
#pragma once

#include <cstdint>
#include <memory>
#include <optional>
#include <set>
#include <stdexcept>
#include <string>
#include <tuple>
#include <unordered_map>
#include <vector>

namespace jenga {

// reference util.hpp:11-21
class ConfigError : public std::runtime_error {
 public:
  explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
class InvariantError : public std::logic_error {
 public:
  explicit InvariantError(const std::string& m) : std::logic_error(m) {}
};

#define JENGA_CHECK(cond, msg)                                                  \
  do {                                                                          \
    if (!(cond)) throw ::jenga::InvariantError(std::string(msg) + " [" #cond "]"); \
  } while (0)

uint64_t checked_mul(uint64_t a, uint64_t b, const char* what);
uint64_t checked_add(uint64_t a, uint64_t b, const char* what);

// splitmix64 finalizer (reference util.hpp:47-55) and FNV-1a (:57-64): the
// prefix-cache block keys must hash identically to the reference's.
inline uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
inline uint64_t mix64(uint64_t a, uint64_t b) { return mix64(a ^ mix64(b)); }
uint64_t hash_str(const std::string& s);

// ---------------------------------------------------------------- geometry
enum class LayerKind : int {
  kFullAttention = 0,
  kSlidingWindow = 1,
  kMamba = 2,
  kCrossAttention = 3,
  kVisionEmbedding = 4,
};
const char* layer_kind_name(LayerKind k);
LayerKind layer_kind_from_name(const std::string& s);

struct LayerGroupSpec {
  std::string name;
  LayerKind kind = LayerKind::kFullAttention;
  uint32_t num_layers = 0;
  uint64_t bytes_per_token_per_layer = 0;
  uint32_t tokens_per_page = 1;
  uint64_t window_tokens = 0;
  uint64_t checkpoint_interval_tokens = 0;
  bool stores_image_tokens() const {
    return kind == LayerKind::kCrossAttention || kind == LayerKind::kVisionEmbedding;
  }
};

struct ModelSpec {
  std::string name;
  std::vector<LayerGroupSpec> groups;
  void validate() const;
  bool has_cross_attention() const;
  bool decoder_stores_images() const { return !has_cross_attention(); }
};

uint64_t small_page_size(const LayerGroupSpec& g);
uint64_t lcm_page_size(const ModelSpec& spec);
double lcm_blowup_ratio(const ModelSpec& spec);
ModelSpec parse_model_spec_json(const std::string& text);

// ---------------------------------------------------------------- ids
struct LargePageId {
  uint32_t index = UINT32_MAX;
  bool valid() const { return index != UINT32_MAX; }
  friend bool operator==(LargePageId a, LargePageId b) { return a.index == b.index; }
};
struct SmallPageId {
  LargePageId large;
  uint32_t slot = 0;
  friend bool operator==(const SmallPageId& a, const SmallPageId& b) {
    return a.large == b.large && a.slot == b.slot;
  }
};

inline constexpr uint64_t kNoRequest = UINT64_MAX;
enum class SmallPageState : uint8_t { kEmpty = 0, kEvictable = 1, kUsed = 2 };

struct SmallPageRecord {
  SmallPageState state = SmallPageState::kEmpty;
  bool has_cache_key = false;
  uint64_t associated_request = kNoRequest;
  uint64_t last_access = 0;
  uint64_t prefix_length = 0;
  uint64_t cache_key = 0;
};

// Lowest-set-bit search over a dense bitmap with one summary word per 64
// words: find_first is two ctz scans, set/clear are O(1).  Replaces the
// reference's ordered std::set free lists (lcm_allocator.hpp:57,
// type_allocator.hpp:179) with identical lowest-index-first order.
class FirstFitBitmap {
 public:
  void resize(uint64_t nbits);
  void set(uint64_t i);
  void clear(uint64_t i);
  bool test(uint64_t i) const { return (words_[i >> 6] >> (i & 63)) & 1ULL; }
  uint64_t find_first() const;  // UINT64_MAX when empty
  uint64_t count() const { return count_; }
  uint64_t size() const { return nbits_; }

 private:
  uint64_t nbits_ = 0, count_ = 0;
  std::vector<uint64_t> words_, summary_, top_;
};

// ---------------------------------------------------------------- level 1
// reference lcm_allocator.hpp:29-59 / lcm_allocator.cpp:7-40
class LargePagePool {
 public:
  LargePagePool(uint64_t capacity_bytes, uint64_t large_page_bytes);
  std::optional<LargePageId> request_large_page(int owner);
  void return_large_page(LargePageId id);
  bool is_free(LargePageId id) const;
  int owner_of(LargePageId id) const;
  uint32_t num_pages() const { return static_cast<uint32_t>(owners_.size()); }
  uint32_t num_free() const { return static_cast<uint32_t>(free_.count()); }
  uint64_t large_page_bytes() const { return page_bytes_; }
  uint64_t free_bytes() const { return uint64_t{num_free()} * page_bytes_; }
  uint64_t reserved_remainder_bytes() const { return remainder_; }
  void check_conservation() const;

 private:
  uint64_t page_bytes_ = 0, remainder_ = 0;
  std::vector<int16_t> owners_;  // -1 = free
  FirstFitBitmap free_;
};

// ---------------------------------------------------------------- level 2
struct GroupGeometry {
  std::string group_name;
  uint64_t small_page_bytes = 0;
  uint32_t slots_per_large = 1;
};

struct UnitEvictionCandidate {
  uint64_t lru_timestamp = 0;
  uint64_t max_prefix_length = 0;
  uint32_t first_index = 0;
  bool better_than(const UnitEvictionCandidate& o) const {
    if (lru_timestamp != o.lru_timestamp) return lru_timestamp < o.lru_timestamp;
    if (max_prefix_length != o.max_prefix_length) return max_prefix_length > o.max_prefix_length;
    return first_index < o.first_index;
  }
};

struct FragmentationReport {
  uint64_t used_bytes = 0, evictable_bytes = 0, empty_stranded_bytes = 0;
};

// reference type_allocator.hpp:81-182.  Jenga geometry only (LCM >= every
// small page, so one unit == one large page).
class TypeAllocator {
 public:
  TypeAllocator(GroupGeometry geo, int owner_id, LargePagePool* pool);
  const GroupGeometry& geometry() const { return geo_; }

  std::optional<SmallPageId> try_allocate_associated(uint64_t request);
  std::optional<SmallPageId> try_allocate_from_new_unit(uint64_t request);
  std::optional<SmallPageId> try_allocate_any(uint64_t request);
  std::optional<SmallPageId> lru_evictable_small() const;
  uint64_t evict_small(SmallPageId id);
  void allocate_slot(SmallPageId id, uint64_t request);
  void free(SmallPageId id, std::optional<uint64_t> cache_key);
  void pin(SmallPageId id, uint64_t request);
  void touch(SmallPageId id, uint64_t step);
  void set_prefix_length(SmallPageId id, uint64_t len);
  const SmallPageRecord& record(SmallPageId id) const;
  bool tracks(SmallPageId id) const;
  std::vector<UnitEvictionCandidate> fully_evictable_units() const;
  std::vector<uint64_t> clear_unit(uint32_t first_index);
  FragmentationReport fragmentation_report() const;

  uint64_t used_pages() const { return used_; }
  uint64_t evictable_pages() const { return lru_live_; }
  uint64_t empty_pages() const { return empty_.count(); }
  uint64_t owned_units() const { return owned_units_; }
  bool has_associated_empty(uint64_t request) const;
  void check_invariants() const;

  uint64_t global_index(uint32_t large, uint32_t slot) const {
    return uint64_t{large} * geo_.slots_per_large + slot;
  }
  SmallPageId from_global(uint64_t g) const {
    return SmallPageId{LargePageId{static_cast<uint32_t>(g / geo_.slots_per_large)},
                       static_cast<uint32_t>(g % geo_.slots_per_large)};
  }

 private:
  struct Unit {
    bool owned = false;
    uint32_t empty_count = 0, evictable_count = 0;
    std::vector<SmallPageRecord> slots;  // allocated while owned
  };
  using LruKey = std::tuple<uint64_t, uint64_t, uint64_t>;  // (last_access, ~prefix, global)

  Unit& unit_of(SmallPageId id);
  const Unit& unit_of(SmallPageId id) const;
  SmallPageRecord& rec(SmallPageId id);
  void index_on_empty(uint64_t g, const SmallPageRecord& r);
  void unindex_on_empty(uint64_t g, const SmallPageRecord& r);
  void release_unit(uint32_t large);
  static LruKey lru_key(const SmallPageRecord& r, uint64_t g) {
    return LruKey{r.last_access, UINT64_MAX - r.prefix_length, g};
  }
  bool lru_entry_live(const LruKey& k) const;
  void lru_push(const LruKey& k);
  void lru_drop_stale_top() const;
  void lru_rebuild() const;

  GroupGeometry geo_;
  int owner_id_;
  LargePagePool* pool_;
  std::vector<Unit> units_;               // indexed by large page index
  uint64_t owned_units_ = 0;
  // Eviction order: a lazy-deletion min-heap of LruKey (front = the reference's
  // LRU victim).  A pin or eviction only changes the page's state and a touch
  // pushes the page's new key, so the entries they leave behind are stale:
  // an entry is live while its page is evictable with exactly that key.  Stale
  // entries are dropped when they surface at the front and by a rebuild once
  // they outnumber the live ones (pins of tens of thousands of cached pages
  // per admission wave no longer rebalance an ordered set).
  mutable std::vector<LruKey> lru_heap_;
  uint64_t lru_live_ = 0;                 // evictable pages
  // unit in fully_evictable_ by unit index (erase by iterator)
  FirstFitBitmap empty_;                  // global indices of empty owned slots
  // request -> its associated empty slots (global indices, kept sorted)
  std::unordered_map<uint64_t, std::vector<uint64_t>> empty_by_request_;
  std::set<uint32_t> fully_evictable_;    // units whose every slot is evictable
  std::vector<std::set<uint32_t>::iterator> fe_it_;
  uint64_t used_ = 0;
};

// ---------------------------------------------------------------- prefix cache
// reference prefix_cache.hpp:20-80
struct BlockContent {
  uint64_t key = 0, parent_key = 0;
  std::vector<uint64_t> tokens;
  bool matches(const BlockContent& o) const {
    return key == o.key && parent_key == o.parent_key && tokens == o.tokens;
  }
};
uint64_t block_chain_salt(const std::string& group_name);
uint64_t chain_block_key(uint64_t parent, const std::vector<uint64_t>& tokens);

// reference prefix_cache.hpp:20-75 semantics: per group, chain key -> the
// cached pages holding that content, in registration order.  Stored as an
// open-addressing table (the keys are already mixed 64-bit chain hashes) over a
// pool of entries chained per key, so a lookup costs a slot probe and an entry
// read instead of a node-based hash map's chain of dependent cache misses —
// admission under prefix caching does hundreds of them per request.
class PrefixCache {
 public:
  explicit PrefixCache(size_t n) : groups_(n) {}
  void register_block(size_t g, const BlockContent& c, SmallPageId page);
  void unregister(size_t g, uint64_t key, SmallPageId page);
  std::optional<SmallPageId> find(size_t g, const BlockContent& c) const;
  uint64_t entries(size_t g) const;

 private:
  static constexpr uint32_t kNil = UINT32_MAX;
  struct Entry {
    BlockContent content;
    SmallPageId page;
    uint32_t next = kNil;
  };
  struct Slot {
    uint64_t key = 0;
    uint32_t head = kNil, tail = kNil;  // entries of this key, registration order
    uint8_t state = 0;                  // 0 empty, 1 live, 2 tombstone
  };
  struct Table {
    std::vector<Slot> slots;  // power-of-two size
    std::vector<Entry> pool;
    std::vector<uint32_t> free;
    uint64_t occupied = 0;    // live + tombstone slots
    uint64_t entries = 0;
  };
  static size_t home(uint64_t key, size_t mask) { return static_cast<size_t>(key ^ (key >> 31)) & mask; }
  static const Slot* probe(const Table& t, uint64_t key);
  static Slot& insert_slot(Table& t, uint64_t key);
  static void rehash(Table& t, size_t capacity);
  std::vector<Table> groups_;
};

// ---------------------------------------------------------------- prefix sets
// Sorted disjoint inclusive ranges of valid prefix lengths (reference
// range_set.hpp:14-39 semantics).
class PrefixRangeSet {
 public:
  void append(uint64_t v) { append_range(v, v); }
  void append_range(uint64_t lo, uint64_t hi);
  bool contains(uint64_t v) const;
  uint64_t max_value() const { return r_.empty() ? 0 : r_.back().second; }
  static PrefixRangeSet intersect(const PrefixRangeSet& a, const PrefixRangeSet& b);
  const std::vector<std::pair<uint64_t, uint64_t>>& ranges() const { return r_; }

 private:
  std::vector<std::pair<uint64_t, uint64_t>> r_;
};

// reference layer_policies.cpp:9-77
std::vector<uint64_t> required_tokens(const LayerGroupSpec& g, uint64_t p, bool* defined);
PrefixRangeSet possible_prefixes(const LayerGroupSpec& g, const std::vector<bool>& is_hit);
// reference prefix_cache.cpp:25-57
PrefixRangeSet stored_to_global_prefixes(const PrefixRangeSet& valid, const std::vector<uint64_t>& stored_positions,
                                         uint64_t sequence_length);
uint64_t find_longest_common_prefix(const std::vector<PrefixRangeSet>& per_group);

struct GroupLookupInput {
  std::vector<uint64_t> stored_positions;
  std::vector<BlockContent> blocks;
  std::vector<uint64_t> block_end_ordinal;
};
struct LookupResult {
  uint64_t hit_length = 0;
  std::vector<std::vector<std::pair<uint64_t, SmallPageId>>> pinned;  // per group (block, page)
};

// ---------------------------------------------------------------- engine
struct AllocResult {
  SmallPageId page;
  int step = 0;
};

// reference kv_allocator.hpp:62-119 (Jenga strategy: one LCM pool).
class KvAllocator {
 public:
  KvAllocator(const ModelSpec& spec, uint64_t budget_bytes);
  size_t num_groups() const { return spec_.groups.size(); }
  const LayerGroupSpec& group(size_t g) const { return spec_.groups[g]; }
  const ModelSpec& spec() const { return spec_; }
  TypeAllocator& type_allocator(size_t g) { return *types_[g]; }
  const TypeAllocator& type_allocator(size_t g) const { return *types_[g]; }
  LargePagePool& pool() { return *pool_; }
  const LargePagePool& pool() const { return *pool_; }
  PrefixCache& cache() { return cache_; }
  const PrefixCache& cache() const { return cache_; }

  std::optional<AllocResult> allocate(size_t g, uint64_t request);
  void free(size_t g, SmallPageId page, const std::optional<BlockContent>& cached);
  void pin(size_t g, SmallPageId page, uint64_t request);
  std::optional<LargePageId> evict_lru_large_page();
  // reference kv_allocator.cpp:241-303
  LookupResult lookup_and_pin(const std::vector<GroupLookupInput>& inputs, uint64_t sequence_length,
                              uint64_t request);
  void set_request_aware(bool on) { request_aware_ = on; }
  uint64_t budget_bytes() const { return budget_; }
  const uint64_t* alloc_step_counts() const { return step_counts_; }
  void check_invariants() const;

 private:
  ModelSpec spec_;
  uint64_t budget_ = 0;
  bool request_aware_ = true;
  std::unique_ptr<LargePagePool> pool_;
  std::vector<std::unique_ptr<TypeAllocator>> types_;
  PrefixCache cache_;
  uint64_t step_counts_[6] = {0, 0, 0, 0, 0, 0};
};

// ---------------------------------------------------------------- address map
struct ByteRange {
  uint64_t begin = 0, end = 0;
};
struct LayerView {
  uint64_t start_offset = 0, page_stride = 0, exec_page_size = 0;
};

// reference memory_layout.hpp:34-69
class AddressMap {
 public:
  explicit AddressMap(const ModelSpec& spec);
  uint64_t large_page_bytes() const { return large_; }
  size_t num_groups() const { return spec_.groups.size(); }
  uint64_t small_page_bytes(size_t g) const { return small_[g]; }
  uint64_t per_layer_bytes(size_t g) const { return per_layer_[g]; }
  uint32_t slots_per_large(size_t g) const { return slots_[g]; }
  uint64_t global_page_index(size_t g, SmallPageId p) const;
  ByteRange address_of(size_t g, uint32_t layer, SmallPageId p) const;
  LayerView layer_view(size_t g, uint32_t layer) const;
  ByteRange view_address(size_t g, uint32_t layer, SmallPageId p) const;

 private:
  ModelSpec spec_;
  uint64_t large_ = 0;
  std::vector<uint64_t> small_, per_layer_;
  std::vector<uint32_t> slots_;
};

// ---------------------------------------------------------------- policies
// reference layer_policies.cpp:79-120
bool needs_token(const LayerGroupSpec& g, uint64_t i, uint64_t new_tokens,
                 uint64_t consumed_tokens);
std::pair<uint64_t, uint64_t> accessed_range(const LayerGroupSpec& g, uint64_t prev_tokens,
                                             uint64_t new_tokens);

// ---------------------------------------------------------------- page lists
// The per-(request, group) page lists of reference simulator.hpp:123-139,
// maintained with the semantics of store_position / free_block /
// release_all_pages (simulator.cpp:196-327).
class PageLists {
 public:
  PageLists(KvAllocator* kv, bool prefix_caching);

  struct Block {
    SmallPageId page;
    bool live = false;
  };
  struct GroupRuntime {
    uint64_t stored = 0;
    std::vector<uint64_t> stored_positions;
    std::vector<Block> blocks;
    std::vector<BlockContent> chain;
    uint64_t freed_blocks = 0, held_tokens = 0, live_blocks = 0;
    std::optional<SmallPageId> working_page;
    uint64_t checkpoints = 0;
    uint64_t consumed_held = 0;      // vision: consumed ordinals still held
    uint64_t consumed_ordinals = 0;  // vision: ordinals consumed by prefill
    // Bumped (to a PageLists-wide unique value) whenever the list changes other
    // than by appending blocks at the tail or freeing its leading live block:
    // a table mirror (jenga_pages_pack_deltas) then resends the whole row.
    uint64_t epoch = 0;
  };
  struct ImageSpan {
    uint64_t begin = 0, end = 0;  // prompt positions, inclusive
  };
  struct Request {
    uint64_t id = 0;
    std::vector<uint64_t> tokens;
    std::vector<uint8_t> is_image;
    std::vector<uint64_t> image_ordinal;  // per position (image tokens only)
    std::vector<GroupRuntime> groups;
    bool needs_release = false;  // set by a failed (OOM) append
    uint64_t prompt_len = 0;     // admit(): prefill target
    uint64_t consumed = 0;       // admit(): prompt positions prefilled (hits included)
    // Mamba checkpoint pages pinned by a prefix hit, per group: the state to
    // copy into the working page before decoding resumes (the reference pins
    // them and never adopts them, simulator.cpp:409-414).
    std::vector<std::optional<SmallPageId>> restore;
    // Defer sliding-window frees while a prefill chunk's attention still
    // needs keys that left the window (the reference's suppress_window_free,
    // simulator.cpp:466-500); apply_window_free() performs them.
    bool defer_window_free = false;
    // full_reuse vision mode: window frees suppressed until the prompt is
    // written (simulator.cpp:466-500)
    bool suppress_window_free = false;
    std::vector<ImageSpan> images;  // admit(): maximal runs of one image
    uint64_t draft_len = 0;         // speculative: draft sequence length
  };
  // reference simulator.hpp:25 (EngineConfig::vision_mode)
  enum class VisionMode { kAllocateOnDemand = 0, kFullyAllocatedReuse = 1 };

  void add_request(uint64_t id);
  bool has_request(uint64_t id) const { return index_.count(id) != 0; }
  // decode_one-style append of one position to every group storing it
  // (vision-embedding groups excluded, as prefill_some / decode do).
  // Returns false on OOM (caller preempts).
  bool append(uint64_t id, uint64_t token, bool is_image, uint64_t image_ordinal,
              uint64_t now);
  bool store_position(uint64_t id, size_t g, uint64_t pos, uint64_t now);
  void release(uint64_t id, bool allow_cache, uint64_t now);
  const Request& request(uint64_t id) const;
  bool group_stores_position(size_t g, const Request& r, uint64_t pos) const;

  // Admission (reference simulator.cpp:435-452): install the prompt and, with
  // prefix caching, pin and adopt the longest cached prefix.  Returns the hit
  // length (prompt positions already resident).
  // Vision pages are stored here too (on_demand: embeddings of images the
  // hit does not cover; full_reuse: all prompt KV up front); *oom set when
  // one of those allocations failed.
  uint64_t admit(uint64_t id, const std::vector<uint64_t>& tokens, const std::vector<uint8_t>& is_image,
                 const std::vector<uint64_t>& image_ordinals, uint64_t now, bool* oom = nullptr);
  // Chunked prefill of up to `budget` positions (reference simulator.cpp:
  // 504-547): on_demand mode frees consumed vision-embedding pages, and the
  // prompt's last position finishes the prefill (finish_prefill, :484-502).
  // Returns positions consumed; *oom set when an allocation failed.
  uint64_t prefill(uint64_t id, uint64_t budget, uint64_t now, bool* oom);
  // Vision-embedding handling at admit / prefill (simulator.cpp:453-476,
  // 525-542); set before admitting requests.
  void set_vision_mode(VisionMode m) { vision_mode_ = m; }
  VisionMode vision_mode() const { return vision_mode_; }
  // reference simulator.cpp:568-597: drop the newest `count` stored
  // positions of group g, freeing pages that empty out.
  void rollback_newest(uint64_t id, size_t g, uint64_t count, uint64_t now);
  // reference speculative_decode_one (simulator.cpp:600-640): the draft
  // groups ("draft." prefix, simulator.cpp:76-78) store propose_k positions,
  // the propose_k - accepted rejected ones roll back, then the target groups
  // store n_target = max(accepted, 1) tokens (fewer when the request ends).
  // Returns false on OOM (the request must be released).
  bool speculative_decode(uint64_t id, uint32_t propose_k, uint64_t accepted, const uint64_t* target_tokens,
                          uint64_t n_target, uint64_t now);
  bool is_draft_group(size_t g) const { return draft_flags_[g] != 0; }
  // reference simulator.cpp:347-358
  void refresh_mamba_checkpoints(uint64_t id, uint64_t now);
  // The Mamba restore fix: forget (and free) a pinned checkpoint page once
  // the caller has copied it into the working page.
  void finish_restore(uint64_t id, size_t g, uint64_t now);
  void set_defer_window_free(uint64_t id, bool on) { req(id).defer_window_free = on; }
  // reference finish_prefill's deferred frees (simulator.cpp:484-500)
  void apply_window_free(uint64_t id, uint64_t now);
  bool fix_mamba_restore = true;  // false: keep the reference's pinned-page leak

  // Mamba checkpoint snapshots: store_position allocates a checkpoint page
  // every k stored positions and frees it straight into the prefix cache
  // (simulator.cpp:231-242) — a byte model with no bytes.  On the device the
  // working state at that ordinal must be copied into the page before anyone
  // can hit it; each allocation is queued here and drained by the caller
  // (take_checkpoint_copies), which drops copies whose page was evicted from
  // the cache in the meantime (it may already belong to another request).
  struct CheckpointCopy {
    uint64_t request = 0;
    uint32_t g = 0;
    uint64_t ordinal = 0;          // stored ordinal the state corresponds to
    SmallPageId working, checkpoint;
    BlockContent key;              // cache key the page was registered under
  };
  std::vector<CheckpointCopy> take_checkpoint_copies();

 private:
  Request& req(uint64_t id);
  bool store_position(Request& r, size_t g, uint64_t pos, uint64_t now);
  std::vector<GroupLookupInput> build_lookup_inputs(const Request& r) const;
  void append_chain(Request& r, size_t g);
  void free_block(Request& r, size_t g, uint64_t b, bool allow_cache, uint64_t now);
  void finish_prefill(Request& r, uint64_t now);
  uint64_t adopt_prefix(Request& r, uint64_t now);
  void reset_groups(Request& r);  // fresh GroupRuntimes, new epochs
  void bump(GroupRuntime& rt) { rt.epoch = ++epoch_counter_; }

  uint64_t epoch_counter_ = 0;
  std::vector<CheckpointCopy> checkpoint_copies_;

  KvAllocator* kv_;
  bool prefix_caching_;
  VisionMode vision_mode_ = VisionMode::kAllocateOnDemand;
  std::vector<uint8_t> draft_flags_;
  std::vector<Request> requests_;
  std::unordered_map<uint64_t, size_t> index_;
};

}  // namespace jenga
