// The two-level Jenga allocator.  Decision order and tie-breaks reproduce the
// reference exactly (cited per method) so page lists are bit-identical for
// identical operation sequences; the data structures are our own (bitmap
// first-fit instead of ordered sets, flat unit tables instead of maps).
#include <algorithm>
#include <functional>

#include "jenga_host.hpp"

namespace jenga {

// ------------------------------------------------------------ FirstFitBitmap
void FirstFitBitmap::resize(uint64_t nbits) {
  nbits_ = nbits;
  count_ = 0;
  const uint64_t nw = (nbits + 63) / 64;
  const uint64_t ns = (nw + 63) / 64;
  const uint64_t nt = (ns + 63) / 64;
  words_.assign(nw, 0);
  summary_.assign(ns, 0);
  top_.assign(nt, 0);
}

void FirstFitBitmap::set(uint64_t i) {
  uint64_t& w = words_[i >> 6];
  const uint64_t bit = 1ULL << (i & 63);
  if (w & bit) return;
  w |= bit;
  ++count_;
  const uint64_t wi = i >> 6;
  summary_[wi >> 6] |= 1ULL << (wi & 63);
  const uint64_t si = wi >> 6;
  top_[si >> 6] |= 1ULL << (si & 63);
}

void FirstFitBitmap::clear(uint64_t i) {
  uint64_t& w = words_[i >> 6];
  const uint64_t bit = 1ULL << (i & 63);
  if (!(w & bit)) return;
  w &= ~bit;
  --count_;
  if (w == 0) {
    const uint64_t wi = i >> 6;
    uint64_t& s = summary_[wi >> 6];
    s &= ~(1ULL << (wi & 63));
    if (s == 0) {
      const uint64_t si = wi >> 6;
      top_[si >> 6] &= ~(1ULL << (si & 63));
    }
  }
}

uint64_t FirstFitBitmap::find_first() const {
  if (count_ == 0) return UINT64_MAX;
  for (uint64_t t = 0; t < top_.size(); ++t) {
    if (top_[t] == 0) continue;
    const uint64_t si = t * 64 + __builtin_ctzll(top_[t]);
    const uint64_t wi = si * 64 + __builtin_ctzll(summary_[si]);
    return wi * 64 + __builtin_ctzll(words_[wi]);
  }
  return UINT64_MAX;
}

// ------------------------------------------------------------ LargePagePool
// reference lcm_allocator.cpp:7-19
LargePagePool::LargePagePool(uint64_t capacity_bytes, uint64_t large_page_bytes)
    : page_bytes_(large_page_bytes) {
  if (large_page_bytes == 0) throw ConfigError("large page size must be positive");
  const uint64_t count = capacity_bytes / large_page_bytes;
  if (count > UINT32_MAX - 1) throw ConfigError("pool would exceed the page index space");
  remainder_ = capacity_bytes - count * large_page_bytes;
  owners_.assign(count, -1);
  free_.resize(count);
  for (uint64_t i = 0; i < count; ++i) free_.set(i);
}

// reference lcm_allocator.cpp:21-29: lowest index first.
std::optional<LargePageId> LargePagePool::request_large_page(int owner) {
  const uint64_t i = free_.find_first();
  if (i == UINT64_MAX) return std::nullopt;
  JENGA_CHECK(owner >= 0, "large page owner must be named");
  free_.clear(i);
  owners_[i] = static_cast<int16_t>(owner);
  return LargePageId{static_cast<uint32_t>(i)};
}

// reference lcm_allocator.cpp:31-40
void LargePagePool::return_large_page(LargePageId id) {
  JENGA_CHECK(id.index < owners_.size(), "large page index out of range");
  if (owners_[id.index] < 0)
    throw InvariantError("double free of large page " + std::to_string(id.index));
  owners_[id.index] = -1;
  JENGA_CHECK(!free_.test(id.index), "large page already on free list");
  free_.set(id.index);
}

bool LargePagePool::is_free(LargePageId id) const {
  JENGA_CHECK(id.index < owners_.size(), "large page index out of range");
  return owners_[id.index] < 0;
}

int LargePagePool::owner_of(LargePageId id) const {
  JENGA_CHECK(id.index < owners_.size(), "large page index out of range");
  return owners_[id.index];
}

void LargePagePool::check_conservation() const {
  uint64_t owned = 0;
  for (uint64_t i = 0; i < owners_.size(); ++i) {
    const bool fr = owners_[i] < 0;
    JENGA_CHECK(fr == free_.test(i), "free list disagrees with ownership");
    if (!fr) ++owned;
  }
  JENGA_CHECK(owned + free_.count() == owners_.size(), "pool pages leaked");
}

// ------------------------------------------------------------ TypeAllocator
TypeAllocator::TypeAllocator(GroupGeometry geo, int owner_id, LargePagePool* pool)
    : geo_(std::move(geo)), owner_id_(owner_id), pool_(pool) {
  JENGA_CHECK(pool_ != nullptr, "type allocator needs a pool");
  JENGA_CHECK(geo_.slots_per_large >= 1, "slots_per_large must be >= 1");
  units_.resize(pool_->num_pages());
  empty_.resize(uint64_t{pool_->num_pages()} * geo_.slots_per_large);
  fe_it_.resize(pool_->num_pages());
}

TypeAllocator::Unit& TypeAllocator::unit_of(SmallPageId id) {
  JENGA_CHECK(id.large.index < units_.size() && units_[id.large.index].owned,
              "small page outside owned large pages");
  return units_[id.large.index];
}

const TypeAllocator::Unit& TypeAllocator::unit_of(SmallPageId id) const {
  JENGA_CHECK(id.large.index < units_.size() && units_[id.large.index].owned,
              "small page outside owned large pages");
  return units_[id.large.index];
}

SmallPageRecord& TypeAllocator::rec(SmallPageId id) {
  Unit& u = unit_of(id);
  JENGA_CHECK(id.slot < u.slots.size(), "slot out of range");
  return u.slots[id.slot];
}

const SmallPageRecord& TypeAllocator::record(SmallPageId id) const {
  const Unit& u = unit_of(id);
  JENGA_CHECK(id.slot < u.slots.size(), "slot out of range");
  return u.slots[id.slot];
}

bool TypeAllocator::tracks(SmallPageId id) const {
  return id.large.index < units_.size() && units_[id.large.index].owned &&
         id.slot < geo_.slots_per_large;
}

bool TypeAllocator::has_associated_empty(uint64_t request) const {
  auto it = empty_by_request_.find(request);
  return it != empty_by_request_.end() && !it->second.empty();
}

// reference type_allocator.cpp:239-258 (index_on_empty / unindex_on_empty)
void TypeAllocator::index_on_empty(uint64_t g, const SmallPageRecord& r) {
  empty_.set(g);
  if (r.associated_request != kNoRequest) {
    auto& v = empty_by_request_[r.associated_request];
    v.insert(std::lower_bound(v.begin(), v.end(), g), g);
  }
}

void TypeAllocator::unindex_on_empty(uint64_t g, const SmallPageRecord& r) {
  empty_.clear(g);
  if (r.associated_request != kNoRequest) {
    auto it = empty_by_request_.find(r.associated_request);
    if (it != empty_by_request_.end()) {
      auto& v = it->second;
      auto pos = std::lower_bound(v.begin(), v.end(), g);
      if (pos != v.end() && *pos == g) v.erase(pos);
      if (v.empty()) empty_by_request_.erase(it);
    }
  }
}

// Step 1 — reference type_allocator.cpp:76-83
std::optional<SmallPageId> TypeAllocator::try_allocate_associated(uint64_t request) {
  auto it = empty_by_request_.find(request);
  if (it == empty_by_request_.end() || it->second.empty()) return std::nullopt;
  const SmallPageId id = from_global(it->second.front());
  allocate_slot(id, request);
  return id;
}

// Step 2 — reference type_allocator.cpp:85-108 (one large page per unit)
std::optional<SmallPageId> TypeAllocator::try_allocate_from_new_unit(uint64_t request) {
  if (pool_->num_free() < 1) return std::nullopt;
  auto page = pool_->request_large_page(owner_id_);
  JENGA_CHECK(page.has_value(), "pool free count lied");
  const uint32_t first = page->index;
  Unit& u = units_[first];
  JENGA_CHECK(!u.owned, "unit already tracked");
  u.owned = true;
  u.slots.assign(geo_.slots_per_large, SmallPageRecord{});
  u.empty_count = geo_.slots_per_large;
  u.evictable_count = 0;
  for (auto& s : u.slots) s.associated_request = request;
  ++owned_units_;
  for (uint32_t s = 0; s < geo_.slots_per_large; ++s)
    index_on_empty(global_index(first, s), u.slots[s]);
  const SmallPageId id{LargePageId{first}, 0};
  allocate_slot(id, request);
  return id;
}

// Step 4 — reference type_allocator.cpp:110-115
std::optional<SmallPageId> TypeAllocator::try_allocate_any(uint64_t request) {
  const uint64_t g = empty_.find_first();
  if (g == UINT64_MAX) return std::nullopt;
  const SmallPageId id = from_global(g);
  allocate_slot(id, request);
  return id;
}

// Step 5 candidate — reference type_allocator.cpp:117-120
bool TypeAllocator::lru_entry_live(const LruKey& k) const {
  const uint64_t g = std::get<2>(k);
  const SmallPageId id = from_global(g);
  const Unit& u = units_[id.large.index];
  if (!u.owned || id.slot >= u.slots.size()) return false;
  const SmallPageRecord& r = u.slots[id.slot];
  return r.state == SmallPageState::kEvictable && lru_key(r, g) == k;
}

void TypeAllocator::lru_rebuild() const {
  lru_heap_.clear();
  for (uint32_t first = 0; first < units_.size(); ++first) {
    const Unit& u = units_[first];
    if (!u.owned || u.evictable_count == 0) continue;
    for (uint32_t s = 0; s < u.slots.size(); ++s)
      if (u.slots[s].state == SmallPageState::kEvictable) lru_heap_.push_back(lru_key(u.slots[s], global_index(first, s)));
  }
  std::make_heap(lru_heap_.begin(), lru_heap_.end(), std::greater<LruKey>());
}

void TypeAllocator::lru_push(const LruKey& k) {
  if (lru_heap_.size() >= 2 * lru_live_ + 4096) {
    lru_rebuild();  // already holds k when the page is evictable with it
    return;
  }
  lru_heap_.push_back(k);
  std::push_heap(lru_heap_.begin(), lru_heap_.end(), std::greater<LruKey>());
}

void TypeAllocator::lru_drop_stale_top() const {
  while (!lru_heap_.empty() && !lru_entry_live(lru_heap_.front())) {
    std::pop_heap(lru_heap_.begin(), lru_heap_.end(), std::greater<LruKey>());
    lru_heap_.pop_back();
  }
}

std::optional<SmallPageId> TypeAllocator::lru_evictable_small() const {
  if (lru_live_ == 0) return std::nullopt;
  lru_drop_stale_top();
  JENGA_CHECK(!lru_heap_.empty(), "LRU heap lost an evictable page");
  return from_global(std::get<2>(lru_heap_.front()));
}

// reference type_allocator.cpp:122-138
uint64_t TypeAllocator::evict_small(SmallPageId id) {
  Unit& u = unit_of(id);
  SmallPageRecord& r = u.slots[id.slot];
  JENGA_CHECK(r.state == SmallPageState::kEvictable, "evict_small on a non-evictable page");
  JENGA_CHECK(r.has_cache_key, "evictable page lost its cache key");
  const uint64_t key = r.cache_key;
  const uint64_t g = global_index(id.large.index, id.slot);
  lru_live_--;  // its heap entry goes stale with the state change
  if (u.evictable_count == u.slots.size()) fully_evictable_.erase(fe_it_[id.large.index]);
  u.evictable_count--;
  r.state = SmallPageState::kEmpty;
  r.has_cache_key = false;
  r.cache_key = 0;
  u.empty_count++;
  index_on_empty(g, r);
  return key;
}

// reference type_allocator.cpp:140-151
void TypeAllocator::allocate_slot(SmallPageId id, uint64_t request) {
  Unit& u = unit_of(id);
  SmallPageRecord& r = u.slots[id.slot];
  JENGA_CHECK(r.state == SmallPageState::kEmpty, "allocate_slot on a non-empty page");
  unindex_on_empty(global_index(id.large.index, id.slot), r);
  u.empty_count--;
  r.state = SmallPageState::kUsed;
  r.associated_request = request;
  r.prefix_length = 0;
  used_++;
}

// reference type_allocator.cpp:153-175
void TypeAllocator::free(SmallPageId id, std::optional<uint64_t> cache_key) {
  Unit& u = unit_of(id);
  SmallPageRecord& r = u.slots[id.slot];
  if (r.state != SmallPageState::kUsed)
    throw InvariantError("double free of small page (group '" + geo_.group_name + "')");
  used_--;
  const uint64_t g = global_index(id.large.index, id.slot);
  if (cache_key.has_value()) {
    r.state = SmallPageState::kEvictable;
    r.cache_key = *cache_key;
    r.has_cache_key = true;
    u.evictable_count++;
    if (u.evictable_count == u.slots.size()) fe_it_[id.large.index] = fully_evictable_.insert(id.large.index).first;
    lru_live_++;
    lru_push(lru_key(r, g));
    return;
  }
  r.state = SmallPageState::kEmpty;
  r.has_cache_key = false;
  u.empty_count++;
  index_on_empty(g, r);
  if (u.empty_count == u.slots.size()) release_unit(id.large.index);
}

// reference type_allocator.cpp:177-190
void TypeAllocator::pin(SmallPageId id, uint64_t request) {
  Unit& u = unit_of(id);
  SmallPageRecord& r = u.slots[id.slot];
  JENGA_CHECK(r.state == SmallPageState::kEvictable, "pin on a non-evictable page");
  lru_live_--;  // its heap entry goes stale with the state change
  if (u.evictable_count == u.slots.size()) fully_evictable_.erase(fe_it_[id.large.index]);
  u.evictable_count--;
  r.state = SmallPageState::kUsed;
  r.has_cache_key = false;
  r.cache_key = 0;
  r.associated_request = request;
  used_++;
}

// reference type_allocator.cpp:192-203
void TypeAllocator::touch(SmallPageId id, uint64_t step) {
  SmallPageRecord& r = rec(id);
  if (r.state == SmallPageState::kEvictable && r.last_access != step) {
    r.last_access = step;  // the old entry goes stale
    lru_push(lru_key(r, global_index(id.large.index, id.slot)));
  } else {
    r.last_access = step;
  }
}

// reference type_allocator.cpp:205-216
void TypeAllocator::set_prefix_length(SmallPageId id, uint64_t len) {
  SmallPageRecord& r = rec(id);
  if (r.state == SmallPageState::kEvictable && r.prefix_length != len) {
    r.prefix_length = len;  // the old entry goes stale
    lru_push(lru_key(r, global_index(id.large.index, id.slot)));
  } else {
    r.prefix_length = len;
  }
}

// reference type_allocator.cpp:218-228
void TypeAllocator::release_unit(uint32_t large) {
  JENGA_CHECK(large < units_.size() && units_[large].owned, "release of an unowned unit");
  Unit& u = units_[large];
  JENGA_CHECK(u.empty_count == u.slots.size(), "release of a non-empty unit");
  for (uint32_t s = 0; s < u.slots.size(); ++s)
    unindex_on_empty(global_index(large, s), u.slots[s]);
  pool_->return_large_page(LargePageId{large});
  u.owned = false;
  u.slots.clear();
  u.slots.shrink_to_fit();
  u.empty_count = u.evictable_count = 0;
  --owned_units_;
}

// reference type_allocator.cpp:230-244 (units in ascending first index)
std::vector<UnitEvictionCandidate> TypeAllocator::fully_evictable_units() const {
  std::vector<UnitEvictionCandidate> out;
  out.reserve(fully_evictable_.size());
  for (uint32_t first : fully_evictable_) {
    const Unit& u = units_[first];
    UnitEvictionCandidate c;
    c.first_index = first;
    for (const auto& s : u.slots) {
      c.lru_timestamp = std::max(c.lru_timestamp, s.last_access);
      c.max_prefix_length = std::max(c.max_prefix_length, s.prefix_length);
    }
    out.push_back(c);
  }
  return out;
}

// reference type_allocator.cpp:246-259
std::vector<uint64_t> TypeAllocator::clear_unit(uint32_t first_index) {
  JENGA_CHECK(first_index < units_.size() && units_[first_index].owned,
              "clear of an unowned unit");
  Unit& u = units_[first_index];
  JENGA_CHECK(u.evictable_count == u.slots.size(), "clear of a unit with non-evictable pages");
  std::vector<uint64_t> keys;
  keys.reserve(u.slots.size());
  for (uint32_t s = 0; s < geo_.slots_per_large; ++s)
    keys.push_back(evict_small(SmallPageId{LargePageId{first_index}, s}));
  release_unit(first_index);
  return keys;
}

// reference type_allocator.cpp:261-281
FragmentationReport TypeAllocator::fragmentation_report() const {
  FragmentationReport r;
  for (const Unit& u : units_) {
    if (!u.owned) continue;
    for (const auto& s : u.slots) {
      switch (s.state) {
        case SmallPageState::kUsed: r.used_bytes += geo_.small_page_bytes; break;
        case SmallPageState::kEvictable: r.evictable_bytes += geo_.small_page_bytes; break;
        case SmallPageState::kEmpty: r.empty_stranded_bytes += geo_.small_page_bytes; break;
      }
    }
  }
  return r;
}

// reference type_allocator.cpp:293-337
void TypeAllocator::check_invariants() const {
  uint64_t used = 0, evictable = 0, empty = 0, owned = 0, fully = 0;
  JENGA_CHECK(std::is_heap(lru_heap_.begin(), lru_heap_.end(), std::greater<LruKey>()), "LRU heap order broken");
  std::set<LruKey> heap_live;
  for (const LruKey& k : lru_heap_)
    if (lru_entry_live(k)) heap_live.insert(k);
  for (uint32_t first = 0; first < units_.size(); ++first) {
    const Unit& u = units_[first];
    if (!u.owned) continue;
    ++owned;
    JENGA_CHECK(u.slots.size() == geo_.slots_per_large, "unit slot count mismatch");
    uint32_t ue = 0, uv = 0;
    for (uint32_t s = 0; s < u.slots.size(); ++s) {
      const auto& r = u.slots[s];
      const uint64_t g = global_index(first, s);
      switch (r.state) {
        case SmallPageState::kUsed:
          ++used;
          JENGA_CHECK(r.associated_request != kNoRequest, "used page without request");
          JENGA_CHECK(!r.has_cache_key, "used page holds a cache key");
          JENGA_CHECK(!empty_.test(g), "used page on the empty index");
          break;
        case SmallPageState::kEvictable:
          ++evictable;
          ++uv;
          JENGA_CHECK(r.has_cache_key, "evictable page without cache key");
          JENGA_CHECK(heap_live.count(lru_key(r, g)) == 1, "evictable page missing from LRU index");
          break;
        case SmallPageState::kEmpty:
          ++empty;
          ++ue;
          JENGA_CHECK(!r.has_cache_key, "empty page holds a cache key");
          JENGA_CHECK(empty_.test(g), "empty page missing from index");
          break;
      }
    }
    JENGA_CHECK(ue == u.empty_count, "unit empty count drifted");
    JENGA_CHECK(uv == u.evictable_count, "unit evictable count drifted");
    JENGA_CHECK(ue < u.slots.size(), "fully-empty unit not released");
    const bool is_fully = uv == u.slots.size();
    JENGA_CHECK(is_fully == (fully_evictable_.count(first) == 1), "fully-evictable index drifted");
    if (is_fully) ++fully;
  }
  JENGA_CHECK(owned == owned_units_, "owned unit count drifted");
  JENGA_CHECK(used == used_, "used count drifted");
  JENGA_CHECK(evictable == lru_live_ && evictable == heap_live.size(), "LRU index size drifted");
  JENGA_CHECK(empty == empty_.count(), "empty index size drifted");
  JENGA_CHECK(fully == fully_evictable_.size(), "fully-evictable set size drifted");
}

// ------------------------------------------------------------ PrefixCache
// reference prefix_cache.cpp:9-18
uint64_t block_chain_salt(const std::string& group_name) {
  return mix64(hash_str(group_name), 0x6a656e6761ULL);
}

uint64_t chain_block_key(uint64_t parent, const std::vector<uint64_t>& tokens) {
  uint64_t h = parent;
  for (uint64_t t : tokens) h = mix64(h, t);
  return h;
}

// reference prefix_cache.cpp:59-100
const PrefixCache::Slot* PrefixCache::probe(const Table& t, uint64_t key) {
  if (t.slots.empty()) return nullptr;
  const size_t mask = t.slots.size() - 1;
  for (size_t i = home(key, mask);; i = (i + 1) & mask) {
    const Slot& s = t.slots[i];
    if (s.state == 0) return nullptr;
    if (s.state == 1 && s.key == key) return &s;
  }
}

void PrefixCache::rehash(Table& t, size_t capacity) {
  std::vector<Slot> old;
  old.swap(t.slots);
  t.slots.assign(capacity, Slot{});
  t.occupied = 0;
  const size_t mask = capacity - 1;
  for (const Slot& s : old) {
    if (s.state != 1) continue;
    size_t i = home(s.key, mask);
    while (t.slots[i].state != 0) i = (i + 1) & mask;
    t.slots[i] = s;
    ++t.occupied;
  }
}

PrefixCache::Slot& PrefixCache::insert_slot(Table& t, uint64_t key) {
  if (t.slots.empty() || (t.occupied + 1) * 2 > t.slots.size()) {
    size_t live = 0;
    for (const Slot& s : t.slots) live += s.state == 1;
    size_t cap = 64;
    while (cap < (live + 1) * 4) cap *= 2;  // <= 1/4 live after a rebuild (tombstones dropped)
    rehash(t, cap);
  }
  const size_t mask = t.slots.size() - 1;
  Slot* tomb = nullptr;
  for (size_t i = home(key, mask);; i = (i + 1) & mask) {
    Slot& s = t.slots[i];
    if (s.state == 1 && s.key == key) return s;
    if (s.state == 2 && tomb == nullptr) tomb = &s;
    if (s.state == 0) {
      Slot& dst = tomb != nullptr ? *tomb : s;
      if (tomb == nullptr) ++t.occupied;
      dst = Slot{key, kNil, kNil, 1};
      return dst;
    }
  }
}

void PrefixCache::register_block(size_t g, const BlockContent& c, SmallPageId page) {
  JENGA_CHECK(g < groups_.size(), "group index out of range");
  Table& t = groups_[g];
  uint32_t e;
  if (!t.free.empty()) {
    e = t.free.back();
    t.free.pop_back();
    t.pool[e] = Entry{c, page, kNil};
  } else {
    e = static_cast<uint32_t>(t.pool.size());
    t.pool.push_back(Entry{c, page, kNil});
  }
  Slot& s = insert_slot(t, c.key);
  if (s.tail == kNil) s.head = e;
  else t.pool[s.tail].next = e;
  s.tail = e;
  ++t.entries;
}

void PrefixCache::unregister(size_t g, uint64_t key, SmallPageId page) {
  JENGA_CHECK(g < groups_.size(), "group index out of range");
  Table& t = groups_[g];
  Slot* s = const_cast<Slot*>(probe(t, key));
  if (s == nullptr) return;
  // every entry of the key holding this page (the reference erases them all)
  uint32_t prev = kNil;
  for (uint32_t e = s->head; e != kNil;) {
    const uint32_t next = t.pool[e].next;
    if (t.pool[e].page == page) {
      if (prev == kNil) s->head = next;
      else t.pool[prev].next = next;
      if (s->tail == e) s->tail = prev;
      t.pool[e].content.tokens.clear();
      t.free.push_back(e);
      --t.entries;
    } else {
      prev = e;
    }
    e = next;
  }
  if (s->head == kNil) s->state = 2;  // tombstone
}

std::optional<SmallPageId> PrefixCache::find(size_t g, const BlockContent& c) const {
  JENGA_CHECK(g < groups_.size(), "group index out of range");
  const Table& t = groups_[g];
  const Slot* s = probe(t, c.key);
  if (s == nullptr) return std::nullopt;
  for (uint32_t e = s->head; e != kNil; e = t.pool[e].next)
    if (t.pool[e].content.matches(c)) return t.pool[e].page;
  return std::nullopt;
}

uint64_t PrefixCache::entries(size_t g) const {
  JENGA_CHECK(g < groups_.size(), "group index out of range");
  return groups_[g].entries;
}

// ------------------------------------------------------------ KvAllocator
// reference kv_allocator.cpp:67-79 (build_geometry, kJenga) + :136-152
KvAllocator::KvAllocator(const ModelSpec& spec, uint64_t budget_bytes)
    : spec_(spec), budget_(budget_bytes), cache_(spec.groups.size()) {
  spec_.validate();
  if (budget_bytes == 0) throw ConfigError("memory budget must be positive");
  if (spec_.groups.size() > 32000) throw ConfigError("too many layer groups");
  const uint64_t page = lcm_page_size(spec_);
  pool_ = std::make_unique<LargePagePool>(budget_bytes, page);
  for (size_t g = 0; g < spec_.groups.size(); ++g) {
    const uint64_t small = small_page_size(spec_.groups[g]);
    JENGA_CHECK(page % small == 0, "LCM page not divisible by small page");
    types_.push_back(std::make_unique<TypeAllocator>(
        GroupGeometry{spec_.groups[g].name, small, static_cast<uint32_t>(page / small)},
        static_cast<int>(g), pool_.get()));
  }
}

// Five-step allocation — reference kv_allocator.cpp:154-197
std::optional<AllocResult> KvAllocator::allocate(size_t g, uint64_t request) {
  JENGA_CHECK(g < types_.size(), "group index out of range");
  TypeAllocator& ta = *types_[g];
  if (request_aware_) {
    if (auto id = ta.try_allocate_associated(request)) {
      step_counts_[1]++;
      return AllocResult{*id, 1};
    }
  } else if (auto id = ta.try_allocate_any(request)) {
    step_counts_[1]++;
    return AllocResult{*id, 1};
  }
  if (auto id = ta.try_allocate_from_new_unit(request)) {
    step_counts_[2]++;
    return AllocResult{*id, 2};
  }
  while (pool_->num_free() < 1) {
    if (!evict_lru_large_page()) break;
  }
  if (auto id = ta.try_allocate_from_new_unit(request)) {
    step_counts_[3]++;
    return AllocResult{*id, 3};
  }
  if (request_aware_) {
    if (auto id = ta.try_allocate_any(request)) {
      step_counts_[4]++;
      return AllocResult{*id, 4};
    }
  }
  if (auto sid = ta.lru_evictable_small()) {
    const uint64_t key = ta.evict_small(*sid);
    cache_.unregister(g, key, *sid);
    ta.allocate_slot(*sid, request);
    step_counts_[5]++;
    return AllocResult{*sid, 5};
  }
  return std::nullopt;
}

// reference kv_allocator.cpp:199-208
void KvAllocator::free(size_t g, SmallPageId page, const std::optional<BlockContent>& cached) {
  JENGA_CHECK(g < types_.size(), "group index out of range");
  if (cached.has_value()) {
    types_[g]->free(page, cached->key);
    cache_.register_block(g, *cached, page);
  } else {
    types_[g]->free(page, std::nullopt);
  }
}

// reference kv_allocator.cpp:210-216
void KvAllocator::pin(size_t g, SmallPageId page, uint64_t request) {
  JENGA_CHECK(g < types_.size(), "group index out of range");
  const auto& r = types_[g]->record(page);
  JENGA_CHECK(r.has_cache_key, "pin of a page without cache key");
  cache_.unregister(g, r.cache_key, page);
  types_[g]->pin(page, request);
}

// reference kv_allocator.cpp:218-239
std::optional<LargePageId> KvAllocator::evict_lru_large_page() {
  std::optional<UnitEvictionCandidate> best;
  size_t best_group = 0;
  for (size_t g = 0; g < types_.size(); ++g) {
    for (const auto& c : types_[g]->fully_evictable_units()) {
      if (!best.has_value() || c.better_than(*best)) {
        best = c;
        best_group = g;
      }
    }
  }
  if (!best.has_value()) return std::nullopt;
  const std::vector<uint64_t> keys = types_[best_group]->clear_unit(best->first_index);
  for (uint32_t s = 0; s < keys.size(); ++s)
    cache_.unregister(best_group, keys[s], SmallPageId{LargePageId{best->first_index}, s});
  return LargePageId{best->first_index};
}

// reference kv_allocator.cpp:335-347 (byte conservation)
void KvAllocator::check_invariants() const {
  pool_->check_conservation();
  for (const auto& t : types_) t->check_invariants();
  uint64_t total = pool_->free_bytes() + pool_->reserved_remainder_bytes();
  for (const auto& t : types_)
    total += (t->used_pages() + t->evictable_pages() + t->empty_pages()) *
             t->geometry().small_page_bytes;
  JENGA_CHECK(total == budget_, "byte conservation violated");
}

}  // namespace jenga
