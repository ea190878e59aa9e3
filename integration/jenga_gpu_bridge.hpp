// jenga_gpu_bridge.hpp — the reference-side binding of the B200 path.
//
// Added next to the reference headers (proj/include/jenga); compiled against
// them and linked with libjenga_b200.so.  The reference's allocator stays the
// host API (KvAllocator / AddressMap / LayerView, kv_allocator.hpp:62-119,
// memory_layout.hpp:25-69); this header only turns its page lists into device
// block tables and its LayerView into kernel launches through the C ABI of
// include/jenga_gpu.h, mapping status codes back onto the reference's
// exception types (util.hpp:11-21).  tests/bridge/bridge_harness.cpp compiles
// exactly this file (INTEGRATION.md §1 quotes it verbatim).
#pragma once

#include <cuda_runtime_api.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "jenga/kv_allocator.hpp"
#include "jenga/memory_layout.hpp"
#include "jenga/util.hpp"
#include "jenga_gpu.h"

namespace jenga::gpu {

inline void check(int rc) {
  switch (rc) {
    case JENGA_OK: return;
    case JENGA_ERR_CONFIG: throw ConfigError(jenga_last_error());
    case JENGA_ERR_INVARIANT: throw InvariantError(jenga_last_error());
    default: throw std::runtime_error(jenga_last_error());
  }
}

inline void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// The device image of the allocator's LCM pool: one arena of
// num_pages x large_page_bytes (LargePagePool sizing, lcm_allocator.cpp:7-19).
class Arena {
 public:
  Arena(KvAllocator& kv, int device) {
    const LargePagePool& pool = kv.pool_of(0);  // the Jenga strategy has one pool
    check(jenga_arena_create(device, pool.num_pages(), pool.large_page_bytes(), &arena_));
  }
  ~Arena() { jenga_arena_destroy(arena_); }
  Arena(const Arena&) = delete;
  Arena& operator=(const Arena&) = delete;
  void* base() const { return jenga_arena_base(arena_); }
  uint64_t bytes() const { return jenga_arena_bytes(arena_); }

 private:
  jenga_arena* arena_ = nullptr;
};

// One request's page list in one group, as the caller's per-request
// bookkeeping holds it (SimEngine's GroupRuntime, simulator.hpp:123-139):
// the SmallPageId of every logical block, the leading dead blocks a sliding
// window freed (simulator.cpp:272-280) and the stored ordinals.
struct PageList {
  std::vector<SmallPageId> blocks;
  uint64_t first_live = 0;
  uint64_t stored = 0;
};

// Device block table of one group: int32 [batch][max_blocks] AddressMap
// global page indices (-1 dead / absent), seq_lens[batch], and the slot of
// each request's newest stored ordinal.
class DeviceTables {
 public:
  DeviceTables(int max_batch, int max_blocks) : max_batch_(max_batch), max_blocks_(max_blocks) {
    check_cuda(cudaMalloc(reinterpret_cast<void**>(&table_), sizeof(int32_t) * max_batch * max_blocks),
               "cudaMalloc block_table");
    check_cuda(cudaMalloc(reinterpret_cast<void**>(&seq_lens_), sizeof(int32_t) * max_batch), "cudaMalloc seq_lens");
    check_cuda(cudaMalloc(reinterpret_cast<void**>(&slots_), sizeof(int64_t) * max_batch), "cudaMalloc slot_mapping");
    check_cuda(cudaMalloc(&csr_, sizeof(int32_t) * (3 * max_batch + 1) + sizeof(jenga_small_page) * max_batch *
                                                                            static_cast<size_t>(max_blocks)),
               "cudaMalloc page lists");
  }
  ~DeviceTables() {
    cudaFree(table_);
    cudaFree(seq_lens_);
    cudaFree(slots_);
    cudaFree(csr_);
  }
  DeviceTables(const DeviceTables&) = delete;
  DeviceTables& operator=(const DeviceTables&) = delete;

  // Page lists -> CSR -> device (AddressMap::global_page_index on the device,
  // memory_layout.cpp:22-27).  Synchronous on `s` for the host staging.
  void build(const AddressMap& map, size_t g, const std::vector<PageList>& lists, cudaStream_t s) {
    const int batch = static_cast<int>(lists.size());
    if (batch > max_batch_) throw ConfigError("batch exceeds the block table");
    std::vector<int32_t> offsets(batch + 1, 0), first_live(batch), stored(batch);
    std::vector<jenga_small_page> pages;
    for (int b = 0; b < batch; ++b) {
      const PageList& pl = lists[b];
      if (pl.blocks.size() > static_cast<size_t>(max_blocks_)) throw ConfigError("request wider than the table");
      for (const SmallPageId& p : pl.blocks) pages.push_back(jenga_small_page{p.large.index, p.slot});
      offsets[b + 1] = static_cast<int32_t>(pages.size());
      first_live[b] = static_cast<int32_t>(pl.first_live);
      stored[b] = static_cast<int32_t>(pl.stored);
    }
    int32_t* d_off = static_cast<int32_t*>(csr_);
    int32_t* d_live = d_off + max_batch_ + 1;
    int32_t* d_stored = d_live + max_batch_;
    auto* d_pages = reinterpret_cast<jenga_small_page*>(d_stored + max_batch_);
    check_cuda(cudaMemcpyAsync(d_off, offsets.data(), sizeof(int32_t) * (batch + 1), cudaMemcpyHostToDevice, s),
               "page-list upload");
    check_cuda(cudaMemcpyAsync(d_live, first_live.data(), sizeof(int32_t) * batch, cudaMemcpyHostToDevice, s),
               "page-list upload");
    check_cuda(cudaMemcpyAsync(d_stored, stored.data(), sizeof(int32_t) * batch, cudaMemcpyHostToDevice, s),
               "page-list upload");
    if (!pages.empty())
      check_cuda(cudaMemcpyAsync(d_pages, pages.data(), sizeof(jenga_small_page) * pages.size(),
                                 cudaMemcpyHostToDevice, s),
                 "page-list upload");
    check(jenga_build_block_tables(d_off, d_pages, d_live, d_stored, batch, map.slots_per_large(g),
                                   map.group(g).tokens_per_page, max_blocks_, table_, slots_, seq_lens_, s));
    check_cuda(cudaStreamSynchronize(s), "page-list upload");  // host staging goes out of scope
  }

  int32_t* table() const { return table_; }
  int32_t* seq_lens() const { return seq_lens_; }
  int64_t* slots() const { return slots_; }
  int max_blocks() const { return max_blocks_; }

 private:
  int max_batch_, max_blocks_;
  int32_t* table_ = nullptr;
  int32_t* seq_lens_ = nullptr;
  int64_t* slots_ = nullptr;
  void* csr_ = nullptr;
};

inline jenga_layer_view to_c(const LayerView& v) {  // memory_layout.hpp:25-32
  return jenga_layer_view{v.start_offset, v.page_stride, v.exec_page_size};
}

// Attention over the needs_token ordinals of every request of a layer
// (layer_policies.cpp:105-120): the device half of SimEngine::decode_one
// (simulator.cpp:549-566) once store_position placed the new token.
inline void decode_layer(const Arena& arena, const LayerView& v, LayerKind kind, uint64_t window,
                         const void* q, void* out, const DeviceTables& t, int batch, int hq, int hkv, int d,
                         uint32_t tpp, float scale, float softcap, void* ws, size_t ws_bytes, cudaStream_t s) {
  check(jenga_paged_decode(arena.base(), to_c(v), static_cast<int>(kind), JENGA_BF16, window, q, out, t.table(),
                           t.seq_lens(), batch, t.max_blocks(), hq, hkv, d, tpp, scale, softcap, ws, ws_bytes, s));
}

// The same step with the new token's K/V written into its slot (the
// table's newest slot) by the decode launch itself.
inline void decode_layer_append(const Arena& arena, const LayerView& v, LayerKind kind, uint64_t window,
                                const void* q, const void* k_new, const void* v_new, void* out,
                                const DeviceTables& t, int batch, int hq, int hkv, int d, uint32_t tpp, float scale,
                                float softcap, void* ws, size_t ws_bytes, cudaStream_t s) {
  check(jenga_paged_decode_append(arena.base(), to_c(v), static_cast<int>(kind), JENGA_BF16, window, q, k_new,
                                  v_new, t.slots(), out, t.table(), t.seq_lens(), batch, t.max_blocks(), hq, hkv, d,
                                  tpp, scale, softcap, ws, ws_bytes, s));
}

}  // namespace jenga::gpu
