// bridge_harness.cpp — TEST INFRASTRUCTURE ONLY (built by oracle/build_oracle.py
// into oracle/_ref/libjenga_bridge_test.so when /root/reference is present;
// loaded by tests/test_gpu_bridge.py).
//
// A reference-side worker, exactly as INTEGRATION.md §1 describes one: the
// UNMODIFIED reference allocator (proj/src, public API only — KvAllocator,
// AddressMap, LayerView) produces the page lists, and the reference-side
// bridge integration/jenga_gpu_bridge.hpp turns them into device block tables
// and fused decode launches through libjenga_b200.so's C ABI.  Everything
// the test needs to check the device against the C oracle is copied back.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <optional>
#include <string>
#include <vector>

#include "jenga/model_config.hpp"
#include "jenga_gpu_bridge.hpp"

namespace {

// store_position's page-list bookkeeping for text positions (simulator.cpp:
// 217-282) over the reference allocator: a block per tokens_per_page stored
// ordinals, sliding-window blocks freed once they left the window.
void store(jenga::KvAllocator& kv, size_t g, uint64_t request, jenga::gpu::PageList& pl) {
  const jenga::LayerGroupSpec& grp = kv.group(g);
  pl.stored++;
  const uint64_t t = grp.tokens_per_page;
  const uint64_t bidx = (pl.stored - 1) / t;
  if (bidx >= pl.blocks.size()) {
    auto res = kv.allocate(g, request);
    if (!res) throw jenga::ConfigError("reference allocator out of memory");
    pl.blocks.push_back(res->page);
  }
  if (grp.kind == jenga::LayerKind::kSlidingWindow && pl.stored > grp.window_tokens) {
    const uint64_t exited = pl.stored - grp.window_tokens;
    while ((pl.first_live + 1) * t <= exited) kv.free(g, pl.blocks[pl.first_live++], std::nullopt);
  }
}

}  // namespace

// Groups of the spec must be attention groups (full / sliding window).  The
// requests store positions in the order `sequence` lists them (request index
// per stored position, n_positions long); the LAST position of every request
// is the decode token whose K/V the fused launch appends.  Per group g:
//   pages_out[g][cap][2], offsets_out[g][n_req+1], first_live_out / stored_out
//   [g][n_req]: the reference page lists (CSR);
//   table_out[g][n_req][max_blocks], seq_out[g][n_req], slot_out[g][n_req]:
//   the device block tables the bridge built;
//   q / k_new / v_new / out [g][n_req][h][d] bf16: layer `layer`'s decode.
// arena_init (arena_bytes) is the arena before the step; arena_out after it.
extern "C" __attribute__((visibility("default"))) int bridge_run(
    const char* spec_json, uint64_t budget, int n_req, const int32_t* sequence, int64_t n_positions, int max_blocks,
    int cap, int32_t* pages_out, int32_t* offsets_out, int32_t* first_live_out, int32_t* stored_out,
    int32_t* table_out, int32_t* seq_out, int64_t* slot_out, const uint8_t* arena_init, uint64_t arena_bytes,
    int layer, const void* q, const void* k_new, const void* v_new, void* out, uint8_t* arena_out, int hq, int hkv,
    int d, float softcap, char* err, int err_cap) {
  try {
    const jenga::ModelSpec spec = jenga::parse_model_spec_json(spec_json);
    jenga::KvAllocator kv(spec, jenga::AllocStrategy::kJenga, budget);
    const jenga::AddressMap map(spec);
    const size_t G = spec.groups.size();
    std::vector<std::vector<jenga::gpu::PageList>> lists(G, std::vector<jenga::gpu::PageList>(n_req));
    for (int64_t i = 0; i < n_positions; ++i) {
      const int r = sequence[i];
      if (r < 0 || r >= n_req) throw jenga::ConfigError("request index out of range");
      for (size_t g = 0; g < G; ++g) store(kv, g, static_cast<uint64_t>(r), lists[g][r]);
    }
    kv.check_invariants();

    jenga::gpu::Arena arena(kv, 0);
    if (arena.bytes() != arena_bytes) throw jenga::ConfigError("arena size mismatch");
    jenga::gpu::check_cuda(cudaMemcpy(arena.base(), arena_init, arena_bytes, cudaMemcpyHostToDevice), "arena init");
    cudaStream_t s = nullptr;
    jenga::gpu::check_cuda(cudaStreamCreate(&s), "stream");
    const size_t row = static_cast<size_t>(n_req) * hq * d * 2, krow = static_cast<size_t>(n_req) * hkv * d * 2;
    void *dq = nullptr, *dk = nullptr, *dv = nullptr, *dout = nullptr, *ws = nullptr;
    const size_t ws_bytes = jenga_paged_decode_workspace_size(n_req, hq, hkv, d, max_blocks, 16);
    jenga::gpu::check_cuda(cudaMalloc(&dq, row), "q");
    jenga::gpu::check_cuda(cudaMalloc(&dout, row), "out");
    jenga::gpu::check_cuda(cudaMalloc(&dk, krow), "k");
    jenga::gpu::check_cuda(cudaMalloc(&dv, krow), "v");
    jenga::gpu::check_cuda(cudaMalloc(&ws, ws_bytes), "workspace");
    jenga::gpu::check_cuda(cudaMemset(ws, 0, ws_bytes), "workspace");
    for (size_t g = 0; g < G; ++g) {
      // the reference page lists, as the caller holds them
      int32_t* off = offsets_out + g * (n_req + 1);
      int32_t* pg = pages_out + g * static_cast<size_t>(cap) * 2;
      off[0] = 0;
      for (int r = 0; r < n_req; ++r) {
        const auto& pl = lists[g][r];
        if (off[r] + static_cast<int64_t>(pl.blocks.size()) > cap) throw jenga::ConfigError("cap too small");
        for (size_t b = 0; b < pl.blocks.size(); ++b) {
          pg[2 * (off[r] + b)] = static_cast<int32_t>(pl.blocks[b].large.index);
          pg[2 * (off[r] + b) + 1] = static_cast<int32_t>(pl.blocks[b].slot);
        }
        off[r + 1] = off[r] + static_cast<int32_t>(pl.blocks.size());
        first_live_out[g * n_req + r] = static_cast<int32_t>(pl.first_live);
        stored_out[g * n_req + r] = static_cast<int32_t>(pl.stored);
      }
      // through the bridge: tables, then one fused decode-append launch
      jenga::gpu::DeviceTables t(n_req, max_blocks);
      t.build(map, g, lists[g], s);
      jenga::gpu::check_cuda(cudaMemcpy(table_out + g * static_cast<size_t>(n_req) * max_blocks, t.table(),
                                        sizeof(int32_t) * n_req * max_blocks, cudaMemcpyDeviceToHost), "table");
      jenga::gpu::check_cuda(cudaMemcpy(seq_out + g * n_req, t.seq_lens(), sizeof(int32_t) * n_req,
                                        cudaMemcpyDeviceToHost), "seq_lens");
      jenga::gpu::check_cuda(cudaMemcpy(slot_out + g * n_req, t.slots(), sizeof(int64_t) * n_req,
                                        cudaMemcpyDeviceToHost), "slots");
      const auto* qh = static_cast<const uint8_t*>(q) + g * row;
      jenga::gpu::check_cuda(cudaMemcpy(dq, qh, row, cudaMemcpyHostToDevice), "q");
      jenga::gpu::check_cuda(cudaMemcpy(dk, static_cast<const uint8_t*>(k_new) + g * krow, krow,
                                        cudaMemcpyHostToDevice), "k");
      jenga::gpu::check_cuda(cudaMemcpy(dv, static_cast<const uint8_t*>(v_new) + g * krow, krow,
                                        cudaMemcpyHostToDevice), "v");
      const jenga::LayerGroupSpec& grp = spec.groups[g];
      jenga::gpu::decode_layer_append(arena, map.layer_view(g, static_cast<uint32_t>(layer)), grp.kind,
                                      grp.window_tokens, dq, dk, dv, dout, t, n_req, hq, hkv, d,
                                      grp.tokens_per_page, 1.0f / std::sqrt(static_cast<float>(d)), softcap, ws,
                                      ws_bytes, s);
      jenga::gpu::check_cuda(cudaStreamSynchronize(s), "decode");
      jenga::gpu::check_cuda(cudaMemcpy(static_cast<uint8_t*>(out) + g * row, dout, row, cudaMemcpyDeviceToHost),
                             "out");
    }
    jenga::gpu::check_cuda(cudaMemcpy(arena_out, arena.base(), arena_bytes, cudaMemcpyDeviceToHost), "arena");
    cudaFree(dq);
    cudaFree(dk);
    cudaFree(dv);
    cudaFree(dout);
    cudaFree(ws);
    cudaStreamDestroy(s);
    return 0;
  } catch (const std::exception& e) {
    std::snprintf(err, static_cast<size_t>(err_cap), "%s", e.what());
    return 1;
  }
}
