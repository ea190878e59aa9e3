// Block-table and slot-mapping construction on the device.
//
// Input is the allocator's page lists in CSR form — for request b the
// SmallPageIds {large, slot} of its logical blocks 0..count-1, of which the
// leading first_live_block[b] are dead (sliding-window blocks freed at
// simulator.cpp:272-280).  Output is the AddressMap global page index
// (reference memory_layout.cpp:22-27: large*slots_per_large + slot) per
// logical block, -1 for dead/absent blocks, and the slot of a token:
// global*tpp + (ordinal-1)%tpp.
#include "common.cuh"

namespace {

__global__ void __launch_bounds__(256) build_tables_kernel(
    const int32_t* __restrict__ offsets, const jenga_small_page* __restrict__ pages,
    const int32_t* __restrict__ first_live, const int32_t* __restrict__ n_stored, int batch,
    uint32_t slots_per_large, uint32_t tpp, int max_blocks, int32_t* __restrict__ table,
    int64_t* __restrict__ slot_mapping, int32_t* __restrict__ seq_lens) {
  const int b = blockIdx.y;
  if (b >= batch) return;
  const int begin = offsets[b];
  const int count = offsets[b + 1] - begin;
  const int live0 = first_live ? first_live[b] : 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < max_blocks; i += gridDim.x * blockDim.x) {
    int32_t v = -1;
    if (i < count && i >= live0) {
      const jenga_small_page p = pages[begin + i];
      v = static_cast<int32_t>(static_cast<uint64_t>(p.large) * slots_per_large + p.slot);
    }
    table[static_cast<int64_t>(b) * max_blocks + i] = v;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const int n = n_stored ? n_stored[b] : 0;
    if (seq_lens) seq_lens[b] = n;
    if (slot_mapping) {
      int64_t slot = -1;
      if (n > 0) {
        const int blk = (n - 1) / static_cast<int>(tpp);
        if (blk < count && blk >= live0) {
          const jenga_small_page p = pages[begin + blk];
          const int64_t g = static_cast<int64_t>(p.large) * slots_per_large + p.slot;
          slot = g * tpp + (n - 1) % static_cast<int>(tpp);
        }
      }
      slot_mapping[b] = slot;
    }
  }
}

__global__ void __launch_bounds__(256) slot_mapping_kernel(const int32_t* __restrict__ table,
                                                           int max_blocks, const int32_t* __restrict__ req,
                                                           const int32_t* __restrict__ ord, int n,
                                                           uint32_t tpp, int64_t* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int o = ord[t];
  int64_t slot = -1;
  if (o >= 1) {
    const int blk = (o - 1) / static_cast<int>(tpp);
    if (blk < max_blocks) {
      const int32_t g = table[static_cast<int64_t>(req[t]) * max_blocks + blk];
      if (g >= 0) slot = static_cast<int64_t>(g) * tpp + (o - 1) % static_cast<int>(tpp);
    }
  }
  out[t] = slot;
}

// Apply a delta buffer (jenga_pages_pack_deltas) to one group's device table:
//   [0] n_records [1] n_rows [2] max_blocks [3] seq [4] ack [5..7] 0 |
//   int64 slots[n_rows] | int32 seq_lens[n_rows] (+1 pad if n_rows is odd) |
//   int32 (flat entry, value)[n_records] (8-byte aligned)
// `delta` is device memory (a copy of the host buffer); the launch writes the
// buffer's sequence number to `ack` (word 4 of the host buffer, pinned memory
// the device can store to), which tells the next pack its predecessor landed.
__global__ void __launch_bounds__(256) apply_deltas_kernel(const int32_t* __restrict__ delta,
                                                            int32_t* __restrict__ ack, int max_batch,
                                                            int max_blocks, int32_t* __restrict__ table,
                                                            int32_t* __restrict__ seq_lens,
                                                            int64_t* __restrict__ slot_mapping) {
  const int n_rec = delta[0];
  const int rows_packed = delta[1];
  const int n_rows = min(rows_packed, max_batch);
  if (delta[2] != max_blocks) return;  // a buffer packed for another table: leave it untouched
  if (ack != nullptr && blockIdx.x == 0 && threadIdx.x == 0) *reinterpret_cast<volatile int32_t*>(ack) = delta[3];
  const int64_t entries = static_cast<int64_t>(max_batch) * max_blocks;
  const int64_t* slots = reinterpret_cast<const int64_t*>(delta + 8);
  const int32_t* seqs = delta + 8 + 2 * rows_packed;
  const int2* rec = reinterpret_cast<const int2*>(seqs + rows_packed + (rows_packed & 1));
  const int stride = gridDim.x * blockDim.x;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_rows; i += stride) {
    if (seq_lens) seq_lens[i] = seqs[i];
    if (slot_mapping) slot_mapping[i] = slots[i];
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_rec; i += stride) {
    const int2 r = rec[i];
    if (r.x >= 0 && r.x < entries) table[r.x] = r.y;
  }
}

}  // namespace

JENGA_EXPORT int jenga_upload_page_list_deltas(const void* delta, int32_t* ack, int max_batch, int max_blocks,
                                               int32_t* block_table, int32_t* seq_lens, int64_t* slot_mapping,
                                               void* stream) {
  using namespace jenga_dev;
  if (delta == nullptr || block_table == nullptr || max_batch < 0 || max_blocks <= 0 ||
      reinterpret_cast<uintptr_t>(delta) % 8 != 0)
    return set_error(JENGA_ERR_ARG, "jenga_upload_page_list_deltas: invalid arguments");
  if (max_batch == 0) return JENGA_OK;
  apply_deltas_kernel<<<4, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const int32_t*>(delta), ack, max_batch, max_blocks, block_table, seq_lens, slot_mapping);
  note_launch(static_cast<cudaStream_t>(stream), kLaunchSerializing);
  return check_launch("apply_deltas_kernel");
}

JENGA_EXPORT int jenga_build_block_tables(const int32_t* offsets, const jenga_small_page* pages,
                                          const int32_t* first_live_block, const int32_t* n_stored,
                                          int batch, uint32_t slots_per_large, uint32_t tokens_per_page,
                                          int max_blocks, int32_t* block_table, int64_t* slot_mapping,
                                          int32_t* seq_lens, void* stream) {
  using namespace jenga_dev;
  if (batch < 0 || max_blocks < 0 || offsets == nullptr || block_table == nullptr ||
      tokens_per_page == 0 || slots_per_large == 0)
    return set_error(JENGA_ERR_ARG, "jenga_build_block_tables: invalid arguments");
  if (batch == 0 || (max_blocks == 0 && slot_mapping == nullptr && seq_lens == nullptr)) return JENGA_OK;
  const int threads = 256;
  const int gx = max_blocks > 0 ? (max_blocks + threads - 1) / threads : 1;
  dim3 grid(gx, batch);
  build_tables_kernel<<<grid, threads, 0, static_cast<cudaStream_t>(stream)>>>(
      offsets, pages, first_live_block, n_stored, batch, slots_per_large, tokens_per_page, max_blocks,
      block_table, slot_mapping, seq_lens);
  note_launch(static_cast<cudaStream_t>(stream), kLaunchSerializing);
  return check_launch("build_tables_kernel");
}

JENGA_EXPORT int jenga_slot_mapping(const int32_t* block_table, int max_blocks, const int32_t* req,
                                    const int32_t* ord, int n_tokens, uint32_t tokens_per_page,
                                    int64_t* slot_mapping, void* stream) {
  using namespace jenga_dev;
  if (n_tokens < 0 || tokens_per_page == 0 || (n_tokens > 0 && (!block_table || !req || !ord || !slot_mapping)))
    return set_error(JENGA_ERR_ARG, "jenga_slot_mapping: invalid arguments");
  if (n_tokens == 0) return JENGA_OK;
  slot_mapping_kernel<<<(n_tokens + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      block_table, max_blocks, req, ord, n_tokens, tokens_per_page, slot_mapping);
  note_launch(static_cast<cudaStream_t>(stream), kLaunchSerializing);
  return check_launch("slot_mapping_kernel");
}
