// reshape_and_cache: scatter new K/V rows into their small-page slots, and
// the Mamba state / checkpoint-page copies.
//
// Slot layout inside one layer's slice of a small page (our definition of the
// bytes the reference only sizes, memory_layout.cpp:16-17):
//     slice = [Hkv] x [K | V] x [tpp] x [D]   (exec_page_size = 2*Hkv*tpp*D*e)
// head-major: token `off` of head h is one contiguous D*e row, and one
// head's K and V tiles of a page are a single contiguous 2*tpp*D*e run (the
// DRAM-locality choice measured in profiles/r01_sweeps.md).  Source and destination
// rows are both contiguous, so one warp moves a 256..512-B row with 16-B
// vector stores — fully coalesced on both sides.
#include "common.cuh"

namespace {

// One thread per 16-byte chunk of one (token, head, K|V) row.
__global__ void __launch_bounds__(256) reshape_and_cache_kernel(
    uint8_t* __restrict__ arena, uint64_t start_offset, uint64_t page_stride, int hkv, int row_bytes,
    uint32_t tpp, const uint8_t* __restrict__ key, const uint8_t* __restrict__ value,
    int64_t token_stride_bytes, const int64_t* __restrict__ slots, int n_tokens) {
  const int chunks_per_row = row_bytes >> 4;
  // PDL: let the decode kernel that follows get resident now; wait for our own
  // prerequisites (the previous layer's decode) before touching the arena.
  jenga_dev::pdl_launch_dependents();
  jenga_dev::pdl_wait();
  const int64_t total = static_cast<int64_t>(n_tokens) * hkv * 2 * chunks_per_row;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % chunks_per_row);
    int64_t r = i / chunks_per_row;
    const int kv = static_cast<int>(r % 2);
    r /= 2;
    const int h = static_cast<int>(r % hkv);
    const int t = static_cast<int>(r / hkv);
    const int64_t slot = slots[t];
    if (slot < 0) continue;
    const int64_t page = slot / tpp;
    const int64_t off = slot % tpp;
    const uint8_t* src = (kv ? value : key) + t * token_stride_bytes + static_cast<int64_t>(h) * row_bytes +
                         (c << 4);
    uint8_t* dst = arena + start_offset + page * page_stride +
                   ((static_cast<int64_t>(h) * 2 + kv) * tpp + off) * row_bytes + (c << 4);
    jenga_dev::st_v4(dst, jenga_dev::ld_nc_v4(src));
  }
}

// dst[b] <- src[b], `bytes` per item, 16-B vectors, 4 in flight per thread.
__global__ void __launch_bounds__(256) paged_copy_kernel(const uint8_t* __restrict__ src_base,
                                                         uint64_t src_off, uint64_t src_stride,
                                                         const int64_t* __restrict__ src_idx,
                                                         uint8_t* __restrict__ dst_base, uint64_t dst_off,
                                                         uint64_t dst_stride,
                                                         const int64_t* __restrict__ dst_idx,
                                                         uint64_t bytes) {
  const int b = blockIdx.y;
  const int64_t si = src_idx ? src_idx[b] : b;
  const int64_t di = dst_idx ? dst_idx[b] : b;
  if (si < 0 || di < 0) return;
  const uint8_t* s = src_base + src_off + si * src_stride;
  uint8_t* d = dst_base + dst_off + di * dst_stride;
  const uint64_t nvec = bytes >> 4;
  const uint64_t step = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + 3 * step < nvec; i += 4 * step) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = jenga_dev::ld_nc_v4(s + ((i + u * step) << 4));
#pragma unroll
    for (int u = 0; u < 4; ++u) jenga_dev::st_v4(d + ((i + u * step) << 4), v[u]);
  }
  for (; i < nvec; i += step) jenga_dev::st_v4(d + (i << 4), jenga_dev::ld_nc_v4(s + (i << 4)));
}

// Token rows <-> pages.  Row t (row_bytes) of the token at slot s = page*tpp +
// off is cut into piece_bytes pieces; piece p sits in layer p / ppl, sub-slice
// q = p % ppl of the page-layer layout:
//     arena + start + layer*layer_stride + page*page_stride + (q*tpp + off)*piece_bytes
// ppl = 1, piece = row: a vision-embedding group's own pages ([tpp][row]).
// ppl = 2*Hkv, piece = D*e: the K|V, head rows reshape_and_cache will write
// for that same token — the full_reuse overlay parks an embedding exactly in
// its own token's unwritten KV bytes, so writing one token's KV never touches
// another token's parked embedding.  One thread per 16-byte chunk.
template <bool kScatter>
__global__ void __launch_bounds__(256) token_rows_kernel(uint8_t* __restrict__ arena, uint64_t start_offset,
                                                         uint64_t layer_stride, uint64_t page_stride, uint32_t tpp,
                                                         uint32_t ppl, uint32_t piece_chunks, uint32_t row_chunks,
                                                         uint8_t* __restrict__ rows, int64_t row_stride,
                                                         const int64_t* __restrict__ slots, int n_tokens) {
  const int64_t total = static_cast<int64_t>(n_tokens) * row_chunks;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int t = static_cast<int>(i / row_chunks);
    const uint32_t c = static_cast<uint32_t>(i - static_cast<int64_t>(t) * row_chunks);
    const uint32_t piece = c / piece_chunks, pc = c - piece * piece_chunks;
    const uint32_t layer = piece / ppl, q = piece - layer * ppl;
    uint8_t* row = rows + t * row_stride + (static_cast<int64_t>(c) << 4);
    const int64_t slot = slots[t];
    if (slot < 0) {
      if (!kScatter) jenga_dev::st_v4(row, make_uint4(0, 0, 0, 0));
      continue;
    }
    const int64_t page = slot / tpp, off = slot - page * tpp;
    uint8_t* cell = arena + start_offset + layer * layer_stride + page * page_stride +
                    ((static_cast<int64_t>(q) * tpp + off) * piece_chunks + pc) * 16;
    if (kScatter)
      jenga_dev::st_v4(cell, jenga_dev::ld_nc_v4(row));
    else
      jenga_dev::st_v4(row, jenga_dev::ld_nc_v4(cell));
  }
}

int launch_token_rows(bool scatter, void* arena_base, jenga_layer_view view, uint32_t num_layers,
                      uint32_t pieces_per_layer, uint32_t piece_bytes, uint32_t tpp, void* rows, uint64_t row_bytes,
                      int64_t row_stride_bytes, const int64_t* slots, int n_tokens, void* stream) {
  using namespace jenga_dev;
  const char* what = scatter ? "jenga_token_rows_scatter" : "jenga_token_rows_gather";
  if (!arena_base || (n_tokens > 0 && (!rows || !slots)) || n_tokens < 0 || tpp == 0 || pieces_per_layer == 0 ||
      piece_bytes == 0 || num_layers == 0 || row_bytes == 0)
    return set_error(JENGA_ERR_ARG, std::string(what) + ": invalid arguments");
  if (piece_bytes % 16 || row_bytes % piece_bytes || row_stride_bytes % 16 || view.start_offset % 16 ||
      view.page_stride % 16 || view.exec_page_size % 16)
    return set_error(JENGA_ERR_UNSUPPORTED, std::string(what) + ": pieces and rows must be 16-byte multiples");
  if (static_cast<uint64_t>(pieces_per_layer) * tpp * piece_bytes > view.exec_page_size)
    return set_error(JENGA_ERR_CONFIG, std::string(what) + ": pieces_per_layer*tpp*piece_bytes exceeds the layer slice");
  if (row_bytes > static_cast<uint64_t>(num_layers) * pieces_per_layer * piece_bytes)
    return set_error(JENGA_ERR_CONFIG, std::string(what) + ": row larger than the token's bytes in the group");
  if (n_tokens == 0) return JENGA_OK;
  const uint32_t row_chunks = static_cast<uint32_t>(row_bytes / 16);
  const int64_t total = static_cast<int64_t>(n_tokens) * row_chunks;
  const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16));
  auto kern = scatter ? token_rows_kernel<true> : token_rows_kernel<false>;
  kern<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<uint8_t*>(arena_base), view.start_offset, view.exec_page_size, view.page_stride, tpp,
      pieces_per_layer, piece_bytes / 16, row_chunks, static_cast<uint8_t*>(rows), row_stride_bytes, slots, n_tokens);
  return check_launch(scatter ? "token_rows_kernel<scatter>" : "token_rows_kernel<gather>");
}

int launch_paged_copy(const void* src_base, uint64_t src_off, uint64_t src_stride, const int64_t* src_idx,
                      void* dst_base, uint64_t dst_off, uint64_t dst_stride, const int64_t* dst_idx,
                      uint64_t bytes, int n, void* stream, const char* what) {
  using namespace jenga_dev;
  if (n <= 0 || bytes == 0) return JENGA_OK;
  if (bytes % 16 != 0 || src_off % 16 != 0 || dst_off % 16 != 0 || src_stride % 16 != 0 ||
      dst_stride % 16 != 0)
    return set_error(JENGA_ERR_UNSUPPORTED, std::string(what) + ": sizes/offsets must be 16-byte multiples");
  const uint64_t nvec = bytes >> 4;
  int gx = static_cast<int>(std::min<uint64_t>((nvec + 1023) / 1024, 512));
  if (gx < 1) gx = 1;
  dim3 grid(gx, n);
  paged_copy_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint8_t*>(src_base), src_off, src_stride, src_idx, static_cast<uint8_t*>(dst_base),
      dst_off, dst_stride, dst_idx, bytes);
  return check_launch(what);
}

}  // namespace

JENGA_EXPORT int jenga_reshape_and_cache(void* arena_base, jenga_layer_view view, int dtype, int num_kv_heads,
                                         int head_dim, uint32_t tokens_per_page, const void* key,
                                         const void* value, int64_t kv_token_stride,
                                         const int64_t* slot_mapping, int n_tokens, void* stream) {
  using namespace jenga_dev;
  const int e = dtype_bytes(dtype);
  if (e == 0 || num_kv_heads <= 0 || head_dim <= 0 || tokens_per_page == 0 || n_tokens < 0)
    return set_error(JENGA_ERR_ARG, "jenga_reshape_and_cache: invalid arguments");
  const int row_bytes = head_dim * e;
  if (view.exec_page_size != 2ull * num_kv_heads * tokens_per_page * row_bytes)
    return set_error(JENGA_ERR_CONFIG,
                     "jenga_reshape_and_cache: exec_page_size != 2*Hkv*tpp*D*dtype (layer view mismatch)");
  if (row_bytes % 16 != 0 || view.start_offset % 16 != 0 || view.page_stride % 16 != 0)
    return set_error(JENGA_ERR_UNSUPPORTED, "jenga_reshape_and_cache: rows must be 16-byte aligned");
  if (n_tokens == 0) return JENGA_OK;
  const int64_t total = static_cast<int64_t>(n_tokens) * num_kv_heads * 2 * (row_bytes / 16);
  const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16));
  launch_maybe_pdl(reshape_and_cache_kernel, dim3(blocks), dim3(256), 0, static_cast<cudaStream_t>(stream),
                   static_cast<uint8_t*>(arena_base), view.start_offset, view.page_stride, num_kv_heads, row_bytes,
                   tokens_per_page, static_cast<const uint8_t*>(key), static_cast<const uint8_t*>(value),
                   kv_token_stride * e, slot_mapping, n_tokens);
  return check_launch("reshape_and_cache_kernel");
}

JENGA_EXPORT int jenga_mamba_state_gather(const void* arena_base, jenga_layer_view view,
                                          const int64_t* page_globals, int batch, void* dense, void* stream) {
  return launch_paged_copy(arena_base, view.start_offset, view.page_stride, page_globals, dense, 0,
                           view.exec_page_size, nullptr, view.exec_page_size, batch, stream,
                           "mamba_state_gather");
}

JENGA_EXPORT int jenga_mamba_state_scatter(void* arena_base, jenga_layer_view view,
                                           const int64_t* page_globals, int batch, const void* dense,
                                           void* stream) {
  return launch_paged_copy(dense, 0, view.exec_page_size, nullptr, arena_base, view.start_offset,
                           view.page_stride, page_globals, view.exec_page_size, batch, stream,
                           "mamba_state_scatter");
}

JENGA_EXPORT int jenga_page_copy(void* arena_base, uint64_t small_page_bytes, const int64_t* src_globals,
                                 const int64_t* dst_globals, int n_pages, void* stream) {
  return launch_paged_copy(arena_base, 0, small_page_bytes, src_globals, arena_base, 0, small_page_bytes,
                           dst_globals, small_page_bytes, n_pages, stream, "page_copy");
}

JENGA_EXPORT int jenga_token_rows_scatter(void* arena_base, jenga_layer_view view, uint32_t num_layers,
                                          uint32_t pieces_per_layer, uint32_t piece_bytes, uint32_t tokens_per_page,
                                          const void* rows, uint64_t row_bytes, int64_t row_stride_bytes,
                                          const int64_t* slot_mapping, int n_tokens, void* stream) {
  return launch_token_rows(true, arena_base, view, num_layers, pieces_per_layer, piece_bytes, tokens_per_page,
                           const_cast<void*>(rows), row_bytes, row_stride_bytes, slot_mapping, n_tokens, stream);
}

JENGA_EXPORT int jenga_token_rows_gather(const void* arena_base, jenga_layer_view view, uint32_t num_layers,
                                         uint32_t pieces_per_layer, uint32_t piece_bytes, uint32_t tokens_per_page,
                                         void* rows, uint64_t row_bytes, int64_t row_stride_bytes,
                                         const int64_t* slot_mapping, int n_tokens, void* stream) {
  return launch_token_rows(false, const_cast<void*>(arena_base), view, num_layers, pieces_per_layer, piece_bytes,
                           tokens_per_page, rows, row_bytes, row_stride_bytes, slot_mapping, n_tokens, stream);
}
