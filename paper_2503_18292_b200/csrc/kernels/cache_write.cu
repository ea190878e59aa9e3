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
#include <array>
#include <cstdio>

#include "decode_common.cuh"

namespace {

// Division by a run-time constant for dividends < 2^31: q = umulhi(n, m) >> s
// with m = ceil(2^(31+l) / d), l = ceil(log2 d) (Granlund-Montgomery).
struct FastDiv {
  uint32_t d = 1, m = 0, s = 0;
  FastDiv() = default;
  explicit FastDiv(uint32_t div) : d(div) {
    if (d <= 1) return;
    uint32_t l = 0;
    while ((1ull << l) < d) ++l;
    m = static_cast<uint32_t>(((1ull << (31 + l)) + d - 1) / d);
    s = l - 1;
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const { return d == 1 ? n : (__umulhi(n, m) >> s); }
};

// One thread per 16-byte chunk of one (token, head, K|V) row, four chunks in
// flight per thread (loads first, then stores); index math by multiply-shift
// (the host launches at most 2^30 chunks at a time).
constexpr int kRcUnroll = 4;

__global__ void __launch_bounds__(256) reshape_and_cache_kernel(
    uint8_t* __restrict__ arena, uint64_t start_offset, uint64_t page_stride, uint32_t row_bytes, uint32_t tpp,
    FastDiv per_token, FastDiv per_row, FastDiv by_tpp, const uint8_t* __restrict__ key,
    const uint8_t* __restrict__ value, int64_t token_stride_bytes, const int64_t* __restrict__ slots, uint32_t total) {
  // PDL: let the decode kernel that follows get resident now; wait for our own
  // prerequisites (the previous layer's decode) before touching the arena.
  jenga_dev::pdl_launch_dependents();
  jenga_dev::pdl_wait();
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < total; i0 += kRcUnroll * stride) {
    uint4 v[kRcUnroll];
    uint8_t* dst[kRcUnroll];
#pragma unroll
    for (int u = 0; u < kRcUnroll; ++u) {
      dst[u] = nullptr;
      const uint32_t i = i0 + u * stride;
      if (i >= total) continue;
      const uint32_t t = per_token.div(i);            // token
      const uint32_t w = i - t * per_token.d;         // chunk within the token's 2*Hkv rows
      const uint32_t row = per_row.div(w);            // (head, K|V) = (row >> 1, row & 1)
      const uint32_t c = w - row * per_row.d;
      const int64_t slot = slots[t];
      if (slot < 0) continue;
      uint64_t page;
      uint32_t off;
      if (slot < (1ll << 31)) {
        const uint32_t s32 = static_cast<uint32_t>(slot);
        const uint32_t pg = by_tpp.div(s32);
        page = pg;
        off = s32 - pg * tpp;
      } else {
        page = static_cast<uint64_t>(slot) / tpp;
        off = static_cast<uint32_t>(static_cast<uint64_t>(slot) - page * tpp);
      }
      v[u] = jenga_dev::ld_nc_v4(((row & 1u) ? value : key) + t * token_stride_bytes + (row >> 1) * row_bytes +
                                 (c << 4));
      // head-major slice: row (h, kv) of token `off` at ((2h + kv) * tpp + off) * row_bytes
      dst[u] = arena + start_offset + page * page_stride + static_cast<uint64_t>(row * tpp + off) * row_bytes +
               (c << 4);
    }
#pragma unroll
    for (int u = 0; u < kRcUnroll; ++u)
      if (dst[u] != nullptr) jenga_dev::st_v4(dst[u], v[u]);
  }
}

// dst[b] <- src[b], `nvec` 16-byte units per item, through the TMA bulk-copy
// engine: a persistent grid, each CTA owning an equal contiguous share of the
// flattened (item, unit) space; one elected thread streams it in <= kCopyChunk
// pieces (never crossing an item) through a kCopyStages-deep shared-memory ring
// (cp.async.bulk global->shared, completion on an mbarrier, then
// cp.async.bulk shared->global).  The thread refills the stage of the
// previous chunk as soon as its store has finished reading shared memory, so
// kCopyStages-1 loads stay in flight; items with a negative index are skipped.
// 16 KiB x 6 stages, 2 CTAs per SM (2 x 96 KiB rings per SM): the fastest of
// the chunk / depth / occupancy sweep in profiles/r01_copy_sweep.jsonl.
#ifndef JENGA_COPY_STAGES
#define JENGA_COPY_STAGES 6
#endif
#ifndef JENGA_COPY_CTAS_PER_SM
#define JENGA_COPY_CTAS_PER_SM 2
#endif
constexpr int kCopyChunkBytes = 16384;
constexpr int kCopyStages = JENGA_COPY_STAGES;
constexpr int kCopyCtasPerSm = JENGA_COPY_CTAS_PER_SM;

struct CopyArgs {
  const uint8_t* src_base;
  uint64_t src_off, src_stride;
  const int64_t* src_idx;
  uint8_t* dst_base;
  uint64_t dst_off, dst_stride;
  const int64_t* dst_idx;
  uint64_t nvec;  // 16-byte units per item
  int n;
  int src_keep, dst_keep;  // 1: L2 evict_last (a dense staging buffer reused next kernel), 0: evict_first
  float scale;     // kScale kernels: every fp32 element is multiplied by it on the way through
  int early;       // 1: the first kCopyStages loads may precede griddepcontrol.wait (common.cuh, column writers)
};

struct CopyChunk {
  const uint8_t* s;
  uint8_t* d;
  uint32_t bytes;
};

template <int kCopyChunk>
__device__ __forceinline__ bool next_copy_chunk(const CopyArgs& a, uint64_t& pos, uint64_t hi, CopyChunk& c) {
  while (pos < hi) {
    const uint64_t b = pos / a.nvec;
    const uint64_t off = pos - b * a.nvec;
    const uint64_t end = min(hi, (b + 1) * a.nvec);
    const int64_t si = a.src_idx ? a.src_idx[b] : static_cast<int64_t>(b);
    const int64_t di = a.dst_idx ? a.dst_idx[b] : static_cast<int64_t>(b);
    if (si < 0 || di < 0) {
      pos = end;
      continue;
    }
    const uint64_t len = min(end - pos, static_cast<uint64_t>(kCopyChunk / 16));
    c.s = a.src_base + a.src_off + si * a.src_stride + off * 16;
    c.d = a.dst_base + a.dst_off + di * a.dst_stride + off * 16;
    c.bytes = static_cast<uint32_t>(len * 16);
    pos += len;
    return true;
  }
  return false;
}

__device__ __forceinline__ void bulk_s2g(void* gmem_dst, const void* smem_src, uint32_t bytes, uint64_t policy) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;\n" ::"l"(gmem_dst),
               "r"(jenga_dev::smem_u32(smem_src)), "r"(bytes), "l"(policy)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}

// Scaling copies (the in-place Mamba state update) run 4 warps per CTA: the
// shared-memory scale pass of a 16 KiB chunk by one warp serialised ~0.5 us per chunk
// behind the bulk copies.
#ifndef JENGA_COPY_SCALE_THREADS
#define JENGA_COPY_SCALE_THREADS 128
#endif
template <bool kScale>
constexpr int copy_threads() { return kScale ? JENGA_COPY_SCALE_THREADS : 32; }

template <int kCopyChunk, int kCopyStages, bool kScale>
__global__ void __launch_bounds__(copy_threads<kScale>()) paged_copy_kernel(const CopyArgs a) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ uint64_t full[kCopyStages];
  // PDL: the next kernel may get resident; our reads/writes wait for the previous one.
  jenga_dev::pdl_launch_dependents();
  if (!kScale && threadIdx.x != 0) return;
  const uint64_t total = a.nvec * static_cast<uint64_t>(a.n);
  uint64_t pos = total * blockIdx.x / gridDim.x;
  const uint64_t hi = total * (blockIdx.x + 1) / gridDim.x;
  if (pos >= hi) return;
  const bool leader = threadIdx.x == 0;
  if (leader) {
    for (int i = 0; i < kCopyStages; ++i) jenga_dev::mbar_init(&full[i], 1);
    jenga_dev::fence_mbar_init();
  }
  if (kScale) __syncthreads();
  if (!a.early) jenga_dev::pdl_wait();
  // arena pages stream through L2 once; a dense staging buffer (Mamba state
  // between gather, the SSM update and scatter) is kept resident
  const uint64_t src_pol = a.src_keep ? jenga_dev::l2_policy_evict_last() : jenga_dev::l2_policy_evict_first();
  const uint64_t dst_pol = a.dst_keep ? jenga_dev::l2_policy_evict_last() : jenga_dev::l2_policy_evict_first();
  CopyChunk ring_c[kCopyStages];
  int issued = 0;
  bool more = true;
  // every lane walks the same chunk sequence (the scale needs all 32 of them);
  // only the leader issues the bulk copies
  auto issue = [&](int j) {
    CopyChunk c;
    if (!next_copy_chunk<kCopyChunk>(a, pos, hi, c)) return false;
    const int st = j % kCopyStages;
    ring_c[st] = c;
    if (leader) {
      jenga_dev::mbar_arrive_expect_tx(&full[st], c.bytes);
      jenga_dev::bulk_g2s_evict_first(ring + st * kCopyChunk, c.s, c.bytes, &full[st], src_pol);
    }
    return true;
  };
  for (; issued < kCopyStages && (more = issue(issued)); ++issued) {
  }
  // early: the ring filled while the previous grid drained; every store and
  // later load follows its completion
  if (a.early) jenga_dev::pdl_wait();
  for (int k = 0; k < issued; ++k) {
    const int st = k % kCopyStages;
    jenga_dev::mbar_wait(&full[st], (k / kCopyStages) & 1);
    if (kScale) {
      float4* f = reinterpret_cast<float4*>(ring + st * kCopyChunk);
      for (uint32_t i = threadIdx.x; i < ring_c[st].bytes / 16; i += blockDim.x) {
        float4 x = f[i];
        x.x *= a.scale;
        x.y *= a.scale;
        x.z *= a.scale;
        x.w *= a.scale;
        f[i] = x;
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic writes -> bulk-copy reads
      __syncthreads();
    }
    if (leader) {
      bulk_s2g(ring_c[st].d, ring + st * kCopyChunk, ring_c[st].bytes, dst_pol);
      if (k >= 1 && more) asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
    }
    if (k >= 1 && more) {
      // chunk k-1's store has read its stage: refill it with chunk k-1+kCopyStages
      if (kScale) __syncthreads();
      if ((more = issue(issued))) ++issued;
    }
  }
  if (leader) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
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
  note_launch(static_cast<cudaStream_t>(stream), kLaunchSerializing);
  return check_launch(scatter ? "token_rows_kernel<scatter>" : "token_rows_kernel<gather>");
}

template <int CHUNK, int STAGES, bool kScale = false>
int launch_copy(const CopyArgs& args, int ctas_per_sm, void* stream, const char* what) {
  constexpr int smem = CHUNK * STAGES;
  auto kern = paged_copy_kernel<CHUNK, STAGES, kScale>;
  static std::atomic<uint64_t> configured{0};
  if (int rc = jenga_decode::configure_smem(kern, smem, configured)) return rc;
  // enough CTAs to fill every SM, none without at least one chunk of work
  const uint64_t chunks = (args.nvec * 16 * static_cast<uint64_t>(args.n) + CHUNK - 1) / CHUNK;
  const int grid = static_cast<int>(
      std::min<uint64_t>(chunks, static_cast<uint64_t>(jenga_dev::num_sms()) * std::max(1, ctas_per_sm)));
  jenga_dev::launch_maybe_pdl(kern, dim3(grid), dim3(copy_threads<kScale>()), smem, static_cast<cudaStream_t>(stream),
                              args);
  return jenga_dev::check_launch(what);
}

int launch_paged_copy(const void* src_base, uint64_t src_off, uint64_t src_stride, const int64_t* src_idx,
                      void* dst_base, uint64_t dst_off, uint64_t dst_stride, const int64_t* dst_idx,
                      uint64_t bytes, int n, void* stream, const char* what, int src_keep, int dst_keep,
                      const float* scale = nullptr, bool column_writer = false) {
  using namespace jenga_dev;
  if (n <= 0 || bytes == 0) return JENGA_OK;
  if (bytes % 16 != 0 || src_off % 16 != 0 || dst_off % 16 != 0 || src_stride % 16 != 0 ||
      dst_stride % 16 != 0 || reinterpret_cast<uintptr_t>(src_base) % 16 || reinterpret_cast<uintptr_t>(dst_base) % 16)
    return set_error(JENGA_ERR_UNSUPPORTED, std::string(what) + ": sizes/offsets must be 16-byte multiples");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // an in-place column writer (src == dst run on one page grid) may load
  // early behind other column writers with disjoint columns
#ifndef JENGA_COPY_EARLY
#define JENGA_COPY_EARLY 1  // 0: profiling variant without the early state loads
#endif
  const bool early = JENGA_COPY_EARLY && column_writer && early_columns_ok(s, dst_stride, dst_off, bytes);
  const CopyArgs args{static_cast<const uint8_t*>(src_base), src_off, src_stride, src_idx,
                      static_cast<uint8_t*>(dst_base), dst_off, dst_stride, dst_idx, bytes / 16, n,
                      src_keep, dst_keep, scale ? *scale : 1.f, early ? 1 : 0};
  const int rc = scale != nullptr && *scale != 1.f
                     ? launch_copy<kCopyChunkBytes, kCopyStages, true>(args, kCopyCtasPerSm, stream, what)
                     : launch_copy<kCopyChunkBytes, kCopyStages>(args, kCopyCtasPerSm, stream, what);
  if (column_writer)
    note_column_writer(s, dst_stride, dst_off, bytes);
  else
    note_launch(s, kLaunchArenaWriterPdl);
  return rc;
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
  const uint64_t per_token = static_cast<uint64_t>(num_kv_heads) * 2 * (row_bytes / 16);
  const int max_tokens = static_cast<int>(std::max<uint64_t>(1, (1ull << 30) / per_token));
  const auto* k8 = static_cast<const uint8_t*>(key);
  const auto* v8 = static_cast<const uint8_t*>(value);
  for (int t0 = 0; t0 < n_tokens; t0 += max_tokens) {  // 32-bit chunk indices per launch
    const int nt = std::min(max_tokens, n_tokens - t0);
    const uint32_t total = static_cast<uint32_t>(nt * per_token);
    const int blocks = static_cast<int>(
        std::min<uint64_t>((total + 256 * kRcUnroll - 1) / (256 * kRcUnroll), static_cast<uint64_t>(num_sms()) * 8));
    launch_maybe_pdl(reshape_and_cache_kernel, dim3(blocks), dim3(256), 0, static_cast<cudaStream_t>(stream),
                     static_cast<uint8_t*>(arena_base), view.start_offset, view.page_stride,
                     static_cast<uint32_t>(row_bytes), tokens_per_page, FastDiv(static_cast<uint32_t>(per_token)),
                     FastDiv(static_cast<uint32_t>(row_bytes / 16)), FastDiv(tokens_per_page),
                     k8 + static_cast<int64_t>(t0) * kv_token_stride * e, v8 + static_cast<int64_t>(t0) * kv_token_stride * e,
                     kv_token_stride * e, slot_mapping + t0, total);
  }
  note_launch(static_cast<cudaStream_t>(stream), kLaunchArenaWriterPdl);
  return check_launch("reshape_and_cache_kernel");
}

JENGA_EXPORT int jenga_mamba_state_gather(const void* arena_base, jenga_layer_view view,
                                          const int64_t* page_globals, int batch, void* dense, void* stream) {
  return launch_paged_copy(arena_base, view.start_offset, view.page_stride, page_globals, dense, 0,
                           view.exec_page_size, nullptr, view.exec_page_size, batch, stream,
                           "mamba_state_gather", 0, 1);
}

JENGA_EXPORT int jenga_mamba_state_scatter(void* arena_base, jenga_layer_view view,
                                           const int64_t* page_globals, int batch, const void* dense,
                                           void* stream) {
  return launch_paged_copy(dense, 0, view.exec_page_size, nullptr, arena_base, view.start_offset,
                           view.page_stride, page_globals, view.exec_page_size, batch, stream,
                           "mamba_state_scatter", 1, 0);
}

JENGA_EXPORT int jenga_mamba_state_update(void* arena_base, jenga_layer_view view, uint32_t num_layers,
                                          const int64_t* page_globals, int batch, float decay, void* stream) {
  if (num_layers == 0 || view.exec_page_size % 16 != 0)
    return jenga_dev::set_error(JENGA_ERR_ARG, "jenga_mamba_state_update: invalid arguments");
  if (static_cast<uint64_t>(num_layers) * view.exec_page_size > view.page_stride)
    return jenga_dev::set_error(JENGA_ERR_CONFIG, "jenga_mamba_state_update: layers beyond the small page");
  // the layers' slices of one page are contiguous: one run per request, read
  // and written back in place through the same addresses
  const uint64_t run = static_cast<uint64_t>(num_layers) * view.exec_page_size;
  return launch_paged_copy(arena_base, view.start_offset, view.page_stride, page_globals, arena_base,
                           view.start_offset, view.page_stride, page_globals, run, batch, stream,
                           "mamba_state_update", 0, 0, &decay, /*column_writer=*/true);
}

JENGA_EXPORT int jenga_page_copy(void* arena_base, uint64_t small_page_bytes, const int64_t* src_globals,
                                 const int64_t* dst_globals, int n_pages, void* stream) {
  return launch_paged_copy(arena_base, 0, small_page_bytes, src_globals, arena_base, 0, small_page_bytes,
                           dst_globals, small_page_bytes, n_pages, stream, "page_copy", 0, 0);
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
