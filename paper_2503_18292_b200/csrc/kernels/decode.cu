// Paged decode attention through Jenga's two-level page table.
//
// Addressing is exactly the reference kernel contract (memory_layout.cpp:41-55,
// PAPER.md:830-838): a layer is {start_offset, page_stride, exec_page_size}
// and a block table of AddressMap global page indices; the bytes of (page,
// layer) start at arena + start_offset + global*page_stride.  Inside the
// slice K/V are [Hkv][K|V][tpp][D] (cache_write.cu), so the tpp K rows and
// then the tpp V rows of one (page, head) are contiguous bulk copies.
//
// Liveness follows LayerPolicy::needs_token (layer_policies.cpp:105-120):
// full / cross attend ordinals 1..n; sliding window attends i + W > n, i.e.
// 0-based [n-W, n).  Leading SWA blocks freed by the allocator
// (simulator.cpp:272-280) carry -1 in the block table and are never touched.
//
// Kernel structure (one CTA per (split, kv-head, request)):
//   warp 4        producer: per 16-token tile, one elected lane issues
//                 cp.async.bulk copies of the K and V rows into an NS-stage
//                 shared-memory ring, completion on an mbarrier (expect_tx).
//   warps 0..3    consumers: tile i is consumed by warp i%4; each warp keeps
//                 its own online-softmax state for its G query heads, so
//                 there is no CTA barrier in the steady state.  q.k partials
//                 are reduced with a transpose-butterfly (31 shuffles for
//                 32 (token, head) dot products), softmax max/sum by warp
//                 shuffles, then P.V accumulates in fp32 registers.
//   epilogue      4 warp states merge through shared memory; splits of one
//                 (request, head) merge in-kernel: the last CTA to finish
//                 (atomic ticket) combines the partials — no second launch.
#include <algorithm>
#include <mutex>

#include "decode_common.cuh"

namespace {

using namespace jenga_decode;

template <int NB>
__device__ __forceinline__ void load_words(const uint8_t* p, uint32_t* w) {
  if constexpr (NB % 16 == 0) {
#pragma unroll
    for (int i = 0; i < NB / 16; ++i) {
      const uint4 v = *reinterpret_cast<const uint4*>(p + 16 * i);
      w[4 * i] = v.x; w[4 * i + 1] = v.y; w[4 * i + 2] = v.z; w[4 * i + 3] = v.w;
    }
  } else if constexpr (NB == 8) {
    const uint2 v = *reinterpret_cast<const uint2*>(p);
    w[0] = v.x; w[1] = v.y;
  } else {
    static_assert(NB == 4, "unsupported per-lane width");
    w[0] = *reinterpret_cast<const uint32_t*>(p);
  }
}

// Sum NV per-lane partials so that each lane ends with one full sum.
// Lane l then holds index k = l (NV == 32) or k = l >> 1 (NV == 16).
template <int NV>
__device__ __forceinline__ float transpose_reduce(float (&v)[NV], int lane) {
  static_assert(NV == 16 || NV == 32, "NV must be 16 or 32");
  int nv = NV;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    if (nv > 1) {
      const int half = nv / 2;
      const bool upper = (lane & off) != 0;
#pragma unroll
      for (int i = 0; i < NV / 2; ++i) {
        if (i < half) {
          const float send = upper ? v[i] : v[i + half];
          const float keep = upper ? v[i + half] : v[i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      }
      nv = half;
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], off);
    }
  }
  return v[0];
}

template <typename T, int D, int G, int NS>
__global__ void __launch_bounds__(kThreads) paged_decode_kernel(const DecodeParams p) {
  static_assert(D % 64 == 0 || D == 64, "head_dim must be 64, 128 or 256");
  constexpr int E = jenga_dev::DT<T>::kBytes;
  constexpr int EPL = D / 32;             // elements per lane per row
  constexpr int LANE_BYTES = EPL * E;
  constexpr int ROW = D * E;
  constexpr int TILE_BYTES = kTile * ROW;
  constexpr int STAGE_BYTES = 2 * TILE_BYTES;
  constexpr int SUB = (32 / G) < kTile ? (32 / G) : kTile;  // tokens per reduction
  constexpr int NSUB = kTile / SUB;
  constexpr int NV = SUB * G;
  constexpr int SHIFT = NV == 16 ? 1 : 0;
  static_assert(NS % kConsumerWarps == 0, "stage ring must be a multiple of the consumer count");
  constexpr int MERGE_BYTES = (kConsumerWarps * G * D + kConsumerWarps * G * 2) * 4;
  constexpr int BAR_OFFSET = (NS * STAGE_BYTES > MERGE_BYTES ? NS * STAGE_BYTES : MERGE_BYTES);


  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + BAR_OFFSET);
  uint64_t* empty = full + NS;
  int* s_flag = reinterpret_cast<int*>(empty + NS);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // Grid order (head, request, split): see decode_tc.cu.
  const int b = grid_request(p);
  const int h = blockIdx.x;
  const int split = grid_split(p);

  const Work wk = assign_work(p, b, split);
  if (split >= wk.nsplit) return;
  const int n = wk.n, lo = wk.lo, nsplit = wk.nsplit, t_begin = wk.t_begin, t_count = wk.t_count;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      jenga_dev::mbar_init(&full[i], 1);
      jenga_dev::mbar_init(&empty[i], 1);
    }
    jenga_dev::fence_mbar_init();
  }
  __syncthreads();

  const int64_t head_chunk = static_cast<int64_t>(p.tpp) * ROW;  // bytes of one (page, head) K chunk
  const int64_t v_offset = head_chunk;  // head-major slice: [Hkv][K|V][tpp][D]
  const uint8_t* layer_base = p.arena + p.start_offset + static_cast<int64_t>(h) * 2 * head_chunk;
  const int32_t* table = p.table + static_cast<int64_t>(b) * p.max_blocks;

  if (warp == kConsumerWarps) {
    // ------------------------------------------------ producer
    if (lane == 0) {
      const uint64_t policy = jenga_dev::l2_policy_evict_first();
      for (int it = 0; it < t_count; ++it) {
        const int st = it % NS;
        if (it >= NS) jenga_dev::mbar_wait(&empty[st], ((it / NS) & 1) ^ 1);
        uint8_t* ks = smem + st * STAGE_BYTES;
        uint8_t* vs = ks + TILE_BYTES;
        const int tok0 = (t_begin + it) * kTile;
        if (p.tpp >= kTile) {
          const int blk = tok0 / p.tpp;
          const int32_t page = table[blk];
          if (page >= 0) {
            const uint8_t* src = layer_base + static_cast<int64_t>(page) * p.page_stride +
                                 static_cast<int64_t>(tok0 % p.tpp) * ROW;
            jenga_dev::mbar_arrive_expect_tx(&full[st], 2 * TILE_BYTES);
            jenga_dev::bulk_g2s_evict_first(ks, src, TILE_BYTES, &full[st], policy);
            jenga_dev::bulk_g2s_evict_first(vs, src + v_offset, TILE_BYTES, &full[st], policy);
          } else {
            jenga_dev::mbar_arrive_expect_tx(&full[st], 0);
          }
        } else {
          const int pieces = kTile / p.tpp;
          const uint32_t piece_bytes = static_cast<uint32_t>(p.tpp * ROW);
          uint32_t total = 0;
          for (int pc = 0; pc < pieces; ++pc) {
            const int tok = tok0 + pc * p.tpp;
            const int blk = tok / p.tpp;
            if (tok < n && blk < p.max_blocks && table[blk] >= 0) total += 2 * piece_bytes;
          }
          jenga_dev::mbar_arrive_expect_tx(&full[st], total);
          for (int pc = 0; pc < pieces; ++pc) {
            const int tok = tok0 + pc * p.tpp;
            const int blk = tok / p.tpp;
            if (tok >= n || blk >= p.max_blocks) continue;
            const int32_t page = table[blk];
            if (page < 0) continue;
            const uint8_t* src = layer_base + static_cast<int64_t>(page) * p.page_stride;
            jenga_dev::bulk_g2s_evict_first(ks + pc * piece_bytes, src, piece_bytes, &full[st], policy);
            jenga_dev::bulk_g2s_evict_first(vs + pc * piece_bytes, src + v_offset, piece_bytes, &full[st],
                                            policy);
          }
        }
      }
    }
    return;
  }

  // -------------------------------------------------- consumers
  float qf[G][EPL];
  {
    const T* qb = static_cast<const T*>(p.q) + (static_cast<int64_t>(b) * p.hq + h * G) * D;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      uint32_t w[LANE_BYTES / 4];
      load_words<LANE_BYTES>(reinterpret_cast<const uint8_t*>(qb + g * D + lane * EPL), w);
      jenga_dev::unpack<T, EPL>(w, qf[g]);
#pragma unroll
      for (int e = 0; e < EPL; ++e) qf[g][e] *= p.qscale;
    }
  }
  float m[G], l[G], acc[G][EPL];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    m[g] = -INFINITY;
    l[g] = 0.f;
#pragma unroll
    for (int e = 0; e < EPL; ++e) acc[g][e] = 0.f;
  }
  const int my_k = lane >> SHIFT;   // reduction index held by this lane
  const int my_g = my_k % G;
  const int my_t = my_k / G;

  for (int it = warp; it < t_count; it += kConsumerWarps) {
    const int st = it % NS;
    jenga_dev::mbar_wait(&full[st], (it / NS) & 1);
    const uint8_t* ks = smem + st * STAGE_BYTES;
    const uint8_t* vs = ks + TILE_BYTES;
    const int tok0 = (t_begin + it) * kTile;
#pragma unroll
    for (int sub = 0; sub < NSUB; ++sub) {
      float part[NV];
#pragma unroll
      for (int tt = 0; tt < SUB; ++tt) {
        uint32_t w[LANE_BYTES / 4];
        float kf[EPL];
        load_words<LANE_BYTES>(ks + (sub * SUB + tt) * ROW + lane * LANE_BYTES, w);
        jenga_dev::unpack<T, EPL>(w, kf);
#pragma unroll
        for (int g = 0; g < G; ++g) {
          float d = 0.f;
#pragma unroll
          for (int e = 0; e < EPL; ++e) d = fmaf(qf[g][e], kf[e], d);
          part[tt * G + g] = d;
        }
      }
      float s = transpose_reduce<NV>(part, lane);
      const int tok = tok0 + sub * SUB + my_t;
      const bool valid = tok >= lo && tok < n;
      if (p.cap_log2 > 0.f) s = p.cap_log2 * tanhf(s * p.inv_cap);
      s = valid ? s : -INFINITY;
      // per-head max over this sub-tile's tokens
      float cm = s;
#pragma unroll
      for (int off = (G << SHIFT); off < 32; off <<= 1) cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, off));
      float mnew[G], alpha[G];
      float m_mine = -INFINITY;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        mnew[g] = fmaxf(m[g], __shfl_sync(0xffffffffu, cm, g << SHIFT));
        alpha[g] = mnew[g] == -INFINITY ? 1.f : jenga_dev::fast_exp2(m[g] - mnew[g]);
        if (my_g == g) m_mine = mnew[g];
      }
      const float pr = (s == -INFINITY) ? 0.f : jenga_dev::fast_exp2(s - m_mine);
      float ps = pr;
#pragma unroll
      for (int off = (G << SHIFT); off < 32; off <<= 1) ps += __shfl_xor_sync(0xffffffffu, ps, off);
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float lsum = __shfl_sync(0xffffffffu, ps, g << SHIFT);
        l[g] = l[g] * alpha[g] + lsum;
        m[g] = mnew[g];
#pragma unroll
        for (int e = 0; e < EPL; ++e) acc[g][e] *= alpha[g];
      }
#pragma unroll
      for (int tt = 0; tt < SUB; ++tt) {
        const int t2 = tok0 + sub * SUB + tt;
        if (t2 < lo || t2 >= n) continue;  // warp-uniform; masked rows may hold stale bytes
        uint32_t w[LANE_BYTES / 4];
        float vf[EPL];
        load_words<LANE_BYTES>(vs + (sub * SUB + tt) * ROW + lane * LANE_BYTES, w);
        jenga_dev::unpack<T, EPL>(w, vf);
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const float pg = __shfl_sync(0xffffffffu, pr, (tt * G + g) << SHIFT);
#pragma unroll
          for (int e = 0; e < EPL; ++e) acc[g][e] = fmaf(pg, vf[e], acc[g][e]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) jenga_dev::mbar_arrive(&empty[st]);
  }

  // -------------------------------------------------- merge the 4 warps
  // All consumers are past their last full-barrier wait and the producer's
  // copies for this CTA have all been consumed, so the ring can be reused.
  consumers_sync();
  float* s_acc = reinterpret_cast<float*>(smem);                  // [4][G][D]
  float* s_ml = s_acc + kConsumerWarps * G * D;                   // [4][G][2]
#pragma unroll
  for (int g = 0; g < G; ++g) {
#pragma unroll
    for (int e = 0; e < EPL; ++e) s_acc[(warp * G + g) * D + lane * EPL + e] = acc[g][e];
    if (lane == 0) {
      s_ml[(warp * G + g) * 2] = m[g];
      s_ml[(warp * G + g) * 2 + 1] = l[g];
    }
  }
  merge_epilogue<T, G, D>(p, s_acc, s_ml, s_flag, nsplit, split, b, h);
}



// The workspace is sized for the finest split the launcher may pick.
constexpr int kMinTilesPerSplit = 8;

int splits_for(int max_blocks, int tpp, int tiles_per_split) {
  const int64_t max_tokens = static_cast<int64_t>(max_blocks) * tpp;
  const int64_t max_tiles = (max_tokens + kTile - 1) / kTile + 1;
  return static_cast<int>((max_tiles + tiles_per_split - 1) / tiles_per_split);
}

// Tiles per CTA, sized by bytes: a CTA pays a fixed prologue / merge cost, so
// it should stream ~512-768 KiB of one head's K+V.  head_dim 256: 32 tiles
// (512 KiB); head_dim <= 128: 96 * 128/D tiles (768 KiB) — measured +7% (Llama
// vision) and +10% (Jamba attention) over 32 tiles at D=128
// (profiles/r01_sweeps.md).
int tiles_per_split(int head_dim) {
  return head_dim >= 256 ? kTilesPerSplit : 96 * 128 / std::max(head_dim, 16);
}

// Wave-aware split count for the tensor-core kernel (three CTAs per SM).  With
// requests of similar length the (KV head, request, split) CTAs finish in
// ceil(CTAs / slots) rounds, so a split count that leaves the last round
// mostly empty wastes up to a round; the launcher picks the split count s
// minimising rounds(s) x (tiles per CTA(s) + per-CTA overhead), never below
// kMinTilesPerSplit tiles per CTA (the workspace granularity).  The overhead
// (prologue, ring fill, split merge) is JENGA_SPLIT_OVERHEAD_TILES tiles of
// streaming time; < 0 keeps the byte-sized splits of tiles_per_split().
#ifndef JENGA_SPLIT_OVERHEAD_TILES
#define JENGA_SPLIT_OVERHEAD_TILES 32
#endif
int wave_tiles_per_split(int64_t pairs, int64_t max_tiles, int64_t slots, int fallback) {
  if (JENGA_SPLIT_OVERHEAD_TILES < 0 || pairs <= 0 || max_tiles <= 0 || slots <= 0) return fallback;
  int64_t best_s = 1;
  double best = 0.0;
  const int64_t s_max = std::max<int64_t>(1, max_tiles / kMinTilesPerSplit);
  for (int64_t sp = 1; sp <= s_max; ++sp) {
    const int64_t per = (max_tiles + sp - 1) / sp;
    const int64_t rounds = (pairs * sp + slots - 1) / slots;
    const double cost = static_cast<double>(rounds) * static_cast<double>(per + JENGA_SPLIT_OVERHEAD_TILES);
    if (sp == 1 || cost < best * 0.999) {
      best = cost;
      best_s = sp;
    }
  }
  return static_cast<int>(std::max<int64_t>(kMinTilesPerSplit, (max_tiles + best_s - 1) / best_s));
}

template <typename T, int D, int G>
int launch_typed(const DecodeParams& prm, int batch, cudaStream_t stream) {
  constexpr int NS = 4;
  constexpr int STAGE = 2 * kTile * D * sizeof(T);
  const int ring = NS * STAGE;
  const int merge = (kConsumerWarps * G * D + kConsumerWarps * G * 2) * 4;
  const int smem = std::max(ring, merge) + 2 * NS * 8 + 16;
  auto kern = paged_decode_kernel<T, D, G, NS>;
  static std::atomic<uint64_t> configured{0};
  if (int rc = configure_smem(kern, smem, configured)) return rc;
  const dim3 grid = decode_grid(prm, batch);
  kern<<<grid, kThreads, smem, stream>>>(prm);
  jenga_dev::note_launch(stream, jenga_dev::kLaunchSerializing);
  return jenga_dev::check_launch("paged_decode_kernel");
}

template <typename T, int D>
int dispatch_g(int G, const DecodeParams& prm, int batch, cudaStream_t s) {
  switch (G) {
    case 1: return launch_typed<T, D, 1>(prm, batch, s);
    case 2: return launch_typed<T, D, 2>(prm, batch, s);
    case 4: return launch_typed<T, D, 4>(prm, batch, s);
    case 8: return launch_typed<T, D, 8>(prm, batch, s);
  }
  return jenga_dev::set_error(JENGA_ERR_UNSUPPORTED, "paged_decode: query heads per kv head must be 1, 2, 4 or 8");
}

template <typename T>
int dispatch_d(int D, int G, const DecodeParams& prm, int batch, cudaStream_t s) {
  switch (D) {
    case 64: return dispatch_g<T, 64>(G, prm, batch, s);
    case 128: return dispatch_g<T, 128>(G, prm, batch, s);
    case 256: return dispatch_g<T, 256>(G, prm, batch, s);
  }
  return jenga_dev::set_error(JENGA_ERR_UNSUPPORTED, "paged_decode: head_dim must be 64, 128 or 256");
}

}  // namespace

JENGA_EXPORT size_t jenga_paged_decode_workspace_size(int batch, int num_q_heads, int num_kv_heads, int head_dim,
                                                      int max_blocks, uint32_t tokens_per_page) {
  if (batch <= 0 || num_kv_heads <= 0 || num_q_heads <= 0 || tokens_per_page == 0) return 0;
  const int64_t ms = splits_for(max_blocks, static_cast<int>(tokens_per_page), kMinTilesPerSplit);
  const int64_t bh = static_cast<int64_t>(batch) * num_kv_heads;
  const int64_t G = num_q_heads / num_kv_heads;
  const int64_t counters = ((bh * 4 + 16 + 255) / 256) * 256;
  return static_cast<size_t>(counters + bh * ms * G * head_dim * 4 + bh * ms * G * 2 * 4);
}

namespace {
int paged_decode_impl(void* arena_base, jenga_layer_view view, int kind, int dtype, uint64_t window, const void* q,
                      void* out, const int32_t* block_table, const int32_t* seq_lens, int batch, int max_blocks,
                      int num_q_heads, int num_kv_heads, int head_dim, uint32_t tokens_per_page, float scale,
                      float softcap, void* workspace, size_t workspace_bytes, const void* k_new, const void* v_new,
                      const int64_t* new_slots, void* stream) {
  using namespace jenga_dev;
  if (batch < 0 || num_kv_heads <= 0 || num_q_heads <= 0 || num_q_heads % num_kv_heads != 0 ||
      tokens_per_page == 0 || max_blocks <= 0 || !arena_base || !q || !out || !block_table || !seq_lens)
    return set_error(JENGA_ERR_ARG, "jenga_paged_decode: invalid arguments");
  if (kind != JENGA_KIND_FULL && kind != JENGA_KIND_SLIDING_WINDOW && kind != JENGA_KIND_CROSS_ATTENTION)
    return set_error(JENGA_ERR_UNSUPPORTED, "jenga_paged_decode: kind must be full, sliding_window or cross");
  if (kind == JENGA_KIND_SLIDING_WINDOW && window == 0)
    return set_error(JENGA_ERR_CONFIG, "jenga_paged_decode: sliding window needs window >= 1");
  const int e = dtype_bytes(dtype);
  if (e == 0) return set_error(JENGA_ERR_UNSUPPORTED, "jenga_paged_decode: unsupported dtype");
  const uint64_t expect = 2ull * num_kv_heads * tokens_per_page * head_dim * e;
  if (view.exec_page_size != expect)
    return set_error(JENGA_ERR_CONFIG, "jenga_paged_decode: exec_page_size != 2*Hkv*tpp*D*dtype");
  if (view.start_offset % 16 || view.page_stride % 16)
    return set_error(JENGA_ERR_UNSUPPORTED, "jenga_paged_decode: layer view must be 16-byte aligned");
  const int tpp = static_cast<int>(tokens_per_page);
  if (!(tpp % kTile == 0 || kTile % tpp == 0))
    return set_error(JENGA_ERR_UNSUPPORTED, "jenga_paged_decode: tokens_per_page must divide 16 or be a multiple of 16");
  const size_t need = jenga_paged_decode_workspace_size(batch, num_q_heads, num_kv_heads, head_dim, max_blocks,
                                                        tokens_per_page);
  if (workspace == nullptr || workspace_bytes < need)
    return set_error(JENGA_ERR_ARG, "jenga_paged_decode: workspace too small");
  if (batch == 0) return JENGA_OK;

  DecodeParams prm{};
  prm.arena = static_cast<const uint8_t*>(arena_base);
  prm.start_offset = view.start_offset;
  prm.page_stride = view.page_stride;
  prm.q = q;
  prm.out = out;
  prm.table = block_table;
  prm.seq_lens = seq_lens;
  prm.kind = kind;
  prm.window = static_cast<int64_t>(window);
  prm.max_blocks = max_blocks;
  prm.hq = num_q_heads;
  prm.hkv = num_kv_heads;
  prm.tpp = tpp;
  prm.tiles_per_split = tiles_per_split(head_dim);
  if ((dtype == JENGA_BF16 || dtype == JENGA_F16) && tpp % kTile == 0) {
    // the tiles a request at full table width can need in this launch
    int64_t max_tiles = (static_cast<int64_t>(max_blocks) * tpp + kTile - 1) / kTile;
    if (kind == JENGA_KIND_SLIDING_WINDOW)
      max_tiles = std::min<int64_t>(max_tiles, (static_cast<int64_t>(window) + kTile - 1) / kTile + 1);
    prm.tiles_per_split = wave_tiles_per_split(static_cast<int64_t>(batch) * num_kv_heads, max_tiles,
                                               static_cast<int64_t>(num_sms()) * decode_ctas_per_sm(head_dim), prm.tiles_per_split);
  }
  prm.batch = batch;
  prm.max_splits = splits_for(max_blocks, tpp, prm.tiles_per_split);
  if (kind == JENGA_KIND_SLIDING_WINDOW) {
    // live ordinals (n-W, n] span at most ceil(W/16)+1 tiles: no grid slices for
    // splits a window can never reach (the table is still indexed by absolute block)
    const int64_t win_tiles = (static_cast<int64_t>(window) + kTile - 1) / kTile + 1;
    const int64_t ws = (win_tiles + prm.tiles_per_split - 1) / prm.tiles_per_split;
    if (ws < prm.max_splits) prm.max_splits = static_cast<int>(ws);
  }
  if (softcap > 0.f) {
    prm.qscale = scale;
    prm.cap_log2 = softcap * kLog2e;
    prm.inv_cap = 1.f / softcap;
  } else {
    prm.qscale = scale * kLog2e;
    prm.cap_log2 = 0.f;
    prm.inv_cap = 0.f;
  }
  const int64_t bh = static_cast<int64_t>(batch) * num_kv_heads;
  const int64_t G = num_q_heads / num_kv_heads;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  const int64_t counters = ((bh * 4 + 16 + 255) / 256) * 256;
  prm.counters = reinterpret_cast<int*>(ws);
  prm.part_acc = reinterpret_cast<float*>(ws + counters);
  prm.part_ml = prm.part_acc + bh * prm.max_splits * G * head_dim;

  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if ((dtype == JENGA_BF16 || dtype == JENGA_F16) && tpp % kTile == 0) {
    prm.k_new = k_new;  // the tensor-core kernel fuses the append
    prm.v_new = v_new;
    prm.new_slots = new_slots;
    prm.early_kv = jenga_dev::early_kv_ok(s) ? 1 : 0;
    const int rc = launch_decode_tc(prm, dtype, head_dim, static_cast<int>(G), batch, s);
    if (rc != JENGA_ERR_UNSUPPORTED) return rc;
    prm.k_new = prm.v_new = nullptr;
    prm.new_slots = nullptr;
  }
  if (k_new != nullptr) {  // CUDA-core kernel: write the new token first, then attend
    const int rc = jenga_reshape_and_cache(arena_base, view, dtype, num_kv_heads, head_dim, tokens_per_page, k_new,
                                           v_new, static_cast<int64_t>(num_kv_heads) * head_dim, new_slots, batch,
                                           stream);
    if (rc != JENGA_OK) return rc;
  }
  switch (dtype) {
    case JENGA_F32: return dispatch_d<float>(head_dim, static_cast<int>(G), prm, batch, s);
    case JENGA_BF16: return dispatch_d<__nv_bfloat16>(head_dim, static_cast<int>(G), prm, batch, s);
    case JENGA_F16: return dispatch_d<__half>(head_dim, static_cast<int>(G), prm, batch, s);
  }
  return set_error(JENGA_ERR_UNSUPPORTED, "jenga_paged_decode: unsupported dtype");
}
}  // namespace

JENGA_EXPORT int jenga_paged_decode(void* arena_base, jenga_layer_view view, int kind, int dtype, uint64_t window,
                                    const void* q, void* out, const int32_t* block_table, const int32_t* seq_lens,
                                    int batch, int max_blocks, int num_q_heads, int num_kv_heads, int head_dim,
                                    uint32_t tokens_per_page, float scale, float softcap, void* workspace,
                                    size_t workspace_bytes, void* stream) {
  return paged_decode_impl(arena_base, view, kind, dtype, window, q, out, block_table, seq_lens, batch, max_blocks,
                           num_q_heads, num_kv_heads, head_dim, tokens_per_page, scale, softcap, workspace,
                           workspace_bytes, nullptr, nullptr, nullptr, stream);
}

JENGA_EXPORT int jenga_paged_decode_append(void* arena_base, jenga_layer_view view, int kind, int dtype,
                                           uint64_t window, const void* q, const void* key, const void* value,
                                           const int64_t* slot_mapping, void* out, const int32_t* block_table,
                                           const int32_t* seq_lens, int batch, int max_blocks, int num_q_heads,
                                           int num_kv_heads, int head_dim, uint32_t tokens_per_page, float scale,
                                           float softcap, void* workspace, size_t workspace_bytes, void* stream) {
  if (kind == JENGA_KIND_CROSS_ATTENTION)
    return jenga_dev::set_error(JENGA_ERR_UNSUPPORTED,
                                "jenga_paged_decode_append: cross-attention KV is static during decode");
  if (batch > 0 && (key == nullptr || value == nullptr || slot_mapping == nullptr))
    return jenga_dev::set_error(JENGA_ERR_ARG, "jenga_paged_decode_append: key, value and slot_mapping required");
  return paged_decode_impl(arena_base, view, kind, dtype, window, q, out, block_table, seq_lens, batch, max_blocks,
                           num_q_heads, num_kv_heads, head_dim, tokens_per_page, scale, softcap, workspace,
                           workspace_bytes, key, value, slot_mapping, stream);
}
