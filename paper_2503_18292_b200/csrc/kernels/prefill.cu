// Chunked-prefill paged attention (the reference's
// prefill_some stores a chunk of positions per step, simulator.cpp:504-547).
//
// Request b contributes C_b query tokens — its newest ordinals, 0-based
// positions n_b - C_b .. n_b - 1 — whose K/V were already scattered into the
// arena by reshape_and_cache.  Query position i attends key j iff j <= i
// (causal), additionally j + W > i for sliding windows (needs_token at
// length i + 1, layer_policies.cpp:105-120); cross attention attends all n_b
// image keys.
//
// One CTA = (query block of 128 rows, KV head, request); rows are
// (token, query head) pairs r = t*G + g, so a block holds 128/G tokens.
//   producer warp   one TMA 3-D box load of the Q block ([T][Hq][D] viewed
//                   with box {64, G, 128/G}; row r lands on swizzle line r),
//                   then streams 16-token K/V tiles through a shared ring
//                   (same 2-D arena tensor map as decode).
//   8 MMA warps     16 rows each, FlashAttention-2 style on the tensor cores:
//                   S = Q K^T (m16n8k16, K^T via ldmatrix), P kept in
//                   registers as the A operand of O += P V (V via
//                   ldmatrix.trans), fp32 online softmax per row.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <map>
#include <mutex>

#include "decode_common.cuh"

namespace jenga_dev {
bool arena_extent(const void* base, uint64_t* bytes);
}

namespace jenga_decode {
int launch_prefill_tc5(const void* arena, uint64_t start_offset, uint64_t page_stride, void* out, const int32_t* cu_q,
                       const int32_t* table, const int32_t* seq_lens, int kind, int64_t window, int max_blocks,
                       int hq, int hkv, int tpp, int q_blocks_128, float qscale, float cap_log2, float inv_cap,
                       int dtype, int head_dim, int batch, int total_tokens, const void* q, cudaStream_t s);
}

namespace {

using namespace jenga_decode;

constexpr int kRows = 128;             // query rows per CTA
constexpr int kMmaWarps = kRows / 16;  // 8
constexpr int kPThreads = (kMmaWarps + 1) * 32;
constexpr int kBoxCols = 64;
constexpr int kKvBox = kTile * 128;    // 64 x 16 box of K or V

struct PrefillParams {
  const uint8_t* arena;
  uint64_t start_offset, page_stride;
  void* out;
  const int32_t* cu_q;
  const int32_t* table;
  const int32_t* seq_lens;
  int kind;
  int64_t window;
  int max_blocks, hq, hkv, tpp, q_blocks;
  float qscale, cap_log2, inv_cap;
};

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_trans(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}

template <typename T>
__device__ __forceinline__ void mma16816(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%0, %1, %2, %3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  } else {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%0, %1, %2, %3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
}

template <typename T>
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
  } else {
    __half2 v = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
  }
}

__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, int32_t c0, int32_t c1, int32_t c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];\n" ::"r"(jenga_dev::smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(jenga_dev::smem_u32(bar))
      : "memory");
}

template <typename T, int D, int G, int NS>
__global__ void __launch_bounds__(kPThreads, 1)
    paged_prefill_kernel(const PrefillParams p, const __grid_constant__ CUtensorMap kv_map,
                         const __grid_constant__ CUtensorMap q_map) {
  constexpr int NBOX = D / kBoxCols;
  constexpr int QB = kRows / G;                 // tokens per query block
  constexpr int Q_BOX = kRows * 128;            // one 64-col box of the Q block
  constexpr int Q_BYTES = NBOX * Q_BOX;
  constexpr int TILE = NBOX * kKvBox;           // K (or V) of 16 tokens, one head
  constexpr int STAGE = 2 * TILE;
  constexpr int KS = D / 16;                    // k-steps over head_dim
  constexpr int NT = D / 8;                     // n-tiles of O

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (jenga_dev::smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* qs = smem;
  uint8_t* ring = smem + Q_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + NS * STAGE);
  uint64_t* empty = full + NS;
  uint64_t* q_full = empty + NS;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int c_len = p.cu_q[b + 1] - p.cu_q[b];
  const int t0 = qb * QB;  // first token of this block within the request's chunk
  if (t0 >= c_len) return;
  const int n = p.seq_lens[b];
  const int pos0 = n - c_len + t0;                       // position of token t0
  const int pos1 = n - c_len + min(t0 + QB, c_len) - 1;  // last position in the block
  int key_lo = 0, key_hi = pos1;
  if (p.kind == JENGA_KIND_CROSS_ATTENTION) key_hi = n - 1;
  if (p.kind == JENGA_KIND_SLIDING_WINDOW && pos0 + 1 > p.window) key_lo = static_cast<int>(pos0 + 1 - p.window);
  const int tile_lo = key_lo / kTile, tile_hi = key_hi / kTile;
  const int ntiles = key_hi >= key_lo ? tile_hi - tile_lo + 1 : 0;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      jenga_dev::mbar_init(&full[i], 1);
      jenga_dev::mbar_init(&empty[i], kMmaWarps);
    }
    jenga_dev::mbar_init(q_full, 1);
    jenga_dev::fence_mbar_init();
  }
  __syncthreads();
  const int32_t* table = p.table + static_cast<int64_t>(b) * p.max_blocks;

  if (warp == kMmaWarps) {
    if (lane == 0) {  // producer
      jenga_dev::prefetch_tmap(&kv_map);
      jenga_dev::prefetch_tmap(&q_map);
      jenga_dev::mbar_arrive_expect_tx(q_full, Q_BYTES);
#pragma unroll
      for (int bx = 0; bx < NBOX; ++bx)
        tma_load_3d(qs + bx * Q_BOX, &q_map, bx * kBoxCols, h * G, p.cu_q[b] + t0, q_full);
      const uint64_t policy = jenga_dev::l2_policy_evict_first();
      const int64_t row_bytes = D * 2;
      const int64_t base_row = static_cast<int64_t>(p.start_offset) / row_bytes + static_cast<int64_t>(h) * 2 * p.tpp;
      const int64_t page_rows = static_cast<int64_t>(p.page_stride) / row_bytes;
      const int v_rows = p.tpp;  // head-major slice
      for (int it = 0; it < ntiles; ++it) {
        const int st = it % NS;
        if (it >= NS) jenga_dev::mbar_wait(&empty[st], ((it / NS) & 1) ^ 1);
        const int tok = (tile_lo + it) * kTile;
        const int32_t row =
            static_cast<int32_t>(base_row + static_cast<int64_t>(table[tok / p.tpp]) * page_rows + tok % p.tpp);
        uint8_t* ks = ring + st * STAGE;
        jenga_dev::mbar_arrive_expect_tx(&full[st], STAGE);
#pragma unroll
        for (int bx = 0; bx < NBOX; ++bx) {
          jenga_dev::tma_load_2d(ks + bx * kKvBox, &kv_map, bx * kBoxCols, row, &full[st], policy);
          jenga_dev::tma_load_2d(ks + TILE + bx * kKvBox, &kv_map, bx * kBoxCols, row + v_rows, &full[st], policy);
        }
      }
    }
    return;
  }

  // ------------------------------------------------ MMA warps (16 rows each)
  const int g4 = lane >> 2, c4 = lane & 3, x7 = lane & 7;
  const int r_lo = warp * 16 + g4, r_hi = r_lo + 8;  // rows owned by this lane
  const int tok_lo = t0 + r_lo / G, tok_hi = t0 + r_hi / G;
  const int ipos_lo = n - c_len + tok_lo, ipos_hi = n - c_len + tok_hi;  // query positions
  const bool row_ok_lo = tok_lo < c_len, row_ok_hi = tok_hi < c_len;
  float o[NT][4];
#pragma unroll
  for (int j = 0; j < NT; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float m_lo = -INFINITY, m_hi = -INFINITY, l_lo = 0.f, l_hi = 0.f;

  // Q fragment addresses (A operand, rows warp*16.., ldmatrix x4 order)
  const int qa_row = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
  const int qa_half = lane >> 4;
  // K^T fragment addresses (B operand: rows = tokens, cols = D)
  const int kb_tok = (lane & 7) + (lane >> 4) * 8;
  const int kb_half = (lane >> 3) & 1;
  // V fragment addresses (B operand via .trans: rows = tokens)
  const int vb_tok = (lane & 7) + ((lane >> 3) & 1) * 8;
  const int vb_chunk = lane >> 4;
  const uint32_t qs_u = jenga_dev::smem_u32(qs);

  jenga_dev::mbar_wait(q_full, 0);
  for (int it = 0; it < ntiles; ++it) {
    const int st = it % NS;
    jenga_dev::mbar_wait(&full[st], (it / NS) & 1);
    const uint32_t ks_u = jenga_dev::smem_u32(ring + st * STAGE);
    const uint32_t vs_u = ks_u + TILE;
    const int ktok0 = (tile_lo + it) * kTile;
    // ---- S = Q K^T : 16 rows x 16 keys
    float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      uint32_t a[4], bk[4];
      const int qc = 2 * k + qa_half;
      ldsm_x4(a, qs_u + (qc >> 3) * Q_BOX + qa_row * 128 + (((qc & 7) ^ x7) << 4));
      const int kc = 2 * k + kb_half;
      ldsm_x4(bk, ks_u + (kc >> 3) * kKvBox + kb_tok * 128 + (((kc & 7) ^ x7) << 4));
      mma16816<T>(s0, a[0], a[1], a[2], a[3], bk[0], bk[1]);
      mma16816<T>(s1, a[0], a[1], a[2], a[3], bk[2], bk[3]);
    }
    // ---- mask + scale: key j = ktok0 + {2c, 2c+1} (s0) / + 8 (s1)
    float sv[8] = {s0[0], s0[1], s1[0], s1[1], s0[2], s0[3], s1[2], s1[3]};  // [lo row: 4][hi row: 4]
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int j = ktok0 + (e & 2 ? 8 : 0) + 2 * c4 + (e & 1);
      const int ipos = e < 4 ? ipos_lo : ipos_hi;
      bool ok = j >= key_lo && j <= (p.kind == JENGA_KIND_CROSS_ATTENTION ? n - 1 : ipos);
      if (p.kind == JENGA_KIND_SLIDING_WINDOW) ok = ok && j + p.window > ipos;
      float x = sv[e] * p.qscale;
      if (p.cap_log2 > 0.f) x = p.cap_log2 * tanhf(x * p.inv_cap);
      sv[e] = ok ? x : -INFINITY;
    }
    float t_lo = fmaxf(fmaxf(sv[0], sv[1]), fmaxf(sv[2], sv[3]));
    float t_hi = fmaxf(fmaxf(sv[4], sv[5]), fmaxf(sv[6], sv[7]));
#pragma unroll
    for (int off = 1; off < 4; off <<= 1) {
      t_lo = fmaxf(t_lo, __shfl_xor_sync(0xffffffffu, t_lo, off));
      t_hi = fmaxf(t_hi, __shfl_xor_sync(0xffffffffu, t_hi, off));
    }
    const float n_lo = fmaxf(m_lo, t_lo), n_hi = fmaxf(m_hi, t_hi);
    const float a_lo = n_lo == -INFINITY ? 1.f : jenga_dev::fast_exp2(m_lo - n_lo);
    const float a_hi = n_hi == -INFINITY ? 1.f : jenga_dev::fast_exp2(m_hi - n_hi);
    m_lo = n_lo;
    m_hi = n_hi;
    float pv[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float mm = e < 4 ? n_lo : n_hi;
      pv[e] = sv[e] == -INFINITY ? 0.f : jenga_dev::fast_exp2(sv[e] - mm);
    }
    l_lo = l_lo * a_lo + pv[0] + pv[1] + pv[2] + pv[3];
    l_hi = l_hi * a_hi + pv[4] + pv[5] + pv[6] + pv[7];
    if (__any_sync(0xffffffffu, a_lo != 1.f || a_hi != 1.f)) {
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        o[j][0] *= a_lo;
        o[j][1] *= a_lo;
        o[j][2] *= a_hi;
        o[j][3] *= a_hi;
      }
    }
    // P as the A operand (k = 16 keys): FA2 register re-use of the S layout
    const uint32_t pa0 = pack2<T>(pv[0], pv[1]);  // row lo, keys 2c..
    const uint32_t pa1 = pack2<T>(pv[4], pv[5]);  // row hi, keys 2c..
    const uint32_t pa2 = pack2<T>(pv[2], pv[3]);  // row lo, keys 8+2c..
    const uint32_t pa3 = pack2<T>(pv[6], pv[7]);  // row hi, keys 8+2c..
    // masked keys of a boundary tile may hold non-finite bytes: 0 * NaN = NaN
    // inside the MMA, so warp 0 zeroes those V rows once per tile (all warps
    // read them only after the named barrier below).
    const bool boundary = ktok0 < key_lo || ktok0 + kTile - 1 > (p.kind == JENGA_KIND_CROSS_ATTENTION ? n - 1 : pos1);
    if (boundary) {
      asm volatile("bar.sync 2, %0;\n" ::"n"(kMmaWarps * 32) : "memory");
      if (warp == 0) {
        const int kmax = p.kind == JENGA_KIND_CROSS_ATTENTION ? n - 1 : pos1;
        for (int r = 0; r < kTile; ++r) {
          const int j = ktok0 + r;
          if (j >= key_lo && j <= kmax) continue;
          for (int c = lane; c < NBOX * 8; c += 32)
            *reinterpret_cast<uint4*>(ring + st * STAGE + TILE + (c >> 3) * kKvBox + r * 128 + ((c & 7) << 4)) =
                make_uint4(0, 0, 0, 0);
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      }
      asm volatile("bar.sync 2, %0;\n" ::"n"(kMmaWarps * 32) : "memory");
    }
    // ---- O += P V
#pragma unroll
    for (int j = 0; j < NT; j += 2) {
      uint32_t bv[4];
      const int vc = j + vb_chunk;
      ldsm_x4_trans(bv, vs_u + (vc >> 3) * kKvBox + vb_tok * 128 + (((vc & 7) ^ x7) << 4));
      mma16816<T>(o[j], pa0, pa1, pa2, pa3, bv[0], bv[1]);
      mma16816<T>(o[j + 1], pa0, pa1, pa2, pa3, bv[2], bv[3]);
    }
    __syncwarp();
    if (lane == 0) jenga_dev::mbar_arrive(&empty[st]);
  }
  // ---- normalise and store rows (token, head) of this lane
#pragma unroll
  for (int off = 1; off < 4; off <<= 1) {
    l_lo += __shfl_xor_sync(0xffffffffu, l_lo, off);
    l_hi += __shfl_xor_sync(0xffffffffu, l_hi, off);
  }
  const float inv_lo = l_lo > 0.f ? 1.f / l_lo : 0.f, inv_hi = l_hi > 0.f ? 1.f / l_hi : 0.f;
  T* out = static_cast<T*>(p.out);
  const int64_t tq_lo = p.cu_q[b] + tok_lo, tq_hi = p.cu_q[b] + tok_hi;
  const int qh_lo = h * G + r_lo % G, qh_hi = h * G + r_hi % G;
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const int d = 8 * j + 2 * c4;
    if (row_ok_lo)
      *reinterpret_cast<uint32_t*>(out + (tq_lo * p.hq + qh_lo) * D + d) = pack2<T>(o[j][0] * inv_lo, o[j][1] * inv_lo);
    if (row_ok_hi)
      *reinterpret_cast<uint32_t*>(out + (tq_hi * p.hq + qh_hi) * D + d) = pack2<T>(o[j][2] * inv_hi, o[j][3] * inv_hi);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

template <typename T, int D, int G>
int launch_prefill(const PrefillParams& prm, int dtype, int batch, int total_tokens, const void* q, cudaStream_t s) {
  constexpr int NS = 4;
  constexpr int NBOX = D / kBoxCols;
  constexpr int QB = kRows / G;
  const int smem = NBOX * kRows * 128 + NS * 2 * NBOX * kKvBox + (2 * NS + 1) * 8 + 1024;
  auto fn = encode_fn();
  if (fn == nullptr) return jenga_dev::set_error(JENGA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  uint64_t bytes = 0;
  if (!jenga_dev::arena_extent(prm.arena, &bytes))
    return jenga_dev::set_error(JENGA_ERR_ARG, "jenga_paged_prefill: arena_base must come from jenga_arena_create");
  const CUtensorMapDataType dt =
      dtype == JENGA_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUtensorMap kv_map, q_map;
  {
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(D), bytes / (D * 2)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(D) * 2};
    cuuint32_t box[2] = {kBoxCols, kTile};
    cuuint32_t es[2] = {1, 1};
    if (fn(&kv_map, dt, 2, const_cast<uint8_t*>(prm.arena), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS)
      return jenga_dev::set_error(JENGA_ERR_CUDA, "prefill: KV tensor map encode failed");
  }
  {
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(prm.hq),
                          static_cast<cuuint64_t>(total_tokens)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(D) * 2, static_cast<cuuint64_t>(prm.hq) * D * 2};
    cuuint32_t box[3] = {kBoxCols, static_cast<cuuint32_t>(G), static_cast<cuuint32_t>(QB)};
    cuuint32_t es[3] = {1, 1, 1};
    if (fn(&q_map, dt, 3, const_cast<void*>(q), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS)
      return jenga_dev::set_error(JENGA_ERR_CUDA, "prefill: Q tensor map encode failed");
  }
  auto kern = paged_prefill_kernel<T, D, G, NS>;
  static std::atomic<uint64_t> configured{0};
  if (int rc = configure_smem(kern, smem, configured)) return rc;
  dim3 grid(prm.q_blocks, prm.hkv, batch);
  kern<<<grid, kPThreads, smem, s>>>(prm, kv_map, q_map);
  return jenga_dev::check_launch("paged_prefill_kernel");
}

template <typename T, int D>
int dispatch_g(int G, const PrefillParams& prm, int dtype, int batch, int total, const void* q, cudaStream_t s) {
  switch (G) {
    case 1: return launch_prefill<T, D, 1>(prm, dtype, batch, total, q, s);
    case 2: return launch_prefill<T, D, 2>(prm, dtype, batch, total, q, s);
    case 4: return launch_prefill<T, D, 4>(prm, dtype, batch, total, q, s);
    case 8: return launch_prefill<T, D, 8>(prm, dtype, batch, total, q, s);
  }
  return jenga_dev::set_error(JENGA_ERR_UNSUPPORTED, "paged_prefill: query heads per kv head must be 1, 2, 4 or 8");
}

template <typename T>
int dispatch_d(int D, int G, const PrefillParams& prm, int dtype, int batch, int total, const void* q,
               cudaStream_t s) {
  switch (D) {
    case 64: return dispatch_g<T, 64>(G, prm, dtype, batch, total, q, s);
    case 128: return dispatch_g<T, 128>(G, prm, dtype, batch, total, q, s);
    case 256: return dispatch_g<T, 256>(G, prm, dtype, batch, total, q, s);
  }
  return jenga_dev::set_error(JENGA_ERR_UNSUPPORTED, "paged_prefill: head_dim must be 64, 128 or 256");
}

}  // namespace

JENGA_EXPORT int jenga_paged_prefill(void* arena_base, jenga_layer_view view, int kind, int dtype, uint64_t window,
                                     const void* q, void* out, const int32_t* cu_q, int total_tokens,
                                     int max_chunk, const int32_t* block_table, const int32_t* seq_lens, int batch,
                                     int max_blocks, int num_q_heads, int num_kv_heads, int head_dim,
                                     uint32_t tokens_per_page, float scale, float softcap, void* stream) {
  using namespace jenga_dev;
  if (batch < 0 || num_kv_heads <= 0 || num_q_heads <= 0 || num_q_heads % num_kv_heads != 0 ||
      tokens_per_page == 0 || max_blocks <= 0 || total_tokens < 0 || max_chunk < 0 || !arena_base || !q || !out ||
      !cu_q || !block_table || !seq_lens)
    return set_error(JENGA_ERR_ARG, "jenga_paged_prefill: invalid arguments");
  if (kind != JENGA_KIND_FULL && kind != JENGA_KIND_SLIDING_WINDOW && kind != JENGA_KIND_CROSS_ATTENTION)
    return set_error(JENGA_ERR_UNSUPPORTED, "jenga_paged_prefill: kind must be full, sliding_window or cross");
  if (kind == JENGA_KIND_SLIDING_WINDOW && window == 0)
    return set_error(JENGA_ERR_CONFIG, "jenga_paged_prefill: sliding window needs window >= 1");
  if (dtype != JENGA_BF16 && dtype != JENGA_F16)
    return set_error(JENGA_ERR_UNSUPPORTED, "jenga_paged_prefill: bf16 / fp16 KV only (tensor-core path)");
  if (view.exec_page_size != 2ull * num_kv_heads * tokens_per_page * head_dim * 2)
    return set_error(JENGA_ERR_CONFIG, "jenga_paged_prefill: exec_page_size != 2*Hkv*tpp*D*dtype");
  if (tokens_per_page % kTile != 0 || view.start_offset % (head_dim * 2) || view.page_stride % (head_dim * 2))
    return set_error(JENGA_ERR_UNSUPPORTED, "jenga_paged_prefill: tokens_per_page must be a multiple of 16");
  if (batch == 0 || total_tokens == 0) return JENGA_OK;
  const int G = num_q_heads / num_kv_heads;
  PrefillParams prm{};
  prm.arena = static_cast<const uint8_t*>(arena_base);
  prm.start_offset = view.start_offset;
  prm.page_stride = view.page_stride;
  prm.out = out;
  prm.cu_q = cu_q;
  prm.table = block_table;
  prm.seq_lens = seq_lens;
  prm.kind = kind;
  prm.window = static_cast<int64_t>(window);
  prm.max_blocks = max_blocks;
  prm.hq = num_q_heads;
  prm.hkv = num_kv_heads;
  prm.tpp = static_cast<int>(tokens_per_page);
  prm.q_blocks = (max_chunk + kRows / G - 1) / (kRows / G);
  if (softcap > 0.f) {
    prm.qscale = scale;
    prm.cap_log2 = softcap * kLog2e;
    prm.inv_cap = 1.f / softcap;
  } else {
    prm.qscale = scale * kLog2e;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int rc = jenga_decode::launch_prefill_tc5(arena_base, prm.start_offset, prm.page_stride, out, cu_q,
                                                  block_table, seq_lens, kind, prm.window, max_blocks, num_q_heads,
                                                  num_kv_heads, prm.tpp, prm.q_blocks, prm.qscale, prm.cap_log2,
                                                  prm.inv_cap, dtype, head_dim, batch, total_tokens, q, s);
  if (rc != JENGA_ERR_UNSUPPORTED) return rc;
  if (dtype == JENGA_BF16) return dispatch_d<__nv_bfloat16>(head_dim, G, prm, dtype, batch, total_tokens, q, s);
  return dispatch_d<__half>(head_dim, G, prm, dtype, batch, total_tokens, q, s);
}
