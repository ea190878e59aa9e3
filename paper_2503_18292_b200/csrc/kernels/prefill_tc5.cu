// Chunked-prefill paged attention on the 5th-generation tensor cores
// (tcgen05.mma + TMEM), bf16/fp16.  Rows are (token, query head) pairs
// r = t*G + g, 128 rows per query block.  Two kernels:
//  * paged_prefill_tc5_wide_kernel (head_dim 128 and 256): persistent clusters of 2
//    CTAs walking (query pair, KV head, request) units, tcgen05.mma.cta_group::2
//    with M = 256 over two adjacent query blocks, 128-key tiles (S = Q K^T issued
//    with N = 128), Q in shared memory (TMA), TMEM = O plus S buffers so S runs
//    ahead of the softmax; each SM holds half of every K/V tile (its 64 keys of K,
//    its half of head_dim of V); 8 softmax warps (two per TMEM lane quarter, each
//    owning half of the key columns), a TMA producer warp and a whole-warp MMA
//    issuer; output staged in shared memory and written by TMA stores.
//  * paged_prefill_tc5_kernel (head_dim 64): one CTA per query block,
//    cta_group::1, 64-key tiles, Q in TMEM (its single 64-column chunk is too
//    narrow to split V across a pair).
// Softmax (both): thread r owns query row r = TMEM lane r of S and O
// (32x32b tcgen05.ld); scores masked with the reference liveness rule
// (layer_policies.cpp:105-120), exponentiated against a lazily updated row max
// (O rescaled in TMEM only when the max grows by more than 2^8); P written back
// over its S columns (tcgen05.st) -- the TMEM A operand of O += P V.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>
#include <utility>

#include "decode_common.cuh"

namespace jenga_dev {
bool arena_extent(const void* base, uint64_t* bytes);
}

namespace {

using namespace jenga_decode;

constexpr int kRows = 128;
constexpr int kSoftWarps = 4;
constexpr int kProducerWarp = 4;
constexpr int kMmaWarp = 5;
constexpr int kT5Threads = 6 * 32;
constexpr int kBoxCols = 64;
constexpr float kRescaleThreshold = 8.f;  // log2 units: P <= 2^8 between rescales

struct Prefill5Params {
  const uint8_t* arena;
  uint64_t start_offset, page_stride;
  const void* q;
  void* out;
  const int32_t* cu_q;
  const int32_t* table;
  const int32_t* seq_lens;
  int kind;
  int64_t window;
  int max_blocks, hq, hkv, tpp, q_blocks, batch;
  float qscale, cap_log2, inv_cap;
};

// ---------------------------------------------------------------- tcgen05
__device__ __forceinline__ uint64_t umma_desc(uint32_t smem_addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  // sm100 shared-memory matrix descriptor, 128-byte swizzle (layout type 2),
  // version 1; addresses / offsets in 16-byte units.
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;  // version
  d |= 2ull << 61;  // SWIZZLE_128B
  return d;
}

// kind::f16 instruction descriptor: f32 accumulate, bf16 (1) or f16 (0)
// inputs, A K-major, B K-major (b_mn = 0) or MN-major (1), M x N.
template <typename T>
__device__ __forceinline__ uint32_t idesc_f16(int m, int n, int b_mn) {
  const uint32_t fmt = std::is_same<T, __nv_bfloat16>::value ? 1u : 0u;
  return (1u << 4) | (fmt << 7) | (fmt << 10) | (static_cast<uint32_t>(b_mn) << 16) |
         (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}




// cta_group::1 whole-warp forms (the head_dim 64 kernel).
__device__ __forceinline__ void umma_ts_w(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma_commit_w(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
          jenga_dev::smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t addr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// Two 32-column TMEM loads behind one tcgen05.wait::ld.
__device__ __forceinline__ void tmem_ld64(uint32_t addr, float (&v)[64]) {
  uint32_t r[64];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%64];\n"
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%32, %33, %34, %35, %36, %37, %38, %39, %40, %41, %42, %43, %44, "
      "%45, %46, %47, %48, %49, %50, %51, %52, %53, %54, %55, %56, %57, %58, %59, %60, %61, %62, %63}, [%65];\n"
      "tcgen05.wait::ld.sync.aligned;\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]),
        "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]),
        "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]),
        "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),
        "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(addr), "r"(addr + 32)
      : "memory");
#pragma unroll
  for (int i = 0; i < 64; ++i) v[i] = __uint_as_float(r[i]);
}

// Two 32-column TMEM loads (any two column offsets) behind one tcgen05.wait::ld.
__device__ __forceinline__ void tmem_ld32x2(uint32_t a0, uint32_t a1, float (&v)[32], float (&w)[32]) {
  uint32_t r[64];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%64];\n"
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%32, %33, %34, %35, %36, %37, %38, %39, %40, %41, %42, %43, %44, "
      "%45, %46, %47, %48, %49, %50, %51, %52, %53, %54, %55, %56, %57, %58, %59, %60, %61, %62, %63}, [%65];\n"
      "tcgen05.wait::ld.sync.aligned;\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]),
        "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]),
        "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]),
        "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),
        "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(a0), "r"(a1)
      : "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    v[i] = __uint_as_float(r[i]);
    w[i] = __uint_as_float(r[32 + i]);
  }
}

__device__ __forceinline__ void tmem_st32u(uint32_t addr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};\n" ::"r"(addr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
      : "memory");
}


__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

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

// Single-CTA 3-D / 4-D TMA loads (box at {0, row, c2[, 0]}).
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, int32_t row, int32_t c2, uint64_t* bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;\n" ::"r"(jenga_dev::smem_u32(dst)),
      "l"(tmap), "r"(0), "r"(row), "r"(c2), "r"(jenga_dev::smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const void* tmap, int32_t row, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %2, %2}], [%4], %5;\n" ::"r"(jenga_dev::smem_u32(dst)),
      "l"(tmap), "r"(0), "r"(row), "r"(jenga_dev::smem_u32(bar)), "l"(policy)
      : "memory");
}

// Warp-cooperative look-ahead over one request's block table for the TMA
// producer: lane l holds table[base + l] (cur) and table[base + 32 + l] (nxt),
// so a page lookup is a shuffle instead of a dependent global load per 16-row
// piece (which serialised ~6 L2 round trips into every tile).  Lookups must be
// warp-uniform and non-decreasing; indices clamp to the last block like the
// direct form table[min(blk, max_blocks - 1)].
struct PageLookahead {
  const int32_t* table;
  int max_blocks, base, cur, nxt;
  __device__ __forceinline__ int load(int i, int lane) const {
    return __ldg(table + min(i + lane, max_blocks - 1));
  }
  __device__ __forceinline__ void init(const int32_t* t, int mb, int first, int lane) {
    table = t;
    max_blocks = mb;
    base = first;
    cur = load(base, lane);
    nxt = load(base + 32, lane);
  }
  __device__ __forceinline__ int32_t get(int blk, int lane) {
    while (blk >= base + 32) {
      base += 32;
      cur = nxt;
      nxt = load(base + 32, lane);
    }
    return __shfl_sync(0xffffffffu, cur, blk - base);
  }
};

// D = head_dim, G = query heads per KV head, KT = KV tokens per tile,
// NS = K/V ring stages.
template <typename T, int D, int G, int KT, int NS>
__global__ void __launch_bounds__(kT5Threads, 1)
    paged_prefill_tc5_kernel(const Prefill5Params p, const __grid_constant__ CUtensorMap k_map,
                             const __grid_constant__ CUtensorMap v_map) {
  // Same box layouts as the CTA-pair kernel, whole tile per CTA:
  //   K: [8-key group][chunk][8 rows][128 B], one 4-D box per 16-key page piece;
  //   V: [16-key piece][chunk][16 rows][128 B], one 3-D box per piece.
  constexpr int NBOX = D / kBoxCols;          // 64-column chunks of head_dim
  constexpr int QB = kRows / G;               // tokens per query block
  constexpr int K_GROUP = NBOX * 8 * 128;     // one 8-key group, all chunks
  constexpr int V_PIECE = NBOX * kTile * 128; // one 16-key piece, all chunks
  constexpr int KV_BYTES = NBOX * KT * 128;   // K (or V) of one tile, one head
  constexpr int STAGE = 2 * KV_BYTES;
  constexpr int PIECES = KT / kTile;          // 16-row TMA boxes per tile chunk
  constexpr int Q_COL = D;                    // Q: D/2 packed columns after O
  constexpr int S_COL = D + D / 2;            // S double buffer (P overwrites its S in place)
  constexpr uint32_t TMEM_COLS = S_COL + 2 * KT <= 256 ? 256 : 512;
  static_assert(KT == 64, "KV tile is 64 tokens");
  static_assert(S_COL + 2 * KT <= 512, "TMEM budget");

  extern __shared__ uint8_t smem_raw[];
  uint8_t* ring = smem_raw + ((1024 - (jenga_dev::smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + NS * STAGE);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = kv_full + NS;
  uint64_t* s_full = kv_empty + NS;
  uint64_t* p_full = s_full + 2;
  uint64_t* p_empty = p_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(p_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int c_len = p.cu_q[b + 1] - p.cu_q[b];
  const int t0 = qb * QB;
  if (t0 >= c_len) return;
  const int n = p.seq_lens[b];
  const bool cross = p.kind == JENGA_KIND_CROSS_ATTENTION;
  const int pos0 = n - c_len + t0;
  const int pos1 = n - c_len + min(t0 + QB, c_len) - 1;
  int key_lo = 0;
  const int key_hi = cross ? n - 1 : pos1;
  if (p.kind == JENGA_KIND_SLIDING_WINDOW && pos0 + 1 > p.window) key_lo = static_cast<int>(pos0 + 1 - p.window);
  const int tile_lo = key_lo / KT;
  const int ntiles = key_hi >= key_lo ? key_hi / KT - tile_lo + 1 : 0;

  if (threadIdx.x == 0) {
    jenga_dev::mbar_init(q_full, kSoftWarps);
    for (int i = 0; i < NS; ++i) {
      jenga_dev::mbar_init(&kv_full[i], 1);
      jenga_dev::mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      jenga_dev::mbar_init(&s_full[i], 1);
      jenga_dev::mbar_init(&p_full[i], kSoftWarps);
      jenga_dev::mbar_init(&p_empty[i], 1);
    }
    jenga_dev::fence_mbar_init();
  }
  if (warp == kMmaWarp) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     jenga_dev::smem_u32(tmem_slot)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int32_t* table = p.table + static_cast<int64_t>(b) * p.max_blocks;

  if (warp == kProducerWarp) {  // the whole warp walks the table; lane 0 issues
    if (lane == 0) {
      jenga_dev::prefetch_tmap(&k_map);
      jenga_dev::prefetch_tmap(&v_map);
    }
    const uint64_t policy = jenga_dev::l2_policy_evict_first();
    const int64_t row_bytes = D * 2;
    const int64_t base_row = static_cast<int64_t>(p.start_offset) / row_bytes + static_cast<int64_t>(h) * 2 * p.tpp;
    const int64_t page_rows = static_cast<int64_t>(p.page_stride) / row_bytes;
    const int v_rows = p.tpp;  // head-major slice
    PageLookahead pl;
    pl.init(table, p.max_blocks, tile_lo * KT / p.tpp, lane);
    for (int j = 0; j < ntiles; ++j) {
      const int st = j % NS;
      if (j >= NS) jenga_dev::mbar_wait(&kv_empty[st], ((j / NS) & 1) ^ 1);
      uint8_t* ks = ring + st * STAGE;
      if (lane == 0) jenga_dev::mbar_arrive_expect_tx(&kv_full[st], STAGE);
      for (int pc = 0; pc < PIECES; ++pc) {
        const int tok = (tile_lo + j) * KT + pc * kTile;
        const int32_t page = pl.get(tok / p.tpp, lane);
        const int32_t row = static_cast<int32_t>(base_row + static_cast<int64_t>(max(page, 0)) * page_rows +
                                                 tok % p.tpp);
        if (lane == 0) {
          tma_load_4d(ks + pc * 2 * K_GROUP, &k_map, row, &kv_full[st], policy);
          tma_load_3d(ks + KV_BYTES + pc * V_PIECE, &v_map, row + v_rows, 0, &kv_full[st], policy);
        }
      }
    }
  } else if (warp == kMmaWarp) {
    {  // the whole warp runs the loop; elect.sync issues (as in the 128-key kernel)
      const uint32_t id_s = idesc_f16<T>(kRows, KT, 0);
      const uint32_t id_o = idesc_f16<T>(kRows, D, 1);
      // O += P_jj V_jj: P (bf16/fp16, packed over S) from TMEM, V [KT][D] MN-major
      auto issue_pv = [&](int jj) {
        const int sb = jj & 1;
        jenga_dev::mbar_wait(&p_full[sb], (jj >> 1) & 1);
        tc_fence_after();
        const uint32_t v_u = jenga_dev::smem_u32(ring + (jj % NS) * STAGE + KV_BYTES);
#pragma unroll
        for (int k = 0; k < KT / 16; ++k)
          umma_ts_w(tmem, tmem + S_COL + sb * KT + k * 8, umma_desc(v_u + k * V_PIECE, kTile * 128, 1024), id_o,
                  (jj > 0 || k > 0) ? 1u : 0u);
        umma_commit_w(&p_empty[sb]);          // O updated
        umma_commit_w(&kv_empty[jj % NS]);    // K/V stage free
      };
      jenga_dev::mbar_wait(q_full, 0);
      // In-order issue: S_{j} (into the buffer P_{j-2} occupied) follows PV_{j-2}.
      for (int j = 0; j < ntiles; ++j) {
        const int st = j % NS, sb = j & 1;
        jenga_dev::mbar_wait(&kv_full[st], (j / NS) & 1);
        tc_fence_after();
        const uint32_t k_u = jenga_dev::smem_u32(ring + st * STAGE);
#pragma unroll
        for (int k = 0; k < D / 16; ++k)   // S = Q K^T: Q from TMEM, K [KT][D] K-major
          umma_ts_w(tmem + S_COL + sb * KT, tmem + Q_COL + k * 8,
                  umma_desc(k_u + (k >> 2) * 1024 + (k & 3) * 32, 16, K_GROUP), id_s, k > 0 ? 1u : 0u);
        umma_commit_w(&s_full[sb]);
        if (j >= 1) issue_pv(j - 1);
      }
      if (ntiles > 0) issue_pv(ntiles - 1);
    }
  } else {
    // ------------------------------------------ softmax / correction warps
    const int r = threadIdx.x;  // query row == TMEM lane
    const uint32_t lane_addr = static_cast<uint32_t>(warp * 32) << 16;
    const int tok = t0 + r / G;
    const bool row_ok = tok < c_len;
    const int ipos = n - c_len + tok;
    // Q row -> TMEM (D/2 packed columns), read once from global
    {
      const uint4* qrow = reinterpret_cast<const uint4*>(
          static_cast<const T*>(p.q) + (static_cast<int64_t>(p.cu_q[b] + tok) * p.hq + h * G + r % G) * D);
#pragma unroll 1
      for (int c = 0; c < D / 64; ++c) {
        uint32_t w[32];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint4 x = row_ok ? jenga_dev::ld_nc_v4(qrow + c * 8 + i) : make_uint4(0, 0, 0, 0);
          w[4 * i] = x.x;
          w[4 * i + 1] = x.y;
          w[4 * i + 2] = x.z;
          w[4 * i + 3] = x.w;
        }
        tmem_st32u(tmem + lane_addr + Q_COL + c * 32, w);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) jenga_dev::mbar_arrive(q_full);
    }
    // row r attends keys [lo_r, hi_r] (empty range for padding rows)
    int lo_r = 0, hi_r = cross ? n - 1 : ipos;
    if (p.kind == JENGA_KIND_SLIDING_WINDOW && static_cast<int64_t>(ipos) + 1 > p.window)
      lo_r = static_cast<int>(ipos + 1 - p.window);
    if (!row_ok || hi_r < lo_r) lo_r = hi_r = 1 << 30;
    const uint32_t span = static_cast<uint32_t>(hi_r - lo_r);
    const bool softcap = p.cap_log2 > 0.f;
    const float sc = softcap ? 1.f : p.qscale;  // scores -> log2 domain
    const float qi = p.qscale * p.inv_cap;
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < ntiles; ++j) {
      const int sb = j & 1;
      const int ktok0 = (tile_lo + j) * KT;
      jenga_dev::mbar_wait(&s_full[sb], (j >> 1) & 1);
      tc_fence_after();
      static_assert(KT == 64, "one 64-column S load");
      float s[KT];
      tmem_ld64(tmem + lane_addr + S_COL + sb * KT, s);  // both halves behind one wait
      if (softcap) {
#pragma unroll
        for (int i = 0; i < KT; ++i) s[i] = p.cap_log2 * tanhf(s[i] * qi);
      }
      if (ktok0 < lo_r || ktok0 + KT - 1 > hi_r) {  // boundary tile for this row
#pragma unroll
        for (int i = 0; i < KT; ++i)
          s[i] = static_cast<uint32_t>(ktok0 + i - lo_r) <= span ? s[i] : -INFINITY;
      }
      float mt = -INFINITY;
#pragma unroll
      for (int i = 0; i < KT; ++i) mt = fmaxf(mt, s[i]);
      mt *= sc;
      // Grow the reference max only when it moved by > 2^8 (P stays <= 256);
      // tcgen05.ld/st are warp-collective, so the warp rescales together.
      if (__any_sync(0xffffffffu, mt > m_used + kRescaleThreshold)) {
        const float m_new = fmaxf(m_used, mt);
        if (j >= 1) {  // O holds P_0..P_{j-1} V: wait for the last PV, rescale rows
          const float alpha = m_used == -INFINITY ? 1.f : jenga_dev::fast_exp2(m_used - m_new);
          jenga_dev::mbar_wait(&p_empty[(j - 1) & 1], ((j - 1) >> 1) & 1);
          tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < D; c += 32) {
            float v[32];
            tmem_ld32(tmem + lane_addr + c, v);
            uint32_t u[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) u[i] = __float_as_uint(v[i] * alpha);
            tmem_st32u(tmem + lane_addr + c, u);
          }
          tmem_st_wait();
          l *= alpha;
        }
        m_used = m_new;
      }
      uint32_t pk[KT / 2];
      float rs0 = 0.f, rs1 = 0.f;
      const float neg = m_used == -INFINITY ? 0.f : -m_used;  // masked: exp2(-inf) = 0
#pragma unroll
      for (int i = 0; i < KT; i += 2) {
        const float a = jenga_dev::fast_exp2(fmaf(s[i], sc, neg));
        const float bb = jenga_dev::fast_exp2(fmaf(s[i + 1], sc, neg));
        rs0 += a;
        rs1 += bb;
        pk[i / 2] = pack2<T>(a, bb);
      }
      l += rs0 + rs1;
      // P_j over S_j's first KT/2 columns (the A operand of O += P_j V_j)
#pragma unroll
      for (int c = 0; c < KT / 2; c += 32) {
        uint32_t w[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) w[i] = pk[c + i];
        tmem_st32u(tmem + lane_addr + S_COL + sb * KT + c, w);
      }
      tmem_st_wait();
      // masked keys of a boundary tile may hold non-finite V bytes (0*NaN = NaN
      // in the MMA): zero those V rows; 128 threads cover KT rows x NBOX chunks
      if (ktok0 < key_lo || ktok0 + KT - 1 > key_hi) {
        uint8_t* vs = ring + (j % NS) * STAGE + KV_BYTES;
        for (int idx = r; idx < KT * NBOX; idx += kRows) {
          const int vrow = idx % KT, chunk = idx / KT;
          const int key = ktok0 + vrow;
          if (key >= key_lo && key <= key_hi) continue;
          uint4* line = reinterpret_cast<uint4*>(vs + (vrow / kTile) * V_PIECE + chunk * kTile * 128 +
                                                 (vrow % kTile) * 128);
#pragma unroll
          for (int c = 0; c < 8; ++c) line[c] = make_uint4(0, 0, 0, 0);
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) jenga_dev::mbar_arrive(&p_full[sb]);
    }
    // ---- epilogue: O / l -> out
    if (ntiles > 0) jenga_dev::mbar_wait(&p_empty[(ntiles - 1) & 1], ((ntiles - 1) >> 1) & 1);
    tc_fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
    T* outp = static_cast<T*>(p.out) + (static_cast<int64_t>(p.cu_q[b] + tok) * p.hq + h * G + r % G) * D;
#pragma unroll 1
    for (int c = 0; c < D; c += 32) {
      float v[32];
      if (ntiles > 0) {
        tmem_ld32(tmem + lane_addr + c, v);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = 0.f;
      }
      if (row_ok) {
#pragma unroll
        for (int i = 0; i < 32; i += 8)
          *reinterpret_cast<uint4*>(outp + c + i) = make_uint4(pack2<T>(v[i] * inv, v[i + 1] * inv),
                                                               pack2<T>(v[i + 2] * inv, v[i + 3] * inv),
                                                               pack2<T>(v[i + 4] * inv, v[i + 5] * inv),
                                                               pack2<T>(v[i + 6] * inv, v[i + 7] * inv));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(TMEM_COLS));
  }
}

// ---------------------------------------------------------------- 2-SM pair
// Same algorithm on a CTA pair (cluster of 2, cta_group::2): the leader issues
// M=256 MMAs over both CTAs' 128 query rows (adjacent query blocks of one
// (request, KV head)); each CTA holds HALF of every K/V tile — K rows of its
// half of the tile's keys, V columns of its half of head_dim — so each SM
// streams half the K/V bytes per flop.  TMA loads of both CTAs complete on the
// leader's barrier; the leader's commits are multicast to both CTAs; the
// peer's softmax warps arrive remotely on the leader's q_full / p_full.
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t map_to_cta0(const void* p) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;\n" : "=r"(r) : "r"(jenga_dev::smem_u32(p)));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// Remote arrive on the leader's barrier.  The default (.release.cta) form is a
// bare SYNCS.ARRIVE; P visibility to the MMA comes from tcgen05.wait::st +
// tcgen05.fence::before_thread_sync.  Only generic shared-memory writes the
// leader's MMA must see (zeroed V rows) need the cluster-scope release, whose
// MEMBAR.GPU + ERRBAR cost ~25% of the kernel when paid every tile.
__device__ __forceinline__ void arrive_cta0(uint32_t cluster_bar) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_bar) : "memory");
}
// Cluster-scope release arrive out of line: inlined under a branch, ptxas
// predicates its MEMBAR.GPU / ERRBAR sequence, whose fixed stall cycles are paid
// even when predicated off (~5% of the 128-key kernel).
__device__ __noinline__ void arrive_cta0_release_ool(uint32_t cluster_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_bar) : "memory");
}
__device__ __forceinline__ void expect_tx_cta0(uint32_t cluster_bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cluster.b64 _, [%0], %1;\n" ::"r"(cluster_bar), "r"(bytes)
               : "memory");
}
// 3-D box over the arena viewed as [chunk][row][64 cols] (dim0 = 64 columns,
// dim1 = rows at row_bytes, dim2 = 64-column chunks at 128 B): one TMA covers
// several head_dim chunks of a run of rows, landing chunk-major in shared memory.
__device__ __forceinline__ void tma_load_3d_pair(void* dst, const void* tmap, int32_t c1, int32_t c2,
                                                 uint32_t cluster_bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;\n" ::"r"(jenga_dev::smem_u32(dst)),
      "l"(tmap), "r"(cluster_bar), "r"(0), "r"(c1), "r"(c2), "l"(policy)
      : "memory");
}
// 4-D box over the arena as [8-row half][chunk][row][64 cols]: one TMA loads a
// 16-row page piece of every head_dim chunk in the K layout [half][chunk][8 rows].
__device__ __forceinline__ void tma_load_4d_pair(void* dst, const void* tmap, int32_t row, uint32_t cluster_bar,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], %7;\n" ::"r"(jenga_dev::smem_u32(dst)),
      "l"(tmap), "r"(cluster_bar), "r"(0), "r"(row), "r"(0), "r"(0), "l"(policy)
      : "memory");
}

#ifndef JENGA_PF_TRACE_Q
#define JENGA_PF_TRACE_Q 0  // TMEM lane quarter (SM sub-partition) whose softmax warps are traced
#endif
#ifdef JENGA_PF_TRACE
// Profiling-only (variant builds): clock64 stamps of the pipeline events of the
// first CTA pair's leader, [event][tile] for tiles < 64.
__device__ long long g_pf_trace[16][64];
#define PF_TRACE(ev, j) \
  do { if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (j) < 64) g_pf_trace[ev][j] = clock64(); } while (0)
#else
#define PF_TRACE(ev, j) do { } while (0)
#endif

// Q rows of one CTA: 4-D box {64 columns, G heads, QB tokens, 1 chunk} over q viewed as
// [chunk][token][head][64 columns], landing as rows r = t*G + g of 128 B (swizzled).
__device__ __forceinline__ void tma_load_q_pair(void* dst, const void* tmap, int32_t head, int32_t token, int32_t chunk,
                                                uint32_t cluster_bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];\n" ::"r"(jenga_dev::smem_u32(dst)),
      "l"(tmap), "r"(cluster_bar), "r"(0), "r"(head), "r"(token), "r"(chunk)
      : "memory");
}
// Whole-warp forms: the warp runs the issue loop convergently (operands are
// warp-uniform, so they stay in uniform registers) and elect.sync picks the one
// issuing lane inside the asm -- no per-instruction ELECT / BRA.U.ANY loop or
// R2UR round trips, which capped the single-thread issuer at ~90 cycles per MMA.
__device__ __forceinline__ void umma2_ss_w(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma2_ts_w(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc,
                                           uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void umma2_commit_both_w(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}\n" ::"r"(
          jenga_dev::smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}

// Packed f32x2 FMA / add (FFMA2 / FADD2 on sm_100a: two lanes per issue slot).
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.ftz.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.ftz.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
// exp2_fma for two lanes, the polynomial on FFMA2.
__device__ __forceinline__ float2 exp2_fma2(float2 x) {
  x.x = fmaxf(x.x, -127.f);
  x.y = fmaxf(x.y, -127.f);
  const float2 t = fadd2(x, make_float2(12582912.f, 12582912.f));
  const float2 f = fadd2(x, fadd2(make_float2(12582912.f, 12582912.f), make_float2(-t.x, -t.y)));
  float2 q = ffma2(make_float2(0.0555041086f, 0.0555041086f), f, make_float2(0.2402264923f, 0.2402264923f));
  q = ffma2(q, f, make_float2(0.6931471806f, 0.6931471806f));
  q = ffma2(q, f, make_float2(1.f, 1.f));
  return make_float2(__int_as_float(__float_as_int(q.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(q.y) + (__float_as_int(t.y) << 23)));
}

#ifndef JENGA_PF_SPLITO
#define JENGA_PF_SPLITO 1
#endif

// Pairs (of every 4 pairs of S columns) whose exponentials the 128-key kernel
// computes on the FMA pipe instead of the MUFU.
#ifndef JENGA_PF_EMU2
#define JENGA_PF_EMU2 1
#endif

template <typename T, int D, int G, int NSK, int NSV>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__((2 * kSoftWarps + 2) * 32, 1)
    paged_prefill_tc5_wide_kernel(const Prefill5Params p, const __grid_constant__ CUtensorMap k_map,
                                  const __grid_constant__ CUtensorMap v_map, const __grid_constant__ CUtensorMap q_map) {
  // 128-key tiles on a CTA pair (cta_group::2, M = 256 query rows, 128 per CTA).
  // S = Q K^T is issued with N = 128 keys (64-key instructions run the tensor
  // core at ~72%: they cannot be issued faster than ~45 cycles each), so Q lives
  // in shared memory (SS MMA) and TMEM holds O (D columns) plus NSB = (512 - D) / 128
  // S buffers: 2 at head_dim 256, 3 at 128.  The MMA issuer keeps S NSB - 1 tiles
  // ahead of the softmax (S(j + NSB) is issued right after O += P(j) V(j), which
  // frees its buffer), so the softmax never waits for a tile's scores.
  // Softmax: 8 warps, two per TMEM lane quarter; warp w owns query rows
  // 32 (w & 3) .. + 31 and key columns 64 (w >> 2) .. + 63 of every S tile (the row
  // max is exchanged between the two warps of a row through shared memory), so two
  // warps per SM sub-partition keep the MUFU busy through each other's loads,
  // reductions and TMEM stores.
  // K and V stream through separate rings (K of tile j + 1 is needed before V of
  // tile j): K slot released when the tile's S MMAs complete, V slot when its PV
  // MMAs complete.
  // Persistent: one CTA pair per two SMs walks the work units (request, KV head,
  // pair of query blocks), ordered heaviest first (the last query blocks of a causal
  // chunk attend the most keys) and dealt to the clusters boustrophedon.  Tile-indexed state
  // (rings, S buffers, P handoffs) runs on a per-CTA tile counter across units, so
  // the next unit's Q (TMA, once the last S MMA of the unit read the old one) and
  // K/V stream in while the current unit's last tiles and epilogue run; TMEM and
  // barriers are set up once.  Shared-memory layouts (128-byte swizzle):
  //   Q: [chunk c][128 rows][128 B]              (one 4-D TMA box {64, G heads, QB tokens, 1} per chunk)
  //   K: [8-key group][chunk c][8 rows][128 B]   (one 4-D TMA box per 16-key piece; this CTA's 64 keys)
  //   V: [16-key piece][chunk c][16 rows][128 B] (one 3-D box per piece; this CTA's half of head_dim)
  constexpr int KT = 128;
  constexpr int NBOX = D / kBoxCols;
  constexpr int VB = NBOX / 2;
  constexpr int QB = kRows / G;
  constexpr int KH = KT / 2;
  constexpr int K_GROUP = NBOX * 8 * 128;
  constexpr int K_BYTES = (KH / 8) * K_GROUP;
  constexpr int V_PIECE = VB * kTile * 128;
  constexpr int V_BYTES = (KT / kTile) * V_PIECE;
  constexpr int Q_BYTES = NBOX * kRows * 128;
  // SPLITO (head_dim 128): one O accumulator per key half, so each softmax warp keeps
  // its own running max / sum and the two warps of a lane quarter never synchronise
  // per tile (their load / max / store phases drift apart and overlap each other's
  // exponentials); the halves are merged once at the end.  TMEM: O_0 | O_1 | 2 S.
  constexpr bool SPLITO = JENGA_PF_SPLITO && D == 128;
  constexpr int NO = SPLITO ? 2 : 1;          // O accumulators
  constexpr int NPH = SPLITO ? 2 : 1;         // P handoffs (p_full / p_empty) per S buffer
  constexpr int NSB = (512 - NO * D) / KT;    // S buffers
  constexpr int S_COL0 = NO * D;
  constexpr int HC = KT / 2;                  // S columns per softmax warp
  constexpr uint32_t TMEM_COLS = 512;
  static_assert(NBOX % 2 == 0 && NO * D + NSB * KT == 512, "128-key kernel shape");
  constexpr int SW = 2 * kSoftWarps, PW = SW, MW = SW + 1;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* qs = smem_raw + ((1024 - (jenga_dev::smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* kring = qs + Q_BYTES;
  uint8_t* vring = kring + NSK * K_BYTES;
  uint8_t* ostage = vring + NSV * V_BYTES;    // output staging, 2 KiB per softmax warp
  float* red = reinterpret_cast<float*>(ostage + kRows * 128);  // [tile parity][half][row]
  uint64_t* bars = reinterpret_cast<uint64_t*>(red + 2 * 2 * kRows);
  uint64_t* q_full = bars;                    // leader: all softmax warps of the pair
  uint64_t* k_full = bars + 1;                // leader: both CTAs' TMA bytes
  uint64_t* k_empty = k_full + NSK;           // both: multicast commit
  uint64_t* v_full = k_empty + NSK;
  uint64_t* v_empty = v_full + NSV;
  uint64_t* s_full = v_empty + NSV;           // both: multicast commit      [buffer]
  uint64_t* p_full = s_full + NSB;            // leader: the softmax warps   [buffer][half]
  uint64_t* p_empty = p_full + NSB * NPH;     // both: multicast commit      [buffer][half]
  uint64_t* q_empty = p_empty + NSB * NPH;     // both: multicast commit after a unit's last S MMA
  uint64_t* o_free = q_empty + 1;              // leader: all softmax warps, after a unit's O readout
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_free + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) PF_TRACE(15, 0);  // kernel entry (trace variant)
  const int cid = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  const int npairs = (p.q_blocks + 1) / 2;
  const int nunits = npairs * p.hkv * p.batch;
  struct Unit {
    int b, h, pt0, c_len, n, key_lo, key_hi, tile_lo, ntiles;
    bool live;
  };
  // unit u -> (query pair, KV head, request): the query pairs of one (request, head)
  // are consecutive -- units in flight together share that K/V through L2 (spreading
  // them over heads first measured 11% slower) -- last (heaviest) pair first
  auto unit_at = [&](int u) {
    Unit x;
    const int qp = npairs - 1 - u % npairs;
    x.h = (u / npairs) % p.hkv;
    x.b = u / (npairs * p.hkv);
    x.c_len = p.cu_q[x.b + 1] - p.cu_q[x.b];
    x.pt0 = 2 * qp * QB;
    x.live = x.pt0 < x.c_len;
    x.n = p.seq_lens[x.b];
    const int pos0 = x.n - x.c_len + x.pt0;
    const int pos1 = x.n - x.c_len + min(x.pt0 + 2 * QB, x.c_len) - 1;  // union of the pair's query rows
    x.key_lo = 0;
    x.key_hi = p.kind == JENGA_KIND_CROSS_ATTENTION ? x.n - 1 : pos1;
    if (p.kind == JENGA_KIND_SLIDING_WINDOW && pos0 + 1 > p.window) x.key_lo = static_cast<int>(pos0 + 1 - p.window);
    x.tile_lo = x.key_lo / KT;
    x.ntiles = x.live && x.key_hi >= x.key_lo ? x.key_hi / KT - x.tile_lo + 1 : 0;
    return x;
  };
  const bool cross = p.kind == JENGA_KIND_CROSS_ATTENTION;
  // this cluster's k-th unit: rounds of `nclusters` units dealt boustrophedon (the
  // cluster that got a round's heaviest unit gets the next round's lightest), which
  // evens out the per-cluster totals of the heaviest-first unit order
  auto snake = [&](int k) { return k * nclusters + ((k & 1) ? nclusters - 1 - cid : cid); };

  if (threadIdx.x == 0) {
    jenga_dev::mbar_init(q_full, 1);
    for (int i = 0; i < NSK; ++i) {
      jenga_dev::mbar_init(&k_full[i], 1);
      jenga_dev::mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < NSV; ++i) {
      jenga_dev::mbar_init(&v_full[i], 1);
      jenga_dev::mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < NSB; ++i) jenga_dev::mbar_init(&s_full[i], 1);
    for (int i = 0; i < NSB * NPH; ++i) {
      jenga_dev::mbar_init(&p_full[i], 2 * SW / NPH);
      jenga_dev::mbar_init(&p_empty[i], 1);
    }
    jenga_dev::mbar_init(q_empty, 1);
    jenga_dev::mbar_init(o_free, 2 * SW);
    jenga_dev::fence_mbar_init();
  }
  if (warp == MW) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     jenga_dev::smem_u32(tmem_slot)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  tc_fence_before();
  cluster_sync();  // barriers of both CTAs initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == PW) {
    // Lane l < 8 owns the 16-key page piece l of every tile: its block index by
    // multiply-shift division, its page from the warp's table look-ahead (lane i
    // holds table[base + i] / table[base + 32 + i]) by one shuffle, its arena row
    // by one multiply-add; the lanes then issue their own TMA boxes.  Per unit, the
    // unit's Q first (once the previous unit's last S MMA has read the old Q).
    if (lane == 0) {
      jenga_dev::prefetch_tmap(&k_map);
      jenga_dev::prefetch_tmap(&v_map);
      jenga_dev::prefetch_tmap(&q_map);
    }
    const uint64_t policy = jenga_dev::l2_policy_evict_first();
    const int64_t row_bytes = D * 2;
    const int64_t page_rows = static_cast<int64_t>(p.page_stride) / row_bytes;
    const uint32_t tpp = static_cast<uint32_t>(p.tpp);
    uint32_t lg = 0;
    while ((1u << lg) < tpp) ++lg;
    const uint32_t dm = static_cast<uint32_t>(((1ull << (31 + lg)) + tpp - 1) / tpp), ds = lg - 1;  // tpp >= 16
    const int mb = p.max_blocks;
    const int piece = lane & 7;
    const int k_lane0 = static_cast<int>(rank) * (KH / kTile);  // this CTA's half of the keys
    int g0 = 0, nu = 0;  // tiles / live units this CTA processed before the current unit
    for (int k = 0, u = cid; u < nunits; ++k, u = snake(k)) {
      const Unit x = unit_at(u);
      if (x.ntiles == 0) continue;
      {  // Q of this unit: this CTA's 128 rows, one box per 64-column chunk
        if (nu > 0) jenga_dev::mbar_wait(q_empty, (nu - 1) & 1);
        const uint32_t qf0 = map_to_cta0(q_full);
        if (lane == 0 && rank == 0) expect_tx_cta0(qf0, 2 * Q_BYTES);
        if (lane < NBOX)
          tma_load_q_pair(qs + lane * kRows * 128, &q_map, x.h * G, p.cu_q[x.b] + x.pt0 + static_cast<int>(rank) * QB,
                          lane, qf0);
      }
      const int32_t* table = p.table + static_cast<int64_t>(x.b) * mb;
      const int64_t base_row = static_cast<int64_t>(p.start_offset) / row_bytes + static_cast<int64_t>(x.h) * 2 * p.tpp;
      int base = static_cast<int>(static_cast<uint32_t>(x.tile_lo * KT) / tpp);
      int cur = __ldg(table + min(base + lane, mb - 1)), nxt = __ldg(table + min(base + 32 + lane, mb - 1));
      auto row_for = [&](int jj) {  // warp-uniform call; this lane's piece of tile jj
        const uint32_t tok = static_cast<uint32_t>((x.tile_lo + jj) * KT + piece * kTile);
        const int blk = static_cast<int>(__umulhi(tok, dm) >> ds);
        const int off = static_cast<int>(tok - static_cast<uint32_t>(blk) * tpp);
        const int blk0 = __shfl_sync(0xffffffffu, blk, 0);
        while (blk0 >= base + 32) {
          base += 32;
          cur = nxt;
          nxt = __ldg(table + min(base + 32 + lane, mb - 1));
        }
        const int rel = blk - base;  // < 64: a tile spans at most 8 blocks
        const int a = __shfl_sync(0xffffffffu, cur, rel & 31), c = __shfl_sync(0xffffffffu, nxt, rel & 31);
        const int32_t page = rel < 32 ? a : c;
        return static_cast<int32_t>(base_row + static_cast<int64_t>(max(page, 0)) * page_rows + off);
      };
      auto issue_k = [&](int jj, int32_t row) {
        const int gg = g0 + jj, st = gg % NSK;
        if (gg >= NSK) jenga_dev::mbar_wait(&k_empty[st], ((gg / NSK) & 1) ^ 1);
        const uint32_t full0 = map_to_cta0(&k_full[st]);
#ifdef JENGA_PF_NOLOAD
        if (lane == 0 && rank == 0) arrive_cta0(full0);  // timing-only variant: no K/V traffic
        return;
#endif
        if (lane == 0 && rank == 0) expect_tx_cta0(full0, 2 * K_BYTES);
        if (lane >= k_lane0 && lane < k_lane0 + KH / kTile)
          tma_load_4d_pair(kring + st * K_BYTES + (lane - k_lane0) * 2 * K_GROUP, &k_map, row, full0, policy);
      };
      auto issue_v = [&](int jj, int32_t row) {
        const int gg = g0 + jj, st = gg % NSV;
        if (gg >= NSV) jenga_dev::mbar_wait(&v_empty[st], ((gg / NSV) & 1) ^ 1);
        const uint32_t full0 = map_to_cta0(&v_full[st]);
#ifdef JENGA_PF_NOLOAD
        if (lane == 0 && rank == 0) arrive_cta0(full0);
        return;
#endif
        if (lane == 0 && rank == 0) expect_tx_cta0(full0, 2 * V_BYTES);
        if (lane < KT / kTile)
          tma_load_3d_pair(vring + st * V_BYTES + lane * V_PIECE, &v_map, row + p.tpp, static_cast<int>(rank) * VB,
                           full0, policy);
      };
      int32_t row_cur = row_for(0), row_nxt = 0;
      issue_k(0, row_cur);
      for (int j = 0; j < x.ntiles; ++j) {
        if (j + 1 < x.ntiles) {  // K runs one tile ahead of V
          row_nxt = row_for(j + 1);
          issue_k(j + 1, row_nxt);
        }
        issue_v(j, row_cur);
        row_cur = row_nxt;
      }
      g0 += x.ntiles;
      ++nu;
    }
  } else if (warp == MW) {
    if (rank == 0) {  // the whole warp runs the loop; elect.sync issues
      const uint32_t id_s = idesc_f16<T>(2 * kRows, KT, 0);
      const uint32_t id_o = idesc_f16<T>(2 * kRows, D, 1);
      // descriptors as base + constant (one add per MMA on the uniform datapath)
      const uint64_t q_desc0 = umma_desc(jenga_dev::smem_u32(qs), 16, 1024);
      const uint64_t k_desc0 = umma_desc(jenga_dev::smem_u32(kring), 16, K_GROUP);
      const uint64_t v_desc0 = umma_desc(jenga_dev::smem_u32(vring), kTile * 128, 1024);
      int g0 = 0, nu = 0;
      for (int k = 0, u = cid; u < nunits; ++k, u = snake(k)) {
        const Unit x = unit_at(u);
        if (x.ntiles == 0) continue;
        auto wait_v = [&](int jj) {
          const int gg = g0 + jj;
          jenga_dev::mbar_wait(&v_full[gg % NSV], (gg / NSV) & 1);
          tc_fence_after();
        };
        // boundary tiles (first / last) get V rows zeroed by the softmax threads after
        // s_full: their S is issued only once V has landed too
        auto wait_k = [&](int jj) {
          const int gg = g0 + jj;
          jenga_dev::mbar_wait(&k_full[gg % NSK], (gg / NSK) & 1);
          tc_fence_after();
          const int kt0 = (x.tile_lo + jj) * KT;
          if (kt0 < x.key_lo || kt0 + KT - 1 > x.key_hi) wait_v(jj);
        };
        auto issue_s = [&](int jj) {  // S(jj) = Q K_jj^T into buffer gg % NSB
          wait_k(jj);
          const int gg = g0 + jj;
          const uint64_t kd = k_desc0 + ((gg % NSK) * K_BYTES >> 4);
          const uint32_t d = tmem + S_COL0 + (gg % NSB) * KT;
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint32_t off = ((k >> 2) * 1024 + (k & 3) * 32) >> 4;
            umma2_ss_w(d, q_desc0 + (((k >> 2) * kRows * 128 + (k & 3) * 32) >> 4), kd + off, id_s, k > 0 ? 1u : 0u);
          }
          umma2_commit_both_w(&s_full[gg % NSB]);
          umma2_commit_both_w(&k_empty[gg % NSK]);
          if (jj == x.ntiles - 1) umma2_commit_both_w(q_empty);  // the unit's last read of Q
          if (lane == 0) PF_TRACE(2, gg);
        };
        auto issue_pv = [&](int jj) {  // O_h += P_h(jj) V_h,jj for each key half h (one half without SPLITO)
          const int gg = g0 + jj;
          const uint64_t vd = v_desc0 + ((gg % NSV) * V_BYTES >> 4);
          const uint32_t a = tmem + S_COL0 + (gg % NSB) * KT;
          constexpr int KPH = KT / 16 / NPH;  // 16-key MMAs per handoff
#pragma unroll
          for (int hh = 0; hh < NPH; ++hh) {
            jenga_dev::mbar_wait(&p_full[(gg % NSB) * NPH + hh], (gg / NSB) & 1);
            if (lane == 0 && hh == 0) PF_TRACE(0, gg);
            tc_fence_after();
            if (hh == 0) wait_v(jj);
#pragma unroll
            for (int k = 0; k < KPH; ++k) {
              const int kk = hh * KPH + k;
              // P of key half kk / 4 sits in that half's own first 32 S columns
              umma2_ts_w(tmem + hh * D, a + (kk >> 2) * HC + (kk & 3) * 8, vd + (kk * V_PIECE >> 4), id_o,
                         (jj > 0 || k > 0) ? 1u : 0u);
            }
            umma2_commit_both_w(&p_empty[(gg % NSB) * NPH + hh]);
          }
          umma2_commit_both_w(&v_empty[gg % NSV]);
        };
        jenga_dev::mbar_wait(q_full, nu & 1);
        if (lane == 0) PF_TRACE(3, nu);
        tc_fence_after();
        for (int j = 0; j < NSB - 1 && j < x.ntiles; ++j) issue_s(j);
        for (int j = 0; j < x.ntiles; ++j) {
          // S(j + NSB - 1) goes to the buffer PV(j - 1) released (in order), ahead of PV(j)
          if (j + NSB - 1 < x.ntiles) issue_s(j + NSB - 1);
          if (j == 0 && nu > 0) {  // O is overwritten by this unit's first PV: the previous unit read it out
            jenga_dev::mbar_wait(o_free, (nu - 1) & 1);
            tc_fence_after();
          }
          issue_pv(j);
        }
        g0 += x.ntiles;
        ++nu;
      }
    }
  } else {
    const int hf = warp >> 2;                   // column half of every S tile / O
    const int r = threadIdx.x & (kRows - 1);    // query row == TMEM lane
    const uint32_t lane_addr = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t p_full0 = map_to_cta0(&p_full[0]);
    const uint32_t o_free0 = map_to_cta0(o_free);
    const uint32_t pair_bar = 1 + (warp & 3);   // named barrier of the two warps sharing these rows
    int g0 = 0, nus = 0;
    for (int k = 0, u = cid; u < nunits; ++k, u = snake(k)) {
    const Unit x = unit_at(u);
    if (!x.live) continue;
    const int ntiles = x.ntiles, tile_lo = x.tile_lo, key_lo = x.key_lo, key_hi = x.key_hi, n = x.n;
    const int t0 = x.pt0 + static_cast<int>(rank) * QB;
    const int tok = t0 + r / G;
    const bool row_ok = tok < x.c_len;
    const int ipos = n - x.c_len + tok;
    int lo_r = 0, hi_r = cross ? n - 1 : ipos;
    if (p.kind == JENGA_KIND_SLIDING_WINDOW && static_cast<int64_t>(ipos) + 1 > p.window)
      lo_r = static_cast<int>(ipos + 1 - p.window);
    if (!row_ok || hi_r < lo_r) lo_r = hi_r = 1 << 30;
    const uint32_t span = static_cast<uint32_t>(hi_r - lo_r);
    const bool softcap = p.cap_log2 > 0.f;
    const float sc = softcap ? 1.f : p.qscale;
    const float qi = p.qscale * p.inv_cap;
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < ntiles; ++j) {
      const int gg = g0 + j;
      const int sb = gg % NSB;
      const uint32_t s_addr = tmem + lane_addr + S_COL0 + sb * KT;
      const int kc0 = (tile_lo + j) * KT + hf * HC;   // key of this warp's first column
      jenga_dev::mbar_wait(&s_full[sb], (gg / NSB) & 1);
      if ((warp & 3) == JENGA_PF_TRACE_Q && lane == 0 && rank == 0) PF_TRACE(4 + 6 * hf, gg);
      tc_fence_after();
#ifdef JENGA_PF_NOSOFTMAX
      if (true) {  // timing-only variant: hand the tile straight back to the MMA issuer
        tc_fence_before();
        __syncwarp();
        if (lane == 0) arrive_cta0(p_full0 + 8u * (sb * NPH + (SPLITO ? hf : 0)));
        continue;
      }
#endif
      float s[HC];
      tmem_ld64(s_addr + hf * HC, s);
      if ((warp & 3) == JENGA_PF_TRACE_Q && lane == 0 && rank == 0) PF_TRACE(5 + 6 * hf, gg);
      if (softcap) {
#pragma unroll
        for (int i = 0; i < HC; ++i) s[i] = p.cap_log2 * tanhf(s[i] * qi);
      }
      if (kc0 < lo_r || kc0 + HC - 1 > hi_r) {
#pragma unroll
        for (int i = 0; i < HC; ++i)
          s[i] = static_cast<uint32_t>(kc0 + i - lo_r) <= span ? s[i] : -INFINITY;
      }
      float m8[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) m8[i] = s[i];
#pragma unroll
      for (int i = 8; i < HC; i += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) m8[u] = fmaxf(m8[u], s[i + u]);
      }
      float mt = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])), fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
      mt *= sc;
      if constexpr (SPLITO) {
        // this warp's own running max over its key half; O_hf rescaled alone
        if (__any_sync(0xffffffffu, mt > m_used + kRescaleThreshold)) {
          const float m_new = fmaxf(m_used, mt);
          if (j >= 1) {
            const float alpha = m_used == -INFINITY ? 1.f : jenga_dev::fast_exp2(m_used - m_new);
            jenga_dev::mbar_wait(&p_empty[((gg - 1) % NSB) * NPH + hf], ((gg - 1) / NSB) & 1);
            tc_fence_after();
#pragma unroll 1
            for (int c = hf * D; c < (hf + 1) * D; c += 32) {
              float v[32];
              tmem_ld32(tmem + lane_addr + c, v);
              uint32_t u[32];
#pragma unroll
              for (int i = 0; i < 32; ++i) u[i] = __float_as_uint(v[i] * alpha);
              tmem_st32u(tmem + lane_addr + c, u);
            }
            tmem_st_wait();
            l *= alpha;
          }
          m_used = m_new;
        }
      } else {
      // Rescale test for the row: its max over both halves.  The two warps of these
      // rows first OR their "some row grew by more than 2^8" votes with one
      // barrier reduction; only then (rarely, after the first tiles) do they
      // exchange the half-row maxima through shared memory.
      uint32_t grow;
      asm volatile("{\n\t.reg .pred p, q;\n\tsetp.gt.f32 p, %1, %2;\n\tbar.red.or.pred q, %3, %4, p;\n\tselp.u32 %0, 1, 0, q;\n\t}\n"
                   : "=r"(grow) : "f"(mt), "f"(m_used + kRescaleThreshold), "r"(pair_bar), "n"(64) : "memory");
      if (grow) {
        float* rd = red + (j & 1) * 2 * kRows;
        rd[hf * kRows + r] = mt;
        asm volatile("bar.sync %0, %1;\n" ::"r"(pair_bar), "n"(64) : "memory");
        mt = fmaxf(mt, rd[(hf ^ 1) * kRows + r]);
        const float m_new = fmaxf(m_used, mt);
        if (j >= 1) {
          const float alpha = m_used == -INFINITY ? 1.f : jenga_dev::fast_exp2(m_used - m_new);
          jenga_dev::mbar_wait(&p_empty[(gg - 1) % NSB], ((gg - 1) / NSB) & 1);
          tc_fence_after();
#pragma unroll 1
          for (int c = hf * (D / 2); c < (hf + 1) * (D / 2); c += 32) {
            float v[32];
            tmem_ld32(tmem + lane_addr + c, v);
            uint32_t u[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) u[i] = __float_as_uint(v[i] * alpha);
            tmem_st32u(tmem + lane_addr + c, u);
          }
          tmem_st_wait();
          l *= alpha;
        }
        m_used = m_new;
      }
      }
      const float neg = m_used == -INFINITY ? 0.f : -m_used;
      float2 rs[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
      uint32_t pk[HC / 2];
      const float2 sc2 = make_float2(sc, sc), neg2 = make_float2(neg, neg);
#pragma unroll
      for (int i = 0; i < HC; i += 2) {
        const float2 x = ffma2(make_float2(s[i], s[i + 1]), sc2, neg2);
        float2 e;
        if (((i >> 1) & 3) >= 4 - JENGA_PF_EMU2)
          e = exp2_fma2(x);
        else
          e = make_float2(jenga_dev::fast_exp2(x.x), jenga_dev::fast_exp2(x.y));
        rs[(i >> 1) & 3] = fadd2(rs[(i >> 1) & 3], e);
        pk[i / 2] = pack2<T>(e.x, e.y);
      }
      // P (bf16 pairs) over the first 32 of this warp's own 64 S columns: the other
      // warp of the lane quarter may still be reading its half of S (SPLITO: no per-tile sync)
      tmem_st32u(s_addr + hf * HC, pk);
      {
        const float2 t = fadd2(fadd2(rs[0], rs[1]), fadd2(rs[2], rs[3]));
        l += t.x + t.y;
      }
      tmem_st_wait();
      if ((warp & 3) == JENGA_PF_TRACE_Q && lane == 0 && rank == 0) PF_TRACE(6 + 6 * hf, gg);
      // zero this CTA's V columns of keys outside the pair's range; the issuer waited
      // for this tile's V before S(j), so s_full(j) implies it has landed
      const int ktok0 = (tile_lo + j) * KT;
      const bool boundary = ktok0 < key_lo || ktok0 + KT - 1 > key_hi;
      if (boundary) {
        // SPLITO: each half zeroes the V rows its own PV reads (it hands off alone)
        uint8_t* vs = vring + (gg % NSV) * V_BYTES;
        constexpr int ZR = SPLITO ? HC : KT;   // V rows zeroed by this group of threads
        const int zr0 = SPLITO ? hf * HC : 0;
        for (int idx = SPLITO ? r : static_cast<int>(threadIdx.x); idx < ZR * VB; idx += (SPLITO ? kRows : SW * 32)) {
          const int vrow = zr0 + idx % ZR, chunk = idx / ZR;
          const int key = ktok0 + vrow;
          if (key >= key_lo && key <= key_hi) continue;
          uint4* line = reinterpret_cast<uint4*>(vs + (vrow / kTile) * V_PIECE + chunk * kTile * 128 +
                                                 (vrow % kTile) * 128);
#pragma unroll
          for (int c = 0; c < 8; ++c) line[c] = make_uint4(0, 0, 0, 0);
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      }
      tc_fence_before();
      __syncwarp();
      if ((warp & 3) == JENGA_PF_TRACE_Q && lane == 0 && rank == 0) PF_TRACE(7 + 6 * hf, gg);
      if (lane == 0) {
        const uint32_t pf = p_full0 + 8u * (sb * NPH + (SPLITO ? hf : 0));
        if (boundary)
          arrive_cta0_release_ool(pf);
        else
          arrive_cta0(pf);
      }
    }
    if (ntiles > 0) {
      const int gl = g0 + ntiles - 1;  // the unit's last tile
#pragma unroll
      for (int hh = 0; hh < NPH; ++hh)
        jenga_dev::mbar_wait(&p_empty[(gl % NSB) * NPH + hh], (gl / NSB) & 1);
    }
    if (warp == 0 && lane == 0 && rank == 0) PF_TRACE(8, nus);
    tc_fence_after();
    // merge the halves: row sum (and, SPLITO, the two accumulators' scales)
    float a_own = 1.f, a_oth = 1.f;
    {
      float* rd = red + (ntiles & 1) * 2 * kRows;  // the parity the last tile's exchange did not use
      float* rm = red + ((ntiles & 1) ^ 1) * 2 * kRows;
      rd[hf * kRows + r] = l;
      if (SPLITO) rm[hf * kRows + r] = m_used;
      asm volatile("bar.sync %0, %1;\n" ::"r"(pair_bar), "n"(64) : "memory");
      const float l_oth = rd[(hf ^ 1) * kRows + r];
      if (SPLITO) {
        const float m_oth = rm[(hf ^ 1) * kRows + r];
        const float m = fmaxf(m_used, m_oth);
        a_own = m_used == -INFINITY ? 0.f : jenga_dev::fast_exp2(m_used - m);
        a_oth = m_oth == -INFINITY ? 0.f : jenga_dev::fast_exp2(m_oth - m);
      }
      l = l * a_own + l_oth * a_oth;
      asm volatile("bar.sync %0, %1;\n" ::"r"(pair_bar), "n"(64) : "memory");  // slots reusable by the next unit
    }
    if (warp == 0 && lane == 0 && rank == 0) PF_TRACE(9, nus);
    const float inv = l > 0.f ? 1.f / l : 0.f;
    const float a0 = (hf == 0 ? a_own : a_oth) * inv, a1 = (hf == 0 ? a_oth : a_own) * inv;
    T* outp = static_cast<T*>(p.out) + (static_cast<int64_t>(p.cu_q[x.b] + tok) * p.hq + x.h * G + r % G) * D;
    // Output in 32-column steps.  Each warp stages its 32 rows' 64-byte pieces in its
    // own 2 KiB of shared memory (XOR-swizzled, conflict-free both ways) and reads them
    // back transposed, four lanes per row, so every store instruction writes 8 rows x
    // 64 contiguous bytes -- 8 L2 lines instead of 32 (rows are (token, head) pairs
    // 256-512 B apart in out; the per-thread row stores and a TMA-store staging with
    // CTA-wide barriers both left the epilogue at ~6k cycles).  O is handed back to the
    // MMA issuer (o_free) after each warp's last TMEM load.
    uint8_t* wst = ostage + warp * 2048;
    const int64_t row0 = static_cast<int64_t>(p.cu_q[x.b] + t0) * p.hq + x.h * G;  // out row of r = 0
    constexpr int OSTEPS = D / 2 / 32;
#pragma unroll 1
    for (int it = 0; it < OSTEPS; ++it) {
      const int c = hf * (D / 2) + it * 32;
      float v[32];
      if (ntiles > 0) {
        if constexpr (SPLITO) {
          float w[32];
          tmem_ld32x2(tmem + lane_addr + c, tmem + lane_addr + D + c, v, w);
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = v[i] * a0 + w[i] * a1;
        } else {
          tmem_ld32(tmem + lane_addr + c, v);
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] *= inv;
        }
        if (it == OSTEPS - 1) {  // O read out: the next unit's first PV may overwrite it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) arrive_cta0(o_free0);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = 0.f;
      }
      // stage: row `lane` of this warp, piece q at slot (lane & 1) * 4 + (q ^ ((lane >> 1) & 3))
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<uint4*>(wst + lane * 64 + ((q ^ ((lane >> 1) & 3)) << 4)) =
            make_uint4(pack2<T>(v[8 * q], v[8 * q + 1]), pack2<T>(v[8 * q + 2], v[8 * q + 3]),
                       pack2<T>(v[8 * q + 4], v[8 * q + 5]), pack2<T>(v[8 * q + 6], v[8 * q + 7]));
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int rr = (lane >> 2) + 8 * k, q = lane & 3;  // warp-local row, piece
        const uint4 d = *reinterpret_cast<const uint4*>(wst + rr * 64 + ((q ^ ((rr >> 1) & 3)) << 4));
        const int rw = (warp & 3) * 32 + rr;  // CTA row
        if (t0 + rw / G < x.c_len) {
          T* dst = static_cast<T*>(p.out) + (row0 + static_cast<int64_t>(rw / G) * p.hq + rw % G) * D + c + q * 8;
          *reinterpret_cast<uint4*>(dst) = d;
        }
      }
      __syncwarp();
    }
    if (warp == 0 && lane == 0 && rank == 0) PF_TRACE(1, nus);
    ++nus;
    g0 += ntiles;
    }
  }
  if (warp == 0 && lane == 0) PF_TRACE(14, 0);  // softmax epilogue done (trace variant)
  tc_fence_before();
  cluster_sync();  // the peer's last remote arrivals and MMAs are done
  if (warp == MW) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(TMEM_COLS));
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

// K as [half][chunk][8 rows] 4-D boxes (one per 16-key page piece) and V as
// [chunk][16 rows] 3-D boxes of `v_chunks` 64-column chunks, over the arena
// viewed as [chunk][row][64 columns] (dim1 steps rows, dim2 steps chunks at 128 B).
int encode_kv_maps(const Prefill5Params& prm, int dtype, int D, int v_chunks, CUtensorMap* k_map,
                   CUtensorMap* v_map) {
  auto fn = encode_fn();
  if (fn == nullptr) return jenga_dev::set_error(JENGA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  uint64_t bytes = 0;
  if (!jenga_dev::arena_extent(prm.arena, &bytes))
    return jenga_dev::set_error(JENGA_ERR_ARG, "jenga_paged_prefill: arena_base must come from jenga_arena_create");
  const CUtensorMapDataType dt =
      dtype == JENGA_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  const cuuint32_t nbox = static_cast<cuuint32_t>(D / kBoxCols);
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(kBoxCols), bytes / (D * 2), nbox};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(D) * 2, 128};
  cuuint32_t es[4] = {1, 1, 1, 1};
  cuuint32_t vbox[3] = {kBoxCols, kTile, static_cast<cuuint32_t>(v_chunks)};
  if (fn(v_map, dt, 3, const_cast<uint8_t*>(prm.arena), dims, strides, vbox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS)
    return jenga_dev::set_error(JENGA_ERR_CUDA, "prefill: V tensor map encode failed");
  cuuint64_t kdims[4] = {static_cast<cuuint64_t>(kBoxCols), bytes / (D * 2), nbox, 2};
  cuuint64_t kstrides[3] = {static_cast<cuuint64_t>(D) * 2, 128, static_cast<cuuint64_t>(D) * 2 * 8};
  cuuint32_t kbox[4] = {kBoxCols, 8, nbox, 2};
  if (fn(k_map, dt, 4, const_cast<uint8_t*>(prm.arena), kdims, kstrides, kbox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS)
    return jenga_dev::set_error(JENGA_ERR_CUDA, "prefill: K tensor map encode failed");
  return JENGA_OK;
}

template <typename T, int D, int G, int KT, int NS>
int launch_tc5(const Prefill5Params& prm, int dtype, cudaStream_t s, int batch) {
  constexpr int NBOX = D / kBoxCols;
  const int smem = NS * 2 * NBOX * KT * 128 + (1 + 2 * NS + 6) * 8 + 16 + 1024;
  CUtensorMap k_map, v_map;
  if (int rc = encode_kv_maps(prm, dtype, D, NBOX, &k_map, &v_map)) return rc;
  auto kern = paged_prefill_tc5_kernel<T, D, G, KT, NS>;
  static std::atomic<uint64_t> configured{0};
  if (int rc = configure_smem(kern, smem, configured)) return rc;
  dim3 grid(prm.q_blocks, prm.hkv, batch);
  kern<<<grid, kT5Threads, smem, s>>>(prm, k_map, v_map);
  return jenga_dev::check_launch("paged_prefill_tc5_kernel");
}

template <typename T, int D, int G, int NSK, int NSV>
int launch_tc5_wide(const Prefill5Params& prm, int dtype, cudaStream_t s, int batch, int total_tokens) {
  constexpr int NBOX = D / kBoxCols;
  constexpr int K_BYTES = (64 / 8) * NBOX * 8 * 128, V_BYTES = 8 * (NBOX / 2) * kTile * 128;
  constexpr int Q_BYTES = NBOX * kRows * 128;
  const int smem = Q_BYTES + NSK * K_BYTES + NSV * V_BYTES + kRows * 128 + 2 * 2 * kRows * 4 +
                   (1 + 2 * NSK + 2 * NSV + 12) * 8 + 16 + 1024;  // 12 >= NSB * (1 + 2 * NPH) + 2
  CUtensorMap k_map, v_map, q_map;
  if (int rc = encode_kv_maps(prm, dtype, D, NBOX / 2, &k_map, &v_map)) return rc;
  {  // q [T][Hq][D] as [chunk][token][head][64 columns]
    const CUtensorMapDataType dt =
        dtype == JENGA_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    cuuint64_t dims[4] = {static_cast<cuuint64_t>(kBoxCols), static_cast<cuuint64_t>(prm.hq),
                          static_cast<cuuint64_t>(total_tokens), static_cast<cuuint64_t>(NBOX)};
    cuuint64_t strides[3] = {static_cast<cuuint64_t>(D) * 2, static_cast<cuuint64_t>(prm.hq) * D * 2, 128};
    cuuint32_t box[4] = {kBoxCols, G, kRows / G, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (encode_fn()(&q_map, dt, 4, const_cast<void*>(prm.q), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return jenga_dev::set_error(JENGA_ERR_CUDA,
                                  "prefill: q tensor map encode failed (q must be 16-byte aligned)");
  }
  auto kern = paged_prefill_tc5_wide_kernel<T, D, G, NSK, NSV>;
  static std::atomic<uint64_t> configured{0};
  if (int rc = configure_smem(kern, smem, configured)) return rc;
  // Persistent: one CTA pair per two SMs (fewer when there are fewer work units), so a
  // unit's prologue (Q, first K/V, first S) overlaps the previous unit's tail.  Against
  // one CTA pair per unit (hardware-scheduled): 256-token chunks at 2k +18%, D=128
  // +2..+11%, SWA +4%, D=256 full 2k chunks at 8k -1.7% (profiles/r02_prefill_experiments.md).
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return jenga_dev::set_error(JENGA_ERR_CUDA, "jenga_paged_prefill: cannot query the SM count");
  const int64_t units = static_cast<int64_t>((prm.q_blocks + 1) / 2) * prm.hkv * batch;
  const int64_t clusters = std::min<int64_t>(units, std::max(sms / 2, 1));
  kern<<<dim3(static_cast<unsigned>(2 * clusters)), (2 * kSoftWarps + 2) * 32, smem, s>>>(prm, k_map, v_map, q_map);
  return jenga_dev::check_launch("paged_prefill_tc5_wide_kernel");
}

template <typename T, int D, int NSK, int NSV>
int dispatch_wide(int G, const Prefill5Params& prm, int dtype, cudaStream_t s, int batch, int total_tokens) {
  switch (G) {
    case 1: return launch_tc5_wide<T, D, 1, NSK, NSV>(prm, dtype, s, batch, total_tokens);
    case 2: return launch_tc5_wide<T, D, 2, NSK, NSV>(prm, dtype, s, batch, total_tokens);
    case 4: return launch_tc5_wide<T, D, 4, NSK, NSV>(prm, dtype, s, batch, total_tokens);
    case 8: return launch_tc5_wide<T, D, 8, NSK, NSV>(prm, dtype, s, batch, total_tokens);
  }
  return JENGA_ERR_UNSUPPORTED;
}

#ifndef JENGA_PF_NSK256
#define JENGA_PF_NSK256 2
#endif
#ifndef JENGA_PF_NSV256
#define JENGA_PF_NSV256 2
#endif

template <typename T, int D, int NS>
int dispatch_g(int G, const Prefill5Params& prm, int dtype, cudaStream_t s, int batch) {
  switch (G) {
    case 1: return launch_tc5<T, D, 1, 64, NS>(prm, dtype, s, batch);
    case 2: return launch_tc5<T, D, 2, 64, NS>(prm, dtype, s, batch);
    case 4: return launch_tc5<T, D, 4, 64, NS>(prm, dtype, s, batch);
    case 8: return launch_tc5<T, D, 8, 64, NS>(prm, dtype, s, batch);
  }
  return JENGA_ERR_UNSUPPORTED;
}

// Kernel per head_dim: persistent CTA pairs (cta_group::2, M = 256, 128-key tiles) at
// 256 and 128 -- each SM streams half of every K/V tile (K ring 2 / V ring 2 stages at
// 256, 5 / 5 at 128); one CTA per query block with 64-key tiles at 64, whose single
// 64-column chunk is too narrow to split V across a pair.
template <typename T>
int dispatch_d(int D, int G, const Prefill5Params& prm, int dtype, cudaStream_t s, int batch, int total_tokens) {
  switch (D) {
    case 256: return dispatch_wide<T, 256, JENGA_PF_NSK256, JENGA_PF_NSV256>(G, prm, dtype, s, batch, total_tokens);
    case 128: return dispatch_wide<T, 128, 5, 5>(G, prm, dtype, s, batch, total_tokens);
    case 64: return dispatch_g<T, 64, 6>(G, prm, dtype, s, batch);
  }
  return jenga_dev::set_error(JENGA_ERR_UNSUPPORTED, "jenga_paged_prefill: head_dim must be 64, 128 or 256");
}

}  // namespace

#ifdef JENGA_PF_TRACE
JENGA_EXPORT int jenga_debug_prefill_trace(long long* dst) {
  return cudaMemcpyFromSymbol(dst, g_pf_trace, sizeof(g_pf_trace)) == cudaSuccess ? 0 : -1;
}
#endif

// Chunked-prefill paged attention (the reference's
// prefill_some stores a chunk of positions per step, simulator.cpp:504-547).
// Request b contributes C_b query tokens — its newest ordinals, 0-based
// positions n_b - C_b .. n_b - 1 — whose K/V were already scattered into the
// arena by reshape_and_cache.  Query position i attends key j iff j <= i
// (causal), additionally j + W > i for sliding windows (needs_token at length
// i + 1, layer_policies.cpp:105-120); cross attention attends all n_b image keys.
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
  const int G = num_q_heads / num_kv_heads;
  if (G != 1 && G != 2 && G != 4 && G != 8)
    return set_error(JENGA_ERR_UNSUPPORTED, "jenga_paged_prefill: query heads per kv head must be 1, 2, 4 or 8");
  if (batch == 0 || total_tokens == 0) return JENGA_OK;
  Prefill5Params prm{};
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
  prm.q_blocks = (max_chunk + kRows / G - 1) / (kRows / G);  // 128 (token, query head) rows per block
  if (softcap > 0.f) {
    prm.qscale = scale;
    prm.cap_log2 = softcap * kLog2e;
    prm.inv_cap = 1.f / softcap;
  } else {
    prm.qscale = scale * kLog2e;
  }
  prm.q = q;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  prm.batch = batch;
  const int rc = dtype == JENGA_BF16 ? dispatch_d<__nv_bfloat16>(head_dim, G, prm, dtype, s, batch, total_tokens)
                                     : dispatch_d<__half>(head_dim, G, prm, dtype, s, batch, total_tokens);
  if (rc == JENGA_OK) note_launch(s, kLaunchSerializing);
  return rc;
}
