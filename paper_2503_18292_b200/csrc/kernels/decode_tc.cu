// Paged decode attention, tensor-core variant (bf16 / fp16 KV, page sizes that
// are multiples of 16 tokens).  Same contract, work split and epilogue as the
// CUDA-core kernel in decode.cu; the differences are the data movement and
// the math:
//
//  * K/V tiles move with TMA tensor loads (cp.async.bulk.tensor -> UTMALDG) over
//    the whole arena viewed as rows of D elements, row = one token of one
//    (page, layer, K|V, head): row index = (start_offset + global*page_stride +
//    ((2h + kv)*tpp + off)*D*e) / (D*e).  One head per CTA (default): ONE 4-D
//    box {64 cols, 16 rows, D/64 chunks, K|V} per 16-token tile; several heads:
//    64 x 16 2-D boxes.  Tiles land with the 128-byte swizzle, so ldmatrix is
//    conflict-free.
//  * Fused append (jenga_paged_decode_append): the warp whose tile holds the
//    newest token writes that token's K/V to its slot and into the staged tile.
//  * One CTA serves HG KV heads of a request: a pipeline stage holds the same
//    16-token tile of all HG heads, which are adjacent in the head-major
//    page-layer slice ([Hkv][K|V][tpp][D]), so each stage is one contiguous
//    HG x 16 KiB run of K and V.  Long contiguous runs keep DRAM row locality high under the
//    page-layer layout, where one layer is only a 128 KiB slice of every
//    2.75 MiB page (measured: the busiest DRAM channels idle ~18% with 8 KiB
//    runs).
//  * S^T = K . Q^T and O^T += V^T . P^T run on the tensor cores with
//    mma.sync m16n8k16 (fp32 accumulate): tokens on M (16 per tile), the G
//    query heads of one KV head on N (padded to 8), head_dim as K for QK and
//    as M for PV.  P is re-laid from the S accumulator into the PV operand
//    with movmatrix (8x8 transpose), never touching shared memory.
//  * online softmax in fp32 registers: per-head tile max via 3 shuffles,
//    lazy rescale of the O accumulators only when a max moved.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <map>
#include <mutex>
#include <tuple>

#include "decode_common.cuh"

namespace jenga_dev {
bool arena_extent(const void* base, uint64_t* bytes);
}

namespace {

using namespace jenga_decode;

constexpr int kBoxCols = 64;            // elements per swizzle row (128 B)
constexpr int kBoxBytes = kTile * 128;  // one 64 x 16 box

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

__device__ __forceinline__ uint32_t movm_trans(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;\n" : "=r"(y) : "r"(x));
  return y;
}

template <typename T>
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%0, %1, %2, %3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  } else {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%0, %1, %2, %3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
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

// Shared-memory budget per CTA for the stage ring: 1 CTA/SM when a CTA owns
// 4 heads, 2 when it owns 2, 3 when it owns 1 (~192 KiB in flight per SM).
template <int HG>
constexpr int ring_budget() {
  return HG >= 4 ? 196608 : (HG == 2 ? 98304 : 65536);
}

// Ring depth: a multiple of the rounds (kConsumerWarps / HG) so each slot is
// always consumed by the same warps — a warp that skipped a use of a slot
// could otherwise wait on a parity two phases ahead and pass early.
template <int D, int HG>
constexpr int stages() {
  constexpr int rounds = kConsumerWarps / HG;
  constexpr int stage = 2 * HG * kTile * D * 2;
  constexpr int ns = (ring_budget<HG>() / stage) / rounds * rounds;
  return ns < rounds ? rounds : (ns > 12 ? 12 : ns);
}

// ------------------------------------------------------------ per-warp math
// One consumer warp's running state for one KV head: Q^T fragments (the B
// operand of S^T = K Q^T), the O^T accumulators and the online-softmax
// statistics of the two query heads this lane's fragments hold.
template <int D>
struct HeadState {
  static constexpr int K = D / 16;
  uint32_t bq[K][2];
  float o[K][4];
  float m0, m1, l0, l1;  // query heads 2*c4, 2*c4+1
};

template <typename T, int D, int G>
__device__ __forceinline__ void head_begin(HeadState<D>& st, const DecodeParams& p, int b, int h, int lane) {
  const int r4 = lane >> 2, c4 = lane & 3;
  const uint32_t* qrow = reinterpret_cast<const uint32_t*>(static_cast<const T*>(p.q) +
                                                           (static_cast<int64_t>(b) * p.hq + h * G + r4) * D);
#pragma unroll
  for (int k = 0; k < HeadState<D>::K; ++k) {
    st.bq[k][0] = r4 < G ? __ldg(qrow + (16 * k + 2 * c4) / 2) : 0u;
    st.bq[k][1] = r4 < G ? __ldg(qrow + (16 * k + 8 + 2 * c4) / 2) : 0u;
    st.o[k][0] = st.o[k][1] = st.o[k][2] = st.o[k][3] = 0.f;
  }
  st.m0 = st.m1 = -INFINITY;
  st.l0 = st.l1 = 0.f;
}

// One 16-token tile of one head: ks/vs are the head's K and V tiles (NBOX
// swizzled 64x16 boxes each) in shared memory.
template <typename T, int D>
__device__ __forceinline__ void head_tile(HeadState<D>& st, uint8_t* ks, uint8_t* vs, int tok0, int lo, int n,
                                          const DecodeParams& p, int lane) {
  constexpr int KS = HeadState<D>::K;
  constexpr int NBOX = D / kBoxCols;
  const int r4 = lane >> 2;
  const int k_row = (lane & 7) + ((lane >> 3) & 1) * 8;  // K tile row fed by this lane
  const int k_half = lane >> 4;                           // which 8-wide D half
  const int v_tok = (lane & 7) + (lane >> 4) * 8;         // V tile token row fed by this lane
  const int v_half = (lane >> 3) & 1;
  const int x7 = lane & 7;                                // == row & 7 for both
  const uint32_t ks_u = jenga_dev::smem_u32(ks), vs_u = jenga_dev::smem_u32(vs);

  // ---- S^T = K . Q^T  (16 tokens x 8 heads, fp32)
  float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int k = 0; k < KS; ++k) {
    const int chunk = 2 * k + k_half;
    uint32_t a[4];
    ldsm_x4(a, ks_u + (chunk >> 3) * kBoxBytes + k_row * 128 + (((chunk & 7) ^ x7) << 4));
    mma16816<T>(s, a, st.bq[k][0], st.bq[k][1]);
  }
  // ---- scale, soft-cap, mask (needs_token), online softmax
  const int ta = tok0 + r4, tb = ta + 8;
  const bool va = ta >= lo && ta < n, vb = tb >= lo && tb < n;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float x = s[i] * p.qscale;
    if (p.cap_log2 > 0.f) x = p.cap_log2 * tanhf(x * p.inv_cap);
    s[i] = x;
  }
  s[0] = va ? s[0] : -INFINITY;
  s[1] = va ? s[1] : -INFINITY;
  s[2] = vb ? s[2] : -INFINITY;
  s[3] = vb ? s[3] : -INFINITY;
  float t0 = fmaxf(s[0], s[2]), t1 = fmaxf(s[1], s[3]);
#pragma unroll
  for (int off = 4; off < 32; off <<= 1) {
    t0 = fmaxf(t0, __shfl_xor_sync(0xffffffffu, t0, off));
    t1 = fmaxf(t1, __shfl_xor_sync(0xffffffffu, t1, off));
  }
  const float n0 = fmaxf(st.m0, t0), n1 = fmaxf(st.m1, t1);
  const float a0 = n0 == -INFINITY ? 1.f : jenga_dev::fast_exp2(st.m0 - n0);
  const float a1 = n1 == -INFINITY ? 1.f : jenga_dev::fast_exp2(st.m1 - n1);
  st.m0 = n0;
  st.m1 = n1;
  const float p0 = va ? jenga_dev::fast_exp2(s[0] - n0) : 0.f;
  const float p1 = va ? jenga_dev::fast_exp2(s[1] - n1) : 0.f;
  const float p2 = vb ? jenga_dev::fast_exp2(s[2] - n0) : 0.f;
  const float p3 = vb ? jenga_dev::fast_exp2(s[3] - n1) : 0.f;
  st.l0 = st.l0 * a0 + p0 + p2;
  st.l1 = st.l1 * a1 + p1 + p3;
  if (__any_sync(0xffffffffu, a0 != 1.f || a1 != 1.f)) {
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      st.o[k][0] *= a0;
      st.o[k][1] *= a1;
      st.o[k][2] *= a0;
      st.o[k][3] *= a1;
    }
  }
  // P^T as the B operand of O^T += V^T P^T (k = tokens, n = heads)
  const uint32_t pb0 = movm_trans(pack2<T>(p0, p1));
  const uint32_t pb1 = movm_trans(pack2<T>(p2, p3));
  // masked rows of a boundary tile may hold stale / non-finite bytes:
  // zero this head's rows so 0 * V cannot produce NaN inside the MMA.
  if (tok0 < lo || tok0 + kTile > n) {
    for (int r = 0; r < kTile; ++r) {
      const int t = tok0 + r;
      if (t >= lo && t < n) continue;
      for (int c = lane; c < NBOX * 8; c += 32)
        *reinterpret_cast<uint4*>(vs + (c >> 3) * kBoxBytes + r * 128 + ((c & 7) << 4)) = make_uint4(0, 0, 0, 0);
    }
    // order these generic-proxy writes before the TMA refill of this stage
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncwarp();
  }
  // ---- O^T += V^T . P^T  (D x 8 heads)
#pragma unroll
  for (int k = 0; k < KS; ++k) {
    const int chunk = 2 * k + v_half;
    uint32_t a[4];
    ldsm_x4_trans(a, vs_u + (chunk >> 3) * kBoxBytes + v_tok * 128 + (((chunk & 7) ^ x7) << 4));
    mma16816<T>(st.o[k], a, pb0, pb1);
  }
}

// Fused append: the warp whose tile holds the newest token (tile row `row`)
// writes that token's K and V rows of its head into the arena slot AND into
// the staged tile (the TMA brought the slot's previous bytes), so the
// reshape_and_cache launch and its dependency disappear from the step.
// 16-byte unit u of 64-column chunk c sits at c*kBoxBytes + row*128 + ((u ^ (row & 7)) << 4).
template <typename T, int D>
__device__ __forceinline__ void patch_newest(const DecodeParams& p, uint8_t* ks, uint8_t* vs, int b, int h, int row,
                                             int lane) {
  constexpr int UNITS = D * 2 / 16;  // 16-byte units per row
  const int64_t slot = p.new_slots[b];
  if (slot < 0) return;
  const int64_t page = slot / p.tpp, off = slot - page * p.tpp;
  uint8_t* dst = const_cast<uint8_t*>(p.arena) + p.start_offset + page * p.page_stride +
                 (static_cast<int64_t>(2 * h) * p.tpp + off) * (D * 2);
  const int64_t src = (static_cast<int64_t>(b) * p.hkv + h) * (D * 2);
  for (int i = lane; i < UNITS; i += 32) {
    const int c = i >> 3, u = i & 7;
    const uint4 kx = jenga_dev::ld_nc_v4(static_cast<const uint8_t*>(p.k_new) + src + i * 16);
    const uint4 vx = jenga_dev::ld_nc_v4(static_cast<const uint8_t*>(p.v_new) + src + i * 16);
    const int sm = c * kBoxBytes + row * 128 + ((u ^ (row & 7)) << 4);
    *reinterpret_cast<uint4*>(ks + sm) = kx;
    *reinterpret_cast<uint4*>(vs + sm) = vx;
    jenga_dev::st_v4(dst + i * 16, kx);
    jenga_dev::st_v4(dst + static_cast<int64_t>(p.tpp) * (D * 2) + i * 16, vx);
  }
  // generic-proxy writes into a TMA stage: order them before its next refill
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncwarp();
}

// Reduce the per-lane l partials and write this warp's unnormalised state to
// the merge area s_acc[warp][G][D] / s_ml[warp][G][2].
template <int D, int G>
__device__ __forceinline__ void head_store(HeadState<D>& st, float* s_acc, float* s_ml, int warp, int lane) {
#pragma unroll
  for (int off = 4; off < 32; off <<= 1) {
    st.l0 += __shfl_xor_sync(0xffffffffu, st.l0, off);
    st.l1 += __shfl_xor_sync(0xffffffffu, st.l1, off);
  }
  const int r4 = lane >> 2, c4 = lane & 3;
  const int q0 = 2 * c4, q1 = q0 + 1;
#pragma unroll
  for (int k = 0; k < HeadState<D>::K; ++k) {
    const int d = 16 * k + r4;
    if (q0 < G) {
      s_acc[(warp * G + q0) * D + d] = st.o[k][0];
      s_acc[(warp * G + q0) * D + d + 8] = st.o[k][2];
    }
    if (q1 < G) {
      s_acc[(warp * G + q1) * D + d] = st.o[k][1];
      s_acc[(warp * G + q1) * D + d + 8] = st.o[k][3];
    }
  }
  if (r4 == 0) {
    if (q0 < G) {
      s_ml[(warp * G + q0) * 2] = st.m0;
      s_ml[(warp * G + q0) * 2 + 1] = st.l0;
    }
    if (q1 < G) {
      s_ml[(warp * G + q1) * 2] = st.m1;
      s_ml[(warp * G + q1) * 2 + 1] = st.l1;
    }
  }
}

// TMA loads of one tile (16 tokens) of HG heads into a stage: K of heads
// h0..h0+HG-1, then their V (head-major slice: head h's K rows at 2*h*tpp,
// its V rows tpp later).
template <int D, int HG>
__device__ __forceinline__ void load_stage(const CUtensorMap* tmap, uint8_t* stage, uint64_t* bar, int32_t row,
                                           int tpp, int v_rows, uint64_t policy, bool kv_box) {
  constexpr int NBOX = D / kBoxCols;
  constexpr int TILE_BYTES = NBOX * kBoxBytes;
  jenga_dev::mbar_arrive_expect_tx(bar, 2 * HG * TILE_BYTES);
  if (HG == 1 && kv_box) {
    // one 4-D box = the head's K and V tiles of the page: {64 cols, 16 rows, NBOX
    // chunks, K|V}, landing [K|V][chunk][16 rows][128 B] — the ldmatrix layout
    jenga_dev::tma_load_4d_row(stage, tmap, row, bar, policy);
    return;
  }
#pragma unroll
  for (int hl = 0; hl < HG; ++hl)
#pragma unroll
    for (int bx = 0; bx < NBOX; ++bx)
      jenga_dev::tma_load_2d(stage + hl * TILE_BYTES + bx * kBoxBytes, tmap, bx * kBoxCols, row + hl * 2 * tpp,
                             bar, policy);
#pragma unroll
  for (int hl = 0; hl < HG; ++hl)
#pragma unroll
    for (int bx = 0; bx < NBOX; ++bx)
      jenga_dev::tma_load_2d(stage + (HG + hl) * TILE_BYTES + bx * kBoxBytes, tmap, bx * kBoxCols,
                             row + v_rows + hl * 2 * tpp, bar, policy);
}

// Arena row of the first K row of (page of token tok0, head h0).
__device__ __forceinline__ int32_t tile_row(const DecodeParams& p, const int32_t* table, int h0, int tok0,
                                            int64_t row_bytes) {
  const int64_t base_row = static_cast<int64_t>(p.start_offset) / row_bytes + static_cast<int64_t>(h0) * 2 * p.tpp;
  const int64_t page_rows = static_cast<int64_t>(p.page_stride) / row_bytes;
  return static_cast<int32_t>(base_row + static_cast<int64_t>(table[tok0 / p.tpp]) * page_rows + tok0 % p.tpp);
}

// ------------------------------------------------------------ grid kernel
// One CTA per (KV-head group, request, split).
template <typename T, int D, int G, int HG, int NS>
__global__ void __launch_bounds__(kThreads, HG >= 4 ? 1 : (HG == 2 ? 2 : 3))
    paged_decode_tc_kernel(const DecodeParams p, const __grid_constant__ CUtensorMap tmap) {
  static_assert(D % kBoxCols == 0, "head_dim must be a multiple of 64");
  static_assert(G <= 8, "at most 8 query heads per KV head (N = 8)");
  static_assert(kConsumerWarps % HG == 0, "heads per CTA must divide the consumer warps");
  constexpr int TILE_BYTES = (D / kBoxCols) * kBoxBytes;  // 16 tokens x D x 2 B, one head
  constexpr int STAGE_BYTES = 2 * HG * TILE_BYTES;
  constexpr int ROUNDS = kConsumerWarps / HG;            // warps per head
  constexpr int MERGE_BYTES = (kConsumerWarps * G * D + kConsumerWarps * G * 2) * 4;
  constexpr int RING = NS * STAGE_BYTES;
  constexpr int BAR_OFFSET = RING > MERGE_BYTES ? RING : MERGE_BYTES;

  extern __shared__ uint8_t smem_raw[];
  // 128-byte swizzled TMA destinations want 1024-byte aligned boxes.
  uint8_t* smem = smem_raw + ((1024 - (jenga_dev::smem_u32(smem_raw) & 1023)) & 1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + BAR_OFFSET);
  uint64_t* empty = full + NS;
  int* s_flag = reinterpret_cast<int*>(empty + NS);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int b = grid_request(p);
  const int h0 = blockIdx.x * HG;  // first KV head of this CTA
  const int split = grid_split(p);
  const Work wk = assign_work(p, b, split);
  if (split >= wk.nsplit) return;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      jenga_dev::mbar_init(&full[i], 1);
      jenga_dev::mbar_init(&empty[i], HG);  // every head's warp releases the stage
    }
    jenga_dev::fence_mbar_init();
  }
  __syncthreads();
  // PDL: the next kernel in the stream may become resident now.  Block
  // tables / seq_lens come from a non-PDL kernel and are complete; q, the
  // newest token's K/V (reshape_and_cache) and the reused workspace are only
  // touched after pdl_wait().
  jenga_dev::pdl_launch_dependents();

  const int32_t* table = p.table + static_cast<int64_t>(b) * p.max_blocks;

  if (warp == kConsumerWarps) {
    if (lane == 0) {  // producer: one elected lane
      jenga_dev::prefetch_tmap(&tmap);
      const uint64_t policy = jenga_dev::l2_policy_evict_first();
      const int v_rows = p.tpp;
      bool waited = false;
      // the next tile's arena row is read one iteration ahead, so the block-table
      // load is off the empty-slot -> refill path
      int32_t row = wk.t_count > 0 ? tile_row(p, table, h0, wk.t_begin * kTile, D * 2) : 0;
      for (int it = 0; it < wk.t_count; ++it) {
        const int st = it % NS;
        const int tok0 = (wk.t_begin + it) * kTile;
        const int32_t next = it + 1 < wk.t_count ? tile_row(p, table, h0, tok0 + kTile, D * 2) : 0;
        if (it >= NS) jenga_dev::mbar_wait(&empty[st], ((it / NS) & 1) ^ 1);
        if (!waited && tok0 + kTile >= wk.n && p.k_new == nullptr) {  // the tile holding the newest token
          jenga_dev::pdl_wait();  // (fused append patches that row itself: no wait)
          waited = true;
        }
        load_stage<D, HG>(&tmap, smem + st * STAGE_BYTES, &full[st], row, p.tpp, v_rows, policy, p.kv_box != 0);
        row = next;
      }
    }
    return;
  }

  const int hl = warp % HG;      // local head of this warp
  const int round = warp / HG;   // which of the ROUNDS stage streams
  HeadState<D> hs;
  jenga_dev::pdl_wait();  // q and the workspace belong to the previous kernels until here
  head_begin<T, D, G>(hs, p, b, h0 + hl, lane);
  for (int it = round; it < wk.t_count; it += ROUNDS) {
    const int st = it % NS;
    jenga_dev::mbar_wait(&full[st], (it / NS) & 1);
    uint8_t* stage = smem + st * STAGE_BYTES;
    const int tok0 = (wk.t_begin + it) * kTile;
    if (p.k_new != nullptr && wk.n - 1 >= tok0 && wk.n - 1 < tok0 + kTile)
      patch_newest<T, D>(p, stage + hl * TILE_BYTES, stage + (HG + hl) * TILE_BYTES, b, h0 + hl, wk.n - 1 - tok0, lane);
    head_tile<T, D>(hs, stage + hl * TILE_BYTES, stage + (HG + hl) * TILE_BYTES, tok0, wk.lo, wk.n, p, lane);
    __syncwarp();
    if (lane == 0) jenga_dev::mbar_arrive(&empty[st]);
  }
  consumers_sync();
  float* s_acc = reinterpret_cast<float*>(smem);  // [4][G][D] (the ring is drained)
  float* s_ml = s_acc + kConsumerWarps * G * D;   // [4][G][2]
  head_store<D, G>(hs, s_acc, s_ml, warp, lane);
  merge_epilogue<T, G, D, HG>(p, s_acc, s_ml, s_flag, wk.nsplit, split, b, h0);
}

// ------------------------------------------------------------ persistent kernel
// gridDim.x CTAs (a few per SM) pull work items (request, head group, split)
// from a global atomic queue.  The producer keeps streaming tiles across item
// boundaries, so the TMA ring never drains between items and there is no
// wave-quantisation tail; the consumers merge each item while the next one's
// tiles are already landing.  Items are enumerated request by request from a
// per-CTA prefix over the requests' split counts (needs batch <= kMaxPersistB).
constexpr int kMaxPersistB = 2048;
constexpr int kItemSlots = 4;

struct ItemDesc {
  int b, h0, split, n, lo, nsplit, t_begin, t_count, seq0, stop;
};

template <typename T, int D, int G, int HG, int NS>
__global__ void __launch_bounds__(kThreads, HG >= 4 ? 1 : (HG == 2 ? 2 : 3))
    paged_decode_tc_persistent(const DecodeParams p, const __grid_constant__ CUtensorMap tmap) {
  constexpr int TILE_BYTES = (D / kBoxCols) * kBoxBytes;
  constexpr int STAGE_BYTES = 2 * HG * TILE_BYTES;
  constexpr int ROUNDS = kConsumerWarps / HG;
  constexpr int MERGE_BYTES = (kConsumerWarps * G * D + kConsumerWarps * G * 2) * 4;
  constexpr int RING = NS * STAGE_BYTES;
  static_assert(NS % ROUNDS == 0, "slots must map to fixed consumer warps");

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (jenga_dev::smem_u32(smem_raw) & 1023)) & 1023);
  float* s_acc = reinterpret_cast<float*>(smem + RING);     // separate from the ring:
  float* s_ml = s_acc + kConsumerWarps * G * D;             // the producer keeps filling it
  ItemDesc* items = reinterpret_cast<ItemDesc*>(smem + RING + MERGE_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(items + kItemSlots);
  uint64_t* empty = full + NS;
  uint64_t* item_full = empty + NS;
  uint64_t* item_empty = item_full + kItemSlots;
  int* s_flag = reinterpret_cast<int*>(item_empty + kItemSlots);
  int* s_prefix = s_flag + 4;  // [batch + 1] item prefix over requests

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int groups = p.hkv / HG;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      jenga_dev::mbar_init(&full[i], 1);
      jenga_dev::mbar_init(&empty[i], HG);
    }
    for (int i = 0; i < kItemSlots; ++i) {
      jenga_dev::mbar_init(&item_full[i], 1);
      jenga_dev::mbar_init(&item_empty[i], kConsumerWarps);
    }
    jenga_dev::fence_mbar_init();
  }
  if (warp == 0) {  // items per request -> exclusive prefix (one warp scan)
    const int per = (p.batch + 31) / 32;
    int local = 0;
    for (int i = 0; i < per; ++i) {
      const int bb = lane * per + i;
      if (bb < p.batch) local += assign_work(p, bb, 0).nsplit * groups;
    }
    int incl = local;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += v;
    }
    int run = incl - local;
    for (int i = 0; i < per; ++i) {
      const int bb = lane * per + i;
      if (bb < p.batch) {
        s_prefix[bb] = run;
        run += assign_work(p, bb, 0).nsplit * groups;
      }
    }
    if (lane == 31) s_prefix[p.batch] = incl;
  }
  __syncthreads();
  const int total = s_prefix[p.batch];

  if (warp == kConsumerWarps) {
    if (lane == 0) {  // producer: fetch items, stream their tiles
      jenga_dev::prefetch_tmap(&tmap);
      const uint64_t policy = jenga_dev::l2_policy_evict_first();
      const int v_rows = p.tpp;
      int seq = 0;
      for (int ic = 0;; ++ic) {
        const int j = ic % kItemSlots;
        if (ic >= kItemSlots) jenga_dev::mbar_wait(&item_empty[j], ((ic / kItemSlots) & 1) ^ 1);
        const int item = atomicAdd(&p.work[0], 1);
        ItemDesc d{};
        if (item >= total) {
          d.stop = 1;
          items[j] = d;
          jenga_dev::mbar_arrive(&item_full[j]);
          break;
        }
        int lo_b = 0, hi_b = p.batch - 1;  // last request with prefix <= item
        while (lo_b < hi_b) {
          const int mid = (lo_b + hi_b + 1) >> 1;
          if (s_prefix[mid] <= item) lo_b = mid;
          else hi_b = mid - 1;
        }
        const int r = item - s_prefix[lo_b];
        d.b = lo_b;
        d.split = r / groups;
        d.h0 = (r % groups) * HG;
        const Work wk = assign_work(p, d.b, d.split);
        d.n = wk.n;
        d.lo = wk.lo;
        d.nsplit = wk.nsplit;
        d.t_begin = wk.t_begin;
        d.t_count = wk.t_count;
        d.seq0 = seq;
        items[j] = d;
        jenga_dev::mbar_arrive(&item_full[j]);  // release: the descriptor is visible to its waiters
        const int32_t* table = p.table + static_cast<int64_t>(d.b) * p.max_blocks;
        for (int it = 0; it < d.t_count; ++it, ++seq) {
          const int st = seq % NS;
          if (seq >= NS) jenga_dev::mbar_wait(&empty[st], ((seq / NS) & 1) ^ 1);
          const int tok0 = (d.t_begin + it) * kTile;
          load_stage<D, HG>(&tmap, smem + st * STAGE_BYTES, &full[st], tile_row(p, table, d.h0, tok0, D * 2), p.tpp,
                            v_rows, policy, p.kv_box != 0);
        }
      }
    }
  } else {
    const int hl = warp % HG;
    const int round = warp / HG;
    HeadState<D> hs;
    for (int ic = 0;; ++ic) {
      const int j = ic % kItemSlots;
      jenga_dev::mbar_wait(&item_full[j], (ic / kItemSlots) & 1);
      const ItemDesc d = items[j];
      __syncwarp();
      if (lane == 0) jenga_dev::mbar_arrive(&item_empty[j]);
      if (d.stop) break;
      head_begin<T, D, G>(hs, p, d.b, d.h0 + hl, lane);
      // this warp owns the global tiles seq with seq % ROUNDS == round (NS % ROUNDS == 0,
      // so every use of a slot is consumed by the same warps)
      int it = (round - d.seq0 % ROUNDS + ROUNDS) % ROUNDS;
      for (; it < d.t_count; it += ROUNDS) {
        const int seq = d.seq0 + it;
        const int st = seq % NS;
        jenga_dev::mbar_wait(&full[st], (seq / NS) & 1);
        uint8_t* stage = smem + st * STAGE_BYTES;
        head_tile<T, D>(hs, stage + hl * TILE_BYTES, stage + (HG + hl) * TILE_BYTES, (d.t_begin + it) * kTile, d.lo,
                        d.n, p, lane);
        __syncwarp();
        if (lane == 0) jenga_dev::mbar_arrive(&empty[st]);
      }
      consumers_sync();  // the previous item's merge has finished reading s_acc
      head_store<D, G>(hs, s_acc, s_ml, warp, lane);
      merge_epilogue<T, G, D, HG>(p, s_acc, s_ml, s_flag, d.nsplit, d.split, d.b, d.h0);
    }
  }
  // the last CTA out re-arms the queue for the next launch / graph replay
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&p.work[1], 1) == static_cast<int>(gridDim.x) - 1) {
      p.work[0] = 0;
      p.work[1] = 0;
      __threadfence();
    }
  }
}

// ------------------------------------------------------------ host side
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

// Views of the arena, encoded once per (arena, D, dtype, tpp, kind):
//  * 2-D [rows][D] with 64 x 16 boxes (several heads per CTA);
//  * 4-D {64 cols, rows, D/64 chunks at 128 B, K|V at tpp rows} with one box =
//    a whole head's K and V tile of a page (one head per CTA): 1 TMA op per 16 KiB
//    instead of 2*D/64 (measured on the prefill producer: TMA op count, not bytes,
//    bounded delivery).
int tensor_map(const void* base, int D, int dtype, int tpp, bool kv_box, CUtensorMap* out) {
  static std::mutex mu;
  static std::map<std::tuple<uintptr_t, uint64_t, int, int, int, bool>, CUtensorMap> cache;
  uint64_t bytes = 0;
  if (!jenga_dev::arena_extent(base, &bytes)) return JENGA_ERR_UNSUPPORTED;  // not a jenga arena
  // keyed by the extent too: a new arena may reuse a freed arena's address
  const auto key = std::make_tuple(reinterpret_cast<uintptr_t>(base), bytes, D, dtype, kv_box ? tpp : 0, kv_box);
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return JENGA_OK;
  }
  auto fn = encode_fn();
  if (fn == nullptr) return jenga_dev::set_error(JENGA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const uint64_t row_bytes = static_cast<uint64_t>(D) * 2;
  const CUtensorMapDataType dt =
      dtype == JENGA_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  CUtensorMap m;
  CUresult r;
  if (kv_box) {
    cuuint64_t dims[4] = {static_cast<cuuint64_t>(kBoxCols), bytes / row_bytes, static_cast<cuuint64_t>(D / kBoxCols),
                          2};
    cuuint64_t strides[3] = {row_bytes, 128, static_cast<cuuint64_t>(tpp) * row_bytes};
    cuuint32_t box[4] = {static_cast<cuuint32_t>(kBoxCols), static_cast<cuuint32_t>(kTile),
                         static_cast<cuuint32_t>(D / kBoxCols), 2};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    r = fn(&m, dt, 4, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(D), bytes / row_bytes};
    cuuint64_t strides[1] = {row_bytes};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(kBoxCols), static_cast<cuuint32_t>(kTile)};
    cuuint32_t estr[2] = {1, 1};
    r = fn(&m, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS)
    return jenga_dev::set_error(JENGA_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
  cache[key] = m;
  *out = m;
  return JENGA_OK;
}

// Persistent scheduling only with JENGA_DECODE_PERSISTENT=1: measured slower
// than three grid CTAs per SM on the bench shapes (profiles/r01_sweeps.md).
bool use_persistent(int batch) {
  static const int v = [] {
    const char* e = std::getenv("JENGA_DECODE_PERSISTENT");
    return e ? std::atoi(e) : 0;
  }();
  return v != 0 && batch <= kMaxPersistB;
}

template <typename T, int D, int G, int HG>
int launch_tc(const DecodeParams& prm, const CUtensorMap& tmap, int batch, cudaStream_t stream) {
  constexpr int STAGE = 2 * HG * kTile * D * 2;
  constexpr int MERGE = (kConsumerWarps * G * D + kConsumerWarps * G * 2) * 4;
  constexpr int CTAS_PER_SM = HG >= 4 ? 1 : (HG == 2 ? 2 : 3);
  if (use_persistent(batch) && prm.k_new == nullptr) {
    // ring budget net of the separate merge area, a multiple of the rounds
    constexpr int ROUNDS = kConsumerWarps / HG;
    constexpr int BUDGET = ring_budget<HG>() - MERGE;
    constexpr int NSR = (BUDGET / STAGE) / ROUNDS * ROUNDS;
    constexpr int NS = NSR < ROUNDS ? ROUNDS : (NSR > 12 ? 12 : NSR);
    const int smem = NS * STAGE + MERGE + kItemSlots * static_cast<int>(sizeof(ItemDesc)) +
                     (2 * NS + 2 * kItemSlots) * 8 + 16 + (batch + 1) * 4 + 1024;
    auto kern = paged_decode_tc_persistent<T, D, G, HG, NS>;
    static std::atomic<uint64_t> configured{0};
    if (int rc = configure_smem(kern, smem, configured)) return rc;
    int per_sm = 0;  // resident CTAs per SM at this shared-memory size
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem) != cudaSuccess || per_sm < 1)
      per_sm = 1;
    kern<<<jenga_dev::num_sms() * std::min(per_sm, CTAS_PER_SM), kThreads, smem, stream>>>(prm, tmap);
    return jenga_dev::check_launch("paged_decode_tc_persistent");
  }
  constexpr int NS = stages<D, HG>();
  const int smem = std::max(NS * STAGE, MERGE) + 2 * NS * 8 + 16 + 1024;
  auto kern = paged_decode_tc_kernel<T, D, G, HG, NS>;
  static std::atomic<uint64_t> configured{0};
  if (int rc = configure_smem(kern, smem, configured)) return rc;
  const dim3 grid = decode_grid(prm, batch, HG);
  jenga_dev::launch_maybe_pdl(kern, grid, dim3(kThreads), smem, stream, prm, tmap);
  return jenga_dev::check_launch("paged_decode_tc_kernel");
}

template <typename T, int D, int G>
int dispatch_hg(int hg, const DecodeParams& prm, const CUtensorMap& m, int batch, cudaStream_t s) {
  switch (hg) {
    case 1: return launch_tc<T, D, G, 1>(prm, m, batch, s);
    case 2: return launch_tc<T, D, G, 2>(prm, m, batch, s);
    case 4: return launch_tc<T, D, G, 4>(prm, m, batch, s);
  }
  return JENGA_ERR_UNSUPPORTED;
}

template <typename T, int D>
int dispatch_g(int G, int hg, const DecodeParams& prm, const CUtensorMap& m, int batch, cudaStream_t s) {
  switch (G) {
    case 1: return dispatch_hg<T, D, 1>(hg, prm, m, batch, s);
    case 2: return dispatch_hg<T, D, 2>(hg, prm, m, batch, s);
    case 4: return dispatch_hg<T, D, 4>(hg, prm, m, batch, s);
    case 8: return dispatch_hg<T, D, 8>(hg, prm, m, batch, s);
  }
  return JENGA_ERR_UNSUPPORTED;
}

template <typename T>
int dispatch_d(int D, int G, int hg, const DecodeParams& prm, const CUtensorMap& m, int batch, cudaStream_t s) {
  switch (D) {
    case 64: return dispatch_g<T, 64>(G, hg, prm, m, batch, s);
    case 128: return dispatch_g<T, 128>(G, hg, prm, m, batch, s);
    case 256: return dispatch_g<T, 256>(G, hg, prm, m, batch, s);
  }
  return JENGA_ERR_UNSUPPORTED;
}

// One 4-D box per (page, head) K+V tile (default); JENGA_DECODE_KV_BOX=0 selects
// the 2-D boxes for A/B runs.
bool use_kv_box() {
  static const bool v = [] {
    const char* e = std::getenv("JENGA_DECODE_KV_BOX");
    return e == nullptr || std::atoi(e) != 0;
  }();
  return v;
}

// KV heads per CTA: 1 by default — three 1-head CTAs per SM overlap each
// other's prologue/epilogue and measured fastest on the Gemma shard
// (profiles/r01_sweeps.md); JENGA_DECODE_HEADS_PER_CTA=2|4 selects the
// multi-head variants.
int heads_per_cta(int hkv) {
  static const int forced = [] {
    const char* e = std::getenv("JENGA_DECODE_HEADS_PER_CTA");
    return e ? std::atoi(e) : 0;
  }();
  for (int hg : {forced, 1})
    if ((hg == 1 || hg == 2 || hg == 4) && hkv % hg == 0) return hg;
  return 1;
}

}  // namespace

namespace jenga_decode {

int launch_decode_tc(const DecodeParams& prm, int dtype, int head_dim, int G, int batch, cudaStream_t stream) {
  if (prm.tpp % kTile != 0 || head_dim % kBoxCols != 0 || G > 8) return JENGA_ERR_UNSUPPORTED;
  if (prm.start_offset % (head_dim * 2) || prm.page_stride % (head_dim * 2)) return JENGA_ERR_UNSUPPORTED;
  const int hg = heads_per_cta(prm.hkv);
  CUtensorMap m;
  DecodeParams p2 = prm;
  p2.kv_box = hg == 1 && use_kv_box();
  const int rc = tensor_map(prm.arena, head_dim, dtype, prm.tpp, p2.kv_box != 0, &m);
  if (rc != JENGA_OK) return rc;
  if (dtype == JENGA_BF16) return dispatch_d<__nv_bfloat16>(head_dim, G, hg, p2, m, batch, stream);
  if (dtype == JENGA_F16) return dispatch_d<__half>(head_dim, G, hg, p2, m, batch, stream);
  return JENGA_ERR_UNSUPPORTED;
}

}  // namespace jenga_decode
