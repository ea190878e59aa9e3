// Paged decode attention, tensor-core variant (bf16 / fp16 KV, page sizes that
// are multiples of 16 tokens).  Same contract, work split and epilogue as the
// CUDA-core kernel in decode.cu; the differences are the data movement and
// the math:
//
//  * K/V tiles move with TMA tensor loads (cp.async.bulk.tensor -> UTMALDG) over
//    the whole arena viewed as rows of D elements, row = one token of one
//    (page, layer, K|V, head): row index = (start_offset + global*page_stride +
//    ((2h + kv)*tpp + off)*D*e) / (D*e).  ONE 4-D box {64 cols, 16 rows, D/64
//    chunks, K|V} per 16-token tile brings a head's K and V tiles of a page
//    (the head-major page-layer slice [Hkv][K|V][tpp][D] makes them one
//    contiguous 2*16*D*e run).  Tiles land with the 128-byte swizzle, so
//    ldmatrix is conflict-free.
//  * Fused append (jenga_paged_decode_append): the warp whose tile holds the
//    newest token writes that token's K/V to its slot and into the staged tile.
//  * One CTA per (KV head, request, split); three CTAs per SM overlap each
//    other's prologue and merge (multi-head CTAs measured 9% slower on the
//    Gemma shard, profiles/r01_sweeps.md).
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

// Stage ring: decode_ring_bytes(D) per CTA (decode_common.cuh),
// a multiple of the four consumer warps so each slot is always consumed by the
// same warp — a warp that skipped a use of a slot could otherwise wait on a
// parity two phases ahead and pass early.
template <int D>
constexpr int stages() {
  constexpr int CW = decode_consumer_warps(D);
  constexpr int stage = 2 * kTile * D * 2;
  constexpr int ns = (decode_ring_bytes(D) / stage) / CW * CW;
  return ns < CW ? CW : (ns > 12 ? 12 : ns);
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

// TMA load of one 16-token tile of one head into a stage: ONE 4-D box
// {64 cols, 16 rows, D/64 chunks, K|V} = the head's K and V tiles of the page,
// landing [K|V][chunk][16 rows][128 B] — the ldmatrix layout.
template <int D>
__device__ __forceinline__ void load_stage(const CUtensorMap* tmap, uint8_t* stage, uint64_t* bar, int32_t row,
                                           uint64_t policy) {
  constexpr int TILE_BYTES = (D / kBoxCols) * kBoxBytes;
  jenga_dev::mbar_arrive_expect_tx(bar, 2 * TILE_BYTES);
  jenga_dev::tma_load_4d_row(stage, tmap, row, bar, policy);
}

// Arena row of the first K row of (page of token tok0, head h).  tok0 is below
// max_blocks*tpp (assign_work clamps n), so the table index stays in the row.
__device__ __forceinline__ int32_t tile_row(const DecodeParams& p, const int32_t* table, int h, int tok0,
                                            int64_t row_bytes) {
  const int64_t base_row = static_cast<int64_t>(p.start_offset) / row_bytes + static_cast<int64_t>(h) * 2 * p.tpp;
  const int64_t page_rows = static_cast<int64_t>(p.page_stride) / row_bytes;
  return static_cast<int32_t>(base_row + static_cast<int64_t>(table[tok0 / p.tpp]) * page_rows + tok0 % p.tpp);
}

// ------------------------------------------------------------ grid kernel
// One CTA per (KV head, request, split).
template <typename T, int D, int G, int NS>
__global__ void __launch_bounds__((decode_consumer_warps(D) + 1) * 32, decode_ctas_per_sm(D))
    paged_decode_tc_kernel(const DecodeParams p, const __grid_constant__ CUtensorMap tmap) {
  constexpr int CW = decode_consumer_warps(D);
  static_assert(D % kBoxCols == 0, "head_dim must be a multiple of 64");
  static_assert(G <= 8, "at most 8 query heads per KV head (N = 8)");
  static_assert(NS % CW == 0, "slots must map to fixed consumer warps");
  constexpr int TILE_BYTES = (D / kBoxCols) * kBoxBytes;  // 16 tokens x D x 2 B, one head
  constexpr int STAGE_BYTES = 2 * TILE_BYTES;
  constexpr int MERGE_BYTES = (CW * G * D + CW * G * 2) * 4;
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
  const int h = blockIdx.x;
  const int split = grid_split(p);
  const Work wk = assign_work(p, b, split);
  if (split >= wk.nsplit) return;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      jenga_dev::mbar_init(&full[i], 1);
      jenga_dev::mbar_init(&empty[i], 1);
    }
    jenga_dev::fence_mbar_init();
  }
  __syncthreads();
  // PDL: the next kernel in the stream may become resident now.  Block
  // tables / seq_lens come from a kernel launched without the attribute and
  // are complete; q, the newest token's K/V and the reused workspace are only
  // touched after pdl_wait().
  jenga_dev::pdl_launch_dependents();

  const int32_t* table = p.table + static_cast<int64_t>(b) * p.max_blocks;

  if (warp == CW) {
    if (lane == 0) {  // producer: one elected lane
      jenga_dev::prefetch_tmap(&tmap);
      const uint64_t policy = jenga_dev::l2_policy_evict_first();
      // an arena writer that let us start early may still be running: wait
      // for it before the first load (common.cuh, PDL ordering contract)
      bool waited = p.early_kv == 0;
      if (waited) jenga_dev::pdl_wait();
      // the next tile's arena row is read one iteration ahead, so the block-table
      // load is off the empty-slot -> refill path
      int32_t row = wk.t_count > 0 ? tile_row(p, table, h, wk.t_begin * kTile, D * 2) : 0;
      for (int it = 0; it < wk.t_count; ++it) {
        const int st = it % NS;
        const int tok0 = (wk.t_begin + it) * kTile;
        const int32_t next = it + 1 < wk.t_count ? tile_row(p, table, h, tok0 + kTile, D * 2) : 0;
        if (it >= NS) jenga_dev::mbar_wait(&empty[st], ((it / NS) & 1) ^ 1);
        if (!waited && tok0 + kTile >= wk.n && p.k_new == nullptr) {  // the tile holding the newest token
          jenga_dev::pdl_wait();  // (fused append patches that row itself: no wait)
          waited = true;
        }
        load_stage<D>(&tmap, smem + st * STAGE_BYTES, &full[st], row, policy);
        row = next;
      }
    }
    return;
  }

  HeadState<D> hs;
  jenga_dev::pdl_wait();  // q and the workspace belong to the previous kernels until here
  head_begin<T, D, G>(hs, p, b, h, lane);
  for (int it = warp; it < wk.t_count; it += CW) {
    const int st = it % NS;
    jenga_dev::mbar_wait(&full[st], (it / NS) & 1);
    uint8_t* stage = smem + st * STAGE_BYTES;
    const int tok0 = (wk.t_begin + it) * kTile;
    if (p.k_new != nullptr && wk.n - 1 >= tok0 && wk.n - 1 < tok0 + kTile)
      patch_newest<T, D>(p, stage, stage + TILE_BYTES, b, h, wk.n - 1 - tok0, lane);
    head_tile<T, D>(hs, stage, stage + TILE_BYTES, tok0, wk.lo, wk.n, p, lane);
    __syncwarp();
    if (lane == 0) jenga_dev::mbar_arrive(&empty[st]);
  }
  consumers_sync<CW>();
  float* s_acc = reinterpret_cast<float*>(smem);  // [CW][G][D] (the ring is drained)
  float* s_ml = s_acc + CW * G * D;               // [CW][G][2]
  head_store<D, G>(hs, s_acc, s_ml, warp, lane);
  merge_epilogue<T, G, D, 1, CW>(p, s_acc, s_ml, s_flag, wk.nsplit, split, b, h);
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

// The arena as a 4-D tensor {64 cols, rows, D/64 chunks at 128 B, K|V at tpp
// rows}: one box = a whole head's K and V tile of a page, 1 TMA op per
// 2*16*D*e bytes (op count, not bytes, bounded delivery in the prefill
// producer; the 2-D 64 x 16 box variant measured 1% / 4.5% slower on the
// Gemma / Llama-vision decode steps).  Encoded once per (arena, D, dtype, tpp).
int tensor_map(const void* base, int D, int dtype, int tpp, CUtensorMap* out) {
  static std::mutex mu;
  static std::map<std::tuple<uintptr_t, uint64_t, int, int, int>, CUtensorMap> cache;
  uint64_t bytes = 0;
  if (!jenga_dev::arena_extent(base, &bytes)) return JENGA_ERR_UNSUPPORTED;  // not a jenga arena
  // keyed by the extent too: a new arena may reuse a freed arena's address
  const auto key = std::make_tuple(reinterpret_cast<uintptr_t>(base), bytes, D, dtype, tpp);
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
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(kBoxCols), bytes / row_bytes, static_cast<cuuint64_t>(D / kBoxCols),
                        2};
  cuuint64_t strides[3] = {row_bytes, 128, static_cast<cuuint64_t>(tpp) * row_bytes};
  cuuint32_t box[4] = {static_cast<cuuint32_t>(kBoxCols), static_cast<cuuint32_t>(kTile),
                       static_cast<cuuint32_t>(D / kBoxCols), 2};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult r = fn(&m, dt, 4, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return jenga_dev::set_error(JENGA_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
  cache[key] = m;
  *out = m;
  return JENGA_OK;
}

template <typename T, int D, int G>
int launch_tc(const DecodeParams& prm, const CUtensorMap& tmap, int batch, cudaStream_t stream) {
  constexpr int STAGE = 2 * kTile * D * 2;
  constexpr int CW = decode_consumer_warps(D);
  constexpr int MERGE = (CW * G * D + CW * G * 2) * 4;
  constexpr int NS = stages<D>();
  const int smem = std::max(NS * STAGE, MERGE) + 2 * NS * 8 + 16 + 1024;
  auto kern = paged_decode_tc_kernel<T, D, G, NS>;
  static std::atomic<uint64_t> configured{0};
  if (int rc = configure_smem(kern, smem, configured)) return rc;
  // Launches of at most two waves go out as clusters of 4 KV heads of one
  // request (co-scheduled on one GPC): +1.3% on the Gemma G=8 shard (one
  // partial wave), +0.8% on Llama-vision (1.7 waves), neutral at G=4 / Jamba,
  // -2.4% on the prefix mix (7 waves: cluster-granular refills fragment the
  // SMs), hence the wave bound (profiles/r02_decode_experiments.md).
  const dim3 grid = decode_grid(prm, batch);
  const int64_t ctas = static_cast<int64_t>(grid.x) * grid.y * grid.z;
  const int64_t slots = static_cast<int64_t>(jenga_dev::num_sms()) * decode_ctas_per_sm(D);
  if (JENGA_DECODE_CLUSTER > 1 && prm.hkv % JENGA_DECODE_CLUSTER == 0 && ctas <= 2 * slots) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3((CW + 1) * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = JENGA_DECODE_CLUSTER;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    if (cudaLaunchKernelEx(&cfg, kern, prm, tmap) == cudaSuccess) return jenga_dev::check_launch("paged_decode_tc_kernel");
    (void)cudaGetLastError();  // cluster shape not schedulable here: plain launch below
  }
  {
    jenga_dev::launch_maybe_pdl(kern, grid, dim3((CW + 1) * 32), smem, stream, prm, tmap);
  }
  return jenga_dev::check_launch("paged_decode_tc_kernel");
}

template <typename T, int D>
int dispatch_g(int G, const DecodeParams& prm, const CUtensorMap& m, int batch, cudaStream_t s) {
  switch (G) {
    case 1: return launch_tc<T, D, 1>(prm, m, batch, s);
    case 2: return launch_tc<T, D, 2>(prm, m, batch, s);
    case 4: return launch_tc<T, D, 4>(prm, m, batch, s);
    case 8: return launch_tc<T, D, 8>(prm, m, batch, s);
  }
  return JENGA_ERR_UNSUPPORTED;
}

template <typename T>
int dispatch_d(int D, int G, const DecodeParams& prm, const CUtensorMap& m, int batch, cudaStream_t s) {
  switch (D) {
    case 64: return dispatch_g<T, 64>(G, prm, m, batch, s);
    case 128: return dispatch_g<T, 128>(G, prm, m, batch, s);
    case 256: return dispatch_g<T, 256>(G, prm, m, batch, s);
  }
  return JENGA_ERR_UNSUPPORTED;
}

}  // namespace

namespace jenga_decode {

int launch_decode_tc(const DecodeParams& prm, int dtype, int head_dim, int G, int batch, cudaStream_t stream) {
  if (prm.tpp % kTile != 0 || head_dim % kBoxCols != 0 || G > 8) return JENGA_ERR_UNSUPPORTED;
  if (prm.start_offset % (head_dim * 2) || prm.page_stride % (head_dim * 2)) return JENGA_ERR_UNSUPPORTED;
  CUtensorMap m;
  const int rc = tensor_map(prm.arena, head_dim, dtype, prm.tpp, &m);
  if (rc != JENGA_OK) return rc;
  if (dtype == JENGA_BF16) return dispatch_d<__nv_bfloat16>(head_dim, G, prm, m, batch, stream);
  if (dtype == JENGA_F16) return dispatch_d<__half>(head_dim, G, prm, m, batch, stream);
  return JENGA_ERR_UNSUPPORTED;
}

}  // namespace jenga_decode
