// Pieces shared by the two paged-decode kernels (decode.cu: CUDA-core math
// for fp32 / odd page sizes; decode_tc.cu: tensor-core math for bf16/fp16):
// launch parameters, the split-KV work assignment and the epilogue that
// merges the four consumer warps and then the splits of one (request, head).
#pragma once

#include "common.cuh"

namespace jenga_decode {

constexpr int kTile = 16;  // tokens per pipeline stage
constexpr int kConsumerWarps = 4;
constexpr int kThreads = (kConsumerWarps + 1) * 32;
constexpr float kLog2e = 1.4426950408889634f;
constexpr int kTilesPerSplit = 32;  // 512 tokens per CTA
// Tensor-core decode residency per head_dim: CTAs per SM and the stage-ring
// bytes of each.  Measured (profiles/r02_sweep_residency.jsonl): two 64 KiB
// rings per SM at head_dim 256, four 48 KiB rings at 128 and below.
// Compile-time so profiling variants (build.py --variant) can sweep them.
#ifndef JENGA_DECODE_CTAS_PER_SM_D256
#define JENGA_DECODE_CTAS_PER_SM_D256 2
#endif
#ifndef JENGA_DECODE_RING_BYTES_D256
#define JENGA_DECODE_RING_BYTES_D256 65536
#endif
#ifndef JENGA_DECODE_CTAS_PER_SM_D128
#define JENGA_DECODE_CTAS_PER_SM_D128 4
#endif
#ifndef JENGA_DECODE_RING_BYTES_D128
#define JENGA_DECODE_RING_BYTES_D128 49152
#endif
__host__ __device__ constexpr int decode_ctas_per_sm(int head_dim) {
  return head_dim >= 256 ? JENGA_DECODE_CTAS_PER_SM_D256 : JENGA_DECODE_CTAS_PER_SM_D128;
}
__host__ __device__ constexpr int decode_ring_bytes(int head_dim) {
  return head_dim >= 256 ? JENGA_DECODE_RING_BYTES_D256 : JENGA_DECODE_RING_BYTES_D128;
}
// KV heads per thread-block cluster for launches of at most two waves
// (decode_tc.cu launch_tc); 1 disables clusters (profiling variant).
#ifndef JENGA_DECODE_CLUSTER
#define JENGA_DECODE_CLUSTER 4
#endif
// Consumer warps per CTA (each owns the stages s with s % CW == its index).
#ifndef JENGA_DECODE_CONSUMERS_D256
#define JENGA_DECODE_CONSUMERS_D256 4
#endif
#ifndef JENGA_DECODE_CONSUMERS_D128
#define JENGA_DECODE_CONSUMERS_D128 4
#endif
__host__ __device__ constexpr int decode_consumer_warps(int head_dim) {
  return head_dim >= 256 ? JENGA_DECODE_CONSUMERS_D256 : JENGA_DECODE_CONSUMERS_D128;
}

struct DecodeParams {
  const uint8_t* arena;
  uint64_t start_offset;
  uint64_t page_stride;
  const void* q;
  void* out;
  const int32_t* table;
  const int32_t* seq_lens;
  int kind;
  int64_t window;
  int max_blocks;
  int hq;
  int hkv;
  int tpp;
  int tiles_per_split;
  int max_splits;
  int batch;
  float qscale;    // scale*log2e, or scale when soft-capping
  float cap_log2;  // softcap*log2e (0: off)
  float inv_cap;   // 1/softcap
  float* part_acc; // [B][Hkv][max_splits][G][D]
  float* part_ml;  // [B][Hkv][max_splits][G][2]
  int* counters;   // [B][Hkv]
  // 1: the producer may stream K/V before griddepcontrol.wait (no early-
  // triggering arena writer is still in the PDL chain, common.cuh)
  int early_kv;
  // Fused append (jenga_paged_decode_append): the newest token's K/V rows
  // [B][Hkv][D] and slots; nullptr = plain decode (K/V already in the arena).
  const void* k_new;
  const void* v_new;
  const int64_t* new_slots;
};

// Grid = (Hkv, batch, max_splits).
__device__ __forceinline__ int grid_request(const DecodeParams&) { return blockIdx.y; }
__device__ __forceinline__ int grid_split(const DecodeParams&) { return blockIdx.z; }
inline dim3 decode_grid(const DecodeParams& p, int batch) { return dim3(p.hkv, batch, p.max_splits); }

// Live ordinals of request b (LayerPolicy::needs_token, layer_policies.cpp:
// 105-120) cut into splits of whole 16-token tiles.
struct Work {
  int n, lo, nsplit, t_begin, t_count;
};

__device__ __forceinline__ Work assign_work(const DecodeParams& p, int b, int split) {
  Work w;
  // a length beyond the table width is clamped to the blocks the table holds,
  // so no kernel ever indexes past the request's row
  w.n = min(p.seq_lens[b], p.max_blocks * p.tpp);
  w.lo = 0;
  if (p.kind == JENGA_KIND_SLIDING_WINDOW && w.n > p.window) w.lo = static_cast<int>(w.n - p.window);
  const int tile_lo = w.lo / kTile;
  const int tile_hi = (w.n + kTile - 1) / kTile;
  const int ntiles = w.n > 0 ? tile_hi - tile_lo : 0;
  int ns = (ntiles + p.tiles_per_split - 1) / p.tiles_per_split;
  w.nsplit = max(1, min(ns, p.max_splits));
  const int per = ntiles / w.nsplit, rem = ntiles % w.nsplit;
  w.t_begin = tile_lo + split * per + min(split, rem);
  w.t_count = per + (split < rem ? 1 : 0);
  return w;
}

template <int CW = kConsumerWarps>
__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;\n" ::"n"(CW * 32) : "memory");
}

// Called by the 128 consumer threads after each warp w wrote its unnormalised
// state to s_acc[w][G][D] / s_ml[w][G][{m, l}] (m in log2 units, -inf = no
// live token).  Writes out[b][h*G+g][:] directly when the request has one
// split; otherwise stores the CTA partial and the last CTA of (b, h) to
// finish (atomic ticket) combines all splits and re-arms the ticket.
//
// HG KV heads per CTA: warp w holds local head w % HG of round w / HG, so
// head hl merges warps {hl, hl + HG, ...}.  The CTA covers heads
// [h0, h0 + HG); one ticket per (request, head group).
template <typename T, int G, int D, int HG = 1, int CW = kConsumerWarps>
__device__ __forceinline__ void merge_epilogue(const DecodeParams& p, const float* s_acc, const float* s_ml,
                                               int* s_flag, int nsplit, int split, int b, int h0) {
  constexpr int R = CW / HG;  // warps per head
  consumers_sync<CW>();
  const int tid = threadIdx.x;
  const int64_t b_h0 = static_cast<int64_t>(b) * p.hkv + h0;
  T* outp = static_cast<T*>(p.out) + (static_cast<int64_t>(b) * p.hq + h0 * G) * D;
  for (int i = tid; i < HG * G * D; i += CW * 32) {
    const int hl = i / (G * D);
    const int j = i - hl * G * D;
    const int g = j / D;
    float M = -INFINITY;
#pragma unroll
    for (int r = 0; r < R; ++r) M = fmaxf(M, s_ml[((r * HG + hl) * G + g) * 2]);
    float a = 0.f, L = 0.f;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int w = r * HG + hl;
      const float mw = s_ml[(w * G + g) * 2];
      const float wt = mw == -INFINITY ? 0.f : jenga_dev::fast_exp2(mw - M);
      a += wt * s_acc[(w * G) * D + j];
      L += wt * s_ml[(w * G + g) * 2 + 1];
    }
    if (nsplit == 1) {
      outp[i] = jenga_dev::DT<T>::from_f(L > 0.f ? a / L : 0.f);
    } else {
      const int64_t slot = (b_h0 + hl) * p.max_splits + split;
      p.part_acc[slot * G * D + j] = a;
      if (j % D == 0) {
        p.part_ml[(slot * G + g) * 2] = M;
        p.part_ml[(slot * G + g) * 2 + 1] = L;
      }
    }
  }
  if (nsplit == 1) return;

  __threadfence();
  consumers_sync<CW>();
  if (tid == 0) {
    const int ticket = atomicAdd(&p.counters[b_h0], 1);
    *s_flag = (ticket == nsplit - 1) ? 1 : 0;
  }
  consumers_sync<CW>();
  if (*s_flag == 0) return;
  __threadfence();
  for (int i = tid; i < HG * G * D; i += CW * 32) {
    const int hl = i / (G * D);
    const int j = i - hl * G * D;
    const int g = j / D;
    const int64_t slot0 = (b_h0 + hl) * p.max_splits;
    float M = -INFINITY;
    for (int s2 = 0; s2 < nsplit; ++s2) M = fmaxf(M, __ldcg(&p.part_ml[((slot0 + s2) * G + g) * 2]));
    float a = 0.f, L = 0.f;
    for (int s2 = 0; s2 < nsplit; ++s2) {
      const float ms = __ldcg(&p.part_ml[((slot0 + s2) * G + g) * 2]);
      const float wt = ms == -INFINITY ? 0.f : jenga_dev::fast_exp2(ms - M);
      a += wt * __ldcg(&p.part_acc[(slot0 + s2) * G * D + j]);
      L += wt * __ldcg(&p.part_ml[((slot0 + s2) * G + g) * 2 + 1]);
    }
    outp[i] = jenga_dev::DT<T>::from_f(L > 0.f ? a / L : 0.f);
  }
  if (tid == 0) p.counters[b_h0] = 0;  // re-arm for the next launch / graph replay
}

// Opt a kernel in to >48 KB dynamic shared memory once per device.
template <typename K>
int configure_smem(K kern, int smem, std::atomic<uint64_t>& configured) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(configured.load() & bit)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess)
      return jenga_dev::set_error(JENGA_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    configured.fetch_or(bit);
  }
  return JENGA_OK;
}

// Tensor-core path (decode_tc.cu); returns JENGA_ERR_UNSUPPORTED when the
// shape is not covered so the caller can use the CUDA-core kernel.
int launch_decode_tc(const DecodeParams& prm, int dtype, int head_dim, int G, int batch, cudaStream_t stream);

}  // namespace jenga_decode
