// Shared device helpers for the sm_100a kernels: mbarrier pipeline, 1-D bulk
// copies (cp.async.bulk -> UBLKCP), 2-D TMA tensor loads, dtype traits,
// launch bookkeeping and the C-ABI error plumbing.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>

#include "../../../include/jenga_gpu.h"

#define JENGA_EXPORT extern "C" __attribute__((visibility("default")))

namespace jenga_dev {

// Set by every launcher; read by jenga_kernel_launch_count().
extern std::atomic<uint64_t> g_launches;
int set_error(int code, const std::string& msg);

inline int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(JENGA_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return JENGA_OK;
}

// ------------------------------------------------------------ dtype traits
template <typename T> struct DT;
template <> struct DT<float> {
  static constexpr int kBytes = 4;
  __device__ static __forceinline__ float to_f(float x) { return x; }
  __device__ static __forceinline__ float from_f(float x) { return x; }
};
template <> struct DT<__nv_bfloat16> {
  static constexpr int kBytes = 2;
  __device__ static __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
  __device__ static __forceinline__ __nv_bfloat16 from_f(float x) { return __float2bfloat16_rn(x); }
};
template <> struct DT<__half> {
  static constexpr int kBytes = 2;
  __device__ static __forceinline__ float to_f(__half x) { return __half2float(x); }
  __device__ static __forceinline__ __half from_f(float x) { return __float2half_rn(x); }
};

// Unpack N contiguous elements held in 32-bit words to fp32.
template <typename T, int N>
__device__ __forceinline__ void unpack(const uint32_t* w, float* out) {
  if constexpr (sizeof(T) == 4) {
#pragma unroll
    for (int i = 0; i < N; ++i) out[i] = __uint_as_float(w[i]);
  } else if constexpr (std::is_same<T, __nv_bfloat16>::value) {
#pragma unroll
    for (int i = 0; i < N / 2; ++i) {
      out[2 * i] = __uint_as_float(w[i] << 16);
      out[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  } else {
#pragma unroll
    for (int i = 0; i < N / 2; ++i) {
      const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
      out[2 * i] = f.x;
      out[2 * i + 1] = f.y;
    }
  }
}

// ------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}\n" ::"r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// 1-D bulk copy global -> shared, completion counted on `bar` (UBLKCP).
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gmem_src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Same, with an L2 evict-first hint: KV pages are streamed exactly once per step.
__device__ __forceinline__ void bulk_g2s_evict_first(void* smem_dst, const void* gmem_src,
                                                     uint32_t bytes, uint64_t* bar,
                                                     uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], "
      "%2, [%3], %4;\n" ::"r"(smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}

// 2-D TMA tensor load (UTMALDG) of box {c0, c1} into swizzled shared memory.
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const void* tmap, int32_t c0, int32_t c1,
                                            uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(smem_u32(smem_dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// 4-D TMA tensor load (UTMALDG.4D) of the box at {0, row, 0, 0}.
__device__ __forceinline__ void tma_load_4d_row(void* smem_dst, const void* tmap, int32_t row, uint64_t* bar,
                                                uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %2, %2}], [%4], %5;\n" ::"r"(smem_u32(smem_dst)),
      "l"(tmap), "r"(0), "r"(row), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// L2 prefetch of a 2-D TMA box (no shared-memory destination): raises the
// bytes in flight beyond what the shared-memory ring can hold.
__device__ __forceinline__ void tma_prefetch_2d(const void* tmap, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];\n" ::"l"(tmap), "r"(c0), "r"(c1)
               : "memory");
}

__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}

// One-line L2 prefetch: used to warm the address translation of a page
// several tiles before its bulk load is issued.
__device__ __forceinline__ void prefetch_line_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p));
}

__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(tmap) : "memory");
}

__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_v4(void* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// Programmatic dependent launch (PDL): a kernel launched with the
// programmatic-serialization attribute may start while the previous kernel
// in the stream is still finishing.  launch_dependents lets the *next* kernel
// start early; wait blocks until every prerequisite grid has completed and
// its writes are visible.  Both are no-ops for a normal launch.
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

int num_sms();  // SMs of the current device (cached per device)

// PDL ordering contract.  Kernels launched with the programmatic attribute may
// start before their predecessor in the stream has finished; every kernel
// reads the previous kernels' outputs only after griddepcontrol.wait — except
// the decode producer, which streams K/V tiles early.  That is safe only when
// no kernel still in the PDL chain writes arena bytes a later decode reads.
// The arena writers that trigger their dependents early (reshape_and_cache,
// the page copies) mark the stream; a launch without the attribute (table
// builds, prefill, token rows) fully serialises the stream and clears the
// mark; decode launches leave it as it is (their only arena write is the
// newest token's row, which the consumer itself patches or waits for).  The
// decode launcher asks early_kv_ok(): false -> its producer waits first.
//
// Column writers: the in-place Mamba state update writes only bytes
// [start, start + len) of every page of stride `stride` (one run of layer
// slices per page).  It records that footprint instead of the blanket mark, and
// it may itself load its state before griddepcontrol.wait when every pending
// writer is such a column writer on the same page grid with disjoint columns
// (early_columns_ok) — consecutive Mamba layers then stream their states while
// the previous layer drains.  The page-index arrays they read early come, like
// block tables, from launches without the attribute.
enum LaunchClass { kLaunchArenaWriterPdl = 0, kLaunchSerializing = 1 };
void note_launch(cudaStream_t stream, LaunchClass c);
void note_column_writer(cudaStream_t stream, uint64_t stride, uint64_t start, uint64_t len);
bool early_kv_ok(cudaStream_t stream);
bool early_columns_ok(cudaStream_t stream, uint64_t stride, uint64_t start, uint64_t len);

// Launch with the programmatic-stream-serialization attribute.
template <typename... KArgs, typename... Args>
cudaError_t launch_maybe_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                             Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

inline int dtype_bytes(int dtype) {
  switch (dtype) {
    case JENGA_F32: return 4;
    case JENGA_BF16: return 2;
    case JENGA_F16: return 2;
  }
  return 0;
}

}  // namespace jenga_dev
