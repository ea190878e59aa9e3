// One contiguous HBM arena per GPU: the device image of the reference's
// LargePagePool capacity (lcm_allocator.cpp:7-19, pages = capacity / LCM).
// Large page i occupies bytes [i*LCM, (i+1)*LCM); small page g of a group is
// at g*small_page_bytes (memory_layout.cpp:29-39), so the arena is addressed
// purely by the AddressMap arithmetic — no per-layer tensors.
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "common.cuh"

namespace jenga_dev {
std::atomic<uint64_t> g_launches{0};
}  // namespace jenga_dev

// The host half owns jenga_last_error(); kernels report through it too.
extern "C" const char* jenga_last_error(void);
namespace jenga_host_err {
int set(int code, const char* msg);
}

namespace jenga_dev {
int set_error(int code, const std::string& msg) { return jenga_host_err::set(code, msg.c_str()); }

namespace {
std::mutex g_stream_mu;
// (device, stream) -> the early-triggering arena writers still possibly in the
// PDL chain: `unknown` for any writer without a footprint, else the column
// footprints [start, start + len) of every page of stride `stride`.
struct PendingWriters {
  bool unknown = false;
  std::vector<std::tuple<uint64_t, uint64_t, uint64_t>> cols;  // (stride, start, len)
};
std::map<std::pair<int, uintptr_t>, PendingWriters> g_pending;

std::pair<int, uintptr_t> stream_key(cudaStream_t s) {
  int dev = 0;
  cudaGetDevice(&dev);
  return {dev, reinterpret_cast<uintptr_t>(s)};
}
}  // namespace

void note_launch(cudaStream_t stream, LaunchClass c) {
  std::lock_guard<std::mutex> lock(g_stream_mu);
  if (c == kLaunchArenaWriterPdl)
    g_pending[stream_key(stream)].unknown = true;
  else
    g_pending.erase(stream_key(stream));
}

void note_column_writer(cudaStream_t stream, uint64_t stride, uint64_t start, uint64_t len) {
  std::lock_guard<std::mutex> lock(g_stream_mu);
  auto& w = g_pending[stream_key(stream)];
  if (w.cols.size() >= 64) w.unknown = true;  // bounded bookkeeping: degrade to "unknown"
  else w.cols.emplace_back(stride, start, len);
}

bool early_kv_ok(cudaStream_t stream) {
  std::lock_guard<std::mutex> lock(g_stream_mu);
  return g_pending.count(stream_key(stream)) == 0;
}

bool early_columns_ok(cudaStream_t stream, uint64_t stride, uint64_t start, uint64_t len) {
  std::lock_guard<std::mutex> lock(g_stream_mu);
  auto it = g_pending.find(stream_key(stream));
  if (it == g_pending.end()) return true;
  if (it->second.unknown) return false;
  for (const auto& [s, b, l] : it->second.cols)  // same page grid, disjoint columns
    if (s != stride || (start < b + l && b < start + len)) return false;
  return true;
}

int num_sms() {
  int dev = 0, v = 148;
  cudaGetDevice(&dev);
  static std::atomic<int> cached[64] = {};
  if (dev < 64 && cached[dev].load()) return cached[dev].load();
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  if (dev < 64) cached[dev].store(v);
  return v;
}
}  // namespace jenga_dev

struct jenga_arena {
  int device = 0;
  void* base = nullptr;
  uint64_t bytes = 0;
};

// Registry of live arenas: kernels that build TMA tensor maps over the whole
// arena look their extent up by base pointer.
namespace {
std::mutex g_arena_mu;
std::map<uintptr_t, uint64_t> g_arenas;
}  // namespace

namespace jenga_dev {
bool arena_extent(const void* base, uint64_t* bytes) {
  std::lock_guard<std::mutex> lock(g_arena_mu);
  auto it = g_arenas.find(reinterpret_cast<uintptr_t>(base));
  if (it == g_arenas.end()) return false;
  *bytes = it->second;
  return true;
}
}  // namespace jenga_dev

JENGA_EXPORT int jenga_arena_create(int device, uint64_t num_large_pages, uint64_t large_page_bytes,
                                    jenga_arena** out) {
  using namespace jenga_dev;
  if (out == nullptr || large_page_bytes == 0) return set_error(JENGA_ERR_ARG, "invalid arena arguments");
  uint64_t bytes = 0;
  if (__builtin_mul_overflow(num_large_pages, large_page_bytes, &bytes))
    return set_error(JENGA_ERR_CONFIG, "byte arithmetic overflow in arena size");
  if (large_page_bytes % 16 != 0)
    return set_error(JENGA_ERR_CONFIG, "large page bytes must be a multiple of 16 for vector access");
  int prev = 0;
  cudaGetDevice(&prev);
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return set_error(JENGA_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  void* p = nullptr;
  e = cudaMalloc(&p, bytes ? bytes : 256);
  cudaSetDevice(prev);
  if (e != cudaSuccess)
    return set_error(JENGA_ERR_CUDA, std::string("arena cudaMalloc(") + std::to_string(bytes) +
                                         "): " + cudaGetErrorString(e));
  auto* a = new jenga_arena;
  a->device = device;
  a->base = p;
  a->bytes = bytes;
  {
    std::lock_guard<std::mutex> lock(g_arena_mu);
    g_arenas[reinterpret_cast<uintptr_t>(p)] = bytes;
  }
  *out = a;
  return JENGA_OK;
}

JENGA_EXPORT void jenga_arena_destroy(jenga_arena* arena) {
  if (arena == nullptr) return;
  int prev = 0;
  cudaGetDevice(&prev);
  {
    std::lock_guard<std::mutex> lock(g_arena_mu);
    g_arenas.erase(reinterpret_cast<uintptr_t>(arena->base));
  }
  cudaSetDevice(arena->device);
  cudaFree(arena->base);
  cudaSetDevice(prev);
  delete arena;
}

JENGA_EXPORT void* jenga_arena_base(const jenga_arena* arena) { return arena ? arena->base : nullptr; }
JENGA_EXPORT uint64_t jenga_arena_bytes(const jenga_arena* arena) { return arena ? arena->bytes : 0; }

JENGA_EXPORT uint64_t jenga_kernel_launch_count(void) {
  return jenga_dev::g_launches.load(std::memory_order_relaxed);
}
