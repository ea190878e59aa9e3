/*
 * jenga_oracle.c — CPU ORACLE for the B200 Jenga hot path.  TEST
 * INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py as the checker; never
 * linked into or called by the product (paper_2503_18292_b200/).
 *
 * A plain-C restatement of the reference algorithm for this path, each
 * function citing the reference file:line it follows (paths relative to the
 * reference repository root).  Integer/byte work is restated exactly; the
 * attention arithmetic (absent from the reference) is restated in
 * fp64 from its definition over the same byte arena and the reference's
 * liveness masks.
 *
 * Parity pinning: the address-map and block-table arithmetic is pinned to the
 * reference's own golden vectors (proj/tests/test_memory_layout.cpp:67-191)
 * and to the reference library itself built under oracle/_ref; the attention
 * outputs are "parity unpinned" by the reference (no reference kernel exists)
 * and are pinned only by their definition (softmax(q.K^T*scale).V over the
 * live ordinals of layer_policies.cpp:105-120).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ERR_CONFIG 1
#define ORC_ERR_INVARIANT 2

enum { ORC_FULL = 0, ORC_SWA = 1, ORC_MAMBA = 2, ORC_CROSS = 3, ORC_VISION = 4 };
enum { ORC_F32 = 0, ORC_BF16 = 1, ORC_F16 = 2 };

/* proj/src/model_config.cpp:85-89 — bytes/token/layer x layers x tokens/page,
 * overflow-checked (util.hpp:31-37). */
int orc_small_page_size(uint64_t bptl, uint64_t num_layers, uint64_t tpp, uint64_t* out) {
  uint64_t a;
  if (__builtin_mul_overflow(bptl, num_layers, &a)) return ORC_ERR_CONFIG;
  if (__builtin_mul_overflow(a, tpp, out)) return ORC_ERR_CONFIG;
  return ORC_OK;
}

static uint64_t gcd_u64(uint64_t a, uint64_t b) {
  while (b) {
    uint64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}

/* proj/src/model_config.cpp:93-107 — LCM folded over the small pages. */
int orc_lcm_page_size(const uint64_t* small, int n, uint64_t* out) {
  uint64_t l = 1;
  for (int i = 0; i < n; ++i) {
    uint64_t g = gcd_u64(l, small[i]);
    if (__builtin_mul_overflow(l / g, small[i], &l)) return ORC_ERR_CONFIG;
  }
  *out = l;
  return ORC_OK;
}

/* proj/src/memory_layout.cpp:22-27 */
int orc_global_page_index(uint32_t large, uint32_t slot, uint32_t slots_per_large, uint64_t* out) {
  if (slot >= slots_per_large) return ORC_ERR_INVARIANT;
  *out = (uint64_t)large * slots_per_large + slot;
  return ORC_OK;
}

/* proj/src/memory_layout.cpp:29-39 */
int orc_address_of(uint64_t large_bytes, uint64_t small_bytes, uint64_t per_layer, uint32_t num_layers,
                   uint32_t slots_per_large, uint32_t layer, uint32_t large, uint32_t slot, uint64_t* begin,
                   uint64_t* end) {
  if (layer >= num_layers || slot >= slots_per_large) return ORC_ERR_INVARIANT;
  *begin = (uint64_t)large * large_bytes + (uint64_t)slot * small_bytes + (uint64_t)layer * per_layer;
  *end = *begin + per_layer;
  return ORC_OK;
}

/* proj/src/memory_layout.cpp:41-55 — LayerView and view address. */
int orc_view_address(uint64_t small_bytes, uint64_t per_layer, uint32_t num_layers, uint32_t slots_per_large,
                     uint32_t layer, uint32_t large, uint32_t slot, uint64_t* begin, uint64_t* end) {
  if (layer >= num_layers || slot >= slots_per_large) return ORC_ERR_INVARIANT;
  uint64_t start = (uint64_t)layer * per_layer;
  uint64_t g = (uint64_t)large * slots_per_large + slot;
  *begin = start + g * small_bytes;
  *end = *begin + per_layer;
  return ORC_OK;
}

/* Block tables: logical block b of request r -> AddressMap global index of
 * its SmallPageId (memory_layout.cpp:22-27); -1 for blocks freed out of the
 * window (simulator.cpp:272-280, leading dead prefix) and for padding.
 * slot_out[r] = slot of the newest stored ordinal n: global*tpp + (n-1)%tpp. */
int orc_build_block_tables(const int32_t* offsets, const uint32_t* pages /* [N][2] */,
                           const int32_t* first_live, const int32_t* n_stored, int batch,
                           uint32_t slots_per_large, uint32_t tpp, int max_blocks, int32_t* table,
                           int64_t* slot_out, int32_t* seq_out) {
  for (int r = 0; r < batch; ++r) {
    int begin = offsets[r], count = offsets[r + 1] - begin;
    int live0 = first_live ? first_live[r] : 0;
    if (count > max_blocks) return ORC_ERR_INVARIANT;
    for (int i = 0; i < max_blocks; ++i) {
      int32_t v = -1;
      if (i < count && i >= live0) {
        uint64_t g;
        if (orc_global_page_index(pages[2 * (begin + i)], pages[2 * (begin + i) + 1], slots_per_large, &g))
          return ORC_ERR_INVARIANT;
        v = (int32_t)g;
      }
      table[(int64_t)r * max_blocks + i] = v;
    }
    int n = n_stored ? n_stored[r] : 0;
    if (seq_out) seq_out[r] = n;
    if (slot_out) {
      int64_t s = -1;
      if (n > 0) {
        int blk = (n - 1) / (int)tpp;
        if (blk < count && blk >= live0) {
          uint64_t g = (uint64_t)pages[2 * (begin + blk)] * slots_per_large + pages[2 * (begin + blk) + 1];
          s = (int64_t)g * tpp + (n - 1) % (int)tpp;
        }
      }
      slot_out[r] = s;
    }
  }
  return ORC_OK;
}

static inline double ld_elem(const uint8_t* p, int dtype) {
  if (dtype == ORC_F32) {
    float f;
    memcpy(&f, p, 4);
    return (double)f;
  }
  uint16_t h;
  memcpy(&h, p, 2);
  if (dtype == ORC_BF16) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    memcpy(&f, &u, 4);
    return (double)f;
  }
  /* IEEE fp16 */
  uint32_t sign = (h >> 15) & 1, exp = (h >> 10) & 0x1f, man = h & 0x3ff;
  double v;
  if (exp == 0) v = ldexp((double)man, -24);
  else if (exp == 31) v = man ? NAN : INFINITY;
  else v = ldexp((double)(man | 0x400), (int)exp - 25);
  return sign ? -v : v;
}

static inline int dtype_size(int dtype) { return dtype == ORC_F32 ? 4 : 2; }

/* Slice layout of one (small page, layer): [Hkv][K|V][tpp][D] of dtype, so
 * exec_page_size = 2*Hkv*tpp*D*e (memory_layout.cpp:16-17 sizes it as
 * bytes_per_token_per_layer*tpp with bptl = 2*Hkv*D*e). */
static inline int64_t slice_row(int kv, int h, int hkv, int tpp, int off) {
  (void)hkv;
  return (((int64_t)h * 2 + kv) * tpp + off);
}

/* reshape_and_cache: row t of K/V -> slot s = page*tpp + off. */
int orc_reshape_and_cache(uint8_t* arena, uint64_t start_offset, uint64_t page_stride, int dtype, int hkv, int d,
                          int tpp, const uint8_t* key, const uint8_t* value, int64_t token_stride_elems,
                          const int64_t* slots, int n_tokens) {
  int e = dtype_size(dtype);
  int64_t row = (int64_t)d * e;
  for (int t = 0; t < n_tokens; ++t) {
    if (slots[t] < 0) continue;
    int64_t page = slots[t] / tpp, off = slots[t] % tpp;
    for (int h = 0; h < hkv; ++h) {
      for (int kv = 0; kv < 2; ++kv) {
        const uint8_t* src = (kv ? value : key) + (int64_t)t * token_stride_elems * e + h * row;
        uint8_t* dst = arena + start_offset + page * page_stride + slice_row(kv, h, hkv, tpp, (int)off) * row;
        memcpy(dst, src, (size_t)row);
      }
    }
  }
  return ORC_OK;
}

typedef struct {
  const uint8_t* arena;
  uint64_t start_offset, page_stride;
  int kind, dtype;
  int64_t window;
  const uint8_t* q;
  double* out;
  const int32_t* table;
  const int32_t* seq_lens;
  int batch, max_blocks, hq, hkv, d, tpp;
  double scale, softcap;
  int rc;
} decode_args;

/* One (request, kv head): softmax(q.K^T*scale [softcap]).V over the live
 * ordinals — full/cross: 1..n; sliding window: i + W > n
 * (layer_policies.cpp:105-120), i.e. 0-based [n-W, n). fp64 throughout. */
static int decode_one(const decode_args* a, int b, int h, double* s) {
  int e = dtype_size(a->dtype), G = a->hq / a->hkv;
  int64_t row = (int64_t)a->d * e;
  int n = a->seq_lens[b];
  int lo = 0;
  if (a->kind == ORC_SWA && n > a->window) lo = (int)(n - a->window);
  for (int g = 0; g < G; ++g) {
    int qh = h * G + g;
    const uint8_t* qp = a->q + ((int64_t)b * a->hq + qh) * row;
    double* op = a->out + ((int64_t)b * a->hq + qh) * a->d;
    for (int x = 0; x < a->d; ++x) op[x] = 0.0;
    if (n <= lo) continue;
    double m = -INFINITY;
    for (int t = lo; t < n; ++t) {
      int blk = t / a->tpp, off = t % a->tpp;
      if (blk >= a->max_blocks) return ORC_ERR_INVARIANT;
      int32_t page = a->table[(int64_t)b * a->max_blocks + blk];
      if (page < 0) return ORC_ERR_INVARIANT; /* a live ordinal on a freed page */
      const uint8_t* kp = a->arena + a->start_offset + (int64_t)page * a->page_stride +
                          slice_row(0, h, a->hkv, a->tpp, off) * row;
      double dot = 0.0;
      for (int x = 0; x < a->d; ++x) dot += ld_elem(qp + x * e, a->dtype) * ld_elem(kp + x * e, a->dtype);
      dot *= a->scale;
      if (a->softcap > 0.0) dot = a->softcap * tanh(dot / a->softcap);
      s[t - lo] = dot;
      if (dot > m) m = dot;
    }
    double l = 0.0;
    for (int t = lo; t < n; ++t) {
      double p = exp(s[t - lo] - m);
      l += p;
      int blk = t / a->tpp, off = t % a->tpp;
      int32_t page = a->table[(int64_t)b * a->max_blocks + blk];
      const uint8_t* vp = a->arena + a->start_offset + (int64_t)page * a->page_stride +
                          slice_row(1, h, a->hkv, a->tpp, off) * row;
      for (int x = 0; x < a->d; ++x) op[x] += p * ld_elem(vp + x * e, a->dtype);
    }
    for (int x = 0; x < a->d; ++x) op[x] /= l;
  }
  return ORC_OK;
}

typedef struct {
  decode_args* a;
  int first, stride;
} worker_args;

static void* decode_worker(void* p) {
  worker_args* w = (worker_args*)p;
  decode_args* a = w->a;
  int maxn = 1;
  for (int b = 0; b < a->batch; ++b)
    if (a->seq_lens[b] > maxn) maxn = a->seq_lens[b];
  double* s = (double*)malloc(sizeof(double) * (size_t)maxn);
  if (!s) {
    a->rc = ORC_ERR_CONFIG;
    return NULL;
  }
  for (int i = w->first; i < a->batch * a->hkv; i += w->stride) {
    int rc = decode_one(a, i / a->hkv, i % a->hkv, s);
    if (rc) a->rc = rc;
  }
  free(s);
  return NULL;
}

/* Paged decode over the two-level table; out is fp64 [B][Hq][D].
 * nthreads > 1 splits (request, head) pairs across POSIX threads. */
int orc_paged_decode(const uint8_t* arena, uint64_t start_offset, uint64_t page_stride, int kind, int dtype,
                     int64_t window, const uint8_t* q, double* out, const int32_t* table, const int32_t* seq_lens,
                     int batch, int max_blocks, int hq, int hkv, int d, int tpp, double scale, double softcap,
                     int nthreads) {
  if (hkv <= 0 || hq % hkv || tpp <= 0) return ORC_ERR_CONFIG;
  if (kind != ORC_FULL && kind != ORC_SWA && kind != ORC_CROSS) return ORC_ERR_CONFIG;
  decode_args a = {arena, start_offset, page_stride, kind, dtype, window, q, out, table, seq_lens,
                   batch, max_blocks, hq, hkv, d, tpp, scale, softcap, ORC_OK};
  if (nthreads < 1) nthreads = 1;
  if (nthreads == 1) {
    worker_args w = {&a, 0, 1};
    decode_worker(&w);
    return a.rc;
  }
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
  worker_args* wa = (worker_args*)malloc(sizeof(worker_args) * (size_t)nthreads);
  for (int i = 0; i < nthreads; ++i) {
    wa[i].a = &a;
    wa[i].first = i;
    wa[i].stride = nthreads;
    pthread_create(&th[i], NULL, decode_worker, &wa[i]);
  }
  for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
  free(th);
  free(wa);
  return a.rc;
}

/* Chunked prefill attention (reference prefill_some, simulator.cpp:504-547,
 * stores the chunk's positions): request b owns query
 * tokens [cu_q[b], cu_q[b+1]) which are its newest C_b ordinals, i.e. 0-based
 * positions n_b - C_b .. n_b - 1 with n_b = seq_lens[b].  Query position i
 * attends key j iff j <= i (causal) and, for sliding windows, j + W > i
 * (needs_token at length i+1, layer_policies.cpp:105-120); cross attention
 * attends all n_b keys.  q/out [T][Hq][D], out fp64. */
int orc_paged_prefill(const uint8_t* arena, uint64_t start_offset, uint64_t page_stride, int kind, int dtype,
                      int64_t window, const uint8_t* q, double* out, const int32_t* cu_q, const int32_t* table,
                      const int32_t* seq_lens, int batch, int max_blocks, int hq, int hkv, int d, int tpp,
                      double scale, double softcap) {
  if (hkv <= 0 || hq % hkv || tpp <= 0) return ORC_ERR_CONFIG;
  const int e = dtype_size(dtype), G = hq / hkv;
  const int64_t row = (int64_t)d * e;
  for (int b = 0; b < batch; ++b) {
    const int n = seq_lens[b], c = cu_q[b + 1] - cu_q[b];
    if (c > n && kind != ORC_CROSS) return ORC_ERR_INVARIANT;
    double* s = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    for (int t = 0; t < c; ++t) {
      const int i = n - c + t;  /* 0-based position of this query */
      int lo = 0, hi = i;       /* inclusive key range */
      if (kind == ORC_CROSS) hi = n - 1;
      if (kind == ORC_SWA && i + 1 > window) lo = (int)(i + 1 - window);
      for (int qh = 0; qh < hq; ++qh) {
        const int h = qh / G;
        const uint8_t* qp = q + ((int64_t)(cu_q[b] + t) * hq + qh) * row;
        double* op = out + ((int64_t)(cu_q[b] + t) * hq + qh) * d;
        for (int x = 0; x < d; ++x) op[x] = 0.0;
        double m = -INFINITY;
        for (int j = lo; j <= hi; ++j) {
          const int32_t page = table[(int64_t)b * max_blocks + j / tpp];
          if (page < 0) { free(s); return ORC_ERR_INVARIANT; }
          const uint8_t* kp = arena + start_offset + (int64_t)page * page_stride + slice_row(0, h, hkv, tpp, j % tpp) * row;
          double dot = 0.0;
          for (int x = 0; x < d; ++x) dot += ld_elem(qp + x * e, dtype) * ld_elem(kp + x * e, dtype);
          dot *= scale;
          if (softcap > 0.0) dot = softcap * tanh(dot / softcap);
          s[j] = dot;
          if (dot > m) m = dot;
        }
        double l = 0.0;
        for (int j = lo; j <= hi; ++j) {
          const double p = exp(s[j] - m);
          l += p;
          const int32_t page = table[(int64_t)b * max_blocks + j / tpp];
          const uint8_t* vp = arena + start_offset + (int64_t)page * page_stride + slice_row(1, h, hkv, tpp, j % tpp) * row;
          for (int x = 0; x < d; ++x) op[x] += p * ld_elem(vp + x * e, dtype);
        }
        if (l > 0) for (int x = 0; x < d; ++x) op[x] /= l;
      }
    }
    free(s);
  }
  return ORC_OK;
}

/* Mamba last-token state (simulator.cpp:222-244: one working page per
 * request; the layer's slice is exec_page_size bytes at start+global*stride). */
int orc_mamba_gather(const uint8_t* arena, uint64_t start_offset, uint64_t page_stride, uint64_t exec_bytes,
                     const int64_t* page_globals, int batch, uint8_t* dense) {
  for (int b = 0; b < batch; ++b) {
    if (page_globals[b] < 0) continue;
    memcpy(dense + (int64_t)b * exec_bytes, arena + start_offset + page_globals[b] * page_stride, exec_bytes);
  }
  return ORC_OK;
}

int orc_mamba_scatter(uint8_t* arena, uint64_t start_offset, uint64_t page_stride, uint64_t exec_bytes,
                      const int64_t* page_globals, int batch, const uint8_t* dense) {
  for (int b = 0; b < batch; ++b) {
    if (page_globals[b] < 0) continue;
    memcpy(arena + start_offset + page_globals[b] * page_stride, dense + (int64_t)b * exec_bytes, exec_bytes);
  }
  return ORC_OK;
}

/* In-place state step over layers [l0, l0 + num_layers) of each request's
 * working page: the layers' slices are one contiguous run (page-layer layout,
 * memory_layout.cpp:29-55); every fp32 state element is multiplied by decay
 * (the stand-in for the selective-scan update, whose math is out of scope). */
int orc_mamba_update(uint8_t* arena, uint64_t start_offset, uint64_t page_stride, uint64_t exec_bytes,
                     uint32_t num_layers, const int64_t* page_globals, int batch, float decay) {
  const uint64_t n = exec_bytes * num_layers / 4;
  for (int b = 0; b < batch; ++b) {
    if (page_globals[b] < 0) continue;
    float* s = (float*)(arena + start_offset + page_globals[b] * page_stride);
    for (uint64_t i = 0; i < n; ++i) s[i] = s[i] * decay;
  }
  return ORC_OK;
}

/* Checkpoint snapshot (simulator.cpp:231-242): whole small page copy. */
int orc_page_copy(uint8_t* arena, uint64_t small_page_bytes, const int64_t* src, const int64_t* dst, int n) {
  for (int i = 0; i < n; ++i) {
    if (src[i] < 0 || dst[i] < 0) continue;
    memmove(arena + dst[i] * small_page_bytes, arena + src[i] * small_page_bytes, small_page_bytes);
  }
  return ORC_OK;
}

/* Token rows <-> pages: the vision-embedding page path (simulator.cpp:453-476,
 * 525-542).  Piece p of row t lives in layer
 * p / ppl, sub-slice q = p % ppl, at
 *   start + layer*layer_stride + page*page_stride + (q*tpp + off)*piece
 * for slot = page*tpp + off (the page-layer address of memory_layout.cpp:
 * 41-55 plus our intra-slice layout).  Negative slots: scatter skips, gather
 * yields zeros. */
static uint8_t* orc_row_piece(uint8_t* arena, uint64_t start, uint64_t layer_stride, uint64_t page_stride,
                              uint32_t tpp, uint32_t ppl, uint32_t piece, int64_t slot, uint64_t p) {
  const uint64_t layer = p / ppl, q = p % ppl;
  const uint64_t page = (uint64_t)slot / tpp, off = (uint64_t)slot % tpp;
  return arena + start + layer * layer_stride + page * page_stride + (q * tpp + off) * piece;
}

int orc_token_rows_scatter(uint8_t* arena, uint64_t start, uint64_t layer_stride, uint64_t page_stride, uint32_t tpp,
                           uint32_t ppl, uint32_t piece, const uint8_t* rows, uint64_t row_bytes, int64_t row_stride,
                           const int64_t* slots, int n) {
  if (piece == 0 || row_bytes % piece) return ORC_ERR_CONFIG;
  for (int t = 0; t < n; ++t) {
    if (slots[t] < 0) continue;
    for (uint64_t p = 0; p < row_bytes / piece; ++p)
      memcpy(orc_row_piece(arena, start, layer_stride, page_stride, tpp, ppl, piece, slots[t], p),
             rows + (int64_t)t * row_stride + p * piece, piece);
  }
  return ORC_OK;
}

int orc_token_rows_gather(uint8_t* arena, uint64_t start, uint64_t layer_stride, uint64_t page_stride, uint32_t tpp,
                          uint32_t ppl, uint32_t piece, uint8_t* rows, uint64_t row_bytes, int64_t row_stride,
                          const int64_t* slots, int n) {
  if (piece == 0 || row_bytes % piece) return ORC_ERR_CONFIG;
  for (int t = 0; t < n; ++t) {
    uint8_t* row = rows + (int64_t)t * row_stride;
    if (slots[t] < 0) {
      memset(row, 0, row_bytes);
      continue;
    }
    for (uint64_t p = 0; p < row_bytes / piece; ++p)
      memcpy(row + p * piece, orc_row_piece(arena, start, layer_stride, page_stride, tpp, ppl, piece, slots[t], p),
             piece);
  }
  return ORC_OK;
}
