/* ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product.
 *
 * CPU restatement of the paged multi-LoRA apply, the operation P-LoRA's
 * unpublished CUDA kernels perform.  Only tests/, the
 * smoke check and bench.py's cpu_baseline / --impl reference legs load it.
 *
 * Math: PAPER.md:64-69 (Eq. 1), W = W0 + B·A with B ∈ R^{d×r}, A ∈ R^{r×k};
 * applied per token as y_t += scale · (x_t · A_{a(t)}ᵀ) · B_{a(t)}ᵀ (no α/r
 * factor in Eq. 1, so scale defaults to 1).
 *
 * Adapter dimensioning follows include/lorasim/adapter.hpp:15-23 and
 * src/adapter.cpp:22-26 (param_count = adapted · r · (d + k)); every weight
 * read goes through the per-adapter page table exactly as
 * PagePool::translate does (src/memory.cpp:55-62): logical page = off / P,
 * physical byte = entries[off / P] · P + off % P, with ceil(S/P) pages per
 * adapter (src/memory.cpp:14-16).
 *
 * In-adapter layout (the build's own contract; the reference fixes only S
 * and ceil(S/P)): for layer l in [0, L) and projection p in
 * [0, n_proj), in that order, one block [A (r × d_in[p], row-major) |
 * Bᵀ (r × d_out[p], row-major)].
 *
 * Rounding points mirror the CUDA path: v = x·Aᵀ is accumulated in double
 * and kept as fp32 (decode / BGMV semantics, v_bf16 = 0) or rounded to bf16
 * (prefill / SGMV semantics, v_bf16 = 1); Δy is accumulated in double and
 * y is rounded once to its storage type.
 *
 * Parity of this arithmetic is UNPINNED by the reference (no reference code
 * computes x·Aᵀ·Bᵀ); page tables fed to it come from the
 * reference PagePool itself (oracle/_ref).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_MAX_PROJ 8

typedef struct {
  uint32_t n_layers;
  uint32_t n_proj;
  uint32_t d_in[ORACLE_MAX_PROJ];
  uint32_t d_out[ORACLE_MAX_PROJ];
  uint32_t esize; /* 2 = bf16, 4 = fp32 */
} oracle_model;

static inline float bf16_to_f32(uint16_t h) {
  uint32_t u = ((uint32_t)h) << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

static inline uint16_t f32_to_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40u); /* quiet NaN */
  u += 0x7fffu + ((u >> 16) & 1u);                                           /* RNE */
  return (uint16_t)(u >> 16);
}

uint64_t oracle_block_elems(const oracle_model* m, uint32_t r, uint32_t proj) {
  return (uint64_t)r * ((uint64_t)m->d_in[proj] + m->d_out[proj]);
}

/* Byte offset of block (layer, proj) inside a rank-r adapter. */
uint64_t oracle_block_offset(const oracle_model* m, uint32_t r, uint32_t layer, uint32_t proj) {
  uint64_t per_layer = 0, before = 0;
  for (uint32_t p = 0; p < m->n_proj; ++p) {
    if (p < proj) before += oracle_block_elems(m, r, p);
    per_layer += oracle_block_elems(m, r, p);
  }
  return ((uint64_t)layer * per_layer + before) * m->esize;
}

/* S = adapted · r · (d + k) · bytes_per_param (src/adapter.cpp:22-26,52-59). */
uint64_t oracle_adapter_bytes(const oracle_model* m, uint32_t r) {
  uint64_t per_layer = 0;
  for (uint32_t p = 0; p < m->n_proj; ++p) per_layer += oracle_block_elems(m, r, p);
  return per_layer * m->n_layers * m->esize;
}

/* Scatter an adapter's logical bytes into a host image of the arena. */
void oracle_scatter_pages(uint8_t* arena, uint64_t page_bytes, const uint32_t* entries,
                          uint64_t n_entries, const uint8_t* src, uint64_t bytes) {
  for (uint64_t i = 0; i < n_entries; ++i) {
    uint64_t off = i * page_bytes;
    if (off >= bytes) break;
    uint64_t len = bytes - off < page_bytes ? bytes - off : page_bytes;
    memcpy(arena + (uint64_t)entries[i] * page_bytes, src + off, len);
  }
}

/* Gather an adapter's logical bytes back out of a host arena image. */
void oracle_gather_pages(const uint8_t* arena, uint64_t page_bytes, const uint32_t* entries,
                         uint64_t n_entries, uint8_t* dst, uint64_t bytes) {
  for (uint64_t i = 0; i < n_entries; ++i) {
    uint64_t off = i * page_bytes;
    if (off >= bytes) break;
    uint64_t len = bytes - off < page_bytes ? bytes - off : page_bytes;
    memcpy(dst + off, arena + (uint64_t)entries[i] * page_bytes, len);
  }
}

typedef struct {
  const oracle_model* m;
  const uint8_t* arena;
  uint64_t page_bytes;
  const uint32_t* entries;
  const uint64_t* table_off;
  const uint32_t* ranks;
  uint32_t layer, proj;
  const uint8_t* x;
  uint8_t* y;
  float scale;
  int v_bf16;
  /* segments: tokens grouped by adapter */
  uint32_t n_seg;
  const uint32_t* seg_adapter;
  const uint32_t* seg_start;
  const uint32_t* seg_tokens;
  volatile uint32_t next; /* work counter */
  pthread_mutex_t mu;
} job_t;

static inline double load_elem(const uint8_t* p, uint32_t es) {
  if (es == 2) {
    uint16_t h;
    memcpy(&h, p, 2);
    return (double)bf16_to_f32(h);
  }
  float f;
  memcpy(&f, p, 4);
  return (double)f;
}

static inline void store_elem(uint8_t* p, uint32_t es, double v) {
  if (es == 2) {
    uint16_t h = f32_to_bf16((float)v);
    memcpy(p, &h, 2);
  } else {
    float f = (float)v;
    memcpy(p, &f, 4);
  }
}

/* Physical address of logical byte `off` of adapter a (PagePool::translate). */
static inline const uint8_t* paged_addr(const job_t* J, uint32_t a, uint64_t off) {
  uint64_t logical = off / J->page_bytes;
  uint32_t phys = J->entries[J->table_off[a] + logical];
  return J->arena + (uint64_t)phys * J->page_bytes + off % J->page_bytes;
}

/* n consecutive elements of adapter a from logical byte `off`, translated
 * once per page (every element lies inside one page: pages are multiples
 * of the element size). */
static void load_row(const job_t* J, uint32_t a, uint64_t off, uint32_t n, double* out) {
  const uint32_t es = J->m->esize;
  uint32_t k = 0;
  while (k < n) {
    const uint64_t o = off + (uint64_t)k * es;
    const uint64_t in_page = o % J->page_bytes;
    uint64_t m = (J->page_bytes - in_page) / es;
    if (m > n - k) m = n - k;
    const uint8_t* p = paged_addr(J, a, o);
    for (uint64_t i = 0; i < m; ++i) out[k + i] = load_elem(p + i * es, es);
    k += (uint32_t)m;
  }
}

static void run_segment(job_t* J, uint32_t s) {
  const oracle_model* m = J->m;
  const uint32_t es = m->esize;
  const uint32_t a = J->seg_adapter[s];
  const uint32_t r = J->ranks[a];
  const uint32_t din = m->d_in[J->proj], dout = m->d_out[J->proj];
  const uint32_t t0 = J->seg_start[s], nt = J->seg_start[s + 1] - t0;
  const uint64_t blk = oracle_block_offset(m, r, J->layer, J->proj);
  const uint64_t boff = blk + (uint64_t)r * din * es; /* start of Bᵀ */

  double* v = (double*)calloc((size_t)nt * r, sizeof(double));
  double* acc = (double*)calloc((size_t)nt * dout, sizeof(double));
  double* row = (double*)malloc(sizeof(double) * (din > dout ? din : dout));
  double* xs = (double*)malloc(sizeof(double) * (size_t)nt * din);
  for (uint32_t i = 0; i < nt; ++i) { /* the segment's x rows, converted once */
    const uint8_t* xt = J->x + (uint64_t)J->seg_tokens[t0 + i] * din * es;
    for (uint32_t k = 0; k < din; ++k) xs[(uint64_t)i * din + k] = load_elem(xt + (uint64_t)k * es, es);
  }

  /* shrink: v[t][j] = sum_k x[t][k] · A[j][k] */
  for (uint32_t j = 0; j < r; ++j) {
    load_row(J, a, blk + (uint64_t)j * din * es, din, row);
    for (uint32_t i = 0; i < nt; ++i) {
      const double* xt = xs + (uint64_t)i * din;
      double sum = 0.0;
      for (uint32_t k = 0; k < din; ++k) sum += xt[k] * row[k];
      v[(uint64_t)i * r + j] = sum;
    }
  }
  /* rounding point of the intermediate (fp32 for BGMV, bf16 for SGMV) */
  for (uint64_t q = 0; q < (uint64_t)nt * r; ++q) {
    float f = (float)v[q];
    v[q] = J->v_bf16 ? (double)bf16_to_f32(f32_to_bf16(f)) : (double)f;
  }
  /* expand: acc[t][o] = sum_j v[t][j] · Bᵀ[j][o] */
  for (uint32_t j = 0; j < r; ++j) {
    load_row(J, a, boff + (uint64_t)j * dout * es, dout, row);
    for (uint32_t i = 0; i < nt; ++i) {
      double vj = v[(uint64_t)i * r + j];
      double* at = acc + (uint64_t)i * dout;
      for (uint32_t o = 0; o < dout; ++o) at[o] += vj * row[o];
    }
  }
  for (uint32_t i = 0; i < nt; ++i) {
    uint8_t* yt = J->y + (uint64_t)J->seg_tokens[t0 + i] * dout * es;
    const double* at = acc + (uint64_t)i * dout;
    for (uint32_t o = 0; o < dout; ++o) {
      uint8_t* p = yt + (uint64_t)o * es;
      store_elem(p, es, load_elem(p, es) + (double)J->scale * at[o]);
    }
  }
  free(v);
  free(acc);
  free(row);
  free(xs);
}

static void* worker(void* arg) {
  job_t* J = (job_t*)arg;
  for (;;) {
    pthread_mutex_lock(&J->mu);
    uint32_t s = J->next++;
    pthread_mutex_unlock(&J->mu);
    if (s >= J->n_seg) break;
    run_segment(J, s);
  }
  return NULL;
}

/* Paged LoRA apply over one (layer, proj).  token_adapter[t] < 0 = no LoRA.
 * Returns 0, or -1 on a malformed argument (unknown adapter / bad esize). */
int oracle_paged_lora_apply(const oracle_model* m, const uint8_t* arena, uint64_t page_bytes,
                            const uint32_t* entries, const uint64_t* table_off,
                            const uint32_t* ranks, uint32_t n_adapters, uint32_t layer,
                            uint32_t proj, const void* x, void* y, const int32_t* token_adapter,
                            uint32_t T, float scale, int v_bf16, int nthreads) {
  if (!m || (m->esize != 2 && m->esize != 4) || proj >= m->n_proj || layer >= m->n_layers)
    return -1;
  /* group tokens by adapter (stable: ascending key, then token order) */
  uint32_t* count = (uint32_t*)calloc(n_adapters + 1, sizeof(uint32_t));
  for (uint32_t t = 0; t < T; ++t) {
    int32_t a = token_adapter[t];
    if (a < 0) continue;
    if ((uint32_t)a >= n_adapters || ranks[a] == 0) {
      free(count);
      return -1;
    }
    count[a]++;
  }
  uint32_t n_seg = 0;
  for (uint32_t a = 0; a < n_adapters; ++a) n_seg += count[a] ? 1 : 0;
  uint32_t* seg_adapter = (uint32_t*)malloc(sizeof(uint32_t) * (n_seg + 1));
  uint32_t* seg_start = (uint32_t*)malloc(sizeof(uint32_t) * (n_seg + 1));
  uint32_t* seg_tokens = (uint32_t*)malloc(sizeof(uint32_t) * (T + 1));
  uint32_t* cursor = (uint32_t*)calloc(n_adapters + 1, sizeof(uint32_t));
  uint32_t s = 0, pos = 0;
  for (uint32_t a = 0; a < n_adapters; ++a) {
    if (!count[a]) continue;
    seg_adapter[s] = a;
    seg_start[s] = pos;
    cursor[a] = pos;
    pos += count[a];
    ++s;
  }
  seg_start[n_seg] = pos;
  for (uint32_t t = 0; t < T; ++t) {
    int32_t a = token_adapter[t];
    if (a >= 0) seg_tokens[cursor[a]++] = t;
  }

  job_t J;
  memset(&J, 0, sizeof(J));
  J.m = m;
  J.arena = arena;
  J.page_bytes = page_bytes;
  J.entries = entries;
  J.table_off = table_off;
  J.ranks = ranks;
  J.layer = layer;
  J.proj = proj;
  J.x = (const uint8_t*)x;
  J.y = (uint8_t*)y;
  J.scale = scale;
  J.v_bf16 = v_bf16;
  J.n_seg = n_seg;
  J.seg_adapter = seg_adapter;
  J.seg_start = seg_start;
  J.seg_tokens = seg_tokens;
  J.next = 0;
  pthread_mutex_init(&J.mu, NULL);
  if (nthreads < 1) nthreads = 1;
  if (nthreads == 1) {
    worker(&J);
  } else {
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nthreads);
    for (int i = 0; i < nthreads; ++i) pthread_create(&th[i], NULL, worker, &J);
    for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
    free(th);
  }
  pthread_mutex_destroy(&J.mu);
  free(count);
  free(cursor);
  free(seg_adapter);
  free(seg_start);
  free(seg_tokens);
  return 0;
}

/* Helpers exposed for tests: bf16 rounding as the oracle does it. */
uint16_t oracle_f32_to_bf16(float f) { return f32_to_bf16(f); }
float oracle_bf16_to_f32(uint16_t h) { return bf16_to_f32(h); }
