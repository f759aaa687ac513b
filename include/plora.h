/*
 * plora.h — C ABI of the B200-native P-LoRA hot path (libplora.so).
 *
 * This is the drop-in boundary.  Plain pointers and sizes only; no torch or
 * C++ types.  Every entry point names the reference interface it replaces as
 * file:line under /root/reference/proj (the lorasim C++ library; the paper's
 * GPU op that the reference only bills as a cost-model constant is cited to
 * PAPER.md).  INTEGRATION.md shows the ctypes / C++ bindings a maintainer adds.
 *
 * Error convention (reference: include/lorasim/errors.hpp:9-24,
 * src/memory.cpp:19-47): functions return int status codes.
 *   >= 0  success, or an AllocStatus value for plora_pool_alloc
 *         (memory.hpp:18-22: 0 ok, 1 out_of_memory, 2 fragmentation_failure)
 *   <  0  an error; plora_last_error() returns the message of the most recent
 *         error on the calling thread.  The C++ wrapper (plora.hpp) rethrows
 *         the same exception types the reference throws.
 *
 * Threading: one owner thread per pool/store.  Device work
 * is stream-ordered on the cudaStream_t the caller passes (NULL = legacy
 * default stream).
 */
#ifndef PLORA_H_
#define PLORA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ status */
#define PLORA_OK 0
#define PLORA_OUT_OF_MEMORY 1         /* AllocStatus::out_of_memory (memory.hpp:20) */
#define PLORA_FRAGMENTATION_FAILURE 2 /* AllocStatus::fragmentation_failure (memory.hpp:21) */
#define PLORA_E_VALIDATION (-1)       /* lorasim::ValidationError (errors.hpp:9-13)  */
#define PLORA_E_LOGIC (-2)            /* std::logic_error (memory.cpp:20-21,42-47)   */
#define PLORA_E_CONFIG (-3)           /* lorasim::ConfigError (errors.hpp:15-19)     */
#define PLORA_E_PARSE (-4)            /* lorasim::ParseError (errors.hpp:21-25)      */
#define PLORA_E_CUDA (-5)             /* CUDA runtime failure (new: device path)     */
#define PLORA_E_NOMEM (-6)            /* host allocation failure                     */

typedef void* plora_stream_t; /* a cudaStream_t, passed through opaquely */

/* Message of the last error raised on this thread ("" if none). */
const char* plora_last_error(void);
const char* plora_version(void);
/* Number of device kernels this process launched through libplora (all
 * entry points, all threads).  Evidence for bench.py's gpu_launches. */
uint64_t plora_kernel_launch_count(void);

/* ------------------------------------------------- adapter model (L1) ----
 * Replaces LoraDims::validate / param_count (include/lorasim/adapter.hpp:15-26,
 * src/adapter.cpp:12-26) and AdapterSizeTable (adapter.hpp:32-47,
 * src/adapter.cpp:28-50). */
int plora_lora_dims_validate(uint32_t d, uint32_t k, uint32_t r, uint32_t adapted_matrices,
                             uint32_t bytes_per_param);
int plora_param_count(uint32_t d, uint32_t k, uint32_t r, uint32_t adapted_matrices,
                      uint32_t bytes_per_param, uint64_t* out);

typedef struct plora_size_table plora_size_table;
/* AdapterSizeTable(anchor_rank, anchor_bytes, linear_fallback) (adapter.cpp:28-35);
 * anchor (8, 13 MiB, 1) is the reference default. */
int plora_size_table_create(uint32_t anchor_rank, uint64_t anchor_bytes, int linear_fallback,
                            plora_size_table** out);
void plora_size_table_destroy(plora_size_table* t);
int plora_size_table_set(plora_size_table* t, uint32_t rank, uint64_t bytes); /* adapter.cpp:37-40 */
int plora_size_table_bytes_for(const plora_size_table* t, uint32_t rank,
                               uint64_t* out); /* adapter.cpp:43-50 */
/* load_catalog_json (adapter.cpp:81-108): a JSON array of {"id": string,
 * "rank": uint[, "size_bytes": uint]}; bytes default to sizes (NULL = the
 * default table) at the rank; base dims d, k, adapted, bytes_per_param.
 * Fills up to cap entries (ranks, bytes, and ids as NUL-terminated strings
 * of at most id_stride - 1 bytes at ids_out + i·id_stride; any output may be
 * NULL) and returns the catalog size, or a negative status: ConfigError
 * (cannot open), ParseError (malformed, not an array, entry without id or
 * rank), ValidationError (empty catalog, invalid dims). */
int64_t plora_load_catalog_json(const char* path, const plora_size_table* sizes, uint32_t d,
                                uint32_t k, uint32_t adapted, uint32_t bytes_per_param,
                                uint32_t* ranks_out, uint64_t* bytes_out, char* ids_out,
                                uint64_t id_stride, uint64_t cap);
/* generate_catalog (adapter.cpp:110-144): ranks/bytes of `count` adapters
 * keyed 0..count-1 (ids "a000".. in catalog order).  sizes NULL = default table. */
int plora_generate_catalog(uint32_t count, const uint32_t* mix_ranks, const double* mix_weights,
                           uint64_t n_mix, uint64_t seed, const plora_size_table* sizes,
                           uint32_t d, uint32_t k, uint32_t adapted_matrices,
                           uint32_t bytes_per_param, uint32_t* ranks_out, uint64_t* bytes_out);

/* ---------------------------------------------------- page pool (L2) -----
 * Replaces lorasim::PagePool (include/lorasim/memory.hpp:39-83,
 * src/memory.cpp:7-146).  Placement is bit-identical to the reference:
 * alloc takes the lowest free physical indices (memory.cpp:18-38), compact
 * moves pages >= live into the lowest free slots walking adapter-key then
 * logical order (memory.cpp:71-89).  Backed by a two-level bitmap instead of
 * std::set, so alloc/free cost O(pages/64) instead of O(pages·log N). */
typedef struct plora_pool plora_pool;

typedef struct {
  double external_frag; /* FragmentationReport (memory.hpp:24-28) */
  double internal_frag;
  double utilization;
} plora_frag_report;

/* A compaction relocation (new: compact() in the reference returns only the
 * count, memory.cpp:71-89; the device needs the moves). */
typedef struct {
  uint32_t adapter;
  uint32_t logical;
  uint32_t src; /* physical page before */
  uint32_t dst; /* physical page after  */
} plora_reloc;

int plora_pool_create(uint64_t page_bytes, uint32_t total_pages,
                      plora_pool** out); /* memory.cpp:7-12 */
void plora_pool_destroy(plora_pool* p);
uint32_t plora_pool_pages_needed(const plora_pool* p, uint64_t bytes); /* memory.cpp:14-16 */
/* >= 0: AllocStatus (0 ok / 1 out_of_memory, pool unchanged);
 * PLORA_E_VALIDATION on 0 bytes; PLORA_E_LOGIC if already allocated.  memory.cpp:18-38 */
int plora_pool_alloc(plora_pool* p, uint32_t adapter, uint64_t weight_bytes);
int plora_pool_free(plora_pool* p, uint32_t adapter); /* memory.cpp:40-53; E_LOGIC on double free */
int plora_pool_translate(const plora_pool* p, uint32_t adapter, uint32_t logical,
                         uint32_t* phys); /* memory.cpp:55-62 */
/* PagePool::table (memory.cpp:64-69).  *entries stays valid until the next
 * mutation of the pool. */
int plora_pool_table(const plora_pool* p, uint32_t adapter, const uint32_t** entries,
                     uint32_t* n_entries, uint64_t* weight_bytes);
int plora_pool_has(const plora_pool* p, uint32_t adapter); /* memory.hpp:60 */
/* PagePool::compact (memory.cpp:71-89).  *moved = relocation count; the
 * relocation list stays readable through plora_pool_last_relocations. */
int plora_pool_compact(plora_pool* p, uint64_t* moved);
int plora_pool_last_relocations(const plora_pool* p, const plora_reloc** relocs, uint64_t* n);
void plora_pool_report(const plora_pool* p, plora_frag_report* out); /* memory.cpp:91-100 */
uint32_t plora_pool_free_pages(const plora_pool* p);                  /* memory.hpp:62 */
uint32_t plora_pool_total_pages(const plora_pool* p);                 /* memory.hpp:63 */
uint64_t plora_pool_page_bytes(const plora_pool* p);                  /* memory.hpp:64 */
uint64_t plora_pool_used_bytes(const plora_pool* p);                  /* memory.hpp:65 */
uint64_t plora_pool_allocated_bytes(const plora_pool* p);             /* memory.hpp:66-68 */
uint64_t plora_pool_total_bytes(const plora_pool* p);                 /* memory.hpp:69-71 */
/* PagePool::resident (memory.cpp:116-121): ascending keys; returns count. */
uint64_t plora_pool_resident(const plora_pool* p, uint32_t* out, uint64_t cap);
int plora_pool_check_invariants(const plora_pool* p); /* memory.cpp:123-146 */
/* PagePool::dump().dump() (memory.cpp:102-114): byte-identical JSON text.
 * Writes up to cap bytes (NUL-terminated when it fits); *len = full length. */
int plora_pool_dump(const plora_pool* p, char* buf, uint64_t cap, uint64_t* len);

/* ------------------------------------------- prefetch policy (L2) --------
 * Replaces include/lorasim/prefetch.hpp:11-72 / src/prefetch.cpp:1-114. */
typedef struct {
  double theta, alpha, beta, gamma, tau_ms, freq_half_life_ms, staging_fraction;
} plora_policy;

#define PLORA_NOT_RESIDENT 0 /* Residency (prefetch.hpp:23) */
#define PLORA_STAGING 1
#define PLORA_RESIDENT 2

typedef struct { /* AdapterDynamics (prefetch.hpp:26-37) */
  int32_t status;
  uint32_t busy;
  double last_access_ms;
  double decayed_count;
  double decay_stamp_ms;
  double prediction;
  int32_t transfer_active;
  int32_t reserved;
} plora_dynamics;

void plora_policy_default(plora_policy* p);     /* prefetch.hpp:11-21 defaults */
int plora_policy_validate(const plora_policy* p); /* prefetch.cpp:8-19 */
void plora_dynamics_init(plora_dynamics* d);
void plora_record_access(plora_dynamics* d, double now_ms, double half_life_ms); /* :21-25 */
double plora_decayed_at(const plora_dynamics* d, double now_ms, double half_life_ms); /* :27-32 */
double plora_recency_score(double last_access_ms, double now_ms, double tau_ms); /* :34-38 */
double plora_eviction_score(const plora_dynamics* d, const plora_policy* p, double now_ms,
                            double max_freq); /* :40-47 */
/* scored_residents (:49-64): ascending (score, key); returns count. */
uint64_t plora_scored_residents(const plora_dynamics* dyn, uint64_t n, const plora_policy* p,
                                double now_ms, double* scores, uint32_t* keys);
/* select_prefetch (:66-91): returns number of picks written to out. */
uint64_t plora_select_prefetch(const double* probabilities, uint64_t n_probs,
                               const plora_dynamics* dyn, uint64_t n, const plora_policy* p,
                               const uint64_t* units_for, uint64_t n_units,
                               uint64_t staging_budget_units, uint32_t* out);
/* plan_evictions (:93-112): returns 1 if satisfied, 0 if not. */
int plora_plan_evictions(uint64_t bytes_needed, uint64_t free_bytes, const uint32_t* eligible,
                         uint64_t n_eligible, const uint64_t* bytes_for, uint64_t n_bytes,
                         uint32_t* victims, uint64_t* n_victims);

/* ----------------------------------- synthetic workload (host input) -----
 * generate_synthetic (include/lorasim/workload.hpp:36-63, src/workload.cpp:59-144),
 * restated bit-identically (same libstdc++ engines/distributions).  Adapter
 * ids "a%0*d" are returned as their integer index. */
typedef struct {
  uint32_t num_adapters;
  double base_rate;
  double diurnal_amplitude;
  double period_s;
  uint32_t hot_set_size;
  double hot_rotation_s;
  double hot_share;
  double rotation_jitter;
  double burstiness_cv;
  double input_median, input_sigma, output_median, output_sigma;
  uint32_t max_tokens;
} plora_synthetic_profile;
void plora_synthetic_profile_default(plora_synthetic_profile* p); /* workload.hpp:19-50 */
/* Returns the number of requests (<0 on error); fills at most cap. */
int64_t plora_generate_synthetic(const plora_synthetic_profile* p, double duration_s,
                                 uint64_t seed, double* arrival_ms, uint32_t* adapter,
                                 uint32_t* input_tokens, uint32_t* output_tokens, uint64_t cap);

/* --------------------------------------- device adapter store (new) -----
 * The page pool's physical pages backed by ONE HBM arena
 * (total_pages · page_bytes, one cudaMalloc) plus a device page table and an
 * adapter directory.  Bookkeeping stays in the host plora_pool.
 *
 * Model shape: n_layers × n_proj adapted matrices (Llama-7B q/v: 32 × 2,
 * adapter.hpp:19 adapted_matrices = 64).  In-adapter layout, for l in
 * [0,L), p in [0,n_proj): block [A (r × d_in[p]) | Bᵀ (r × d_out[p])],
 * row-major; so S = r·L·Σ(d_in+d_out)·esize = param_count·bytes_per_param
 * (adapter.cpp:22-26,52-59). */
#define PLORA_MAX_PROJ 8
#define PLORA_BF16 0
#define PLORA_F32 1

typedef struct {
  uint32_t n_layers;
  uint32_t n_proj;
  uint32_t d_in[PLORA_MAX_PROJ];
  uint32_t d_out[PLORA_MAX_PROJ];
  uint32_t dtype; /* PLORA_BF16 or PLORA_F32: weights, x and y */
} plora_model;

uint64_t plora_model_adapter_bytes(const plora_model* m, uint32_t rank);
uint64_t plora_model_block_offset(const plora_model* m, uint32_t rank, uint32_t layer,
                                  uint32_t proj);

typedef struct plora_store plora_store;
/* pool is borrowed and must outlive the store; page_bytes must be a power of
 * two >= 16.  max_adapters bounds adapter keys (dense, AdapterKey memory.hpp:16). */
int plora_store_create(plora_pool* pool, int device, const plora_model* model,
                       uint32_t max_adapters, plora_store** out);
void plora_store_destroy(plora_store* s);
void* plora_store_arena(const plora_store* s); /* device base pointer */
/* Register adapter key -> rank (the AdapterSpec.dims.r, adapter.hpp:51-61). */
int plora_store_register(plora_store* s, uint32_t adapter, uint32_t rank);
int plora_store_rank(const plora_store* s, uint32_t adapter, uint32_t* rank);

#define PLORA_COPY_CE 0 /* copy engines: cudaMemcpyAsync per contiguous physical run;
                          src may be host (pinned or pageable) or device memory (UVA) */
#define PLORA_COPY_SM 1 /* SM page-scatter kernel reading mapped pinned host memory */
/* Page scatter H2D: copy the adapter's logical bytes (host, ideally pinned)
 * into its physical pages (pool table).  The reference models this transfer
 * as processor-shared PCIe time (src/engine.cpp:197-288); here it is real. */
int plora_store_write_pages(plora_store* s, uint32_t adapter, const void* host_src,
                            uint64_t bytes, int mode, plora_stream_t stream);
/* Gather the adapter's logical bytes back to host (parity checks). */
int plora_store_read_pages(plora_store* s, uint32_t adapter, void* host_dst, uint64_t bytes,
                           plora_stream_t stream);
/* Publish the adapter's page table to the device and mark it resident: the
 * promotion point of src/engine.cpp:406-414. */
int plora_store_publish(plora_store* s, uint32_t adapter, plora_stream_t stream);
/* Withdraw residency (before PagePool::free / eviction, src/engine.cpp:294-304). */
int plora_store_retire(plora_store* s, uint32_t adapter, plora_stream_t stream);
int plora_store_is_published(const plora_store* s, uint32_t adapter);
/* Apply compaction relocations on device (page_move_d2d) and republish the
 * affected tables (src/memory.cpp:71-89, idle trigger src/engine.cpp:486-497). */
int plora_store_apply_relocations(plora_store* s, const plora_reloc* relocs, uint64_t n,
                                  plora_stream_t stream);

/* ------------------------------------------------ host adapter store -----
 * The pinned host copy of every adapter the engine pages in (SURVEY §8(f)
 * row 4): one page-aligned pinned region with an offset index, optionally
 * file-backed ("PLHS": header, index, align-aligned images; opened with mmap
 * + cudaHostRegister).  Adapter sizes: plora_param_count (adapter.cpp:12-26);
 * the engine's transfer sources point into it (plora_engine_set_source). */
typedef struct plora_hoststore plora_hoststore;
int plora_hoststore_create(const uint64_t* bytes, const uint32_t* ranks, uint32_t n,
                           uint64_t align, plora_hoststore** out);
int plora_hoststore_open(const char* path, plora_hoststore** out);
int plora_hoststore_save(const plora_hoststore* s, const char* path);
void plora_hoststore_destroy(plora_hoststore* s);
uint32_t plora_hoststore_count(const plora_hoststore* s);
int plora_hoststore_entry(const plora_hoststore* s, uint32_t key, void** ptr, uint64_t* bytes,
                          uint32_t* rank);
int plora_hoststore_bytes(const plora_hoststore* s, uint64_t* data_bytes);

/* --------------------------------------- paged LoRA forward op (new) -----
 * The op the reference bills as cost_model prefill_ms / step_ms
 * (include/lorasim/cost_model.hpp:32-40 at src/engine.cpp:355,510);
 * math PAPER.md:64-69.  A batch plan groups tokens by adapter once per batch
 * and is reused for every (layer, proj) call of the step. */
typedef struct plora_plan plora_plan;
/* token_adapter: HOST array, adapter key per token or -1 (no LoRA).  Every
 * referenced adapter must be published.  Uploads the plan on `stream`. */
int plora_plan_create(plora_store* s, const int32_t* token_adapter, uint32_t n_tokens,
                      plora_stream_t stream, plora_plan** out);
/* Rebuild an existing plan for a new batch, reusing its buffers. */
int plora_plan_update(plora_plan* plan, const int32_t* token_adapter, uint32_t n_tokens,
                      plora_stream_t stream);
void plora_plan_destroy(plora_plan* plan);
uint32_t plora_plan_num_segments(const plora_plan* plan);

/* y[t, :] += scale · (x[t, :] · Aᵀ) · Bᵀ for every token, A/B of adapter
 * a(t) at (layer, proj) read through the device page table.  x: [T, d_in]
 * with row stride x_stride elements; y: [T, d_out] with row stride y_stride.
 * The intermediate v = x·Aᵀ is kept in fp32. */
int plora_bgmv(plora_plan* plan, uint32_t layer, uint32_t proj, const void* x,
               uint64_t x_stride, void* y, uint64_t y_stride, float scale,
               plora_stream_t stream);
/* Every projection p of `layer` at once (they read the same x, as q/k/v of
 * an attention block do): ys[p] += scale · (x · A_pᵀ) · B_pᵀ with row stride
 * y_strides[p].  bf16 stores with equal input widths: one shrink launch and
 * one expand launch for all projections (bgmv_warp.cu), bit-identical to
 * per-projection plora_bgmv calls; else one plora_bgmv per projection. */
int plora_bgmv_layer(plora_plan* plan, uint32_t layer, const void* x, uint64_t x_stride,
                     void* const* ys, const uint64_t* y_strides, float scale,
                     plora_stream_t stream);
/* Layers [layer0, layer0 + n_layers) of plora_bgmv_layer in one call, for
 * inputs that are all ready (a LoRA-only decode step, speculative/multi-layer
 * batching): one shrink launch and one expand launch cover every layer
 * (bgmv_warp.cu; the layers' work items interleaved, heaviest first), so the
 * per-launch ramp and drain are paid once.  Layer layer0 + i reads
 * x + i·x_layer_stride and updates ys[p] + i·y_layer_strides[p] (all strides
 * in elements).  Deterministic and bit for bit equal to n_layers
 * plora_bgmv_layer calls.  bf16 stores with equal input widths; otherwise one
 * plora_bgmv_layer per layer.  (plora_debug_set_bgmv_impl selects the
 * cluster kernel or the round-2 hybrid pair of clusters + streaming kernel.) */
int plora_bgmv_layers(plora_plan* plan, uint32_t layer0, uint32_t n_layers, const void* x,
                      uint64_t x_stride, uint64_t x_layer_stride, void* const* ys,
                      const uint64_t* y_strides, const uint64_t* y_layer_strides, float scale,
                      plora_stream_t stream);
/* Same contract, prefill path (tcgen05 tensor cores; v rounded to the
 * storage dtype between shrink and expand). */
int plora_sgmv(plora_plan* plan, uint32_t layer, uint32_t proj, const void* x,
               uint64_t x_stride, void* y, uint64_t y_stride, float scale,
               plora_stream_t stream);
/* Every projection of `layer` at once, prefill path (as plora_bgmv_layer):
 * with two projections of equal shape the shrink reads each x chunk once
 * for both and one expand launch covers both; otherwise one plora_sgmv
 * call per projection. */
int plora_sgmv_layer(plora_plan* plan, uint32_t layer, const void* x, uint64_t x_stride,
                     void* const* ys, const uint64_t* y_strides, float scale,
                     plora_stream_t stream);
/* Prefill with the base projection fused in: for every
 * token row t of the plan (with or without an adapter)
 *   y[t] = x[t] · W0ᵀ + bf16(scale · x[t] · A_{a(t)}ᵀ) · B_{a(t)}ᵀ
 * w0: the base weight [d_out, d_in] (row stride w0_stride elements), y is
 * overwritten.  bf16 store, rank <= 128, d_in % 64 == 0, d_out % 256 == 0. */
int plora_sgmv_fused(plora_plan* plan, uint32_t layer, uint32_t proj, const void* x,
                     uint64_t x_stride, const void* w0, uint64_t w0_stride, void* y,
                     uint64_t y_stride, float scale, plora_stream_t stream);
/* Every projection of `layer` (they share x): one shrink for both when their
 * shapes allow (x read once), then one fused GEMM per projection.
 * w0s[p] / w0_strides[p]: projection p's base weight [d_out, d_in]. */
int plora_sgmv_fused_layer(plora_plan* plan, uint32_t layer, const void* x, uint64_t x_stride,
                           const void* const* w0s, const uint64_t* w0_strides, void* const* ys,
                           const uint64_t* y_strides, float scale, plora_stream_t stream);

/* ------------------- tensor-parallel decode (new; BASELINE cfg5) -----
 * The S-LoRA scheme for a column-parallel base projection (hidden-dim
 * sharded 70B config; the reference has no multi-GPU path).
 * TP rank i of N shrinks rows [i·r/N, (i+1)·r/N) of every adapter into
 * v_part [n_tokens × rs] fp32 (rs = plora_tp_shard_rows), the caller
 * all-gathers v_part over the TP group into v_gathered [N][n_tokens][rs]
 * (rank-major, e.g. ncclAllGather), and the expand adds
 * scale · v · Bᵀ[:, i·d_out/N : (i+1)·d_out/N] into the rank's output shard
 * y_shard [n_tokens × d_out/N].  Every adapter rank must be divisible by N;
 * bf16 stores only.  Kernels: warp items (bgmv_warp.cu) — K-sliced shrink
 * items whose per-job partial sums are added in slice order by the job's
 * last item (deterministic), column-shard expand items. */
uint32_t plora_tp_shard_rows(const plora_plan* plan, uint32_t tp_size);
int plora_bgmv_tp_shrink(plora_plan* plan, uint32_t layer, uint32_t proj, uint32_t tp_rank,
                         uint32_t tp_size, const void* x, uint64_t x_stride, float* v_part,
                         plora_stream_t stream);
int plora_bgmv_tp_expand(plora_plan* plan, uint32_t layer, uint32_t proj, uint32_t tp_rank,
                         uint32_t tp_size, const float* v_gathered, void* y_shard,
                         uint64_t y_stride, float scale, plora_stream_t stream);
/* The all-gather fused into the shrink (peer-write, no collective call).
 * Each rank holds v_gathered [tp_size][n_tokens][rs] fp32 and a flag array of
 * tp_size uint32 (zero-initialised), both in memory every rank can address
 * (CUDA IPC / symmetric memory over NVLink; peer_*[d] = rank d's copy).
 * shrink_push stores this rank's v rows straight into every rank's
 * v_gathered (block tp_rank) as they are produced; its last CTA then adds 1
 * to slot tp_rank of every rank's flag array (release, system scope).
 * expand_wait waits until every slot of the local flag array is >= 1
 * (acquire), expands, and its last CTA takes 1 from every slot — so the
 * protocol is the same on every call and CUDA-graph replays are safe.  A
 * rank's v_gathered may be rewritten by a peer's next call once that peer
 * passed this rank's expand: callers alternate two buffers by call parity
 * (an even number of calls per captured graph).  tp_size <= 8. */
int plora_bgmv_tp_shrink_push(plora_plan* plan, uint32_t layer, uint32_t proj, uint32_t tp_rank,
                              uint32_t tp_size, const void* x, uint64_t x_stride,
                              float* const* peer_v_gathered, uint32_t* const* peer_flags,
                              plora_stream_t stream);
int plora_bgmv_tp_expand_wait(plora_plan* plan, uint32_t layer, uint32_t proj, uint32_t tp_rank,
                              uint32_t tp_size, const float* v_gathered, uint32_t* flags,
                              void* y_shard, uint64_t y_stride, float scale, plora_stream_t stream);

/* ------------------------------------ loading / prefetch engine (new) -----
 * The reference simulator's residency control restated on CUDA streams and
 * events: Simulation::ensure_loading / evict (src/engine.cpp:292-333),
 * transfers (:197-288), do_boundary / admit_requests / issue_prefetches /
 * maybe_compact (:406-497), on_arrival / on_round (:515-571).  Transfers
 * are real page scatters of caller-owned pinned host images; demand loads
 * run on a high-priority stream and preempt prefetch at chunk granularity;
 * prefetched adapters are promoted (device table published) at the next
 * boundary.  One owner thread per engine; the engine's own pump thread
 * keeps prefetch copies flowing between boundaries. */
#define PLORA_COPY_AUTO 2 /* CE for pages >= 64 KiB, SM scatter kernel below */
#define PLORA_ADMIT_LOADING 0 /* weights in flight (demand priority) */
#define PLORA_ADMIT_READY 1   /* resident and published */
#define PLORA_ADMIT_FAILED 2  /* could not allocate (engine.cpp:427-431) */
typedef struct {
  plora_policy policy;
  int32_t copy_mode;  /* PLORA_COPY_CE / _SM / _AUTO */
  int32_t prefetch;   /* issue_prefetches enabled (RunConfig policy.prefetch) */
  int32_t compaction; /* idle compaction (engine.cpp:486-497) */
  int32_t reserved;
  uint64_t chunk_bytes;             /* prefetch issue granularity */
  uint64_t prefetch_inflight_bytes; /* prefetch bytes in flight at most */
} plora_engine_config;
typedef struct { /* MetricsReport counters (include/lorasim/engine.hpp:66-98) */
  uint64_t arrivals, hits, demand_loads, prefetch_issued, promotions, evictions;
  uint64_t admission_failures, upgrades, compactions, relocations, prediction_rounds;
  uint64_t transfers_completed, bytes_h2d;
  double transfer_ms;        /* Σ per-transfer device time (first chunk -> done) */
  double demand_transfer_ms; /* the demand share of it */
  double predictor_ms;       /* async predictor worker busy time */
  uint64_t in_flight, staged, resident;
  int32_t copy_mode, reserved;
  /* per-interval prediction accuracy (engine.cpp:598-633): Σ tp/(tp+fp+fn)
   * over the scored intervals, their count, and the summed tp / fp / fn */
  double acc_sum;
  uint64_t acc_intervals, acc_tp, acc_fp, acc_fn;
} plora_engine_stats;
/* One decision-log row (DecisionLogRow, include/lorasim/engine.hpp:61;
 * engine.cpp:304, 330, 412, 435, 495): action, adapter (0xffffffff: none),
 * time, score (eviction score / prefetch probability) and a detail value
 * (bytes for loads, relocations for compact). */
#define PLORA_DECISION_EVICT 0
#define PLORA_DECISION_PREFETCH 1
#define PLORA_DECISION_DEMAND_LOAD 2
#define PLORA_DECISION_PROMOTE 3
#define PLORA_DECISION_ADMISSION_FAILURE 4
#define PLORA_DECISION_COMPACT 5
typedef struct {
  double t_ms, score;
  uint32_t adapter, action;
  uint64_t detail;
} plora_decision;
typedef struct plora_engine plora_engine;
typedef struct plora_predictor plora_predictor;
void plora_engine_config_default(plora_engine_config* c);
int plora_engine_create(plora_store* s, const plora_engine_config* cfg, plora_engine** out);
void plora_engine_destroy(plora_engine* e);
/* Host image of a registered adapter (plora_model_adapter_bytes(rank) bytes,
 * caller-owned; pinned for PLORA_COPY_SM and for asynchronous CE copies). */
int plora_engine_set_source(plora_engine* e, uint32_t adapter, const void* host_src,
                            uint64_t bytes);
/* NULL detaches.  async = 0: observe/predict_all run inline (the
 * reference's synchronous semantics).  async = 1: a worker thread owns the
 * predictor; a round applies the last completed prediction set and requests
 * the next (one round of lag), keeping the LSTM off the decode loop. */
int plora_engine_attach_predictor(plora_engine* e, plora_predictor* p, int async);
/* Wait for the async predictor to drain queued observations and finish the
 * requested round, then apply its predictions. */
int plora_engine_flush_predictor(plora_engine* e);
/* Request arrival (engine.cpp:515-545): access statistics, predictor
 * observation, reactive demand load.  Returns 1 if resident at arrival. */
int plora_engine_on_arrival(plora_engine* e, uint32_t adapter, double now_ms,
                            plora_stream_t compute);
/* Prediction round (engine.cpp:547-561): predict_all of the attached predictor. */
int plora_engine_round(plora_engine* e, double now_ms, plora_stream_t compute);
/* External predictions (oracle mode, engine.cpp:562-571); -1 = no prediction. */
int plora_engine_set_predictions(plora_engine* e, const double* probs, uint64_t n);
/* Admission (engine.cpp:416-457): PLORA_ADMIT_READY / _LOADING / _FAILED;
 * pins the adapter (busy) until plora_engine_release. */
int plora_engine_acquire(plora_engine* e, uint32_t adapter, double now_ms,
                         plora_stream_t compute);
/* Make `compute` wait (device-side) for a loading adapter and publish it. */
int plora_engine_wait_ready(plora_engine* e, uint32_t adapter, plora_stream_t compute);
int plora_engine_release(plora_engine* e, uint32_t adapter); /* finish_request :358-372 */
/* Batch boundary (engine.cpp:406-414): completions, promotions, prefetch
 * issue, idle compaction.  Table updates are ordered on `compute`.
 * Returns the number of transfers observed complete. */
int plora_engine_boundary(plora_engine* e, double now_ms, plora_stream_t compute);
/* Batched forms for a serving loop: arrivals (returns the hit count),
 * admission of distinct adapters (status per entry; wait != 0 makes
 * `compute` wait device-side for loading ones), release. */
int64_t plora_engine_on_arrivals(plora_engine* e, const uint32_t* adapters, uint64_t n,
                                 double now_ms, plora_stream_t compute);
int plora_engine_admit(plora_engine* e, const uint32_t* adapters, uint64_t n, double now_ms,
                       plora_stream_t compute, int wait, int32_t* status);
int plora_engine_release_many(plora_engine* e, const uint32_t* adapters, uint64_t n);
int plora_engine_sync(plora_engine* e); /* wait for every issued copy */
int plora_engine_status(const plora_engine* e, uint32_t adapter, plora_dynamics* out);
void plora_engine_get_stats(const plora_engine* e, plora_engine_stats* out);
/* Decision log rows [start, start + cap) into out; returns the total count. */
uint64_t plora_engine_decisions(const plora_engine* e, uint64_t start, plora_decision* out,
                                uint64_t cap);
int plora_engine_set_decision_log(plora_engine* e, int enabled); /* default on; off clears */
/* Interval length and warm-up of the accuracy scoring (predictor interval_ms,
 * run.warmup_s); defaults 1000 ms and 0. */
int plora_engine_set_accuracy_interval(plora_engine* e, double interval_ms, double warmup_ms);
int plora_engine_streams(const plora_engine* e, plora_stream_t* demand, plora_stream_t* prefetch);

/* ----------------------------------------------- demand predictor (host) ---
 * The LSTM that drives predictor-based prefetch: PredictorModel
 * (include/lorasim/lstm.hpp:11-85) and OnlinePredictor
 * (include/lorasim/predictor.hpp:12-111).  Same parameter layout, seeded
 * initialisation, BPTT, Adam and LSW1 file format; windows are row-major
 * [n, window] doubles. */
typedef struct {
  uint32_t window, hidden, layers, embedding_dim, num_adapters;
  double learning_rate, adam_beta1, adam_beta2, adam_eps;
} plora_lstm_config; /* PredictorConfig, lstm.hpp:19-33 */
typedef struct {
  plora_lstm_config model;
  double interval_ms;
  uint32_t train_every, batch_size, replay_capacity;
} plora_predictor_config; /* OnlinePredictorConfig, predictor.hpp:45-51 */
void plora_lstm_config_default(plora_lstm_config* c);
void plora_predictor_config_default(plora_predictor_config* c);
/* Summed clamped binary cross-entropy (lstm.hpp:35-37). */
int plora_cross_entropy(const double* p, const double* y, uint64_t n, double* out);

typedef struct plora_lstm plora_lstm;
int plora_lstm_create(const plora_lstm_config* cfg, uint64_t seed, plora_lstm** out);
void plora_lstm_destroy(plora_lstm* m); /* no-op for predictor-owned models */
uint64_t plora_lstm_param_count(const plora_lstm* m);
double* plora_lstm_parameters(plora_lstm* m); /* mutable view of θ */
void plora_lstm_get_config(const plora_lstm* m, plora_lstm_config* out);
int plora_lstm_forward(const plora_lstm* m, const uint32_t* adapters, const double* windows,
                       uint64_t n, double* probs);
int plora_lstm_loss(const plora_lstm* m, const uint32_t* adapters, const double* windows,
                    const double* labels, uint64_t n, double* out);
int plora_lstm_gradient(const plora_lstm* m, const uint32_t* adapters, const double* windows,
                        const double* labels, uint64_t n, double* grad);
int plora_lstm_train_step(plora_lstm* m, const uint32_t* adapters, const double* windows,
                          const double* labels, uint64_t n, double* loss);
int plora_lstm_save(const plora_lstm* m, const char* path);
int plora_lstm_load(const char* path, plora_lstm** out);

int plora_predictor_create(const plora_predictor_config* cfg, uint64_t seed,
                           plora_predictor** out);
void plora_predictor_destroy(plora_predictor* p);
plora_lstm* plora_predictor_model(plora_predictor* p); /* borrowed */
int plora_predictor_observe(plora_predictor* p, uint32_t adapter, double t_ms);
int plora_predictor_roll_to(plora_predictor* p, double t_ms);
/* 1 = trained one batch (loss written), 0 = replay buffer empty. */
int plora_predictor_train_step(plora_predictor* p, double* loss);
/* Predictions for every known adapter in key order; returns the count (may
 * exceed cap; only cap entries written) or a negative status. */
/* Run predict_all's LSTM forward on CUDA device `device` (FP64, the same
 * summation order as the host path; differs only by exp/tanh rounding), or
 * on the host threads (device = -1, the default).  New for the 100 ms
 * prediction round at production adapter counts. */
int plora_predictor_set_device(plora_predictor* p, int device);
int64_t plora_predictor_predict_all(plora_predictor* p, double now_ms, uint32_t* adapters,
                                    double* probs, uint64_t cap);
int plora_predictor_window(const plora_predictor* p, uint32_t adapter, double* out);
/* 1 if the adapter has been observed (OnlinePredictor::known, predictor.hpp:77). */
int plora_predictor_known(const plora_predictor* p, uint32_t adapter);
typedef struct {
  uint64_t observed, train_steps, known, buffered;
  int64_t current_interval;
  double last_loss;
} plora_predictor_stats_t;
void plora_predictor_stats(const plora_predictor* p, plora_predictor_stats_t* out);
/* Replay buffer entry i (0 = oldest): ReplayBuffer::at (predictor.hpp:31). */
int plora_predictor_buffer_at(const plora_predictor* p, uint64_t i, uint32_t* adapter,
                              double* window, double* label);

/* ------------------------------------------------------------ diagnostics
 * Device timestamps of the next decode / prefill launches, for the
 * diagnostics scripts: cluster kernel (scripts/trace_bgmv.py), streaming
 * kernel (scripts/trace_stream.py), single-layer warp-item calls (per item
 * start / end %globaltimer, scripts/trace_warp_layer.py), persistent SGMV
 * expand (scripts/trace_sgmv_expand.py).  dev_buf = NULL disables tracing. */
int plora_debug_set_trace(void* dev_buf, uint64_t bytes);
/* Diagnostics: the bf16 decode kernel behind plora_bgmv* — 0 warp items
 * (bgmv_warp.cu, the default); 1 the streaming kernel alone (bgmv_stream.cu);
 * 2 thread-block clusters only (bgmv_cluster.cu); 3 clusters with the hybrid
 * streaming share for plora_bgmv_layers (the round-2 pair).  Applies to plans
 * built afterwards for the hybrid split.  The tensor-parallel halves run on
 * warp items, or on the streaming kernel with impl 1. */
int plora_debug_set_bgmv_impl(int impl);
/* Diagnostics for the streaming kernel: 1 consumers skip the math, 2 no
 * weight copies (results are then wrong; timing ablation only). */
int plora_debug_set_bgmv_flags(uint32_t flags);
/* Diagnostics: L2 bulk prefetch of the streaming decode kernel's weight rows
 * two items ahead of its shared-memory ring (1) or off (0, the default:
 * measured slower, profiles/r02i_stream_prefetch_ablation.txt). */
int plora_debug_set_stream_prefetch(uint32_t on);
/* Diagnostics: plans built afterwards give the streaming kernel at most
 * `ctas` CTAs (0 = one per SM). */
int plora_debug_set_stream_ctas(uint32_t ctas);
/* Adapters with at least `min_tokens` tokens in a decode batch leave the
 * decode kernels for the tensor-core SGMV path (their tokens gathered into a
 * child plan, run concurrently on a second stream).  Applies to plans built
 * afterwards; 0 disables.  Default 160 (profiles/r02o_route_warp.txt). */
int plora_debug_set_route_tokens(uint32_t min_tokens);
/* Tokens of the plan's batch that take the routed SGMV path. */
int plora_debug_plan_routed(const plora_plan* plan, uint32_t* n_tokens);
/* Diagnostics: the hybrid decode launch's streaming share = spare SMs / SMs ×
 * factor of the weight rows (default 0.95; plans built afterwards), and a
 * plan's split: {spare SMs, share fraction, clusters, streaming CTAs}. */
int plora_debug_set_hybrid_share(double factor);
int plora_debug_plan_hybrid(const plora_plan* plan, double out[4]);
/* Diagnostics: also run plora_bgmv_layer (one layer) as the hybrid pair. */
int plora_debug_set_hybrid_per_layer(int on);
/* Launch geometry the plan chose for the bf16 decode op of projection
 * `proj`: out[0..7] = {cluster size, input slice, output slice, A-row ring
 * slots, Bᵀ-row ring slots, dynamic smem bytes, clusters, chunks}. */
int plora_debug_plan_geom(const plora_plan* plan, uint32_t proj, uint32_t out[8]);
/* Timing experiments only (results are wrong while set): the next SGMV
 * shrink launches skip their 1 = weight gathers, 2 = MMAs, 4 = x loads,
 * 16 = epilogue; 32 = the split reduction launch, 8 = the expand launch;
 * the expand skips its 64 = y reduce-adds, 128 = Bᵀ gathers, 256 = MMAs,
 * 512 = everything after its prologue.  0 restores the op. */
int plora_debug_set_sgmv_flags(uint32_t flags);

#ifdef __cplusplus
}
#endif
#endif /* PLORA_H_ */
