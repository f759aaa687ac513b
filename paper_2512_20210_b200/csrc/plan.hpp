// Batch plan: tokens grouped by adapter (segments) and the work lists the
// persistent kernels consume.  Built on the host once per batch and reused
// for every (layer, proj) call of the step — the "translation once per
// batch" of PAPER.md:136.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <vector>

#include "store.hpp"

namespace plora {

// ---------------------------------------------------------------- BGMV
constexpr uint32_t kExpandBit = 0x80000000u;
constexpr uint32_t kStopUnit = 0xffffffffu;
constexpr uint32_t kMaxUnitTok = 4;           // tokens per work unit
constexpr uint32_t kShrinkWeightBytes = 32768;  // A rows per shrink unit
constexpr uint32_t kSlotWeightBytes = 32768;    // Bᵀ tile per expand CTA
constexpr uint32_t kSlotAuxBytes = 16384;       // x rows (shrink) / y rows (expand)
constexpr uint32_t kMaxShrinkRows = 8;          // one warp per rank row
constexpr uint32_t kMaxBgmvRank = 256;

// A BGMV work unit, fully resolved on the host (64 bytes): the producer warp
// needs no dependent loads besides the page table.
struct BgmvUnit {
  uint32_t kind_seg;  // segment | kExpandBit for expand units
  uint32_t off;       // first rank row (shrink) or first output column (expand)
  uint32_t count;     // rows (shrink) or columns (expand)
  uint32_t table_off; // adapter's first entry in the device page table
  uint32_t rank;
  uint32_t voff;      // fp32 index of v for this unit's first token (row stride rpad4)
  uint32_t ntok;      // tokens (<= kMaxUnitTok)
  uint32_t n_shrink;  // expand: shrink units of the segment to wait for
  uint32_t tok[kMaxUnitTok];  // x / y row indices
  uint32_t kc;        // shrink: K chunk (0: full rows)
  uint32_t nkc;       // expand: number of K-chunk partial planes of v to sum (1)
  uint32_t vstride;   // expand: floats between consecutive partial planes
  uint32_t pad;
};
static_assert(sizeof(BgmvUnit) == 64, "BgmvUnit layout");

// Expand split: RG row groups × CT column threads (RG·CT = kBgmvConsumers),
// CB = CT · VEC columns, so the Bᵀ tile r × CB fits one 32 KiB slot and a
// thread holds <= 8 rank rows.
constexpr uint32_t kBgmvConsumers = 256;
constexpr uint32_t kRedBytes = 16384;  // expand cross-group reduction buffer
#ifdef __CUDACC__
__host__ __device__
#endif
inline uint32_t expand_rg(uint32_t rank) {
  uint32_t rg = 1;
  while (rg * 8 < rank) rg <<= 1;
  return rg;  // <= 32 for rank <= 256
}

#ifdef __CUDACC__
__host__ __device__
#endif
inline uint32_t rpad4(uint32_t r) { return (r + 3) & ~3u; }

// Columns per fp32 expand unit: RG·CB = 256 threads × 4 columns.
#ifdef __CUDACC__
__host__ __device__
#endif
inline uint32_t expand_cols(uint32_t rank, uint32_t esize) {
  if (esize == 2) {
    const uint32_t r16 = (rank + 15) & ~15u;
    uint32_t cb = 1024;
    while (cb * r16 > 16384) cb >>= 1;
    return cb;  // 1024 (r <= 16) ... 64 (r <= 256)
  }
  return (kBgmvConsumers / expand_rg(rank)) * 4;
}

struct ProjWork {
  uint32_t n_units = 0;
  uint32_t n_shrink = 0;   // units [0, n_shrink) are shrink, the rest expand
  uint32_t units_off = 0;  // into the unit array
};

// ------------------------------------------------ bf16 BGMV (clusters)
// A job = one adapter's tokens (<= kJobTok of them) at one (layer, proj);
// it is cut into chunks of <= kChunkRows rank rows.  Every CTA of a cluster
// of CS CTAs walks the same chunk list, CTA c owning input slice c (shrink,
// K-split) and output slice c (expand, N-split); partial v rows cross the
// cluster through distributed shared memory.
constexpr uint32_t kJobTok = 4;
constexpr uint32_t kChunkRows = 8;
constexpr uint32_t kChunkFirst = 1, kChunkLast = 2;
// the job's adapter has further jobs in the batch (more than kJobTok tokens):
// its pages are read again, so they are kept in L2 (evict_last) instead of
// streamed through it (evict_first)
constexpr uint32_t kChunkReuse = 4;

struct ClusterJob {  // 32 bytes; uploaded for the tensor-parallel path (tp.cu)
  uint32_t table_off;
  uint32_t rank;
  uint32_t ntok;
  uint32_t pad;
  uint32_t tok[kJobTok];
};
static_assert(sizeof(ClusterJob) == 32, "ClusterJob layout");

// Self-contained chunk record (32 bytes): the kernel's producer loads it
// ahead of time and forwards it to the consumers through shared memory, so
// no consumer ever waits on a dependent global load.
struct ClusterChunk {
  uint32_t table_off;  // adapter's first entry in the device page table
  uint16_t rank;
  uint8_t ntok;
  uint8_t flags;       // kChunkFirst | kChunkLast of the job
  uint16_t row0;
  uint8_t nrows;
  uint8_t proj;        // index into the launch's projection list (plora_bgmv_layer)
  uint32_t jord;       // job ordinal within the cluster's list (job buffer jord & 1)
  uint32_t tok[kJobTok];  // x / y row of each job token
};
static_assert(sizeof(ClusterChunk) == 32, "ClusterChunk layout");

// Launch geometry of one projection (host-side, decided at plan build).
struct ClusterGeom {
  uint32_t cs = 0;          // CTAs per cluster
  uint32_t ks = 0, ns = 0;  // input / output slice widths (elements)
  uint32_t na = 0, nbs = 0;         // ring depths: A-row slots, Bᵀ-row slots
  uint32_t a_bytes = 0, b_bytes = 0;  // slot sizes
  uint32_t jb_bytes = 0, smem = 0;
  uint32_t n_clusters = 0;  // clusters launched (<= co-resident clusters)
};
ClusterGeom cluster_geom(uint32_t d_in, uint32_t d_out, int device);

struct ClusterWork {
  ClusterGeom geom;
  uint32_t chunks_off = 0;  // into the chunk array
  uint32_t cl_off = 0;      // into the cluster offset array (n_clusters + 1 entries)
};

// ------------------------------------------------ bf16 BGMV (streaming)
// bgmv_stream.cu: persistent, one CTA per SM, no cross-CTA exchange.  A job
// is <= JT tokens of one adapter at one (layer, proj).  Its shrink is cut
// into S items (<= 16 rank rows, full K: v = x·A[rows]ᵀ exact in fp32, written
// to a v plane) and its expand into E items (one column block of <= 1024
// output columns, all rank rows: y[:, block] += scale · v · Bᵀ[:, block]);
// an E item waits (acquire) on its job's v counter.  Every item streams
// 16 weight rows × <= 1024 elements per stage.
constexpr uint32_t kStreamKC = 1024;     // elements per stage row segment
constexpr uint32_t kStreamExpand = 0x80000000u;
struct StreamItem {  // 64 bytes, fully resolved on the host
  uint32_t kind;       // kStreamExpand | launch projection index
  uint32_t job;        // job index (counter slot within a (layer, proj) plane)
  uint32_t table_off;  // adapter's first entry in the device page table
  uint32_t rank_ntok;  // rank | ntok << 16
  uint32_t off;        // S: first rank row; E: first output column
  uint32_t n;          // S: rank rows (<= 16); E: columns (<= kStreamKC)
  uint32_t v_off;      // floats into a v plane: the job's [rank][JT] block
  uint32_t ns_ne;      // v elements of the job (rank · ntok, each released by its own store) | E items << 16
  uint32_t tok[8];     // x / y rows of the job's tokens
};
static_assert(sizeof(StreamItem) == 64, "StreamItem layout");

constexpr uint32_t kMaxTp = 8;  // TP ranks of the fused peer-write all-gather
struct StreamTp {  // a tensor-parallel half on the streaming kernel (tp.cu)
  uint32_t mode;      // 1 shrink (S items; v -> v_out), 2 expand (E items; v from v_in)
  uint32_t tp_size, n_tokens, rs_max;
  float* v_out;
  const float* v_in;
  const StreamItem* items;
  const uint32_t* cta_off;
  // fused all-gather.  Shrink: v rows also go straight into every rank's
  // gathered buffer (peer memory; rank block already applied), then the last
  // CTA adds 1 to this rank's slot of every rank's flag array.  Expand: wait
  // until every slot of the local flag array is >= 1, and the last CTA takes
  // 1 from each (consumed: graph replays see the same protocol).
  uint32_t n_dst;
  float* dst[kMaxTp];
  uint32_t* flags[kMaxTp];  // shrink: &flag_array_of_rank_d[tp_rank]
  uint32_t* done;           // this launch's CTA-completion counter (zero between calls)
  uint32_t* wait;           // expand: the local flag array [tp_size]
};

struct StreamWork {  // one launch variant (a projection, or every projection of a layer)
  uint32_t items_off = 0;  // into the item array
  uint32_t cta_off = 0;    // into the CTA offset array (ctas + 1 entries)
  uint32_t ctas = 0;
  uint32_t np = 0;
  uint32_t projs[PLORA_MAX_PROJ] = {};
};

// ------------------------------------------------ bf16 BGMV (warp items)
// bgmv_warp.cu, the default decode op: two launches, shrink then expand, each
// a flat list of warp-sized work items (no shared-memory ring, no clusters,
// no cross-CTA waits: the launch boundary orders v).  A job = <= 4 tokens of
// one adapter at one (layer, proj).
//   S item: <= kWarpRows(ntok) rank rows of A over one of the list's `ks`
//           K slices; its fp32 partial of v[tok][row] goes to that slice's
//           plane of the job's v block [ks][ntok][rank].
//   E item: one column block of <= kWarpCols(ntok) outputs over every rank
//           row; y[tok][block] = bf16(y + scale · Σ_row v[tok][row] · Bᵀ[row][block])
//           with v = the K-slice partials summed in slice order.
constexpr uint32_t kWarpJobTok = 4;
#ifdef __CUDACC__
__host__ __device__
#endif
constexpr uint32_t kWarpRows(uint32_t ntok) { return ntok <= 2 ? 8u : 4u; }
#ifdef __CUDACC__
__host__ __device__
#endif
constexpr uint32_t kWarpCols(uint32_t ntok) { return ntok <= 2 ? 512u : 256u; }
// Single-layer calls (plora_bgmv / plora_bgmv_layer): E items of jobs with
// >= kWarpSplitRows rank rows come in pairs — the two warps of one CTA take
// rows [0, h) and [h, r) of the same column block (h = ceil(r / 2)) and the
// first adds the second's partial sums (shared memory, fixed order) before
// the y epilogue: half the stream per warp for the widest adapters, which set
// the tail of a single layer's call (cfg2 34.6 -> 32.5 us).  Multi-layer
// launches keep whole items (the pairs measured 3 % slower there,
// profiles/r02o_warp_split.txt), so the two launch forms differ in the fp32
// summation order of those adapters' rows (<= 1 bf16 ulp of y).
constexpr uint32_t kWarpSplitRows = 64;
constexpr uint32_t kWarpSplit = 1u << 26;   // meta: a member of a split pair
constexpr uint32_t kWarpSecond = 1u << 27;  // meta: the pair's second half (rows [h, r))
struct WarpItem {  // 32 bytes, self-contained
  uint32_t table_off;  // adapter's first entry in the device page table
  uint32_t meta;       // rank (bits 0-8) | ntok (9-11) | launch projection (12-15) | n (16-25) | flags (26-27)
  uint32_t off;        // S: first rank row | K slice << 16; E: first output column
  uint32_t v_off;      // floats into the launch's per-layer v plane: the job's [ks][ntok][rank] block
  uint32_t tok[kWarpJobTok];
};
static_assert(sizeof(WarpItem) == 32, "WarpItem layout");

// A tensor-parallel half on the warp-item kernels (tp.cu; the default).
//   shrink (half 1): S items = (job, <= kWarpRows rows of the rank's shard,
//     K slice of `ks`); each writes its partial sums to `part` at the job's
//     block [ks][ntok][rs]; the job's last item (counter at cnt[v_off]) sums
//     the slices in order into v_out[tok][shard row] and / or every dst[d]
//     (fused all-gather), and with dst the launch's last job adds 1 to every
//     flags[d] (this rank's slot of rank d's flag array).
//   expand (half 2): E items = (job, <= kWarpCols columns of the shard), every
//     rank row, v read from v_in = [N][T][rs_max]; with `wait` the items first
//     wait for every local flag slot >= 1 and the launch's last item takes 1
//     from each.
struct WarpTp {
  uint32_t half = 0;
  const WarpItem* items = nullptr;
  uint32_t n_items = 0, ks = 1, njobs = 0;
  uint32_t tp_size = 1, tp_rank = 0, rs_max = 0, n_tokens = 0;
  float* part = nullptr;
  uint32_t* cnt = nullptr;
  float* v_out = nullptr;
  uint32_t n_dst = 0;
  float* dst[kMaxTp] = {};
  uint32_t* flags[kMaxTp] = {};
  uint32_t* done = nullptr;  // zero between calls
  const float* v_in = nullptr;
  uint32_t* wait = nullptr;
  uint32_t narrow = 0;  // expand: items of <= 256 columns (else kWarpCols)
};
struct WarpWork {  // one launch variant (a projection, or every projection of a layer)
  uint32_t s_off = 0, ns = 0;  // S items [s_off, s_off + ns) of the item array
  uint32_t e_off = 0, ne = 0;  // E items (multi-layer launches)
  uint32_t e1_off = 0, ne1 = 0;  // E items of single-layer calls (split pairs)
  uint32_t np = 0;
  uint32_t projs[PLORA_MAX_PROJ] = {};
  uint32_t ks = 1;             // K slices of the S items (v partial planes per job)
  uint64_t vplane = 0;         // floats of v per launched layer
};

// ---------------------------------------------------------------- SGMV
// A run = maximal stretch of consecutive tokens with the same adapter
// (Punica's seg_indptr formulation); tiles are 128-row slices of runs.
struct SgmvTile {
  uint32_t row0;       // first x / y row of the tile
  uint32_t nrows;      // valid rows (<= 128)
  uint32_t table_off;
  uint32_t rank;
};

// Fused base-GEMM + LoRA prefill (sgmv_fused.cu): every token row is in
// exactly one 128-row tile of a run (adapter runs and runs of tokens without
// an adapter); vtile indexes the run's SGMV tile (its V rows), ~0u for none.
struct GemmTile {
  uint32_t row0, nrows, table_off, rank, vtile, pad[3];
};

// One SGMV shrink work item: a unit (one tile, or two consecutive full tiles
// of one run, tile_b = ~0u otherwise) × one K slice, self-contained so the
// kernel reads one 32-byte record per item.
struct SgmvItem {
  uint32_t tile_a, tile_b, row0_a, row0_b, table_off, rank, split, pad;
};

// Persistent SGMV shrink schedule of one projection: CTA c runs the work
// items items[item_off + cta[cta_off + c] .. cta[cta_off + c + 1]), heaviest
// first (LPT over the CTAs).
struct SgmvSched {
  uint32_t splits = 0, ctas = 0, item_off = 0, cta_off = 0;
};

}  // namespace plora

struct plora_plan {
  plora_store* store = nullptr;
  uint32_t n_tokens = 0;
  uint32_t n_seg = 0;
  uint32_t max_rank = 0;
  uint64_t v_elems = 0;
  plora::ProjWork proj[PLORA_MAX_PROJ];
  plora::ClusterWork cwork[PLORA_MAX_PROJ];
  plora::ClusterWork cwork_layer;  // every projection of a layer in one launch (same d_in, d_out)
  uint32_t n_layer_proj = 0;       // 0: the projections' shapes differ, no fused launch
  uint32_t n_tiles = 0;

  std::vector<plora::BgmvUnit> units;
  std::vector<plora::SgmvTile> tiles;
  std::vector<plora::ClusterJob> cjobs;
  std::vector<plora::ClusterChunk> cchunks;
  std::vector<uint32_t> ccl_off;
  std::vector<uint32_t> ccl_jobs;  // jobs per cluster list (indexed like ccl_off; 0 at each list's end entry)
  plora::ClusterChunk* d_cchunks = nullptr;
  plora::ClusterJob* d_cjobs = nullptr;
  char* h_pinned = nullptr;
  uint64_t h_cap = 0;
  char* d_buf = nullptr;
  uint64_t d_cap = 0;
  plora::BgmvUnit* d_units = nullptr;
  plora::SgmvTile* d_tiles = nullptr;
  float* d_v = nullptr;
  uint64_t v_cap = 0;
  uint32_t* d_sync = nullptr;  // [0] ticket, [1] exit count, [2..] per-segment shrink done
  uint64_t sync_cap = 0;
  // SGMV: split-K partials of V (fp32), V tiles (bf16, 128 × 128 per tile)
  float* d_vpart = nullptr;
  uint64_t vpart_cap = 0;  // floats
  char* d_vbuf = nullptr;
  uint64_t vbuf_cap = 0;   // bytes
  // SGMV shrink units: pairs of consecutive full tiles of one run (they share
  // the adapter's A chunks), {tile, tile or ~0u}
  std::vector<uint32_t> sunits;
  uint32_t n_sunits = 0;
  plora::SgmvSched ssched[PLORA_MAX_PROJ];
  plora::SgmvSched ssched_layer;  // both projections from one x chunk (splits 0: unavailable)
  uint32_t vpart_parts = 0;       // K splits the partial regions are sized for
  std::vector<plora::GemmTile> gtiles;
  plora::GemmTile* d_gtiles = nullptr;
  std::vector<plora::SgmvItem> sitems;
  std::vector<uint32_t> scta;
  plora::SgmvItem* d_sitems = nullptr;
  uint32_t* d_scta = nullptr;
  // bf16 streaming BGMV (bgmv_stream.cu)
  uint32_t s_jt = 4;       // tokens per job (4 or 8)
  uint32_t s_njobs = 0;    // jobs per (layer, proj) plane
  uint64_t s_vplane = 0;   // floats per (layer, proj) v plane
  plora::StreamWork swork[PLORA_MAX_PROJ];
  plora::StreamWork swork_layer;  // every projection of a layer (equal shapes), ctas 0: none
  std::vector<plora::StreamItem> stitems;
  std::vector<uint32_t> stcta;
  plora::StreamItem* d_stitems = nullptr;
  uint32_t* d_stcta = nullptr;
  float* d_sv = nullptr;       // v planes: n_layers · n_proj · s_vplane floats
  uint64_t sv_cap = 0;
  uint32_t* d_scnt = nullptr;  // per plane: s_njobs S-item counters, then s_njobs E-done counters
  uint64_t scnt_cap = 0;
  void build_stream(const std::vector<std::vector<uint32_t>>& seg_toks,
                    const std::vector<uint32_t>& seg_rank, const std::vector<uint32_t>& seg_table);
  // bf16 warp-item BGMV (bgmv_warp.cu, the default decode op)
  plora::WarpWork wwork[PLORA_MAX_PROJ];
  plora::WarpWork wwork_layer;  // every projection of a layer (equal d_in), np 0: none
  std::vector<plora::WarpItem> witems;
  plora::WarpItem* d_witems = nullptr;
  float* d_wv = nullptr;        // v planes: n_layers · max vplane floats
  uint64_t wv_cap = 0;
  // hybrid decode launch (plora_bgmv_layers): the clusters' share and the
  // streaming kernel's share on the SMs the clusters leave idle, run
  // concurrently on `stream` and `aux_stream` (fork / join by events)
  std::vector<uint8_t> seg_hyb;
  uint32_t hyb_spare = 0;             // SMs the streaming share runs on (0: no hybrid)
  double hyb_frac = 0.0;              // the streaming share's fraction of the weight rows
  plora::ClusterWork cwork_hyb;
  plora::StreamWork swork_hyb;
  cudaStream_t aux_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t upload_done = nullptr;
  // tensor-parallel halves (tp.cu): streaming-kernel item lists per
  // (tp_rank, tp_size, proj, half), built on first use, dropped on rebuild
  struct TpWork {
    plora::StreamWork w;
    plora::WarpTp wt;                      // the warp-item path (default): items / partials / counters in d_items
    plora::StreamItem* d_items = nullptr;  // items, then the CTA offsets (one allocation, freed by drop_tp)
    uint32_t* d_cta = nullptr;
    uint32_t* d_done = nullptr;            // fused all-gather: CTAs of the shrink done (zero between calls)
    char* h_stage = nullptr;               // pinned source of the upload
  };
  std::map<uint64_t, TpWork> tpw;
  void drop_tp();
  // Many-token adapters (>= route_min_tokens() tokens in the batch) leave the
  // decode kernels: their tokens, gathered in adapter order, form a child
  // plan that runs the tensor-core SGMV path (bgmv.cu launch_routed), on its
  // own stream, concurrently with the decode kernels over the other adapters.
  std::vector<uint8_t> seg_route;    // per segment (adapter) of the batch
  plora_plan* route = nullptr;       // the child plan (never routes itself)
  bool no_route = false;
  uint32_t n_route = 0;              // routed tokens (0: none this batch)
  std::vector<uint32_t> route_perm;  // routed row i -> the batch's token row
  uint32_t* d_route_perm = nullptr;  // (in d_buf)
  char* d_route_ws = nullptr;        // one layer: gathered x, then y deltas per projection
  uint64_t route_ws_cap = 0;
  cudaStream_t route_stream = nullptr;
  cudaEvent_t ev_rfork = nullptr, ev_rjoin = nullptr;

  void build(const int32_t* token_adapter, uint32_t n, cudaStream_t stream);
};

namespace plora {
// Diagnostics buffer set by plora_debug_set_trace (nullptr if absent or too small).
uint64_t* trace_buffer(uint64_t need_bytes);
// Tensor-parallel decode halves (tp.cu).
// bf16 decode op (bgmv_cluster.cu): 4-CTA clusters, DSMEM exchange of v.
void launch_bgmv_cluster(const plora_plan& plan, uint32_t layer, uint32_t proj, const void* x,
                         uint64_t x_stride, void* y, uint64_t y_stride, float scale,
                         cudaStream_t stream);
// Streaming bf16 BGMV (bgmv_stream.cu): the projections `w` was built for,
// layers [layer0, layer0 + n_layers); layer layer0 + i reads x + i·x_lstride
// and updates ys[j] + i·y_lstrides[j] (elements).
// One tensor-parallel half (single projection `w.projs[0]`, one layer); y is
// pre-shifted by the caller so that column c of the output is y + c.
void launch_bgmv_stream_tp(const plora_plan& plan, const StreamWork& w, const StreamTp& tp,
                           uint32_t layer, const void* x, uint64_t x_stride, void* y,
                           uint64_t y_stride, float scale, cudaStream_t stream);
void launch_bgmv_stream(const plora_plan& plan, const StreamWork& w, uint32_t layer0,
                        uint32_t n_layers, const void* x, uint64_t x_stride, uint64_t x_lstride,
                        void* const* ys, const uint64_t* y_strides, const uint64_t* y_lstrides,
                        float scale, cudaStream_t stream);
uint32_t stream_max_ctas(int device, uint32_t jt);
// Warp-item bf16 BGMV (bgmv_warp.cu): shrink launch then expand launch over
// the projections `w` was built for, layers [layer0, layer0 + n_layers)
// (strides as launch_bgmv_stream).
void launch_bgmv_warp(const plora_plan& plan, const WarpWork& w, uint32_t layer0, uint32_t n_layers,
                      const void* x, uint64_t x_stride, uint64_t x_lstride, void* const* ys,
                      const uint64_t* y_strides, const uint64_t* y_lstrides, float scale,
                      cudaStream_t stream);
void launch_bgmv_warp_tp(const plora_plan& plan, const WarpTp& t, uint32_t layer, uint32_t proj, const void* x,
                         uint64_t x_stride, void* y, uint64_t y_stride, float scale, cudaStream_t stream);
// plora_debug_set_bgmv_impl: 0 (default) warp items, 1 streaming kernel,
// 2 clusters, 3 the hybrid pair (clusters + streaming share)
uint32_t bgmv_impl();
bool hybrid_enabled();  // impl 3
uint32_t route_min_tokens();  // plora_debug_set_route_tokens (0: never route)
double hybrid_share_factor();  // streaming share = spare SMs / SMs × this (of the weight bytes)
// Every projection of `layer` (they read the same x) in one launch.
void launch_bgmv_cluster_layer(const plora_plan& plan, uint32_t layer, const void* x,
                               uint64_t x_stride, void* const* ys, const uint64_t* y_strides,
                               float scale, cudaStream_t stream);
// Layers [layer0, layer0 + n_layers), every projection, in one launch: the
// clusters stay resident and stream layer l + 1's pages right behind layer
// l's.  Layer l's x rows start l·x_lstride elements after x, projection p's
// y rows y_lstrides[p] elements after the previous layer's.
void launch_bgmv_cluster_layers(const plora_plan& plan, uint32_t layer0, uint32_t n_layers,
                                const void* x, uint64_t x_stride, uint64_t x_lstride,
                                void* const* ys, const uint64_t* y_strides,
                                const uint64_t* y_lstrides, float scale, cudaStream_t stream,
                                const ClusterWork* work = nullptr);  // default: plan.cwork_layer
}  // namespace plora
