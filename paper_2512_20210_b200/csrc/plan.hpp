// Batch plan: tokens grouped by adapter (segments) and the work lists the
// persistent kernels consume.  Built on the host once per batch and reused
// for every (layer, proj) call of the step — the "translation once per
// batch" of PAPER.md:136.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
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
  cudaEvent_t upload_done = nullptr;

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
                                const uint64_t* y_lstrides, float scale, cudaStream_t stream);
}  // namespace plora
