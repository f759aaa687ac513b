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
  uint32_t kc;        // shrink: K chunk (bf16 path: d_in split in kShrinkK slices)
  uint32_t nkc;       // expand: number of K-chunk partial planes of v to sum
  uint32_t vstride;   // expand: floats between consecutive partial planes
  uint32_t pad;
};
static_assert(sizeof(BgmvUnit) == 64, "BgmvUnit layout");

// bf16 shrink units: 16 rank rows (the MMA M) × kShrinkK input columns.
constexpr uint32_t kShrinkK = 1024;
constexpr uint32_t kShrinkRows16 = 16;
// bf16 ring slot: shrink 16 rows + 4 x rows of (kShrinkK·2 + 16) bytes;
// expand Bᵀ tile r16 × (CB·2 + 16) + per token: y segment + K-partial v rows.
constexpr uint32_t kRingSlotBytes = 53248;
constexpr uint32_t kRingRowPad = 16;

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

// Columns per expand unit.  bf16 (tensor-core path): the Bᵀ tile r16 × CB
// (rank padded to the MMA K of 16) fits 32 KiB; fp32 (CUDA-core path): RG·CB
// = 256 threads × 4 columns.
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

// ---------------------------------------------------------------- SGMV
// A run = maximal stretch of consecutive tokens with the same adapter
// (Punica's seg_indptr formulation); tiles are 128-row slices of runs.
struct SgmvTile {
  uint32_t row0;       // first x / y row of the tile
  uint32_t nrows;      // valid rows (<= 128)
  uint32_t table_off;
  uint32_t rank;
};

}  // namespace plora

struct plora_plan {
  plora_store* store = nullptr;
  uint32_t n_tokens = 0;
  uint32_t n_seg = 0;
  uint32_t max_rank = 0;
  uint64_t v_elems = 0;
  plora::ProjWork proj[PLORA_MAX_PROJ];
  uint32_t n_tiles = 0;

  std::vector<plora::BgmvUnit> units;
  std::vector<plora::SgmvTile> tiles;
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
  cudaEvent_t upload_done = nullptr;

  void build(const int32_t* token_adapter, uint32_t n, cudaStream_t stream);
};

namespace plora {
// bf16 decode op (bgmv_ring.cu): persistent TMA ring + warp-level tensor cores.
void launch_bgmv_ring(const plora_plan& plan, uint32_t layer, uint32_t proj, const void* x,
                      uint64_t x_stride, void* y, uint64_t y_stride, float scale,
                      cudaStream_t stream);
}  // namespace plora
