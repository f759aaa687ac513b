// Batch plan: tokens grouped by adapter (segments) and the work-unit lists
// the persistent kernels consume.  Built on the host once per batch and
// reused for every (layer, proj) call of the step — the "translation once
// per batch" of PAPER.md:136.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "store.hpp"

namespace plora {

// One segment = the tokens of one adapter in this batch.  32 bytes.
struct SegDesc {
  uint32_t table_off;  // adapter's first entry in the device page table
  uint32_t rank;
  uint32_t tok_start;  // into the token list
  uint32_t n_tok;
  uint32_t voff;       // fp32 offset of this segment's v = x·Aᵀ block
  uint32_t n_shrink;   // shrink units the expand units of this segment wait for
  uint32_t adapter;
  uint32_t pad;
};

// Work unit: x = segment | kind << 31 (0 shrink, 1 expand); y = first rank
// row (shrink) or first output column (expand).
constexpr uint32_t kExpandBit = 0x80000000u;
constexpr uint32_t kShrinkRows = 8;  // one warp per rank row, 8 warps per CTA
constexpr uint32_t kThreads = 256;

// Rank rows per thread group in the expand: rows are split over RG groups of
// CT = 256/RG column-threads so a thread holds <= 4 rows of Bᵀ (ranks up to
// 128 in one batch of loads; larger ranks loop).
#ifdef __CUDACC__
__host__ __device__
#endif
inline uint32_t expand_rg(uint32_t rank) {
  return rank <= 16 ? 4u : (rank <= 32 ? 8u : (rank <= 64 ? 16u : 32u));
}

struct ProjUnits {
  uint32_t n_units = 0;
  uint32_t units_off = 0;  // into the unit array
  uint32_t smem = 0;       // dynamic shared memory for this proj's launch
};

}  // namespace plora

struct plora_plan {
  plora_store* store = nullptr;
  uint32_t n_tokens = 0;
  uint32_t n_seg = 0;
  uint32_t max_rank = 0;
  uint64_t v_elems = 0;
  plora::ProjUnits proj[PLORA_MAX_PROJ];

  // host staging (pinned) and device mirror of: segs | toks | units
  std::vector<plora::SegDesc> segs;
  std::vector<uint32_t> toks;
  std::vector<uint2> units;
  char* h_pinned = nullptr;
  uint64_t h_cap = 0;
  char* d_buf = nullptr;
  uint64_t d_cap = 0;
  plora::SegDesc* d_segs = nullptr;
  uint32_t* d_toks = nullptr;
  uint2* d_units = nullptr;
  float* d_v = nullptr;
  uint64_t v_cap = 0;
  uint32_t* d_sync = nullptr;  // [0] ticket, [1] exit count, [2..] per-segment done
  uint64_t sync_cap = 0;
  cudaEvent_t upload_done = nullptr;

  void build(const int32_t* token_adapter, uint32_t n, cudaStream_t stream);
};
