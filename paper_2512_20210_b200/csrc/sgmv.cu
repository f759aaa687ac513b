// Paged multi-LoRA prefill op (gathered SGMV) on the 5th-generation tensor
// cores (tcgen05 + TMEM) for sm_100a.
//
// y[t, :] += scale · bf16(x[t, :] · Aᵀ) · Bᵀ for the tokens of each run (a
// stretch of consecutive tokens with one adapter).  The
// reference bills this as cost_model.prefill_ms (cost_model.hpp:32-34,
// src/engine.cpp:355).
//
// Two kernels per (layer, proj) call, chained by programmatic dependent
// launch, each with enough CTAs to keep every SM streaming (a 128-token tile
// is 1 MiB of x and 2 MiB of y read-modify-write; one CTA per tile would be
// latency-bound on its own serial stream):
//
//  shrink  CTA (tile, k-split): V_part[128 × r16] = X[128, ks] · A[r, ks]ᵀ
//          over a d_in/KS slice.  Warp 0 TMA-loads x chunks [128 × 64]
//          (SWIZZLE_128B) into a 4-stage ring; warps 1-3 gather the
//          adapter's A rows with 16-byte cp.async pieces, each translated
//          through the device page table, straight into the UMMA K-major
//          SW128 layout (rank zero-padded to 16 in smem only); warp 4 issues
//          tcgen05.mma (M = 128, N = r16) into TMEM; warps 4-7 store the fp32
//          partial.  The last CTA of a tile (arrival counter) sums the KS
//          partials in split order (deterministic) and writes V in bf16 — the
//          rounding point between shrink and expand.
//  expand  CTA (tile, 8 column blocks of 64): D[128 × 64] = V · Bᵀ[:, block]
//          (tcgen05, K = r16) per block, with the V tile loaded once by TMA,
//          the Bᵀ blocks gathered from pages (MN-major SW128), two TMEM
//          accumulators; the epilogue stages bf16(scale · D) in shared
//          memory and TMA reduce-adds it into y (the read-modify-write happens
//          in L2; rows of a partial tile that belong to the next run add 0).
//          y therefore sees one extra bf16 rounding of the LoRA delta.
// Rank <= 128; d_in % 64 == 0; d_out % 128 == 0; bf16 stores (otherwise the
// exact CUDA-core BGMV path runs, see plora_sgmv).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>
#include <mutex>

#include "plan.hpp"
#include "ptx.cuh"

using namespace plora;

namespace plora {
void check_io(const plora_plan* plan, uint32_t layer, uint32_t proj, const void* x,
              uint64_t x_stride, void* y, uint64_t y_stride);
}

extern "C" int plora_bgmv(plora_plan* plan, uint32_t layer, uint32_t proj, const void* x,
                          uint64_t x_stride, void* y, uint64_t y_stride, float scale,
                          plora_stream_t stream);

namespace {

uint32_t g_sgmv_dbg = 0;  // plora_debug_set_sgmv_flags

constexpr int kThreads = 256;
constexpr uint32_t kTileM = 128;
constexpr uint32_t kChunkK = 64;   // shrink K per stage (one 128-byte swizzle row)
constexpr uint32_t kBlockN = 128;  // expand output columns per CTA
constexpr uint32_t kMaxRank = 128;
constexpr uint32_t kTmemCols = 128;
constexpr int kGatherThreads = 96;   // expand: warps 1-3
constexpr int kSGather = 192;       // shrink: warps 1-3 and 5-7 (5-7 are idle until the epilogue)
constexpr int kEGather = 96;        // expand: warps 1-3

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ uint32_t swz(uint32_t row, uint32_t chunk) {
  // 128-byte swizzle inside an 8-row × 128-byte atom
  return (row >> 3) * 1024 + (row & 7) * 128 + ((chunk ^ (row & 7)) << 4);
}

struct PagedSrc {
  const char* arena;
  const uint32_t* table;
  uint32_t table_off;
  uint32_t log2_page;
  __device__ const char* at(uint64_t off) const {
    const uint32_t phys = __ldg(table + table_off + static_cast<uint32_t>(off >> log2_page));
    return arena + (static_cast<uint64_t>(phys) << log2_page) + (off & ((1ull << log2_page) - 1));
  }
};

// ------------------------------------------------------------------ shrink
constexpr int kSStages = 4;  // a deep per-CTA ring beats more CTAs here (measured: 2 stages x3 CTAs 108 us, 3x2 92, 4x1 75)
constexpr uint32_t kSStageBytes = 49152;  // X [2 tiles][128 × 64] 32 KiB + A [r16 × 64] <= 16 KiB
constexpr uint32_t kSTmemCols = 2 * kTmemCols;  // one accumulator per tile of the unit

struct ShrinkArgs {
  const char* arena;
  const uint32_t* table;
  const SgmvTile* tiles;
  const uint32_t* units;  // [unit] {tile, tile or ~0u}
  float* vpart;      // [tile][split][128][128] fp32
  __nv_bfloat16* vbuf;  // [tile][128][128] bf16
  uint32_t* tcnt;    // [tile] arrivals
  uint64_t blk_mult;
  uint32_t log2_page;
  uint32_t d_in;
  uint32_t splits;
  uint32_t dbg;  // diagnostics (plora_debug_set_sgmv_flags): 1 no A gather, 2 no MMA, 4 no x load, 16 no epilogue, 32 no reduction
};

struct SSmem {
  static constexpr uint32_t stages = 0;  // 1024-aligned
  static constexpr uint32_t bars = stages + kSStages * kSStageBytes;
  static constexpr uint32_t n_bars = 2 * kSStages + 1;  // full[4], empty[4], v_full
  static constexpr uint32_t tmem_slot = bars + n_bars * 8;
  static constexpr uint32_t flag = tmem_slot + 8;
  static constexpr uint32_t total = flag + 8;
  static constexpr uint32_t alloc = total + 1024;  // alignment slack
};

__global__ void __launch_bounds__(kThreads, 1)
    sgmv_shrink_kernel(const ShrinkArgs p, const __grid_constant__ CUtensorMap tmap_x) {
  extern __shared__ char smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SSmem::bars);
  uint64_t* empty = full + kSStages;
  uint64_t* v_full = full + 2 * kSStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SSmem::tmem_slot);
  volatile uint32_t* last_flag = reinterpret_cast<uint32_t*>(smem + SSmem::flag);

  const uint32_t unit = blockIdx.x / p.splits, split = blockIdx.x % p.splits;
  const uint32_t tile_a = p.units[2 * unit], tile_b = p.units[2 * unit + 1];
  const uint32_t nt = tile_b != 0xffffffffu ? 2 : 1;  // tiles sharing the A chunks
  const SgmvTile tile = p.tiles[tile_a];
  const uint32_t row0_b = nt == 2 ? p.tiles[tile_b].row0 : 0;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t r = tile.rank, r16 = (r + 15) & ~15u;
  const uint32_t kslice = p.d_in / p.splits, NK = kslice / kChunkK, k0 = split * kslice;
  const uint64_t blk = static_cast<uint64_t>(r) * p.blk_mult * 2;  // A block, bytes
  const PagedSrc src{p.arena, p.table, tile.table_off, p.log2_page};

  ptx::pdl_launch_dependents();  // the expand may start gathering its weights
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSStages; ++s) {
      ptx::mbar_init(&full[s], 1 + kSGather);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(v_full, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 4) ptx::tmem_alloc(tmem_slot, kSTmemCols);
  if (warp == 0 && lane == 0) ptx::prefetch_tmap(&tmap_x);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer (x chunks)
    if (lane == 0) {
      ptx::pdl_wait();  // x is written by earlier kernels in the stream
      for (uint32_t kc = 0; kc < NK; ++kc) {
        const uint32_t st = kc % kSStages, ph = (kc / kSStages) & 1u;
        ptx::mbar_wait(&empty[st], ph ^ 1u);
        if (p.dbg & 4u) {
          ptx::mbar_arrive(&full[st]);
          continue;
        }
        ptx::mbar_arrive_expect_tx(&full[st], nt * kTileM * kChunkK * 2);
        ptx::tma_load_2d(smem + SSmem::stages + st * kSStageBytes, &tmap_x,
                         static_cast<int32_t>(k0 + kc * kChunkK), static_cast<int32_t>(tile.row0),
                         &full[st]);
        if (nt == 2)
          ptx::tma_load_2d(smem + SSmem::stages + st * kSStageBytes + kTileM * kChunkK * 2, &tmap_x,
                           static_cast<int32_t>(k0 + kc * kChunkK), static_cast<int32_t>(row0_b),
                           &full[st]);
      }
    }
  }
  if (warp >= 1 && warp != 4) {
    // ----------------------------------------------- A gathers (paged rows)
    // Thread wt owns rank rows wt and wt + 96.  With pages >= 256 B a row's
    // 128-byte piece of a chunk lies in one page: one page-table lookup per
    // row per chunk, issued a chunk ahead (before the slot wait), so the
    // lookups never serialise the copies.  Smaller pages: per-piece lookups.
    const uint32_t wt = warp < 4 ? threadIdx.x - 32 : threadIdx.x - 160 + 96;
    const bool fast = p.log2_page >= 8;
    const uint32_t n0 = wt, n1 = wt + kSGather;
    auto row_off = [&](uint32_t n, uint32_t kc) {
      return blk + (static_cast<uint64_t>(n) * p.d_in + k0 + kc * kChunkK) * 2;
    };
    auto lookup = [&](uint32_t n, uint32_t kc) -> uint32_t {
      return (fast && n < r && kc < NK) ? __ldg(p.table + tile.table_off + static_cast<uint32_t>(row_off(n, kc) >> p.log2_page)) : 0u;
    };
    uint32_t ph0 = lookup(n0, 0), ph1 = lookup(n1, 0);
    const uint64_t pmask = (1ull << p.log2_page) - 1;
    for (uint32_t kc = 0; kc < NK; ++kc) {
      const uint32_t st = kc % kSStages, ph = (kc / kSStages) & 1u;
      const uint32_t nx0 = lookup(n0, kc + 1), nx1 = lookup(n1, kc + 1);  // next chunk, in flight
      ptx::mbar_wait(&empty[st], ph ^ 1u);
      char* wdst = smem + SSmem::stages + st * kSStageBytes + 2 * kTileM * kChunkK * 2;
#pragma unroll
      for (uint32_t h = 0; h < 1; ++h) {  // r16 <= 128 < 192 threads: one row each
        const uint32_t n = h ? n1 : n0;
        if (n >= r16 || (p.dbg & 1u)) continue;
        if (n >= r) {
#pragma unroll
          for (uint32_t c = 0; c < 8; ++c) ptx::cp_async_16(wdst + swz(n, c), p.arena, 0);  // zero padding
        } else if (fast) {
          const uint64_t off = row_off(n, kc);
          const char* base = p.arena + (static_cast<uint64_t>(h ? ph1 : ph0) << p.log2_page) + (off & pmask);
#pragma unroll
          for (uint32_t c = 0; c < 8; ++c) ptx::cp_async_16(wdst + swz(n, c), base + c * 16, 16);
        } else {
          for (uint32_t c = 0; c < 8; ++c)
            ptx::cp_async_16(wdst + swz(n, c), src.at(row_off(n, kc) + c * 16), 16);
        }
      }
      ptx::cp_async_mbar_arrive_noinc(&full[st]);
      ph0 = nx0;
      ph1 = nx1;
    }
  }
  if (warp >= 4) {
    if (warp == 4 && lane == 0) {
      // ------------------------------------------------------- MMA issuer
      const uint32_t idesc = ptx::idesc_bf16_f32(kTileM, r16, false, false);
      const uint32_t sbase = ptx::smem_u32(smem + SSmem::stages);
      for (uint32_t kc = 0; kc < NK; ++kc) {
        const uint32_t st = kc % kSStages, ph = (kc / kSStages) & 1u;
        ptx::mbar_wait(&full[st], ph);
        if (p.dbg & 2u) {
          ptx::mbar_arrive(&empty[st]);
          continue;
        }
        ptx::fence_proxy_async_shared();
        ptx::tc_fence_after();
        const uint32_t xa = sbase + st * kSStageBytes, xb = xa + kTileM * kChunkK * 2;
        const uint32_t wa = xa + 2 * kTileM * kChunkK * 2;
#pragma unroll
        for (uint32_t k = 0; k < kChunkK / 16; ++k) {
          const uint64_t wd = ptx::smem_desc_sw128(wa + k * 32, 16, 1024);
          ptx::umma_f16(tmem, ptx::smem_desc_sw128(xa + k * 32, 16, 1024), wd, idesc, (kc | k) != 0);
          if (nt == 2)
            ptx::umma_f16(tmem + kTmemCols, ptx::smem_desc_sw128(xb + k * 32, 16, 1024), wd, idesc,
                          (kc | k) != 0);
        }
        ptx::umma_commit(&empty[st]);
      }
      ptx::umma_commit(v_full);
    }
    __syncwarp();
  }
  // --------------------------------------------- epilogue (all 8 warps)
  // Warp w reads TMEM lanes 32·(w % 4) (its lane quarter), columns of half
  // w / 4.  Partials are [tile][split] blocks of 128 × r16 fp32, rows of
  // r16/4 16-byte chunks with chunk j of row m stored at j ^ (m & swm):
  // staged through the (now idle) stage buffers without bank conflicts,
  // written with one bulk copy, and read back coalesced by the reducing CTA.
  ptx::mbar_wait(v_full, 0);
  ptx::tc_fence_after();
  {
    const uint32_t m = (warp & 3) * 32 + lane;  // tile row == TMEM lane
    const uint32_t lane_base = ((warp & 3) * 32) << 16;
    const uint32_t nch = r16 / 4, swm = min(8u, nch & (0u - nch)) - 1u;
    const uint32_t tile_floats = kTileM * r16;
    for (uint32_t t = 0; t < ((p.dbg & 16u) ? 0u : nt); ++t) {
      const uint32_t tile_i = t ? tile_b : tile_a;
      float* stg = reinterpret_cast<float*>(smem + SSmem::stages + t * kTileM * kMaxRank * 4);
      for (uint32_t cc = warp >> 2; cc < r16 / 16; cc += 2) {
        uint32_t rv[16];
        ptx::tmem_ld_32x32b_x16(tmem + lane_base + t * kTmemCols + cc * 16, rv);
        ptx::tmem_ld_wait();
#pragma unroll
        for (uint32_t i = 0; i < 4; ++i)
          reinterpret_cast<uint4*>(stg + m * r16)[(cc * 4 + i) ^ (m & swm)] =
              make_uint4(rv[4 * i], rv[4 * i + 1], rv[4 * i + 2], rv[4 * i + 3]);
      }
      ptx::fence_proxy_async_shared();
      __syncthreads();
      if (threadIdx.x == 0) {
        float* dst = p.vpart + (static_cast<uint64_t>(tile_i) * p.splits + split) * kTileM * kMaxRank;
        ptx::bulk_s2g(dst, stg, tile_floats * 4);
        ptx::bulk_commit();
        ptx::bulk_wait_all();  // written, not just read: the count below publishes it
        ptx::fence_proxy_async_global();
        __threadfence();
        *last_flag = atomicAdd(p.tcnt + tile_i, 1u) == p.splits - 1;
      }
      __syncthreads();
      if (*last_flag && !(p.dbg & 32u)) {
        // split-K reduction by the tile's last CTA, in split order; 4 float4
        // per thread and two splits per step keep 8 loads in flight
        __threadfence();
        constexpr uint32_t kU = 4;
        constexpr uint32_t kSplitStride = kTileM * kMaxRank / 4;  // float4s
        const float4* v0 = reinterpret_cast<const float4*>(
            p.vpart + static_cast<uint64_t>(tile_i) * p.splits * kTileM * kMaxRank);
        __nv_bfloat16* vb = p.vbuf + static_cast<uint64_t>(tile_i) * kTileM * kMaxRank;
        const uint32_t n4 = tile_floats / 4;
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
        for (uint32_t f0 = threadIdx.x; f0 < n4; f0 += kU * kThreads) {
          float4 acc[kU];
#pragma unroll
          for (uint32_t u = 0; u < kU; ++u) acc[u] = z;
          for (uint32_t sp = 0; sp < p.splits; sp += 2) {
            float4 q0[kU], q1[kU];
#pragma unroll
            for (uint32_t u = 0; u < kU; ++u) {
              const uint32_t f = f0 + u * kThreads;
              q0[u] = f < n4 ? __ldcg(v0 + sp * kSplitStride + f) : z;
              q1[u] = f < n4 && sp + 1 < p.splits ? __ldcg(v0 + (sp + 1) * kSplitStride + f) : z;
            }
#pragma unroll
            for (uint32_t u = 0; u < kU; ++u) {
              acc[u].x += q0[u].x; acc[u].y += q0[u].y; acc[u].z += q0[u].z; acc[u].w += q0[u].w;
              acc[u].x += q1[u].x; acc[u].y += q1[u].y; acc[u].z += q1[u].z; acc[u].w += q1[u].w;
            }
          }
#pragma unroll
          for (uint32_t u = 0; u < kU; ++u) {
            const uint32_t f = f0 + u * kThreads;
            if (f >= n4) continue;
            const uint32_t row = f / nch, j = (f % nch) ^ (row & swm);
            uint2 o;
            __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&o);
            h[0] = __floats2bfloat162_rn(acc[u].x, acc[u].y);
            h[1] = __floats2bfloat162_rn(acc[u].z, acc[u].w);
            *reinterpret_cast<uint2*>(vb + row * kMaxRank + j * 4) = o;
          }
        }
        if (threadIdx.x == 0) p.tcnt[tile_i] = 0;  // graph-replayable
      }
      __syncthreads();  // last_flag and the staging buffer are reused by the next tile
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, kSTmemCols);
  }
}

// ------------------------------------------------------------------ expand
// CTA (tile, group of kGroupBlocks 64-column blocks): the V tile is loaded
// once; the Bᵀ block of block b goes to stage b % 2 and the MMA to TMEM
// accumulator b % 2, so the epilogue of block b overlaps the gather and MMA
// of block b + 1.  The epilogue never reads y: it stages bf16(scale · D) in
// shared memory and TMA reduce-adds the tile into y (the add happens in L2),
// with the rows of a partial tile that belong to the next run zeroed.
constexpr uint32_t kEBlockN = 64;     // output columns per block (one 128-byte swizzle row)
constexpr uint32_t kGroupBlocks = 8;  // blocks per CTA (512 columns)
constexpr uint32_t kETmemCols = 2 * kEBlockN;
// warps 0 TMA, 1-3 Bᵀ gathers, 4-7 epilogue, 8 MMA issuer (its own warp: the
// epilogue releases the accumulators the MMA loop waits for)
constexpr int kEThreads = 288;

struct ExpandArgs {
  const char* arena;
  const uint32_t* table;
  const SgmvTile* tiles;
  char* y;
  uint64_t y_stride_b;
  uint64_t blk_mult;
  uint32_t log2_page;
  uint32_t d_in;
  uint32_t d_out;
  uint32_t ngroups;  // column groups per tile
  float scale;
};

struct ESmem {  // ~97 KB: two expand CTAs per SM
  static constexpr uint32_t v = 0;                  // [2 atoms][128 rows × 128 B] SW128 (K-major)
  static constexpr uint32_t y = v + 32768;          // [2 stages][128 rows × 128 B] SW128
  static constexpr uint32_t b = y + 2 * 16384;      // [2 stages][r16 × 128 B] MN-major SW128
  static constexpr uint32_t bars = b + 2 * 16384;
  // v_full, (unused) [4], b_full[2], b_empty[2], acc_full[2], acc_empty[2]
  static constexpr uint32_t n_bars = 13;
  static constexpr uint32_t tmem_slot = bars + n_bars * 8;
  static constexpr uint32_t total = tmem_slot + 8;
  static constexpr uint32_t alloc = total + 1024;
};

__global__ void __launch_bounds__(kEThreads, 2)
    sgmv_expand_kernel(const ExpandArgs p, const __grid_constant__ CUtensorMap tmap_y,
                       const __grid_constant__ CUtensorMap tmap_v) {
  extern __shared__ char smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* v_full = reinterpret_cast<uint64_t*>(smem + ESmem::bars);
  uint64_t* y_full = v_full + 1;
  uint64_t* y_empty = v_full + 3;
  uint64_t* b_full = v_full + 5;
  uint64_t* b_empty = v_full + 7;
  uint64_t* acc_full = v_full + 9;
  uint64_t* acc_empty = v_full + 11;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + ESmem::tmem_slot);

  const uint32_t tile_i = blockIdx.x / p.ngroups, grp = blockIdx.x % p.ngroups;
  const SgmvTile tile = p.tiles[tile_i];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t r = tile.rank, r16 = (r + 15) & ~15u;
  const uint64_t bt = (static_cast<uint64_t>(r) * p.blk_mult + static_cast<uint64_t>(r) * p.d_in) * 2;
  const PagedSrc src{p.arena, p.table, tile.table_off, p.log2_page};
  const uint32_t nblk = min(kGroupBlocks, p.d_out / kEBlockN - grp * kGroupBlocks);
  const uint32_t col_base = grp * kGroupBlocks * kEBlockN;
  const uint32_t vboxes = r16 > 64 ? 2 : 1;

  if (threadIdx.x == 0) {
    ptx::mbar_init(v_full, 1);
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&y_full[i], 1);
      ptx::mbar_init(&y_empty[i], 1);
      ptx::mbar_init(&b_full[i], kEGather);
      ptx::mbar_init(&b_empty[i], 1);
      ptx::mbar_init(&acc_full[i], 1);
      ptx::mbar_init(&acc_empty[i], 1);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 4) ptx::tmem_alloc(tmem_slot, kETmemCols);
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmap_y);
    ptx::prefetch_tmap(&tmap_v);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ----------------------------------------------- TMA: V tile once
    if (lane == 0) {
      ptx::pdl_wait();  // V comes from the shrink (and y may be read by earlier kernels)
      ptx::mbar_arrive_expect_tx(v_full, vboxes * 16384);
      for (uint32_t bx = 0; bx < vboxes; ++bx)
        ptx::tma_load_2d(smem + ESmem::v + bx * 16384, &tmap_v, static_cast<int32_t>(bx * 64),
                         static_cast<int32_t>(tile_i * kTileM), v_full);
    }
  } else if (warp < 4) {
    // ----------------------------------- Bᵀ block gathers (paged rows)
    // Thread wt owns rank rows wt and wt + 96; with pages >= 256 B a row's
    // 256-byte block slice lies in one page (one lookup, issued a block ahead).
    const uint32_t wt = threadIdx.x - 32;
    const bool fast = p.log2_page >= 7;  // a row's 128-byte block slice lies in one page
    const uint64_t pmask = (1ull << p.log2_page) - 1;
    auto row_off = [&](uint32_t j, uint32_t b) {
      return bt + (static_cast<uint64_t>(j) * p.d_out + col_base + b * kEBlockN) * 2;
    };
    auto lookup = [&](uint32_t j, uint32_t b) -> uint32_t {
      return (fast && j < r && b < nblk) ? __ldg(p.table + tile.table_off + static_cast<uint32_t>(row_off(j, b) >> p.log2_page)) : 0u;
    };
    uint32_t ph0 = lookup(wt, 0), ph1 = lookup(wt + kEGather, 0);
    for (uint32_t b = 0; b < nblk; ++b) {
      const uint32_t st = b & 1u, ph = (b >> 1) & 1u;
      const uint32_t nx0 = lookup(wt, b + 1), nx1 = lookup(wt + kEGather, b + 1);
      ptx::mbar_wait(&b_empty[st], ph ^ 1u);
      char* bs = smem + ESmem::b + st * 16384;
#pragma unroll
      for (uint32_t h = 0; h < 2; ++h) {  // rows wt and wt + 96
        const uint32_t j = wt + h * kEGather;
        if (j >= r16) continue;
        const uint64_t off = row_off(j, b);
        const char* base = p.arena + (static_cast<uint64_t>(h ? ph1 : ph0) << p.log2_page) + (off & pmask);
#pragma unroll
        for (uint32_t q = 0; q < 8; ++q) {
          char* dst = bs + swz(j, q);
          if (j >= r)
            ptx::cp_async_16(dst, p.arena, 0);
          else if (fast)
            ptx::cp_async_16(dst, base + q * 16, 16);
          else
            ptx::cp_async_16(dst, src.at(off + q * 16), 16);
        }
      }
      ptx::cp_async_mbar_arrive_noinc(&b_full[st]);
      ph0 = nx0;
      ph1 = nx1;
    }
  } else if (warp == 8) {
    if (lane == 0) {
      // ------------------------------------------------------- MMA issuer
      const uint32_t idesc = ptx::idesc_bf16_f32(kTileM, kEBlockN, false, true);
      const uint32_t vbase = ptx::smem_u32(smem + ESmem::v);
      const uint32_t lbo = r16 * 128;  // unused with one 64-column group
      ptx::mbar_wait(v_full, 0);
      for (uint32_t b = 0; b < nblk; ++b) {
        const uint32_t st = b & 1u, ph = (b >> 1) & 1u;
        ptx::mbar_wait(&b_full[st], ph);
        ptx::mbar_wait(&acc_empty[st], ph ^ 1u);
        ptx::fence_proxy_async_shared();
        ptx::tc_fence_after();
        const uint32_t bbase = ptx::smem_u32(smem + ESmem::b + st * 16384);
        for (uint32_t kk = 0; kk < r16 / 16; ++kk)
          ptx::umma_f16(tmem + st * kEBlockN,
                        ptx::smem_desc_sw128(vbase + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                        ptx::smem_desc_sw128(bbase + kk * 2048, lbo, 1024), idesc, kk != 0);
        ptx::umma_commit(&b_empty[st]);
        ptx::umma_commit(&acc_full[st]);
      }
    }
  } else {
    // ------------------------------------------------- epilogue (warps 4-7)
    const uint32_t m = (warp - 4) * 32 + lane;  // tile row == TMEM lane
    const uint32_t lane_base = ((warp & 3) * 32) << 16;
    const bool live = m < tile.nrows;  // rows past the run belong to the next one: add 0
    for (uint32_t b = 0; b < nblk; ++b) {
      const uint32_t st = b & 1u, ph = (b >> 1) & 1u;
      const uint32_t col0 = col_base + b * kEBlockN;
      char* ys = smem + ESmem::y + st * 16384;
      if (b >= 2) {  // the reduce-store of block b - 2 must have read stage st
        if (warp == 4 && lane == 0) ptx::bulk_wait_read_n<1>();
        ptx::named_bar_sync(1, 128);
      }
      ptx::mbar_wait(&acc_full[st], ph);
      ptx::tc_fence_after();
#pragma unroll 1
      for (uint32_t q = 0; q < kEBlockN / 16; ++q) {  // 16 columns = two 16-byte chunks
        uint32_t rv[16];
        ptx::tmem_ld_32x32b_x16(tmem + lane_base + st * kEBlockN + q * 16, rv);
        ptx::tmem_ld_wait();
#pragma unroll
        for (uint32_t hh = 0; hh < 2; ++hh) {
          const uint32_t ya = ptx::smem_u32(ys + swz(m, q * 2 + hh));
          uint32_t o[4];
#pragma unroll
          for (int i = 0; i < 4; ++i)
            o[i] = live ? pack_bf16x2(p.scale * __uint_as_float(rv[hh * 8 + 2 * i]),
                                      p.scale * __uint_as_float(rv[hh * 8 + 2 * i + 1]))
                        : 0u;
          asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(ya), "r"(o[0]), "r"(o[1]),
                       "r"(o[2]), "r"(o[3]) : "memory");
        }
      }
      ptx::tc_fence_before();
      ptx::fence_proxy_async_shared();  // generic-proxy smem writes -> TMA
      ptx::named_bar_sync(1, 128);
      if (warp == 4 && lane == 0) {
        ptx::mbar_arrive(&acc_empty[st]);
        ptx::tma_reduce_add_2d(&tmap_y, static_cast<int32_t>(col0), static_cast<int32_t>(tile.row0), ys);
        ptx::bulk_commit();
      }
    }
    if (warp == 4 && lane == 0) ptx::bulk_wait_all();
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, kETmemCols);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  if (!fn) throw CudaError("cuTensorMapEncodeTiled unavailable");
  return fn;
}


void make_tmap_2d(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows,
                  uint64_t row_stride_b, uint32_t box_cols, uint32_t box_rows) {
  const cuuint64_t dims[2] = {cols, std::max<uint64_t>(rows, 1)};
  const cuuint64_t strides[1] = {row_stride_b};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult cr = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                            strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string(cr));
}

}  // namespace

extern "C" int plora_debug_set_sgmv_flags(uint32_t flags) {
  g_sgmv_dbg = flags;
  return PLORA_OK;
}

extern "C" int plora_sgmv(plora_plan* plan, uint32_t layer, uint32_t proj, const void* x,
                          uint64_t x_stride, void* y, uint64_t y_stride, float scale,
                          plora_stream_t stream) {
  return guard([&] {
    if (!plan) throw ValidationError("null plan");
    check_io(plan, layer, proj, x, x_stride, y, y_stride);
    const plora_store& st = *plan->store;
    const ModelGeom& g = st.geom;
    const uint32_t din = g.m.d_in[proj], dout = g.m.d_out[proj];
    // The tensor-core path: bf16, rank <= 128, d_in % 64 == 0, d_out % 128 == 0.
    // Anything else (fp32 storage, wider ranks, odd widths) runs the exact
    // CUDA-core BGMV path, which handles every segment length.
    if (g.esize != 2 || plan->max_rank > kMaxRank || din % kChunkK || dout % kBlockN)
      return plora_bgmv(plan, layer, proj, x, x_stride, y, y_stride, scale, stream);
    if (plan->n_tiles == 0) return 0;
    DeviceCtx ctx(st.device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const uint32_t splits = sgmv_splits(plan->n_tiles, din);
    CUtensorMap tmap_x, tmap_y, tmap_v;
    make_tmap_2d(&tmap_x, x, din, plan->n_tokens, x_stride * 2, kChunkK, kTileM);
    make_tmap_2d(&tmap_y, y, dout, plan->n_tokens, y_stride * 2, 64, kTileM);
    make_tmap_2d(&tmap_v, plan->d_vbuf, kMaxRank, static_cast<uint64_t>(plan->n_tiles) * kTileM,
                 kMaxRank * 2, 64, kTileM);
    static bool attr = false;
    if (!attr) {
      PLORA_CUDA(cudaFuncSetAttribute(sgmv_shrink_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(SSmem::alloc)));
      PLORA_CUDA(cudaFuncSetAttribute(sgmv_expand_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(ESmem::alloc)));
      attr = true;
    }
    cudaLaunchAttribute pdl[1];
    pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl[0].val.programmaticStreamSerializationAllowed = 1;

    ShrinkArgs sa{};
    sa.arena = st.arena;
    sa.table = st.d_table;
    sa.tiles = plan->d_tiles;
    sa.units = plan->d_sunits;
    sa.vpart = plan->d_vpart;
    sa.vbuf = reinterpret_cast<__nv_bfloat16*>(plan->d_vbuf);
    sa.tcnt = plan->d_tcnt;
    sa.blk_mult = g.blk_mult(layer, proj);
    sa.log2_page = st.log2_page;
    sa.d_in = din;
    sa.splits = splits;
    sa.dbg = g_sgmv_dbg;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(plan->n_sunits * splits);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = SSmem::alloc;
    cfg.stream = s;
    cfg.attrs = pdl;
    cfg.numAttrs = 1;
    PLORA_CUDA(cudaLaunchKernelEx(&cfg, sgmv_shrink_kernel, sa, tmap_x));
    count_launch();
    if (g_sgmv_dbg & 8u) return 0;

    ExpandArgs ea{};
    ea.arena = st.arena;
    ea.table = st.d_table;
    ea.tiles = plan->d_tiles;
    ea.y = static_cast<char*>(y);
    ea.y_stride_b = y_stride * 2;
    ea.blk_mult = g.blk_mult(layer, proj);
    ea.log2_page = st.log2_page;
    ea.d_in = din;
    ea.d_out = dout;
    ea.ngroups = (dout / kEBlockN + kGroupBlocks - 1) / kGroupBlocks;
    ea.scale = scale;
    cfg.gridDim = dim3(plan->n_tiles * ea.ngroups);
    cfg.blockDim = dim3(kEThreads);
    cfg.dynamicSmemBytes = ESmem::alloc;
    PLORA_CUDA(cudaLaunchKernelEx(&cfg, sgmv_expand_kernel, ea, tmap_y, tmap_v));
    count_launch();
    return 0;
  });
}
