// Paged multi-LoRA prefill op (gathered SGMV) on the 5th-generation tensor
// cores (tcgen05 + TMEM) for sm_100a.
//
// y[t, :] += scale · bf16(x[t, :] · Aᵀ) · Bᵀ for the tokens of each run (a
// stretch of consecutive tokens with one adapter).  The
// reference bills this as cost_model.prefill_ms (cost_model.hpp:32-34,
// src/engine.cpp:355).
//
// Three kernels per (layer, proj) call, chained by programmatic dependent
// launch:
//
//  shrink  persistent, one CTA per SM: LPT-scheduled work items, each a
//          unit (one 128-token tile, or two consecutive full tiles of one
//          run sharing every A chunk) × one K slice.  Warp 0 TMA-loads x
//          chunks [128 × 64] (SWIZZLE_128B) into a 4-stage ring; warps 1-6
//          gather the adapter's A rows with 16-byte cp.async pieces, each
//          translated through the device page table, straight into the UMMA
//          K-major SW128 layout (rank zero-padded to 16 in smem only); warp 7
//          issues tcgen05.mma (M = 128, N = r16) into one of two TMEM
//          accumulator sets; warps 8-11 bulk-copy the fp32 partial out while
//          the next item streams.
//  reduce  sums the K-slice partials in split order (deterministic) and
//          writes V in bf16 — the rounding point between shrink and expand.
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
#include "tmap.cuh"

using namespace plora;

namespace plora {
void check_io(const plora_plan* plan, uint32_t layer, uint32_t proj, const void* x,
              uint64_t x_stride, void* y, uint64_t y_stride);
}

extern "C" int plora_bgmv(plora_plan* plan, uint32_t layer, uint32_t proj, const void* x,
                          uint64_t x_stride, void* y, uint64_t y_stride, float scale,
                          plora_stream_t stream);

namespace {
using namespace plora::tmap;

uint32_t g_sgmv_dbg = 0;  // plora_debug_set_sgmv_flags
constexpr uint32_t kDbgPersistentExpand = 1u << 20;  // run the persistent expand (measured slower) instead of the tiled one

constexpr uint32_t kTileM = 128;
constexpr uint32_t kChunkK = 64;   // shrink K per stage (one 128-byte swizzle row)
constexpr uint32_t kBlockN = 128;  // expand output columns per CTA
constexpr uint32_t kMaxRank = 128;
constexpr uint32_t kTmemCols = 128;
constexpr int kSGather = 192;       // shrink: warps 1-6
constexpr int kEGather = 96;        // expand: warps 1-3

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// ------------------------------------------------------------------ shrink
// Persistent: one CTA per SM runs its LPT-scheduled work items, each a unit
// (one tile, or two consecutive full tiles of one run that share every A
// chunk) × one K slice.  The stage ring runs across items; the TMEM
// accumulators are double-buffered, so the epilogue of item i (TMEM ->
// shared -> bulk copy of the fp32 partial) overlaps the loads and MMAs of
// item i + 1.  sgmv_reduce_kernel then sums the K-slice partials in split
// order (deterministic) into the bf16 V tiles.
//   warp 0      TMA producer of the x chunks (one 128 × 64 box per tile)
//   warps 1-6   A gathers: rank row n of the chunk, page-table lookup a chunk ahead
//   warp 7      MMA issuer (and TMEM allocator)
//   warps 8-11  epilogue (warp 8 + q reads TMEM lanes 32q..32q+31)
constexpr int kSStages = 4;
constexpr uint32_t kSStageBytes = 49152;  // 16 KiB parts: x of each tile, then A of each projection
constexpr uint32_t kSThreads = 384;
constexpr uint32_t kStgBytes = 8192;  // per epilogue warp: 32 rows × 64 fp32
constexpr uint32_t kSTmemCols = 512;  // [buffer][tile][128 columns]

struct ShrinkArgs {
  const char* arena;
  const uint32_t* table;
  const SgmvTile* tiles;
  const SgmvItem* items;
  const uint32_t* cta_items;  // [cta + 1] offsets into items
  float* vpart;               // [proj][tile][split] blocks of 128 × 128 fp32 (128 × r16 used)
  uint64_t vpart_pstride;     // floats between projection regions
  uint64_t blk_mult[2];       // per projection of the x chunk
  uint32_t np;                // projections sharing each x chunk (nt · np <= 2)
  uint32_t log2_page;
  uint32_t d_in;
  uint32_t splits;
  uint32_t dbg;  // diagnostics (plora_debug_set_sgmv_flags): 1 no A gather, 2 no MMA, 4 no x load, 16 no epilogue
  uint32_t g4;   // pages >= 256 B: A rows by TMA gather4 over the arena viewed as 128-byte rows
};

struct SSmem {
  static constexpr uint32_t stages = 0;  // 1024-aligned
  static constexpr uint32_t stg = stages + kSStages * kSStageBytes;
  static constexpr uint32_t bars = stg + 4 * kStgBytes;
  static constexpr uint32_t n_bars = 2 * kSStages + 4;  // full, empty, tfull[2], tempty[2]
  static constexpr uint32_t tmem_slot = bars + n_bars * 8;
  static constexpr uint32_t total = tmem_slot + 8;
  static constexpr uint32_t alloc = total + 1024;  // alignment slack
};

struct UnitInfo {
  uint32_t tile_a, tile_b, nt, row0_a, row0_b, r, r16, table_off, split;
};

__device__ __forceinline__ UnitInfo unit_info(const SgmvItem* it) {
  const uint4 a = __ldg(reinterpret_cast<const uint4*>(it));
  const uint4 b = __ldg(reinterpret_cast<const uint4*>(it) + 1);
  UnitInfo u;
  u.tile_a = a.x;
  u.tile_b = a.y;
  u.nt = a.y != 0xffffffffu ? 2 : 1;
  u.row0_a = a.z;
  u.row0_b = a.w;
  u.table_off = b.x;
  u.r = b.y;
  u.r16 = (b.y + 15) & ~15u;
  u.split = b.z;
  return u;
}

// Partial block layout (floats): [quarter q][pass][32 rows][pw], pass = 64
// columns (pw = min(64, r16 - 64·pass)); 16-byte chunk j of row i stored at
// j ^ (i & swm(pw)) so the staging writes are free of bank conflicts.
__device__ __forceinline__ uint32_t part_swm(uint32_t pw4) { return min(8u, pw4 & (0u - pw4)) - 1u; }

__global__ void __launch_bounds__(kSThreads, 1)
    sgmv_shrink_kernel(const ShrinkArgs p, const __grid_constant__ CUtensorMap tmap_x,
                       const __grid_constant__ CUtensorMap tmap_arena) {
  extern __shared__ char smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + SSmem::bars);
  uint64_t* empty = full + kSStages;
  uint64_t* tfull = full + 2 * kSStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + SSmem::tmem_slot);

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t it0 = p.cta_items[blockIdx.x], it1 = p.cta_items[blockIdx.x + 1];
  const uint32_t kslice = p.d_in / p.splits, NK = kslice / kChunkK;

  ptx::pdl_launch_dependents();  // the expand may start gathering its weights
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSStages; ++s) {
      ptx::mbar_init(&full[s], 1 + kSGather);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], 4);  // one arrival per epilogue warp
    }
    ptx::fence_mbar_init();
  }
  if (warp == 7) ptx::tmem_alloc(tmem_slot, kSTmemCols);
  if (warp == 0 && lane == 0) ptx::prefetch_tmap(&tmap_x);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer (x chunks)
    if (lane == 0) {
      ptx::pdl_wait();  // x is written by earlier kernels in the stream
      uint32_t g = 0;
      for (uint32_t it = it0; it < it1; ++it) {
        const UnitInfo u = unit_info(p.items + it);
        const uint32_t k0 = u.split * kslice;
        for (uint32_t kc = 0; kc < NK; ++kc, ++g) {
          const uint32_t st = g % kSStages, ph = (g / kSStages) & 1u;
          ptx::mbar_wait(&empty[st], ph ^ 1u);
          if (p.dbg & 4u) {
            ptx::mbar_arrive(&full[st]);
            continue;
          }
          char* xs = smem + SSmem::stages + st * kSStageBytes;
          ptx::mbar_arrive_expect_tx(&full[st], u.nt * kTileM * kChunkK * 2);
          ptx::tma_load_2d(xs, &tmap_x, static_cast<int32_t>(k0 + kc * kChunkK),
                           static_cast<int32_t>(u.row0_a), &full[st]);
          if (u.nt == 2)
            ptx::tma_load_2d(xs + kTileM * kChunkK * 2, &tmap_x, static_cast<int32_t>(k0 + kc * kChunkK),
                             static_cast<int32_t>(u.row0_b), &full[st]);
        }
      }
    }
  } else if (warp <= 6) {
    // ----------------------------------------------- A gathers (paged rows)
    // Thread n owns rank row n (r16 <= 128 < 192).  A row's K slice spans
    // few pages: the thread keeps the current page's frame and the next
    // one's (looked up a page ahead), so a lookup never stalls a chunk.
    // The next item's record is fetched one item ahead.
    const uint32_t n = threadIdx.x - 32;
    const bool fast = p.log2_page >= 8;
    const uint64_t pmask = (1ull << p.log2_page) - 1;
    uint32_t g = 0;
    UnitInfo un = it0 < it1 ? unit_info(p.items + it0) : UnitInfo{};
    for (uint32_t it = it0; it < it1; ++it) {
      const UnitInfo u = un;
      if (it + 1 < it1) un = unit_info(p.items + it + 1);
      const uint32_t k0 = u.split * kslice;
      const PagedSrc src{p.arena, p.table, u.table_off, p.log2_page};
      const bool live = fast && n < u.r;
      uint64_t off0[2];
      uint32_t lp[2], lp_last[2], e_cur[2], e_nxt[2];
#pragma unroll
      for (uint32_t q = 0; q < 2; ++q) {  // this row of each projection's A block
        const uint64_t blk = static_cast<uint64_t>(u.r) * (q ? p.blk_mult[1] : p.blk_mult[0]) * 2;
        off0[q] = blk + (static_cast<uint64_t>(n) * p.d_in + k0) * 2;
        lp_last[q] = static_cast<uint32_t>((off0[q] + kslice * 2 - 1) >> p.log2_page);
        lp[q] = static_cast<uint32_t>(off0[q] >> p.log2_page);
        const bool lq = live && q < p.np;
        e_cur[q] = lq ? __ldg(p.table + u.table_off + lp[q]) : 0u;
        e_nxt[q] = lq && lp[q] < lp_last[q] ? __ldg(p.table + u.table_off + lp[q] + 1) : 0u;
      }
      for (uint32_t kc = 0; kc < NK; ++kc, ++g) {
        const uint32_t st = g % kSStages, ph = (g / kSStages) & 1u;
#pragma unroll
        for (uint32_t q = 0; q < 2; ++q) {
          const uint64_t off = off0[q] + kc * kChunkK * 2;
          if (live && q < p.np && (off >> p.log2_page) != lp[q]) {  // crossed into the next page
            lp[q] = static_cast<uint32_t>(off >> p.log2_page);
            e_cur[q] = e_nxt[q];
            e_nxt[q] = lp[q] < lp_last[q] ? __ldg(p.table + u.table_off + lp[q] + 1) : 0u;
          }
        }
        ptx::mbar_wait(&empty[st], ph ^ 1u);
        // Groups of four real rows go by one TMA gather4 (its row indices
        // collected by the group's first lane); padding rows and the rows of
        // a partial last group by 16-byte cp.async.
        // Every other group of four goes by cp.async instead: the TMA unit
        // (gather4 moves 512 B per op) and the LSU pipes then share the rows
        // (profiles/r02l_sgmv_g4_split.txt: shrink 60.2 -> 54.4 us at cfg3).
        // Diagnostics: 16384 all by gather4, 4096 one in four by cp.async,
        // 8192 three in four, 2048 all.
        const uint32_t gi = (n >> 2) & 3u;
        const bool by_lsu = (p.dbg & 2048u) || ((p.dbg & 4096u) ? gi == 3u
                                               : (p.dbg & 8192u) ? gi != 0u
                                               : !(p.dbg & 16384u) && (gi & 1u));
        const bool g4 = p.g4 && (n | 3u) < u.r && !by_lsu;
        if (p.g4 && !(p.dbg & 1u)) {
#pragma unroll
          for (uint32_t q = 0; q < 2; ++q) {
            if (q >= p.np) break;
            const uint64_t off = off0[q] + kc * kChunkK * 2;
            const int32_t row = static_cast<int32_t>(((static_cast<uint64_t>(e_cur[q]) << p.log2_page) +
                                                      (off & pmask)) >> 7);
            const uint32_t l0 = lane & ~3u;
            const int32_t r0 = __shfl_sync(0xffffffffu, row, l0), r1 = __shfl_sync(0xffffffffu, row, l0 + 1);
            const int32_t r2 = __shfl_sync(0xffffffffu, row, l0 + 2), r3 = __shfl_sync(0xffffffffu, row, l0 + 3);
            if (g4 && (lane & 3u) == 0) {
              char* wdst = smem + SSmem::stages + st * kSStageBytes + (u.nt + q) * kTileM * kChunkK * 2;
              ptx::mbar_expect_tx(&full[st], 4 * kChunkK * 2);
              ptx::tma_gather4(wdst + n * kChunkK * 2, &tmap_arena, 0, r0, r1, r2, r3, &full[st]);
            }
          }
        }
        if (n < u.r16 && !g4 && !(p.dbg & 1u)) {
#pragma unroll
          for (uint32_t q = 0; q < 2; ++q) {
            if (q >= p.np) break;
            char* wdst = smem + SSmem::stages + st * kSStageBytes + (u.nt + q) * kTileM * kChunkK * 2;
            const uint64_t off = off0[q] + kc * kChunkK * 2;
            if (n >= u.r) {
#pragma unroll
              for (uint32_t c = 0; c < 8; ++c) ptx::cp_async_16(wdst + swz(n, c), p.arena, 0);  // zero padding
            } else if (fast) {
              const char* base = p.arena + (static_cast<uint64_t>(e_cur[q]) << p.log2_page) + (off & pmask);
#pragma unroll
              for (uint32_t c = 0; c < 8; ++c) ptx::cp_async_16(wdst + swz(n, c), base + c * 16, 16);
            } else {
              for (uint32_t c = 0; c < 8; ++c) ptx::cp_async_16(wdst + swz(n, c), src.at(off + c * 16), 16);
            }
          }
        }
        ptx::cp_async_mbar_arrive_noinc(&full[st]);
      }
    }
  } else if (warp == 7) {
    // ------------------------------------------------------- MMA issuer
    if (lane == 0) {
      const uint32_t sbase = ptx::smem_u32(smem + SSmem::stages);
      uint32_t g = 0;
      for (uint32_t it = it0, i = 0; it < it1; ++it, ++i) {
        const UnitInfo u = unit_info(p.items + it);
        const uint32_t buf = i & 1u, tb = tmem + buf * 2 * kTmemCols;
        const uint32_t idesc = ptx::idesc_bf16_f32(kTileM, u.r16, false, false);
        ptx::mbar_wait(&tempty[buf], ((i >> 1) & 1u) ^ 1u);  // epilogue of item i - 2 read it
        ptx::tc_fence_after();
        for (uint32_t kc = 0; kc < NK; ++kc, ++g) {
          const uint32_t st = g % kSStages, ph = (g / kSStages) & 1u;
          ptx::mbar_wait(&full[st], ph);
          if (p.dbg & 2u) {
            ptx::mbar_arrive(&empty[st]);
            continue;
          }
          ptx::fence_proxy_async_shared();
          ptx::tc_fence_after();
          // accumulators: tile t against the A chunk (np = 1), or the one tile
          // against projection q's A chunk (np = 2), in TMEM columns 128 · (t | q)
          const uint32_t xa = sbase + st * kSStageBytes;
          constexpr uint32_t kPart = kTileM * kChunkK * 2;
          const uint32_t wa = xa + u.nt * kPart;  // first A chunk
          const bool second = u.nt == 2 || p.np == 2;
#pragma unroll
          for (uint32_t k = 0; k < kChunkK / 16; ++k) {
            const uint64_t x0 = ptx::smem_desc_sw128(xa + k * 32, 16, 1024);
            const uint64_t w0 = ptx::smem_desc_sw128(wa + k * 32, 16, 1024);
            ptx::umma_f16(tb, x0, w0, idesc, (kc | k) != 0);
            if (second) {
              const uint64_t x1 = p.np == 2 ? x0 : ptx::smem_desc_sw128(xa + kPart + k * 32, 16, 1024);
              const uint64_t w1 = p.np == 2 ? ptx::smem_desc_sw128(wa + kPart + k * 32, 16, 1024) : w0;
              ptx::umma_f16(tb + kTmemCols, x1, w1, idesc, (kc | k) != 0);
            }
          }
          ptx::umma_commit(&empty[st]);
        }
        ptx::umma_commit(&tfull[buf]);
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue
    const uint32_t q = warp - 8;
    const uint32_t lane_base = (q * 32) << 16;
    float* stg = reinterpret_cast<float*>(smem + SSmem::stg + q * kStgBytes);
    for (uint32_t it = it0, i = 0; it < it1; ++it, ++i) {
      const UnitInfo u = unit_info(p.items + it);
      const uint32_t buf = i & 1u, tb = tmem + buf * 2 * kTmemCols;
      ptx::mbar_wait(&tfull[buf], (i >> 1) & 1u);
      ptx::tc_fence_after();
      const uint32_t nacc = (p.dbg & 16u) ? 0u : u.nt * p.np;
      for (uint32_t a = 0; a < nacc; ++a) {
        const uint32_t t = a / p.np, pj = a - t * p.np;
        const uint32_t tile_i = t ? u.tile_b : u.tile_a;
        float* blk = p.vpart + pj * p.vpart_pstride +
                     (static_cast<uint64_t>(tile_i) * p.splits + u.split) * kTileM * kMaxRank + q * 32 * u.r16;
        for (uint32_t pass = 0; pass * 64 < u.r16; ++pass) {
          const uint32_t pw = min(64u, u.r16 - pass * 64), pw4 = pw / 4, swm = part_swm(pw4);
          if (lane == 0) ptx::bulk_wait_read_n<0>();  // the staging buffer's last copy has read it
          __syncwarp();
          for (uint32_t cc = 0; cc < pw / 16; ++cc) {
            uint32_t rv[16];
            ptx::tmem_ld_32x32b_x16(tb + lane_base + a * kTmemCols + pass * 64 + cc * 16, rv);
            ptx::tmem_ld_wait();
#pragma unroll
            for (uint32_t c = 0; c < 4; ++c)
              reinterpret_cast<uint4*>(stg + lane * pw)[(cc * 4 + c) ^ (lane & swm)] =
                  make_uint4(rv[4 * c], rv[4 * c + 1], rv[4 * c + 2], rv[4 * c + 3]);
          }
          ptx::fence_proxy_async_shared();
          __syncwarp();
          if (lane == 0) {
            ptx::bulk_s2g(blk + pass * 32 * 64, stg, 32 * pw * 4);
            ptx::bulk_commit();
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty[buf]);  // TMEM buffer free for item i + 2
    }
    if (lane == 0) ptx::bulk_wait_all();  // partials written before the grid completes
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 7) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, kSTmemCols);
  }
}

// ------------------------------------------------------------------ reduce
// V tile i = bf16(Σ_split partial[i][split]), summed in split order.  Block
// (tile, quarter) reads its quarter's float4s of every split coalesced.
constexpr uint32_t kRThreads = 256;

struct ReduceArgs {
  const SgmvTile* tiles;
  const float* vpart;
  __nv_bfloat16* vbuf;  // [proj][tile][128][128] bf16
  uint64_t vpart_pstride;  // floats between projection regions
  uint32_t n_tiles;
  uint32_t splits;
  float scale;  // V = bf16(scale · Σ partials): 1 for plora_sgmv, the LoRA scale when fused
};

__global__ void __launch_bounds__(kRThreads) sgmv_reduce_kernel(const ReduceArgs p) {
  ptx::pdl_launch_dependents();
  const uint32_t pj = blockIdx.x / (4 * p.n_tiles), rest = blockIdx.x - pj * 4 * p.n_tiles;
  const uint32_t tile = rest >> 2, qq = rest & 3;
  const uint32_t r16 = (p.tiles[tile].rank + 15) & ~15u, q4 = 8 * r16;  // float4s per quarter
  constexpr uint32_t kSplitStride = kTileM * kMaxRank / 4;  // float4s
  const float4* v0 = reinterpret_cast<const float4*>(p.vpart + pj * p.vpart_pstride) +
                     static_cast<uint64_t>(tile) * p.splits * kSplitStride + qq * q4;
  __nv_bfloat16* vb = p.vbuf + (static_cast<uint64_t>(pj) * p.n_tiles + tile) * kTileM * kMaxRank;
  ptx::pdl_wait();  // the shrink's partials
  constexpr uint32_t kU = 4;
  for (uint32_t f0 = threadIdx.x; f0 < q4; f0 += kU * kRThreads) {
    float4 acc[kU];
#pragma unroll
    for (uint32_t c = 0; c < kU; ++c) acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (uint32_t sp = 0; sp < p.splits; sp += 2) {
      float4 a0[kU], a1[kU];
#pragma unroll
      for (uint32_t c = 0; c < kU; ++c) {
        const uint32_t f = f0 + c * kRThreads;
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
        a0[c] = f < q4 ? __ldcg(v0 + sp * kSplitStride + f) : z;
        a1[c] = f < q4 && sp + 1 < p.splits ? __ldcg(v0 + (sp + 1) * kSplitStride + f) : z;
      }
#pragma unroll
      for (uint32_t c = 0; c < kU; ++c) {
        acc[c].x += a0[c].x; acc[c].y += a0[c].y; acc[c].z += a0[c].z; acc[c].w += a0[c].w;
        acc[c].x += a1[c].x; acc[c].y += a1[c].y; acc[c].z += a1[c].z; acc[c].w += a1[c].w;
      }
    }
#pragma unroll
    for (uint32_t c = 0; c < kU; ++c) {
      const uint32_t f = f0 + c * kRThreads;
      if (f >= q4) continue;
      const uint32_t pass = f / 512, rem = f - pass * 512;
      const uint32_t pw4 = min(16u, r16 / 4 - pass * 16), row = rem / pw4, jp = rem - row * pw4;
      const uint32_t j = jp ^ (row & part_swm(pw4));
      uint2 o;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&o);
      h[0] = __floats2bfloat162_rn(p.scale * acc[c].x, p.scale * acc[c].y);
      h[1] = __floats2bfloat162_rn(p.scale * acc[c].z, p.scale * acc[c].w);
      *reinterpret_cast<uint2*>(vb + (qq * 32 + row) * kMaxRank + pass * 64 + j * 4) = o;
    }
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
// epilogue releases the accumulators the MMA loop waits for).  (Eight
// epilogue warps measured slower: the y stream, not the epilogue, bounds it.)
constexpr int kEThreads = 288;
constexpr uint32_t kEEpiThreads = 128;

struct ExpandArgs {
  const char* arena;
  const uint32_t* table;
  const SgmvTile* tiles;
  uint64_t blk_mult[2];  // per projection (CTA (proj, tile, group))
  uint32_t log2_page;
  uint32_t d_in;
  uint32_t d_out;
  uint32_t n_tiles;
  uint32_t ngroups;  // column groups per tile
  uint32_t np;       // projections of the call (persistent expand)
  uint64_t* trace;   // diagnostics (plora_debug_set_trace): [cta][block < kPTrace][8] SM clocks, or nullptr
  float scale;
  uint32_t dbg;  // diagnostics: 64 no y reduce-add, 128 no Bᵀ gather, 256 no MMA, 512 prologue only
  uint32_t g4;   // pages >= 256 B: Bᵀ rows by TMA gather4 (see ShrinkArgs::g4)
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
    sgmv_expand_kernel(const ExpandArgs p, const __grid_constant__ CUtensorMap tmap_y0,
                       const __grid_constant__ CUtensorMap tmap_y1,
                       const __grid_constant__ CUtensorMap tmap_v,
                       const __grid_constant__ CUtensorMap tmap_arena) {
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

  const uint32_t per_proj = p.n_tiles * p.ngroups;
  const uint32_t pj = blockIdx.x / per_proj, tile_i = (blockIdx.x % per_proj) / p.ngroups,
                 grp = blockIdx.x % p.ngroups;
  const CUtensorMap* tmap_y = pj ? &tmap_y1 : &tmap_y0;
  const SgmvTile tile = p.tiles[tile_i];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t r = tile.rank, r16 = (r + 15) & ~15u;
  const uint64_t bt = (static_cast<uint64_t>(r) * (pj ? p.blk_mult[1] : p.blk_mult[0]) +
                       static_cast<uint64_t>(r) * p.d_in) * 2;
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
      ptx::mbar_init(&acc_empty[i], kEEpiThreads / 32);  // each epilogue warp, once its TMEM reads are done
    }
    ptx::fence_mbar_init();
  }
  if (warp == 4) ptx::tmem_alloc(tmem_slot, kETmemCols);
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(tmap_y);
    ptx::prefetch_tmap(&tmap_v);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (p.dbg & 512u) {
  } else if (warp == 0) {
    // ----------------------------------------------- TMA: V tile once
    if (lane == 0) {
      ptx::pdl_wait();  // V comes from the shrink (and y may be read by earlier kernels)
      ptx::mbar_arrive_expect_tx(v_full, vboxes * 16384);
      for (uint32_t bx = 0; bx < vboxes; ++bx)
        ptx::tma_load_2d(smem + ESmem::v + bx * 16384, &tmap_v, static_cast<int32_t>(bx * 64),
                         static_cast<int32_t>((pj * p.n_tiles + tile_i) * kTileM), v_full);
    }
  } else if (warp < 4) {
    // ----------------------------------- Bᵀ block gathers (paged rows)
    // Thread wt owns rank rows wt and wt + 96.  A row's 1 KiB group slice
    // spans few pages: the thread keeps each row's current page frame and
    // the next one's (looked up a page ahead), so no block waits on a lookup.
    const uint32_t wt = threadIdx.x - 32;
    const bool fast = p.log2_page >= 7;  // a row's 128-byte block slice lies in one page
    const uint64_t pmask = (1ull << p.log2_page) - 1;
    auto row_off = [&](uint32_t j, uint32_t b) {
      return bt + (static_cast<uint64_t>(j) * p.d_out + col_base + b * kEBlockN) * 2;
    };
    uint32_t lp[2], lp_last[2], e_cur[2], e_nxt[2];
#pragma unroll
    for (uint32_t h = 0; h < 2; ++h) {
      const uint32_t j = wt + h * kEGather;
      const bool live = fast && j < r && nblk > 0;
      lp[h] = static_cast<uint32_t>(row_off(j, 0) >> p.log2_page);
      lp_last[h] = live ? static_cast<uint32_t>((row_off(j, nblk - 1) + kEBlockN * 2 - 1) >> p.log2_page) : 0u;
      e_cur[h] = live ? __ldg(p.table + tile.table_off + lp[h]) : 0u;
      e_nxt[h] = live && lp[h] < lp_last[h] ? __ldg(p.table + tile.table_off + lp[h] + 1) : 0u;
    }
    for (uint32_t b = 0; b < nblk; ++b) {
      const uint32_t st = b & 1u, ph = (b >> 1) & 1u;
#pragma unroll
      for (uint32_t h = 0; h < 2; ++h) {
        const uint32_t j = wt + h * kEGather;
        const uint32_t lpb = static_cast<uint32_t>(row_off(j, b) >> p.log2_page);
        if (fast && j < r && lpb != lp[h]) {  // crossed into the next page
          lp[h] = lpb;
          e_cur[h] = e_nxt[h];
          e_nxt[h] = lpb < lp_last[h] ? __ldg(p.table + tile.table_off + lpb + 1) : 0u;
        }
      }
      ptx::mbar_wait(&b_empty[st], ph ^ 1u);
      char* bs = smem + ESmem::b + st * 16384;
      // groups of four real rows by TMA gather4 (row indices collected by the
      // group's first lane), the rest by 16-byte cp.async
      bool g4[2];
#pragma unroll
      for (uint32_t h = 0; h < 2; ++h) {
        const uint32_t j = wt + h * kEGather;
        // (unlike the shrink, sending half the rows by cp.async here measured
        // slower: 178.0 vs 164.5 us per layer call, profiles/r02l_sgmv_g4_split.txt)
        g4[h] = p.g4 && (j | 3u) < r;
        if (p.g4 && !(p.dbg & 128u)) {
          const int32_t row = static_cast<int32_t>(
              ((static_cast<uint64_t>(e_cur[h]) << p.log2_page) + (row_off(j, b) & pmask)) >> 7);
          const uint32_t l0 = lane & ~3u;
          const int32_t r0 = __shfl_sync(0xffffffffu, row, l0), r1 = __shfl_sync(0xffffffffu, row, l0 + 1);
          const int32_t r2 = __shfl_sync(0xffffffffu, row, l0 + 2), r3 = __shfl_sync(0xffffffffu, row, l0 + 3);
          if (g4[h] && (lane & 3u) == 0) {
            ptx::mbar_expect_tx(&b_full[st], 4 * kEBlockN * 2);
            ptx::tma_gather4(bs + j * kEBlockN * 2, &tmap_arena, 0, r0, r1, r2, r3, &b_full[st]);
          }
        }
      }
#pragma unroll
      for (uint32_t h = 0; h < 2; ++h) {  // rows wt and wt + 96
        const uint32_t j = wt + h * kEGather;
        if (j >= r16 || g4[h] || (p.dbg & 128u)) continue;
        const uint64_t off = row_off(j, b);
        const char* base = p.arena + (static_cast<uint64_t>(e_cur[h]) << p.log2_page) + (off & pmask);
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
        for (uint32_t kk = 0; kk < ((p.dbg & 256u) ? 0u : r16 / 16); ++kk)
          ptx::umma_f16(tmem + st * kEBlockN,
                        ptx::smem_desc_sw128(vbase + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                        ptx::smem_desc_sw128(bbase + kk * 2048, lbo, 1024), idesc, kk != 0);
        ptx::umma_commit(&b_empty[st]);
        ptx::umma_commit(&acc_full[st]);
      }
    }
  } else {
    // ------------------------------------------------- epilogue (warps 4-7)
    const uint32_t m = (warp & 3) * 32 + lane;  // tile row == TMEM lane
    const uint32_t lane_base = ((warp & 3) * 32) << 16;
    const bool live = m < tile.nrows;  // rows past the run belong to the next one: add 0
    for (uint32_t b = 0; b < nblk; ++b) {
      const uint32_t st = b & 1u, ph = (b >> 1) & 1u;
      const uint32_t col0 = col_base + b * kEBlockN;
      char* ys = smem + ESmem::y + st * 16384;
      if (b >= 2) {  // the reduce-store of block b - 2 must have read stage st
        if (warp == 4 && lane == 0) ptx::bulk_wait_read_n<1>();
        ptx::named_bar_sync(1, kEEpiThreads);
      }
      ptx::mbar_wait(&acc_full[st], ph);
      ptx::tc_fence_after();
      // the warp's 32 rows × 64 columns in one TMEM round trip, then the
      // accumulator goes back to the MMA warp before the smem writes
      uint32_t rv[kEBlockN / 16][16];
#pragma unroll
      for (uint32_t q = 0; q < kEBlockN / 16; ++q)
        ptx::tmem_ld_32x32b_x16(tmem + lane_base + st * kEBlockN + q * 16, rv[q]);
      ptx::tmem_ld_wait();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&acc_empty[st]);  // one arrival per epilogue warp
#pragma unroll
      for (uint32_t q = 0; q < kEBlockN / 16; ++q) {  // 16 columns = two 16-byte chunks
#pragma unroll
        for (uint32_t hh = 0; hh < 2; ++hh) {
          const uint32_t ya = ptx::smem_u32(ys + swz(m, q * 2 + hh));
          uint32_t o[4];
#pragma unroll
          for (int i = 0; i < 4; ++i)
            o[i] = live ? pack_bf16x2(p.scale * __uint_as_float(rv[q][hh * 8 + 2 * i]),
                                      p.scale * __uint_as_float(rv[q][hh * 8 + 2 * i + 1]))
                        : 0x80008000u;  // bf16 -0.0: the exact additive identity of the reduce-add
          asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(ya), "r"(o[0]), "r"(o[1]),
                       "r"(o[2]), "r"(o[3]) : "memory");
        }
      }
      ptx::fence_proxy_async_shared();  // generic-proxy smem writes -> TMA
      ptx::named_bar_sync(1, kEEpiThreads);
      if (warp == 4 && lane == 0) {
        if (!(p.dbg & 64u)) ptx::tma_reduce_add_2d(tmap_y, static_cast<int32_t>(col0), static_cast<int32_t>(tile.row0), ys);
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

// ------------------------------------------------------- persistent expand
// An alternative to sgmv_expand_kernel, selected by plora_debug_set_sgmv_flags
// bit 20 and measured SLOWER at cfg3 (layer call 173 vs 165 us,
// profiles/r02o_sgmv_persistent_expand.txt): its per-block pipeline (Bᵀ
// gather4 latency ~1.6 us under load, ~0.45 us of epilogue per block on the
// critical chain) ends up serial per SM, where the tiled grid's two resident
// CTAs per SM overlap one CTA's setup and drain with the other's blocks.
// One CTA per SM walks a contiguous range of the call's
// 64-column output blocks, ordered (proj, tile, block) — ~111 blocks per SM at
// cfg3 — so the per-CTA setup (barriers, TMEM, the first V load) and the final
// drain are paid once per SM instead of once per 512 columns, and the block
// pipeline runs kPStages deep across tile boundaries:
//   warp 0      TMA of the V tiles, two stages (the next tile's V streams
//               while the current tile's blocks run)
//   warps 1-8   Bᵀ block gathers into kPStages stages: groups of four rows
//               by TMA gather4, spread round-robin over the eight warps (a
//               warp issues its lanes' TMA ops one after another, ~84 cycles
//               each), the remaining rows by 16-byte cp.async
//   warps 9-16  epilogue, two groups of four warps taking alternate blocks:
//               TMEM -> bf16(scale · D) -> staging buffer -> TMA reduce-add
//               into y
//   warp 17     MMA issuer into kPStages TMEM accumulators of 64 columns
// Same arithmetic as sgmv_expand_kernel (bit-identical y).
constexpr uint32_t kPStages = 6;      // Bᵀ block stages (gather4 latency under load is ~1.6 us)
constexpr uint32_t kPAcc = 4;         // TMEM accumulators of 64 columns (k % 4; group k % 2)
constexpr uint32_t kPGatherWarps = 8;
constexpr uint32_t kPGather = kPGatherWarps * 32;
constexpr uint32_t kPEpi0 = 1 + kPGatherWarps;  // first epilogue warp
constexpr uint32_t kPMma = kPEpi0 + 8;
constexpr int kPThreads = (kPMma + 1) * 32;
constexpr uint32_t kPVStages = 3;  // V tiles in flight: a unit's V loads two units ahead
struct PSmem {  // ~225 KB: one CTA per SM
  static constexpr uint32_t v = 0;                        // [kPVStages][2 atoms][128 rows × 128 B] SW128
  static constexpr uint32_t y = v + kPVStages * 32768;    // [8 epilogue warps][32 rows × 128 B] SW128
  static constexpr uint32_t b = y + 8 * 4096;             // [kPStages][r16 × 128 B] MN-major SW128
  static constexpr uint32_t bars = b + kPStages * 16384;
  // v_full[V], v_empty[V], b_full[S], b_empty[S], acc_full[A], acc_empty[A]
  static constexpr uint32_t n_bars = 2 * kPVStages + 2 * kPStages + 2 * kPAcc;
  static constexpr uint32_t tmem_slot = bars + n_bars * 8;
  static constexpr uint32_t total = tmem_slot + 8;
  static constexpr uint32_t alloc = total + 1024;
};
static_assert(PSmem::alloc <= 232448, "persistent expand shared memory");
constexpr uint32_t kPTrace = 128;
__device__ __forceinline__ void ptrace(const ExpandArgs& p, uint32_t k, int f) {
  if (p.trace && k < kPTrace) p.trace[(blockIdx.x * kPTrace + k) * 8 + f] = clock64();
}

// Work units: (proj, tile, group of kPUnitBlocks 64-column blocks), dealt
// round-robin to the CTAs (unit i to CTA i mod grid), so at any moment the
// CTAs work on a window of ~grid consecutive units — a few segments, whose
// Bᵀ rows the neighbouring CTAs read from L2 — as the round-1 tiled grid did
// (dealing contiguous ranges spread the CTAs over every tile at once and
// tripled the gather time).
constexpr uint32_t kPUnitBlocks = 4;
struct Unit {
  uint32_t tile, pj, b0, b1;  // tile, projection, block range [b0, b1)
  __device__ void set(uint32_t ui, uint32_t ngrp, uint32_t nbt, uint32_t n_tiles) {
    const uint32_t tu = ui / ngrp, grp = ui - tu * ngrp;
    pj = tu / n_tiles;
    tile = tu - pj * n_tiles;
    b0 = grp * kPUnitBlocks;
    b1 = min(nbt, b0 + kPUnitBlocks);
  }
};

__global__ void __launch_bounds__(kPThreads, 1)
    sgmv_expand_persistent_kernel(const ExpandArgs p, const __grid_constant__ CUtensorMap tmap_y0,
                                  const __grid_constant__ CUtensorMap tmap_y1,
                                  const __grid_constant__ CUtensorMap tmap_v,
                                  const __grid_constant__ CUtensorMap tmap_arena) {
  extern __shared__ char smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* v_full = reinterpret_cast<uint64_t*>(smem + PSmem::bars);
  uint64_t* v_empty = v_full + kPVStages;
  uint64_t* b_full = v_empty + kPVStages;
  uint64_t* b_empty = b_full + kPStages;
  uint64_t* acc_full = b_empty + kPStages;
  uint64_t* acc_empty = acc_full + kPAcc;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + PSmem::tmem_slot);

  const uint32_t nbt = p.d_out / kEBlockN;  // blocks per tile row
  const uint32_t ngrp = (nbt + kPUnitBlocks - 1) / kPUnitBlocks;
  const uint32_t n_units = p.np * p.n_tiles * ngrp;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (uint32_t i = 0; i < kPVStages; ++i) {
      ptx::mbar_init(&v_full[i], 1);
      ptx::mbar_init(&v_empty[i], 1);
    }
    for (uint32_t i = 0; i < kPStages; ++i) {
      // gather4 mode: one arrival per gather warp (after its lanes' expect_tx);
      // otherwise every gather thread's cp.async completion arrives
      ptx::mbar_init(&b_full[i], p.g4 ? kPGatherWarps : kPGather);
      ptx::mbar_init(&b_empty[i], 1);
    }
    for (uint32_t i = 0; i < kPAcc; ++i) {
      ptx::mbar_init(&acc_full[i], 1);
      ptx::mbar_init(&acc_empty[i], kEEpiThreads / 32);
    }
    ptx::fence_mbar_init();
  }
  if (warp == kPEpi0) ptx::tmem_alloc(tmem_slot, kPAcc * kEBlockN);
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmap_y0);
    ptx::prefetch_tmap(&tmap_y1);
    ptx::prefetch_tmap(&tmap_v);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  Unit un;

  if (p.dbg & 512u) {
  } else if (warp == 0) {
    // ------------------------------------ TMA: the V tile of each unit
    if (lane == 0) {
      ptx::pdl_wait();  // V comes from the shrink (and y may be read by earlier kernels)
      uint32_t vi = 0;
      for (uint32_t ui = blockIdx.x; ui < n_units; ui += gridDim.x, ++vi) {
        un.set(ui, ngrp, nbt, p.n_tiles);
        const uint32_t vs = vi % kPVStages, vph = (vi / kPVStages) & 1u;
        const uint32_t r16 = (p.tiles[un.tile].rank + 15) & ~15u;
        const uint32_t vboxes = r16 > 64 ? 2 : 1;
        ptx::mbar_wait(&v_empty[vs], vph ^ 1u);
        ptx::mbar_arrive_expect_tx(&v_full[vs], vboxes * 16384);
        for (uint32_t bx = 0; bx < vboxes; ++bx)
          ptx::tma_load_2d(smem + PSmem::v + vs * 32768 + bx * 16384, &tmap_v, static_cast<int32_t>(bx * 64),
                           static_cast<int32_t>((un.pj * p.n_tiles + un.tile) * kTileM), &v_full[vs]);
      }
    }
  } else if (warp <= kPGatherWarps) {
    // ----------------------------------- Bᵀ block gathers (paged rows)
    // gather4 mode (pages >= 256 B): lane l of gather warp w issues the
    // gather4 of row group q = l · 8 + w (rows 4q..4q+3, looked up by itself;
    // a warp issues its lanes' TMA ops one after another, so the groups are
    // spread over all eight warps).  Rows r..r16-1 (zero V columns) get
    // copies of row r - 1: finite values, so they add exact zeros.
    // Completion is all transaction bytes plus one arrival per warp.
    // Otherwise thread gt copies row gt by cp.async (zero-filled padding) and
    // every thread's completion arrives.  Page entries are cached per row and
    // logical page (a 2 KiB page holds 16 blocks of a row).
    const uint32_t gt = threadIdx.x - 32, gw = warp - 1;
    const uint32_t q = lane * kPGatherWarps + gw;
    const bool fast = p.log2_page >= 7;  // a row's 128-byte block slice lies in one page
    const uint64_t pmask = (1ull << p.log2_page) - 1;
    uint64_t rowoff[5];  // the rows' offsets at block 0: group q's four, row gt
    uint32_t lp[5], le[5];
    uint32_t k = 0;
    for (uint32_t ui = blockIdx.x; ui < n_units; ui += gridDim.x) {
      un.set(ui, ngrp, nbt, p.n_tiles);
      const SgmvTile t = p.tiles[un.tile];
      const uint32_t r = t.rank, r16 = (r + 15) & ~15u;
      const uint64_t bt = (static_cast<uint64_t>(r) * (un.pj ? p.blk_mult[1] : p.blk_mult[0]) +
                           static_cast<uint64_t>(r) * p.d_in) * 2;
#pragma unroll
      for (uint32_t i = 0; i < 4; ++i) rowoff[i] = bt + static_cast<uint64_t>(min(q * 4 + i, r - 1)) * p.d_out * 2;
      rowoff[4] = bt + static_cast<uint64_t>(gt) * p.d_out * 2;
#pragma unroll
      for (int i = 0; i < 5; ++i) lp[i] = ~0u;
      auto entry = [&](int i, uint64_t off) {
        const uint32_t pg = static_cast<uint32_t>(off >> p.log2_page);
        if (pg != lp[i]) {
          lp[i] = pg;
          le[i] = __ldg(p.table + t.table_off + pg);
        }
        return le[i];
      };
      for (uint32_t b = un.b0; b < un.b1; ++b, ++k) {
        const uint32_t st = k % kPStages, ph = (k / kPStages) & 1u;
        const uint32_t cb = b * kEBlockN * 2;  // the block's byte offset in a row
        int32_t row[4];
        if (p.g4 && q * 4 < r16) {  // (looked up before the stage wait)
#pragma unroll
          for (uint32_t i = 0; i < 4; ++i) {
            const uint64_t off = rowoff[i] + cb;
            row[i] = static_cast<int32_t>(((static_cast<uint64_t>(entry(i, off)) << p.log2_page) + (off & pmask)) >> 7);
          }
        }
        ptx::mbar_wait(&b_empty[st], ph ^ 1u);
        if (gt == 0) ptrace(p, k, 0);
        char* bs = smem + PSmem::b + st * 16384;
        if (p.g4) {
          if (q * 4 < r16 && !(p.dbg & 128u)) {
            ptx::mbar_expect_tx(&b_full[st], 4 * kEBlockN * 2);
            ptx::tma_gather4(bs + q * 4 * kEBlockN * 2, &tmap_arena, 0, row[0], row[1], row[2], row[3], &b_full[st]);
          }
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&b_full[st]);
        } else {
          const uint32_t j = gt;
          if (j < r16 && !(p.dbg & 128u)) {
            const uint64_t off = rowoff[4] + cb;
            const PagedSrc src{p.arena, p.table, t.table_off, p.log2_page};
            const char* base = fast && j < r ? p.arena + (static_cast<uint64_t>(entry(4, off)) << p.log2_page) + (off & pmask)
                                             : p.arena;
#pragma unroll
            for (uint32_t c = 0; c < 8; ++c) {
              char* dst = bs + swz(j, c);
              if (j >= r)
                ptx::cp_async_16(dst, p.arena, 0);
              else if (fast)
                ptx::cp_async_16(dst, base + c * 16, 16);
              else
                ptx::cp_async_16(dst, src.at(off + c * 16), 16);
            }
          }
          ptx::cp_async_mbar_arrive_noinc(&b_full[st]);
        }
        if (gt == 0) ptrace(p, k, 1);
      }
    }
  } else if (warp == kPMma) {
    if (lane == 0) {
      // ------------------------------------------------------- MMA issuer
      const uint32_t idesc = ptx::idesc_bf16_f32(kTileM, kEBlockN, false, true);
      uint32_t k = 0, vi = 0;
      for (uint32_t ui = blockIdx.x; ui < n_units; ui += gridDim.x, ++vi) {
        un.set(ui, ngrp, nbt, p.n_tiles);
        const uint32_t r16 = (p.tiles[un.tile].rank + 15) & ~15u, vs = vi % kPVStages;
        ptx::mbar_wait(&v_full[vs], (vi / kPVStages) & 1u);
        const uint32_t vbase = ptx::smem_u32(smem + PSmem::v + vs * 32768);
        for (uint32_t b = un.b0; b < un.b1; ++b, ++k) {
          const uint32_t st = k % kPStages, ph = (k / kPStages) & 1u;
          const uint32_t as = k % kPAcc, aph = (k / kPAcc) & 1u;
          ptx::mbar_wait(&b_full[st], ph);
          ptrace(p, k, 2);
          ptx::mbar_wait(&acc_empty[as], aph ^ 1u);
          ptrace(p, k, 3);
          ptx::fence_proxy_async_shared();
          ptx::tc_fence_after();
          const uint32_t bbase = ptx::smem_u32(smem + PSmem::b + st * 16384);
          for (uint32_t kk = 0; kk < ((p.dbg & 256u) ? 0u : r16 / 16); ++kk)
            ptx::umma_f16(tmem + as * kEBlockN, ptx::smem_desc_sw128(vbase + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                          ptx::smem_desc_sw128(bbase + kk * 2048, r16 * 128, 1024), idesc, kk != 0);
          ptx::umma_commit(&b_empty[st]);
          ptx::umma_commit(&acc_full[as]);
        }
        ptx::umma_commit(&v_empty[vs]);  // the unit's last block: its V stage is free
      }
    }
  } else {
    // ------------------------------------------------ epilogue (two groups)
    // Every warp stages its own 32 rows and reduce-adds them itself (a 64 × 32
    // box): no barrier across the group, and each warp waits only for its own
    // earlier reduce-add before reusing its staging buffer.
    const uint32_t quad = warp & 3;             // TMEM lane quadrant (each group covers all four)
    const uint32_t m = quad * 32 + lane;        // tile row == TMEM lane
    const uint32_t lane_base = (quad * 32) << 16;
    const uint32_t eg = (warp - kPEpi0) >> 2;   // group: blocks k ≡ eg (mod 2)
    char* ys = smem + PSmem::y + (warp - kPEpi0) * 4096;
    uint32_t k = 0, n = 0;
    for (uint32_t ui = blockIdx.x; ui < n_units; ui += gridDim.x) {
      un.set(ui, ngrp, nbt, p.n_tiles);
      const SgmvTile tile = p.tiles[un.tile];
      const bool live = m < tile.nrows;  // rows past the run belong to the next one: add -0
      const bool any = quad * 32 < tile.nrows;
      for (uint32_t b = un.b0; b < un.b1; ++b, ++k) {
        if ((k & 1u) != eg) continue;
        const uint32_t as = k % kPAcc, aph = (k / kPAcc) & 1u;
        if (n >= 1) {  // this warp's previous reduce-add must have read the buffer
          if (lane == 0) ptx::bulk_wait_read_n<0>();
          __syncwarp();
        }
        ++n;
        if (lane == 0 && quad == 0) ptrace(p, k, 7);
        ptx::mbar_wait(&acc_full[as], aph);
        if (lane == 0 && quad == 0) ptrace(p, k, 4);
        ptx::tc_fence_after();
        uint32_t rv[kEBlockN / 16][16];
#pragma unroll
        for (uint32_t c = 0; c < kEBlockN / 16; ++c)
          ptx::tmem_ld_32x32b_x16(tmem + lane_base + as * kEBlockN + c * 16, rv[c]);
        ptx::tmem_ld_wait();
        if (lane == 0 && quad == 0) ptrace(p, k, 5);
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&acc_empty[as]);
#pragma unroll
        for (uint32_t c = 0; c < kEBlockN / 16; ++c) {
#pragma unroll
          for (uint32_t hh = 0; hh < 2; ++hh) {
            const uint32_t ya = ptx::smem_u32(ys + swz(lane, c * 2 + hh));
            uint32_t o[4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
              o[i] = live ? pack_bf16x2(p.scale * __uint_as_float(rv[c][hh * 8 + 2 * i]),
                                        p.scale * __uint_as_float(rv[c][hh * 8 + 2 * i + 1]))
                          : 0x80008000u;  // bf16 -0.0: the exact additive identity of the reduce-add
            asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(ya), "r"(o[0]), "r"(o[1]),
                         "r"(o[2]), "r"(o[3]) : "memory");
          }
        }
        ptx::fence_proxy_async_shared();  // generic-proxy smem writes -> TMA
        __syncwarp();
        if (lane == 0) {
          if (quad == 0) ptrace(p, k, 6);
          if (any && !(p.dbg & 64u))  // (a warp whose rows all belong to the next run adds nothing)
            ptx::tma_reduce_add_2d(un.pj ? &tmap_y1 : &tmap_y0, static_cast<int32_t>(b * kEBlockN),
                                   static_cast<int32_t>(tile.row0 + quad * 32), ys);
          ptx::bulk_commit();
        }
      }
    }
    if (lane == 0) ptx::bulk_wait_all();
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == kPEpi0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, kPAcc * kEBlockN);
  }
}

}  // namespace

extern "C" int plora_debug_set_sgmv_flags(uint32_t flags) {
  g_sgmv_dbg = flags;
  return PLORA_OK;
}

namespace plora {

// Shrink + split reduction of `np` projections (<= 2) that share x: V tiles
// (bf16, scaled by v_scale) in plan->d_vbuf, projection j's at tile offset
// j · n_tiles.  np = 2 reads each x chunk once for both (plan->ssched_layer).
void sgmv_shrink_reduce_n(plora_plan* plan, uint32_t layer, const uint32_t* projs, uint32_t np,
                          const void* x, uint64_t x_stride, float v_scale, cudaStream_t s) {
  const plora_store& st = *plan->store;
  const ModelGeom& g = st.geom;
  const uint32_t din = g.m.d_in[projs[0]];
  const SgmvSched& sc = np == 1 ? plan->ssched[projs[0]] : plan->ssched_layer;
  CUtensorMap tmap_x, tmap_arena;
  make_tmap_2d(&tmap_x, x, din, plan->n_tokens, x_stride * 2, kChunkK, kTileM);
  // the arena as rows of 128 bytes (64 bf16): TMA gather4 of A row segments
  const uint64_t arena_rows = (static_cast<uint64_t>(st.pool->pool.total_pages()) << st.log2_page) >> 7;
  const bool g4 = st.log2_page >= 8 && arena_rows < (1ull << 31);
  make_tmap_2d(&tmap_arena, st.arena, kChunkK, g4 ? arena_rows : 1, kChunkK * 2, kChunkK, 1);
  set_smem_once(reinterpret_cast<const void*>(sgmv_shrink_kernel), static_cast<int>(SSmem::alloc));
  cudaLaunchAttribute pdl[1];
  pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl[0].val.programmaticStreamSerializationAllowed = 1;
  const uint64_t pstride = static_cast<uint64_t>(plan->vpart_parts) * plan->n_tiles * kTileM * kMaxRank;
  ShrinkArgs sa{};
  sa.arena = st.arena;
  sa.table = st.d_table;
  sa.items = plan->d_sitems + sc.item_off;
  sa.cta_items = plan->d_scta + sc.cta_off;
  sa.vpart = plan->d_vpart;
  sa.vpart_pstride = pstride;
  for (uint32_t j = 0; j < 2; ++j) sa.blk_mult[j] = g.blk_mult(layer, projs[j < np ? j : 0]);
  sa.np = np;
  sa.log2_page = st.log2_page;
  sa.d_in = din;
  sa.splits = sc.splits;
  sa.dbg = g_sgmv_dbg;
  sa.g4 = g4 ? 1u : 0u;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(sc.ctas);
  cfg.blockDim = dim3(kSThreads);
  cfg.dynamicSmemBytes = SSmem::alloc;
  cfg.stream = s;
  cfg.attrs = pdl;
  cfg.numAttrs = 1;
  PLORA_CUDA(cudaLaunchKernelEx(&cfg, sgmv_shrink_kernel, sa, tmap_x, tmap_arena));
  count_launch();
  if (!(g_sgmv_dbg & 32u)) {
    ReduceArgs ra{plan->d_tiles, plan->d_vpart, reinterpret_cast<__nv_bfloat16*>(plan->d_vbuf),
                  pstride, plan->n_tiles, sc.splits, v_scale};
    cfg.gridDim = dim3(np * plan->n_tiles * 4);
    cfg.blockDim = dim3(kRThreads);
    cfg.dynamicSmemBytes = 0;
    PLORA_CUDA(cudaLaunchKernelEx(&cfg, sgmv_reduce_kernel, ra));
    count_launch();
  }
}

void sgmv_shrink_reduce(plora_plan* plan, uint32_t layer, uint32_t proj, const void* x,
                        uint64_t x_stride, float v_scale, cudaStream_t s) {
  sgmv_shrink_reduce_n(plan, layer, &proj, 1, x, x_stride, v_scale, s);
}

// The tensor-core SGMV of `np` projections sharing x (equal d_in, d_out):
// one shrink + reduction, one expand launch over (proj, tile, group) CTAs.
static void sgmv_run(plora_plan* plan, uint32_t layer, const uint32_t* projs, uint32_t np, const void* x,
              uint64_t x_stride, void* const* ys, const uint64_t* y_strides, float scale,
              cudaStream_t s) {
  const plora_store& st = *plan->store;
  const ModelGeom& g = st.geom;
  const uint32_t din = g.m.d_in[projs[0]], dout = g.m.d_out[projs[0]];
  sgmv_shrink_reduce_n(plan, layer, projs, np, x, x_stride, 1.0f, s);
  if (g_sgmv_dbg & 8u) return;
  CUtensorMap tmap_y[2], tmap_v;
  for (uint32_t j = 0; j < 2; ++j) {
    const uint32_t jj = j < np ? j : 0;
    make_tmap_2d(&tmap_y[j], ys[jj], dout, plan->n_tokens, y_strides[jj] * 2, 64, kTileM);
  }
  make_tmap_2d(&tmap_v, plan->d_vbuf, kMaxRank, static_cast<uint64_t>(np) * plan->n_tiles * kTileM,
               kMaxRank * 2, 64, kTileM);
  set_smem_once(reinterpret_cast<const void*>(sgmv_expand_kernel), static_cast<int>(ESmem::alloc));
  cudaLaunchAttribute pdl[1];
  pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl[0].val.programmaticStreamSerializationAllowed = 1;
  ExpandArgs ea{};
  ea.arena = st.arena;
  ea.table = st.d_table;
  ea.tiles = plan->d_tiles;
  for (uint32_t j = 0; j < 2; ++j) ea.blk_mult[j] = g.blk_mult(layer, projs[j < np ? j : 0]);
  ea.log2_page = st.log2_page;
  ea.d_in = din;
  ea.d_out = dout;
  ea.n_tiles = plan->n_tiles;
  ea.ngroups = (dout / kEBlockN + kGroupBlocks - 1) / kGroupBlocks;
  ea.np = np;
  ea.scale = scale;
  ea.dbg = g_sgmv_dbg;
  CUtensorMap tmap_arena;
  const uint64_t arena_rows = (static_cast<uint64_t>(st.pool->pool.total_pages()) << st.log2_page) >> 7;
  const bool g4 = st.log2_page >= 8 && arena_rows < (1ull << 31);
  make_tmap_2d(&tmap_arena, st.arena, kEBlockN, g4 ? arena_rows : 1, kEBlockN * 2, kEBlockN, 1);
  ea.g4 = g4 ? 1u : 0u;
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(kEThreads);
  cfg.stream = s;
  cfg.attrs = pdl;
  cfg.numAttrs = 1;
  if (!(g_sgmv_dbg & kDbgPersistentExpand)) {  // the default: one CTA per (proj, tile, 512 columns)
    cfg.gridDim = dim3(np * plan->n_tiles * ea.ngroups);
    cfg.dynamicSmemBytes = ESmem::alloc;
    PLORA_CUDA(cudaLaunchKernelEx(&cfg, sgmv_expand_kernel, ea, tmap_y[0], tmap_y[1], tmap_v, tmap_arena));
  } else {
    for (uint32_t j = 0; j < 2; ++j) {  // 64 × 32 boxes: every epilogue warp reduce-adds its own rows
      const uint32_t jj = j < np ? j : 0;
      make_tmap_2d(&tmap_y[j], ys[jj], dout, plan->n_tokens, y_strides[jj] * 2, 64, 32);
    }
    set_smem_once(reinterpret_cast<const void*>(sgmv_expand_persistent_kernel), static_cast<int>(PSmem::alloc));
    cfg.blockDim = dim3(kPThreads);
    const uint64_t units = static_cast<uint64_t>(np) * plan->n_tiles *
                           ((dout / kEBlockN + kPUnitBlocks - 1) / kPUnitBlocks);
    cfg.gridDim = dim3(static_cast<uint32_t>(std::min<uint64_t>(std::max(1, st.num_sms), units)));
    cfg.dynamicSmemBytes = PSmem::alloc;
    ea.trace = trace_buffer(static_cast<uint64_t>(cfg.gridDim.x) * kPTrace * 64);
    PLORA_CUDA(cudaLaunchKernelEx(&cfg, sgmv_expand_persistent_kernel, ea, tmap_y[0], tmap_y[1], tmap_v,
                                  tmap_arena));
  }
  count_launch();
}

static bool tc_path(const plora_plan* plan, uint32_t proj) {
  const ModelGeom& g = plan->store->geom;
  // bf16, rank <= 128, d_in % 64 == 0, d_out % 128 == 0; anything else (fp32
  // storage, wider ranks, odd widths) runs the exact CUDA-core BGMV path,
  // which handles every segment length.
  // The gathered rows are addressed as 128-byte arena rows (gather4 indices,
  // 16-byte cp.async groups of 128 B): every (layer, proj) block of every
  // rank must start on a 128-byte boundary, i.e. rank · blk_mult · 2 ≡ 0 mod
  // 128 for rank 1 — blk_mult ≡ 0 (mod 64) for every layer.
  return g.esize == 2 && plan->max_rank <= kMaxRank && g.m.d_in[proj] % kChunkK == 0 &&
         g.m.d_out[proj] % kBlockN == 0 && g.blocks_aligned_128(proj);
}

}  // namespace plora

extern "C" int plora_sgmv(plora_plan* plan, uint32_t layer, uint32_t proj, const void* x,
                          uint64_t x_stride, void* y, uint64_t y_stride, float scale,
                          plora_stream_t stream) {
  return guard([&] {
    if (!plan) throw ValidationError("null plan");
    check_io(plan, layer, proj, x, x_stride, y, y_stride);
    if (!tc_path(plan, proj))
      return plora_bgmv(plan, layer, proj, x, x_stride, y, y_stride, scale, stream);
    if (plan->n_tiles == 0) return 0;
    DeviceCtx ctx(plan->store->device);
    void* ys[1] = {y};
    const uint64_t ystr[1] = {y_stride};
    sgmv_run(plan, layer, &proj, 1, x, x_stride, ys, ystr, scale, static_cast<cudaStream_t>(stream));
    return 0;
  });
}

extern "C" int plora_sgmv_layer(plora_plan* plan, uint32_t layer, const void* x, uint64_t x_stride,
                                void* const* ys, const uint64_t* y_strides, float scale,
                                plora_stream_t stream) {
  return guard([&] {
    if (!plan) throw ValidationError("null plan");
    if (!ys || !y_strides) throw ValidationError("null ys / y_strides");
    const ModelGeom& g = plan->store->geom;
    const uint32_t np = g.m.n_proj;
    for (uint32_t j = 0; j < np; ++j) check_io(plan, layer, j, x, x_stride, ys[j], y_strides[j]);
    bool joint = np == 2 && plan->ssched_layer.splits != 0;
    for (uint32_t j = 0; j < np; ++j)
      joint = joint && tc_path(plan, j) && g.m.d_in[j] == g.m.d_in[0] && g.m.d_out[j] == g.m.d_out[0];
    if (!joint) {  // one call per projection
      for (uint32_t j = 0; j < np; ++j) {
        const int rc = plora_sgmv(plan, layer, j, x, x_stride, ys[j], y_strides[j], scale, stream);
        if (rc != 0) return rc;
      }
      return 0;
    }
    if (plan->n_tiles == 0) return 0;
    DeviceCtx ctx(plan->store->device);
    const uint32_t projs[2] = {0, 1};
    sgmv_run(plan, layer, projs, 2, x, x_stride, ys, y_strides, scale, static_cast<cudaStream_t>(stream));
    return 0;
  });
}
