// Base projection GEMM with the paged LoRA fused in (prefill, §8(f) row 3):
//
//   y[t, :] = x[t, :] · W0ᵀ + bf16(scale · x[t, :] · A_{a(t)}ᵀ) · B_{a(t)}ᵀ
//
// for every token t (tokens without an adapter get the base product only).
// The standalone SGMV is HBM-bound (AI ≈ 41 flop/B); inside the base GEMM
// the LoRA expand is r16 more K-steps of the same accumulator and the whole
// op is tensor-bound.  The shrink (x·Aᵀ, split-K over pages) and its split
// reduction run first (sgmv.cu, V pre-scaled); this kernel then computes
//
//   D[128 × 256] = X[128, d_in] · W0[256, d_in]ᵀ  +  V[128, r16] · Bᵀ[r16, 256]
//
// per (run tile, 256-column block) item.  Persistent, one CTA per SM, items
// taken round-robin in tile-major order (the ~150 items in flight share ~9 x
// tiles and all of W0 through L2).
//   warp 0      TMA: x [128 × 64] and W0 [256 × 64] chunks (SW128, K-major)
//               into a 4-stage ring; for the LoRA K-steps the V chunk.
//   warps 1-4   Bᵀ gathers for the LoRA K-steps: rank rows × 256 columns from
//               the adapter's pages (MN-major SW128, four 64-column groups).
//   warp 5      tcgen05.mma issuer: M=128 N=256 K=16 for the base, four
//               M=128 N=64 MMAs per LoRA K-step, into one of two TMEM
//               accumulators (2 × 256 columns).
//   warps 8-11  epilogue: TMEM -> bf16 -> swizzled smem -> TMA store per
//               64-column slab (rows of a partial tile are stored per row:
//               the rows past it belong to the next run's tile).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include "plan.hpp"
#include "ptx.cuh"
#include "tmap.cuh"

using namespace plora;

namespace plora {
void check_io(const plora_plan* plan, uint32_t layer, uint32_t proj, const void* x,
              uint64_t x_stride, void* y, uint64_t y_stride);
void sgmv_shrink_reduce(plora_plan* plan, uint32_t layer, uint32_t proj, const void* x,
                        uint64_t x_stride, float v_scale, cudaStream_t s);
void sgmv_shrink_reduce_n(plora_plan* plan, uint32_t layer, const uint32_t* projs, uint32_t np,
                          const void* x, uint64_t x_stride, float v_scale, cudaStream_t s);
}  // namespace plora

namespace {
using namespace plora::tmap;

constexpr uint32_t kBM = 128, kBN = 256, kBK = 64;
constexpr int kFStages = 4;
constexpr uint32_t kXBytes = kBM * kBK * 2;           // 16 KiB
constexpr uint32_t kWBytes = kBN * kBK * 2;           // 32 KiB
constexpr uint32_t kFStageBytes = kXBytes + kWBytes;  // 48 KiB
constexpr uint32_t kSlabBytes = kBM * 64 * 2;         // 16 KiB: 64 output columns
constexpr uint32_t kFThreads = 384;
constexpr uint32_t kFGather = 128;  // warps 1-4
constexpr uint32_t kFTmemCols = 512;
constexpr uint32_t kMaxRank = 128;

struct FArgs {
  const char* arena;
  const uint32_t* table;
  const GemmTile* tiles;
  char* y;
  uint64_t y_stride_b;
  uint64_t bt_mult;  // Bᵀ block of a rank-r adapter starts at element r · bt_mult
  uint32_t log2_page;
  uint32_t d_in, d_out;
  uint32_t n_items, nb;  // items = tiles × nb column blocks, tile-major
  uint32_t g4;           // Bᵀ rows by TMA gather4 over the arena viewed as 128-byte rows
};

struct FSmem {
  static constexpr uint32_t stages = 0;  // 1024-aligned
  static constexpr uint32_t slab = stages + kFStages * kFStageBytes;
  static constexpr uint32_t bars = slab + 2 * kSlabBytes;
  // full[4], empty[4], bfull[4], tfull[2], tempty[2]
  static constexpr uint32_t n_bars = 3 * kFStages + 4;
  static constexpr uint32_t tmem_slot = bars + n_bars * 8;
  static constexpr uint32_t total = tmem_slot + 8;
  static constexpr uint32_t alloc = total + 1024;
};

__device__ __forceinline__ uint32_t lora_chunks(uint32_t rank) {
  return rank ? (((rank + 15) & ~15u) + kBK - 1) / kBK : 0u;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

__global__ void __launch_bounds__(kFThreads, 1)
    sgmv_fused_kernel(const FArgs p, const __grid_constant__ CUtensorMap tmap_x,
                      const __grid_constant__ CUtensorMap tmap_w,
                      const __grid_constant__ CUtensorMap tmap_v,
                      const __grid_constant__ CUtensorMap tmap_y,
                      const __grid_constant__ CUtensorMap tmap_arena) {
  extern __shared__ char smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + FSmem::bars);
  uint64_t* empty = full + kFStages;
  uint64_t* bfull = full + 2 * kFStages;
  uint64_t* tfull = full + 3 * kFStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + FSmem::tmem_slot);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t NKb = p.d_in / kBK;

  ptx::pdl_launch_dependents();
  if (threadIdx.x == 0) {
    for (int s = 0; s < kFStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
      ptx::mbar_init(&bfull[s], kFGather);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], 4);  // one arrival per epilogue warp
    }
    ptx::fence_mbar_init();
  }
  if (warp == 5) ptx::tmem_alloc(tmem_slot, kFTmemCols);
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmap_x);
    ptx::prefetch_tmap(&tmap_w);
    ptx::prefetch_tmap(&tmap_v);
    ptx::prefetch_tmap(&tmap_y);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    if (lane == 0) {
      ptx::pdl_wait();  // x and V come from earlier kernels in the stream
      uint32_t g = 0;
      for (uint32_t item = blockIdx.x; item < p.n_items; item += gridDim.x) {
        const GemmTile t = p.tiles[item / p.nb];
        const int32_t n0 = static_cast<int32_t>((item % p.nb) * kBN);
        const uint32_t nk = NKb + lora_chunks(t.rank);
        for (uint32_t kc = 0; kc < nk; ++kc, ++g) {
          const uint32_t st = g % kFStages, ph = (g / kFStages) & 1u;
          ptx::mbar_wait(&empty[st], ph ^ 1u);
          char* sx = smem + FSmem::stages + st * kFStageBytes;
          if (kc < NKb) {
            ptx::mbar_arrive_expect_tx(&full[st], kFStageBytes);
            ptx::tma_load_2d(sx, &tmap_x, static_cast<int32_t>(kc * kBK), static_cast<int32_t>(t.row0),
                             &full[st]);
            ptx::tma_load_2d(sx + kXBytes, &tmap_w, static_cast<int32_t>(kc * kBK), n0, &full[st]);
          } else {
            ptx::mbar_arrive_expect_tx(&full[st], kXBytes);
            ptx::tma_load_2d(sx, &tmap_v, static_cast<int32_t>((kc - NKb) * kBK),
                             static_cast<int32_t>(t.vtile * kBM), &full[st]);
          }
        }
      }
    }
  } else if (warp <= 4) {
    // ------------------------------------------- Bᵀ gathers (LoRA K-steps)
    // A LoRA chunk is 64 rank rows × 256 columns: piece (row, group) = one
    // 128-byte row segment of a 64-column group, two pieces per thread; four
    // consecutive lanes hold four consecutive rows of one group, so with
    // pages >= 512 B a group of real rows goes by one TMA gather4.
    // The threads wait for every chunk's slot, base chunks included: a parity
    // wait must never run two ring laps ahead of the barrier.  Base chunks
    // arrive nowhere.
    const uint32_t tid = threadIdx.x - 32;
    const bool fast = p.log2_page >= 9;  // a row's 512-byte block slice lies in one page
    uint32_t g = 0;
    for (uint32_t item = blockIdx.x; item < p.n_items; item += gridDim.x) {
      const GemmTile t = p.tiles[item / p.nb];
      const uint32_t n0 = (item % p.nb) * kBN;
      const uint32_t nl = lora_chunks(t.rank), r = t.rank, r16 = (r + 15) & ~15u;
      const uint64_t bt = static_cast<uint64_t>(r) * p.bt_mult * 2;
      const PagedSrc src{p.arena, p.table, t.table_off, p.log2_page};
      for (uint32_t c = 0; c < NKb; ++c, ++g) ptx::mbar_wait(&empty[g % kFStages], ((g / kFStages) & 1u) ^ 1u);
      for (uint32_t l = 0; l < nl; ++l, ++g) {
        const uint32_t st = g % kFStages, ph = (g / kFStages) & 1u;
        uint32_t phys[2];
        uint64_t off[2];
#pragma unroll
        for (uint32_t h = 0; h < 2; ++h) {  // page lookups before the slot wait
          const uint32_t pc = tid + h * kFGather, krow = (pc & 3) + 4 * (pc >> 4), grp = (pc >> 2) & 3;
          const uint32_t j = l * kBK + krow;
          off[h] = bt + (static_cast<uint64_t>(j) * p.d_out + n0 + grp * 64) * 2;
          phys[h] = (fast && j < r) ? __ldg(p.table + t.table_off + static_cast<uint32_t>(off[h] >> p.log2_page)) : 0u;
        }
        ptx::mbar_wait(&empty[st], ph ^ 1u);
        char* bs = smem + FSmem::stages + st * kFStageBytes + kXBytes;
        bool g4[2];
#pragma unroll
        for (uint32_t h = 0; h < 2; ++h) {
          const uint32_t pc = tid + h * kFGather, krow = (pc & 3) + 4 * (pc >> 4), grp = (pc >> 2) & 3;
          const uint32_t j = l * kBK + krow;
          g4[h] = p.g4 && fast && (j | 3u) < r;
          if (p.g4 && fast) {
            const int32_t row = static_cast<int32_t>(
                ((static_cast<uint64_t>(phys[h]) << p.log2_page) + (off[h] & ((1ull << p.log2_page) - 1))) >> 7);
            const uint32_t l0 = lane & ~3u;
            const int32_t r0 = __shfl_sync(0xffffffffu, row, l0), r1 = __shfl_sync(0xffffffffu, row, l0 + 1);
            const int32_t r2 = __shfl_sync(0xffffffffu, row, l0 + 2), r3 = __shfl_sync(0xffffffffu, row, l0 + 3);
            if (g4[h] && (lane & 3u) == 0) {
              ptx::mbar_expect_tx(&bfull[st], 4 * 128);
              ptx::tma_gather4(bs + grp * 8192 + krow * 128, &tmap_arena, 0, r0, r1, r2, r3, &bfull[st]);
            }
          }
        }
#pragma unroll
        for (uint32_t h = 0; h < 2; ++h) {
          const uint32_t pc = tid + h * kFGather, krow = (pc & 3) + 4 * (pc >> 4), grp = (pc >> 2) & 3;
          const uint32_t j = l * kBK + krow;
          if (j >= r16 || g4[h]) continue;  // the MMA stops at r16
          char* dst = bs + grp * 8192;
          const char* base = p.arena + (static_cast<uint64_t>(phys[h]) << p.log2_page) +
                             (off[h] & ((1ull << p.log2_page) - 1));
#pragma unroll
          for (uint32_t q = 0; q < 8; ++q) {
            if (j >= r)
              ptx::cp_async_16(dst + swz(krow, q), p.arena, 0);  // rank padding: zeros
            else if (fast)
              ptx::cp_async_16(dst + swz(krow, q), base + q * 16, 16);
            else
              ptx::cp_async_16(dst + swz(krow, q), src.at(off[h] + q * 16), 16);
          }
        }
        ptx::cp_async_mbar_arrive_noinc(&bfull[st]);
      }
    }
  } else if (warp == 5) {
    // ------------------------------------------------------- MMA issuer
    if (lane == 0) {
      const uint32_t id_base = ptx::idesc_bf16_f32(kBM, kBN, false, false);
      const uint32_t id_lora = ptx::idesc_bf16_f32(kBM, 64, false, true);
      const uint32_t sbase = ptx::smem_u32(smem + FSmem::stages);
      uint32_t g = 0, bph = 0;  // bph: bfull parity per slot (bit st)
      for (uint32_t item = blockIdx.x, i = 0; item < p.n_items; item += gridDim.x, ++i) {
        const GemmTile t = p.tiles[item / p.nb];
        const uint32_t nk = NKb + lora_chunks(t.rank), r16 = (t.rank + 15) & ~15u;
        const uint32_t buf = i & 1u, tb = tmem + buf * kBN;
        ptx::mbar_wait(&tempty[buf], ((i >> 1) & 1u) ^ 1u);
        ptx::tc_fence_after();
        for (uint32_t kc = 0; kc < nk; ++kc, ++g) {
          const uint32_t st = g % kFStages, ph = (g / kFStages) & 1u;
          ptx::mbar_wait(&full[st], ph);
          const uint32_t xa = sbase + st * kFStageBytes, wa = xa + kXBytes;
          if (kc < NKb) {
            ptx::tc_fence_after();
#pragma unroll
            for (uint32_t k = 0; k < kBK / 16; ++k)
              ptx::umma_f16(tb, ptx::smem_desc_sw128(xa + k * 32, 16, 1024),
                            ptx::smem_desc_sw128(wa + k * 32, 16, 1024), id_base, (kc | k) != 0);
          } else {
            ptx::mbar_wait(&bfull[st], (bph >> st) & 1u);
            bph ^= 1u << st;
            ptx::fence_proxy_async_shared();  // cp.async (generic proxy) -> tensor core
            ptx::tc_fence_after();
            const uint32_t ksteps = min(kBK, r16 - (kc - NKb) * kBK) / 16;
            for (uint32_t kk = 0; kk < ksteps; ++kk)
#pragma unroll
              for (uint32_t grp = 0; grp < 4; ++grp)
                ptx::umma_f16(tb + grp * 64, ptx::smem_desc_sw128(xa + kk * 32, 16, 1024),
                              ptx::smem_desc_sw128(wa + grp * 8192 + kk * 2048, kMaxRank * 128, 1024),
                              id_lora, 1u);
          }
          ptx::umma_commit(&empty[st]);
        }
        ptx::umma_commit(&tfull[buf]);
      }
    }
    __syncwarp();
  } else if (warp >= 8) {
    // ------------------------------------------------------------ epilogue
    const uint32_t q4 = warp & 3, m = q4 * 32 + lane;
    const uint32_t lane_base = (q4 * 32) << 16;
    const bool leader = warp == 8 && lane == 0;
    uint32_t slabs = 0;  // TMA stores issued (staging buffer = slabs & 1)
    for (uint32_t item = blockIdx.x, i = 0; item < p.n_items; item += gridDim.x, ++i) {
      const GemmTile t = p.tiles[item / p.nb];
      const uint32_t n0 = (item % p.nb) * kBN;
      const uint32_t buf = i & 1u, tb = tmem + buf * kBN;
      const bool full_tile = t.nrows == kBM;
      ptx::mbar_wait(&tfull[buf], (i >> 1) & 1u);
      ptx::tc_fence_after();
      for (uint32_t sl = 0; sl < kBN / 64; ++sl) {
        uint32_t rv[4][16];
#pragma unroll
        for (uint32_t c = 0; c < 4; ++c) ptx::tmem_ld_32x32b_x16(tb + lane_base + sl * 64 + c * 16, rv[c]);
        ptx::tmem_ld_wait();
        if (full_tile) {
          char* ob = smem + FSmem::slab + (slabs & 1u) * kSlabBytes;
          if (slabs >= 2) {  // the store issued from this buffer two slabs ago has read it
            if (leader) ptx::bulk_wait_read_n<1>();
            ptx::named_bar_sync(1, 128);
          }
#pragma unroll
          for (uint32_t c = 0; c < 4; ++c)
#pragma unroll
            for (uint32_t hh = 0; hh < 2; ++hh) {
              uint32_t o[4];
#pragma unroll
              for (int e = 0; e < 4; ++e)
                o[e] = pack_bf16x2(__uint_as_float(rv[c][hh * 8 + 2 * e]),
                                   __uint_as_float(rv[c][hh * 8 + 2 * e + 1]));
              asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(ptx::smem_u32(ob + swz(m, c * 2 + hh))),
                           "r"(o[0]), "r"(o[1]), "r"(o[2]), "r"(o[3]) : "memory");
            }
          ptx::fence_proxy_async_shared();
          ptx::named_bar_sync(1, 128);
          if (leader) {
            ptx::tma_store_2d(&tmap_y, static_cast<int32_t>(n0 + sl * 64), static_cast<int32_t>(t.row0), ob);
            ptx::bulk_commit();
          }
          ++slabs;
        } else if (m < t.nrows) {  // partial tile: this row only
          uint4* dst = reinterpret_cast<uint4*>(p.y + static_cast<uint64_t>(t.row0 + m) * p.y_stride_b +
                                                static_cast<uint64_t>(n0 + sl * 64) * 2);
#pragma unroll
          for (uint32_t c = 0; c < 4; ++c)
#pragma unroll
            for (uint32_t hh = 0; hh < 2; ++hh) {
              uint32_t o[4];
#pragma unroll
              for (int e = 0; e < 4; ++e)
                o[e] = pack_bf16x2(__uint_as_float(rv[c][hh * 8 + 2 * e]),
                                   __uint_as_float(rv[c][hh * 8 + 2 * e + 1]));
              dst[c * 2 + hh] = make_uint4(o[0], o[1], o[2], o[3]);
            }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty[buf]);  // accumulator free for item i + 2
    }
    if (leader) ptx::bulk_wait_all();
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, kFTmemCols);
  }
}

}  // namespace

namespace {

void check_fused(const plora_plan* plan, uint32_t proj, const void* w0, uint64_t w0_stride) {
  const ModelGeom& g = plan->store->geom;
  const uint32_t din = g.m.d_in[proj], dout = g.m.d_out[proj];
  if (!w0) throw ValidationError("null base weight");
  if (g.esize != 2) throw ValidationError("plora_sgmv_fused needs a bf16 store");
  if (plan->max_rank > kMaxRank) throw ValidationError("plora_sgmv_fused: rank > 128");
  if (din % kBK || dout % kBN)
    throw ValidationError("plora_sgmv_fused needs d_in % 64 == 0 and d_out % 256 == 0");
  if (w0_stride < din) throw ValidationError("base weight row stride < d_in");
  if (!g.blocks_aligned_128(proj))
    throw ValidationError("plora_sgmv_fused needs every (layer, proj) block on a 128-byte boundary "
                          "(sum of the projection widths and their prefixes multiples of 64)");
}

// The fused GEMM of one projection; its V tiles start at tile row v_tile0 of
// the V buffer (projection j of a joint shrink: j · n_tiles).
void launch_fused(plora_plan* plan, uint32_t layer, uint32_t proj, const void* x, uint64_t x_stride,
                  const void* w0, uint64_t w0_stride, void* y, uint64_t y_stride, uint64_t v_tile0,
                  cudaStream_t s) {
  const plora_store& st = *plan->store;
  const ModelGeom& g = st.geom;
  const uint32_t din = g.m.d_in[proj], dout = g.m.d_out[proj];
  CUtensorMap tmap_x, tmap_w, tmap_v, tmap_y;
  make_tmap_2d(&tmap_x, x, din, plan->n_tokens, x_stride * 2, kBK, kBM);
  make_tmap_2d(&tmap_w, w0, din, dout, w0_stride * 2, kBK, kBN);
  const char* vbase = plan->n_tiles ? plan->d_vbuf + v_tile0 * kBM * kMaxRank * 2 : static_cast<const char*>(x);
  make_tmap_2d(&tmap_v, vbase, kMaxRank, std::max<uint64_t>(plan->n_tiles, 1) * kBM, kMaxRank * 2, kBK, kBM);
  make_tmap_2d(&tmap_y, y, dout, plan->n_tokens, y_stride * 2, 64, kBM);
  set_smem_once(reinterpret_cast<const void*>(sgmv_fused_kernel), static_cast<int>(FSmem::alloc));
  FArgs a{};
  a.arena = st.arena;
  a.table = st.d_table;
  a.tiles = plan->d_gtiles;
  a.y = static_cast<char*>(y);
  a.y_stride_b = y_stride * 2;
  a.bt_mult = g.blk_mult(layer, proj) + din;  // Bᵀ follows A (r · d_in elements)
  a.log2_page = st.log2_page;
  a.d_in = din;
  a.d_out = dout;
  a.nb = dout / kBN;
  a.n_items = static_cast<uint32_t>(plan->gtiles.size()) * a.nb;
  CUtensorMap tmap_arena;
  const uint64_t arena_rows = (static_cast<uint64_t>(st.pool->pool.total_pages()) << st.log2_page) >> 7;
  const bool g4 = st.log2_page >= 9 && arena_rows < (1ull << 31);
  make_tmap_2d(&tmap_arena, st.arena, 64, g4 ? arena_rows : 1, 128, 64, 1);
  a.g4 = g4 ? 1u : 0u;
  cudaLaunchAttribute pdl[1];
  pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(std::min<uint32_t>(static_cast<uint32_t>(st.num_sms), a.n_items));
  cfg.blockDim = dim3(kFThreads);
  cfg.dynamicSmemBytes = FSmem::alloc;
  cfg.stream = s;
  cfg.attrs = pdl;
  cfg.numAttrs = 1;
  PLORA_CUDA(cudaLaunchKernelEx(&cfg, sgmv_fused_kernel, a, tmap_x, tmap_w, tmap_v, tmap_y, tmap_arena));
  count_launch();
}

}  // namespace

extern "C" int plora_sgmv_fused(plora_plan* plan, uint32_t layer, uint32_t proj, const void* x,
                                uint64_t x_stride, const void* w0, uint64_t w0_stride, void* y,
                                uint64_t y_stride, float scale, plora_stream_t stream) {
  return guard([&] {
    if (!plan) throw ValidationError("null plan");
    check_io(plan, layer, proj, x, x_stride, y, y_stride);
    check_fused(plan, proj, w0, w0_stride);
    if (plan->gtiles.empty()) return 0;
    DeviceCtx ctx(plan->store->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (plan->n_tiles) sgmv_shrink_reduce(plan, layer, proj, x, x_stride, scale, s);
    launch_fused(plan, layer, proj, x, x_stride, w0, w0_stride, y, y_stride, 0, s);
    return 0;
  });
}

extern "C" int plora_sgmv_fused_layer(plora_plan* plan, uint32_t layer, const void* x,
                                      uint64_t x_stride, const void* const* w0s,
                                      const uint64_t* w0_strides, void* const* ys,
                                      const uint64_t* y_strides, float scale, plora_stream_t stream) {
  return guard([&] {
    if (!plan) throw ValidationError("null plan");
    if (!w0s || !w0_strides || !ys || !y_strides) throw ValidationError("null weight / output arrays");
    const ModelGeom& g = plan->store->geom;
    const uint32_t np = g.m.n_proj;
    for (uint32_t j = 0; j < np; ++j) {
      check_io(plan, layer, j, x, x_stride, ys[j], y_strides[j]);
      check_fused(plan, j, w0s[j], w0_strides[j]);
    }
    if (plan->gtiles.empty()) return 0;
    DeviceCtx ctx(plan->store->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const bool joint = np == 2 && plan->ssched_layer.splits != 0 && g.m.d_in[1] == g.m.d_in[0];
    if (joint) {  // one shrink reads x once for both projections' V
      const uint32_t projs[2] = {0, 1};
      if (plan->n_tiles) sgmv_shrink_reduce_n(plan, layer, projs, 2, x, x_stride, scale, s);
      for (uint32_t j = 0; j < 2; ++j)
        launch_fused(plan, layer, j, x, x_stride, w0s[j], w0_strides[j], ys[j], y_strides[j],
                     static_cast<uint64_t>(j) * plan->n_tiles, s);
      return 0;
    }
    for (uint32_t j = 0; j < np; ++j) {
      if (plan->n_tiles) sgmv_shrink_reduce(plan, layer, j, x, x_stride, scale, s);
      launch_fused(plan, layer, j, x, x_stride, w0s[j], w0_strides[j], ys[j], y_strides[j], 0, s);
    }
    return 0;
  });
}
