// Paged multi-LoRA prefill op (gathered SGMV) on the 5th-generation tensor
// cores (tcgen05 + TMEM) for sm_100a.
//
// y[t, :] += scale · bf16(x[t, :] · Aᵀ) · Bᵀ for the tokens of each run (a
// stretch of consecutive tokens with one adapter).  The
// reference bills this as cost_model.prefill_ms (cost_model.hpp:32-34,
// src/engine.cpp:355).
//
// One CTA per 128-token tile of a run, 8 warps:
//   warp 5      TMA producer: x tile [128 × 64] per K-chunk (2-D tensor map,
//               128-byte swizzle) into a 4-stage smem ring;
//   warps 6-7   page-gather producers: cp.async 16-byte pieces of the
//               adapter's A rows (shrink) / Bᵀ rows (expand), each piece
//               translated through the device page table, written straight
//               into the UMMA canonical SW128 layouts (K-major for A,
//               MN-major for Bᵀ); ranks are zero-padded to a multiple of 16
//               in shared memory only — no contiguous adapter is built;
//   warp 4      MMA issuer (one thread): shrink V[128 × r16] += X · Aᵀ over
//               d_in/64 chunks into TMEM, then expand D[128 × 128] = V · Bᵀ
//               per 128-column chunk into two TMEM buffers (double-buffered
//               against the epilogue);
//   warps 0-3   epilogue: V (TMEM) -> bf16 -> smem (A operand of the
//               expand); then per chunk D (TMEM) + y -> y, with the y row
//               prefetched before the accumulator is ready.
// Rank up to 128 (TMEM columns: V 128 + 2 × 128 accumulators of 512).
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

constexpr int kThreads = 256;
constexpr int kStages = 4;
constexpr uint32_t kTileM = 128;
constexpr uint32_t kChunkK = 64;    // shrink K per stage (one 128-byte swizzle row)
constexpr uint32_t kChunkN = 128;   // expand N per stage / accumulator
constexpr uint32_t kMaxRank = 128;
constexpr uint32_t kStageBytes = 32768;  // X 16 KiB + A 16 KiB, or Bᵀ r16 × 128 × 2
constexpr uint32_t kVBytes = kTileM * kMaxRank * 2;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kAccCol0 = 128;  // expand accumulators at columns 128 and 256
constexpr int kWeightProducers = 64;

struct SgmvArgs {
  const char* arena;
  const uint32_t* table;
  const SgmvTile* tiles;
  char* y;
  uint64_t y_stride_b;
  uint64_t blk_mult;
  uint32_t log2_page;
  uint32_t d_in;
  uint32_t d_out;
  float scale;
};

struct Smem {
  static constexpr uint32_t stages = 0;  // 1024-aligned
  static constexpr uint32_t v = stages + kStages * kStageBytes;
  static constexpr uint32_t bars = v + kVBytes;
  // full[4], empty[4], v_full, v_ready, acc_full[2], acc_empty[2]
  static constexpr uint32_t n_bars = 2 * kStages + 6;
  static constexpr uint32_t tmem_slot = bars + n_bars * 8;
  static constexpr uint32_t total = tmem_slot + 16;
  static constexpr uint32_t alloc = total + 1024;  // alignment slack
};

__device__ __forceinline__ uint32_t swz(uint32_t row, uint32_t chunk) {
  // 128-byte swizzle inside an 8-row × 128-byte atom
  return (row >> 3) * 1024 + (row & 7) * 128 + ((chunk ^ (row & 7)) << 4);
}

__device__ __forceinline__ const char* paged_src(const SgmvArgs& p, uint32_t table_off,
                                                 uint64_t off) {
  const uint32_t phys = __ldg(p.table + table_off + static_cast<uint32_t>(off >> p.log2_page));
  return p.arena + (static_cast<uint64_t>(phys) << p.log2_page) +
         (off & ((1ull << p.log2_page) - 1));
}

__global__ void __launch_bounds__(kThreads, 1)
    sgmv_tc_kernel(const SgmvArgs p, const __grid_constant__ CUtensorMap tmap_x) {
  extern __shared__ char smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Smem::bars);
  uint64_t* full = bars;
  uint64_t* empty = bars + kStages;
  uint64_t* v_full = bars + 2 * kStages;
  uint64_t* v_ready = v_full + 1;
  uint64_t* acc_full = v_full + 2;
  uint64_t* acc_empty = v_full + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + Smem::tmem_slot);

  const SgmvTile tile = p.tiles[blockIdx.x];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t r = tile.rank, r16 = (r + 15) & ~15u;
  const uint32_t NK = p.d_in / kChunkK, NC = p.d_out / kChunkN;
  const uint64_t blk = static_cast<uint64_t>(r) * p.blk_mult * 2;       // A block, bytes
  const uint64_t bt = blk + static_cast<uint64_t>(r) * p.d_in * 2;       // Bᵀ block, bytes

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], 1 + kWeightProducers);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(v_full, 1);
    ptx::mbar_init(v_ready, kTileM);
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&acc_full[b], 1);
      ptx::mbar_init(&acc_empty[b], kTileM);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 4) ptx::tmem_alloc(tmem_slot, kTmemCols);
  if (warp == 5 && lane == 0) ptx::prefetch_tmap(&tmap_x);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 5) {
    // ------------------------------------------------ TMA producer (x tiles)
    if (lane == 0) {
      uint32_t it = 0;
      for (uint32_t kc = 0; kc < NK; ++kc, ++it) {
        const uint32_t st = it % kStages, ph = (it / kStages) & 1u;
        ptx::mbar_wait(&empty[st], ph ^ 1u);
        ptx::mbar_arrive_expect_tx(&full[st], kTileM * kChunkK * 2);
        ptx::tma_load_2d(smem + Smem::stages + st * kStageBytes, &tmap_x,
                         static_cast<int32_t>(kc * kChunkK), static_cast<int32_t>(tile.row0),
                         &full[st]);
      }
      for (uint32_t nc = 0; nc < NC; ++nc, ++it) {
        const uint32_t st = it % kStages, ph = (it / kStages) & 1u;
        ptx::mbar_wait(&empty[st], ph ^ 1u);
        ptx::mbar_arrive(&full[st]);
      }
    }
  } else if (warp >= 6) {
    // ------------------------------------------- page-gather producers (A, Bᵀ)
    const uint32_t wt = threadIdx.x - 6 * 32;
    uint32_t it = 0;
    for (uint32_t kc = 0; kc < NK; ++kc, ++it) {
      const uint32_t st = it % kStages, ph = (it / kStages) & 1u;
      ptx::mbar_wait(&empty[st], ph ^ 1u);
      char* wdst = smem + Smem::stages + st * kStageBytes + kTileM * kChunkK * 2;
      for (uint32_t q = wt; q < r16 * 8; q += kWeightProducers) {
        const uint32_t n = q >> 3, c = q & 7;
        if (n < r) {
          const uint64_t off = blk + (static_cast<uint64_t>(n) * p.d_in + kc * kChunkK + c * 8) * 2;
          ptx::cp_async_16(wdst + swz(n, c), paged_src(p, tile.table_off, off), 16);
        } else {
          ptx::cp_async_16(wdst + swz(n, c), p.arena, 0);  // zero rank padding
        }
      }
      ptx::cp_async_mbar_arrive_noinc(&full[st]);
    }
    const uint32_t lbo = (r16 / 8) * 1024;  // N-group stride of the MN-major Bᵀ tile
    for (uint32_t nc = 0; nc < NC; ++nc, ++it) {
      const uint32_t st = it % kStages, ph = (it / kStages) & 1u;
      ptx::mbar_wait(&empty[st], ph ^ 1u);
      char* bdst = smem + Smem::stages + st * kStageBytes;
      for (uint32_t q = wt; q < r16 * 16; q += kWeightProducers) {
        const uint32_t j = q >> 4, g = (q >> 3) & 1, c = q & 7;
        char* dst = bdst + g * lbo + swz(j, c);
        if (j < r) {
          const uint64_t off =
              bt + (static_cast<uint64_t>(j) * p.d_out + nc * kChunkN + g * 64 + c * 8) * 2;
          ptx::cp_async_16(dst, paged_src(p, tile.table_off, off), 16);
        } else {
          ptx::cp_async_16(dst, p.arena, 0);
        }
      }
      ptx::cp_async_mbar_arrive_noinc(&full[st]);
    }
  } else if (warp == 4) {
    // --------------------------------------------------------- MMA issuer
    if (lane == 0) {
      const uint32_t idesc_s = ptx::idesc_bf16_f32(kTileM, r16, false, false);
      const uint32_t idesc_e = ptx::idesc_bf16_f32(kTileM, kChunkN, false, true);
      const uint32_t sbase = ptx::smem_u32(smem + Smem::stages);
      const uint32_t vbase = ptx::smem_u32(smem + Smem::v);
      uint32_t it = 0;
      for (uint32_t kc = 0; kc < NK; ++kc, ++it) {
        const uint32_t st = it % kStages, ph = (it / kStages) & 1u;
        ptx::mbar_wait(&full[st], ph);
        ptx::fence_proxy_async_shared();
        ptx::tc_fence_after();
        const uint32_t xa = sbase + st * kStageBytes, wa = xa + kTileM * kChunkK * 2;
#pragma unroll
        for (uint32_t k = 0; k < kChunkK / 16; ++k)
          ptx::umma_f16(tmem, ptx::smem_desc_sw128(xa + k * 32, 16, 1024),
                        ptx::smem_desc_sw128(wa + k * 32, 16, 1024), idesc_s, (kc | k) != 0);
        ptx::umma_commit(&empty[st]);
      }
      ptx::umma_commit(v_full);
      ptx::mbar_wait(v_ready, 0);
      ptx::tc_fence_after();
      const uint32_t lbo = (r16 / 8) * 1024;
      for (uint32_t nc = 0; nc < NC; ++nc, ++it) {
        const uint32_t buf = nc & 1u;
        ptx::mbar_wait(&acc_empty[buf], ((nc >> 1) & 1u) ^ 1u);
        const uint32_t st = it % kStages, ph = (it / kStages) & 1u;
        ptx::mbar_wait(&full[st], ph);
        ptx::fence_proxy_async_shared();
        ptx::tc_fence_after();
        const uint32_t ba = sbase + st * kStageBytes;
        for (uint32_t kk = 0; kk < r16 / 16; ++kk)
          ptx::umma_f16(tmem + kAccCol0 + buf * kChunkN,
                        ptx::smem_desc_sw128(vbase + (kk >> 2) * (kTileM * 128) + (kk & 3) * 32,
                                             16, 1024),
                        ptx::smem_desc_sw128(ba + kk * 2048, lbo, 1024), idesc_e, kk != 0);
        ptx::umma_commit(&empty[st]);
        ptx::umma_commit(&acc_full[buf]);
      }
    }
  } else {
    // ------------------------------------------------- epilogue (warps 0-3)
    const uint32_t m = warp * 32 + lane;  // tile row == TMEM lane
    const uint32_t lane_base = (warp * 32) << 16;
    ptx::mbar_wait(v_full, 0);
    ptx::tc_fence_after();
    char* vs = smem + Smem::v;
    for (uint32_t cc = 0; cc < r16 / 16; ++cc) {
      uint32_t rv[16];
      ptx::tmem_ld_32x32b_x16(tmem + lane_base + cc * 16, rv);
      ptx::tmem_ld_wait();
      uint4 pk[2];
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(pk);
#pragma unroll
      for (int i = 0; i < 8; ++i)
        h[i] = __floats2bfloat162_rn(__uint_as_float(rv[2 * i]), __uint_as_float(rv[2 * i + 1]));
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const uint32_t chunk = cc * 2 + hh;  // 16-byte chunk along K
        *reinterpret_cast<uint4*>(vs + (chunk >> 3) * (kTileM * 128) + swz(m, chunk & 7)) = pk[hh];
      }
    }
    ptx::fence_proxy_async_shared();
    ptx::mbar_arrive(v_ready);

    const bool valid = m < tile.nrows;
    char* yrow = p.y + static_cast<uint64_t>(tile.row0 + m) * p.y_stride_b;
    for (uint32_t nc = 0; nc < NC; ++nc) {
      const uint32_t buf = nc & 1u;
      uint4 yv[16];
      uint4* yp = reinterpret_cast<uint4*>(yrow + static_cast<uint64_t>(nc) * kChunkN * 2);
      if (valid) {
#pragma unroll
        for (int i = 0; i < 16; ++i) yv[i] = yp[i];
      }
      ptx::mbar_wait(&acc_full[buf], (nc >> 1) & 1u);
      ptx::tc_fence_after();
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        uint32_t rv[16];
        ptx::tmem_ld_32x32b_x16(tmem + lane_base + kAccCol0 + buf * kChunkN + q * 16, rv);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          __nv_bfloat162* hy = reinterpret_cast<__nv_bfloat162*>(&yv[q * 2 + hh]);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            float2 f = __bfloat1622float2(hy[i]);
            f.x = fmaf(p.scale, __uint_as_float(rv[hh * 8 + 2 * i]), f.x);
            f.y = fmaf(p.scale, __uint_as_float(rv[hh * 8 + 2 * i + 1]), f.y);
            hy[i] = __floats2bfloat162_rn(f.x, f.y);
          }
        }
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&acc_empty[buf]);
      if (valid) {
#pragma unroll
        for (int i = 0; i < 16; ++i) yp[i] = yv[i];
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, kTmemCols);
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

}  // namespace

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
    if (g.esize != 2 || plan->max_rank > kMaxRank || din % kChunkK || dout % kChunkN)
      return plora_bgmv(plan, layer, proj, x, x_stride, y, y_stride, scale, stream);
    if (plan->n_tiles == 0) return 0;
    DeviceCtx ctx(st.device);
    CUtensorMap tmap;
    const cuuint64_t dims[2] = {din, std::max<uint64_t>(plan->n_tokens, 1)};
    const cuuint64_t strides[1] = {x_stride * 2};
    const cuuint32_t box[2] = {kChunkK, kTileM};
    const cuuint32_t estr[2] = {1, 1};
    CUresult cr = encode_fn()(&tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(x),
                              dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string(cr));
    SgmvArgs a{};
    a.arena = st.arena;
    a.table = st.d_table;
    a.tiles = plan->d_tiles;
    a.y = static_cast<char*>(y);
    a.y_stride_b = y_stride * 2;
    a.blk_mult = g.blk_mult(layer, proj);
    a.log2_page = st.log2_page;
    a.d_in = din;
    a.d_out = dout;
    a.scale = scale;
    static bool attr = false;
    if (!attr) {
      PLORA_CUDA(cudaFuncSetAttribute(sgmv_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(Smem::alloc)));
      attr = true;
    }
    sgmv_tc_kernel<<<plan->n_tiles, kThreads, Smem::alloc, static_cast<cudaStream_t>(stream)>>>(
        a, tmap);
    PLORA_CUDA(cudaGetLastError());
    count_launch();
    return 0;
  });
}
