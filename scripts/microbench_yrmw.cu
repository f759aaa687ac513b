// microbench: the SGMV expand's y read-modify-write alone.  y = 16384 x 4096
// bf16 (128 MiB) updated in 128 x 64 tiles (16 KiB) from shared memory:
//   0  TMA reduce-add (cp.reduce.async.bulk.tensor .add: the add in L2), the
//      product's expand epilogue
//   1  TMA load of the tile, add in registers, TMA store
//   2  TMA store only (no read: a lower bound, wrong result)
// Persistent-ish grid of 296 CTAs (2 per SM) of 128 threads, each walking
// tiles round-robin with a 2-deep staging ring; CUDA events, 20 reps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_y scripts/microbench_yrmw.cu -lcuda
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int M = 16384, N = 4096, TM = 128, TN = 64;
constexpr int TNW = 128;  // wide reduce-add boxes (mode 5)
constexpr int TILES = (M / TM) * (N / TN);

__device__ __forceinline__ uint32_t su(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int MODE>
__global__ void __launch_bounds__(128) yrmw(const __grid_constant__ CUtensorMap tm) {
  extern __shared__ __align__(1024) char smem[];
  __shared__ __align__(8) uint64_t bar[2];
  char* buf = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  const uint32_t tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t k = 0;
  for (uint32_t t = blockIdx.x; t < TILES; t += gridDim.x, ++k) {
    const uint32_t st = k & 1, ph = (k >> 1) & 1;
    char* b = buf + st * 16384;
    const int c0 = (t % (N / TN)) * TN, r0 = (t / (N / TN)) * TM;
    if (k >= 2) {  // this stage's previous store / reduce has read the buffer
      if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      __syncthreads();
    }
    if (MODE == 1) {
      if (tid == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[st])), "r"(16384) : "memory");
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(su(b)), "l"(&tm), "r"(c0), "r"(r0), "r"(su(&bar[st])) : "memory");
      }
      asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(su(&bar[st])), "r"(ph) : "memory");
    }
    // each thread: one row of 64 values (128 B) -> add 1.0 (or write 1.0)
    uint4* row = reinterpret_cast<uint4*>(b + tid * 128);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      uint4 v = MODE == 1 ? row[c] : make_uint4(0, 0, 0, 0);
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
      for (int i = 0; i < 4; ++i) h[i] = __hadd2(h[i], __floats2bfloat162_rn(1.f, 1.f));
      row[c] = v;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      if (MODE == 0)
        asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%1, %2}], [%3];"
                     ::"l"(&tm), "r"(c0), "r"(r0), "r"(su(b)) : "memory");
      else
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                     ::"l"(&tm), "r"(c0), "r"(r0), "r"(su(b)) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// 5: TMA reduce-add of 128 x 128 boxes (32 KiB, SWIZZLE_NONE): half the ops
__global__ void __launch_bounds__(128) yrmw_wide(const __grid_constant__ CUtensorMap tm) {
  extern __shared__ __align__(1024) char smem[];
  char* buf = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  const uint32_t tid = threadIdx.x;
  constexpr int TILESW = (M / TM) * (N / TNW);
  uint32_t k = 0;
  for (uint32_t t = blockIdx.x; t < TILESW; t += gridDim.x, ++k) {
    char* b = buf + (k & 1) * 32768;
    const int c0 = (t % (N / TNW)) * TNW, r0 = (t / (N / TNW)) * TM;
    if (k >= 2) {
      if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      __syncthreads();
    }
    uint4* row = reinterpret_cast<uint4*>(b + tid * 256);
#pragma unroll
    for (int c = 0; c < 16; ++c) {
      uint4 v = make_uint4(0, 0, 0, 0);
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
      for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(1.f, 1.f);
      row[c] = v;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%1, %2}], [%3];"
                   ::"l"(&tm), "r"(c0), "r"(r0), "r"(su(b)) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// 3: plain CUDA — every thread one row's 64 columns of a tile: 8 x 16-byte
//    loads, add, 8 x 16-byte stores (the layout an epilogue thread holds)
__global__ void __launch_bounds__(128) yrmw_plain(__nv_bfloat16* y) {
  for (uint32_t t = blockIdx.x; t < TILES; t += gridDim.x) {
    const int c0 = (t % (N / TN)) * TN, r0 = (t / (N / TN)) * TM;
    uint4* row = reinterpret_cast<uint4*>(y + static_cast<size_t>(r0 + threadIdx.x) * N + c0);
    uint4 v[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) v[c] = __ldcg(row + c);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v[c]);
#pragma unroll
      for (int i = 0; i < 4; ++i) h[i] = __hadd2(h[i], __floats2bfloat162_rn(1.f, 1.f));
      __stcg(row + c, v[c]);
    }
  }
}

// 4: plain CUDA, coalesced: a warp's 32 lanes cover 512 contiguous bytes
__global__ void __launch_bounds__(256) yrmw_flat(uint4* y, size_t n) {
  for (size_t i = blockIdx.x * 256ull + threadIdx.x; i < n; i += gridDim.x * 256ull) {
    uint4 v = __ldcs(y + i);
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
    for (int k = 0; k < 4; ++k) h[k] = __hadd2(h[k], __floats2bfloat162_rn(1.f, 1.f));
    __stcs(y + i, v);
  }
}

int main() {
  void* y;
  CK(cudaMalloc(&y, size_t(M) * N * 2));
  CK(cudaMemset(y, 0, size_t(M) * N * 2));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q{};
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap tm;
  const cuuint64_t dims[2] = {N, M};
  const cuuint64_t strides[1] = {N * 2ull};
  const cuuint32_t box[2] = {TN, TM};
  const cuuint32_t es[2] = {1, 1};
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, y, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n");
    return 1;
  }
  const int smem = 2 * 16384 + 1024;
  CK(cudaFuncSetAttribute(yrmw<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(yrmw<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(yrmw<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  char* flush;
  CK(cudaMalloc(&flush, 256 << 20));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[3] = {"TMA reduce-add (product)", "TMA load + add + TMA store", "TMA store only (no read)"};
  for (int grid : {296, 592, 888})
    for (int m = 0; m < 3; ++m) {
      float tot = 0.f;
      for (int i = 0; i < 20; ++i) {
        cudaMemset(flush, i, 256 << 20);
        cudaEventRecord(e0);
        if (m == 0) yrmw<0><<<grid, 128, smem>>>(tm);
        if (m == 1) yrmw<1><<<grid, 128, smem>>>(tm);
        if (m == 2) yrmw<2><<<grid, 128, smem>>>(tm);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        tot += ms;
      }
      const double us = tot / 20 * 1e3, bytes = (m == 2 ? 1.0 : 2.0) * M * N * 2;
      printf("grid %4d  %-28s %8.1f us  %6.2f TB/s DRAM\n", grid, names[m], us, bytes / (us * 1e-6) / 1e12);
    }
  {
    CUtensorMap tw;
    const cuuint32_t boxw[2] = {TNW, TM};
    if (enc(&tw, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, y, dims, strides, boxw, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      printf("encode (wide) failed\n");
      return 1;
    }
    const int smw = 2 * 32768 + 1024;
    CK(cudaFuncSetAttribute(yrmw_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, smw));
    for (int grid : {296, 444, 888}) {
      float tot = 0.f;
      for (int i = 0; i < 20; ++i) {
        cudaMemset(flush, i, 256 << 20);
        cudaEventRecord(e0);
        yrmw_wide<<<grid, 128, smw>>>(tw);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        tot += ms;
      }
      const double us = tot / 20 * 1e3;
      printf("grid %4d  %-28s %8.1f us  %6.2f TB/s DRAM\n", grid, "TMA reduce-add 128x128 boxes", us,
             2.0 * M * N * 2 / (us * 1e-6) / 1e12);
    }
  }
  for (int grid : {1184, 2368, 4736}) {
    for (int m = 0; m < 2; ++m) {
      float tot = 0.f;
      for (int i = 0; i < 20; ++i) {
        cudaMemset(flush, i, 256 << 20);
        cudaEventRecord(e0);
        if (m == 0) yrmw_plain<<<grid, 128>>>(static_cast<__nv_bfloat16*>(y));
        else yrmw_flat<<<grid, 256>>>(static_cast<uint4*>(y), size_t(M) * N / 8);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        tot += ms;
      }
      const double us = tot / 20 * 1e3;
      printf("grid %4d  %-28s %8.1f us  %6.2f TB/s DRAM\n", grid, m ? "plain ld/st, flat coalesced" : "plain ld/st, row per thread",
             us, 2.0 * M * N * 2 / (us * 1e-6) / 1e12);
    }
  }
  return 0;
}
