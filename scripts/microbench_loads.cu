// Microbenchmark: achievable HBM read bandwidth on B200 for the load
// mechanisms a paged-LoRA kernel can use, as a function of piece size and
// bytes in flight per SM.  Reads `pieces` chunks of `piece` bytes at
// pseudo-random page-aligned offsets (like a scattered page table).
//   mode 0: cp.async.bulk (1-D TMA) into smem, one mbarrier per CTA-iteration
//   mode 1: LDG.128 by all threads, accumulate into a register (kept live)
//   mode 2: cp.async 16 B (LDGSTS) into smem
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb microbench_loads.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void bulk_kernel(const char* src, uint64_t n_pages, uint32_t page, uint32_t piece,
                            uint32_t per_cta_bytes, uint32_t iters, unsigned long long* sink) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  uint32_t phase = 0;
  uint64_t h = blockIdx.x * 0x9E3779B97F4A7C15ull;
  for (uint32_t it = 0; it < iters; ++it) {
    if (threadIdx.x < 32) {
      const uint32_t n = per_cta_bytes / piece;
      if (threadIdx.x == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                     "r"(per_cta_bytes));
      __syncwarp();
      for (uint32_t q = threadIdx.x; q < n; q += 32) {
        uint64_t x = (h + it * 7919ull + q) * 0xD1B54A32D192ED03ull;
        x ^= x >> 29;
        const uint64_t pg = x % n_pages;
        const uint64_t off = pg * page + (q * piece) % page;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                "r"(smem_u32(smem + q * piece)),
            "l"(src + off), "r"(piece), "r"(smem_u32(&bar))
            : "memory");
      }
    }
    uint32_t ok = 0;
    while (!ok)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(ok)
          : "r"(smem_u32(&bar)), "r"(phase));
    phase ^= 1;
    __syncthreads();
  }
  if (threadIdx.x == 0) atomicAdd(sink, static_cast<unsigned long long>(smem[7]));
}

__global__ void ldg_kernel(const char* src, uint64_t n_pages, uint32_t page, uint32_t piece,
                           uint32_t per_cta_bytes, uint32_t iters, unsigned long long* sink) {
  uint64_t h = blockIdx.x * 0x9E3779B97F4A7C15ull;
  uint32_t acc = 0;
  const uint32_t vec_per_piece = piece / 16;
  for (uint32_t it = 0; it < iters; ++it) {
    const uint32_t n = per_cta_bytes / 16;
    uint4 v[8];
    for (uint32_t i0 = threadIdx.x; i0 < n; i0 += blockDim.x * 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t i = i0 + u * blockDim.x;
        const uint32_t q = i / vec_per_piece, e = i % vec_per_piece;
        uint64_t x = (h + it * 7919ull + q) * 0xD1B54A32D192ED03ull;
        x ^= x >> 29;
        const uint64_t off = (x % n_pages) * page + (q * piece) % page + e * 16;
        if (i < n) {
          asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                       : "l"(src + off));
        } else {
          v[u] = make_uint4(0, 0, 0, 0);
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].w;
    }
  }
  if (acc == 0x12345678) atomicAdd(sink, 1ull);
}

__global__ void ldgsts_kernel(const char* src, uint64_t n_pages, uint32_t page, uint32_t piece,
                              uint32_t per_cta_bytes, uint32_t iters, unsigned long long* sink) {
  extern __shared__ __align__(128) char smem[];
  uint64_t h = blockIdx.x * 0x9E3779B97F4A7C15ull;
  const uint32_t vec_per_piece = piece / 16;
  for (uint32_t it = 0; it < iters; ++it) {
    const uint32_t n = per_cta_bytes / 16;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
      const uint32_t q = i / vec_per_piece, e = i % vec_per_piece;
      uint64_t x = (h + it * 7919ull + q) * 0xD1B54A32D192ED03ull;
      x ^= x >> 29;
      const uint64_t off = (x % n_pages) * page + (q * piece) % page + e * 16;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem + i * 16)),
                   "l"(src + off)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    __syncthreads();
  }
  if (threadIdx.x == 0) atomicAdd(sink, static_cast<unsigned long long>(smem[5]));
}

int main() {
  const uint64_t bytes = 4ull << 30;  // 4 GiB source (>> L2)
  char* src;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 1, bytes);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint32_t page = 2048;
  const uint64_t n_pages = bytes / page;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (void* fnp : {(void*)bulk_kernel, (void*)ldgsts_kernel})
    cudaFuncSetAttribute(fnp, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  printf("mode piece per_cta ctas_per_sm threads GB/s\n");
  for (int mode = 0; mode < 3; ++mode) {
    for (uint32_t piece : {512u, 2048u}) {
      for (uint32_t per_cta : {16384u, 32768u, 65536u}) {
        for (uint32_t cps : {1u, 2u, 4u, 8u}) {
          if (per_cta * cps > 200 * 1024 && mode != 1) continue;
          const uint32_t threads = mode == 0 ? 64 : 256;
          const uint32_t grid = sms * cps;
          const uint32_t iters = static_cast<uint32_t>((2ull << 30) / (uint64_t(per_cta) * grid)) + 1;
          auto run = [&]() {
            if (mode == 0)
              bulk_kernel<<<grid, threads, per_cta>>>(src, n_pages, page, piece, per_cta, iters, sink);
            else if (mode == 1)
              ldg_kernel<<<grid, threads>>>(src, n_pages, page, piece, per_cta, iters, sink);
            else
              ldgsts_kernel<<<grid, threads, per_cta>>>(src, n_pages, page, piece, per_cta, iters, sink);
          };
          run();
          cudaEventRecord(e0);
          run();
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          cudaError_t err = cudaGetLastError();
          const double gb = double(per_cta) * grid * iters / 1e9;
          printf("%d %u %u %u %u %.0f %s\n", mode, piece, per_cta, cps, threads, gb / (ms / 1e3),
                 err == cudaSuccess ? "" : cudaGetErrorString(err));
        }
      }
    }
  }
  return 0;
}
