// microbench: issue cost and throughput of 1-D TMA bulk copies (2 KiB page
// pieces into shared memory), the producer pattern of bgmv_stream.cu.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_bulk scripts/microbench_bulk.cu
// Each CTA runs W producer warps; each warp owns S slots of R rows x 2 KiB and
// loops: wait slot's full barrier (previous fill landed), re-issue R copies
// (one per lane, lanes 0..R-1, or all by lane 0) from pseudo-random pages of a
// large arena, arrive_expect_tx.  Reports the issue time per stage (clock64
// around the copy issue) and the achieved GB/s over all SMs.
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool try_wait(uint64_t* b, uint32_t ph) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(smem_u32(b)), "r"(ph) : "memory");
  return ok;
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

template <int MODE>  // 0: one copy per lane; 1: lane 0 issues all; 2: 2 KiB copies split in halves per lane pair
__global__ void k(const char* arena, uint64_t npages, int W, int S, int R, int iters, unsigned long long* issue_cyc,
                  unsigned long long* tot_cyc) {
  extern __shared__ __align__(128) char sm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm);
  char* data = sm + 1024;
  if (threadIdx.x == 0) {
    for (int i = 0; i < W * S; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned long long t_issue = 0;
  const long long t0 = clock64();
  uint64_t seed = (blockIdx.x * 131 + w) * 2654435761ull;
  for (int it = 0; it < iters; ++it) {
    const int s = it % S;
    uint64_t* bar = &bars[w * S + s];
    char* slot = data + (size_t)(w * S + s) * R * 2048;
    if (it >= S) {
      const uint32_t ph = ((it / S) - 1) & 1;
      while (!try_wait(bar, ph)) {
      }
    }
    const long long a = clock64();
    uint64_t pg[32];
    if (MODE == 1) {
      if (lane == 0) {
        for (int r = 0; r < R; ++r) {
          seed = seed * 6364136223846793005ull + 1442695040888963407ull;
          bulk(slot + r * 2048, arena + ((seed >> 20) % npages) * 2048, 2048, bar);
        }
        expect_tx(bar, R * 2048);
      }
    } else {
      seed = seed * 6364136223846793005ull + 1442695040888963407ull;
      const uint64_t mine = ((seed >> 20) + lane * 7919) % npages;
      if (MODE == 0) {
        if (lane < R) bulk(slot + lane * 2048, arena + mine * 2048, 2048, bar);
      } else {
        const int r = lane >> 1, h = lane & 1;
        if (r < R) bulk(slot + r * 2048 + h * 1024, arena + mine * 2048 + h * 1024, 1024, bar);
      }
      __syncwarp();
      if (lane == 0) expect_tx(bar, R * 2048);
    }
    __syncwarp();
    t_issue += clock64() - a;
    (void)pg;
  }
  // drain
  for (int s = 0; s < S && s < iters; ++s) {
    const int last = ((iters - 1 - s) / S) * S + s;
    while (!try_wait(&bars[w * S + s], (last / S) & 1)) {
    }
  }
  const long long t1 = clock64();
  if (lane == 0) {
    atomicAdd(issue_cyc, t_issue);
    atomicMax(tot_cyc, (unsigned long long)(t1 - t0));
  }
}

int main() {
  const uint64_t npages = (6ull << 30) / 2048;  // 6 GiB arena (> L2)
  char* arena;
  cudaMalloc(&arena, npages * 2048);
  cudaMemset(arena, 1, npages * 2048);
  unsigned long long *ic, *tc;
  cudaMalloc(&ic, 8);
  cudaMalloc(&tc, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto run = [&](auto kern, const char* name, int ctas, int W, int S, int R, int iters) {
    const int smem = 1024 + W * S * R * 2048;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaMemset(ic, 0, 8);
    cudaMemset(tc, 0, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kern<<<ctas, W * 32, smem>>>(arena, npages, W, S, R, 4, ic, tc);  // warm
    cudaDeviceSynchronize();
    cudaMemset(ic, 0, 8);
    cudaEventRecord(e0);
    kern<<<ctas, W * 32, smem>>>(arena, npages, W, S, R, iters, ic, tc);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long hi, ht;
    cudaMemcpy(&hi, ic, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&ht, tc, 8, cudaMemcpyDeviceToHost);
    const double bytes = double(ctas) * W * iters * R * 2048;
    printf("%-10s ctas=%3d warps=%d slots/warp=%d rows=%2d (%3d KB in flight/SM): issue %.0f cycles/stage, %.0f GB/s (%.1f GB/s/SM)\n",
           name, ctas, W, S, R, W * S * R * 2, double(hi) / (double(ctas) * W * iters), bytes / ms / 1e6,
           bytes / ms / 1e6 / ctas);
  };
  for (int ctas : {1, sms}) {
    run(k<0>, "per-lane", ctas, 5, 1, 16, 2000);
    run(k<1>, "lane0", ctas, 5, 1, 16, 2000);
    run(k<2>, "half-lanes", ctas, 5, 1, 16, 2000);
    run(k<0>, "per-lane", ctas, 5, 2, 8, 2000);
    run(k<0>, "per-lane", ctas, 10, 1, 8, 2000);
    run(k<0>, "per-lane", ctas, 6, 1, 16, 2000);
    run(k<0>, "per-lane", ctas, 3, 1, 32, 2000);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
