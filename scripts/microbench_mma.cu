// Microbenchmark: legacy warp-level mma.sync throughput / latency on B200
// (sm_100a), m16n8k16 and m16n8k8 bf16 -> fp32, as a function of warps per
// SM and independent accumulator chains per warp.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_mma microbench_mma.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

template <int CHAINS, bool K16>
__global__ void mma_kernel(int iters, float* out, long long* cycles) {
  float d[CHAINS][4] = {};
  uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, threadIdx.x * 5u, threadIdx.x * 7u};
  uint32_t b[2] = {threadIdx.x * 11u, threadIdx.x * 13u};
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      if (K16)
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
            "{%8,%9}, {%0,%1,%2,%3};"
            : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      else
        asm volatile(
            "mma.sync.aligned.m16n8k8.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
            "{%0,%1,%2,%3};"
            : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
            : "r"(a[0]), "r"(a[1]), "r"(b[0]));
    }
  }
  long long t1 = clock64();
  float s = 0;
  for (int c = 0; c < CHAINS; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = t1 - t0;
}

template <int CHAINS, bool K16>
void run(int warps, float* out, long long* dcyc) {
  const int iters = 4096;
  mma_kernel<CHAINS, K16><<<148, warps * 32>>>(iters, out, dcyc);
  cudaDeviceSynchronize();
  long long cyc;
  cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
  const double per = double(cyc) / (double(iters) * CHAINS);
  const double fma = (K16 ? 2048.0 : 1024.0) * warps / per;  // FMA per clock per SM
  printf("%s warps/SM=%2d chains=%d: %.1f cycles per mma per warp, %.0f FMA/clk/SM\n",
         K16 ? "m16n8k16" : "m16n8k8 ", warps, CHAINS, per, fma);
}

int main() {
  float* out;
  long long* dcyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&dcyc, 8);
  for (int w : {1, 4, 8, 16}) {
    run<1, true>(w, out, dcyc);
    run<4, true>(w, out, dcyc);
    run<1, false>(w, out, dcyc);
    run<4, false>(w, out, dcyc);
  }
  return 0;
}
