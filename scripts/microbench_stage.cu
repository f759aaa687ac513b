// microbench: per-stage consumer math of bgmv_stream (S stage: 8 x (ldsm.x4 + ldsm.x2 + mma.16816) per warp)
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t smem_u32(const void* p){return (uint32_t)__cvta_generic_to_shared(p);}
__device__ __forceinline__ void ldsm_x4(uint32_t a, uint32_t (&r)[4]){asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];":"=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]):"r"(a));}
__device__ __forceinline__ void ldsm_x2(uint32_t a, uint32_t (&r)[2]){asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];":"=r"(r[0]),"=r"(r[1]):"r"(a));}
__device__ __forceinline__ void mma(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]){
 asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};":"+f"(d[0]),"+f"(d[1]),"+f"(d[2]),"+f"(d[3]):"r"(a[0]),"r"(a[1]),"r"(a[2]),"r"(a[3]),"r"(b[0]),"r"(b[1]));}
constexpr uint32_t kRowB = 2064;
template<int WARPS, bool BATCH>
__global__ void k(int iters, float* out, long long* cyc){
  extern __shared__ char sm[];
  const uint32_t lane=threadIdx.x&31, w=threadIdx.x>>5;
  const uint32_t a_off = ((lane&7) + ((lane>>3)&1)*8)*kRowB + (lane>>4)*16;
  const uint32_t x_off = 16*kRowB + ((lane&7)&3)*kRowB + ((lane>>3)&1)*16;
  const uint32_t base = smem_u32(sm);
  float d[2][4]={};
  __syncthreads();
  long long t0=clock64();
  for(int it=0; it<iters; ++it){
    const uint32_t sb = base + (it&3)*0;  // same slot
    if (BATCH) {
      uint32_t fa[8][4], fb[8][2];
      #pragma unroll
      for(int j=0;j<8;++j){ const uint32_t kk = w + j*WARPS; ldsm_x4(sb+a_off+kk*32, fa[j]); ldsm_x2(sb+x_off+kk*32, fb[j]); }
      #pragma unroll
      for(int j=0;j<8;++j) mma(d[j&1], fa[j], fb[j]);
    } else {
      #pragma unroll
      for(int j=0;j<8;++j){ const uint32_t kk = w + j*WARPS; uint32_t fa[4], fb[2]; ldsm_x4(sb+a_off+kk*32, fa); ldsm_x2(sb+x_off+kk*32, fb); mma(d[j&1], fa, fb);}
    }
  }
  long long t1=clock64();
  out[blockIdx.x*blockDim.x+threadIdx.x]=d[0][0]+d[1][1];
  if(threadIdx.x==0&&blockIdx.x==0) *cyc=t1-t0;
}
int main(){
  float* out; long long* dc; cudaMalloc(&out, 148*1024*4); cudaMalloc(&dc,8);
  const int smem = 20*kRowB+1024;
  auto run=[&](auto kern, int warps, const char* name){
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<148, warps*32, smem>>>(1000, out, dc); cudaDeviceSynchronize();
    long long c; cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
    printf("%s warps=%d: %.1f cycles per stage (8 k-steps per warp)\n", name, warps, c/1000.0);
  };
  run(k<8,false>, 8, "serial"); run(k<8,true>, 8, "batched");
  run(k<16,true>, 16, "batched"); run(k<4,true>, 4, "batched");
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
