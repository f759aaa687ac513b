// microbench: the single-layer decode shrink's data path alone (cfg2: 960
// warp items of 8 rank rows x 8 KiB, rows scattered over 2 KiB pages), three
// ways of moving a warp's 64 KiB into shared memory, no math:
//   0  per-lane cp.async.cg 16 B pieces into a 32-unit (16 KiB) ring per warp
//      (the product's bgmv_warp shrink)
//   1  1-D TMA bulk copies of 512 B units (one row's chunk), 8 lanes issuing,
//      a 4-chunk ring (16 KiB) with one mbarrier per chunk slot
//   2  1-D TMA bulk copies of whole 2 KiB page pieces, 4 lanes issuing one
//      row-page each, a ring of 8 pieces (16 KiB)
// 2-warp CTAs, 36 KiB of smem per CTA (as the product), CUDA events, 20 reps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_s scripts/microbench_sphase.cu
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int ITEMS = 960, ROWS = 8, ROWB = 8192, PAGE = 2048;
constexpr int SMEM_WARP = 18432;  // 36 units x 512 B (ring + y area, as the product)

__device__ __forceinline__ uint32_t su(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void cpa16(uint32_t d, const void* s) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(s) : "memory");
}
__device__ __forceinline__ void bulk(uint32_t d, const void* s, uint32_t n, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(d), "l"(s), "r"(n), "r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c)); }
__device__ __forceinline__ void expect(uint32_t b, uint32_t n) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(n) : "memory");
}
__device__ __forceinline__ void mwait(uint32_t b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(b), "r"(ph) : "memory");
}

template <int MODE, int NS2 = 8>
__global__ void __launch_bounds__(64) sphase(const char* arena, const uint32_t* table, float* out) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t bars[2][16];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t item = blockIdx.x * 2 + warp;
  if (item >= ITEMS) return;
  const uint32_t* tab = table + item * (ROWS * ROWB / PAGE);  // the item's 32 pages
  char* ring = smem + warp * SMEM_WARP;
  float acc = 0.f;
  if (MODE == 0) {
    constexpr int RG = 32, LA = RG / ROWS;  // chunks ahead (16 chunks of 512 B per row)
    auto issue = [&](int c, int i) {
      const uint32_t off = i * ROWB + c * 512 + lane * 16;
      const bool v = c < 16;
      const char* src = arena + (static_cast<uint64_t>(tab[off / PAGE]) * PAGE) + off % PAGE;
      if (v) cpa16(su(ring + ((c % LA) * ROWS + i) * 512 + lane * 16), src);
      asm volatile("cp.async.commit_group;");
    };
    for (int c = 0; c < LA; ++c) for (int i = 0; i < ROWS; ++i) issue(c, i);
    for (int c = 0; c < 16; ++c)
      for (int i = 0; i < ROWS; ++i) {
        asm volatile("cp.async.wait_group %0;" ::"n"(RG - 1));
        acc += *reinterpret_cast<const float*>(ring + ((c % LA) * ROWS + i) * 512 + lane * 16);
        issue(c + LA, i);
      }
    asm volatile("cp.async.wait_group 0;");
  } else if (MODE == 1) {
    constexpr int NS = 4;  // chunk slots of 8 rows x 512 B
    const uint32_t b0 = su(&bars[warp][0]);
    if (lane == 0) for (int s = 0; s < NS; ++s) mbar_init(b0 + s * 8, 1);
    __syncwarp();
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    auto issue = [&](int c) {
      if (c >= 16) return;
      const int s = c % NS;
      if (lane == 0) expect(b0 + s * 8, ROWS * 512);
      __syncwarp();
      if (lane < ROWS) {
        const uint32_t off = lane * ROWB + c * 512;
        bulk(su(ring + (s * ROWS + lane) * 512), arena + static_cast<uint64_t>(tab[off / PAGE]) * PAGE + off % PAGE, 512,
             b0 + s * 8);
      }
    };
    for (int c = 0; c < NS; ++c) issue(c);
    for (int c = 0; c < 16; ++c) {
      mwait(b0 + (c % NS) * 8, (c / NS) & 1);
      for (int i = 0; i < ROWS; ++i) acc += *reinterpret_cast<const float*>(ring + ((c % NS) * ROWS + i) * 512 + lane * 16);
      __syncwarp();
      issue(c + NS);
    }
  } else {
    constexpr int NS = NS2;  // 2 KiB piece slots; piece k = (page chunk k / 8, row k % 8)
    const uint32_t b0 = su(&bars[warp][0]);
    if (lane == 0) for (int s = 0; s < NS; ++s) mbar_init(b0 + s * 8, 1);
    __syncwarp();
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    auto issue = [&](int k) {  // pieces k .. k+3 by lanes 0..3
      if (k >= 32) return;
      if (lane < 4) {
        const int kk = k + lane, s = kk % NS;
        const uint32_t off = (kk % ROWS) * ROWB + (kk / ROWS) * PAGE;
        expect(b0 + s * 8, PAGE);
        bulk(su(ring + s * PAGE), arena + static_cast<uint64_t>(tab[off / PAGE]) * PAGE, PAGE, b0 + s * 8);
      }
    };
    for (int k = 0; k < NS; k += 4) issue(k);
    for (int k = 0; k < 32; ++k) {
      mwait(b0 + (k % NS) * 8, (k / NS) & 1);
      acc += *reinterpret_cast<const float*>(ring + (k % NS) * PAGE + lane * 16);
      __syncwarp();
      if (k % 4 == 3) issue(k + NS - 3);
    }
  }
  if (acc == 123.f) out[item] = acc;
}

int main() {
  const uint64_t pages = 3ull << 20;  // 6 GiB arena of 2 KiB pages
  char* arena;
  uint32_t* table;
  float* out;
  CK(cudaMalloc(&arena, pages * PAGE));
  CK(cudaMemset(arena, 1, pages * PAGE));
  std::vector<uint32_t> t(ITEMS * 32);
  std::mt19937 rng(5);
  for (auto& v : t) v = rng() % pages;
  CK(cudaMalloc(&table, t.size() * 4));
  CK(cudaMemcpy(table, t.data(), t.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&out, ITEMS * 4));
  char* flush;
  CK(cudaMalloc(&flush, 256 << 20));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](auto kern, int smem, const char* name, const uint32_t* tb) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    float tot = 0.f;
    for (int i = 0; i < 20; ++i) {
      cudaMemset(flush, i, 256 << 20);
      cudaEventRecord(e0);
      kern<<<ITEMS / 2, 64, smem>>>(arena, tb, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      tot += ms;
    }
    const double us = tot / 20 * 1e3;
    printf("%-52s %7.2f us  %6.2f TB/s\n", name, us, ITEMS * 65536.0 / (us * 1e-6) / 1e12);
  };
  std::vector<uint32_t> ts(ITEMS * 32);
  for (size_t i = 0; i < ts.size(); ++i) ts[i] = static_cast<uint32_t>(i);
  uint32_t* tseq;
  CK(cudaMalloc(&tseq, ts.size() * 4));
  CK(cudaMemcpy(tseq, ts.data(), ts.size() * 4, cudaMemcpyHostToDevice));
  for (int rep = 0; rep < 2; ++rep) {
    run(sphase<0>, 2 * SMEM_WARP, "cp.async 16B/lane, 16 KiB ring, random pages", table);
    run(sphase<2, 8>, 2 * SMEM_WARP, "bulk 2KiB pieces, 16 KiB ring, random pages", table);
    run(sphase<2, 4>, 2 * SMEM_WARP, "bulk 2KiB pieces, 8 KiB ring, random pages", table);
    run(sphase<2, 16>, 2 * 2 * SMEM_WARP, "bulk 2KiB pieces, 32 KiB ring, random pages", table);
    run(sphase<0>, 2 * SMEM_WARP, "cp.async 16B/lane, 16 KiB ring, sequential pages", tseq);
    run(sphase<2, 8>, 2 * SMEM_WARP, "bulk 2KiB pieces, 16 KiB ring, sequential pages", tseq);
    run(sphase<2, 16>, 2 * 2 * SMEM_WARP, "bulk 2KiB pieces, 32 KiB ring, sequential pages", tseq);
  }
  // an empty launch for the launch + event overhead
  float tot = 0.f;
  for (int i = 0; i < 20; ++i) {
    cudaEventRecord(e0);
    sphase<0><<<1, 64, 2 * SMEM_WARP>>>(arena, table, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    tot += ms;
  }
  printf("one-CTA launch (launch + 1 item): %.2f us\n", tot / 20 * 1e3);
  return 0;
}
