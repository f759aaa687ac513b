// microbench: warp-per-item LDG streaming decode at cfg2 shapes, two phases
// (S: v = x·Aᵀ over groups of R rank rows; E: y += v·Bᵀ over 1024-column
// blocks), paged rows read through a scattered page table with 16-byte
// ld.global.nc.  Question it answers: how close does a plain load-stream
// design (no TMA, no smem ring, no clusters) get to the HBM read roofline
// for the 32-layer decode step?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_ldg scripts/microbench_ldg.cu
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e = (x);                                                           \
    if (e != cudaSuccess) {                                                        \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);     \
      return 1;                                                                    \
    }                                                                              \
  } while (0)

constexpr int H = 4096, L = 32, P = 2, NA = 128, T = 2, NTOK = NA * T;
constexpr int LOGP = 11;

__device__ __forceinline__ uint4 ldw(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void bf8(const uint4& a, float (&f)[8]) {
  const uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}

template <int R, int MATH>
__global__ void __launch_bounds__(256) kS(const char* __restrict__ arena, const uint32_t* __restrict__ table,
                                          const uint4* __restrict__ items, int n_items,
                                          const __nv_bfloat16* __restrict__ x, float* __restrict__ v) {
  const int wi = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (wi >= n_items) return;
  const uint4 it = items[wi];  // a, lp, j0, toff
  const uint32_t a = it.x, lp = it.y, j0 = it.z, toff = it.w, r = 8u << (a & 3);
  const uint64_t base = static_cast<uint64_t>(lp) * r * 16384 + static_cast<uint64_t>(j0) * 8192;
  const uint32_t pg0 = static_cast<uint32_t>(base >> LOGP);
  const uint32_t ent = __ldg(table + toff + pg0 + lane);  // R*4 == 32 pages
  const char* xr[T];
#pragma unroll
  for (int t = 0; t < T; ++t)
    xr[t] = reinterpret_cast<const char*>(x) + ((static_cast<uint64_t>(lp / P) * NTOK + a * T + t) * H) * 2;
  float acc[R][T];
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int t = 0; t < T; ++t) acc[i][t] = 0.f;
#pragma unroll 2
  for (int c = 0; c < 16; ++c) {
    uint4 xv[T];
#pragma unroll
    for (int t = 0; t < T; ++t) xv[t] = __ldg(reinterpret_cast<const uint4*>(xr[t] + c * 512 + lane * 16));
    uint4 w[R];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const uint32_t e = __shfl_sync(0xffffffffu, ent, i * 4 + (c >> 2));
      w[i] = ldw(arena + (static_cast<uint64_t>(e) << LOGP) + (c & 3) * 512 + lane * 16);
    }
    if (MATH) {
#pragma unroll
      for (int t = 0; t < T; ++t) {
        float xf[8];
        bf8(xv[t], xf);
#pragma unroll
        for (int i = 0; i < R; ++i) {
          float wf[8];
          bf8(w[i], wf);
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[i][t] = fmaf(wf[e], xf[e], acc[i][t]);
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < R; ++i) acc[i][0] += __uint_as_float(w[i].x ^ w[i].y ^ w[i].z ^ w[i].w);
    }
  }
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int t = 0; t < T; ++t) {
      float s = acc[i][t];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) v[(static_cast<uint64_t>(lp) * NTOK + a * T + t) * 64 + j0 + i] = s;
    }
}

template <int NS, int MATH>
__global__ void __launch_bounds__(256) kE(const char* __restrict__ arena, const uint32_t* __restrict__ table,
                                          const uint4* __restrict__ items, int n_items, const float* __restrict__ v,
                                          __nv_bfloat16* __restrict__ y) {
  const int wi = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (wi >= n_items) return;
  const uint4 it = items[wi];  // a, lp, cb, toff
  const uint32_t a = it.x, lp = it.y, cb = it.z, toff = it.w, r = 8u << (a & 3);
  const uint64_t bt = static_cast<uint64_t>(lp) * r * 16384 + static_cast<uint64_t>(r) * 8192;
  const uint32_t pb = static_cast<uint32_t>(bt >> LOGP) + cb;
  const uint32_t e0 = lane < r ? __ldg(table + toff + pb + lane * 4) : 0u;
  const uint32_t e1 = lane + 32 < r ? __ldg(table + toff + pb + (lane + 32) * 4) : 0u;
  float vv[T][2];
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const float* vr = v + (static_cast<uint64_t>(lp) * NTOK + a * T + t) * 64;
    vv[t][0] = lane < r ? vr[lane] : 0.f;
    vv[t][1] = lane + 32 < r ? vr[lane + 32] : 0.f;
  }
  float acc[NS][8][T];
#pragma unroll
  for (int s = 0; s < NS; ++s)
#pragma unroll
    for (int e = 0; e < 8; ++e)
#pragma unroll
      for (int t = 0; t < T; ++t) acc[s][e][t] = 0.f;
#pragma unroll 4
  for (uint32_t j = 0; j < r; ++j) {
    const uint32_t e = __shfl_sync(0xffffffffu, j < 32 ? e0 : e1, j & 31);
    uint4 w[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) w[s] = ldw(arena + (static_cast<uint64_t>(e) << LOGP) + s * 512 + lane * 16);
    float vt[T];
#pragma unroll
    for (int t = 0; t < T; ++t) vt[t] = __shfl_sync(0xffffffffu, j < 32 ? vv[t][0] : vv[t][1], j & 31);
    if (MATH) {
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        float wf[8];
        bf8(w[s], wf);
#pragma unroll
        for (int ee = 0; ee < 8; ++ee)
#pragma unroll
          for (int t = 0; t < T; ++t) acc[s][ee][t] = fmaf(vt[t], wf[ee], acc[s][ee][t]);
      }
    } else {
#pragma unroll
      for (int s = 0; s < NS; ++s) acc[s][0][0] += __uint_as_float(w[s].x ^ w[s].y ^ w[s].z ^ w[s].w);
    }
  }
#pragma unroll
  for (int t = 0; t < T; ++t)
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      uint4* yp = reinterpret_cast<uint4*>(y + (static_cast<uint64_t>(lp) * NTOK + a * T + t) * H + cb * 1024 +
                                           s * 256 + lane * 8);
      uint4 yv = *yp;
      float f[8];
      bf8(yv, f);
      uint32_t o[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * i] + acc[s][2 * i][t], f[2 * i + 1] + acc[s][2 * i + 1][t]);
        o[i] = *reinterpret_cast<uint32_t*>(&h);
      }
      *yp = make_uint4(o[0], o[1], o[2], o[3]);
    }
}

__device__ __forceinline__ void fh(float& acc, uint32_t a, uint32_t b) {  // acc += a.lo*b.lo + a.hi*b.hi (bf16 pairs)
  asm("{\n\t.reg .b16 al, ah, bl, bh;\n\tmov.b32 {al, ah}, %1;\n\tmov.b32 {bl, bh}, %2;\n\t"
      "fma.rn.f32.bf16 %0, al, bl, %0;\n\tfma.rn.f32.bf16 %0, ah, bh, %0;\n\t}"
      : "+f"(acc) : "r"(a), "r"(b));
}
__device__ __forceinline__ void ffma2(float& a0, float& a1, float w0, float w1, float v) {
  uint64_t acc, ww, vv;
  asm("mov.b64 %0, {%1, %2};" : "=l"(acc) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(ww) : "f"(w0), "f"(w1));
  asm("mov.b64 %0, {%1, %1};" : "=l"(vv) : "f"(v));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(ww), "l"(vv));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(acc));
}

// S v2: FHFMA (no conversions), loads of chunk c+1 issued before the math of chunk c
template <int R>
__global__ void __launch_bounds__(256) kS2(const char* __restrict__ arena, const uint32_t* __restrict__ table,
                                           const uint4* __restrict__ items, int n_items,
                                           const __nv_bfloat16* __restrict__ x, float* __restrict__ v) {
  const int wi = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (wi >= n_items) return;
  const uint4 it = items[wi];
  const uint32_t a = it.x, lp = it.y, j0 = it.z, toff = it.w, r = 8u << (a & 3);
  const uint64_t base = static_cast<uint64_t>(lp) * r * 16384 + static_cast<uint64_t>(j0) * 8192;
  const uint32_t pg0 = static_cast<uint32_t>(base >> LOGP);
  const uint32_t ent = __ldg(table + toff + pg0 + lane);
  const char* xr[T];
#pragma unroll
  for (int t = 0; t < T; ++t)
    xr[t] = reinterpret_cast<const char*>(x) + ((static_cast<uint64_t>(lp / P) * NTOK + a * T + t) * H) * 2;
  float acc[R][T];
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int t = 0; t < T; ++t) acc[i][t] = 0.f;
  auto ld = [&](int c, uint4 (&w)[R], uint4 (&xv)[T]) {
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const uint32_t e = __shfl_sync(0xffffffffu, ent, i * 4 + (c >> 2));
      w[i] = ldw(arena + (static_cast<uint64_t>(e) << LOGP) + (c & 3) * 512 + lane * 16);
    }
#pragma unroll
    for (int t = 0; t < T; ++t) xv[t] = __ldg(reinterpret_cast<const uint4*>(xr[t] + c * 512 + lane * 16));
  };
  uint4 w[R], xv[T];
  ld(0, w, xv);
#pragma unroll 1
  for (int c = 0; c < 16; ++c) {
    uint4 wn[R], xn[T];
    if (c + 1 < 16) ld(c + 1, wn, xn);
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
      for (int t = 0; t < T; ++t) {
        fh(acc[i][t], w[i].x, xv[t].x);
        fh(acc[i][t], w[i].y, xv[t].y);
        fh(acc[i][t], w[i].z, xv[t].z);
        fh(acc[i][t], w[i].w, xv[t].w);
      }
#pragma unroll
    for (int i = 0; i < R; ++i) w[i] = wn[i];
#pragma unroll
    for (int t = 0; t < T; ++t) xv[t] = xn[t];
  }
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int t = 0; t < T; ++t) {
      float s = acc[i][t];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) v[(static_cast<uint64_t>(lp) * NTOK + a * T + t) * 64 + j0 + i] = s;
    }
}

// E v2: NS 256-column sub-blocks, rows in groups of G with the next group's
// loads in flight during the math; FFMA2 on converted weight pairs
template <int NS, int G>
__global__ void __launch_bounds__(256) kE2(const char* __restrict__ arena, const uint32_t* __restrict__ table,
                                           const uint4* __restrict__ items, int n_items, const float* __restrict__ v,
                                           __nv_bfloat16* __restrict__ y) {
  const int wi = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (wi >= n_items) return;
  const uint4 it = items[wi];  // a, lp, col0 (elements), toff
  const uint32_t a = it.x, lp = it.y, col0 = it.z, toff = it.w, r = 8u << (a & 3);
  const uint64_t bt = static_cast<uint64_t>(lp) * r * 16384 + static_cast<uint64_t>(r) * 8192 + col0 * 2;
  const uint32_t pb = static_cast<uint32_t>(bt >> LOGP);
  const uint32_t inpg = static_cast<uint32_t>(bt & 2047);
  const uint32_t e0 = lane < r ? __ldg(table + toff + pb + lane * 4) : 0u;
  const uint32_t e1 = lane + 32 < r ? __ldg(table + toff + pb + (lane + 32) * 4) : 0u;
  float vv[T][2];
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const float* vr = v + (static_cast<uint64_t>(lp) * NTOK + a * T + t) * 64;
    vv[t][0] = lane < r ? vr[lane] : 0.f;
    vv[t][1] = lane + 32 < r ? vr[lane + 32] : 0.f;
  }
  float acc[NS][8][T];
#pragma unroll
  for (int s = 0; s < NS; ++s)
#pragma unroll
    for (int e = 0; e < 8; ++e)
#pragma unroll
      for (int t = 0; t < T; ++t) acc[s][e][t] = 0.f;
  auto ld = [&](uint32_t j0, uint4 (&w)[G][NS]) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t j = j0 + g;
      const uint32_t e = __shfl_sync(0xffffffffu, j < 32 ? e0 : e1, j & 31);
#pragma unroll
      for (int s = 0; s < NS; ++s)
        w[g][s] = ldw(arena + (static_cast<uint64_t>(e) << LOGP) + inpg + s * 512 + lane * 16);
    }
  };
  uint4 w[G][NS];
  ld(0, w);
#pragma unroll 1
  for (uint32_t j0 = 0; j0 < r; j0 += G) {
    uint4 wn[G][NS];
    if (j0 + G < r) ld(j0 + G, wn);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t j = j0 + g;
      float vt[T];
#pragma unroll
      for (int t = 0; t < T; ++t) vt[t] = __shfl_sync(0xffffffffu, j < 32 ? vv[t][0] : vv[t][1], j & 31);
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        float wf[8];
        bf8(w[g][s], wf);
#pragma unroll
        for (int t = 0; t < T; ++t)
#pragma unroll
          for (int e = 0; e < 8; e += 2) ffma2(acc[s][e][t], acc[s][e + 1][t], wf[e], wf[e + 1], vt[t]);
      }
    }
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int s = 0; s < NS; ++s) w[g][s] = wn[g][s];
  }
#pragma unroll
  for (int t = 0; t < T; ++t)
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      uint4* yp = reinterpret_cast<uint4*>(y + (static_cast<uint64_t>(lp) * NTOK + a * T + t) * H + col0 +
                                           s * 256 + lane * 8);
      uint4 yv = *yp;
      float f[8];
      bf8(yv, f);
      uint32_t o[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * i] + acc[s][2 * i][t], f[2 * i + 1] + acc[s][2 * i + 1][t]);
        o[i] = *reinterpret_cast<uint32_t*>(&h);
      }
      *yp = make_uint4(o[0], o[1], o[2], o[3]);
    }
}

__device__ __forceinline__ void cpa16(uint32_t dst, const void* src, uint32_t n) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ uint4 lds16(uint32_t a) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
  return r;
}

// E v3: per-lane cp.async ring of D rows (NS 16-byte chunks per row per lane) in shared memory
template <int NS, int D, int WPB>
__global__ void __launch_bounds__(WPB * 32) kE3(const char* __restrict__ arena, const uint32_t* __restrict__ table,
                                                const uint4* __restrict__ items, int n_items,
                                                const float* __restrict__ v, __nv_bfloat16* __restrict__ y) {
  extern __shared__ __align__(16) char sm[];
  const int w = threadIdx.x >> 5, wi = blockIdx.x * WPB + w, lane = threadIdx.x & 31;
  if (wi >= n_items) return;
  const uint32_t ring = static_cast<uint32_t>(__cvta_generic_to_shared(sm)) + w * (D * NS * 512) + lane * 16;
  const uint4 it = items[wi];
  const uint32_t a = it.x, lp = it.y, col0 = it.z, toff = it.w, r = 8u << (a & 3);
  const uint64_t bt = static_cast<uint64_t>(lp) * r * 16384 + static_cast<uint64_t>(r) * 8192 + col0 * 2;
  const uint32_t pb = static_cast<uint32_t>(bt >> LOGP);
  const uint32_t inpg = static_cast<uint32_t>(bt & 2047);
  const uint32_t e0 = lane < r ? __ldg(table + toff + pb + lane * 4) : 0u;
  const uint32_t e1 = lane + 32 < r ? __ldg(table + toff + pb + (lane + 32) * 4) : 0u;
  auto issue = [&](uint32_t j) {
    const uint32_t e = __shfl_sync(0xffffffffu, (j & 32) ? e1 : e0, j & 31);
    const uint32_t slot = ring + (j % D) * (NS * 512);
#pragma unroll
    for (int s = 0; s < NS; ++s)
      cpa16(slot + s * 512, arena + (static_cast<uint64_t>(e) << LOGP) + inpg + s * 512 + lane * 16, j < r ? 16 : 0);
    cpa_commit();
  };
#pragma unroll
  for (int d = 0; d < D - 1; ++d) issue(d);
  float vv[T][2];
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const float* vr = v + (static_cast<uint64_t>(lp) * NTOK + a * T + t) * 64;
    vv[t][0] = lane < r ? vr[lane] : 0.f;
    vv[t][1] = lane + 32 < r ? vr[lane + 32] : 0.f;
  }
  float acc[NS][8][T];
#pragma unroll
  for (int s = 0; s < NS; ++s)
#pragma unroll
    for (int e = 0; e < 8; ++e)
#pragma unroll
      for (int t = 0; t < T; ++t) acc[s][e][t] = 0.f;
#pragma unroll 1
  for (uint32_t j = 0; j < r; ++j) {
    issue(j + D - 1);
    cpa_wait<D - 1>();
    const uint32_t slot = ring + (j % D) * (NS * 512);
    float vt[T];
#pragma unroll
    for (int t = 0; t < T; ++t) vt[t] = __shfl_sync(0xffffffffu, (j & 32) ? vv[t][1] : vv[t][0], j & 31);
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const uint4 wv = lds16(slot + s * 512);
      float wf[8];
      bf8(wv, wf);
#pragma unroll
      for (int t = 0; t < T; ++t)
#pragma unroll
        for (int e = 0; e < 8; e += 2) ffma2(acc[s][e][t], acc[s][e + 1][t], wf[e], wf[e + 1], vt[t]);
    }
  }
  cpa_wait<0>();
#pragma unroll
  for (int t = 0; t < T; ++t)
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      uint4* yp = reinterpret_cast<uint4*>(y + (static_cast<uint64_t>(lp) * NTOK + a * T + t) * H + col0 +
                                           s * 256 + lane * 8);
      uint4 yv = *yp;
      float f[8];
      bf8(yv, f);
      uint32_t o[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * i] + acc[s][2 * i][t], f[2 * i + 1] + acc[s][2 * i + 1][t]);
        o[i] = *reinterpret_cast<uint32_t*>(&h);
      }
      *yp = make_uint4(o[0], o[1], o[2], o[3]);
    }
}

// S v3: per-lane cp.async ring over (chunk c, row i) units, D units deep; x by LDG one chunk ahead
template <int R, int D, int WPB>
__global__ void __launch_bounds__(WPB * 32) kS3(const char* __restrict__ arena, const uint32_t* __restrict__ table,
                                                const uint4* __restrict__ items, int n_items,
                                                const __nv_bfloat16* __restrict__ x, float* __restrict__ v) {
  extern __shared__ __align__(16) char sm[];
  const int w = threadIdx.x >> 5, wi = blockIdx.x * WPB + w, lane = threadIdx.x & 31;
  if (wi >= n_items) return;
  const uint32_t ring = static_cast<uint32_t>(__cvta_generic_to_shared(sm)) + w * (D * 512) + lane * 16;
  const uint4 it = items[wi];
  const uint32_t a = it.x, lp = it.y, j0 = it.z, toff = it.w, r = 8u << (a & 3);
  const uint64_t base = static_cast<uint64_t>(lp) * r * 16384 + static_cast<uint64_t>(j0) * 8192;
  const uint32_t pg0 = static_cast<uint32_t>(base >> LOGP);
  const uint32_t ent = __ldg(table + toff + pg0 + lane);
  constexpr int NU = 16 * R;  // units
  auto issue = [&](int u) {
    const int c = u / R, i = u % R;
    const uint32_t e = __shfl_sync(0xffffffffu, ent, (i * 4 + (c >> 2)) & 31);
    cpa16(ring + (u % D) * 512, arena + (static_cast<uint64_t>(e) << LOGP) + (c & 3) * 512 + lane * 16, u < NU ? 16 : 0);
    cpa_commit();
  };
#pragma unroll
  for (int d = 0; d < D - 1; ++d) issue(d);
  const char* xr[T];
#pragma unroll
  for (int t = 0; t < T; ++t)
    xr[t] = reinterpret_cast<const char*>(x) + ((static_cast<uint64_t>(lp / P) * NTOK + a * T + t) * H) * 2;
  float acc[R][T];
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int t = 0; t < T; ++t) acc[i][t] = 0.f;
  uint4 xv[T];
#pragma unroll
  for (int t = 0; t < T; ++t) xv[t] = __ldg(reinterpret_cast<const uint4*>(xr[t] + lane * 16));
#pragma unroll 1
  for (int c = 0; c < 16; ++c) {
    uint4 xn[T];
#pragma unroll
    for (int t = 0; t < T; ++t)
      xn[t] = c + 1 < 16 ? __ldg(reinterpret_cast<const uint4*>(xr[t] + (c + 1) * 512 + lane * 16)) : xv[t];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int u = c * R + i;
      issue(u + D - 1);
      cpa_wait<D - 1>();
      const uint4 wv = lds16(ring + (u % D) * 512);
#pragma unroll
      for (int t = 0; t < T; ++t) {
        fh(acc[i][t], wv.x, xv[t].x);
        fh(acc[i][t], wv.y, xv[t].y);
        fh(acc[i][t], wv.z, xv[t].z);
        fh(acc[i][t], wv.w, xv[t].w);
      }
    }
#pragma unroll
    for (int t = 0; t < T; ++t) xv[t] = xn[t];
  }
  cpa_wait<0>();
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int t = 0; t < T; ++t) {
      float s = acc[i][t];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) v[(static_cast<uint64_t>(lp) * NTOK + a * T + t) * 64 + j0 + i] = s;
    }
}

int main() {
  // adapters: rank 8 << (a % 4); bytes r · L · P · 2H · 2 = r MiB; pages r · 512
  std::vector<uint32_t> toff(NA);
  uint64_t npages = 0, wbytes = 0;
  for (int a = 0; a < NA; ++a) {
    toff[a] = static_cast<uint32_t>(npages);
    npages += (8u << (a & 3)) * 512u;
  }
  wbytes = npages << LOGP;
  std::vector<uint32_t> perm(npages);
  for (uint64_t i = 0; i < npages; ++i) perm[i] = static_cast<uint32_t>(i);
  std::mt19937_64 rng(7);
  std::shuffle(perm.begin(), perm.end(), rng);
  std::vector<uint4> si, ei;
  for (int lp = 0; lp < L * P; ++lp)
    for (int a = 0; a < NA; ++a) {
      const uint32_t r = 8u << (a & 3);
      for (uint32_t j0 = 0; j0 < r; j0 += 8) si.push_back(make_uint4(a, lp, j0, toff[a]));
      for (uint32_t cb = 0; cb < 4; ++cb) ei.push_back(make_uint4(a, lp, cb, toff[a]));
    }
  // big first (LPT-ish for the hardware scheduler)
  std::stable_sort(ei.begin(), ei.end(), [](const uint4& p, const uint4& q) { return (p.x & 3) > (q.x & 3); });
  char* arena;
  uint32_t* table;
  uint4 *dsi, *dei;
  __nv_bfloat16 *x, *y;
  float* v;
  CK(cudaMalloc(&arena, wbytes));
  CK(cudaMemset(arena, 0x3c, wbytes));
  CK(cudaMalloc(&table, npages * 4));
  CK(cudaMemcpy(table, perm.data(), npages * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&dsi, si.size() * 16));
  CK(cudaMalloc(&dei, ei.size() * 16));
  CK(cudaMemcpy(dsi, si.data(), si.size() * 16, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dei, ei.data(), ei.size() * 16, cudaMemcpyHostToDevice));
  const uint64_t xe = static_cast<uint64_t>(L) * NTOK * H, ye = static_cast<uint64_t>(L) * P * NTOK * H;
  CK(cudaMalloc(&x, xe * 2));
  CK(cudaMalloc(&y, ye * 2));
  CK(cudaMemset(x, 0x3c, xe * 2));
  CK(cudaMemset(y, 0, ye * 2));
  CK(cudaMalloc(&v, static_cast<uint64_t>(L) * P * NTOK * 64 * 4));
  char* flush;
  CK(cudaMalloc(&flush, 512ull << 20));
  const double alg = wbytes + xe * 2.0 + ye * 4.0;
  printf("weights %.3f GB, algorithmic %.3f GB per step, S items %zu, E items %zu\n", wbytes / 1e9, alg / 1e9,
         si.size(), ei.size());
  cudaEvent_t e0, e1, e2;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventCreate(&e2);
  const int gs = static_cast<int>((si.size() + 7) / 8), ge = static_cast<int>((ei.size() + 7) / 8);
  for (int math = 0; math < 2; ++math) {
    float ts = 0, te = 0, best = 1e9;
    const int iters = 10;
    for (int i = 0; i < iters + 2; ++i) {
      cudaMemsetAsync(flush, i, 512ull << 20);
      cudaEventRecord(e0);
      if (math) kS<8, 1><<<gs, 256>>>(arena, table, dsi, (int)si.size(), x, v);
      else kS<8, 0><<<gs, 256>>>(arena, table, dsi, (int)si.size(), x, v);
      cudaEventRecord(e1);
      if (math) kE<4, 1><<<ge, 256>>>(arena, table, dei, (int)ei.size(), v, y);
      else kE<4, 0><<<ge, 256>>>(arena, table, dei, (int)ei.size(), v, y);
      cudaEventRecord(e2);
      CK(cudaEventSynchronize(e2));
      float a, b;
      cudaEventElapsedTime(&a, e0, e1);
      cudaEventElapsedTime(&b, e1, e2);
      if (i >= 2) {
        ts += a;
        te += b;
        best = std::min(best, a + b);
      }
    }
    ts /= iters;
    te /= iters;
    const double sb = wbytes / 2.0 + xe * 2.0, eb = wbytes / 2.0 + ye * 4.0;
    printf("math=%d  S %.1f us (%.0f GB/s)  E %.1f us (%.0f GB/s)  step %.1f us  best %.1f us  -> %.0f GB/s (frac %.3f of 6453)\n",
           math, ts * 1e3, sb / ts / 1e6, te * 1e3, eb / te / 1e6, (ts + te) * 1e3, best * 1e3,
           alg / (ts + te) / 1e6, alg / (ts + te) / 1e6 / 6453.4);
  }

  // v2 variants: E items of 512 columns (NS 2) and 256 (NS 1)
  for (int ns : {1, 2, 4}) {
    std::vector<uint4> ev2;
    for (int lp = 0; lp < L * P; ++lp)
      for (int a = 0; a < NA; ++a)
        for (uint32_t c = 0; c < H; c += 256 * ns) ev2.push_back(make_uint4(a, lp, c, toff[a]));
    std::stable_sort(ev2.begin(), ev2.end(), [](const uint4& p, const uint4& q) { return (p.x & 3) > (q.x & 3); });
    uint4* de2;
    CK(cudaMalloc(&de2, ev2.size() * 16));
    CK(cudaMemcpy(de2, ev2.data(), ev2.size() * 16, cudaMemcpyHostToDevice));
    const int g2 = static_cast<int>((ev2.size() + 7) / 8);
    for (int gsz : {2, 4}) {
      float ts = 0, te = 0;
      const int iters = 10;
      for (int i = 0; i < iters + 2; ++i) {
        cudaMemsetAsync(flush, i, 512ull << 20);
        cudaEventRecord(e0);
        kS2<8><<<gs, 256>>>(arena, table, dsi, (int)si.size(), x, v);
        cudaEventRecord(e1);
        if (ns == 1 && gsz == 2) kE2<1, 2><<<g2, 256>>>(arena, table, de2, (int)ev2.size(), v, y);
        if (ns == 1 && gsz == 4) kE2<1, 4><<<g2, 256>>>(arena, table, de2, (int)ev2.size(), v, y);
        if (ns == 2 && gsz == 2) kE2<2, 2><<<g2, 256>>>(arena, table, de2, (int)ev2.size(), v, y);
        if (ns == 2 && gsz == 4) kE2<2, 4><<<g2, 256>>>(arena, table, de2, (int)ev2.size(), v, y);
        if (ns == 4 && gsz == 2) kE2<4, 2><<<g2, 256>>>(arena, table, de2, (int)ev2.size(), v, y);
        if (ns == 4 && gsz == 4) kE2<4, 4><<<g2, 256>>>(arena, table, de2, (int)ev2.size(), v, y);
        cudaEventRecord(e2);
        CK(cudaEventSynchronize(e2));
        float a, b;
        cudaEventElapsedTime(&a, e0, e1);
        cudaEventElapsedTime(&b, e1, e2);
        if (i >= 2) {
          ts += a;
          te += b;
        }
      }
      ts /= iters;
      te /= iters;
      const double sb = wbytes / 2.0 + xe * 2.0, eb = wbytes / 2.0 + ye * 4.0;
      printf("v2 NS=%d G=%d  S %.1f us (%.0f GB/s)  E %.1f us (%.0f GB/s)  step %.1f us -> %.0f GB/s (frac %.3f)\n", ns,
             gsz, ts * 1e3, sb / ts / 1e6, te * 1e3, eb / te / 1e6, (ts + te) * 1e3, alg / (ts + te) / 1e6,
             alg / (ts + te) / 1e6 / 6453.4);
    }
    CK(cudaGetLastError());
  }

  // v3: cp.async rings
  {
    std::vector<uint4> ev2;
    for (int lp = 0; lp < L * P; ++lp)
      for (int a = 0; a < NA; ++a)
        for (uint32_t c = 0; c < H; c += 512) ev2.push_back(make_uint4(a, lp, c, toff[a]));
    std::stable_sort(ev2.begin(), ev2.end(), [](const uint4& p, const uint4& q) { return (p.x & 3) > (q.x & 3); });
    uint4* de2;
    CK(cudaMalloc(&de2, ev2.size() * 16));
    CK(cudaMemcpy(de2, ev2.data(), ev2.size() * 16, cudaMemcpyHostToDevice));
    auto runv = [&](const char* name, auto launchS, auto launchE) -> int {
      float ts = 0, te = 0;
      const int iters = 10;
      for (int i = 0; i < iters + 2; ++i) {
        cudaMemsetAsync(flush, i, 512ull << 20);
        cudaEventRecord(e0);
        launchS();
        cudaEventRecord(e1);
        launchE();
        cudaEventRecord(e2);
        CK(cudaEventSynchronize(e2));
        float a, b;
        cudaEventElapsedTime(&a, e0, e1);
        cudaEventElapsedTime(&b, e1, e2);
        if (i >= 2) { ts += a; te += b; }
      }
      ts /= iters; te /= iters;
      const double sb = wbytes / 2.0 + xe * 2.0, eb = wbytes / 2.0 + ye * 4.0;
      printf("%s  S %.1f us (%.0f GB/s)  E %.1f us (%.0f GB/s)  step %.1f us -> frac %.3f\n", name, ts * 1e3,
             sb / ts / 1e6, te * 1e3, eb / te / 1e6, (ts + te) * 1e3, alg / (ts + te) / 1e6 / 6453.4);
      CK(cudaGetLastError());
      return 0;
    };
    const int ne = (int)ev2.size(), ns = (int)si.size();
#define RUN3(DS, WS, DE, WE)                                                                                  \
    {                                                                                                         \
      const int smS = WS * DS * 512, smE = WE * DE * 2 * 512;                                                \
      cudaFuncSetAttribute(kS3<8, DS, WS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smS);                \
      cudaFuncSetAttribute(kE3<2, DE, WE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smE);                \
      runv("v3 S(D=" #DS ",W=" #WS ") E(D=" #DE ",W=" #WE ")",                                              \
           [&] { kS3<8, DS, WS><<<(ns + WS - 1) / WS, WS * 32, smS>>>(arena, table, dsi, ns, x, v); },      \
           [&] { kE3<2, DE, WE><<<(ne + WE - 1) / WE, WE * 32, smE>>>(arena, table, de2, ne, v, y); });      \
    }
    RUN3(8, 8, 4, 8)
    RUN3(12, 8, 6, 8)
    RUN3(16, 8, 8, 8)
    RUN3(16, 4, 8, 4)
    RUN3(24, 4, 12, 4)
    RUN3(12, 16, 6, 16)
  }
  CK(cudaGetLastError());
  return 0;
}
