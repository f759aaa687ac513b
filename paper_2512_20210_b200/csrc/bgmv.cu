// Paged multi-LoRA decode op (gathered BGMV) for sm_100a.
//
// y[t, :] += scale · (x[t, :] · A_{a(t)}ᵀ) · B_{a(t)}ᵀ
//
// The reference only bills this op as a cost-model constant
// (include/lorasim/cost_model.hpp:32-40, billed at src/engine.cpp:355,510);
// weights are read straight out of the paged arena through the device page
// table (PagePool::translate semantics, src/memory.cpp:55-62).
//
// Design (HBM-bound: AI ≈ 1.8 flop/B at Llama-7B decode shapes).  Two
// streaming kernels per (layer, proj) call, chained with Programmatic
// Dependent Launch:
//
//  shrink  one CTA per (segment, <= 8 rank rows, <= 2 tokens): warp 0 issues
//          1-D TMA bulk copies (cp.async.bulk, one per page piece, L2
//          evict-first) of the rows — one contiguous logical range of the
//          adapter — and of the tokens' x rows into shared memory, all on one
//          mbarrier; then warp w dots row w with the x rows and warp-reduces
//          v = x·Aᵀ (fp32) into an L2-resident workspace.  It triggers the
//          dependent launch as soon as it starts.
//  expand  one CTA per (segment, <= 2 tokens, column block CB): it issues the
//          bulk copies of its Bᵀ tile (r × CB, r row pieces) and the y rows
//          BEFORE griddepcontrol.wait, so its weight stream overlaps the
//          shrink grid; after the wait it reads v, splits rows over RG groups
//          (<= 8 rows per thread), reduces in shared memory and stores y.
//
// Units are equal-byte slices built on the host (plan.cu); every adapter's
// weights are read once per call regardless of its token count.  Several
// CTAs per SM (48-80 KiB of smem each) keep >= 100 KiB in flight per SM.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstring>

#include "plan.hpp"
#include "ptx.cuh"

using namespace plora;

namespace {

constexpr int kThreads = 256;
constexpr uint32_t kExpandTok = 2;  // tokens per expand pass (reduction buffer)

struct BgmvArgs {
  const char* arena;
  const uint32_t* table;
  const BgmvUnit* units;
  float* v;
  const char* x;
  char* y;
  uint64_t x_stride_b;
  uint64_t y_stride_b;
  uint64_t blk_mult;  // block (layer, proj) starts at element rank · blk_mult
  uint32_t log2_page;
  uint32_t d_in;
  uint32_t d_out;
  float scale;
};

template <typename T>
struct VecOps;

template <>
struct VecOps<__nv_bfloat16> {
  static constexpr int N = 8;
  __device__ static __forceinline__ void unpack(const uint4& a, float (&f)[8]) {
    const __nv_bfloat162* pa = reinterpret_cast<const __nv_bfloat162*>(&a);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 t = __bfloat1622float2(pa[i]);
      f[2 * i] = t.x;
      f[2 * i + 1] = t.y;
    }
  }
  __device__ static __forceinline__ uint4 pack(const float (&f)[8]) {
    uint4 r;
    __nv_bfloat162* pr = reinterpret_cast<__nv_bfloat162*>(&r);
#pragma unroll
    for (int i = 0; i < 4; ++i) pr[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
    return r;
  }
};

template <>
struct VecOps<float> {
  static constexpr int N = 4;
  __device__ static __forceinline__ void unpack(const uint4& a, float (&f)[4]) {
    f[0] = __uint_as_float(a.x);
    f[1] = __uint_as_float(a.y);
    f[2] = __uint_as_float(a.z);
    f[3] = __uint_as_float(a.w);
  }
  __device__ static __forceinline__ uint4 pack(const float (&f)[4]) {
    return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]),
                      __float_as_uint(f[3]));
  }
};

__device__ __forceinline__ float warp_sum(float a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  return a;
}

__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// Bulk-copy the logical byte range [lo, lo + bytes) of an adapter into smem
// at dst, one cp.async.bulk per page piece, lanes in parallel.
__device__ __forceinline__ void gather_range(const BgmvArgs& p, uint32_t table_off, uint64_t lo,
                                             uint32_t bytes, char* dst, uint64_t* bar,
                                             uint64_t policy, uint32_t lane) {
  const uint32_t L = p.log2_page;
  const uint64_t hi = lo + bytes, p0 = lo >> L, p1 = (hi - 1) >> L;
  for (uint64_t pg = p0 + lane; pg <= p1; pg += 32) {
    const uint64_t a = max(lo, pg << L), b = min(hi, (pg + 1) << L);
    const uint32_t phys = __ldg(p.table + table_off + static_cast<uint32_t>(pg));
    ptx::bulk_g2s_hint(dst + (a - lo),
                       p.arena + (static_cast<uint64_t>(phys) << L) + (a & ((1ull << L) - 1)),
                       static_cast<uint32_t>(b - a), bar, policy);
  }
}

// ------------------------------------------------------------------ shrink
template <typename T>
__global__ void __launch_bounds__(kThreads) bgmv_shrink_kernel(const BgmvArgs p) {
  using V = VecOps<T>;
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t bar;
  pdl_launch_dependents();  // the expand grid may start streaming Bᵀ now
  const BgmvUnit u = p.units[blockIdx.x];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rowbytes = p.d_in * sizeof(T);
  const uint32_t rpu = min(kMaxShrinkRows, kShrinkWeightBytes / rowbytes);
  char* W = smem;                   // [count <= rpu][d_in]
  char* X = smem + rpu * rowbytes;  // [ntok][d_in]
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) ptx::mbar_arrive_expect_tx(&bar, (u.count + u.ntok) * rowbytes);
    __syncwarp();
    const uint64_t base =
        (static_cast<uint64_t>(u.rank) * p.blk_mult + static_cast<uint64_t>(u.off) * p.d_in) *
        sizeof(T);
    gather_range(p, u.table_off, base, u.count * rowbytes, W, &bar, ptx::policy_evict_first(),
                 lane);
    if (lane < u.ntok)
      ptx::bulk_g2s(X + lane * rowbytes, p.x + u.tok[lane] * p.x_stride_b, rowbytes, &bar);
  }
  ptx::mbar_wait(&bar, 0);
  if (warp < u.count) {
    const uint32_t nvec = p.d_in / V::N;
    const uint4* w = reinterpret_cast<const uint4*>(W + warp * rowbytes);
    const uint4* xs = reinterpret_cast<const uint4*>(X);
    float acc[kMaxUnitTok];
#pragma unroll
    for (int t = 0; t < kMaxUnitTok; ++t) acc[t] = 0.f;
#pragma unroll 4
    for (uint32_t c = lane; c < nvec; c += 32) {
      float wf[V::N];
      V::unpack(w[c], wf);
#pragma unroll
      for (int t = 0; t < kMaxUnitTok; ++t) {
        if (t < u.ntok) {
          float xf[V::N];
          V::unpack(xs[t * nvec + c], xf);
          float a = acc[t];
#pragma unroll
          for (int e = 0; e < V::N; ++e) a = fmaf(wf[e], xf[e], a);
          acc[t] = a;
        }
      }
    }
#pragma unroll
    for (int t = 0; t < kMaxUnitTok; ++t) {
      if (t < u.ntok) {
        const float s = warp_sum(acc[t]);
        if (lane == 0) p.v[u.voff + t * rpad4(u.rank) + u.off + warp] = s;
      }
    }
  }
}

// ------------------------------------------------------------------ expand
struct ExpandSmem {
  // [0, kSlotWeightBytes)            Bᵀ tile, row j at j · CB · esize
  // [.., + kSlotAuxBytes)            y rows, token t at t · CB · esize
  // [.., + kRedBytes)                cross-group partial sums
  // [.., + kMaxUnitTok·256·4)        v rows of the unit's tokens
  static constexpr uint32_t y = kSlotWeightBytes;
  static constexpr uint32_t red = y + kSlotAuxBytes;
  static constexpr uint32_t v = red + kRedBytes;
  static constexpr uint32_t total = v + kMaxUnitTok * kMaxBgmvRank * 4;
};

template <typename T, int RG>
__device__ __forceinline__ void expand_compute(const BgmvArgs& p, const BgmvUnit& u, char* smem) {
  using V = VecOps<T>;
  constexpr int CT = kBgmvConsumers / RG;
  constexpr int CB = CT * V::N;
  const uint32_t tid = threadIdx.x, rg = tid / CT, ct = tid % CT;
  const uint32_t rp = rpad4(u.rank);
  const uint4* Bs = reinterpret_cast<const uint4*>(smem);
  const uint4* Ys = reinterpret_cast<const uint4*>(smem + ExpandSmem::y);
  float* red = reinterpret_cast<float*>(smem + ExpandSmem::red);
  const float* Vs = reinterpret_cast<const float*>(smem + ExpandSmem::v);
  // this thread's rows of Bᵀ, converted once and reused by every token pass
  constexpr int kRows = 8;
  for (uint32_t t0 = 0; t0 < u.ntok; t0 += kExpandTok) {
    const uint32_t nt = min(kExpandTok, u.ntok - t0);
    float acc[kExpandTok][V::N];
#pragma unroll
    for (int t = 0; t < kExpandTok; ++t)
#pragma unroll
      for (int e = 0; e < V::N; ++e) acc[t][e] = 0.f;
    for (uint32_t j0 = rg; j0 < u.rank; j0 += RG * kRows) {
#pragma unroll
      for (int i = 0; i < kRows; ++i) {
        const uint32_t j = j0 + i * RG;
        if (j < u.rank) {
          float bf[V::N];
          V::unpack(Bs[j * CT + ct], bf);
#pragma unroll
          for (int t = 0; t < kExpandTok; ++t) {
            if (t < nt) {
              const float vt = Vs[(t0 + t) * rp + j];
#pragma unroll
              for (int e = 0; e < V::N; ++e) acc[t][e] = fmaf(vt, bf[e], acc[t][e]);
            }
          }
        }
      }
    }
    if constexpr (RG == 1) {
      if (ct * V::N < u.count) {
#pragma unroll
        for (int t = 0; t < kExpandTok; ++t) {
          if (t < nt) {
            float yv[V::N];
            V::unpack(Ys[(t0 + t) * CT + ct], yv);
#pragma unroll
            for (int e = 0; e < V::N; ++e) yv[e] = fmaf(p.scale, acc[t][e], yv[e]);
            *reinterpret_cast<uint4*>(p.y + u.tok[t0 + t] * p.y_stride_b +
                                      static_cast<uint64_t>(u.off + ct * V::N) * sizeof(T)) =
                V::pack(yv);
          }
        }
      }
    } else {
#pragma unroll
      for (int t = 0; t < kExpandTok; ++t) {
        if (t < nt) {
          float4* dst = reinterpret_cast<float4*>(red + (t * RG + rg) * CB + ct * V::N);
#pragma unroll
          for (int e = 0; e < V::N; e += 4)
            dst[e / 4] = make_float4(acc[t][e], acc[t][e + 1], acc[t][e + 2], acc[t][e + 3]);
        }
      }
      __syncthreads();
      for (uint32_t o = tid; o < nt * CT; o += kThreads) {
        const uint32_t t = o / CT, cc = o - t * CT;
        if (cc * V::N < u.count) {
          float s[V::N];
#pragma unroll
          for (int e = 0; e < V::N; ++e) s[e] = 0.f;
#pragma unroll
          for (int g = 0; g < RG; ++g) {
            const float4* src = reinterpret_cast<const float4*>(red + (t * RG + g) * CB + cc * V::N);
#pragma unroll
            for (int e = 0; e < V::N; e += 4) {
              const float4 q = src[e / 4];
              s[e] += q.x;
              s[e + 1] += q.y;
              s[e + 2] += q.z;
              s[e + 3] += q.w;
            }
          }
          float yv[V::N];
          V::unpack(Ys[(t0 + t) * CT + cc], yv);
#pragma unroll
          for (int e = 0; e < V::N; ++e) yv[e] = fmaf(p.scale, s[e], yv[e]);
          *reinterpret_cast<uint4*>(p.y + u.tok[t0 + t] * p.y_stride_b +
                                    static_cast<uint64_t>(u.off + cc * V::N) * sizeof(T)) =
              V::pack(yv);
        }
      }
      __syncthreads();
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(kThreads) bgmv_expand_kernel(const BgmvArgs p) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t bar;
  const BgmvUnit u = p.units[blockIdx.x];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rg = expand_rg(u.rank);
  const uint32_t cb = (kBgmvConsumers / rg) * (16 / sizeof(T));
  const uint32_t segbytes = u.count * sizeof(T);  // one row's column segment
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  // Bᵀ tile + y rows do not depend on the shrink grid: stream them now.
  if (warp == 0) {
    if (lane == 0) ptx::mbar_arrive_expect_tx(&bar, (u.rank + u.ntok) * segbytes);
    __syncwarp();
    const uint64_t policy = ptx::policy_evict_first();
    const uint64_t bt = (static_cast<uint64_t>(u.rank) * p.blk_mult +
                         static_cast<uint64_t>(u.rank) * p.d_in + u.off) * sizeof(T);
    const uint32_t L = p.log2_page;
    // rows j: [bt + j·d_out·esize, + segbytes), usually one page piece each
    for (uint32_t j = lane; j < u.rank; j += 32) {
      const uint64_t lo = bt + static_cast<uint64_t>(j) * p.d_out * sizeof(T), hi = lo + segbytes;
      for (uint64_t pg = lo >> L; pg <= ((hi - 1) >> L); ++pg) {
        const uint64_t a = max(lo, pg << L), b = min(hi, (pg + 1) << L);
        const uint32_t phys = __ldg(p.table + u.table_off + static_cast<uint32_t>(pg));
        ptx::bulk_g2s_hint(smem + j * cb * sizeof(T) + (a - lo),
                           p.arena + (static_cast<uint64_t>(phys) << L) + (a & ((1ull << L) - 1)),
                           static_cast<uint32_t>(b - a), &bar, policy);
      }
    }
    if (lane < u.ntok)
      ptx::bulk_g2s(smem + ExpandSmem::y + lane * cb * sizeof(T),
                    p.y + u.tok[lane] * p.y_stride_b + static_cast<uint64_t>(u.off) * sizeof(T),
                    segbytes, &bar);
  }
  // v = x·Aᵀ comes from the shrink grid
  pdl_wait();
  {
    const uint32_t rp = rpad4(u.rank);
    float* vs = reinterpret_cast<float*>(smem + ExpandSmem::v);
    for (uint32_t i = threadIdx.x; i < u.ntok * rp; i += kThreads) vs[i] = __ldcg(p.v + u.voff + i);
  }
  ptx::mbar_wait(&bar, 0);
  __syncthreads();
  switch (rg) {
    case 1: expand_compute<T, 1>(p, u, smem); break;
    case 2: expand_compute<T, 2>(p, u, smem); break;
    case 4: expand_compute<T, 4>(p, u, smem); break;
    case 8: expand_compute<T, 8>(p, u, smem); break;
    case 16: expand_compute<T, 16>(p, u, smem); break;
    default: expand_compute<T, 32>(p, u, smem); break;
  }
}

template <typename T>
void launch(const BgmvArgs& a, const ProjWork& pw, const BgmvUnit* d_units, uint32_t shrink_smem,
            cudaStream_t s) {
  set_smem_once(reinterpret_cast<const void*>(bgmv_shrink_kernel<T>), 200 * 1024);
  set_smem_once(reinterpret_cast<const void*>(bgmv_expand_kernel<T>), static_cast<int>(ExpandSmem::total));
  BgmvArgs sa = a;
  sa.units = d_units;
  if (pw.n_shrink) {
    bgmv_shrink_kernel<T><<<pw.n_shrink, kThreads, shrink_smem, s>>>(sa);
    PLORA_CUDA(cudaGetLastError());
    count_launch();
  }
  const uint32_t n_expand = pw.n_units - pw.n_shrink;
  if (n_expand) {
    BgmvArgs ea = a;
    ea.units = d_units + pw.n_shrink;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(n_expand);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = ExpandSmem::total;
    cfg.stream = s;
    cudaLaunchAttribute attrs[1];
    attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 1;
    PLORA_CUDA(cudaLaunchKernelEx(&cfg, bgmv_expand_kernel<T>, ea));
    count_launch();
  }
}

}  // namespace

namespace plora {

void check_io(const plora_plan* plan, uint32_t layer, uint32_t proj, const void* x,
              uint64_t x_stride, void* y, uint64_t y_stride) {
  const ModelGeom& g = plan->store->geom;
  if (layer >= g.m.n_layers) throw ValidationError("layer " + std::to_string(layer) + " out of range");
  if (proj >= g.m.n_proj) throw ValidationError("proj " + std::to_string(proj) + " out of range");
  const uint32_t vec = 16 / g.esize;
  if (x_stride < g.m.d_in[proj] || y_stride < g.m.d_out[proj])
    throw ValidationError("row stride smaller than the projection width");
  if (x_stride % vec || y_stride % vec)
    throw ValidationError("row strides must be multiples of 16 bytes");
  if (plan->n_tokens && (!x || !y)) throw ValidationError("null x or y");
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) % 16)
    throw ValidationError("x and y must be 16-byte aligned");
}

}  // namespace plora

namespace {
int g_hybrid_per_layer = 0;  // plora_debug_set_hybrid_per_layer
// bf16 decode kernel: 0 warp items (bgmv_warp.cu, the default); 1 the
// streaming kernel alone (bgmv_stream.cu); 2 clusters only (bgmv_cluster.cu);
// 3 clusters, and for multi-layer launches the hybrid with a streaming share
// on the SMs the clusters leave idle (the round-2 pair)
int g_bgmv_impl = 0;
}  // namespace

namespace plora {
uint32_t bgmv_impl() { return static_cast<uint32_t>(g_bgmv_impl); }
bool hybrid_enabled() { return g_bgmv_impl == 3; }
double g_hybrid_factor = 0.95;
double hybrid_share_factor() { return g_hybrid_factor; }
}  // namespace plora

namespace plora {
// The hybrid decode launch: the streaming share forks onto the plan's aux
// stream, the clusters run on `stream`, and `stream` joins the aux stream
// (the two shares touch disjoint adapters and y rows).
void launch_hybrid(plora_plan* plan, uint32_t layer0, uint32_t n_layers, const void* x,
                   uint64_t x_stride, uint64_t x_lstride, void* const* ys, const uint64_t* y_strides,
                   const uint64_t* y_lstrides, float scale, cudaStream_t s) {
  if (!plan->aux_stream) {
    PLORA_CUDA(cudaStreamCreateWithFlags(&plan->aux_stream, cudaStreamNonBlocking));
    PLORA_CUDA(cudaEventCreateWithFlags(&plan->ev_fork, cudaEventDisableTiming));
    PLORA_CUDA(cudaEventCreateWithFlags(&plan->ev_join, cudaEventDisableTiming));
  }
  PLORA_CUDA(cudaEventRecord(plan->ev_fork, s));
  PLORA_CUDA(cudaStreamWaitEvent(plan->aux_stream, plan->ev_fork, 0));
  launch_bgmv_cluster_layers(*plan, layer0, n_layers, x, x_stride, x_lstride, ys, y_strides, y_lstrides,
                             scale, s, &plan->cwork_hyb);
  launch_bgmv_stream(*plan, plan->swork_hyb, layer0, n_layers, x, x_stride, x_lstride, ys, y_strides,
                     y_lstrides, scale, plan->aux_stream);
  PLORA_CUDA(cudaEventRecord(plan->ev_join, plan->aux_stream));
  PLORA_CUDA(cudaStreamWaitEvent(s, plan->ev_join, 0));
}
}  // namespace plora

namespace {
// ---- many-token adapters on the tensor-core path (plan.cu: plan->route)
// plora_debug_set_route_tokens.  160: with the warp-item decode kernels the
// routed SGMV side costs ~100 us per layer call however few tiles it has (its
// persistent shrink needs whole SMs, which the decode CTAs hold), so routing
// pays only for adapters of >= ~160 tokens (profiles/r02o_route_warp.txt;
// the cluster kernel's break-even was 48, profiles/r02j_route_sweep.txt).
uint32_t g_route_min = 160;

// xg[i, :] = x[perm[i], :]: the routed tokens' rows, in adapter order
__global__ void route_gather_kernel(const char* __restrict__ x, uint64_t x_stride_b,
                                    const uint32_t* __restrict__ perm, uint32_t n, uint32_t row_v,
                                    uint4* __restrict__ xg) {
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < static_cast<uint64_t>(n) * row_v;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t i = static_cast<uint32_t>(e / row_v), c = static_cast<uint32_t>(e - static_cast<uint64_t>(i) * row_v);
    xg[e] = __ldg(reinterpret_cast<const uint4*>(x + perm[i] * x_stride_b) + c);
  }
}

// y[perm[i], :] = bf16(y + yg[i, :]) for every projection (blockIdx.y): yg
// holds bf16(scale · delta), the value the SGMV expand reduce-adds into y
struct ScatterArgs {
  const uint4* yg[PLORA_MAX_PROJ];
  char* y[PLORA_MAX_PROJ];
  uint64_t y_stride_b[PLORA_MAX_PROJ];
  uint32_t row_v[PLORA_MAX_PROJ];
  const uint32_t* perm;
  uint32_t n;
};
__global__ void route_scatter_kernel(const ScatterArgs a) {
  const uint32_t p = blockIdx.y, row_v = a.row_v[p];
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < static_cast<uint64_t>(a.n) * row_v;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t i = static_cast<uint32_t>(e / row_v), c = static_cast<uint32_t>(e - static_cast<uint64_t>(i) * row_v);
    uint4* yp = reinterpret_cast<uint4*>(a.y[p] + a.perm[i] * a.y_stride_b[p]) + c;
    const uint4 d = a.yg[p][e];
    uint4 v = *yp;
    uint32_t* vw = reinterpret_cast<uint32_t*>(&v);
    const uint32_t* dw = reinterpret_cast<const uint32_t*>(&d);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const __nv_bfloat162 o = __floats2bfloat162_rn(__uint_as_float(vw[k] << 16) + __uint_as_float(dw[k] << 16),
                                                     __uint_as_float(vw[k] & 0xffff0000u) +
                                                         __uint_as_float(dw[k] & 0xffff0000u));
      vw[k] = *reinterpret_cast<const uint32_t*>(&o);
    }
    *yp = v;
  }
}
}  // namespace

namespace plora {
uint32_t route_min_tokens() { return g_route_min; }

// The routed adapters of layers [layer0, layer0 + n_layers), projections
// `projs`, forked onto the plan's route stream: per layer, gather their x
// rows, run the tensor-core SGMV (plora_sgmv / plora_sgmv_layer on the child
// plan) into zeroed bf16 deltas, and add the deltas into their y rows.  The
// caller joins with join_routed after its own launches (the decode kernels
// touch the other tokens' rows only).  Returns false if nothing is routed.
bool launch_routed(plora_plan* plan, uint32_t layer0, uint32_t n_layers, const uint32_t* projs,
                   uint32_t np, const void* x, uint64_t x_stride, uint64_t x_lstride, void* const* ys,
                   const uint64_t* y_strides, const uint64_t* y_lstrides, float scale, cudaStream_t s) {
  if (!plan->route || plan->n_route == 0) return false;
  const ModelGeom& g = plan->store->geom;
  if (!plan->route_stream) {
    PLORA_CUDA(cudaStreamCreateWithFlags(&plan->route_stream, cudaStreamNonBlocking));
    PLORA_CUDA(cudaEventCreateWithFlags(&plan->ev_rfork, cudaEventDisableTiming));
    PLORA_CUDA(cudaEventCreateWithFlags(&plan->ev_rjoin, cudaEventDisableTiming));
  }
  cudaStream_t rs = plan->route_stream;
  PLORA_CUDA(cudaEventRecord(plan->ev_rfork, s));
  PLORA_CUDA(cudaStreamWaitEvent(rs, plan->ev_rfork, 0));
  const uint32_t n = plan->n_route, din = g.m.d_in[projs[0]];
  char* xg = plan->d_route_ws;
  char* yg[PLORA_MAX_PROJ];
  uint64_t ygs[PLORA_MAX_PROJ];
  uint64_t ybytes = 0;
  char* yb = xg + static_cast<uint64_t>(n) * din * 2;
  for (uint32_t j = 0; j < np; ++j) {
    yg[j] = yb + ybytes;
    ygs[j] = g.m.d_out[projs[j]];
    ybytes += static_cast<uint64_t>(n) * g.m.d_out[projs[j]] * 2;
  }
  const uint32_t blocks = std::min<uint32_t>(1024, (n * (din / 8) + 255) / 256);
  for (uint32_t l = 0; l < n_layers; ++l) {
    route_gather_kernel<<<blocks, 256, 0, rs>>>(static_cast<const char*>(x) + l * x_lstride * 2, x_stride * 2,
                                                plan->d_route_perm, n, din / 8, reinterpret_cast<uint4*>(xg));
    PLORA_CUDA(cudaGetLastError());
    count_launch();
    PLORA_CUDA(cudaMemsetAsync(yb, 0, ybytes, rs));
    int rc;
    if (np == g.m.n_proj && np > 1)
      rc = plora_sgmv_layer(plan->route, layer0 + l, xg, din, reinterpret_cast<void* const*>(yg), ygs, scale, rs);
    else
      rc = plora_sgmv(plan->route, layer0 + l, projs[0], xg, din, yg[0], ygs[0], scale, rs);
    if (rc < 0) throw CudaError(std::string("routed SGMV: ") + plora_last_error());
    ScatterArgs sa{};
    uint32_t vmax = 0;
    for (uint32_t j = 0; j < np; ++j) {
      sa.yg[j] = reinterpret_cast<const uint4*>(yg[j]);
      sa.y[j] = static_cast<char*>(ys[j]) + (y_lstrides ? l * y_lstrides[j] * 2 : 0);
      sa.y_stride_b[j] = y_strides[j] * 2;
      sa.row_v[j] = g.m.d_out[projs[j]] / 8;
      vmax = std::max(vmax, sa.row_v[j]);
    }
    sa.perm = plan->d_route_perm;
    sa.n = n;
    route_scatter_kernel<<<dim3(std::min<uint32_t>(1024, (n * vmax + 255) / 256), np), 256, 0, rs>>>(sa);
    PLORA_CUDA(cudaGetLastError());
    count_launch();
  }
  PLORA_CUDA(cudaEventRecord(plan->ev_rjoin, rs));
  return true;
}

void join_routed(plora_plan* plan, cudaStream_t s) {
  PLORA_CUDA(cudaStreamWaitEvent(s, plan->ev_rjoin, 0));
}
}  // namespace plora

extern "C" int plora_debug_set_route_tokens(uint32_t min_tokens) {
  g_route_min = min_tokens;  // plans built afterwards
  return 0;
}

extern "C" int plora_debug_plan_routed(const plora_plan* plan, uint32_t* n_tokens) {
  using namespace plora;
  return guard([&] {
    if (!plan || !n_tokens) throw ValidationError("null plan or n_tokens");
    *n_tokens = plan->route ? plan->n_route : 0u;
    return 0;
  });
}

extern "C" int plora_debug_set_hybrid_per_layer(int on) {
  g_hybrid_per_layer = on;
  return 0;
}

extern "C" int plora_debug_set_hybrid_share(double factor) {
  plora::g_hybrid_factor = factor;  // plans built afterwards
  return 0;
}

extern "C" int plora_debug_plan_hybrid(const plora_plan* plan, double out[4]) {
  using namespace plora;
  return guard([&] {
    if (!plan || !out) throw ValidationError("null plan or out");
    out[0] = plan->hyb_spare;                       // SMs the streaming share runs on (0: none)
    out[1] = plan->hyb_frac;                        // its fraction of the step's weight rows
    out[2] = plan->cwork_hyb.geom.n_clusters;       // clusters of the cluster share
    out[3] = plan->swork_hyb.ctas;                  // CTAs of the streaming share
    return 0;
  });
}

extern "C" int plora_debug_set_bgmv_impl(int impl) {
  g_bgmv_impl = impl;
  return 0;
}

extern "C" int plora_bgmv(plora_plan* plan, uint32_t layer, uint32_t proj, const void* x,
                          uint64_t x_stride, void* y, uint64_t y_stride, float scale,
                          plora_stream_t stream) {
  return guard([&] {
    if (!plan) throw ValidationError("null plan");
    check_io(plan, layer, proj, x, x_stride, y, y_stride);
    const plora_store& st = *plan->store;
    const ModelGeom& g = st.geom;
    const ProjWork& pw = plan->proj[proj];
    DeviceCtx ctx(st.device);
    if (g.esize == 2) {  // bf16: the streaming op (bgmv_stream.cu) or the cluster op
      cudaStream_t s = static_cast<cudaStream_t>(stream);
      void* ys[1] = {y};
      const uint64_t yst[1] = {y_stride};
      const bool routed = launch_routed(plan, layer, 1, &proj, 1, x, x_stride, 0, ys, yst, nullptr, scale, s);
      if (g_bgmv_impl == 0)
        launch_bgmv_warp(*plan, plan->wwork[proj], layer, 1, x, x_stride, 0, ys, yst, nullptr, scale, s);
      else if (g_bgmv_impl != 1)
        launch_bgmv_cluster(*plan, layer, proj, x, x_stride, y, y_stride, scale, s);
      else
        launch_bgmv_stream(*plan, plan->swork[proj], layer, 1, x, x_stride, 0, ys, yst, nullptr, scale, s);
      if (routed) join_routed(plan, s);
      return 0;
    }
    if (pw.n_units == 0) return 0;  // no LoRA token in the batch
    BgmvArgs a{};
    a.arena = st.arena;
    a.table = st.d_table;
    a.v = plan->d_v;
    a.x = static_cast<const char*>(x);
    a.y = static_cast<char*>(y);
    a.x_stride_b = x_stride * g.esize;
    a.y_stride_b = y_stride * g.esize;
    a.blk_mult = g.blk_mult(layer, proj);
    a.log2_page = st.log2_page;
    a.d_in = g.m.d_in[proj];
    a.d_out = g.m.d_out[proj];
    a.scale = scale;
    const uint32_t rowbytes = a.d_in * g.esize;
    const uint32_t rpu = std::min<uint32_t>(kMaxShrinkRows, kShrinkWeightBytes / rowbytes);
    const uint32_t nts = std::min<uint32_t>(kMaxUnitTok, kSlotAuxBytes / rowbytes);
    const uint32_t shrink_smem = (rpu + nts) * rowbytes;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const BgmvUnit* units = plan->d_units + pw.units_off;
    launch<float>(a, pw, units, shrink_smem, s);
    return 0;
  });
}

extern "C" int plora_bgmv_layers(plora_plan* plan, uint32_t layer0, uint32_t n_layers,
                                 const void* x, uint64_t x_stride, uint64_t x_layer_stride,
                                 void* const* ys, const uint64_t* y_strides,
                                 const uint64_t* y_layer_strides, float scale,
                                 plora_stream_t stream) {
  return guard([&] {
    if (!plan) throw ValidationError("null plan");
    if (!ys || !y_strides || !y_layer_strides) throw ValidationError("null ys / strides");
    if (n_layers == 0) return 0;
    const plora_store& st = *plan->store;
    const ModelGeom& g = st.geom;
    if (layer0 + static_cast<uint64_t>(n_layers) > g.m.n_layers)
      throw ValidationError("layers [" + std::to_string(layer0) + ", " +
                            std::to_string(layer0 + n_layers) + ") out of range");
    const uint32_t vec = 16 / g.esize;
    if (x_layer_stride % vec) throw ValidationError("layer strides must be multiples of 16 bytes");
    for (uint32_t p = 0; p < g.m.n_proj; ++p) {
      if (g.m.d_in[p] != g.m.d_in[0])
        throw ValidationError("plora_bgmv_layers: projections read different input widths");
      if (y_layer_strides[p] % vec) throw ValidationError("layer strides must be multiples of 16 bytes");
      check_io(plan, layer0, p, x, x_stride, ys[p], y_strides[p]);
    }
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    uint32_t all[PLORA_MAX_PROJ];
    for (uint32_t p = 0; p < g.m.n_proj; ++p) all[p] = p;
    auto routed = [&] {
      return launch_routed(plan, layer0, n_layers, all, g.m.n_proj, x, x_stride, x_layer_stride, ys,
                           y_strides, y_layer_strides, scale, s);
    };
    if (g.esize == 2 && g_bgmv_impl == 0 && plan->wwork_layer.np == g.m.n_proj) {
      DeviceCtx ctx(st.device);
      const bool r = routed();
      launch_bgmv_warp(*plan, plan->wwork_layer, layer0, n_layers, x, x_stride, x_layer_stride, ys,
                       y_strides, y_layer_strides, scale, s);
      if (r) join_routed(plan, s);
      return 0;
    }
    if (g.esize == 2 && g_bgmv_impl == 1 && plan->swork_layer.np == g.m.n_proj) {
      DeviceCtx ctx(st.device);
      const bool r = routed();
      launch_bgmv_stream(*plan, plan->swork_layer, layer0, n_layers, x, x_stride, x_layer_stride,
                         ys, y_strides, y_layer_strides, scale, s);
      if (r) join_routed(plan, s);
      return 0;
    }
    if (g.esize == 2 && g_bgmv_impl == 3 && plan->hyb_spare && plan->n_layer_proj == g.m.n_proj &&
        n_layers * g.m.n_proj <= 256) {
      DeviceCtx ctx(st.device);
      const bool r = routed();
      launch_hybrid(plan, layer0, n_layers, x, x_stride, x_layer_stride, ys, y_strides, y_layer_strides,
                    scale, s);
      if (r) join_routed(plan, s);
      return 0;
    }
    const bool one = g.esize == 2 && plan->n_layer_proj == g.m.n_proj &&
                     n_layers * g.m.n_proj <= 256;
    if (one) {
      DeviceCtx ctx(st.device);
      const bool r = routed();
      launch_bgmv_cluster_layers(*plan, layer0, n_layers, x, x_stride, x_layer_stride, ys,
                                 y_strides, y_layer_strides, scale, s);
      if (r) join_routed(plan, s);
      return 0;
    }
    std::vector<void*> yl(g.m.n_proj);
    for (uint32_t i = 0; i < n_layers; ++i) {
      for (uint32_t p = 0; p < g.m.n_proj; ++p)
        yl[p] = static_cast<char*>(ys[p]) + i * y_layer_strides[p] * g.esize;
      const int rc = plora_bgmv_layer(plan, layer0 + i, static_cast<const char*>(x) + i * x_layer_stride * g.esize,
                                      x_stride, yl.data(), y_strides, scale, stream);
      if (rc < 0) return rc;
    }
    return 0;
  });
}

extern "C" int plora_bgmv_layer(plora_plan* plan, uint32_t layer, const void* x,
                                uint64_t x_stride, void* const* ys, const uint64_t* y_strides,
                                float scale, plora_stream_t stream) {
  return guard([&] {
    if (!plan) throw ValidationError("null plan");
    if (!ys || !y_strides) throw ValidationError("null ys or y_strides");
    const plora_store& st = *plan->store;
    const ModelGeom& g = st.geom;
    for (uint32_t p = 0; p < g.m.n_proj; ++p) {
      if (g.m.d_in[p] != g.m.d_in[0])
        throw ValidationError("plora_bgmv_layer: projections read different input widths");
      check_io(plan, layer, p, x, x_stride, ys[p], y_strides[p]);
    }
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    uint32_t all[PLORA_MAX_PROJ];
    for (uint32_t p = 0; p < g.m.n_proj; ++p) all[p] = p;
    auto routed = [&] {
      return launch_routed(plan, layer, 1, all, g.m.n_proj, x, x_stride, 0, ys, y_strides, nullptr, scale, s);
    };
    if (g.esize == 2 && g_bgmv_impl == 0 && plan->wwork_layer.np == g.m.n_proj) {
      DeviceCtx ctx(st.device);
      const bool r = routed();
      launch_bgmv_warp(*plan, plan->wwork_layer, layer, 1, x, x_stride, 0, ys, y_strides, nullptr, scale, s);
      if (r) join_routed(plan, s);
      return 0;
    }
    if (g.esize == 2 && g_bgmv_impl == 1 && plan->swork_layer.np == g.m.n_proj) {
      DeviceCtx ctx(st.device);
      const uint64_t zero[PLORA_MAX_PROJ] = {};
      const bool r = routed();
      launch_bgmv_stream(*plan, plan->swork_layer, layer, 1, x, x_stride, 0, ys, y_strides, zero, scale, s);
      if (r) join_routed(plan, s);
      return 0;
    }
    if (g.esize == 2 && g_bgmv_impl == 3 && g_hybrid_per_layer && plan->hyb_spare &&
        plan->n_layer_proj == g.m.n_proj) {
      DeviceCtx ctx(st.device);
      const uint64_t zero[PLORA_MAX_PROJ] = {};
      const bool r = routed();
      launch_hybrid(plan, layer, 1, x, x_stride, 0, ys, y_strides, zero, scale, s);
      if (r) join_routed(plan, s);
      return 0;
    }
    if (g.esize == 2 && plan->n_layer_proj == g.m.n_proj) {
      DeviceCtx ctx(st.device);
      const bool r = routed();
      launch_bgmv_cluster_layer(*plan, layer, x, x_stride, ys, y_strides, scale, s);
      if (r) join_routed(plan, s);
      return 0;
    }
    for (uint32_t p = 0; p < g.m.n_proj; ++p) {  // shapes differ: one launch per projection
      const int rc = plora_bgmv(plan, layer, p, x, x_stride, ys[p], y_strides[p], scale, stream);
      if (rc < 0) return rc;
    }
    return 0;
  });
}
