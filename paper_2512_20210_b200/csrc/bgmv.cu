// Paged multi-LoRA decode op (gathered BGMV) for sm_100a, plus the batch
// plan it runs from.
//
// y[t, :] += scale · (x[t, :] · A_{a(t)}ᵀ) · B_{a(t)}ᵀ
//
// The reference only bills this op as a cost-model constant
// (include/lorasim/cost_model.hpp:32-40, billed at src/engine.cpp:355,510);
// the weights are read straight out of the paged arena through the device
// page table (PagePool::translate semantics, src/memory.cpp:55-62).
//
// Design (HBM-bound, AI ≈ 1.8 flop/B at Llama-7B decode shapes):
//  * One persistent kernel per (layer, proj) call, grid = SMs × occupancy,
//    pulling work units from an atomic ticket.  Units are equal-byte slices:
//      shrink (segment, 8 rank rows): one warp per row of A streams d_in
//        elements with 16-byte loads (16 in flight per lane), dots them with
//        the segment's x rows staged in shared memory, warp-shuffle reduces
//        and writes v (fp32) to an L2-resident workspace;
//      expand (segment, column block): each thread holds <= 4 rank rows of
//        Bᵀ for 8 (bf16) output columns, loaded BEFORE waiting on the
//        segment's shrink counter, then reduces across row groups in shared
//        memory and read-modify-writes y once.
//    All shrink units precede all expand units in ticket order, so an expand
//    unit only ever waits on units already held by running CTAs — no
//    deadlock regardless of residency.  The last CTA out resets the ticket
//    and counters, so the launch is graph-capturable.
//  * Each adapter's weights are read exactly once per call regardless of how
//    many of its tokens are in the batch (tokens are grouped by adapter).
//  * Page lookups: one __ldg of the page table per 16-byte vector (L1-hot;
//    4 B per page of weights).
#include <cuda_bf16.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <numeric>

#include "plan.hpp"

using namespace plora;

namespace {

constexpr uint32_t kTokChunk = 4;   // tokens per shared-memory chunk (shrink)
constexpr uint32_t kExpTok = 2;     // tokens per accumulation chunk (expand)
constexpr int kShrinkVecs = 8;      // 16-byte loads in flight per lane (shrink)
constexpr int kExpandRows = 4;      // Bᵀ rows held per thread (expand)

struct BgmvArgs {
  const char* arena;
  const uint32_t* table;
  const SegDesc* segs;
  const uint32_t* toks;
  const uint2* units;
  float* v;
  uint32_t* sync;  // [0] ticket, [1] exit, [2 + s] shrink-done of segment s
  const void* x;
  void* y;
  uint64_t x_stride;
  uint64_t y_stride;
  uint64_t blk_mult;  // block (layer, proj) starts at element rank · blk_mult
  uint32_t log2_page;
  uint32_t n_units;
  uint32_t n_seg;
  uint32_t d_in;
  uint32_t d_out;
  float scale;
};

__device__ __forceinline__ uint4 ld_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Address of logical byte `off` of an adapter through its page table.
__device__ __forceinline__ const uint4* paged(const BgmvArgs& p, uint32_t table_off,
                                              uint64_t off) {
  const uint32_t phys = __ldg(p.table + table_off + static_cast<uint32_t>(off >> p.log2_page));
  return reinterpret_cast<const uint4*>(p.arena + (static_cast<uint64_t>(phys) << p.log2_page) +
                                        (off & ((1ull << p.log2_page) - 1)));
}

template <typename T>
struct VecOps;

template <>
struct VecOps<__nv_bfloat16> {
  static constexpr int N = 8;
  __device__ static __forceinline__ float dot(const uint4& a, const uint4& b) {
    const __nv_bfloat162* pa = reinterpret_cast<const __nv_bfloat162*>(&a);
    const __nv_bfloat162* pb = reinterpret_cast<const __nv_bfloat162*>(&b);
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 fa = __bfloat1622float2(pa[i]);
      float2 fb = __bfloat1622float2(pb[i]);
      s = fmaf(fa.x, fb.x, s);
      s = fmaf(fa.y, fb.y, s);
    }
    return s;
  }
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
  __device__ static __forceinline__ float dot(const uint4& a, const uint4& b) {
    float s = __uint_as_float(a.x) * __uint_as_float(b.x);
    s = fmaf(__uint_as_float(a.y), __uint_as_float(b.y), s);
    s = fmaf(__uint_as_float(a.z), __uint_as_float(b.z), s);
    s = fmaf(__uint_as_float(a.w), __uint_as_float(b.w), s);
    return s;
  }
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

// ---------------------------------------------------------------- shrink
template <typename T>
__device__ void shrink_unit(const BgmvArgs& p, const SegDesc& sd, uint32_t seg, uint32_t j0,
                            char* smem) {
  using V = VecOps<T>;
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t j = j0 + warp;
  const bool active = j < sd.rank;  // warp-uniform
  const uint32_t nvec = p.d_in / V::N;
  uint4* xs = reinterpret_cast<uint4*>(smem);
  const uint64_t row_byte =
      (static_cast<uint64_t>(sd.rank) * p.blk_mult + static_cast<uint64_t>(j) * p.d_in) * sizeof(T);

  for (uint32_t tc = 0; tc < sd.n_tok; tc += kTokChunk) {
    const uint32_t nch = min(kTokChunk, sd.n_tok - tc);
    // the weight loads do not depend on x: issue them first
    uint4 w[kShrinkVecs];
    float acc[kTokChunk];
#pragma unroll
    for (uint32_t t = 0; t < kTokChunk; ++t) acc[t] = 0.f;
    uint32_t c0 = lane;
    if (active) {
#pragma unroll
      for (int g = 0; g < kShrinkVecs; ++g) {
        const uint32_t c = c0 + 32u * g;
        if (c < nvec) w[g] = ld_stream(paged(p, sd.table_off, row_byte + 16ull * c));
      }
    }
    for (uint32_t i = threadIdx.x; i < nch * nvec; i += blockDim.x) {
      const uint32_t t = i / nvec, c = i - t * nvec;
      const uint32_t tok = p.toks[sd.tok_start + tc + t];
      xs[t * nvec + c] = __ldg(reinterpret_cast<const uint4*>(static_cast<const T*>(p.x) +
                                                              tok * p.x_stride) + c);
    }
    __syncthreads();
    if (active) {
      while (true) {
#pragma unroll
        for (int g = 0; g < kShrinkVecs; ++g) {
          const uint32_t c = c0 + 32u * g;
          if (c < nvec) {
#pragma unroll
            for (uint32_t t = 0; t < kTokChunk; ++t)
              if (t < nch) acc[t] += V::dot(w[g], xs[t * nvec + c]);
          }
        }
        c0 += 32u * kShrinkVecs;
        if (c0 >= nvec) break;
#pragma unroll
        for (int g = 0; g < kShrinkVecs; ++g) {
          const uint32_t c = c0 + 32u * g;
          if (c < nvec) w[g] = ld_stream(paged(p, sd.table_off, row_byte + 16ull * c));
        }
      }
#pragma unroll
      for (uint32_t t = 0; t < kTokChunk; ++t) {
        float a = acc[t];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        acc[t] = a;
      }
      if (lane == 0) {
        for (uint32_t t = 0; t < nch; ++t)
          p.v[sd.voff + (tc + t) * sd.rank + j] = acc[t];
        __threadfence();
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(p.sync + 2 + seg, 1u);
  }
}

// ---------------------------------------------------------------- expand
template <typename T, int RG>
__device__ void expand_unit(const BgmvArgs& p, const SegDesc& sd, uint32_t seg, uint32_t c0,
                            char* smem) {
  using V = VecOps<T>;
  constexpr int CT = kThreads / RG;  // column threads
  constexpr int CB = CT * V::N;      // columns per unit
  const uint32_t rg = threadIdx.x / CT, ct = threadIdx.x % CT;
  const uint32_t col = c0 + ct * V::N;
  const bool col_ok = col < p.d_out;
  const uint32_t r = sd.rank;
  const uint64_t bt_byte =
      (static_cast<uint64_t>(r) * p.blk_mult + static_cast<uint64_t>(r) * p.d_in) * sizeof(T);
  const uint32_t n_i = rg < r ? (r - rg + RG - 1) / RG : 0;  // rows j = rg + RG·i

  uint4 b[kExpandRows];
#define PLORA_LOAD_ROWS(i0)                                                                  \
  _Pragma("unroll") for (int e = 0; e < kExpandRows; ++e) {                                  \
    const uint32_t i_ = (i0) + e;                                                            \
    if (col_ok && i_ < n_i) {                                                                \
      const uint32_t jj = rg + RG * i_;                                                      \
      b[e] = ld_stream(paged(p, sd.table_off,                                                \
                             bt_byte + (static_cast<uint64_t>(jj) * p.d_out + col) * sizeof(T))); \
    }                                                                                        \
  }
  PLORA_LOAD_ROWS(0u)  // Bᵀ does not depend on v: prefetch before waiting

  if (threadIdx.x == 0) {
    const uint32_t* flag = p.sync + 2 + seg;
    while (ld_acquire(flag) < sd.n_shrink) __nanosleep(32);
  }
  __syncthreads();

  float* vs = reinterpret_cast<float*>(smem);  // [kExpTok][r]
  float* red = vs + ((kExpTok * r + 3) & ~3u);  // [RG][kExpTok][CB]
  bool first = true;
  for (uint32_t tc = 0; tc < sd.n_tok; tc += kExpTok) {
    const uint32_t nch = min(kExpTok, sd.n_tok - tc);
    for (uint32_t i = threadIdx.x; i < nch * r; i += blockDim.x)
      vs[i] = __ldcg(p.v + sd.voff + tc * r + i);
    __syncthreads();
    float acc[kExpTok][V::N];
#pragma unroll
    for (uint32_t t = 0; t < kExpTok; ++t)
#pragma unroll
      for (int k = 0; k < V::N; ++k) acc[t][k] = 0.f;
    for (uint32_t i0 = 0; i0 < n_i; i0 += kExpandRows) {
      if (!first) { PLORA_LOAD_ROWS(i0) }
      first = false;
#pragma unroll
      for (int e = 0; e < kExpandRows; ++e) {
        const uint32_t i = i0 + e;
        if (i < n_i) {
          const uint32_t jj = rg + RG * i;
          float bf[V::N];
          V::unpack(b[e], bf);
#pragma unroll
          for (uint32_t t = 0; t < kExpTok; ++t) {
            if (t < nch) {
              const float vt = vs[t * r + jj];
#pragma unroll
              for (int k = 0; k < V::N; ++k) acc[t][k] = fmaf(vt, bf[k], acc[t][k]);
            }
          }
        }
      }
    }
    first = false;
    // partial sums of this row group
#pragma unroll
    for (uint32_t t = 0; t < kExpTok; ++t) {
      float4* dst = reinterpret_cast<float4*>(red + (rg * kExpTok + t) * CB + ct * V::N);
#pragma unroll
      for (int k = 0; k < V::N; k += 4)
        dst[k / 4] = make_float4(acc[t][k], acc[t][k + 1], acc[t][k + 2], acc[t][k + 3]);
    }
    __syncthreads();
    for (uint32_t o = threadIdx.x; o < nch * CT; o += blockDim.x) {
      const uint32_t t = o / CT, cc = o - t * CT;
      const uint32_t colo = c0 + cc * V::N;
      if (colo < p.d_out) {
        float sum[V::N];
#pragma unroll
        for (int k = 0; k < V::N; ++k) sum[k] = 0.f;
#pragma unroll
        for (int g = 0; g < RG; ++g) {
          const float4* src =
              reinterpret_cast<const float4*>(red + (g * kExpTok + t) * CB + cc * V::N);
#pragma unroll
          for (int k = 0; k < V::N; k += 4) {
            float4 q = src[k / 4];
            sum[k] += q.x;
            sum[k + 1] += q.y;
            sum[k + 2] += q.z;
            sum[k + 3] += q.w;
          }
        }
        const uint32_t tok = p.toks[sd.tok_start + tc + t];
        uint4* yp = reinterpret_cast<uint4*>(static_cast<T*>(p.y) + tok * p.y_stride + colo);
        float yv[V::N];
        V::unpack(*yp, yv);
#pragma unroll
        for (int k = 0; k < V::N; ++k) yv[k] = fmaf(p.scale, sum[k], yv[k]);
        *yp = V::pack(yv);
      }
    }
    __syncthreads();
  }
#undef PLORA_LOAD_ROWS
}

template <typename T>
__global__ void __launch_bounds__(kThreads, 2) bgmv_paged_kernel(const BgmvArgs p) {
  extern __shared__ __align__(16) char smem[];
  __shared__ uint32_t s_unit;
  __shared__ uint32_t s_last;
  while (true) {
    if (threadIdx.x == 0) s_unit = atomicAdd(p.sync, 1u);
    __syncthreads();
    const uint32_t u = s_unit;
    __syncthreads();
    if (u >= p.n_units) break;
    const uint2 un = p.units[u];
    const uint32_t seg = un.x & ~kExpandBit;
    const SegDesc sd = p.segs[seg];
    if (!(un.x & kExpandBit)) {
      shrink_unit<T>(p, sd, seg, un.y, smem);
    } else {
      switch (expand_rg(sd.rank)) {
        case 4: expand_unit<T, 4>(p, sd, seg, un.y, smem); break;
        case 8: expand_unit<T, 8>(p, sd, seg, un.y, smem); break;
        case 16: expand_unit<T, 16>(p, sd, seg, un.y, smem); break;
        default: expand_unit<T, 32>(p, sd, seg, un.y, smem); break;
      }
    }
  }
  // last CTA out resets the ticket and the per-segment counters
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(p.sync + 1, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    for (uint32_t i = threadIdx.x; i < p.n_seg; i += blockDim.x) p.sync[2 + i] = 0;
    if (threadIdx.x == 0) {
      p.sync[0] = 0;
      p.sync[1] = 0;
    }
  }
}

// Occupancy cache: (kernel, smem) -> resident CTAs per SM.
int blocks_per_sm(const void* fn, uint32_t smem) {
  static std::map<std::pair<const void*, uint32_t>, int> cache;
  auto key = std::make_pair(fn, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  static std::map<const void*, uint32_t> attr_set;
  if (smem > 48 * 1024 && attr_set[fn] < smem) {
    PLORA_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
    attr_set[fn] = smem;
  }
  int n = 0;
  PLORA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, kThreads, smem));
  cache[key] = std::max(n, 1);
  return cache[key];
}

uint32_t expand_cols(uint32_t rank, uint32_t esize) {
  return (kThreads / expand_rg(rank)) * (16 / esize);
}

}  // namespace

// ------------------------------------------------------------------ plan
void plora_plan::build(const int32_t* token_adapter, uint32_t n, cudaStream_t stream) {
  const plora_store& st = *store;
  const ModelGeom& g = st.geom;
  // group tokens by adapter: validate residency first (host shadow)
  std::vector<uint32_t> count;
  count.assign(st.max_adapters, 0);
  for (uint32_t t = 0; t < n; ++t) {
    const int32_t a = token_adapter[t];
    if (a < 0) continue;
    if (static_cast<uint32_t>(a) >= st.max_adapters)
      throw ValidationError("token " + std::to_string(t) + " names adapter " + std::to_string(a) +
                            " >= max_adapters");
    if (!st.slots[a].published)
      throw ValidationError("token " + std::to_string(t) + " names adapter " + std::to_string(a) +
                            " which is not resident (publish it first)");
    ++count[a];
  }
  segs.clear();
  toks.assign(n, 0);
  std::vector<uint32_t> cursor(st.max_adapters, 0);
  uint32_t pos = 0;
  max_rank = 0;
  v_elems = 0;
  for (uint32_t a = 0; a < st.max_adapters; ++a) {
    if (!count[a]) continue;
    SegDesc sd{};
    sd.table_off = st.h_dir[a].table_off;
    sd.rank = st.h_dir[a].rank;
    sd.tok_start = pos;
    sd.n_tok = count[a];
    sd.voff = static_cast<uint32_t>(v_elems);
    sd.n_shrink = (sd.rank + kShrinkRows - 1) / kShrinkRows;
    sd.adapter = a;
    cursor[a] = pos;
    pos += count[a];
    v_elems += static_cast<uint64_t>(sd.n_tok) * sd.rank;
    max_rank = std::max(max_rank, sd.rank);
    segs.push_back(sd);
  }
  if (v_elems > 0xffffffffull) throw ValidationError("batch too large for one plan");
  for (uint32_t t = 0; t < n; ++t)
    if (token_adapter[t] >= 0) toks[cursor[token_adapter[t]]++] = t;
  toks.resize(pos);
  n_tokens = n;
  n_seg = static_cast<uint32_t>(segs.size());

  // segment order for scheduling: largest rank first (longest dependency
  // chains start earliest), ties by adapter key
  std::vector<uint32_t> order(n_seg);
  std::iota(order.begin(), order.end(), 0u);
  std::stable_sort(order.begin(), order.end(),
                   [&](uint32_t x, uint32_t y) { return segs[x].rank > segs[y].rank; });

  units.clear();
  for (uint32_t p = 0; p < g.m.n_proj; ++p) {
    ProjUnits& pu = proj[p];
    pu.units_off = static_cast<uint32_t>(units.size());
    for (uint32_t s : order)
      for (uint32_t j0 = 0; j0 < segs[s].rank; j0 += kShrinkRows) units.push_back(make_uint2(s, j0));
    for (uint32_t s : order) {
      const uint32_t cb = expand_cols(segs[s].rank, g.esize);
      for (uint32_t c0 = 0; c0 < g.m.d_out[p]; c0 += cb) units.push_back(make_uint2(s | kExpandBit, c0));
    }
    pu.n_units = static_cast<uint32_t>(units.size()) - pu.units_off;
    // shared memory: max(shrink x staging, expand v + reduction)
    const uint32_t shrink_smem = kTokChunk * g.m.d_in[p] * g.esize;
    // expand: v chunk [kExpTok][max_rank] + partials [RG][kExpTok][CB] floats,
    // and RG · CB = kThreads · (16 / esize) for every rank
    const uint32_t expand_smem =
        (((kExpTok * max_rank + 3) & ~3u) + kExpTok * kThreads * (16 / g.esize)) * 4;
    pu.smem = std::max(shrink_smem, expand_smem);
  }

  // pack segs | toks | units into one pinned buffer and upload once
  auto align = [](uint64_t v) { return (v + 255) & ~255ull; };
  const uint64_t seg_b = align(segs.size() * sizeof(SegDesc));
  const uint64_t tok_b = align(toks.size() * sizeof(uint32_t));
  const uint64_t unit_b = align(units.size() * sizeof(uint2));
  const uint64_t total = std::max<uint64_t>(seg_b + tok_b + unit_b, 256);
  DeviceCtx ctx(st.device);
  if (upload_done) PLORA_CUDA(cudaEventSynchronize(upload_done));  // pinned buffer reuse
  if (h_cap < total) {
    if (h_pinned) cudaFreeHost(h_pinned);
    h_pinned = nullptr;
    PLORA_CUDA(cudaMallocHost(&h_pinned, total));
    h_cap = total;
  }
  if (d_cap < total) {
    if (d_buf) {
      PLORA_CUDA(cudaStreamSynchronize(stream));
      cudaFree(d_buf);
    }
    d_buf = nullptr;
    PLORA_CUDA(cudaMalloc(&d_buf, total));
    d_cap = total;
  }
  std::memcpy(h_pinned, segs.data(), segs.size() * sizeof(SegDesc));
  std::memcpy(h_pinned + seg_b, toks.data(), toks.size() * sizeof(uint32_t));
  std::memcpy(h_pinned + seg_b + tok_b, units.data(), units.size() * sizeof(uint2));
  d_segs = reinterpret_cast<SegDesc*>(d_buf);
  d_toks = reinterpret_cast<uint32_t*>(d_buf + seg_b);
  d_units = reinterpret_cast<uint2*>(d_buf + seg_b + tok_b);
  PLORA_CUDA(cudaMemcpyAsync(d_buf, h_pinned, seg_b + tok_b + unit_b, cudaMemcpyHostToDevice,
                             stream));
  if (!upload_done) PLORA_CUDA(cudaEventCreateWithFlags(&upload_done, cudaEventDisableTiming));
  PLORA_CUDA(cudaEventRecord(upload_done, stream));

  if (v_cap < std::max<uint64_t>(v_elems, 1)) {
    if (d_v) {
      PLORA_CUDA(cudaStreamSynchronize(stream));
      cudaFree(d_v);
    }
    d_v = nullptr;
    v_cap = std::max<uint64_t>(v_elems, 1024);
    PLORA_CUDA(cudaMalloc(&d_v, v_cap * sizeof(float)));
  }
  if (sync_cap < 2ull + n_seg) {
    if (d_sync) {
      PLORA_CUDA(cudaStreamSynchronize(stream));
      cudaFree(d_sync);
    }
    d_sync = nullptr;
    sync_cap = std::max<uint64_t>(2ull + n_seg, 1024);
    PLORA_CUDA(cudaMalloc(&d_sync, sync_cap * sizeof(uint32_t)));
    PLORA_CUDA(cudaMemsetAsync(d_sync, 0, sync_cap * sizeof(uint32_t), stream));
  }
}

namespace {

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

}  // namespace

extern "C" {

int plora_plan_create(plora_store* s, const int32_t* token_adapter, uint32_t n_tokens,
                      plora_stream_t stream, plora_plan** out) {
  return guard([&] {
    if (!s) throw ValidationError("null store");
    if (n_tokens && !token_adapter) throw ValidationError("null token_adapter");
    auto plan = std::make_unique<plora_plan>();
    plan->store = s;
    plan->build(token_adapter, n_tokens, static_cast<cudaStream_t>(stream));
    *out = plan.release();
    return 0;
  });
}

int plora_plan_update(plora_plan* plan, const int32_t* token_adapter, uint32_t n_tokens,
                      plora_stream_t stream) {
  return guard([&] {
    if (!plan) throw ValidationError("null plan");
    if (n_tokens && !token_adapter) throw ValidationError("null token_adapter");
    plan->build(token_adapter, n_tokens, static_cast<cudaStream_t>(stream));
    return 0;
  });
}

void plora_plan_destroy(plora_plan* plan) {
  if (!plan) return;
  DeviceCtx ctx(plan->store->device);
  if (plan->upload_done) {
    cudaEventSynchronize(plan->upload_done);
    cudaEventDestroy(plan->upload_done);
  }
  cudaDeviceSynchronize();
  cudaFreeHost(plan->h_pinned);
  cudaFree(plan->d_buf);
  cudaFree(plan->d_v);
  cudaFree(plan->d_sync);
  delete plan;
}

uint32_t plora_plan_num_segments(const plora_plan* plan) { return plan ? plan->n_seg : 0; }

int plora_bgmv(plora_plan* plan, uint32_t layer, uint32_t proj, const void* x,
               uint64_t x_stride, void* y, uint64_t y_stride, float scale,
               plora_stream_t stream) {
  return guard([&] {
    if (!plan) throw ValidationError("null plan");
    check_io(plan, layer, proj, x, x_stride, y, y_stride);
    const plora_store& st = *plan->store;
    const ModelGeom& g = st.geom;
    const ProjUnits& pu = plan->proj[proj];
    if (pu.n_units == 0) return 0;
    DeviceCtx ctx(st.device);
    BgmvArgs a{};
    a.arena = st.arena;
    a.table = st.d_table;
    a.segs = plan->d_segs;
    a.toks = plan->d_toks;
    a.units = plan->d_units + pu.units_off;
    a.v = plan->d_v;
    a.sync = plan->d_sync;
    a.x = x;
    a.y = y;
    a.x_stride = x_stride;
    a.y_stride = y_stride;
    a.blk_mult = g.blk_mult(layer, proj);
    a.log2_page = st.log2_page;
    a.n_units = pu.n_units;
    a.n_seg = plan->n_seg;
    a.d_in = g.m.d_in[proj];
    a.d_out = g.m.d_out[proj];
    a.scale = scale;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const void* fn = g.esize == 2 ? reinterpret_cast<const void*>(bgmv_paged_kernel<__nv_bfloat16>)
                                  : reinterpret_cast<const void*>(bgmv_paged_kernel<float>);
    const int per_sm = blocks_per_sm(fn, pu.smem);
    const uint32_t grid = std::min<uint32_t>(pu.n_units, static_cast<uint32_t>(per_sm * st.num_sms));
    if (g.esize == 2) {
      bgmv_paged_kernel<__nv_bfloat16><<<grid, kThreads, pu.smem, s>>>(a);
    } else {
      bgmv_paged_kernel<float><<<grid, kThreads, pu.smem, s>>>(a);
    }
    PLORA_CUDA(cudaGetLastError());
    count_launch();
    return 0;
  });
}

}  // extern "C"
