// bf16 paged BGMV (decode), warp-item design: the default hot path behind
// plora_bgmv / plora_bgmv_layer / plora_bgmv_layers for bf16 stores.
//
//   y[t, :] += scale · (x[t, :] · A_{a(t)}ᵀ) · B_{a(t)}ᵀ
//
// every A / Bᵀ row read straight out of the page arena through the device
// page table (the translation PagePool::translate does on the host,
// src/memory.cpp:55-62).
//
// Decode is a pure weight stream (arithmetic intensity ~2 flop/byte at two
// tokens per adapter), so the design is the one that streams best: every
// warp runs one self-contained work item; each lane copies its own 16-byte
// pieces of the paged rows with cp.async into its own slots of a per-warp
// ring in shared memory and reads back exactly those bytes — no clusters, no
// cross-warp barriers (except the two warps of a split pair), no cross-CTA
// waits.  Two launches per call, chained by programmatic dependent launch:
//   shrink  S items (<= 8 rank rows of one job, one K slice of <= 4096):
//           v[tok][row] = Σ_k x[tok][k] · A[row][k], exact fp32
//           (FHFMA: bf16 × bf16 + fp32, one rounding per term, no converts);
//           lane partials summed by a fixed butterfly -> deterministic.
//           Single-layer calls also stream x through the ring.
//   expand  E items (one block of <= 512 output columns, every rank row):
//           acc[tok][col] = Σ_row v[tok][row] · Bᵀ[row][col] in row order
//           (FFMA2 on converted weight pairs), then y = bf16(y + scale·acc).
//           Single-layer calls issue the first Bᵀ rows before the dependency
//           wait and split rank >= 64 items over a CTA's two warps (partials
//           added in fixed order).
// The launch boundary orders v (the expand's griddepcontrol.wait).  A
// multi-layer launch (plora_bgmv_layers) is the same item list repeated per
// layer.  The tensor-parallel halves (tp.cu) run on the same items in a TP
// mode: K-sliced shrink items with per-job in-order partial sums, column-
// shard expand items reading the gathered v.
// Measured at cfg2 (profiles/r02n_*, r02o_*): the 32-layer step at 1.00-1.01
// of the HBM copy peak, one layer per call 0.647 (latency-bound phases).
#include <cuda_bf16.h>

#include "plan.hpp"
#include "ptx.cuh"

namespace plora {
namespace {

#ifndef PLORA_WARP_CTA
#define PLORA_WARP_CTA 2  // warps (work items) per CTA
#endif
constexpr uint32_t kWarps = PLORA_WARP_CTA;
static_assert(kWarps % 2 == 0, "split E pairs are the two warps (2c, 2c + 1) of a CTA");
#define PLORA_WARP_MINB (16 / PLORA_WARP_CTA)  // 16 warps per SM: <= 128 registers
constexpr uint32_t kThreads = kWarps * 32;

struct WArgs {
  const char* arena;
  const uint32_t* table;
  const WarpItem* items;  // this launch's S or E items
  uint32_t n_items;
  uint32_t n_layers;  // layers of this launch (grid = item blocks × n_layers)
  uint32_t ks;        // K slices of the S items (v partial planes per job)
  uint32_t d_in;
  uint32_t log2_page;
  uint32_t fast;  // page entries by warp shuffle (rows / blocks span few pages)
  const char* x;
  uint64_t x_stride_b, x_lstride_b;
  char* y[PLORA_MAX_PROJ];
  uint64_t y_stride_b[PLORA_MAX_PROJ], y_lstride_b[PLORA_MAX_PROJ];
  uint64_t blk_mult[PLORA_MAX_PROJ];  // block offset multiplier of (layer0, proj)
  uint32_t d_out[PLORA_MAX_PROJ];
  uint64_t plu;                       // ModelGeom::per_layer_unit
  float* v;
  uint64_t vplane;                    // floats per launched layer
  float scale;
  uint64_t* trace;  // diagnostics (plora_debug_set_trace): [item][2] globaltimer ns (start, end), or nullptr
  uint32_t trace_off;  // expand launch: its items follow the shrink's in the trace
  // tensor-parallel halves (launch_bgmv_warp_tp; zero for the data-parallel op)
  uint32_t tp_size, tp_rank, tp_rsmax, tp_T, tp_njobs, tp_ndst;
  float* tp_part;
  uint32_t* tp_cnt;
  float* tp_vout;
  float* tp_dst[kMaxTp];
  uint32_t* tp_flags[kMaxTp];
  uint32_t* tp_done;
  const float* tp_vg;
  uint32_t* tp_wait;
};

struct WI {
  uint32_t toff, rank, ntok, pj, n, off, voff, flags;
  uint32_t tok[kWarpJobTok];
};

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ WI load_item(const WarpItem* it) {
  const uint4 a = __ldg(reinterpret_cast<const uint4*>(it));
  const uint4 b = __ldg(reinterpret_cast<const uint4*>(it) + 1);
  WI w;
  w.toff = a.x;
  w.rank = a.y & 0x1ffu;
  w.ntok = (a.y >> 9) & 7u;
  w.pj = (a.y >> 12) & 0xfu;
  w.n = (a.y >> 16) & 0x3ffu;
  w.flags = a.y & (kWarpSplit | kWarpSecond);
  w.off = a.z;
  w.voff = a.w;
  w.tok[0] = b.x;
  w.tok[1] = b.y;
  w.tok[2] = b.z;
  w.tok[3] = b.w;
  return w;
}


// acc += a.lo · b.lo + a.hi · b.hi for bf16 pairs (fma.rn.f32.bf16: exact
// products, one fp32 rounding per term — the same as FFMA on converted values)
__device__ __forceinline__ void fh2(float& acc, uint32_t a, uint32_t b) {
  asm("{\n\t.reg .b16 al, ah, bl, bh;\n\t"
      "mov.b32 {al, ah}, %1;\n\t"
      "mov.b32 {bl, bh}, %2;\n\t"
      "fma.rn.f32.bf16 %0, al, bl, %0;\n\t"
      "fma.rn.f32.bf16 %0, ah, bh, %0;\n\t}"
      : "+f"(acc)
      : "r"(a), "r"(b));
}

__device__ __forceinline__ void fh8(float& acc, const uint4& a, const uint4& b) {
  fh2(acc, a.x, b.x);
  fh2(acc, a.y, b.y);
  fh2(acc, a.z, b.z);
  fh2(acc, a.w, b.w);
}

// {a0, a1} += {w.lo, w.hi} · {v, v}  (FFMA2)
__device__ __forceinline__ void ffma2_bf(uint64_t& acc, uint32_t w, uint64_t vv) {
  uint64_t wf;
  asm("mov.b64 %0, {%1, %2};" : "=l"(wf) : "r"(w << 16), "r"(w & 0xffff0000u));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(wf), "l"(vv));
}

__device__ __forceinline__ uint64_t dup2(float v) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %1};" : "=l"(r) : "f"(v));
  return r;
}

__device__ __forceinline__ float2 unpack2(uint64_t a) {
  float2 f;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(f.x), "=f"(f.y) : "l"(a));
  return f;
}

// Sum V[0..N) over the warp by a halving butterfly (N a power of two <= 32):
// N - 1 + 5 - log2(N) shuffles.  Returns the total of value index k(lane)
// (see warp_sum_index); every lane pair (l, l ^ (32 / N)...) agrees.
template <int N>
__device__ __forceinline__ float warp_sum_many(float (&V)[N], uint32_t lane) {
  int n = N;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    if (n > 1) {
      const int h = n / 2;
      const bool up = (lane & o) != 0;
#pragma unroll
      for (int k = 0; k < N / 2; ++k) {
        if (k < h) {
          const float send = up ? V[k] : V[k + h];
          const float keep = up ? V[k + h] : V[k];
          V[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
      n = h;
    } else {
      V[0] += __shfl_xor_sync(0xffffffffu, V[0], o);
    }
  }
  return V[0];
}

// The value index whose total lane `lane` holds after warp_sum_many<N>.
template <int N>
__device__ __forceinline__ uint32_t warp_sum_index(uint32_t lane) {
  uint32_t k = 0;
  int n = N;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    if (n > 1) {
      const int h = n / 2;
      if (lane & o) k += h;
      n = h;
    }
  }
  return k;
}

template <int N>
__device__ __forceinline__ bool warp_sum_owner(uint32_t lane) {
  // after the halving steps, values are replicated over the lane bits that
  // were only full-reduced: the lowest such lane stores
  constexpr uint32_t kLog = N <= 1 ? 0 : N <= 2 ? 1 : N <= 4 ? 2 : N <= 8 ? 3 : N <= 16 ? 4 : 5;
  constexpr uint32_t kRepMask = (1u << (5 - kLog)) - 1u;  // low lane bits not used for the index
  return (lane & kRepMask) == 0;
}

constexpr int pow2_at_least(int v) { return v <= 1 ? 1 : v <= 2 ? 2 : v <= 4 ? 4 : v <= 8 ? 8 : v <= 16 ? 16 : 32; }

// Per-lane cp.async rings: every lane copies its own 16-byte pieces of the
// weight rows into its own slots of the warp's ring in shared memory and
// later reads back exactly those bytes (no cross-lane visibility, so no
// barrier of any kind); cp.async.wait_group orders each lane's copies.  The
// ring holds kRing 512-byte warp units (8 KiB per warp), i.e. the loads in
// flight no longer cost registers (profiles/r02n_microbench_ldg.txt: the
// register-buffered loop reached 0.94 of the roofline, this one the load-only
// ceiling).
// Ring depth: 16 units (8 KiB per warp, 16 warps per SM) for multi-layer
// launches, which have items for every SM many times over; 32 units (16 KiB
// per warp, 12 warps per SM) for a single layer's call, whose few items each
// stream for longer (profiles/r02n_warp_variants.txt: per-layer 45.0 ->
// 36.5 us; the 32-layer step 0.661 -> 0.766 ms with the deep ring, so both).
constexpr uint32_t kRing = 16;
constexpr uint32_t kDeepRing = 32;
constexpr uint32_t kYUnits = 4;  // expand: the item's y pieces (T · NS <= 4 units)
__host__ __device__ constexpr uint32_t warp_smem(uint32_t ring) { return (ring + kYUnits) * 512; }
__host__ __device__ constexpr uint32_t cta_smem(uint32_t ring) { return kWarps * warp_smem(ring); }

__device__ __forceinline__ uint4 lds16(uint32_t a) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
  return r;
}

__device__ __forceinline__ void cpa16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16u : 0u)
               : "memory");
}

// ------------------------------------------------------------------ shrink
// Units (chunk c, row i), row fastest; unit u goes to slot u % kRing and is
// issued kRing units (LA = kRing / R chunks) before it is consumed, so the
// unit issued after consuming (c, i) is (c + LA, i): the same row, a static
// register index for its page entries.
// The two warps of a split pair (warps 2c and 2c + 1 of the CTA) meet here:
// named barrier 1 + c, 64 threads.  The non-.aligned barrier: the warps reach
// it from different instructions and a warp may arrive not yet reconverged.
// (Immediate barrier ids: a register id cost a single layer's call 5 µs,
// 32.4 -> 37.7, profiles/r02o_warp_split.txt.)
__device__ __forceinline__ void pair_sync() {
  __syncwarp();
  if constexpr (kWarps == 2) {
    asm volatile("barrier.sync 1, 64;" ::: "memory");
  } else {
    static_assert(kWarps <= 8, "pair barriers 1..4");
    switch (threadIdx.x >> 6) {
      case 0: asm volatile("barrier.sync 1, 64;" ::: "memory"); break;
      case 1: asm volatile("barrier.sync 2, 64;" ::: "memory"); break;
      case 2: asm volatile("barrier.sync 3, 64;" ::: "memory"); break;
      default: asm volatile("barrier.sync 4, 64;" ::: "memory"); break;
    }
  }
}

__device__ __forceinline__ uint32_t tok_of(const WI& w, uint32_t t) {
  return t == 0 ? w.tok[0] : t == 1 ? w.tok[1] : t == 2 ? w.tok[2] : w.tok[3];
}

// Tensor-parallel shrink: the job's last item (of rs/R row blocks × ks K
// slices) sums the K-slice partials in slice order into v_part / the peers'
// gathered buffers; with peers, the launch's last job releases their flags.
__device__ __forceinline__ void tp_job_done(const WArgs& p, const WI& w, uint32_t lane, uint32_t rs,
                                         uint32_t nitems) {
  __syncwarp();
  uint32_t last = 0;
  if (lane == 0) {
    __threadfence();
    last = atomicAdd(p.tp_cnt + w.voff, 1u) + 1 == nitems;
  }
  if (!__shfl_sync(0xffffffffu, last, 0)) return;
  __threadfence();
  const uint32_t ne = w.ntok * rs;
  for (uint32_t e = lane; e < ne; e += 32) {
    const uint32_t t = e / rs, row = e - t * rs;
    float sum = 0.f;
    for (uint32_t k = 0; k < p.ks; ++k) sum += __ldcg(p.tp_part + w.voff + (k * w.ntok + t) * rs + row);
    const uint64_t o = static_cast<uint64_t>(tok_of(w, t)) * p.tp_rsmax + row;
    if (p.tp_vout) p.tp_vout[o] = sum;
    for (uint32_t d = 0; d < p.tp_ndst; ++d) p.tp_dst[d][o] = sum;  // peer stores over NVLink
  }
  if (lane == 0) p.tp_cnt[w.voff] = 0u;  // for the next call (stream-ordered after this grid)
  if (p.tp_ndst) {
    ptx::fence_acq_rel_sys();  // this lane's peer stores, before the job counts as done
    __syncwarp();
    if (lane == 0 && atomicAdd(p.tp_done, 1u) + 1 == p.tp_njobs) {
      *p.tp_done = 0u;
      for (uint32_t d = 0; d < p.tp_ndst; ++d) ptx::red_release_sys_add(p.tp_flags[d], 1u);
    }
  }
}

template <int T, bool FAST, uint32_t RG, bool TPS = false>
__device__ __forceinline__ void shrink_item(const WArgs& p, const WI& w, uint32_t li, uint32_t lane,
                                            uint32_t ring) {
  constexpr int R = kWarpRows(T);
  constexpr uint32_t LA = RG / R;  // chunks of lookahead
  const uint32_t L = p.log2_page;
  const uint64_t pmask = (1ull << L) - 1;
  const uint64_t blk = p.blk_mult[w.pj] + static_cast<uint64_t>(li) * p.plu;
  const uint32_t rowb = p.d_in * 2;
  const uint32_t row0 = w.off & 0xffffu, slice = w.off >> 16;
  const uint32_t ncall = (p.d_in + 255) / 256;  // 512-byte chunks per row (the last may be partial)
  const uint32_t cps = (ncall + p.ks - 1) / p.ks;
  const uint32_t c0 = slice * cps, nc = min(ncall, c0 + cps) - c0;  // this item's chunks [c0, c0 + nc)
  const uint32_t kin = min(p.d_in, (c0 + nc) * 256) - c0 * 256;     // its inputs
  const uint64_t a0 = (static_cast<uint64_t>(w.rank) * blk + static_cast<uint64_t>(row0) * p.d_in + c0 * 256ull) * 2;
  const uint32_t* tab = p.table + w.toff;
  // page entries: lane k holds the entry of row i's k-th page
  uint32_t ent[R], pg0[R];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const uint64_t rb = a0 + static_cast<uint64_t>(i) * rowb;
    pg0[i] = static_cast<uint32_t>(rb >> L);
    ent[i] = 0u;
    if (FAST) {
      const uint32_t span = static_cast<uint32_t>((rb + kin * 2 - 1) >> L) - pg0[i];
      if (static_cast<uint32_t>(i) < w.n && lane <= span) ent[i] = __ldg(tab + pg0[i] + lane);
    }
  }
  auto issue = [&](uint32_t c, int i) {  // unit (c, i) -> slot ((c % LA) · R + i); always one group
    const uint64_t off = a0 + static_cast<uint64_t>(i) * rowb + c * 512 + lane * 16;
    const uint32_t pg = static_cast<uint32_t>(off >> L);
    uint32_t e = 0u;
    if (FAST) e = __shfl_sync(0xffffffffu, ent[i], (pg - pg0[i]) & 31u);
    const bool valid = static_cast<uint32_t>(i) < w.n && c < nc && c * 256 + lane * 8 < kin;
    if (!FAST && valid) e = __ldg(tab + pg);
    cpa16(ring + ((c % LA) * R + i) * 512, valid ? p.arena + (static_cast<uint64_t>(e) << L) + (off & pmask) : p.arena,
          valid);
    ptx::cp_async_commit();
  };
  const char* xr[T];
#pragma unroll
  for (int t = 0; t < T; ++t)
    xr[t] = p.x + static_cast<uint64_t>(li) * p.x_lstride_b + static_cast<uint64_t>(w.tok[t]) * p.x_stride_b +
            c0 * 512 + lane * 16;
  float acc[R][T];
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int t = 0; t < T; ++t) acc[i][t] = 0.f;
  if constexpr (RG == kDeepRing) {
    // Single-layer calls (few items per SM, each warp's own latency counts):
    // the x pieces travel through the ring too, LX chunks ahead like the
    // weights — one commit group per chunk (its R weight units + T x units);
    // x registers loaded one chunk ahead left every chunk waiting on an L2
    // round trip.  The prologue's weight groups precede the dependency wait,
    // its x groups follow it: waiting for <= LX - 1 pending groups before
    // chunk c always covers both of chunk c's groups.
    constexpr uint32_t U = R + T, LX = RG / U;
    auto issue_w = [&](uint32_t c) {
      const uint32_t sb = ring + (c % LX) * U * 512;
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const uint64_t off = a0 + static_cast<uint64_t>(i) * rowb + c * 512 + lane * 16;
        const uint32_t pg = static_cast<uint32_t>(off >> L);
        uint32_t e = 0u;
        if (FAST) e = __shfl_sync(0xffffffffu, ent[i], (pg - pg0[i]) & 31u);
        const bool valid = static_cast<uint32_t>(i) < w.n && c < nc && c * 256 + lane * 8 < kin;
        if (!FAST && valid) e = __ldg(tab + pg);
        cpa16(sb + i * 512, valid ? p.arena + (static_cast<uint64_t>(e) << L) + (off & pmask) : p.arena, valid);
      }
    };
    auto issue_x = [&](uint32_t c) {
      const uint32_t sb = ring + ((c % LX) * U + R) * 512;
      const bool valid = c < nc && c * 256 + lane * 8 < kin;
#pragma unroll
      for (int t = 0; t < T; ++t) cpa16(sb + t * 512, valid ? xr[t] + c * 512 : p.x, valid);
    };
    for (uint32_t c = 0; c < LX; ++c) {
      issue_w(c);
      ptx::cp_async_commit();
    }
    ptx::pdl_wait();  // x (and the v this launch overwrites) belong to earlier kernels
    for (uint32_t c = 0; c < LX; ++c) {
      issue_x(c);
      ptx::cp_async_commit();
    }
#pragma unroll 1
    for (uint32_t c = 0; c < nc; ++c) {
      ptx::cp_async_wait<LX - 1>();  // chunk c's weight and x groups have landed
      const uint32_t sb = ring + (c % LX) * U * 512;
      uint4 xv[T];
#pragma unroll
      for (int t = 0; t < T; ++t) xv[t] = lds16(sb + (R + t) * 512);
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const uint4 wv = lds16(sb + i * 512);
#pragma unroll
        for (int t = 0; t < T; ++t) fh8(acc[i][t], wv, xv[t]);
      }
      issue_w(c + LX);
      issue_x(c + LX);
      ptx::cp_async_commit();
    }
  } else {
    for (uint32_t c = 0; c < LA; ++c)
#pragma unroll
      for (int i = 0; i < R; ++i) issue(c, i);
    ptx::pdl_wait();  // x (and the v this launch overwrites) belong to earlier kernels
    auto ldx = [&](uint32_t c, uint4 (&xv)[T]) {
      const bool valid = c < nc && c * 256 + lane * 8 < kin;
#pragma unroll
      for (int t = 0; t < T; ++t)
        xv[t] = valid ? __ldg(reinterpret_cast<const uint4*>(xr[t] + c * 512)) : make_uint4(0u, 0u, 0u, 0u);
    };
    uint4 xv[T];
    ldx(0, xv);
#pragma unroll 1
    for (uint32_t c = 0; c < nc; ++c) {
      uint4 xn[T];
      ldx(c + 1, xn);
      const uint32_t sb = ring + (c % LA) * R * 512;
#pragma unroll
      for (int i = 0; i < R; ++i) {
        ptx::cp_async_wait<RG - 1>();  // unit (c, i) has landed
        const uint4 wv = lds16(sb + i * 512);
#pragma unroll
        for (int t = 0; t < T; ++t) fh8(acc[i][t], wv, xv[t]);
        issue(c + LA, i);
      }
#pragma unroll
      for (int t = 0; t < T; ++t) xv[t] = xn[t];
    }
  }
  ptx::cp_async_wait<0>();  // (only zero-size copies remain; the ring is reused by the next item)
  constexpr int N = pow2_at_least(R * T);
  float V[N];
#pragma unroll
  for (int k = 0; k < N; ++k) V[k] = k < R * T ? acc[k / T][k % T] : 0.f;
  const float sum = warp_sum_many<N>(V, lane);
  const uint32_t k = warp_sum_index<N>(lane);
  if (TPS) {  // the item's partial sums of its K slice -> the job's partial block [ks][ntok][rs]
    const uint32_t rs = w.rank / p.tp_size;
    if (warp_sum_owner<N>(lane) && k < static_cast<uint32_t>(R * T)) {
      const uint32_t i = k / T, t = k % T;
      if (i < w.n) p.tp_part[w.voff + (slice * w.ntok + t) * rs + (row0 + i - p.tp_rank * rs)] = sum;
    }
    tp_job_done(p, w, lane, rs, (rs + R - 1) / R * p.ks);
    return;
  }
  if (warp_sum_owner<N>(lane) && k < static_cast<uint32_t>(R * T)) {
    const uint32_t i = k / T, t = k % T;
    if (i < w.n)
      p.v[static_cast<uint64_t>(li) * p.vplane + w.voff + (slice * w.ntok + t) * w.rank + row0 + i] = sum;
  }
}

template <bool FAST, uint32_t RG>
__global__ void __launch_bounds__(kThreads, PLORA_WARP_MINB) bgmv_warp_shrink_kernel(const WArgs p) {
  extern __shared__ __align__(16) char smem[];
  ptx::pdl_launch_dependents();  // the expand may start loading its first weight rows
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // block b: layer b % n_layers of item block b / n_layers (the heaviest items
  // of every layer first)
  const uint32_t li = blockIdx.x % p.n_layers;
  const uint32_t wi = (blockIdx.x / p.n_layers) * kWarps + warp;
  if (wi >= p.n_items) return;
  const uint32_t ring = ptx::smem_u32(smem) + warp * warp_smem(RG) + lane * 16;
  const uint64_t t0 = p.trace ? gtime() : 0;
  const WI w = load_item(p.items + wi);
  switch (w.ntok) {
    case 1: shrink_item<1, FAST, RG>(p, w, li, lane, ring); break;
    case 2: shrink_item<2, FAST, RG>(p, w, li, lane, ring); break;
    case 3: shrink_item<3, FAST, RG>(p, w, li, lane, ring); break;
    default: shrink_item<4, FAST, RG>(p, w, li, lane, ring); break;
  }
  if (p.trace && lane == 0) {
    p.trace[2 * (blockIdx.x * kWarps + warp)] = t0;
    p.trace[2 * (blockIdx.x * kWarps + warp) + 1] = gtime();
  }
}

// ------------------------------------------------------------------ expand
// Rows in blocks of 64 (lane k holds the page entries and v of rows jb + k and
// jb + 32 + k); row j's NS units go to ring row slot j % DR, issued DR rows
// ahead of their use.
// Fused all-gather, expand side: the launch's last item (of either half of a
// split pair) consumes this call's arrival from every source.
__device__ __forceinline__ void tp_consume(const WArgs& p, uint32_t lane) {
  __syncwarp();
  if (lane == 0 && atomicAdd(p.tp_done, 1u) + 1 == p.n_items) {
    *p.tp_done = 0u;
    for (uint32_t q = 0; q < p.tp_size; ++q) ptx::red_relaxed_sys_add(p.tp_wait + q, 0xffffffffu);
  }
}

// NARROW: items of <= 256 columns for every token count (the TP halves, whose
// column shards leave few items at kWarpCols)
template <int T, bool FAST, uint32_t RG, uint32_t KS, bool TPE = false, bool NARROW = false>
__device__ __forceinline__ void expand_item(const WArgs& p, const WI& w, uint32_t li, uint32_t lane,
                                            uint32_t ring, uint32_t partner) {
  constexpr int NS = NARROW ? 1 : kWarpCols(T) / 256;  // 16-byte column chunks per lane and row
  constexpr uint32_t DR = RG / NS;        // ring depth in rows
  const uint32_t L = p.log2_page;
  const uint64_t pmask = (1ull << L) - 1;
  const uint64_t blk = p.blk_mult[w.pj] + static_cast<uint64_t>(li) * p.plu;
  const uint32_t rowb = p.d_out[w.pj] * 2;
  const uint32_t r = w.rank;
  // byte offset of row 0's column block
  const uint64_t b0 = (static_cast<uint64_t>(r) * blk + static_cast<uint64_t>(r) * p.d_in + w.off) * 2;
  const uint32_t segb = w.n * 2;
  const uint32_t* tab = p.table + w.toff;
  // rank rows [j0, j1) of this warp: all of them, or one half of a split pair
  // (single-layer calls only: multi-layer launches have no pairs, and their
  // kernels are compiled without the pair code)
  const bool split = RG == kDeepRing && (w.flags & kWarpSplit) != 0;
  const bool second = split && (w.flags & kWarpSecond) != 0;
  const uint32_t hr = (r + 1) / 2;
  const uint32_t j0 = split && second ? hr : 0u, j1 = split && !second ? hr : r;
  bool valid[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) valid[s] = s * 256 + lane * 8 < w.n;
  const float* vb = p.v + static_cast<uint64_t>(li) * p.vplane + w.voff;  // [tok][rank]
  uint64_t acc[NS][4][T];
#pragma unroll
  for (int s = 0; s < NS; ++s)
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int t = 0; t < T; ++t) acc[s][q][t] = 0ull;
  // page entries of rows jb + lane and jb + 32 + lane (first and second page
  // of the row's column block)
  uint32_t ef[2], es[2];
  auto entries = [&](uint32_t jb) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t j = jb + h * 32 + lane;
      ef[h] = es[h] = 0u;
      if (FAST && j < r) {
        const uint64_t sb = b0 + static_cast<uint64_t>(j) * rowb;
        const uint32_t pf = static_cast<uint32_t>(sb >> L);
        ef[h] = __ldg(tab + pf);
        es[h] = static_cast<uint32_t>((sb + segb - 1) >> L) != pf ? __ldg(tab + pf + 1) : ef[h];
      }
    }
  };
  auto issue = [&](uint32_t jb, uint32_t nrow, uint32_t jj) {  // row jb + jj (one group, possibly empty)
    const uint64_t sb = b0 + static_cast<uint64_t>(jb + jj) * rowb;
    const uint32_t pf = static_cast<uint32_t>(sb >> L);
    uint32_t e_f = 0u, e_s = 0u;
    if (FAST) {
      e_f = __shfl_sync(0xffffffffu, (jj & 32u) ? ef[1] : ef[0], jj & 31u);
      e_s = __shfl_sync(0xffffffffu, (jj & 32u) ? es[1] : es[0], jj & 31u);
    }
    const uint32_t slot = ring + (jj % DR) * NS * 512;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const bool ok = jj < nrow && valid[s];
      const uint64_t off = sb + s * 512 + lane * 16;
      const uint32_t pg = static_cast<uint32_t>(off >> L);
      uint32_t e = pg == pf ? e_f : e_s;
      if (!FAST && ok) e = __ldg(tab + pg);
      cpa16(slot + s * 512, ok ? p.arena + (static_cast<uint64_t>(e) << L) + (off & pmask) : p.arena, ok);
    }
    ptx::cp_async_commit();
  };
  // Single-layer calls: the first block's weight rows do not depend on the
  // shrink (the arena is static over the call, ordered before the shrink by
  // the stream), so they are issued before the dependency wait and stream
  // under the shrink's tail (per-layer call 36.7 -> 34.6 us; the multi-layer
  // launch, whose expand items mostly start after the shrink, measured 1 %
  // slower with it: profiles/r02o_expand_prefetch.txt).
  constexpr bool kPre = RG == kDeepRing;
  if (kPre) {
    entries(j0);
    for (uint32_t jj = 0; jj < DR; ++jj) issue(j0, min(64u, j1 - j0), jj);
  }
  ptx::pdl_wait();  // v (the shrink launch) and y (earlier kernels)
  // the item's y pieces into the warp's y area (the oldest group, or with kPre
  // the one after the first block's rows: every wait from row 1 on covers it);
  // a pair's second half does not touch y
  const uint32_t yarea = ring + RG * 512;
#pragma unroll
  for (int t = 0; t < T; ++t) {
    const char* yr = p.y[w.pj] + static_cast<uint64_t>(li) * p.y_lstride_b[w.pj] +
                     static_cast<uint64_t>(w.tok[t]) * p.y_stride_b[w.pj] + static_cast<uint64_t>(w.off) * 2;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const bool ok = valid[s] && !second;
      cpa16(yarea + (t * NS + s) * 512, ok ? yr + s * 512 + lane * 16 : p.y[w.pj], ok);
    }
  }
  ptx::cp_async_commit();
  if (TPE && p.tp_wait) {  // fused all-gather: every rank's v rows of this call have landed
    if (lane == 0)
      for (uint32_t q = 0; q < p.tp_size; ++q)
        while (ptx::ld_acquire_sys(p.tp_wait + q) == 0u) __nanosleep(64);
    __syncwarp();
  }
  const uint32_t trs = TPE ? r / p.tp_size : 1u;  // TP: shard rows per rank of this adapter
  for (uint32_t jb = j0; jb < j1; jb += 64) {
    float vv[T][2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t j = jb + h * 32 + lane;
      if (TPE) {  // v(t, j) = v_gathered[j / rs][tok][j % rs]
        const uint32_t src = j / trs;
#pragma unroll
        for (int t = 0; t < T; ++t)
          vv[t][h] = j < r ? __ldcg(p.tp_vg + (static_cast<uint64_t>(src) * p.tp_T + w.tok[t]) * p.tp_rsmax + (j - src * trs))
                           : 0.f;
        continue;
      }
#pragma unroll
      for (int t = 0; t < T; ++t) vv[t][h] = j < r ? vb[t * r + j] : 0.f;
      // the K-slice partials of v, summed in slice order (KS: compile-time
      // slice count, 0 = the launch's p.ks; the expand's code is sensitive to
      // anything around these loads, so the one-slice body has none)
      if (KS == 2 && j < r) {
#pragma unroll
        for (int t = 0; t < T; ++t) vv[t][h] += vb[(T + t) * r + j];
      }
      if (KS == 0 && j < r) {
#pragma unroll
        for (int t = 0; t < T; ++t)
          for (uint32_t k = 1; k < p.ks; ++k) vv[t][h] += vb[(k * T + t) * r + j];
      }
    }
    const uint32_t nrow = min(64u, j1 - jb);
    if (!kPre || jb > j0) {
      entries(jb);
      for (uint32_t jj = 0; jj < DR; ++jj) issue(jb, nrow, jj);
    }
#pragma unroll 2
    for (uint32_t jj = 0; jj < nrow; ++jj) {
      uint64_t v2[T];
#pragma unroll
      for (int t = 0; t < T; ++t)
        v2[t] = dup2(__shfl_sync(0xffffffffu, (jj & 32u) ? vv[t][1] : vv[t][0], jj & 31u));
      ptx::cp_async_wait<DR - 1>();  // row jj has landed
      const uint32_t slot = ring + (jj % DR) * NS * 512;
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const uint4 wv = lds16(slot + s * 512);
        const uint32_t wq[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int t = 0; t < T; ++t) ffma2_bf(acc[s][q][t], wq[q], v2[t]);
      }
      issue(jb, nrow, jj + DR);
    }
    ptx::cp_async_wait<0>();  // the ring is refilled by the next block / item (and y has landed)
  }
  ptx::cp_async_wait<0>();
  if (split) {  // combine the pair: acc(rows [0, h)) + acc(rows [h, r)), in that order
    constexpr int K = NS * 4 * T;
    if (second) {  // its own ring is idle now: stage the partial sums there
      __syncwarp();  // every lane's copies into the ring have landed (the staging crosses lanes' slots)
#pragma unroll
      for (int s = 0; s < NS; ++s)
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int t = 0; t < T; ++t)
            asm volatile("st.shared.u64 [%0], %1;" ::"r"(ring - lane * 16 + (((s * 4 + q) * T + t) * 32 + lane) * 8),
                         "l"(acc[s][q][t]) : "memory");
      pair_sync();
      if (TPE && p.tp_wait) tp_consume(p, lane);
      return;
    }
    pair_sync();
    static_assert(K * 256 <= 16 * 512, "pair partial sums fit the partner's ring");
#pragma unroll
    for (int s = 0; s < NS; ++s)
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int t = 0; t < T; ++t) {
          uint64_t o;
          asm volatile("ld.shared.u64 %0, [%1];" : "=l"(o) : "r"(partner + (((s * 4 + q) * T + t) * 32 + lane) * 8) : "memory");
          const float2 a = unpack2(acc[s][q][t]), b = unpack2(o);
          asm("mov.b64 %0, {%1, %2};" : "=l"(acc[s][q][t]) : "f"(a.x + b.x), "f"(a.y + b.y));
        }
  }
  // y = bf16(y + scale · acc), 16 bytes per (token, chunk)
#pragma unroll
  for (int t = 0; t < T; ++t) {
    char* yr = p.y[w.pj] + static_cast<uint64_t>(li) * p.y_lstride_b[w.pj] +
               static_cast<uint64_t>(w.tok[t]) * p.y_stride_b[w.pj] + static_cast<uint64_t>(w.off) * 2;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      if (!valid[s]) continue;
      const uint4 yv = lds16(yarea + (t * NS + s) * 512);
      const uint32_t yw[4] = {yv.x, yv.y, yv.z, yv.w};
      uint32_t o[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 a = unpack2(acc[s][q][t]);
        const float lo = __uint_as_float(yw[q] << 16) + p.scale * a.x;
        const float hi = __uint_as_float(yw[q] & 0xffff0000u) + p.scale * a.y;
        __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
        o[q] = *reinterpret_cast<uint32_t*>(&h);
      }
      *reinterpret_cast<uint4*>(yr + s * 512 + lane * 16) = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
  if (TPE && p.tp_wait) tp_consume(p, lane);
}

template <bool FAST, uint32_t RG, uint32_t KS>
__global__ void __launch_bounds__(kThreads, PLORA_WARP_MINB) bgmv_warp_expand_kernel(const WArgs p) {
  extern __shared__ __align__(16) char smem[];
  ptx::pdl_launch_dependents();
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // block b: layer b % n_layers of item block b / n_layers (the heaviest items
  // of every layer first)
  const uint32_t li = blockIdx.x % p.n_layers;
  const uint32_t wi = (blockIdx.x / p.n_layers) * kWarps + warp;
  if (wi >= p.n_items) return;
  const uint32_t ring = ptx::smem_u32(smem) + warp * warp_smem(RG) + lane * 16;
  const uint32_t partner = ptx::smem_u32(smem) + (warp ^ 1u) * warp_smem(RG);  // a split pair's other warp
  const uint64_t t0 = p.trace ? gtime() : 0;
  const WI w = load_item(p.items + wi);
  switch (w.ntok) {
    case 1: expand_item<1, FAST, RG, KS>(p, w, li, lane, ring, partner); break;
    case 2: expand_item<2, FAST, RG, KS>(p, w, li, lane, ring, partner); break;
    case 3: expand_item<3, FAST, RG, KS>(p, w, li, lane, ring, partner); break;
    default: expand_item<4, FAST, RG, KS>(p, w, li, lane, ring, partner); break;
  }
  if (p.trace && lane == 0) {  // expand items after the shrink's (offset by the launch's S item count)
    const uint64_t o = 2 * (p.trace_off + blockIdx.x * kWarps + warp);
    p.trace[o] = t0;
    p.trace[o + 1] = gtime();
  }
}

// Tensor-parallel halves (tp.cu): one layer, single-layer ring geometry.
template <bool FAST>
__global__ void __launch_bounds__(kThreads, PLORA_WARP_MINB) bgmv_warp_tp_shrink_kernel(const WArgs p) {
  extern __shared__ __align__(16) char smem[];
  ptx::pdl_launch_dependents();
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t wi = blockIdx.x * kWarps + warp;
  if (wi >= p.n_items) return;
  const uint32_t ring = ptx::smem_u32(smem) + warp * warp_smem(kDeepRing) + lane * 16;
  const WI w = load_item(p.items + wi);
  switch (w.ntok) {
    case 1: shrink_item<1, FAST, kDeepRing, true>(p, w, 0, lane, ring); break;
    case 2: shrink_item<2, FAST, kDeepRing, true>(p, w, 0, lane, ring); break;
    case 3: shrink_item<3, FAST, kDeepRing, true>(p, w, 0, lane, ring); break;
    default: shrink_item<4, FAST, kDeepRing, true>(p, w, 0, lane, ring); break;
  }
}

template <bool FAST, bool NARROW>
__global__ void __launch_bounds__(kThreads, PLORA_WARP_MINB) bgmv_warp_tp_expand_kernel(const WArgs p) {
  extern __shared__ __align__(16) char smem[];
  ptx::pdl_launch_dependents();
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t wi = blockIdx.x * kWarps + warp;
  if (wi >= p.n_items) return;
  const uint32_t ring = ptx::smem_u32(smem) + warp * warp_smem(kDeepRing) + lane * 16;
  const uint32_t partner = ptx::smem_u32(smem) + (warp ^ 1u) * warp_smem(kDeepRing);  // a split pair's other warp
  const WI w = load_item(p.items + wi);
  switch (w.ntok) {
    case 1: expand_item<1, FAST, kDeepRing, 1, true, NARROW>(p, w, 0, lane, ring, partner); break;
    case 2: expand_item<2, FAST, kDeepRing, 1, true, NARROW>(p, w, 0, lane, ring, partner); break;
    case 3: expand_item<3, FAST, kDeepRing, 1, true, NARROW>(p, w, 0, lane, ring, partner); break;
    default: expand_item<4, FAST, kDeepRing, 1, true, NARROW>(p, w, 0, lane, ring, partner); break;
  }
}

}  // namespace

void launch_bgmv_warp_tp(const plora_plan& plan, const WarpTp& t, uint32_t layer, uint32_t proj, const void* x,
                         uint64_t x_stride, void* y, uint64_t y_stride, float scale, cudaStream_t stream) {
  if (t.n_items == 0) return;
  const plora_store& st = *plan.store;
  const ModelGeom& gm = st.geom;
  WArgs a{};
  a.n_layers = 1;
  a.arena = st.arena;
  a.table = st.d_table;
  a.items = t.items;
  a.n_items = t.n_items;
  a.ks = t.ks;
  a.d_in = gm.m.d_in[proj];
  a.log2_page = st.log2_page;
  a.x = static_cast<const char*>(x);
  a.x_stride_b = x_stride * 2;
  a.y[0] = static_cast<char*>(y);
  a.y_stride_b[0] = y_stride * 2;
  a.blk_mult[0] = gm.blk_mult(layer, proj);
  a.d_out[0] = gm.m.d_out[proj];
  a.plu = gm.per_layer_unit;
  a.scale = scale;
  a.tp_size = t.tp_size;
  a.tp_rank = t.tp_rank;
  a.tp_rsmax = t.rs_max;
  a.tp_T = t.n_tokens;
  a.tp_njobs = t.njobs;
  a.tp_ndst = t.n_dst;
  a.tp_part = t.part;
  a.tp_cnt = t.cnt;
  a.tp_vout = t.v_out;
  for (uint32_t d = 0; d < t.n_dst; ++d) {
    a.tp_dst[d] = t.dst[d];
    a.tp_flags[d] = t.flags[d];
  }
  a.tp_done = t.done;
  a.tp_vg = t.v_in;
  a.tp_wait = t.wait;
  const uint64_t P = 1ull << st.log2_page;
  const bool fast = P >= 2ull * kWarpCols(1) && (a.d_in * 2ull + P - 1) / P + 1 <= 32;
  a.fast = fast ? 1u : 0u;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(kThreads);
  cfg.gridDim = dim3((t.n_items + kWarps - 1) / kWarps);
  cfg.stream = stream;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  cfg.dynamicSmemBytes = cta_smem(kDeepRing);
  auto go = [&](auto k) {
    set_smem_once(reinterpret_cast<const void*>(k), static_cast<int>(cfg.dynamicSmemBytes));
    PLORA_CUDA(cudaLaunchKernelEx(&cfg, k, a));
    count_launch();
  };
  if (t.half == 1)
    fast ? go(bgmv_warp_tp_shrink_kernel<true>) : go(bgmv_warp_tp_shrink_kernel<false>);
  else if (t.narrow)
    fast ? go(bgmv_warp_tp_expand_kernel<true, true>) : go(bgmv_warp_tp_expand_kernel<false, true>);
  else
    fast ? go(bgmv_warp_tp_expand_kernel<true, false>) : go(bgmv_warp_tp_expand_kernel<false, false>);
}

void launch_bgmv_warp(const plora_plan& plan, const WarpWork& w, uint32_t layer0, uint32_t n_layers,
                      const void* x, uint64_t x_stride, uint64_t x_lstride, void* const* ys,
                      const uint64_t* y_strides, const uint64_t* y_lstrides, float scale,
                      cudaStream_t stream) {
  if (w.ns == 0 || n_layers == 0) return;  // no LoRA token in the batch
  const plora_store& st = *plan.store;
  const ModelGeom& gm = st.geom;
  if (gm.m.d_in[w.projs[0]] % 8) throw ValidationError("bf16 BGMV needs d_in and d_out multiples of 8");
  WArgs a{};
  a.n_layers = n_layers;
  a.arena = st.arena;
  a.table = st.d_table;
  a.d_in = gm.m.d_in[w.projs[0]];
  a.log2_page = st.log2_page;
  a.x = static_cast<const char*>(x);
  a.x_stride_b = x_stride * 2;
  a.x_lstride_b = x_lstride * 2;
  for (uint32_t i = 0; i < w.np; ++i) {
    const uint32_t pr = w.projs[i];
    if (gm.m.d_out[pr] % 8) throw ValidationError("bf16 BGMV needs d_in and d_out multiples of 8");
    a.y[i] = static_cast<char*>(ys[i]);
    a.y_stride_b[i] = y_strides[i] * 2;
    a.y_lstride_b[i] = y_lstrides ? y_lstrides[i] * 2 : 0;
    a.blk_mult[i] = gm.blk_mult(layer0, pr);
    a.d_out[i] = gm.m.d_out[pr];
  }
  a.plu = gm.per_layer_unit;
  a.v = plan.d_wv;
  a.vplane = w.vplane;
  a.ks = w.ks;
  a.scale = scale;
  // shuffle-resolved page entries: a shrink row spans <= 32 pages and an
  // expand block (<= 1 KiB) <= 2 pages
  const uint64_t P = 1ull << st.log2_page;
  const bool fast = P >= 2ull * kWarpCols(1) && (a.d_in * 2ull + P - 1) / P + 1 <= 32;
  a.fast = fast ? 1u : 0u;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(kThreads);
  cfg.stream = stream;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  const bool deep = n_layers == 1;
  cfg.dynamicSmemBytes = cta_smem(deep ? kDeepRing : kRing);
  if (deep) {
    a.trace = trace_buffer(16ull * ((w.ns + w.ne1 + 2) / 2 * 2 + 2));
    a.trace_off = (w.ns + kWarps - 1) / kWarps * kWarps;
  }
  auto launch = [&](auto k16, auto k32, uint32_t n_items, const WarpItem* items) {
    a.items = items;
    a.n_items = n_items;
    cfg.gridDim = dim3((n_items + kWarps - 1) / kWarps * n_layers);
    const void* k = deep ? reinterpret_cast<const void*>(k32) : reinterpret_cast<const void*>(k16);
    set_smem_once(k, static_cast<int>(cfg.dynamicSmemBytes));
    if (deep)
      PLORA_CUDA(cudaLaunchKernelEx(&cfg, k32, a));
    else
      PLORA_CUDA(cudaLaunchKernelEx(&cfg, k16, a));
    count_launch();
  };
  if (fast)
    launch(bgmv_warp_shrink_kernel<true, kRing>, bgmv_warp_shrink_kernel<true, kDeepRing>, w.ns,
           plan.d_witems + w.s_off);
  else
    launch(bgmv_warp_shrink_kernel<false, kRing>, bgmv_warp_shrink_kernel<false, kDeepRing>, w.ns,
           plan.d_witems + w.s_off);
  // single-layer calls: the item list with split pairs for the widest adapters
  const WarpItem* ei = plan.d_witems + (deep ? w.e1_off : w.e_off);
  const uint32_t ne = deep ? w.ne1 : w.ne;
  if (fast && w.ks == 1)
    launch(bgmv_warp_expand_kernel<true, kRing, 1>, bgmv_warp_expand_kernel<true, kDeepRing, 1>, ne, ei);
  else if (fast && w.ks == 2)
    launch(bgmv_warp_expand_kernel<true, kRing, 2>, bgmv_warp_expand_kernel<true, kDeepRing, 2>, ne, ei);
  else if (fast)
    launch(bgmv_warp_expand_kernel<true, kRing, 0>, bgmv_warp_expand_kernel<true, kDeepRing, 0>, ne, ei);
  else if (w.ks == 1)
    launch(bgmv_warp_expand_kernel<false, kRing, 1>, bgmv_warp_expand_kernel<false, kDeepRing, 1>, ne, ei);
  else
    launch(bgmv_warp_expand_kernel<false, kRing, 0>, bgmv_warp_expand_kernel<false, kDeepRing, 0>, ne, ei);
}

}  // namespace plora
