// bf16 paged BGMV: persistent, warp-specialized TMA ring + warp-level tensor
// cores.  This is the decode hot path behind plora_bgmv for bf16 stores.
//
// y[t, :] += scale · (x[t, :] · A_{a(t)}ᵀ) · B_{a(t)}ᵀ,
// weights read through the device page table (src/memory.cpp:55-62).
//
//  * One CTA per SM: 4 producer warps (one per ring slot) + 2 consumer
//    groups of 4 warps (even / odd slots), 4 × 48 KiB slots.  Measured on
//    this B200 (profiles/r01_microbench_loads.txt): 1-D TMA bulk copies
//    sustain ~7 TB/s once >= ~128 KiB per SM are in flight (LDG/LDGSTS
//    streams top out near 2.8 TB/s).  A per-unit device trace
//    (scripts/trace_bgmv.py) showed each unit's issue costs ~2 µs of
//    dependent latency (descriptor, page-table lookups): four producer warps
//    run four such chains in parallel and two consumer groups compute two
//    units at once.
//  * Static schedule: CTA c owns local units k = 0, 1, ... = global units
//    c + k·G of the plan's LPT-ordered list (every shrink unit before every
//    expand unit); unit k goes to slot k % 4 (producer warp k % 4) and to
//    consumer group k % 2.  No atomics; a blocked expand only ever has
//    expands behind it, and every shrink counter is published before its
//    group waits again, so the schedule cannot deadlock.
//  * Producer: per unit, one cp.async.bulk per page piece (weights, L2
//    evict-first), one per x / y row, zero rows for rank padding; for an
//    expand, after those are in flight, it acquires the segment's shrink
//    counter and copies v through the async proxy.
//  * Shrink unit (<= 8 rank rows, <= 2 tokens): mma.sync m16n8k16,
//    D[tok][row] = x · Wᵀ (tokens padded to M = 16), K split over 4 warps
//    with 4 independent accumulators each, reduced in smem; v = x·Aᵀ (fp32).
//  * Expand unit (<= 4 tokens, CB columns): D[tok][col] = v · Bᵀ with v as
//    bf16 hi + lo (two MMAs, ~16 mantissa bits), A fragments built once per
//    k-step for 8 column tiles at a time; y += scale·D stored directly.
#include <cuda_bf16.h>

#include <algorithm>

#include "plan.hpp"
#include "ptx.cuh"

namespace plora {
namespace {

constexpr int kSlots = 4;
constexpr uint32_t kSlotBytes = kRingSlotBytes;  // see plan.hpp
constexpr int kGroupWarps = 4;          // consumer warps per group
constexpr int kGroups = 2;
constexpr int kGroupThreads = kGroupWarps * 32;
constexpr int kConsumers = kGroups * kGroupThreads;
constexpr int kProducers = kSlots;      // one producer warp per slot
constexpr int kThreads = kConsumers + kProducers * 32;
constexpr uint32_t kRowPad = 16;        // conflict-free ldmatrix rows
constexpr int kPre = 8;                 // page pieces per producer lane resolved ahead
constexpr int kTiles = 8;               // expand column tiles per accumulator pass
constexpr uint32_t kStop = 0xffffffffu;
constexpr uint32_t kTraceUnits = 64;

__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ uint64_t now_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void trace_put(const uint64_t* base, uint32_t k, int field,
                                          uint64_t value) {
  if (base && k < kTraceUnits)
    const_cast<uint64_t*>(base)[(blockIdx.x * kTraceUnits + k) * 8 + field] = value;
}

struct RingArgs {
  const char* arena;
  const uint32_t* table;
  const BgmvUnit* units;
  const char* zeros;  // >= 2 KiB of zero bytes (rank-padding rows)
  float* v;
  uint32_t* sync;     // [1] exit count, [2 + s] shrink units done for segment s
  uint64_t* trace;    // diagnostics (plora_debug_set_trace) or nullptr
  const char* x;
  char* y;
  uint64_t x_stride_b;
  uint64_t y_stride_b;
  uint64_t blk_mult;
  uint32_t log2_page;
  uint32_t n_units;
  uint32_t n_seg;
  uint32_t d_in;
  uint32_t d_out;
  float scale;
};

struct Smem {
  static constexpr uint32_t slots = 0;
  static constexpr uint32_t vs = kSlots * kSlotBytes;                            // [2][4][256] f32
  static constexpr uint32_t red = vs + kGroups * kMaxUnitTok * kMaxBgmvRank * 4; // [2][4][16][8]
  static constexpr uint32_t hdr = red + kGroups * kGroupWarps * 16 * 8 * 4;
  static constexpr uint32_t bars = hdr + kSlots * sizeof(BgmvUnit);
  static constexpr uint32_t total = bars + 2 * kSlots * 8;
};

struct Geom {  // per-unit copy geometry (identical in producer and consumers)
  uint32_t stride;    // smem row stride of the weight tile
  uint32_t aux;       // smem offset of x rows (shrink) / y rows (expand)
  uint32_t segbytes;  // bytes per copied row segment
  uint32_t r16;       // expand: rank padded to 16
  uint32_t cb;        // expand: columns per unit
};

__device__ __forceinline__ Geom geom(const RingArgs& p, const BgmvUnit& u) {
  Geom g;
  if (!(u.kind_seg & kExpandBit)) {
    // 16 rank rows × one kShrinkK-wide K chunk (the last chunk may be narrower)
    g.stride = kShrinkK * 2 + kRowPad;
    g.aux = kShrinkRows16 * g.stride;
    g.segbytes = min(kShrinkK, p.d_in - u.kc * kShrinkK) * 2;
    g.r16 = 0;
    g.cb = 0;
  } else {
    g.cb = expand_cols(u.rank, 2);
    g.stride = g.cb * 2 + kRowPad;
    g.r16 = (u.rank + 15) & ~15u;
    g.aux = g.r16 * g.stride;
    g.segbytes = u.count * 2;
  }
  return g;
}

// Piece q of a unit's weight copies: (row, page k) of the unit's rows.
__device__ __forceinline__ bool piece(const RingArgs& p, const BgmvUnit& u, const Geom& g,
                                      uint32_t q, uint32_t ppr, uint64_t& src, uint32_t& dst,
                                      uint32_t& len, uint32_t& page) {
  const uint32_t L = p.log2_page;
  const uint32_t row = q / ppr, k = q - row * ppr;
  uint64_t lo;
  if (!(u.kind_seg & kExpandBit)) {
    if (row >= u.count) return false;
    lo = (static_cast<uint64_t>(u.rank) * p.blk_mult +
          static_cast<uint64_t>(u.off + row) * p.d_in + u.kc * kShrinkK) * 2;
  } else {
    if (row >= u.rank) return false;
    lo = (static_cast<uint64_t>(u.rank) * p.blk_mult + static_cast<uint64_t>(u.rank) * p.d_in +
          static_cast<uint64_t>(row) * p.d_out + u.off) * 2;
  }
  const uint64_t hi = lo + g.segbytes;
  const uint64_t pg = (lo >> L) + k;
  const uint64_t a = max(lo, pg << L), b = min(hi, (pg + 1) << L);
  if (a >= b) return false;
  src = a & ((1ull << L) - 1);  // offset within the page; the page base is added later
  dst = row * g.stride + static_cast<uint32_t>(a - lo);
  len = static_cast<uint32_t>(b - a);
  page = static_cast<uint32_t>(pg);
  return true;
}

// Producer warp w fills slot w with local units w, w + 4, w + 8, ...
__device__ void producer(const RingArgs& p, char* smem, uint32_t w) {
  const uint32_t lane = threadIdx.x & 31;
  BgmvUnit* hdr = reinterpret_cast<BgmvUnit*>(smem + Smem::hdr);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Smem::bars);
  uint64_t* empty = full + kSlots;
  const uint64_t evict_first = ptx::policy_evict_first();
  const uint32_t G = gridDim.x, step = G * kSlots;
  char* sb = smem + Smem::slots + w * kSlotBytes;
  uint32_t u = blockIdx.x + w * G;
  BgmvUnit rec{};
  if (u < p.n_units) rec = p.units[u];
  for (uint32_t k = w, it = 0;; k += kSlots, ++it, u += step) {
    const uint32_t phase = it & 1u;
    const bool live = u < p.n_units;
    if (lane == 0) trace_put(p.trace, k, 4, now_ns());
    BgmvUnit next{};
    if (u + step < p.n_units) next = p.units[u + step];  // descriptor prefetch
    Geom g{};
    uint32_t ppr = 0, n = 0;
    uint64_t src[kPre];
    uint32_t dst[kPre], len[kPre];
#pragma unroll
    for (int m = 0; m < kPre; ++m) len[m] = 0;
    if (live) {
      g = geom(p, rec);
      ppr = ((g.segbytes - 1) >> p.log2_page) + 2;
      n = ((rec.kind_seg & kExpandBit) ? rec.rank : rec.count) * ppr;
#pragma unroll
      for (int m = 0; m < kPre; ++m) {  // page-table lookups before the slot wait
        const uint32_t q = lane + 32u * m;
        uint32_t page;
        if (q < n && piece(p, rec, g, q, ppr, src[m], dst[m], len[m], page)) {
          src[m] += static_cast<uint64_t>(__ldg(p.table + rec.table_off + page)) << p.log2_page;
        } else {
          len[m] = 0;
        }
      }
    }
    if (lane == 0) trace_put(p.trace, k, 5, now_ns());
    ptx::mbar_wait(&empty[w], phase ^ 1u);
    if (lane == 0) trace_put(p.trace, k, 6, now_ns());
    if (!live) {
      if (lane == 0) {
        hdr[w].kind_seg = kStop;
        ptx::mbar_arrive(&full[w]);
      }
      break;
    }
    const bool expand = rec.kind_seg & kExpandBit;
    const uint32_t vbytes = rec.ntok * rpad4(rec.rank) * 4;  // one K-partial plane
    uint32_t tx = (expand ? rec.rank : rec.count) * g.segbytes + rec.ntok * g.segbytes;
    if (expand) tx += (g.r16 - rec.rank) * g.segbytes + rec.nkc * vbytes;
    if (lane == 0) {
      hdr[w] = rec;
      ptx::mbar_arrive_expect_tx(&full[w], tx);
    }
    __syncwarp();
#pragma unroll
    for (int m = 0; m < kPre; ++m)
      if (len[m]) ptx::bulk_g2s_hint(sb + dst[m], p.arena + src[m], len[m], &full[w], evict_first);
    for (uint32_t q = lane + 32u * kPre; q < n; q += 32) {  // very small pages only
      uint64_t s;
      uint32_t d, l, page;
      if (piece(p, rec, g, q, ppr, s, d, l, page))
        ptx::bulk_g2s_hint(sb + d,
                           p.arena + s +
                               (static_cast<uint64_t>(__ldg(p.table + rec.table_off + page))
                                << p.log2_page),
                           l, &full[w], evict_first);
    }
    // Everything below reads data written by earlier kernels in the stream
    // (activations, v, counters): with programmatic dependent launch the
    // weight copies above may run ahead of the previous call's grid.
    if (it == 0) pdl_wait();
    if (!expand) {
      if (lane < rec.ntok)
        ptx::bulk_g2s(sb + g.aux + lane * g.stride,
                      p.x + rec.tok[lane] * p.x_stride_b + rec.kc * kShrinkK * 2, g.segbytes,
                      &full[w]);
    } else {
      if (lane < rec.ntok)
        ptx::bulk_g2s(sb + g.aux + lane * g.cb * 2,
                      p.y + rec.tok[lane] * p.y_stride_b + static_cast<uint64_t>(rec.off) * 2,
                      g.segbytes, &full[w]);
      for (uint32_t j = rec.rank + lane; j < g.r16; j += 32)  // zero rank-padding rows
        ptx::bulk_g2s(sb + j * g.stride, p.zeros, g.segbytes, &full[w]);
      // v = x·Aᵀ of this segment: acquire its shrink counter (the Bᵀ / y copies
      // above are already in flight), then copy v through the async proxy.
      if (lane == 0) {
        const uint32_t* flag = p.sync + 2 + (rec.kind_seg & ~kExpandBit);
        while (ptx::ld_acquire_gpu(flag) < rec.n_shrink) __nanosleep(32);
        ptx::fence_proxy_async_global();
      }
      __syncwarp();
      if (lane < rec.nkc)  // one copy per K-partial plane
        ptx::bulk_g2s(sb + g.aux + rec.ntok * g.cb * 2 + lane * vbytes,
                      p.v + rec.voff + lane * rec.vstride, vbytes, &full[w]);
    }
    if (lane == 0) {
      trace_put(p.trace, k, 0, now_ns());
      trace_put(p.trace, k, 3, (static_cast<uint64_t>(expand) << 32) | tx);
    }
    rec = next;
  }
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// gw = warp index within the consumer group, gt = thread index within it.
// D[row][tok] = W · xᵀ over one K chunk: A = 16 rank rows (ldmatrix), B = the
// unit's tokens straight from smem into registers (N = 8, lanes of absent
// tokens hold zeros), K split over the group's 4 warps, 4 accumulators each.
__device__ __forceinline__ void shrink(const RingArgs& p, const BgmvUnit& u, const Geom& g,
                                       char* sb, float (*red)[16][8], uint32_t gw, uint32_t gt,
                                       uint32_t bar_id) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t ri = (lane & 7) + ((lane >> 3) & 1) * 8;  // rows >= count: stale, discarded
  const uint32_t a_base = ptx::smem_u32(sb + ri * g.stride + (lane >> 4) * 16);
  const uint32_t gq = lane >> 2, c = lane & 3;
  const bool has_tok = gq < u.ntok;
  const char* xrow = sb + g.aux + (has_tok ? gq : 0) * g.stride + c * 4;
  float d[4][4] = {};
  const uint32_t ksteps = g.segbytes / 32;
  uint32_t ks = gw;
  for (; ks + 3 * kGroupWarps < ksteps; ks += 4 * kGroupWarps) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t k = ks + j * kGroupWarps;
      uint32_t a[4], b[2];
      ptx::ldsm_x4(a_base + k * 32, a);
      b[0] = has_tok ? *reinterpret_cast<const uint32_t*>(xrow + k * 32) : 0u;
      b[1] = has_tok ? *reinterpret_cast<const uint32_t*>(xrow + k * 32 + 16) : 0u;
      ptx::mma_bf16_16816(d[j], a, b);
    }
  }
  for (; ks < ksteps; ks += kGroupWarps) {
    uint32_t a[4], b[2];
    ptx::ldsm_x4(a_base + ks * 32, a);
    b[0] = has_tok ? *reinterpret_cast<const uint32_t*>(xrow + ks * 32) : 0u;
    b[1] = has_tok ? *reinterpret_cast<const uint32_t*>(xrow + ks * 32 + 16) : 0u;
    ptx::mma_bf16_16816(d[0], a, b);
  }
  // d0/d1 = (row gq, tokens 2c, 2c+1), d2/d3 = (row gq + 8, tokens 2c, 2c+1)
#pragma unroll
  for (int e = 0; e < 4; ++e)
    red[gw][gq + (e >> 1) * 8][2 * c + (e & 1)] = d[0][e] + d[1][e] + d[2][e] + d[3][e];
  ptx::named_bar_sync(bar_id, kGroupThreads);
  if (gt < u.ntok * u.count) {
    const uint32_t i = gt / u.ntok, t = gt - i * u.ntok;
    float s = 0.f;
#pragma unroll
    for (int w2 = 0; w2 < kGroupWarps; ++w2) s += red[w2][i][t];
    p.v[u.voff + t * rpad4(u.rank) + u.off + i] = s;
  }
}

__device__ __forceinline__ void expand(const RingArgs& p, const BgmvUnit& u, const Geom& g,
                                       char* sb, float (*vs)[kMaxBgmvRank], uint32_t gw,
                                       uint32_t gt, uint32_t bar_id) {
  const uint32_t lane = threadIdx.x & 31;
  // v rows arrived in the slot (the producer acquired the segment counter)
  const uint32_t rp = rpad4(u.rank);
  const float* vsl = reinterpret_cast<const float*>(sb + g.aux + u.ntok * g.cb * 2);
  const uint32_t plane = u.ntok * rp;
  for (uint32_t i = gt; i < kMaxUnitTok * g.r16; i += kGroupThreads) {
    const uint32_t t = i / g.r16, j = i - t * g.r16;
    float s = 0.f;
    if (t < u.ntok && j < u.rank)
      for (uint32_t kc = 0; kc < u.nkc; ++kc) s += vsl[kc * plane + t * rp + j];
    vs[t][j] = s;
  }
  ptx::named_bar_sync(bar_id, kGroupThreads);
  const uint32_t gq = lane >> 2, c = lane & 3;
  const uint32_t tg = min(gq, kMaxUnitTok - 1);
  const float gate = gq < u.ntok ? 1.f : 0.f;
  const uint32_t ksteps = g.r16 / 16;
  const uint32_t b_base = ptx::smem_u32(sb + (lane & 15) * g.stride);
  const char* Y = sb + g.aux;
  const uint32_t n_tiles = u.count / 8;
  // this warp owns column tiles gw, gw + 4, ...; 8 of them per accumulator pass
  for (uint32_t t0 = gw; t0 < n_tiles; t0 += kTiles * kGroupWarps) {
    float d[kTiles][4] = {};
    for (uint32_t kk = 0; kk < ksteps; ++kk) {
      const uint32_t j0 = kk * 16 + 2 * c;
      const float v0 = gate * vs[tg][j0], v1 = gate * vs[tg][j0 + 1];
      const float v8 = gate * vs[tg][j0 + 8], v9 = gate * vs[tg][j0 + 9];
      const uint32_t h0 = pack_bf16x2(v0, v1), h2 = pack_bf16x2(v8, v9);
      const float2 f0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&h0));
      const float2 f2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&h2));
      const uint32_t ahi[4] = {h0, 0u, h2, 0u};
      const uint32_t alo[4] = {pack_bf16x2(v0 - f0.x, v1 - f0.y), 0u,
                               pack_bf16x2(v8 - f2.x, v9 - f2.y), 0u};
#pragma unroll
      for (int i = 0; i < kTiles; ++i) {
        const uint32_t nt = t0 + i * kGroupWarps;
        if (nt < n_tiles) {
          uint32_t b[2];
          ptx::ldsm_x2_trans(b_base + kk * 16 * g.stride + nt * 16, b);
          ptx::mma_bf16_16816(d[i], ahi, b);
          ptx::mma_bf16_16816(d[i], alo, b);
        }
      }
    }
    if (gq < u.ntok) {  // d0/d1 = (token gq, columns nt·8 + 2c, +1): fire-and-forget store
      char* yrow = p.y + u.tok[gq] * p.y_stride_b;
#pragma unroll
      for (int i = 0; i < kTiles; ++i) {
        const uint32_t nt = t0 + i * kGroupWarps;
        if (nt < n_tiles) {
          const uint32_t col = nt * 8 + 2 * c;
          const float2 yo = __bfloat1622float2(
              *reinterpret_cast<const __nv_bfloat162*>(Y + gq * g.cb * 2 + col * 2));
          *reinterpret_cast<__nv_bfloat162*>(yrow + static_cast<uint64_t>(u.off + col) * 2) =
              __floats2bfloat162_rn(fmaf(p.scale, d[i][0], yo.x), fmaf(p.scale, d[i][1], yo.y));
        }
      }
    }
  }
}

// Consumer group grp processes local units grp, grp + 2, ... (slots k % 4).
__device__ void consumer(const RingArgs& p, char* smem, uint32_t grp) {
  const BgmvUnit* hdr = reinterpret_cast<const BgmvUnit*>(smem + Smem::hdr);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Smem::bars);
  uint64_t* empty = full + kSlots;
  float (*red)[16][8] =
      reinterpret_cast<float (*)[16][8]>(smem + Smem::red) + grp * kGroupWarps;
  pdl_wait();  // consumers write v / y / counters: the previous call must be done
  float (*vs)[kMaxBgmvRank] =
      reinterpret_cast<float (*)[kMaxBgmvRank]>(smem + Smem::vs) + grp * kMaxUnitTok;
  const uint32_t gt = threadIdx.x - grp * kGroupThreads, gw = gt >> 5;
  const uint32_t bar_id = 1 + grp;
  uint32_t pending = kStop;  // segment whose shrink unit still has to be published
  for (uint32_t k = grp;; k += kGroups) {
    const uint32_t slot = k % kSlots, phase = (k / kSlots) & 1u;
    if (pending != kStop) {
      if (gt == kGroupThreads - 32) {  // last warp publishes while the others wait for data
        __threadfence();
        atomicAdd(p.sync + 2 + pending, 1u);
      }
      pending = kStop;
    }
    ptx::mbar_wait(&full[slot], phase);
    if (gt == 0) trace_put(p.trace, k, 1, now_ns());
    const BgmvUnit u = hdr[slot];
    if (u.kind_seg == kStop) break;
    char* sb = smem + Smem::slots + slot * kSlotBytes;
    const Geom g = geom(p, u);
    if (!(u.kind_seg & kExpandBit)) {
      shrink(p, u, g, sb, red, gw, gt, bar_id);
      pending = u.kind_seg;
    } else {
      expand(p, u, g, sb, vs, gw, gt, bar_id);
    }
    ptx::named_bar_sync(bar_id, kGroupThreads);  // slot + group scratch free
    if (gt == 0) {
      trace_put(p.trace, k, 2, now_ns());
      ptx::mbar_arrive(&empty[slot]);
    }
  }
  if (pending != kStop && gt == kGroupThreads - 32) {
    __threadfence();
    atomicAdd(p.sync + 2 + pending, 1u);
  }
}

__global__ void __launch_bounds__(kThreads, 1) bgmv_ring_kernel(const RingArgs p) {
  extern __shared__ __align__(128) char smem[];
  __shared__ uint32_t s_last;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Smem::bars);
  uint64_t* empty = full + kSlots;
  pdl_launch_dependents();  // the next call may start streaming its weights
  if (threadIdx.x == 0) {
    for (int s = 0; s < kSlots; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x >= kConsumers)
    producer(p, smem, (threadIdx.x - kConsumers) >> 5);
  else
    consumer(p, smem, threadIdx.x / kGroupThreads);
  __syncthreads();
  // the last CTA out resets the per-segment counters (graph-replayable)
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(p.sync + 1, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    for (uint32_t i = threadIdx.x; i < p.n_seg; i += blockDim.x) p.sync[2 + i] = 0;
    if (threadIdx.x == 0) p.sync[1] = 0;
  }
}

uint64_t* g_trace = nullptr;
uint64_t g_trace_bytes = 0;

}  // namespace

uint64_t* trace_buffer(uint64_t need_bytes) { return g_trace_bytes >= need_bytes ? g_trace : nullptr; }

// Launch the bf16 decode op for one (layer, proj); see plora_bgmv.
void launch_bgmv_ring(const plora_plan& plan, uint32_t layer, uint32_t proj, const void* x,
                      uint64_t x_stride, void* y, uint64_t y_stride, float scale,
                      cudaStream_t stream) {
  const plora_store& st = *plan.store;
  const ModelGeom& gm = st.geom;
  const ProjWork& pw = plan.proj[proj];
  if (pw.n_units == 0) return;
  if (gm.m.d_in[proj] * 2 > kSlotAuxBytes)
    throw ValidationError("bf16 BGMV needs d_in <= 8192");
  RingArgs a{};
  a.arena = st.arena;
  a.table = st.d_table;
  a.units = plan.d_units + pw.units_off;
  a.zeros = st.d_zeros;
  a.v = plan.d_v;
  a.sync = plan.d_sync;
  a.x = static_cast<const char*>(x);
  a.y = static_cast<char*>(y);
  a.x_stride_b = x_stride * 2;
  a.y_stride_b = y_stride * 2;
  a.blk_mult = gm.blk_mult(layer, proj);
  a.log2_page = st.log2_page;
  a.n_units = pw.n_units;
  a.n_seg = plan.n_seg;
  a.d_in = gm.m.d_in[proj];
  a.d_out = gm.m.d_out[proj];
  a.scale = scale;
  const uint32_t grid = std::min<uint32_t>(pw.n_units, static_cast<uint32_t>(st.num_sms));
  a.trace = g_trace_bytes >= static_cast<uint64_t>(grid) * kTraceUnits * 64 ? g_trace : nullptr;
  static bool attr = false;
  if (!attr) {
    PLORA_CUDA(cudaFuncSetAttribute(bgmv_ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(Smem::total)));
    attr = true;
  }
  // programmatic dependent launch: this call's weight streaming may overlap
  // the previous call's tail (the kernel waits before touching activations)
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = Smem::total;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  PLORA_CUDA(cudaLaunchKernelEx(&cfg, bgmv_ring_kernel, a));
  count_launch();
}

}  // namespace plora

extern "C" int plora_debug_set_trace(void* dev_buf, uint64_t bytes) {
  plora::g_trace = static_cast<uint64_t*>(dev_buf);
  plora::g_trace_bytes = dev_buf ? bytes : 0;
  return 0;
}
