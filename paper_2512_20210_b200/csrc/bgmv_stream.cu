// bf16 paged BGMV (decode), streaming design: the hot path behind
// plora_bgmv / plora_bgmv_layer / plora_bgmv_layers for bf16 stores.
//
//   y[t, :] += scale · (x[t, :] · A_{a(t)}ᵀ) · B_{a(t)}ᵀ
//
// with every A / Bᵀ row read straight out of the page arena through the
// device page table (the translation PagePool::translate does on the host,
// src/memory.cpp:55-62).
//
// Decomposition (plan.hpp, StreamItem).  A job = <= JT tokens of one adapter
// at one (layer, proj).  Its shrink is cut into S items of <= 16 rank rows with
// the full K (v[row][tok] = x[tok] · A[row] computed exactly in fp32 inside
// one CTA and stored to the job's block of a v plane), its expand into E
// items, one per block of <= 1024 output columns over all rank rows
// (y[tok][block] += scale · Σ_row v[row][tok] · Bᵀ[row][block]).  An E item
// waits on its job's S-item counter (release / acquire at gpu scope); the
// host schedules every CTA's S items before its E items and orders E items
// by the simulated completion time of their jobs' S items, so the wait is
// rarely taken.  No cluster, no per-chunk exchange: a CTA never waits for a
// peer's progress except through those counters, and every SM streams.
//
// One CTA per SM, persistent over its host-built item list (and, for
// plora_bgmv_layers, over n_layers passes of it).  Every item streams in
// stages of 16 weight rows × <= 1024 elements (32 KiB at Llama-7B widths):
//   producer warps 8-9   alternate stages: wait for the slot, issue one 1-D
//                        TMA bulk copy per page piece of the stage's weight
//                        rows (L2 evict-first; page-table entries fetched an
//                        item ahead with cp.async), the stage's activations
//                        (S: the tokens' x rows; E: the 16 rows of v and, on the
//                        item's last stage, the tokens' y rows) and a header.
//   consumer warps 0-7   S: mma.sync m16n8k16 (tokens as M, 8 rank rows as
//                        N), k-steps split over the warps, partials summed in
//                        a fixed order at the item's last stage -> v.
//                        E: mma.sync m16n8k8 (16 output columns as M, token ×
//                        {bf16 hi, lo} of the fp32 v as N — ~16 mantissa bits
//                        of v), accumulators in registers across the item's
//                        stages; y read (staged) and written once per item.
// Deterministic: every sum has a fixed order independent of the schedule.
#include <cuda_bf16.h>

#include <algorithm>
#include <map>
#include <mutex>

#include "plan.hpp"
#include "ptx.cuh"

namespace plora {
namespace {

constexpr uint32_t kKC = kStreamKC;
constexpr uint32_t kRowB = kKC * 2 + 16;  // smem row stride: 16 B pad -> conflict-free ldmatrix
constexpr uint32_t kWRows = 16;           // weight rows per stage (one MMA K / M of 16)
constexpr uint32_t kCWarps = 8;
constexpr uint32_t kCThreads = kCWarps * 32;
constexpr uint32_t kEntPW = 64;           // page-table entries of one item per producer warp (fast path)
template <uint32_t JT>
constexpr uint32_t kPubBufs = JT == 4 ? 4 : 2;  // S-item partial buffers between the consumers and the publisher
constexpr uint32_t kLook = 4;             // producer lookahead (items)
constexpr uint32_t kRecRing = 2 * kLook;  // item records in flight
constexpr uint32_t kPf = 2;               // L2 prefetch distance (items; <= kLook - 1)
constexpr uint32_t kSmemBudget = 227 * 1024;
constexpr uint32_t kStop = 0xffffffffu;
constexpr uint32_t kHdrWords = 16;

struct SArgs {
  const char* arena;
  const uint32_t* table;
  const StreamItem* items;  // this launch's items
  const uint32_t* cta_off;  // [grid + 1]
  const char* x;
  uint64_t x_stride_b, x_lstride_b;
  char* y[PLORA_MAX_PROJ];
  uint64_t y_stride_b[PLORA_MAX_PROJ], y_lstride_b[PLORA_MAX_PROJ];
  uint64_t blk_mult[PLORA_MAX_PROJ];  // block offset multiplier of (layer0, proj)
  uint32_t plane0[PLORA_MAX_PROJ];    // v / counter plane of (layer0, proj)
  uint64_t plu;                       // ModelGeom::per_layer_unit
  float* v;
  uint64_t vplane;                    // floats per plane
  uint32_t* cnt;                      // per plane: njobs S counters, then njobs E-done counters
  uint32_t njobs, plane_lstride;      // planes between consecutive layers
  uint32_t n_layers;
  uint32_t log2_page, d_in, d_out;
  uint32_t nslots, slot_bytes, off_hdr, off_bar, off_ring, off_part;
  uint32_t fast;  // every weight row segment of a stage lies inside one page
  float scale;
  uint64_t* trace;  // diagnostics (plora_debug_set_trace): [cta][stage][4] SM clocks, or nullptr
  uint32_t dbg;     // diagnostics (plora_debug_set_bgmv_flags): 1 consumers skip the math, 2 no weight copies
  uint32_t pf;      // L2 prefetch of the weight rows kPf items ahead (fast path)
  // tensor-parallel halves (tp.cu; 0: the data-parallel op).  1 = shrink: S
  // items only, v stored as fp32 tp_v[tok][v_off + row] (the v_part layout);
  // 2 = expand: E items only, v read from the all-gathered tp_vg[N][T][rs_max]
  // (row j of a rank-r adapter lives in rank block j / (r/N)).  No counters.
  uint32_t tp, tp_size, tp_T, tp_rsmax;
  float* tp_v;
  const float* tp_vg;
  // fused peer-write all-gather (StreamTp): shrink destinations and flags,
  // expand wait
  uint32_t tp_ndst;
  float* tp_dst[kMaxTp];
  uint32_t* tp_flags[kMaxTp];
  uint32_t* tp_done;
  uint32_t* tp_wait;  // [tp_size] per-source arrivals (expand)
};

constexpr uint32_t kTraceStages = 512;
__device__ __forceinline__ void tput(const SArgs& p, uint32_t gs, uint32_t f, uint64_t v) {
  if (p.trace && gs < kTraceStages) p.trace[(blockIdx.x * kTraceStages + gs) * 12 + f] = v;
}

// Smem slot: [16 weight rows][JT activation rows (S: x, E: y)][v: 16 × JT fp32];
// n slots (one producer warp each), as many as 227 KiB hold
template <uint32_t JT>
struct Slot {
  static constexpr uint32_t aux = kWRows * kRowB;
  static constexpr uint32_t vrows = aux + JT * kRowB;
  static constexpr uint32_t bytes = (vrows + kWRows * JT * 4 + 127) / 128 * 128;
  static constexpr uint32_t n = JT == 4 ? 5 : 4;
  static constexpr uint32_t threads = kCThreads + n * 32 + 32;  // consumers, producers, publisher
};

struct Item {  // a StreamItem read from a smem ring, resolved for pass li
  uint32_t expand, pj, job, table_off, rank, ntok, off, n, v_off, ns, ne, li;
  uint64_t blk;
  __device__ Item(const uint32_t* w, const SArgs& p, uint32_t pass) {
    expand = w[0] >> 31;
    pj = w[0] & 0xffu;
    job = w[1];
    table_off = w[2];
    rank = w[3] & 0xffffu;
    ntok = w[3] >> 16;
    off = w[4];
    n = w[5];
    v_off = w[6];
    ns = w[7] & 0xffffu;
    ne = w[7] >> 16;
    li = pass;
    blk = p.blk_mult[pj] + static_cast<uint64_t>(pass) * p.plu;
  }
  __device__ uint32_t stages(const SArgs& p) const {
    return expand ? (rank + kWRows - 1) / kWRows : (p.d_in + kKC - 1) / kKC;
  }
  __device__ uint32_t plane(const SArgs& p) const { return p.plane0[pj] + li * p.plane_lstride; }
};

// Logical byte range of weight row i of stage st (S: A row off + i, K slice
// st; E: Bᵀ row 8·st + i, columns [off, off + n)).
__device__ __forceinline__ void row_seg(const SArgs& p, const Item& it, uint32_t st, uint32_t i,
                                        uint64_t& lo, uint32_t& len) {
  if (!it.expand) {
    const uint32_t k0 = st * kKC;
    lo = (static_cast<uint64_t>(it.rank) * it.blk + static_cast<uint64_t>(it.off + i) * p.d_in + k0) * 2;
    len = min(kKC, p.d_in - k0) * 2;
  } else {
    lo = (static_cast<uint64_t>(it.rank) * (it.blk + p.d_in) +
          static_cast<uint64_t>(st * kWRows + i) * p.d_out + it.off) * 2;
    len = it.n * 2;
  }
}

__device__ __forceinline__ uint32_t stage_rows(const Item& it, uint32_t st) {
  return it.expand ? min(kWRows, it.rank - st * kWRows) : it.n;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ void cp_async_4(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void red_release_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ---------------------------------------------------------------- producer
// One producer warp per slot: warp pw issues the CTA's stages g ≡ pw (mod
// kPW) into slot pw — wait for the slot, one bulk copy per page piece of the
// stage's weight rows (lanes 0-15), the stage's activation rows (lanes
// 16-23: x, or y on an E item's last stage), v (lane 24, after the job's
// counter says it is complete), then the header and the expect_tx arrival.
// A warp's bulk copies issue one lane at a time, so stages issue in
// parallel across the warps.  Records and (fast path) the page-table entries
// of this warp's stages are fetched kLook items ahead with cp.async.
template <uint32_t JT>
__device__ void producer(const SArgs& p, char* smem, uint32_t pw) {
  constexpr uint32_t kPW = Slot<JT>::n;
  const uint32_t lane = threadIdx.x & 31;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.off_bar);
  uint64_t* empty = full + kPW;
  uint32_t* hdr = reinterpret_cast<uint32_t*>(smem + p.off_hdr) + pw * kHdrWords;
  uint32_t* recring = reinterpret_cast<uint32_t*>(smem + p.off_ring) + pw * (kRecRing * 16 + kLook * kEntPW);
  uint32_t* entring = recring + kRecRing * 16;
  const uint32_t c0 = __ldg(p.cta_off + blockIdx.x), nc = __ldg(p.cta_off + blockIdx.x + 1) - c0;
  const uint32_t nv = nc * p.n_layers;
  const uint32_t L = p.log2_page;
  const uint64_t pmask = (1ull << L) - 1;
  const uint64_t ef = ptx::policy_evict_first();
  char* sb = smem + pw * p.slot_bytes;
  const uint32_t* recg = reinterpret_cast<const uint32_t*>(p.items + c0);
  auto fetch_rec = [&](uint32_t v) {
    if (v < nv && lane < 4)
      ptx::cp_async_16(recring + (v % kRecRing) * 16 + lane * 4, recg + (v % nc) * 16 + lane * 4, 16);
  };
  // page-table entries of this warp's stages of item v (first global stage
  // gv): entry of (its j-th stage, row i) at j · kWRows + i (fast path)
  auto fetch_ent = [&](uint32_t v, uint32_t gv) {
    if (!p.fast || v >= nv) return;
    const Item it(recring + (v % kRecRing) * 16, p, v / nc);
    uint32_t* ent = entring + (v % kLook) * kEntPW;
    const uint32_t nst = it.stages(p), st0 = (pw + kPW - gv % kPW) % kPW;
    const uint32_t mine = st0 < nst ? (nst - st0 + kPW - 1) / kPW : 0u;
    for (uint32_t e = lane; e < mine * kWRows; e += 32) {
      const uint32_t st = st0 + (e / kWRows) * kPW, i = e % kWRows;
      if (i < stage_rows(it, st)) {
        uint64_t lo;
        uint32_t len;
        row_seg(p, it, st, i, lo, len);
        cp_async_4(ptx::smem_u32(ent + e), p.table + it.table_off + static_cast<uint32_t>(lo >> L));
      }
    }
  };
  for (uint32_t v = 0; v < kRecRing; ++v) fetch_rec(v);
  ptx::cp_async_commit();
  cp_async_wait_group<0>();
  __syncwarp();
  uint32_t g_ent = 0;  // first global stage of the next item whose entries are fetched
  for (uint32_t v = 0; v < kLook; ++v) {
    fetch_ent(v, g_ent);
    if (v < nv) g_ent += Item(recring + (v % kRecRing) * 16, p, v / nc).stages(p);
    ptx::cp_async_commit();
  }
  ptx::pdl_wait();  // activations, v planes and counters belong to the previous call until here
  if (p.tp_wait) {  // fused all-gather: every rank's v rows of this call have landed
    if (lane == 0)
      for (uint32_t r = 0; r < p.tp_size; ++r)
        while (ptx::ld_acquire_sys(p.tp_wait + r) == 0u) __nanosleep(128);
    __syncwarp();
  }
  uint32_t ph = 0, g = 0;  // parity of this warp's slot; global stage number
  // L2 prefetch of this warp's stages kPf items ahead: DRAM -> L2 runs that
  // far ahead of the shared-memory ring, whose depth the smem budget caps
  auto prefetch_item = [&](uint32_t vp, uint32_t gp) {
    const Item ip(recring + (vp % kRecRing) * 16, p, vp / nc);
    const uint32_t* entp = entring + (vp % kLook) * kEntPW;
    const uint32_t nstp = ip.stages(p);
    for (uint32_t st = (pw + kPW - gp % kPW) % kPW, j = 0; st < nstp; st += kPW, ++j) {
      if (lane < stage_rows(ip, st)) {
        uint64_t lo;
        uint32_t len;
        row_seg(p, ip, st, lane, lo, len);
        ptx::bulk_prefetch_l2(p.arena + (static_cast<uint64_t>(entp[j * kWRows + lane]) << L) + (lo & pmask), len);
      }
    }
  };
  uint32_t g_pf = 0;  // first global stage of item v + kPf
  if (p.fast && p.pf) {
    for (uint32_t v = 0; v < kPf && v < nv; ++v) g_pf += Item(recring + (v % kRecRing) * 16, p, v / nc).stages(p);
  }
#pragma unroll 1
  for (uint32_t v = 0; v < nv; ++v) {
    cp_async_wait_group<kLook - 1 - kPf>();  // entries of v + kPf, record of v + kLook
    __syncwarp();
    const uint32_t* rw = recring + (v % kRecRing) * 16;
    const Item it(rw, p, v / nc);
    const uint32_t* ent = entring + (v % kLook) * kEntPW;
    const uint32_t nst = it.stages(p);
    const uint32_t plane = it.plane(p);
    const uint32_t st0 = (pw + kPW - g % kPW) % kPW;  // this warp's first stage of the item
    if (p.fast && p.pf && v + kPf < nv) {
      prefetch_item(v + kPf, g_pf);
      g_pf += Item(recring + ((v + kPf) % kRecRing) * 16, p, (v + kPf) / nc).stages(p);
    }
    if (it.expand && st0 < nst && p.tp == 0) {  // v of the job must be complete
      if (lane == 0) {
        const uint64_t tw = clock64();
        const uint32_t* c = p.cnt + static_cast<uint64_t>(plane) * 2 * p.njobs + it.job;
        while (ptx::ld_acquire_gpu(c) < it.ns) __nanosleep(64);
        ptx::fence_proxy_async_global();  // generic-proxy v stores -> async-proxy (TMA) reads
        tput(p, g + st0, 3, clock64() - tw);
      }
      __syncwarp();
    }
#pragma unroll 1
    for (uint32_t st = st0, j = 0; st < nst; st += kPW, ++j) {
      const uint32_t gs = g + st;
      if (lane == 0) tput(p, gs, 4, clock64());
      ptx::mbar_wait_backoff(&empty[pw], ph ^ 1u, 64);
      if (lane == 0) tput(p, gs, 0, clock64());
      const uint32_t rows = stage_rows(it, st);
      uint32_t bytes = 0;
      // ---- weight rows
      if (p.dbg & 2u) {
        bytes = 0;
      } else if (p.fast) {
        uint64_t lo;
        uint32_t len;
        row_seg(p, it, st, lane < rows ? lane : 0u, lo, len);
        if (lane < rows)
          ptx::bulk_g2s_hint(sb + lane * kRowB,
                             p.arena + (static_cast<uint64_t>(ent[j * kWRows + lane]) << L) + (lo & pmask),
                             len, &full[pw], ef);
        bytes = rows * len;
      } else {  // generic pages: every piece translated on the spot
        for (uint32_t i = 0; i < rows; ++i) {
          uint64_t lo;
          uint32_t len;
          row_seg(p, it, st, i, lo, len);
          const uint64_t hi = lo + len;
          const uint64_t np = ((hi - 1) >> L) - (lo >> L) + 1;
          for (uint64_t q = lane; q < np; q += 32) {
            const uint64_t page = (lo >> L) + q;
            const uint64_t a = max(lo, page << L), b = min(hi, (page + 1) << L);
            const uint32_t phys = __ldg(p.table + it.table_off + static_cast<uint32_t>(page));
            ptx::bulk_g2s_hint(sb + i * kRowB + static_cast<uint32_t>(a - lo),
                               p.arena + (static_cast<uint64_t>(phys) << L) + (a & pmask),
                               static_cast<uint32_t>(b - a), &full[pw], ef);
          }
          bytes += len;
        }
      }
      // ---- activations
      const bool last = st + 1 == nst;
      if (!it.expand) {
        const uint32_t k0 = st * kKC, kb = min(kKC, p.d_in - k0) * 2;
        if (lane >= 16 && lane - 16 < it.ntok)
          ptx::bulk_g2s(sb + Slot<JT>::aux + (lane - 16) * kRowB,
                        p.x + it.li * p.x_lstride_b + static_cast<uint64_t>(rw[8 + lane - 16]) * p.x_stride_b + k0 * 2,
                        kb, &full[pw]);
        bytes += it.ntok * kb;
      } else {
        if (p.tp == 2) {
          // v rows st·16 .. st·16 + 15 of the job from the gathered shards,
          // split into the fragment words the consumers read (as the
          // publisher stores them): word ((row pair)·JT + tok)·2 + {hi, lo}
          uint32_t* vw = reinterpret_cast<uint32_t*>(sb + Slot<JT>::vrows);
          const uint32_t rs = it.rank / p.tp_size;
          for (uint32_t e = lane; e < kWRows * JT; e += 32) {
            const uint32_t rp = e / (2 * JT), t = (e / 2) % JT, part = e & 1u;
            float v2[2];
#pragma unroll
            for (uint32_t q = 0; q < 2; ++q) {
              const uint32_t j = st * kWRows + 2 * rp + q;
              v2[q] = (j < it.rank && t < it.ntok)  // L2 (peers write it during the call's lifetime)
                          ? __ldcg(p.tp_vg + (static_cast<uint64_t>(j / rs) * p.tp_T + rw[8 + t]) * p.tp_rsmax + j % rs)
                          : 0.f;
            }
            const __nv_bfloat16 h0 = __float2bfloat16_rn(v2[0]), h1 = __float2bfloat16_rn(v2[1]);
            vw[e] = part ? pack_bf16x2(v2[0] - __bfloat162float(h0), v2[1] - __bfloat162float(h1))
                         : (static_cast<uint32_t>(__bfloat16_as_ushort(h1)) << 16) | __bfloat16_as_ushort(h0);
          }
          if (lane != 0) ptx::mbar_arrive(&full[pw]);  // each lane releases its own words (count 32)
        } else {
          if (lane == 24)
            ptx::bulk_g2s(sb + Slot<JT>::vrows,
                          p.v + static_cast<uint64_t>(plane) * p.vplane + it.v_off + st * kWRows * JT,
                          kWRows * JT * 4, &full[pw]);  // the job's v block is padded to 16 rows
          bytes += kWRows * JT * 4;
        }
        if (last) {
          if (lane >= 16 && lane - 16 < it.ntok)
            ptx::bulk_g2s(sb + Slot<JT>::aux + (lane - 16) * kRowB,
                          p.y[it.pj] + it.li * p.y_lstride_b[it.pj] +
                              static_cast<uint64_t>(rw[8 + lane - 16]) * p.y_stride_b[it.pj] + it.off * 2ull,
                          it.n * 2, &full[pw]);
          bytes += it.ntok * it.n * 2;
        }
      }
      if (lane == 0) tput(p, gs, 5, clock64());
      if (lane == 0) {  // the stage header, released by the arrival
        hdr[0] = (it.expand << 31) | ((st == 0) << 30) | (last << 29) | (it.pj << 16) | rows;
        hdr[1] = it.job;
        hdr[2] = it.ntok;
        hdr[3] = it.expand ? it.n : min(kKC, p.d_in - st * kKC);
        hdr[4] = it.v_off;
        hdr[5] = it.off;
        hdr[6] = plane;
        hdr[7] = (it.li << 16) | (it.expand ? it.ne : it.n);
#pragma unroll
        for (int t = 0; t < 8; ++t) hdr[8 + t] = rw[8 + t];
        ptx::mbar_arrive_expect_tx(&full[pw], bytes);
      }
      __syncwarp();
      ph ^= 1u;
    }
    g += nst;
    __syncwarp();  // record ring slot v is refilled below
    if (v + kLook < nv) {
      fetch_ent(v + kLook, g_ent);
      g_ent += Item(recring + ((v + kLook) % kRecRing) * 16, p, (v + kLook) / nc).stages(p);
    }
    fetch_rec(v + kRecRing);
    ptx::cp_async_commit();
  }
  // the stop marker goes to the owner of stage g
  if (g % kPW == pw) {
    ptx::mbar_wait(&empty[pw], ph ^ 1u);
    if (lane == 0) hdr[0] = kStop;
    if (lane == 0 || p.tp == 2) ptx::mbar_arrive(&full[pw]);  // (TP expand: the full count is 32)
  }
  cp_async_wait_group<0>();
}

// ---------------------------------------------------------------- consumers
// Every consumer warp takes a 1/8 slice of every stage (S: k-steps, E:
// 16-column tiles) and releases the slot on its own (empty count = 8).
//  S stage  D[row][tok] += A[row, k] · x[tok, k]: m16n8k16 with the 16
//           weight rows as M (ldmatrix.x4) and the tokens as N (x rows,
//           ldmatrix.x2); at the item's last stage the warps' partials are
//           summed in a fixed order by warp 0, stored to the v plane and
//           released (one red.release per element).
//  E stage  Dᵀ[col][tok] += Bᵀ[row, col]ᵀ · v[row][tok]: m16n8k16 with 16
//           output columns as M (ldmatrix.x4.trans of 16 Bᵀ rows) and N =
//           4 tokens × {bf16 hi, lo} of the fp32 v; accumulators live in
//           registers across the item's stages.
template <uint32_t JT>
__device__ void consumers(const SArgs& p, char* smem) {
  constexpr uint32_t NT = JT / 4;                  // 4-token groups of the expand's N
  constexpr uint32_t kTiles = kKC / 16 / kCWarps;  // 16-column tiles per warp (8)
  constexpr uint32_t kKSteps = kKC / 16 / kCWarps; // k-steps per warp per S stage (8)
  const uint32_t tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const uint32_t gq = lane >> 2, cc = lane & 3;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.off_bar);
  uint64_t* empty = full + p.nslots;
  const uint32_t* hdr = reinterpret_cast<const uint32_t*>(smem + p.off_hdr);
  float* part = reinterpret_cast<float*>(smem + p.off_part);  // [kPubBufs<JT>][warp][16 rows][JT]
  // ldmatrix lane offsets: 16 rows × 16 columns as four 8 × 8 matrices
  // (lanes 8j..8j+7 address matrix j: rows +8 for j & 1 (non-trans A) ...)
  const uint32_t a_off = ((lane & 7) + ((lane >> 3) & 1) * 8) * kRowB + (lane >> 4) * 16;  // S: W (M x K)
  const uint32_t x_off = Slot<JT>::aux + ((lane & 7) < JT ? (lane & 7) : 0) * kRowB + ((lane >> 3) & 1) * 16;
  const uint32_t t_off = ((lane & 7) + (lane >> 4) * 8) * kRowB + ((lane >> 3) & 1) * 16;  // E: Bᵀ, .trans
  ptx::pdl_wait();
  float sd[2][4] = {};  // two independent MMA chains
  float acc[kTiles][NT][4];
  uint32_t s_items = 0, s = 0, ph = 0;
#pragma unroll 1
  for (uint32_t gs = 0;; ++gs) {
    if (p.dbg & 32u) ptx::mbar_wait(&full[s], ph);
    else ptx::mbar_wait_spin(&full[s], ph);
    if (tid == 0) tput(p, gs, 1, clock64());
    const uint4 h0 = *reinterpret_cast<const uint4*>(hdr + s * kHdrWords);
    const uint4 h1 = *reinterpret_cast<const uint4*>(hdr + s * kHdrWords + 4);
    if (h0.x == kStop) {  // after every consumer warp handed off its last partials: tell the publisher
      ptx::named_bar_sync(1, kCThreads);
      if (tid == 0) ptx::mbar_arrive(empty + p.nslots + 2 * kPubBufs<JT>);  // cdone
      break;
    }
    const uint32_t expand = h0.x >> 31, first = (h0.x >> 30) & 1u, last = (h0.x >> 29) & 1u;
    const uint32_t pj = (h0.x >> 16) & 0xffu, rows = h0.x & 0xffffu;
    const uint32_t job = h0.y, ntok = h0.z, width = h0.w;
    const uint32_t v_off = h1.x, off = h1.y, plane = h1.z, li_n = h1.w;
    const uint32_t sbase = ptx::smem_u32(smem + s * p.slot_bytes);
    if (tid == 0) tput(p, gs, 8, (expand << 2) | (first << 1) | last);
    if (p.dbg & 1u) {
      // diagnostics: release the slot without the math (S items still publish v)
      if (!expand && last && w == 0 && lane == 0)
        red_release_add(p.cnt + static_cast<uint64_t>(plane) * 2 * p.njobs + job, ntok * rows);
    } else if (!expand) {
      // ---------------- shrink stage
      if (first) {
#pragma unroll
        for (int i = 0; i < 4; ++i) sd[0][i] = sd[1][i] = 0.f;
      }
      const uint32_t ksteps = (p.dbg & 4u) ? 0u : (width + 15) / 16;
      const bool half_tail = (width & 15u) != 0;
      // k-steps w, w + 8, ... (interleaved: smem banks), in two batches of four
      // whose fragments are all loaded before their MMAs
#pragma unroll
      for (uint32_t b = 0; b < kKSteps; b += 4) {
        uint32_t fa[4][4], fb[4][2];
#pragma unroll
        for (uint32_t j = 0; j < 4; ++j) {
          const uint32_t k = w + (b + j) * kCWarps;
          if (k < ksteps) {
            ptx::ldsm_x4(sbase + a_off + k * 32, fa[j]);
            ptx::ldsm_x2(sbase + x_off + k * 32, fb[j]);
            if (half_tail && k + 1 == ksteps) {  // k 8..15 of the last step lie past the slice
              fa[j][2] = fa[j][3] = 0u;
              fb[j][1] = 0u;
            }
          }
        }
#pragma unroll
        for (uint32_t j = 0; j < 4; ++j)
          if (w + (b + j) * kCWarps < ksteps) ptx::mma_bf16_16816(sd[j & 1], fa[j], fb[j]);
      }
      if (last) {  // hand the warps' partials to the publisher warp
        const uint32_t pbuf = s_items % kPubBufs<JT>;
        uint64_t* pready = empty + p.nslots;  // [kPubBufs<JT>] partials written (8 warps)
        uint64_t* pfree = pready + kPubBufs<JT>;  // [kPubBufs<JT>] publisher done with the buffer
        if (s_items >= kPubBufs<JT>) ptx::mbar_wait(&pfree[pbuf], ((s_items / kPubBufs<JT>) - 1) & 1u);
        float* pw = part + (pbuf * kCWarps + w) * kWRows * JT;
        if (2 * cc < JT) {  // d[0..1]: (row gq, tok 2cc..2cc+1); d[2..3]: row gq + 8
          pw[gq * JT + 2 * cc] = sd[0][0] + sd[1][0];
          pw[gq * JT + 2 * cc + 1] = sd[0][1] + sd[1][1];
          pw[(gq + 8) * JT + 2 * cc] = sd[0][2] + sd[1][2];
          pw[(gq + 8) * JT + 2 * cc + 1] = sd[0][3] + sd[1][3];
        }
        if (w == 0 && lane == 0) {  // the item's coordinates
          uint32_t* meta = reinterpret_cast<uint32_t*>(part + kPubBufs<JT> * kCWarps * kWRows * JT) + pbuf * 16;
          meta[0] = plane;
          meta[1] = p.tp ? v_off : v_off + off * JT;  // TP: the item's first shard row
          meta[2] = rows;
          meta[3] = ntok;
          meta[4] = job;
#pragma unroll
          for (uint32_t t = 0; t < 8; ++t) meta[8 + t] = hdr[s * kHdrWords + 8 + t];
        }
        ptx::mbar_arrive(&pready[pbuf]);  // every consumer thread: its own writes precede it
        ++s_items;
      }
    } else {
      // ---------------- expand stage
      if (first) {
#pragma unroll
        for (uint32_t t = 0; t < kTiles; ++t)
#pragma unroll
          for (uint32_t q = 0; q < NT; ++q)
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[t][q][i] = 0.f;
      }
      // B operand (16 rows × 8 columns n = 2·tok + part, the bf16 hi / lo of
      // v[row][tok]): this lane supplies rows 2cc, 2cc+1 (b0) and 2cc+8,
      // 2cc+9 (b1) of column gq; rows >= `rows` and tokens >= ntok are 0
      const uint32_t* vw = reinterpret_cast<const uint32_t*>(smem + s * p.slot_bytes + Slot<JT>::vrows);
      uint32_t bv[NT][2];
#pragma unroll
      for (uint32_t q = 0; q < NT; ++q) {  // (row pair cc / cc + 4, token tq, part gq & 1)
        const uint32_t tq = q * 4 + (gq >> 1);
        bv[q][0] = vw[(cc * JT + tq) * 2 + (gq & 1u)];
        bv[q][1] = vw[((cc + 4) * JT + tq) * 2 + (gq & 1u)];
      }
      // stale Bᵀ rows (>= rows) of a short stage: mask their halves of the A
      // fragment (v's pad rows are zero, but stale smem may hold non-finite bits)
      const uint32_t m_lo = (2 * cc < rows ? 0x0000ffffu : 0u) | (2 * cc + 1 < rows ? 0xffff0000u : 0u);
      const uint32_t m_hi = (2 * cc + 8 < rows ? 0x0000ffffu : 0u) | (2 * cc + 9 < rows ? 0xffff0000u : 0u);
      const uint32_t ntiles = (p.dbg & 8u) ? 0u : (width + 15) / 16;
      uint32_t a[kTiles][4];  // all of this warp's fragments first (one dependent round trip)
#pragma unroll
      for (uint32_t j = 0; j < kTiles; ++j)  // a partial last tile reads stale columns: not stored
        if (w + j * kCWarps < ntiles) ptx::ldsm_x4_trans(sbase + t_off + (w + j * kCWarps) * 32, a[j]);
      if (rows < kWRows) {
#pragma unroll
        for (uint32_t j = 0; j < kTiles; ++j) {
          a[j][0] &= m_lo;
          a[j][1] &= m_lo;
          a[j][2] &= m_hi;
          a[j][3] &= m_hi;
        }
      }
#pragma unroll
      for (uint32_t j = 0; j < kTiles; ++j)
        if (w + j * kCWarps < ntiles)
#pragma unroll
          for (uint32_t q = 0; q < NT; ++q) ptx::mma_bf16_16816(acc[j][q], a[j], bv[q]);
      if (tid == 0) tput(p, gs, 9, clock64());
      if (last && !(p.dbg & 16u)) {  // y[tok][c0 + col] = bf16(y + scale · (hi + lo)), once per item
        // the new values overwrite the staged y rows in place (each warp
        // owns its 16-column tiles), then go out as 16-byte stores
        const uint32_t li = li_n >> 16;
        char* ysm = smem + s * p.slot_bytes + Slot<JT>::aux;
        const uint32_t* toks = hdr + s * kHdrWords + 8;
#pragma unroll
        for (uint32_t q = 0; q < NT; ++q) {
          const uint32_t tok = q * 4 + cc;
          if (tok < ntok) {
            __nv_bfloat16* yrow = reinterpret_cast<__nv_bfloat16*>(ysm + tok * kRowB);
#pragma unroll
            for (uint32_t j = 0; j < kTiles; ++j) {
              const uint32_t t = w + j * kCWarps;
              if (t < ntiles) {
                const uint32_t c = t * 16 + gq;
                yrow[c] = __float2bfloat16_rn(fmaf(p.scale, acc[j][q][0] + acc[j][q][1], __bfloat162float(yrow[c])));
                yrow[c + 8] = __float2bfloat16_rn(fmaf(p.scale, acc[j][q][2] + acc[j][q][3], __bfloat162float(yrow[c + 8])));
              }
            }
          }
        }
        __syncwarp();
        // this warp's tiles of every token: (token, tile, 16-byte half) per lane
        const uint32_t nchunks = ntok * kTiles * 2;
        for (uint32_t e = lane; e < nchunks; e += 32) {
          const uint32_t tok = e / (kTiles * 2), j = (e / 2) % kTiles, hh = e & 1u;
          const uint32_t t = w + j * kCWarps, c = t * 16 + hh * 8;
          if (t < ntiles && c < width) {
            const uint4 v = *reinterpret_cast<const uint4*>(ysm + tok * kRowB + c * 2);
            char* yg = p.y[pj] + li * p.y_lstride_b[pj] + toks[tok] * p.y_stride_b[pj] +
                       (static_cast<uint64_t>(off) + c) * 2;
            *reinterpret_cast<uint4*>(yg) = v;
          }
        }
      }
    }
    ptx::mbar_arrive(&empty[s]);  // every consumer thread releases its own reads of the slot
    if (lane == 0) {
      if (w == 0) tput(p, gs, 2, clock64());
      if (w == 0 && expand && last && p.tp == 0) {  // the job's last E item resets its counters for the next call
        uint32_t* c = p.cnt + static_cast<uint64_t>(plane) * 2 * p.njobs;
        const uint32_t ne = li_n & 0xffffu;
        if (atomicAdd(c + p.njobs + job, 1u) + 1 == ne) {
          c[job] = 0u;
          c[p.njobs + job] = 0u;
        }
      }
    }
    if (++s == p.nslots) {
      s = 0;
      ph ^= 1u;
    }
  }
}

// Publisher warp: sums each S item's 8 warp partials in a fixed order,
// stores v and releases it (one red.release per S item, after the warp's
// stores are ordered by __syncwarp), off the consumers' critical path.
template <uint32_t JT>
__device__ void publisher(const SArgs& p, char* smem) {
  const uint32_t lane = threadIdx.x & 31;
  uint64_t* pready = reinterpret_cast<uint64_t*>(smem + p.off_bar) + 2 * p.nslots;
  uint64_t* pfree = pready + kPubBufs<JT>;
  const float* part = reinterpret_cast<const float*>(smem + p.off_part);
  const uint32_t* metas = reinterpret_cast<const uint32_t*>(part + kPubBufs<JT> * kCWarps * kWRows * JT);
  uint64_t* cdone = pfree + kPubBufs<JT>;  // the consumers have exited
  ptx::pdl_wait();
  for (uint32_t i = 0;; ++i) {
    const uint32_t pbuf = i % kPubBufs<JT>;
    // wait for the partials, or for the consumers' exit (they raise the stop word)
    bool done = false;
    while (!ptx::mbar_try_wait(&pready[pbuf], (i / kPubBufs<JT>) & 1u)) {
      __nanosleep(128);
      if (ptx::mbar_test_wait(cdone, 0)) {
        // every consumer arrival precedes cdone: one more look, then stop
        done = !ptx::mbar_try_wait(&pready[pbuf], (i / kPubBufs<JT>) & 1u);
        break;
      }
    }
    if (done) return;
    const uint32_t* meta = metas + pbuf * 16;
    const uint32_t plane = meta[0], vbase = meta[1], rows = meta[2], ntok = meta[3], job = meta[4];
    const float* pb = part + pbuf * kCWarps * kWRows * JT;
    if (p.tp == 1) {  // tensor-parallel shrink: v_part[tok][shard row] in fp32
      for (uint32_t e = lane; e < kWRows * JT; e += 32) {
        const uint32_t r = e / JT, t = e % JT;
        float vv = 0.f;
#pragma unroll
        for (uint32_t ww = 0; ww < kCWarps; ++ww) vv += pb[ww * kWRows * JT + e];
        if (t < ntok && r < rows) {
          const uint64_t o = static_cast<uint64_t>(meta[8 + t]) * p.tp_rsmax + vbase + r;
          if (p.tp_v) p.tp_v[o] = vv;
          for (uint32_t d = 0; d < p.tp_ndst; ++d) p.tp_dst[d][o] = vv;  // peer stores over NVLink
        }
      }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&pfree[pbuf]);
      continue;
    }
    // v is stored as the expand's B fragments want it: per row pair, token and
    // part (bf16 hi / lo of the fp32 value), a 32-bit word holding rows 2i, 2i+1
    __nv_bfloat16* vg = reinterpret_cast<__nv_bfloat16*>(p.v + static_cast<uint64_t>(plane) * p.vplane + vbase);
#pragma unroll
    for (uint32_t e = lane; e < kWRows * JT; e += 32) {
      const uint32_t r = e / JT, t = e % JT;
      float vv = 0.f;
#pragma unroll
      for (uint32_t ww = 0; ww < kCWarps; ++ww) vv += pb[ww * kWRows * JT + e];
      if (t < ntok && r < rows) {
        const __nv_bfloat16 hi = __float2bfloat16_rn(vv);
        const __nv_bfloat16 lo = __float2bfloat16_rn(vv - __bfloat162float(hi));
        const uint32_t wi = ((r >> 1) * JT + t) * 2;  // word of (row pair, token, hi)
        vg[2 * wi + (r & 1u)] = hi;
        vg[2 * (wi + 1) + (r & 1u)] = lo;
      }
    }
    __syncwarp();  // every lane's v stores are ordered before lane 0's release
    if (lane == 0) {
      red_release_add(p.cnt + static_cast<uint64_t>(plane) * 2 * p.njobs + job, rows * ntok);
      ptx::mbar_arrive(&pfree[pbuf]);
    }
  }
}

template <uint32_t JT>
__global__ void __launch_bounds__(Slot<JT>::threads, 1) bgmv_stream_kernel(const SArgs p) {
  extern __shared__ __align__(128) char smem[];
  ptx::pdl_launch_dependents();
  if (threadIdx.x == 0) {
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + p.off_bar);
    for (uint32_t s = 0; s < p.nslots; ++s) {
      ptx::mbar_init(&full[s], p.tp == 2 ? 32 : 1);  // the slot's producer (every lane in TP expand) + tx
      ptx::mbar_init(&full[p.nslots + s], kCThreads);  // empty: every consumer thread's release
    }
    for (uint32_t b = 0; b < kPubBufs<JT>; ++b) {
      ptx::mbar_init(&full[2 * p.nslots + b], kCThreads);     // partials of an S item written
      ptx::mbar_init(&full[2 * p.nslots + kPubBufs<JT> + b], 1);  // publisher done with the buffer
    }
    ptx::mbar_init(&full[2 * p.nslots + 2 * kPubBufs<JT>], 1);  // cdone: the consumers have exited
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x >= kCThreads + Slot<JT>::n * 32)
    publisher<JT>(p, smem);
  else if (threadIdx.x >= kCThreads)
    producer<JT>(p, smem, (threadIdx.x - kCThreads) >> 5);
  else
    consumers<JT>(p, smem);
  if (p.tp_ndst || p.tp_wait) {  // fused all-gather: the last CTA to finish signals
    __syncthreads();  // this CTA's peer stores (or flag reads) precede thread 0's atomic
    if (threadIdx.x == 0) {
      if (p.tp_ndst) ptx::fence_acq_rel_sys();  // the peer stores, before this CTA's count
      if (atomicAdd(p.tp_done, 1u) + 1 == gridDim.x) {
        *p.tp_done = 0u;  // for the next call (stream-ordered after this grid)
        if (p.tp_ndst) {  // shrink: one arrival in this rank's slot of every rank's flags
          ptx::fence_acq_rel_sys();  // every CTA's stores (observed through the count) first
          for (uint32_t d = 0; d < p.tp_ndst; ++d) ptx::red_release_sys_add(p.tp_flags[d], 1u);
        }
        if (p.tp_wait)  // expand: consume this call's arrival from every source
          for (uint32_t r = 0; r < p.tp_size; ++r) ptx::red_relaxed_sys_add(p.tp_wait + r, 0xffffffffu);
      }
    }
  }
}

uint32_t g_stream_dbg = 0;
uint32_t g_stream_pf = 0;  // plora_debug_set_stream_prefetch (measured slower: off)
uint32_t g_stream_ctas = 0;  // plora_debug_set_stream_ctas

struct Geom {
  uint32_t nslots, slot_bytes, off_hdr, off_bar, off_ring, off_part, smem;
};

template <uint32_t JT>
Geom geom() {
  Geom g{};
  g.slot_bytes = Slot<JT>::bytes;
  const uint32_t ring = Slot<JT>::n * (kRecRing * 16 + kLook * kEntPW) * 4;
  const uint32_t part = kPubBufs<JT> * (kCWarps * JT * kWRows + 16) * 4;
  const uint32_t per_slot = g.slot_bytes + kHdrWords * 4 + 16;
  const uint32_t fixed = ring + part + kHdrWords * 4 + 4 * kPubBufs<JT> * 8 + 256;
  g.nslots = Slot<JT>::n;
  (void)per_slot;
  g.off_hdr = g.nslots * g.slot_bytes;
  g.off_bar = g.off_hdr + (g.nslots + 1) * kHdrWords * 4;  // + the consumers' exit word
  g.off_ring = (g.off_bar + (2 * g.nslots + 2 * kPubBufs<JT> + 1) * 8 + 127) / 128 * 128;
  g.off_part = g.off_ring + ring;
  g.smem = g.off_part + part;
  return g;
}

template <uint32_t JT>
void launch_jt(const plora_plan& plan, const StreamWork& w, uint32_t layer0, uint32_t n_layers,
               const void* x, uint64_t x_stride, uint64_t x_lstride, void* const* ys,
               const uint64_t* y_strides, const uint64_t* y_lstrides, float scale,
               cudaStream_t stream, const StreamTp* tp = nullptr) {
  const plora_store& st = *plan.store;
  const ModelGeom& gm = st.geom;
  const Geom g = geom<JT>();
  if (g.nslots < 2 || g.smem > kSmemBudget) throw CudaError("bgmv_stream: shared-memory plan does not fit");
  static std::once_flag once;
  std::call_once(once, [&] {
    PLORA_CUDA(cudaFuncSetAttribute(bgmv_stream_kernel<JT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kSmemBudget)));
  });
  SArgs a{};
  a.arena = st.arena;
  a.table = st.d_table;
  a.items = (tp ? tp->items : plan.d_stitems) + w.items_off;
  a.cta_off = (tp ? tp->cta_off : plan.d_stcta) + w.cta_off;
  if (tp) {
    a.tp = tp->mode;
    a.tp_size = tp->tp_size;
    a.tp_T = tp->n_tokens;
    a.tp_rsmax = tp->rs_max;
    a.tp_v = tp->v_out;
    a.tp_vg = tp->v_in;
    a.tp_ndst = tp->n_dst;
    for (uint32_t d = 0; d < tp->n_dst; ++d) {
      a.tp_dst[d] = tp->dst[d];
      a.tp_flags[d] = tp->flags[d];
    }
    a.tp_done = tp->done;
    a.tp_wait = tp->wait;
  }
  a.x = static_cast<const char*>(x);
  a.x_stride_b = x_stride * 2;
  a.x_lstride_b = x_lstride * 2;
  const uint32_t NPT = gm.m.n_proj;
  for (uint32_t i = 0; i < w.np; ++i) {
    const uint32_t pr = w.projs[i];
    a.y[i] = static_cast<char*>(ys[i]);
    a.y_stride_b[i] = y_strides[i] * 2;
    a.y_lstride_b[i] = y_lstrides ? y_lstrides[i] * 2 : 0;
    a.blk_mult[i] = gm.blk_mult(layer0, pr);
    a.plane0[i] = layer0 * NPT + pr;
  }
  a.plu = gm.per_layer_unit;
  a.v = plan.d_sv;
  a.vplane = plan.s_vplane;
  a.cnt = plan.d_scnt;
  a.njobs = plan.s_njobs;
  a.plane_lstride = NPT;
  a.n_layers = n_layers;
  a.log2_page = st.log2_page;
  a.d_in = gm.m.d_in[w.projs[0]];
  a.d_out = gm.m.d_out[w.projs[0]];
  a.nslots = g.nslots;
  a.slot_bytes = g.slot_bytes;
  a.off_hdr = g.off_hdr;
  a.off_bar = g.off_bar;
  a.off_ring = g.off_ring;
  a.off_part = g.off_part;
  const uint64_t P = 1ull << st.log2_page;
  bool fast = P % (kKC * 2) == 0 && a.d_in % kKC == 0 && a.d_out % kKC == 0 &&
              gm.per_layer_unit % kKC == 0 && a.d_in <= 16 * kKC;  // <= 16 stages per item
  for (uint32_t i = 0; i < w.np; ++i) fast = fast && gm.prefix[w.projs[i]] % kKC == 0;
  a.fast = fast ? 1u : 0u;
  a.scale = scale;
  a.trace = trace_buffer(static_cast<uint64_t>(w.ctas) * kTraceStages * 96);
  a.dbg = g_stream_dbg;
  a.pf = g_stream_pf;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(w.ctas);
  cfg.blockDim = dim3(Slot<JT>::threads);
  cfg.dynamicSmemBytes = g.smem;
  cfg.stream = stream;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  PLORA_CUDA(cudaLaunchKernelEx(&cfg, bgmv_stream_kernel<JT>, a));
  count_launch();
}

}  // namespace

void launch_bgmv_stream(const plora_plan& plan, const StreamWork& w, uint32_t layer0,
                        uint32_t n_layers, const void* x, uint64_t x_stride, uint64_t x_lstride,
                        void* const* ys, const uint64_t* y_strides, const uint64_t* y_lstrides,
                        float scale, cudaStream_t stream) {
  if (w.ctas == 0 || n_layers == 0) return;  // no LoRA token in the batch
  if (plan.store->geom.m.d_in[w.projs[0]] % 8 || plan.store->geom.m.d_out[w.projs[0]] % 8)
    throw ValidationError("bf16 BGMV needs d_in and d_out multiples of 8");
  if (plan.s_jt == 8)
    launch_jt<8>(plan, w, layer0, n_layers, x, x_stride, x_lstride, ys, y_strides, y_lstrides, scale, stream);
  else
    launch_jt<4>(plan, w, layer0, n_layers, x, x_stride, x_lstride, ys, y_strides, y_lstrides, scale, stream);
}

void launch_bgmv_stream_tp(const plora_plan& plan, const StreamWork& w, const StreamTp& tp,
                           uint32_t layer, const void* x, uint64_t x_stride, void* y,
                           uint64_t y_stride, float scale, cudaStream_t stream) {
  if (w.ctas == 0) return;
  void* ys[1] = {y};
  const uint64_t yst[1] = {y_stride};
  launch_jt<4>(plan, w, layer, 1, x, x_stride, 0, ys, yst, nullptr, scale, stream, &tp);
}

extern "C" int plora_debug_set_stream_prefetch(uint32_t on) {
  g_stream_pf = on;
  return 0;
}

extern "C" int plora_debug_set_bgmv_flags(uint32_t flags) {
  g_stream_dbg = flags;
  return 0;
}

uint32_t stream_max_ctas(int device, uint32_t jt) {
  // one CTA per SM (the kernel holds ~210 KB of shared memory)
  static std::mutex mu;
  static std::map<int, int> sms;
  std::lock_guard<std::mutex> lk(mu);
  auto it = sms.find(device);
  if (it == sms.end()) {
    int n = 0;
    PLORA_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device));
    it = sms.emplace(device, n).first;
  }
  (void)jt;
  const uint32_t n = static_cast<uint32_t>(it->second);
  return g_stream_ctas ? std::min(n, g_stream_ctas) : n;
}

extern "C" int plora_debug_set_stream_ctas(uint32_t ctas) {
  g_stream_ctas = ctas;  // plans built afterwards use at most `ctas` CTAs (0: one per SM)
  return 0;
}

}  // namespace plora
