// Tensor-parallel paged LoRA for the hidden-dim-sharded configuration
// (BASELINE cfg5, Llama-2-70B q/v): the S-LoRA scheme for a column-parallel
// base projection, split into the two halves a collective sits between.
//
//   shrink   v_part[t, j] = x[t, :] · A[row_i(j), :]ᵀ for this TP rank's rows
//            row_i(j) = tp_rank · r/N + j, j < r/N, of every adapter
//            (r = the token's adapter rank; x is replicated, as the input of
//            a column-parallel layer is)
//   (all-gather of v_part over the TP group: NCCL / torch.distributed —
//    v_gathered = [N][T][rs_max], rank-major)
//   expand   y_shard[t, c] += scale · Σ_j v(t, j) · Bᵀ[j, col0 + c] over this
//            rank's output columns [col0, col0 + d_out/N), v(t, j) read from
//            the gathered buffer at [j / (r/N)][t][j % (r/N)]
//
// Every rank's pool holds the full adapter (same page layout as the
// data-parallel path); each rank streams only its shard of A and of Bᵀ, so
// the HBM traffic per GPU is 1/N of the adapter.  Math: PAPER.md:64-69; the
// reference has no multi-GPU path.
//
// Both halves run on the warp-item decode kernels (bgmv_warp.cu,
// launch_bgmv_warp_tp; the default):
//   shrink  = items (job, <= kWarpRows shard rows, K slice of >= 4 chunks;
//             the fewest power-of-two slices giving >= 6 items per SM); each
//             writes its partial sums, and the job's last item sums the
//             slices in order into v_part (or every rank's gathered buffer,
//             with the fused all-gather).
//   expand  = items (job, <= kWarpCols columns of the rank's shard) over
//             every rank row, v read from v_gathered; rank >= 64 as split
//             pairs on a CTA's two warps.
// With plora_debug_set_bgmv_impl(1) they run on the round-2 streaming kernel
// (bgmv_stream.cu) instead: one persistent CTA per SM, weight rows moved
// page by page with 1-D TMA bulk copies, mma.sync consumers.  The item lists
// depend on (batch, proj, tp_rank, tp_size) only; they are built and
// uploaded on a plan's first call for that key (outside stream capture) and
// reused by every layer.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstddef>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <queue>

#include "plan.hpp"
#include "ptx.cuh"

using namespace plora;

namespace {

struct TpGeom {
  uint32_t d_in, d_out, rs_max, ncols, col0;
};

TpGeom tp_check(const plora_plan& plan, uint32_t layer, uint32_t proj, uint32_t tp_rank,
                uint32_t tp_size) {
  const plora_store& st = *plan.store;
  const ModelGeom& g = st.geom;
  if (g.esize != 2) throw ValidationError("tensor-parallel LoRA needs a bf16 store");
  if (layer >= g.m.n_layers || proj >= g.m.n_proj) throw ValidationError("layer / proj out of range");
  if (tp_size == 0 || tp_rank >= tp_size) throw ValidationError("tp_rank must be < tp_size");
  const uint32_t din = g.m.d_in[proj], dout = g.m.d_out[proj];
  if (din % 8 || dout % (8 * tp_size)) throw ValidationError("d_in % 8 and d_out % (8 tp_size) must be 0");
  if (plan.max_rank > 256) throw ValidationError("tensor-parallel LoRA: rank > 256");
  for (const ClusterJob& j : plan.cjobs)
    if (j.rank % tp_size)
      throw ValidationError("adapter rank " + std::to_string(j.rank) + " is not divisible by tp_size " +
                            std::to_string(tp_size));
  TpGeom t{};
  t.d_in = din;
  t.d_out = dout;
  t.rs_max = (plan.max_rank + tp_size - 1) / tp_size;
  t.ncols = dout / tp_size;
  t.col0 = tp_rank * t.ncols;
  return t;
}

// The item list of one half for (proj, tp_rank, tp_size): items are
// LPT-assigned by streamed bytes to one CTA per SM.
plora_plan::TpWork& tp_work(plora_plan& plan, uint32_t proj, uint32_t tp_rank, uint32_t tp_size,
                            uint32_t half, const TpGeom& tg, cudaStream_t stream) {
  const uint64_t key = (static_cast<uint64_t>(half) << 48) | (static_cast<uint64_t>(proj) << 40) |
                       (static_cast<uint64_t>(tp_size) << 20) | tp_rank;
  auto found = plan.tpw.find(key);
  if (found != plan.tpw.end()) return found->second;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  PLORA_CUDA(cudaStreamIsCapturing(stream, &cs));
  if (cs != cudaStreamCaptureStatusNone)
    throw ValidationError("the first tensor-parallel call of a plan for (proj, tp_rank, tp_size) uploads its "
                          "item list and must run outside stream capture");
  struct Cand {
    StreamItem it;
    double cost;
  };
  std::vector<Cand> cands;
  const double ovh = 4096.0;  // per-item overhead in byte equivalents (as plan.cu)
  for (uint32_t jn = 0; jn < plan.cjobs.size(); ++jn) {
    const ClusterJob& j = plan.cjobs[jn];
    StreamItem base{};
    base.job = jn;
    base.table_off = j.table_off;
    base.rank_ntok = j.rank | (j.ntok << 16);
    for (uint32_t t = 0; t < kJobTok; ++t) base.tok[t] = t < j.ntok ? j.tok[t] : 0u;
    if (half == 1) {
      const uint32_t rs = j.rank / tp_size;
      for (uint32_t r0 = 0; r0 < rs; r0 += 16) {
        Cand c{base, 0.0};
        c.it.kind = 0;
        c.it.off = tp_rank * rs + r0;  // absolute A row
        c.it.n = std::min<uint32_t>(16, rs - r0);
        c.it.v_off = r0;  // shard row of v_part
        c.cost = 2.0 * c.it.n * tg.d_in + 1.0 * j.ntok * tg.d_in + ovh;
        cands.push_back(c);
      }
    } else {
      for (uint32_t c0 = tg.col0; c0 < tg.col0 + tg.ncols;) {
        const uint32_t c1 = std::min(tg.col0 + tg.ncols, (c0 / kStreamKC + 1) * kStreamKC);
        Cand c{base, 0.0};
        c.it.kind = kStreamExpand;
        c.it.off = c0;  // absolute output column
        c.it.n = c1 - c0;
        c.cost = 2.0 * j.rank * c.it.n + 4.0 * j.ntok * c.it.n + ovh;
        cands.push_back(c);
        c0 = c1;
      }
    }
  }
  std::stable_sort(cands.begin(), cands.end(), [](const Cand& a, const Cand& b) { return a.cost > b.cost; });
  const uint32_t ctas =
      std::min<uint32_t>(stream_max_ctas(plan.store->device, 4), static_cast<uint32_t>(cands.size()));
  std::vector<std::vector<uint32_t>> lists(ctas);
  using Load = std::pair<double, uint32_t>;
  std::priority_queue<Load, std::vector<Load>, std::greater<Load>> heap;
  for (uint32_t c = 0; c < ctas; ++c) heap.emplace(0.0, c);
  for (uint32_t k = 0; k < cands.size(); ++k) {
    Load l = heap.top();
    heap.pop();
    lists[l.second].push_back(k);
    heap.emplace(l.first + cands[k].cost, l.second);
  }
  std::vector<StreamItem> items;
  std::vector<uint32_t> cta_off;
  for (uint32_t c = 0; c < ctas; ++c) {
    cta_off.push_back(static_cast<uint32_t>(items.size()));
    for (uint32_t k : lists[c]) items.push_back(cands[k].it);
  }
  cta_off.push_back(static_cast<uint32_t>(items.size()));
  plora_plan::TpWork w;
  w.w.ctas = ctas;
  w.w.np = 1;
  w.w.projs[0] = proj;
  const uint64_t ib = items.size() * sizeof(StreamItem), cb = cta_off.size() * sizeof(uint32_t);
  DeviceCtx ctx(plan.store->device);
  // items, CTA offsets, then the fused all-gather's CTA-completion counter
  const uint64_t db = (ib + cb + 15) / 16 * 16;
  PLORA_CUDA(cudaMalloc(&w.d_items, db + 16));
  w.d_cta = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(w.d_items) + ib);
  w.d_done = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(w.d_items) + db);
  PLORA_CUDA(cudaMallocHost(&w.h_stage, db + 16));
  std::memset(w.h_stage, 0, db + 16);
  std::memcpy(w.h_stage, items.data(), ib);
  std::memcpy(w.h_stage + ib, cta_off.data(), cb);
  PLORA_CUDA(cudaMemcpyAsync(w.d_items, w.h_stage, db + 16, cudaMemcpyHostToDevice, stream));
  return plan.tpw.emplace(key, w).first->second;
}

// The warp-item lists of one half (the default TP path): shrink items are
// (job, <= kWarpRows(ntok) shard rows, K slice of 4 chunks = 1024 inputs) —
// ~16 KiB each, so even a TP = 8 shard gives every SM several — and expand
// items (job, <= kWarpCols(ntok) columns of the shard), heaviest first.  One
// allocation: items, then (shrink) the per-job partial blocks and their
// counters, then the launch counter; counters start at zero and every call
// leaves them at zero.
plora_plan::TpWork& tp_work_warp(plora_plan& plan, uint32_t proj, uint32_t tp_rank, uint32_t tp_size,
                                 uint32_t half, const TpGeom& tg, cudaStream_t stream) {
  const uint64_t key = (1ull << 56) | (static_cast<uint64_t>(half) << 48) | (static_cast<uint64_t>(proj) << 40) |
                       (static_cast<uint64_t>(tp_size) << 20) | tp_rank;
  auto found = plan.tpw.find(key);
  if (found != plan.tpw.end()) return found->second;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  PLORA_CUDA(cudaStreamIsCapturing(stream, &cs));
  if (cs != cudaStreamCaptureStatusNone)
    throw ValidationError("the first tensor-parallel call of a plan for (proj, tp_rank, tp_size) uploads its "
                          "item list and must run outside stream capture");
  const uint32_t ncall = (tg.d_in + 255) / 256;
  // expand items: kWarpCols columns, or 256 when that leaves fewer than 4
  // items per SM (narrow shards at TP >= 4: rank 0 of cfg5 at TP 4 / 8
  // 18.7 -> 15.2 / 16.6 -> 14.8 us; wide shards measured slower narrow)
  uint64_t wide_items = 0;
  for (const ClusterJob& j : plan.cjobs) wide_items += (tg.ncols + kWarpCols(j.ntok) - 1) / kWarpCols(j.ntok);
  const bool narrow = half == 2 && wide_items < 4ull * std::max(1, plan.store->num_sms);
  // K slices of the shrink: the fewest (a power of two, slices of >= 4
  // chunks) that give >= 6 items per SM — cfg5 measured best at ~900-1400
  // items for every TP size (profiles/r02o_tp_warp.txt: fewer leave SMs idle,
  // more add per-item and partial-sum overhead)
  uint32_t ks = 1;
  if (half == 1) {
    uint64_t blocks = 0;
    for (const ClusterJob& j : plan.cjobs) blocks += (j.rank / tp_size + kWarpRows(j.ntok) - 1) / kWarpRows(j.ntok);
    const uint64_t target = 6ull * std::max(1, plan.store->num_sms);
    while (blocks * ks < target && (ncall + 2 * ks - 1) / (2 * ks) >= 4) ks *= 2;
  }
  std::vector<WarpItem> items, pairs;  // pairs: split expand items (adjacent)
  uint64_t pfl = 0;  // shrink: partial floats
  for (const ClusterJob& j : plan.cjobs) {
    WarpItem base{};
    base.table_off = j.table_off;
    for (uint32_t t = 0; t < kWarpJobTok; ++t) base.tok[t] = t < j.ntok ? j.tok[t] : 0u;
    auto meta = [&](uint32_t n) { return j.rank | (j.ntok << 9) | (n << 16); };
    if (half == 1) {
      const uint32_t rs = j.rank / tp_size, R = kWarpRows(j.ntok);
      base.v_off = static_cast<uint32_t>(pfl);
      for (uint32_t k = 0; k < ks; ++k)
        for (uint32_t r0 = 0; r0 < rs; r0 += R) {
          WarpItem it = base;
          it.meta = meta(std::min(R, rs - r0));
          it.off = (tp_rank * rs + r0) | (k << 16);  // absolute A row | K slice
          items.push_back(it);
        }
      pfl += static_cast<uint64_t>(ks) * j.ntok * rs;
    } else {
      const uint32_t C = narrow ? 256u : kWarpCols(j.ntok);
      for (uint32_t c0 = tg.col0; c0 < tg.col0 + tg.ncols; c0 += C) {
        WarpItem it = base;
        it.meta = meta(std::min(C, tg.col0 + tg.ncols - c0));
        it.off = c0;  // absolute output column
        if (j.rank >= kWarpSplitRows) {  // split pair: rows [0, h) / [h, r) on a CTA's two warps
          it.meta |= kWarpSplit;
          pairs.push_back(it);
          it.meta |= kWarpSecond;
          pairs.push_back(it);
        } else {
          items.push_back(it);
        }
      }
    }
  }
  if (pfl > 0xffffffffull) throw ValidationError("batch too large for one plan");
  auto cost = [&](const WarpItem& it) {
    return half == 1 ? (it.meta >> 16) & 0x3ffu : (it.meta & 0x1ffu) * ((it.meta >> 16) & 0x3ffu);
  };
  std::stable_sort(items.begin(), items.end(), [&](const WarpItem& a, const WarpItem& b) { return cost(a) > cost(b); });
  if (!pairs.empty()) {  // pairs first, heaviest first, each on an even position
    std::vector<uint32_t> pi(pairs.size() / 2);
    std::iota(pi.begin(), pi.end(), 0u);
    std::stable_sort(pi.begin(), pi.end(),
                     [&](uint32_t a, uint32_t b) { return cost(pairs[2 * a]) > cost(pairs[2 * b]); });
    std::vector<WarpItem> all;
    for (uint32_t k : pi) {
      all.push_back(pairs[2 * k]);
      all.push_back(pairs[2 * k + 1]);
    }
    all.insert(all.end(), items.begin(), items.end());
    items.swap(all);
  }
  const uint64_t ib = items.size() * sizeof(WarpItem);
  const uint64_t pb = pfl * 4;                    // partials
  const uint64_t total = ib + 2 * pb + 16;        // items | partials | counters | launch counter
  plora_plan::TpWork w;
  DeviceCtx ctx(plan.store->device);
  char* d = nullptr;
  PLORA_CUDA(cudaMalloc(&d, total));
  w.d_items = reinterpret_cast<StreamItem*>(d);
  PLORA_CUDA(cudaMallocHost(&w.h_stage, total));
  std::memset(w.h_stage, 0, total);
  std::memcpy(w.h_stage, items.data(), ib);
  PLORA_CUDA(cudaMemcpyAsync(d, w.h_stage, total, cudaMemcpyHostToDevice, stream));
  w.wt.half = half;
  w.wt.narrow = narrow ? 1u : 0u;
  w.wt.items = reinterpret_cast<const WarpItem*>(d);
  w.wt.n_items = static_cast<uint32_t>(items.size());
  w.wt.ks = ks;
  w.wt.njobs = static_cast<uint32_t>(plan.cjobs.size());
  w.wt.tp_size = tp_size;
  w.wt.tp_rank = tp_rank;
  w.wt.rs_max = tg.rs_max;
  w.wt.n_tokens = plan.n_tokens;
  w.wt.part = reinterpret_cast<float*>(d + ib);
  w.wt.cnt = reinterpret_cast<uint32_t*>(d + ib + pb);
  w.wt.done = reinterpret_cast<uint32_t*>(d + ib + 2 * pb);
  return plan.tpw.emplace(key, w).first->second;
}

struct TpFlags {
  uint32_t* flags[kMaxTp];
  uint32_t n;
};
// A rank with no LoRA token still completes its share of the fused all-gather.
__global__ void tp_flag_bump_kernel(const TpFlags f) {
  if (threadIdx.x < f.n) ptx::red_release_sys_add(f.flags[threadIdx.x], 1u);
}

__global__ void tp_flag_consume_kernel(uint32_t* flags, uint32_t n) {
  if (threadIdx.x < n) {
    while (ptx::ld_acquire_sys(flags + threadIdx.x) == 0u) __nanosleep(128);
    ptx::red_relaxed_sys_add(flags + threadIdx.x, 0xffffffffu);
  }
}

}  // namespace

// One rank's expand; flags != nullptr: first wait for the fused all-gather
// (every rank's shrink_push of this call has added 1 to its slot), and
// consume those arrivals at the end.
namespace {
int tp_expand(plora_plan* plan, uint32_t layer, uint32_t proj, uint32_t tp_rank, uint32_t tp_size,
              const float* v_gathered, uint32_t* flags, void* y_shard, uint64_t y_stride, float scale,
              plora_stream_t stream) {
  if (!plan) throw ValidationError("null plan");
  const TpGeom tg = tp_check(*plan, layer, proj, tp_rank, tp_size);
  if (plan->cjobs.empty()) {
    if (flags) {  // no LoRA token: still take this call's arrivals
      if (tp_size > kMaxTp) throw ValidationError("fused all-gather: tp_size > " + std::to_string(kMaxTp));
      DeviceCtx ctx(plan->store->device);
      tp_flag_consume_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(flags, tp_size);
      PLORA_CUDA(cudaGetLastError());
      count_launch();
    }
    return 0;
  }
  if (!v_gathered || !y_shard) throw ValidationError("null v_gathered or y_shard");
  if (y_stride < tg.ncols || y_stride % 8 || reinterpret_cast<uintptr_t>(y_shard) % 16)
    throw ValidationError("y_shard must be 16-byte aligned with a row stride >= d_out/tp_size, multiple of 8");
  DeviceCtx ctx(plan->store->device);
  const cudaStream_t s = static_cast<cudaStream_t>(stream);
  // the kernel addresses output column c (absolute in d_out) at y + c
  char* y = static_cast<char*>(y_shard) - static_cast<ptrdiff_t>(tg.col0) * 2;
  if (flags && tp_size > kMaxTp) throw ValidationError("fused all-gather: tp_size > " + std::to_string(kMaxTp));
  if (bgmv_impl() != 1) {  // warp items (default)
    WarpTp t = tp_work_warp(*plan, proj, tp_rank, tp_size, 2, tg, s).wt;
    t.v_in = v_gathered;
    t.wait = flags;
    launch_bgmv_warp_tp(*plan, t, layer, proj, nullptr, 0, y, y_stride, scale, s);
    return 0;
  }
  const plora_plan::TpWork& w = tp_work(*plan, proj, tp_rank, tp_size, 2, tg, s);
  StreamTp tp{};
  tp.mode = 2;
  tp.tp_size = tp_size;
  tp.n_tokens = plan->n_tokens;
  tp.rs_max = tg.rs_max;
  tp.v_in = v_gathered;
  tp.items = w.d_items;
  tp.cta_off = w.d_cta;
  if (flags) {
    tp.wait = flags;
    tp.done = w.d_done;
  }
  launch_bgmv_stream_tp(*plan, w.w, tp, layer, nullptr, 0, y, y_stride, scale, s);
  return 0;
}
}  // namespace

extern "C" {

uint32_t plora_tp_shard_rows(const plora_plan* plan, uint32_t tp_size) {
  if (!plan || tp_size == 0) return 0;
  return (plan->max_rank + tp_size - 1) / tp_size;
}

int plora_bgmv_tp_shrink(plora_plan* plan, uint32_t layer, uint32_t proj, uint32_t tp_rank,
                         uint32_t tp_size, const void* x, uint64_t x_stride, float* v_part,
                         plora_stream_t stream) {
  return guard([&] {
    if (!plan) throw ValidationError("null plan");
    const TpGeom tg = tp_check(*plan, layer, proj, tp_rank, tp_size);
    if (plan->cjobs.empty()) return 0;
    if (!x || !v_part) throw ValidationError("null x or v_part");
    if (x_stride < tg.d_in || x_stride % 8 || reinterpret_cast<uintptr_t>(x) % 16)
      throw ValidationError("x must be 16-byte aligned with a row stride >= d_in, multiple of 8");
    DeviceCtx ctx(plan->store->device);
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (bgmv_impl() != 1) {  // warp items (default)
      WarpTp t = tp_work_warp(*plan, proj, tp_rank, tp_size, 1, tg, s).wt;
      t.v_out = v_part;
      launch_bgmv_warp_tp(*plan, t, layer, proj, x, x_stride, nullptr, 0, 1.f, s);
      return 0;
    }
    const plora_plan::TpWork& w = tp_work(*plan, proj, tp_rank, tp_size, 1, tg, s);
    StreamTp tp{};
    tp.mode = 1;
    tp.tp_size = tp_size;
    tp.n_tokens = plan->n_tokens;
    tp.rs_max = tg.rs_max;
    tp.v_out = v_part;
    tp.items = w.d_items;
    tp.cta_off = w.d_cta;
    launch_bgmv_stream_tp(*plan, w.w, tp, layer, x, x_stride, nullptr, 0, 1.f, s);
    return 0;
  });
}

int plora_bgmv_tp_shrink_push(plora_plan* plan, uint32_t layer, uint32_t proj, uint32_t tp_rank,
                              uint32_t tp_size, const void* x, uint64_t x_stride,
                              float* const* peer_v_gathered, uint32_t* const* peer_flags,
                              plora_stream_t stream) {
  return guard([&] {
    if (!plan) throw ValidationError("null plan");
    const TpGeom tg = tp_check(*plan, layer, proj, tp_rank, tp_size);
    if (tp_size > kMaxTp) throw ValidationError("fused all-gather: tp_size > " + std::to_string(kMaxTp));
    if (!peer_v_gathered || !peer_flags) throw ValidationError("null peer buffers");
    for (uint32_t d = 0; d < tp_size; ++d)
      if (!peer_v_gathered[d] || !peer_flags[d]) throw ValidationError("null peer buffer " + std::to_string(d));
    if (!x) throw ValidationError("null x");
    if (x_stride < tg.d_in || x_stride % 8 || reinterpret_cast<uintptr_t>(x) % 16)
      throw ValidationError("x must be 16-byte aligned with a row stride >= d_in, multiple of 8");
    DeviceCtx ctx(plan->store->device);
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    StreamTp tp{};
    tp.mode = 1;
    tp.tp_size = tp_size;
    tp.n_tokens = plan->n_tokens;
    tp.rs_max = tg.rs_max;
    tp.n_dst = tp_size;
    const uint64_t block = static_cast<uint64_t>(tp_rank) * plan->n_tokens * tg.rs_max;  // this rank's rows
    for (uint32_t d = 0; d < tp_size; ++d) {
      tp.dst[d] = peer_v_gathered[d] + block;
      tp.flags[d] = peer_flags[d] + tp_rank;  // this rank's slot of rank d's flag array
    }
    if (plan->cjobs.empty()) {  // nothing to write: still tell every rank this call is done
      TpFlags f{};
      f.n = tp_size;
      for (uint32_t d = 0; d < tp_size; ++d) f.flags[d] = peer_flags[d] + tp_rank;
      tp_flag_bump_kernel<<<1, 32, 0, s>>>(f);
      PLORA_CUDA(cudaGetLastError());
      count_launch();
      return 0;
    }
    if (bgmv_impl() != 1) {  // warp items (default)
      WarpTp t = tp_work_warp(*plan, proj, tp_rank, tp_size, 1, tg, s).wt;
      t.n_dst = tp_size;
      for (uint32_t d = 0; d < tp_size; ++d) {
        t.dst[d] = tp.dst[d];
        t.flags[d] = tp.flags[d];
      }
      launch_bgmv_warp_tp(*plan, t, layer, proj, x, x_stride, nullptr, 0, 1.f, s);
      return 0;
    }
    const plora_plan::TpWork& w = tp_work(*plan, proj, tp_rank, tp_size, 1, tg, s);
    tp.items = w.d_items;
    tp.cta_off = w.d_cta;
    tp.done = w.d_done;
    launch_bgmv_stream_tp(*plan, w.w, tp, layer, x, x_stride, nullptr, 0, 1.f, s);
    return 0;
  });
}

int plora_bgmv_tp_expand_wait(plora_plan* plan, uint32_t layer, uint32_t proj, uint32_t tp_rank,
                              uint32_t tp_size, const float* v_gathered, uint32_t* flags,
                              void* y_shard, uint64_t y_stride, float scale, plora_stream_t stream) {
  return guard([&] {
    if (!flags) throw ValidationError("null flags");
    return tp_expand(plan, layer, proj, tp_rank, tp_size, v_gathered, flags, y_shard, y_stride, scale, stream);
  });
}

int plora_bgmv_tp_expand(plora_plan* plan, uint32_t layer, uint32_t proj, uint32_t tp_rank,
                         uint32_t tp_size, const float* v_gathered, void* y_shard,
                         uint64_t y_stride, float scale, plora_stream_t stream) {
  return guard([&] {
    return tp_expand(plan, layer, proj, tp_rank, tp_size, v_gathered, nullptr, y_shard, y_stride, scale, stream);
  });
}

}  // extern "C"
