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
// Both kernels are plain streaming kernels (HBM-bound, ~1.8 flop/B): the
// work per rank at 70B shapes is small and the all-gather message is T·r/N
// fp32 per rank (4-32 KiB in total), so the call is latency-bound.
#include <cuda_bf16.h>

#include <algorithm>

#include "plan.hpp"

using namespace plora;

namespace plora {
void check_io(const plora_plan* plan, uint32_t layer, uint32_t proj, const void* x,
              uint64_t x_stride, void* y, uint64_t y_stride);
}

namespace {

struct TpArgs {
  const char* arena;
  const uint32_t* table;
  const ClusterJob* jobs;
  const char* x;       // shrink: [T, d_in]
  uint64_t x_stride_b;
  float* v;            // shrink: v_part [T, rs_max]; expand: v_gathered [N][T][rs_max]
  char* y;             // expand: [T, d_out / N] (this rank's column shard)
  uint64_t y_stride_b;
  uint64_t blk_mult;
  uint32_t log2_page;
  uint32_t d_in, d_out;
  uint32_t tp_rank, tp_size;
  uint32_t rs_max;     // row stride of v_part (floats)
  uint32_t n_tokens;
  uint32_t col0, ncols;
  float scale;
};

__device__ __forceinline__ const char* paged(const TpArgs& p, uint32_t table_off, uint64_t off) {
  const uint32_t phys = __ldg(p.table + table_off + static_cast<uint32_t>(off >> p.log2_page));
  return p.arena + (static_cast<uint64_t>(phys) << p.log2_page) + (off & ((1ull << p.log2_page) - 1));
}

__device__ __forceinline__ float bf_lo(uint32_t u) { return __uint_as_float(u << 16); }
__device__ __forceinline__ float bf_hi(uint32_t u) { return __uint_as_float(u & 0xffff0000u); }

// One warp per (job, shard row): lanes stride the row in 16-byte vectors
// (each vector inside one page: pages are >= 16 B and 16-byte aligned).
__global__ void __launch_bounds__(128) tp_shrink_kernel(const TpArgs p) {
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const ClusterJob job = p.jobs[blockIdx.x];
  const uint32_t rs = job.rank / p.tp_size;
  const uint32_t j = blockIdx.y * 4 + warp;
  if (j >= rs) return;
  const uint32_t row = p.tp_rank * rs + j;
  const uint64_t base = (static_cast<uint64_t>(job.rank) * p.blk_mult + static_cast<uint64_t>(row) * p.d_in) * 2;
  float acc[kJobTok] = {0.f, 0.f, 0.f, 0.f};
  // unrolled so several (page-table lookup -> load) chains are in flight
#pragma unroll 8
  for (uint32_t v8 = lane; v8 < p.d_in / 8; v8 += 32) {
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(paged(p, job.table_off, base + v8 * 16ull)));
#pragma unroll
    for (uint32_t t = 0; t < kJobTok; ++t) {
      if (t < job.ntok) {
        const uint4 xv = __ldg(reinterpret_cast<const uint4*>(p.x + job.tok[t] * p.x_stride_b + v8 * 16ull));
        acc[t] = fmaf(bf_lo(a.x), bf_lo(xv.x), acc[t]);
        acc[t] = fmaf(bf_hi(a.x), bf_hi(xv.x), acc[t]);
        acc[t] = fmaf(bf_lo(a.y), bf_lo(xv.y), acc[t]);
        acc[t] = fmaf(bf_hi(a.y), bf_hi(xv.y), acc[t]);
        acc[t] = fmaf(bf_lo(a.z), bf_lo(xv.z), acc[t]);
        acc[t] = fmaf(bf_hi(a.z), bf_hi(xv.z), acc[t]);
        acc[t] = fmaf(bf_lo(a.w), bf_lo(xv.w), acc[t]);
        acc[t] = fmaf(bf_hi(a.w), bf_hi(xv.w), acc[t]);
      }
    }
  }
#pragma unroll
  for (uint32_t t = 0; t < kJobTok; ++t) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[t] += __shfl_xor_sync(0xffffffffu, acc[t], o);
    if (lane == 0 && t < job.ntok) p.v[static_cast<uint64_t>(job.tok[t]) * p.rs_max + j] = acc[t];
  }
}

// One CTA per (job, 256-column block of the shard): thread = 4 columns; v of
// the job's tokens staged in shared memory from the gathered buffer.
constexpr uint32_t kExpCols = 256;
constexpr uint32_t kMaxTpRank = 256;

__global__ void __launch_bounds__(64) tp_expand_kernel(const TpArgs p) {
  __shared__ float vs[kJobTok][kMaxTpRank];
  const ClusterJob job = p.jobs[blockIdx.x];
  const uint32_t r = job.rank, rs = r / p.tp_size;
  for (uint32_t i = threadIdx.x; i < kJobTok * r; i += blockDim.x) {
    const uint32_t t = i / r, jj = i - t * r;
    vs[t][jj] = t < job.ntok ? p.v[(static_cast<uint64_t>(jj / rs) * p.n_tokens + job.tok[t]) * p.rs_max + jj % rs]
                             : 0.f;
  }
  __syncthreads();
  const uint32_t c = blockIdx.y * kExpCols + threadIdx.x * 4;  // column within the shard
  if (c >= p.ncols) return;
  const uint64_t bt = (static_cast<uint64_t>(r) * p.blk_mult + static_cast<uint64_t>(r) * p.d_in) * 2;
  float acc[kJobTok][4] = {};
#pragma unroll 8
  for (uint32_t jj = 0; jj < r; ++jj) {
    const uint64_t off = bt + (static_cast<uint64_t>(jj) * p.d_out + p.col0 + c) * 2;
    const uint2 b = __ldg(reinterpret_cast<const uint2*>(paged(p, job.table_off, off)));
    const float b0 = bf_lo(b.x), b1 = bf_hi(b.x), b2 = bf_lo(b.y), b3 = bf_hi(b.y);
#pragma unroll
    for (uint32_t t = 0; t < kJobTok; ++t) {
      const float v = vs[t][jj];
      acc[t][0] = fmaf(v, b0, acc[t][0]);
      acc[t][1] = fmaf(v, b1, acc[t][1]);
      acc[t][2] = fmaf(v, b2, acc[t][2]);
      acc[t][3] = fmaf(v, b3, acc[t][3]);
    }
  }
#pragma unroll
  for (uint32_t t = 0; t < kJobTok; ++t) {
    if (t >= job.ntok) continue;
    uint2* yp = reinterpret_cast<uint2*>(p.y + job.tok[t] * p.y_stride_b + c * 2ull);
    uint2 yo = *yp;
    __nv_bfloat162 lo = __floats2bfloat162_rn(fmaf(p.scale, acc[t][0], bf_lo(yo.x)),
                                              fmaf(p.scale, acc[t][1], bf_hi(yo.x)));
    __nv_bfloat162 hi = __floats2bfloat162_rn(fmaf(p.scale, acc[t][2], bf_lo(yo.y)),
                                              fmaf(p.scale, acc[t][3], bf_hi(yo.y)));
    yo.x = *reinterpret_cast<uint32_t*>(&lo);
    yo.y = *reinterpret_cast<uint32_t*>(&hi);
    *yp = yo;
  }
}

TpArgs tp_args(const plora_plan& plan, uint32_t layer, uint32_t proj, uint32_t tp_rank,
               uint32_t tp_size) {
  const plora_store& st = *plan.store;
  const ModelGeom& g = st.geom;
  if (g.esize != 2) throw ValidationError("tensor-parallel LoRA needs a bf16 store");
  if (layer >= g.m.n_layers || proj >= g.m.n_proj) throw ValidationError("layer / proj out of range");
  if (tp_size == 0 || tp_rank >= tp_size) throw ValidationError("tp_rank must be < tp_size");
  const uint32_t din = g.m.d_in[proj], dout = g.m.d_out[proj];
  if (din % 8 || dout % (4 * tp_size)) throw ValidationError("d_in % 8 and d_out % (4 tp_size) must be 0");
  if (plan.max_rank > kMaxTpRank) throw ValidationError("tensor-parallel LoRA: rank > 256");
  for (const ClusterJob& j : plan.cjobs)
    if (j.rank % tp_size)
      throw ValidationError("adapter rank " + std::to_string(j.rank) + " is not divisible by tp_size " +
                            std::to_string(tp_size));
  TpArgs a{};
  a.arena = st.arena;
  a.table = st.d_table;
  a.jobs = plan.d_cjobs;
  a.blk_mult = g.blk_mult(layer, proj);
  a.log2_page = st.log2_page;
  a.d_in = din;
  a.d_out = dout;
  a.tp_rank = tp_rank;
  a.tp_size = tp_size;
  a.rs_max = (plan.max_rank + tp_size - 1) / tp_size;
  a.n_tokens = plan.n_tokens;
  a.ncols = dout / tp_size;
  a.col0 = tp_rank * a.ncols;
  return a;
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
    TpArgs a = tp_args(*plan, layer, proj, tp_rank, tp_size);
    if (plan->cjobs.empty()) return 0;
    if (!x || !v_part) throw ValidationError("null x or v_part");
    if (x_stride < a.d_in || x_stride % 8 || reinterpret_cast<uintptr_t>(x) % 16)
      throw ValidationError("x must be 16-byte aligned with a row stride >= d_in, multiple of 8");
    DeviceCtx ctx(plan->store->device);
    a.x = static_cast<const char*>(x);
    a.x_stride_b = x_stride * 2;
    a.v = v_part;
    const uint32_t rows = a.rs_max;
    tp_shrink_kernel<<<dim3(static_cast<uint32_t>(plan->cjobs.size()), (rows + 3) / 4), 128, 0,
                       static_cast<cudaStream_t>(stream)>>>(a);
    PLORA_CUDA(cudaGetLastError());
    count_launch();
    return 0;
  });
}

int plora_bgmv_tp_expand(plora_plan* plan, uint32_t layer, uint32_t proj, uint32_t tp_rank,
                         uint32_t tp_size, const float* v_gathered, void* y_shard,
                         uint64_t y_stride, float scale, plora_stream_t stream) {
  return guard([&] {
    if (!plan) throw ValidationError("null plan");
    TpArgs a = tp_args(*plan, layer, proj, tp_rank, tp_size);
    if (plan->cjobs.empty()) return 0;
    if (!v_gathered || !y_shard) throw ValidationError("null v_gathered or y_shard");
    if (y_stride < a.ncols || y_stride % 4 || reinterpret_cast<uintptr_t>(y_shard) % 8)
      throw ValidationError("y_shard must be 8-byte aligned with a row stride >= d_out/tp_size, multiple of 4");
    DeviceCtx ctx(plan->store->device);
    a.v = const_cast<float*>(v_gathered);
    a.y = static_cast<char*>(y_shard);
    a.y_stride_b = y_stride * 2;
    a.scale = scale;
    tp_expand_kernel<<<dim3(static_cast<uint32_t>(plan->cjobs.size()), (a.ncols + kExpCols - 1) / kExpCols),
                       64, 0, static_cast<cudaStream_t>(stream)>>>(a);
    PLORA_CUDA(cudaGetLastError());
    count_launch();
    return 0;
  });
}

}  // extern "C"
