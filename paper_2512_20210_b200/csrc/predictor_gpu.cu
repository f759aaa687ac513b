// predict_all on the GPU: the LSTM forward (lstm.cpp:88-174, batched over
// every known adapter as predictor.cpp:109-143 does) in FP64 on one device,
// for engines whose 100 ms prediction round a host
// forward cannot meet at production adapter counts.
//
// Same parameter layout as the host re-host (predictor.cpp): per layer W
// (4H × in), U (4H × H), b (4H), column-major, gates [i, f, g, o]; head w
// (H), b; embeddings E × A.  Every gate sum is accumulated in the host's order
// (b, then W·x over k ascending, then U·h) with explicitly rounded multiplies
// and adds (no FMA contraction), so the result differs from the host path
// only through the exp / tanh implementations (~1 ulp).
//
// One CTA per block of EB examples, one thread per gate row: the layers run
// as a wavefront over time steps (layer l at step t only needs layer l-1's
// output at step t), so per-example state is h, c of every layer and z.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "predictor_gpu.hpp"

namespace plora {
namespace {

constexpr uint32_t kEB = 8;          // examples per CTA
constexpr uint32_t kMaxLayers = 4;

struct FwdArgs {
  const double* theta;
  const double* windows;   // [n][T]
  const uint32_t* adapters;
  double* out;             // [n] probabilities
  uint32_t n, H, E, T, layers;
  uint64_t w_off[kMaxLayers], u_off[kMaxLayers], b_off[kMaxLayers];
  uint64_t head_w, head_b, emb;
};

__device__ __forceinline__ double sigmoid_d(double x) {  // lstm.cpp:12-16
  if (x >= 0) return 1.0 / (1.0 + exp(-x));
  const double e = exp(x);
  return e / (1.0 + e);
}

__global__ void lstm_forward_kernel(const FwdArgs p) {
  extern __shared__ double sm[];
  const uint32_t H = p.H, G = 4 * H, L = p.layers, in0 = 1 + p.E;
  const uint32_t e0 = blockIdx.x * kEB, ne = min(kEB, p.n - e0);
  // smem: x0 [EB][in0] (layer-0 input of the step), h / c [L][EB][H], z [EB][G]
  double* x0 = sm;
  double* h = x0 + kEB * in0;
  double* c = h + L * kEB * H;
  double* z = c + L * kEB * H;
  for (uint32_t i = threadIdx.x; i < L * kEB * H; i += blockDim.x) h[i] = c[i] = 0.0;
  for (uint32_t i = threadIdx.x; i < kEB * in0; i += blockDim.x) {
    const uint32_t e = i / in0, k = i % in0;
    x0[i] = (e < ne && k > 0) ? p.theta[p.emb + static_cast<uint64_t>(p.adapters[e0 + e]) * p.E + (k - 1)] : 0.0;
  }
  __syncthreads();
  const uint32_t r = threadIdx.x;
  for (uint32_t t = 0; t < p.T; ++t) {
    if (threadIdx.x < ne) x0[threadIdx.x * in0] = p.windows[static_cast<uint64_t>(e0 + threadIdx.x) * p.T + t];
    __syncthreads();
    for (uint32_t l = 0; l < L; ++l) {
      const uint32_t in = l == 0 ? in0 : H;
      const double* xs = l == 0 ? x0 : h + (l - 1) * kEB * H;  // layer l-1's h at this step
      const uint32_t xstride = l == 0 ? in0 : H;
      const double* hl = h + l * kEB * H;
      if (r < G) {
        const double* W = p.theta + p.w_off[l];
        const double* U = p.theta + p.u_off[l];
        double acc[kEB];
        const double bv = p.theta[p.b_off[l] + r];
#pragma unroll
        for (uint32_t e = 0; e < kEB; ++e) acc[e] = bv;
        for (uint32_t k = 0; k < in; ++k) {
          const double wv = W[static_cast<uint64_t>(k) * G + r];
#pragma unroll
          for (uint32_t e = 0; e < kEB; ++e) acc[e] = __dadd_rn(acc[e], __dmul_rn(wv, xs[e * xstride + k]));
        }
        for (uint32_t k = 0; k < H; ++k) {
          const double uv = U[static_cast<uint64_t>(k) * G + r];
#pragma unroll
          for (uint32_t e = 0; e < kEB; ++e) acc[e] = __dadd_rn(acc[e], __dmul_rn(uv, hl[e * H + k]));
        }
#pragma unroll
        for (uint32_t e = 0; e < kEB; ++e) z[e * G + r] = acc[e];
      }
      __syncthreads();  // z complete; every read of this layer's h (and of h[l-1]) done
      for (uint32_t i = threadIdx.x; i < kEB * H; i += blockDim.x) {
        const uint32_t e = i / H, j = i % H;
        const double* ze = z + e * G;
        const double gi = sigmoid_d(ze[j]), gf = sigmoid_d(ze[H + j]);
        const double gg = tanh(ze[2 * H + j]), go = sigmoid_d(ze[3 * H + j]);
        double* ce = c + l * kEB * H;
        const double ct = __dadd_rn(__dmul_rn(gf, ce[i]), __dmul_rn(gi, gg));
        ce[i] = ct;
        h[l * kEB * H + i] = __dmul_rn(go, tanh(ct));
      }
      __syncthreads();
    }
  }
  // head on the last layer's final h
  if (threadIdx.x < ne) {
    const double* hl = h + (L - 1) * kEB * H + threadIdx.x * H;
    double logit = p.theta[p.head_b];
    for (uint32_t j = 0; j < H; ++j) logit = __dadd_rn(logit, __dmul_rn(p.theta[p.head_w + j], hl[j]));
    p.out[e0 + threadIdx.x] = sigmoid_d(logit);
  }
}

#define PG_CUDA(x)                                                                       \
  do {                                                                                   \
    cudaError_t err_ = (x);                                                              \
    if (err_ != cudaSuccess) throw std::runtime_error(std::string("predict_all GPU: ") + \
                                                      cudaGetErrorString(err_));         \
  } while (0)

}  // namespace

struct GpuLstm::Impl {
  int device = 0;
  cudaStream_t stream = nullptr;
  double* d_theta = nullptr;
  double* d_win = nullptr;
  uint32_t* d_ad = nullptr;
  double* d_out = nullptr;
  double* h_stage = nullptr;  // pinned: theta | windows | adapters | out
  std::size_t cap_theta = 0, cap_n = 0, cap_stage = 0;
};

GpuLstm::GpuLstm(int device) : impl_(new Impl) {
  impl_->device = device;
  int cur = 0;
  PG_CUDA(cudaGetDevice(&cur));
  PG_CUDA(cudaSetDevice(device));
  PG_CUDA(cudaStreamCreateWithFlags(&impl_->stream, cudaStreamNonBlocking));
  PG_CUDA(cudaSetDevice(cur));
}

int GpuLstm::device() const { return impl_->device; }

GpuLstm::~GpuLstm() {
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(impl_->device);
  cudaFree(impl_->d_theta);
  cudaFree(impl_->d_win);
  cudaFree(impl_->d_ad);
  cudaFree(impl_->d_out);
  cudaFreeHost(impl_->h_stage);
  if (impl_->stream) cudaStreamDestroy(impl_->stream);
  cudaSetDevice(cur);
}

void GpuLstm::forward(const GpuLstmShape& s, const double* theta, std::size_t n_theta,
                      const uint32_t* adapters, const double* windows, std::size_t n,
                      double* out) {
  if (n == 0) return;
  if (s.layers > kMaxLayers || 4 * s.hidden > 1024)
    throw std::runtime_error("predict_all GPU: layers <= 4 and 4 * hidden <= 1024 required");
  Impl& m = *impl_;
  int cur = 0;
  PG_CUDA(cudaGetDevice(&cur));
  PG_CUDA(cudaSetDevice(m.device));
  auto grow = [&](auto*& ptr, std::size_t& cap, std::size_t need, std::size_t esz) {
    if (cap >= need) return;
    cudaFree(ptr);
    ptr = nullptr;
    PG_CUDA(cudaMalloc(reinterpret_cast<void**>(&ptr), need * esz));
    cap = need;
  };
  grow(m.d_theta, m.cap_theta, n_theta, sizeof(double));
  if (m.cap_n < n) {
    cudaFree(m.d_win);
    cudaFree(m.d_ad);
    cudaFree(m.d_out);
    PG_CUDA(cudaMalloc(&m.d_win, n * s.window * sizeof(double)));
    PG_CUDA(cudaMalloc(&m.d_ad, n * sizeof(uint32_t)));
    PG_CUDA(cudaMalloc(&m.d_out, n * sizeof(double)));
    m.cap_n = n;
  }
  // one pinned staging copy up (theta, windows, adapters), one down (probabilities)
  const std::size_t stage = n_theta + n * s.window + (n + 1) / 2 + n;
  if (m.cap_stage < stage) {
    cudaFreeHost(m.h_stage);
    m.h_stage = nullptr;
    PG_CUDA(cudaMallocHost(&m.h_stage, stage * sizeof(double)));
    m.cap_stage = stage;
  }
  double* hs = m.h_stage;
  std::memcpy(hs, theta, n_theta * sizeof(double));
  std::memcpy(hs + n_theta, windows, n * s.window * sizeof(double));
  std::memcpy(hs + n_theta + n * s.window, adapters, n * sizeof(uint32_t));
  double* hout = hs + n_theta + n * s.window + (n + 1) / 2;
  PG_CUDA(cudaMemcpyAsync(m.d_theta, hs, n_theta * sizeof(double), cudaMemcpyHostToDevice, m.stream));
  PG_CUDA(cudaMemcpyAsync(m.d_win, hs + n_theta, n * s.window * sizeof(double), cudaMemcpyHostToDevice,
                          m.stream));
  PG_CUDA(cudaMemcpyAsync(m.d_ad, hs + n_theta + n * s.window, n * sizeof(uint32_t),
                          cudaMemcpyHostToDevice, m.stream));
  FwdArgs a{};
  a.theta = m.d_theta;
  a.windows = m.d_win;
  a.adapters = m.d_ad;
  a.out = m.d_out;
  a.n = static_cast<uint32_t>(n);
  a.H = s.hidden;
  a.E = s.embedding_dim;
  a.T = s.window;
  a.layers = s.layers;
  for (uint32_t l = 0; l < s.layers; ++l) {
    a.w_off[l] = s.w_off[l];
    a.u_off[l] = s.u_off[l];
    a.b_off[l] = s.b_off[l];
  }
  a.head_w = s.head_w;
  a.head_b = s.head_b;
  a.emb = s.emb;
  const uint32_t G = 4 * s.hidden;
  const uint32_t threads = std::max<uint32_t>(64, (G + 31) / 32 * 32);
  const std::size_t smem = (kEB * (1 + s.embedding_dim) + 2 * s.layers * kEB * s.hidden + kEB * G) * sizeof(double);
  if (smem > 48 * 1024)
    PG_CUDA(cudaFuncSetAttribute(lstm_forward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
  const uint32_t blocks = static_cast<uint32_t>((n + kEB - 1) / kEB);
  lstm_forward_kernel<<<blocks, threads, smem, m.stream>>>(a);
  PG_CUDA(cudaGetLastError());
  PG_CUDA(cudaMemcpyAsync(hout, m.d_out, n * sizeof(double), cudaMemcpyDeviceToHost, m.stream));
  PG_CUDA(cudaStreamSynchronize(m.stream));
  std::memcpy(out, hout, n * sizeof(double));
  PG_CUDA(cudaSetDevice(cur));
}

}  // namespace plora
