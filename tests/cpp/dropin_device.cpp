// The C++ face of the device path (include/plora.hpp): PagePool ->
// DeviceStore -> BatchPlan -> bgmv / sgmv_layer on a small model, checked
// against a double-precision host computation of y += s·(x·Aᵀ)·Bᵀ.
// Built and run by tests/test_cpp_dropin.py (compile-only without a GPU).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "plora.hpp"

namespace {

uint16_t to_bf16(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7fffu + ((u >> 16) & 1u);  // round to nearest even
  return static_cast<uint16_t>(u >> 16);
}
float from_bf16(uint16_t h) {
  const uint32_t u = static_cast<uint32_t>(h) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}
float pseudo(uint64_t i) {  // deterministic values in [-1, 1)
  i = (i + 0x9e3779b97f4a7c15ull) * 0xbf58476d1ce4e5b9ull;
  i ^= i >> 31;
  return static_cast<float>(i % 2001) / 1000.f - 1.f;
}

}  // namespace

int main() {
  const uint32_t L = 2, d_in = 256, d_out = 256, T = 6;
  plora_model m{};
  m.n_layers = L;
  m.n_proj = 2;
  for (uint32_t p = 0; p < 2; ++p) {
    m.d_in[p] = d_in;
    m.d_out[p] = d_out;
  }
  m.dtype = PLORA_BF16;
  const uint32_t ranks[2] = {8, 16};
  plora::PagePool pool(2048, 4096);
  plora::DeviceStore store(pool, 0, m, 4);
  std::vector<std::vector<uint16_t>> img(2);
  for (uint32_t a = 0; a < 2; ++a) {
    const uint64_t bytes = plora_model_adapter_bytes(&m, ranks[a]);
    img[a].resize(bytes / 2);
    for (uint64_t i = 0; i < img[a].size(); ++i) img[a][i] = to_bf16(0.25f * pseudo(a * 1000003 + i));
    if (pool.alloc(a, bytes) != plora::AllocStatus::ok) return 2;
    store.register_adapter(a, ranks[a]);
    store.write_pages(a, img[a].data(), bytes);
    store.publish(a);
  }
  const std::vector<int32_t> ta = {1, 0, -1, 1, 0, 1};
  plora::BatchPlan plan(store, ta);
  std::vector<uint16_t> xh(T * d_in), yh(2 * T * d_out);
  for (uint32_t i = 0; i < xh.size(); ++i) xh[i] = to_bf16(pseudo(7777 + i));
  for (uint32_t i = 0; i < yh.size(); ++i) yh[i] = to_bf16(pseudo(99999 + i));
  void *x = nullptr, *y = nullptr;
  if (cudaMalloc(&x, xh.size() * 2) != cudaSuccess || cudaMalloc(&y, yh.size() * 2) != cudaSuccess) return 3;
  cudaMemcpy(x, xh.data(), xh.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(y, yh.data(), yh.size() * 2, cudaMemcpyHostToDevice);
  const uint32_t layer = 1;
  const float scale = 0.5f;
  char* yb = static_cast<char*>(y);
  plora::bgmv(plan, layer, 0, x, d_in, yb, d_out, scale);  // projection 0, decode path
  void* ys[2] = {yb, yb + T * d_out * 2};
  const uint64_t lds[2] = {d_out, d_out};
  plora::sgmv_layer(plan, layer, x, d_in, ys, lds, scale);  // both projections, prefill path
  std::vector<uint16_t> out(yh.size());
  cudaMemcpy(out.data(), y, out.size() * 2, cudaMemcpyDeviceToHost);
  double worst = 0.0, ymax = 0.0;
  for (uint32_t p = 0; p < 2; ++p) {
    const int applications = p == 0 ? 2 : 1;  // projection 0 got bgmv and sgmv_layer
    for (uint32_t t = 0; t < T; ++t) {
      const int32_t a = ta[t];
      for (uint32_t n = 0; n < d_out; ++n) {
        double ref = from_bf16(yh[(p * T + t) * d_out + n]);
        if (a >= 0) {
          const uint32_t r = ranks[a];
          const uint64_t blk = plora_model_block_offset(&m, r, layer, p) / 2;  // elements
          double dn = 0.0;
          for (uint32_t j = 0; j < r; ++j) {
            double v = 0.0;
            for (uint32_t k = 0; k < d_in; ++k)
              v += from_bf16(xh[t * d_in + k]) * from_bf16(img[a][blk + j * d_in + k]);
            dn += v * from_bf16(img[a][blk + r * d_in + j * d_out + n]);
          }
          ref += applications * scale * dn;
        }
        const double got = from_bf16(out[(p * T + t) * d_out + n]);
        worst = std::fmax(worst, std::fabs(got - ref));
        ymax = std::fmax(ymax, std::fabs(ref));
      }
    }
  }
  cudaFree(x);
  cudaFree(y);
  const double rel = worst / ymax;
  std::printf("dropin device rel err %.3e\n", rel);
  if (!(rel <= 1e-2)) return 1;
  std::printf("dropin device ok\n");
  return 0;
}
