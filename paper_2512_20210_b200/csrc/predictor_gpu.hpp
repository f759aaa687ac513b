// GPU predict_all (predictor_gpu.cu): the host predictor's LSTM forward in
// FP64 on one device.  Plain C++ interface so predictor.cpp (host compiler)
// can call it.
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>

namespace plora {

struct GpuLstmShape {
  uint32_t hidden, embedding_dim, window, layers;
  uint64_t w_off[4], u_off[4], b_off[4];
  uint64_t head_w, head_b, emb;
};

class GpuLstm {
 public:
  explicit GpuLstm(int device);
  ~GpuLstm();
  GpuLstm(const GpuLstm&) = delete;
  GpuLstm& operator=(const GpuLstm&) = delete;
  int device() const;
  // out[i] = sigmoid(logit) of example i (adapters[i], windows[i·window ..])
  void forward(const GpuLstmShape& s, const double* theta, std::size_t n_theta,
               const uint32_t* adapters, const double* windows, std::size_t n, double* out);

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};

}  // namespace plora
