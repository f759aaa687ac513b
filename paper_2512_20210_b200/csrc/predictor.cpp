// Host-side demand predictor — the input of the predictor-driven prefetch
// hook.  Eigen-free C++ restatement of the reference's stacked LSTM
// (include/lorasim/lstm.hpp:11-85, src/lstm.cpp:1-331) and online predictor
// (include/lorasim/predictor.hpp:12-111, src/predictor.cpp:1-155).  It stays
// on the CPU as the north star asks; predict_all over ~1000 adapters is
// threaded across the batch.
//
// Same parameter layout (per layer W(4H×in), U(4H×H), b(4H), head w(H), b,
// embeddings E×A; column-major, gates [i, f, g, o]), same initialization
// (mt19937_64(seed), U(-1/√H, 1/√H)), same BPTT equations and Adam update,
// same replay sampling and interval bookkeeping.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <deque>
#include <fstream>
#include <random>
#include <thread>
#include <vector>

#include "common.hpp"
#include "predictor_gpu.hpp"

namespace plora {
namespace {

constexpr double kClamp = 1e-7;     // lstm.cpp:10
constexpr double kProbEps = 1e-12;  // predictor.cpp:11

double sigmoid(double x) {  // lstm.cpp:12-16
  if (x >= 0) return 1.0 / (1.0 + std::exp(-x));
  double e = std::exp(x);
  return e / (1.0 + e);
}

double clamped_ce(double p, double y) {  // lstm.cpp:22-25
  double q = std::min(1.0 - kClamp, std::max(kClamp, p));
  return -(y * std::log(q) + (1.0 - y) * std::log(1.0 - q));
}

// z[r] = b[r] + Σ_k W[k·G + r]·x[k] + Σ_k U[k·G + r]·h[k] for the G = 4H gate
// rows, summed in that order (blocks of 32 rows kept in registers across k).
// Cloned per host ISA; with -ffp-contract=off every clone rounds identically.
__attribute__((target_clones("avx512f", "avx2", "default")))
void gate_sums(const double* b, const double* W, const double* U, const double* x,
               const double* h, std::size_t in, std::size_t H, double* z) {
  constexpr std::size_t kRB = 32;
  const std::size_t G = 4 * H;
  std::size_t r0 = 0;
  for (; r0 + kRB <= G; r0 += kRB) {
    double acc[kRB];
    for (std::size_t i = 0; i < kRB; ++i) acc[i] = b[r0 + i];
    for (std::size_t k = 0; k < in; ++k) {
      const double xv = x[k];
      const double* col = W + k * G + r0;
      for (std::size_t i = 0; i < kRB; ++i) acc[i] += col[i] * xv;
    }
    for (std::size_t k = 0; k < H; ++k) {
      const double hv = h[k];
      const double* col = U + k * G + r0;
      for (std::size_t i = 0; i < kRB; ++i) acc[i] += col[i] * hv;
    }
    for (std::size_t i = 0; i < kRB; ++i) z[r0 + i] = acc[i];
  }
  for (std::size_t r = r0; r < G; ++r) {  // a last partial block
    double a = b[r];
    for (std::size_t k = 0; k < in; ++k) a += W[k * G + r] * x[k];
    for (std::size_t k = 0; k < H; ++k) a += U[k * G + r] * h[k];
    z[r] = a;
  }
}

template <class F>
void parallel_for(std::size_t n, std::size_t grain, F&& f) {
  const std::size_t hw = std::max<std::size_t>(1, std::thread::hardware_concurrency());
  const std::size_t nt = std::min(hw, (n + grain - 1) / grain);
  if (nt <= 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> th;
  const std::size_t chunk = (n + nt - 1) / nt;
  for (std::size_t i = 0; i < nt; ++i) {
    const std::size_t lo = i * chunk, hi = std::min(n, lo + chunk);
    if (lo < hi) th.emplace_back([&f, lo, hi] { f(lo, hi); });
  }
  for (auto& t : th) t.join();
}

}  // namespace

struct Example {
  uint32_t adapter = 0;
  std::vector<double> window;
  double label = 0.0;
};

class Lstm {
 public:
  Lstm(const plora_lstm_config& cfg, uint64_t seed) : c_(cfg) {
    // PredictorConfig::validate (lstm.cpp:29-35)
    if (c_.window < 1) throw ValidationError("predictor window must be >= 1");
    if (c_.hidden < 1) throw ValidationError("hidden units must be >= 1");
    if (c_.layers < 1) throw ValidationError("layers must be >= 1");
    if (c_.num_adapters < 1) throw ValidationError("predictor needs >= 1 adapter");
    if (c_.learning_rate <= 0) throw ValidationError("learning rate must be positive");
    in0_ = 1 + c_.embedding_dim;
    const std::size_t H = c_.hidden;
    std::size_t off = 0;
    for (uint32_t l = 0; l < c_.layers; ++l) {  // lstm.cpp:59-70
      const std::size_t in = l == 0 ? in0_ : H;
      w_off_.push_back(off);
      off += 4 * H * in;
      u_off_.push_back(off);
      off += 4 * H * H;
      b_off_.push_back(off);
      off += 4 * H;
    }
    head_w_off_ = off;
    off += H;
    head_b_off_ = off;
    off += 1;
    emb_off_ = off;
    off += static_cast<std::size_t>(c_.embedding_dim) * c_.num_adapters;
    theta_.resize(off);
    std::mt19937_64 rng(seed);  // lstm.cpp:75-78
    const double bound = 1.0 / std::sqrt(static_cast<double>(H));
    std::uniform_real_distribution<double> dist(-bound, bound);
    for (auto& v : theta_) v = dist(rng);
    m_.assign(off, 0.0);
    v_.assign(off, 0.0);
  }

  const plora_lstm_config& cfg() const { return c_; }
  GpuLstmShape gpu_shape() const {
    GpuLstmShape s{};
    s.hidden = c_.hidden;
    s.embedding_dim = c_.embedding_dim;
    s.window = c_.window;
    s.layers = c_.layers;
    for (uint32_t l = 0; l < c_.layers && l < 4; ++l) {
      s.w_off[l] = w_off_[l];
      s.u_off[l] = u_off_[l];
      s.b_off[l] = b_off_[l];
    }
    s.head_w = head_w_off_;
    s.head_b = head_b_off_;
    s.emb = emb_off_;
    return s;
  }
  std::vector<double>& theta() { return theta_; }
  const std::vector<double>& theta() const { return theta_; }

  void validate_batch(const std::vector<Example>& batch) const {
    if (batch.empty()) throw ValidationError("empty batch");
    for (const auto& ex : batch) {
      if (ex.window.size() != c_.window)
        throw ValidationError("window length " + std::to_string(ex.window.size()) +
                              " does not match configured window " + std::to_string(c_.window));
      if (ex.adapter >= c_.num_adapters) throw ValidationError("adapter index out of range");
    }
  }

  // Per-example recurrence (lstm.cpp:120-173).  When `cache` is non-null it
  // receives gates/states [layer][t][4·H + 3·H] for the backward pass.
  double logit_one(const Example& ex, std::vector<double>* cache) const {
    const std::size_t H = c_.hidden, E = c_.embedding_dim, T = c_.window;
    std::vector<double> x(std::max<std::size_t>(in0_, H) * T), xn(H * T);
    for (std::size_t t = 0; t < T; ++t) {
      x[t * in0_] = ex.window[t];
      for (std::size_t e = 0; e < E; ++e)
        x[t * in0_ + 1 + e] = theta_[emb_off_ + ex.adapter * E + e];
    }
    std::vector<double> z(4 * H), h(H), c(H);
    std::size_t in = in0_;
    const std::size_t per_t = 7 * H;  // i f g o c tanh_c h
    for (uint32_t l = 0; l < c_.layers; ++l) {
      const double* W = theta_.data() + w_off_[l];
      const double* U = theta_.data() + u_off_[l];
      const double* b = theta_.data() + b_off_[l];
      std::fill(h.begin(), h.end(), 0.0);
      std::fill(c.begin(), c.end(), 0.0);
      for (std::size_t t = 0; t < T; ++t) {
        std::copy(b, b + 4 * H, z.begin());
        const double* xt = x.data() + t * in;
        for (std::size_t k = 0; k < in; ++k) {
          const double xv = xt[k];
          const double* col = W + k * 4 * H;
          for (std::size_t r = 0; r < 4 * H; ++r) z[r] += col[r] * xv;
        }
        for (std::size_t k = 0; k < H; ++k) {
          const double hv = h[k];
          const double* col = U + k * 4 * H;
          for (std::size_t r = 0; r < 4 * H; ++r) z[r] += col[r] * hv;
        }
        double* cl = cache ? cache->data() + (l * T + t) * per_t : nullptr;
        for (std::size_t j = 0; j < H; ++j) {
          const double gi = sigmoid(z[j]), gf = sigmoid(z[H + j]);
          const double gg = std::tanh(z[2 * H + j]), go = sigmoid(z[3 * H + j]);
          const double ct = gf * c[j] + gi * gg, tc = std::tanh(ct), ht = go * tc;
          c[j] = ct;
          h[j] = ht;
          if (cl) {
            cl[j] = gi;
            cl[H + j] = gf;
            cl[2 * H + j] = gg;
            cl[3 * H + j] = go;
            cl[4 * H + j] = ct;
            cl[5 * H + j] = tc;
            cl[6 * H + j] = ht;
          }
          xn[t * H + j] = ht;  // feeds the next layer
        }
      }
      x.swap(xn);
      xn.assign(H * T, 0.0);
      in = H;
    }
    double logit = theta_[head_b_off_];
    for (std::size_t j = 0; j < H; ++j) logit += theta_[head_w_off_ + j] * h[j];
    return logit;
  }

  // Inference over many examples (predict_all): examples in chunks of kFwdChunk
  // share every pass over W / U (the reference's batched Eigen products,
  // lstm.cpp:130-161), the gate sums of each example accumulated in the same
  // order as logit_one, so the result is bit-identical to it.
  static constexpr std::size_t kFwdChunk = 16;
  void logits_chunk(const Example* ex, std::size_t n, double* out) const {
    const std::size_t H = c_.hidden, E = c_.embedding_dim, T = c_.window, G = 4 * H;
    const std::size_t in_max = std::max<std::size_t>(in0_, H);
    std::vector<double> x(n * T * in_max), xn(n * T * H), z(n * G), h(n * H), c(n * H);
    for (std::size_t e = 0; e < n; ++e)
      for (std::size_t t = 0; t < T; ++t) {
        double* xt = x.data() + (e * T + t) * in0_;
        xt[0] = ex[e].window[t];
        for (std::size_t q = 0; q < E; ++q) xt[1 + q] = theta_[emb_off_ + ex[e].adapter * E + q];
      }
    std::size_t in = in0_;
    for (uint32_t l = 0; l < c_.layers; ++l) {
      const double* W = theta_.data() + w_off_[l];
      const double* U = theta_.data() + u_off_[l];
      const double* b = theta_.data() + b_off_[l];
      std::fill(h.begin(), h.end(), 0.0);
      std::fill(c.begin(), c.end(), 0.0);
      for (std::size_t t = 0; t < T; ++t) {
        // z = b + W·x_t + U·h, per (example, gate row) summed over k in order
        for (std::size_t e = 0; e < n; ++e)
          gate_sums(b, W, U, x.data() + (e * T + t) * in, h.data() + e * H, in, H, z.data() + e * G);
        for (std::size_t e = 0; e < n; ++e) {
          const double* ze = z.data() + e * G;
          double* he = h.data() + e * H;
          double* ce = c.data() + e * H;
          for (std::size_t j = 0; j < H; ++j) {
            const double gi = sigmoid(ze[j]), gf = sigmoid(ze[H + j]);
            const double gg = std::tanh(ze[2 * H + j]), go = sigmoid(ze[3 * H + j]);
            const double ct = gf * ce[j] + gi * gg, ht = go * std::tanh(ct);
            ce[j] = ct;
            he[j] = ht;
            xn[(e * T + t) * H + j] = ht;  // feeds the next layer
          }
        }
      }
      x.swap(xn);
      in = H;
    }
    for (std::size_t e = 0; e < n; ++e) {
      double logit = theta_[head_b_off_];
      for (std::size_t j = 0; j < H; ++j) logit += theta_[head_w_off_ + j] * h[e * H + j];
      out[e] = logit;
    }
  }

  std::vector<double> forward(const std::vector<Example>& batch) const {
    validate_batch(batch);
    std::vector<double> out(batch.size());
    const std::size_t nch = (batch.size() + kFwdChunk - 1) / kFwdChunk;
    parallel_for(nch, 1, [&](std::size_t lo, std::size_t hi) {
      for (std::size_t q = lo; q < hi; ++q) {
        const std::size_t b0 = q * kFwdChunk, n = std::min(kFwdChunk, batch.size() - b0);
        logits_chunk(batch.data() + b0, n, out.data() + b0);
        for (std::size_t i = b0; i < b0 + n; ++i) out[i] = sigmoid(out[i]);
      }
    });
    return out;
  }

  double loss_on(const std::vector<Example>& batch) const {  // lstm.cpp:183-188
    auto p = forward(batch);
    double total = 0.0;
    for (std::size_t b = 0; b < batch.size(); ++b) total += clamped_ce(p[b], batch[b].label);
    return total / static_cast<double>(batch.size());
  }

  // d(mean CE)/dθ by backpropagation through time (lstm.cpp:190-281).
  // d(mean CE)/dθ.  Examples are processed in fixed chunks of kGradChunk
  // (threads over chunks), partial gradients summed in chunk order, so the
  // result does not depend on the host's thread count.
  static constexpr std::size_t kGradChunk = 8;
  std::vector<double> gradient(const std::vector<Example>& batch) const {
    validate_batch(batch);
    const std::size_t B = batch.size(), P = theta_.size();
    const std::size_t n_chunks = (B + kGradChunk - 1) / kGradChunk;
    std::vector<double> part(n_chunks * P, 0.0);
    parallel_for(n_chunks, 1, [&](std::size_t lo, std::size_t hi) {
      for (std::size_t c = lo; c < hi; ++c)
        grad_range(batch, c * kGradChunk, std::min(B, (c + 1) * kGradChunk), part.data() + c * P);
    });
    std::vector<double> grad(part.begin(), part.begin() + P);
    for (std::size_t c = 1; c < n_chunks; ++c) {
      const double* q = part.data() + c * P;
      for (std::size_t i = 0; i < P; ++i) grad[i] += q[i];
    }
    return grad;
  }

  void grad_range(const std::vector<Example>& batch, std::size_t b0, std::size_t b1,
                  double* grad) const {
    const std::size_t B = batch.size(), H = c_.hidden, E = c_.embedding_dim, T = c_.window;
    const std::size_t per_t = 7 * H;
    std::vector<double> cache(c_.layers * T * per_t);
    std::vector<double> dh_ext(T * H), dx_below(T * std::max<std::size_t>(in0_, H));
    std::vector<double> dz(4 * H), dh(H), dc(H), dc_next(H), dh_carry(H), xs(T * in0_);
    for (std::size_t b = b0; b < b1; ++b) {
      const Example& ex = batch[b];
      const double z = logit_one(ex, &cache);
      const double dlogit = (sigmoid(z) - ex.label) / static_cast<double>(B);
      const double* h_top = cache.data() + ((c_.layers - 1) * T + (T - 1)) * per_t + 6 * H;
      for (std::size_t j = 0; j < H; ++j) grad[head_w_off_ + j] += h_top[j] * dlogit;
      grad[head_b_off_] += dlogit;
      std::fill(dh_ext.begin(), dh_ext.end(), 0.0);
      for (std::size_t j = 0; j < H; ++j) dh_ext[(T - 1) * H + j] = theta_[head_w_off_ + j] * dlogit;
      for (std::size_t t = 0; t < T; ++t) {
        xs[t * in0_] = ex.window[t];
        for (std::size_t e = 0; e < E; ++e)
          xs[t * in0_ + 1 + e] = theta_[emb_off_ + ex.adapter * E + e];
      }
      for (int l = static_cast<int>(c_.layers) - 1; l >= 0; --l) {
        const std::size_t in = l == 0 ? in0_ : H;
        const double* W = theta_.data() + w_off_[l];
        const double* U = theta_.data() + u_off_[l];
        double* gW = grad + w_off_[l];
        double* gU = grad + u_off_[l];
        double* gb = grad + b_off_[l];
        std::fill(dc_next.begin(), dc_next.end(), 0.0);
        std::fill(dh_carry.begin(), dh_carry.end(), 0.0);
        for (int t = static_cast<int>(T) - 1; t >= 0; --t) {
          const double* cl = cache.data() + (l * T + t) * per_t;
          const double *gi = cl, *gf = cl + H, *gg = cl + 2 * H, *go = cl + 3 * H, *tc = cl + 5 * H;
          const double* c_prev = t > 0 ? cache.data() + (l * T + t - 1) * per_t + 4 * H : nullptr;
          const double* h_prev = t > 0 ? cache.data() + (l * T + t - 1) * per_t + 6 * H : nullptr;
          for (std::size_t j = 0; j < H; ++j) {
            const double dhj = dh_ext[t * H + j] + dh_carry[j];
            const double dO = dhj * tc[j];
            const double dcj = dc_next[j] + dhj * go[j] * (1.0 - tc[j] * tc[j]);
            const double di = dcj * gg[j], dg = dcj * gi[j];
            const double df = dcj * (c_prev ? c_prev[j] : 0.0);
            dc_next[j] = dcj * gf[j];
            dz[j] = di * gi[j] * (1.0 - gi[j]);
            dz[H + j] = df * gf[j] * (1.0 - gf[j]);
            dz[2 * H + j] = dg * (1.0 - gg[j] * gg[j]);
            dz[3 * H + j] = dO * go[j] * (1.0 - go[j]);
          }
          const double* x_t = l == 0 ? xs.data() + t * in0_
                                     : cache.data() + ((l - 1) * T + t) * per_t + 6 * H;
          for (std::size_t k = 0; k < in; ++k) {
            const double xv = x_t[k];
            double* col = gW + k * 4 * H;
            for (std::size_t r = 0; r < 4 * H; ++r) col[r] += dz[r] * xv;
          }
          if (h_prev)
            for (std::size_t k = 0; k < H; ++k) {
              const double hv = h_prev[k];
              double* col = gU + k * 4 * H;
              for (std::size_t r = 0; r < 4 * H; ++r) col[r] += dz[r] * hv;
            }
          for (std::size_t r = 0; r < 4 * H; ++r) gb[r] += dz[r];
          for (std::size_t k = 0; k < H; ++k) {  // dh_carry = Uᵀ dz
            const double* col = U + k * 4 * H;
            double s = 0.0;
            for (std::size_t r = 0; r < 4 * H; ++r) s += col[r] * dz[r];
            dh_carry[k] = s;
          }
          for (std::size_t k = 0; k < in; ++k) {  // dx_below = Wᵀ dz
            const double* col = W + k * 4 * H;
            double s = 0.0;
            for (std::size_t r = 0; r < 4 * H; ++r) s += col[r] * dz[r];
            dx_below[t * in + k] = s;
          }
        }
        if (l > 0) {
          for (std::size_t t = 0; t < T; ++t)
            for (std::size_t j = 0; j < H; ++j) dh_ext[t * H + j] = dx_below[t * H + j];
        } else {
          double* g_emb = grad + emb_off_ + ex.adapter * E;
          for (std::size_t t = 0; t < T; ++t)
            for (std::size_t e = 0; e < E; ++e) g_emb[e] += dx_below[t * in0_ + 1 + e];
        }
      }
    }
  }

  double train_step(const std::vector<Example>& batch) {  // lstm.cpp:283-296
    const double loss = loss_on(batch);
    const std::vector<double> g = gradient(batch);
    ++t_;
    const double b1 = c_.adam_beta1, b2 = c_.adam_beta2;
    const double mc = 1.0 - std::pow(b1, static_cast<double>(t_));
    const double vc = 1.0 - std::pow(b2, static_cast<double>(t_));
    for (std::size_t i = 0; i < theta_.size(); ++i) {
      m_[i] = b1 * m_[i] + (1.0 - b1) * g[i];
      v_[i] = b2 * v_[i] + (1.0 - b2) * g[i] * g[i];
      theta_[i] -= c_.learning_rate * (m_[i] / mc) / (std::sqrt(v_[i] / vc) + c_.adam_eps);
    }
    return loss;
  }

  void save(const std::string& path) const {  // lstm.cpp:298-309 ("LSW1")
    std::ofstream out(path, std::ios::binary);
    if (!out) throw ConfigError("cannot write model file: " + path);
    const char magic[4] = {'L', 'S', 'W', '1'};
    out.write(magic, 4);
    const uint32_t dims[5] = {c_.window, c_.hidden, c_.layers, c_.embedding_dim, c_.num_adapters};
    out.write(reinterpret_cast<const char*>(dims), sizeof(dims));
    out.write(reinterpret_cast<const char*>(theta_.data()),
              static_cast<std::streamsize>(theta_.size() * sizeof(double)));
  }

  static Lstm* load(const std::string& path) {  // lstm.cpp:311-331
    std::ifstream in(path, std::ios::binary);
    if (!in) throw ConfigError("cannot open model file: " + path);
    char magic[4];
    in.read(magic, 4);
    if (!in || magic[0] != 'L' || magic[1] != 'S' || magic[2] != 'W' || magic[3] != '1')
      throw ParseError("bad model file magic in " + path);
    uint32_t dims[5];
    in.read(reinterpret_cast<char*>(dims), sizeof(dims));
    if (!in) throw ParseError("truncated model header in " + path);
    plora_lstm_config cfg;
    plora_lstm_config_default(&cfg);
    cfg.window = dims[0];
    cfg.hidden = dims[1];
    cfg.layers = dims[2];
    cfg.embedding_dim = dims[3];
    cfg.num_adapters = dims[4];
    auto* m = new Lstm(cfg, 0);
    in.read(reinterpret_cast<char*>(m->theta_.data()),
            static_cast<std::streamsize>(m->theta_.size() * sizeof(double)));
    if (!in) {
      delete m;
      throw ParseError("truncated model weights in " + path);
    }
    return m;
  }

 private:
  plora_lstm_config c_;
  std::size_t in0_ = 0;
  std::vector<std::size_t> w_off_, u_off_, b_off_;
  std::size_t head_w_off_ = 0, head_b_off_ = 0, emb_off_ = 0;
  std::vector<double> theta_, m_, v_;
  uint64_t t_ = 0;
};

// OnlinePredictor (predictor.hpp:54-111, predictor.cpp:41-155)
class Online {
 public:
  Online(const plora_predictor_config& cfg, uint64_t seed)
      : cfg_(cfg), model_(cfg.model, seed), series_(cfg.model.num_adapters), rng_(seed ^ 0xA5A5A5A5ull) {
    if (cfg_.interval_ms <= 0) throw ValidationError("interval_ms must be positive");
    if (cfg_.train_every == 0) throw ValidationError("train_every must be >= 1");
    if (cfg_.batch_size == 0) throw ValidationError("batch_size must be >= 1");
  }

  Lstm& model() { return model_; }
  // predict_all's forward on a GPU (device >= 0) or on the host (-1)
  void set_device(int device) {
    gpu_.reset(device >= 0 ? new GpuLstm(device) : nullptr);
    cache_interval_ = -1;  // recompute on the next call
  }
  int device() const { return gpu_ ? gpu_->device() : -1; }

  void observe(uint32_t adapter, double t_ms) {  // predictor.cpp:86-98
    if (adapter >= series_.size()) throw ValidationError("adapter index out of range in observe()");
    roll_to(t_ms);
    Series& s = series_[adapter];
    if (!s.seen) {
      s.seen = true;
      ++known_;
    }
    ++s.current;
    ++observed_;
    if (observed_ % cfg_.train_every == 0) train_step(nullptr);
  }

  void roll_to(double t_ms) {  // predictor.cpp:81-84
    const auto target = static_cast<int64_t>(std::floor(t_ms / cfg_.interval_ms));
    while (interval_ < target) close_interval();
  }

  bool train_step(double* loss) {  // predictor.cpp:100-107
    if (buf_.empty()) return false;
    auto batch = sample(cfg_.batch_size);
    last_loss_ = model_.train_step(batch);
    ++train_steps_;
    cache_interval_ = -1;
    if (loss) *loss = last_loss_;
    return true;
  }

  // predictor.cpp:109-143: one prediction per known adapter (adapter order), cached per interval
  const std::vector<std::pair<uint32_t, double>>& predict_all(double now_ms) {
    roll_to(now_ms);
    if (known_ == 0) {
      cache_.clear();
      return cache_;
    }
    if (cache_interval_ == interval_ && cache_known_ == known_) return cache_;
    std::vector<Example> batch;
    std::vector<uint32_t> ids;
    for (uint32_t a = 0; a < series_.size(); ++a) {
      if (!series_[a].seen) continue;
      Example ex;
      ex.adapter = a;
      ex.window = normalized(series_[a]);
      batch.push_back(std::move(ex));
      ids.push_back(a);
    }
    std::vector<double> probs;
    if (gpu_) {  // FP64 forward on the device (plora_predictor_set_device)
      const std::size_t T = model_.cfg().window;
      std::vector<double> win(batch.size() * T);
      for (std::size_t i = 0; i < batch.size(); ++i)
        std::copy(batch[i].window.begin(), batch[i].window.end(), win.begin() + i * T);
      probs.resize(batch.size());
      gpu_->forward(model_.gpu_shape(), model_.theta().data(), model_.theta().size(), ids.data(),
                    win.data(), ids.size(), probs.data());
    } else {
      probs = model_.forward(batch);
    }
    cache_.resize(ids.size());
    for (std::size_t i = 0; i < ids.size(); ++i)
      cache_[i] = {ids[i], std::min(1.0 - kProbEps, std::max(kProbEps, probs[i]))};
    cache_interval_ = interval_;
    cache_known_ = known_;
    return cache_;
  }

  std::vector<double> window_for(uint32_t adapter) const {
    if (adapter >= series_.size()) throw ValidationError("adapter index out of range in window_for()");
    return normalized(series_[adapter]);
  }

  const Example& buffer_at(uint64_t i) const {
    if (i >= buf_.size()) throw ValidationError("replay buffer index out of range");
    return buf_[i];
  }
  bool known(uint32_t adapter) const {
    if (adapter >= series_.size()) throw ValidationError("adapter index out of range in known()");
    return series_[adapter].seen;
  }
  uint64_t observed() const { return observed_; }
  int64_t current_interval() const { return interval_; }
  uint64_t train_steps() const { return train_steps_; }
  uint64_t known() const { return known_; }
  uint64_t buffer_size() const { return buf_.size(); }
  double last_loss() const { return last_loss_; }

 private:
  struct Series {
    std::deque<uint32_t> ring;
    double run_max = 0.0;
    uint32_t current = 0;
    bool seen = false;
  };

  std::vector<double> normalized(const Series& s) const {  // predictor.cpp:52-60
    const std::size_t w = cfg_.model.window;
    std::vector<double> out(w, 0.0);
    const double denom = std::max(1.0, s.run_max);
    const std::size_t pad = w - s.ring.size();
    for (std::size_t i = 0; i < s.ring.size(); ++i) out[pad + i] = static_cast<double>(s.ring[i]) / denom;
    return out;
  }

  void close_interval() {  // predictor.cpp:62-79
    const std::size_t w = cfg_.model.window;
    for (uint32_t a = 0; a < series_.size(); ++a) {
      Series& s = series_[a];
      if (!s.seen) continue;
      Example ex;
      ex.adapter = a;
      ex.window = normalized(s);
      ex.label = s.current > 0 ? 1.0 : 0.0;
      push(std::move(ex));
      s.ring.push_back(s.current);
      if (s.ring.size() > w) s.ring.pop_front();
      s.run_max = std::max(s.run_max, static_cast<double>(s.current));
      s.current = 0;
    }
    ++interval_;
  }

  void push(Example ex) {  // ReplayBuffer::push (predictor.cpp:14-18)
    if (cfg_.replay_capacity == 0) return;
    if (buf_.size() == cfg_.replay_capacity) buf_.pop_front();
    buf_.push_back(std::move(ex));
  }

  std::vector<Example> sample(std::size_t n) {  // ReplayBuffer::sample (predictor.cpp:20-39)
    std::vector<Example> out;
    if (buf_.empty() || n == 0) return out;
    out.reserve(n);
    if (buf_.size() >= n) {
      std::vector<std::size_t> idx(buf_.size());
      for (std::size_t i = 0; i < idx.size(); ++i) idx[i] = i;
      for (std::size_t i = 0; i < n; ++i) {
        std::uniform_int_distribution<std::size_t> pick(i, idx.size() - 1);
        std::swap(idx[i], idx[pick(rng_)]);
        out.push_back(buf_[idx[i]]);
      }
    } else {
      std::uniform_int_distribution<std::size_t> pick(0, buf_.size() - 1);
      for (std::size_t i = 0; i < n; ++i) out.push_back(buf_[pick(rng_)]);
    }
    return out;
  }

  plora_predictor_config cfg_;
  Lstm model_;
  std::unique_ptr<GpuLstm> gpu_;
  std::vector<Series> series_;
  int64_t interval_ = 0;
  uint64_t observed_ = 0, train_steps_ = 0, known_ = 0;
  double last_loss_ = 0.0;
  std::deque<Example> buf_;
  std::mt19937_64 rng_;
  int64_t cache_interval_ = -1;
  uint64_t cache_known_ = 0;
  std::vector<std::pair<uint32_t, double>> cache_;
};

}  // namespace plora

using namespace plora;

struct plora_lstm {
  Lstm* m;
  bool owned;
};
struct plora_predictor {
  Online p;
  plora_lstm view;
};

namespace {
std::vector<Example> make_batch(const plora_lstm* m, const uint32_t* adapters,
                                const double* windows, const double* labels, uint64_t n) {
  const uint32_t w = m->m->cfg().window;
  std::vector<Example> b(n);
  for (uint64_t i = 0; i < n; ++i) {
    b[i].adapter = adapters[i];
    b[i].window.assign(windows + i * w, windows + (i + 1) * w);
    b[i].label = labels ? labels[i] : 0.0;
  }
  return b;
}
}  // namespace

extern "C" {

void plora_lstm_config_default(plora_lstm_config* c) {  // lstm.hpp:21-33
  c->window = 30;
  c->hidden = 64;
  c->layers = 2;
  c->embedding_dim = 8;
  c->num_adapters = 0;
  c->learning_rate = 1e-3;
  c->adam_beta1 = 0.9;
  c->adam_beta2 = 0.999;
  c->adam_eps = 1e-8;
}

void plora_predictor_config_default(plora_predictor_config* c) {  // predictor.hpp:45-51
  plora_lstm_config_default(&c->model);
  c->interval_ms = 1000.0;
  c->train_every = 100;
  c->batch_size = 64;
  c->replay_capacity = 10000;
}

int plora_cross_entropy(const double* p, const double* y, uint64_t n, double* out) {
  return guard([&] {  // lstm.cpp:37-44
    double total = 0.0;
    for (uint64_t i = 0; i < n; ++i) total += clamped_ce(p[i], y[i]);
    *out = total;
    return 0;
  });
}

int plora_lstm_create(const plora_lstm_config* cfg, uint64_t seed, plora_lstm** out) {
  return guard([&] {
    *out = new plora_lstm{new Lstm(*cfg, seed), true};
    return 0;
  });
}

void plora_lstm_destroy(plora_lstm* m) {
  if (m && m->owned) delete m->m;
  if (m && m->owned) delete m;
}

uint64_t plora_lstm_param_count(const plora_lstm* m) { return m->m->theta().size(); }
double* plora_lstm_parameters(plora_lstm* m) { return m->m->theta().data(); }
void plora_lstm_get_config(const plora_lstm* m, plora_lstm_config* out) { *out = m->m->cfg(); }

int plora_lstm_forward(const plora_lstm* m, const uint32_t* adapters, const double* windows,
                       uint64_t n, double* probs) {
  return guard([&] {
    auto p = m->m->forward(make_batch(m, adapters, windows, nullptr, n));
    std::memcpy(probs, p.data(), n * sizeof(double));
    return 0;
  });
}

int plora_lstm_loss(const plora_lstm* m, const uint32_t* adapters, const double* windows,
                    const double* labels, uint64_t n, double* out) {
  return guard([&] {
    *out = m->m->loss_on(make_batch(m, adapters, windows, labels, n));
    return 0;
  });
}

int plora_lstm_gradient(const plora_lstm* m, const uint32_t* adapters, const double* windows,
                        const double* labels, uint64_t n, double* grad) {
  return guard([&] {
    auto g = m->m->gradient(make_batch(m, adapters, windows, labels, n));
    std::memcpy(grad, g.data(), g.size() * sizeof(double));
    return 0;
  });
}

int plora_lstm_train_step(plora_lstm* m, const uint32_t* adapters, const double* windows,
                          const double* labels, uint64_t n, double* loss) {
  return guard([&] {
    *loss = m->m->train_step(make_batch(m, adapters, windows, labels, n));
    return 0;
  });
}

int plora_lstm_save(const plora_lstm* m, const char* path) {
  return guard([&] {
    m->m->save(path);
    return 0;
  });
}

int plora_lstm_load(const char* path, plora_lstm** out) {
  return guard([&] {
    *out = new plora_lstm{Lstm::load(path), true};
    return 0;
  });
}

int plora_predictor_create(const plora_predictor_config* cfg, uint64_t seed,
                           plora_predictor** out) {
  return guard([&] {
    auto* p = new plora_predictor{Online(*cfg, seed), {nullptr, false}};
    p->view.m = &p->p.model();
    *out = p;
    return 0;
  });
}

void plora_predictor_destroy(plora_predictor* p) { delete p; }

plora_lstm* plora_predictor_model(plora_predictor* p) { return &p->view; }

int plora_predictor_observe(plora_predictor* p, uint32_t adapter, double t_ms) {
  return guard([&] {
    p->p.observe(adapter, t_ms);
    return 0;
  });
}

int plora_predictor_roll_to(plora_predictor* p, double t_ms) {
  return guard([&] {
    p->p.roll_to(t_ms);
    return 0;
  });
}

int plora_predictor_train_step(plora_predictor* p, double* loss) {
  return guard([&] { return p->p.train_step(loss) ? 1 : 0; });
}

int plora_predictor_set_device(plora_predictor* p, int device) {
  return guard([&] {
    if (!p) throw ValidationError("null predictor");
    try {
      p->p.set_device(device);
    } catch (const std::runtime_error& e) {
      throw CudaError(e.what());
    }
    return 0;
  });
}

int64_t plora_predictor_predict_all(plora_predictor* p, double now_ms, uint32_t* adapters,
                                    double* probs, uint64_t cap) {
  int64_t n = 0;
  const int rc = guard([&] {
    const std::vector<std::pair<uint32_t, double>>* vp = nullptr;
    try {
      vp = &p->p.predict_all(now_ms);
    } catch (const std::runtime_error& e) {  // GPU forward failures are CUDA errors
      if (dynamic_cast<const ValidationError*>(&e) || dynamic_cast<const ConfigError*>(&e) ||
          dynamic_cast<const ParseError*>(&e) || dynamic_cast<const CudaError*>(&e))
        throw;
      throw CudaError(e.what());
    }
    const auto& v = *vp;
    n = static_cast<int64_t>(v.size());
    for (uint64_t i = 0; i < v.size() && i < cap; ++i) {
      adapters[i] = v[i].first;
      probs[i] = v[i].second;
    }
    return 0;
  });
  return rc ? rc : n;
}

int plora_predictor_window(const plora_predictor* p, uint32_t adapter, double* out) {
  return guard([&] {
    auto w = const_cast<plora_predictor*>(p)->p.window_for(adapter);
    std::memcpy(out, w.data(), w.size() * sizeof(double));
    return 0;
  });
}

int plora_predictor_known(const plora_predictor* p, uint32_t adapter) {
  return guard([&] { return p->p.known(adapter) ? 1 : 0; });
}

void plora_predictor_stats(const plora_predictor* p, plora_predictor_stats_t* out) {
  const Online& o = p->p;
  out->observed = o.observed();
  out->train_steps = o.train_steps();
  out->known = o.known();
  out->buffered = o.buffer_size();
  out->current_interval = o.current_interval();
  out->last_loss = o.last_loss();
}

int plora_predictor_buffer_at(const plora_predictor* p, uint64_t i, uint32_t* adapter,
                              double* window, double* label) {
  return guard([&] {
    const Example& ex = p->p.buffer_at(i);
    if (adapter) *adapter = ex.adapter;
    if (window) std::memcpy(window, ex.window.data(), ex.window.size() * sizeof(double));
    if (label) *label = ex.label;
    return 0;
  });
}

}  // extern "C"
