// C ABI for the host-side pieces: errors, adapter model, page pool and the
// synthetic workload generator.  Each function cites the reference code it
// restates (paths under /root/reference/proj).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <map>
#include <random>
#include <string>
#include <vector>

#include "common.hpp"
#include "pagepool.hpp"
#include "store.hpp"

namespace plora {
namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_launches{0};
}  // namespace

void set_last_error(const std::string& msg) { g_last_error = msg; }
void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// adapter.cpp:12-20
static void validate_dims(uint32_t d, uint32_t k, uint32_t r, uint32_t adapted, uint32_t bpp) {
  if (r < 1) throw ValidationError("rank must be >= 1");
  if (r >= std::min(d, k))
    throw ValidationError("rank must be < min(d, k), got r=" + std::to_string(r));
  if (adapted < 1) throw ValidationError("adapted_matrices must be >= 1");
  if (bpp != 1 && bpp != 2 && bpp != 4)
    throw ValidationError("bytes_per_param must be 1, 2 or 4");
}

// adapter.cpp:22-26
static uint64_t param_count(uint32_t d, uint32_t k, uint32_t r, uint32_t adapted, uint32_t bpp) {
  validate_dims(d, k, r, adapted, bpp);
  return static_cast<uint64_t>(adapted) * r * (static_cast<uint64_t>(d) + k);
}

}  // namespace plora

using namespace plora;

// AdapterSizeTable (adapter.hpp:32-47)
struct plora_size_table {
  std::map<uint32_t, uint64_t> table;
  uint32_t anchor_rank = 8;
  uint64_t anchor_bytes = 13ull << 20;
  bool linear_fallback = true;

  uint64_t bytes_for(uint32_t rank) const {  // adapter.cpp:43-50
    auto it = table.find(rank);
    if (it != table.end()) return it->second;
    if (!linear_fallback)
      throw ConfigError("no size configured for rank " + std::to_string(rank) +
                        " and linear fallback is disabled");
    return anchor_bytes * rank / anchor_rank;
  }
};


extern "C" {

const char* plora_last_error(void) { return plora::g_last_error.c_str(); }
const char* plora_version(void) { return "plora-b200 0.1.0 (sm_100a)"; }
uint64_t plora_kernel_launch_count(void) { return plora::g_launches.load(); }

// ---------------------------------------------------------------- adapter model
int plora_lora_dims_validate(uint32_t d, uint32_t k, uint32_t r, uint32_t adapted,
                             uint32_t bpp) {
  return guard([&] {
    validate_dims(d, k, r, adapted, bpp);
    return 0;
  });
}

int plora_param_count(uint32_t d, uint32_t k, uint32_t r, uint32_t adapted, uint32_t bpp,
                      uint64_t* out) {
  return guard([&] {
    *out = param_count(d, k, r, adapted, bpp);
    return 0;
  });
}

int plora_size_table_create(uint32_t anchor_rank, uint64_t anchor_bytes, int linear_fallback,
                            plora_size_table** out) {
  return guard([&] {
    // adapter.cpp:28-35
    if (anchor_rank == 0 || anchor_bytes == 0)
      throw ConfigError("size table anchor must be positive");
    auto* t = new plora_size_table();
    t->anchor_rank = anchor_rank;
    t->anchor_bytes = anchor_bytes;
    t->linear_fallback = linear_fallback != 0;
    *out = t;
    return 0;
  });
}

void plora_size_table_destroy(plora_size_table* t) { delete t; }

int plora_size_table_set(plora_size_table* t, uint32_t rank, uint64_t bytes) {
  return guard([&] {
    // adapter.cpp:37-40
    if (bytes == 0) throw ConfigError("adapter size must be positive");
    t->table[rank] = bytes;
    return 0;
  });
}

int plora_size_table_bytes_for(const plora_size_table* t, uint32_t rank, uint64_t* out) {
  return guard([&] {
    *out = t->bytes_for(rank);
    return 0;
  });
}

int plora_generate_catalog(uint32_t count, const uint32_t* mix_ranks, const double* mix_weights,
                           uint64_t n_mix, uint64_t seed, const plora_size_table* sizes,
                           uint32_t d, uint32_t k, uint32_t adapted, uint32_t bpp,
                           uint32_t* ranks_out, uint64_t* bytes_out) {
  return guard([&] {
    // adapter.cpp:110-144 (ids are the dense index; the zero-padded string id
    // "a%0*u" is derivable by the caller)
    if (count == 0) throw ValidationError("catalog count must be >= 1");
    if (n_mix == 0) throw ConfigError("rank mix is empty");
    std::vector<double> weights;
    for (uint64_t i = 0; i < n_mix; ++i) {
      if (mix_weights[i] < 0) throw ConfigError("rank mix weights must be nonnegative");
      weights.push_back(mix_weights[i]);
    }
    plora_size_table def;
    const plora_size_table& st = sizes ? *sizes : def;
    std::mt19937_64 rng(seed ^ 0x9e3779b97f4a7c15ull);
    std::discrete_distribution<std::size_t> pick(weights.begin(), weights.end());
    for (uint32_t i = 0; i < count; ++i) {
      uint32_t r = mix_ranks[pick(rng)];
      validate_dims(d, k, r, adapted, bpp);  // AdapterSpec::sized -> validate
      uint64_t b = st.bytes_for(r);
      if (b == 0) throw ValidationError("adapter weight_bytes must be > 0");
      ranks_out[i] = r;
      bytes_out[i] = b;
    }
    return 0;
  });
}

// ------------------------------------------------------------------- page pool
int plora_pool_create(uint64_t page_bytes, uint32_t total_pages, plora_pool** out) {
  return guard([&] {
    *out = new plora_pool{PagePool(page_bytes, total_pages), {}};
    return 0;
  });
}

void plora_pool_destroy(plora_pool* p) { delete p; }

uint32_t plora_pool_pages_needed(const plora_pool* p, uint64_t bytes) {
  return p->pool.pages_needed(bytes);
}

int plora_pool_alloc(plora_pool* p, uint32_t adapter, uint64_t weight_bytes) {
  return guard([&] { return static_cast<int>(p->pool.alloc(adapter, weight_bytes)); });
}

int plora_pool_free(plora_pool* p, uint32_t adapter) {
  return guard([&] {
    p->pool.free(adapter);
    return 0;
  });
}

int plora_pool_translate(const plora_pool* p, uint32_t adapter, uint32_t logical,
                         uint32_t* phys) {
  return guard([&] {
    *phys = p->pool.translate(adapter, logical);
    return 0;
  });
}

int plora_pool_table(const plora_pool* p, uint32_t adapter, const uint32_t** entries,
                     uint32_t* n_entries, uint64_t* weight_bytes) {
  return guard([&] {
    const PageTable& t = p->pool.table(adapter);
    if (entries) *entries = t.entries.data();
    if (n_entries) *n_entries = static_cast<uint32_t>(t.entries.size());
    if (weight_bytes) *weight_bytes = t.weight_bytes;
    return 0;
  });
}

int plora_pool_has(const plora_pool* p, uint32_t adapter) { return p->pool.has(adapter) ? 1 : 0; }

int plora_pool_compact(plora_pool* p, uint64_t* moved) {
  return guard([&] {
    uint64_t m = p->pool.compact();
    if (moved) *moved = m;
    return 0;
  });
}

int plora_pool_last_relocations(const plora_pool* p, const plora_reloc** relocs, uint64_t* n) {
  const auto& r = p->pool.last_relocations();
  if (relocs) *relocs = r.data();
  if (n) *n = r.size();
  return 0;
}

void plora_pool_report(const plora_pool* p, plora_frag_report* out) {
  FragmentationReport r = p->pool.report();
  out->external_frag = r.external_frag;
  out->internal_frag = r.internal_frag;
  out->utilization = r.utilization;
}

uint32_t plora_pool_free_pages(const plora_pool* p) { return p->pool.free_pages(); }
uint32_t plora_pool_total_pages(const plora_pool* p) { return p->pool.total_pages(); }
uint64_t plora_pool_page_bytes(const plora_pool* p) { return p->pool.page_bytes(); }
uint64_t plora_pool_used_bytes(const plora_pool* p) { return p->pool.used_bytes(); }
uint64_t plora_pool_allocated_bytes(const plora_pool* p) { return p->pool.allocated_bytes(); }
uint64_t plora_pool_total_bytes(const plora_pool* p) { return p->pool.total_bytes(); }

uint64_t plora_pool_resident(const plora_pool* p, uint32_t* out, uint64_t cap) {
  auto r = p->pool.resident();
  for (uint64_t i = 0; i < r.size() && i < cap; ++i) out[i] = r[i];
  return r.size();
}

int plora_pool_check_invariants(const plora_pool* p) {
  return guard([&] {
    p->pool.check_invariants();
    return 0;
  });
}

int plora_pool_dump(const plora_pool* p, char* buf, uint64_t cap, uint64_t* len) {
  return guard([&] {
    std::string s = p->pool.dump();
    if (len) *len = s.size();
    if (buf && cap) {
      uint64_t n = std::min<uint64_t>(cap - 1, s.size());
      std::memcpy(buf, s.data(), n);
      buf[n] = '\0';
    }
    return 0;
  });
}

// ------------------------------------------------------------ synthetic workload
void plora_synthetic_profile_default(plora_synthetic_profile* p) {
  // workload.hpp:19-50 member initializers
  p->num_adapters = 20;
  p->base_rate = 50.0;
  p->diurnal_amplitude = 0.0;
  p->period_s = 3600.0;
  p->hot_set_size = 5;
  p->hot_rotation_s = 7.0;
  p->hot_share = 0.9;
  p->rotation_jitter = 0.0;
  p->burstiness_cv = 1.0;
  p->input_median = 256.0;
  p->input_sigma = 0.6;
  p->output_median = 128.0;
  p->output_sigma = 0.6;
  p->max_tokens = 8192;
}

namespace {
// workload.cpp:26-31
uint32_t clamp_tokens(double v, uint32_t max_tokens) {
  if (!(v >= 1.0)) return 1;
  if (v > max_tokens) return max_tokens;
  return static_cast<uint32_t>(std::llround(v));
}
}  // namespace

int64_t plora_generate_synthetic(const plora_synthetic_profile* pp, double duration_s,
                                 uint64_t seed, double* arrival_ms, uint32_t* adapter,
                                 uint32_t* input_tokens, uint32_t* output_tokens, uint64_t cap) {
  int64_t count = 0;
  int rc = guard([&] {
    const plora_synthetic_profile& p = *pp;
    // SyntheticProfile::validate (workload.cpp:45-57)
    if (p.num_adapters < 1) throw ValidationError("num_adapters must be >= 1");
    if (p.base_rate <= 0) throw ValidationError("base_rate must be positive");
    if (p.diurnal_amplitude < 0 || p.diurnal_amplitude > 1)
      throw ValidationError("diurnal_amplitude must be in [0, 1]");
    if (p.period_s <= 0) throw ValidationError("period must be positive");
    if (p.hot_set_size < 1 || p.hot_set_size > p.num_adapters)
      throw ValidationError("hot_set_size must be in [1, num_adapters]");
    if (p.hot_rotation_s <= 0) throw ValidationError("hot_rotation_s must be positive");
    if (p.hot_share < 0 || p.hot_share > 1) throw ValidationError("hot_share must be in [0, 1]");
    if (p.rotation_jitter < 0 || p.rotation_jitter >= 1)
      throw ValidationError("rotation_jitter must be in [0, 1)");
    if (p.burstiness_cv <= 0) throw ValidationError("burstiness_cv must be positive");
    if (duration_s <= 0) throw ValidationError("duration must be positive");

    // workload.cpp:59-144
    constexpr double kPi = 3.14159265358979323846;
    std::mt19937_64 rng(seed);
    const uint32_t num_groups = (p.num_adapters + p.hot_set_size - 1) / p.hot_set_size;
    std::vector<double> rotation_ends;
    {
      std::uniform_real_distribution<double> u(-1.0, 1.0);
      double t = 0.0;
      while (t < duration_s) {
        double len = p.hot_rotation_s;
        if (p.rotation_jitter > 0) len *= 1.0 + p.rotation_jitter * u(rng);
        t += std::max(len, 1e-3);
        rotation_ends.push_back(t);
      }
    }
    auto group_at = [&](double t_s) -> uint32_t {
      auto it = std::upper_bound(rotation_ends.begin(), rotation_ends.end(), t_s);
      return static_cast<uint32_t>(it - rotation_ends.begin()) % num_groups;
    };
    const double rate_max = p.base_rate * (1.0 + p.diurnal_amplitude);
    auto rate_at = [&](double t_s) {
      return p.base_rate * (1.0 + p.diurnal_amplitude * std::sin(2.0 * kPi * t_s / p.period_s));
    };
    const double shape = 1.0 / (p.burstiness_cv * p.burstiness_cv);
    std::gamma_distribution<double> gap(shape, 1.0 / (rate_max * shape));
    std::uniform_real_distribution<double> accept(0.0, 1.0);
    std::uniform_int_distribution<uint32_t> hot_pick(0, p.hot_set_size - 1);
    auto sample_len = [&](double median, double sigma) {  // workload.cpp:33-43
      std::normal_distribution<double> n(std::log(median), sigma);
      return clamp_tokens(std::exp(n(rng)), p.max_tokens);
    };
    double t = 0.0;
    while (true) {
      t += gap(rng);
      if (t >= duration_s) break;
      if (accept(rng) > rate_at(t) / rate_max) continue;
      uint32_t g = group_at(t);
      uint32_t idx;
      if (accept(rng) < p.hot_share) {
        idx = (g * p.hot_set_size + hot_pick(rng)) % p.num_adapters;
      } else {
        uint32_t cold = p.num_adapters - p.hot_set_size;
        if (cold == 0) {
          idx = (g * p.hot_set_size + hot_pick(rng)) % p.num_adapters;
        } else {
          std::uniform_int_distribution<uint32_t> cold_pick(0, cold - 1);
          uint32_t o = cold_pick(rng);
          uint32_t hot_base = (g * p.hot_set_size) % p.num_adapters;
          idx = (hot_base + p.hot_set_size + o) % p.num_adapters;
        }
      }
      uint32_t in = sample_len(p.input_median, p.input_sigma);
      uint32_t out = sample_len(p.output_median, p.output_sigma);
      if (static_cast<uint64_t>(count) < cap) {
        arrival_ms[count] = t * 1000.0;
        adapter[count] = idx;
        input_tokens[count] = in;
        output_tokens[count] = out;
      }
      ++count;
    }
    return 0;
  });
  return rc ? rc : count;
}

}  // extern "C"
