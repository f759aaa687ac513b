// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference sources, compiled in place
// from /root/reference/proj/src/{memory,prefetch,adapter,workload}.cpp by
// oracle/Makefile into oracle/_ref/libref.so.  Only tests/, the smoke check
// and bench.py's cpu_baseline leg load it, and only as the checker.
//
// Wrapped reference entry points (file:line under /root/reference/proj):
//   PagePool            include/lorasim/memory.hpp:39-83, src/memory.cpp:7-146
//   prefetch policy     include/lorasim/prefetch.hpp:11-72, src/prefetch.cpp:1-114
//   adapter model       include/lorasim/adapter.hpp:15-76, src/adapter.cpp:12-144
//   generate_synthetic  include/lorasim/workload.hpp:36-63, src/workload.cpp:59-144
//   LSTM scalar oracle  tests/support/lstm_reference.hpp (the reference's own
//                       Eigen-free test oracle for PredictorModel::forward)
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "lorasim/adapter.hpp"
#include "lorasim/memory.hpp"
#include "lorasim/prefetch.hpp"
#include "lorasim/workload.hpp"
#include "support/lstm_reference.hpp"

using namespace lorasim;

namespace {
thread_local std::string g_err;

// 0 ok; -1 ValidationError; -2 logic_error; -3 ConfigError; -4 other; -5 ParseError
template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const ParseError& e) {
    g_err = e.what();
    return -5;
  } catch (const ValidationError& e) {
    g_err = e.what();
    return -1;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return -3;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return -2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -4;
  }
}

struct DynC {  // mirrors plora_dynamics in include/plora.h
  int32_t status;
  uint32_t busy;
  double last_access_ms;
  double decayed_count;
  double decay_stamp_ms;
  double prediction;
  int32_t transfer_active;
  int32_t pad;
};

struct PolicyC {  // mirrors plora_policy in include/plora.h
  double theta, alpha, beta, gamma, tau_ms, freq_half_life_ms, staging_fraction;
};

AdapterDynamics to_dyn(const DynC& d) {
  AdapterDynamics o;
  o.status = static_cast<Residency>(d.status);
  o.busy = d.busy;
  o.last_access_ms = d.last_access_ms;
  o.decayed_count = d.decayed_count;
  o.decay_stamp_ms = d.decay_stamp_ms;
  o.prediction = d.prediction;
  o.transfer_active = d.transfer_active != 0;
  return o;
}

PrefetchPolicy to_policy(const PolicyC& p) {
  PrefetchPolicy o;
  o.theta = p.theta;
  o.alpha = p.alpha;
  o.beta = p.beta;
  o.gamma = p.gamma;
  o.tau_ms = p.tau_ms;
  o.freq_half_life_ms = p.freq_half_life_ms;
  o.staging_fraction = p.staging_fraction;
  return o;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- PagePool ----------------------------------------------------------------
int ref_pool_create(uint64_t page_bytes, uint32_t total_pages, void** out) {
  return guard([&] { *out = new PagePool(page_bytes, total_pages); });
}
void ref_pool_destroy(void* p) { delete static_cast<PagePool*>(p); }
uint32_t ref_pool_pages_needed(void* p, uint64_t bytes) {
  return static_cast<PagePool*>(p)->pages_needed(bytes);
}
// >=0: AllocStatus; <0: error
int ref_pool_alloc(void* p, uint32_t a, uint64_t bytes) {
  int st = 0;
  int rc = guard([&] { st = static_cast<int>(static_cast<PagePool*>(p)->alloc(a, bytes)); });
  return rc ? rc : st;
}
int ref_pool_free(void* p, uint32_t a) {
  return guard([&] { static_cast<PagePool*>(p)->free(a); });
}
int ref_pool_translate(void* p, uint32_t a, uint32_t logical, uint32_t* out) {
  return guard([&] { *out = static_cast<PagePool*>(p)->translate(a, logical); });
}
int ref_pool_table(void* p, uint32_t a, uint32_t* entries, uint64_t cap, uint64_t* n,
                   uint64_t* weight_bytes) {
  return guard([&] {
    const PageTable& t = static_cast<PagePool*>(p)->table(a);
    *n = t.entries.size();
    *weight_bytes = t.weight_bytes;
    if (entries)
      std::memcpy(entries, t.entries.data(),
                  sizeof(uint32_t) * std::min<uint64_t>(cap, t.entries.size()));
  });
}
int ref_pool_has(void* p, uint32_t a) { return static_cast<PagePool*>(p)->has(a) ? 1 : 0; }
uint64_t ref_pool_compact(void* p) { return static_cast<PagePool*>(p)->compact(); }
void ref_pool_report(void* p, double* out3) {
  auto r = static_cast<PagePool*>(p)->report();
  out3[0] = r.external_frag;
  out3[1] = r.internal_frag;
  out3[2] = r.utilization;
}
uint32_t ref_pool_free_pages(void* p) { return static_cast<PagePool*>(p)->free_pages(); }
uint32_t ref_pool_total_pages(void* p) { return static_cast<PagePool*>(p)->total_pages(); }
uint64_t ref_pool_used_bytes(void* p) { return static_cast<PagePool*>(p)->used_bytes(); }
uint64_t ref_pool_allocated_bytes(void* p) {
  return static_cast<PagePool*>(p)->allocated_bytes();
}
uint64_t ref_pool_total_bytes(void* p) { return static_cast<PagePool*>(p)->total_bytes(); }
int ref_pool_check_invariants(void* p) {
  return guard([&] { static_cast<PagePool*>(p)->check_invariants(); });
}
uint64_t ref_pool_resident(void* p, uint32_t* out, uint64_t cap) {
  auto r = static_cast<PagePool*>(p)->resident();
  for (uint64_t i = 0; i < r.size() && i < cap; ++i) out[i] = r[i];
  return r.size();
}
// Returns needed length (excluding NUL); copies when buf is large enough.
uint64_t ref_pool_dump(void* p, char* buf, uint64_t cap) {
  std::string s = static_cast<PagePool*>(p)->dump().dump();
  if (buf && cap > s.size()) std::memcpy(buf, s.c_str(), s.size() + 1);
  return s.size();
}

// ---- prefetch policy ------------------------------------------------------------
int ref_policy_validate(const PolicyC* p) {
  return guard([&] { to_policy(*p).validate(); });
}
double ref_recency_score(double last, double now, double tau) {
  return recency_score(last, now, tau);
}
double ref_decayed_at(const DynC* d, double now, double half_life) {
  return to_dyn(*d).decayed_at(now, half_life);
}
void ref_record_access(DynC* d, double now, double half_life) {
  AdapterDynamics o = to_dyn(*d);
  o.record_access(now, half_life);
  d->last_access_ms = o.last_access_ms;
  d->decayed_count = o.decayed_count;
  d->decay_stamp_ms = o.decay_stamp_ms;
}
double ref_eviction_score(const DynC* d, const PolicyC* p, double now, double max_freq) {
  return eviction_score(to_dyn(*d), to_policy(*p), now, max_freq);
}
uint64_t ref_scored_residents(const DynC* dyn, uint64_t n, const PolicyC* p, double now,
                              double* scores, uint32_t* keys) {
  std::vector<AdapterDynamics> v;
  for (uint64_t i = 0; i < n; ++i) v.push_back(to_dyn(dyn[i]));
  auto r = scored_residents(v, to_policy(*p), now);
  for (uint64_t i = 0; i < r.size(); ++i) {
    scores[i] = r[i].first;
    keys[i] = r[i].second;
  }
  return r.size();
}
uint64_t ref_select_prefetch(const double* probs, uint64_t n_probs, const DynC* dyn,
                             uint64_t n, const PolicyC* p, const uint64_t* units,
                             uint64_t n_units, uint64_t budget, uint32_t* out) {
  std::vector<double> pr(probs, probs + n_probs);
  std::vector<AdapterDynamics> v;
  for (uint64_t i = 0; i < n; ++i) v.push_back(to_dyn(dyn[i]));
  std::vector<uint64_t> u(units, units + n_units);
  auto r = select_prefetch(pr, v, to_policy(*p), u, budget);
  for (uint64_t i = 0; i < r.size(); ++i) out[i] = r[i];
  return r.size();
}
int ref_plan_evictions(uint64_t need, uint64_t free_bytes, const uint32_t* eligible,
                       uint64_t n_elig, const uint64_t* bytes_for, uint64_t n_bytes,
                       uint32_t* victims, uint64_t* n_victims) {
  std::vector<AdapterKey> e(eligible, eligible + n_elig);
  std::vector<uint64_t> b(bytes_for, bytes_for + n_bytes);
  auto plan = plan_evictions(need, free_bytes, e, b);
  *n_victims = plan.victims.size();
  for (uint64_t i = 0; i < plan.victims.size(); ++i) victims[i] = plan.victims[i];
  return plan.satisfied ? 1 : 0;
}

// ---- adapter model --------------------------------------------------------------
int ref_param_count(uint32_t d, uint32_t k, uint32_t r, uint32_t adapted, uint32_t bpp,
                    uint64_t* out) {
  return guard([&] { *out = param_count(LoraDims{d, k, r, adapted, bpp}); });
}
int ref_size_table_bytes(uint32_t anchor_rank, uint64_t anchor_bytes, int linear,
                         const uint32_t* ranks, const uint64_t* bytes, uint64_t n_set,
                         uint32_t rank, uint64_t* out) {
  return guard([&] {
    AdapterSizeTable t(anchor_rank, anchor_bytes, linear != 0);
    for (uint64_t i = 0; i < n_set; ++i) t.set(ranks[i], bytes[i]);
    *out = t.bytes_for(rank);
  });
}
int ref_generate_catalog(uint32_t count, const uint32_t* mix_ranks, const double* mix_w,
                         uint64_t n_mix, uint64_t seed, uint32_t d, uint32_t k,
                         uint32_t adapted, uint32_t bpp, uint32_t* ranks_out,
                         uint64_t* bytes_out) {
  return guard([&] {
    RankMix mix;
    for (uint64_t i = 0; i < n_mix; ++i) mix.emplace_back(mix_ranks[i], mix_w[i]);
    LoraDims base{d, k, 8, adapted, bpp};
    auto cat = generate_catalog(count, mix, seed, AdapterSizeTable{}, base);
    for (uint32_t i = 0; i < count; ++i) {
      ranks_out[i] = cat[i].dims.r;
      bytes_out[i] = cat[i].weight_bytes;
    }
  });
}

// load_catalog_json over the reference's own parser: returns the entry count
// (ranks / bytes filled up to cap) or a negative status (ref_last_error).
int64_t ref_load_catalog_json(const char* path, uint32_t* ranks_out, uint64_t* bytes_out,
                              uint64_t cap) {
  int64_t n = -1;
  const int rc = guard([&] {
    LoraDims base{4096, 4096, 8, 64, 2};
    auto cat = load_catalog_json(path, AdapterSizeTable{}, base);
    n = static_cast<int64_t>(cat.size());
    for (uint64_t i = 0; i < cat.size() && i < cap; ++i) {
      ranks_out[i] = cat[i].dims.r;
      bytes_out[i] = cat[i].weight_bytes;
    }
  });
  return rc == 0 ? n : rc;
}

// ---- synthetic workload -------------------------------------------------------
// Returns number of requests (or -1 on error); fills up to cap entries.
int64_t ref_generate_synthetic(uint32_t num_adapters, double base_rate, double diurnal,
                               double period_s, uint32_t hot_set, double hot_rotation_s,
                               double hot_share, double jitter, double cv,
                               double duration_s, uint64_t seed, double* arrival_ms,
                               uint32_t* adapter_idx, uint32_t* in_tok, uint32_t* out_tok,
                               uint64_t cap) {
  std::vector<Request> reqs;
  int rc = guard([&] {
    SyntheticProfile p;
    p.num_adapters = num_adapters;
    p.base_rate = base_rate;
    p.diurnal_amplitude = diurnal;
    p.period_s = period_s;
    p.hot_set_size = hot_set;
    p.hot_rotation_s = hot_rotation_s;
    p.hot_share = hot_share;
    p.rotation_jitter = jitter;
    p.burstiness_cv = cv;
    reqs = generate_synthetic(p, duration_s, seed);
  });
  if (rc) return -1;
  for (uint64_t i = 0; i < reqs.size() && i < cap; ++i) {
    arrival_ms[i] = reqs[i].arrival_ms;
    adapter_idx[i] = static_cast<uint32_t>(std::stoul(reqs[i].adapter_id.substr(1)));
    in_tok[i] = reqs[i].input_tokens;
    out_tok[i] = reqs[i].output_tokens;
  }
  return static_cast<int64_t>(reqs.size());
}

// lstm_reference::forward_probability (tests/support/lstm_reference.hpp)
double ref_lstm_forward_probability(uint32_t window, uint32_t hidden, uint32_t layers,
                                    uint32_t embedding_dim, uint32_t num_adapters,
                                    const double* theta, uint32_t adapter, const double* w) {
  lstm_reference::Shape s{window, hidden, layers, embedding_dim, num_adapters};
  return lstm_reference::forward_probability(s, theta, adapter,
                                             std::vector<double>(w, w + window));
}

}  // extern "C"
