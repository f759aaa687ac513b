// Prefetch / eviction policy — the host half of the predictor-driven
// prefetch hook.  Restates /root/reference/proj/src/prefetch.cpp:1-114
// operation for operation so the doubles (and hence orderings) are
// identical to the reference's.
#include <algorithm>
#include <cmath>
#include <utility>
#include <vector>

#include "common.hpp"

namespace plora {
namespace {

double decayed_at(const plora_dynamics& d, double now_ms, double half_life_ms) {
  // prefetch.cpp:27-32
  if (d.decayed_count == 0.0) return 0.0;
  double dt = now_ms - d.decay_stamp_ms;
  if (dt <= 0) return d.decayed_count;
  return d.decayed_count * std::exp2(-dt / half_life_ms);
}

double recency(double last_access_ms, double now_ms, double tau_ms) {
  // prefetch.cpp:34-38
  if (last_access_ms < 0) return 0.0;
  double dt = std::max(0.0, now_ms - last_access_ms);
  return std::exp(-dt / tau_ms);
}

double score(const plora_dynamics& d, const plora_policy& p, double now_ms, double max_freq) {
  // prefetch.cpp:40-47
  double lru = recency(d.last_access_ms, now_ms, p.tau_ms);
  double freq = max_freq > 0 ? decayed_at(d, now_ms, p.freq_half_life_ms) / max_freq : 0.0;
  return p.alpha * lru + p.beta * freq + p.gamma * d.prediction;
}

}  // namespace
}  // namespace plora

using namespace plora;

extern "C" {

void plora_policy_default(plora_policy* p) {
  // prefetch.hpp:11-21
  p->theta = 0.5;
  p->alpha = 0.3;
  p->beta = 0.3;
  p->gamma = 0.4;
  p->tau_ms = 60'000.0;
  p->freq_half_life_ms = 120'000.0;
  p->staging_fraction = 0.1;
}

int plora_policy_validate(const plora_policy* p) {
  return guard([&] {
    // prefetch.cpp:8-19
    if (p->theta <= 0.0 || p->theta >= 1.0)
      throw ValidationError("theta must be strictly inside (0, 1)");
    if (p->alpha < 0 || p->beta < 0 || p->gamma < 0)
      throw ValidationError("score weights must be nonnegative");
    if (p->alpha + p->beta + p->gamma <= 0)
      throw ValidationError("at least one score weight must be positive");
    if (p->tau_ms <= 0) throw ValidationError("tau must be positive");
    if (p->freq_half_life_ms <= 0) throw ValidationError("half-life must be positive");
    if (p->staging_fraction < 0 || p->staging_fraction > 1)
      throw ValidationError("staging_fraction must be in [0, 1]");
    return 0;
  });
}

void plora_dynamics_init(plora_dynamics* d) {
  // prefetch.hpp:26-37 member initializers
  d->status = PLORA_NOT_RESIDENT;
  d->busy = 0;
  d->last_access_ms = -1.0;
  d->decayed_count = 0.0;
  d->decay_stamp_ms = 0.0;
  d->prediction = 0.0;
  d->transfer_active = 0;
  d->reserved = 0;
}

void plora_record_access(plora_dynamics* d, double now_ms, double half_life_ms) {
  // prefetch.cpp:21-25
  d->decayed_count = decayed_at(*d, now_ms, half_life_ms) + 1.0;
  d->decay_stamp_ms = now_ms;
  d->last_access_ms = now_ms;
}

double plora_decayed_at(const plora_dynamics* d, double now_ms, double half_life_ms) {
  return decayed_at(*d, now_ms, half_life_ms);
}

double plora_recency_score(double last_access_ms, double now_ms, double tau_ms) {
  return recency(last_access_ms, now_ms, tau_ms);
}

double plora_eviction_score(const plora_dynamics* d, const plora_policy* p, double now_ms,
                            double max_freq) {
  return score(*d, *p, now_ms, max_freq);
}

uint64_t plora_scored_residents(const plora_dynamics* dyn, uint64_t n, const plora_policy* p,
                                double now_ms, double* scores, uint32_t* keys) {
  // prefetch.cpp:49-64
  double max_freq = 0.0;
  for (uint64_t a = 0; a < n; ++a)
    if (dyn[a].status == PLORA_RESIDENT)
      max_freq = std::max(max_freq, decayed_at(dyn[a], now_ms, p->freq_half_life_ms));
  std::vector<std::pair<double, uint32_t>> out;
  for (uint64_t a = 0; a < n; ++a) {
    if (dyn[a].status != PLORA_RESIDENT) continue;
    out.emplace_back(score(dyn[a], *p, now_ms, max_freq), static_cast<uint32_t>(a));
  }
  std::sort(out.begin(), out.end());
  for (std::size_t i = 0; i < out.size(); ++i) {
    scores[i] = out[i].first;
    keys[i] = out[i].second;
  }
  return out.size();
}

uint64_t plora_select_prefetch(const double* probabilities, uint64_t n_probs,
                               const plora_dynamics* dyn, uint64_t n, const plora_policy* p,
                               const uint64_t* units_for, uint64_t n_units,
                               uint64_t staging_budget_units, uint32_t* out) {
  // prefetch.cpp:66-91
  std::vector<std::pair<double, uint32_t>> candidates;
  for (uint64_t a = 0; a < n; ++a) {
    if (a >= n_probs) break;
    double pr = probabilities[a];
    if (pr <= p->theta) continue;  // strict inequality gate
    if (dyn[a].status != PLORA_NOT_RESIDENT) continue;
    if (dyn[a].transfer_active) continue;
    candidates.emplace_back(-pr, static_cast<uint32_t>(a));
  }
  std::sort(candidates.begin(), candidates.end());
  uint64_t budget = staging_budget_units, k = 0;
  for (const auto& [negp, a] : candidates) {
    uint64_t need = a < n_units ? units_for[a] : 1;
    if (need > budget) continue;  // skip-if-too-big, then continue
    budget -= need;
    out[k++] = a;
  }
  return k;
}

int plora_plan_evictions(uint64_t bytes_needed, uint64_t free_bytes, const uint32_t* eligible,
                         uint64_t n_eligible, const uint64_t* bytes_for, uint64_t n_bytes,
                         uint32_t* victims, uint64_t* n_victims) {
  // prefetch.cpp:93-112
  (void)n_bytes;
  *n_victims = 0;
  if (free_bytes >= bytes_needed) return 1;
  uint64_t freed = free_bytes;
  for (uint64_t i = 0; i < n_eligible; ++i) {
    victims[(*n_victims)++] = eligible[i];
    freed += bytes_for[eligible[i]];
    if (freed >= bytes_needed) return 1;
  }
  *n_victims = 0;  // unsatisfiable: caller queues the request
  return 0;
}

}  // extern "C"
