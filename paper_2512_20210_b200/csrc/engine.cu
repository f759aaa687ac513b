// Real-time loading / prefetch engine: the reference simulator's residency
// control (src/engine.cpp:197-333 transfers + ensure_loading/evict,
// :406-484 do_boundary/admit_requests/issue_prefetches/maybe_compact,
// :515-582 on_arrival/on_round) restated on CUDA streams and events instead
// of modelled time.
//
//   * a transfer is a real page scatter of the adapter's pinned host image
//     into its physical pages (copy engines per contiguous run, or the SM
//     scatter kernel for small scattered pages), issued in chunks;
//   * demand transfers go on a high-priority stream, all chunks at once;
//     prefetch chunks go on a low-priority stream and are only issued while
//     no demand transfer is in flight, with a bounded number of bytes in
//     flight ("demand loads preempt prefetch bandwidth entirely",
//     engine.cpp:214-221, at chunk granularity);
//   * completion is observed by polling events at batch boundaries;
//     demanded weights are published at once, prefetched ones are staged and
//     promoted at the next boundary (engine.cpp:270-288, 406-414);
//   * page reuse after an eviction is ordered after every kernel already
//     enqueued on the compute stream by an event fence on both copy streams;
//   * a pump thread keeps the prefetch copy queue fed between boundaries
//     (it sleeps on the oldest in-flight chunk's event); every entry point
//     and the pump serialise on one mutex — one owner thread per engine as
//     in the reference, the pump being the engine's own.
#include <nvtx3/nvToolsExt.h>
#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <thread>
#include <vector>

#include "plan.hpp"
#include "store.hpp"

namespace plora {
namespace {

constexpr uint64_t kDefaultChunk = 1ull << 20;       // bytes per prefetch chunk
constexpr uint64_t kDefaultPrefetchInflight = 4ull << 20;

struct Transfer {
  bool demand = false;
  uint32_t next_page = 0;  // first logical page not yet issued
  uint32_t n_pages = 0;
  uint64_t bytes = 0;
  cudaEvent_t start = nullptr;  // timing: first chunk issued
  cudaEvent_t done = nullptr;   // recorded after the last chunk
  bool fully_issued = false;
  bool upgraded = false;
};

}  // namespace
}  // namespace plora

using namespace plora;

struct plora_engine {
  plora_store* store = nullptr;
  plora_policy policy{};
  int copy_mode = PLORA_COPY_CE;
  bool prefetch_enabled = true;
  bool compaction_enabled = true;
  uint64_t chunk_bytes = kDefaultChunk;
  uint64_t prefetch_inflight_cap = kDefaultPrefetchInflight;

  uint32_t A = 0;
  std::vector<plora_dynamics> dyn;
  std::vector<double> probs;
  std::vector<uint64_t> bytes, units;
  std::vector<const char*> src, src_dev;

  std::map<uint32_t, Transfer> transfers;  // ordered: deterministic polling
  std::set<uint32_t> staged_ready, prefetch_staged;
  uint64_t staging_total_units = 0;

  cudaStream_t demand_stream = nullptr, prefetch_stream = nullptr;
  cudaEvent_t fence = nullptr;
  std::deque<std::pair<cudaEvent_t, uint64_t>> prefetch_chunks;  // in-flight prefetch chunks
  uint64_t prefetch_inflight = 0;
  std::vector<cudaEvent_t> event_pool, timing_pool;

  plora_predictor* predictor = nullptr;
  plora_engine_stats st{};

  // ---- decision log (engine.cpp:635-640, written as decisions.csv by
  // report.cpp:106-113): every evict / prefetch / demand_load / promote /
  // admission_failure / compact with its time and score
  std::vector<plora_decision> decisions;
  bool log_decisions = true;
  void log(double t, uint32_t action, uint32_t adapter, double score, uint64_t detail = 0) {
    if (log_decisions) decisions.push_back(plora_decision{t, score, adapter, action, detail});
  }

  // ---- per-interval prediction accuracy (engine.cpp:547-561 snapshots the
  // predicted set {p > theta} of the known adapters when an interval starts;
  // :598-633 scores each closed interval as tp / (tp + fp + fn))
  double acc_interval_ms = 1000.0, acc_warmup_ms = 0.0;
  std::vector<uint8_t> seen;
  int64_t last_snapshot = -1;
  std::map<int64_t, std::pair<std::vector<uint32_t>, std::vector<uint32_t>>> snapshots;  // known, predicted
  std::map<int64_t, std::set<uint32_t>> actual;
  int64_t interval_of(double t) const { return static_cast<int64_t>(std::floor(t / acc_interval_ms)); }
  void snapshot(double now) {
    const int64_t k = interval_of(now);
    if (k <= last_snapshot) return;
    last_snapshot = k;
    auto& sn = snapshots[k];
    for (uint32_t a = 0; a < A; ++a) {
      if (!seen[a]) continue;
      sn.first.push_back(a);
      if (probs[a] > policy.theta) sn.second.push_back(a);
    }
  }
  void evaluate(double now) {
    const int64_t cur = interval_of(now);
    while (!snapshots.empty() && snapshots.begin()->first < cur) {
      const int64_t k = snapshots.begin()->first;
      const auto& [known, predicted] = snapshots.begin()->second;
      std::set<uint32_t> act;
      auto it = actual.find(k);
      if (it != actual.end())
        for (uint32_t a : it->second)
          if (std::binary_search(known.begin(), known.end(), a)) act.insert(a);
      uint64_t tp = 0, fp = 0, fn = 0;
      for (uint32_t a : predicted) (act.count(a) ? tp : fp) += 1;
      for (uint32_t a : act)
        if (!std::binary_search(predicted.begin(), predicted.end(), a)) ++fn;
      if (tp + fp + fn > 0 && static_cast<double>(k) * acc_interval_ms >= acc_warmup_ms) {
        st.acc_sum += static_cast<double>(tp) / static_cast<double>(tp + fp + fn);
        ++st.acc_intervals;
        st.acc_tp += tp;
        st.acc_fp += fp;
        st.acc_fn += fn;
      }
      snapshots.erase(snapshots.begin());
    }
    while (!actual.empty() && actual.begin()->first < cur &&
           (snapshots.empty() || actual.begin()->first < snapshots.begin()->first))
      actual.erase(actual.begin());
  }

  // Asynchronous predictor service: observations are queued to a worker
  // thread that owns the predictor (observe -> periodic train_step,
  // predict_all on round requests); a round applies the most recent
  // completed prediction set and requests the next, so the LSTM never sits
  // on the decode loop's critical path (predictions lag by one round).
  struct PredictorService {
    plora_predictor* p = nullptr;
    std::mutex m;
    std::condition_variable cv, idle;
    std::vector<std::pair<uint32_t, double>> obs;
    bool round_req = false, busy = false, stop = false, have = false;
    double round_now = 0;
    std::vector<uint32_t> ids;
    std::vector<double> probs;
    std::string error;
    std::thread th;
    double busy_ms = 0;

    void loop(uint32_t A) {
      std::vector<uint32_t> id(A);
      std::vector<double> pr(A);
      std::unique_lock<std::mutex> lk(m);
      while (true) {
        cv.wait(lk, [&] { return stop || !obs.empty() || round_req; });
        if (stop) break;
        std::vector<std::pair<uint32_t, double>> batch;
        batch.swap(obs);
        const bool rq = round_req;
        const double now = round_now;
        round_req = false;
        busy = true;
        lk.unlock();
        const auto t0 = std::chrono::steady_clock::now();
        std::string err;
        for (const auto& [a, t] : batch)
          if (plora_predictor_observe(p, a, t) != 0) err = plora_last_error();
        int64_t n = 0;
        if (rq) {
          n = plora_predictor_predict_all(p, now, id.data(), pr.data(), A);
          if (n < 0) err = plora_last_error();
        }
        const double dt = std::chrono::duration<double, std::milli>(
                              std::chrono::steady_clock::now() - t0).count();
        lk.lock();
        busy_ms += dt;
        if (!err.empty()) error = err;
        if (rq && n >= 0) {
          ids.assign(id.begin(), id.begin() + std::min<int64_t>(n, A));
          probs.assign(pr.begin(), pr.begin() + std::min<int64_t>(n, A));
          have = true;
        }
        busy = false;
        idle.notify_all();
      }
    }
  };
  std::unique_ptr<PredictorService> svc;

  void stop_service() {
    if (!svc) return;
    {
      std::lock_guard<std::mutex> lk(svc->m);
      svc->stop = true;
    }
    svc->cv.notify_all();
    if (svc->th.joinable()) svc->th.join();
    svc.reset();
  }

  void apply_predictions(const uint32_t* ids, const double* p, int64_t n) {
    std::fill(probs.begin(), probs.end(), -1.0);
    for (int64_t i = 0; i < n && i < static_cast<int64_t>(A); ++i) {
      probs[ids[i]] = p[i];
      dyn[ids[i]].prediction = p[i];
    }
  }

  double now_ms = 0.0;  // time of the current API call (decision log)
  mutable std::mutex mu;
  std::condition_variable cv;
  std::thread pump;
  bool stop = false;

  // ------------------------------------------------------------- events
  cudaEvent_t get_event(bool timing) {
    auto& pool = timing ? timing_pool : event_pool;
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    PLORA_CUDA(cudaEventCreateWithFlags(
        &e, cudaEventBlockingSync | (timing ? 0u : static_cast<unsigned>(cudaEventDisableTiming))));
    return e;
  }
  void put_event(cudaEvent_t e, bool timing) {
    if (e) (timing ? timing_pool : event_pool).push_back(e);
  }

  // A demand transfer whose copies are still running (engine.cpp:214-221).
  cudaEvent_t active_demand_event() const {
    for (const auto& [a, t] : transfers)
      if (t.demand && (!t.fully_issued || cudaEventQuery(t.done) == cudaErrorNotReady))
        return t.fully_issued ? t.done : nullptr;
    return nullptr;
  }
  bool demand_active() const {
    for (const auto& [a, t] : transfers)
      if (t.demand && (!t.fully_issued || cudaEventQuery(t.done) == cudaErrorNotReady))
        return true;
    return false;
  }

  // ------------------------------------------------------ chunk issuance
  void issue_pages(uint32_t a, Transfer& t, uint32_t n, cudaStream_t stream) {
    scatter_pages(*store, a, src[a], src_dev[a], t.next_page, n, t.bytes, copy_mode, stream);
    t.next_page += n;
  }

  void finish_issue(uint32_t a, Transfer& t, cudaStream_t stream) {
    t.done = get_event(true);
    PLORA_CUDA(cudaEventRecord(t.done, stream));
    t.fully_issued = true;
    (void)a;
  }

  // Issue every remaining page of a demanded transfer on the demand stream.
  // An upgraded prefetch joins the chunks it already issued on the prefetch
  // stream first, so `done` covers the whole image.
  void issue_all_demand(uint32_t a, Transfer& t) {
    if (t.fully_issued) return;
    if (t.upgraded || t.next_page > 0) {
      cudaEvent_t j = get_event(false);
      PLORA_CUDA(cudaEventRecord(j, prefetch_stream));
      PLORA_CUDA(cudaStreamWaitEvent(demand_stream, j, 0));
      put_event(j, false);
    }
    if (t.next_page < t.n_pages) issue_pages(a, t, t.n_pages - t.next_page, demand_stream);
    finish_issue(a, t, demand_stream);
  }

  void retire_prefetch_chunks() {
    while (!prefetch_chunks.empty()) {
      cudaError_t q = cudaEventQuery(prefetch_chunks.front().first);
      if (q == cudaErrorNotReady) break;
      PLORA_CUDA(q);
      prefetch_inflight -= prefetch_chunks.front().second;
      put_event(prefetch_chunks.front().first, false);
      prefetch_chunks.pop_front();
    }
  }

  // Feed prefetch chunks while no demand transfer is active (engine.cpp:214-221).
  void pump_prefetch() {
    retire_prefetch_chunks();
    if (demand_active()) return;
    const uint64_t P = store->pool->pool.page_bytes();
    const uint32_t chunk_pages = static_cast<uint32_t>(std::max<uint64_t>(1, chunk_bytes / P));
    for (auto& [a, t] : transfers) {
      if (t.demand || t.fully_issued) continue;
      while (t.next_page < t.n_pages && prefetch_inflight < prefetch_inflight_cap) {
        const uint32_t n = std::min(chunk_pages, t.n_pages - t.next_page);
        issue_pages(a, t, n, prefetch_stream);
        cudaEvent_t e = get_event(false);
        PLORA_CUDA(cudaEventRecord(e, prefetch_stream));
        const uint64_t b = static_cast<uint64_t>(n) * P;
        prefetch_chunks.emplace_back(e, b);
        prefetch_inflight += b;
      }
      if (t.next_page == t.n_pages) finish_issue(a, t, prefetch_stream);
      if (prefetch_inflight >= prefetch_inflight_cap) break;
    }
  }

  // ------------------------------------------------- transfers (real time)
  void start_transfer(uint32_t a, bool demand) {  // engine.cpp:250-259
    Transfer t;
    t.demand = demand;
    t.bytes = bytes[a];
    t.n_pages = static_cast<uint32_t>(units[a]);
    cudaStream_t s = demand ? demand_stream : prefetch_stream;
    if (copy_mode == PLORA_COPY_SM) store->upload_table(a, s);
    t.start = get_event(true);
    PLORA_CUDA(cudaEventRecord(t.start, s));
    dyn[a].transfer_active = 1;
    dyn[a].status = PLORA_STAGING;
    auto& slot = transfers.emplace(a, t).first->second;
    if (demand) issue_all_demand(a, slot);
    else cv.notify_one();
  }

  void publish(uint32_t a, cudaStream_t compute) {
    PLORA_CUDA(cudaGetLastError());
    if (plora_store_publish(store, a, compute) != 0)
      throw CudaError(std::string("publish failed: ") + plora_last_error());
  }

  void complete_transfer(uint32_t a, Transfer& t, cudaStream_t compute) {  // :269-288
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, t.start, t.done) == cudaSuccess) {
      st.transfer_ms += ms;
      if (t.demand) st.demand_transfer_ms += ms;
    }
    st.bytes_h2d += t.bytes;
    ++st.transfers_completed;
    put_event(t.start, true);
    put_event(t.done, true);
    const bool demand = t.demand;
    // the compute stream orders after the copies (already complete when
    // observed by polling; a device-side wait for plora_engine_wait_ready)
    PLORA_CUDA(cudaStreamWaitEvent(compute, t.done, 0));
    transfers.erase(a);
    dyn[a].transfer_active = 0;
    if (demand) {  // demanded weights become usable immediately
      dyn[a].status = PLORA_RESIDENT;
      prefetch_staged.erase(a);
      publish(a, compute);
    } else {
      staged_ready.insert(a);  // promoted at the next batch boundary
    }
  }

  int poll_transfers(cudaStream_t compute) {
    int done = 0;
    std::vector<uint32_t> finished;
    for (auto& [a, t] : transfers) {
      if (!t.fully_issued) continue;
      cudaError_t q = cudaEventQuery(t.done);
      if (q == cudaErrorNotReady) continue;
      PLORA_CUDA(q);
      finished.push_back(a);
    }
    for (uint32_t a : finished) {
      complete_transfer(a, transfers.at(a), compute);
      ++done;
    }
    return done;
  }

  // --------------------------------------------------- allocation/eviction
  void evict(uint32_t a, double score, cudaStream_t compute) {  // engine.cpp:294-304
    if (dyn[a].busy > 0 || dyn[a].transfer_active)
      throw std::logic_error("evicting an adapter with in-flight work");
    if (plora_store_retire(store, a, compute) != 0)
      throw CudaError(std::string("retire failed: ") + plora_last_error());
    store->pool->pool.free(a);
    dyn[a].status = PLORA_NOT_RESIDENT;
    staged_ready.erase(a);
    ++st.evictions;
    log(now_ms, PLORA_DECISION_EVICT, a, score);
    // pages of `a` may still be read by kernels already on the compute
    // stream: order every later copy after them
    PLORA_CUDA(cudaEventRecord(fence, compute));
    PLORA_CUDA(cudaStreamWaitEvent(demand_stream, fence, 0));
    PLORA_CUDA(cudaStreamWaitEvent(prefetch_stream, fence, 0));
  }

  // engine.cpp:310-333
  bool ensure_loading(uint32_t a, bool for_prefetch, double candidate_p, double now,
                      cudaStream_t compute) {
    if (dyn[a].status != PLORA_NOT_RESIDENT || dyn[a].transfer_active) return false;
    if (!src[a]) throw ValidationError("adapter " + std::to_string(a) + " has no host image");
    std::vector<double> scores(A);
    std::vector<uint32_t> keys(A);
    while (true) {
      const int stc = static_cast<int>(store->pool->pool.alloc(a, bytes[a]));
      if (stc == PLORA_OK) break;
      const uint64_t n = plora_scored_residents(dyn.data(), A, &policy, now, scores.data(),
                                                keys.data());
      bool found = false;
      uint32_t victim = 0;
      double vs = 0;
      for (uint64_t i = 0; i < n; ++i) {
        const uint32_t k = keys[i];
        if (dyn[k].busy > 0 || dyn[k].transfer_active) continue;
        if (for_prefetch && scores[i] >= policy.gamma * candidate_p) break;
        found = true;
        victim = k;
        vs = scores[i];
        break;
      }
      if (!found) return false;
      evict(victim, vs, compute);
    }
    nvtxRangePushA(for_prefetch ? "plora.transfer.prefetch" : "plora.transfer.demand");
    start_transfer(a, !for_prefetch);
    nvtxRangePop();
    if (!for_prefetch) ++st.demand_loads;
    log(now, for_prefetch ? PLORA_DECISION_PREFETCH : PLORA_DECISION_DEMAND_LOAD, a,
        for_prefetch ? candidate_p : 0.0, bytes[a]);
    return true;
  }

  void promote_staged(cudaStream_t compute) {  // engine.cpp:406-414
    for (uint32_t a : staged_ready) {
      dyn[a].status = PLORA_RESIDENT;
      prefetch_staged.erase(a);
      ++st.promotions;
      log(now_ms, PLORA_DECISION_PROMOTE, a, 0.0);
      publish(a, compute);
    }
    staged_ready.clear();
  }

  void issue_prefetches(double now, cudaStream_t compute) {  // engine.cpp:459-471
    if (!prefetch_enabled) return;
    uint64_t used = 0;
    for (uint32_t a : prefetch_staged) used += units[a];
    if (used >= staging_total_units) return;
    std::vector<uint32_t> picks(A);
    const uint64_t n = plora_select_prefetch(probs.data(), A, dyn.data(), A, &policy,
                                             units.data(), A, staging_total_units - used,
                                             picks.data());
    for (uint64_t i = 0; i < n; ++i) {
      const uint32_t a = picks[i];
      if (!src[a]) continue;  // no host image: cannot be staged
      if (ensure_loading(a, true, probs[a], now, compute)) {
        ++st.prefetch_issued;
        prefetch_staged.insert(a);
      }
    }
  }

  void maybe_compact(cudaStream_t compute) {  // engine.cpp:486-497
    if (!compaction_enabled || !transfers.empty()) return;
    for (const auto& d : dyn)
      if (d.busy) return;
    PagePool& pool = store->pool->pool;
    const std::size_t moved = pool.compact();
    if (moved == 0) return;
    const auto& rel = pool.last_relocations();
    if (plora_store_apply_relocations(store, rel.data(), rel.size(), compute) != 0)
      throw CudaError(std::string("relocation failed: ") + plora_last_error());
    st.relocations += moved;
    ++st.compactions;
    log(now_ms, PLORA_DECISION_COMPACT, 0xffffffffu, 0.0, moved);
    PLORA_CUDA(cudaEventRecord(fence, compute));
    PLORA_CUDA(cudaStreamWaitEvent(demand_stream, fence, 0));
    PLORA_CUDA(cudaStreamWaitEvent(prefetch_stream, fence, 0));
  }

  // Pump thread: feed prefetch chunks between boundaries.
  void pump_loop() {
    DeviceCtx ctx(store->device);
    std::unique_lock<std::mutex> lk(mu);
    while (!stop) {
      cudaEvent_t wait_on = nullptr;
      try {
        cudaEvent_t dem = active_demand_event();
        if (dem) {
          wait_on = dem;
        } else if (!demand_active()) {
          pump_prefetch();
          if (!prefetch_chunks.empty()) wait_on = prefetch_chunks.front().first;
        }
      } catch (const std::exception&) {
        pump_error = true;  // surfaced by the next boundary
      }
      bool issuing_pending = false;
      for (const auto& [a, t] : transfers)
        if (!t.demand && !t.fully_issued) issuing_pending = true;
      if (wait_on) {
        lk.unlock();
        cudaEventSynchronize(wait_on);  // blocking-sync event: the thread sleeps
        lk.lock();
      } else if (issuing_pending || demand_active()) {
        cv.wait_for(lk, std::chrono::microseconds(50));
      } else {
        cv.wait(lk);
      }
    }
  }
  bool pump_error = false;

  void check_key(uint32_t a) const {
    if (a >= A) throw ValidationError("adapter key " + std::to_string(a) + " out of range");
    if (!store->slots[a].rank)
      throw ValidationError("adapter " + std::to_string(a) + " is not registered");
  }
};

namespace {
plora_engine* E(plora_engine* e) {
  if (!e) throw ValidationError("null engine");
  return e;
}
}  // namespace

extern "C" {

void plora_engine_config_default(plora_engine_config* c) {
  plora_policy_default(&c->policy);
  c->copy_mode = PLORA_COPY_AUTO;
  c->prefetch = 1;
  c->compaction = 1;
  c->chunk_bytes = kDefaultChunk;
  c->prefetch_inflight_bytes = kDefaultPrefetchInflight;
}

int plora_engine_create(plora_store* s, const plora_engine_config* cfg, plora_engine** out) {
  return guard([&] {
    if (!s) throw ValidationError("null store");
    if (plora_policy_validate(&cfg->policy) != 0) throw ValidationError(plora_last_error());
    auto e = std::make_unique<plora_engine>();
    e->store = s;
    e->policy = cfg->policy;
    const uint64_t P = s->pool->pool.page_bytes();
    int mode = cfg->copy_mode;
    if (mode == PLORA_COPY_AUTO) mode = P >= (64u << 10) ? PLORA_COPY_CE : PLORA_COPY_SM;
    if (mode != PLORA_COPY_CE && mode != PLORA_COPY_SM)
      throw ValidationError("unknown copy mode " + std::to_string(cfg->copy_mode));
    e->copy_mode = mode;
    e->prefetch_enabled = cfg->prefetch != 0;
    e->compaction_enabled = cfg->compaction != 0;
    e->chunk_bytes = std::max<uint64_t>(cfg->chunk_bytes, P);
    e->prefetch_inflight_cap = std::max<uint64_t>(cfg->prefetch_inflight_bytes, e->chunk_bytes);
    e->A = s->max_adapters;
    e->dyn.resize(e->A);
    for (auto& d : e->dyn) plora_dynamics_init(&d);
    e->probs.assign(e->A, -1.0);
    e->seen.assign(e->A, 0);
    e->bytes.assign(e->A, 0);
    e->units.assign(e->A, 0);
    e->src.assign(e->A, nullptr);
    e->src_dev.assign(e->A, nullptr);
    // engine.cpp:76-80: staging budget = staging_fraction · pool pages
    e->staging_total_units = static_cast<uint64_t>(cfg->policy.staging_fraction *
                                                   s->pool->pool.total_pages());
    DeviceCtx ctx(s->device);
    int lo = 0, hi = 0;
    PLORA_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));  // hi = greatest priority
    PLORA_CUDA(cudaStreamCreateWithPriority(&e->demand_stream, cudaStreamNonBlocking, hi));
    PLORA_CUDA(cudaStreamCreateWithPriority(&e->prefetch_stream, cudaStreamNonBlocking, lo));
    PLORA_CUDA(cudaEventCreateWithFlags(&e->fence, cudaEventDisableTiming));
    plora_engine* raw = e.get();
    e->pump = std::thread([raw] { raw->pump_loop(); });
    *out = e.release();
    return 0;
  });
}

void plora_engine_destroy(plora_engine* e) {
  if (!e) return;
  e->stop_service();
  {
    std::lock_guard<std::mutex> lk(e->mu);
    e->stop = true;
  }
  e->cv.notify_all();
  if (e->pump.joinable()) e->pump.join();
  DeviceCtx ctx(e->store->device);
  cudaStreamSynchronize(e->demand_stream);
  cudaStreamSynchronize(e->prefetch_stream);
  for (auto& [a, t] : e->transfers) {
    if (t.start) cudaEventDestroy(t.start);
    if (t.done) cudaEventDestroy(t.done);
  }
  for (auto& c : e->prefetch_chunks) cudaEventDestroy(c.first);
  for (auto ev : e->event_pool) cudaEventDestroy(ev);
  for (auto ev : e->timing_pool) cudaEventDestroy(ev);
  cudaEventDestroy(e->fence);
  cudaStreamDestroy(e->demand_stream);
  cudaStreamDestroy(e->prefetch_stream);
  delete e;
}

int plora_engine_set_source(plora_engine* e, uint32_t adapter, const void* host_src,
                            uint64_t bytes) {
  return guard([&] {
    E(e)->check_key(adapter);
    std::lock_guard<std::mutex> lk(e->mu);
    const uint64_t need = e->store->geom.adapter_bytes(e->store->slots[adapter].rank);
    if (bytes != need)
      throw ValidationError("adapter " + std::to_string(adapter) + " image is " +
                            std::to_string(bytes) + " bytes; its rank needs " +
                            std::to_string(need));
    if (!host_src) throw ValidationError("null host image");
    DeviceCtx ctx(e->store->device);
    e->src[adapter] = static_cast<const char*>(host_src);
    e->src_dev[adapter] =
        e->copy_mode == PLORA_COPY_SM ? mapped_source(host_src, bytes) : nullptr;
    e->bytes[adapter] = bytes;
    e->units[adapter] = e->store->pool->pool.pages_needed(bytes);
    return 0;
  });
}

int plora_engine_attach_predictor(plora_engine* e, plora_predictor* p, int async) {
  return guard([&] {
    E(e);
    std::lock_guard<std::mutex> lk(e->mu);
    e->stop_service();
    e->predictor = p;
    if (p && async) {
      e->svc = std::make_unique<plora_engine::PredictorService>();
      e->svc->p = p;
      const uint32_t A = e->A;
      auto* sv = e->svc.get();
      e->svc->th = std::thread([sv, A] { sv->loop(A); });
    }
    return 0;
  });
}

int plora_engine_flush_predictor(plora_engine* e) {
  return guard([&] {
    E(e);
    std::lock_guard<std::mutex> lk(e->mu);
    if (!e->svc) return 0;
    auto& sv = *e->svc;
    std::unique_lock<std::mutex> sl(sv.m);
    // on_arrival wakes the worker only every 64 observations: wake it for
    // the tail, or this wait would outlast a sleeping worker
    sv.cv.notify_one();
    sv.idle.wait(sl, [&] { return sv.obs.empty() && !sv.round_req && !sv.busy; });
    if (!sv.error.empty()) {  // report a worker failure once, then clear it
      std::string msg;
      msg.swap(sv.error);
      throw ValidationError("predictor worker: " + msg);
    }
    if (sv.have) {
      e->apply_predictions(sv.ids.data(), sv.probs.data(), static_cast<int64_t>(sv.ids.size()));
      sv.have = false;
    }
    return 0;
  });
}

int plora_engine_on_arrival(plora_engine* e, uint32_t adapter, double now_ms,
                            plora_stream_t compute) {
  return guard([&] {  // engine.cpp:515-545
    E(e)->check_key(adapter);
    std::lock_guard<std::mutex> lk(e->mu);
    DeviceCtx ctx(e->store->device);
    nvtxRangePushA("plora.arrival");
    e->now_ms = now_ms;
    plora_dynamics& d = e->dyn[adapter];
    const bool hit = d.status == PLORA_RESIDENT;
    ++e->st.arrivals;
    e->seen[adapter] = 1;
    e->actual[e->interval_of(now_ms)].insert(adapter);
    if (hit) ++e->st.hits;
    plora_record_access(&d, now_ms, e->policy.freq_half_life_ms);
    if (e->svc) {
      std::lock_guard<std::mutex> sl(e->svc->m);
      e->svc->obs.emplace_back(adapter, now_ms);
      if (e->svc->obs.size() >= 64) e->svc->cv.notify_one();
    } else if (e->predictor) {
      if (plora_predictor_observe(e->predictor, adapter, now_ms) != 0)
        throw ValidationError(plora_last_error());
    }
    // reactive demand path: absent adapters start loading at arrival
    if (d.status == PLORA_NOT_RESIDENT && !d.transfer_active)
      e->ensure_loading(adapter, false, 0.0, now_ms, static_cast<cudaStream_t>(compute));
    nvtxRangePop();
    return hit ? 1 : 0;
  });
}

int plora_engine_round(plora_engine* e, double now_ms, plora_stream_t compute) {
  return guard([&] {  // engine.cpp:547-561 (predictive mode)
    E(e);
    std::lock_guard<std::mutex> lk(e->mu);
    if (!e->predictor) throw ValidationError("no predictor attached");
    ++e->st.prediction_rounds;
    e->now_ms = now_ms;
    nvtxRangePushA("plora.round");
    struct Pop {
      plora_engine* e;
      double now;
      ~Pop() {
        e->snapshot(now);
        e->evaluate(now);
        nvtxRangePop();
      }
    } pop{e, now_ms};
    if (e->svc) {  // apply the last completed round, request the next one
      auto& sv = *e->svc;
      std::lock_guard<std::mutex> sl(sv.m);
      if (!sv.error.empty()) {  // report a worker failure once, then clear it
      std::string msg;
      msg.swap(sv.error);
      throw ValidationError("predictor worker: " + msg);
    }
      if (sv.have) {
        e->apply_predictions(sv.ids.data(), sv.probs.data(), static_cast<int64_t>(sv.ids.size()));
        sv.have = false;
      }
      sv.round_req = true;
      sv.round_now = now_ms;
      sv.cv.notify_one();
      return 0;
    }
    std::vector<uint32_t> ids(e->A);
    std::vector<double> p(e->A);
    const int64_t n = plora_predictor_predict_all(e->predictor, now_ms, ids.data(), p.data(),
                                                  e->A);
    if (n < 0) throw ValidationError(plora_last_error());
    e->apply_predictions(ids.data(), p.data(), n);
    (void)compute;
    return 0;
  });
}

int plora_engine_set_predictions(plora_engine* e, const double* probs, uint64_t n) {
  return guard([&] {  // engine.cpp:562-571 (oracle / external predictions)
    E(e);
    std::lock_guard<std::mutex> lk(e->mu);
    if (n > e->A) throw ValidationError("more predictions than adapter keys");
    std::fill(e->probs.begin(), e->probs.end(), -1.0);
    for (uint64_t a = 0; a < n; ++a) {
      e->probs[a] = probs[a];
      e->dyn[a].prediction = probs[a];
    }
    ++e->st.prediction_rounds;
    e->snapshot(e->now_ms);
    e->evaluate(e->now_ms);
    return 0;
  });
}

int plora_engine_acquire(plora_engine* e, uint32_t adapter, double now_ms,
                         plora_stream_t compute_) {
  return guard([&] {  // admit_requests, engine.cpp:416-457
    E(e)->check_key(adapter);
    std::lock_guard<std::mutex> lk(e->mu);
    DeviceCtx ctx(e->store->device);
    cudaStream_t compute = static_cast<cudaStream_t>(compute_);
    plora_dynamics& d = e->dyn[adapter];
    e->now_ms = now_ms;
    if (d.status == PLORA_NOT_RESIDENT && !d.transfer_active) {
      if (!e->ensure_loading(adapter, false, 0.0, now_ms, compute)) {
        ++e->st.admission_failures;
        e->log(now_ms, PLORA_DECISION_ADMISSION_FAILURE, adapter, 0.0);
        return PLORA_ADMIT_FAILED;
      }
    }
    ++d.busy;
    if (e->staged_ready.count(adapter)) {  // staged between boundaries: promote now
      e->staged_ready.erase(adapter);
      d.status = PLORA_RESIDENT;
      e->prefetch_staged.erase(adapter);
      ++e->st.promotions;
      e->publish(adapter, compute);
    }
    if (d.status == PLORA_RESIDENT) return PLORA_ADMIT_READY;
    Transfer& t = e->transfers.at(adapter);
    if (!t.demand) {  // a demanded staging transfer takes demand priority
      t.demand = true;
      t.upgraded = true;
      ++e->st.upgrades;
      e->issue_all_demand(adapter, t);
    }
    return PLORA_ADMIT_LOADING;
  });
}

int plora_engine_wait_ready(plora_engine* e, uint32_t adapter, plora_stream_t compute_) {
  return guard([&] {
    E(e)->check_key(adapter);
    std::lock_guard<std::mutex> lk(e->mu);
    DeviceCtx ctx(e->store->device);
    cudaStream_t compute = static_cast<cudaStream_t>(compute_);
    plora_dynamics& d = e->dyn[adapter];
    if (d.status == PLORA_RESIDENT) return 0;
    auto it = e->transfers.find(adapter);
    if (it == e->transfers.end()) {
      if (e->staged_ready.count(adapter)) {
        e->staged_ready.erase(adapter);
        d.status = PLORA_RESIDENT;
        e->prefetch_staged.erase(adapter);
        ++e->st.promotions;
        e->publish(adapter, compute);
        return 0;
      }
      throw ValidationError("adapter " + std::to_string(adapter) + " is neither resident nor loading");
    }
    Transfer& t = it->second;
    if (!t.demand) {
      t.demand = true;
      t.upgraded = true;
      ++e->st.upgrades;
    }
    e->issue_all_demand(adapter, t);
    // device-side wait inside complete_transfer: the compute stream orders
    // after the copy, the host does not block
    e->complete_transfer(adapter, t, compute);
    return 0;
  });
}

int plora_engine_release(plora_engine* e, uint32_t adapter) {
  return guard([&] {  // finish_request, engine.cpp:358-372
    E(e)->check_key(adapter);
    std::lock_guard<std::mutex> lk(e->mu);
    if (e->dyn[adapter].busy == 0) throw std::logic_error("release without acquire");
    --e->dyn[adapter].busy;
    return 0;
  });
}

int plora_engine_boundary(plora_engine* e, double now_ms, plora_stream_t compute_) {
  return guard([&] {  // do_boundary, engine.cpp:406-414
    E(e);
    std::lock_guard<std::mutex> lk(e->mu);
    DeviceCtx ctx(e->store->device);
    cudaStream_t compute = static_cast<cudaStream_t>(compute_);
    if (e->pump_error) throw CudaError("prefetch pump failed (see CUDA error state)");
    nvtxRangePushA("plora.boundary");
    e->now_ms = now_ms;
    const int done = e->poll_transfers(compute);
    e->promote_staged(compute);
    e->issue_prefetches(now_ms, compute);
    e->maybe_compact(compute);
    e->evaluate(now_ms);
    e->cv.notify_one();
    nvtxRangePop();
    return done;
  });
}

int plora_engine_sync(plora_engine* e) {
  return guard([&] {
    E(e);
    DeviceCtx ctx(e->store->device);
    // wait until the pump has issued every prefetch chunk, then drain both streams
    while (true) {
      {
        std::lock_guard<std::mutex> lk(e->mu);
        bool pending = false;
        for (auto& [a, t] : e->transfers)
          if (!t.fully_issued) pending = true;
        if (!pending) break;
        e->cv.notify_one();
      }
      std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
    PLORA_CUDA(cudaStreamSynchronize(e->demand_stream));
    PLORA_CUDA(cudaStreamSynchronize(e->prefetch_stream));
    return 0;
  });
}

int64_t plora_engine_on_arrivals(plora_engine* e, const uint32_t* adapters, uint64_t n,
                                 double now_ms, plora_stream_t compute) {
  int64_t hits = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const int rc = plora_engine_on_arrival(e, adapters[i], now_ms, compute);
    if (rc < 0) return rc;
    hits += rc;
  }
  return hits;
}

int plora_engine_admit(plora_engine* e, const uint32_t* adapters, uint64_t n, double now_ms,
                       plora_stream_t compute, int wait, int32_t* status) {
  for (uint64_t i = 0; i < n; ++i) {
    int st = plora_engine_acquire(e, adapters[i], now_ms, compute);
    if (st < 0) return st;
    if (st == PLORA_ADMIT_LOADING && wait) {
      const int rc = plora_engine_wait_ready(e, adapters[i], compute);
      if (rc < 0) return rc;
    }
    if (status) status[i] = st;
  }
  return 0;
}

int plora_engine_release_many(plora_engine* e, const uint32_t* adapters, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) {
    const int rc = plora_engine_release(e, adapters[i]);
    if (rc < 0) return rc;
  }
  return 0;
}

int plora_engine_status(const plora_engine* e, uint32_t adapter, plora_dynamics* out) {
  return guard([&] {
    if (!e) throw ValidationError("null engine");
    e->check_key(adapter);
    std::lock_guard<std::mutex> lk(e->mu);
    *out = e->dyn[adapter];
    return 0;
  });
}

void plora_engine_get_stats(const plora_engine* e, plora_engine_stats* out) {
  if (!e || !out) return;
  std::lock_guard<std::mutex> lk(e->mu);
  *out = e->st;
  out->in_flight = e->transfers.size();
  out->staged = e->staged_ready.size();
  uint64_t resident = 0;
  for (const auto& d : e->dyn)
    if (d.status == PLORA_RESIDENT) ++resident;
  out->resident = resident;
  out->copy_mode = e->copy_mode;
  if (e->svc) {
    std::lock_guard<std::mutex> sl(e->svc->m);
    out->predictor_ms = e->svc->busy_ms;
  }
}

uint64_t plora_engine_decisions(const plora_engine* e, uint64_t start, plora_decision* out,
                                uint64_t cap) {
  if (!e) return 0;
  std::lock_guard<std::mutex> lk(e->mu);
  const uint64_t n = e->decisions.size();
  for (uint64_t i = start; i < n && i - start < cap && out; ++i) out[i - start] = e->decisions[i];
  return n;
}

int plora_engine_set_decision_log(plora_engine* e, int enabled) {
  return guard([&] {
    E(e);
    std::lock_guard<std::mutex> lk(e->mu);
    e->log_decisions = enabled != 0;
    if (!enabled) e->decisions.clear();
    return 0;
  });
}

int plora_engine_set_accuracy_interval(plora_engine* e, double interval_ms, double warmup_ms) {
  return guard([&] {  // cfg_.predictor.interval_ms, cfg_.run.warmup_s (engine.cpp:598-633)
    E(e);
    if (!(interval_ms > 0)) throw ValidationError("accuracy interval must be positive");
    std::lock_guard<std::mutex> lk(e->mu);
    e->acc_interval_ms = interval_ms;
    e->acc_warmup_ms = warmup_ms;
    e->snapshots.clear();
    e->actual.clear();
    e->last_snapshot = -1;
    return 0;
  });
}

int plora_engine_streams(const plora_engine* e, plora_stream_t* demand, plora_stream_t* prefetch) {
  return guard([&] {
    if (!e) throw ValidationError("null engine");
    if (demand) *demand = e->demand_stream;
    if (prefetch) *prefetch = e->prefetch_stream;
    return 0;
  });
}

}  // extern "C"
