// plora.hpp — header-only C++ face of libplora.so, shaped like the reference's
// own headers so a lorasim caller can switch by changing includes/namespace:
//
//   lorasim::PagePool        (include/lorasim/memory.hpp:39-83)  -> plora::PagePool
//   lorasim::AllocStatus     (memory.hpp:18-22)                  -> plora::AllocStatus
//   lorasim::ValidationError / ConfigError / ParseError (errors.hpp:9-24)
//                                                                -> same names in plora::
//   std::logic_error on double free / re-alloc                   -> std::logic_error
//
// Every method forwards to the C ABI (include/plora.h) and rethrows the
// reference's exception type for the returned status code.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "plora.h"

namespace plora {

class ValidationError : public std::runtime_error {
 public:
  explicit ValidationError(const std::string& m) : std::runtime_error(m) {}
};
class ConfigError : public std::runtime_error {
 public:
  explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
class ParseError : public std::runtime_error {
 public:
  explicit ParseError(const std::string& m) : std::runtime_error(m) {}
};
class CudaError : public std::runtime_error {
 public:
  explicit CudaError(const std::string& m) : std::runtime_error(m) {}
};

inline int check(int rc) {
  if (rc >= 0) return rc;
  const std::string msg = plora_last_error();
  switch (rc) {
    case PLORA_E_VALIDATION: throw ValidationError(msg);
    case PLORA_E_CONFIG: throw ConfigError(msg);
    case PLORA_E_PARSE: throw ParseError(msg);
    case PLORA_E_CUDA: throw CudaError(msg);
    case PLORA_E_NOMEM: throw std::bad_alloc();
    default: throw std::logic_error(msg);
  }
}

using AdapterKey = std::uint32_t;

enum class AllocStatus { ok = 0, out_of_memory = 1, fragmentation_failure = 2 };

struct FragmentationReport {
  double external_frag = 0.0;
  double internal_frag = 0.0;
  double utilization = 0.0;
};

struct PageTable {
  AdapterKey adapter = 0;
  std::uint64_t weight_bytes = 0;
  std::vector<std::uint32_t> entries;
};

// Drop-in for lorasim::PagePool: identical placement, errors and dump().
class PagePool {
 public:
  PagePool(std::uint64_t page_bytes, std::uint32_t total_pages) {
    check(plora_pool_create(page_bytes, total_pages, &p_));
  }
  ~PagePool() { plora_pool_destroy(p_); }
  PagePool(const PagePool&) = delete;
  PagePool& operator=(const PagePool&) = delete;
  PagePool(PagePool&& o) noexcept : p_(o.p_) { o.p_ = nullptr; }

  std::uint32_t pages_needed(std::uint64_t bytes) const { return plora_pool_pages_needed(p_, bytes); }
  AllocStatus alloc(AdapterKey adapter, std::uint64_t weight_bytes) {
    return static_cast<AllocStatus>(check(plora_pool_alloc(p_, adapter, weight_bytes)));
  }
  void free(AdapterKey adapter) { check(plora_pool_free(p_, adapter)); }
  std::uint32_t translate(AdapterKey adapter, std::uint32_t logical) const {
    std::uint32_t out = 0;
    check(plora_pool_translate(p_, adapter, logical, &out));
    return out;
  }
  std::size_t compact() {
    std::uint64_t moved = 0;
    check(plora_pool_compact(p_, &moved));
    return static_cast<std::size_t>(moved);
  }
  std::vector<plora_reloc> last_relocations() const {
    const plora_reloc* r = nullptr;
    std::uint64_t n = 0;
    plora_pool_last_relocations(p_, &r, &n);
    return std::vector<plora_reloc>(r, r + n);
  }
  FragmentationReport report() const {
    plora_frag_report r{};
    plora_pool_report(p_, &r);
    return FragmentationReport{r.external_frag, r.internal_frag, r.utilization};
  }
  std::string dump() const {  // == lorasim's dump().dump()
    std::uint64_t n = 0;
    check(plora_pool_dump(p_, nullptr, 0, &n));
    std::string s(n + 1, '\0');
    check(plora_pool_dump(p_, s.data(), n + 1, &n));
    s.resize(n);
    return s;
  }
  bool has(AdapterKey adapter) const { return plora_pool_has(p_, adapter) != 0; }
  PageTable table(AdapterKey adapter) const {
    const std::uint32_t* e = nullptr;
    std::uint32_t n = 0;
    PageTable t;
    check(plora_pool_table(p_, adapter, &e, &n, &t.weight_bytes));
    t.adapter = adapter;
    t.entries.assign(e, e + n);
    return t;
  }
  std::uint32_t free_pages() const { return plora_pool_free_pages(p_); }
  std::uint32_t total_pages() const { return plora_pool_total_pages(p_); }
  std::uint64_t page_bytes() const { return plora_pool_page_bytes(p_); }
  std::uint64_t used_bytes() const { return plora_pool_used_bytes(p_); }
  std::uint64_t allocated_bytes() const { return plora_pool_allocated_bytes(p_); }
  std::uint64_t total_bytes() const { return plora_pool_total_bytes(p_); }
  std::vector<AdapterKey> resident() const {
    std::vector<AdapterKey> out(plora_pool_resident(p_, nullptr, 0));
    plora_pool_resident(p_, out.data(), out.size());
    return out;
  }
  void check_invariants() const { check(plora_pool_check_invariants(p_)); }

  plora_pool* handle() const { return p_; }

 private:
  plora_pool* p_ = nullptr;
};

// ------------------------------------------------------ device path (new)
// The adapter pages in HBM behind a PagePool (which must outlive the store).
class DeviceStore {
 public:
  DeviceStore(PagePool& pool, int device, const plora_model& model, std::uint32_t max_adapters) {
    check(plora_store_create(pool.handle(), device, &model, max_adapters, &s_));
  }
  ~DeviceStore() { plora_store_destroy(s_); }
  DeviceStore(const DeviceStore&) = delete;
  DeviceStore& operator=(const DeviceStore&) = delete;

  void register_adapter(AdapterKey a, std::uint32_t rank) { check(plora_store_register(s_, a, rank)); }
  // H2D page scatter of the adapter's logical bytes (start_transfer, engine.cpp:250-259)
  void write_pages(AdapterKey a, const void* host_src, std::uint64_t bytes,
                   int mode = PLORA_COPY_CE, plora_stream_t stream = nullptr) {
    check(plora_store_write_pages(s_, a, host_src, bytes, mode, stream));
  }
  // promotion (engine.cpp:406-414) / eviction (engine.cpp:294-304)
  void publish(AdapterKey a, plora_stream_t stream = nullptr) { check(plora_store_publish(s_, a, stream)); }
  void retire(AdapterKey a, plora_stream_t stream = nullptr) { check(plora_store_retire(s_, a, stream)); }
  bool is_published(AdapterKey a) const { return plora_store_is_published(s_, a) != 0; }

  plora_store* handle() const { return s_; }

 private:
  plora_store* s_ = nullptr;
};

// A batch's tokens grouped by adapter (reused for every (layer, proj) call).
class BatchPlan {
 public:
  BatchPlan(DeviceStore& store, const std::vector<std::int32_t>& token_adapter,
            plora_stream_t stream = nullptr) {
    check(plora_plan_create(store.handle(), token_adapter.data(),
                            static_cast<std::uint32_t>(token_adapter.size()), stream, &p_));
  }
  ~BatchPlan() { plora_plan_destroy(p_); }
  BatchPlan(const BatchPlan&) = delete;
  BatchPlan& operator=(const BatchPlan&) = delete;
  void update(const std::vector<std::int32_t>& token_adapter, plora_stream_t stream = nullptr) {
    check(plora_plan_update(p_, token_adapter.data(), static_cast<std::uint32_t>(token_adapter.size()),
                            stream));
  }
  plora_plan* handle() const { return p_; }

 private:
  plora_plan* p_ = nullptr;
};

// y += scale · (x · Aᵀ) · Bᵀ per token; device pointers, strides in elements.
inline void bgmv(BatchPlan& plan, std::uint32_t layer, std::uint32_t proj, const void* x,
                 std::uint64_t ldx, void* y, std::uint64_t ldy, float scale = 1.f,
                 plora_stream_t stream = nullptr) {
  check(plora_bgmv(plan.handle(), layer, proj, x, ldx, y, ldy, scale, stream));
}
inline void sgmv(BatchPlan& plan, std::uint32_t layer, std::uint32_t proj, const void* x,
                 std::uint64_t ldx, void* y, std::uint64_t ldy, float scale = 1.f,
                 plora_stream_t stream = nullptr) {
  check(plora_sgmv(plan.handle(), layer, proj, x, ldx, y, ldy, scale, stream));
}
// every projection of a layer (they share x): decode / prefill
inline void bgmv_layer(BatchPlan& plan, std::uint32_t layer, const void* x, std::uint64_t ldx,
                       void* const* ys, const std::uint64_t* ldys, float scale = 1.f,
                       plora_stream_t stream = nullptr) {
  check(plora_bgmv_layer(plan.handle(), layer, x, ldx, ys, ldys, scale, stream));
}
inline void sgmv_layer(BatchPlan& plan, std::uint32_t layer, const void* x, std::uint64_t ldx,
                       void* const* ys, const std::uint64_t* ldys, float scale = 1.f,
                       plora_stream_t stream = nullptr) {
  check(plora_sgmv_layer(plan.handle(), layer, x, ldx, ys, ldys, scale, stream));
}
// y = x · W0ᵀ + scale · (x · Aᵀ) · Bᵀ (base projection fused, prefill)
inline void sgmv_fused(BatchPlan& plan, std::uint32_t layer, std::uint32_t proj, const void* x,
                       std::uint64_t ldx, const void* w0, std::uint64_t ldw, void* y,
                       std::uint64_t ldy, float scale = 1.f, plora_stream_t stream = nullptr) {
  check(plora_sgmv_fused(plan.handle(), layer, proj, x, ldx, w0, ldw, y, ldy, scale, stream));
}

// every projection of a layer with its base weight (x read once by the shrink)
inline void sgmv_fused_layer(BatchPlan& plan, std::uint32_t layer, const void* x, std::uint64_t ldx,
                             const void* const* w0s, const std::uint64_t* ldws, void* const* ys,
                             const std::uint64_t* ldys, float scale = 1.f,
                             plora_stream_t stream = nullptr) {
  check(plora_sgmv_fused_layer(plan.handle(), layer, x, ldx, w0s, ldws, ys, ldys, scale, stream));
}

}  // namespace plora
