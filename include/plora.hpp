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

}  // namespace plora
