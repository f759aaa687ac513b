// plora_lorasim.hpp — libplora's page pool with the reference's own types, for
// callers that keep the rest of lorasim (include/lorasim/memory.hpp's
// AllocStatus, FragmentationReport, PageTable, BlockArena and errors.hpp's
// exceptions).  Include it after lorasim/memory.hpp; then the engine's
//
//   std::optional<PagePool> pool_;                          (src/engine.cpp:748)
//
// becomes std::optional<lorasim::PloraPagePool> pool_ and every use compiles
// unchanged: `pool_ ? pool_->alloc(a, b) : arena_->alloc(a, b)` (engine.cpp:293,
// both branches lorasim::AllocStatus), `FragmentationReport rep = pool_ ?
// pool_->report() : arena_->report()` (:587), `pool_->pages_needed(..)`
// (:78), `pool_->free(a)` (:299), `pool_->compact()` (:489), and
// `table(a)` returns a const reference valid until the next mutation, as
// lorasim::PagePool::table does (memory.hpp:65).  Placement, errors and
// dump() are identical to lorasim::PagePool (tests/test_pagepool.py,
// tests/test_cpp_dropin.py::test_engine_excerpt_against_reference).
#pragma once

#include <map>
#include <utility>

#include "plora.hpp"

namespace lorasim {

class PloraPagePool {
 public:
  PloraPagePool(std::uint64_t page_bytes, std::uint32_t total_pages)
      : p_(rethrow([&] { return plora::PagePool(page_bytes, total_pages); })) {}

  std::uint32_t pages_needed(std::uint64_t bytes) const { return p_.pages_needed(bytes); }
  AllocStatus alloc(AdapterKey adapter, std::uint64_t weight_bytes) {
    tables_.erase(adapter);
    return static_cast<AllocStatus>(rethrow([&] { return p_.alloc(adapter, weight_bytes); }));
  }
  void free(AdapterKey adapter) {
    tables_.erase(adapter);
    rethrow([&] {
      p_.free(adapter);
      return 0;
    });
  }
  std::uint32_t translate(AdapterKey adapter, std::uint32_t logical) const {
    return rethrow([&] { return p_.translate(adapter, logical); });
  }
  std::size_t compact() {
    tables_.clear();
    return p_.compact();
  }
  FragmentationReport report() const {
    const plora::FragmentationReport r = p_.report();
    return FragmentationReport{r.external_frag, r.internal_frag, r.utilization};
  }
  nlohmann::json dump() const { return nlohmann::json::parse(p_.dump()); }
  bool has(AdapterKey adapter) const { return p_.has(adapter); }
  const PageTable& table(AdapterKey adapter) const {
    auto it = tables_.find(adapter);
    if (it == tables_.end()) {
      plora::PageTable t = rethrow([&] { return p_.table(adapter); });
      it = tables_.emplace(adapter, PageTable{t.adapter, t.weight_bytes, std::move(t.entries)}).first;
    }
    return it->second;
  }
  std::uint32_t free_pages() const { return p_.free_pages(); }
  std::uint32_t total_pages() const { return p_.total_pages(); }
  std::uint64_t page_bytes() const { return p_.page_bytes(); }
  std::uint64_t used_bytes() const { return p_.used_bytes(); }
  std::uint64_t allocated_bytes() const { return p_.allocated_bytes(); }
  std::uint64_t total_bytes() const { return p_.total_bytes(); }
  std::vector<AdapterKey> resident() const { return p_.resident(); }
  void check_invariants() const {
    rethrow([&] {
      p_.check_invariants();
      return 0;
    });
  }
  plora::PagePool& native() { return p_; }

 private:
  // plora's exception types -> lorasim's (errors.hpp:9-24); logic_error as is
  template <class F>
  static auto rethrow(F&& f) -> decltype(f()) {
    try {
      return f();
    } catch (const plora::ValidationError& e) {
      throw ValidationError(e.what());
    } catch (const plora::ConfigError& e) {
      throw ConfigError(e.what());
    } catch (const plora::ParseError& e) {
      throw ParseError(e.what());
    }
  }
  plora::PagePool p_;
  mutable std::map<AdapterKey, PageTable> tables_;  // table() references, dropped on mutation
};

}  // namespace lorasim
