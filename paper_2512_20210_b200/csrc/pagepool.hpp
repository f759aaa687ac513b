// Host-side page pool: bit-identical placement to lorasim::PagePool
// (include/lorasim/memory.hpp:39-83, src/memory.cpp:7-146) on a two-level
// free bitmap instead of an ordered std::set.
//
//  * alloc   — the `need` lowest free physical indices, ascending, atomic on
//              OOM (memory.cpp:18-38).  Cost O(need + words scanned).
//  * free    — returns pages; logic_error on double free (memory.cpp:40-53).
//  * compact — pages >= live move to the lowest free slots, visiting tables
//              in adapter-key order then logical order (memory.cpp:71-89);
//              additionally records the relocation list for the device.
#pragma once

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "common.hpp"

namespace plora {

using AdapterKey = std::uint32_t;

enum class AllocStatus : int { ok = 0, out_of_memory = 1, fragmentation_failure = 2 };

struct FragmentationReport {
  double external_frag = 0.0;
  double internal_frag = 0.0;
  double utilization = 0.0;
};

struct PageTable {
  AdapterKey adapter = 0;
  std::uint64_t weight_bytes = 0;
  std::vector<std::uint32_t> entries;  // logical i -> physical page
};

class PagePool {
 public:
  PagePool(std::uint64_t page_bytes, std::uint32_t total_pages);

  std::uint32_t pages_needed(std::uint64_t bytes) const;
  AllocStatus alloc(AdapterKey adapter, std::uint64_t weight_bytes);
  void free(AdapterKey adapter);
  std::uint32_t translate(AdapterKey adapter, std::uint32_t logical) const;
  std::size_t compact();
  const std::vector<plora_reloc>& last_relocations() const { return relocs_; }

  FragmentationReport report() const;
  std::string dump() const;  // == nlohmann::json(...).dump() of the reference

  bool has(AdapterKey adapter) const { return tables_.count(adapter) > 0; }
  const PageTable& table(AdapterKey adapter) const;
  std::uint32_t free_pages() const { return free_count_; }
  std::uint32_t total_pages() const { return total_pages_; }
  std::uint64_t page_bytes() const { return page_bytes_; }
  std::uint64_t used_bytes() const { return used_bytes_; }
  std::uint64_t allocated_bytes() const {
    return static_cast<std::uint64_t>(total_pages_ - free_count_) * page_bytes_;
  }
  std::uint64_t total_bytes() const {
    return static_cast<std::uint64_t>(total_pages_) * page_bytes_;
  }
  std::vector<AdapterKey> resident() const;
  void check_invariants() const;

  // Monotone counter bumped by every mutation (alloc/free/compact); lets the
  // device store detect stale published tables.
  std::uint64_t generation() const { return generation_; }

 private:
  bool is_free(std::uint32_t i) const { return (bits_[i >> 6] >> (i & 63)) & 1u; }
  void set_free(std::uint32_t i);
  void set_used(std::uint32_t i);
  std::uint32_t lowest_free_from(std::uint32_t start) const;  // total_pages_ if none

  std::uint64_t page_bytes_;
  std::uint32_t total_pages_;
  std::uint64_t used_bytes_ = 0;
  std::uint32_t free_count_ = 0;
  std::vector<std::uint64_t> bits_;     // bit i: page i is free
  std::vector<std::uint64_t> summary_;  // bit w: bits_[w] != 0
  std::vector<std::int64_t> owner_;     // physical page -> adapter, -1 free
  std::map<AdapterKey, PageTable> tables_;
  std::vector<plora_reloc> relocs_;
  std::uint64_t generation_ = 0;
};

}  // namespace plora
