// See pagepool.hpp.  Reference: /root/reference/proj/src/memory.cpp:7-146.
#include "pagepool.hpp"

#include <algorithm>
#include <set>

namespace plora {

PagePool::PagePool(std::uint64_t page_bytes, std::uint32_t total_pages)
    : page_bytes_(page_bytes), total_pages_(total_pages) {
  // memory.cpp:9
  if (page_bytes_ == 0) throw ValidationError("page size must be positive");
  owner_.assign(total_pages_, -1);
  const std::size_t words = (static_cast<std::size_t>(total_pages_) + 63) / 64;
  bits_.assign(words, ~0ull);
  if (total_pages_ % 64) bits_.back() = (1ull << (total_pages_ % 64)) - 1;
  summary_.assign((words + 63) / 64, 0);
  for (std::size_t w = 0; w < words; ++w)
    if (bits_[w]) summary_[w >> 6] |= 1ull << (w & 63);
  free_count_ = total_pages_;
}

// memory.cpp:14-16 — same u64 arithmetic and u32 truncation as the reference.
std::uint32_t PagePool::pages_needed(std::uint64_t bytes) const {
  return static_cast<std::uint32_t>((bytes + page_bytes_ - 1) / page_bytes_);
}

void PagePool::set_free(std::uint32_t i) {
  const std::uint32_t w = i >> 6;
  bits_[w] |= 1ull << (i & 63);
  summary_[w >> 6] |= 1ull << (w & 63);
}

void PagePool::set_used(std::uint32_t i) {
  const std::uint32_t w = i >> 6;
  bits_[w] &= ~(1ull << (i & 63));
  if (!bits_[w]) summary_[w >> 6] &= ~(1ull << (w & 63));
}

std::uint32_t PagePool::lowest_free_from(std::uint32_t start) const {
  if (start >= total_pages_) return total_pages_;
  std::size_t w = start >> 6;
  std::uint64_t word = bits_[w] & (~0ull << (start & 63));
  if (word) return static_cast<std::uint32_t>((w << 6) + __builtin_ctzll(word));
  // next non-empty word via the summary
  std::size_t sw = (w + 1) >> 6;
  if (sw >= summary_.size()) return total_pages_;
  std::uint64_t s = summary_[sw] & (((w + 1) & 63) ? (~0ull << ((w + 1) & 63)) : ~0ull);
  while (true) {
    if (s) {
      std::size_t nw = (sw << 6) + __builtin_ctzll(s);
      return static_cast<std::uint32_t>((nw << 6) + __builtin_ctzll(bits_[nw]));
    }
    if (++sw >= summary_.size()) return total_pages_;
    s = summary_[sw];
  }
}

// memory.cpp:18-38
AllocStatus PagePool::alloc(AdapterKey adapter, std::uint64_t weight_bytes) {
  if (weight_bytes == 0) throw ValidationError("cannot allocate zero bytes");
  if (tables_.count(adapter))
    throw std::logic_error("adapter " + std::to_string(adapter) + " already allocated");
  const std::uint32_t need = pages_needed(weight_bytes);
  if (free_count_ < need) return AllocStatus::out_of_memory;

  PageTable table;
  table.adapter = adapter;
  table.weight_bytes = weight_bytes;
  table.entries.resize(need);
  const std::int64_t owner = static_cast<std::int64_t>(adapter);
  std::uint32_t got = 0;
  std::uint32_t cursor = 0;
  while (got < need) {
    std::uint32_t i = lowest_free_from(cursor);  // guaranteed < total (free_count_ >= need)
    std::size_t w = i >> 6;
    std::uint64_t word = bits_[w] & (~0ull << (i & 63));
    // take ascending set bits of this word
    std::uint64_t taken = 0;
    while (word && got < need) {
      std::uint64_t low = word & (~word + 1);
      std::uint32_t phys = static_cast<std::uint32_t>((w << 6) + __builtin_ctzll(word));
      table.entries[got++] = phys;
      owner_[phys] = owner;
      taken |= low;
      word &= word - 1;
    }
    bits_[w] &= ~taken;
    if (!bits_[w]) summary_[w >> 6] &= ~(1ull << (w & 63));
    cursor = static_cast<std::uint32_t>((w + 1) << 6);
  }
  free_count_ -= need;
  used_bytes_ += weight_bytes;
  tables_.emplace(adapter, std::move(table));
  ++generation_;
  return AllocStatus::ok;
}

// memory.cpp:40-53
void PagePool::free(AdapterKey adapter) {
  auto it = tables_.find(adapter);
  if (it == tables_.end())
    throw std::logic_error("free of adapter " + std::to_string(adapter) +
                           " which holds no pages");
  const std::int64_t owner = static_cast<std::int64_t>(adapter);
  for (std::uint32_t phys : it->second.entries) {
    if (owner_[phys] != owner)
      throw std::logic_error("page table corruption: page not owned by adapter");
    owner_[phys] = -1;
    set_free(phys);
  }
  free_count_ += static_cast<std::uint32_t>(it->second.entries.size());
  used_bytes_ -= it->second.weight_bytes;
  tables_.erase(it);
  ++generation_;
}

// memory.cpp:55-62
std::uint32_t PagePool::translate(AdapterKey adapter, std::uint32_t logical) const {
  const PageTable& t = table(adapter);
  if (logical >= t.entries.size())
    throw ValidationError("logical page " + std::to_string(logical) +
                          " out of range (adapter has " + std::to_string(t.entries.size()) +
                          " pages)");
  return t.entries[logical];
}

// memory.cpp:64-69
const PageTable& PagePool::table(AdapterKey adapter) const {
  auto it = tables_.find(adapter);
  if (it == tables_.end())
    throw ValidationError("no page table for adapter " + std::to_string(adapter));
  return it->second;
}

// memory.cpp:71-89.  The lowest free slot is monotone during the walk: every
// freed source is >= live > every target, so a forward cursor suffices.
std::size_t PagePool::compact() {
  relocs_.clear();
  const std::uint32_t live = total_pages_ - free_count_;
  std::size_t moved = 0;
  std::uint32_t cursor = 0;
  for (auto& [adapter, table] : tables_) {
    for (std::uint32_t logical = 0; logical < table.entries.size(); ++logical) {
      std::uint32_t& phys = table.entries[logical];
      if (phys < live) continue;
      std::uint32_t target = lowest_free_from(cursor);
      cursor = target + 1;
      set_used(target);
      set_free(phys);
      owner_[target] = owner_[phys];
      owner_[phys] = -1;
      relocs_.push_back(plora_reloc{adapter, logical, phys, target});
      phys = target;
      ++moved;
    }
  }
  if (moved) ++generation_;
  return moved;
}

// memory.cpp:91-100
FragmentationReport PagePool::report() const {
  FragmentationReport r;
  r.external_frag = 0.0;
  std::uint64_t allocated = allocated_bytes();
  r.internal_frag =
      allocated == 0 ? 0.0 : static_cast<double>(allocated - used_bytes_) / allocated;
  r.utilization = static_cast<double>(used_bytes_) / total_bytes();
  return r;
}

// memory.cpp:102-114 — nlohmann::json orders object keys lexicographically
// and dump() is compact, so the text is reproduced byte for byte.
std::string PagePool::dump() const {
  std::string s;
  s.reserve(32 + owner_.size() * 3 + tables_.size() * 64);
  s += "{\"owner\":[";
  for (std::size_t i = 0; i < owner_.size(); ++i) {
    if (i) s += ',';
    s += std::to_string(owner_[i]);
  }
  s += "],\"page_bytes\":";
  s += std::to_string(page_bytes_);
  s += ",\"tables\":{";
  std::map<std::string, const PageTable*> by_name;
  for (const auto& [a, t] : tables_) by_name.emplace(std::to_string(a), &t);
  bool first = true;
  for (const auto& [name, t] : by_name) {
    if (!first) s += ',';
    first = false;
    s += '"';
    s += name;
    s += "\":{\"entries\":[";
    for (std::size_t i = 0; i < t->entries.size(); ++i) {
      if (i) s += ',';
      s += std::to_string(t->entries[i]);
    }
    s += "],\"weight_bytes\":";
    s += std::to_string(t->weight_bytes);
    s += '}';
  }
  s += "},\"total_pages\":";
  s += std::to_string(total_pages_);
  s += '}';
  return s;
}

std::vector<AdapterKey> PagePool::resident() const {
  std::vector<AdapterKey> out;
  out.reserve(tables_.size());
  for (const auto& [adapter, _] : tables_) out.push_back(adapter);
  return out;
}

// memory.cpp:123-146, plus bitmap/summary consistency.
void PagePool::check_invariants() const {
  std::size_t allocated = 0;
  for (auto o : owner_)
    if (o >= 0) ++allocated;
  if (allocated + free_count_ != total_pages_)
    throw std::logic_error("page conservation violated");
  std::size_t bit_free = 0;
  for (std::size_t w = 0; w < bits_.size(); ++w) {
    bit_free += static_cast<std::size_t>(__builtin_popcountll(bits_[w]));
    bool s = (summary_[w >> 6] >> (w & 63)) & 1u;
    if (s != (bits_[w] != 0)) throw std::logic_error("free-bitmap summary out of sync");
  }
  if (bit_free != free_count_) throw std::logic_error("page conservation violated");
  std::vector<char> seen(total_pages_, 0);
  std::uint64_t used = 0;
  std::size_t seen_n = 0;
  for (const auto& [adapter, table] : tables_) {
    if (table.entries.size() != pages_needed(table.weight_bytes))
      throw std::logic_error("page table entry count != ceil(S/P)");
    used += table.weight_bytes;
    for (std::uint32_t phys : table.entries) {
      if (seen[phys]) throw std::logic_error("physical page mapped twice");
      seen[phys] = 1;
      ++seen_n;
      if (owner_[phys] != static_cast<std::int64_t>(adapter))
        throw std::logic_error("owner map does not match page table");
      if (is_free(phys)) throw std::logic_error("allocated page present in free list");
    }
  }
  if (seen_n != allocated) throw std::logic_error("orphan allocated pages");
  if (used != used_bytes_) throw std::logic_error("used byte accounting drifted");
}

}  // namespace plora
