// The reference engine's page-pool call sites (src/engine.cpp:77-78, 293,
// 299, 489, 587), written against lorasim's own types with libplora's pool
// in place of lorasim::PagePool (include/plora_lorasim.hpp), next to the
// reference's BlockArena — and a churn run that drives this pool and the
// reference lorasim::PagePool (oracle/_ref/libref.so) with the same
// operations, comparing tables, reports, errors and dump() after every step.
#include <lorasim/memory.hpp>

#include <cstdio>
#include <optional>
#include <random>
#include <vector>

#include "plora_lorasim.hpp"

using namespace lorasim;

// The engine's members and expressions (a restatement of the call sites,
// not the reference's code).
struct EngineExcerpt {
  std::optional<PloraPagePool> pool_;
  std::optional<BlockArena> arena_;
  std::vector<std::uint64_t> bytes_;
  std::vector<std::uint32_t> units_;

  void make_allocator(bool paged, std::uint64_t page_bytes, std::uint32_t pages, std::uint64_t arena) {
    if (paged) {
      pool_.emplace(page_bytes, pages);                                  // :77
      for (std::size_t a = 0; a < bytes_.size(); ++a) units_[a] = pool_->pages_needed(bytes_[a]);  // :78
    } else {
      arena_.emplace(arena);
    }
  }
  AllocStatus alloc_adapter(std::uint32_t a) {                          // :293
    return pool_ ? pool_->alloc(a, bytes_[a]) : arena_->alloc(a, bytes_[a]);
  }
  void evict(std::uint32_t a) {                                         // :299
    if (pool_) pool_->free(a);
    else arena_->free(a);
  }
  std::size_t compact() { return pool_ ? pool_->compact() : 0; }       // :489
  FragmentationReport report() const {                                  // :587
    FragmentationReport rep = pool_ ? pool_->report() : arena_->report();
    return rep;
  }
};

static int fails = 0;
#define EXPECT(c)                                              \
  do {                                                         \
    if (!(c)) {                                                \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);  \
      ++fails;                                                 \
    }                                                          \
  } while (0)

int main() {
  const std::uint64_t P = 4096;
  const std::uint32_t N = 3000, A = 40;
  EngineExcerpt eng;
  eng.bytes_.resize(A);
  eng.units_.resize(A);
  std::mt19937_64 rng(20240611);
  for (auto& b : eng.bytes_) b = 1 + rng() % (200 * P);
  eng.make_allocator(true, P, N, 0);
  PagePool ref(P, N);  // the reference's own pool
  for (std::uint32_t a = 0; a < A; ++a) EXPECT(eng.units_[a] == ref.pages_needed(eng.bytes_[a]));
  std::vector<bool> live(A, false);
  for (int op = 0; op < 4000; ++op) {
    const std::uint32_t a = static_cast<std::uint32_t>(rng() % A);
    if (op % 250 == 0) EXPECT(eng.compact() == ref.compact());
    if (live[a]) {
      eng.evict(a);
      ref.free(a);
      live[a] = false;
    } else {
      const AllocStatus s = eng.alloc_adapter(a);
      EXPECT(s == ref.alloc(a, eng.bytes_[a]));
      live[a] = s == AllocStatus::ok;
    }
    for (std::uint32_t k = 0; k < A; ++k)
      if (live[k]) EXPECT(eng.pool_->table(k).entries == ref.table(k).entries);
    const FragmentationReport r1 = eng.report(), r2 = ref.report();
    EXPECT(r1.internal_frag == r2.internal_frag && r1.utilization == r2.utilization &&
           r1.external_frag == r2.external_frag);
  }
  EXPECT(eng.pool_->dump() == ref.dump());
  // errors keep lorasim's types
  std::uint32_t dead = 0;
  while (live[dead]) ++dead;
  try {
    eng.pool_->translate(dead, 0);
    EXPECT(false);
  } catch (const ValidationError&) {
  }
  try {
    eng.evict(dead);
    EXPECT(false);
  } catch (const std::logic_error&) {
  }
  // the block-arena branch of the same expressions
  EngineExcerpt blk;
  blk.bytes_ = eng.bytes_;
  blk.units_.resize(A);
  blk.make_allocator(false, 0, 0, 64ull * P * 100);
  EXPECT(blk.alloc_adapter(0) == AllocStatus::ok);
  blk.evict(0);
  (void)blk.report();
  if (fails) return 1;
  std::printf("engine excerpt ok\n");
  return 0;
}
