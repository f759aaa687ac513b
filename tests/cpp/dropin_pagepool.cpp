// C++ drop-in check: the reference's test_memory.cpp scenarios written
// against plora::PagePool (include/plora.hpp) instead of lorasim::PagePool.
#include <cstdio>
#include <stdexcept>

#include "plora.hpp"

#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      std::fprintf(stderr, "CHECK failed line %d: %s\n", __LINE__, #c); \
      return 1;                                                    \
    }                                                              \
  } while (0)

int main() {
  constexpr std::uint64_t MiB = 1ull << 20, kPage = 2 * MiB;
  {  // test_memory.cpp:17-24
    plora::PagePool pool(kPage, 16);
    CHECK(pool.pages_needed(13 * MiB) == 7);
    CHECK(pool.alloc(1, 13 * MiB) == plora::AllocStatus::ok);
    CHECK(pool.table(1).entries.size() == 7);
    CHECK(pool.free_pages() == 9);
    pool.check_invariants();
  }
  {  // :41-48 double free is std::logic_error
    plora::PagePool pool(kPage, 16);
    CHECK(pool.alloc(3, 5 * MiB) == plora::AllocStatus::ok);
    pool.free(3);
    bool threw = false;
    try {
      pool.free(3);
    } catch (const std::logic_error&) {
      threw = true;
    }
    CHECK(threw);
  }
  {  // :50-55 translate out of range is ValidationError
    plora::PagePool pool(kPage, 8);
    CHECK(pool.alloc(0, 3 * kPage) == plora::AllocStatus::ok);
    for (std::uint32_t i = 0; i < 3; ++i) CHECK(pool.translate(0, i) == i);
    bool threw = false;
    try {
      pool.translate(0, 3);
    } catch (const plora::ValidationError&) {
      threw = true;
    }
    CHECK(threw);
  }
  {  // hole reuse then compaction
    plora::PagePool pool(2048, 16);
    pool.alloc(0, 3 * 2048);
    pool.alloc(1, 2 * 2048);
    pool.alloc(2, 4 * 2048);
    pool.free(1);
    pool.alloc(3, 5 * 2048 + 1);
    const std::vector<std::uint32_t> a3{3, 4, 9, 10, 11, 12};
    CHECK(pool.table(3).entries == a3);
    pool.free(0);
    CHECK(pool.compact() == 3);
    const std::vector<std::uint32_t> a3c{3, 4, 9, 0, 1, 2};
    CHECK(pool.table(3).entries == a3c);
    CHECK(pool.last_relocations().size() == 3);
  }
  std::printf("dropin ok\n");
  return 0;
}
