// Host adapter store: the pinned host copy of every
// adapter the engine may page in — one page-aligned, pinned region with an
// offset index, optionally backed by a file ("PLHS").  The engine's transfer
// sources (plora_engine_set_source) point into it, so every demand load or
// prefetch moves that adapter's own bytes.  Adapter sizes follow the
// reference's LoraDims (src/adapter.cpp:12-26, 52-59); the catalog itself
// comes from plora_generate_catalog / load_catalog_json (src/adapter.cpp:81-108).
//
// File layout (little endian):
//   [0, 64)      header: "PLHS", u32 version = 1, u32 n, u64 align, u64 data_off,
//                u64 data_bytes, reserved
//   [64, ...)    index: n × {u64 offset (from data_off), u64 bytes, u32 rank, u32 pad}
//   [data_off,)  adapter images, each at an `align`-aligned offset
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "common.hpp"

namespace {

struct IndexEntry {
  uint64_t offset, bytes;
  uint32_t rank, pad;
};
static_assert(sizeof(IndexEntry) == 24, "index entry layout");

struct Header {
  char magic[4];
  uint32_t version, n;
  uint32_t pad;
  uint64_t align, data_off, data_bytes;
  uint64_t reserved[3];
};
static_assert(sizeof(Header) == 64, "header layout");

uint64_t round_up(uint64_t v, uint64_t a) { return (v + a - 1) / a * a; }

}  // namespace

struct plora_hoststore {
  std::vector<IndexEntry> index;
  uint64_t align = 0;
  char* base = nullptr;       // data region (pinned)
  uint64_t data_bytes = 0;
  // ownership: cudaHostAlloc'ed, or an mmap'ed file registered with CUDA
  bool mapped = false;
  void* map_addr = nullptr;
  uint64_t map_bytes = 0;
};

extern "C" {

int plora_hoststore_create(const uint64_t* bytes, const uint32_t* ranks, uint32_t n, uint64_t align,
                           plora_hoststore** out) {
  using namespace plora;
  return guard([&] {
    if (!out || (n && !bytes)) throw ValidationError("null argument");
    if (align == 0 || (align & (align - 1))) throw ValidationError("align must be a power of two");
    auto s = std::make_unique<plora_hoststore>();
    s->align = align;
    uint64_t off = 0;
    s->index.resize(n);
    for (uint32_t i = 0; i < n; ++i) {
      if (bytes[i] == 0) throw ValidationError("adapter " + std::to_string(i) + " has 0 bytes");
      s->index[i] = IndexEntry{off, bytes[i], ranks ? ranks[i] : 0u, 0u};
      off = round_up(off + bytes[i], align);
    }
    s->data_bytes = off;
    void* p = nullptr;
    if (off) {
      const cudaError_t e = cudaHostAlloc(&p, off, cudaHostAllocPortable);
      if (e != cudaSuccess)
        throw CudaError("host store: cudaHostAlloc(" + std::to_string(off) + "): " + cudaGetErrorString(e));
    }
    s->base = static_cast<char*>(p);
    *out = s.release();
    return 0;
  });
}

int plora_hoststore_open(const char* path, plora_hoststore** out) {
  using namespace plora;
  return guard([&] {
    if (!path || !out) throw ValidationError("null argument");
    const int fd = ::open(path, O_RDONLY);
    if (fd < 0) throw ConfigError(std::string("host store: cannot open ") + path);
    struct stat sb;
    if (fstat(fd, &sb) != 0 || static_cast<uint64_t>(sb.st_size) < sizeof(Header)) {
      ::close(fd);
      throw ParseError(std::string("host store: truncated file ") + path);
    }
    const uint64_t size = static_cast<uint64_t>(sb.st_size);
    void* m = mmap(nullptr, size, PROT_READ, MAP_SHARED, fd, 0);
    ::close(fd);
    if (m == MAP_FAILED) throw ConfigError(std::string("host store: mmap failed for ") + path);
    auto fail = [&](const std::string& msg) {
      munmap(m, size);
      throw ParseError("host store: " + msg + " in " + path);
    };
    Header h;
    std::memcpy(&h, m, sizeof h);
    if (std::memcmp(h.magic, "PLHS", 4) != 0) fail("bad magic");
    if (h.version != 1) fail("unsupported version");
    if (sizeof(Header) + static_cast<uint64_t>(h.n) * sizeof(IndexEntry) > h.data_off ||
        h.data_off + h.data_bytes > size)
      fail("inconsistent header");
    auto s = std::make_unique<plora_hoststore>();
    s->index.resize(h.n);
    std::memcpy(s->index.data(), static_cast<char*>(m) + sizeof(Header), h.n * sizeof(IndexEntry));
    for (const auto& e : s->index)
      if (e.offset + e.bytes > h.data_bytes) fail("index entry past the data region");
    s->align = h.align;
    s->data_bytes = h.data_bytes;
    // zero-copy: pin the file mapping itself (page-rounded; read-only
    // registration), so the engine's copies DMA straight from the page cache
    const uint64_t pg = static_cast<uint64_t>(sysconf(_SC_PAGESIZE));
    const uint64_t reg = round_up(size, pg);
    if (cudaHostRegister(m, reg, cudaHostRegisterPortable | cudaHostRegisterReadOnly) == cudaSuccess) {
      s->mapped = true;
      s->map_addr = m;
      s->map_bytes = reg;
      s->base = static_cast<char*>(m) + h.data_off;
    } else {
      // the platform cannot pin a file mapping: load the images into a pinned buffer
      cudaGetLastError();
      void* p = nullptr;
      const cudaError_t e = cudaHostAlloc(&p, std::max<uint64_t>(h.data_bytes, 1), cudaHostAllocPortable);
      if (e != cudaSuccess) {
        munmap(m, size);
        throw CudaError(std::string("host store: cudaHostAlloc: ") + cudaGetErrorString(e));
      }
      std::memcpy(p, static_cast<char*>(m) + h.data_off, h.data_bytes);
      munmap(m, size);
      s->base = static_cast<char*>(p);
    }
    *out = s.release();
    return 0;
  });
}

int plora_hoststore_save(const plora_hoststore* s, const char* path) {
  using namespace plora;
  return guard([&] {
    if (!s || !path) throw ValidationError("null argument");
    Header h{};
    std::memcpy(h.magic, "PLHS", 4);
    h.version = 1;
    h.n = static_cast<uint32_t>(s->index.size());
    h.align = s->align;
    h.data_off = round_up(sizeof(Header) + s->index.size() * sizeof(IndexEntry), 4096);
    h.data_bytes = s->data_bytes;
    FILE* f = std::fopen(path, "wb");
    if (!f) throw ConfigError(std::string("host store: cannot write ") + path);
    bool ok = std::fwrite(&h, sizeof h, 1, f) == 1 &&
              (s->index.empty() ||
               std::fwrite(s->index.data(), sizeof(IndexEntry), s->index.size(), f) == s->index.size());
    const uint64_t pad = h.data_off - sizeof h - s->index.size() * sizeof(IndexEntry);
    std::vector<char> zeros(pad, 0);
    ok = ok && (pad == 0 || std::fwrite(zeros.data(), 1, pad, f) == pad);
    ok = ok && (s->data_bytes == 0 || std::fwrite(s->base, 1, s->data_bytes, f) == s->data_bytes);
    ok = (std::fclose(f) == 0) && ok;
    if (!ok) throw ConfigError(std::string("host store: short write to ") + path);
    return 0;
  });
}

void plora_hoststore_destroy(plora_hoststore* s) {
  if (!s) return;
  if (s->mapped) {
    cudaHostUnregister(s->map_addr);
    munmap(s->map_addr, s->map_bytes);
  } else if (s->base) {
    cudaFreeHost(s->base);
  }
  delete s;
}

uint32_t plora_hoststore_count(const plora_hoststore* s) {
  return s ? static_cast<uint32_t>(s->index.size()) : 0u;
}

int plora_hoststore_entry(const plora_hoststore* s, uint32_t key, void** ptr, uint64_t* bytes,
                          uint32_t* rank) {
  using namespace plora;
  return guard([&] {
    if (!s) throw ValidationError("null store");
    if (key >= s->index.size())
      throw ValidationError("host store: key " + std::to_string(key) + " out of range");
    const IndexEntry& e = s->index[key];
    if (ptr) *ptr = s->base + e.offset;
    if (bytes) *bytes = e.bytes;
    if (rank) *rank = e.rank;
    return 0;
  });
}

int plora_hoststore_bytes(const plora_hoststore* s, uint64_t* data_bytes) {
  using namespace plora;
  return guard([&] {
    if (!s || !data_bytes) throw ValidationError("null argument");
    *data_bytes = s->data_bytes;
    return 0;
  });
}

}  // extern "C"
