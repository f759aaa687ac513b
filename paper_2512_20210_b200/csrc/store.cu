// Device adapter store: HBM arena + device page table + adapter directory,
// page-scatter H2D (copy engines or an SM kernel over mapped pinned memory),
// D2H gather for parity, and on-device compaction moves.
//
// Reference semantics: PagePool owns placement (src/memory.cpp:18-89); the
// engine transfers S bytes on a demand or prefetch load (src/engine.cpp:
// 250-288) and makes them usable at promotion (src/engine.cpp:406-414).
#include <algorithm>
#include <cstring>
#include <mutex>
#include <set>

#include "store.hpp"

using namespace plora;

void plora::ModelGeom::init(const plora_model& model) {
  m = model;
  if (model.n_proj == 0 || model.n_proj > PLORA_MAX_PROJ)
    throw ValidationError("n_proj must be in [1, " + std::to_string(PLORA_MAX_PROJ) + "]");
  if (model.n_layers == 0) throw ValidationError("n_layers must be >= 1");
  if (model.dtype != PLORA_BF16 && model.dtype != PLORA_F32)
    throw ValidationError("dtype must be PLORA_BF16 or PLORA_F32");
  esize = model.dtype == PLORA_BF16 ? 2 : 4;
  const uint32_t vec = 16 / esize;
  per_layer_unit = 0;
  for (uint32_t p = 0; p < model.n_proj; ++p) {
    if (model.d_in[p] == 0 || model.d_out[p] == 0)
      throw ValidationError("d_in/d_out must be positive");
    if (model.d_in[p] % vec || model.d_out[p] % vec)
      throw ValidationError("d_in/d_out must be multiples of " + std::to_string(vec) +
                            " elements (16-byte vectors)");
    prefix[p] = per_layer_unit;
    per_layer_unit += static_cast<uint64_t>(model.d_in[p]) + model.d_out[p];
  }
  prefix[model.n_proj] = per_layer_unit;
}

namespace {

// One page per warp-iteration: 16-byte vectors, src in mapped pinned host
// memory (PCIe reads), dst in the arena at the physical page.
// Logical pages [first, first + n_pages); `bytes` is the whole image size.
__global__ void page_scatter_h2d_kernel(const uint4* __restrict__ src, char* __restrict__ arena,
                                        const uint32_t* __restrict__ entries, uint32_t first,
                                        uint32_t n_pages, uint32_t log2_page, uint64_t bytes) {
  const uint32_t vec_per_page = (1u << log2_page) / 16;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t n_warps = (gridDim.x * blockDim.x) >> 5;
  const uint64_t n_vec_total = bytes / 16;
  for (uint32_t pg = first + warp; pg < first + n_pages; pg += n_warps) {
    const uint64_t base_vec = static_cast<uint64_t>(pg) * vec_per_page;
    uint4* dst = reinterpret_cast<uint4*>(arena + (static_cast<uint64_t>(entries[pg]) << log2_page));
    for (uint32_t i = lane; i < vec_per_page; i += 32 * 4) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        uint32_t k = i + u * 32;
        if (k < vec_per_page && base_vec + k < n_vec_total) v[u] = src[base_vec + k];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        uint32_t k = i + u * 32;
        if (k < vec_per_page && base_vec + k < n_vec_total) dst[k] = v[u];
      }
    }
  }
}

// Compaction moves: relocation i copies page src -> dst.  Sources (>= live)
// and destinations (< live) are disjoint (src/memory.cpp:71-89), so every
// move is independent.
__global__ void page_move_kernel(char* __restrict__ arena, const uint32_t* __restrict__ pairs,
                                 uint32_t n, uint32_t log2_page) {
  const uint32_t vec_per_page = (1u << log2_page) / 16;
  for (uint32_t r = blockIdx.x; r < n; r += gridDim.x) {
    const uint4* s = reinterpret_cast<const uint4*>(arena + (static_cast<uint64_t>(pairs[2 * r]) << log2_page));
    uint4* d = reinterpret_cast<uint4*>(arena + (static_cast<uint64_t>(pairs[2 * r + 1]) << log2_page));
    for (uint32_t i = threadIdx.x; i < vec_per_page; i += blockDim.x) d[i] = s[i];
  }
}

plora_store* checked(plora_store* s) {
  if (!s) throw ValidationError("null store");
  return s;
}

}  // namespace

void plora_store::ensure_table_capacity(uint64_t need, cudaStream_t stream) {
  if (need <= table_capacity) return;
  uint64_t cap = std::max<uint64_t>(need, table_capacity * 2 + 1024);
  uint32_t* fresh = nullptr;
  PLORA_CUDA(cudaMalloc(&fresh, cap * sizeof(uint32_t)));
  if (d_table) {
    PLORA_CUDA(cudaMemcpyAsync(fresh, d_table, table_used * sizeof(uint32_t),
                               cudaMemcpyDeviceToDevice, stream));
    PLORA_CUDA(cudaStreamSynchronize(stream));
    PLORA_CUDA(cudaFree(d_table));
  }
  d_table = fresh;
  table_capacity = cap;
}

void plora_store::upload_table(uint32_t adapter, cudaStream_t stream) {
  const PageTable& t = pool->pool.table(adapter);
  const AdapterSlot& sl = slots[adapter];
  if (t.entries.size() > sl.table_cap)
    throw ValidationError("adapter " + std::to_string(adapter) + " holds " +
                          std::to_string(t.entries.size()) + " pages but its registered rank " +
                          "reserves " + std::to_string(sl.table_cap));
  // pageable source: the copy is staged before cudaMemcpyAsync returns
  PLORA_CUDA(cudaMemcpyAsync(d_table + sl.table_off, t.entries.data(),
                             t.entries.size() * sizeof(uint32_t), cudaMemcpyHostToDevice,
                             stream));
}

void plora_store::upload_dir(uint32_t adapter, cudaStream_t stream) {
  PLORA_CUDA(cudaMemcpyAsync(d_dir + adapter, &h_dir[adapter], sizeof(DevAdapter),
                             cudaMemcpyHostToDevice, stream));
  // h_dir is pageable: cudaMemcpyAsync stages it before returning, so later
  // host-side edits of the entry cannot race the upload.
}

const char* plora::mapped_source(const void* host_src, uint64_t bytes) {
  if (bytes % 16 || reinterpret_cast<uintptr_t>(host_src) % 16)
    throw ValidationError("SM page scatter needs 16-byte aligned size and source");
  cudaPointerAttributes attr{};
  PLORA_CUDA(cudaPointerGetAttributes(&attr, host_src));
  if (attr.type != cudaMemoryTypeHost)
    throw ValidationError("SM page scatter needs pinned (cudaHostAlloc/Register) host memory");
  return static_cast<const char*>(attr.devicePointer ? attr.devicePointer : host_src);
}

void plora::scatter_pages(plora_store& s, uint32_t adapter, const char* src, const char* src_dev,
                          uint32_t first, uint32_t n, uint64_t bytes, int mode,
                          cudaStream_t stream) {
  if (n == 0) return;
  const PageTable& t = s.pool->pool.table(adapter);
  const uint64_t P = s.pool->pool.page_bytes();
  if (mode == PLORA_COPY_CE) {
    // coalesce runs of consecutive physical pages into one copy each
    uint32_t i = first;
    while (i < first + n) {
      uint32_t j = i + 1;
      while (j < first + n && t.entries[j] == t.entries[j - 1] + 1) ++j;
      const uint64_t off = static_cast<uint64_t>(i) * P;
      const uint64_t len = std::min<uint64_t>(static_cast<uint64_t>(j - i) * P, bytes - off);
      PLORA_CUDA(cudaMemcpyAsync(s.arena + static_cast<uint64_t>(t.entries[i]) * P, src + off,
                                 len, cudaMemcpyDefault, stream));
      i = j;
    }
    return;
  }
  const int blocks = std::min<int>(2 * s.num_sms, static_cast<int>((n + 7) / 8));
  page_scatter_h2d_kernel<<<std::max(blocks, 1), 256, 0, stream>>>(
      reinterpret_cast<const uint4*>(src_dev), s.arena, s.d_table + s.slots[adapter].table_off,
      first, n, s.log2_page, bytes);
  PLORA_CUDA(cudaGetLastError());
  count_launch();
}

extern "C" {

uint64_t plora_model_adapter_bytes(const plora_model* m, uint32_t rank) {
  ModelGeom g;
  try {
    g.init(*m);
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return 0;
  }
  return g.adapter_bytes(rank);
}

uint64_t plora_model_block_offset(const plora_model* m, uint32_t rank, uint32_t layer,
                                  uint32_t proj) {
  ModelGeom g;
  try {
    g.init(*m);
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return 0;
  }
  return static_cast<uint64_t>(rank) * g.blk_mult(layer, proj) * g.esize;
}

int plora_store_create(plora_pool* pool, int device, const plora_model* model,
                       uint32_t max_adapters, plora_store** out) {
  return guard([&] {
    if (!pool) throw ValidationError("null pool");
    const uint64_t P = pool->pool.page_bytes();
    if (P < 16 || (P & (P - 1)))
      throw ValidationError("device store needs a power-of-two page size >= 16 bytes, got " +
                            std::to_string(P));
    if (max_adapters == 0) throw ValidationError("max_adapters must be >= 1");
    auto s = std::make_unique<plora_store>();
    s->pool = pool;
    s->device = device;
    s->geom.init(*model);
    s->max_adapters = max_adapters;
    s->log2_page = static_cast<uint32_t>(__builtin_ctzll(P));
    s->slots.resize(max_adapters);
    s->h_dir.assign(max_adapters, DevAdapter{0, 0, 0, 0});
    DeviceCtx ctx(device);
    PLORA_CUDA(cudaDeviceGetAttribute(&s->num_sms, cudaDevAttrMultiProcessorCount, device));
    const uint64_t arena_bytes = pool->pool.total_bytes();
    if (arena_bytes) PLORA_CUDA(cudaMalloc(&s->arena, arena_bytes));
    PLORA_CUDA(cudaMalloc(&s->d_dir, sizeof(DevAdapter) * max_adapters));
    PLORA_CUDA(cudaMemset(s->d_dir, 0, sizeof(DevAdapter) * max_adapters));
    PLORA_CUDA(cudaMalloc(&s->d_zeros, 4096));
    PLORA_CUDA(cudaMemset(s->d_zeros, 0, 4096));
    PLORA_CUDA(cudaDeviceSynchronize());
    *out = s.release();
    return 0;
  });
}

void plora_store_destroy(plora_store* s) {
  if (!s) return;
  DeviceCtx ctx(s->device);
  cudaDeviceSynchronize();
  cudaFree(s->arena);
  cudaFree(s->d_dir);
  cudaFree(s->d_table);
  cudaFree(s->d_scratch);
  cudaFree(s->d_zeros);
  delete s;
}

void* plora_store_arena(const plora_store* s) { return s ? s->arena : nullptr; }

int plora_store_register(plora_store* s, uint32_t adapter, uint32_t rank) {
  return guard([&] {
    checked(s);
    if (adapter >= s->max_adapters)
      throw ValidationError("adapter key " + std::to_string(adapter) + " >= max_adapters " +
                            std::to_string(s->max_adapters));
    if (rank == 0) throw ValidationError("rank must be >= 1");
    AdapterSlot& sl = s->slots[adapter];
    if (sl.published)
      throw std::logic_error("cannot re-register published adapter " + std::to_string(adapter));
    const uint32_t pages = s->pool->pool.pages_needed(s->geom.adapter_bytes(rank));
    if (sl.rank && pages <= sl.table_cap) {
      sl.rank = rank;
      return 0;
    }
    DeviceCtx ctx(s->device);
    s->ensure_table_capacity(s->table_used + pages, nullptr);
    sl.rank = rank;
    sl.table_off = static_cast<uint32_t>(s->table_used);
    sl.table_cap = pages;
    s->table_used += pages;
    return 0;
  });
}

int plora_store_rank(const plora_store* s, uint32_t adapter, uint32_t* rank) {
  return guard([&] {
    if (!s || adapter >= s->max_adapters || !s->slots[adapter].rank)
      throw ValidationError("adapter " + std::to_string(adapter) + " is not registered");
    *rank = s->slots[adapter].rank;
    return 0;
  });
}

int plora_store_write_pages(plora_store* s, uint32_t adapter, const void* host_src,
                            uint64_t bytes, int mode, plora_stream_t stream_) {
  return guard([&] {
    checked(s);
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    if (adapter >= s->max_adapters || !s->slots[adapter].rank)
      throw ValidationError("adapter " + std::to_string(adapter) + " is not registered");
    if (s->slots[adapter].published)
      throw std::logic_error("write_pages on published adapter " + std::to_string(adapter) +
                             " (retire it first)");
    const PageTable& t = s->pool->pool.table(adapter);
    if (bytes > t.weight_bytes)
      throw ValidationError("write of " + std::to_string(bytes) + " bytes exceeds adapter " +
                            std::to_string(adapter) + "'s " + std::to_string(t.weight_bytes));
    if (bytes == 0) return 0;
    DeviceCtx ctx(s->device);
    const uint64_t P = s->pool->pool.page_bytes();
    const uint32_t n_pages = static_cast<uint32_t>((bytes + P - 1) / P);
    const char* src = static_cast<const char*>(host_src);
    const char* src_dev = nullptr;
    if (mode == PLORA_COPY_SM) {
      src_dev = plora::mapped_source(host_src, bytes);
      s->upload_table(adapter, stream);  // the kernel reads the entries from the device table
    } else if (mode != PLORA_COPY_CE) {
      throw ValidationError("unknown copy mode " + std::to_string(mode));
    }
    plora::scatter_pages(*s, adapter, src, src_dev, 0, n_pages, bytes, mode, stream);
    return 0;
  });
}

int plora_store_read_pages(plora_store* s, uint32_t adapter, void* host_dst, uint64_t bytes,
                           plora_stream_t stream_) {
  return guard([&] {
    checked(s);
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    const PageTable& t = s->pool->pool.table(adapter);
    if (bytes > t.weight_bytes) throw ValidationError("read exceeds the adapter's bytes");
    DeviceCtx ctx(s->device);
    const uint64_t P = s->pool->pool.page_bytes();
    const uint32_t n_pages = static_cast<uint32_t>((bytes + P - 1) / P);
    char* dst = static_cast<char*>(host_dst);
    uint32_t i = 0;
    while (i < n_pages) {
      uint32_t j = i + 1;
      while (j < n_pages && t.entries[j] == t.entries[j - 1] + 1) ++j;
      const uint64_t off = static_cast<uint64_t>(i) * P;
      const uint64_t len = std::min<uint64_t>(static_cast<uint64_t>(j - i) * P, bytes - off);
      PLORA_CUDA(cudaMemcpyAsync(dst + off, s->arena + static_cast<uint64_t>(t.entries[i]) * P,
                                 len, cudaMemcpyDeviceToHost, stream));
      i = j;
    }
    PLORA_CUDA(cudaStreamSynchronize(stream));
    return 0;
  });
}

int plora_store_publish(plora_store* s, uint32_t adapter, plora_stream_t stream_) {
  return guard([&] {
    checked(s);
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    if (adapter >= s->max_adapters || !s->slots[adapter].rank)
      throw ValidationError("adapter " + std::to_string(adapter) + " is not registered");
    const PageTable& t = s->pool->pool.table(adapter);  // ValidationError if unallocated
    AdapterSlot& sl = s->slots[adapter];
    const uint64_t need = s->geom.adapter_bytes(sl.rank);
    if (t.weight_bytes < need)
      throw ValidationError("adapter " + std::to_string(adapter) + " holds " +
                            std::to_string(t.weight_bytes) + " bytes; rank " +
                            std::to_string(sl.rank) + " needs " + std::to_string(need));
    DeviceCtx ctx(s->device);
    s->upload_table(adapter, stream);
    s->h_dir[adapter] = DevAdapter{sl.rank, static_cast<uint32_t>(t.entries.size()), sl.table_off, 1};
    s->upload_dir(adapter, stream);
    sl.published = true;
    return 0;
  });
}

int plora_store_retire(plora_store* s, uint32_t adapter, plora_stream_t stream_) {
  return guard([&] {
    checked(s);
    if (adapter >= s->max_adapters) throw ValidationError("adapter key out of range");
    AdapterSlot& sl = s->slots[adapter];
    if (!sl.published) return 0;
    DeviceCtx ctx(s->device);
    s->h_dir[adapter].resident = 0;
    s->upload_dir(adapter, static_cast<cudaStream_t>(stream_));
    sl.published = false;
    return 0;
  });
}

int plora_store_is_published(const plora_store* s, uint32_t adapter) {
  return s && adapter < s->max_adapters && s->slots[adapter].published ? 1 : 0;
}

int plora_store_apply_relocations(plora_store* s, const plora_reloc* relocs, uint64_t n,
                                  plora_stream_t stream_) {
  return guard([&] {
    checked(s);
    if (n == 0) return 0;
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    DeviceCtx ctx(s->device);
    std::vector<uint32_t> pairs(2 * n);
    std::vector<uint32_t> touched;
    for (uint64_t i = 0; i < n; ++i) {
      pairs[2 * i] = relocs[i].src;
      pairs[2 * i + 1] = relocs[i].dst;
      touched.push_back(relocs[i].adapter);
    }
    if (s->scratch_cap < 2 * n) {
      cudaFree(s->d_scratch);
      s->d_scratch = nullptr;
      PLORA_CUDA(cudaMalloc(&s->d_scratch, 2 * n * sizeof(uint32_t)));
      s->scratch_cap = 2 * n;
    }
    PLORA_CUDA(cudaMemcpyAsync(s->d_scratch, pairs.data(), 2 * n * sizeof(uint32_t),
                               cudaMemcpyHostToDevice, stream));
    const int blocks = static_cast<int>(std::min<uint64_t>(n, 4ull * s->num_sms));
    page_move_kernel<<<blocks, 256, 0, stream>>>(s->arena, s->d_scratch, static_cast<uint32_t>(n),
                                                 s->log2_page);
    PLORA_CUDA(cudaGetLastError());
    count_launch();
    std::sort(touched.begin(), touched.end());
    touched.erase(std::unique(touched.begin(), touched.end()), touched.end());
    for (uint32_t a : touched)
      if (a < s->max_adapters && s->slots[a].published) s->upload_table(a, stream);
    PLORA_CUDA(cudaStreamSynchronize(stream));
    return 0;
  });
}

}  // extern "C"

namespace plora {

void set_smem_once(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  int dev = 0;
  PLORA_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (done.count({dev, kernel})) return;
  PLORA_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done.insert({dev, kernel});
}

}  // namespace plora
