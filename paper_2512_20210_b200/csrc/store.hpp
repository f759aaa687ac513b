// Device adapter store: one HBM arena behind the host PagePool, a device
// page table and an adapter directory.  See include/plora.h.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "common.hpp"
#include "pagepool.hpp"

struct plora_pool {
  plora::PagePool pool;
  mutable std::string dump_cache;
};

namespace plora {

#define PLORA_CUDA(expr)                                                              \
  do {                                                                                \
    cudaError_t _e = (expr);                                                          \
    if (_e != cudaSuccess)                                                            \
      throw ::plora::CudaError(std::string(#expr) + ": " + cudaGetErrorString(_e));   \
  } while (0)

// Opt a kernel into `bytes` of dynamic shared memory, once per (device,
// kernel): the attribute belongs to the device's context, and several host
// threads (the engine's pump, callers) may launch.
void set_smem_once(const void* kernel, int bytes);

// Directory entry for one adapter key, read by every kernel.  16 bytes.
struct DevAdapter {
  uint32_t rank;
  uint32_t n_pages;
  uint32_t table_off;  // first entry of this adapter in the device page table
  uint32_t resident;   // 1 once published (promotion, src/engine.cpp:406-414)
};

// Model-derived addressing (plora_model + in-adapter layout).
struct ModelGeom {
  plora_model m{};
  uint32_t esize = 2;
  uint64_t per_layer_unit = 0;  // Σ_p (d_in[p] + d_out[p]); block elems = rank · this
  uint64_t prefix[PLORA_MAX_PROJ + 1] = {};

  void init(const plora_model& model);
  // element offset of block (layer, proj) inside a rank-r adapter = rank · blk_mult
  uint64_t blk_mult(uint32_t layer, uint32_t proj) const {
    return static_cast<uint64_t>(layer) * per_layer_unit + prefix[proj];
  }
  // Every (layer, proj) A and Bᵀ block of projection `proj` starts on a
  // 128-byte boundary of the adapter for every rank (the tensor-core paths
  // address pages as 128-byte rows).
  bool blocks_aligned_128(uint32_t proj) const {
    return per_layer_unit % 64 == 0 && prefix[proj] % 64 == 0 && m.d_in[proj] % 64 == 0;
  }
  uint64_t adapter_bytes(uint32_t rank) const {
    return static_cast<uint64_t>(rank) * per_layer_unit * m.n_layers * esize;
  }
};

struct AdapterSlot {
  uint32_t rank = 0;       // 0 = unregistered
  uint32_t table_off = 0;
  uint32_t table_cap = 0;  // entries reserved in the device page table
  bool published = false;
};

struct DeviceCtx {  // RAII device guard
  int prev = -1;
  explicit DeviceCtx(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceCtx() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace plora

struct plora_store {
  plora_pool* pool = nullptr;
  int device = 0;
  int num_sms = 148;
  plora::ModelGeom geom;
  uint32_t max_adapters = 0;
  uint32_t log2_page = 0;

  char* arena = nullptr;  // total_pages · page_bytes
  plora::DevAdapter* d_dir = nullptr;
  uint32_t* d_table = nullptr;
  uint64_t table_capacity = 0;  // entries
  uint64_t table_used = 0;

  std::vector<plora::AdapterSlot> slots;
  std::vector<plora::DevAdapter> h_dir;
  uint32_t* d_scratch = nullptr;  // relocation list staging
  char* d_zeros = nullptr;        // 4 KiB of zeros (rank-padding rows of MMA tiles)
  uint64_t scratch_cap = 0;

  void ensure_table_capacity(uint64_t need, cudaStream_t stream);
  void upload_table(uint32_t adapter, cudaStream_t stream);
  void upload_dir(uint32_t adapter, cudaStream_t stream);
};

namespace plora {
// Device alias of a pinned host image for the SM copy path (validates
// alignment and pinning).
const char* mapped_source(const void* host_src, uint64_t bytes);
// Copy logical pages [first, first + n) of the adapter image `src` (`bytes`
// long) into their physical pages.  PLORA_COPY_CE: one cudaMemcpyAsync per
// physically contiguous run.  PLORA_COPY_SM: one scatter-kernel launch
// reading src_dev, page entries from the device table (upload_table first).
void scatter_pages(plora_store& s, uint32_t adapter, const char* src, const char* src_dev,
                   uint32_t first, uint32_t n, uint64_t bytes, int mode, cudaStream_t stream);
}  // namespace plora
