// Shared pieces of the tcgen05 prefill kernels (sgmv.cu, sgmv_fused.cu):
// the 128-byte swizzle of a UMMA operand row, paged weight addressing
// through the device page table, and 2-D TMA tensor maps (bf16, SW128).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>
#include <string>

#include "plan.hpp"

namespace plora {
namespace tmap {

__device__ __forceinline__ uint32_t swz(uint32_t row, uint32_t chunk) {
  // 128-byte swizzle inside an 8-row × 128-byte atom
  return (row >> 3) * 1024 + (row & 7) * 128 + ((chunk ^ (row & 7)) << 4);
}

struct PagedSrc {
  const char* arena;
  const uint32_t* table;
  uint32_t table_off;
  uint32_t log2_page;
  __device__ const char* at(uint64_t off) const {
    const uint32_t phys = __ldg(table + table_off + static_cast<uint32_t>(off >> log2_page));
    return arena + (static_cast<uint64_t>(phys) << log2_page) + (off & ((1ull << log2_page) - 1));
  }
};

inline PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  if (!fn) throw CudaError("cuTensorMapEncodeTiled unavailable");
  return fn;
}

inline void make_tmap_2d(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows,
                         uint64_t row_stride_b, uint32_t box_cols, uint32_t box_rows) {
  const cuuint64_t dims[2] = {cols, std::max<uint64_t>(rows, 1)};
  const cuuint64_t strides[1] = {row_stride_b};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult cr = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                            strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string(cr));
}

}  // namespace tmap
}  // namespace plora
