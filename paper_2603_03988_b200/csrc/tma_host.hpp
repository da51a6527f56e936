// SPDX-License-Identifier: Apache-2.0
// Host-side TMA tensor-map construction. The driver entry point is resolved
// through the runtime (cudaGetDriverEntryPoint) so the library does not link
// libcuda directly.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace sortk {

inline PFN_cuTensorMapEncodeTiled_v12000 tma_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !p) {
      throw std::runtime_error("cuTensorMapEncodeTiled entry point unavailable");
    }
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

inline CUtensorMapSwizzle tma_swizzle(int bytes) {
  switch (bytes) {
    case 0: return CU_TENSOR_MAP_SWIZZLE_NONE;
    case 32: return CU_TENSOR_MAP_SWIZZLE_32B;
    case 64: return CU_TENSOR_MAP_SWIZZLE_64B;
    case 128: return CU_TENSOR_MAP_SWIZZLE_128B;
    case 129: return CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;  // (code 129) the MN-major TF32 UMMA layout
    default: throw std::runtime_error("bad swizzle");
  }
}

// Tensor of rank 2..3, dims[0] innermost (contiguous). strides_bytes has
// rank-1 entries (stride of dims[1], dims[2]).
inline CUtensorMap make_tmap(CUtensorMapDataType dt, const void* base, int rank, const uint64_t* dims,
                             const uint64_t* strides_bytes, const uint32_t* box, int swizzle_bytes) {
  CUtensorMap m;
  uint32_t elem_strides[5] = {1, 1, 1, 1, 1};
  CUresult r = tma_encode_fn()(&m, dt, rank, const_cast<void*>(base),
                               dims, strides_bytes, box, elem_strides,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, tma_swizzle(swizzle_bytes),
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    std::string what = "cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)) + " (base " +
                       std::to_string(reinterpret_cast<uintptr_t>(base)) + ", dims";
    for (int i = 0; i < rank; ++i) what += " " + std::to_string(dims[i]);
    what += ", strides";
    for (int i = 0; i + 1 < rank; ++i) what += " " + std::to_string(strides_bytes[i]);
    what += ", box";
    for (int i = 0; i < rank; ++i) what += " " + std::to_string(box[i]);
    throw std::runtime_error(what + ")");
  }
  return m;
}

inline CUtensorMap make_tmap_bf16(const void* base, int rank, const uint64_t* dims,
                                  const uint64_t* strides_bytes, const uint32_t* box,
                                  int swizzle_bytes) {
  return make_tmap(CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, base, rank, dims, strides_bytes, box, swizzle_bytes);
}

// Row-major [rows, cols] fp32 matrix, box = [box_rows, box_cols].
inline CUtensorMap make_tmap_2d_f32(const void* base, uint64_t rows, uint64_t cols,
                                    uint32_t box_rows, uint32_t box_cols, int swizzle_bytes) {
  uint64_t dims[2] = {cols, rows};
  uint64_t strides[1] = {cols * 4};
  uint32_t box[2] = {box_cols, box_rows};
  return make_tmap(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, base, 2, dims, strides, box, swizzle_bytes);
}

// Row-major [rows, cols] bf16 matrix with row pitch `ld` elements; box = [box_rows, box_cols].
inline CUtensorMap make_tmap_2d(const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                                uint32_t box_rows, uint32_t box_cols, int swizzle_bytes) {
  uint64_t dims[2] = {cols, rows};
  uint64_t strides[1] = {ld * 2};
  uint32_t box[2] = {box_cols, box_rows};
  return make_tmap_bf16(base, 2, dims, strides, box, swizzle_bytes);
}

}  // namespace sortk
