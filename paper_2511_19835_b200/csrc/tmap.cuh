// Host-side TMA tensor-map encoding (cuTensorMapEncodeTiled through the
// runtime's driver entry point: no -lcuda symbol at load time).
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "rsa_internal.cuh"

namespace rsa {

inline PFN_cuTensorMapEncodeTiled_v12000 tmap_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
  }();
  return fn;
}

// The rows of Q/K/V/O as a 4-D bf16 tensor (d, T, heads per batch entry,
// batch) with the geometry's element strides -- any [B, H, T, d] or
// [B, T, H, d] view whose rows are contiguous and 16-byte aligned.  Box
// (box0, box1, 1, 1); swizzle as given (none for row-major staging).
inline bool make_rows_tmap(CUtensorMap* tm, const void* ptr, const Geometry& g, int box0, int box1,
                           CUtensorMapSwizzle swz) {
  auto fn = tmap_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {(cuuint64_t)g.d, (cuuint64_t)g.T, (cuuint64_t)g.hb, (cuuint64_t)(g.H / g.hb)};
  cuuint64_t strides[3] = {(cuuint64_t)g.s_tok * 2, (cuuint64_t)g.s_head * 2, (cuuint64_t)g.s_batch * 2};
  cuuint32_t box[4] = {(cuuint32_t)box0, (cuuint32_t)box1, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return fn(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace rsa
