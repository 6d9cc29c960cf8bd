// Host helper for the tools: cuTensorMapEncodeTiled through the runtime's
// driver entry point (same as paper_2303_05601_b200/csrc/device/util.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

namespace gfx {
inline bool encode_tensor_map_2d(CUtensorMap* map, CUtensorMapDataType dtype, uint32_t, const void* base,
                                 uint64_t inner, uint64_t outer, uint64_t row_stride_bytes, uint32_t box_inner,
                                 uint32_t box_outer, CUtensorMapSwizzle swizzle) {
    using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                            const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                            CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p) return false;
    const cuuint64_t dims[2] = {inner, outer};
    const cuuint64_t strides[1] = {row_stride_bytes};
    const cuuint32_t box[2] = {box_inner, box_outer};
    const cuuint32_t estr[2] = {1, 1};
    return reinterpret_cast<Fn>(p)(map, dtype, 2, const_cast<void*>(base), dims, strides, box, estr,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace gfx
