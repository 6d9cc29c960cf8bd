// Shared device utilities: TMA tensor-map encoding (through the runtime's
// driver entry point, no -lcuda) and the parameter-stream fill kernel for
// request inputs and test tensors.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <mutex>
#include <utility>

#include "common.cuh"
#include "mlp.cuh"
#include "sm100.cuh"

namespace gfx {

namespace {

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        GFX_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || p == nullptr)
            throw CudaError("cuTensorMapEncodeTiled entry point unavailable");
        fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

}  // namespace

int current_device() {
    int dev = 0;
    GFX_CUDA(cudaGetDevice(&dev));
    return dev;
}

int device_sm_count(int dev) {
    static std::mutex mu;
    static std::map<int, int> sms;
    std::lock_guard<std::mutex> lk(mu);
    auto it = sms.find(dev);
    if (it != sms.end()) return it->second;
    int n = 0;
    GFX_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    sms[dev] = n;
    return n;
}

void ensure_max_dynamic_smem(const void* func, int bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, int> done;  // (device, kernel) -> bytes set
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(mu);
    auto it = done.find({dev, func});
    if (it != done.end() && it->second >= bytes) return;
    GFX_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    done[{dev, func}] = bytes;
}

bool encode_tensor_map_2d(CUtensorMap* map, CUtensorMapDataType dtype, uint32_t elem_bytes, const void* base,
                          uint64_t inner, uint64_t outer, uint64_t row_stride_bytes, uint32_t box_inner,
                          uint32_t box_outer, CUtensorMapSwizzle swizzle) {
    (void)elem_bytes;
    const cuuint64_t dims[2] = {inner, outer};
    const cuuint64_t strides[1] = {row_stride_bytes};
    const cuuint32_t box[2] = {box_inner, box_outer};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(map, dtype, 2, const_cast<void*>(base), dims, strides, box, estr,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// Request inputs / test tensors straight from the parameter stream; one
// launch fills `count` consecutive tensors with seeds seed0, seed0+1, ...
__global__ void fill_params_kernel(float* dst, uint64_t n, uint64_t count, uint64_t seed0, uint32_t tensor,
                                   float scaled) {
    const uint64_t total = n * count;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t t = i / n;
        dst[i] = param_at(param_stream(seed0 + t, tensor), i - t * n, scaled);
    }
}

void launch_fill_params(float* dst, uint64_t n, uint64_t seed, uint32_t tensor, float scale, cudaStream_t s,
                        uint64_t count) {
    const uint64_t total = n * count;
    unsigned blocks = static_cast<unsigned>((total + 255) / 256);
    if (blocks > 148 * 32) blocks = 148 * 32;
    if (blocks == 0) blocks = 1;
    fill_params_kernel<<<blocks, 256, 0, s>>>(dst, n, count, seed, tensor, param_scale(scale));
    GFX_CUDA(cudaGetLastError());
}

}  // namespace gfx
