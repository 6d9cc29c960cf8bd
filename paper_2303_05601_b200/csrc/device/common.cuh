#pragma once
// Shared device-side helpers: error mapping to the C-ABI status classes,
// the paged-arena address translation and the parameter stream.
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "gpufaas_b200.h"

namespace gfx {

// CUDA failures surface as GFX_ERR_CUDA through the C-ABI.
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess)
        throw CudaError(std::string(what) + " failed: " + cudaGetErrorString(e) + " (" + file + ":" +
                        std::to_string(line) + ")");
}
#define GFX_CUDA(x) ::gfx::cuda_check((x), #x, __FILE__, __LINE__)

// Per-device launch setup (util.cu). cudaFuncSetAttribute applies to the
// current device's context only, so one process driving several devices sets
// it once per (device, kernel); the SM count is cached per device.
int current_device();
int device_sm_count(int dev);
void ensure_max_dynamic_smem(const void* func, int bytes);

constexpr uint32_t kPageShift = 21;  // 2 MiB arena pages
constexpr uint64_t kPageBytes = uint64_t{1} << kPageShift;
constexpr uint64_t kPageMask = kPageBytes - 1;
static_assert(kPageBytes == GFX_PAGE_BYTES, "page size mismatch with the C-ABI");

// A model's pages in arena order: virtual byte v of the model blob lives at
// arena + (page[v >> 21] << 21) + (v & (2 MiB - 1)). Passed by value as a
// kernel parameter, so a reload (new pages) never races an in-flight launch.
struct PageTable {
    uint32_t n;
    uint32_t page[GFX_MAX_PAGES];
};

__host__ __device__ inline uint64_t mix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}

// Parameter stream of DESIGN.md §4 (bit-identical to oracle/infer_oracle.c):
// value = int24 uniform * (scale * 2^-23), one rounding.
__host__ __device__ inline uint64_t param_stream(uint64_t seed, uint32_t tensor) {
    return mix64(seed ^ (static_cast<uint64_t>(tensor) * 0xD1B54A32D192ED03ULL));
}
__host__ __device__ inline float param_at(uint64_t stream, uint64_t index, float scaled) {
    const uint64_t h = mix64(stream + index);
    const int32_t u = static_cast<int32_t>(h >> 40) - (1 << 23);
    return static_cast<float>(u) * scaled;
}
// scale * 2^-23 (exact: power-of-two scaling of a normal float).
__host__ __device__ inline float param_scale(float scale) { return scale * 0x1.0p-23f; }

}  // namespace gfx
