// Micro-benchmark: per-SM TMA delivery rate. Each CTA (one per SM, `ctas` of
// them) keeps `stages` 1-D bulk copies of `bytes` in flight from an L2-resident
// (or HBM-sized) source into a shared-memory ring and re-issues each as soon as
// it lands, for `iters` copies. Prints GB/s per SM and in total.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//   -I paper_2303_05601_b200/csrc/device -I tools tools/tma_rate.cu -o tools/_bin/tma_rate
#include <cstdio>

#include "sm100.cuh"
#include "util_host.hpp"

using namespace gfx::sm100;

// mode 0: one thread, 1-D bulk copies. mode 1: one thread, 2-D tensor boxes of
// `bytes` (64 bf16 x rows). mode 2: two threads (two warps) each with its own
// ring of 1-D bulk copies. mode 3: one thread alternating bulk and tensor copies.
// mode 4: two lanes of ONE warp, each its own ring. mode 5: one thread, two
// 1-D copies of `bytes` per slot completing on the slot's barrier.
__global__ void __launch_bounds__(64, 1) tma_rate(const char* src, size_t src_bytes, int bytes, int stages, int iters,
                                                  long long* out, const __grid_constant__ CUtensorMap tmap, int mode) {
    extern __shared__ uint8_t raw[];
    uint8_t* sm = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
    __shared__ __align__(8) uint64_t bar[2][16];
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&bar[0][s], 1);
            mbar_init(&bar[1][s], 1);
        }
        mbar_fence_init();
    }
    __syncthreads();
    const int w = mode == 4 ? (threadIdx.x & 31) : threadIdx.x >> 5;
    if (mode == 4) {
        if (threadIdx.x >= 2) return;
    } else if ((threadIdx.x & 31) != 0 || (w == 1 && mode != 2)) {
        return;
    }
    const int per = mode == 5 ? 2 : 1;
    uint8_t* ring = sm + w * stages * bytes * per;
    const int rows = bytes / 128;
    size_t off = (static_cast<size_t>(blockIdx.x * 2 + w) * 7919u * bytes) % src_bytes;
    int row = static_cast<int>((blockIdx.x * 37) % 4096);
    auto issue = [&](int s, int it) {
        mbar_arrive_expect_tx(&bar[w][s], bytes * per);
        if (mode == 5) {
            tma_bulk_g2s(ring + (2 * s + 1) * bytes, src + off, bytes, &bar[w][s]);
            off = (off + static_cast<size_t>(bytes) * 148) % src_bytes;
            tma_bulk_g2s(ring + 2 * s * bytes, src + off, bytes, &bar[w][s]);
            off = (off + static_cast<size_t>(bytes) * 148) % src_bytes;
            return;
        }
        const bool tensor = mode == 1 || (mode == 3 && (it & 1));
        if (tensor) {
            tma_tile2d_g2s(ring + s * bytes, &tmap, 0, row, &bar[w][s]);
            row = (row + rows * 7) % (16384 - rows);
        } else {
            tma_bulk_g2s(ring + s * bytes, src + off, bytes, &bar[w][s]);
            off = (off + static_cast<size_t>(bytes) * 148) % src_bytes;
        }
    };
    const long long t0 = clock64();
    for (int s = 0; s < stages && s < iters; ++s) issue(s, s);
    for (int it = stages; it < iters + stages; ++it) {
        const int s = it % stages;
        mbar_wait(&bar[w][s], ((it / stages) - 1) & 1);
        if (it < iters) issue(s, it);
    }
    const long long t1 = clock64();
    if (w == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
    char* src;
    const size_t big = 4ull << 30;
    cudaMalloc(&src, big);
    cudaMemset(src, 1, big);
    long long *d, h[148];
    cudaMalloc(&d, sizeof h);
    cudaFuncSetAttribute(tma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    // 2-D map over the first 32 MB: [16384 rows x 1024 bf16], boxes of 64 bf16 x (bytes/128) rows, SW128.
    CUtensorMap tm[2];
    for (int i = 0; i < 2; ++i)
        if (!gfx::encode_tensor_map_2d(&tm[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, 1024, 16384, 2048, 64,
                                       i == 0 ? 128 : 256, CU_TENSOR_MAP_SWIZZLE_128B)) {
            printf("tensor map failed\n");
            return 1;
        }
    struct Case {
        size_t src;
        int bytes, stages, ctas, mode;
    } cases[] = {
        {32ull << 20, 16384, 8, 148, 0}, {32ull << 20, 32768, 6, 148, 0}, {32ull << 20, 65536, 3, 148, 0},
        {32ull << 20, 8192, 12, 148, 0}, {32ull << 20, 16384, 8, 148, 1}, {32ull << 20, 32768, 6, 148, 1},
        {32ull << 20, 16384, 6, 148, 2}, {32ull << 20, 16384, 8, 148, 3}, {big, 32768, 6, 148, 0},
        {big, 65536, 3, 148, 0},         {32ull << 20, 16384, 6, 148, 4}, {32ull << 20, 16384, 4, 148, 5},
        {big, 16384, 6, 148, 2},         {big, 16384, 6, 148, 4},
    };
    for (const Case& c : cases) {
        const int iters = 2000;
        tma_rate<<<c.ctas, 64, c.bytes * c.stages * (c.mode == 2 || c.mode == 4 || c.mode == 5 ? 2 : 1) + 1024>>>(
            src, c.src, c.bytes, c.stages, iters, d, tm[c.bytes == 32768 ? 1 : 0], c.mode);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("%s\n", cudaGetErrorString(e));
            return 1;
        }
        cudaMemcpy(h, d, sizeof(long long) * c.ctas, cudaMemcpyDeviceToHost);
        double cyc = 0;
        for (int i = 0; i < c.ctas; ++i) cyc += h[i];
        cyc /= c.ctas;
        const double per_sm = static_cast<double>(c.bytes) * iters / (cyc / 1.9e9) / 1e9;  // GB/s at 1.9 GHz
        const double f = (c.mode == 2 || c.mode == 4 || c.mode == 5) ? 2.0 : 1.0;  // two rings / two copies per slot
        static const char* mn[6] = {"bulk", "tensor", "2 warps", "bulk+tensor", "2 lanes", "2 per slot"};
        printf("%-11s src %5zu MB, %5d B x %2d in flight, %3d SMs: %6.1f B/cycle/SM = %6.1f GB/s/SM, %7.1f GB/s total\n",
               mn[c.mode], c.src >> 20, c.bytes, c.stages, c.ctas, f * c.bytes * iters / cyc, f * per_sm,
               f * per_sm * c.ctas);
    }
    return 0;
}
