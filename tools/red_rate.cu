// L2 reduction throughput on B200: 148 CTAs x 128 threads, each CTA adds a
// 128 x 32 partial (4096 values) into a shared [N][32] buffer, S CTAs per tile
// (as at a K1 layer boundary). Variants: u64 red (coalesced 256 B per warp
// instruction), f32 v4 red, f32 scalar red, plain u64 store, f32 v4 store.
// usage: red_rate  -> one line per variant: µs per boundary (CUDA events, mean of 50)
#include <cstdio>
#include <cuda_runtime.h>

template <int kMode>
__global__ void __launch_bounds__(128) red_kernel(unsigned long long* out64, float* out32, int splits, int reps) {
  for (int rep = 0; rep < reps; ++rep) {
    const int tile = blockIdx.x / splits;
    const int lane = threadIdx.x & 31, q = threadIdx.x >> 5;
    const float v = 1.0f + threadIdx.x;
    if (kMode == 0) {  // u64 red: instruction i -> feature row q*32+i, lane = batch row
        for (int i = 0; i < 32; ++i) {
            unsigned long long* p = out64 + (static_cast<size_t>(tile) * 128 + q * 32 + i) * 32 + lane;
            asm volatile("red.global.add.u64 [%0], %1;" ::"l"(p), "l"(static_cast<unsigned long long>(v) << 9));
        }
    } else if (kMode == 1) {  // f32 v4 red: thread = feature row, 8 x 16 B
        float* p = out32 + (static_cast<size_t>(tile) * 128 + threadIdx.x) * 32;
        for (int b = 0; b < 32; b += 4)
            asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p + b), "f"(v), "f"(v), "f"(v), "f"(v));
    } else if (kMode == 2) {  // f32 scalar red, coalesced 128 B per instruction
        for (int i = 0; i < 32; ++i) {
            float* p = out32 + (static_cast<size_t>(tile) * 128 + q * 32 + i) * 32 + lane;
            asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v));
        }
    } else if (kMode == 3) {  // plain u64 stores to a per-CTA slot (no reduction), same bytes as mode 0
        for (int i = 0; i < 32; ++i) {
            unsigned long long* p = out64 + (static_cast<size_t>(blockIdx.x) * 128 + q * 32 + i) * 32 + lane;
            *reinterpret_cast<volatile unsigned long long*>(p) = static_cast<unsigned long long>(v);
        }
    } else if (kMode == 4) {  // f32 v4 red, coalesced: instruction i covers 512 contiguous bytes
        for (int i = 0; i < 8; ++i) {
            float* p = out32 + (static_cast<size_t>(tile) * 128 + q * 32 + i * 4 + (lane >> 3)) * 32 + (lane & 7) * 4;
            asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v), "f"(v), "f"(v), "f"(v));
        }
    } else if (kMode == 5) {  // u64 red v2? (not in PTX) -> u32 pairs: 2 x red.u32 per word
        for (int i = 0; i < 32; ++i) {
            unsigned* p = reinterpret_cast<unsigned*>(out64 + (static_cast<size_t>(tile) * 128 + q * 32 + i) * 32) + lane;
            asm volatile("red.global.add.u32 [%0], %1;" ::"l"(p), "r"(static_cast<unsigned>(v)));
            asm volatile("red.global.add.u32 [%0], %1;" ::"l"(p + 32), "r"(static_cast<unsigned>(v)));
        }
    }
  }
}

template <int kMode>
float run1(unsigned long long* o64, float* o32, int splits, int grid, int reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 5; ++i) red_kernel<kMode><<<grid, 128>>>(o64, o32, splits, reps);
    cudaEventRecord(a);
    for (int i = 0; i < 50; ++i) red_kernel<kMode><<<grid, 128>>>(o64, o32, splits, reps);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms * 1e3f / 50;
}
template <int kMode>
float run(unsigned long long* o64, float* o32, int splits, int grid) {  // per boundary: (21 reps - 1 rep) / 20
    return (run1<kMode>(o64, o32, splits, grid, 21) - run1<kMode>(o64, o32, splits, grid, 1)) / 20;
}

int main() {
    unsigned long long* o64;
    float* o32;
    cudaMalloc(&o64, 64ull << 20);
    cudaMalloc(&o32, 64ull << 20);
    cudaMemset(o64, 0, 64ull << 20);
    cudaMemset(o32, 0, 64ull << 20);
    const char* names[6] = {"u64 red (256 B/instr)", "f32 v4 red (strided)", "f32 red (128 B/instr)",
                            "u64 plain store", "f32 v4 red (512 B/instr)", "2 x u32 red"};
    for (int splits : {1, 6, 12}) {
        const int grid = 148;
        float t[6] = {run<0>(o64, o32, splits, grid), run<1>(o64, o32, splits, grid), run<2>(o64, o32, splits, grid),
                      run<3>(o64, o32, splits, grid), run<4>(o64, o32, splits, grid), run<5>(o64, o32, splits, grid)};
        for (int m = 0; m < 6; ++m)
            printf("splits %2d  %-26s %7.2f us per boundary\n", splits, names[m], t[m]);
    }
    // empty-kernel launch cost for reference
    return 0;
}
