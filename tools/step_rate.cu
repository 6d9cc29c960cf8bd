// Micro-benchmark: cost of one K1 v6 ring step as seen by the MMA-issuing
// thread — 4 x tf32 SS M128 N64 K8 + 4 x tf32 TS M128 N32 K8 tcgen05.mma,
// plus the per-step tcgen05.commit(s) and mbarrier try_waits — with the other
// parts switched on/off by a mask, one CTA per SM (148). Prints cycles per step
// for the issue loop alone and including the final drain.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//   -I paper_2303_05601_b200/csrc/device tools/step_rate.cu -o tools/_bin/step_rate
#include <cstdio>
#include <cstdlib>

#include "sm100.cuh"

using namespace gfx::sm100;

__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{\n.reg .pred p;\nelect.sync _|p, 0xffffffff;\nselp.u32 %0, 1, 0, p;\n}\n" : "=r"(pred));
    return pred != 0;
}

// mask bits: 1 SS MMAs, 2 TS MMAs, 4 two commits per step, 8 three completed-barrier waits per step,
//            16 tcgen05.fence::after_thread_sync per step
__global__ void __launch_bounds__(128, 1) step_rate(int steps, int mask, long long* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* sm = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
    __shared__ __align__(8) uint64_t bar[4];
    __shared__ uint32_t tmem_base;
    for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
    if (threadIdx.x < 32) tmem_alloc<512>(&tmem_base);
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
        mbar_fence_init();
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = tmem_base;
    const bool warp_mode = mask & 32;  // whole warp 0 runs the loop, one elected lane issues
    if (threadIdx.x == 0) mbar_arrive(&bar[3]);  // one completed phase for the try_wait probes
    __syncwarp();
    if (warp_mode ? threadIdx.x < 32 : threadIdx.x == 0) {
        constexpr uint32_t id64 = umma_idesc<128, 64, 2>();
        constexpr uint32_t id32 = umma_idesc<128, 32, 2>();
        const uint8_t* w = sm;            // 16 KB: 128 rows x 128 B
        const uint8_t* x = sm + 16384;    // 8 KB: 64 rows x 128 B
        const long long t0 = clock64();
        for (int st = 0; st < steps; ++st) {
            const uint32_t acc = tm + static_cast<uint32_t>((st >> 2) & 1) * 64u;
            const uint32_t lo = tm + 128u + static_cast<uint32_t>(st & 7) * 32u;
            if (mask & 8) {
                mbar_wait(&bar[3], 0);
                mbar_wait(&bar[3], 0);
                mbar_wait(&bar[3], 0);
            }
            if (mask & 16) tc_fence_after();
            const bool leader = !warp_mode || elect_one();
            if (leader) {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const uint64_t bd = umma_desc_sw128(x, kk * 32);
                    if (mask & 1) umma_tf32(acc, umma_desc_sw128(w, kk * 32), bd, id64, 1u);
                    if (mask & 2) umma_tf32_ts(acc, lo + 8u * kk, bd, id32, 1u);
                }
                if (mask & 4) {
                    umma_commit(&bar[0]);
                    umma_commit(&bar[1]);
                }
            }
            if (warp_mode) __syncwarp();
        }
        const long long t1 = clock64();
        if (threadIdx.x == 0) {
            umma_commit(&bar[2]);
            mbar_wait(&bar[2], 0);
            const long long t2 = clock64();
            out[2 * blockIdx.x] = t1 - t0;
            out[2 * blockIdx.x + 1] = t2 - t0;
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x < 32) tmem_dealloc<512>(tm);
}

int main() {
    const int sms = 148, steps = 4000;
    long long *d, h[2 * 148];
    cudaMalloc(&d, sizeof h);
    cudaFuncSetAttribute(step_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 50 * 1024);
    const int masks[] = {0, 32, 3, 3 | 4, 31, 3 | 32, 7 | 32, 31 | 32, 4 | 32, 1 | 32, 2 | 32};
    for (int mask : masks) {
        step_rate<<<sms, 128, 50 * 1024>>>(steps, mask, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("mask %d: %s\n", mask, cudaGetErrorString(e));
            return 1;
        }
        cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
        double issue = 0, total = 0;
        for (int i = 0; i < sms; ++i) {
            issue += h[2 * i];
            total += h[2 * i + 1];
        }
        printf("mask %2d (%s%s%s%s%s%s): issue %7.1f cyc/step, with drain %7.1f cyc/step\n", mask, mask & 1 ? "SS " : "",
               mask & 2 ? "TS " : "", mask & 4 ? "commit2 " : "", mask & 8 ? "wait3 " : "", mask & 16 ? "fence " : "", mask & 32 ? "warp" : "",
               issue / sms / steps, total / sms / steps);
    }
    return 0;
}
