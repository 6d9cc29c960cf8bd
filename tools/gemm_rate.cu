// Micro-benchmark: tcgen05 bf16 MMA throughput for GEMM-shaped issue, one CTA
// per SM (148), one elected thread issuing K-loop MMAs (M=128, N in {64, 128,
// 256}, K=16 each) from smem operands rotating over `stages` ring stages, one
// accumulator per tile of `ktiles` 64-wide K stages, commit every `commit_every`
// stages. Reports cycles per MMA and the implied dense bf16 TFLOP/s at 1.9 GHz.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//   -I paper_2303_05601_b200/csrc/device tools/gemm_rate.cu -o tools/_bin/gemm_rate
#include <cstdio>

#include "sm100.cuh"

using namespace gfx::sm100;

template <int N, bool kPair = false>
__global__ void __launch_bounds__(128, 1) gemm_rate(int iters, int stages, int commit_every, int same_d, long long* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* sm = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ uint32_t tmem_base;
    constexpr uint32_t kStage = 16384 + (kPair ? N / 2 : N) * 128;
    for (int i = threadIdx.x; i < static_cast<int>(stages * kStage / 4); i += blockDim.x)
        reinterpret_cast<uint32_t*>(sm)[i] = 0;
    if (threadIdx.x < 32) {
        if (kPair)
            tmem_alloc_pair<512>(&tmem_base);
        else
            tmem_alloc<512>(&tmem_base);
    }
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_fence_init();
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    if (kPair) cluster_sync();
    tc_fence_after();
    const uint32_t tm = tmem_base;
    if (threadIdx.x == 0 && (!kPair || cluster_ctarank() == 0)) {
        constexpr uint32_t idesc = umma_idesc<kPair ? 256 : 128, N, 1>();
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const uint8_t* a0 = sm + (it % stages) * kStage;
            const uint64_t ad = umma_desc_sw128(a0, 0), bd = umma_desc_sw128(a0 + 16384, 0);
            const uint32_t d = tm + (same_d ? 0u : static_cast<uint32_t>((it / 8) & 1) * (N <= 256 ? N : 256));
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                if (kPair)
                    umma_f16_pair(d, ad + kk * 2, bd + kk * 2, idesc, 1u);
                else
                    umma_f16(d, ad + kk * 2, bd + kk * 2, idesc, 1u);
            }
            if ((it + 1) % commit_every == 0) {
                if (kPair)
                    umma_commit_pair_multicast(&bar[0], 0x3);
                else
                    umma_commit(&bar[0]);
            }
        }
        if (kPair)
            umma_commit_pair_multicast(&bar[1], 0x1);
        else
            umma_commit(&bar[1]);
        mbar_wait(&bar[1], 0);
        const long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (kPair) cluster_sync();
    tc_fence_after();
    if (threadIdx.x < 32) {
        if (kPair)
            tmem_dealloc_pair<512>(tm);
        else
            tmem_dealloc<512>(tm);
    }
}

template <int N, bool kPair = false>
void run(int stages, int commit_every, int same_d, long long* d, long long* h) {
    const int sms = 148, iters = 2000;
    const size_t smem = stages * (16384 + (kPair ? N / 2 : N) * 128) + 1024;
    cudaFuncSetAttribute(gemm_rate<N, kPair>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(sms);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kPair ? 2 : 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, gemm_rate<N, kPair>, iters, stages, commit_every, same_d, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("N %d: %s\n", N, cudaGetErrorString(e));
        return;
    }
    cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
    double sum = 0;
    int n = 0;
    for (int i = 0; i < sms; i += kPair ? 2 : 1) sum += h[i], ++n;
    const double cyc = sum / n / (iters * 4.0);
    // per SM: 128 x N x 16 MACs per instruction (pair: each SM its 128 rows)
    const double tf = 2.0 * 128 * N * 16 / cyc * 1.9e9 * 148 / 1e12;
    printf("bf16 SS %s N%3d K16: stages %d commit/%2d %s: %6.1f cyc/MMA -> %6.0f TFLOP/s @1.9GHz\n",
           kPair ? "2SM M256" : "M128    ", N, stages, commit_every, same_d ? "same D " : "2 Ds   ", cyc, tf);
}

int main() {
    long long *d, h[148];
    cudaMalloc(&d, sizeof h);
    cudaMemset(d, 0, sizeof h);
    run<256, true>(4, 1, 1, d, h);
    run<256, true>(6, 1, 1, d, h);
    run<256, true>(6, 16, 1, d, h);
    run<128, true>(6, 1, 1, d, h);
    for (int same : {1}) {
        run<64>(4, 1, same, d, h);
        run<128>(4, 1, same, d, h);
        run<256>(4, 1, same, d, h);
        run<128>(4, 16, same, d, h);
        run<256>(4, 16, same, d, h);
        run<256>(1, 16, same, d, h);
    }
    return 0;
}
