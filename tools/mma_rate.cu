// Micro-benchmark: tcgen05.mma issue-to-completion cost per instruction for the
// K1 shapes (M=128, small N), one CTA per SM, operands in shared memory (SS) or
// A in TMEM (TS). Prints cycles per MMA for a streamed run (one commit at the
// end) and for a chained run (commit + wait every `group` MMAs, like a
// pipeline stage). Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   -I paper_2303_05601_b200/csrc/device tools/mma_rate.cu -o tools/_bin/mma_rate
#include <cstdio>
#include <cstdlib>

#include "sm100.cuh"

using namespace gfx::sm100;

template <int kN, int kFmt, bool kTs>
__global__ void __launch_bounds__(128, 1) mma_rate(int reps, int group, int nacc, long long* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* sm = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tmem_base;
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
    if (threadIdx.x < 32) tmem_alloc<512>(&tmem_base);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_fence_init();
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = tmem_base;
    // `group` < 0: |group| issuing warps (lane 0 of each), 12-MMA unrolled body
    // with compile-time offsets, one accumulator per issuer, no waits.
    const int issuers = group < 0 ? -group : 1;
    if ((threadIdx.x & 31) == 0 && (threadIdx.x >> 5) < issuers) {
        constexpr uint32_t idesc = umma_idesc<128, kN, kFmt>();
        const uint64_t a0 = umma_desc_sw128(sm, 0);            // 128 rows x 128 B
        const uint64_t b0 = umma_desc_sw128(sm + 65536, 0);    // kN rows x 128 B
        uint32_t phase = 0;
        const long long t0 = clock64();
        if (group < 0) {
            const uint32_t d = tm + static_cast<uint32_t>((threadIdx.x >> 5) * 32);
            for (int r = 0; r < reps; r += 12) {
#pragma unroll
                for (int u = 0; u < 12; ++u) {
                    const uint64_t koff = static_cast<uint64_t>((u & 3) * 2);
                    if (kFmt == 2) umma_tf32(d, a0 + koff, b0 + koff, idesc, 1);
                    else umma_f16(d, a0 + koff, b0 + koff, idesc, 1);
                }
            }
        } else {
            for (int r = 0; r < reps; ++r) {
                const uint64_t koff = static_cast<uint64_t>((r & 3) * 2);  // 32-byte K slice (>>4)
                const uint32_t d = tm + static_cast<uint32_t>((r % nacc) * (kN < 64 ? kN : 64));
                if (kTs) {
                    asm volatile(
                        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
                        "r"(tm + 448 + (r & 3) * 8), "l"(b0 + koff), "r"(idesc), "r"(1));
                } else if (kFmt == 2) {
                    umma_tf32(d, a0 + koff, b0 + koff, idesc, 1);
                } else {
                    umma_f16(d, a0 + koff, b0 + koff, idesc, 1);
                }
                if (group > 0 && (r + 1) % group == 0) {
                    umma_commit(&bar);
                    mbar_wait(&bar, phase);
                    phase ^= 1;
                }
            }
        }
        if (threadIdx.x == 0) {
            umma_commit(&bar);
            mbar_wait(&bar, phase);
        }
        const long long t1 = clock64();
        if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x < 32) tmem_dealloc<512>(tm);
}

template <int kN, int kFmt, bool kTs>
void run(const char* name, int reps, int group, int nacc, int sms, long long* d, long long* h) {
    auto k = mma_rate<kN, kFmt, kTs>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    k<<<sms, 128, 100 * 1024>>>(reps, group, nacc, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("%s: %s\n", name, cudaGetErrorString(e));
        exit(1);
    }
    cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
    long long mx = 0, sum = 0;
    for (int i = 0; i < sms; ++i) {
        mx = h[i] > mx ? h[i] : mx;
        sum += h[i];
    }
    printf("%-24s group %3d acc %2d: %7.1f cyc/mma (mean)  %7.1f (max CTA)\n", name, group, nacc, double(sum) / sms / reps,
           double(mx) / reps);
}

int main() {
    int sms = 148;
    long long *d, h[256];
    cudaMalloc(&d, 256 * sizeof(long long));
    const int reps = 12000;
    for (int group : {-1, -2, -4}) {
        run<32, 2, false>("tf32 SS M128 N32 K8 unr", reps, group, 1, sms, d, h);
        run<64, 2, false>("tf32 SS M128 N64 K8 unr", reps, group, 1, sms, d, h);
        run<128, 2, false>("tf32 SS M128 N128 K8 unr", reps, group, 1, sms, d, h);
        run<32, 1, false>("bf16 SS M128 N32 K16 unr", reps, group, 1, sms, d, h);
    }
    run<32, 2, false>("tf32 SS M128 N32 K8", reps, 0, 1, sms, d, h);
    run<32, 2, false>("tf32 SS M128 N32 K8", reps, 1, 1, sms, d, h);
    run<32, 2, false>("tf32 SS M128 N32 K8", reps, 12, 1, sms, d, h);
    return 0;
}
