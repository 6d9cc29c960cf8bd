// Micro-benchmark: per-iteration cost of a single-thread issue loop (lane 0
// only, the rest of the CTA parked at the final barrier) versus a converged
// whole-warp loop whose tcgen05 ops are predicated by elect.sync inside the
// asm block (no C++-level divergence). Body: 4 x tf32 SS M128 N64 K8 MMAs +
// 1 commit per iteration, or empty. One CTA per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//   -I paper_2303_05601_b200/csrc/device tools/issue_rate.cu -o tools/_bin/issue_rate
#include <cstdio>

#include "sm100.cuh"

using namespace gfx::sm100;

__device__ __forceinline__ void mma_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
    asm volatile(
        "{\n.reg .pred p;\nelect.sync _|p, 0xffffffff;\n"
        "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;\n}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc));
}
__device__ __forceinline__ void commit_elect(uint64_t* bar) {
    asm volatile(
        "{\n.reg .pred p;\nelect.sync _|p, 0xffffffff;\n"
        "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(bar))
        : "memory");
}

// mode: 0 lane-0 loop empty, 1 lane-0 loop MMAs, 2 warp loop empty, 3 warp loop MMAs (elect in asm),
//       4 lane-0 loop MMAs, rest of warp 0 also spinning in the same loop doing nothing
__global__ void __launch_bounds__(128, 1) issue_rate(int steps, int mode, long long* out, const char* gsrc, int tma) {
    extern __shared__ uint8_t raw[];
    uint8_t* sm = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
    __shared__ __align__(8) uint64_t bar[2];
    __shared__ uint32_t tmem_base;
    for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
    __shared__ __align__(8) uint64_t tbar[4];
    __shared__ volatile int stop_flag;
    if (threadIdx.x == 0) stop_flag = 0;
    if (threadIdx.x < 32) tmem_alloc<512>(&tmem_base);
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        for (int i = 0; i < 4; ++i) mbar_init(&tbar[i], 1);
        mbar_fence_init();
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = tmem_base;
    constexpr uint32_t id64 = umma_idesc<128, 64, 2>();
    const uint64_t wd = umma_desc_sw128(sm, 0), xd = umma_desc_sw128(sm + 16384, 0);
    long long t0 = 0, t1 = 0;
    // Optional background smem traffic: warp 2 streams 16 KB bulk copies from HBM/L2
    // into a 4-deep ring (64 KB) for as long as the issue loop runs (tma: 0 off, 1 on).
    if (tma && threadIdx.x == 64) {
        uint8_t* ring = sm;
        uint32_t ph[4] = {0, 0, 0, 0};
        size_t off = (static_cast<size_t>(blockIdx.x) * 997) << 14;
        for (int i = 0; i < 4; ++i) {
            mbar_arrive_expect_tx(&tbar[i], 16384);
            tma_bulk_g2s(ring + i * 16384, gsrc + (off & ((1ull << 30) - 1)), 16384, &tbar[i]);
            off += 16384 * 148;
        }
        for (int it = 0; !stop_flag; ++it) {
            const int i = it & 3;
            mbar_wait(&tbar[i], ph[i]);
            ph[i] ^= 1;
            mbar_arrive_expect_tx(&tbar[i], 16384);
            tma_bulk_g2s(ring + i * 16384, gsrc + (off & ((1ull << 30) - 1)), 16384, &tbar[i]);
            off += 16384 * 148;
        }
        for (int i = 0; i < 4; ++i) mbar_wait(&tbar[i], ph[i]);
    }
    if (mode == 0 || mode == 1) {
        if (threadIdx.x == 0) {
            t0 = clock64();
            for (int st = 0; st < steps; ++st) {
                if (mode == 1) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) umma_tf32(tm + (st & 1) * 64, wd + kk * 2, xd + kk * 2, id64, 1u);
                    umma_commit(&bar[0]);
                }
            }
            t1 = clock64();
        }
    } else if (mode == 4 || mode == 5) {
        // lane-0 loop, operands rotating over 8 ring slots of 24 KB (W 16 KB + X 8 KB), like K1 v6;
        // mode 5 adds 4 TS MMAs (A = W_lo from TMEM, N = 32) per iteration
        if (threadIdx.x == 0) {
            constexpr uint32_t id32 = umma_idesc<128, 32, 2>();
            t0 = clock64();
            for (int st = 0; st < steps; ++st) {
                const uint8_t* w = sm + (st & 7) * 24576;
                const uint64_t wds = umma_desc_sw128(w, 0), xds = umma_desc_sw128(w + 16384, 0);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    umma_tf32(tm + (st & 1) * 64, wds + kk * 2, xds + kk * 2, id64, 1u);
                    if (mode == 5) umma_tf32_ts(tm + (st & 1) * 64, tm + 128 + (st & 7) * 32 + kk * 8, xds + kk * 2, id32, 1u);
                }
                umma_commit(&bar[0]);
            }
            t1 = clock64();
        }
    } else if (mode >= 6) {
        // lane-0 loop, TS only (A from TMEM stages rotating over 6 x 64 columns), B = X slot rotating:
        // 6: per kk TS N64 (W_hi) + TS N32 (W_lo)   7: per kk TS N64 only   8: per kk 2 x TS N64 (v5)
        // 9: per kk TS N64 + TS N32, B slot fixed
        if (threadIdx.x == 0) {
            constexpr uint32_t id32 = umma_idesc<128, 32, 2>();
            t0 = clock64();
            for (int st = 0; st < steps; ++st) {
                const uint8_t* x = sm + (mode == 9 ? 0 : (st & 7)) * 24576 + 16384;
                const uint64_t xds = umma_desc_sw128(x, 0);
                const uint32_t hi = tm + 128 + (st % 6) * 64, lo = hi + 32;
                const uint32_t acc = tm + ((st >> 2) & 1) * 64;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    umma_tf32_ts(acc, hi + kk * 8, xds + kk * 2, id64, 1u);
                    if (mode == 6 || mode == 9) umma_tf32_ts(acc, lo + kk * 8, xds + kk * 2, id32, 1u);
                    if (mode == 8) umma_tf32_ts(acc, lo + kk * 8, xds + kk * 2, id64, 1u);
                }
                umma_commit(&bar[0]);
            }
            t1 = clock64();
        }
    } else if (mode >= 10 && mode <= 12) {
        // bf16 SS M128 x N x K16, 4 per iteration (one 64-wide K stage), operands rotating over
        // 4 stages of A (16 KB) + B (N x 128 B): 10 -> N=128, 11 -> N=256, 12 -> N=256 same address
        if (threadIdx.x == 0) {
            const int N = mode == 10 ? 128 : 256;
            const uint32_t idesc = N == 128 ? umma_idesc<128, 128, 1>() : umma_idesc<128, 256, 1>();
            const uint32_t stage = 16384 + N * 128;
            t0 = clock64();
            for (int st = 0; st < steps; ++st) {
                const uint8_t* a0 = sm + (mode == 12 ? 0 : (st & 3)) * stage;
                const uint64_t ad = umma_desc_sw128(a0, 0), bd = umma_desc_sw128(a0 + 16384, 0);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) umma_f16(tm + (st & 1) * 256, ad + kk * 2, bd + kk * 2, idesc, 1u);
                umma_commit(&bar[0]);
            }
            t1 = clock64();
        }
    } else if (mode == 2 || mode == 3) {
        if (threadIdx.x < 32) {
            t0 = clock64();
            for (int st = 0; st < steps; ++st) {
                if (mode == 3) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) mma_elect(tm + (st & 1) * 64, wd + kk * 2, xd + kk * 2, id64);
                    commit_elect(&bar[0]);
                }
            }
            t1 = clock64();
        }
    }
    if (threadIdx.x == 0) {
        umma_commit(&bar[1]);
        mbar_wait(&bar[1], 0);
        const long long t2 = clock64();
        out[2 * blockIdx.x] = t1 - t0;
        out[2 * blockIdx.x + 1] = t2 - t0;
        stop_flag = 1;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x < 32) tmem_dealloc<512>(tm);
}

int main() {
    const int sms = 148;
    long long *d, h[2 * 148];
    cudaMalloc(&d, sizeof h);
    cudaFuncSetAttribute(issue_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 201 * 1024);
    char* gsrc;
    cudaMalloc(&gsrc, 1ull << 30);
    cudaMemset(gsrc, 0, 1ull << 30);
    const char* names[] = {"lane0 empty", "lane0 4xMMA+commit", "warp empty", "warp 4xMMA+commit (elect)",
                           "lane0 4xMMA rotating slots", "lane0 4xSS+4xTS rotating", "TS N64+N32 x4 rot",
                           "TS N64 x4 rot", "TS 2xN64 x4 rot (v5)", "TS N64+N32 x4 fixed B",
                           "bf16 SS N128 K16 x4 rot", "bf16 SS N256 K16 x4 rot", "bf16 SS N256 K16 x4 same"};
    for (int tma : {0}) {
        const int steps = 4000;
        for (int mode = 0; mode < 13; ++mode) {
            issue_rate<<<sms, 128, 201 * 1024>>>(steps, mode, d, gsrc, tma);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("mode %d: %s\n", mode, cudaGetErrorString(e));
                return 1;
            }
            cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
            double issue = 0, total = 0;
            for (int i = 0; i < sms; ++i) {
                issue += h[2 * i];
                total += h[2 * i + 1];
            }
            printf("tma %d %-28s issue %8.1f cyc/iter, incl. drain %8.1f cyc/iter\n", tma, names[mode],
                   issue / sms / steps, total / sms / steps);
        }
    }
    return 0;
}
