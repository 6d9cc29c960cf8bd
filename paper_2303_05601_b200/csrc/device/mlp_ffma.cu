// K1: fp32 linear layer of the MLP model family at batch 32, reading weights
// straight out of the paged HBM arena.
//
//   Y[32 x N] = act(X[32 x K] . W^T + b),  W row-major [N x K] (Linear layout)
//   act = ReLU on hidden layers; the last layer also writes softmax(Y) rows.
//
// Bound: at batch 32 the arithmetic intensity is 16 flop/B of weights, above
// the FFMA ridge (FP32 peak / HBM BW ~ 11 flop/B), so the kernel is FFMA-pipe
// bound; DESIGN.md §5 has the roofline. fp32 throughout (FFMA) because the
// north-star tolerance for fp32 (1e-5 relative) excludes plain TF32.
//
// Structure (one launch per layer):
//   * CTA tile = 64 output features x 32 rows x a K-split; grid = tiles x S,
//     S chosen so the grid covers ~2 CTAs per SM (a batch-32 layer is far too
//     small to fill 148 SMs without splitting K).
//   * 4-stage cp.async pipeline: per 32-wide K step a W tile (64 x 32, 8 KB) and
//     an X tile (32 x 32, 4 KB) land in shared memory. W rows are stored with a
//     16-byte-chunk XOR swizzle (chunk ^ (row & 7)) so the per-lane LDS.128
//     reads of 8 consecutive rows hit 8 distinct bank groups; X reads are
//     warp-uniform broadcasts.
//   * 8 warps = 4 row groups (8 rows) x 2 K halves; each lane owns features
//     (lane, lane+32): 16 accumulators, 64 FFMA per 10 LDS.128.
//   * K halves are reduced through shared memory; K splits through a global
//     workspace reduced by the last-arriving CTA of each feature tile in fixed
//     split order — deterministic, no atomics on data.
//   * Bias + ReLU fused into that epilogue; on the last layer the last tile to
//     finish runs the row softmax (warp-shuffle max/sum) over all 32 rows.
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"
#include "mlp_ffma.cuh"

namespace gfx {

namespace {

constexpr int kRows = 32;      // batch rows per request
constexpr int kTileF = 64;     // output features per CTA
constexpr int kTileK = 32;     // K per pipeline stage
constexpr int kStages = 4;
constexpr int kThreads = 256;

struct __align__(16) Stage {
    float w[kTileF * kTileK];  // 8 KB, swizzled rows
    float x[kRows * kTileK];   // 4 KB
};

__device__ __forceinline__ const char* translate(const char* arena, const uint32_t* pt, uint64_t v) {
    return arena + (static_cast<uint64_t>(pt[v >> kPageShift]) << kPageShift) + (v & kPageMask);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
    const int bytes = valid ? 16 : 0;  // 0 -> zero-fill (out-of-range feature rows)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__global__ void __launch_bounds__(kThreads, 2) mlp_layer_kernel(const __grid_constant__ MlpLayerArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Stage* stages = reinterpret_cast<Stage*>(smem_raw);
    __shared__ uint32_t pt[GFX_MAX_PAGES];
    __shared__ int last_flag;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int tile = blockIdx.x;
    const int split = blockIdx.y;
    const int f0 = tile * kTileF;
    const int K = a.K;
    const int N = a.N;

    for (int i = tid; i < static_cast<int>(a.pt.n); i += kThreads) pt[i] = a.pt.page[i];
    __syncthreads();

    const int kt_total = K / kTileK;
    const int kt_begin = static_cast<int>((static_cast<long long>(kt_total) * split) / a.splits);
    const int kt_end = static_cast<int>((static_cast<long long>(kt_total) * (split + 1)) / a.splits);
    const int nkt = kt_end - kt_begin;

    // Loader assignment: W tile = 64 rows x 8 chunks (2 per thread), X tile =
    // 32 rows x 8 chunks (1 per thread).
    auto load_stage = [&](int slot, int kt) {
        Stage& st = stages[slot];
        const int k0 = kt * kTileK;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int q = tid + i * kThreads;
            const int r = q >> 3;
            const int c = q & 7;
            const int f = f0 + r;
            const bool ok = f < N;
            const uint64_t v = a.w_off + (static_cast<uint64_t>(ok ? f : 0) * K + k0 + 4 * c) * 4;
            cp_async16(&st.w[r * kTileK + ((c ^ (r & 7)) << 2)], translate(a.arena, pt, v), ok);
        }
        {
            const int r = tid >> 3;
            const int c = tid & 7;
            cp_async16(&st.x[r * kTileK + (c << 2)], a.x + static_cast<size_t>(r) * K + k0 + 4 * c, true);
        }
    };

    // Prologue: fill kStages-1 stages.
#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) {
        if (s < nkt) load_stage(s, kt_begin + s);
        cp_async_commit();
    }

    const int rg = warp & 3;   // rows 8rg .. 8rg+7
    const int kh = warp >> 2;  // chunks 4kh .. 4kh+3 of each K step
    float acc0[8], acc1[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) acc0[r] = acc1[r] = 0.0f;

    for (int it = 0; it < nkt; ++it) {
        cp_async_wait<kStages - 2>();
        __syncthreads();
        // Refill the slot consumed in the previous iteration.
        const int nxt = it + kStages - 1;
        if (nxt < nkt) load_stage(nxt % kStages, kt_begin + nxt);
        cp_async_commit();

        const Stage& st = stages[it % kStages];
        const float* wr0 = &st.w[lane * kTileK];
        const float* wr1 = &st.w[(lane + 32) * kTileK];
        const float* xr = &st.x[(rg * 8) * kTileK];
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
            const int c = kh * 4 + cc;
            const int pc = (c ^ (lane & 7)) << 2;  // rows lane and lane+32 share the swizzle
            const float4 w0 = *reinterpret_cast<const float4*>(wr0 + pc);
            const float4 w1 = *reinterpret_cast<const float4*>(wr1 + pc);
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const float4 xv = *reinterpret_cast<const float4*>(xr + r * kTileK + (c << 2));
                acc0[r] = fmaf(w0.x, xv.x, acc0[r]);
                acc0[r] = fmaf(w0.y, xv.y, acc0[r]);
                acc0[r] = fmaf(w0.z, xv.z, acc0[r]);
                acc0[r] = fmaf(w0.w, xv.w, acc0[r]);
                acc1[r] = fmaf(w1.x, xv.x, acc1[r]);
                acc1[r] = fmaf(w1.y, xv.y, acc1[r]);
                acc1[r] = fmaf(w1.z, xv.z, acc1[r]);
                acc1[r] = fmaf(w1.w, xv.w, acc1[r]);
            }
        }
    }
    cp_async_wait<0>();
    __syncthreads();

    // Reduce the two K halves through shared memory (stage buffers are free now).
    float* red = reinterpret_cast<float*>(smem_raw);  // [4 rg][32 lanes][16]
    if (kh == 1) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            red[(rg * 32 + lane) * 16 + r] = acc0[r];
            red[(rg * 32 + lane) * 16 + 8 + r] = acc1[r];
        }
    }
    __syncthreads();

    const int fa = f0 + lane;
    const int fb = f0 + lane + 32;
    if (kh == 0) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            acc0[r] += red[(rg * 32 + lane) * 16 + r];
            acc1[r] += red[(rg * 32 + lane) * 16 + 8 + r];
        }
        if (a.splits > 1) {
            float* ws = a.ws + static_cast<size_t>(split) * kRows * a.ldws;
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const int row = rg * 8 + r;
                ws[static_cast<size_t>(row) * a.ldws + fa] = acc0[r];
                ws[static_cast<size_t>(row) * a.ldws + fb] = acc1[r];
            }
        }
    }

    if (a.splits > 1) {
        // Publish the partial tile; the last CTA of this feature tile reduces.
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            const unsigned prev = atomicAdd(&a.counters[tile], 1u);
            last_flag = prev == static_cast<unsigned>(a.splits - 1);
        }
        __syncthreads();
        if (!last_flag) return;
        __threadfence();
        if (kh == 0) {
#pragma unroll
            for (int r = 0; r < 8; ++r) acc0[r] = acc1[r] = 0.0f;
            for (int s = 0; s < a.splits; ++s) {  // fixed order: deterministic
                const float* ws = a.ws + static_cast<size_t>(s) * kRows * a.ldws;
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    const int row = rg * 8 + r;
                    acc0[r] += __ldcg(&ws[static_cast<size_t>(row) * a.ldws + fa]);
                    acc1[r] += __ldcg(&ws[static_cast<size_t>(row) * a.ldws + fb]);
                }
            }
        }
        if (tid == 0) a.counters[tile] = 0;  // ready for the next launch
    }

    // Epilogue: bias (+ ReLU), store rows.
    float va[8], vb[8];
    if (kh == 0) {
        const float ba = fa < N ? *reinterpret_cast<const float*>(translate(a.arena, pt, a.b_off + 4ull * fa)) : 0.f;
        const float bb = fb < N ? *reinterpret_cast<const float*>(translate(a.arena, pt, a.b_off + 4ull * fb)) : 0.f;
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int row = rg * 8 + r;
            va[r] = acc0[r] + ba;
            vb[r] = acc1[r] + bb;
            if (a.relu) {
                va[r] = fmaxf(va[r], 0.0f);
                vb[r] = fmaxf(vb[r], 0.0f);
            }
            if (fa < N) a.y[static_cast<size_t>(row) * N + fa] = va[r];
            if (fb < N) a.y[static_cast<size_t>(row) * N + fb] = vb[r];
        }
    }
    if (a.probs == nullptr) return;

    // Last layer, softmax in two levels. (1) This tile's per-row partial
    // (max, sum exp) over its 64 features, straight from registers.
    if (kh == 0) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            float m = fmaxf(fa < N ? va[r] : -INFINITY, fb < N ? vb[r] : -INFINITY);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            float e = (fa < N ? expf(va[r] - m) : 0.f) + (fb < N ? expf(vb[r] - m) : 0.f);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
            if (lane == 0) {
                float* st = a.stats + (static_cast<size_t>(tile) * kRows + rg * 8 + r) * 2;
                st[0] = m;
                st[1] = e;
            }
        }
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        const unsigned prev = atomicAdd(&a.counters[a.ntiles], 1u);
        last_flag = prev == static_cast<unsigned>(a.ntiles - 1);
    }
    __syncthreads();
    if (!last_flag) return;
    __threadfence();
    // (2) The last tile combines the partials per row (fixed tile order) ...
    float* rowstat = reinterpret_cast<float*>(smem_raw);  // [32][2]
    if (tid < kRows) {
        float m = -INFINITY;
        for (int t = 0; t < a.ntiles; ++t) m = fmaxf(m, __ldcg(a.stats + (static_cast<size_t>(t) * kRows + tid) * 2));
        float ssum = 0.f;
        for (int t = 0; t < a.ntiles; ++t) {
            const float* st = a.stats + (static_cast<size_t>(t) * kRows + tid) * 2;
            ssum += __ldcg(st + 1) * expf(__ldcg(st) - m);
        }
        rowstat[2 * tid] = m;
        rowstat[2 * tid + 1] = 1.0f / ssum;
    }
    __syncthreads();
    // ... and writes every probability, element-parallel over all 256 threads.
    const int total = kRows * N;
    for (int i = tid; i < total; i += 4 * kThreads) {
        float v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int j = i + u * kThreads;
            v[u] = j < total ? __ldcg(a.y + j) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int j = i + u * kThreads;
            if (j < total) {
                const int row = j / N;
                a.probs[j] = expf(v[u] - rowstat[2 * row]) * rowstat[2 * row + 1];
            }
        }
    }
    if (tid == 0) a.counters[a.ntiles] = 0;
}

}  // namespace

int mlp_layer_splits(int K, int N, int sm_count) {
    const int tiles = (N + kTileF - 1) / kTileF;
    const int kt = K / kTileK;
    // At most one wave of 2 CTAs per SM: a partial second wave idles most SMs.
    int s = (2 * sm_count) / tiles;
    if (s > kt / 2) s = kt / 2;  // >= 2 K steps per CTA
    if (s > kMaxSplits) s = kMaxSplits;
    return s < 1 ? 1 : s;
}

int mlp_layer_tiles(int N) { return (N + kTileF - 1) / kTileF; }

size_t mlp_layer_smem() { return sizeof(Stage) * kStages; }

void launch_mlp_layer(const MlpLayerArgs& a, cudaStream_t stream) {
    if (a.K % kTileK != 0 || a.N % 4 != 0) throw std::runtime_error("mlp layer: K must be a multiple of 32, N of 4");
    static bool attr_set = false;
    const size_t smem = mlp_layer_smem();
    if (!attr_set) {
        GFX_CUDA(cudaFuncSetAttribute(mlp_layer_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
        attr_set = true;
    }
    dim3 grid(static_cast<unsigned>(a.ntiles), static_cast<unsigned>(a.splits));
    mlp_layer_kernel<<<grid, kThreads, smem, stream>>>(a);
    GFX_CUDA(cudaGetLastError());
}

// Request inputs / test tensors straight from the parameter stream.
__global__ void fill_params_kernel(float* dst, uint64_t n, uint64_t stream, float scaled) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        dst[i] = param_at(stream, i, scaled);
}

void launch_fill_params(float* dst, uint64_t n, uint64_t seed, uint32_t tensor, float scale, cudaStream_t s) {
    const uint64_t stream = param_stream(seed, tensor);
    unsigned blocks = static_cast<unsigned>((n + 255) / 256);
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks == 0) blocks = 1;
    fill_params_kernel<<<blocks, 256, 0, s>>>(dst, n, stream, param_scale(scale));
    GFX_CUDA(cudaGetLastError());
}

}  // namespace gfx
