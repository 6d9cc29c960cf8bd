// K1: fp32 linear layer of the MLP model family at batch 32 on the 5th-gen
// tensor cores (tcgen05, kind::tf32) with 3xTF32 error compensation, weights
// streamed by TMA straight out of the paged HBM arena.
//
//   Y[32 x N] = act(X[32 x K] . W^T + b);  computed as D^T[N x 32] = W . X^T
//   ("swap AB": the weight rows fill the 128-row MMA M side, the 32 batch rows
//   are the MMA N side), act = ReLU on hidden layers; the last layer also
//   produces softmax(Y) rows.
//
// Precision: fp32 inputs are split v = hi + lo with hi = v rounded to the
// nearest TF32 value and lo = v - hi (exact). The B operand stacks the batch
// planes [X_hi; X_lo] as 64 MMA columns, so per K=8 slice two MMAs
// (W_lo.[X_hi;X_lo], then W_hi.[X_hi;X_lo]) accumulate all four products into
// a 128 x 64 fp32 TMEM accumulator; the drain adds the two 32-column halves.
// ~fp32 accuracy, which the north-star fp32 tolerance (1e-5) requires — plain
// TF32 would not meet it. (Measured on B200, tools/mma_rate.cu: a tcgen05.mma
// with M=128 costs ~40 cycles at N=32 and ~48 at N=64, so two N=64 MMAs per
// slice are 1.6x cheaper than the classic three N=32 3xTF32 products.)
//
// Bound: batch 32 gives 16 flop per weight byte; three TF32 MMAs per product
// still leave the tensor pipe far from its limit, so the kernel is bound by
// streaming fp32 weights from HBM.
//
// Structure, one CTA per (128-feature tile, K split), 1 CTA per SM:
//   warp 0      TMA producer into a 6-deep landing ring (120 KB in flight per
//               SM covers HBM latency): per 32-wide K step one 1-D bulk copy
//               of the 16 KB pre-swizzled weight tile (the model blob stores W
//               as SWIZZLE_128B K-major 128x32 tiles, so a tile never
//               straddles a 2 MiB arena page) + one 2-D tensor-map copy of the
//               32x32 activation tile;
//   warps 2-5   split each landed tile into hi/lo planes of a 2-deep operand
//               ring (elementwise, so the swizzled layout is preserved),
//               release the landing slot, fence.proxy.async and arrive;
//   warp 1      one elected thread issues 8 tcgen05.mma (4 K slices x 2
//               N=64 products) per stage into a 128x64 fp32 TMEM accumulator and
//               commits the stage back to the producer; accumulators are
//               double-buffered per chunk of 4 K tiles;
//   warps 2-5   drain each finished chunk (tcgen05.ld of their 32-lane TMEM
//               quarter) into fp32 registers while the next chunk runs, then
//               the epilogue: split-K
//               partials through a global workspace reduced by the last CTA of
//               the feature tile in fixed split order (deterministic), bias +
//               ReLU. The classifier softmax is a separate row-parallel kernel.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <stdexcept>

#include "common.cuh"
#include "mlp.cuh"
#include "sm100.cuh"

namespace gfx {

namespace {

using namespace gfx::sm100;

constexpr int kRows = 32;        // batch rows per request = MMA N
constexpr int kTileM = 128;      // output features per CTA = MMA M
constexpr int kTileK = 32;       // fp32 K per stage (= one 128-byte swizzle row)
constexpr int kLand = 8;         // TMA landing ring: raw fp32 tiles in flight from HBM
constexpr int kOps = 6;          // converted operand ring: W hi/lo in TMEM, X hi/lo in smem
constexpr int kThreads = 320;    // 10 warps: TMA, MMA, 4 converters, 4 drain/epilogue
constexpr uint32_t kWBytes = kTileM * kTileK * 4;  // 16 KB
constexpr uint32_t kXBytes = kRows * kTileK * 4;   // 4 KB
constexpr uint32_t kLandBytes = kWBytes + kXBytes;           // 20 KB, 1024-aligned
constexpr uint32_t kOpBytes = 2 * kXBytes;                   // 8 KB: X hi + X lo (W hi/lo live in TMEM)
constexpr int kCounterDone = 128;  // counters[kCounterDone + tile]: splits done reducing
// TMEM: columns [0,128) two 64-column fp32 accumulators (double-buffered
// chunks; columns 0-31 of one = products with X_hi, 32-63 = with X_lo);
// operand stage o: W_hi at 128 + 64o, W_lo at 128 + 64o + 32 (lane = weight row, column = k).
constexpr uint32_t kAccCols = 2 * kRows;
constexpr uint32_t kOpBase = 2 * kAccCols;
constexpr uint32_t kTmemCols = 512;
static_assert(kOpBase + 64 * kOps <= 512, "TMEM budget");
constexpr int kChunk = 4;           // K tiles accumulated in TMEM before draining to fp32 registers

struct Landing {
    uint8_t* w;
    uint8_t* x;
};
__device__ __forceinline__ Landing landing(uint8_t* base, int s) {
    uint8_t* p = base + static_cast<size_t>(s) * kLandBytes;
    return {p, p + kWBytes};
}
struct Operands {
    uint8_t* x_hi;
    uint8_t* x_lo;
};
__device__ __forceinline__ Operands operands(uint8_t* base, int s) {
    uint8_t* p = base + static_cast<size_t>(kLand) * kLandBytes + static_cast<size_t>(s) * kOpBytes;
    return {p, p + kXBytes};
}

__device__ __forceinline__ const char* translate(const char* arena, const uint32_t* pt, uint64_t v) {
    return arena + (static_cast<uint64_t>(pt[v >> kPageShift]) << kPageShift) + (v & kPageMask);
}

// v = hi + lo, hi = v rounded to the nearest TF32 value (exact in TF32),
// lo = v - hi exact in fp32, |lo| <= 2^-11 |v|.
__device__ __forceinline__ void split_tf32(const float4& v, float4& hi, float4& lo) {
    const float* a = reinterpret_cast<const float*>(&v);
    float* h = reinterpret_cast<float*>(&hi);
    float* b = reinterpret_cast<float*>(&lo);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        h[i] = __uint_as_float((__float_as_uint(a[i]) + 0x1000u) & 0xFFFFE000u);
        b[i] = a[i] - h[i];
    }
}

__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 1, 128;\n" ::: "memory"); }  // drain warps
// Programmatic dependent launch: wait for the previous kernel of the stream
// (no-op without the launch attribute) / let the next one start its prologue.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
__device__ __forceinline__ void trace_mark(unsigned long long* tr, int i) {
    if (tr == nullptr) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    tr[(static_cast<size_t>(blockIdx.y) * gridDim.x + blockIdx.x) * 8 + i] = t;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}

__global__ void __launch_bounds__(kThreads, 1)
    mlp_tc_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ MlpLayerArgs a) {
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment by pointer arithmetic on the shared array itself, so
    // every derived pointer stays in the shared window (LDS/STS, not generic).
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ __align__(8) uint64_t land_full[kLand], land_empty[kLand], op_full[kOps], op_empty[kOps];
    __shared__ __align__(8) uint64_t tfull_bar[2], tempty_bar[2];
    __shared__ uint32_t tmem_base_s;
    __shared__ uint32_t pt[GFX_MAX_PAGES];
    __shared__ int last_flag;
    __shared__ float red_m[4][kRows], red_s[4][kRows];
    __shared__ float rowstat[kRows][2];

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    const int tile = blockIdx.x;
    const int split = blockIdx.y;
    const int K = a.K;
    const int N = a.N;
    const int kt_total = K / kTileK;
    const int kt_begin = static_cast<int>((static_cast<long long>(kt_total) * split) / a.splits);
    const int kt_end = static_cast<int>((static_cast<long long>(kt_total) * (split + 1)) / a.splits);
    const int nkt = kt_end - kt_begin;

    if (tid == 0) trace_mark(a.trace, 0);
    for (int i = tid; i < static_cast<int>(a.pt.n); i += kThreads) pt[i] = a.pt.page[i];
    if (tid == 0) {
        for (int s = 0; s < kLand; ++s) {
            mbar_init(&land_full[s], 1);
            mbar_init(&land_empty[s], 128);
        }
        for (int s = 0; s < kOps; ++s) {
            mbar_init(&op_full[s], 128);
            mbar_init(&op_empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull_bar[b], 1);
            mbar_init(&tempty_bar[b], 128);  // the 4 drain warps
        }
        mbar_fence_init();
        tma_prefetch_desc(&tmap_x);
    }
    if (warp == 1) tmem_alloc<kTmemCols>(&tmem_base_s);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_s;
    if (tid == 0) trace_mark(a.trace, 1);

    if (warp == 0) {
        // ---------------- TMA producer ----------------
        if (lane == 0) {
            // Weights do not depend on the previous layer: stream the first
            // landing slots' weight tiles before waiting for it (PDL overlap).
            const int pre = nkt < kLand ? nkt : kLand;
            for (int it = 0; it < pre; ++it) {
                const Landing ld = landing(smem, it);
                mbar_arrive_expect_tx(&land_full[it], kLandBytes);
                const uint64_t v = a.w_off + (static_cast<uint64_t>(tile) * kt_total + kt_begin + it) * kWBytes;
                tma_bulk_g2s(ld.w, translate(a.arena, pt, v), kWBytes, &land_full[it]);
            }
            pdl_wait();
            for (int it = 0; it < pre; ++it)
                tma_tile2d_g2s(landing(smem, it).x, &tmap_x, (kt_begin + it) * kTileK, 0, &land_full[it]);
            trace_mark(a.trace, 2);
            for (int it = pre; it < nkt; ++it) {
                const int s = it % kLand;
                mbar_wait(&land_empty[s], ((it / kLand) & 1) ^ 1);
                const Landing ld = landing(smem, s);
                const int kt = kt_begin + it;
                mbar_arrive_expect_tx(&land_full[s], kLandBytes);
                const uint64_t v = a.w_off + (static_cast<uint64_t>(tile) * kt_total + kt) * kWBytes;
                tma_bulk_g2s(ld.w, translate(a.arena, pt, v), kWBytes, &land_full[s]);
                tma_tile2d_g2s(ld.x, &tmap_x, kt * kTileK, 0, &land_full[s]);
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        if (lane == 0) {
            constexpr uint32_t idesc = umma_idesc<kTileM, 2 * kRows, 2>();  // TF32 x TF32 -> F32, N = 64
            for (int it = 0; it < nkt; ++it) {
                const int s = it % kOps;
                const int chunk = it / kChunk;
                const uint32_t acc_tmem = tmem + static_cast<uint32_t>((chunk & 1) * kAccCols);
                // Chunk c reuses accumulator buffer c&1: wait until chunk c-2 was drained.
                if (it % kChunk == 0 && chunk >= 2) mbar_wait(&tempty_bar[chunk & 1], ((chunk >> 1) & 1) ^ 1);
                mbar_wait(&op_full[s], (it / kOps) & 1);
                tc_fence_after();
                const Operands st = operands(smem, s);
                const uint32_t a_hi = tmem + kOpBase + 64u * static_cast<uint32_t>(s), a_lo = a_hi + 32u;
#pragma unroll
                for (int kk = 0; kk < kTileK / 8; ++kk) {
                    // B = [X_hi; X_lo]: 64 K-major rows (x_lo directly follows x_hi).
                    const uint64_t b = umma_desc_sw128(st.x_hi, kk * 32);
                    const uint32_t ck = static_cast<uint32_t>(kk * 8);  // 8 TMEM columns per K=8 slice
                    if (!(a.ablate & 4)) umma_tf32_ts(acc_tmem, a_lo + ck, b, idesc, ((it % kChunk) | kk) ? 1u : 0u);
                    umma_tf32_ts(acc_tmem, a_hi + ck, b, idesc, ((a.ablate & 4) && ((it % kChunk) | kk) == 0) ? 0u : 1u);
                }
                umma_commit(&op_empty[s]);  // operand buffer free once these MMAs retire
                if (it % kChunk == kChunk - 1 || it == nkt - 1) umma_commit(&tfull_bar[chunk & 1]);
            }
        }
    } else if (warp < 6) {
        // ---------------- converters: hi/lo split into the operand ring ----------------
        const int ct = tid - 64;  // 0..127
        const int q = warp & 3;   // this warp's TMEM lane quarter
        for (int it = 0; it < nkt; ++it) {
            const int s = it % kLand;
            const int o = it % kOps;
            mbar_wait(&land_full[s], (it / kLand) & 1);
            if (it == 0 && ct == 0) trace_mark(a.trace, 3);
            if (it >= kOps) mbar_wait(&op_empty[o], ((it / kOps) & 1) ^ 1);
            const Landing ld = landing(smem, s);
            const Operands op = operands(smem, o);
            if (a.ablate & 2) {
                mbar_arrive(&land_empty[s]);
                mbar_arrive(&op_full[o]);
                continue;
            }
            // This thread owns weight row r = 32q + lane of the tile (its TMEM
            // lane): read the row's 8 swizzled 16-byte chunks (conflict-free),
            // split into hi/lo in registers, store both as 32 TMEM columns.
            const int r = q * 32 + lane;
            const float4* wrow = reinterpret_cast<const float4*>(ld.w + r * 128);
            float whi[32], wlo[32];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float4 v = wrow[j ^ (r & 7)];
                float4 h, l;
                split_tf32(v, h, l);
                whi[4 * j] = h.x; whi[4 * j + 1] = h.y; whi[4 * j + 2] = h.z; whi[4 * j + 3] = h.w;
                wlo[4 * j] = l.x; wlo[4 * j + 1] = l.y; wlo[4 * j + 2] = l.z; wlo[4 * j + 3] = l.w;
            }
            const float4* x = reinterpret_cast<const float4*>(ld.x);
            float4 xv[kXBytes / 16 / 128];
#pragma unroll
            for (int j = 0; j < static_cast<int>(kXBytes / 16 / 128); ++j) xv[j] = x[ct + 128 * j];
            mbar_arrive(&land_empty[s]);  // landing slot back to the TMA producer
            tc_fence_after();             // order after the MMAs that last read stage o
            const uint32_t lane_base = tmem + (static_cast<uint32_t>(q * 32) << 16);
            tmem_st_32x32b_x32(lane_base + kOpBase + 64u * static_cast<uint32_t>(o), whi);
            tmem_st_32x32b_x32(lane_base + kOpBase + 32u + 64u * static_cast<uint32_t>(o), wlo);
#pragma unroll
            for (int j = 0; j < static_cast<int>(kXBytes / 16 / 128); ++j) {
                float4 hi, lo;
                split_tf32(xv[j], hi, lo);
                reinterpret_cast<float4*>(op.x_hi)[ct + 128 * j] = hi;
                reinterpret_cast<float4*>(op.x_lo)[ct + 128 * j] = lo;
            }
            tmem_st_wait();
            tc_fence_before();
            if (!(a.ablate & 1)) fence_proxy_async_smem();
            mbar_arrive(&op_full[o]);
        }
    } else {
        // ---------------- drain + epilogue warps ----------------
        const int ct = tid - 192;  // 0..127
        const int q = warp & 3;    // TMEM lane quarter (warps 6..9 -> 2,3,0,1)
        const int f = tile * kTileM + q * 32 + lane;
        // Bias fetched now; its latency hides behind the whole main loop.
        const float bias = f < N ? *reinterpret_cast<const float*>(translate(a.arena, pt, a.b_off + 4ull * f)) : 0.f;
        const int nchunks = (nkt + kChunk - 1) / kChunk;
        // Accumulator: TMEM lane = feature row of the tile, column = batch row.
        // Each chunk of kChunk K tiles is accumulated by the tensor core, then
        // drained and summed here in fp32 (round-to-nearest) while the next
        // chunk accumulates in the other buffer — short tensor-core
        // accumulation chains keep the fp32 tolerance at any K.
        float acc[kRows];
#pragma unroll
        for (int b = 0; b < kRows; ++b) acc[b] = 0.f;
        for (int c = 0; c < nchunks; ++c) {
            mbar_wait(&tfull_bar[c & 1], (c >> 1) & 1);
            tc_fence_after();
            float ph[kRows], pl[kRows];
            const uint32_t src = tmem + static_cast<uint32_t>((c & 1) * kAccCols) + (static_cast<uint32_t>(q * 32) << 16);
            tmem_ld_32x32b_x32(src + kRows, pl);  // products with X_lo (small)
            tmem_ld_32x32b_x32(src, ph);
#pragma unroll
            for (int b = 0; b < kRows; ++b) acc[b] += ph[b] + pl[b];
            tc_fence_before();
            mbar_arrive(&tempty_bar[c & 1]);
        }
        if (ct == 0) trace_mark(a.trace, 4);

        pdl_trigger();  // main loop done: the next layer may start its prologue
        pdl_wait();     // workspace / counters / output belong to us only after the previous layer
        const bool valid = f < N;  // rows >= N are the zero padding of the last weight tile
        if (a.splits == 1) {
#pragma unroll
            for (int b = 0; b < kRows; ++b) {
                float v = acc[b] + bias;
                if (a.relu) v = fmaxf(v, 0.f);
                if (valid) a.y[static_cast<size_t>(b) * N + f] = v;
            }
        } else {
            // Split-K: publish this CTA's partial ws[tile][split][32][128], wait
            // until all splits of the tile have published (the grid is a single
            // wave, one CTA per SM, so every sibling is resident), then each
            // split reduces its own rows b = split, split+S, ... in fixed split
            // order — deterministic, and the reduction is spread over S CTAs.
            const int fl = q * 32 + lane;
            const size_t blk = static_cast<size_t>(kRows) * kTileM;
            float* base = a.ws + static_cast<size_t>(tile) * a.splits * blk;
#pragma unroll
            for (int b = 0; b < kRows; ++b) base[static_cast<size_t>(split) * blk + b * kTileM + fl] = acc[b];
            __threadfence();
            epi_sync();
            if (ct == 0) {
                atomicAdd(&a.counters[tile], 1u);
                while (ld_acquire(&a.counters[tile]) < static_cast<unsigned>(a.splits)) __nanosleep(64);
            }
            epi_sync();
            // Gather this split's rows of every partial in one round of cp.async
            // (the landing ring is idle now), then sum in fixed split order.
            const int nrows = (kRows - split + a.splits - 1) / a.splits;
            float* red = reinterpret_cast<float*>(smem);  // [nrows][splits][128]
            const int chunks = nrows * a.splits * (kTileM / 4);
            for (int c = ct; c < chunks; c += 128) {
                const int col4 = c % (kTileM / 4), rs = c / (kTileM / 4);
                const int sp = rs % a.splits, ri = rs / a.splits;
                const int b = split + ri * a.splits;
                cp_async16(red + static_cast<size_t>(rs) * kTileM + col4 * 4,
                           base + static_cast<size_t>(sp) * blk + b * kTileM + col4 * 4);
            }
            asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
            epi_sync();
            for (int ri = 0; ri < nrows; ++ri) {
                const int b = split + ri * a.splits;
                float v = 0.f;
                for (int sp = 0; sp < a.splits; ++sp) v += red[static_cast<size_t>(ri * a.splits + sp) * kTileM + fl];
                v += bias;
                if (a.relu) v = fmaxf(v, 0.f);
                if (valid) a.y[static_cast<size_t>(b) * N + f] = v;
            }
            epi_sync();
            if (ct == 0 && atomicAdd(&a.counters[kCounterDone + tile], 1u) == static_cast<unsigned>(a.splits - 1)) {
                a.counters[tile] = 0;  // every sibling has left the spin: reset for the next launch
                a.counters[kCounterDone + tile] = 0;
            }
        }
        if (ct == 0) trace_mark(a.trace, 5);
    }

    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc<kTmemCols>(tmem);
}

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

int mlp_layer_splits(int K, int N, int sm_count) {
    const int tiles = mlp_layer_tiles(N);
    const int kt = K / kTileK;
    int s = sm_count / tiles;  // one wave, one CTA per SM
    if (s > kt) s = kt;
    if (s > kMaxSplits) s = kMaxSplits;
    return s < 1 ? 1 : s;
}

int mlp_layer_tiles(int N) { return (N + kTileM - 1) / kTileM; }

size_t mlp_layer_smem() { return static_cast<size_t>(kLandBytes) * kLand + static_cast<size_t>(kOpBytes) * kOps + 1024; }

void launch_mlp_layer(const MlpLayerArgs& a, cudaStream_t stream, bool pdl) {
    if (a.K % kTileK != 0) throw std::runtime_error("mlp layer: K must be a multiple of 32");
    CUtensorMap tmx;
    if (!encode_tensor_map_2d(&tmx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, a.x, static_cast<uint64_t>(a.K), kRows,
                              static_cast<uint64_t>(a.K) * 4, kTileK, kRows, CU_TENSOR_MAP_SWIZZLE_128B))
        throw CudaError("cuTensorMapEncodeTiled failed for the activation tile map");
    static bool attr_set = false;
    const size_t smem = mlp_layer_smem();
    if (!attr_set) {
        GFX_CUDA(cudaFuncSetAttribute(mlp_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
        attr_set = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(a.ntiles), static_cast<unsigned>(a.splits));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    GFX_CUDA(cudaLaunchKernelEx(&cfg, mlp_tc_kernel, tmx, a));
}

// Row softmax of the classifier logits: one CTA per batch row, 256 threads,
// block-wide max / sum through warp shuffles (K4, HBM/L2-latency bound).
__global__ void __launch_bounds__(256) softmax_rows_kernel(const float* __restrict__ logits,
                                                           float* __restrict__ probs, int C) {
    __shared__ float red[8];
    pdl_wait();
    const int row = blockIdx.x;
    const float* in = logits + static_cast<size_t>(row) * C;
    float* out = probs + static_cast<size_t>(row) * C;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int kPer = 8;  // C <= 2048
    float v[kPer];
    float m = -INFINITY;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
        const int c = threadIdx.x + i * 256;
        v[i] = c < C ? in[c] : -INFINITY;
        m = fmaxf(m, v[i]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) red[warp] = m;
    __syncthreads();
    m = red[0];
#pragma unroll
    for (int w = 1; w < 8; ++w) m = fmaxf(m, red[w]);
    __syncthreads();
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
        const int c = threadIdx.x + i * 256;
        v[i] = c < C ? expf(v[i] - m) : 0.f;
        s += v[i];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    float tot = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) tot += red[w];
    const float inv = 1.0f / tot;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
        const int c = threadIdx.x + i * 256;
        if (c < C) out[c] = v[i] * inv;
    }
}

void launch_softmax_rows(const float* logits, float* probs, int rows, int C, cudaStream_t s) {
    if (C > 2048) throw std::runtime_error("softmax: at most 2048 classes");
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(rows));
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    GFX_CUDA(cudaLaunchKernelEx(&cfg, softmax_rows_kernel, logits, probs, C));
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
