// K5: the whole BERT encoder (all layers) as ONE persistent dataflow launch.
//
// Every op of a post-LN encoder layer is local to a 128-token row block (one
// sequence): QKV(m) -> attention(m, head) -> O-proj(m) + LN1 -> FFN1(m) ->
// FFN2(m) + LN2 -> QKV of the next layer (m). The per-op launches of bert.cu
// pay ~2 µs of fill and ~2-3 µs of tail per GEMM (5 launches per layer) and
// run the N = 768 GEMMs on 96 of 148 SMs; here one CTA per SM pops READY work
// items from a global queue, so row blocks flow through the layers
// independently and the SMs stay busy across op and layer boundaries.
//
// Items:
//   QKV tile (m, n<9), K 768          epilogue: + bias                 -> qkv
//   ATT (m, head)                      S = Q K^T, softmax, O = P V      -> ctx
//   O tile (m, n<3), K 768            epilogue: + bias + x (residual)  -> t
//   FFN1 tile (m, n<ffn/256), K 768   epilogue: + bias, GELU           -> f
//   FFN2 tile (m, n<3), K ffn         epilogue: + bias + h (residual)  -> t
// A residual tile also writes its 256 columns' per-row (mean, M2) of the
// bf16-rounded t; the CTA completing the LAST of a row block's three residual
// tiles combines the statistics and runs that row block's LayerNorm (t -> h,
// resp. t -> the layer output): the same bf16 rounding points as the per-op path.
//
// Dataflow: the CTA that completes an item's last input (a per-(layer, row
// block, op) completion counter, atom.acq_rel) pushes the successor items into
// the queue (st.release into the slot after an atomic tail bump); a CTA pops
// with an atomic head bump and an ld.acquire of the slot. Layer 0's QKV tiles
// are the queue's implicit first entries. A popped item never waits for
// another CTA, so there is no deadlock by construction and no CTA idles on a
// claimed item whose inputs are late (a static claim order did exactly that:
// profiles/r2_k5_flow.md).
//
// CTA roles (640 threads): warps 0-15 epilogue, 16 A producer + queue pops,
// 17 MMA issuer, 18-19 B (weight) producers. One 4-stage ring of 48 KB stages
// (A + two 16 KB weight tiles; for an attention item Q, K, V) and two 256-column
// TMEM accumulators cycle across ALL items of the CTA, so an item's loads and
// MMAs overlap the previous item's epilogue exactly as inside one GEMM. The
// popped items reach the other roles through a 4-slot shared-memory queue.
// Attention: the MMA warp issues S = Q K^T into the accumulator and moves on;
// the epilogue warps compute the softmax, write P over Q/K in the stage and
// one epilogue thread issues O = P V (tcgen05, V MN-major) whose commit frees
// the stage.
//
// Memory ordering between CTAs: a GEMM tile's four store groups wait for their
// TMA stores to complete and fence the async proxy; the epilogue barriers and
// thread 0 fences and bumps the counter (acq_rel), and pushes with release
// stores. The popping producer acquires the slot and fences the async proxy
// before its TMA loads; generic reads of other CTAs' data (LayerNorm) go
// through L2 (ld.cg) after the counter's acquire.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <stdexcept>
#include <vector>

#include "bert.cuh"
#include "bert_dev.cuh"
#include "sm100.cuh"

namespace gfx {

namespace {

using namespace gfx::sm100;
using namespace gfx::bertdev;

constexpr int kFThreads = 640;
constexpr int kFEpiWarps = 16, kFAWarp = 16, kFMmaWarp = 17, kFBWarp0 = 18;
constexpr int kFStages = 4;
constexpr uint32_t kFTile = 16384;              // 128 rows x 64 bf16, K-major SWIZZLE_128B
constexpr uint32_t kFStage = 3 * kFTile;        // A + 2 weight tiles | Q, K, V
constexpr uint32_t kFRing = kFStages * kFStage;  // 192 KB
constexpr uint32_t kFBoxes = 4 * 8192;          // epilogue staging (4 groups x 128 x 32 bf16)
constexpr size_t kFSmem = kFRing + kFBoxes + 1024;
constexpr int kFQueue = 4;
constexpr uint32_t kFCluster = 3;  // CTAs per cluster = a row block's three d-column tiles
constexpr int kFD = 768, kFHeads = 12, kFSeq = 128;

enum FlowOp : uint32_t { kOpQkv = 0, kOpAtt = 1, kOpO = 2, kOpF1 = 3, kOpF2 = 4, kOpEnd = 7 };
// Completion counters per (layer, row block) = the op; then the queue's head and tail.
constexpr int kCSlots = 5;

__host__ __device__ constexpr uint32_t flow_item(uint32_t op, uint32_t l, uint32_t m, uint32_t n) {
    return (op << 29) | (l << 24) | (m << 12) | n;
}
__device__ __forceinline__ uint32_t it_op(uint32_t it) { return it >> 29; }
__device__ __forceinline__ int it_l(uint32_t it) { return static_cast<int>((it >> 24) & 31u); }
__device__ __forceinline__ int it_m(uint32_t it) { return static_cast<int>((it >> 12) & 4095u); }
__device__ __forceinline__ int it_n(uint32_t it) { return static_cast<int>(it & 4095u); }

#ifdef GFX_K5_DEBUG
// Debug build (make K5_DEBUG=1): per CTA and item ordinal j, %globaltimer marks
// [0] item, [1] popped, [2] = [1], [3] first stage in the MMA warp, [4] last
// MMA issued, [5] epilogue saw the accumulator, [6] epilogue done (successors
// pushed), [7] LayerNorm started here (else 0). bert_encoder_flow writes the
// table of one forward to $GFX_K5_TRACE.
constexpr int kFTraceItems = 512;
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define K5_MARK(j, f, v)                                                                          \
    do {                                                                                          \
        if (a.trace && (j) < kFTraceItems)                                                        \
            a.trace[(static_cast<size_t>(blockIdx.x) * kFTraceItems + (j)) * 8 + (f)] = (v);      \
    } while (0)
#else
#define K5_MARK(j, f, v) \
    do {                 \
    } while (0)
#endif

struct FlowMaps {
    CUtensorMap a_in, a_x, a_ctx, a_h, a_f;  // A operands: 64 x 128 boxes, SWIZZLE_128B
    CUtensorMap qkv;                         // attention Q / K / V: 64 x 128 boxes, SWIZZLE_128B
    CUtensorMap y_qkv, y_f, y_h, y_x;        // outputs: 32 x 128 boxes, SWIZZLE_64B
    CUtensorMap r_in, r_x, r_h;              // residuals: 32 x 128 boxes, SWIZZLE_64B
};

struct FlowArgs {
    const char* arena;
    BertLayerOffsets l0;    // layer 0's parameter offsets; layer l = l0 + l * stride
    uint64_t stride;
    uint32_t* slots;        // ready queue of cluster items: item + 1 per pushed entry (zeroed per launch)
    int n_items, n_first;   // all cluster items; layer 0's QKV triples = the queue's implicit first n_first
    uint32_t* cnt;          // [L][M][kCSlots] completion counters, then head, tail (zeroed per launch)
    float2* stats;          // [L][M][2 LayerNorms][3 column tiles][128 rows] (mean, M2) of the pre-LN rows
    __nv_bfloat16 *ctx, *h, *xout;
    int M, L, ffn;
    int xstride;            // rows between consecutive layers' outputs in xout (0: one buffer)
    unsigned long long* trace;  // GFX_K5_DEBUG builds: [grid][kFTraceItems][8], else nullptr
    PageTable pt;
};

// This CTA's unit of a cluster item (op, l, m, t): the O / FFN2 triple is the row
// block's three column tiles, the others are the t-th triple of tiles / heads.
__device__ __forceinline__ uint32_t cta_item(uint32_t cit, uint32_t rank) {
    const uint32_t op = cit >> 29, t = cit & 4095u;
    const uint32_t n = (op == kOpO || op == kOpF2) ? rank : 3u * t + rank;
    return (cit & ~4095u) | n;
}

__global__ void __launch_bounds__(kFThreads, 1)
    encoder_flow_kernel(const __grid_constant__ FlowMaps mp, const __grid_constant__ FlowArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* boxes = smem + kFRing;
    __shared__ __align__(8) uint64_t full_bar[kFStages], empty_bar[kFStages], tfull_bar[2], tempty_bar[2], res_bar[4];
    __shared__ __align__(8) uint64_t o_bar, q_full[kFQueue], q_empty[kFQueue], sib_bar[2];
    __shared__ uint32_t q_item[kFQueue];
    __shared__ uint32_t tmem_s;
    __shared__ float bias_s[256];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = cluster_ctarank();
    const uint32_t* const pt = a.pt.page;
    if (tid == 0) {
        for (int s = 0; s < kFStages; ++s) {
            mbar_init(&full_bar[s], 3);  // A producer (+tx) and both weight producers
            mbar_init(&empty_bar[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull_bar[b], 1);
            mbar_init(&tempty_bar[b], kFEpiWarps);
            mbar_init(&sib_bar[b], kFCluster);  // the cluster's three CTAs' LayerNorm statistics written
        }
        for (int g = 0; g < 4; ++g) mbar_init(&res_bar[g], 1);
        mbar_init(&o_bar, 1);
        for (int q = 0; q < kFQueue; ++q) {
            mbar_init(&q_full[q], 1);
            // Leader's copy: every consumer of the cluster (weight producers, MMA, epilogue
            // warps of each CTA, and the other CTAs' A producers) releases the slot here.
            mbar_init(&q_empty[q], kFCluster * (2 + 1 + kFEpiWarps) + (kFCluster - 1));
        }
        mbar_fence_init();
        tma_prefetch_desc(&mp.a_in), tma_prefetch_desc(&mp.a_x), tma_prefetch_desc(&mp.a_ctx);
        tma_prefetch_desc(&mp.a_h), tma_prefetch_desc(&mp.a_f), tma_prefetch_desc(&mp.qkv);
        tma_prefetch_desc(&mp.y_qkv), tma_prefetch_desc(&mp.y_f), tma_prefetch_desc(&mp.y_h);
        tma_prefetch_desc(&mp.y_x), tma_prefetch_desc(&mp.r_in), tma_prefetch_desc(&mp.r_x);
        tma_prefetch_desc(&mp.r_h);
    }
    if (warp == kFMmaWarp) tmem_alloc<512>(&tmem_s);
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // every CTA's barriers exist before any remote arrive reaches them
    tc_fence_after();
    const uint32_t tmem = tmem_s;
    uint32_t* const qhead = a.cnt + static_cast<size_t>(a.L) * a.M * kCSlots;
    uint32_t* const qtail = qhead + 1;
    auto counter = [&](int l, int m, uint32_t op) { return a.cnt + (static_cast<size_t>(l) * a.M + m) * kCSlots + op; };
    // Make cluster items first .. first + count - 1 (consecutive triples) ready: after the
    // caller's fence, one tail bump and a release store per queue slot.
    auto push = [&](uint32_t first, int count) {
        const uint32_t base = atomicAdd(qtail, static_cast<uint32_t>(count));
        for (int i = 0; i < count; ++i) st_release_gpu_u32(a.slots + base + i, first + static_cast<uint32_t>(i) + 1u);
    };
    const int nk_ffn = a.ffn / 64, nf1 = a.ffn / 256;
    auto nk_of = [&](uint32_t op) { return op == kOpAtt ? 1 : op == kOpF2 ? nk_ffn : kFD / 64; };
    // Consumers of the cluster's item queue: wait for slot j (filled by the leader CTA),
    // read this CTA's unit, release the slot in the leader.
    auto take = [&](int j) {
        const int slot = j % kFQueue;
        mbar_wait_cluster(&q_full[slot], (j / kFQueue) & 1);
        const uint32_t cit = q_item[slot];
        return (cit >> 29) == kOpEnd ? cit : cta_item(cit, rank);
    };
    auto release = [&](int j) { mbar_arrive_remote(&q_empty[j % kFQueue], 0); };

    if (warp == kFAWarp) {
        // ---------------- A producer (leader: pops ready cluster items and hands them to the
        // cluster's three CTAs); loads A (or Q, K, V) of this CTA's unit.
        if (lane == 0) {
            int g = 0;
            for (int j = 0;; ++j) {
                const int slot = j % kFQueue;
                uint32_t it;
                if (rank == 0) {
                    if (j >= kFQueue) mbar_wait(&q_empty[slot], ((j / kFQueue) & 1) ^ 1);
                    const uint32_t idx = atomicAdd(qhead, 1u);
                    uint32_t cit;
                    if (idx >= static_cast<uint32_t>(a.n_items)) {
                        cit = flow_item(kOpEnd, 0, 0, 0);
                    } else if (idx < static_cast<uint32_t>(a.n_first)) {
                        cit = flow_item(kOpQkv, 0, idx / 3, idx % 3);
                    } else {
                        const uint32_t* sl = a.slots + (idx - a.n_first);
                        uint32_t v;
                        while ((v = ld_acquire_gpu_u32(sl)) == 0) __nanosleep(32);
                        cit = v - 1;
                    }
                    for (uint32_t r = 0; r < kFCluster; ++r) {
                        st_cluster_u32(mapa_u32(&q_item[slot], r), cit);
                        mbar_arrive_remote(&q_full[slot], r);
                    }
                    it = (cit >> 29) == kOpEnd ? cit : cta_item(cit, 0);
                    mbar_wait_cluster(&q_full[slot], (j / kFQueue) & 1);  // keep this CTA's own slot phase in step
                } else {
                    it = take(j);
                    release(j);
                }
                K5_MARK(j, 0, it);
                K5_MARK(j, 1, gtimer());
                const uint32_t op = it_op(it);
                if (op == kOpEnd) break;
                fence_proxy_async_global();  // the pusher's release (acquired above) -> the TMA reads below
                const int l = it_l(it), m = it_m(it);
                K5_MARK(j, 2, gtimer());
                const int m0 = m * kFSeq;
                if (op == kOpAtt) {
                    const int s = g % kFStages, h = it_n(it);
                    if (g >= kFStages) mbar_wait(&empty_bar[s], ((g / kFStages) & 1) ^ 1);
                    uint8_t* st = smem + static_cast<size_t>(s) * kFStage;
                    mbar_arrive_expect_tx(&full_bar[s], 3 * kFTile);
                    tma_tile2d_g2s(st, &mp.qkv, h * 64, m0, &full_bar[s]);
                    tma_tile2d_g2s(st + kFTile, &mp.qkv, kFD + h * 64, m0, &full_bar[s]);
                    tma_tile2d_g2s(st + 2 * kFTile, &mp.qkv, 2 * kFD + h * 64, m0, &full_bar[s]);
                    ++g;
                    continue;
                }
                const CUtensorMap* am = op == kOpO ? &mp.a_ctx : op == kOpF1 ? &mp.a_h : op == kOpF2 ? &mp.a_f
                                        : l == 0  ? &mp.a_in
                                                  : &mp.a_x;
                const int row = (op == kOpQkv && l > 0) ? (l - 1) * a.xstride + m0 : m0;
                const int nk = nk_of(op);
                for (int k = 0; k < nk; ++k, ++g) {
                    const int s = g % kFStages;
                    if (g >= kFStages) mbar_wait(&empty_bar[s], ((g / kFStages) & 1) ^ 1);
                    mbar_arrive_expect_tx(&full_bar[s], kFTile);
                    tma_tile2d_g2s(smem + static_cast<size_t>(s) * kFStage, am, k * 64, row, &full_bar[s]);
                }
            }
        }
    } else if (warp >= kFBWarp0) {
        // ---------------- weight producers: tile h of each stage (independent of other CTAs).
        if (lane == 0) {
            const int h = warp - kFBWarp0;
            int g = 0;
            for (int j = 0;; ++j) {
                const uint32_t it = take(j);
                release(j);
                const uint32_t op = it_op(it);
                if (op == kOpEnd) break;
                if (op == kOpAtt) {  // attention: nothing to load, keep the stage's arrival count
                    const int s = g % kFStages;
                    if (g >= kFStages) mbar_wait(&empty_bar[s], ((g / kFStages) & 1) ^ 1);
                    mbar_arrive(&full_bar[s]);
                    ++g;
                    continue;
                }
                const uint64_t lo = a.stride * static_cast<uint64_t>(it_l(it));
                const uint64_t w = lo + (op == kOpQkv ? a.l0.wqkv : op == kOpO ? a.l0.wo : op == kOpF1 ? a.l0.w1 : a.l0.w2);
                const int nk = nk_of(op);
                const uint64_t bt = static_cast<uint64_t>(it_n(it)) * 2 + h;  // 128-row weight tile of the 256 columns
                for (int k = 0; k < nk; ++k, ++g) {
                    const int s = g % kFStages;
                    if (g >= kFStages) mbar_wait(&empty_bar[s], ((g / kFStages) & 1) ^ 1);
                    mbar_arrive_expect_tx(&full_bar[s], kFTile);
                    const uint64_t v = w + (bt * nk + k) * kFTile;
                    tma_bulk_g2s(smem + static_cast<size_t>(s) * kFStage + kFTile * (1 + h), translate(a.arena, pt, v),
                                 kFTile, &full_bar[s]);
                }
            }
        }
    } else if (warp == kFMmaWarp) {
        // ---------------- MMA issuer.
        if (lane == 0) {
            constexpr uint32_t idesc = umma_idesc<128, 256, 1>();    // bf16 x bf16 -> f32
            constexpr uint32_t idesc_s = umma_idesc<128, 128, 1>();  // S = Q K^T
            int g = 0;
            for (int j = 0;; ++j) {
                const uint32_t it = take(j);
                release(j);
                const uint32_t op = it_op(it);
                if (op == kOpEnd) break;
                const int b = j & 1;
                if (j >= 2) mbar_wait(&tempty_bar[b], ((j >> 1) & 1) ^ 1);  // epilogue drained item j - 2
                tc_fence_after();
                const uint32_t acc = tmem + static_cast<uint32_t>(b * 256);
                if (op == kOpAtt) {
                    const int s = g % kFStages;
                    mbar_wait(&full_bar[s], (g / kFStages) & 1);
                    tc_fence_after();
                    uint8_t* st = smem + static_cast<size_t>(s) * kFStage;
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        umma_f16(acc, umma_desc_sw128(st, kk * 32), umma_desc_sw128(st + kFTile, kk * 32), idesc_s,
                                 kk ? 1u : 0u);
                    umma_commit(&tfull_bar[b]);  // the stage is freed by the epilogue's P V commit
                    K5_MARK(j, 3, gtimer());
                    K5_MARK(j, 4, gtimer());
                    ++g;
                    continue;
                }
                const int nk = nk_of(op);
                for (int k = 0; k < nk; ++k, ++g) {
                    const int s = g % kFStages;
                    mbar_wait(&full_bar[s], (g / kFStages) & 1);
                    tc_fence_after();
                    if (k == 0) K5_MARK(j, 3, gtimer());
                    uint8_t* st = smem + static_cast<size_t>(s) * kFStage;
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        umma_f16(acc, umma_desc_sw128(st, kk * 32), umma_desc_sw128(st + kFTile, kk * 32), idesc,
                                 (k | kk) ? 1u : 0u);
                    umma_commit(&empty_bar[s]);
                }
                umma_commit(&tfull_bar[b]);
                K5_MARK(j, 4, gtimer());
            }
        }
    } else {
        // ---------------- epilogue (16 warps): TMEM lane quarter q = warp & 3, column group gp = warp >> 2.
        const int q = warp & 3, gp = warp >> 2, ht = tid & 127, r = q * 32 + lane;
        const uint32_t gbar = 4u + static_cast<uint32_t>(gp);
        auto group_sync = [&] { asm volatile("bar.sync %0, 128;\n" ::"r"(gbar) : "memory"); };
        auto epi_sync = [&] { asm volatile("bar.sync 3, %0;\n" ::"r"(kFEpiWarps * 32) : "memory"); };
        uint8_t* box = boxes + gp * 8192;
        const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
        auto box_chunk = [&](int u) { return box + r * 64 + ((u ^ ((r >> 1) & 3)) << 4); };  // SWIZZLE_64B row r
        int g = 0, na = 0, e = 0, nln = 0;
        for (int j = 0;; ++j) {
            const uint32_t it = take(j);
            __syncwarp();
            if (lane == 0) release(j);
            const uint32_t op = it_op(it);
            if (op == kOpEnd) break;
            const int l = it_l(it), m = it_m(it), n = it_n(it), m0 = m * kFSeq;
            const uint64_t lo = a.stride * static_cast<uint64_t>(l);
            const int b = j & 1, tpar = (j >> 1) & 1;
            const uint32_t acc = tmem + static_cast<uint32_t>(b * 256);
            if (op == kOpAtt) {
                // ---- attention of (row block m, head n): softmax over S in TMEM, P V, ctx.
                const int s = g % kFStages;
                uint8_t* st = smem + static_cast<size_t>(s) * kFStage;
                float* red_max = reinterpret_cast<float*>(boxes);  // [4 groups][128 rows]
                float* red_sum = red_max + 512;
                if (ht == 0) bulk_wait_group_read<0>();  // the staging boxes are free of TMA store reads
                mbar_wait(&tfull_bar[b], tpar);
                tc_fence_after();
                if (tid == 0) K5_MARK(j, 5, gtimer());
                float sv[32];
                tmem_ld_32x32b_x32(acc + static_cast<uint32_t>(gp * 32) + lane_off, sv);
                float mx = sv[0];
#pragma unroll
                for (int i = 1; i < 32; ++i) mx = fmaxf(mx, sv[i]);
                epi_sync();
                red_max[gp * 128 + r] = mx;
                epi_sync();
                mx = fmaxf(fmaxf(red_max[r], red_max[128 + r]), fmaxf(red_max[256 + r], red_max[384 + r]));
                const float off = mx * kAttnScaleLog2;
                float sum = 0.f;
#pragma unroll
                for (int u = 0; u < 4; ++u) {  // 16-byte chunks of 8 keys: keys 32 gp + 8 u ...
                    uint4 w;
                    __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&w);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const float p0 = ex2_approx(fmaf(sv[u * 8 + 2 * k], kAttnScaleLog2, -off));
                        const float p1 = ex2_approx(fmaf(sv[u * 8 + 2 * k + 1], kAttnScaleLog2, -off));
                        sum += p0 + p1;
                        h2[k] = __floats2bfloat162_rn(p0, p1);
                    }
                    const int c = gp * 4 + u, blk = c >> 3, cc = c & 7;  // P: two K-major SW128 blocks of 64 keys
                    *reinterpret_cast<uint4*>(st + blk * 16384 + r * 128 + ((cc ^ (r & 7)) << 4)) = w;
                }
                red_sum[gp * 128 + r] = sum;
                fence_proxy_async_smem();  // P (generic-proxy writes) -> the P V MMA reads
                tc_fence_before();
                epi_sync();
                if (tid == 0) {
                    tc_fence_after();
                    constexpr uint32_t idesc_o = umma_idesc<128, 64, 1>() | (1u << 16);  // B (V) MN-major
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk)
                        umma_f16(acc + 128, umma_desc_sw128(st + (kk >> 2) * 16384, (kk & 3) * 32),
                                 umma_desc_sw128(st + 2 * kFTile, kk * 2048), idesc_o, kk ? 1u : 0u);
                    umma_commit(&empty_bar[s]);
                    umma_commit(&o_bar);
                }
                mbar_wait(&o_bar, na & 1);
                tc_fence_after();
                const float inv = 1.0f / (red_sum[r] + red_sum[128 + r] + red_sum[256 + r] + red_sum[384 + r]);
                float ov[16];
                tmem_ld_32x32b_x16(acc + 128 + static_cast<uint32_t>(gp * 16) + lane_off, ov);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty_bar[b]);
                uint4 o[2];
                __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(o);
#pragma unroll
                for (int k = 0; k < 8; ++k) o2[k] = __floats2bfloat162_rn(ov[2 * k] * inv, ov[2 * k + 1] * inv);
                uint4* dst = reinterpret_cast<uint4*>(a.ctx + static_cast<size_t>(m0 + r) * kFD + n * 64 + gp * 16);
                dst[0] = o[0];
                dst[1] = o[1];
                epi_sync();
                if (tid == 0) {  // the row block's last head makes its O triple ready
                    __threadfence();
                    if (atom_acq_rel_gpu_add(counter(l, m, kOpAtt), 1) == kFHeads - 1) push(flow_item(kOpO, l, m, 0), 1);
                    K5_MARK(j, 6, gtimer());
                }
                ++g;
                ++na;
                continue;
            }
            // ---- GEMM tile epilogue: bias (+ GELU | + residual [+ LayerNorm]), bf16, TMA stores.
            const bool resid = op == kOpO || op == kOpF2;
            const uint64_t boff = lo + (op == kOpQkv ? a.l0.bqkv : op == kOpO ? a.l0.bo : op == kOpF1 ? a.l0.b1 : a.l0.b2);
            const int n0 = n * 256;
            epi_sync();  // the previous item's reads of bias_s / the boxes' scratch are done
            if (tid < 256) bias_s[tid] = *reinterpret_cast<const float*>(translate(a.arena, pt, boff + 4ull * (n0 + tid)));
            epi_sync();
            const CUtensorMap* ym = op == kOpQkv ? &mp.y_qkv : &mp.y_f;
            const CUtensorMap* rm = op == kOpF2 ? &mp.r_h : l == 0 ? &mp.r_in : &mp.r_x;
            const int rrow = (op == kOpO && l > 0) ? (l - 1) * a.xstride + m0 : m0;
            if (resid) {
                // The first chunk's residual box is loaded before the accumulator is ready, and the
                // LayerNorm's gamma / beta lines are pulled into L1 while the MMAs run.
                if (ht == 0) {
                    fence_proxy_async_global();  // residual rows written by other CTAs
                    bulk_wait_group_read<0>();   // this group's previous store has read the box
                    mbar_arrive_expect_tx(&res_bar[gp], 8192);
                    tma_tile2d_g2s(box, rm, n0 + gp * 32, rrow, &res_bar[gp]);
                }
                if (tid < 16) {
                    const uint64_t lnp = lo + (op == kOpO ? (tid < 8 ? a.l0.ln1_g : a.l0.ln1_b) : (tid < 8 ? a.l0.ln2_g : a.l0.ln2_b));
                    const char* pf = translate(a.arena, pt, lnp + 4ull * n0 + 128ull * (tid & 7));
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(pf));
                }
            }
            mbar_wait(&tfull_bar[b], tpar);
            tc_fence_after();
            if (tid == 0) K5_MARK(j, 5, gtimer());
            float st_n = 0.f, st_mean = 0.f, st_m2 = 0.f;  // resid: this row's (count, mean, M2) over its chunks
            uint32_t hold[2][16];                            // resid: the pre-LN bf16 pairs of both chunks
#pragma unroll
            for (int ci = 0; ci < 2; ++ci) {
                const int c = gp + 4 * ci;
                if (!resid || ci == 1) {
                    if (ht == 0) bulk_wait_group_read<0>();  // this group's previous store has read the box
                    group_sync();                            // (resid: every row read the first residual chunk)
                }
                if (resid && ci == 1 && ht == 0) {
                    mbar_arrive_expect_tx(&res_bar[gp], 8192);
                    tma_tile2d_g2s(box, rm, n0 + c * 32, rrow, &res_bar[gp]);
                }
                float v[32];
                tmem_ld_32x32b_x32(acc + static_cast<uint32_t>(c * 32) + lane_off, v);
                if (ci == 1) {  // the accumulator is free for item j + 2
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty_bar[b]);
                }
                const float* bc = bias_s + c * 32;
                if (resid) {
                    // t = bf16(acc + bias + resid) stays in registers; its row statistics feed the
                    // LayerNorm (the values as the LayerNorm reads them).
                    mbar_wait(&res_bar[gp], e & 1);
                    ++e;
                    float sm = 0.f;
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const uint4 w = *reinterpret_cast<const uint4*>(box_chunk(u));
                        const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const int i = u * 8 + 2 * k;
                            const float2 f2 = __bfloat1622float2(h2[k]);
                            const __nv_bfloat162 x2 = __floats2bfloat162_rn(v[i] + bc[i] + f2.x, v[i + 1] + bc[i + 1] + f2.y);
                            hold[ci][u * 4 + k] = *reinterpret_cast<const uint32_t*>(&x2);
                            const float2 xf = __bfloat1622float2(x2);
                            v[i] = xf.x, v[i + 1] = xf.y;
                            sm += xf.x + xf.y;
                        }
                    }
                    const float mc = sm * (1.f / 32.f);
                    float mc2 = 0.f;
#pragma unroll
                    for (int k = 0; k < 32; ++k) mc2 = fmaf(v[k] - mc, v[k] - mc, mc2);
                    if (ci == 0)
                        st_n = 32.f, st_mean = mc, st_m2 = mc2;
                    else
                        chan_combine(st_n, st_mean, st_m2, 32.f, mc, mc2);
                    continue;
                }
                uint4 out[4];
                __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(out);
                if (op == kOpF1) {
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        const float2 gv = gelu2(make_float2(v[2 * k] + bc[2 * k], v[2 * k + 1] + bc[2 * k + 1]));
                        o2[k] = __floats2bfloat162_rn(gv.x, gv.y);
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < 16; ++k) o2[k] = __floats2bfloat162_rn(v[2 * k] + bc[2 * k], v[2 * k + 1] + bc[2 * k + 1]);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) *reinterpret_cast<uint4*>(box_chunk(u)) = out[u];
                fence_proxy_async_smem();  // generic-proxy writes -> the TMA store reads
                group_sync();
                if (ht == 0) {
                    tma_tile2d_s2g(ym, n0 + c * 32, m0, box);
                    bulk_commit_group();
                }
            }
            g += nk_of(op);
            if (!resid) {
                // ---- publish: this group's stores complete, then the row block's counter.
                if (ht == 0) {
                    bulk_wait_group<0>();
                    fence_proxy_async_global();
                }
                epi_sync();
                if (tid == 0) {  // the row block's last QKV (FFN1) tile makes its heads (FFN2 triple) ready
                    __threadfence();
                    const bool qkv = op == kOpQkv;
                    if (atom_acq_rel_gpu_add(counter(l, m, op), 1) == (qkv ? 9u : static_cast<uint32_t>(nf1)) - 1u)
                        push(qkv ? flow_item(kOpAtt, l, m, 0) : flow_item(kOpF2, l, m, 0), qkv ? 4 : 1);
                    K5_MARK(j, 6, gtimer());
                }
                continue;
            }
            // ---- residual tile + LayerNorm. The row block's three column tiles are this cluster's
            // three CTAs: each publishes its per-row (mean, M2) in global memory and signals its
            // siblings (cluster-scope release on their mbarrier; two barriers alternate so a fast
            // sibling's next statistics never land in a phase still being waited on).
            const bool ln1 = op == kOpO;
            float2* const stats = a.stats + ((static_cast<size_t>(l) * a.M + m) * 2 + (ln1 ? 0 : 1)) * 3 * 128;
            float2* part = reinterpret_cast<float2*>(boxes);  // [4 groups][128 rows]
            if (ht == 0) bulk_wait_group_read<0>();
            epi_sync();  // residual boxes read, previous stores read: the boxes are scratch
            part[gp * 128 + r] = make_float2(st_mean, st_m2);
            epi_sync();
            if (gp == 0) {
#pragma unroll
                for (int k = 1; k < 4; ++k) {
                    const float2 p = part[k * 128 + r];
                    chan_combine(st_n, st_mean, st_m2, 64.f, p.x, p.y);
                }
                stats[rank * 128 + r] = make_float2(st_mean, st_m2);
            }
            epi_sync();
            const int sb = nln & 1;
            if (tid == 0) {
                fence_acq_rel_cluster();
                for (uint32_t rr = 0; rr < kFCluster; ++rr) mbar_arrive_remote(&sib_bar[sb], rr);
            }
            mbar_wait_cluster(&sib_bar[sb], (nln >> 1) & 1);
            ++nln;
            float mean, rstd;
            {
                float2 p = __ldcg(stats + r);
                float cnt = 256.f;
                mean = p.x;
                float m2 = p.y;
#pragma unroll
                for (int k = 1; k < kFCluster; ++k) {
                    p = __ldcg(stats + k * 128 + r);
                    chan_combine(cnt, mean, m2, 256.f, p.x, p.y);
                }
                rstd = rsqrtf(m2 * (1.f / kFD) + 1e-12f);
            }
            if (tid == 0) K5_MARK(j, 7, gtimer());
            const uint64_t go = lo + (ln1 ? a.l0.ln1_g : a.l0.ln2_g), bo = lo + (ln1 ? a.l0.ln1_b : a.l0.ln2_b);
            const CUtensorMap* lm = ln1 ? &mp.y_h : &mp.y_x;
            const int lrow = (ln1 ? 0 : l * a.xstride) + m0;
#pragma unroll
            for (int ci = 0; ci < 2; ++ci) {
                const int c = gp + 4 * ci;
                if (ci == 1) {
                    if (ht == 0) bulk_wait_group_read<0>();
                    group_sync();
                }
                const float4* gam = reinterpret_cast<const float4*>(translate(a.arena, pt, go + 4ull * (n0 + c * 32)));
                const float4* bet = reinterpret_cast<const float4*>(translate(a.arena, pt, bo + 4ull * (n0 + c * 32)));
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float4 g0 = __ldg(gam + 2 * u), g1 = __ldg(gam + 2 * u + 1);
                    const float4 b0 = __ldg(bet + 2 * u), b1 = __ldg(bet + 2 * u + 1);
                    const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
                    const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
                    uint4 o;
                    uint32_t* o32 = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint32_t pr = hold[ci][u * 4 + k];
                        const float2 x = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pr));
                        const __nv_bfloat162 y2 = __floats2bfloat162_rn((x.x - mean) * rstd * gg[2 * k] + bb[2 * k],
                                                                        (x.y - mean) * rstd * gg[2 * k + 1] + bb[2 * k + 1]);
                        o32[k] = *reinterpret_cast<const uint32_t*>(&y2);
                    }
                    *reinterpret_cast<uint4*>(box_chunk(u)) = o;
                }
                fence_proxy_async_smem();
                group_sync();
                if (ht == 0) {
                    tma_tile2d_s2g(lm, n0 + c * 32, lrow, box);
                    bulk_commit_group();
                }
            }
            if (ht == 0) {
                bulk_wait_group<0>();
                fence_proxy_async_global();
            }
            epi_sync();
            if (tid == 0) {  // LN1 makes the row block's FFN1 triples ready, LN2 the next layer's QKV triples
                __threadfence();
                if (atom_acq_rel_gpu_add(counter(l, m, op), 1) == kFCluster - 1) {
                    if (ln1)
                        push(flow_item(kOpF1, l, m, 0), nf1 / 3);
                    else if (l + 1 < a.L)
                        push(flow_item(kOpQkv, l + 1, m, 0), 3);
                }
                K5_MARK(j, 6, gtimer());
            }
        }
        if (ht == 0) bulk_wait_group<0>();
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // no remote arrive may target an exited CTA
    tc_fence_after();
    if (warp == kFMmaWarp) tmem_dealloc<512>(tmem);
}

// ------------------------------------------------------------------ host

bool encode_or_throw(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint32_t box_inner,
                     CUtensorMapSwizzle sw, const char* what) {
    if (!encode_tensor_map_2d(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, inner, outer, inner * 2, box_inner, 128,
                              sw))
        throw CudaError(std::string("cuTensorMapEncodeTiled failed (encoder flow: ") + what + ")");
    return true;
}

// Co-resident 3-CTA clusters of the kernel on this device (every CTA must be resident:
// CTAs of one cluster wait for each other). Cached per device.
int flow_clusters() {
    static std::mutex mu;
    static std::map<int, int> cache;
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(dev);
    if (it != cache.end()) return it->second;
    ensure_max_dynamic_smem(reinterpret_cast<const void*>(encoder_flow_kernel), static_cast<int>(kFSmem));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(kFCluster * 64);
    cfg.blockDim = dim3(kFThreads);
    cfg.dynamicSmemBytes = kFSmem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kFCluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    GFX_CUDA(cudaOccupancyMaxActiveClusters(&n, encoder_flow_kernel, &cfg));
    n = std::min(n, device_sm_count(dev) / static_cast<int>(kFCluster));
    if (n < 1) throw std::runtime_error("encoder flow: no 3-CTA cluster fits on this device");
    cache[dev] = n;
    return n;
}

}  // namespace

bool bert_flow_supported(const BertLayout& lay, int batch) {
    if (lay.d != kFD || lay.heads != kFHeads || lay.seq != kFSeq || lay.ffn % 768 || lay.L < 1 || lay.L > 31) return false;
    if (batch < 1 || batch > 4095) return false;
    // Layer l's parameters must sit at layer 0's offsets + l * stride (bert_layout's periodic blob).
    const uint64_t stride = lay.L > 1 ? lay.layer[1].wqkv - lay.layer[0].wqkv : 0;
    for (int l = 0; l < lay.L; ++l) {
        const BertLayerOffsets& o = lay.layer[static_cast<size_t>(l)];
        const BertLayerOffsets& z = lay.layer[0];
        const uint64_t d = stride * static_cast<uint64_t>(l);
        if (o.wqkv != z.wqkv + d || o.bqkv != z.bqkv + d || o.wo != z.wo + d || o.bo != z.bo + d ||
            o.ln1_g != z.ln1_g + d || o.ln1_b != z.ln1_b + d || o.w1 != z.w1 + d || o.b1 != z.b1 + d ||
            o.w2 != z.w2 + d || o.b2 != z.b2 + d || o.ln2_g != z.ln2_g + d || o.ln2_b != z.ln2_b + d)
            return false;
    }
    return true;
}

int bert_encoder_flow(const char* arena, const PageTable& pt, const BertLayout& lay, int batch,
                      const __nv_bfloat16* in, __nv_bfloat16* xout, int xstride, BertWorkspace& ws, cudaStream_t s) {
    if (!bert_flow_supported(lay, batch)) throw std::runtime_error("encoder flow: unsupported BERT shape");
    const int T = batch * kFSeq, M = batch, L = lay.L, F = lay.ffn;
    const int clusters = flow_clusters();
    const int ctas = clusters * static_cast<int>(kFCluster);
    // Queue slots, counters and LayerNorm statistics (sized per shape in the workspace).
    // Cluster items per (layer, row block): 3 QKV, 4 attention, 1 O, ffn / 768 FFN1, 1 FFN2.
    const int n_items = L * M * (3 + 4 + 1 + F / 768 + 1);
    if (ws.flow_L != L || ws.flow_M != M || ws.flow_F != F) {
        if (ws.flow_cnt) GFX_CUDA(cudaFree(ws.flow_cnt));
        if (ws.flow_stats) GFX_CUDA(cudaFree(ws.flow_stats));
        ws.flow_cnt = nullptr;
        ws.flow_stats = nullptr;
        // One allocation: [L][M][kCSlots] counters, head, tail, then n_items queue slots.
        ws.flow_cnt_words = static_cast<size_t>(L) * M * kCSlots + 2 + static_cast<size_t>(n_items);
        GFX_CUDA(cudaMalloc(&ws.flow_cnt, ws.flow_cnt_words * 4));
        GFX_CUDA(cudaMalloc(&ws.flow_stats, static_cast<size_t>(L) * M * 2 * 3 * 128 * sizeof(float2)));
        ws.flow_L = L, ws.flow_M = M, ws.flow_F = F, ws.flow_ctas = ctas;
    }
    FlowMaps mp;
    const CUtensorMapSwizzle k128 = CU_TENSOR_MAP_SWIZZLE_128B, k64 = CU_TENSOR_MAP_SWIZZLE_64B;
    const uint64_t xrows = static_cast<uint64_t>(T) + static_cast<uint64_t>(xstride) * (L - 1);
    encode_or_throw(&mp.a_in, in, kFD, T, 64, k128, "input");
    encode_or_throw(&mp.a_x, xout, kFD, xrows, 64, k128, "layer input");
    encode_or_throw(&mp.a_ctx, ws.ctx, kFD, T, 64, k128, "ctx");
    encode_or_throw(&mp.a_h, ws.h, kFD, T, 64, k128, "h");
    encode_or_throw(&mp.a_f, ws.f, F, T, 64, k128, "f");
    encode_or_throw(&mp.qkv, ws.qkv, 3 * kFD, T, 64, k128, "qkv");
    encode_or_throw(&mp.y_qkv, ws.qkv, 3 * kFD, T, 32, k64, "qkv out");
    encode_or_throw(&mp.y_f, ws.f, F, T, 32, k64, "f out");
    encode_or_throw(&mp.y_h, ws.h, kFD, T, 32, k64, "h out");
    encode_or_throw(&mp.y_x, xout, kFD, xrows, 32, k64, "layer out");
    encode_or_throw(&mp.r_in, in, kFD, T, 32, k64, "input resid");
    encode_or_throw(&mp.r_x, xout, kFD, xrows, 32, k64, "layer input resid");
    encode_or_throw(&mp.r_h, ws.h, kFD, T, 32, k64, "h resid");
    FlowArgs fa{};
    fa.arena = arena;
    fa.l0 = lay.layer[0];
    fa.stride = L > 1 ? lay.layer[1].wqkv - lay.layer[0].wqkv : 0;
    fa.cnt = ws.flow_cnt;
    fa.slots = ws.flow_cnt + static_cast<size_t>(L) * M * kCSlots + 2;
    fa.n_items = n_items;
    fa.n_first = 3 * M;
    fa.ctx = ws.ctx;
    fa.h = ws.h;
    fa.xout = xout;
    fa.stats = static_cast<float2*>(ws.flow_stats);
    fa.M = M;
    fa.L = L;
    fa.ffn = F;
    fa.xstride = xstride;
    fa.pt = pt;
    fa.trace = nullptr;
#ifdef GFX_K5_DEBUG
    static int forwards = 0;
    const char* trace_path = std::getenv("GFX_K5_TRACE");
    const bool tracing = trace_path && ++forwards == 8;  // a warm forward
    const size_t trace_words = static_cast<size_t>(ctas) * kFTraceItems * 8;
    if (tracing) {
        GFX_CUDA(cudaMalloc(&fa.trace, trace_words * 8));
        GFX_CUDA(cudaMemsetAsync(fa.trace, 0, trace_words * 8, s));
    }
#endif
    GFX_CUDA(cudaMemsetAsync(ws.flow_cnt, 0, ws.flow_cnt_words * 4, s));
    ensure_max_dynamic_smem(reinterpret_cast<const void*>(encoder_flow_kernel), static_cast<int>(kFSmem));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(ctas));
    cfg.blockDim = dim3(kFThreads);
    cfg.dynamicSmemBytes = kFSmem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kFCluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    GFX_CUDA(cudaLaunchKernelEx(&cfg, encoder_flow_kernel, mp, fa));
#ifdef GFX_K5_DEBUG
    if (tracing) {
        std::vector<unsigned long long> v(trace_words);
        GFX_CUDA(cudaStreamSynchronize(s));
        GFX_CUDA(cudaMemcpy(v.data(), fa.trace, trace_words * 8, cudaMemcpyDeviceToHost));
        GFX_CUDA(cudaFree(fa.trace));
        if (FILE* f = std::fopen(trace_path, "wb")) {
            const int hdr[4] = {ctas, kFTraceItems, M, L};
            std::fwrite(hdr, sizeof hdr, 1, f);
            std::fwrite(v.data(), 8, v.size(), f);
            std::fclose(f);
        }
    }
#endif
    return 1;
}

}  // namespace gfx
