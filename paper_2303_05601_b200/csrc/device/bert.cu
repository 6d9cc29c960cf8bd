// C5: BERT-base-style encoder (post-LN, bf16 activations, fp32 accumulation)
// served from the paged HBM arena.
//
// Kernels:
//   K2 gemm_bf16_kernel   Y[T x N] = epi(X[T x K] . W^T + b) on tcgen05
//                         (kind::f16, bf16 -> fp32 in TMEM), persistent 128 x 256
//                         tiles, X via a 2-D TMA tensor map, W tiles
//                         (pre-swizzled 16 KB) via 1-D bulk TMA from the arena,
//                         double-buffered TMEM accumulators; fused bias / GELU /
//                         residual epilogue (16 warps) through TMA stores; bf16 out.
//                         Tensor-core bound. Opt-in 2-SM (cta_group::2) variant.
//   K3 attention_tc_kernel softmax(Q K^T / sqrt(64)) V per (sequence, head, query tile),
//                         sequences of 128-512 tokens: one CTA of 8 warps, both
//                         products on tcgen05 (V read MN-major), exact softmax from
//                         TMEM, optional padding mask (valid length per sequence).
//   K4 layernorm_kernel   one warp per token row, 16-byte vector loads, fp32
//                         two-pass statistics; HBM bound.
//   pooler_kernel         tanh(Wp . x_cls + bp) per sequence, fp32 out.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>
#include <map>
#include <mutex>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <stdexcept>

#include "bert.cuh"
#include "bert_dev.cuh"
#include "mlp.cuh"
#include "sm100.cuh"

namespace gfx {

namespace {

using namespace gfx::sm100;

using namespace gfx::bertdev;

#ifdef GFX_K2_DEBUG
// Per-CTA phase marks (debug build only): 0 start, 1 setup, 2 first A issued;
// tile i < 4: 3 + 4i first stage landed (MMA thread), 4 + 4i last MMA issued,
// 5 + 4i epilogue saw the accumulator, 6 + 4i epilogue done; 19 end.
#define K2_MARK(i)                                                                   \
    do {                                                                             \
        if (a.dbg) {                                                                 \
            unsigned long long t_;                                                   \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                   \
            a.dbg[blockIdx.x * 24 + (i)] = t_;                                       \
        }                                                                            \
    } while (0)
// Per-launch span (debug build): [0] earliest CTA start, [1] latest CTA end
// (%globaltimer ns) of one kernel launch; bert_forward prints the forward's
// kernel timeline from these (gaps between launches included).
#define K2_SPAN_BEGIN(tr)                                                            \
    do {                                                                             \
        if ((tr) && threadIdx.x == 0) {                                              \
            unsigned long long t_;                                                   \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                   \
            atomicMin((tr), t_);                                                     \
        }                                                                            \
    } while (0)
#define K2_SPAN_END(tr)                                                              \
    do {                                                                             \
        if ((tr) && threadIdx.x == 0) {                                              \
            unsigned long long t_;                                                   \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                   \
            atomicMax((tr) + 1, t_);                                                 \
        }                                                                            \
    } while (0)
#else
#define K2_MARK(i) \
    do {           \
    } while (0)
#define K2_SPAN_BEGIN(tr) \
    do {                  \
    } while (0)
#define K2_SPAN_END(tr) \
    do {                \
    } while (0)
#endif

// Debug build: kernel spans of one traced forward (bert_forward's 10th call).
#ifdef GFX_K2_DEBUG
struct SpanTrace {
    unsigned long long* buf = nullptr;  // [kMax][2]
    std::vector<const char*> names;
    bool on = false;
    static constexpr int kMax = 256;
};
SpanTrace g_span;
unsigned long long* next_span(const char* name) {
    if (!g_span.on || static_cast<int>(g_span.names.size()) >= SpanTrace::kMax) return nullptr;
    g_span.names.push_back(name);
    return g_span.buf + 2 * (g_span.names.size() - 1);
}
#else
inline unsigned long long* next_span(const char*) { return nullptr; }
#endif

// ------------------------------------------------------------------ K2 GEMM
// Persistent: one CTA per SM loops over 128 x kBN output tiles; the TMEM holds
// two accumulators so the epilogue of tile i overlaps the MMAs of tile i+1.

// Warps: 0-15 epilogue, 16 A producer, 17 MMA issuer, 18-19 B producers (the
// latency-critical roles at the highest ids, which the SMSP arbiter prefers,
// B300_MICROARCH.md; measured within noise of producers/MMA at ids 0/1/18/19).
// A tile's MMA phase runs ~4.2 µs alone but ~4.8 µs (bias epilogue) to ~6 µs
// (GELU epilogue) while the previous tile's epilogue drains the other TMEM
// buffer (make K2_DEBUG=1 per-tile timeline, profiles/r2_k2_bert.md).
constexpr int kGM = 128, kGK = 64, kGThreads = 640;
constexpr int kGEpiWarps = 16, kGAWarp = 16, kGMmaWarp = 17, kGBWarp0 = 18;
constexpr uint32_t kGATile = 128 * 128;  // A: 128 rows x 64 bf16 (16 KB)
constexpr uint32_t kGSmem = 192 * 1024;  // stage ring budget

// kEpiResidLN: bias + residual + the post-LN LayerNorm of the whole d-wide row,
// fused (K4 disappears from the forward). The row's d / 256 column tiles (3 for
// BERT-base, 4 for BERT-large) are computed by the CTAs of one cluster; each
// CTA reduces its tile's per-row (mean, M2) and sends it to every CTA of the
// cluster by st.async into their shared
// memory (DSMEM, completing a tx-counted mbarrier), so the statistics never
// touch global memory and no CTA waits on a flag in L2. One tile per CTA (the
// host falls back to kEpiResid + layernorm_kernel when the row blocks exceed
// the resident clusters).
enum Epi : int { kEpiBias = 0, kEpiGelu = 1, kEpiResid = 2, kEpiResidLN = 3 };

struct GemmArgs {
    unsigned long long* dbg;      // GFX_K2_DEBUG builds: [grid][24] %globaltimer marks, else nullptr
    unsigned long long* span;     // GFX_K2_DEBUG builds: this launch's [start, end] span, else nullptr
    const char* arena;
    uint64_t w_off, b_off;        // weight tiles, fp32 bias
    uint64_t g_off, be_off;       // kEpiResidLN: LayerNorm gamma / beta (fp32)
    __nv_bfloat16* y;             // [T x N]
    const __nv_bfloat16* resid;   // [T x N] (kEpiResid, kEpiResidLN)
    int T, K, N;
    PageTable pt;
};

// kPair: 2-SM tcgen05 (cta_group::2). A CTA pair (cluster of 2) computes a
// 256 x kBN tile: each CTA stages its own 128 rows of A and its half of the
// kBN rows of B (32 KB per K stage instead of 48 KB), the even CTA issues one
// M = 256 MMA per K slice that reads both CTAs' smem, and each CTA's TMEM holds
// its own 128 rows of D for its own epilogue. Halving the per-CTA stage is the
// point: 6 stages (1.6 µs of MMA work) instead of 4 (1.07 µs) cover the TMA
// latency under load, which bounded the single-CTA MMA phase at ~78 % of
// issue rate (multicasting B alone did not help).
// Barriers: every operand load of either CTA is a .cta_group::2 tensor TMA
// whose bytes complete the EVEN CTA's full barrier (the even CTA's producers
// expect both halves), so the issuer waits on one barrier — an earlier version
// relayed the odd CTA's "landed" by a remote arrive, one stage at a time, and
// that relay set a 0.7 µs stage cadence; weights come through a tensor map
// over the whole arena (pre-swizzled tiles, SWIZZLE_NONE boxes); the issuer's
// commits multicast to both CTAs' empty / tfull barriers; both epilogues arrive
// on the even CTA's tempty.
template <int kEpi, int kBN, bool kPair>
__global__ void __launch_bounds__(kGThreads, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_y,
                     const __grid_constant__ CUtensorMap tmap_r, const __grid_constant__ CUtensorMap tmap_w,
                     const __grid_constant__ GemmArgs a) {
    constexpr uint32_t kBBytes = (kPair ? kBN / 2 : kBN) * 128;  // B: this CTA's rows x 64 bf16
    constexpr uint32_t kStage = kGATile + kBBytes;
    constexpr int kStages = static_cast<int>(kGSmem / kStage);
    constexpr uint32_t kTmemCols = 2 * kBN <= 256 ? 256 : 512;
    constexpr bool kLN = kEpi == kEpiResidLN;
    constexpr bool kCluster = kPair || kLN;
    static_assert(!kLN || (kBN == 256 && !kPair), "the fused LayerNorm runs 128 x 256 single-CTA tiles");
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared window
    __shared__ __align__(8) uint64_t full_bar[kStages], empty_bar[kStages], tfull_bar[2], tempty_bar[2], res_bar[4];
    __shared__ __align__(8) uint64_t stat_bar;  // kLN: the three CTAs' row statistics landed
    __shared__ uint32_t tmem_s;
    __shared__ float bias_s[kBN];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) K2_MARK(0);
    K2_SPAN_BEGIN(a.span);
    const int n_tiles = a.N / kBN, m_tiles = a.T / kGM;
    // Tile sequence of this CTA: single -> tiles t = blockIdx.x (step grid);
    // pair -> pair tiles t = cluster id (step clusters), rows 2*(t / n) + rank.
    const uint32_t rank = kPair ? cluster_ctarank() : 0u;
    const int t_first = kPair ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
    const int t_step = kPair ? static_cast<int>(gridDim.x >> 1) : static_cast<int>(gridDim.x);
    const int tiles = kPair ? n_tiles * (m_tiles / 2) : n_tiles * m_tiles;
    const int nk = a.K / kGK;
    auto tile_m0 = [&](int t) { return kPair ? ((t / n_tiles) * 2 + static_cast<int>(rank)) * kGM : (t / n_tiles) * kGM; };
    const int ktiles_row = a.K / kGK;  // blob weight tiles per 128 rows

    // The page table is read straight from the __grid_constant__ parameter (up to
    // GFX_MAX_PAGES entries, 4 KB: no room for a shared-memory copy).
    const uint32_t* const pt = a.pt.page;
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            // One arrive.expect_tx per producer warp: A (warp 0) and each B tile
            // (warps 10, 11). TMA requests of one issuing thread are served one
            // after another (~500 cycles per 16 KB, tools/tma_rate.cu), so the
            // stage's three 16 KB loads come from three threads in parallel.
            mbar_init(&full_bar[s], 1 + kBBytes / kGATile);
            mbar_init(&empty_bar[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull_bar[b], 1);
            mbar_init(&tempty_bar[b], kPair ? 2 * kGEpiWarps : kGEpiWarps);  // epilogue warps (of both CTAs in pair mode)
        }
        for (int g = 0; g < 4; ++g) mbar_init(&res_bar[g], 1);
        if (kLN) mbar_init(&stat_bar, 1);
        mbar_fence_init();
        // n_tiles senders x 128 rows x (mean, M2); remote bytes may land before
        // this CTA's epilogue runs, never before the cluster_sync below.
        if (kLN) mbar_arrive_expect_tx(&stat_bar, static_cast<uint32_t>(n_tiles) * 128 * 8);
        tma_prefetch_desc(&tmap_x);
        tma_prefetch_desc(&tmap_y);
        if (kEpi == kEpiResid || kLN) tma_prefetch_desc(&tmap_r);
        if (kPair) tma_prefetch_desc(&tmap_w);
    }
    // kLN: the residual tile (8 boxes of 128 rows x 32 columns, SWIZZLE_64B) goes
    // into the two ring stages after the tile's last K stage, loaded as soon as
    // the MMAs free them; the normalised output is written over it in place.
    auto ln_box = [&](int c) {
        return smem + static_cast<size_t>((nk + c / 6) % kStages) * kStage + static_cast<size_t>(c % 6) * 8192;
    };
    if (warp == kGMmaWarp) {
        if (kPair)
            tmem_alloc_pair<kTmemCols>(&tmem_s);
        else
            tmem_alloc<kTmemCols>(&tmem_s);
    }
    tc_fence_before();
    __syncthreads();
    if (kCluster) cluster_sync();  // the peers' barriers exist before any remote arrive / st.async reaches them
    tc_fence_after();
    const uint32_t tmem = tmem_s;
    if (tid == 0) K2_MARK(1);

    constexpr int kBTiles = static_cast<int>(kBBytes / kGATile);  // B tiles per stage and CTA
    if (warp == kGAWarp || warp >= kGBWarp0) {
        // Producers: one continuous stage ring across this CTA's tiles. Warp 0
        // loads A (X rows, 2-D tensor map, after the previous kernel: PDL);
        // warp kGBWarp0 + h loads B tile h (weights: pair -> this CTA's half of
        // the kBN rows), independent of the previous kernel.
        const int h = warp - kGBWarp0;
        if (lane == 0 && h < kBTiles) {
            int g = 0;
            if (warp == kGAWarp) {
                pdl_wait();
                K2_MARK(2);
            }
            for (int t = t_first; t < tiles; t += t_step) {
                const int m0 = tile_m0(t), nb = t % n_tiles;
                for (int k = 0; k < nk; ++k, ++g) {
                    const int s = g % kStages;
                    if (g >= kStages) mbar_wait(&empty_bar[s], ((g / kStages) & 1) ^ 1);
                    uint8_t* st = smem + static_cast<size_t>(s) * kStage;
                    if (kPair) {
                        // Both CTAs load their halves; only the even CTA's barrier counts them.
                        if (rank == 0) mbar_arrive_expect_tx(&full_bar[s], 2 * kGATile);
                        if (warp == kGAWarp) {
                            tma_tile2d_g2s_pair(st, &tmap_x, k * kGK, m0, &full_bar[s]);
                        } else {
                            const int bt = nb * (kBN / 128) + static_cast<int>(rank) * kBTiles + h;
                            const uint64_t v = a.w_off + (static_cast<uint64_t>(bt) * ktiles_row + k) * kGATile;
                            const uint64_t row = static_cast<uint64_t>(translate(a.arena, pt, v) - a.arena) / 512;
                            tma_tile2d_g2s_pair(st + kGATile + h * kGATile, &tmap_w, 0, static_cast<int>(row), &full_bar[s]);
                        }
                    } else if (warp == kGAWarp) {
                        mbar_arrive_expect_tx(&full_bar[s], kGATile);
                        tma_tile2d_g2s(st, &tmap_x, k * kGK, m0, &full_bar[s]);
                    } else {
                        const int bt = nb * (kBN / 128) + h;
                        const uint64_t v = a.w_off + (static_cast<uint64_t>(bt) * ktiles_row + k) * kGATile;
                        mbar_arrive_expect_tx(&full_bar[s], kGATile);
                        tma_bulk_g2s(st + kGATile + h * kGATile, translate(a.arena, pt, v), kGATile, &full_bar[s]);
                    }
                }
            }
            if (kLN && warp == kGAWarp) {
                // One tile per CTA: stages nk and nk + 1 are free once the MMAs of
                // K stages nk - kStages and nk + 1 - kStages completed.
                // Chunks 0-5 go to the first stage, 6-7 to the second; the epilogue's
                // first pass (chunks 0-3) waits on res_bar[0] only.
                const int m0 = tile_m0(t_first), n0 = (t_first % n_tiles) * kBN;
                if (g >= kStages) mbar_wait(&empty_bar[g % kStages], ((g / kStages) & 1) ^ 1);
                mbar_arrive_expect_tx(&res_bar[0], 4 * 8192);
                for (int c = 0; c < 4; ++c) tma_tile2d_g2s(ln_box(c), &tmap_r, n0 + c * 32, m0, &res_bar[0]);
                mbar_arrive_expect_tx(&res_bar[1], 4 * 8192);
                for (int c = 4; c < 6; ++c) tma_tile2d_g2s(ln_box(c), &tmap_r, n0 + c * 32, m0, &res_bar[1]);
                if (g + 1 >= kStages) mbar_wait(&empty_bar[(g + 1) % kStages], (((g + 1) / kStages) & 1) ^ 1);
                for (int c = 6; c < 8; ++c) tma_tile2d_g2s(ln_box(c), &tmap_r, n0 + c * 32, m0, &res_bar[1]);
            }
        }
    } else if (warp == kGMmaWarp) {
        if (kPair && rank == 1) {
            // Odd CTA of the pair: nothing to issue (its loads complete the even CTA's barrier).
        } else if (lane == 0) {
            constexpr uint32_t idesc = umma_idesc<kPair ? 2 * kGM : kGM, kBN, 1>();  // BF16 x BF16 -> F32
            int g = 0, i = 0;
            for (int t = t_first; t < tiles; t += t_step, ++i) {
                const int b = i & 1;
                if (i >= 2) mbar_wait(&tempty_bar[b], ((i >> 1) & 1) ^ 1);  // epilogue(s) drained tile i-2
                tc_fence_after();
                const uint32_t acc = tmem + static_cast<uint32_t>(b * kBN);
                for (int k = 0; k < nk; ++k, ++g) {
                    const int s = g % kStages;
                    mbar_wait(&full_bar[s], (g / kStages) & 1);
                    tc_fence_after();
                    if (k == 0 && i < 4) K2_MARK(3 + 4 * i);
                    uint8_t* st = smem + static_cast<size_t>(s) * kStage;
#pragma unroll
                    for (int kk = 0; kk < kGK / 16; ++kk) {  // K = 16 bf16 = 32 bytes per MMA
                        const uint64_t ad = umma_desc_sw128(st, kk * 32), bd = umma_desc_sw128(st + kGATile, kk * 32);
                        if (kPair)
                            umma_f16_pair(acc, ad, bd, idesc, (k | kk) ? 1u : 0u);
                        else
                            umma_f16(acc, ad, bd, idesc, (k | kk) ? 1u : 0u);
                    }
                    if (kPair)
                        umma_commit_pair_multicast(&empty_bar[s], 0x3);
                    else
                        umma_commit(&empty_bar[s]);
                }
                if (kPair)
                    umma_commit_pair_multicast(&tfull_bar[b], 0x3);
                else
                    umma_commit(&tfull_bar[b]);
                if (i < 4) K2_MARK(4 + 4 * i);
            }
        }
    } else if constexpr (kLN) {
        // Fused residual + LayerNorm epilogue (one 128 x 256 tile per CTA, the
        // cluster's n_tiles = d / 256 CTAs hold the row's column tiles). Thread = row
        // r (TMEM lane), group gp = column chunks gp and gp + 4 (32 each).
        // t1 = bf16(acc + bias + resid) stays in registers as bf16 pairs; the
        // row's (mean, M2) is reduced over chunks (registers), groups (shared
        // memory) and CTAs (st.async into every CTA of the cluster), then the
        // normalised row overwrites the thread's own residual bytes in the ring
        // and goes out by TMA stores. Bias / gamma / beta and the statistics
        // scratch live in the (otherwise unused) staging-box region.
        const int q = warp & 3, gp = warp >> 2, r = q * 32 + lane, ht = tid & 127;
        const uint32_t gbar = 4u + static_cast<uint32_t>(gp);
        auto group_sync = [&] { asm volatile("bar.sync %0, 128;\n" ::"r"(gbar) : "memory"); };
        auto epi_sync = [&] { asm volatile("bar.sync 3, %0;\n" ::"r"(kGEpiWarps * 32) : "memory"); };
        float* gam_s = reinterpret_cast<float*>(smem + kGSmem);
        float* bet_s = gam_s + kBN;
        float2* part = reinterpret_cast<float2*>(smem + kGSmem + 4096);   // [4 groups][128 rows]
        float2* xbuf = reinterpret_cast<float2*>(smem + kGSmem + 8192);   // [<= 8 CTAs][128 rows]
        const int t = t_first;
        const int m0 = tile_m0(t), n0 = (t % n_tiles) * kBN;
        for (int c = tid; c < kBN; c += kGEpiWarps * 32) {
            bias_s[c] = *reinterpret_cast<const float*>(translate(a.arena, pt, a.b_off + 4ull * (n0 + c)));
            gam_s[c] = *reinterpret_cast<const float*>(translate(a.arena, pt, a.g_off + 4ull * (n0 + c)));
            bet_s[c] = *reinterpret_cast<const float*>(translate(a.arena, pt, a.be_off + 4ull * (n0 + c)));
        }
        epi_sync();
        mbar_wait(&tfull_bar[0], 0);
        tc_fence_after();
        if (tid == 0) K2_MARK(5);
        pdl_trigger();
        uint32_t hold[2][16];
        float cnt = 32.f, mean = 0.f, m2 = 0.f;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int c = gp + 4 * j;
            float v[32];
            tmem_ld_32x32b_x32(tmem + static_cast<uint32_t>(c * 32) + (static_cast<uint32_t>(q * 32) << 16), v);
            mbar_wait(&res_bar[j], 0);
            const uint8_t* box = ln_box(c);
            float s = 0.f;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint4 w = *reinterpret_cast<const uint4*>(box + r * 64 + ((u ^ ((r >> 1) & 3)) << 4));
                const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int e = u * 8 + 2 * k;
                    const float2 f2 = __bfloat1622float2(h2[k]);
                    const __nv_bfloat162 x2 = __floats2bfloat162_rn(v[e] + bias_s[c * 32 + e] + f2.x,
                                                                    v[e + 1] + bias_s[c * 32 + e + 1] + f2.y);
                    hold[j][u * 4 + k] = *reinterpret_cast<const uint32_t*>(&x2);
                    const float2 xf = __bfloat1622float2(x2);
                    v[e] = xf.x;
                    v[e + 1] = xf.y;
                    s += xf.x + xf.y;
                }
            }
            const float mc = s * (1.f / 32.f);
            float mc2 = 0.f;
#pragma unroll
            for (int e = 0; e < 32; ++e) mc2 = fmaf(v[e] - mc, v[e] - mc, mc2);
            if (j == 0) {
                mean = mc;
                m2 = mc2;
            } else {
                chan_combine(cnt, mean, m2, 32.f, mc, mc2);
            }
        }
        part[gp * 128 + r] = make_float2(mean, m2);
        if (tid == 0) K2_MARK(7);
        epi_sync();
        if (gp == 0) {
#pragma unroll
            for (int g = 1; g < 4; ++g) {
                const float2 p = part[g * 128 + r];
                chan_combine(cnt, mean, m2, 64.f, p.x, p.y);
            }
            const uint32_t my = static_cast<uint32_t>(t % n_tiles);
#pragma unroll
            for (uint32_t dst = 0; dst < static_cast<uint32_t>(n_tiles); ++dst)
                st_async_v2f32(mapa_u32(&xbuf[my * 128 + r], dst), mean, m2, mapa_u32(&stat_bar, dst));
        }
        if (tid == 0) K2_MARK(8);
        mbar_wait(&stat_bar, 0);
        if (tid == 0) K2_MARK(9);
        {
            float2 p = xbuf[r];
            float n_r = 256.f;
            mean = p.x;
            m2 = p.y;
            for (int k = 1; k < n_tiles; ++k) {
                p = xbuf[k * 128 + r];
                chan_combine(n_r, mean, m2, 256.f, p.x, p.y);
            }
        }
        const float rstd = rsqrtf(m2 * (1.f / static_cast<float>(a.N)) + 1e-12f);
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int c = gp + 4 * j;
            uint8_t* box = ln_box(c);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                uint4 o;
                uint32_t* o32 = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int e = c * 32 + u * 8 + 2 * k;
                    const uint32_t pr = hold[j][u * 4 + k];
                    const float2 xf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pr));
                    const __nv_bfloat162 y2 = __floats2bfloat162_rn((xf.x - mean) * rstd * gam_s[e] + bet_s[e],
                                                                    (xf.y - mean) * rstd * gam_s[e + 1] + bet_s[e + 1]);
                    o32[k] = *reinterpret_cast<const uint32_t*>(&y2);
                }
                *reinterpret_cast<uint4*>(box + r * 64 + ((u ^ ((r >> 1) & 3)) << 4)) = o;  // this thread's own residual bytes
            }
        }
        fence_proxy_async_smem();
        group_sync();
        if (ht == 0) {
            tma_tile2d_s2g(&tmap_y, n0 + gp * 32, m0, ln_box(gp));
            tma_tile2d_s2g(&tmap_y, n0 + (gp + 4) * 32, m0, ln_box(gp + 4));
            bulk_commit_group();
        }
        if (tid == 0) K2_MARK(10);
        if (ht == 0) bulk_wait_group_read<0>();
        if (tid == 0) K2_MARK(6);
    } else {
        // Epilogue (16 warps): TMEM lane = token row, column = output feature.
        // Four warps per TMEM lane quarter; group gp takes the 32-column chunks
        // c = gp (mod 4) with its own 8 KB staging box (128 x 32 bf16,
        // SWIZZLE_64B image), named barrier and store thread. FFN1's GELU made
        // the epilogue the bottleneck with 8 warps (~7 µs per 128 x 256 tile
        // against ~4 µs of MMAs).
        const int q = warp & 3, gp = warp >> 2, ct = tid, ht = ct & 127;
        const uint32_t gbar = 4u + static_cast<uint32_t>(gp);
        auto group_sync = [&] { asm volatile("bar.sync %0, 128;\n" ::"r"(gbar) : "memory"); };
        uint8_t* box = smem + kGSmem + gp * 8192;
        int i = 0, e = 0;
        for (int t = t_first; t < tiles; t += t_step, ++i) {
            const int m0 = tile_m0(t), n0 = (t % n_tiles) * kBN;
            const int b = i & 1;
            asm volatile("bar.sync 3, %0;\n" ::"r"(kGEpiWarps * 32) : "memory");  // previous tile's bias reads done
            for (int c = ct; c < kBN; c += kGEpiWarps * 32)
                bias_s[c] = *reinterpret_cast<const float*>(translate(a.arena, pt, a.b_off + 4ull * (n0 + c)));
            asm volatile("bar.sync 3, %0;\n" ::"r"(kGEpiWarps * 32) : "memory");
            mbar_wait(&tfull_bar[b], (i >> 1) & 1);
            tc_fence_after();
            if (ct == 0 && i < 4) K2_MARK(5 + 4 * i);
            if (t + t_step >= tiles) pdl_trigger();  // last tile: let the next kernel start
            const int r = q * 32 + lane;
#pragma unroll 1
            for (int c = gp; c < kBN / 32; c += kGEpiWarps / 4, ++e) {
                if (ht == 0) bulk_wait_group_read<0>();  // this group's previous store has read the box
                group_sync();
                if (kEpi == kEpiResid && ht == 0) {
                    mbar_arrive_expect_tx(&res_bar[gp], 8192);
                    tma_tile2d_g2s(box, &tmap_r, n0 + c * 32, m0, &res_bar[gp]);
                }
                float v[32];
                tmem_ld_32x32b_x32(tmem + static_cast<uint32_t>(b * kBN + c * 32) + (static_cast<uint32_t>(q * 32) << 16), v);
                float rs[32];
                if (kEpi == kEpiResid) {
                    mbar_wait(&res_bar[gp], e & 1);
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const uint4 w = *reinterpret_cast<const uint4*>(box + r * 64 + ((u ^ ((r >> 1) & 3)) << 4));
                        const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const float2 f2 = __bfloat1622float2(h2[j]);
                            rs[u * 8 + 2 * j] = f2.x;
                            rs[u * 8 + 2 * j + 1] = f2.y;
                        }
                    }
                }
                uint4 out[4];
                __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(out);
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    float x0 = v[2 * j] + bias_s[c * 32 + 2 * j];
                    float x1 = v[2 * j + 1] + bias_s[c * 32 + 2 * j + 1];
                    if (kEpi == kEpiGelu) {
                        const float2 g = gelu2(make_float2(x0, x1));
                        x0 = g.x;
                        x1 = g.y;
                    }
                    if (kEpi == kEpiResid) {
                        x0 += rs[2 * j];
                        x1 += rs[2 * j + 1];
                    }
                    o2[j] = __floats2bfloat162_rn(x0, x1);
                }
                if (kEpi == kEpiResid) group_sync();  // every row's residual read before the box is overwritten
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    *reinterpret_cast<uint4*>(box + r * 64 + ((u ^ ((r >> 1) & 3)) << 4)) = out[u];
                fence_proxy_async_smem();  // generic-proxy writes -> the TMA store reads
                group_sync();
                if (ht == 0) {
                    tma_tile2d_s2g(&tmap_y, n0 + c * 32, m0, box);
                    bulk_commit_group();
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {  // accumulator b free for tile i+2 (the issuer's barrier)
                if (kPair && rank == 1)
                    mbar_arrive_remote(&tempty_bar[b], 0);
                else
                    mbar_arrive(&tempty_bar[b]);
            }
            if (ct == 0 && i < 4) K2_MARK(6 + 4 * i);
        }
        // The boxes must stay valid until the stores have read them; the grid's
        // completion (the next kernel's griddepcontrol.wait) covers the writes.
        if (ht == 0) bulk_wait_group_read<0>();
    }
    tc_fence_before();
    __syncthreads();
    if (kCluster) {  // no MMA / remote arrive / st.async may target an exited CTA
        cluster_arrive();  // every CTA's remote writes into its peers have landed (their waits passed)
        cluster_wait();
    }
    tc_fence_after();
    if (tid == 0) K2_MARK(19);
    K2_SPAN_END(a.span);
    if (warp == kGMmaWarp) {
        if (kPair)
            tmem_dealloc_pair<kTmemCols>(tmem);
        else
            tmem_dealloc<kTmemCols>(tmem);
    }
}

// ------------------------------------------------------------------ K3 attention

constexpr int kS = 128, kDh = 64;

// One CTA (8 warps) per (sequence, head, 128-query tile) for sequences of
// 128 kNK tokens (kNK = 1..4: 128 / 256 / 384 / 512): S = Q K^T for all kNK key
// tiles into TMEM (M = 128 queries, N = 128 keys per tile, K = 64: four
// kind::f16 MMAs each — the whole score row is resident, so the softmax is
// exact, no online rescaling), row softmax by the threads owning the row's TMEM
// lane (P = exp((s - max) / 8) unnormalised, bf16, written as the next MMA's
// K-major SWIZZLE_128B A operand), O = P V (M = 128, N = 64, K = 128 kNK: V
// read MN-major straight from its token-major tiles), O / sum. Q, K, V arrive by
// 2-D TMA boxes (64 dims x 128 tokens) from the fused QKV activation.
// Shared memory: [V: kNK x 16 KB][Q 16 KB][K: kNK x 16 KB][pad]; P (kNK x 32 KB)
// overlays Q, K and the pad once the S MMAs have read them. (The first version
// used warp-level mma.sync; 2.7 % of the model's flops took 12 % of its time.)
template <int kNK>
constexpr uint32_t attn_smem() {
    return static_cast<uint32_t>(kNK) * 16384 + static_cast<uint32_t>(kNK) * 32768 + 1024;
}

// 8 warps: warp w owns TMEM lane quarter w & 3 (query rows 32 (w & 3) ..) and key
// half w >> 2 (keys 64 kNK (w >> 2) .. + 64 kNK - 1): each thread takes half a row,
// the two halves exchange their row max and sum through shared memory. (Measured
// against the 4-warp version, one thread per row: the same 1.017 ms per C5
// forward — the kernel's ~9.7 µs after QKV are load and launch latency.)
constexpr int kAttnThreads = 256;
// lengths (nullptr: every sequence full): padding mask — keys j >= lengths[seq] get
// probability 0 (excluded from the row max and sum, as an additive -inf mask).
template <int kNK, bool kMasked>
__global__ void __launch_bounds__(kAttnThreads, kNK == 1 ? 4 : 1) attention_tc_kernel(const __grid_constant__ CUtensorMap tmap_qkv,
                                                                    __nv_bfloat16* __restrict__ ctx, int heads,
                                                                    const int* __restrict__ lengths,
                                                                    unsigned long long* span,
                                                                    unsigned long long* marks) {
    constexpr int kSeq = kNK * kS, kHalf = kSeq / 2;  // tokens per sequence, keys per thread
    // Debug builds: per-CTA %globaltimer marks (0 start, 1 after the PDL wait, 2 Q/K/V landed,
    // 3 S in TMEM, 4 P written, 5 O in TMEM, 6 end); nullptr otherwise.
    auto mark = [&](int i) {
        if (marks && threadIdx.x == 0) {
            unsigned long long t_;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
            marks[blockIdx.x * 8 + i] = t_;
        }
    };
    mark(0);
    constexpr uint32_t kTmemCols = kNK == 1 ? 128 : kNK == 2 ? 256 : 512;
    K2_SPAN_BEGIN(span);
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* vs = sm;
    uint8_t* qs = sm + kNK * 16384;
    uint8_t* ks = qs + 16384;
    uint8_t* ps = qs;  // P: 2 kNK blocks of 64 keys (16 KB each) over Q, K and the pad
    __shared__ __align__(8) uint64_t ld_bar, s_bar, o_bar;
    __shared__ uint32_t tmem_s;
    __shared__ float red_max[2][kS], red_sum[2][kS];
    const int bid = blockIdx.x, qt = bid % kNK, h = (bid / kNK) % heads, seq = bid / (kNK * heads);
    const int d = heads * kDh;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int q = warp & 3, hf = warp >> 2, r = q * 32 + lane;
    if (tid == 0) {
        mbar_init(&ld_bar, 1);
        mbar_init(&s_bar, 1);
        mbar_init(&o_bar, 1);
        mbar_fence_init();
        tma_prefetch_desc(&tmap_qkv);
    }
    if (warp == 0) tmem_alloc<kTmemCols>(&tmem_s);  // S: columns 0 .. 128 kNK - 1; O reuses 0-63 after the softmax
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_s;
    pdl_wait();
    mark(1);
    if (tid == 0) {
        const int row0 = seq * kSeq;
        mbar_arrive_expect_tx(&ld_bar, (1 + 2 * kNK) * 16384);
        tma_tile2d_g2s(qs, &tmap_qkv, h * kDh, row0 + qt * kS, &ld_bar);
#pragma unroll
        for (int j = 0; j < kNK; ++j) {
            tma_tile2d_g2s(ks + j * 16384, &tmap_qkv, d + h * kDh, row0 + j * kS, &ld_bar);
            tma_tile2d_g2s(vs + j * 16384, &tmap_qkv, 2 * d + h * kDh, row0 + j * kS, &ld_bar);
        }
        mbar_wait(&ld_bar, 0);
        mark(2);
        tc_fence_after();
        constexpr uint32_t idesc_s = umma_idesc<128, 128, 1>();  // bf16 x bf16 -> f32, both K-major
#pragma unroll
        for (int j = 0; j < kNK; ++j)
#pragma unroll
            for (int kk = 0; kk < kDh / 16; ++kk)
                umma_f16(tmem + static_cast<uint32_t>(j * kS), umma_desc_sw128(qs, kk * 32),
                         umma_desc_sw128(ks + j * 16384, kk * 32), idesc_s, kk ? 1u : 0u);
        umma_commit(&s_bar);
    }
    pdl_trigger();
    mbar_wait(&s_bar, 0);
    mark(3);
    tc_fence_after();
    const uint32_t row_base = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(hf * kHalf);
    const int nvalid = kMasked ? lengths[seq] - hf * kHalf : kHalf;  // this half's valid keys (<= 0: none)
    float mx = -INFINITY;
#pragma unroll
    for (int c = 0; c < kHalf / 32; ++c) {
        float part[32];
        tmem_ld_32x32b_x32(row_base + static_cast<uint32_t>(c * 32), part);
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (!kMasked || c * 32 + j < nvalid) mx = fmaxf(mx, part[j]);
    }
    red_max[hf][r] = mx;
    __syncthreads();
    mx = fmaxf(red_max[0][r], red_max[1][r]);  // finite: every sequence has >= 1 valid key (host-checked)
    const float off = mx * kAttnScaleLog2;
    float sum = 0.f;
#pragma unroll
    for (int c32 = 0; c32 < kHalf / 32; ++c32) {
        float part[32];
        tmem_ld_32x32b_x32(row_base + static_cast<uint32_t>(c32 * 32), part);
        const int key0 = hf * kHalf + c32 * 32;  // first key of this chunk within the sequence
        uint8_t* pb = ps + (key0 >> 6) * 16384;  // its 64-key P block
#pragma unroll
        for (int q8 = 0; q8 < 4; ++q8) {  // 16-byte chunks of 8 keys
            const int cc = ((key0 & 63) >> 3) + q8;
            uint4 u;
            __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int key = c32 * 32 + q8 * 8 + 2 * j;  // within this half
                const float p0 = !kMasked || key < nvalid ? ex2_approx(fmaf(part[q8 * 8 + 2 * j], kAttnScaleLog2, -off)) : 0.f;
                const float p1 =
                    !kMasked || key + 1 < nvalid ? ex2_approx(fmaf(part[q8 * 8 + 2 * j + 1], kAttnScaleLog2, -off)) : 0.f;
                sum += p0 + p1;
                h2[j] = __floats2bfloat162_rn(p0, p1);
            }
            *reinterpret_cast<uint4*>(pb + r * 128 + ((cc ^ (r & 7)) << 4)) = u;
        }
    }
    red_sum[hf][r] = sum;
    fence_proxy_async_smem();  // P (generic-proxy writes) -> the PV MMA reads
    tc_fence_before();
    __syncthreads();
    mark(4);
    if (tid == 0) {
        tc_fence_after();
        // B = V as an MN-major operand: N = 64 dims contiguous (one 128-byte swizzle
        // span per key), K = keys in 8-key atoms 1024 B apart (SBO), the tiles contiguous.
        constexpr uint32_t idesc_o = umma_idesc<128, kDh, 1>() | (1u << 16);  // b_major = MN
#pragma unroll
        for (int kk = 0; kk < kSeq / 16; ++kk)
            umma_f16(tmem, umma_desc_sw128(ps + (kk >> 2) * 16384, (kk & 3) * 32),
                     umma_desc_sw128(vs, kk * 2048), idesc_o, kk ? 1u : 0u);
        umma_commit(&o_bar);
    }
    mbar_wait(&o_bar, 0);
    mark(5);
    tc_fence_after();
    float o[32];  // this half's 32 output dims of row r
    tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(hf * 32), o);
    const float inv = 1.0f / (red_sum[0][r] + red_sum[1][r]);
    uint4* dst = reinterpret_cast<uint4*>(ctx + (static_cast<size_t>(seq) * kSeq + qt * kS + r) * d + h * kDh + hf * 32);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        uint4 u;
        __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
        for (int j = 0; j < 4; ++j) h2[j] = __floats2bfloat162_rn(o[c * 8 + 2 * j] * inv, o[c * 8 + 2 * j + 1] * inv);
        dst[c] = u;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) tmem_dealloc<kTmemCols>(tmem);
    mark(6);
    K2_SPAN_END(span);
}

// ------------------------------------------------------------------ K4 LayerNorm

template <int kD>
__global__ void __launch_bounds__(256) layernorm_kernel(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y,
                                                        const char* arena, const __grid_constant__ PageTable ptab,
                                                        uint64_t g_off, uint64_t b_off, int rows,
                                                        unsigned long long* span) {
    K2_SPAN_BEGIN(span);
    // One warp per row, kRowsPerWarp rows per warp with every load of a row
    // issued before any math (HBM latency, not arithmetic, bounds this
    // kernel). gamma / beta come straight into registers from the arena (lane
    // l owns columns 8(l + 32i) .. +7, 256 B-aligned vectors: a 16-byte chunk
    // never straddles a page), no shared-memory staging or block barrier.
    constexpr int kPer = kD / 256;  // uint4 (8 bf16) chunks per lane per row
    constexpr int kRowsPerWarp = 2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float gam[kPer * 8], bet[kPer * 8];
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
        const uint64_t c = static_cast<uint64_t>(i * 32 + lane) * 8;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
            const float4 g = *reinterpret_cast<const float4*>(translate(arena, ptab.page, g_off + 4 * (c + 4 * hh)));
            const float4 bb = *reinterpret_cast<const float4*>(translate(arena, ptab.page, b_off + 4 * (c + 4 * hh)));
            gam[i * 8 + 4 * hh] = g.x, gam[i * 8 + 4 * hh + 1] = g.y, gam[i * 8 + 4 * hh + 2] = g.z,
            gam[i * 8 + 4 * hh + 3] = g.w;
            bet[i * 8 + 4 * hh] = bb.x, bet[i * 8 + 4 * hh + 1] = bb.y, bet[i * 8 + 4 * hh + 2] = bb.z,
            bet[i * 8 + 4 * hh + 3] = bb.w;
        }
    }
    pdl_wait();
    const int row0 = (blockIdx.x * 8 + warp) * kRowsPerWarp;
    uint4 raw[kRowsPerWarp][kPer];
#pragma unroll
    for (int rr = 0; rr < kRowsPerWarp; ++rr) {
        const int row = row0 + rr;
        if (row >= rows) break;
        const __nv_bfloat16* xr = x + static_cast<size_t>(row) * kD;
#pragma unroll
        for (int i = 0; i < kPer; ++i) raw[rr][i] = *reinterpret_cast<const uint4*>(xr + (i * 32 + lane) * 8);
    }
#pragma unroll
    for (int rr = 0; rr < kRowsPerWarp; ++rr) {
        const int row = row0 + rr;
        if (row >= rows) break;
        float v[kPer * 8];
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
            const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&raw[rr][i]);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float2 f = __bfloat1622float2(h2[j]);
                v[i * 8 + 2 * j] = f.x;
                v[i * 8 + 2 * j + 1] = f.y;
            }
        }
        float s = 0.f;
#pragma unroll
        for (int i = 0; i < kPer * 8; ++i) s += v[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        const float mean = s / kD;
        float q = 0.f;
#pragma unroll
        for (int i = 0; i < kPer * 8; ++i) {
            const float t = v[i] - mean;
            q += t * t;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
        const float rstd = rsqrtf(q / kD + 1e-12f);
        __nv_bfloat16* yr = y + static_cast<size_t>(row) * kD;
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
            uint4 u;
            __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
            for (int j = 0; j < 4; ++j)
                h2[j] = __floats2bfloat162_rn((v[i * 8 + 2 * j] - mean) * rstd * gam[i * 8 + 2 * j] + bet[i * 8 + 2 * j],
                                              (v[i * 8 + 2 * j + 1] - mean) * rstd * gam[i * 8 + 2 * j + 1] +
                                                  bet[i * 8 + 2 * j + 1]);
            *reinterpret_cast<uint4*>(yr + (i * 32 + lane) * 8) = u;
        }
    }
    K2_SPAN_END(span);
}

// ------------------------------------------------------------------ pooler

// Pooler: out[b][n] = tanh(Wp[n] . x[b, token 0] + bp[n]) for the batch's
// [CLS] rows — a 32 x 768 x 768 product. Block = 8 output features (one warp
// each) x up to kPoolRows sequences (blockIdx.y); the block's [CLS] rows are
// staged in shared memory once; each lane
// holds 3 16-byte chunks of its warp's weight row in registers (swizzled blob
// tile layout, one page translation per chunk).
constexpr int kPoolRows = 64;  // sequences per pooler block (shared memory: 64 x d bf16)
template <int kD>
__global__ void __launch_bounds__(256) pooler_kernel(const __nv_bfloat16* __restrict__ x, float* __restrict__ out,
                                                     const char* arena, const __grid_constant__ PageTable ptab,
                                                     uint64_t w_off, uint64_t b_off, int d, int seq, int batch,
                                                     unsigned long long* span) {
    K2_SPAN_BEGIN(span);
    constexpr int kChunks = kD / 8 / 32;  // 16-byte chunks per lane
    extern __shared__ __align__(16) uint8_t cls_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n = blockIdx.x * 8 + warp;
    uint4 w[kChunks];
    float bias = 0.f;
    if (n < d) {
#pragma unroll
        for (int i = 0; i < kChunks; ++i) {
            const int k = (i * 32 + lane) * 8;
            const uint64_t r = static_cast<uint64_t>(n % 128);
            const uint64_t off = w_off + (static_cast<uint64_t>(n / 128) * (kD / 64) + k / 64) * 16384 + r * 128 +
                                 ((((k % 64) >> 3) ^ (r & 7)) << 4);
            w[i] = *reinterpret_cast<const uint4*>(translate(arena, ptab.page, off));
        }
        bias = *reinterpret_cast<const float*>(translate(arena, ptab.page, b_off + 4ull * n));
    }
    pdl_wait();
    const int b0 = blockIdx.y * kPoolRows, nb = min(kPoolRows, batch - b0);
    for (int i = threadIdx.x; i < nb * kD / 8; i += 256) {
        const int b = i / (kD / 8), c = i % (kD / 8);
        reinterpret_cast<uint4*>(cls_raw)[i] =
            *reinterpret_cast<const uint4*>(x + static_cast<size_t>(b0 + b) * seq * kD + c * 8);
    }
    __syncthreads();
    K2_SPAN_END(span);  // (pooler: start of the per-row loop)
    if (n >= d) return;
    for (int b = 0; b < nb; ++b) {
        float acc = 0.f;
#pragma unroll
        for (int i = 0; i < kChunks; ++i) {
            const uint4 xv = reinterpret_cast<const uint4*>(cls_raw)[b * (kD / 8) + i * 32 + lane];
            const __nv_bfloat162* xh = reinterpret_cast<const __nv_bfloat162*>(&xv);
            const __nv_bfloat162* wh = reinterpret_cast<const __nv_bfloat162*>(&w[i]);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float2 xf = __bfloat1622float2(xh[j]), wf = __bfloat1622float2(wh[j]);
                acc = fmaf(wf.x, xf.x, acc);
                acc = fmaf(wf.y, xf.y, acc);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) out[static_cast<size_t>(b0 + b) * d + n] = tanhf(acc + bias);
    }
}

__global__ void fill_bf16_kernel(__nv_bfloat16* dst, uint64_t n, uint64_t count, uint64_t seed0, uint32_t tensor,
                                 float scaled) {
    const uint64_t total = n * count;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t t = i / n;
        const float v = param_at(param_stream(seed0 + t, tensor), i - t * n, scaled);
        dst[i] = __ushort_as_bfloat16(bf16_bits(v));
    }
}

template <typename Kern, typename... Args>
void launch_pdl(Kern k, dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    GFX_CUDA(cudaLaunchKernelEx(&cfg, k, args...));
}

template <int kEpi, int kBN, bool kPair>
void gemm_bn(const char* arena, const PageTable& pt, uint64_t w_off, uint64_t b_off, const __nv_bfloat16* x,
             __nv_bfloat16* y, const __nv_bfloat16* resid, int T, int K, int N, cudaStream_t s, bool pdl,
             uint64_t g_off = 0, uint64_t be_off = 0) {
    constexpr bool kLN = kEpi == kEpiResidLN;
    CUtensorMap tm;
    if (!encode_tensor_map_2d(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, static_cast<uint64_t>(K),
                              static_cast<uint64_t>(T), static_cast<uint64_t>(K) * 2, kGK, kGM,
                              CU_TENSOR_MAP_SWIZZLE_128B))
        throw CudaError("cuTensorMapEncodeTiled failed (bert gemm)");
    // Output (and residual) as 32-column x 128-row boxes, SWIZZLE_64B: the epilogue's staging layout.
    CUtensorMap tmy, tmr;
    if (!encode_tensor_map_2d(&tmy, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, y, static_cast<uint64_t>(N),
                              static_cast<uint64_t>(T), static_cast<uint64_t>(N) * 2, 32, kGM,
                              CU_TENSOR_MAP_SWIZZLE_64B))
        throw CudaError("cuTensorMapEncodeTiled failed (bert gemm output)");
    if (!encode_tensor_map_2d(&tmr, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, resid ? resid : y, static_cast<uint64_t>(N),
                              static_cast<uint64_t>(T), static_cast<uint64_t>(N) * 2, 32, kGM,
                              CU_TENSOR_MAP_SWIZZLE_64B))
        throw CudaError("cuTensorMapEncodeTiled failed (bert gemm residual)");
    // Pair mode: weight tiles as 16 KB boxes (64 bf16 x 128 rows of 128 B, raw bytes:
    // the tiles are stored pre-swizzled) of a tensor map over the arena span the
    // model's pages cover, so the odd CTA's loads can complete the even CTA's barrier.
    CUtensorMap tmw = tmy;
    if (kPair) {
        uint32_t maxp = 0;
        for (uint32_t i = 0; i < pt.n; ++i) maxp = std::max(maxp, pt.page[i]);
        // 512-byte rows, 32-row boxes: a 16 KB tile as 32 row requests instead of 128.
        const uint64_t rows = (static_cast<uint64_t>(maxp) + 1) * (kPageBytes / 512);
        if (!encode_tensor_map_2d(&tmw, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, arena, 256, rows, 512, 256, 32,
                                  CU_TENSOR_MAP_SWIZZLE_NONE))
            throw CudaError("cuTensorMapEncodeTiled failed (bert gemm arena weights)");
    }
    unsigned long long* span = next_span(kLN ? "gemm+LN" : kEpi == kEpiGelu ? "gemm GELU" : kEpi == kEpiResid ? "gemm resid" : "gemm bias");
    GemmArgs a{nullptr, span, arena, w_off, b_off, g_off, be_off, y, resid, T, K, N, pt};
#ifdef GFX_K2_DEBUG
    static unsigned long long* dbg = nullptr;
    static int calls = 0;
    if (!dbg) GFX_CUDA(cudaMalloc(&dbg, sizeof(unsigned long long) * 24 * 1024));
    const bool report = ++calls > 48 && calls <= 52;  // the second forward's first layer
    if (report) {
        GFX_CUDA(cudaMemsetAsync(dbg, 0, sizeof(unsigned long long) * 24 * 1024, s));
        a.dbg = dbg;
    }
#endif
    const size_t smem = kGSmem + 4 * 8192 + 1024;
    ensure_max_dynamic_smem(reinterpret_cast<const void*>(gemm_bf16_kernel<kEpi, kBN, kPair>), static_cast<int>(smem));
    const int sms = device_sm_count(current_device());
    const int tiles = (T / kGM) * (N / kBN);
    int grid = tiles < sms ? tiles : sms;
    if (kPair) grid &= ~1;
    if (kLN) grid = tiles;  // one 128 x 256 tile per CTA, clusters of N / 256 = 3 (host-checked: ln_fusable)
    if (kPair || kLN) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(kGThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
        attr[1].id = cudaLaunchAttributeClusterDimension;
        attr[1].val.clusterDim.x = kPair ? 2u : static_cast<unsigned>(N / kBN);
        attr[1].val.clusterDim.y = 1;
        attr[1].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 2;
        GFX_CUDA(cudaLaunchKernelEx(&cfg, gemm_bf16_kernel<kEpi, kBN, kPair>, tm, tmy, tmr, tmw, a));
    } else {
        launch_pdl(gemm_bf16_kernel<kEpi, kBN, kPair>, dim3(grid), dim3(kGThreads), smem, s, pdl, tm, tmy, tmr, tmw, a);
    }
#ifdef GFX_K2_DEBUG
    if (report) {
        std::vector<unsigned long long> m(static_cast<size_t>(grid) * 24);
        GFX_CUDA(cudaStreamSynchronize(s));
        GFX_CUDA(cudaMemcpy(m.data(), dbg, m.size() * 8, cudaMemcpyDeviceToHost));
        unsigned long long t0 = ~0ull;
        for (int c = 0; c < grid; ++c) t0 = std::min(t0, m[static_cast<size_t>(c) * 24]);
        std::fprintf(stderr, "[K2 epi %d T %d K %d N %d tile 128x%d pair %d grid %d tiles %d] us: min med max\n", kEpi, T, K,
                     N, kBN, kPair ? 1 : 0, grid, tiles);
        static const char* nm[4] = {"stage0 landed", "last MMA issued", "epi saw acc", "epi done"};
        for (int i = 0; i < 20; ++i) {
            std::vector<double> v;
            for (int c = 0; c < grid; ++c)
                if (m[static_cast<size_t>(c) * 24 + i]) v.push_back((m[static_cast<size_t>(c) * 24 + i] - t0) * 1e-3);
            if (v.empty()) continue;
            std::sort(v.begin(), v.end());
            char n[40];
            if (i < 3) std::snprintf(n, sizeof n, "%s", i == 0 ? "start" : i == 1 ? "setup" : "first A issued");
            else if (i == 19) std::snprintf(n, sizeof n, "end");
            else std::snprintf(n, sizeof n, "tile%d %s", (i - 3) / 4, nm[(i - 3) % 4]);
            std::fprintf(stderr, "  %-24s n=%3zu %7.2f %7.2f %7.2f\n", n, v.size(), v[0], v[v.size() / 2], v.back());
        }
    }
#endif
}

// 128 x 256 tiles: a tcgen05.mma with smem operands costs >= ~119 cycles
// whatever N (tools/gemm_rate.cu: N=256 runs at its 128-cycle floor, N=128 at
// 119 vs 64), so the widest tile wins even when it leaves SMs idle (N = 768:
// 96 tiles). 128 x 192 was measured at ~210 cycles per MMA.
template <int kEpi>
void gemm(const char* arena, const PageTable& pt, uint64_t w_off, uint64_t b_off, const __nv_bfloat16* x,
          __nv_bfloat16* y, const __nv_bfloat16* resid, int T, int K, int N, cudaStream_t s, bool pdl, bool pair) {
    if (T % kGM || N % 128 || K % kGK) throw std::runtime_error("bert gemm: T, N multiple of 128, K of 64");
    // The 2-SM variant (BertWorkspace::gemm_pair) is correct; with the relay removed
    // (.cta_group::2 loads complete the even CTA's barrier) it runs 1.21 ms per
    // forward vs 1.17-1.18 for the single-CTA kernel (was 1.63 with the relay):
    // both advance ~0.45 µs per K stage with ~2 µs TMA latency at 192 KB in
    // flight per SM, so the single-CTA kernel stays the default.
    if (N % 256 == 0 && (T / kGM) % 2 == 0 && pair)
        gemm_bn<kEpi, 256, true>(arena, pt, w_off, b_off, x, y, resid, T, K, N, s, pdl);
    else if (N % 256 == 0)
        gemm_bn<kEpi, 256, false>(arena, pt, w_off, b_off, x, y, resid, T, K, N, s, pdl);
    else
        gemm_bn<kEpi, 128, false>(arena, pt, w_off, b_off, x, y, resid, T, K, N, s, pdl);
}

// Residual GEMM (N = d = 768) with the post-LN LayerNorm fused into its
// epilogue when every 128-row block gets its own resident 3-CTA cluster
// (T <= 128 x max active clusters; 4096 tokens = 32 clusters); otherwise the
// residual GEMM and layernorm_kernel (via `t`).
int ln_max_clusters(int nc) {
    static std::mutex mu;
    static std::map<std::pair<int, int>, int> cache;
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find({dev, nc});
    if (it != cache.end()) return it->second;
    auto k = gemm_bf16_kernel<kEpiResidLN, 256, false>;
    const size_t smem = kGSmem + 4 * 8192 + 1024;
    ensure_max_dynamic_smem(reinterpret_cast<const void*>(k), static_cast<int>(smem));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(nc * 32));
    cfg.blockDim = dim3(kGThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(nc);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    GFX_CUDA(cudaOccupancyMaxActiveClusters(&n, k, &cfg));
    cache[{dev, nc}] = n;
    return n;
}

bool ln_fusable(int T, int N) {
#ifdef GFX_K2_DEBUG
    if (std::getenv("GFX_K2_NOLN")) return false;  // debug A/B only
#endif
    return N % 256 == 0 && N / 256 >= 2 && N / 256 <= 8 && T % kGM == 0 && T / kGM <= ln_max_clusters(N / 256);
}

void gemm_resid_ln(const char* arena, const PageTable& pt, uint64_t w_off, uint64_t b_off, uint64_t g_off,
                   uint64_t be_off, const __nv_bfloat16* x, __nv_bfloat16* y, const __nv_bfloat16* resid,
                   __nv_bfloat16* t, int T, int K, int N, cudaStream_t s, bool pdl, bool pair) {
    if (ln_fusable(T, N)) {
        if (K % kGK) throw std::runtime_error("bert gemm: K multiple of 64");
        gemm_bn<kEpiResidLN, 256, false>(arena, pt, w_off, b_off, x, y, resid, T, K, N, s, pdl, g_off, be_off);
        return;
    }
    gemm<kEpiResid>(arena, pt, w_off, b_off, x, t, resid, T, K, N, s, pdl, pair);
    auto ln = N == 512 ? layernorm_kernel<512> : N == 1024 ? layernorm_kernel<1024> : layernorm_kernel<768>;
    if (N != 512 && N != 768 && N != 1024) throw std::runtime_error("bert layernorm: d must be 512, 768 or 1024");
    launch_pdl(ln, dim3((T + 15) / 16), dim3(256), 0, s, true, static_cast<const __nv_bfloat16*>(t), y, arena, pt, g_off,
               be_off, T, next_span("layernorm"));
}

}  // namespace

// ------------------------------------------------------------------ layout

BertLayout bert_layout(int L, int d, int heads, int ffn, int seq) {
    BertLayout lay;
    lay.L = L;
    lay.d = d;
    lay.heads = heads;
    lay.ffn = ffn;
    lay.seq = seq;
    uint64_t off = 0;
    auto align = [](uint64_t v, uint64_t a) { return (v + a - 1) / a * a; };
    auto wmat = [&](uint64_t n, uint64_t k) {
        off = align(off, 16384);
        const uint64_t at = off;
        off += align(n, 128) * k * 2;
        return at;
    };
    auto vec = [&](uint64_t n) {
        off = align(off, 256);
        const uint64_t at = off;
        off += 4 * n;
        return at;
    };
    for (int l = 0; l < L; ++l) {
        BertLayerOffsets o{};
        o.wqkv = wmat(3 * d, d);
        o.bqkv = vec(3 * d);
        o.wo = wmat(d, d);
        o.bo = vec(d);
        o.ln1_g = vec(d);
        o.ln1_b = vec(d);
        o.w1 = wmat(ffn, d);
        o.b1 = vec(ffn);
        o.w2 = wmat(d, ffn);
        o.b2 = vec(d);
        o.ln2_g = vec(d);
        o.ln2_b = vec(d);
        lay.layer.push_back(o);
    }
    lay.wp = wmat(d, d);
    lay.bp = vec(d);
    lay.bytes = align(off, 256);
    return lay;
}

void BertWorkspace::ensure(int ntok, int d, int ffn) {
    if (ntok <= tokens) return;
    release();
    const size_t T = static_cast<size_t>(ntok);
    GFX_CUDA(cudaMalloc(&x, T * d * 2));
    GFX_CUDA(cudaMalloc(&qkv, T * 3 * d * 2));
    GFX_CUDA(cudaMalloc(&ctx, T * d * 2));
    GFX_CUDA(cudaMalloc(&h, T * d * 2));
    GFX_CUDA(cudaMalloc(&f, T * ffn * 2));
    GFX_CUDA(cudaMalloc(&t, T * d * 2));
    tokens = ntok;
}

void BertWorkspace::ensure_side_stream() {
    if (side) return;
    GFX_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
    GFX_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    GFX_CUDA(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
}

void BertWorkspace::release() {
    for (__nv_bfloat16** p : {&x, &qkv, &ctx, &h, &f, &t}) {
        if (*p) cudaFree(*p);
        *p = nullptr;
    }

    tokens = 0;
    if (side) cudaStreamDestroy(side);
    if (fork) cudaEventDestroy(fork);
    if (join) cudaEventDestroy(join);
    side = nullptr;
    fork = join = nullptr;
    if (flow_cnt) cudaFree(flow_cnt);
    if (flow_stats) cudaFree(flow_stats);
    flow_cnt = nullptr;
    flow_stats = nullptr;
    flow_L = flow_M = flow_F = flow_ctas = 0;
    flow_cnt_words = 0;
}

// The per-op encoder (K2-K4) over sequences [seq0, seq0 + nb) of a request, on stream s:
// every buffer is addressed at the range's first token row, so two ranges can run on two
// streams at once. Layer l's output lands in ws.x (and hidden[l + 1] when debugging).
int encode_rows(const char* arena, const PageTable& pt, const BertLayout& lay, int seq0, int nb,
                const __nv_bfloat16* in, const int* lengths, BertWorkspace& ws, cudaStream_t s,
                __nv_bfloat16* hidden) {
    const int d = lay.d, T = nb * lay.seq;
    const size_t r0 = static_cast<size_t>(seq0) * lay.seq;
    __nv_bfloat16 *xw = ws.x + r0 * d, *qkv = ws.qkv + r0 * 3 * d, *ctx = ws.ctx + r0 * d, *h = ws.h + r0 * d,
                  *f = ws.f + r0 * lay.ffn, *t = ws.t + r0 * d;
    const __nv_bfloat16* x = in + r0 * d;
    const int* len = lengths ? lengths + seq0 : nullptr;
    const size_t hbytes = static_cast<size_t>(T) * d * 2;
    int launches = 0;
    for (int l = 0; l < lay.L; ++l) {
        const BertLayerOffsets& o = lay.layer[static_cast<size_t>(l)];
        gemm<kEpiBias>(arena, pt, o.wqkv, o.bqkv, x, qkv, nullptr, T, d, 3 * d, s, l > 0 && !hidden, ws.gemm_pair);
        {
            CUtensorMap tq;
            if (!encode_tensor_map_2d(&tq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, qkv, static_cast<uint64_t>(3 * d),
                                      static_cast<uint64_t>(T), static_cast<uint64_t>(3 * d) * 2, kDh, kS,
                                      CU_TENSOR_MAP_SWIZZLE_128B))
                throw CudaError("cuTensorMapEncodeTiled failed (attention)");
            const int nk = lay.seq / kS;
            auto att = len ? (nk == 1 ? attention_tc_kernel<1, true> : nk == 2 ? attention_tc_kernel<2, true>
                              : nk == 3 ? attention_tc_kernel<3, true> : attention_tc_kernel<4, true>)
                           : (nk == 1 ? attention_tc_kernel<1, false> : nk == 2 ? attention_tc_kernel<2, false>
                              : nk == 3 ? attention_tc_kernel<3, false> : attention_tc_kernel<4, false>);
            const uint32_t asmem = nk == 1 ? attn_smem<1>() : nk == 2 ? attn_smem<2>() : nk == 3 ? attn_smem<3>() : attn_smem<4>();
            ensure_max_dynamic_smem(reinterpret_cast<const void*>(att), static_cast<int>(asmem));
            unsigned long long* marks = nullptr;
#ifdef GFX_K2_DEBUG
            static unsigned long long* mbuf = nullptr;
            static int att_calls = 0;
            const bool report = ++att_calls == 13;  // the second forward's first layer
            if (report) {
                if (!mbuf) GFX_CUDA(cudaMalloc(&mbuf, sizeof(unsigned long long) * 8 * 8192));
                GFX_CUDA(cudaMemsetAsync(mbuf, 0, sizeof(unsigned long long) * 8 * 8192, s));
                marks = mbuf;
            }
#endif
            launch_pdl(att, dim3(nb * lay.heads * nk), dim3(kAttnThreads), asmem, s, true, tq, ctx, lay.heads, len,
                       next_span("attention"), marks);
#ifdef GFX_K2_DEBUG
            if (report) {
                const int grid = nb * lay.heads * nk;
                std::vector<unsigned long long> m(static_cast<size_t>(grid) * 8);
                GFX_CUDA(cudaStreamSynchronize(s));
                GFX_CUDA(cudaMemcpy(m.data(), mbuf, m.size() * 8, cudaMemcpyDeviceToHost));
                unsigned long long t0 = ~0ull;
                for (int c = 0; c < grid; ++c) t0 = std::min(t0, m[static_cast<size_t>(c) * 8]);
                static const char* nm[7] = {"start", "after PDL wait", "Q/K/V landed", "S in TMEM", "P written", "O in TMEM", "end"};
                std::fprintf(stderr, "[K3 attention, %d CTAs] us after the first CTA start: min p10 median p90 max\n", grid);
                for (int i = 0; i < 7; ++i) {
                    std::vector<double> v;
                    for (int c = 0; c < grid; ++c)
                        if (m[static_cast<size_t>(c) * 8 + i]) v.push_back((m[static_cast<size_t>(c) * 8 + i] - t0) * 1e-3);
                    if (v.empty()) continue;
                    std::sort(v.begin(), v.end());
                    const size_t n = v.size();
                    std::fprintf(stderr, "  %-16s %7.2f %7.2f %7.2f %7.2f %7.2f\n", nm[i], v[0], v[n / 10], v[n / 2],
                                 v[n * 9 / 10], v[n - 1]);
                }
            }
#endif
        }
        gemm_resid_ln(arena, pt, o.wo, o.bo, o.ln1_g, o.ln1_b, ctx, h, x, t, T, d, d, s, true, ws.gemm_pair);
        gemm<kEpiGelu>(arena, pt, o.w1, o.b1, h, f, nullptr, T, d, lay.ffn, s, true, ws.gemm_pair);
        gemm_resid_ln(arena, pt, o.w2, o.b2, o.ln2_g, o.ln2_b, f, xw, h, t, T, lay.ffn, d, s, true, ws.gemm_pair);
        launches += ln_fusable(T, d) ? 5 : 7;
        x = xw;
        if (hidden)
            GFX_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(hidden) + (l + 1) * hbytes, xw, hbytes,
                                     cudaMemcpyDeviceToDevice, s));
    }
    return launches;
}

int bert_forward(const char* arena, const PageTable& pt, const BertLayout& lay, int batch, const __nv_bfloat16* in,
                 float* out, BertWorkspace& ws, cudaStream_t s, __nv_bfloat16* hidden, const int* lengths) {
    const int d = lay.d, T = batch * lay.seq;
    if (lay.seq % kS || lay.seq > 4 * kS || d / lay.heads != kDh || d % lay.heads || (d != 512 && d != 768 && d != 1024))
        throw std::runtime_error("bert: this build serves seq 128 / 256 / 384 / 512, d_head 64, d 512 / 768 / 1024");
    ws.ensure(T, d, lay.ffn);
    int launches = 0;
#ifdef GFX_K2_DEBUG
    static int forwards = 0;
    if (++forwards == 10 && !hidden) {
        if (!g_span.buf) GFX_CUDA(cudaMalloc(&g_span.buf, 16 * SpanTrace::kMax));
        std::vector<unsigned long long> init(2 * SpanTrace::kMax);
        for (int i = 0; i < SpanTrace::kMax; ++i) init[2 * i] = ~0ull, init[2 * i + 1] = 0;
        GFX_CUDA(cudaMemcpyAsync(g_span.buf, init.data(), init.size() * 8, cudaMemcpyHostToDevice, s));
        GFX_CUDA(cudaStreamSynchronize(s));
        g_span.names.clear();
        g_span.on = true;
    }
#endif
    const __nv_bfloat16* x = in;
    const size_t hbytes = static_cast<size_t>(T) * d * 2;
    if (hidden) GFX_CUDA(cudaMemcpyAsync(hidden, in, hbytes, cudaMemcpyDeviceToDevice, s));
    const bool flow = ws.flow && !lengths && bert_flow_supported(lay, batch);  // K5 serves unmasked requests
    if (flow) {
        // K5: every layer in one dataflow launch; with `hidden`, layer l's output lands in hidden[l + 1].
        __nv_bfloat16* xout = hidden ? hidden + static_cast<size_t>(T) * d : ws.x;
        const int xstride = hidden ? T : 0;
        launches += bert_encoder_flow(arena, pt, lay, batch, in, xout, xstride, ws, s);
        x = xout + static_cast<size_t>(lay.L - 1) * xstride * d;
    }
    bool split = false;
    if (!flow) {
        // Per-op launches. A request of >= 64 sequences runs as two halves on two streams
        // (row-partitioned activations: nothing shared but the weights), so each half's
        // kernels fill the other's launch fill, tails and idle SMs (the N = d GEMMs run
        // one tile per CTA on d / 256 x row-block clusters). Measured (BERT-base, 12
        // layers): 64 sequences 1.73 -> 1.59 ms, 128: 3.26 -> 3.17 ms; at 32 the halves'
        // GEMMs quantise worse (0.98 -> 1.02 ms), so smaller requests stay on one stream.
        // The debug path stays serial (and tests check it equals the split result).
        split = !hidden && batch >= 64;
        if (split) {
            ws.ensure_side_stream();
            GFX_CUDA(cudaEventRecord(ws.fork, s));
            GFX_CUDA(cudaStreamWaitEvent(ws.side, ws.fork, 0));
            const int b0 = batch / 2;
            launches += encode_rows(arena, pt, lay, 0, b0, in, lengths, ws, s, nullptr);
            launches += encode_rows(arena, pt, lay, b0, batch - b0, in, lengths, ws, ws.side, nullptr);
            GFX_CUDA(cudaEventRecord(ws.join, ws.side));
            GFX_CUDA(cudaStreamWaitEvent(s, ws.join, 0));
        } else {
            launches += encode_rows(arena, pt, lay, 0, batch, in, lengths, ws, s, hidden);
        }
        x = ws.x;
    }
    auto pool = d == 512 ? pooler_kernel<512> : d == 1024 ? pooler_kernel<1024> : pooler_kernel<768>;
    const int rows = batch < kPoolRows ? batch : kPoolRows;
    ensure_max_dynamic_smem(reinterpret_cast<const void*>(pool), kPoolRows * 1024 * 2);
    launch_pdl(pool, dim3((d + 7) / 8, (batch + kPoolRows - 1) / kPoolRows), dim3(256), static_cast<size_t>(rows) * d * 2,
               s, !hidden && !split, static_cast<const __nv_bfloat16*>(x), out, arena, pt, lay.wp, lay.bp, d, lay.seq, batch,
               next_span("pooler"));
#ifdef GFX_K2_DEBUG
    if (g_span.on) {
        std::vector<unsigned long long> v(2 * g_span.names.size());
        GFX_CUDA(cudaStreamSynchronize(s));
        GFX_CUDA(cudaMemcpy(v.data(), g_span.buf, v.size() * 8, cudaMemcpyDeviceToHost));
        const unsigned long long t0 = v[0];
        double busy = 0;
        std::fprintf(stderr, "[K2 span] T %d: kernel, start, end, duration, gap after previous end (us)\n", T);
        for (size_t i = 0; i < g_span.names.size(); ++i) {
            const double st = (v[2 * i] - t0) * 1e-3, en = (v[2 * i + 1] - t0) * 1e-3;
            const double gap = i ? st - (v[2 * i - 1] - t0) * 1e-3 : 0.0;
            busy += en - st;
            if (i < 16 || i + 2 >= g_span.names.size())
                std::fprintf(stderr, "  %3zu %-12s %9.2f %9.2f %7.2f %7.2f\n", i, g_span.names[i], st, en, en - st, gap);
        }
        std::fprintf(stderr, "  forward %.2f us, sum of kernel spans %.2f us\n",
                     (v[2 * g_span.names.size() - 1] - t0) * 1e-3, busy);
        g_span.on = false;
    }
#endif
    return launches + 1;
}

void bert_gemm_op(const char* arena, const PageTable& pt, const BertLayout& lay, int l, int op,
                  const __nv_bfloat16* x, const __nv_bfloat16* resid, __nv_bfloat16* y, int T, bool pair,
                  cudaStream_t s) {
    if (l < 0 || l >= lay.L) throw std::invalid_argument("bert gemm: bad layer");
    const BertLayerOffsets& o = lay.layer[static_cast<size_t>(l)];
    const int d = lay.d;
    switch (op) {
        case 0: gemm<kEpiBias>(arena, pt, o.wqkv, o.bqkv, x, y, nullptr, T, d, 3 * d, s, false, pair); break;
        case 1: gemm<kEpiResid>(arena, pt, o.wo, o.bo, x, y, resid, T, d, d, s, false, pair); break;
        case 2: gemm<kEpiGelu>(arena, pt, o.w1, o.b1, x, y, nullptr, T, d, lay.ffn, s, false, pair); break;
        case 3: gemm<kEpiResid>(arena, pt, o.w2, o.b2, x, y, resid, T, lay.ffn, d, s, false, pair); break;
        case 4:
        case 5: {
            // The forward's residual + LayerNorm step (fused when ln_fusable, else GEMM + K4 through a scratch).
            __nv_bfloat16* t = nullptr;
            if (!ln_fusable(T, d)) GFX_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&t), static_cast<size_t>(T) * d * 2, s));
            if (op == 4)
                gemm_resid_ln(arena, pt, o.wo, o.bo, o.ln1_g, o.ln1_b, x, y, resid, t, T, d, d, s, false, pair);
            else
                gemm_resid_ln(arena, pt, o.w2, o.b2, o.ln2_g, o.ln2_b, x, y, resid, t, T, lay.ffn, d, s, false, pair);
            if (t) GFX_CUDA(cudaFreeAsync(t, s));
            break;
        }
        default: throw std::invalid_argument("bert gemm: op must be 0..5");
    }
}

void launch_fill_bf16(__nv_bfloat16* dst, uint64_t n, uint64_t seed, uint32_t tensor, float scale, cudaStream_t s,
                      uint64_t count) {
    const uint64_t total = n * count;
    unsigned blocks = static_cast<unsigned>((total + 255) / 256);
    if (blocks > 148 * 32) blocks = 148 * 32;
    if (blocks == 0) blocks = 1;
    fill_bf16_kernel<<<blocks, 256, 0, s>>>(dst, n, count, seed, tensor, param_scale(scale));
    GFX_CUDA(cudaGetLastError());
}

}  // namespace gfx
