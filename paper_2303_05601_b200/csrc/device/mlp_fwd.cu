// K1 v7: the whole fp32 MLP forward of one request (batch 32) in ONE persistent
// cooperative launch on the 5th-gen tensor cores (tcgen05, kind::tf32, 3xTF32
// error compensation), weights streamed by TMA straight out of the paged HBM
// arena. Replaces profile.infer_time_us (proj/src/cluster.cpp:161,167).
//
//   layer l: Y_l[32 x N] = act(X_l[32 x K] . W_l^T + b_l)  as  D^T[N x 32] = W_l . X_l^T
//   (swap AB: 128 weight rows fill the MMA M side, the 32 batch rows are N),
//   act = ReLU on hidden layers; the last layer's rows go through softmax.
//
// Layer 0 (v9) is split dynamically instead: CTAs claim kMlpChunk0-step ranges from a
// per-launch counter, so the CTAs a PDL-chained launch places last (up to ~5 µs late)
// take less of it (profiles/r2_k1_v7.md); the static split below holds for layers >= 1.
//
// Work split (stream-K): a layer is tiles x nkt steps, step s = (feature tile
// s / nkt, K tile s % nkt); the blob stores weight tiles in exactly that order,
// so step s reads the 16 KB tile at w_off + 16 KB * s. CTA c takes the
// contiguous steps [c*S/grid, (c+1)*S/grid): every SM streams the same number
// of weight bytes in every layer (no idle SMs, whatever the layer shape), and a
// CTA whose range crosses a tile boundary contributes to two tiles. Every CTA
// streams the weight tiles of ALL its layers back to back through one TMA ring
// (weights do not depend on activations), so the HBM stays busy across layer
// boundaries; only the activation operands wait.
//
// Layer boundary (v6 needed eight dependent global round trips, a counter-
// based v7 draft five): each CTA adds its partial of a tile straight into the
// layer's output buffer with red.add.u64 (the reduction happens in L2), and
// nothing else — no fence, no counter. Every 64-bit word carries its own
// completion count: word = (fixed-point value << 9) + (K tiles this partial
// covers), so a word is complete when its low 9 bits reach the layer's nkt.
// The consumer's X producer waits until one word of the source tile is
// complete (the tile's contributors reduce all its words at about the same
// time; lanes share what they have seen through shared memory), then
// bulk-copies the 8 KB [32 features x 32 rows] block of its K tile; the
// converter warps check every word's count and re-read any still incomplete
// word from L2, then apply ReLU and the tf32 split while building the MMA
// operand. (Issuing the copies before the tile completed made every early
// ring slot pay its own ~1 µs poll round trip in the converters.) The bias is added once, by the CTA whose range holds the tile's K
// tile 0. Fixed point: value x 2^32 rounded to an integer; integer addition is
// associative, so the reduced value does not depend on the order the partials
// reach L2 and every launch is bit-reproducible; the consumer converts once
// (int64 -> fp32, one rounding). Range |value| < 2^22, resolution 2^-32 (far
// inside the 1e-5 fp32 tolerance for these models).
//
// Precision: the tensor core reads W straight from the landed fp32 tile;
// kind::tf32 uses only the top 19 bits, i.e. W_hi = trunc_tf32(W) (verified on
// B200: the rounded interpretation breaks parity, 1.4e-3). Converter warps form
// W_lo = W - W_hi (exact) into a TMEM ring; activations are split by the
// converters: X_hi = rn_tf32(X), X_lo = X - X_hi (exact). Per 8-wide K slice:
//   D += W_hi . [X_hi; X_lo]   (SS, N = 64: both batch planes at once)
//   D += W_lo . X_hi           (TS, A from TMEM, N = 32)
// i.e. every product but W_lo.X_lo (< 2^-21 relative); the accumulator is
// drained to fp32 registers every kChunk K tiles.
//
// Operand block (smem, per step, 8 KB): 64 rows x 128 B, rows 0-31 = X_hi of
// batch rows 0-31, rows 32-63 = X_lo, SWIZZLE_128B chunk permutation (16-byte
// chunk j of row r at j ^ (r & 7)): the MMA's K-major B operand as is. The raw
// input of the step lands in the same 8 KB (layer 0: 2-D TMA of the 4 KB
// request-input tile into the upper half, row-major swizzled; later layers:
// the previous layer's 8 KB fixed-point output block, feature-major) and is
// converted in place.
//
// Roles (16 warps, one CTA per SM, 8-deep ring: W [8][16 KB] and X [8][8 KB]):
//   warp 0        W producer: 1-D bulk TMA of the pre-swizzled weight tiles, one
//                 32 KB copy per pair of consecutive steps of a layer (half the
//                 requests of one issuing thread, whose TMA requests are served
//                 one after another)
//   warp 14       X producer (one lane: divergent lanes spinning on different
//                 conditions can starve each other): layer 0 issues the 2-D TMA
//                 of the raw input tile, later layers wait for the source tile's
//                 first complete word, then bulk-copy its 8 KB block (16 KB for
//                 a pair of steps). A paired copy completes the first slot's
//                 barrier; the producer arrives on the second slot's barrier so
//                 every barrier still completes once per ring round.
//   warps 2-5/6-9 converters (two groups, alternate steps): W_lo -> TMEM ring,
//                 raw X (completion-checked) -> [X_hi; X_lo] operand (ReLU)
//   warps 1, 15   MMA issuers, alternate accumulator chunks: 8 MMAs per K tile
//                 and one commit per step (step_done frees slot + W_lo stage)
//   warps 10-13   drain (TMEM -> fp32 registers per chunk); per tile partial:
//                 fixed-point words staged in smem (SWIZZLE_128B boxes of 32
//                 features x 16 rows), then one TMA add-reduction per box
//                 (cp.reduce.async.bulk.tensor .add u64, rows >= N clipped by
//                 the tensor map) — the SM hands 32 KB to the TMA engine;
//                 softmax rows at the end; at start they clear the other
//                 parity's buffer for the next launch.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <vector>

#include "common.cuh"
#include "mlp.cuh"
#include "sm100.cuh"

namespace gfx {

namespace {

using namespace gfx::sm100;

constexpr int kRows = 32;     // batch rows per request
constexpr int kTileM = 128;   // output features per tile = MMA M
constexpr int kTileK = 32;    // fp32 K per ring step (one 128-byte swizzle row)
constexpr int kSlots = 8;     // ring depth: 8 x 16 KB = 128 KB of weights in flight per SM
constexpr int kChunk = 4;     // K tiles accumulated in TMEM before a drain
constexpr int kThreads = 16 * 32;
constexpr uint32_t kWBytes = kTileM * kTileK * 4;      // 16 KB
constexpr uint32_t kXBytes = 2 * kRows * kTileK * 4;   // 8 KB: [X_hi; X_lo]
constexpr uint32_t kRaw0Bytes = kRows * kTileK * 4;    // layer-0 raw input tile: 4 KB (upper half of X)
constexpr uint32_t kRawBytes = kRows * kTileK * 8;     // later layers: 8 KB fixed-point block (all of X)
constexpr uint32_t kXRing = kSlots * kWBytes;          // smem: W ring [8][16 KB], then X ring [8][8 KB]
constexpr uint32_t kStageOff = kXRing + kSlots * kXBytes;  // then the drain's 32 KB staging
constexpr uint32_t kAccCols = 2 * kRows;               // 64: X_hi products | X_lo products
constexpr int kAccBufs = 4;                              // accumulator buffers (chunks in flight MMA -> drain)
constexpr uint32_t kLoBase = kAccBufs * kAccCols;        // W_lo ring (one 32-column stage per slot)
constexpr uint32_t kTmemCols = 512;
static_assert(kLoBase + kTileK * kSlots <= kTmemCols, "TMEM budget");
constexpr uint32_t kStageBytes = kTileM * kRows * 8;    // drain staging: 2 halves x 128 features x 16 rows u64
constexpr float kFixScale = 4294967296.0f;               // 2^kMlpFixShift
constexpr float kFixInv = 1.0f / 4294967296.0f;
static_assert(kMlpFixShift == 32, "fixed-point scale");
constexpr int kCountBits = 9;                            // per-word completion count (nkt <= 256)
constexpr unsigned long long kCountMask = (1ull << kCountBits) - 1;
static_assert(kMlpMaxDim / kTileK < (1 << kCountBits), "count field");

__device__ __forceinline__ const char* translate(const char* arena, const uint32_t* pt, uint64_t v) {
    return arena + (static_cast<uint64_t>(pt[v >> kPageShift]) << kPageShift) + (v & kPageMask);
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// Debug build (make K1_DEBUG=1 -> -DGFX_K1_DEBUG): every wait has a watchdog
// that reports the stuck wait (CTA, warp, lane, site, step) and traps.
#ifdef GFX_K1_DEBUG
__device__ __forceinline__ void watchdog(long long& spins, int site, int g) {
    if (++spins == (1ll << 24))
        printf("K1 watchdog: cta %d warp %d lane %d site %d step %d\n", blockIdx.x, threadIdx.x >> 5, threadIdx.x & 31,
               site, g);
    if (spins == (1ll << 26)) __trap();
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// Phase marks per CTA (K1_MARK: first writer wins; K1_SET: last writer wins),
// copied to MlpFwdArgs::dbg[cta][32] at exit: 0 start, 1 setup; per layer
// l < 4 at 2 + 6 l: +0 first W landed, +1 first X word block complete, +2 first
// MMA issued, +3 last MMA complete (drain), +4 last partial's reds issued,
// +5 last step's X complete; 26 end.
#define K1_MARK(i)                                                         \
    do {                                                                   \
        if ((i) < 32) atomicCAS(&k1_marks[(i)], 0ull, gtime());            \
    } while (0)
#define K1_SET(i)                                \
    do {                                         \
        if ((i) < 32) k1_marks[(i)] = gtime();    \
    } while (0)
// Per-step marks of CTA 0 (steps < 96): dbg[grid * 32 + g * 8 + i], i = 0 W issued,
// 1 X issued, 2 W landed, 3 raw landed, 4 operand ready (converter), 5 MMA issued.
#define K1_STEP(g, i)                                                                         \
    do {                                                                                      \
        if (a.dbg && blockIdx.x == 0 && (g) < 96) a.dbg[gridDim.x * 32 + (g) * 8 + (i)] = gtime(); \
    } while (0)
#define K1_WAIT(bar, parity, site, g)                          \
    do {                                                       \
        long long spins_ = 0;                                  \
        while (!mbar_try((bar), (parity))) watchdog(spins_, (site), (g)); \
    } while (0)
#else
#define K1_WAIT(bar, parity, site, g) mbar_wait((bar), (parity))
#define K1_MARK(i) \
    do {           \
    } while (0)
#define K1_SET(i) \
    do {          \
    } while (0)
#define K1_STEP(g, i) \
    do {              \
    } while (0)
#endif
// Layer-output words once all K tiles of their feature tile are reduced into
// them: w[i] is the copy at hand (from the bulk copy), p[i] its address; every
// incomplete word is re-read from L2, all of them in flight at once, until each
// count equals `need`.
template <int kN>
__device__ __forceinline__ void complete_words(unsigned long long (&w)[kN], const unsigned long long* const (&p)[kN],
                                               unsigned need, int site = 0, int g = 0) {
#ifdef GFX_K1_DEBUG
    long long spins = 0;
#else
    (void)site;
    (void)g;
#endif
    for (;;) {
        bool done = true;
#pragma unroll
        for (int i = 0; i < kN; ++i) done &= (w[i] & kCountMask) == need;
        if (done) return;
        __nanosleep(32);
#pragma unroll
        for (int i = 0; i < kN; ++i)
            if ((w[i] & kCountMask) != need) w[i] = ld_relaxed_u64(p[i]);
#ifdef GFX_K1_DEBUG
        watchdog(spins, site, g);
#endif
    }
}
__device__ __forceinline__ float decode_word(unsigned long long w) {
    return __ll2float_rn(static_cast<long long>(w) >> kCountBits) * kFixInv;
}
__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 1, 128;\n" ::: "memory"); }
__device__ __forceinline__ void conv_sync(int group) {
    asm volatile("bar.sync %0, 128;\n" ::"r"(2 + group) : "memory");
}
__device__ __forceinline__ float rn_tf32(float v) {
    return __uint_as_float((__float_as_uint(v) + 0x1000u) & 0xFFFFE000u);
}
// Byte offset of element (row r, column c) in an operand block / weight tile row of 128 B.
__device__ __forceinline__ uint32_t sw128(int r, int c) {
    return static_cast<uint32_t>(r * 128 + ((((c >> 2) ^ (r & 7))) << 4) + (c & 3) * 4);
}

// This CTA's contiguous step range of a layer (stream-K split).
struct Range {
    int s0, s1;
};
__device__ __forceinline__ Range range_of(const MlpFwdLayer& ly, int cta, int grid) {
    const long long steps = static_cast<long long>(ly.tiles) * ly.nkt;
    return {static_cast<int>(steps * cta / grid), static_cast<int>(steps * (cta + 1) / grid)};
}
// End of the segment (steps of one feature tile) that starts at s.
__device__ __forceinline__ int seg_end(const MlpFwdLayer& ly, const Range& r, int s) {
    const int e = (s / ly.nkt + 1) * ly.nkt;
    return e < r.s1 ? e : r.s1;
}

__global__ void __launch_bounds__(kThreads, 1)
    mlp_forward_kernel(const __grid_constant__ MlpFwdArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ __align__(8) uint64_t w_full[kSlots], raw_full[kSlots], ready[kSlots], step_done[kSlots];
    __shared__ __align__(8) uint64_t tfull[kAccBufs], tempty[kAccBufs];
    // Layer-0 claims (a.claim): the W producer's claimed step ranges, read in order by every role.
    constexpr int kQ0 = 8;
    __shared__ __align__(8) uint64_t q0_full[kQ0], q0_empty[kQ0];
    __shared__ int2 q0_range[kQ0];
    __shared__ uint32_t tmem_base_s;
    __shared__ float red_s[2][4];
#ifdef GFX_K1_DEBUG
    __shared__ unsigned long long k1_marks[32];
    if (threadIdx.x < 32) k1_marks[threadIdx.x] = 0;
    __syncthreads();
    if (threadIdx.x == 0) K1_MARK(0);
#endif

    // PDL chain (a.pdl): the next forward may place its CTAs on SMs this one
    // frees (the softmax CTAs finish last), so its weight stream and layer 0 —
    // which share nothing with this launch — overlap this launch's tail. Only
    // what touches the layer-output buffers waits for this grid's predecessor
    // (griddepcontrol.wait: the drain before clearing / reducing, the X
    // producer before polling layer outputs). No-ops without the attribute.
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    const int cta = blockIdx.x;
    const int grid = a.grid;
    const int L = a.L;

    // The page table is read straight from the __grid_constant__ parameter (up to
    // GFX_MAX_PAGES entries, 4 KB: no room for a shared-memory copy).
    const uint32_t* const pt = a.pt.page;
    if (tid == 0) {
        for (int s = 0; s < kSlots; ++s) {
            mbar_init(&w_full[s], 1);
            mbar_init(&raw_full[s], 1);
            mbar_init(&ready[s], 4);      // the 4 converter warps of the step's group
            mbar_init(&step_done[s], 1);  // MMA commit: W, X and W_lo of the step consumed
        }
        for (int b = 0; b < kAccBufs; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 4);  // one arrival per drain warp
        }
        for (int i = 0; i < kQ0; ++i) {
            mbar_init(&q0_full[i], 1);
            mbar_init(&q0_empty[i], 1 + 8 + 2 + 4);  // X producer, converter warps, MMA warps, drain warps
        }
        mbar_fence_init();
        tma_prefetch_desc(&a.tmap_in);
    }
    if (warp == 1) tmem_alloc<kTmemCols>(&tmem_base_s);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_s;
    if (tid == 0) K1_MARK(1);

    // Step ranges of layer l: the static stream-K range once, or (layer 0 under a dynamic
    // split) the W producer's successive claims until its sentinel. A warp-wide role reads a
    // claim with every lane and releases it from lane 0; a single-lane role does both.
    const bool dyn0 = a.claim != nullptr;
    auto next_range = [&](int l, int jq, Range& r, bool single_lane) -> bool {
        if (l != 0 || !dyn0) {
            if (jq) return false;
            r = range_of(a.layer[l], cta, grid);
            return true;
        }
        const int qi = jq % kQ0;
        K1_WAIT(&q0_full[qi], (jq / kQ0) & 1, 12, jq);
        const int2 v = q0_range[qi];
        if (!single_lane) __syncwarp();
        if (single_lane || lane == 0) mbar_arrive(&q0_empty[qi]);
        r = Range{v.x, v.y};
        return v.x >= 0;
    };

    if (warp == 0) {
        // ---------------- W producer: never waits on activations ----------------
        if (lane == 0) {
            int g = 0;
            const int S0 = a.layer[0].tiles * a.layer[0].nkt;
            // Claims are software-pipelined: the atomic for claim j + 1 is issued before claim j's
            // steps, so its L2 round trip overlaps the ring waits instead of stalling the stream.
            unsigned claim_next = dyn0 ? atomicAdd(a.claim, 1u) : 0u;
            for (int l = 0; l < L; ++l) {
                const MlpFwdLayer& ly = a.layer[l];
              for (int jq = 0;; ++jq) {
                Range r;
                if (l == 0 && dyn0) {
                    // Claim the next kMlpChunk0 steps of layer 0 (a CTA that started late — under
                    // the PDL chain launch CTAs start over a ~5 µs window — simply claims fewer).
                    const int qi = jq % kQ0;
                    if (jq >= kQ0) K1_WAIT(&q0_empty[qi], ((jq / kQ0) & 1) ^ 1, 11, jq);
                    const int s0 = static_cast<int>(claim_next) * kMlpChunk0;
                    r = s0 < S0 ? Range{s0, s0 + kMlpChunk0 < S0 ? s0 + kMlpChunk0 : S0} : Range{-1, -1};
                    if (r.s0 >= 0) claim_next = atomicAdd(a.claim, 1u);  // (monotonic: none valid is ever dropped)
                    q0_range[qi] = make_int2(r.s0, r.s1);
                    mbar_arrive(&q0_full[qi]);
                    if (r.s0 < 0) break;
                } else {
                    if (jq) break;
                    r = range_of(ly, cta, grid);
                }
                for (int s = r.s0; s < r.s1;) {
                    const int slot = g % kSlots;
                    const bool pair = (g & 1) == 0 && s + 1 < r.s1;  // steps g, g+1 of this range
                    if (g >= kSlots) K1_WAIT(&step_done[slot], ((g / kSlots) & 1) ^ 1, 1, g);
                    if (pair && g + 1 >= kSlots) K1_WAIT(&step_done[slot + 1], (((g + 1) / kSlots) & 1) ^ 1, 1, g + 1);
                    K1_STEP(g, 0);
                    const uint64_t v = ly.w_off + static_cast<uint64_t>(s) * kWBytes;
                    const char* src = translate(a.arena, pt, v);
                    uint8_t* dst = smem + slot * kWBytes;
                    mbar_arrive_expect_tx(&w_full[slot], pair ? 2 * kWBytes : kWBytes);
                    if (pair && translate(a.arena, pt, v + kWBytes) == src + kWBytes) {
                        tma_bulk_g2s(dst, src, 2 * kWBytes, &w_full[slot]);
                    } else {
                        tma_bulk_g2s(dst, src, kWBytes, &w_full[slot]);
                        if (pair) tma_bulk_g2s(dst + kWBytes, translate(a.arena, pt, v + kWBytes), kWBytes, &w_full[slot]);
                    }
                    if (pair) mbar_arrive(&w_full[slot + 1]);
                    s += pair ? 2 : 1;
                    g += pair ? 2 : 1;
                }
              }
            }
        }
    } else if (warp == 14) {
        // ---------------- X producer: the raw input block of each step ----------------
        if (lane == 0) {
            int g = 0;
            for (int l = 0; l < L; ++l) {
                const MlpFwdLayer& ly = a.layer[l];
                Range r;
              for (int jq = 0; next_range(l, jq, r, true); ++jq) {
                const unsigned long long* src_act = l > 0 ? a.act + a.layer[l - 1].act_off : nullptr;
                int seen = -1;  // last source tile seen complete
                // Wait until source tile kt >> 2 shows a complete word (its partials have landed).
                auto await_source = [&](int kt, int g_) {
                    const int src = kt >> 2;  // the previous layer's feature tile holding these 32 inputs
                    if (src == seen) return;
                    const unsigned long long* w = src_act + static_cast<size_t>(kt) * (kTileK * kRows) + 32 * 32 - 1;
                    unsigned long long v[1] = {ld_relaxed_u64(w)};
                    const unsigned long long* pp[1] = {w};
                    complete_words(v, pp, static_cast<unsigned>(a.layer[l - 1].nkt), 10, g_);
                    seen = src;
                };
                if (l == 1 && jq == 0) asm volatile("griddepcontrol.wait;\n" ::: "memory");  // the buffers' clear by the predecessor
                for (int s = r.s0; s < r.s1;) {
                    const int slot = g % kSlots, kt = s % ly.nkt;
                    const bool pair = l > 0 && (g & 1) == 0 && s + 1 < r.s1;
                    if (g >= kSlots) K1_WAIT(&step_done[slot], ((g / kSlots) & 1) ^ 1, 2, g);
                    if (pair && g + 1 >= kSlots) K1_WAIT(&step_done[slot + 1], (((g + 1) / kSlots) & 1) ^ 1, 2, g + 1);
                    uint8_t* xs = smem + kXRing + slot * kXBytes;
                    K1_STEP(g, 1);
                    if (l == 0) {
                        mbar_arrive_expect_tx(&raw_full[slot], kRaw0Bytes);
                        tma_tile2d_g2s(xs + kRaw0Bytes, &a.tmap_in, kt * kTileK, 0, &raw_full[slot]);
                    } else {
                        const int kt1 = (s + 1) % ly.nkt;  // the pair's second K tile
                        await_source(kt, g);
                        if (pair) await_source(kt1, g + 1);
                        mbar_arrive_expect_tx(&raw_full[slot], pair ? 2 * kRawBytes : kRawBytes);
                        const unsigned long long* b0 = src_act + static_cast<size_t>(kt) * (kTileK * kRows);
                        if (pair && kt1 == kt + 1) {
                            tma_bulk_g2s(xs, b0, 2 * kRawBytes, &raw_full[slot]);
                        } else {
                            tma_bulk_g2s(xs, b0, kRawBytes, &raw_full[slot]);
                            if (pair)
                                tma_bulk_g2s(xs + kRawBytes, src_act + static_cast<size_t>(kt1) * (kTileK * kRows), kRawBytes,
                                             &raw_full[slot]);
                        }
                        if (pair) mbar_arrive(&raw_full[slot + 1]);
                    }
                    s += pair ? 2 : 1;
                    g += pair ? 2 : 1;
                }
              }
            }
        }
    } else if (warp == 1 || warp == 15) {
        // ---------------- MMA issuers: two warps take alternate accumulator chunks ----------------
        // Each issuing warp loops converged (one elected lane issues). With two,
        // one issues while the other waits on its barriers. Chunks never span
        // two tiles; chunks of one tile accumulate in different TMEM buffers and
        // are summed by the drain in chunk order.
        const int issuer = warp == 1 ? 0 : 1;
        constexpr uint32_t idesc64 = umma_idesc<kTileM, 2 * kRows, 2>();  // TF32 x TF32 -> F32, N = 64
        constexpr uint32_t idesc32 = umma_idesc<kTileM, kRows, 2>();      // N = 32
        int g = 0, chunk = 0;
        for (int l = 0; l < L; ++l) {
            const MlpFwdLayer& ly = a.layer[l];
            Range r;
          for (int jq = 0; next_range(l, jq, r, false); ++jq) {
            for (int s = r.s0; s < r.s1;) {
                const int e = seg_end(ly, r, s);
                for (; s < e; ++chunk) {
                    const int len = e - s < kChunk ? e - s : kChunk;
                    if ((chunk & 1) != issuer) {
                        s += len;
                        g += len;
                        continue;
                    }
                    const int buf = chunk % kAccBufs;
                    const uint32_t acc = tmem + static_cast<uint32_t>(buf * kAccCols);
                    if (chunk >= kAccBufs) K1_WAIT(&tempty[buf], ((chunk / kAccBufs) & 1) ^ 1, 4, g);
                    for (int j = 0; j < len; ++j, ++s, ++g) {
                        const int slot = g % kSlots;
                        K1_WAIT(&ready[slot], (g / kSlots) & 1, 5, g);  // W landed, W_lo staged, X operand built
                        tc_fence_after();
                        if (l < 4 && lane == 0) K1_MARK(4 + 6 * l);
                        if (l == 1 && lane == 0 && s == r.s0) K1_MARK(29);
                        const uint64_t bx = umma_desc_sw128(smem + kXRing + slot * kXBytes, 0);
                        const uint64_t aw = umma_desc_sw128(smem + slot * kWBytes, 0);
                        const uint32_t lo = tmem + kLoBase + static_cast<uint32_t>(kTileK * slot);
#pragma unroll
                        for (int kk = 0; kk < kTileK / 8; ++kk) {
                            // +kk*32 bytes = +2 in the descriptor's 16-byte address units
                            umma_tf32_elect(acc, aw + 2 * kk, bx + 2 * kk, idesc64, (j == 0 && kk == 0) ? 0u : 1u);
                            umma_tf32_ts_elect(acc, lo + static_cast<uint32_t>(8 * kk), bx + 2 * kk, idesc32, 1u);
                        }
                        umma_commit_elect(&step_done[slot]);  // slot + W_lo stage free once these MMAs retire
                        if (lane == 0) K1_STEP(g, 5);
                    }
                    umma_commit_elect(&tfull[buf]);
                }
            }
          }
        }
    } else if (warp < 10) {
        // ---------------- converters: W_lo -> TMEM stage, raw X -> operand ----------------
        const int group = (warp - 2) >> 2;
        const int q = warp & 3;            // TMEM lane quarter of this warp
        const int r = q * 32 + lane;       // weight row of the tile = TMEM lane
        int g = 0;
        for (int l = 0; l < L; ++l) {
            const MlpFwdLayer& ly = a.layer[l];
            Range rg;
          for (int jq = 0; next_range(l, jq, rg, false); ++jq) {
            for (int s = rg.s0; s < rg.s1; ++s, ++g) {
                if ((g & 1) != group) continue;
                const int slot = g % kSlots;
                uint8_t* xs = smem + kXRing + slot * kXBytes;
                // The second step of a producer pair (odd g, not the layer's first step
                // here) landed with the first: wait on the first slot's barrier.
                const bool second = (g & 1) && s > rg.s0;
                K1_WAIT(&w_full[second ? slot - 1 : slot], (g / kSlots) & 1, 6, g);
                // The producer's plain arrive on the second slot's barrier (its phase completes at once):
                // consumed here, so every phase of every barrier has a waiter (compute-sanitizer synccheck).
                if (second) K1_WAIT(&w_full[slot], (g / kSlots) & 1, 6, g);
                if (q == 0 && lane == 0) K1_STEP(g, 2);
                if (l < 4 && lane == 0) K1_MARK(2 + 6 * l);
                // Stage `slot` of the W_lo ring was last read by the MMAs of step
                // g - kSlots, which the producer waited on before this tile landed.
                const float4* wrow = reinterpret_cast<const float4*>(smem + slot * kWBytes + r * 128);
                float wlo[32];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const float4 v = wrow[j ^ (r & 7)];
                    wlo[4 * j + 0] = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
                    wlo[4 * j + 1] = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
                    wlo[4 * j + 2] = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
                    wlo[4 * j + 3] = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
                }
                tc_fence_after();
                tmem_st_32x32b_x32(tmem + (static_cast<uint32_t>(q * 32) << 16) + kLoBase + static_cast<uint32_t>(kTileK * slot), wlo);
                if (q == 0 && lane == 0) K1_STEP(g, 6);
                // X: warp q converts K columns 8q .. 8q+7 (16-byte chunks 2q, 2q+1) of all 32 rows; lane = batch row.
                K1_WAIT(&raw_full[second && l > 0 ? slot - 1 : slot], (g / kSlots) & 1, 7, g);
                if (second && l > 0) K1_WAIT(&raw_full[slot], (g / kSlots) & 1, 7, g);
                if (q == 0 && lane == 0) K1_STEP(g, 3);
                if (l == 0 && lane == 0) {
                    K1_MARK(3);
                    K1_SET(7);
                }
                float4 xv[2];
                if (l == 0) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) xv[h] = *reinterpret_cast<const float4*>(xs + kRaw0Bytes + sw128(lane, 8 * q + 4 * h));
                } else {
                    // Fixed-point feature-major block: raw[f][b] at f * 256 + b * 8; words whose
                    // count is short are re-read from L2. Hidden inputs get the ReLU here.
                    const unsigned long long* rawq = reinterpret_cast<const unsigned long long*>(xs);
                    const unsigned long long* gsrc =
                        a.act + a.layer[l - 1].act_off + static_cast<size_t>(s % ly.nkt) * (kTileK * kRows);
                    const unsigned need = static_cast<unsigned>(a.layer[l - 1].nkt);
                    unsigned long long wv[8];
                    const unsigned long long* wp[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        wv[i] = rawq[(8 * q + i) * 32 + lane];
                        wp[i] = gsrc + (8 * q + i) * 32 + lane;
                    }
                    complete_words(wv, wp, need, 3, g);
                    float x[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) x[i] = fmaxf(decode_word(wv[i]), 0.f);
                    if (l < 4 && lane == 0) {
                        K1_MARK(3 + 6 * l);
                        K1_SET(7 + 6 * l);
                    }
                    xv[0] = make_float4(x[0], x[1], x[2], x[3]);
                    xv[1] = make_float4(x[4], x[5], x[6], x[7]);
                    conv_sync(group);  // every warp of the group has read its raw rows before the operand overwrites them
                    if (q == 0 && lane == 0) K1_STEP(g, 7);
                    if (l == 1 && lane == 0) K1_MARK(27);
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    float4 hi, lo;
                    hi.x = rn_tf32(xv[h].x);
                    hi.y = rn_tf32(xv[h].y);
                    hi.z = rn_tf32(xv[h].z);
                    hi.w = rn_tf32(xv[h].w);
                    lo.x = xv[h].x - hi.x;
                    lo.y = xv[h].y - hi.y;
                    lo.z = xv[h].z - hi.z;
                    lo.w = xv[h].w - hi.w;
                    *reinterpret_cast<float4*>(xs + sw128(lane, 8 * q + 4 * h)) = hi;
                    *reinterpret_cast<float4*>(xs + sw128(kRows + lane, 8 * q + 4 * h)) = lo;
                }
                fence_proxy_async_smem();  // generic-proxy writes -> tensor core reads
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&ready[slot]);
                if (l == 1 && lane == 0) K1_MARK(28);
                if (q == 0 && lane == 0) K1_STEP(g, 4);
            }
          }
        }
    } else if (warp < 14) {
        // ---------------- drain + epilogue warps ----------------
        const int ct = tid - 320;          // 0..127
        const int q = warp & 3;            // TMEM lane quarter (warps 10..13 -> 2,3,0,1)
        const int fl = q * 32 + lane;      // feature row within the tile

        // The other parity's buffer, for the next launch, once the previous launch
        // (its owner) has completed; also orders this launch's reductions after it.
        asm volatile("griddepcontrol.wait;\n" ::: "memory");
        for (uint32_t i = static_cast<uint32_t>(cta * 128 + ct); i < a.clear_vec; i += static_cast<uint32_t>(grid * 128))
            a.act_clear[i] = make_uint4(0u, 0u, 0u, 0u);
        // The launch before the predecessor has completed: its claim counter is free for launch + 2.
        if (cta == 0 && ct == 0 && a.claim_reset) atomicExch(a.claim_reset, 0u);
        // Staging (after the ring): half h holds rows 16h..16h+15 as [128 features][128 B], 16-byte chunk j of
        // feature f at j ^ (f & 7) (the TMA SWIZZLE_128B image); warp q owns features 32q..32q+31 of both halves.
        uint8_t* const stg = smem + kStageOff;

        int chunk = 0;
        for (int l = 0; l < L; ++l) {
            const MlpFwdLayer& ly = a.layer[l];
            Range r;
          for (int jq = 0; next_range(l, jq, r, false); ++jq) {
            for (int s = r.s0; s < r.s1;) {
                const int e = seg_end(ly, r, s);
                const int tile = s / ly.nkt;
                const int f = tile * kTileM + fl;
                // Bias row fetched before the MMAs finish (off the boundary's critical path).
                const float bias = (s % ly.nkt) == 0 && f < ly.N
                                       ? *reinterpret_cast<const float*>(translate(a.arena, pt, ly.b_off + 4ull * f))
                                       : 0.f;
                const unsigned long long count = static_cast<unsigned long long>(e - s);  // K tiles of this partial
                float acc[kRows];
#pragma unroll
                for (int b = 0; b < kRows; ++b) acc[b] = 0.f;
                for (; s < e; ++chunk) {
                    const int len = e - s < kChunk ? e - s : kChunk;
                    s += len;
                    K1_WAIT(&tfull[chunk % kAccBufs], (chunk / kAccBufs) & 1, 8, chunk);
                    tc_fence_after();
                    float ph[kRows], pl[kRows];
                    const uint32_t src = tmem + static_cast<uint32_t>((chunk % kAccBufs) * kAccCols) + (static_cast<uint32_t>(q * 32) << 16);
                    tmem_ld_32x32b_x32(src + kRows, pl);  // products with X_lo (small)
                    tmem_ld_32x32b_x32(src, ph);
#pragma unroll
                    for (int b = 0; b < kRows; ++b) acc[b] += ph[b] + pl[b];
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&tempty[chunk % kAccBufs]);
                }
                if (l < 4 && ct == 0 && e == r.s1) K1_SET(5 + 6 * l);
                if (lane == 0) bulk_wait_group_read<0>();  // the previous segment's reductions have read the staging
                __syncwarp();
#pragma unroll
                for (int j = 0; j < kRows / 2; ++j) {
                    const unsigned long long q0 =
                        (static_cast<unsigned long long>(__float2ll_rn((acc[2 * j] + bias) * kFixScale)) << kCountBits) + count;
                    const unsigned long long q1 =
                        (static_cast<unsigned long long>(__float2ll_rn((acc[2 * j + 1] + bias) * kFixScale)) << kCountBits) +
                        count;
                    *reinterpret_cast<ulonglong2*>(stg + (j >> 3) * (kStageBytes / 2) + fl * 128 + (((j & 7) ^ (fl & 7)) << 4)) =
                        make_ulonglong2(q0, q1);
                }
                fence_proxy_async_smem();  // generic-proxy writes -> the TMA engine's reads
                __syncwarp();
                if (lane == 0 && tile * kTileM + q * 32 < ly.N) {  // rows >= N: zero padding, clipped by the map
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        tma_reduce_add_2d(&a.tmap_out[l], 16 * h, tile * kTileM + q * 32, stg + h * (kStageBytes / 2) + q * 4096);
                    bulk_commit_group();
                }
                if (l < 4 && ct == 0) K1_SET(6 + 6 * l);
            }
          }
        }

        if (lane == 0) bulk_wait_group<0>();  // every reduction of this CTA issued and complete

        // Softmax rows: batch row b = cta, from the last layer's words once complete.
        if (cta < kRows) {
            const MlpFwdLayer& ly = a.layer[L - 1];
            const int C = ly.N;
            const unsigned need = static_cast<unsigned>(ly.nkt);
            const unsigned long long* in = a.act + ly.act_off;  // [C][32]
            float* lg = a.logits + static_cast<size_t>(cta) * C;
            float* pr = a.probs + static_cast<size_t>(cta) * C;
            constexpr int kPer = kMlpMaxClasses / 128;
            unsigned long long wv[kPer];
            const unsigned long long* wp[kPer];
#pragma unroll
            for (int i = 0; i < kPer; ++i) {  // columns past C: a complete dummy word
                const int c = ct + i * 128;
                wp[i] = in + static_cast<size_t>(c < C ? c : 0) * kRows + cta;
                wv[i] = c < C ? ld_relaxed_u64(wp[i]) : need;
            }
            complete_words(wv, wp, need, 9, 0);
            float v[kPer];
            float m = -INFINITY;
#pragma unroll
            for (int i = 0; i < kPer; ++i) {
                const int c = ct + i * 128;
                v[i] = c < C ? decode_word(wv[i]) : -INFINITY;
                if (c < C) lg[c] = v[i];
                m = fmaxf(m, v[i]);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (lane == 0) red_s[0][q] = m;
            epi_sync();
            m = fmaxf(fmaxf(red_s[0][0], red_s[0][1]), fmaxf(red_s[0][2], red_s[0][3]));
            float sum = 0.f;
#pragma unroll
            for (int i = 0; i < kPer; ++i) {
                const int c = ct + i * 128;
                v[i] = c < C ? expf(v[i] - m) : 0.f;
                sum += v[i];
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
            if (lane == 0) red_s[1][q] = sum;
            epi_sync();
            const float inv = 1.0f / (red_s[1][0] + red_s[1][1] + red_s[1][2] + red_s[1][3]);
#pragma unroll
            for (int i = 0; i < kPer; ++i) {
                const int c = ct + i * 128;
                if (c < C) pr[c] = v[i] * inv;
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc<kTmemCols>(tmem);
#ifdef GFX_K1_DEBUG
    if (tid == 0) K1_MARK(26);
    __syncthreads();
    if (a.dbg && tid < 32) a.dbg[cta * 32 + tid] = k1_marks[tid];
#endif
}

}  // namespace

void mlp_debug_report(const unsigned long long* dbg, int grid, int L, int model, cudaStream_t s) {
    std::vector<unsigned long long> m(static_cast<size_t>(grid) * 32 + 96 * 8);
    GFX_CUDA(cudaStreamSynchronize(s));
    GFX_CUDA(cudaMemcpy(m.data(), dbg, m.size() * 8, cudaMemcpyDeviceToHost));
    unsigned long long t0 = ~0ull;
    for (int c = 0; c < grid; ++c) t0 = std::min(t0, m[static_cast<size_t>(c) * 32]);
    static const char* nm[6] = {"W landed", "X complete", "MMA first", "MMA done", "reds issued", "last X cplt"};
    std::fprintf(stderr, "[K1 model %d] us after first CTA start: min p10 median p90 max over %d CTAs\n", model, grid);
    for (int i = 0; i < 30; ++i) {
        std::vector<double> v;
        for (int c = 0; c < grid; ++c)
            if (m[static_cast<size_t>(c) * 32 + i]) v.push_back((m[static_cast<size_t>(c) * 32 + i] - t0) * 1e-3);
        if (v.empty() || (i >= 2 && i < 26 && (i - 2) / 6 >= L)) continue;
        std::sort(v.begin(), v.end());
        char name[40];
        if (i == 0) std::snprintf(name, sizeof name, "start");
        else if (i == 1) std::snprintf(name, sizeof name, "setup");
        else if (i == 26) std::snprintf(name, sizeof name, "end");
        else if (i == 27) std::snprintf(name, sizeof name, "L1 grp words cplt");
        else if (i == 28) std::snprintf(name, sizeof name, "L1 ready arrive");
        else if (i == 29) std::snprintf(name, sizeof name, "L1 MMA saw step0");
        else std::snprintf(name, sizeof name, "L%d %s", (i - 2) / 6, nm[(i - 2) % 6]);
        const size_t n = v.size();
        std::fprintf(stderr, "  %-18s %7.2f %7.2f %7.2f %7.2f %7.2f\n", name, v[0], v[n / 10], v[n / 2], v[n * 9 / 10],
                     v[n - 1]);
    }
    std::fprintf(stderr, "  CTA 0 steps (us): W issued, X issued, W landed, raw landed, operand ready, MMA issued, W_lo stored, X read\n");
    for (int g = 0; g < 96; ++g) {
        const unsigned long long* p = m.data() + static_cast<size_t>(grid) * 32 + g * 8;
        if (!p[0] && !p[2]) break;  // (odd steps of a producer pair have no issue mark of their own)
        auto us = [&](unsigned long long t) { return t ? (t - t0) * 1e-3 : -1.0; };
        std::fprintf(stderr, "   %2d %7.2f %7.2f %7.2f %7.2f %7.2f %7.2f %7.2f %7.2f\n", g, us(p[0]), us(p[1]), us(p[2]), us(p[3]),
                     us(p[4]), us(p[5]), us(p[6]), us(p[7]));
    }
    GFX_CUDA(cudaMemset(const_cast<unsigned long long*>(dbg), 0, m.size() * 8));
}

size_t mlp_fwd_smem() { return static_cast<size_t>(kStageOff) + kStageBytes + 1024; }

void launch_mlp_forward(MlpFwdArgs& a, cudaStream_t stream) {
    if (a.L < 1 || a.L > GFX_MAX_LAYERS) throw std::runtime_error("mlp forward: bad layer count");
    uint64_t act = 0;
    for (int l = 0; l < a.L; ++l) {
        const MlpFwdLayer& ly = a.layer[l];
        if (ly.K % kTileK || ly.K <= 0 || ly.N <= 0 || ly.K > kMlpMaxDim || ly.N > kMlpMaxDim ||
            ly.tiles != (ly.N + kTileM - 1) / kTileM || ly.nkt != ly.K / kTileK || ly.act_off != act)
            throw std::runtime_error("mlp forward: unsupported layer shape");
        if (l > 0 && a.layer[l - 1].N != ly.K) throw std::runtime_error("mlp forward: layer widths do not chain");
        act += static_cast<uint64_t>(ly.N) * kRows;
    }
    if (act > kMlpActWords) throw std::runtime_error("mlp forward: layer outputs exceed the workspace");
    if (a.layer[a.L - 1].N > kMlpMaxClasses || a.grid < kRows)
        throw std::runtime_error("mlp forward: at most 2048 classes, grid >= 32");
    // Layer outputs: [N][32] u64 rows, boxes of 16 words x 32 features, SWIZZLE_128B (the drain's staging image).
    for (int l = 0; l < a.L; ++l)
        if (!encode_tensor_map_2d(&a.tmap_out[l], CU_TENSOR_MAP_DATA_TYPE_UINT64, 8, a.act + a.layer[l].act_off, kRows,
                                  static_cast<uint64_t>(a.layer[l].N), kRows * 8, 16, 32, CU_TENSOR_MAP_SWIZZLE_128B))
            throw CudaError("cuTensorMapEncodeTiled failed for a layer output");
    // Layer-0 input tiles: 32 x 32 fp32 boxes of the [32 x K0] request input, SWIZZLE_128B.
    if (!encode_tensor_map_2d(&a.tmap_in, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, a.in, static_cast<uint64_t>(a.layer[0].K),
                              kRows, static_cast<uint64_t>(a.layer[0].K) * 4, kTileK, kRows, CU_TENSOR_MAP_SWIZZLE_128B))
        throw CudaError("cuTensorMapEncodeTiled failed for the request input");
    const size_t smem = mlp_fwd_smem();
    ensure_max_dynamic_smem(reinterpret_cast<const void*>(mlp_forward_kernel), static_cast<int>(smem));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(a.grid));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    // Every CTA must become resident (CTAs wait on each other's partials):
    // cooperative launch, or — on a device this process's one manager owns —
    // a PDL-chained launch whose CTAs take SMs as the previous forward frees them.
    cudaLaunchAttribute attr[1];
    if (a.pdl) {
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
    } else {
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
    }
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    GFX_CUDA(cudaLaunchKernelEx(&cfg, mlp_forward_kernel, a));
}

}  // namespace gfx
