// K1 v6: the whole fp32 MLP forward of one request (batch 32) in ONE persistent
// cooperative launch on the 5th-gen tensor cores (tcgen05, kind::tf32, 3xTF32
// error compensation), weights streamed by TMA straight out of the paged HBM
// arena. Replaces profile.infer_time_us (proj/src/cluster.cpp:161,167).
//
//   layer l: Y_l[32 x N] = act(X_l[32 x K] . W_l^T + b_l)  as  D^T[N x 32] = W_l . X_l^T
//   (swap AB: 128 weight rows fill the MMA M side, the 32 batch rows are N),
//   act = ReLU on hidden layers; the last layer's rows also go through softmax.
//
// Why one launch (profiles/r1_k1_v5_ncu.md): a layer of a C2 model is 7-13 MB
// of weights, 1-2 µs of HBM time, but a per-layer launch cost 12-15 µs of
// prologue, pipeline fill and split-K tail. Here every CTA streams the weight
// tiles of ALL its layers back to back through one TMA ring — weights do not
// depend on activations — so the HBM never idles at a layer boundary; only the
// (small) activation operands wait, on per-tile dataflow flags set by the
// CTAs that reduced the previous layer's tile. No grid barrier, no relaunch.
//
// Work split per layer: unit u = blockIdx.x < tiles x splits -> feature tile
// u % tiles (128 outputs), K split u / tiles (a contiguous range of 32-wide K
// tiles). Split-K partials are reduced by the split CTAs of the tile, each
// owning the batch rows b = split (mod splits), summed in fixed split order
// (deterministic). The reducer writes the next layer's operand directly in the
// tensor-core layout (see "operand block" below), so no CTA re-splits inputs.
//
// Precision (north-star fp32 tolerance 1e-5): the tensor core reads W straight
// from the landed fp32 tile; kind::tf32 uses only the top 19 bits, i.e.
// W_hi = trunc_tf32(W) (verified on B200: taking W_hi as the rounded value
// instead breaks parity, 1.4e-3). Converter warps form W_lo = W - W_hi (exact
// in fp32, |W_lo| < 2^-10 |W|) into a TMEM ring. Activations are pre-split by
// their producer: X_hi = rn_tf32(X), X_lo = X - X_hi (exact). Per 8-wide K slice:
//   D += W_hi . [X_hi; X_lo]   (SS, N = 64: both batch planes at once)
//   D += W_lo . X_hi           (TS, A from TMEM, N = 32; B rows just read)
// Measured per 32-wide K step (tools/issue_rate.cu, rotating ring slots): this
// pair costs ~556 cycles, vs ~1081 with W_hi also from TMEM and ~1007 for the
// two N = 64 TMEM products of K1 v5.
// i.e. every product but W_lo.X_lo (< 2^-21 relative); the accumulator keeps
// the X_hi / X_lo columns apart and is drained to fp32 registers every kChunk
// K tiles (short tensor-core accumulation chains at any K).
//
// Operand block (global, per 32-wide K tile of a layer input, 8 KB): 64 rows x
// 128 B — rows 0-31 = X_hi of batch rows 0-31, rows 32-63 = X_lo — with the
// SWIZZLE_128B chunk permutation (16-byte chunk j of row r at j ^ (r & 7)), so
// a 1-D bulk copy into a 1024-aligned smem slot is the MMA's B operand as is.
//
// Roles (16 warps, one CTA per SM, 8-deep ring of 24 KB slots = W 16 KB + X 8 KB):
//   warp 0        W producer: 1-D bulk TMA of each 16 KB pre-swizzled weight tile
//   warp 14       X producer: layer 0 splits the request input into the slot;
//                 later layers wait for the tile's dataflow flag, bulk TMA 8 KB
//   warps 2-5/6-9 converters (two groups, alternate K tiles): W_lo -> TMEM ring
//   warps 1, 15   MMA issuers, alternate accumulator chunks: 8 MMAs per K tile
//                 and ONE commit per step (slot, operand and W_lo stage share
//                 a step_done barrier)
//   warps 10-13   drain (TMEM -> fp32 registers per chunk) and epilogue
//                 (split-K reduction, bias, ReLU, next-layer operand / logits),
//                 softmax rows at the end.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <stdexcept>

#include "common.cuh"
#include "mlp.cuh"
#include "sm100.cuh"

namespace gfx {

namespace {

using namespace gfx::sm100;

constexpr int kRows = 32;     // batch rows per request
constexpr int kTileM = 128;   // output features per unit = MMA M
constexpr int kTileK = 32;    // fp32 K per ring step (one 128-byte swizzle row)
constexpr int kSlots = 8;     // ring depth: 8 x 16 KB = 128 KB of weights in flight per SM
constexpr int kChunk = 4;     // K tiles accumulated in TMEM before a drain
constexpr int kThreads = 16 * 32;
constexpr uint32_t kWBytes = kTileM * kTileK * 4;      // 16 KB
constexpr uint32_t kXBytes = 2 * kRows * kTileK * 4;   // 8 KB: [X_hi; X_lo]
constexpr uint32_t kSlotBytes = kWBytes + kXBytes;     // 24 KB (1024-aligned)
constexpr uint32_t kAccCols = 2 * kRows;               // 64: X_hi products | X_lo products
constexpr int kAccBufs = 4;                              // accumulator buffers (chunks in flight MMA -> drain)
constexpr uint32_t kLoBase = kAccBufs * kAccCols;        // W_lo ring (one 32-column stage per slot)
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kGatherBytes = 64 * kTileM * 4;     // split-K gather: <= 63 partial rows of 512 B
static_assert(kLoBase + kTileK * kSlots <= kTmemCols, "TMEM budget");

// counters (u32), zero between launches (the last CTA out resets them)
constexpr int kCntArrive = 0;                        // [layer][tile] split partials published
constexpr int kCntDone = GFX_MAX_LAYERS * 64;         // [layer][tile] split rows reduced + written
constexpr int kCntFinal = 2 * GFX_MAX_LAYERS * 64;    // last-layer units finished
// Two banks alternate by launch parity: a launch zeroes the bank the previous
// (stream-ordered, finished) launch used, off its critical path, so no CTA has
// to reset counters at the end.
constexpr int kCntBank = kCntFinal + 64;
static_assert(2 * kCntBank <= kMlpCounters, "counter banks");

__device__ __forceinline__ const char* translate(const char* arena, const uint32_t* pt, uint64_t v) {
    return arena + (static_cast<uint64_t>(pt[v >> kPageShift]) << kPageShift) + (v & kPageMask);
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void wait_count(const unsigned* p, unsigned target) {
    while (ld_acquire(p) < target) {
    }
}
// Release/acquire fence at GPU scope (MEMBAR.ALL.GPU), not __threadfence()'s
// sequentially consistent MEMBAR.SC.GPU: the dataflow flags only need
// "writes before the flag are visible to whoever acquires it".
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 1, 128;\n" ::: "memory"); }
__device__ __forceinline__ float rn_tf32(float v) {
    return __uint_as_float((__float_as_uint(v) + 0x1000u) & 0xFFFFE000u);
}
// Byte offset of element (row r, column c) in an operand block / weight tile row of 128 B.
__device__ __forceinline__ uint32_t sw128(int r, int c) {
    return static_cast<uint32_t>(r * 128 + ((((c >> 2) ^ (r & 7))) << 4) + (c & 3) * 4);
}

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// Per-step timeline of CTA 0 (GFX_TRACE_MLP): 8 %globaltimer marks per ring step.
__device__ __forceinline__ void smark(unsigned long long* tr, int step, int i) {
    if (tr == nullptr || blockIdx.x != 0 || step >= 64) return;
    tr[static_cast<size_t>(gridDim.x) * 32 + step * 8 + i] = gtime();
}
// Per-CTA cycle accounting (GFX_TRACE_MLP): where each role's time goes.
struct Prof {
    long long t = 0;
    __device__ __forceinline__ void start() { t = clock64(); }
    __device__ __forceinline__ void stop(long long& acc) {
        const long long n = clock64();
        acc += n - t;
        t = n;
    }
};
__device__ __forceinline__ void prof_store(unsigned long long* tr, int i, long long v) {
    if (tr) tr[static_cast<size_t>(gridDim.x) * 32 + 576 + blockIdx.x * 16 + i] = static_cast<unsigned long long>(v);
}
// Debug timeline (GFX_TRACE_MLP): %globaltimer per CTA at phase boundaries.
__device__ __forceinline__ void mark(unsigned long long* tr, int i) {
    if (tr == nullptr) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    tr[blockIdx.x * 32 + i] = t;
}

struct Unit {
    bool valid;
    int tile, split, kt0, nkt, kt_total;
};
__device__ __forceinline__ Unit unit_of(const MlpFwdLayer& ly, int cta, int cluster) {
    Unit u{};
    if (cluster) {
        // Cluster mode: the S splits of a tile are adjacent ranks of one cluster
        // (S divides the cluster size), cluster c holds tiles c * (cluster / S) + ...
        const int per = cluster / ly.splits, rank = cta % cluster, lt = rank / ly.splits;
        u.tile = (cta / cluster) * per + lt;
        u.split = rank % ly.splits;
        u.valid = u.tile < ly.tiles;
    } else {
        const int units = ly.tiles * ly.splits;
        u.valid = cta < units;
        u.tile = cta % ly.tiles;
        u.split = cta / ly.tiles;
    }
    if (!u.valid) return u;
    u.kt_total = ly.K / kTileK;
    u.kt0 = static_cast<int>((static_cast<long long>(u.kt_total) * u.split) / ly.splits);
    const int kt1 = static_cast<int>((static_cast<long long>(u.kt_total) * (u.split + 1)) / ly.splits);
    u.nkt = kt1 - u.kt0;
    return u;
}

// Walk of one CTA's weight tiles over all layers (the W producer's order).
struct WIter {
    int l, it;
    Unit u;
};
__device__ __forceinline__ bool witer_seek(const MlpFwdArgs& a, int cta, WIter& w) {
    for (; w.l < a.L; ++w.l) {
        w.u = unit_of(a.layer[w.l], cta, a.cluster);
        if (w.u.valid) {
            w.it = 0;
            return true;
        }
    }
    return false;
}
__device__ __forceinline__ bool witer_first(const MlpFwdArgs& a, int cta, WIter& w) {
    w.l = 0;
    return witer_seek(a, cta, w);
}
__device__ __forceinline__ bool witer_next(const MlpFwdArgs& a, int cta, WIter& w) {
    if (++w.it < w.u.nkt) return true;
    ++w.l;
    return witer_seek(a, cta, w);
}
__device__ __forceinline__ uint64_t witer_off(const MlpFwdArgs& a, const WIter& w) {
    return a.layer[w.l].w_off + (static_cast<uint64_t>(w.u.tile) * w.u.kt_total + w.u.kt0 + w.it) * kWBytes;
}

__global__ void __launch_bounds__(kThreads, 1)
    mlp_forward_kernel(const __grid_constant__ MlpFwdArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ __align__(8) uint64_t w_full[kSlots], ready[kSlots], step_done[kSlots], raw_full[kSlots];
    __shared__ __align__(8) uint64_t tfull[kAccBufs], tempty[kAccBufs];
    __shared__ uint32_t tmem_base_s;
    __shared__ uint32_t pt[GFX_MAX_PAGES];
    __shared__ float red[2][4];
    // Cluster mode: split-K partials arrive by st.async into the gather area
    // (two 16 KB parities), completing rbar[parity]; consumed[parity] = the last
    // layer whose partials this CTA has read from that parity (senders poll it).
    __shared__ __align__(8) uint64_t rbar[2];
    __shared__ int consumed[2];

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    const int cta = blockIdx.x;
    const int L = a.L;
    unsigned* const cnt = a.cnt + (a.epoch & 1u) * kCntBank;

    if (tid == 0) mark(a.trace, 0);
    for (int i = tid; i < static_cast<int>(a.pt.n); i += kThreads) pt[i] = a.pt.page[i];
    if (tid == 0) {
        for (int s = 0; s < kSlots; ++s) {
            mbar_init(&w_full[s], 1);
            // ready: the 4 converter warps (W_lo in TMEM; they saw w_full) + the X
            // producer's arrive.expect_tx, completed by the X bulk copy's bytes —
            // the MMA thread waits on ONE barrier per step (a try_wait costs ~90
            // cycles even when the phase is already complete).
            mbar_init(&ready[s], 5);
            mbar_init(&step_done[s], 1);  // MMA commit: W, X and W_lo of the step consumed
            mbar_init(&raw_full[s], 1);   // layer-0 raw input tile landed
        }
        for (int b = 0; b < kAccBufs; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 4);  // one arrival per drain warp
        }
        mbar_init(&rbar[0], 1);
        mbar_init(&rbar[1], 1);
        consumed[0] = -2;
        consumed[1] = -1;
        mbar_fence_init();
        tma_prefetch_desc(&a.tmap_in);
    }
    if (warp == 1) tmem_alloc<kTmemCols>(&tmem_base_s);
    tc_fence_before();
    __syncthreads();
    if (a.cluster) cluster_sync();  // every CTA's barriers exist before any remote access
    tc_fence_after();
    const uint32_t tmem = tmem_base_s;
    if (tid == 0) mark(a.trace, 1);

    if (warp == 0) {
        // ---------------- W producer: never waits on activations ----------------
        if (lane == 0) {
            long long pw = 0;
            Prof pr;
            WIter cur{};
            bool have = witer_first(a, cta, cur);
            for (int step = 0; have; ++step) {
                const int s = step % kSlots;
                if (step >= kSlots) {
                    pr.start();
                    mbar_wait(&step_done[s], ((step / kSlots) & 1) ^ 1);
                    pr.stop(pw);
                }
                smark(a.trace, step, 0);
                mbar_arrive_expect_tx(&w_full[s], kWBytes);
                tma_bulk_g2s(smem + s * kSlotBytes, translate(a.arena, pt, witer_off(a, cur)), kWBytes, &w_full[s]);
                have = witer_next(a, cta, cur);
            }
            prof_store(a.trace, 8, pw);
        }
    } else if (warp == 14) {
        // ---------------- X producer: the operand block of each step ----------------
        // Layer 0: a 2-D TMA brings the raw 32 x 32 fp32 input tile into the lower
        // half of the slot (rows 32-63 of the SWIZZLE_128B block, same chunk
        // permutation), then the warp splits it in place (lane = batch row):
        // X_hi to rows 0-31, X_lo over the raw row it read. All of a CTA's
        // layer-0 tiles are requested up front (they fit the first ring slots).
        // Later layers: dataflow wait on the previous layer's tile, then one 8 KB
        // bulk copy of the operand block its reducers wrote.
        int step = 0;
        long long px[2] = {0, 0};
        Prof pr;
        for (int l = 0; l < L; ++l) {
            const MlpFwdLayer& ly = a.layer[l];
            const Unit u = unit_of(ly, cta, a.cluster);
            if (!u.valid) continue;
            if (l == 0 && lane < (u.nkt < kSlots ? u.nkt : kSlots)) {
                // one lane per tile: a thread's TMA requests are served one after another
                const int it = lane;
                uint8_t* xs = smem + it * kSlotBytes + kWBytes;
                mbar_arrive_expect_tx(&raw_full[it], kXBytes / 2);
                tma_tile2d_g2s(xs + kXBytes / 2, &a.tmap_in, (u.kt0 + it) * kTileK, 0, &raw_full[it]);
            }
            __syncwarp();
            if (l > 0) {
                // Two lanes issue alternate steps, each its own loop (a thread's TMA
                // requests are served one after another, ~500 cycles each: one lane
                // alone capped the post-boundary step rate at ~0.43 µs). Each lane
                // polls the dataflow counter of a source tile the first time one of
                // its steps needs it.
                const int step0 = step;
                if (lane < 2) {
                    int ready_src = -1;  // last source tile this lane knows complete
                    for (int it = lane; it < u.nkt; it += 2) {
                        const int st = step0 + it, s = st % kSlots, kt = u.kt0 + it;
                        if (st >= kSlots) mbar_wait(&step_done[s], ((st / kSlots) & 1) ^ 1);
                        const int src = kt >> 2;  // the previous layer's feature tile holding these 32 inputs
                        if (src != ready_src) {
                            wait_count(cnt + kCntDone + (l - 1) * 64 + src, static_cast<unsigned>(a.layer[l - 1].splits));
                            fence_proxy_async_global();
                            ready_src = src;
                        }
                        smark(a.trace, st, 1);
                        mbar_arrive_expect_tx(&ready[s], kXBytes);
                        tma_bulk_g2s(smem + s * kSlotBytes + kWBytes,
                                     a.opnd + static_cast<size_t>(l) * kMlpOpndLayerBytes + static_cast<size_t>(kt) * kXBytes,
                                     kXBytes, &ready[s]);
                    }
                }
                __syncwarp();
                step = step0 + u.nkt;
                continue;
            }
            for (int it = 0; it < u.nkt; ++it, ++step) {
                const int s = step % kSlots;
                const int kt = u.kt0 + it;
                uint8_t* xs = smem + s * kSlotBytes + kWBytes;
                pr.start();
                if (step >= kSlots) mbar_wait(&step_done[s], ((step / kSlots) & 1) ^ 1);
                pr.stop(px[0]);
                if (l == 0) {
                    if (it >= kSlots && lane == 0) {  // wider than the ring: request this tile now
                        mbar_arrive_expect_tx(&raw_full[s], kXBytes / 2);
                        tma_tile2d_g2s(xs + kXBytes / 2, &a.tmap_in, kt * kTileK, 0, &raw_full[s]);
                    }
                    __syncwarp();
                    mbar_wait(&raw_full[s], (it / kSlots) & 1);
                    if (lane == 0) smark(a.trace, step, 6);
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        float4* p = reinterpret_cast<float4*>(xs + sw128(kRows + lane, 4 * j));
                        const float4 v = *p;
                        float4 hi, lo;
                        hi.x = rn_tf32(v.x);
                        hi.y = rn_tf32(v.y);
                        hi.z = rn_tf32(v.z);
                        hi.w = rn_tf32(v.w);
                        lo.x = v.x - hi.x;
                        lo.y = v.y - hi.y;
                        lo.z = v.z - hi.z;
                        lo.w = v.w - hi.w;
                        *reinterpret_cast<float4*>(xs + sw128(lane, 4 * j)) = hi;
                        *p = lo;
                    }
                    fence_proxy_async_smem();  // generic-proxy writes -> tensor core reads
                    __syncwarp();
                    if (lane == 0) {
                        smark(a.trace, step, 1);
                        mbar_arrive(&ready[s]);
                    }
                    continue;
                }
            }
        }
        if (lane == 0) {
            prof_store(a.trace, 9, px[0]);
            prof_store(a.trace, 10, px[1]);
        }
    } else if (warp == 1 || warp == 15) {
        // ---------------- MMA issuers: two warps take alternate accumulator chunks ----------------
        // Each issuing warp loops converged (one elected lane issues). One issuer
        // alone left the tensor pipe idle during its per-step barrier waits and
        // commits (~0.3 us of every 0.6 us step); with two, one issues while the
        // other waits. Chunks of one unit accumulate in different TMEM buffers
        // and are summed by the drain in chunk order, so the result is the same
        // whichever issuer ran first.
        const int issuer = warp == 1 ? 0 : 1;
        constexpr uint32_t idesc64 = umma_idesc<kTileM, 2 * kRows, 2>();  // TF32 x TF32 -> F32, N = 64
        constexpr uint32_t idesc32 = umma_idesc<kTileM, kRows, 2>();      // N = 32
        int step = 0, chunk = 0;
        long long pw[6] = {0, 0, 0, 0, 0, 0};
        Prof pr;
        pr.start();
        for (int l = 0; l < L; ++l) {
            const Unit u = unit_of(a.layer[l], cta, a.cluster);
            if (!u.valid) continue;
            for (int c0 = 0; c0 < u.nkt; c0 += kChunk, ++chunk) {
                const int len = u.nkt - c0 < kChunk ? u.nkt - c0 : kChunk;
                if ((chunk & 1) != issuer) {
                    step += len;
                    continue;
                }
                const int buf = chunk % kAccBufs;
                const uint32_t acc = tmem + static_cast<uint32_t>(buf * kAccCols);
                if (chunk >= kAccBufs) mbar_wait(&tempty[buf], ((chunk / kAccBufs) & 1) ^ 1);
                pr.stop(pw[0]);
                for (int j = 0; j < len; ++j, ++step) {
                    const int s = step % kSlots;
                    // W_lo staged (the converters waited on w_full) and X landed.
                    mbar_wait(&ready[s], (step / kSlots) & 1);
                    tc_fence_after();
                    pr.stop(pw[1]);
                    if (lane == 0) smark(a.trace, step, 4);
                    if (lane == 0 && c0 + j == 0 && l < 6) mark(a.trace, 2 + 4 * l);
                    const uint8_t* w = smem + s * kSlotBytes;
                    const uint64_t bx = umma_desc_sw128(w + kWBytes, 0), aw = umma_desc_sw128(w, 0);
                    const uint32_t lo = tmem + kLoBase + static_cast<uint32_t>(kTileK * s);
#pragma unroll
                    for (int kk = 0; kk < kTileK / 8; ++kk) {
                        // +kk*32 bytes = +2 in the descriptor's 16-byte address units
                        umma_tf32_elect(acc, aw + 2 * kk, bx + 2 * kk, idesc64, (j == 0 && kk == 0) ? 0u : 1u);
                        if (!(a.ablate & 2)) umma_tf32_ts_elect(acc, lo + static_cast<uint32_t>(8 * kk), bx + 2 * kk, idesc32, 1u);
                    }
                    pr.stop(pw[5]);
                    if (lane == 0) smark(a.trace, step, 5);
                    umma_commit_elect(&step_done[s]);  // W slot, X slot and W_lo stage s free once these MMAs retire
                    if (lane == 0 && c0 + j == u.nkt - 1 && l < 6) mark(a.trace, 3 + 4 * l);
                    pr.stop(pw[4]);
                }
                umma_commit_elect(&tfull[buf]);
            }
        }
        if (lane == 0 && issuer == 0) {
            for (int i = 0; i < 5; ++i) prof_store(a.trace, i, pw[i]);
            prof_store(a.trace, 13, pw[5]);
            prof_store(a.trace, 15, step);
        }
    } else if (warp < 10) {
        // ---------------- converters: W_lo = W - trunc_tf32(W) into TMEM stage s ----------------
        const int group = (warp - 2) >> 2;
        const int q = warp & 3;            // TMEM lane quarter of this warp
        const int r = q * 32 + lane;       // weight row of the tile = TMEM lane
        const uint32_t mask = (a.ablate & 1) ? 0u : 0xFFFFE000u;
        int step = 0;
        long long pc[3] = {0, 0, 0};
        Prof pr;
        pr.start();
        for (int l = 0; l < L; ++l) {
            const Unit u = unit_of(a.layer[l], cta, a.cluster);
            if (!u.valid) continue;
            for (int it = 0; it < u.nkt; ++it, ++step) {
                if ((step & 1) != group) continue;
                const int s = step % kSlots;
                mbar_wait(&w_full[s], (step / kSlots) & 1);
                pr.stop(pc[0]);
                if (lane == 0 && q == 2) smark(a.trace, step, 2);
                // Stage s of the W_lo ring was last read by the MMAs of step - kSlots,
                // which also freed the landing slot this tile arrived in: step_done
                // of that phase is complete already (the producer waited on it).
                if (a.ablate & 4) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&ready[s]);
                    continue;
                }
                const float4* wrow = reinterpret_cast<const float4*>(smem + s * kSlotBytes + r * 128);
                float wlo[32];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const float4 v = wrow[j ^ (r & 7)];
                    const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const float hi = (a.ablate & 1) ? rn_tf32(e[i]) : __uint_as_float(__float_as_uint(e[i]) & mask);
                        wlo[4 * j + i] = e[i] - hi;
                    }
                }
                pr.stop(pc[2]);
                tc_fence_after();
                tmem_st_32x32b_x32(tmem + (static_cast<uint32_t>(q * 32) << 16) + kLoBase + static_cast<uint32_t>(kTileK * s), wlo);
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&ready[s]);
                pr.stop(pc[2]);
                if (lane == 0 && q == 2) smark(a.trace, step, 3);
            }
        }
        if (warp == 2 && lane == 0)
            for (int i = 0; i < 3; ++i) prof_store(a.trace, 5 + i, pc[i]);
    } else if (warp < 14) {
        // ---------------- drain + epilogue warps ----------------
        const int ct = tid - 320;          // 0..127
        const int q = warp & 3;            // TMEM lane quarter (warps 10..13 -> 2,3,0,1)
        const int fl = q * 32 + lane;      // feature row within the tile

        {  // the other counter bank, for the next launch (see kCntBank)
            unsigned* other = a.cnt + ((a.epoch & 1u) ^ 1u) * kCntBank;
            for (int i = cta * 128 + ct; i < kCntBank; i += gridDim.x * 128) other[i] = 0;
        }
        int chunk = 0;
        uint32_t rph = 0;  // rbar phase bits (cluster mode)
        long long pd[2] = {0, 0};
        Prof pr;
        auto mark_consumed = [&](int l) {  // cluster mode: parity l & 1 of this CTA's buffer is free again
            if (a.cluster && ct == 0) {
                asm volatile("fence.acq_rel.cluster;\n" ::: "memory");
                *reinterpret_cast<volatile int*>(&consumed[l & 1]) = l;
            }
        };
        for (int l = 0; l < L; ++l) {
            const MlpFwdLayer& ly = a.layer[l];
            const Unit u = unit_of(ly, cta, a.cluster);
            if (!u.valid || ly.splits == 1) mark_consumed(l);  // nobody sends this CTA partials of layer l
            if (!u.valid) continue;
            pr.start();
            const bool last = l == L - 1;
            const int N = ly.N;
            const int f = u.tile * kTileM + fl;
            const bool valid = f < N;  // rows >= N are the zero padding of the last weight tile
            const float bias = valid ? *reinterpret_cast<const float*>(translate(a.arena, pt, ly.b_off + 4ull * f)) : 0.f;
            float acc[kRows];
#pragma unroll
            for (int b = 0; b < kRows; ++b) acc[b] = 0.f;
            const int nch = (u.nkt + kChunk - 1) / kChunk;
            for (int c = 0; c < nch; ++c, ++chunk) {
                mbar_wait(&tfull[chunk % kAccBufs], (chunk / kAccBufs) & 1);
                pr.stop(pd[0]);
                if (ct == 0 && a.trace && cta == 0 && chunk < 32) a.trace[static_cast<size_t>(gridDim.x) * 32 + 512 + chunk] = gtime();
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

            if (ct == 0 && l < 6) mark(a.trace, 4 + 4 * l);
            // Where row b of feature f goes.
            char* const nxt = last ? nullptr : a.opnd + static_cast<size_t>(l + 1) * kMlpOpndLayerBytes + static_cast<size_t>(f >> 5) * kXBytes;
            auto emit = [&](int b, float v) {
                v += bias;
                if (!last) {
                    v = fmaxf(v, 0.f);
                    if (valid) {
                        const float hi = rn_tf32(v);
                        *reinterpret_cast<float*>(nxt + sw128(b, f & 31)) = hi;
                        *reinterpret_cast<float*>(nxt + sw128(kRows + b, f & 31)) = v - hi;
                    }
                } else if (valid) {
                    a.logits[static_cast<size_t>(b) * N + f] = v;
                }
            };
            const int S = ly.splits;
            if (S == 1) {
#pragma unroll
                for (int b = 0; b < kRows; ++b) emit(b, acc[b]);
            } else if (a.cluster) {
                // The tile's S splits are cluster ranks base .. base + S - 1; split o
                // owns rows b = o (mod S). Every split st.asyncs its partial rows into
                // the owner's receive buffer [src split][row / S][feature] (a warp's
                // 32 features of a row = 128 contiguous bytes), completing the
                // owner's rbar; the owner sums in split order. No global round trip.
                const int par = l & 1, per = kRows / S;
                const int base = cta % a.cluster - u.split;
                float* rb = reinterpret_cast<float*>(smem + kSlots * kSlotBytes) + par * (kRows * kTileM);
                if (ct < S) {  // the destination's parity buffer was read for layer l - 2
                    const uint32_t ra = mapa_u32(&consumed[par], static_cast<uint32_t>(base + ct));
                    while (ld_acquire_cluster_s32(ra) < l - 2) {
                    }
                }
                epi_sync();
                if (ct == 0) {
                    if (l == 0) mark(a.trace, 18);
                    mbar_arrive_expect_tx(&rbar[par], kRows * kTileM * 4);
                }
                const uint32_t rb_mine = smem_u32(rb) + static_cast<uint32_t>((u.split * per * kTileM + fl) * 4);
#pragma unroll
                for (int b = 0; b < kRows; ++b) {
                    const int o = b % S, jj = b / S;
                    const uint32_t rank = static_cast<uint32_t>(base + o);
                    uint32_t dst, mb;
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(dst) : "r"(rb_mine + jj * kTileM * 4), "r"(rank));
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(mb) : "r"(smem_u32(&rbar[par])), "r"(rank));
                    st_async_f32(dst, acc[b], mb);
                }
                mbar_wait(&rbar[par], (rph >> par) & 1u);
                rph ^= 1u << par;
                if (ct == 0 && l < 2) mark(a.trace, 26 + 2 * l);
                for (int jj = 0; jj < per; ++jj) {
                    float v = 0.f;
                    for (int sp = 0; sp < S; ++sp) v += rb[(sp * per + jj) * kTileM + fl];
                    emit(u.split + jj * S, v);
                }
                epi_sync();  // every thread has read the buffer
                mark_consumed(l);
                if (ct == 0 && l < 2) mark(a.trace, 27 + 2 * l);
            } else {
                // Publish this unit's partial [32][128], wait for the tile's
                // siblings (co-resident: cooperative launch), reduce rows
                // b = split (mod S) in fixed split order.
                float* tp = a.part + static_cast<size_t>(l) * kMlpPartLayerFloats +
                            static_cast<size_t>(u.tile) * S * (kRows * kTileM);
                float* mine = tp + static_cast<size_t>(u.split) * (kRows * kTileM);
#pragma unroll
                for (int b = 0; b < kRows; ++b) __stcg(mine + b * kTileM + fl, acc[b]);
                epi_sync();  // CTA-scope ordering; thread 0's gpu fence is cumulative over it
                if (ct == 0) {
                    if (l == 0) mark(a.trace, 18);
                    fence_acq_rel_gpu();
                    if (l == 0) mark(a.trace, 19);
                    atomicAdd(cnt + kCntArrive + l * 64 + u.tile, 1u);
                    if (l == 0) mark(a.trace, 20);
                    wait_count(cnt + kCntArrive + l * 64 + u.tile, static_cast<unsigned>(S));  // acquire
                    if (l == 0) mark(a.trace, 21);
                }
                epi_sync();
                if (ct == 0 && l < 2) mark(a.trace, 26 + 2 * l);
                // One round of 16-byte cp.async gathers every partial row this
                // split reduces (ri-th owned row, split sp) into the gather area.
                const int nrows = (kRows - u.split + S - 1) / S;
                float* gat = reinterpret_cast<float*>(smem + kSlots * kSlotBytes);
                // Lane = 16-byte column chunk of a 512-byte partial row; the 4
                // warps take the (row, split) pairs round robin (no divisions).
                {
                    const int w4 = ct >> 5;
                    int rs = 0;
                    for (int ri = 0; ri < nrows; ++ri) {
                        const float* row = tp + (u.split + ri * S) * kTileM + lane * 4;
                        for (int sp = 0; sp < S; ++sp, ++rs)
                            if ((rs & 3) == w4)
                                cp_async16(gat + static_cast<size_t>(rs) * kTileM + lane * 4,
                                           row + static_cast<size_t>(sp) * (kRows * kTileM));
                    }
                }
                if (ct == 0 && l == 0) mark(a.trace, 22);
                asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
                epi_sync();
                if (ct == 0 && l == 0) mark(a.trace, 23);
                for (int ri = 0; ri < nrows; ++ri) {
                    const float* g = gat + static_cast<size_t>(ri * S) * kTileM + fl;
                    float v = 0.f;
#pragma unroll 8
                    for (int sp = 0; sp < S; ++sp) v += g[sp * kTileM];
                    emit(u.split + ri * S, v);
                }
                if (ct == 0 && l < 2) mark(a.trace, 27 + 2 * l);
            }
            fence_proxy_async_global();
            if (ct == 0 && l == 0) mark(a.trace, 24);
            epi_sync();
            if (ct == 0) {
                if (l == 0) mark(a.trace, 25);
                fence_acq_rel_gpu();
                if (l == 0) mark(a.trace, 30);
                atomicAdd(cnt + kCntDone + l * 64 + u.tile, 1u);
                if (last) atomicAdd(cnt + kCntFinal, 1u);
                if (l < 6) mark(a.trace, 5 + 4 * l);
            }
            pr.stop(pd[1]);
        }
        if (ct == 0) {
            prof_store(a.trace, 11, pd[0]);
            prof_store(a.trace, 12, pd[1]);
        }

        // Softmax of the logits: batch row b = cta, after every last-layer unit finished.
        if (cta < kRows) {
            const MlpFwdLayer& ly = a.layer[L - 1];
            const int C = ly.N;
            if (ct == 0) wait_count(cnt + kCntFinal, static_cast<unsigned>(ly.tiles * ly.splits));
            epi_sync();
            const float* in = a.logits + static_cast<size_t>(cta) * C;
            float* out = a.probs + static_cast<size_t>(cta) * C;
            constexpr int kPer = 2048 / 128;
            float v[kPer];
            float m = -INFINITY;
#pragma unroll
            for (int i = 0; i < kPer; ++i) {
                const int c = ct + i * 128;
                v[i] = c < C ? __ldcg(in + c) : -INFINITY;
                m = fmaxf(m, v[i]);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (lane == 0) red[0][q] = m;
            epi_sync();
            m = fmaxf(fmaxf(red[0][0], red[0][1]), fmaxf(red[0][2], red[0][3]));
            float sum = 0.f;
#pragma unroll
            for (int i = 0; i < kPer; ++i) {
                const int c = ct + i * 128;
                v[i] = c < C ? expf(v[i] - m) : 0.f;
                sum += v[i];
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
            if (lane == 0) red[1][q] = sum;
            epi_sync();
            const float inv = 1.0f / (red[1][0] + red[1][1] + red[1][2] + red[1][3]);
#pragma unroll
            for (int i = 0; i < kPer; ++i) {
                const int c = ct + i * 128;
                if (c < C) out[c] = v[i] * inv;
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (a.cluster) cluster_sync();  // no CTA leaves while a peer may still write into its smem
    tc_fence_after();
    if (tid == 0) mark(a.trace, 31);
    if (warp == 1) tmem_dealloc<kTmemCols>(tmem);
}

}  // namespace

int mlp_fwd_splits(int K, int N, int grid, int cluster) {
    const int tiles = (N + kTileM - 1) / kTileM;
    const int kt = K / kTileK;
    if (cluster) {  // the largest S dividing the cluster whose tiles fit the co-resident clusters
        for (int s = cluster; s > 1; s >>= 1)
            if (s <= kt && (tiles + cluster / s - 1) / (cluster / s) <= grid / cluster) return s;
        return 1;
    }
    int s = grid / tiles;
    if (s > kt) s = kt;
    if (s > kRows) s = kRows;
    return s < 1 ? 1 : s;
}

int mlp_fwd_cluster_grid(int cluster) {
    // Co-resident CTAs when launched in clusters of `cluster` (one CTA per SM).
    const size_t smem = mlp_fwd_smem();
    GFX_CUDA(cudaFuncSetAttribute(mlp_forward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(cluster));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(cluster);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    GFX_CUDA(cudaOccupancyMaxActiveClusters(&n, mlp_forward_kernel, &cfg));
    return n * cluster;
}

size_t mlp_trace_words(int grid) { return static_cast<size_t>(48) * grid + 576; }

// Debug report of a traced launch (GFX_TRACE_MLP=1): per-phase %globaltimer marks
// (µs after the first CTA started; min / median / max over CTAs), CTA 0's
// per-step timeline and the per-role cycle accounting.
void mlp_trace_report(const std::vector<unsigned long long>& tr, int grid, int L, int model) {
    struct {
        int grid, L;
    } f{grid, L};
    unsigned long long t0 = ~0ull;
    const size_t nct = static_cast<size_t>(f.grid) * 32;
    for (size_t i = 0; i < nct; i += 32) t0 = std::min(t0, tr[i]);
    static const char* names[4] = {"mma first", "mma last", "epi start", "tile done"};
    std::fprintf(stderr, "[trace] model %d grid %d\n", model, f.grid);
    for (int ph = 0; ph < 32; ++ph) {
        std::vector<double> v;
        for (size_t i = 0; i < nct; i += 32)
            if (tr[i + static_cast<size_t>(ph)]) v.push_back((tr[i + static_cast<size_t>(ph)] - t0) * 1e-3);
        if (v.empty()) continue;
        std::sort(v.begin(), v.end());
        char nm[32];
        if (ph == 0) std::snprintf(nm, sizeof nm, "start");
        else if (ph == 1) std::snprintf(nm, sizeof nm, "setup");
        else if (ph == 31) std::snprintf(nm, sizeof nm, "end");
        else if (ph >= 26 && ph < 30) std::snprintf(nm, sizeof nm, "L%d %s", (ph - 26) / 2, ph % 2 ? "gathered" : "siblings");
        else if (ph >= 18 && ph <= 30 && f.L <= 4) {
            static const char* sub[13] = {"L0 part stored", "L0 fenced", "L0 arrived", "L0 sib seen", "L0 cp.async issued",
                                          "L0 cp.async done", "L0 emitted", "L0 done-sync", "", "", "", "", "L0 done fenced"};
            std::snprintf(nm, sizeof nm, "%s", sub[ph - 18]);
        }
        else std::snprintf(nm, sizeof nm, "L%d %s", (ph - 2) / 4, names[(ph - 2) % 4]);
        std::fprintf(stderr, "  %-16s n=%3zu %8.2f %8.2f %8.2f\n", nm, v.size(), v.front(), v[v.size() / 2],
                     v.back());
    }
    std::fprintf(stderr, "  CTA 0 steps (us): Wreq Xreq Wlanded WloDone xFull mmaIssued rawLanded\n");
    for (int st = 0; st < 64; ++st) {
        const unsigned long long* p = tr.data() + nct + st * 8;
        if (!p[0] && !p[5]) break;
        auto us = [&](unsigned long long t) { return t ? (t - t0) * 1e-3 : -1.0; };
        std::fprintf(stderr, "   %2d %7.2f %7.2f %7.2f %7.2f %7.2f %7.2f %7.2f\n", st, us(p[0]), us(p[1]), us(p[2]),
                     us(p[3]), us(p[4]), us(p[5]), us(p[6]));
    }
    static const char* pn[16] = {"mma: wait tempty", "mma: wait ready", "", "",
                                 "mma: commits+rest", "conv: wait w_full", "", "conv: work",
                                 "wprod: wait slot", "xprod: wait slot", "xprod: wait flag", "drain: wait tfull",
                                 "drain: epilogue", "mma: MMAs", "", "steps"};
    std::fprintf(stderr, "  cycles per CTA, mean over CTAs with work (per step in brackets):\n");
    for (int i = 0; i < 16; ++i) {
        if (!pn[i][0]) continue;
        double sum = 0, steps = 0;
        int n = 0;
        for (int c = 0; c < f.grid; ++c) {
            const unsigned long long st = tr[nct + 576 + c * 16 + 15];
            if (!st) continue;
            sum += static_cast<double>(tr[nct + 576 + c * 16 + i]);
            steps += static_cast<double>(st);
            ++n;
        }
        if (n) std::fprintf(stderr, "   %-22s %10.0f  (%7.1f)\n", pn[i], sum / n, sum / steps);
    }
    }

size_t mlp_fwd_smem() { return static_cast<size_t>(kSlotBytes) * kSlots + kGatherBytes + 1024; }

void launch_mlp_forward(MlpFwdArgs& a, cudaStream_t stream) {
    if (a.L < 1 || a.L > GFX_MAX_LAYERS) throw std::runtime_error("mlp forward: bad layer count");
    for (int l = 0; l < a.L; ++l) {
        const MlpFwdLayer& ly = a.layer[l];
        if (ly.K % kTileK || ly.K > kMlpMaxDim || ly.N > kMlpMaxDim || ly.tiles > 64 || ly.tiles * ly.splits > a.grid)
            throw std::runtime_error("mlp forward: unsupported layer shape");
        if (a.cluster && (a.cluster % ly.splits || (ly.tiles + a.cluster / ly.splits - 1) / (a.cluster / ly.splits) >
                                                        a.grid / a.cluster))
            throw std::runtime_error("mlp forward: layer does not fit the cluster map");
        if (l > 0 && a.layer[l - 1].N != ly.K) throw std::runtime_error("mlp forward: layer widths do not chain");
    }
    if (a.layer[a.L - 1].N > 2048 || a.grid < kRows) throw std::runtime_error("mlp forward: at most 2048 classes, grid >= 32");
    // Layer-0 input tiles: 32 x 32 fp32 boxes of the [32 x K0] request input, SWIZZLE_128B.
    if (!encode_tensor_map_2d(&a.tmap_in, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, a.in, static_cast<uint64_t>(a.layer[0].K),
                              kRows, static_cast<uint64_t>(a.layer[0].K) * 4, kTileK, kRows, CU_TENSOR_MAP_SWIZZLE_128B))
        throw CudaError("cuTensorMapEncodeTiled failed for the request input");
    static bool attr_set = false;
    const size_t smem = mlp_fwd_smem();
    if (!attr_set) {
        GFX_CUDA(cudaFuncSetAttribute(mlp_forward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
        attr_set = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(a.grid));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;  // every CTA co-resident: the dataflow waits need it
    attr[0].val.cooperative = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = static_cast<unsigned>(a.cluster ? a.cluster : 1);
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    static const bool no_coop = std::getenv("GFX_MLP_NOCOOP") != nullptr;  // debug A/B
    cfg.numAttrs = a.cluster ? 2 : (no_coop ? 0 : 1);
    GFX_CUDA(cudaLaunchKernelEx(&cfg, mlp_forward_kernel, a));
}

}  // namespace gfx
