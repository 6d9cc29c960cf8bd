#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <vector>

#include "common.cuh"

namespace gfx {

// Fills `count` consecutive tensors of n values, tensor t from seed + t.
void launch_fill_params(float* dst, uint64_t n, uint64_t seed, uint32_t tensor, float scale, cudaStream_t s,
                        uint64_t count = 1);

// K1 v7: whole forward in one persistent cooperative launch (mlp_fwd.cu).
constexpr int kMlpMaxDim = 8192;
constexpr int kMlpMaxClasses = 2048;
// Layer outputs as 64-bit words (fixed-point value x 2^32 << 9 | completion
// count), feature-major [N][32], reduced in L2 by the split-K partials
// (red.add.u64: associative, so the sum is the same whatever order the
// partials arrive in). One buffer per launch parity; Σ_l N_l x 32 words used.
constexpr int kMlpFixShift = 32;
constexpr size_t kMlpActWords = static_cast<size_t>(GFX_MAX_LAYERS) * kMlpMaxDim * 32;

struct MlpFwdLayer {
    uint64_t w_off, b_off;  // model-blob offsets of the weight tiles and the bias
    int K, N;
    int tiles, nkt;         // 128-row feature tiles, 32-wide K tiles
    uint32_t act_off;       // words: this layer's output [N][32] in the act buffer
};

struct MlpFwdArgs {
    CUtensorMap tmap_in;    // layer-0 input tiles (filled by launch_mlp_forward)
    CUtensorMap tmap_out[GFX_MAX_LAYERS];  // layer outputs [N][32] u64, 32 x 16 boxes (filled by launch_mlp_forward)
    const char* arena;
    const float* in;        // [32 x K0] request input, row-major
    float* logits;          // [32 x C]
    float* probs;           // [32 x C] softmax rows
    unsigned long long* act;  // this launch's layer outputs (all zero at launch)
    uint4* act_clear;         // the other parity's buffer: cleared here for the next launch
    uint32_t clear_vec;       // 16-byte vectors of act_clear the previous launch dirtied
    unsigned long long* dbg;  // GFX_K1_DEBUG builds: [grid][32] phase marks (%globaltimer), else unused
    int L;
    int grid;
    int pdl;                  // 1: chained to the previous launch by PDL (device owned by one manager), 0: cooperative
    // Layer 0 split dynamically (nullptr: static stream-K ranges like the other layers):
    // CTAs claim kMlpChunk0-step ranges from *claim (zero at launch); CTA 0 zeroes
    // *claim_reset (the counter of launch + 2) once the previous launch completed.
    unsigned* claim;
    unsigned* claim_reset;
    MlpFwdLayer layer[GFX_MAX_LAYERS];
    PageTable pt;
};

constexpr int kMlpChunk0 = 4;  // layer-0 steps per dynamic claim (two paired 32 KB weight copies)
size_t mlp_fwd_smem();
// GFX_K1_DEBUG builds: phase-mark table of the last launch (stderr).
void mlp_debug_report(const unsigned long long* dbg, int grid, int L, int model, cudaStream_t s);
// Validates the shapes, fills the tensor map and launches on `stream`.
void launch_mlp_forward(MlpFwdArgs& a, cudaStream_t stream);

// Weight tiles of the blob: 128 x 32 fp32, K-major SWIZZLE_128B image (16 KB).
constexpr int kWTileRows = 128;
constexpr int kWTileK = 32;
__host__ __device__ inline uint64_t wtile_offset(uint64_t n, uint64_t k, uint64_t K) {
    const uint64_t mt = n / kWTileRows, r = n % kWTileRows, kt = k / kWTileK, kk = k % kWTileK;
    const uint64_t tile = mt * (K / kWTileK) + kt;
    return tile * (kWTileRows * kWTileK * 4) + r * 128 + (((kk >> 2) ^ (r & 7)) << 4) + (kk & 3) * 4;
}

}  // namespace gfx
