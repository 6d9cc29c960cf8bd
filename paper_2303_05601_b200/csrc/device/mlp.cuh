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

// K1 v6: whole forward in one persistent cooperative launch (mlp_fwd.cu).
constexpr int kMlpMaxDim = 8192;
constexpr size_t kMlpOpndLayerBytes = static_cast<size_t>(kMlpMaxDim / 32) * 8192;  // operand blocks per layer input
constexpr size_t kMlpPartLayerFloats = static_cast<size_t>(160) * 32 * 128;        // split-K partials per layer
constexpr int kMlpCounters = 8192;

struct MlpFwdLayer {
    uint64_t w_off, b_off;  // model-blob offsets of the weight tiles and the bias
    int K, N;
    int tiles, splits;      // units = tiles x splits <= grid
};

struct MlpFwdArgs {
    CUtensorMap tmap_in;    // layer-0 input tiles (filled by launch_mlp_forward)
    const char* arena;
    const float* in;        // [32 x K0] request input, row-major
    float* logits;          // [32 x C]
    float* probs;           // [32 x C] softmax rows
    char* opnd;             // operand blocks, layer l's input at opnd + l * kMlpOpndLayerBytes
    float* part;            // split-K partials, layer l at part + l * kMlpPartLayerFloats
    unsigned* cnt;          // kMlpCounters dataflow counters: two banks, bank (epoch & 1) zero at launch
    unsigned epoch;         // launch sequence number on this workspace (stream-ordered)
    int L;
    int grid;
    int cluster;            // 0, or 8: split-K reduced through cluster DSMEM (GFX_MLP_CLUSTER=1)
    int ablate;             // debug bitmask (0 in production): 1 = W_hi taken as rn_tf32 instead of trunc
    unsigned long long* trace;  // debug (GFX_TRACE_MLP): [grid][32] %globaltimer marks, else nullptr
    MlpFwdLayer layer[GFX_MAX_LAYERS];
    PageTable pt;
};

int mlp_fwd_splits(int K, int N, int grid, int cluster = 0);
int mlp_fwd_cluster_grid(int cluster);
size_t mlp_fwd_smem();
void launch_mlp_forward(MlpFwdArgs& a, cudaStream_t stream);
// Debug timeline (GFX_TRACE_MLP): buffer size in 64-bit words and the stderr report.
size_t mlp_trace_words(int grid);
void mlp_trace_report(const std::vector<unsigned long long>& trace, int grid, int layers, int model);

// Weight tiles of the blob: 128 x 32 fp32, K-major SWIZZLE_128B image (16 KB).
constexpr int kWTileRows = 128;
constexpr int kWTileK = 32;
__host__ __device__ inline uint64_t wtile_offset(uint64_t n, uint64_t k, uint64_t K) {
    const uint64_t mt = n / kWTileRows, r = n % kWTileRows, kt = k / kWTileK, kk = k % kWTileK;
    const uint64_t tile = mt * (K / kWTileK) + kt;
    return tile * (kWTileRows * kWTileK * 4) + r * 128 + (((kk >> 2) ^ (r & 7)) << 4) + (kk & 3) * 4;
}

}  // namespace gfx
