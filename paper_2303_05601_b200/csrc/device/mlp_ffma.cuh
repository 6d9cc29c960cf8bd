#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "common.cuh"

namespace gfx {

constexpr int kMaxSplits = 32;

struct MlpLayerArgs {
    const float* x;        // [32 x K] activations, row-major, device
    float* y;              // [32 x N] output rows
    float* probs;          // last layer: [32 x N] softmax rows; else nullptr
    const char* arena;     // arena base
    uint64_t w_off;        // model-blob offset of W [N x K]
    uint64_t b_off;        // model-blob offset of b [N]
    int K, N;
    int splits, ntiles;
    int relu;
    int ldws;              // leading dimension of the split-K workspace
    float* ws;             // [splits][32][ldws]
    unsigned* counters;    // [ntiles + 1], zero between launches
    float* stats;          // last layer: [ntiles][32][2] per-tile softmax partials
    PageTable pt;
};

int mlp_layer_splits(int K, int N, int sm_count);
int mlp_layer_tiles(int N);
size_t mlp_layer_smem();
void launch_mlp_layer(const MlpLayerArgs& a, cudaStream_t stream);
void launch_fill_params(float* dst, uint64_t n, uint64_t seed, uint32_t tensor, float scale, cudaStream_t s);

}  // namespace gfx
