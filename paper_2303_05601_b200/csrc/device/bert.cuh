#pragma once
// C5 model family: BERT-base-style post-LN transformer encoder in bf16
// (fp32 accumulation), batch of sequences per request, pooled fp32 output.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace gfx {

// Blob layout of one BERT model: weight matrices as 16 KB
// K-major SWIZZLE_128B tiles of 128 rows x 64 bf16 (16 KB-aligned, rows padded
// to 128); biases and LayerNorm parameters fp32 (256 B-aligned).
struct BertLayerOffsets {
    uint64_t wqkv, bqkv, wo, bo, ln1_g, ln1_b, w1, b1, w2, b2, ln2_g, ln2_b;
};
struct BertLayout {
    int L = 0, d = 0, heads = 0, ffn = 0, seq = 0;
    std::vector<BertLayerOffsets> layer;
    uint64_t wp = 0, bp = 0;  // pooler
    uint64_t bytes = 0;
};
BertLayout bert_layout(int L, int d, int heads, int ffn, int seq);

// Parameter tensors of layer l: 16*l + {0 Wqkv, 1 bqkv, 2 Wo, 3 bo, 4 ln1_g,
// 5 ln1_b, 6 W1, 7 b1, 8 W2, 9 b2, 10 ln2_g, 11 ln2_b}; pooler 16*L + {0 Wp, 1 bp}.
enum BertTensor : uint32_t {
    kWqkv = 0, kBqkv, kWo, kBo, kLn1G, kLn1B, kW1, kB1, kW2, kB2, kLn2G, kLn2B
};

__host__ __device__ inline uint64_t bf16_tile_offset(uint64_t n, uint64_t k, uint64_t K) {
    // 128 x 64 bf16 tile = 128 rows x 128 B, 16-byte chunk XOR (row & 7).
    const uint64_t mt = n / 128, r = n % 128, kt = k / 64, kk = k % 64;
    const uint64_t tile = mt * (K / 64) + kt;
    return tile * 16384 + r * 128 + (((kk >> 3) ^ (r & 7)) << 4) + (kk & 7) * 2;
}

// Round-to-nearest-even fp32 -> bf16 bits (matches the oracle's restatement).
__host__ __device__ inline uint16_t bf16_bits(float f) {
#ifdef __CUDA_ARCH__
    uint32_t u = __float_as_uint(f);
#else
    uint32_t u;
    memcpy(&u, &f, 4);
#endif
    if ((u & 0x7F800000u) == 0x7F800000u) return static_cast<uint16_t>(u >> 16);  // inf / nan
    u += 0x7FFFu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}

struct BertWorkspace {
    int tokens = 0;
    bool gemm_pair = false;  // 2-SM (cta_group::2) GEMMs where the shape allows (gfx_arena_set_option)
    bool flow = false;       // the encoder dataflow kernel K5 instead of per-op launches (K2-K4)
    __nv_bfloat16 *x = nullptr, *qkv = nullptr, *ctx = nullptr, *h = nullptr, *f = nullptr, *t = nullptr;
    // K5: dataflow counters + ready-queue slots for one (layers, row blocks, ffn) shape.
    uint32_t* flow_cnt = nullptr;
    void* flow_stats = nullptr;  // per-row LayerNorm statistics of the residual tiles
    int flow_L = 0, flow_M = 0, flow_F = 0, flow_ctas = 0;
    size_t flow_cnt_words = 0;
    // Second stream (+ fork / join events) for the two-half per-op forward, created on first use
    // on the device current at the time (the manager's).
    cudaStream_t side = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    void ensure(int tokens, int d, int ffn);
    void ensure_side_stream();
    void release();
};

// K5 (bert_flow.cu): all encoder layers as one persistent dataflow launch.
// Layer l's output goes to xout + l * xstride rows (xstride 0: one buffer,
// rewritten in place per row block); layer 0 reads `in`.
bool bert_flow_supported(const BertLayout& lay, int batch);
int bert_encoder_flow(const char* arena, const PageTable& pt, const BertLayout& lay, int batch,
                      const __nv_bfloat16* in, __nv_bfloat16* xout, int xstride, BertWorkspace& ws, cudaStream_t s);

// One forward of a resident BERT model: in = [batch*seq x d] bf16 embeddings,
// out = [batch x d] fp32 pooled output. Returns kernel launches.
// lengths (device, [batch] int32 in 1..seq, optional): padding mask — sequence b
// attends to its first lengths[b] tokens.
int bert_forward(const char* arena, const PageTable& pt, const BertLayout& lay, int batch,
                 const __nv_bfloat16* in, float* out, BertWorkspace& ws, cudaStream_t s,
                 __nv_bfloat16* hidden = nullptr,  // debug: [L+1][T][d] hidden states
                 const int* lengths = nullptr);

// Test hook: one K2 GEMM of layer l with its fused epilogue. op 0: QKV (+bias),
// 1: attention output (+bias +resid), 2: FFN1 (+bias, GELU), 3: FFN2 (+bias +resid);
// 4 / 5: ops 1 / 3 followed by LayerNorm 1 / 2 (the forward's fused residual + LN step).
void bert_gemm_op(const char* arena, const PageTable& pt, const BertLayout& lay, int l, int op,
                  const __nv_bfloat16* x, const __nv_bfloat16* resid, __nv_bfloat16* y, int T, bool pair,
                  cudaStream_t s);

// Fill `count` bf16 tensors of n values from the parameter stream (inputs).
void launch_fill_bf16(__nv_bfloat16* dst, uint64_t n, uint64_t seed, uint32_t tensor, float scale, cudaStream_t s,
                      uint64_t count = 1);

}  // namespace gfx
