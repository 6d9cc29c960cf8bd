"""Library baseline for K2/K3/K4: the C5 BERT-base shapes (T = 32 x 128 tokens,
d 768, 12 heads, FFN 3072, bf16) through cuBLAS (torch.nn.functional.linear ->
cublasLt with bias epilogue), torch SDPA (flash) and torch LayerNorm, timed with
CUDA events on the current stream, warm, back to back. Not product code: it is
the number the hand-written kernels are compared with (profiles/r2_k2_bert.md).
usage: python tools/cublas_bert.py [iters]"""
import json
import sys

import torch
import torch.nn.functional as F

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 50
dev = torch.device("cuda:0")
torch.manual_seed(0)
B, S, D, H, FF, L = 32, 128, 768, 12, 3072, 12
T = B * S
bf = torch.bfloat16


def timed(fn, n=iters):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3  # us


out = {"gemm_us": {}, "gemm_tflops": {}}
x = torch.randn(T, D, device=dev, dtype=bf)
h = torch.randn(T, FF, device=dev, dtype=bf)
for name, K, N, src in (("qkv", D, 3 * D, x), ("oproj", D, D, x), ("ffn1", D, FF, x), ("ffn2", FF, D, h)):
    w = torch.randn(N, K, device=dev, dtype=bf) * 0.02
    b = torch.randn(N, device=dev, dtype=bf)
    us = timed(lambda: F.linear(src, w, b))
    out["gemm_us"][name] = round(us, 2)
    out["gemm_tflops"][name] = round(2.0 * T * K * N / us / 1e6, 1)

# One encoder layer (post-LN, like the product's) and the 12-layer forward.
Wqkv = torch.randn(3 * D, D, device=dev, dtype=bf) * 0.02
bqkv = torch.zeros(3 * D, device=dev, dtype=bf)
Wo = torch.randn(D, D, device=dev, dtype=bf) * 0.02
bo = torch.zeros(D, device=dev, dtype=bf)
W1 = torch.randn(FF, D, device=dev, dtype=bf) * 0.02
b1 = torch.zeros(FF, device=dev, dtype=bf)
W2 = torch.randn(D, FF, device=dev, dtype=bf) * 0.02
b2 = torch.zeros(D, device=dev, dtype=bf)
g = torch.ones(D, device=dev, dtype=bf)
be = torch.zeros(D, device=dev, dtype=bf)


def layer(x):
    qkv = F.linear(x, Wqkv, bqkv).view(B, S, 3, H, D // H).permute(2, 0, 3, 1, 4)
    ctx = F.scaled_dot_product_attention(qkv[0], qkv[1], qkv[2])
    ctx = ctx.transpose(1, 2).reshape(T, D)
    x = F.layer_norm(F.linear(ctx, Wo, bo) + x, (D,), g, be)
    f = F.gelu(F.linear(x, W1, b1))
    return F.layer_norm(F.linear(f, W2, b2) + x, (D,), g, be)


def forward():
    y = x
    for _ in range(L):
        y = layer(y)
    return y


with torch.no_grad():
    out["attention_us"] = round(timed(lambda: F.scaled_dot_product_attention(
        *torch.randn(3, B, H, S, D // H, device=dev, dtype=bf).unbind(0))), 2)
    out["layer_us"] = round(timed(lambda: layer(x)), 2)
    out["forward_ms"] = round(timed(forward, max(5, iters // 5)) / 1e3, 4)
    g_graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_graph):
        forward()
    out["forward_graph_ms"] = round(timed(g_graph.replay, max(5, iters // 5)) / 1e3, 4)
flops = L * (2.0 * T * (4 * D * D + 2 * D * FF) + 4.0 * T * S * D)
out["forward_tflops_graph"] = round(flops / (out["forward_graph_ms"] * 1e-3) / 1e12, 1)
out["note"] = "torch eager / CUDA graph: cuBLAS(Lt) linear with bias, SDPA, layer_norm, erf GELU; bf16; warm; CUDA events"
print(json.dumps(out))
