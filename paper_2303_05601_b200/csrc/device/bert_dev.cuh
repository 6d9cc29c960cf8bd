#pragma once
// Device helpers shared by the BERT kernels (bert.cu: per-op K2-K4, bert_flow.cu:
// the whole-encoder dataflow kernel K5).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "common.cuh"

namespace gfx::bertdev {

// Arena virtual offset -> address through the model's page table.
__device__ __forceinline__ const char* translate(const char* arena, const uint32_t* pt, uint64_t v) {
    return arena + (static_cast<uint64_t>(pt[v >> kPageShift]) << kPageShift) + (v & kPageMask);
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// GELU(x) = x/2 (1 + erf(x / sqrt 2)) with erf from Abramowitz & Stegun 7.1.26
// (|error| <= 1.5e-7, far below the bf16 output's 2^-9 relative resolution):
// one rcp, one ex2 and 8 FMAs instead of erff's branchy ~30 instructions — the
// FFN1 epilogue was the bottleneck of that GEMM (~6 µs per 128 x 256 tile
// against ~4.2 µs of MMAs).
__device__ __forceinline__ float gelu(float x) {
    const float z = fabsf(x) * 0.70710678118654752f;
    float t;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(fmaf(0.3275911f, z, 1.0f)));
    const float poly =
        t * fmaf(fmaf(fmaf(fmaf(1.061405429f, t, -1.453152027f), t, 1.421413741f), t, -0.284496736f), t, 0.254829592f);
    float e;  // exp(-z^2) = 2^(-z^2 log2 e)
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-z * z * 1.4426950408889634f));
    const float erf_abs = 1.0f - poly * e;
    return 0.5f * x * (1.0f + copysignf(erf_abs, x));
}

// GELU of two values with the same A&S 7.1.26 erf, in sm_100's packed fp32x2
// arithmetic (FFMA2 / FMUL2 issue one instruction for both lanes): with
// h(x) = 0.5 erfc(|x| / sqrt 2) = 0.5 poly(t) exp(-x^2 / 2), t = 1 / (1 + p |x| / sqrt 2),
// GELU(x) = x Phi(x) = max(x, 0) - |x| h(x) for either sign (the 0.5 and the
// 1/sqrt 2 are folded into the constants). ~9 issue slots per value instead
// of ~25: the FFN1 epilogue (64 GELUs per thread per tile) was issue-bound.
__device__ __forceinline__ float2 gelu2(float2 x) {
    const float2 a = make_float2(fabsf(x.x), fabsf(x.y));
    const float2 d = __ffma2_rn(a, make_float2(0.23164189f, 0.23164189f), make_float2(1.0f, 1.0f));
    float2 t;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t.x) : "f"(d.x));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t.y) : "f"(d.y));
    float2 p = __ffma2_rn(make_float2(0.5307027145f, 0.5307027145f), t, make_float2(-0.7265760135f, -0.7265760135f));
    p = __ffma2_rn(p, t, make_float2(0.7107068705f, 0.7107068705f));
    p = __ffma2_rn(p, t, make_float2(-0.142248368f, -0.142248368f));
    p = __ffma2_rn(p, t, make_float2(0.127414796f, 0.127414796f));
    p = __fmul2_rn(p, t);
    const float2 w = __fmul2_rn(x, __fmul2_rn(x, make_float2(-0.72134752044f, -0.72134752044f)));  // -x^2 log2(e) / 2
    float2 e;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.x) : "f"(w.x));
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e.y) : "f"(w.y));
    const float2 h = __fmul2_rn(p, e);
    return __ffma2_rn(make_float2(-a.x, -a.y), h, make_float2(fmaxf(x.x, 0.f), fmaxf(x.y, 0.f)));
}

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Chan et al. pairwise combination of (count, mean, M2) partial statistics.
__device__ __forceinline__ void chan_combine(float& n_a, float& mean_a, float& m2_a, float n_b, float mean_b, float m2_b) {
    const float n = n_a + n_b, dlt = mean_b - mean_a;
    mean_a = fmaf(dlt, n_b / n, mean_a);
    m2_a = m2_a + m2_b + dlt * dlt * (n_a * n_b / n);
    n_a = n;
}

// 1/sqrt(64) * log2(e): attention scores scaled into the exp2 domain.
constexpr float kAttnScaleLog2 = 0.125f * 1.4426950408889634f;

}  // namespace gfx::bertdev
