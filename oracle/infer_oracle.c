/* ORACLE / TEST INFRASTRUCTURE ONLY — see gpufaas_oracle.h.
 *
 * CPU numerics restatement of the inference models the B200 build serves.
 * The reference has no inference implementation (its "inference" is the
 * profiled constant infer_time_us, proj/src/cluster.cpp:161,167), so this is
 * "parity unpinned" with respect to the reference: it restates the model
 * definition of DESIGN.md §4 with fp64 accumulation and the product's fp32
 * rounding points (each layer output rounded to fp32 before the next layer).
 */
#define _POSIX_C_SOURCE 200809L
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#include "gpufaas_oracle.h"

/* splitmix64 finaliser (public-domain constants) */
static uint64_t mix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ULL;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
    return x ^ (x >> 31);
}

/* value = (int24 uniform) * (scale * 2^-23): exact int->float, exact power-of-two
 * scaling, one rounding in the final multiply. DESIGN.md §4. */
float orc_param_value(uint64_t model_seed, uint32_t tensor, uint64_t index, float scale) {
    uint64_t stream = mix64(model_seed ^ ((uint64_t)tensor * 0xD1B54A32D192ED03ULL));
    uint64_t h = mix64(stream + index);
    int32_t u = (int32_t)(h >> 40) - (1 << 23);
    float s = scale * 0x1.0p-23f;
    return (float)u * s;
}

void orc_fill_params(uint64_t model_seed, uint32_t tensor, uint64_t n, float scale, float* out) {
    uint64_t stream = mix64(model_seed ^ ((uint64_t)tensor * 0xD1B54A32D192ED03ULL));
    float s = scale * 0x1.0p-23f;
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t h = mix64(stream + i);
        int32_t u = (int32_t)(h >> 40) - (1 << 23);
        out[i] = (float)u * s;
    }
}

typedef struct {
    const float* in;   /* B x K */
    const float* w;    /* N x K */
    const float* b;    /* N */
    float* out;        /* B x N */
    int B, K, N, relu, t, nt;
} job;

static void* layer_worker(void* arg) {
    job* j = arg;
    for (int n = j->t; n < j->N; n += j->nt) {
        const float* wr = j->w + (size_t)n * (size_t)j->K;
        for (int r = 0; r < j->B; ++r) {
            const float* xr = j->in + (size_t)r * (size_t)j->K;
            double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
            int k = 0;
            for (; k + 3 < j->K; k += 4) {
                a0 += (double)xr[k] * (double)wr[k];
                a1 += (double)xr[k + 1] * (double)wr[k + 1];
                a2 += (double)xr[k + 2] * (double)wr[k + 2];
                a3 += (double)xr[k + 3] * (double)wr[k + 3];
            }
            for (; k < j->K; ++k) a0 += (double)xr[k] * (double)wr[k];
            double acc = (double)j->b[n] + ((a0 + a1) + (a2 + a3));
            float v = (float)acc;
            if (j->relu && v < 0.0f) v = 0.0f;
            j->out[(size_t)r * (size_t)j->N + (size_t)n] = v;
        }
    }
    return NULL;
}

static void run_layer(const float* in, const float* w, const float* b, float* out, int B, int K, int N,
                      int relu, int threads) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t th[256];
    job jobs[256];
    for (int t = 0; t < threads; ++t) {
        jobs[t] = (job){in, w, b, out, B, K, N, relu, t, threads};
        if (t) pthread_create(&th[t], NULL, layer_worker, &jobs[t]);
    }
    layer_worker(&jobs[0]);
    for (int t = 1; t < threads; ++t) pthread_join(th[t], NULL);
}

/* Weight tensor of layer l is tensor id 2l (row-major N x K, PyTorch Linear
 * layout), its bias is tensor 2l+1; scale = 1/sqrt(K). */
int orc_mlp_forward(uint64_t model_seed, int n_layers, const int32_t* dims, int batch, const float* x,
                    float* logits, float* probs, int threads) {
    int maxd = 0;
    for (int l = 0; l <= n_layers; ++l) if (dims[l] > maxd) maxd = dims[l];
    float* cur = malloc((size_t)batch * (size_t)maxd * sizeof(float));
    float* nxt = malloc((size_t)batch * (size_t)maxd * sizeof(float));
    if (!cur || !nxt) { free(cur); free(nxt); return -1; }
    memcpy(cur, x, (size_t)batch * (size_t)dims[0] * sizeof(float));
    for (int l = 0; l < n_layers; ++l) {
        int K = dims[l], N = dims[l + 1];
        float scale = (float)(1.0 / sqrt((double)K));
        float* w = malloc((size_t)N * (size_t)K * sizeof(float));
        float* b = malloc((size_t)N * sizeof(float));
        if (!w || !b) { free(w); free(b); free(cur); free(nxt); return -1; }
        orc_fill_params(model_seed, (uint32_t)(2 * l), (uint64_t)N * (uint64_t)K, scale, w);
        orc_fill_params(model_seed, (uint32_t)(2 * l + 1), (uint64_t)N, scale, b);
        run_layer(cur, w, b, nxt, batch, K, N, l + 1 < n_layers, threads);
        free(w);
        free(b);
        float* t = cur; cur = nxt; nxt = t;
    }
    int C = dims[n_layers];
    memcpy(logits, cur, (size_t)batch * (size_t)C * sizeof(float));
    if (probs) {
        for (int r = 0; r < batch; ++r) {
            const float* lr = cur + (size_t)r * (size_t)C;
            double m = lr[0];
            for (int c = 1; c < C; ++c) if (lr[c] > m) m = lr[c];
            double s = 0;
            for (int c = 0; c < C; ++c) s += exp((double)lr[c] - m);
            for (int c = 0; c < C; ++c) probs[(size_t)r * (size_t)C + (size_t)c] = (float)(exp((double)lr[c] - m) / s);
        }
    }
    free(cur);
    free(nxt);
    return 0;
}
