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
        /* four batch rows per pass over the weight row (fp64 accumulation, two
         * partial sums per row, combined in a fixed order) */
        int r = 0;
        for (; r + 3 < j->B; r += 4) {
            const float* x0 = j->in + (size_t)r * (size_t)j->K;
            const float* x1 = x0 + j->K;
            const float* x2 = x1 + j->K;
            const float* x3 = x2 + j->K;
            double a0 = 0, b0 = 0, a1 = 0, b1 = 0, a2 = 0, b2 = 0, a3 = 0, b3 = 0;
            int k = 0;
            for (; k + 1 < j->K; k += 2) {
                const double w0 = wr[k], w1 = wr[k + 1];
                a0 += (double)x0[k] * w0;
                b0 += (double)x0[k + 1] * w1;
                a1 += (double)x1[k] * w0;
                b1 += (double)x1[k + 1] * w1;
                a2 += (double)x2[k] * w0;
                b2 += (double)x2[k + 1] * w1;
                a3 += (double)x3[k] * w0;
                b3 += (double)x3[k + 1] * w1;
            }
            for (; k < j->K; ++k) {
                a0 += (double)x0[k] * wr[k];
                a1 += (double)x1[k] * wr[k];
                a2 += (double)x2[k] * wr[k];
                a3 += (double)x3[k] * wr[k];
            }
            const double acc[4] = {a0 + b0, a1 + b1, a2 + b2, a3 + b3};
            for (int i = 0; i < 4; ++i) {
                float v = (float)((double)j->b[n] + acc[i]);
                if (j->relu && v < 0.0f) v = 0.0f;
                j->out[(size_t)(r + i) * (size_t)j->N + (size_t)n] = v;
            }
        }
        for (; r < j->B; ++r) {
            const float* xr = j->in + (size_t)r * (size_t)j->K;
            double a0 = 0, b0 = 0;
            int k = 0;
            for (; k + 1 < j->K; k += 2) {
                a0 += (double)xr[k] * (double)wr[k];
                b0 += (double)xr[k + 1] * (double)wr[k + 1];
            }
            for (; k < j->K; ++k) a0 += (double)xr[k] * (double)wr[k];
            float v = (float)((double)j->b[n] + (a0 + b0));
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
struct orc_mlp {
    int n_layers;
    int32_t dims[ORC_MAX_LAYERS + 1];
    float* w[ORC_MAX_LAYERS];
    float* b[ORC_MAX_LAYERS];
};

orc_mlp* orc_mlp_create(uint64_t model_seed, int n_layers, const int32_t* dims) {
    if (n_layers < 1 || n_layers > ORC_MAX_LAYERS) return NULL;
    orc_mlp* m = calloc(1, sizeof *m);
    if (!m) return NULL;
    m->n_layers = n_layers;
    memcpy(m->dims, dims, (size_t)(n_layers + 1) * sizeof(int32_t));
    for (int l = 0; l < n_layers; ++l) {
        const int K = dims[l], N = dims[l + 1];
        const float scale = (float)(1.0 / sqrt((double)K));
        m->w[l] = malloc((size_t)N * (size_t)K * sizeof(float));
        m->b[l] = malloc((size_t)N * sizeof(float));
        if (!m->w[l] || !m->b[l]) {
            orc_mlp_free(m);
            return NULL;
        }
        orc_fill_params(model_seed, (uint32_t)(2 * l), (uint64_t)N * (uint64_t)K, scale, m->w[l]);
        orc_fill_params(model_seed, (uint32_t)(2 * l + 1), (uint64_t)N, scale, m->b[l]);
    }
    return m;
}

void orc_mlp_free(orc_mlp* m) {
    if (!m) return;
    for (int l = 0; l < m->n_layers; ++l) {
        free(m->w[l]);
        free(m->b[l]);
    }
    free(m);
}

int orc_mlp_run(const orc_mlp* m, int batch, const float* x, float* logits, float* probs, int threads) {
    const int n_layers = m->n_layers;
    const int32_t* dims = m->dims;
    int maxd = 0;
    for (int l = 0; l <= n_layers; ++l) if (dims[l] > maxd) maxd = dims[l];
    float* cur = malloc((size_t)batch * (size_t)maxd * sizeof(float));
    float* nxt = malloc((size_t)batch * (size_t)maxd * sizeof(float));
    if (!cur || !nxt) { free(cur); free(nxt); return -1; }
    memcpy(cur, x, (size_t)batch * (size_t)dims[0] * sizeof(float));
    for (int l = 0; l < n_layers; ++l) {
        run_layer(cur, m->w[l], m->b[l], nxt, batch, dims[l], dims[l + 1], l + 1 < n_layers, threads);
        float* t = cur; cur = nxt; nxt = t;
    }
    int C = dims[n_layers];
    memcpy(logits, cur, (size_t)batch * (size_t)C * sizeof(float));
    if (probs) {
        for (int r = 0; r < batch; ++r) {
            const float* lr = cur + (size_t)r * (size_t)C;
            double mx = lr[0];
            for (int c = 1; c < C; ++c) if (lr[c] > mx) mx = lr[c];
            double s = 0;
            for (int c = 0; c < C; ++c) s += exp((double)lr[c] - mx);
            for (int c = 0; c < C; ++c) probs[(size_t)r * (size_t)C + (size_t)c] = (float)(exp((double)lr[c] - mx) / s);
        }
    }
    free(cur);
    free(nxt);
    return 0;
}

int orc_mlp_forward(uint64_t model_seed, int n_layers, const int32_t* dims, int batch, const float* x,
                    float* logits, float* probs, int threads) {
    orc_mlp* m = orc_mlp_create(model_seed, n_layers, dims);
    if (!m) return -1;
    const int rc = orc_mlp_run(m, batch, x, logits, probs, threads);
    orc_mlp_free(m);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* BERT-base-style encoder (C5), restated from DESIGN.md §4:
 * post-LN layers  qkv = XWqkv^T+b; ctx = softmax(QK^T/8)V per head;
 *                 h = LN1(X + ctx Wo^T + bo); f = GELU(h W1^T + b1);
 *                 X = LN2(h + f W2^T + b2);  pooled = tanh(Wp x_cls + bp).
 * fp64 accumulation; activations rounded to bf16 where the product stores
 * bf16 (every GEMM/attention/LN output); attention probabilities rounded to
 * bf16 for the P.V product, normaliser from unrounded values; LN eps 1e-12. */

static float bf16_round(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7F800000u) != 0x7F800000u) u += 0x7FFFu + ((u >> 16) & 1u);
    u &= 0xFFFF0000u;
    float r;
    memcpy(&r, &u, 4);
    return r;
}

typedef struct {
    const float* a;  /* T x K */
    const float* w;  /* N x K */
    double* out;     /* T x N */
    int T, K, N, t, nt;
} gjob;

/* Test hook: accumulate GEMMs in fp32 (k order) instead of fp64 — used only to
 * measure the network's intrinsic sensitivity to accumulation precision. */
static int g_acc32 = 0;
void orc_set_acc32(int on) { g_acc32 = on; }

static void* gemm_worker(void* arg) {
    gjob* j = arg;
    if (g_acc32) {
        for (int n = j->t; n < j->N; n += j->nt) {
            const float* wr = j->w + (size_t)n * (size_t)j->K;
            for (int r = 0; r < j->T; ++r) {
                const float* ar = j->a + (size_t)r * (size_t)j->K;
                float a = 0.f;
                for (int k = 0; k < j->K; ++k) a = fmaf(ar[k], wr[k], a);
                j->out[(size_t)r * (size_t)j->N + (size_t)n] = a;
            }
        }
        return NULL;
    }
    for (int n = j->t; n < j->N; n += j->nt) {
        const float* wr = j->w + (size_t)n * (size_t)j->K;
        for (int r = 0; r < j->T; ++r) {
            const float* ar = j->a + (size_t)r * (size_t)j->K;
            double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
            int k = 0;
            for (; k + 3 < j->K; k += 4) {
                a0 += (double)ar[k] * wr[k];
                a1 += (double)ar[k + 1] * wr[k + 1];
                a2 += (double)ar[k + 2] * wr[k + 2];
                a3 += (double)ar[k + 3] * wr[k + 3];
            }
            for (; k < j->K; ++k) a0 += (double)ar[k] * wr[k];
            j->out[(size_t)r * (size_t)j->N + (size_t)n] = (a0 + a1) + (a2 + a3);
        }
    }
    return NULL;
}

static void par_gemm(const float* a, const float* w, double* out, int T, int K, int N, int threads) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t th[256];
    gjob jobs[256];
    for (int t = 0; t < threads; ++t) {
        jobs[t] = (gjob){a, w, out, T, K, N, t, threads};
        if (t) pthread_create(&th[t], NULL, gemm_worker, &jobs[t]);
    }
    gemm_worker(&jobs[0]);
    for (int t = 1; t < threads; ++t) pthread_join(th[t], NULL);
}

/* bf16 weight matrix [n x k] of tensor id, values rounded to bf16 */
static float* bert_mat(uint64_t seed, uint32_t tensor, int n, int k) {
    float* w = malloc((size_t)n * (size_t)k * sizeof(float));
    orc_fill_params(seed, tensor, (uint64_t)n * (uint64_t)k, (float)(1.0 / sqrt((double)k)), w);
    for (size_t i = 0; i < (size_t)n * (size_t)k; ++i) w[i] = bf16_round(w[i]);
    return w;
}
static float* bert_vec(uint64_t seed, uint32_t tensor, int n, float scale, float shift) {
    float* v = malloc((size_t)n * sizeof(float));
    orc_fill_params(seed, tensor, (uint64_t)n, scale, v);
    for (int i = 0; i < n; ++i) v[i] = shift + v[i];
    return v;
}

static void layernorm_rows(const float* x, float* y, const float* g, const float* b, int T, int d) {
    for (int t = 0; t < T; ++t) {
        const float* xr = x + (size_t)t * (size_t)d;
        double mean = 0, var = 0;
        for (int i = 0; i < d; ++i) mean += xr[i];
        mean /= d;
        for (int i = 0; i < d; ++i) var += (xr[i] - mean) * (xr[i] - mean);
        var /= d;
        const double rstd = 1.0 / sqrt(var + 1e-12);
        for (int i = 0; i < d; ++i) y[(size_t)t * (size_t)d + (size_t)i] = bf16_round((float)((xr[i] - mean) * rstd * g[i] + b[i]));
    }
}

/* One encoder layer l on x (in place): fp64 accumulation, bf16 rounding points.
 * lengths (NULL: every sequence is full): sequence s attends to its first
 * lengths[s] keys only (padding mask: keys j >= len excluded from the softmax,
 * as transformers' additive -inf attention mask); every query row is computed. */
static int bert_layer(uint64_t seed, int l, int d, int heads, int ffn, int seq, int batch, float* x, int threads,
                      const int32_t* lengths) {
    const int T = batch * seq, dh = d / heads;
    float* qkv = malloc((size_t)T * 3 * (size_t)d * sizeof(float));
    float* ctx = malloc((size_t)T * (size_t)d * sizeof(float));
    float* h = malloc((size_t)T * (size_t)d * sizeof(float));
    float* t1 = malloc((size_t)T * (size_t)d * sizeof(float));
    float* f = malloc((size_t)T * (size_t)ffn * sizeof(float));
    double* acc = malloc((size_t)T * (size_t)(ffn > 3 * d ? ffn : 3 * d) * sizeof(double));
    double* srow = malloc((size_t)seq * sizeof(double));
    if (!qkv || !ctx || !h || !t1 || !f || !acc || !srow) return -1;
    const uint32_t t0 = 16u * (uint32_t)l;
    float* wqkv = bert_mat(seed, t0 + 0, 3 * d, d);
    float* bqkv = bert_vec(seed, t0 + 1, 3 * d, 0.02f, 0.f);
    float* wo = bert_mat(seed, t0 + 2, d, d);
    float* bo = bert_vec(seed, t0 + 3, d, 0.02f, 0.f);
    float* g1 = bert_vec(seed, t0 + 4, d, 0.1f, 1.f);
    float* be1 = bert_vec(seed, t0 + 5, d, 0.1f, 0.f);
    float* w1 = bert_mat(seed, t0 + 6, ffn, d);
    float* b1 = bert_vec(seed, t0 + 7, ffn, 0.02f, 0.f);
    float* w2 = bert_mat(seed, t0 + 8, d, ffn);
    float* b2 = bert_vec(seed, t0 + 9, d, 0.02f, 0.f);
    float* g2 = bert_vec(seed, t0 + 10, d, 0.1f, 1.f);
    float* be2 = bert_vec(seed, t0 + 11, d, 0.1f, 0.f);
    /* QKV projection */
    par_gemm(x, wqkv, acc, T, d, 3 * d, threads);
    for (int t = 0; t < T; ++t)
        for (int n = 0; n < 3 * d; ++n)
            qkv[(size_t)t * 3 * (size_t)d + (size_t)n] = bf16_round((float)(acc[(size_t)t * 3 * (size_t)d + (size_t)n] + bqkv[n]));
    /* attention per (sequence, head) */
    for (int s = 0; s < batch; ++s)
        for (int hh = 0; hh < heads; ++hh)
            for (int i = 0; i < seq; ++i) {
                const int nk = lengths ? lengths[s] : seq; /* valid keys of this sequence */
                const float* q = qkv + ((size_t)s * seq + (size_t)i) * 3 * (size_t)d + (size_t)hh * dh;
                double m = -INFINITY;
                for (int j = 0; j < nk; ++j) {
                    const float* k = qkv + ((size_t)s * seq + (size_t)j) * 3 * (size_t)d + (size_t)d + (size_t)hh * dh;
                    double sc = 0;
                    for (int e = 0; e < dh; ++e) sc += (double)q[e] * k[e];
                    srow[j] = sc;
                    if (sc > m) m = sc;
                }
                double lsum = 0;
                for (int j = 0; j < nk; ++j) {
                    srow[j] = exp((srow[j] - m) * 0.125);
                    lsum += srow[j];
                }
                for (int e = 0; e < dh; ++e) {
                    double o = 0;
                    for (int j = 0; j < nk; ++j) {
                        const float* v = qkv + ((size_t)s * seq + (size_t)j) * 3 * (size_t)d + 2 * (size_t)d + (size_t)hh * dh;
                        o += (double)bf16_round((float)srow[j]) * v[e];
                    }
                    ctx[((size_t)s * seq + (size_t)i) * (size_t)d + (size_t)hh * dh + (size_t)e] = bf16_round((float)(o / lsum));
                }
            }
    /* output projection + residual, LN1 */
    par_gemm(ctx, wo, acc, T, d, d, threads);
    for (size_t i = 0; i < (size_t)T * (size_t)d; ++i) t1[i] = bf16_round((float)(acc[i] + bo[i % (size_t)d] + x[i]));
    layernorm_rows(t1, h, g1, be1, T, d);
    /* FFN */
    par_gemm(h, w1, acc, T, d, ffn, threads);
    for (size_t i = 0; i < (size_t)T * (size_t)ffn; ++i) {
        const double v = acc[i] + b1[i % (size_t)ffn];
        f[i] = bf16_round((float)(0.5 * v * (1.0 + erf(v * 0.70710678118654752))));
    }
    par_gemm(f, w2, acc, T, ffn, d, threads);
    for (size_t i = 0; i < (size_t)T * (size_t)d; ++i) t1[i] = bf16_round((float)(acc[i] + b2[i % (size_t)d] + h[i]));
    layernorm_rows(t1, x, g2, be2, T, d);
    free(wqkv); free(bqkv); free(wo); free(bo); free(g1); free(be1);
    free(w1); free(b1); free(w2); free(b2); free(g2); free(be2);
    free(qkv); free(ctx); free(h); free(t1); free(f); free(acc); free(srow);
    return 0;
}

static void bits_to_float(const uint16_t* b, float* x, size_t n) {
    for (size_t i = 0; i < n; ++i) {
        uint32_t u = (uint32_t)b[i] << 16;
        memcpy(&x[i], &u, 4);
    }
}
static void float_to_bits(const float* x, uint16_t* b, size_t n) {
    for (size_t i = 0; i < n; ++i) {
        uint32_t u;
        memcpy(&u, &x[i], 4);
        b[i] = (uint16_t)(u >> 16); /* values are already bf16-exact */
    }
}

/* Pooler on each sequence's first token. */
static void bert_pool(uint64_t seed, int L, int d, int seq, int batch, const float* x, float* pooled) {
    const uint32_t tp = 16u * (uint32_t)L;
    float* wp = bert_mat(seed, tp + 0, d, d);
    float* bp = bert_vec(seed, tp + 1, d, 0.02f, 0.f);
    for (int s = 0; s < batch; ++s)
        for (int n = 0; n < d; ++n) {
            const float* xr = x + (size_t)s * seq * (size_t)d;
            double a = 0;
            for (int k = 0; k < d; ++k) a += (double)wp[(size_t)n * d + (size_t)k] * xr[k];
            pooled[(size_t)s * d + (size_t)n] = (float)tanh(a + bp[n]);
        }
    free(wp);
    free(bp);
}

int orc_bert_layer(uint64_t seed, int l, int d, int heads, int ffn, int seq, int batch, const uint16_t* x_in,
                   uint16_t* x_out, int threads) {
    const size_t n = (size_t)batch * seq * (size_t)d;
    float* x = malloc(n * sizeof(float));
    if (!x) return -1;
    bits_to_float(x_in, x, n);
    int rc = bert_layer(seed, l, d, heads, ffn, seq, batch, x, threads, NULL);
    float_to_bits(x, x_out, n);
    free(x);
    return rc;
}

int orc_bert_layer_masked(uint64_t seed, int l, int d, int heads, int ffn, int seq, int batch, const int32_t* lengths,
                          const uint16_t* x_in, uint16_t* x_out, int threads) {
    for (int s = 0; s < batch; ++s)
        if (lengths[s] < 1 || lengths[s] > seq) return -1;
    const size_t n = (size_t)batch * seq * (size_t)d;
    float* x = malloc(n * sizeof(float));
    if (!x) return -1;
    bits_to_float(x_in, x, n);
    int rc = bert_layer(seed, l, d, heads, ffn, seq, batch, x, threads, lengths);
    float_to_bits(x, x_out, n);
    free(x);
    return rc;
}

int orc_bert_pool(uint64_t seed, int L, int d, int seq, int batch, const uint16_t* x_bits, float* pooled) {
    const size_t n = (size_t)batch * seq * (size_t)d;
    float* x = malloc(n * sizeof(float));
    if (!x) return -1;
    bits_to_float(x_bits, x, n);
    bert_pool(seed, L, d, seq, batch, x, pooled);
    free(x);
    return 0;
}

int orc_bert_forward(uint64_t seed, int L, int d, int heads, int ffn, int seq, int batch, const uint16_t* x_bits,
                     float* pooled, int threads) {
    const size_t n = (size_t)batch * seq * (size_t)d;
    float* x = malloc(n * sizeof(float));
    if (!x) return -1;
    bits_to_float(x_bits, x, n);
    for (int l = 0; l < L; ++l)
        if (bert_layer(seed, l, d, heads, ffn, seq, batch, x, threads, NULL)) { free(x); return -1; }
    bert_pool(seed, L, d, seq, batch, x, pooled);
    free(x);
    return 0;
}
