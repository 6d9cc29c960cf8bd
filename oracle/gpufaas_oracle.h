/* ORACLE / TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference GPU function-execution control plane
 * (arXiv 2303.05601 reference simulator, /root/reference/proj) plus the CPU
 * numerics restatement of the inference models the B200 build executes.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library; the product never links it.
 *
 * Pinning: the control-plane restatement is checked field-by-field against
 * the compiled UNMODIFIED reference (oracle/_ref/libgpufaas_ref.so) and against
 * the golden digests of SURVEY.md Appendix B.1 (tests/golden/). The inference
 * restatement has no reference to pin against (the reference has no GPU or
 * inference code): "parity unpinned" for numerics; it is a
 * fp64-accumulating restatement of the model definition in DESIGN.md §4.
 *
 * Canonical digests (shared with oracle/ref_shim.cpp and the product):
 *   decision digest = FNV-1a-64 over, per decision in order:
 *       i32 kind, i32 request_id, i32 gpu_id, i32 from_local_queue,
 *       i32 false_miss, i32 skip_count, i64 completion_us, i64 load_us,
 *       i64 infer_us, i32 n_evicted, then each evicted model id + '\0'
 *     (little-endian raw bytes).
 *   request digest  = FNV-1a-64 over, per request: i64 dispatched_at_us,
 *       i64 completed_at_us, i32 skip_count.
 *   log digest      = FNV-1a-64 over the EventLogger JSON-lines bytes
 *       (proj/src/engine.cpp:63-98).
 */
#ifndef GPUFAAS_ORACLE_H
#define GPUFAAS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int32_t gpu_count;
    int32_t policy; /* 0 lb, 1 lalb, 2 lalbo3 (proj/include/gpufaas/sched.hpp:17) */
    int32_t o3_limit;
    int32_t working_set;
    int32_t per_minute_total;
    int32_t duration_minutes;
    int32_t use_synthetic_trace;
    int32_t syn_function_count;
    int32_t syn_minutes;
    int32_t syn_draws_per_minute;
    int32_t debug_checks;
    int32_t log_events; /* 0 none, 1 log, 2 log + caches */
    int32_t use_reference_scheduler; /* ignored: the oracle has one scheduler */
    int32_t pipeline; /* extension: pipelined GPUs (one staged task behind the running one); 0 = reference */
    double capacity_mb;
    double syn_zipf_exponent;
    uint64_t seed;
    uint64_t syn_seed;
} orc_sim_config;

typedef struct {
    int64_t request_count;
    double total_sim_time_s;
    int32_t has_latency, has_ratios, has_time;
    int32_t max_skip_count;
    double avg_latency_s, latency_variance_s2;
    double cache_miss_ratio, false_miss_ratio;
    double avg_top_model_duplicates, utilization_busy, utilization_infer_only;
    int64_t hits, misses, false_misses, local_enqueues, evictions;
    int32_t top_model_idx;
    int32_t pad_;
} orc_report;

const char* orc_sim_last_error(void);
void* orc_sim_run(const char* catalog_csv, const char* trace_csv, const orc_sim_config* cfg);
void* orc_sim_run_stream(const char* catalog_csv, const orc_sim_config* cfg, int n,
                         const int32_t* model_idx, const int64_t* arrival_us);
int64_t orc_sim_num_decisions(void* h);
int64_t orc_sim_num_requests(void* h);
double orc_sim_run_ns(void* h);
void orc_sim_get_decisions(void* h, int32_t* ints7, int64_t* times3);
void orc_sim_get_requests(void* h, int32_t* model_idx, int64_t* arrival, int64_t* dispatched,
                          int64_t* completed, int32_t* skip);
/* evicted model indices of decision i (catalog rows), returns count */
int32_t orc_sim_get_evicted(void* h, int64_t i, int32_t* out, int32_t cap);
void orc_sim_get_report(void* h, orc_report* out);
uint64_t orc_sim_decision_digest(void* h);
uint64_t orc_sim_request_digest(void* h);
uint64_t orc_sim_log_digest(void* h);
int64_t orc_sim_log_size(void* h);
const char* orc_sim_log(void* h);
void orc_sim_free(void* h);

/* Synthetic Azure-style trace as CSV (proj/src/trace.cpp:156-192). Caller frees with orc_free. */
char* orc_synthetic_trace_csv(int function_count, int minutes, int draws, double zipf, uint64_t seed);
void orc_free(void* p);

/* Raw mt19937_64 stream (proj/include/gpufaas/rng.hpp:11-30) for KATs. */
void orc_mt19937_64(uint64_t seed, int64_t n, uint64_t* out);

/* ---------------- inference numerics restatement (infer_oracle.c) ---------------- */
/* Deterministic parameter / input generation shared bit-for-bit with the product
 * (DESIGN.md §4): counter-based splitmix64 → 24-bit uniform → float. */
float orc_param_value(uint64_t model_seed, uint32_t tensor, uint64_t index, float scale);
void orc_fill_params(uint64_t model_seed, uint32_t tensor, uint64_t n, float scale, float* out);

/* fp32 MLP classifier forward with fp64 accumulation:
 *   h_0 = x (B x d_0); h_{l+1} = relu(h_l W_l^T + b_l) for l < L-1;
 *   logits = h_{L-1} W_{L-1}^T + b_{L-1}; probs = softmax(logits) per row.
 * dims has L+1 entries. Weights/biases generated from model_seed. Uses up to
 * `threads` POSIX threads. */
int orc_mlp_forward(uint64_t model_seed, int n_layers, const int32_t* dims, int batch,
                    const float* x, float* logits, float* probs, int threads);

/* The same forward on a model whose parameters were generated once
 * (orc_mlp_create), so a CPU baseline times the forward alone. */
#define ORC_MAX_LAYERS 16
typedef struct orc_mlp orc_mlp;
orc_mlp* orc_mlp_create(uint64_t model_seed, int n_layers, const int32_t* dims);
int orc_mlp_run(const orc_mlp* m, int batch, const float* x, float* logits, float* probs, int threads);
void orc_mlp_free(orc_mlp* m);

/* BERT-base-style encoder (C5) forward, fp64 accumulation with the product's
 * bf16 rounding points. x_bits: [batch*seq x d] bf16 bit patterns;
 * pooled: [batch x d] fp32. */
int orc_bert_forward(uint64_t seed, int L, int d, int heads, int ffn, int seq, int batch, const uint16_t* x_bits,
                     float* pooled, int threads);
/* Teacher-forced pieces: encoder layer l applied to a given bf16 input, and the
 * pooler applied to a given final hidden state. */
int orc_bert_layer(uint64_t seed, int l, int d, int heads, int ffn, int seq, int batch, const uint16_t* x_in,
                   uint16_t* x_out, int threads);
/* orc_bert_layer with a padding mask: sequence s attends to its first lengths[s]
 * keys (1 <= lengths[s] <= seq). Returns -1 on a bad length. */
int orc_bert_layer_masked(uint64_t seed, int l, int d, int heads, int ffn, int seq, int batch, const int32_t* lengths,
                          const uint16_t* x_in, uint16_t* x_out, int threads);
int orc_bert_pool(uint64_t seed, int L, int d, int seq, int batch, const uint16_t* x_bits, float* pooled);
/* Test hook: fp32 (k-order) GEMM accumulation, to measure intrinsic sensitivity. */
void orc_set_acc32(int on);

#ifdef __cplusplus
}
#endif
#endif
