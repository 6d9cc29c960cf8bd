/* gpufaas_b200.h — C-ABI of the B200 GPU function-execution path.
 *
 * Host code (the C++ control plane under include/gpufaas/) reaches CUDA only
 * through these entry points: plain pointers, sizes and int status codes, no
 * exceptions and no torch types across the boundary. The reference has no FFI
 * of its own; each entry point names the reference interface
 * whose profiled constant it replaces with real device work:
 *
 *   gfx_arena_create   <- GpuState::capacity_mb_ accounting
 *                         (proj/include/gpufaas/cluster.hpp:74-77)
 *   gfx_load_h2d       <- profile.load_time_us charged on a miss
 *                         (proj/src/cluster.cpp:163-167)
 *   gfx_fetch_p2p      <- the false-miss reload (proj/src/sched.cpp:117,127;
 *                         locations(): proj/src/cluster.cpp:69-72)
 *   gfx_evict          <- ClusterState::evict_one (proj/src/cluster.cpp:117-129)
 *   gfx_infer          <- profile.infer_time_us (proj/src/cluster.cpp:161,167)
 *   gfx_event_*        <- ClusterState::complete (proj/src/cluster.cpp:176-187)
 *   gfx_replay         <- run_stream (proj/src/engine.cpp:100-173) driving
 *                         one GPU manager per device
 *   gfx_sim_*          <- run()/run_stream() of the control plane alone, with
 *                         canonical digests (see oracle/gpufaas_oracle.h)
 *
 * Status codes: 0 = ok, GFX_ERR_DOMAIN (1) = the reference's std::runtime_error
 * class (bad input, model cannot fit, ...), GFX_ERR_INTERNAL (2) = its
 * std::logic_error class (invariant violation), GFX_ERR_CUDA (3) = CUDA
 * failure or no device. gfx_last_error() holds the message (thread-local).
 * INTEGRATION.md shows the ctypes / C++ bindings.
 */
#ifndef GPUFAAS_B200_H
#define GPUFAAS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GFX_OK 0
#define GFX_ERR_DOMAIN 1
#define GFX_ERR_INTERNAL 2
#define GFX_ERR_CUDA 3

#define GFX_PAGE_BYTES (2u << 20) /* HBM arena page: 2 MiB */
#define GFX_MAX_PAGES 1024        /* largest model: 2 GiB (the page table travels by value in kernel parameters) */
#define GFX_MAX_LAYERS 16

/* ---------------------------------------------------------------- sim ABI */
typedef struct {
    int32_t gpu_count;
    int32_t policy; /* 0 lb, 1 lalb, 2 lalbo3 */
    int32_t o3_limit;
    int32_t working_set;
    int32_t per_minute_total;
    int32_t duration_minutes;
    int32_t use_synthetic_trace;
    int32_t syn_function_count;
    int32_t syn_minutes;
    int32_t syn_draws_per_minute;
    int32_t debug_checks;
    int32_t log_events; /* 0 none, 1 events, 2 events + cache contents */
    int32_t use_reference_scheduler; /* unused by the product */
    int32_t pipeline; /* extension: pipelined GPUs (SchedulerConfig::pipeline); 0 = reference semantics */
    double capacity_mb;
    double syn_zipf_exponent;
    uint64_t seed;
    uint64_t syn_seed;
} gfx_sim_config;

const char* gfx_sim_last_error(void);
void* gfx_sim_run(const char* catalog_csv, const char* trace_csv, const gfx_sim_config* cfg);
void* gfx_sim_run_stream(const char* catalog_csv, const gfx_sim_config* cfg, int n,
                         const int32_t* model_idx, const int64_t* arrival_us);
/* Extension: run_live() (see gfx_replay_run_live) against a
 * timed stand-in device on which every task takes its catalog duration /
 * time_scale of real time and reports those durations as measured (for
 * ema_alpha > 0). Request times are real microseconds. */
void* gfx_sim_run_live_timed(const char* catalog_csv, const char* trace_csv, const gfx_sim_config* cfg,
                             double time_scale, double ema_alpha);
/* Extension: convert an Azure Functions 2019 invocation
 * file ("HashOwner,HashApp,HashFunction,Trigger,1..1440") into the trace CSV
 * ("function_id,m1..mN") of its top_k functions by invocations over the first
 * max_minutes (0 = all), streaming (O(top_k x minutes) memory).
 * Returns 0, or -1 with gfx_sim_last_error(). */
int gfx_sim_azure_convert(const char* in_path, const char* out_path, int top_k, int max_minutes,
                          int64_t* rows_read, int64_t* rows_kept);
int64_t gfx_sim_num_decisions(void* h);
int64_t gfx_sim_num_requests(void* h);
double gfx_sim_run_ns(void* h);
void gfx_sim_get_decisions(void* h, int32_t* ints7, int64_t* times3);
void gfx_sim_get_requests(void* h, int32_t* model_idx, int64_t* arrival, int64_t* dispatched,
                          int64_t* completed, int32_t* skip);
uint64_t gfx_sim_decision_digest(void* h);
uint64_t gfx_sim_request_digest(void* h);
uint64_t gfx_sim_log_digest(void* h);
int64_t gfx_sim_log_size(void* h);
const char* gfx_sim_log(void* h);
const char* gfx_sim_report_json(void* h);
void gfx_sim_free(void* h);

/* ------------------------------------------------------------ data plane */
typedef struct gfx_arena_s* gfx_arena_t; /* one per device: the GPU manager */
typedef struct gfx_event_s* gfx_event_t;

#define GFX_MODEL_MLP 1  /* fp32 MLP classifier: relu(xW^T+b) ... softmax */
#define GFX_MODEL_BERT 2 /* bf16 post-LN transformer encoder + tanh pooler (C5) */

typedef struct {
    int32_t family;             /* GFX_MODEL_* */
    int32_t n_layers;           /* MLP: linear layers; BERT: encoder layers */
    int32_t dims[GFX_MAX_LAYERS + 1]; /* MLP: dims[0] = input features, dims[L] = classes;
                                         BERT: {d_model, heads, ffn, seq} */
    int32_t batch;              /* MLP: rows per request (32); BERT: sequences per request */
    int32_t pad_;
    uint64_t seed;              /* parameter stream */
} gfx_model_desc;

const char* gfx_last_error(void);
int gfx_device_count(int* out);
int gfx_device_init(int dev, int enable_peers);

/* Model repository in pinned host memory (the paper's host-side model store).
 * Builds the model's parameter blob; idx is the catalog row. */
int gfx_model_register(int model_idx, const gfx_model_desc* desc);
int gfx_model_bytes(int model_idx, uint64_t* bytes);
int gfx_model_pages(int model_idx, int32_t* pages);
/* Bytes of one request's input / output tensors for this model. */
int gfx_model_io_bytes(int model_idx, uint64_t* in_bytes, uint64_t* out_bytes);
int gfx_models_clear(void);

/* Pre-allocated HBM arena of `capacity_bytes` (multiple of GFX_PAGE_BYTES)
 * plus the manager's streams and workspaces on device `dev`. */
int gfx_arena_create(int dev, uint64_t capacity_bytes, gfx_arena_t* out);
int gfx_arena_destroy(gfx_arena_t a);
int gfx_arena_reset(gfx_arena_t a); /* synchronise, evict everything */
int gfx_arena_free_pages(gfx_arena_t a, int32_t* out);
/* Explicit manager options (no environment switches on the product path). */
#define GFX_OPT_GEMM_PAIR 1 /* BERT GEMMs on 2-SM (cta_group::2) tiles where the shape allows; default 0 */
#define GFX_OPT_BERT_FLOW 2 /* BERT forward as the encoder dataflow kernel K5 (one launch) instead of per-op K2-K4 launches; default 0 */
int gfx_arena_set_option(gfx_arena_t a, int32_t option, int32_t value);
int gfx_arena_resident(gfx_arena_t a, int model_idx, int32_t* out);

/* Cache operations. Each is asynchronous on the manager's streams; `done`
 * (optional) receives an event that fires when the operation completes. */
int gfx_load_h2d(gfx_arena_t a, int model_idx, gfx_event_t* done);
int gfx_fetch_p2p(gfx_arena_t dst, gfx_arena_t src, int model_idx, gfx_event_t* done);
int gfx_evict(gfx_arena_t a, int model_idx);
/* One batched inference of a resident model (DEVICE pointers on the arena's device).
 * MLP:  in [batch x dims[0]] fp32, out [2][batch x classes] fp32 (logits, softmax).
 * BERT: in [batch*seq x d] bf16 embeddings, out [batch x d] fp32 pooled output. */
int gfx_infer(gfx_arena_t a, int model_idx, const void* in, void* out, int batch, gfx_event_t* done);

/* Bench: n back-to-back inferences of resident models models[i] on the compute
 * stream (input i at in + i * in_stride, output at out + (i % 2) * out_stride,
 * device pointers), bracketed by two CUDA events; *ms = their elapsed time.
 * Synchronous. The dominant kernel's average launch duration = *ms / n. */
int gfx_infer_sequence(gfx_arena_t a, const int32_t* models, int n, const void* in, uint64_t in_stride, void* out,
                       uint64_t out_stride, double* ms);

/* Test/debug: BERT inference that also copies every layer's hidden state into
 * hidden ([L+1][batch*seq][d] bf16, device) for teacher-forced parity checks. */
int gfx_infer_debug(gfx_arena_t a, int model_idx, const void* in, void* out, int batch, void* hidden);

/* BERT inference of padded sequences: lengths (HOST, [batch] int32, each in
 * 1..seq) = valid tokens per sequence; attention ignores keys at or beyond a
 * sequence's length (the additive -inf padding mask of BERT serving). hidden:
 * optional, as gfx_infer_debug (then synchronous). Status 1 on a bad length. */
int gfx_infer_masked(gfx_arena_t a, int model_idx, const void* in, void* out, int batch, const int32_t* lengths,
                     void* hidden, gfx_event_t* done);

/* Test/debug: one encoder GEMM of a resident BERT model with its fused epilogue,
 * on `tokens` rows (bf16, device pointers). op 0: QKV (+bias) [tokens x 3d];
 * 1: attention output (+bias, +resid) [tokens x d]; 2: FFN1 (+bias, GELU)
 * [tokens x ffn]; 3: FFN2 (+bias, +resid) [tokens x d]; 4 / 5: op 1 / 3 followed
 * by LayerNorm 1 / 2 (the forward's fused residual + LayerNorm step). Synchronous. */
int gfx_bert_gemm(gfx_arena_t a, int model_idx, int layer, int op, const void* x, const void* resid, void* y,
                  int tokens);

int gfx_event_query(gfx_event_t e); /* 0 done, 1 pending */
int gfx_event_sync(gfx_event_t e);
int gfx_event_release(gfx_event_t e);

/* Copy helpers for tests / e2e (host<->device through the manager's stream). */
int gfx_device_alloc(gfx_arena_t a, uint64_t bytes, void** out);
int gfx_device_free(gfx_arena_t a, void* p);
int gfx_memcpy_h2d(gfx_arena_t a, void* dst, const void* src, uint64_t bytes);
int gfx_memcpy_d2h(gfx_arena_t a, void* dst, const void* src, uint64_t bytes);
int gfx_synchronize(gfx_arena_t a);
/* Fill `n` fp32 values on device with the parameter stream (seed, tensor). */
int gfx_fill_params(gfx_arena_t a, float* dst, uint64_t n, uint64_t seed, uint32_t tensor, float scale);
uint64_t gfx_input_seed(int request_id);
/* Same stream generated on the host (no device needed). */
int gfx_host_fill_params(float* dst, uint64_t n, uint64_t seed, uint32_t tensor, float scale);
/* The model's request input for request_id, generated on the host (fp32 or bf16 bits). */
int gfx_host_fill_input(int model_idx, int request_id, void* dst, uint64_t bytes);

/* ---------------------------------------------------------------- replay */
/* Trace replay: the control plane (scheduler + cluster state, bit-exact with
 * the reference) drives one GPU manager per device; every dispatch becomes
 * evict -> (H2D | NVLink P2P) -> batched inference in decision order. */
typedef struct {
    const char* catalog_csv;
    const char* trace_csv;       /* NULL -> synthetic trace of cfg */
    gfx_sim_config cfg;
    int32_t n_devices;           /* devices backing cfg.gpu_count GPUs (1 or cfg.gpu_count) */
    int32_t first_device;
    int32_t only_gpu;            /* >= 0: execute only this GPU's decisions (one rank per GPU) */
    int32_t use_p2p;             /* false misses fetch from the peer holder over NVLink */
    int32_t host_io;             /* 1: inputs from pinned host, outputs back to host (e2e) */
    int32_t record_kernels;      /* CUDA-event timing of every inference (its L+1 kernels, PDL-chained) */
    int32_t record_requests;     /* per-request service-time events */
    int32_t keep_outputs;        /* keep every request's output (parity checks) */
    const void* host_inputs;     /* host_io: [n_requests][in_bytes] pinned, else NULL */
    void* host_outputs;          /* host_io: [n_requests][out_bytes] or NULL */
} gfx_replay_args;

typedef struct {
    int64_t n_requests;
    int64_t n_decisions;
    int64_t hits, misses, false_misses, local_enqueues, evictions;
    int64_t loads_h2d, loads_p2p;
    int64_t kernel_launches;
    uint64_t decision_digest;
    uint64_t h2d_bytes;          /* model weight bytes host->device */
    uint64_t p2p_bytes;
    uint64_t io_h2d_bytes;       /* request inputs (host_io) */
    uint64_t io_d2h_bytes;       /* request outputs (host_io) */
    double device_ms;            /* CUDA-event time of the whole replay (max over devices) */
    double host_ms;              /* wall time of the call */
    double sched_ms;             /* host time spent in the control plane */
    double kernel_ms;            /* sum over inferences of their kernel-chain event time (record_kernels) */
    double h2d_ms;               /* sum of model-load event times */
    double service_p50_ms, service_p99_ms; /* per-request device service time (record_requests) */
    double sim_p50_s, sim_p99_s, sim_avg_latency_s; /* virtual-time latency from the schedule */
    double mlp_flops;            /* algorithmic flops of all inferences */
    double mlp_weight_bytes;     /* algorithmic weight+activation bytes of all inferences */
    double p2p_ms;               /* sum of peer-fetch (NVLink) event times */
} gfx_replay_result;

/* Reusable replay context: managers, device buffers and timing events are
 * created once; every gfx_replay_run() replays the whole trace from an empty
 * cache (one bench step). */
typedef struct gfx_replay_s* gfx_replay_t;
int gfx_replay_create(const gfx_replay_args* args, gfx_replay_t* out);
int gfx_replay_run(gfx_replay_t r, gfx_replay_result* out);
/* Extension (no reference counterpart): live closed-loop serving of
 * the same trace. Arrivals are compressed to arrival / time_scale and released
 * in real time; each GPU's completion is observed on the device (an event after
 * its inference) and triggers the scheduler, so the schedule follows the
 * device, not the catalog's predicted times. sim_p50_s / sim_p99_s /
 * sim_avg_latency_s then hold REAL request latencies (seconds, arrival to
 * observed completion) and decision_digest is not reproducible. ema_alpha > 0:
 * each model's planned load/infer times follow the event-measured device
 * durations (exponential moving average; 0 keeps the catalog's). Needs every
 * GPU in this process (only_gpu < 0). */
int gfx_replay_run_live(gfx_replay_t r, double time_scale, double ema_alpha, gfx_replay_result* out);
/* Per-request outputs of the last run (keep_outputs): [n_requests][out_bytes]. */
int gfx_replay_outputs(gfx_replay_t r, void* host, uint64_t bytes);
/* Per-request model row and device service time (ms) of the last run. */
int gfx_replay_requests(gfx_replay_t r, int32_t* model_idx, double* service_ms, int64_t n);
/* One process per GPU (only_gpu >= 0, use_p2p): NVLink peer fetch between
 * processes. Each rank exports its arena and flag words as a CUDA IPC blob,
 * the ranks exchange blobs (e.g. an all-gather over torch.distributed), and
 * every rank imports all gpu_count blobs (index = GPU id) before the first
 * run. Ordering is device-side (cuStreamWaitValue32 / WriteValue32 on the
 * flag words); page tables of peer arenas are derived from the shared
 * deterministic schedule. Replaces nothing in the reference (its loads are
 * constants, proj/src/cluster.cpp:163-167). */
uint64_t gfx_replay_ipc_blob_bytes(void);
int gfx_replay_ipc_export(gfx_replay_t r, void* blob, uint64_t bytes);
int gfx_replay_ipc_import(gfx_replay_t r, const void* blobs, int32_t n);
int gfx_replay_destroy(gfx_replay_t r);
/* create + run + destroy */
int gfx_replay(const gfx_replay_args* args, gfx_replay_result* out);

/* ------------------------------------------------------------ cluster (N1) */
/* One GPU Manager daemon process per GPU (gfx_managerd: the paper's GPU Manager,
 * PAPER.md:288-303, owning that GPU's pre-allocated HBM arena, copy/compute
 * streams and pinned model store), fed by the global cache manager — the
 * reference control plane (scheduler + ClusterState,
 * proj/include/gpufaas/cluster.hpp:88-140) in the calling process — over one
 * POSIX shared-memory segment with a command ring and a completion ring per GPU.
 * gfx_cluster_run replays the deterministic schedule (run_stream, bit-exact
 * with the reference); gfx_cluster_run_live serves the trace in real time with
 * device-observed completions (run_live) — with one process per GPU. False
 * misses fetch from the holder daemon's arena over NVLink (CUDA IPC, device-side
 * ordering by stream memory operations on IPC-mapped flag words). Each daemon
 * builds request i's input on the device from its parameter stream
 * (gfx_input_seed) and keeps every output for gfx_cluster_output. */
typedef struct gfx_cluster_s* gfx_cluster_t;
typedef struct {
    const char* catalog_csv;
    const char* trace_csv;         /* NULL -> synthetic trace of cfg */
    gfx_sim_config cfg;            /* gpu_count <= 8 */
    const gfx_model_desc* models;  /* catalog row i = models[i] (checked by seed), at most 64 */
    int32_t n_models;
    int32_t use_p2p;               /* false misses fetch from the holder daemon (NVLink / CUDA IPC) */
    const int32_t* devices;        /* CUDA device of each GPU (NULL: device 0 for all = emulated peers) */
    int32_t spawn;                 /* 1: start gfx_managerd processes (next to the library); 0: they attach themselves */
    int32_t pad_;
    const char* shm_name;          /* NULL: a unique name (spawn = 1); spawn = 0 needs the name the daemons use */
} gfx_cluster_args;
const char* gfx_cluster_last_error(void);
int gfx_cluster_create(const gfx_cluster_args* args, gfx_cluster_t* out);
int gfx_cluster_run(gfx_cluster_t c, gfx_replay_result* out);
int gfx_cluster_run_live(gfx_cluster_t c, double time_scale, double ema_alpha, gfx_replay_result* out);
/* Output of request_id in the last run (fetched from the daemon that served it). */
int gfx_cluster_output(gfx_cluster_t c, int32_t request_id, void* host, uint64_t bytes);
int gfx_cluster_request_gpu(gfx_cluster_t c, int32_t request_id, int32_t* gpu);
int gfx_cluster_destroy(gfx_cluster_t c); /* stops the daemons */
/* The daemon loop: attach to the segment as GPU gpu_index, serve until stopped.
 * Returns 0 when stopped, nonzero on failure (the message is in the segment). */
int gfx_managerd_serve(const char* shm_name, int32_t gpu_index);
/* Test: a forked producer pushes n commands through a shared-memory command
 * ring; the caller pops and checks them in order (no device needed). */
int gfx_cluster_ring_selftest(int64_t n);

#ifdef __cplusplus
}
#endif
#endif /* GPUFAAS_B200_H */
