#pragma once
// Per-B200 GPU Manager (the paper's GPU Manager, whose
// cache bookkeeping the reference models in proj/src/cluster.cpp): owns a
// pre-allocated HBM arena of 2 MiB pages, a copy stream for model loads
// (pinned-host H2D or NVLink peer fetch) and a compute stream for batched
// inference, and executes the cache operations the control plane decides.
//
// Arena layout: capacity / 2 MiB pages in one cudaMalloc. A model occupies
// ceil(bytes / 2 MiB) pages anywhere in the arena (page table passed by value
// to every kernel), so the reference's sum-of-sizes capacity model
// (proj/src/cluster.cpp:107,133-147) is exact: any model set whose page
// counts fit the budget fits physically — no fragmentation, no compaction.
#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <mutex>
#include <set>
#include <vector>

#include "common.cuh"
#include "gpufaas_b200.h"
#include "bert.cuh"
#include "mlp.cuh"

namespace gfx {

// One model of the pinned host model store.
struct ModelBlob {
    gfx_model_desc desc{};
    uint64_t bytes = 0;
    uint32_t pages = 0;
    std::vector<uint64_t> w_off, b_off;  // per layer, offsets in the blob
    float* host = nullptr;               // pinned (cudaHostAlloc)
    double flops = 0;                    // per inference
    double alg_bytes = 0;                // per inference: weights + biases + in/out activations
    uint64_t in_bytes = 0, out_bytes = 0;  // one request's input / output tensors
    BertLayout bert;                     // GFX_MODEL_BERT
    ~ModelBlob();
};

class ModelStore {
public:
    static ModelStore& get();
    void add(int idx, const gfx_model_desc& desc);
    const ModelBlob& at(int idx) const;
    bool has(int idx) const;
    void clear();
    int max_dim() const;

private:
    mutable std::mutex mu_;
    std::vector<std::unique_ptr<ModelBlob>> blobs_;
};

// Arena pages a model occupies (its blob layout, without building the blob).
uint32_t model_pages(const gfx_model_desc& desc);

// Blob layout of an MLP: per layer the weight tiles (16 KB,
// 16 KB-aligned, N padded to 128 rows) then b [N] fp32 (256 B-aligned).
void mlp_layout(const gfx_model_desc& d, std::vector<uint64_t>& w_off, std::vector<uint64_t>& b_off,
                uint64_t& bytes);

struct KernelTimer {  // optional per-launch CUDA-event timing
    std::vector<cudaEvent_t> ev;
    size_t used = 0;
    cudaEvent_t next();
};

// Declares that another process also runs GPU managers on device `dev` (two
// daemons / replay ranks on one GPU in tests and emulation): K1 then keeps the
// cooperative launch instead of the PDL chain (see GpuManager::infer).
void mark_device_shared(int dev);

class GpuManager {
public:
    GpuManager(int device, uint64_t capacity_bytes, int manager_id);
    ~GpuManager();
    GpuManager(const GpuManager&) = delete;
    GpuManager& operator=(const GpuManager&) = delete;

    int device() const { return device_; }
    uint32_t total_pages() const { return npages_; }
    uint32_t free_pages() const { return static_cast<uint32_t>(free_.size()); }
    bool resident(int model) const;

    // Cache operations (asynchronous; host bookkeeping is immediate).
    void evict(int model);
    // Returns bytes copied. src == nullptr -> pinned host store.
    uint64_t load(int model, GpuManager* src);
    // BERT only: lengths (HOST, [batch] int32 in 1..seq) = padding mask per sequence.
    void infer(int model, const void* in, void* out, void* debug_hidden = nullptr, const int32_t* lengths = nullptr);
    void reset();  // synchronise and drop every resident model
    // Test hook: one BERT GEMM (bert_gemm_op) of a resident model on the compute stream.
    void bert_gemm(int model, int layer, int op, const void* x, const void* resid, void* y, int tokens);

    // Cross-process peers (one process per GPU): fetch a model from another
    // rank's arena mapped into this process by CUDA IPC, `src_pages` being that
    // arena's page table for the model; the copy stream first waits until the
    // 32-bit word `wait_addr` >= `wait_value` (the holder's load is done).
    uint64_t load_remote(int model, const char* src_arena, const std::vector<uint32_t>& src_pages,
                         const uint32_t* wait_addr, uint32_t wait_value);
    // Stream memory operations on the copy stream (device-side cross-process ordering).
    void copy_wait_geq(const uint32_t* addr, uint32_t value);
    void copy_write(uint32_t* addr, uint32_t value);

    cudaStream_t compute_stream() const { return compute_; }
    cudaStream_t copy_stream() const { return copy_; }
    cudaEvent_t loaded_event(int model) const;
    void add_reader(int model, cudaEvent_t e);  // peer fetch in flight from our pages
    const std::vector<uint32_t>& pages_of(int model) const;
    char* arena() const { return arena_; }
    void activate() const;  // cudaSetDevice
    void set_gemm_pair(bool on) { bert_ws_.gemm_pair = on; }
    void set_bert_flow(bool on) { bert_ws_.flow = on; }

    // Instrumentation (all optional).
    KernelTimer* layer_timer = nullptr;   // records around every inference
    KernelTimer* load_timer = nullptr;    // records around every pinned-host model load
    KernelTimer* p2p_timer = nullptr;     // records around every peer (NVLink) fetch
    int64_t kernel_launches = 0;

private:
    struct Slot {
        bool live = false;
        std::vector<uint32_t> pages;
        cudaEvent_t loaded = nullptr;       // copy stream, after the load
        cudaEvent_t last_use = nullptr;     // compute stream, after the last inference
        std::vector<cudaEvent_t> readers;   // peer fetches out of our pages
    };
    Slot& slot(int model);
    void build_page_table(const Slot& s, PageTable& pt) const;
    Slot& allocate(int model, const ModelBlob& blob);

    int device_;
    int id_;
    uint32_t npages_ = 0;
    char* arena_ = nullptr;
    std::set<uint32_t> free_;  // lowest-first allocation keeps page runs contiguous
    std::vector<Slot> slots_;
    cudaStream_t compute_ = nullptr, copy_ = nullptr;
    int sm_count_ = 148;
    // inference workspaces
    BertWorkspace bert_ws_;
    int* bert_lengths_ = nullptr;  // device copy of a masked request's sequence lengths
    int bert_lengths_cap_ = 0;
    // K1 forward workspace: layer outputs, two banks by launch parity
    unsigned long long* fwd_act_ = nullptr;
    unsigned fwd_epoch_ = 0;      // launches of the forward kernel on this manager's workspace
    unsigned* fwd_claim_ = nullptr;  // K1 layer-0 claim counters, one per launch mod 4 (zero when due)
    uint32_t act_dirty_[2] = {0, 0};  // words of each act bank written and not yet cleared
};

}  // namespace gfx
