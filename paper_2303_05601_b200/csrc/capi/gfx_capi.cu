// C-ABI of the data plane and the trace replay (declared in include/gpufaas_b200.h).
//
// The replay is the product path end to end: the bit-exact control plane
// (gpufaas::run_stream with the Scheduler) emits decisions; an
// ExecutionListener turns each dispatch into device work on the GPU manager
// of the chosen GPU — evict victims, load the model (pinned-host H2D, or
// NVLink peer fetch when another GPU holds it), run the batched inference —
// in decision order per GPU. Host enqueue runs ahead of the device; streams
// and events carry every dependency, so the host never blocks on the GPU
// until the end-of-replay synchronisation.
#include <cuda_runtime.h>

#include <algorithm>
#include <deque>
#include <cstring>
#include <set>
#include <chrono>
#include <cmath>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "capi_common.hpp"
#include "gpufaas/engine.hpp"
#include "gpufaas_b200.h"
#include "manager.cuh"

using gfx::GpuManager;
using gfx::KernelTimer;
using gfx::ModelStore;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    return gpufaas::capi::guarded_call(g_err, std::forward<F>(f));
}

double elapsed_ms(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0;
    GFX_CUDA(cudaEventElapsedTime(&ms, a, b));
    return ms;
}

using gpufaas::capi::percentile;

}  // namespace

struct gfx_arena_s {
    std::unique_ptr<GpuManager> mgr;
};
struct gfx_event_s {
    cudaEvent_t ev = nullptr;
    int device = 0;
};

// ---------------------------------------------------------------- replay

struct gfx_replay_s : gpufaas::ExecutionListener {
    gfx_replay_args args{};
    std::string catalog_csv, trace_csv;
    gpufaas::Catalog catalog;
    std::vector<gpufaas::Request> requests;
    std::vector<std::unique_ptr<GpuManager>> mgrs;  // index = GPU id (nullptr if not executed here)
    std::vector<int> dev_of;
    // device buffers per device
    struct DevBufs {
        char* inputs = nullptr;    // [n][in_bytes]
        char* outputs = nullptr;   // [n][out_bytes] (keep/host_io) or [2][out_bytes] ring
        cudaStream_t io_in = nullptr, io_out = nullptr;
        cudaEvent_t start = nullptr, stop = nullptr;
    };
    std::vector<DevBufs> bufs;  // per GPU id
    size_t in_bytes = 0, out_bytes = 0;
    int family = 0;
    bool full_outputs = false;
    // timing: events per GPU (an event belongs to the device current at its creation)
    struct Timers {
        KernelTimer layer, load, p2p, req;
    };
    std::vector<Timers> timers;  // per GPU id
    std::vector<cudaEvent_t> req_start, req_end;
    std::vector<int> req_gpu;
    // ---- cross-process peers (one process per GPU, only_gpu mode) ----
    // Another rank's GPU: its arena and flag words mapped by CUDA IPC, plus a
    // host shadow of its page allocator. The shadow is exact because every
    // rank runs the same bit-exact control plane and a manager allocates the
    // lowest free pages (GpuManager::allocate), so the page table of any model
    // on any GPU is known here without asking that rank.
    struct RemoteArena {
        char* arena = nullptr;
        uint32_t* flags = nullptr;
        uint32_t npages = 0;
        std::set<uint32_t> free;
        std::vector<std::vector<uint32_t>> pages;
        void reset() {
            free.clear();
            for (uint32_t p = 0; p < npages; ++p) free.insert(p);
            for (auto& v : pages) v.clear();
        }
        void evict(int m) {
            for (uint32_t p : pages[static_cast<size_t>(m)]) free.insert(p);
            pages[static_cast<size_t>(m)].clear();
        }
        void load(int m, uint32_t n) {
            auto& v = pages[static_cast<size_t>(m)];
            v.clear();
            for (uint32_t i = 0; i < n; ++i) {
                v.push_back(*free.begin());
                free.erase(free.begin());
            }
        }
    };
    std::vector<RemoteArena> remotes;  // index = GPU id (unused for only_gpu)
    // This rank's flag words (device, IPC-exported), written by peers' copy
    // streams: loaded[s][m] = loads of model m completed on GPU s (so far, all
    // runs), read_done[m][r] = fetches of our model m completed by GPU r.
    uint32_t* flags = nullptr;
    bool ipc = false;
    size_t M = 0;
    std::vector<uint32_t> load_cnt;   // [G][M] loads decided so far (all runs)
    std::vector<uint32_t> fetch_cnt;  // [G src][M][G reader] peer fetches decided so far
    size_t fl_loaded(int g, int m) const { return static_cast<size_t>(g) * M + static_cast<size_t>(m); }
    size_t fl_read(int m, int r) const {
        return static_cast<size_t>(gpu_count()) * M + static_cast<size_t>(m) * gpu_count() + static_cast<size_t>(r);
    }
    uint32_t& fetches(int src, int m, int r) {
        return fetch_cnt[(static_cast<size_t>(src) * M + static_cast<size_t>(m)) * gpu_count() + static_cast<size_t>(r)];
    }
    bool remote_fetch(int gpu, int source) const {
        return ipc && args.use_p2p && source >= 0 && source != gpu;
    }
    // Host bookkeeping of every GPU's dispatch (all ranks see the whole stream).
    void track(int gpu, int model, bool hit, const std::vector<int>& evicted, int source) {
        if (hit) return;
        const bool mine = gpu == args.only_gpu;
        for (int v : evicted)
            if (!mine) remotes[static_cast<size_t>(gpu)].evict(v);
        if (remote_fetch(gpu, source)) ++fetches(source, model, gpu);
        if (!mine) remotes[static_cast<size_t>(gpu)].load(model, ModelStore::get().at(model).pages);
        ++load_cnt[fl_loaded(gpu, model)];
    }
    // Before our pages of model v are reused: every peer fetch of v decided so far has completed.
    void wait_peer_reads(GpuManager& m, int v) {
        for (int r = 0; r < gpu_count(); ++r) {
            const uint32_t c = fetches(args.only_gpu, v, r);
            if (c) m.copy_wait_geq(flags + fl_read(v, r), c);
        }
    }

    // counters of the current run
    gfx_replay_result res{};
    std::vector<cudaEvent_t> pending_in;  // per GPU: event of the last input copy

    int gpu_count() const { return args.cfg.gpu_count; }

    void setup() {
        std::istringstream cin_(catalog_csv);
        catalog = gpufaas::parse_catalog_csv(cin_, "catalog");
        requests = gpufaas::capi::make_requests(args.cfg, catalog, args.trace_csv ? trace_csv.c_str() : nullptr);
        const int G = gpu_count();
        if (G <= 0) throw std::invalid_argument("gpu_count must be positive");
        if (args.n_devices != 1 && args.n_devices != G)
            throw std::invalid_argument("n_devices must be 1 or cfg.gpu_count");
        // Every catalog model must be registered and its charge must cover its pages.
        for (size_t i = 0; i < catalog.size(); ++i) {
            const gfx::ModelBlob& b = ModelStore::get().at(static_cast<int>(i));
            // Catalog row i must be the model registered at index i (its parameter
            // stream is seeded by the FNV-1a hash of the model id).
            uint64_t h = 14695981039346656037ULL;
            for (unsigned char c : catalog.profiles()[i].model_id) {
                h ^= c;
                h *= 1099511628211ULL;
            }
            if (b.desc.seed != h)
                throw std::invalid_argument("model registered at index " + std::to_string(i) + " is not catalog row '" +
                                            catalog.profiles()[i].model_id + "'");
            const double need = 2.0 * b.pages;
            if (catalog.profiles()[i].occupation_mb < need)
                throw std::invalid_argument("catalog occupation_mb of '" + catalog.profiles()[i].model_id +
                                            "' is below its " + std::to_string(b.pages) + " arena pages");
            if (i == 0) {
                in_bytes = b.in_bytes;
                out_bytes = b.out_bytes;
                family = b.desc.family;
            } else if (b.in_bytes != in_bytes || b.out_bytes != out_bytes || b.desc.family != family) {
                throw std::invalid_argument("all models of a replay must share family and request tensor shapes");
            }
        }
        full_outputs = args.keep_outputs || args.host_io;
        const uint64_t pages = static_cast<uint64_t>(args.cfg.capacity_mb / 2.0);
        const uint64_t cap_bytes = pages * gfx::kPageBytes;
        mgrs.resize(static_cast<size_t>(G));
        bufs.resize(static_cast<size_t>(G));
        dev_of.resize(static_cast<size_t>(G));
        pending_in.assign(static_cast<size_t>(G), nullptr);
        timers.resize(static_cast<size_t>(G));
        const size_t n = requests.size();
        for (int g = 0; g < G; ++g) {
            dev_of[g] = args.first_device + (args.n_devices == 1 ? 0 : g);
            if (args.only_gpu >= 0 && g != args.only_gpu) continue;
            mgrs[g] = std::make_unique<GpuManager>(dev_of[g], cap_bytes, g);
            mgrs[g]->layer_timer = args.record_kernels ? &timers[g].layer : nullptr;
            mgrs[g]->load_timer = &timers[g].load;
            mgrs[g]->p2p_timer = &timers[g].p2p;
            DevBufs& b = bufs[g];
            GFX_CUDA(cudaSetDevice(dev_of[g]));
            // Inputs: every request this GPU might serve (ids are global).
            GFX_CUDA(cudaMalloc(&b.inputs, in_bytes * std::max<size_t>(n, 1)));
            GFX_CUDA(cudaMalloc(&b.outputs, out_bytes * (full_outputs ? std::max<size_t>(n, 1) : 2)));
            GFX_CUDA(cudaStreamCreateWithFlags(&b.io_in, cudaStreamNonBlocking));
            GFX_CUDA(cudaStreamCreateWithFlags(&b.io_out, cudaStreamNonBlocking));
            GFX_CUDA(cudaEventCreate(&b.start));
            GFX_CUDA(cudaEventCreate(&b.stop));
            if (!args.host_io) {
                // HBM-resident inputs, generated once outside the timed region.
                if (family == GFX_MODEL_BERT)
                    gfx::launch_fill_bf16(reinterpret_cast<__nv_bfloat16*>(b.inputs), in_bytes / 2, gfx_input_seed(0),
                                          0xFFFFFFFFu, 1.0f, mgrs[g]->compute_stream(), n);
                else
                    gfx::launch_fill_params(reinterpret_cast<float*>(b.inputs), in_bytes / 4, gfx_input_seed(0),
                                            0xFFFFFFFFu, 1.0f, mgrs[g]->compute_stream(), n);
            }
            GFX_CUDA(cudaDeviceSynchronize());
        }
        if (args.use_p2p && args.n_devices > 1) {
            for (int a = 0; a < G; ++a)
                for (int b2 = 0; b2 < G; ++b2) {
                    if (a == b2 || !mgrs[a] || !mgrs[b2]) continue;
                    int ok = 0;
                    GFX_CUDA(cudaDeviceCanAccessPeer(&ok, dev_of[a], dev_of[b2]));
                    if (ok) {
                        GFX_CUDA(cudaSetDevice(dev_of[a]));
                        cudaError_t e = cudaDeviceEnablePeerAccess(dev_of[b2], 0);
                        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) GFX_CUDA(e);
                        cudaGetLastError();
                    }
                }
        }
        req_start.assign(n, nullptr);
        req_end.assign(n, nullptr);
        req_gpu.assign(n, -1);
        M = catalog.size();
        if (args.only_gpu >= 0) {
            GFX_CUDA(cudaSetDevice(dev_of[static_cast<size_t>(args.only_gpu)]));
            const size_t words = 2 * static_cast<size_t>(G) * M;
            GFX_CUDA(cudaMalloc(&flags, words * 4));
            GFX_CUDA(cudaMemset(flags, 0, words * 4));
            GFX_CUDA(cudaDeviceSynchronize());
            load_cnt.assign(static_cast<size_t>(G) * M, 0);
            fetch_cnt.assign(static_cast<size_t>(G) * M * static_cast<size_t>(G), 0);
        }
    }

    struct IpcBlob {
        cudaIpcMemHandle_t arena;
        cudaIpcMemHandle_t flags;
        uint64_t arena_pages;
        int32_t gpu;
        int32_t models;
        char uuid[16];  // the exporting process's device (ranks sharing one B200 -> cooperative K1)
    };

    void ipc_export(void* out, uint64_t bytes) {
        if (args.only_gpu < 0) throw std::invalid_argument("ipc export needs only_gpu (one process per GPU)");
        if (bytes < sizeof(IpcBlob)) throw std::invalid_argument("ipc blob buffer too small");
        GpuManager& m = *mgrs[static_cast<size_t>(args.only_gpu)];
        m.activate();
        IpcBlob b{};
        GFX_CUDA(cudaIpcGetMemHandle(&b.arena, m.arena()));
        GFX_CUDA(cudaIpcGetMemHandle(&b.flags, flags));
        b.arena_pages = m.total_pages();
        b.gpu = args.only_gpu;
        b.models = static_cast<int32_t>(M);
        cudaDeviceProp prop{};
        GFX_CUDA(cudaGetDeviceProperties(&prop, dev_of[static_cast<size_t>(args.only_gpu)]));
        std::memcpy(b.uuid, &prop.uuid, sizeof b.uuid);
        std::memcpy(out, &b, sizeof b);
    }

    void ipc_import(const void* blobs, int n) {
        if (args.only_gpu < 0) throw std::invalid_argument("ipc import needs only_gpu (one process per GPU)");
        if (n != gpu_count()) throw std::invalid_argument("ipc import needs one blob per GPU");
        GFX_CUDA(cudaSetDevice(dev_of[static_cast<size_t>(args.only_gpu)]));
        remotes.assign(static_cast<size_t>(n), RemoteArena{});
        const IpcBlob* b = static_cast<const IpcBlob*>(blobs);
        const int my = args.only_gpu;
        for (int g = 0; g < n; ++g)
            if (g != my && std::memcmp(b[g].uuid, b[my].uuid, sizeof b[g].uuid) == 0)
                gfx::mark_device_shared(dev_of[static_cast<size_t>(my)]);
        for (int g = 0; g < n; ++g) {
            if (b[g].gpu != g || static_cast<size_t>(b[g].models) != M)
                throw std::invalid_argument("ipc blob " + std::to_string(g) + " is not GPU " + std::to_string(g) +
                                            " of the same catalog");
            if (g == args.only_gpu) continue;
            RemoteArena& ra = remotes[static_cast<size_t>(g)];
            void* p = nullptr;
            GFX_CUDA(cudaIpcOpenMemHandle(&p, b[g].arena, cudaIpcMemLazyEnablePeerAccess));
            ra.arena = static_cast<char*>(p);
            GFX_CUDA(cudaIpcOpenMemHandle(&p, b[g].flags, cudaIpcMemLazyEnablePeerAccess));
            ra.flags = static_cast<uint32_t*>(p);
            ra.npages = static_cast<uint32_t>(b[g].arena_pages);
            ra.pages.assign(M, {});
            ra.reset();
        }
        ipc = true;
    }

    void on_begin_execution(int gpu, const gpufaas::Request& req, int model, bool hit,
                            const std::vector<int>& evicted, int source, gpufaas::SimTime, gpufaas::SimTime) override {
        if (ipc) track(gpu, model, hit, evicted, source);
        if (args.only_gpu >= 0 && gpu != args.only_gpu) return;
        GpuManager& m = *mgrs[static_cast<size_t>(gpu)];
        DevBufs& b = bufs[static_cast<size_t>(gpu)];
        const int rid = req.request_id;
        KernelTimer& rt = timers[static_cast<size_t>(gpu)].req;
        m.activate();
        cudaEvent_t e0 = nullptr;
        req_gpu[rid] = gpu;
        if (args.record_requests) {
            e0 = rt.next();
            req_start[rid] = e0;
        }
        LiveTask live_t{};
        LiveTask* lt = live_mode ? &live_t : nullptr;
        if (!hit) {
            if (e0) GFX_CUDA(cudaEventRecord(e0, m.copy_stream()));
            if (lt) {
                lt->ls = rt.next();
                GFX_CUDA(cudaEventRecord(lt->ls, m.copy_stream()));
            }
            for (int v : evicted) {
                if (ipc) wait_peer_reads(m, v);
                m.evict(v);
            }
            GpuManager* src = nullptr;
            if (args.use_p2p && source >= 0 && mgrs[static_cast<size_t>(source)] &&
                mgrs[static_cast<size_t>(source)]->resident(model))
                src = mgrs[static_cast<size_t>(source)].get();
            if (remote_fetch(gpu, source)) {
                // Another rank holds it: NVLink fetch out of its IPC-mapped
                // arena once its load counter shows the load complete, then
                // tell it our read is done (it waits on that before reusing
                // the pages).
                RemoteArena& ra = remotes[static_cast<size_t>(source)];
                const uint64_t bytes = m.load_remote(model, ra.arena, ra.pages[static_cast<size_t>(model)],
                                                     flags + fl_loaded(source, model),
                                                     load_cnt[fl_loaded(source, model)]);
                m.copy_write(ra.flags + fl_read(model, gpu), fetches(source, model, gpu));
                res.loads_p2p++;
                res.p2p_bytes += bytes;
            } else {
                const uint64_t bytes = m.load(model, src);
                if (src) {
                    res.loads_p2p++;
                    res.p2p_bytes += bytes;
                } else {
                    res.loads_h2d++;
                    res.h2d_bytes += bytes;
                }
            }
            if (ipc)  // our load of `model` is complete: publish the count to every peer
                for (int r = 0; r < gpu_count(); ++r)
                    if (r != gpu) m.copy_write(remotes[static_cast<size_t>(r)].flags + fl_loaded(gpu, model),
                                               load_cnt[fl_loaded(gpu, model)]);
            if (lt) {
                lt->le = rt.next();
                GFX_CUDA(cudaEventRecord(lt->le, m.copy_stream()));
            }
        } else if (e0) {
            GFX_CUDA(cudaEventRecord(e0, m.compute_stream()));
        }
        char* in = b.inputs + static_cast<size_t>(rid) * in_bytes;
        char* out = b.outputs + (full_outputs ? static_cast<size_t>(rid) : static_cast<size_t>(rid & 1)) * out_bytes;
        if (args.host_io) {
            // e2e: this request's input crosses PCIe inside the timed region.
            GFX_CUDA(cudaMemcpyAsync(in, static_cast<const char*>(args.host_inputs) + static_cast<size_t>(rid) * in_bytes,
                                     in_bytes, cudaMemcpyHostToDevice, b.io_in));
            cudaEvent_t ein = rt.next();
            GFX_CUDA(cudaEventRecord(ein, b.io_in));
            GFX_CUDA(cudaStreamWaitEvent(m.compute_stream(), ein, 0));
            res.io_h2d_bytes += in_bytes;
        }
        if (lt) {
            if (lt->le) GFX_CUDA(cudaStreamWaitEvent(m.compute_stream(), lt->le, 0));
            lt->is = rt.next();
            GFX_CUDA(cudaEventRecord(lt->is, m.compute_stream()));
        }
        m.infer(model, in, out);
        if (lt) {
            lt->ie = rt.next();
            GFX_CUDA(cudaEventRecord(lt->ie, m.compute_stream()));
        }
        const gfx::ModelBlob& blob = ModelStore::get().at(model);
        res.mlp_flops += blob.flops;
        res.mlp_weight_bytes += blob.alg_bytes;
        if (args.record_requests) {
            cudaEvent_t e1 = rt.next();
            GFX_CUDA(cudaEventRecord(e1, m.compute_stream()));
            req_end[rid] = e1;
        }
        if (args.host_io) {
            cudaEvent_t done = rt.next();
            GFX_CUDA(cudaEventRecord(done, m.compute_stream()));
            GFX_CUDA(cudaStreamWaitEvent(b.io_out, done, 0));
            GFX_CUDA(cudaMemcpyAsync(static_cast<char*>(args.host_outputs) + static_cast<size_t>(rid) * out_bytes, out,
                                     out_bytes, cudaMemcpyDeviceToHost, b.io_out));
            res.io_d2h_bytes += out_bytes;
        }
        if (live_mode) {
            // Live mode: the engine polls this to learn the request finished (output included).
            lt->done = rt.next();
            GFX_CUDA(cudaEventRecord(lt->done, args.host_io ? b.io_out : m.compute_stream()));
            live_q[static_cast<size_t>(gpu)].push_back(live_t);
        }
    }

    void on_complete(int, int, gpufaas::SimTime) override {}

    // Live closed-loop serving (gpufaas::run_live): completions are observed
    // on the device instead of predicted.
    // Per GPU, a FIFO of dispatched tasks (two deep with pipelined GPUs): load
    // (copy stream) and inference (compute stream) events for measured(), and
    // the completion event done() polls; the engine retires the front.
    struct LiveTask {
        cudaEvent_t ls = nullptr, le = nullptr, is = nullptr, ie = nullptr, done = nullptr;
    };
    struct LiveExec : gpufaas::LiveExecutor {
        gfx_replay_s* r = nullptr;
        bool done(int gpu) override {
            const auto& q = r->live_q[static_cast<size_t>(gpu)];
            if (q.empty()) return true;
            const cudaError_t st = cudaEventQuery(q.front().done);
            if (st == cudaErrorNotReady) return false;
            GFX_CUDA(st);
            return true;
        }
        void retire(int gpu) override {
            auto& q = r->live_q[static_cast<size_t>(gpu)];
            if (!q.empty()) q.pop_front();
        }
        bool measured(int gpu, gpufaas::SimTime* load_us, gpufaas::SimTime* infer_us) override {
            const auto& q = r->live_q[static_cast<size_t>(gpu)];
            if (q.empty()) return false;
            const LiveTask& t = q.front();
            if (!t.is) return false;
            *load_us = t.ls ? std::max<gpufaas::SimTime>(1, std::llround(elapsed_ms(t.ls, t.le) * 1e3)) : 0;
            *infer_us = std::max<gpufaas::SimTime>(1, std::llround(elapsed_ms(t.is, t.ie) * 1e3));
            return true;
        }
    };
    bool live_mode = false;
    double live_scale = 0.0, live_alpha = 0.0;
    std::vector<std::deque<LiveTask>> live_q;

    void run_live(double time_scale, double ema_alpha, gfx_replay_result* out) {
        if (args.only_gpu >= 0) throw std::invalid_argument("live mode runs every GPU in one process (only_gpu < 0)");
        if (!(time_scale > 0)) throw std::invalid_argument("live mode needs a positive time_scale");
        live_mode = true;
        live_scale = time_scale;
        live_alpha = ema_alpha;
        live_q.assign(static_cast<size_t>(gpu_count()), {});
        try {
            run(out);
        } catch (...) {
            live_mode = false;
            throw;
        }
        live_mode = false;
    }

    void run(gfx_replay_result* out) {
        res = gfx_replay_result{};
        for (Timers& t : timers) t.layer.used = t.load.used = t.p2p.used = t.req.used = 0;
        std::fill(req_start.begin(), req_start.end(), nullptr);
        std::fill(req_end.begin(), req_end.end(), nullptr);
        const int G = gpu_count();
        for (int g = 0; g < G; ++g) {
            if (!mgrs[g]) continue;
            if (ipc)  // peers may still be reading our pages from the previous run
                for (int v = 0; v < static_cast<int>(M); ++v) wait_peer_reads(*mgrs[g], v);
            mgrs[g]->reset();
            mgrs[g]->kernel_launches = 0;
        }
        for (RemoteArena& ra : remotes)
            if (ra.arena) ra.reset();
        const auto h0 = std::chrono::steady_clock::now();
        for (int g = 0; g < G; ++g) {
            if (!mgrs[g]) continue;
            GpuManager& m = *mgrs[g];
            m.activate();
            GFX_CUDA(cudaEventRecord(bufs[g].start, m.compute_stream()));
            for (cudaStream_t s : {m.copy_stream(), bufs[g].io_in, bufs[g].io_out})
                GFX_CUDA(cudaStreamWaitEvent(s, bufs[g].start, 0));
        }
        gpufaas::SimConfig cfg = gpufaas::capi::to_sim_config(args.cfg);
        const auto s0 = std::chrono::steady_clock::now();
        gpufaas::SimResult sim;
        if (live_mode) {
            LiveExec ex;
            ex.r = this;
            sim = gpufaas::run_live(cfg, catalog, requests, live_scale, this, ex, nullptr, live_alpha);
        } else {
            sim = gpufaas::run_stream(cfg, catalog, requests, nullptr, nullptr, this);
        }
        const auto s1 = std::chrono::steady_clock::now();
        for (int g = 0; g < G; ++g) {
            if (!mgrs[g]) continue;
            GpuManager& m = *mgrs[g];
            m.activate();
            for (cudaStream_t s : {m.copy_stream(), bufs[g].io_in, bufs[g].io_out}) {
                cudaEvent_t e = timers[static_cast<size_t>(g)].req.next();
                GFX_CUDA(cudaEventRecord(e, s));
                GFX_CUDA(cudaStreamWaitEvent(m.compute_stream(), e, 0));
            }
            GFX_CUDA(cudaEventRecord(bufs[g].stop, m.compute_stream()));
        }
        double dev_ms = 0;
        for (int g = 0; g < G; ++g) {
            if (!mgrs[g]) continue;
            GFX_CUDA(cudaSetDevice(dev_of[g]));
            GFX_CUDA(cudaEventSynchronize(bufs[g].stop));
            dev_ms = std::max(dev_ms, elapsed_ms(bufs[g].start, bufs[g].stop));
        }
        const auto h1 = std::chrono::steady_clock::now();

        res.n_requests = static_cast<int64_t>(sim.requests.size());
        res.n_decisions = static_cast<int64_t>(sim.decisions.size());
        res.hits = sim.report.hits;
        res.misses = sim.report.misses;
        res.false_misses = sim.report.false_misses;
        res.local_enqueues = sim.report.local_enqueues;
        res.evictions = sim.report.evictions;
        res.decision_digest = gpufaas::capi::decision_digest(sim.decisions);
        res.device_ms = dev_ms;
        res.host_ms = std::chrono::duration<double, std::milli>(h1 - h0).count();
        res.sched_ms = std::chrono::duration<double, std::milli>(s1 - s0).count();
        for (int g = 0; g < G; ++g)
            if (mgrs[g]) res.kernel_launches += mgrs[g]->kernel_launches;
        for (size_t g = 0; g < timers.size(); ++g) {
            if (!mgrs[g]) continue;
            GFX_CUDA(cudaSetDevice(dev_of[g]));
            const Timers& t = timers[g];
            for (size_t i = 0; i + 1 < t.layer.used; i += 2) res.kernel_ms += elapsed_ms(t.layer.ev[i], t.layer.ev[i + 1]);
            for (size_t i = 0; i + 1 < t.load.used; i += 2) res.h2d_ms += elapsed_ms(t.load.ev[i], t.load.ev[i + 1]);
            for (size_t i = 0; i + 1 < t.p2p.used; i += 2) res.p2p_ms += elapsed_ms(t.p2p.ev[i], t.p2p.ev[i + 1]);
        }
        if (args.record_requests) {
            std::vector<double> svc;
            for (size_t r = 0; r < req_start.size(); ++r)
                if (req_start[r] && req_end[r]) {
                    GFX_CUDA(cudaSetDevice(dev_of[static_cast<size_t>(req_gpu[r])]));
                    svc.push_back(elapsed_ms(req_start[r], req_end[r]));
                }
            res.service_p50_ms = percentile(svc, 50);
            res.service_p99_ms = percentile(svc, 99);
            service_ms = std::move(svc);
        }
        res.sim_p50_s = gpufaas::latency_percentile_s(sim.requests, 50);
        res.sim_p99_s = gpufaas::latency_percentile_s(sim.requests, 99);
        res.sim_avg_latency_s = sim.report.avg_latency_s.value_or(0.0);
        last_models.clear();
        for (const gpufaas::Request& r : sim.requests) last_models.push_back(catalog.index_of(r.model_id));
        *out = res;
    }

    std::vector<double> service_ms;
    std::vector<int32_t> last_models;

    ~gfx_replay_s() override {
        for (size_t g = 0; g < bufs.size(); ++g) {
            if (!mgrs[g]) continue;
            cudaSetDevice(dev_of[g]);
            cudaDeviceSynchronize();
            cudaFree(bufs[g].inputs);
            cudaFree(bufs[g].outputs);
            cudaStreamDestroy(bufs[g].io_in);
            cudaStreamDestroy(bufs[g].io_out);
            cudaEventDestroy(bufs[g].start);
            cudaEventDestroy(bufs[g].stop);
        }
        for (Timers& tm : timers)
            for (KernelTimer* t : {&tm.layer, &tm.load, &tm.p2p, &tm.req})
                for (cudaEvent_t e : t->ev) cudaEventDestroy(e);
        for (RemoteArena& ra : remotes) {
            if (ra.arena) cudaIpcCloseMemHandle(ra.arena);
            if (ra.flags) cudaIpcCloseMemHandle(ra.flags);
        }
        if (flags) cudaFree(flags);
    }
};

extern "C" {

const char* gfx_last_error(void) { return g_err.c_str(); }

int gfx_device_count(int* out) {
    return guarded([&] {
        int n = 0;
        GFX_CUDA(cudaGetDeviceCount(&n));
        *out = n;
    });
}

int gfx_device_init(int dev, int enable_peers) {
    return guarded([&] {
        GFX_CUDA(cudaSetDevice(dev));
        GFX_CUDA(cudaFree(nullptr));
        if (enable_peers) {
            int n = 0;
            GFX_CUDA(cudaGetDeviceCount(&n));
            for (int p = 0; p < n; ++p) {
                if (p == dev) continue;
                int ok = 0;
                GFX_CUDA(cudaDeviceCanAccessPeer(&ok, dev, p));
                if (!ok) continue;
                cudaError_t e = cudaDeviceEnablePeerAccess(p, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) GFX_CUDA(e);
                cudaGetLastError();
            }
        }
    });
}

int gfx_model_register(int model_idx, const gfx_model_desc* desc) {
    return guarded([&] { ModelStore::get().add(model_idx, *desc); });
}
int gfx_model_bytes(int model_idx, uint64_t* bytes) {
    return guarded([&] { *bytes = ModelStore::get().at(model_idx).bytes; });
}
int gfx_model_pages(int model_idx, int32_t* pages) {
    return guarded([&] { *pages = static_cast<int32_t>(ModelStore::get().at(model_idx).pages); });
}
int gfx_model_io_bytes(int model_idx, uint64_t* in_bytes, uint64_t* out_bytes) {
    return guarded([&] {
        const gfx::ModelBlob& b = ModelStore::get().at(model_idx);
        *in_bytes = b.in_bytes;
        *out_bytes = b.out_bytes;
    });
}
int gfx_host_fill_input(int model_idx, int request_id, void* dst, uint64_t bytes) {
    return guarded([&] {
        const gfx::ModelBlob& b = ModelStore::get().at(model_idx);
        if (bytes < b.in_bytes) throw std::invalid_argument("input buffer too small");
        const uint64_t st = gfx::param_stream(gfx_input_seed(request_id), 0xFFFFFFFFu);
        const float sc = gfx::param_scale(1.0f);
        if (b.desc.family == GFX_MODEL_BERT) {
            uint16_t* o = static_cast<uint16_t*>(dst);
            for (uint64_t i = 0; i < b.in_bytes / 2; ++i) o[i] = gfx::bf16_bits(gfx::param_at(st, i, sc));
        } else {
            float* o = static_cast<float*>(dst);
            for (uint64_t i = 0; i < b.in_bytes / 4; ++i) o[i] = gfx::param_at(st, i, sc);
        }
    });
}
int gfx_models_clear(void) {
    return guarded([&] { ModelStore::get().clear(); });
}

int gfx_arena_create(int dev, uint64_t capacity_bytes, gfx_arena_t* out) {
    return guarded([&] {
        auto a = std::make_unique<gfx_arena_s>();
        a->mgr = std::make_unique<GpuManager>(dev, capacity_bytes, 0);
        *out = a.release();
    });
}
int gfx_arena_destroy(gfx_arena_t a) {
    return guarded([&] { delete a; });
}
int gfx_arena_reset(gfx_arena_t a) {
    return guarded([&] { a->mgr->reset(); });
}
int gfx_arena_free_pages(gfx_arena_t a, int32_t* out) {
    return guarded([&] { *out = static_cast<int32_t>(a->mgr->free_pages()); });
}
int gfx_arena_set_option(gfx_arena_t a, int32_t option, int32_t value) {
    return guarded([&] {
        if ((option != GFX_OPT_GEMM_PAIR && option != GFX_OPT_BERT_FLOW) || (value != 0 && value != 1))
            throw std::invalid_argument("unknown arena option or value");
        if (option == GFX_OPT_GEMM_PAIR)
            a->mgr->set_gemm_pair(value != 0);
        else
            a->mgr->set_bert_flow(value != 0);
    });
}
int gfx_arena_resident(gfx_arena_t a, int model_idx, int32_t* out) {
    return guarded([&] { *out = a->mgr->resident(model_idx) ? 1 : 0; });
}

static void make_event(GpuManager& m, cudaStream_t s, gfx_event_t* done) {
    if (!done) return;
    auto e = std::make_unique<gfx_event_s>();
    e->device = m.device();
    GFX_CUDA(cudaEventCreateWithFlags(&e->ev, cudaEventDisableTiming));
    GFX_CUDA(cudaEventRecord(e->ev, s));
    *done = e.release();
}

int gfx_load_h2d(gfx_arena_t a, int model_idx, gfx_event_t* done) {
    return guarded([&] {
        a->mgr->load(model_idx, nullptr);
        make_event(*a->mgr, a->mgr->copy_stream(), done);
    });
}
int gfx_fetch_p2p(gfx_arena_t dst, gfx_arena_t src, int model_idx, gfx_event_t* done) {
    return guarded([&] {
        if (!src->mgr->resident(model_idx)) throw std::invalid_argument("peer does not hold the model");
        dst->mgr->load(model_idx, src->mgr.get());
        make_event(*dst->mgr, dst->mgr->copy_stream(), done);
    });
}
int gfx_evict(gfx_arena_t a, int model_idx) {
    return guarded([&] { a->mgr->evict(model_idx); });
}
int gfx_infer(gfx_arena_t a, int model_idx, const void* in, void* out, int batch, gfx_event_t* done) {
    return guarded([&] {
        if (batch != ModelStore::get().at(model_idx).desc.batch)
            throw std::invalid_argument("batch does not match the registered model");
        a->mgr->infer(model_idx, in, out);
        make_event(*a->mgr, a->mgr->compute_stream(), done);
    });
}

int gfx_infer_sequence(gfx_arena_t a, const int32_t* models, int n, const void* in, uint64_t in_stride, void* out,
                       uint64_t out_stride, double* ms) {
    return guarded([&] {
        if (n <= 0) throw std::invalid_argument("empty inference sequence");
        GpuManager& m = *a->mgr;
        m.activate();
        cudaEvent_t e0, e1;
        GFX_CUDA(cudaEventCreate(&e0));
        GFX_CUDA(cudaEventCreate(&e1));
        GFX_CUDA(cudaEventRecord(e0, m.compute_stream()));
        for (int i = 0; i < n; ++i)
            m.infer(models[i], static_cast<const char*>(in) + static_cast<size_t>(i) * in_stride,
                    static_cast<char*>(out) + static_cast<size_t>(i % 2) * out_stride);
        GFX_CUDA(cudaEventRecord(e1, m.compute_stream()));
        GFX_CUDA(cudaEventSynchronize(e1));
        *ms = elapsed_ms(e0, e1);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    });
}

int gfx_infer_masked(gfx_arena_t a, int model_idx, const void* in, void* out, int batch, const int32_t* lengths,
                     void* hidden, gfx_event_t* done) {
    return guarded([&] {
        const gfx::ModelBlob& b = ModelStore::get().at(model_idx);
        if (b.desc.family != GFX_MODEL_BERT) throw std::invalid_argument("gfx_infer_masked: BERT models only");
        if (batch != b.desc.batch) throw std::invalid_argument("batch does not match the registered model");
        if (!lengths) throw std::invalid_argument("gfx_infer_masked: lengths required");
        a->mgr->infer(model_idx, in, out, hidden, lengths);
        if (hidden) GFX_CUDA(cudaStreamSynchronize(a->mgr->compute_stream()));
        make_event(*a->mgr, a->mgr->compute_stream(), done);
    });
}
int gfx_infer_debug(gfx_arena_t a, int model_idx, const void* in, void* out, int batch, void* hidden) {
    return guarded([&] {
        const gfx::ModelBlob& b = ModelStore::get().at(model_idx);
        if (b.desc.family != GFX_MODEL_BERT) throw std::invalid_argument("gfx_infer_debug: BERT models only");
        if (batch != b.desc.batch) throw std::invalid_argument("batch does not match the registered model");
        a->mgr->infer(model_idx, in, out, hidden);
        GFX_CUDA(cudaStreamSynchronize(a->mgr->compute_stream()));
    });
}

int gfx_bert_gemm(gfx_arena_t a, int model_idx, int layer, int op, const void* x, const void* resid, void* y,
                  int tokens) {
    return guarded([&] {
        a->mgr->bert_gemm(model_idx, layer, op, x, resid, y, tokens);
        GFX_CUDA(cudaStreamSynchronize(a->mgr->compute_stream()));
    });
}

int gfx_event_query(gfx_event_t e) {
    cudaSetDevice(e->device);
    const cudaError_t r = cudaEventQuery(e->ev);
    if (r == cudaSuccess) return 0;
    if (r == cudaErrorNotReady) {
        cudaGetLastError();
        return 1;
    }
    g_err = cudaGetErrorString(r);
    return -GFX_ERR_CUDA;
}
int gfx_event_sync(gfx_event_t e) {
    return guarded([&] {
        GFX_CUDA(cudaSetDevice(e->device));
        GFX_CUDA(cudaEventSynchronize(e->ev));
    });
}
int gfx_event_release(gfx_event_t e) {
    return guarded([&] {
        if (e) {
            cudaEventDestroy(e->ev);
            delete e;
        }
    });
}

int gfx_device_alloc(gfx_arena_t a, uint64_t bytes, void** out) {
    return guarded([&] {
        a->mgr->activate();
        GFX_CUDA(cudaMalloc(out, bytes));
    });
}
int gfx_device_free(gfx_arena_t a, void* p) {
    return guarded([&] {
        a->mgr->activate();
        GFX_CUDA(cudaFree(p));
    });
}
int gfx_memcpy_h2d(gfx_arena_t a, void* dst, const void* src, uint64_t bytes) {
    return guarded([&] {
        a->mgr->activate();
        GFX_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, a->mgr->compute_stream()));
        GFX_CUDA(cudaStreamSynchronize(a->mgr->compute_stream()));
    });
}
int gfx_memcpy_d2h(gfx_arena_t a, void* dst, const void* src, uint64_t bytes) {
    return guarded([&] {
        a->mgr->activate();
        GFX_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, a->mgr->compute_stream()));
        GFX_CUDA(cudaStreamSynchronize(a->mgr->compute_stream()));
    });
}
int gfx_synchronize(gfx_arena_t a) {
    return guarded([&] {
        a->mgr->activate();
        GFX_CUDA(cudaStreamSynchronize(a->mgr->copy_stream()));
        GFX_CUDA(cudaStreamSynchronize(a->mgr->compute_stream()));
    });
}
int gfx_fill_params(gfx_arena_t a, float* dst, uint64_t n, uint64_t seed, uint32_t tensor, float scale) {
    return guarded([&] {
        a->mgr->activate();
        gfx::launch_fill_params(dst, n, seed, tensor, scale, a->mgr->compute_stream());
        GFX_CUDA(cudaStreamSynchronize(a->mgr->compute_stream()));
    });
}
int gfx_host_fill_params(float* dst, uint64_t n, uint64_t seed, uint32_t tensor, float scale) {
    return guarded([&] {
        const uint64_t stream = gfx::param_stream(seed, tensor);
        const float scaled = gfx::param_scale(scale);
        for (uint64_t i = 0; i < n; ++i) dst[i] = gfx::param_at(stream, i, scaled);
    });
}
uint64_t gfx_input_seed(int request_id) { return 0xC0FFEE0000000000ULL + static_cast<uint64_t>(request_id); }

int gfx_replay_create(const gfx_replay_args* args, gfx_replay_t* out) {
    return guarded([&] {
        auto r = std::make_unique<gfx_replay_s>();
        r->args = *args;
        r->catalog_csv = args->catalog_csv ? args->catalog_csv : "";
        if (args->trace_csv) r->trace_csv = args->trace_csv;
        r->args.catalog_csv = r->catalog_csv.c_str();
        r->args.trace_csv = args->trace_csv ? r->trace_csv.c_str() : nullptr;
        r->setup();
        *out = r.release();
    });
}
int gfx_replay_run(gfx_replay_t r, gfx_replay_result* out) {
    return guarded([&] { r->run(out); });
}
int gfx_replay_run_live(gfx_replay_t r, double time_scale, double ema_alpha, gfx_replay_result* out) {
    return guarded([&] { r->run_live(time_scale, ema_alpha, out); });
}
int gfx_replay_outputs(gfx_replay_t r, void* host, uint64_t bytes) {
    return guarded([&] {
        if (!r->full_outputs) throw std::invalid_argument("replay was created without keep_outputs");
        const size_t n = r->requests.size();
        if (bytes < n * r->out_bytes) throw std::invalid_argument("output buffer too small");
        for (size_t g = 0; g < r->mgrs.size(); ++g) {
            if (!r->mgrs[g]) continue;
            GFX_CUDA(cudaSetDevice(r->dev_of[g]));
            GFX_CUDA(cudaDeviceSynchronize());
        }
        // Each request's output lives on the GPU that served it in the last run.
        for (size_t i = 0; i < n; ++i) {
            const int g = r->req_gpu[i] >= 0 ? r->req_gpu[i] : (r->args.only_gpu >= 0 ? r->args.only_gpu : 0);
            if (!r->mgrs[static_cast<size_t>(g)]) continue;
            GFX_CUDA(cudaSetDevice(r->dev_of[static_cast<size_t>(g)]));
            GFX_CUDA(cudaMemcpy(static_cast<char*>(host) + i * r->out_bytes,
                                r->bufs[static_cast<size_t>(g)].outputs + i * r->out_bytes, r->out_bytes,
                                cudaMemcpyDeviceToHost));
        }
    });
}
int gfx_replay_requests(gfx_replay_t r, int32_t* model_idx, double* service_ms, int64_t n) {
    return guarded([&] {
        for (int64_t i = 0; i < n && static_cast<size_t>(i) < r->last_models.size(); ++i) {
            if (model_idx) model_idx[i] = r->last_models[static_cast<size_t>(i)];
            if (service_ms)
                service_ms[i] = (r->req_start[static_cast<size_t>(i)] && r->req_end[static_cast<size_t>(i)])
                                    ? elapsed_ms(r->req_start[static_cast<size_t>(i)], r->req_end[static_cast<size_t>(i)])
                                    : -1.0;
        }
    });
}
uint64_t gfx_replay_ipc_blob_bytes(void) { return sizeof(gfx_replay_s::IpcBlob); }
int gfx_replay_ipc_export(gfx_replay_t r, void* blob, uint64_t bytes) {
    return guarded([&] { r->ipc_export(blob, bytes); });
}
int gfx_replay_ipc_import(gfx_replay_t r, const void* blobs, int32_t n) {
    return guarded([&] { r->ipc_import(blobs, n); });
}
int gfx_replay_destroy(gfx_replay_t r) {
    return guarded([&] { delete r; });
}
int gfx_replay(const gfx_replay_args* args, gfx_replay_result* out) {
    gfx_replay_t r = nullptr;
    int rc = gfx_replay_create(args, &r);
    if (rc) return rc;
    rc = gfx_replay_run(r, out);
    gfx_replay_destroy(r);
    return rc;
}

}  // extern "C"
