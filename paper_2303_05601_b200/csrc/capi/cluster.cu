// N1: the paper's per-GPU GPU Manager as its own process — one gfx_managerd
// daemon per B200 owning that GPU's pre-allocated HBM arena, streams and pinned
// host model store — fed by the global cache manager (the process calling
// gfx_cluster_*: the reference control plane, scheduler + ClusterState,
// proj/include/gpufaas/cluster.hpp:88-140) over ONE POSIX shared-memory
// segment: per GPU a command ring (coordinator -> daemon) and a completion ring
// (daemon -> coordinator), both single-producer / single-consumer.
//
// Why: one process per GPU is how the path runs on a multi-GPU node, and the
// non-deterministic live mode (completions observed on the device drive the
// scheduler) cannot be replayed independently by each rank, so a single
// decision producer must feed every GPU — the reference's own structure
// (the scheduler is one sequential thread).
//
// A dispatch (ExecutionListener::on_begin_execution, the hook where the
// reference adds load_time_us / infer_time_us, proj/src/cluster.cpp:159-168)
// becomes one EXEC command: the LRU victims to evict, the load (pinned-host H2D,
// or an NVLink fetch out of the lowest-id holder's arena,
// proj/src/cluster.cpp:69-72 / proj/src/sched.cpp:117,127) and the inference.
// The coordinator keeps a shadow of every daemon's page allocator (a daemon
// allocates the lowest free pages, deterministically), so a fetch command
// carries the holder's page table. Cross-daemon ordering is device-side, as in
// the replay's one-process-per-GPU mode: each daemon's flag words are CUDA-IPC
// mapped by every peer; a holder's copy stream publishes its cumulative load
// count of a model into every peer's flags after each load
// (cuStreamWriteValue32); a fetcher's copy stream waits for the count the
// coordinator saw when it decided the fetch (cuStreamWaitValue32), copies, and
// writes its cumulative fetch count back into the holder's flags; a holder
// waits for every fetch decided so far before reusing a victim's pages. The
// daemon reports each request's completion (device events polled on the host)
// with its measured load and inference durations; in live mode those
// completions are the scheduling points.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <fcntl.h>
#include <signal.h>
#include <spawn.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <sys/wait.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstring>
#include <deque>
#include <memory>
#include <set>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "capi_common.hpp"
#include "gpufaas/engine.hpp"
#include "gpufaas_b200.h"
#include "manager.cuh"

extern char** environ;

namespace {

using gfx::GpuManager;
using gfx::ModelStore;

thread_local std::string g_err;

constexpr uint32_t kMagic = 0x47465843u;  // "GFXC"
constexpr int kMaxGpus = 8;
constexpr int kMaxModels = 64;
constexpr int kMaxEvict = 16;
constexpr int kRingSlots = 64;
constexpr size_t kMailboxBytes = 256 * 1024;  // one request's output (MLP: 2 x 32 x 1000 fp32)

enum Op : int32_t { kOpExec = 1, kOpReset = 2, kOpOutput = 3, kOpStats = 4, kOpStop = 5 };
enum DoneKind : int32_t { kDoneRequest = 1, kDoneReset = 2, kDoneOutput = 3, kDoneStats = 4, kDoneError = 5 };

struct Cmd {
    int32_t op;
    int32_t request;
    int32_t model;
    int32_t hit;
    int32_t n_evict;
    int32_t source;        // miss: -1 = pinned-host load, else the peer GPU holding the model
    uint32_t wait_loaded;  // fetch: the holder's cumulative load count of `model` to wait for
    uint32_t my_loaded;    // miss: this GPU's cumulative load count of `model` after this load
    uint32_t fetch_done;   // fetch: this GPU's cumulative fetch count of `model` out of `source`
    int32_t evict[kMaxEvict];
    uint32_t evict_reads[kMaxEvict][kMaxGpus];  // fetches of each victim by each reader so far
    uint32_t n_src_pages;
    uint32_t src_pages[GFX_MAX_PAGES];  // the holder's page table of `model`
};

struct Done {
    int32_t kind;
    int32_t request;
    int64_t load_ns;   // copy-stream time of the load (0 on a hit)
    int64_t infer_ns;  // compute-stream time of the inference
    double device_ms;  // stats: device time since the reset (all streams joined)
    int64_t launches;  // stats: kernel launches since the reset
};

template <typename T, int N>
struct Ring {  // single producer, single consumer, across processes (lock-free 64-bit atomics)
    alignas(64) std::atomic<uint64_t> head;
    alignas(64) std::atomic<uint64_t> tail;
    T slot[N];
    bool try_push(const T& v) {
        const uint64_t h = head.load(std::memory_order_relaxed);
        if (h - tail.load(std::memory_order_acquire) >= static_cast<uint64_t>(N)) return false;
        slot[h % N] = v;
        head.store(h + 1, std::memory_order_release);
        return true;
    }
    bool try_pop(T& v) {
        const uint64_t t = tail.load(std::memory_order_relaxed);
        if (t == head.load(std::memory_order_acquire)) return false;
        v = slot[t % N];
        tail.store(t + 1, std::memory_order_release);
        return true;
    }
};

struct IpcBlob {
    cudaIpcMemHandle_t arena;
    cudaIpcMemHandle_t flags;
    uint64_t arena_pages;
};

struct GpuBlock {
    std::atomic<int32_t> state;  // 0 starting, 1 ready (IPC blob published), -1 failed
    int32_t device;
    char error[512];
    IpcBlob ipc;
    Ring<Cmd, kRingSlots> cmd;
    Ring<Done, kRingSlots> done;
    alignas(64) uint8_t mailbox[kMailboxBytes];
};

struct Shm {
    uint32_t magic;
    int32_t gpu_count;
    int32_t n_models;
    int32_t n_requests;  // output slots each daemon keeps
    int32_t use_p2p;
    int32_t pad_;
    uint64_t arena_bytes;
    std::atomic<int32_t> peers_ready;  // every daemon's IPC blob is published
    gfx_model_desc models[kMaxModels];
    GpuBlock gpu[kMaxGpus];
};

constexpr size_t flag_words(int G, int M) { return 2 * static_cast<size_t>(G) * static_cast<size_t>(M); }
constexpr size_t fl_loaded(int M, int s, int m) { return static_cast<size_t>(s) * M + m; }
constexpr size_t fl_read(int G, int M, int m, int r) {
    return static_cast<size_t>(G) * M + static_cast<size_t>(m) * G + r;
}

Shm* map_shm(const char* name, bool create, int* fd_out) {
    const int fd = shm_open(name, create ? (O_CREAT | O_EXCL | O_RDWR) : O_RDWR, 0600);
    if (fd < 0) throw std::runtime_error(std::string("shm_open ") + name + ": " + std::strerror(errno));
    if (create && ftruncate(fd, sizeof(Shm)) != 0) {
        close(fd);
        throw std::runtime_error(std::string("ftruncate shm: ") + std::strerror(errno));
    }
    struct stat st{};
    if (!create && (fstat(fd, &st) != 0 || static_cast<size_t>(st.st_size) < sizeof(Shm))) {
        close(fd);  // created but not sized yet: the caller retries
        throw std::runtime_error("shm segment not ready");
    }
    void* p = mmap(nullptr, sizeof(Shm), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    if (p == MAP_FAILED) {
        close(fd);
        throw std::runtime_error(std::string("mmap shm: ") + std::strerror(errno));
    }
    *fd_out = fd;
    return static_cast<Shm*>(p);
}

// ------------------------------------------------------------------ daemon

struct Daemon {
    Shm* shm = nullptr;
    int fd = -1;
    int gpu = 0, G = 0, M = 0;
    std::unique_ptr<GpuManager> mgr;
    uint32_t* flags = nullptr;              // ours (device), written by peers
    std::vector<char*> peer_arena;          // IPC-mapped
    std::vector<uint32_t*> peer_flags;      // IPC-mapped
    char* in = nullptr;                     // one request input (filled on the device per request)
    char* outs = nullptr;                   // [n_requests][out_bytes]
    size_t in_bytes = 0, out_bytes = 0;
    int family = 0;
    struct Task {
        int32_t request;
        cudaEvent_t ls, le, is, ie;
        bool loaded;
    };
    std::deque<Task> inflight;
    std::vector<cudaEvent_t> pool;
    cudaEvent_t t0 = nullptr, t1 = nullptr;

    cudaEvent_t event() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        GFX_CUDA(cudaEventCreate(&e));
        return e;
    }

    void push_done(const Done& d) {
        while (!shm->gpu[gpu].done.try_push(d)) std::this_thread::yield();
    }

    void setup() {
        GpuBlock& b = shm->gpu[gpu];
        G = shm->gpu_count;
        M = shm->n_models;
        GFX_CUDA(cudaSetDevice(b.device));
        for (int i = 0; i < M; ++i)  // a rank may have registered the models already (same process)
            if (!ModelStore::get().has(i) || ModelStore::get().at(i).desc.seed != shm->models[i].seed)
                ModelStore::get().add(i, shm->models[i]);
        const gfx::ModelBlob& b0 = ModelStore::get().at(0);
        in_bytes = b0.in_bytes;
        out_bytes = b0.out_bytes;
        family = b0.desc.family;
        if (out_bytes > kMailboxBytes) throw std::invalid_argument("request output larger than the mailbox");
        for (int g = 0; g < G; ++g)  // another daemon serves a GPU on this device
            if (g != gpu && shm->gpu[g].device == b.device) gfx::mark_device_shared(b.device);
        mgr = std::make_unique<GpuManager>(b.device, shm->arena_bytes, gpu);
        GFX_CUDA(cudaMalloc(&flags, flag_words(G, M) * 4));
        GFX_CUDA(cudaMemset(flags, 0, flag_words(G, M) * 4));
        GFX_CUDA(cudaMalloc(&in, in_bytes));
        GFX_CUDA(cudaMalloc(&outs, out_bytes * static_cast<size_t>(std::max(1, shm->n_requests))));
        GFX_CUDA(cudaEventCreate(&t0));
        GFX_CUDA(cudaEventCreate(&t1));
        GFX_CUDA(cudaDeviceSynchronize());
        GFX_CUDA(cudaIpcGetMemHandle(&b.ipc.arena, mgr->arena()));
        GFX_CUDA(cudaIpcGetMemHandle(&b.ipc.flags, flags));
        b.ipc.arena_pages = mgr->total_pages();
        b.state.store(1, std::memory_order_release);
        // Peers' arenas and flag words, once every daemon has published its blob.
        while (shm->peers_ready.load(std::memory_order_acquire) == 0) std::this_thread::sleep_for(std::chrono::milliseconds(1));
        peer_arena.assign(G, nullptr);
        peer_flags.assign(G, nullptr);
        for (int g = 0; g < G; ++g) {
            if (g == gpu || !shm->use_p2p) continue;
            void* p = nullptr;
            GFX_CUDA(cudaIpcOpenMemHandle(&p, shm->gpu[g].ipc.arena, cudaIpcMemLazyEnablePeerAccess));
            peer_arena[g] = static_cast<char*>(p);
            GFX_CUDA(cudaIpcOpenMemHandle(&p, shm->gpu[g].ipc.flags, cudaIpcMemLazyEnablePeerAccess));
            peer_flags[g] = static_cast<uint32_t*>(p);
        }
    }

    void exec(const Cmd& c) {
        GpuManager& m = *mgr;
        m.activate();
        Task t{c.request, nullptr, nullptr, event(), event(), !c.hit};
        if (!c.hit) {
            t.ls = event();
            t.le = event();
            GFX_CUDA(cudaEventRecord(t.ls, m.copy_stream()));
            for (int i = 0; i < c.n_evict; ++i) {
                const int v = c.evict[i];
                for (int r = 0; r < G; ++r)  // every fetch of our pages of v decided so far has completed
                    if (c.evict_reads[i][r]) m.copy_wait_geq(flags + fl_read(G, M, v, r), c.evict_reads[i][r]);
                m.evict(v);
            }
            if (c.source >= 0) {
                if (!peer_arena[c.source]) throw std::logic_error("peer fetch without an IPC-mapped peer");
                const std::vector<uint32_t> sp(c.src_pages, c.src_pages + c.n_src_pages);
                m.load_remote(c.model, peer_arena[c.source], sp, flags + fl_loaded(M, c.source, c.model), c.wait_loaded);
                m.copy_write(peer_flags[c.source] + fl_read(G, M, c.model, gpu), c.fetch_done);
            } else {
                m.load(c.model, nullptr);
            }
            GFX_CUDA(cudaEventRecord(t.le, m.copy_stream()));
            if (shm->use_p2p)  // our load of the model is complete: publish the count to every peer
                for (int r = 0; r < G; ++r)
                    if (r != gpu) m.copy_write(peer_flags[r] + fl_loaded(M, gpu, c.model), c.my_loaded);
        }
        // The request's input (its parameter stream) and the inference.
        const uint64_t seed = gfx_input_seed(c.request);
        if (family == GFX_MODEL_BERT)
            gfx::launch_fill_bf16(reinterpret_cast<__nv_bfloat16*>(in), in_bytes / 2, seed, 0xFFFFFFFFu, 1.0f,
                                  m.compute_stream());
        else
            gfx::launch_fill_params(reinterpret_cast<float*>(in), in_bytes / 4, seed, 0xFFFFFFFFu, 1.0f,
                                    m.compute_stream());
        GFX_CUDA(cudaEventRecord(t.is, m.compute_stream()));
        m.infer(c.model, in, outs + static_cast<size_t>(c.request) * out_bytes);
        GFX_CUDA(cudaEventRecord(t.ie, m.compute_stream()));
        inflight.push_back(t);
    }

    bool poll_inflight() {  // report the oldest task once its inference finished
        if (inflight.empty()) return false;
        Task& t = inflight.front();
        for (cudaEvent_t e : {t.ie, t.le}) {  // the inference, and the load's end on the copy stream
            if (!e) continue;
            const cudaError_t st = cudaEventQuery(e);
            if (st == cudaErrorNotReady) return false;
            GFX_CUDA(st);
        }
        float li = 0, ii = 0;
        if (t.loaded) GFX_CUDA(cudaEventElapsedTime(&li, t.ls, t.le));
        GFX_CUDA(cudaEventElapsedTime(&ii, t.is, t.ie));
        Done d{kDoneRequest, t.request, static_cast<int64_t>(li * 1e6), static_cast<int64_t>(ii * 1e6), 0.0, 0};
        push_done(d);
        for (cudaEvent_t e : {t.ls, t.le, t.is, t.ie})
            if (e) pool.push_back(e);
        inflight.pop_front();
        return true;
    }

    void drain() {
        while (!inflight.empty()) poll_inflight();
    }

    int serve() {
        GpuBlock& b = shm->gpu[gpu];
        for (;;) {
            Cmd c;
            bool busy = poll_inflight();
            if (b.cmd.try_pop(c)) {
                busy = true;
                switch (c.op) {
                    case kOpExec:
                        exec(c);
                        break;
                    case kOpReset: {
                        drain();
                        mgr->reset();
                        mgr->kernel_launches = 0;
                        GFX_CUDA(cudaEventRecord(t0, mgr->compute_stream()));
                        GFX_CUDA(cudaStreamWaitEvent(mgr->copy_stream(), t0, 0));
                        push_done(Done{kDoneReset, -1, 0, 0, 0.0, 0});
                        break;
                    }
                    case kOpStats: {
                        drain();
                        cudaEvent_t j = event();
                        GFX_CUDA(cudaEventRecord(j, mgr->copy_stream()));
                        GFX_CUDA(cudaStreamWaitEvent(mgr->compute_stream(), j, 0));
                        GFX_CUDA(cudaEventRecord(t1, mgr->compute_stream()));
                        GFX_CUDA(cudaEventSynchronize(t1));
                        float ms = 0;
                        GFX_CUDA(cudaEventElapsedTime(&ms, t0, t1));
                        pool.push_back(j);
                        push_done(Done{kDoneStats, -1, 0, 0, ms, mgr->kernel_launches});
                        break;
                    }
                    case kOpOutput: {
                        drain();
                        GFX_CUDA(cudaMemcpy(b.mailbox, outs + static_cast<size_t>(c.request) * out_bytes, out_bytes,
                                            cudaMemcpyDeviceToHost));
                        push_done(Done{kDoneOutput, c.request, 0, 0, 0.0, static_cast<int64_t>(out_bytes)});
                        break;
                    }
                    case kOpStop:
                        drain();
                        return 0;
                    default:
                        throw std::logic_error("unknown daemon command");
                }
            }
            if (!busy) std::this_thread::yield();
        }
    }

    ~Daemon() {
        if (mgr) {
            mgr->activate();
            cudaDeviceSynchronize();
            for (size_t g = 0; g < peer_arena.size(); ++g) {
                if (peer_arena[g]) cudaIpcCloseMemHandle(peer_arena[g]);
                if (peer_flags[g]) cudaIpcCloseMemHandle(peer_flags[g]);
            }
            for (cudaEvent_t e : pool) cudaEventDestroy(e);
            if (flags) cudaFree(flags);
            if (in) cudaFree(in);
            if (outs) cudaFree(outs);
            mgr.reset();
        }
        if (shm) munmap(shm, sizeof(Shm));
        if (fd >= 0) close(fd);
    }
};

// ------------------------------------------------------------------ coordinator

std::string library_dir() {
    Dl_info info{};
    if (dladdr(reinterpret_cast<void*>(&library_dir), &info) == 0 || !info.dli_fname) return ".";
    std::string p = info.dli_fname;
    const size_t k = p.rfind('/');
    return k == std::string::npos ? std::string(".") : p.substr(0, k);
}

}  // namespace

struct gfx_cluster_s : gpufaas::ExecutionListener, gpufaas::LiveExecutor {
    std::string name, catalog_csv, trace_csv;
    bool have_trace = false;
    gfx_sim_config sc{};
    gpufaas::Catalog catalog;
    std::vector<gpufaas::Request> requests;
    Shm* shm = nullptr;
    int fd = -1;
    int G = 0, M = 0;
    bool use_p2p = false;
    std::vector<pid_t> pids;
    std::vector<uint32_t> model_pages;
    // shadow of every daemon's page allocator (lowest free pages first, like GpuManager::allocate)
    struct Shadow {
        std::set<uint32_t> free;
        std::vector<std::vector<uint32_t>> pages;
    };
    std::vector<Shadow> shadow;
    std::vector<uint32_t> load_cnt;   // [G][M] loads decided so far (all runs)
    std::vector<uint32_t> fetch_cnt;  // [G src][M][G reader] fetches decided so far (all runs)
    // per-run state
    std::vector<std::deque<int32_t>> dispatched;  // per GPU, requests in dispatch order
    std::vector<std::deque<Done>> completed;      // per GPU, completion records in order
    std::vector<int32_t> req_gpu;
    gfx_replay_result res{};

    uint32_t& fetches(int src, int m, int r) {
        return fetch_cnt[(static_cast<size_t>(src) * M + m) * G + r];
    }

    void check_children() {
        for (size_t g = 0; g < pids.size(); ++g) {
            if (pids[g] <= 0) continue;
            int status = 0;
            if (waitpid(pids[g], &status, WNOHANG) == pids[g]) {
                pids[g] = -1;
                throw gfx::CudaError("gfx_managerd of GPU " + std::to_string(g) + " exited: " + shm->gpu[g].error);
            }
        }
    }

    // Pulls every completion record the daemons have posted.
    void drain_done() {
        Done d;
        for (int g = 0; g < G; ++g)
            while (shm->gpu[g].done.try_pop(d)) {
                if (d.kind == kDoneError) throw gfx::CudaError("gfx_managerd of GPU " + std::to_string(g) + ": " +
                                                               shm->gpu[g].error);
                completed[static_cast<size_t>(g)].push_back(d);
            }
    }

    void push(int g, const Cmd& c) {
        auto t0 = std::chrono::steady_clock::now();
        while (!shm->gpu[g].cmd.try_push(c)) {
            drain_done();  // a daemon blocked on a full completion ring would never pop commands
            check_children();
            std::this_thread::yield();
            if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120))
                throw gfx::CudaError("gfx_managerd of GPU " + std::to_string(g) + " stopped taking commands");
        }
    }

    // Blocks until GPU g posted a record of `kind`; returns it (request records stay queued).
    Done wait_kind(int g, int32_t kind) {
        auto t0 = std::chrono::steady_clock::now();
        for (;;) {
            drain_done();
            auto& q = completed[static_cast<size_t>(g)];
            for (auto it = q.begin(); it != q.end(); ++it)
                if (it->kind == kind) {
                    Done d = *it;
                    q.erase(it);
                    return d;
                }
            check_children();
            std::this_thread::sleep_for(std::chrono::microseconds(50));
            if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(600))
                throw gfx::CudaError("timeout waiting for gfx_managerd of GPU " + std::to_string(g));
        }
    }

    void start(const gfx_cluster_args& a) {
        catalog_csv = a.catalog_csv ? a.catalog_csv : "";
        have_trace = a.trace_csv != nullptr;
        if (have_trace) trace_csv = a.trace_csv;
        sc = a.cfg;
        std::istringstream cin_(catalog_csv);
        catalog = gpufaas::parse_catalog_csv(cin_, "catalog");
        requests = gpufaas::capi::make_requests(sc, catalog, have_trace ? trace_csv.c_str() : nullptr);
        G = sc.gpu_count;
        M = a.n_models;
        use_p2p = a.use_p2p != 0;
        if (G < 1 || G > kMaxGpus) throw std::invalid_argument("cluster: 1..8 GPUs");
        if (M < 1 || M > kMaxModels || static_cast<size_t>(M) != catalog.size())
            throw std::invalid_argument("cluster: one model description per catalog row (at most 64)");
        for (int i = 0; i < M; ++i) {
            const gfx_model_desc& d = a.models[i];
            uint64_t h = 14695981039346656037ULL;  // catalog row i must be model i (seed = FNV-1a of the id)
            for (unsigned char ch : catalog.profiles()[static_cast<size_t>(i)].model_id) {
                h ^= ch;
                h *= 1099511628211ULL;
            }
            if (d.seed != h) throw std::invalid_argument("cluster: model " + std::to_string(i) + " is not catalog row '" +
                                                         catalog.profiles()[static_cast<size_t>(i)].model_id + "'");
            model_pages.push_back(gfx::model_pages(d));
            if (catalog.profiles()[static_cast<size_t>(i)].occupation_mb < 2.0 * model_pages.back())
                throw std::invalid_argument("cluster: catalog occupation_mb below the model's arena pages");
        }
        const uint64_t pages = static_cast<uint64_t>(sc.capacity_mb / 2.0);
        static std::atomic<int> seq{0};
        name = a.shm_name ? a.shm_name
                          : "/gfx_cluster_" + std::to_string(getpid()) + "_" + std::to_string(seq.fetch_add(1));
        shm = map_shm(name.c_str(), true, &fd);
        std::memset(static_cast<void*>(shm), 0, sizeof(Shm));
        shm->gpu_count = G;
        shm->n_models = M;
        shm->n_requests = static_cast<int32_t>(requests.size());
        shm->use_p2p = use_p2p ? 1 : 0;
        shm->arena_bytes = pages * gfx::kPageBytes;
        for (int i = 0; i < M; ++i) shm->models[i] = a.models[i];
        for (int g = 0; g < G; ++g) shm->gpu[g].device = a.devices ? a.devices[g] : 0;
        __atomic_store_n(&shm->magic, kMagic, __ATOMIC_RELEASE);  // header complete: daemons may attach
        shadow.assign(static_cast<size_t>(G), {});
        for (Shadow& s : shadow) {
            for (uint32_t p = 0; p < pages; ++p) s.free.insert(p);
            s.pages.assign(static_cast<size_t>(M), {});
        }
        load_cnt.assign(static_cast<size_t>(G) * M, 0);
        fetch_cnt.assign(static_cast<size_t>(G) * M * G, 0);
        if (a.spawn) {
            const std::string exe = library_dir() + "/gfx_managerd";
            for (int g = 0; g < G; ++g) {
                const std::string gs = std::to_string(g);
                char* argv[] = {const_cast<char*>(exe.c_str()), const_cast<char*>(name.c_str()),
                                const_cast<char*>(gs.c_str()), nullptr};
                pid_t pid = -1;
                if (posix_spawn(&pid, exe.c_str(), nullptr, nullptr, argv, environ) != 0)
                    throw std::runtime_error("cannot start " + exe);
                pids.push_back(pid);
            }
        }
        auto t0 = std::chrono::steady_clock::now();
        for (int g = 0; g < G; ++g)
            for (;;) {
                const int st = shm->gpu[g].state.load(std::memory_order_acquire);
                if (st == 1) break;
                if (st < 0) throw gfx::CudaError("gfx_managerd of GPU " + std::to_string(g) + ": " + shm->gpu[g].error);
                check_children();
                if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(600))
                    throw gfx::CudaError("gfx_managerd of GPU " + std::to_string(g) + " did not start");
                std::this_thread::sleep_for(std::chrono::milliseconds(5));
            }
        shm->peers_ready.store(1, std::memory_order_release);
        dispatched.assign(static_cast<size_t>(G), {});
        completed.assign(static_cast<size_t>(G), {});
    }

    // ---- the dispatch hook (ExecutionListener)
    void on_begin_execution(int gpu, const gpufaas::Request& req, int model, bool hit, const std::vector<int>& evicted,
                            int source, gpufaas::SimTime, gpufaas::SimTime) override {
        Cmd c{};
        c.op = kOpExec;
        c.request = req.request_id;
        c.model = model;
        c.hit = hit ? 1 : 0;
        c.source = -1;
        if (!hit) {
            if (evicted.size() > static_cast<size_t>(kMaxEvict)) throw std::logic_error("cluster: too many victims");
            Shadow& sh = shadow[static_cast<size_t>(gpu)];
            c.n_evict = static_cast<int32_t>(evicted.size());
            for (size_t i = 0; i < evicted.size(); ++i) {
                const int v = evicted[i];
                c.evict[i] = v;
                for (int r = 0; r < G; ++r) c.evict_reads[i][r] = fetches(gpu, v, r);
                for (uint32_t p : sh.pages[static_cast<size_t>(v)]) sh.free.insert(p);
                sh.pages[static_cast<size_t>(v)].clear();
            }
            if (use_p2p && source >= 0 && source != gpu) {
                const std::vector<uint32_t>& sp = shadow[static_cast<size_t>(source)].pages[static_cast<size_t>(model)];
                if (sp.size() != model_pages[static_cast<size_t>(model)]) throw std::logic_error("cluster: holder shadow");
                c.source = source;
                c.wait_loaded = load_cnt[static_cast<size_t>(source) * M + model];
                c.fetch_done = ++fetches(source, model, gpu);
                c.n_src_pages = static_cast<uint32_t>(sp.size());
                std::copy(sp.begin(), sp.end(), c.src_pages);
                ++res.loads_p2p;
            } else {
                ++res.loads_h2d;
            }
            auto& mine = sh.pages[static_cast<size_t>(model)];
            mine.clear();
            for (uint32_t i = 0; i < model_pages[static_cast<size_t>(model)]; ++i) {
                mine.push_back(*sh.free.begin());
                sh.free.erase(sh.free.begin());
            }
            c.my_loaded = ++load_cnt[static_cast<size_t>(gpu) * M + model];
        }
        req_gpu[static_cast<size_t>(req.request_id)] = gpu;
        dispatched[static_cast<size_t>(gpu)].push_back(req.request_id);
        push(gpu, c);
    }
    void on_complete(int, int, gpufaas::SimTime) override {}

    // ---- live completions (LiveExecutor): the front dispatched task of a GPU has finished
    const Done* front_done(int g) {
        drain_done();
        auto& d = dispatched[static_cast<size_t>(g)];
        if (d.empty()) return nullptr;
        for (const Done& x : completed[static_cast<size_t>(g)])
            if (x.kind == kDoneRequest && x.request == d.front()) return &x;
        return nullptr;
    }
    bool done(int g) override {
        if (dispatched[static_cast<size_t>(g)].empty()) return true;
        check_children();
        return front_done(g) != nullptr;
    }
    bool measured(int g, gpufaas::SimTime* load_us, gpufaas::SimTime* infer_us) override {
        const Done* d = front_done(g);
        if (!d) return false;
        *load_us = d->load_ns > 0 ? std::max<gpufaas::SimTime>(1, (d->load_ns + 500) / 1000) : 0;
        *infer_us = std::max<gpufaas::SimTime>(1, (d->infer_ns + 500) / 1000);
        return true;
    }
    void retire(int g) override {
        auto& d = dispatched[static_cast<size_t>(g)];
        if (d.empty()) return;
        auto& q = completed[static_cast<size_t>(g)];
        for (auto it = q.begin(); it != q.end(); ++it)
            if (it->kind == kDoneRequest && it->request == d.front()) {
                q.erase(it);
                break;
            }
        d.pop_front();
    }

    void run(bool live, double time_scale, double alpha, gfx_replay_result* out) {
        if (live && !(time_scale > 0)) throw std::invalid_argument("live mode needs a positive time_scale");
        res = gfx_replay_result{};
        req_gpu.assign(requests.size(), -1);
        for (int g = 0; g < G; ++g) {
            dispatched[static_cast<size_t>(g)].clear();
            completed[static_cast<size_t>(g)].clear();
        }
        // Every request of the previous run finished (its fetches with it), so the
        // daemons can drop their residents; the shadows restart from empty arenas.
        for (int g = 0; g < G; ++g) push(g, Cmd{kOpReset});
        for (int g = 0; g < G; ++g) wait_kind(g, kDoneReset);
        for (Shadow& s : shadow) {
            for (auto& v : s.pages) {
                for (uint32_t p : v) s.free.insert(p);
                v.clear();
            }
        }
        const gpufaas::SimConfig cfg = gpufaas::capi::to_sim_config(sc);
        const auto h0 = std::chrono::steady_clock::now();
        gpufaas::SimResult sim = live ? gpufaas::run_live(cfg, catalog, requests, time_scale, this, *this, nullptr, alpha)
                                      : gpufaas::run_stream(cfg, catalog, requests, nullptr, nullptr, this);
        const auto h1 = std::chrono::steady_clock::now();
        double dev_ms = 0;
        for (int g = 0; g < G; ++g) push(g, Cmd{kOpStats});
        for (int g = 0; g < G; ++g) {
            const Done d = wait_kind(g, kDoneStats);
            dev_ms = std::max(dev_ms, d.device_ms);
            res.kernel_launches += d.launches;
        }
        res.n_requests = static_cast<int64_t>(sim.requests.size());
        res.n_decisions = static_cast<int64_t>(sim.decisions.size());
        res.hits = sim.report.hits;
        res.misses = sim.report.misses;
        res.false_misses = sim.report.false_misses;
        res.local_enqueues = sim.report.local_enqueues;
        res.evictions = sim.report.evictions;
        res.decision_digest = gpufaas::capi::decision_digest(sim.decisions);
        res.device_ms = dev_ms;
        res.host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count();
        res.sched_ms = std::chrono::duration<double, std::milli>(h1 - h0).count();
        res.sim_p50_s = gpufaas::latency_percentile_s(sim.requests, 50);
        res.sim_p99_s = gpufaas::latency_percentile_s(sim.requests, 99);
        res.sim_avg_latency_s = sim.report.avg_latency_s.value_or(0.0);
        *out = res;
    }

    void output(int32_t rid, void* host, uint64_t bytes) {
        if (rid < 0 || static_cast<size_t>(rid) >= req_gpu.size() || req_gpu[static_cast<size_t>(rid)] < 0)
            throw std::invalid_argument("request was not served in the last run");
        const int g = req_gpu[static_cast<size_t>(rid)];
        Cmd c{};
        c.op = kOpOutput;
        c.request = rid;
        push(g, c);
        const Done d = wait_kind(g, kDoneOutput);
        if (bytes < static_cast<uint64_t>(d.launches)) throw std::invalid_argument("output buffer too small");
        std::memcpy(host, shm->gpu[g].mailbox, static_cast<size_t>(d.launches));
    }

    ~gfx_cluster_s() override {
        if (shm) {
            for (int g = 0; g < G; ++g) {
                Cmd c{};
                c.op = kOpStop;
                for (int i = 0; i < 1000 && !shm->gpu[g].cmd.try_push(c); ++i) std::this_thread::sleep_for(std::chrono::milliseconds(1));
            }
            for (pid_t& p : pids) {
                if (p <= 0) continue;
                int status = 0;
                for (int i = 0; i < 3000 && waitpid(p, &status, WNOHANG) == 0; ++i)
                    std::this_thread::sleep_for(std::chrono::milliseconds(10));
                if (waitpid(p, &status, WNOHANG) == 0) {
                    kill(p, SIGKILL);
                    waitpid(p, &status, 0);
                }
            }
            munmap(shm, sizeof(Shm));
        }
        if (fd >= 0) close(fd);
        if (!name.empty()) shm_unlink(name.c_str());
    }
};

extern "C" {

const char* gfx_cluster_last_error(void) { return g_err.c_str(); }

int gfx_cluster_create(const gfx_cluster_args* args, gfx_cluster_t* out) {
    return gpufaas::capi::guarded_call(g_err, [&] {
        auto c = std::make_unique<gfx_cluster_s>();
        c->start(*args);
        *out = c.release();
    });
}

int gfx_cluster_run(gfx_cluster_t c, gfx_replay_result* out) {
    return gpufaas::capi::guarded_call(g_err, [&] { c->run(false, 0.0, 0.0, out); });
}

int gfx_cluster_run_live(gfx_cluster_t c, double time_scale, double ema_alpha, gfx_replay_result* out) {
    return gpufaas::capi::guarded_call(g_err, [&] { c->run(true, time_scale, ema_alpha, out); });
}

int gfx_cluster_output(gfx_cluster_t c, int32_t request_id, void* host, uint64_t bytes) {
    return gpufaas::capi::guarded_call(g_err, [&] { c->output(request_id, host, bytes); });
}

int gfx_cluster_request_gpu(gfx_cluster_t c, int32_t request_id, int32_t* gpu) {
    return gpufaas::capi::guarded_call(g_err, [&] {
        if (request_id < 0 || static_cast<size_t>(request_id) >= c->req_gpu.size())
            throw std::invalid_argument("request id out of range");
        *gpu = c->req_gpu[static_cast<size_t>(request_id)];
    });
}

int gfx_cluster_destroy(gfx_cluster_t c) {
    return gpufaas::capi::guarded_call(g_err, [&] { delete c; });
}

int gfx_cluster_ring_selftest(int64_t n) {
    // A forked producer pushes n commands through a shared-memory ring; this
    // process pops them and checks order and payload (no device needed).
    return gpufaas::capi::guarded_call(g_err, [&] {
        using R = Ring<Cmd, kRingSlots>;
        void* mem = mmap(nullptr, sizeof(R), PROT_READ | PROT_WRITE, MAP_SHARED | MAP_ANONYMOUS, -1, 0);
        if (mem == MAP_FAILED) throw std::runtime_error("mmap failed");
        R* ring = new (mem) R();
        const pid_t pid = fork();
        if (pid < 0) throw std::runtime_error("fork failed");
        if (pid == 0) {
            for (int64_t i = 0; i < n; ++i) {
                Cmd c{};
                c.op = kOpExec;
                c.request = static_cast<int32_t>(i);
                c.model = static_cast<int32_t>(i * 7 % 1000);
                c.src_pages[GFX_MAX_PAGES - 1] = static_cast<uint32_t>(i);
                while (!ring->try_push(c)) {
                }
            }
            _exit(0);
        }
        std::string bad;
        for (int64_t i = 0; i < n && bad.empty(); ++i) {
            Cmd c;
            while (!ring->try_pop(c)) {
            }
            if (c.request != i || c.model != i * 7 % 1000 || c.src_pages[GFX_MAX_PAGES - 1] != static_cast<uint32_t>(i))
                bad = "ring item " + std::to_string(i) + " out of order or torn";
        }
        int status = 0;
        waitpid(pid, &status, 0);
        munmap(mem, sizeof(R));
        if (!bad.empty()) throw std::logic_error(bad);
        if (!WIFEXITED(status) || WEXITSTATUS(status) != 0) throw std::runtime_error("ring producer failed");
    });
}

int gfx_managerd_serve(const char* shm_name, int32_t gpu_index) {
    Daemon d;
    try {
        // The coordinator may create the segment after a rank started its daemon (spawn = 0).
        for (int i = 0;; ++i) {
            try {
                d.shm = map_shm(shm_name, false, &d.fd);
                break;
            } catch (const std::runtime_error&) {
                if (i >= 12000) throw;  // 60 s
                std::this_thread::sleep_for(std::chrono::milliseconds(5));
            }
        }
        for (int i = 0; __atomic_load_n(&d.shm->magic, __ATOMIC_ACQUIRE) != kMagic; ++i) {
            if (i >= 60000) throw std::runtime_error("segment never initialised");
            std::this_thread::sleep_for(std::chrono::milliseconds(1));
        }
        if (gpu_index < 0 || gpu_index >= d.shm->gpu_count) throw std::invalid_argument("gpu index out of range");
        d.gpu = gpu_index;
        d.setup();
        return d.serve();
    } catch (const std::exception& e) {
        if (d.shm) {
            std::snprintf(d.shm->gpu[gpu_index].error, sizeof d.shm->gpu[gpu_index].error, "%s", e.what());
            d.shm->gpu[gpu_index].state.store(-1, std::memory_order_release);
            Done x{kDoneError, -1, 0, 0, 0.0, 0};
            d.shm->gpu[gpu_index].done.try_push(x);
        }
        std::fprintf(stderr, "gfx_managerd %d: %s\n", gpu_index, e.what());
        return 1;
    }
}

}  // extern "C"
