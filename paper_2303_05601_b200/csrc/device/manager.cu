// GPU Manager implementation — see manager.cuh.
#include "manager.cuh"

#include <cuda.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <thread>

namespace gfx {

namespace {
constexpr int kMaxDim = 8192;  // widest layer the inference workspace supports
constexpr int kBatch = 32;
}  // namespace

// ------------------------------------------------------------- model store

ModelBlob::~ModelBlob() {
    if (host) cudaFreeHost(host);
}

void mlp_layout(const gfx_model_desc& d, std::vector<uint64_t>& w_off, std::vector<uint64_t>& b_off,
                uint64_t& bytes) {
    w_off.clear();
    b_off.clear();
    uint64_t off = 0;
    auto align = [](uint64_t v, uint64_t a) { return (v + a - 1) & ~(a - 1); };
    for (int l = 0; l < d.n_layers; ++l) {
        const uint64_t K = static_cast<uint64_t>(d.dims[l]);
        const uint64_t N = static_cast<uint64_t>(d.dims[l + 1]);
        const uint64_t Npad = align(N, kWTileRows);
        off = align(off, 16384);  // tiles never straddle a 2 MiB page
        w_off.push_back(off);
        off += 4 * K * Npad;
        off = align(off, 256);
        b_off.push_back(off);
        off += 4 * N;
    }
    bytes = align(off, 256);
}

uint32_t model_pages(const gfx_model_desc& desc) {
    uint64_t bytes = 0;
    if (desc.family == GFX_MODEL_BERT) {
        bytes = bert_layout(desc.n_layers, desc.dims[0], desc.dims[1], desc.dims[2], desc.dims[3]).bytes;
    } else if (desc.family == GFX_MODEL_MLP) {
        if (desc.n_layers < 1 || desc.n_layers > GFX_MAX_LAYERS) throw std::invalid_argument("bad layer count");
        std::vector<uint64_t> w, b;
        mlp_layout(desc, w, b, bytes);
    } else {
        throw std::invalid_argument("unsupported model family");
    }
    return static_cast<uint32_t>((bytes + kPageBytes - 1) / kPageBytes);
}

ModelStore& ModelStore::get() {
    static ModelStore store;
    return store;
}

namespace {

// BERT parameter blob: bf16 weight tiles, fp32 vectors.
void build_bert_blob(ModelBlob& blob) {
    const gfx_model_desc& d = blob.desc;
    const BertLayout& lay = blob.bert;
    char* base = reinterpret_cast<char*>(blob.host);
    std::vector<std::thread> pool;
    struct Mat {
        uint64_t off, n, k;
        uint32_t tensor;
    };
    struct Vec {
        uint64_t off, n;
        uint32_t tensor;
        float scale, shift;
    };
    std::vector<Mat> mats;
    std::vector<Vec> vecs;
    const uint64_t D = static_cast<uint64_t>(lay.d), F = static_cast<uint64_t>(lay.ffn);
    const float sd = static_cast<float>(1.0 / std::sqrt(static_cast<double>(D)));
    const float sf = static_cast<float>(1.0 / std::sqrt(static_cast<double>(F)));
    for (int l = 0; l < lay.L; ++l) {
        const BertLayerOffsets& o = lay.layer[static_cast<size_t>(l)];
        const uint32_t t0 = 16u * static_cast<uint32_t>(l);
        mats.push_back({o.wqkv, 3 * D, D, t0 + kWqkv});
        mats.push_back({o.wo, D, D, t0 + kWo});
        mats.push_back({o.w1, F, D, t0 + kW1});
        mats.push_back({o.w2, D, F, t0 + kW2});
        vecs.push_back({o.bqkv, 3 * D, t0 + kBqkv, 0.02f, 0.f});
        vecs.push_back({o.bo, D, t0 + kBo, 0.02f, 0.f});
        vecs.push_back({o.b1, F, t0 + kB1, 0.02f, 0.f});
        vecs.push_back({o.b2, D, t0 + kB2, 0.02f, 0.f});
        vecs.push_back({o.ln1_g, D, t0 + kLn1G, 0.1f, 1.f});
        vecs.push_back({o.ln1_b, D, t0 + kLn1B, 0.1f, 0.f});
        vecs.push_back({o.ln2_g, D, t0 + kLn2G, 0.1f, 1.f});
        vecs.push_back({o.ln2_b, D, t0 + kLn2B, 0.1f, 0.f});
    }
    const uint32_t tp = 16u * static_cast<uint32_t>(lay.L);
    mats.push_back({lay.wp, D, D, tp + 0});
    vecs.push_back({lay.bp, D, tp + 1, 0.02f, 0.f});
    for (const Vec& v : vecs) {
        const uint64_t st = param_stream(d.seed, v.tensor);
        const float sc = param_scale(v.scale);
        float* dst = reinterpret_cast<float*>(base + v.off);
        for (uint64_t i = 0; i < v.n; ++i) dst[i] = v.shift + param_at(st, i, sc);
    }
    unsigned nthreads = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    for (unsigned t = 0; t < nthreads; ++t)
        pool.emplace_back([&, t] {
            for (const Mat& m : mats) {
                const uint64_t st = param_stream(d.seed, m.tensor);
                const float sc = param_scale(m.k == F ? sf : sd);
                const uint64_t total = m.n * m.k, chunk = (total + nthreads - 1) / nthreads;
                const uint64_t lo = std::min<uint64_t>(total, t * chunk), hi = std::min<uint64_t>(total, lo + chunk);
                for (uint64_t i = lo; i < hi; ++i) {
                    const uint64_t n = i / m.k, k = i % m.k;
                    *reinterpret_cast<uint16_t*>(base + m.off + bf16_tile_offset(n, k, m.k)) =
                        bf16_bits(param_at(st, i, sc));
                }
            }
        });
    for (auto& th : pool) th.join();
    const double T = static_cast<double>(d.batch) * lay.seq;
    blob.flops = lay.L * (2.0 * T * (3 * D * D + D * D + 2 * D * F) + 4.0 * T * lay.seq * D) + 2.0 * d.batch * D * D;
    blob.alg_bytes = static_cast<double>(blob.bytes) + T * D * 2 + d.batch * D * 4.0;
    blob.in_bytes = static_cast<uint64_t>(T) * D * 2;
    blob.out_bytes = static_cast<uint64_t>(d.batch) * D * 4;
}

}  // namespace

void ModelStore::add(int idx, const gfx_model_desc& desc) {
    if (idx < 0) throw std::invalid_argument("model index must be >= 0");
    if (desc.family == GFX_MODEL_BERT) {
        const int L = desc.n_layers, D = desc.dims[0], H = desc.dims[1], F = desc.dims[2], S = desc.dims[3];
        if (L < 1 || (D != 512 && D != 768 && D != 1024) || H * 64 != D || F % 256 || F < 256 || S % 128 || S < 128 ||
            S > 512 || desc.batch < 1)
            throw std::invalid_argument("bert: supported shapes are d = 512 / 768 / 1024 with d / 64 heads, seq 128 / "
                                        "256 / 384 / 512, ffn % 256 == 0");
        auto blob = std::make_unique<ModelBlob>();
        blob->desc = desc;
        blob->bert = bert_layout(L, D, H, F, S);
        blob->bytes = blob->bert.bytes;
        blob->pages = static_cast<uint32_t>((blob->bytes + kPageBytes - 1) / kPageBytes);
        if (blob->pages > GFX_MAX_PAGES) throw std::invalid_argument("model larger than the page-table limit");
        GFX_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&blob->host), blob->bytes, cudaHostAllocDefault));
        std::memset(blob->host, 0, blob->bytes);
        build_bert_blob(*blob);
        std::lock_guard<std::mutex> lk(mu_);
        if (static_cast<size_t>(idx) >= blobs_.size()) blobs_.resize(static_cast<size_t>(idx) + 1);
        blobs_[static_cast<size_t>(idx)] = std::move(blob);
        return;
    }
    if (desc.family != GFX_MODEL_MLP) throw std::invalid_argument("unsupported model family");
    if (desc.n_layers < 1 || desc.n_layers > GFX_MAX_LAYERS) throw std::invalid_argument("bad layer count");
    if (desc.batch != kBatch) throw std::invalid_argument("batch must be 32");
    for (int l = 0; l <= desc.n_layers; ++l)
        if (desc.dims[l] <= 0 || desc.dims[l] > kMaxDim) throw std::invalid_argument("bad layer width");
    for (int l = 0; l < desc.n_layers; ++l)
        if (desc.dims[l] % 32 != 0 || desc.dims[l + 1] % 4 != 0)
            throw std::invalid_argument("layer inputs must be multiples of 32, outputs of 4");

    auto blob = std::make_unique<ModelBlob>();
    blob->desc = desc;
    mlp_layout(desc, blob->w_off, blob->b_off, blob->bytes);
    blob->pages = static_cast<uint32_t>((blob->bytes + kPageBytes - 1) / kPageBytes);
    if (blob->pages > GFX_MAX_PAGES) throw std::invalid_argument("model larger than the page-table limit");
    GFX_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&blob->host), blob->bytes, cudaHostAllocDefault));
    std::memset(blob->host, 0, blob->bytes);

    // Parameters, generated in parallel on the host.
    struct Job {
        float* dst;
        uint64_t n;        // values
        uint64_t K;        // > 0: weight matrix [n / K x K] written as swizzled tiles
        uint64_t stream;
        float scaled;
    };
    std::vector<Job> jobs;
    double flops = 0, wbytes = 0;
    for (int l = 0; l < desc.n_layers; ++l) {
        const uint64_t K = static_cast<uint64_t>(desc.dims[l]);
        const uint64_t N = static_cast<uint64_t>(desc.dims[l + 1]);
        const float scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(K)));
        char* base = reinterpret_cast<char*>(blob->host);
        jobs.push_back({reinterpret_cast<float*>(base + blob->w_off[l]), K * N, K,
                        param_stream(desc.seed, static_cast<uint32_t>(2 * l)), param_scale(scale)});
        jobs.push_back({reinterpret_cast<float*>(base + blob->b_off[l]), N, 0,
                        param_stream(desc.seed, static_cast<uint32_t>(2 * l + 1)), param_scale(scale)});
        flops += 2.0 * kBatch * static_cast<double>(K) * static_cast<double>(N);
        wbytes += 4.0 * static_cast<double>(K * N + N) + 4.0 * kBatch * static_cast<double>(K + N);
    }
    blob->flops = flops;
    blob->alg_bytes = wbytes;
    blob->in_bytes = static_cast<uint64_t>(kBatch) * desc.dims[0] * 4;
    blob->out_bytes = static_cast<uint64_t>(2) * kBatch * desc.dims[desc.n_layers] * 4;
    unsigned nthreads = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < nthreads; ++t)
        pool.emplace_back([&, t] {
            for (const Job& j : jobs) {
                const uint64_t chunk = (j.n + nthreads - 1) / nthreads;
                const uint64_t lo = std::min<uint64_t>(j.n, t * chunk), hi = std::min<uint64_t>(j.n, lo + chunk);
                if (j.K == 0) {
                    for (uint64_t i = lo; i < hi; ++i) j.dst[i] = param_at(j.stream, i, j.scaled);
                } else {
                    char* dst = reinterpret_cast<char*>(j.dst);
                    for (uint64_t i = lo; i < hi; ++i)  // logical W[n][k] = stream[n*K + k]
                        *reinterpret_cast<float*>(dst + wtile_offset(i / j.K, i % j.K, j.K)) =
                            param_at(j.stream, i, j.scaled);
                }
            }
        });
    for (auto& th : pool) th.join();

    std::lock_guard<std::mutex> lk(mu_);
    if (static_cast<size_t>(idx) >= blobs_.size()) blobs_.resize(static_cast<size_t>(idx) + 1);
    blobs_[static_cast<size_t>(idx)] = std::move(blob);
}

const ModelBlob& ModelStore::at(int idx) const {
    std::lock_guard<std::mutex> lk(mu_);
    if (idx < 0 || static_cast<size_t>(idx) >= blobs_.size() || !blobs_[static_cast<size_t>(idx)])
        throw std::invalid_argument("model " + std::to_string(idx) + " is not registered");
    return *blobs_[static_cast<size_t>(idx)];
}

bool ModelStore::has(int idx) const {
    std::lock_guard<std::mutex> lk(mu_);
    return idx >= 0 && static_cast<size_t>(idx) < blobs_.size() && blobs_[static_cast<size_t>(idx)];
}

void ModelStore::clear() {
    std::lock_guard<std::mutex> lk(mu_);
    blobs_.clear();
}

// ------------------------------------------------------------- timer

cudaEvent_t KernelTimer::next() {
    if (used == ev.size()) {
        cudaEvent_t e;
        GFX_CUDA(cudaEventCreate(&e));
        ev.push_back(e);
    }
    return ev[used++];
}

// ------------------------------------------------------------- manager

// Managers per device in this process. K1 chains its launches by PDL only on a
// device one manager owns: two managers' persistent forwards on one device
// (the emulated fleets, or another process's manager: mark_device_shared)
// could each hold part of the SMs while waiting for their own missing CTAs,
// so a shared device keeps the cooperative launch.
namespace {
std::mutex g_dev_mu;
std::map<int, int> g_dev_managers;
std::map<int, bool> g_dev_shared;  // other processes run managers on the device
}  // namespace

void mark_device_shared(int dev) {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    g_dev_shared[dev] = true;
}

GpuManager::GpuManager(int device, uint64_t capacity_bytes, int manager_id) : device_(device), id_(manager_id) {
    {
        std::lock_guard<std::mutex> lk(g_dev_mu);
        ++g_dev_managers[device];
    }
    if (capacity_bytes == 0 || capacity_bytes % kPageBytes != 0)
        throw std::invalid_argument("arena capacity must be a positive multiple of 2 MiB");
    activate();
    npages_ = static_cast<uint32_t>(capacity_bytes / kPageBytes);
    GFX_CUDA(cudaMalloc(&arena_, capacity_bytes));
    for (uint32_t p = 0; p < npages_; ++p) free_.insert(p);
    GFX_CUDA(cudaStreamCreateWithFlags(&compute_, cudaStreamNonBlocking));
    GFX_CUDA(cudaStreamCreateWithFlags(&copy_, cudaStreamNonBlocking));
    sm_count_ = device_sm_count(device_);
    GFX_CUDA(cudaMalloc(&fwd_act_, sizeof(unsigned long long) * 2 * kMlpActWords));
    GFX_CUDA(cudaMemset(fwd_act_, 0, sizeof(unsigned long long) * 2 * kMlpActWords));
    GFX_CUDA(cudaMalloc(&fwd_claim_, sizeof(unsigned) * 4));
    GFX_CUDA(cudaMemset(fwd_claim_, 0, sizeof(unsigned) * 4));
    GFX_CUDA(cudaDeviceSynchronize());
}

GpuManager::~GpuManager() {
    {
        std::lock_guard<std::mutex> lk(g_dev_mu);
        --g_dev_managers[device_];
    }
    cudaSetDevice(device_);
    cudaStreamSynchronize(compute_);
    cudaStreamSynchronize(copy_);
    for (Slot& s : slots_) {
        if (s.loaded) cudaEventDestroy(s.loaded);
        if (s.last_use) cudaEventDestroy(s.last_use);
    }
    cudaFree(arena_);
    cudaFree(fwd_act_);
    cudaFree(fwd_claim_);
    bert_ws_.release();
    if (bert_lengths_) cudaFree(bert_lengths_);
    bert_lengths_ = nullptr;
    bert_lengths_cap_ = 0;
    cudaStreamDestroy(compute_);
    cudaStreamDestroy(copy_);
}

void GpuManager::activate() const { GFX_CUDA(cudaSetDevice(device_)); }

GpuManager::Slot& GpuManager::slot(int model) {
    if (model < 0) throw std::invalid_argument("negative model index");
    if (static_cast<size_t>(model) >= slots_.size()) slots_.resize(static_cast<size_t>(model) + 1);
    Slot& s = slots_[static_cast<size_t>(model)];
    if (!s.loaded) {
        GFX_CUDA(cudaEventCreateWithFlags(&s.loaded, cudaEventDisableTiming));
        GFX_CUDA(cudaEventCreateWithFlags(&s.last_use, cudaEventDisableTiming));
    }
    return s;
}

bool GpuManager::resident(int model) const {
    return model >= 0 && static_cast<size_t>(model) < slots_.size() && slots_[static_cast<size_t>(model)].live;
}

cudaEvent_t GpuManager::loaded_event(int model) const {
    if (!resident(model)) throw std::logic_error("loaded_event of non-resident model");
    return slots_[static_cast<size_t>(model)].loaded;
}

const std::vector<uint32_t>& GpuManager::pages_of(int model) const {
    if (!resident(model)) throw std::logic_error("pages_of non-resident model");
    return slots_[static_cast<size_t>(model)].pages;
}

void GpuManager::add_reader(int model, cudaEvent_t e) {
    // One entry per reader event: a re-fetch by the same manager re-records the
    // same event, and waiting on its latest record covers every earlier one.
    std::vector<cudaEvent_t>& r = slot(model).readers;
    if (std::find(r.begin(), r.end(), e) == r.end()) r.push_back(e);
}

// ClusterState::evict_one (proj/src/cluster.cpp:117-129) on device: the pages
// return to the pool at once (host bookkeeping), and the copy stream — the
// only writer of arena pages — is ordered after every pending reader of them
// (the model's last inference and any peer fetch out of them), so a later
// load can never overwrite weights still in use.
void GpuManager::evict(int model) {
    Slot& s = slot(model);
    if (!s.live) throw std::logic_error("evict of non-resident model " + std::to_string(model));
    activate();
    GFX_CUDA(cudaStreamWaitEvent(copy_, s.last_use, 0));
    for (cudaEvent_t r : s.readers) GFX_CUDA(cudaStreamWaitEvent(copy_, r, 0));
    s.readers.clear();
    for (uint32_t p : s.pages) free_.insert(p);
    s.pages.clear();
    s.live = false;
}

// Lowest free pages first (deterministic: peers replay it as a shadow, see
// gfx_capi.cu RemoteArena).
GpuManager::Slot& GpuManager::allocate(int model, const ModelBlob& blob) {
    Slot& s = slot(model);
    if (s.live) throw std::logic_error("load of resident model " + std::to_string(model));
    if (free_.size() < blob.pages)
        throw std::logic_error("arena out of pages: the control plane's capacity model and the arena disagree");
    s.pages.clear();
    for (uint32_t i = 0; i < blob.pages; ++i) {
        s.pages.push_back(*free_.begin());
        free_.erase(free_.begin());
    }
    return s;
}

namespace {
using StreamWaitValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using StreamWriteValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
template <typename Fn>
Fn driver_fn(const char* name) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    GFX_CUDA(cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || p == nullptr) throw CudaError(std::string(name) + " entry point unavailable");
    return reinterpret_cast<Fn>(p);
}
}  // namespace

void GpuManager::copy_wait_geq(const uint32_t* addr, uint32_t value) {
    static StreamWaitValue32Fn fn = driver_fn<StreamWaitValue32Fn>("cuStreamWaitValue32");
    activate();
    if (fn(copy_, reinterpret_cast<CUdeviceptr>(addr), value, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
        throw CudaError("cuStreamWaitValue32 failed");
}

void GpuManager::copy_write(uint32_t* addr, uint32_t value) {
    static StreamWriteValue32Fn fn = driver_fn<StreamWriteValue32Fn>("cuStreamWriteValue32");
    activate();
    // Default flags: the write is ordered after (and fenced behind) the prior copies of the stream.
    if (fn(copy_, reinterpret_cast<CUdeviceptr>(addr), value, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
        throw CudaError("cuStreamWriteValue32 failed");
}

// NVLink fetch from another process's arena (IPC-mapped): the same page-run
// copies as the in-process peer path, ordered by a device-side wait on the
// holder's load counter instead of an event.
uint64_t GpuManager::load_remote(int model, const char* src_arena, const std::vector<uint32_t>& sp,
                                 const uint32_t* wait_addr, uint32_t wait_value) {
    const ModelBlob& blob = ModelStore::get().at(model);
    if (sp.size() != blob.pages) throw std::logic_error("remote page table does not match the model");
    activate();
    Slot& s = allocate(model, blob);
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    copy_wait_geq(wait_addr, wait_value);  // outside the timed copy: the holder's load may still run
    if (p2p_timer) {
        t0 = p2p_timer->next();
        t1 = p2p_timer->next();
        GFX_CUDA(cudaEventRecord(t0, copy_));
    }
    uint32_t i = 0;
    while (i < blob.pages) {
        uint32_t j = i + 1;
        while (j < blob.pages && s.pages[j] == s.pages[j - 1] + 1 && sp[j] == sp[j - 1] + 1) ++j;
        const uint64_t off = static_cast<uint64_t>(i) * kPageBytes;
        const uint64_t len = std::min<uint64_t>(static_cast<uint64_t>(j - i) * kPageBytes, blob.bytes - off);
        GFX_CUDA(cudaMemcpyAsync(arena_ + static_cast<uint64_t>(s.pages[i]) * kPageBytes,
                                 src_arena + static_cast<uint64_t>(sp[i]) * kPageBytes, len, cudaMemcpyDeviceToDevice,
                                 copy_));
        i = j;
    }
    if (p2p_timer) GFX_CUDA(cudaEventRecord(t1, copy_));
    GFX_CUDA(cudaEventRecord(s.loaded, copy_));
    s.live = true;
    GFX_CUDA(cudaStreamWaitEvent(compute_, s.loaded, 0));
    return blob.bytes;
}

// The load that replaces profile.load_time_us (proj/src/cluster.cpp:163-167).
uint64_t GpuManager::load(int model, GpuManager* src) {
    const ModelBlob& blob = ModelStore::get().at(model);
    activate();
    Slot& s = allocate(model, blob);
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    if (src) GFX_CUDA(cudaStreamWaitEvent(copy_, src->loaded_event(model), 0));  // holder's copy complete
    KernelTimer* timer = src ? p2p_timer : load_timer;
    if (timer) {
        t0 = timer->next();
        t1 = timer->next();
        GFX_CUDA(cudaEventRecord(t0, copy_));
    }
    if (src == nullptr) {
        // Pinned-host H2D, one copy per run of contiguous destination pages.
        const char* host = reinterpret_cast<const char*>(blob.host);
        uint32_t i = 0;
        while (i < blob.pages) {
            uint32_t j = i + 1;
            while (j < blob.pages && s.pages[j] == s.pages[j - 1] + 1) ++j;
            const uint64_t off = static_cast<uint64_t>(i) * kPageBytes;
            const uint64_t len = std::min<uint64_t>(static_cast<uint64_t>(j - i) * kPageBytes, blob.bytes - off);
            GFX_CUDA(cudaMemcpyAsync(arena_ + static_cast<uint64_t>(s.pages[i]) * kPageBytes, host + off, len,
                                     cudaMemcpyHostToDevice, copy_));
            i = j;
        }
    } else {
        // NVLink peer fetch from the holder's arena (false miss): wait until
        // the holder's copy is complete, copy runs contiguous on both sides,
        // and register the fetch as a reader of the holder's pages.
        const std::vector<uint32_t>& sp = src->pages_of(model);
        uint32_t i = 0;
        while (i < blob.pages) {
            uint32_t j = i + 1;
            while (j < blob.pages && s.pages[j] == s.pages[j - 1] + 1 && sp[j] == sp[j - 1] + 1) ++j;
            const uint64_t off = static_cast<uint64_t>(i) * kPageBytes;
            const uint64_t len = std::min<uint64_t>(static_cast<uint64_t>(j - i) * kPageBytes, blob.bytes - off);
            GFX_CUDA(cudaMemcpyPeerAsync(arena_ + static_cast<uint64_t>(s.pages[i]) * kPageBytes, device_,
                                         src->arena() + static_cast<uint64_t>(sp[i]) * kPageBytes, src->device(),
                                         len, copy_));
            i = j;
        }
    }
    if (timer) GFX_CUDA(cudaEventRecord(t1, copy_));
    GFX_CUDA(cudaEventRecord(s.loaded, copy_));
    if (src) src->add_reader(model, s.loaded);
    s.live = true;
    // Inference of this model on the compute stream starts after the load.
    GFX_CUDA(cudaStreamWaitEvent(compute_, s.loaded, 0));
    return blob.bytes;
}

void GpuManager::build_page_table(const Slot& s, PageTable& pt) const {
    pt.n = static_cast<uint32_t>(s.pages.size());
    for (size_t i = 0; i < s.pages.size(); ++i) pt.page[i] = s.pages[i];
}

// The batched inference that replaces profile.infer_time_us
// (proj/src/cluster.cpp:161,167): MLP -> one K1 launch (the whole forward),
// BERT -> the K2-K4 chain, on the compute stream.
void GpuManager::infer(int model, const void* in_v, void* out_v, void* debug_hidden, const int32_t* lengths) {
    const ModelBlob& blob = ModelStore::get().at(model);
    Slot& s = slot(model);
    if (!s.live) throw std::logic_error("inference of non-resident model " + std::to_string(model));
    if (lengths && blob.desc.family != GFX_MODEL_BERT) throw std::invalid_argument("sequence lengths: BERT models only");
    activate();
    if (blob.desc.family == GFX_MODEL_BERT) {
        PageTable pt;
        build_page_table(s, pt);
        const int* dlen = nullptr;
        if (lengths) {
            const int batch = blob.desc.batch, seq = blob.bert.seq;
            for (int b = 0; b < batch; ++b)
                if (lengths[b] < 1 || lengths[b] > seq)
                    throw std::invalid_argument("sequence length " + std::to_string(lengths[b]) + " outside 1.." +
                                                std::to_string(seq));
            if (bert_lengths_cap_ < batch) {
                if (bert_lengths_) GFX_CUDA(cudaFree(bert_lengths_));
                GFX_CUDA(cudaMalloc(&bert_lengths_, sizeof(int) * static_cast<size_t>(batch)));
                bert_lengths_cap_ = batch;
            }
            // Ordered on the compute stream before the forward; the host array may be reused on return
            // (pageable source: the copy is staged before cudaMemcpyAsync returns).
            GFX_CUDA(cudaMemcpyAsync(bert_lengths_, lengths, sizeof(int) * static_cast<size_t>(batch),
                                     cudaMemcpyHostToDevice, compute_));
            dlen = bert_lengths_;
        }
        if (layer_timer) GFX_CUDA(cudaEventRecord(layer_timer->next(), compute_));
        kernel_launches += bert_forward(arena_, pt, blob.bert, blob.desc.batch,
                                        static_cast<const __nv_bfloat16*>(in_v), static_cast<float*>(out_v), bert_ws_,
                                        compute_, static_cast<__nv_bfloat16*>(debug_hidden), dlen);
        if (layer_timer) GFX_CUDA(cudaEventRecord(layer_timer->next(), compute_));
        GFX_CUDA(cudaEventRecord(s.last_use, compute_));
        return;
    }
    MlpFwdArgs f{};
    f.arena = arena_;
    build_page_table(s, f.pt);
    f.in = static_cast<const float*>(in_v);
    f.L = blob.desc.n_layers;
    f.logits = static_cast<float*>(out_v);
    f.probs = f.logits + static_cast<size_t>(kBatch) * blob.desc.dims[f.L];
    f.grid = sm_count_;
    {
        std::lock_guard<std::mutex> lk(g_dev_mu);
        f.pdl = g_dev_managers[device_] == 1 && !g_dev_shared[device_] ? 1 : 0;
    }
    uint32_t act = 0;
    for (int l = 0; l < f.L; ++l) {
        MlpFwdLayer& ly = f.layer[l];
        ly.w_off = blob.w_off[l];
        ly.b_off = blob.b_off[l];
        ly.K = blob.desc.dims[l];
        ly.N = blob.desc.dims[l + 1];
        ly.tiles = (ly.N + kWTileRows - 1) / kWTileRows;
        ly.nkt = ly.K / kWTileK;
        ly.act_off = act;
        act += static_cast<uint32_t>(ly.N) * kBatch;
    }
    // Launch parity p uses act bank p (zeroed by the previous launch) and
    // clears bank p^1 up to what the previous launch (parity p^1) dirtied.
    const unsigned p = fwd_epoch_ & 1u;
    f.act = fwd_act_ + p * kMlpActWords;
    f.act_clear = reinterpret_cast<uint4*>(fwd_act_ + (p ^ 1u) * kMlpActWords);
    f.clear_vec = act_dirty_[p ^ 1u] / 2;
    // Layer 0 dynamically split: this launch claims from counter epoch % 4 and zeroes
    // counter (epoch + 2) % 4 once its predecessor completed (then launch epoch - 2, its
    // last user, has completed too; launch epoch + 2 cannot start before every CTA of this
    // launch has left its SM).
    f.claim = fwd_claim_ + (fwd_epoch_ & 3u);
    f.claim_reset = fwd_claim_ + ((fwd_epoch_ + 2u) & 3u);
#ifdef GFX_K1_DEBUG
    // Four consecutive launches (8..11 of every 64) mark into their own tables,
    // then one report: the chain's per-launch CTA start / end spread (does the
    // next forward's CTAs start before this one's last CTA ends?) and launch 10's
    // phase table.
    constexpr size_t kDbgWords = 32 * 1024 + 96 * 8;
    static unsigned long long* dbg = nullptr;
    static unsigned launches = 0;
    if (!dbg) {
        GFX_CUDA(cudaMalloc(&dbg, sizeof(unsigned long long) * kDbgWords * 4));
        GFX_CUDA(cudaMemset(dbg, 0, sizeof(unsigned long long) * kDbgWords * 4));
    }
    const unsigned ph = ++launches % 64;
    f.dbg = ph >= 8 && ph <= 11 ? dbg + kDbgWords * (ph - 8) : nullptr;
#endif
    if (layer_timer) GFX_CUDA(cudaEventRecord(layer_timer->next(), compute_));
    launch_mlp_forward(f, compute_);
#ifdef GFX_K1_DEBUG
    if (ph == 11) {
        std::vector<unsigned long long> m(kDbgWords * 4);
        GFX_CUDA(cudaStreamSynchronize(compute_));
        GFX_CUDA(cudaMemcpy(m.data(), dbg, m.size() * 8, cudaMemcpyDeviceToHost));
        unsigned long long t0 = ~0ull;
        for (int c = 0; c < f.grid; ++c) t0 = std::min(t0, m[static_cast<size_t>(c) * 32]);
        std::fprintf(stderr, "[K1 chain, pdl %d] us from launch 8's first CTA: start min/max, end min/median/max\n", f.pdl);
        for (int k = 0; k < 4; ++k) {
            std::vector<double> st, en;
            for (int c = 0; c < f.grid; ++c) {
                st.push_back((m[kDbgWords * k + static_cast<size_t>(c) * 32] - t0) * 1e-3);
                en.push_back((m[kDbgWords * k + static_cast<size_t>(c) * 32 + 26] - t0) * 1e-3);
            }
            std::sort(st.begin(), st.end());
            std::sort(en.begin(), en.end());
            std::fprintf(stderr, "  launch %d: start %7.2f %7.2f  end %7.2f %7.2f %7.2f\n", 8 + k, st.front(), st.back(),
                         en.front(), en[en.size() / 2], en.back());
        }
        mlp_debug_report(dbg + kDbgWords * 2, f.grid, f.L, model, compute_);
        GFX_CUDA(cudaMemset(dbg, 0, sizeof(unsigned long long) * kDbgWords * 4));
    }
#endif
    act_dirty_[p ^ 1u] = 0;
    act_dirty_[p] = act;
    ++fwd_epoch_;
    ++kernel_launches;
    if (layer_timer) GFX_CUDA(cudaEventRecord(layer_timer->next(), compute_));
    GFX_CUDA(cudaEventRecord(s.last_use, compute_));
}

void GpuManager::bert_gemm(int model, int layer, int op, const void* x, const void* resid, void* y, int tokens) {
    const ModelBlob& blob = ModelStore::get().at(model);
    Slot& s = slot(model);
    if (!s.live) throw std::logic_error("gemm of non-resident model " + std::to_string(model));
    if (blob.desc.family != GFX_MODEL_BERT) throw std::invalid_argument("bert_gemm: BERT models only");
    activate();
    PageTable pt;
    build_page_table(s, pt);
    bert_gemm_op(arena_, pt, blob.bert, layer, op, static_cast<const __nv_bfloat16*>(x),
                 static_cast<const __nv_bfloat16*>(resid), static_cast<__nv_bfloat16*>(y), tokens, bert_ws_.gemm_pair,
                 compute_);
    GFX_CUDA(cudaEventRecord(s.last_use, compute_));
}

void GpuManager::reset() {
    activate();
    GFX_CUDA(cudaStreamSynchronize(copy_));
    GFX_CUDA(cudaStreamSynchronize(compute_));
    for (Slot& s : slots_) {
        for (uint32_t p : s.pages) free_.insert(p);
        s.pages.clear();
        s.readers.clear();
        s.live = false;
    }
    // A run may have ended mid-way (an exception after a launch): clear both banks.
    for (unsigned p = 0; p < 2; ++p)
        if (act_dirty_[p])
            GFX_CUDA(cudaMemset(fwd_act_ + p * kMlpActWords, 0, sizeof(unsigned long long) * act_dirty_[p]));
    act_dirty_[0] = act_dirty_[1] = 0;
    GFX_CUDA(cudaMemset(fwd_claim_, 0, sizeof(unsigned) * 4));
    fwd_epoch_ = 0;
    GFX_CUDA(cudaDeviceSynchronize());
}

}  // namespace gfx
