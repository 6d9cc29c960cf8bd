// gfx_sim_*: C-ABI view of the product control plane (catalog -> workload ->
// run_stream) with the same struct layout and canonical digests as the
// oracle (oracle/gpufaas_oracle.h) and the reference shim, so the parity
// tests drive all three identically. Declared in include/gpufaas_b200.h.
#include <chrono>
#include <cstdint>
#include <deque>
#include <exception>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "gpufaas/engine.hpp"
#include "gpufaas_b200.h"

using namespace gpufaas;

namespace {

thread_local std::string g_err;

struct SimHandle {
    SimResult result;
    std::vector<int> model_idx;
    std::string log;
    std::string report_json;
    double run_ns = 0;
};

constexpr std::uint64_t kBasis = 14695981039346656037ULL;
std::uint64_t fnv(std::uint64_t h, const void* p, std::size_t n) {
    const auto* b = static_cast<const unsigned char*>(p);
    for (std::size_t i = 0; i < n; ++i) {
        h ^= b[i];
        h *= 1099511628211ULL;
    }
    return h;
}
template <typename T>
std::uint64_t fnv_v(std::uint64_t h, T v) { return fnv(h, &v, sizeof v); }

}  // namespace

namespace gpufaas::capi {

SimConfig to_sim_config(const gfx_sim_config& c) {
    SimConfig cfg;
    cfg.gpu_count = c.gpu_count;
    cfg.capacity_mb = c.capacity_mb;
    if (c.policy < 0 || c.policy > 2) throw std::invalid_argument("policy must be 0 (lb), 1 (lalb) or 2 (lalbo3)");
    cfg.scheduler.policy = c.policy == 0 ? Policy::LB : c.policy == 1 ? Policy::LALB : Policy::LALBO3;
    cfg.scheduler.o3_limit = c.o3_limit;
    cfg.workload.working_set_size = c.working_set;
    cfg.workload.per_minute_total = c.per_minute_total;
    cfg.workload.duration_minutes = c.duration_minutes;
    cfg.workload.seed = c.seed;
    cfg.use_synthetic_trace = c.use_synthetic_trace != 0;
    cfg.synthetic.function_count = c.syn_function_count;
    cfg.synthetic.minutes = c.syn_minutes;
    cfg.synthetic.draws_per_minute = c.syn_draws_per_minute;
    cfg.synthetic.zipf_exponent = c.syn_zipf_exponent;
    cfg.synthetic.seed = c.syn_seed;
    cfg.debug_checks = c.debug_checks != 0;
    cfg.scheduler.pipeline = c.pipeline != 0;
    return cfg;
}

std::vector<Request> make_requests(const gfx_sim_config& c, const Catalog& cat, const char* trace_csv) {
    const SimConfig cfg = to_sim_config(c);
    TraceMatrix trace;
    if (trace_csv && !c.use_synthetic_trace) {
        std::istringstream in(trace_csv);
        trace = parse_trace_csv(in, "trace");
    } else {
        trace = make_synthetic_trace(cfg.synthetic);
    }
    return synthesize_workload(trace, cfg.workload, cat);
}

}  // namespace gpufaas::capi

extern "C" {

const char* gfx_sim_last_error(void) { return g_err.c_str(); }

static void* finish(const gfx_sim_config& c, const Catalog& cat, std::vector<Request> reqs) {
    auto* h = new SimHandle();
    h->model_idx.reserve(reqs.size());
    for (const Request& r : reqs) h->model_idx.push_back(cat.index_of(r.model_id));
    std::ostringstream log;
    EventLogger logger(log, c.log_events == 2);
    const SimConfig cfg = gpufaas::capi::to_sim_config(c);
    const auto t0 = std::chrono::steady_clock::now();
    h->result = run_stream(cfg, cat, std::move(reqs), c.log_events ? &logger : nullptr);
    h->run_ns = std::chrono::duration<double, std::nano>(std::chrono::steady_clock::now() - t0).count();
    h->log = log.str();
    h->report_json = report_to_json(h->result.report).dump();
    return h;
}

void* gfx_sim_run(const char* catalog_csv, const char* trace_csv, const gfx_sim_config* c) {
    try {
        std::istringstream in(catalog_csv);
        const Catalog cat = parse_catalog_csv(in, "catalog");
        return finish(*c, cat, gpufaas::capi::make_requests(*c, cat, trace_csv));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void* gfx_sim_run_stream(const char* catalog_csv, const gfx_sim_config* c, int n, const int32_t* model_idx,
                         const int64_t* arrival_us) {
    try {
        std::istringstream in(catalog_csv);
        const Catalog cat = parse_catalog_csv(in, "catalog");
        std::vector<Request> reqs(static_cast<std::size_t>(n));
        for (int i = 0; i < n; ++i) {
            reqs[i].request_id = i;
            reqs[i].model_id = cat.profiles().at(static_cast<std::size_t>(model_idx[i])).model_id;
            reqs[i].arrival_us = arrival_us[i];
        }
        return finish(*c, cat, std::move(reqs));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

// Live closed-loop mode on a timed stand-in device: each dispatched task
// "runs" for its catalog duration / time_scale of real time. Exercises
// run_live()'s real-time loop and live ClusterState without a GPU.
void* gfx_sim_run_live_timed(const char* catalog_csv, const char* trace_csv, const gfx_sim_config* c,
                             double time_scale, double ema_alpha) {
    // Per GPU a FIFO of tasks; a load starts when the copy engine is free, an
    // inference when its load and the previous inference are done.
    struct Timed : ExecutionListener, LiveExecutor {
        using clock = std::chrono::steady_clock;
        struct Task {
            clock::time_point due;
            SimTime load, infer;
        };
        const Catalog* cat = nullptr;
        std::vector<std::deque<Task>> q;
        std::vector<clock::time_point> copy_free, compute_free;
        double scale = 1;
        void on_begin_execution(int gpu, const Request& r, int, bool hit, const std::vector<int>&, int, SimTime,
                                SimTime) override {
            const ModelProfile& p = cat->lookup(r.model_id);
            const std::size_t g = static_cast<std::size_t>(gpu);
            Task t{};
            t.load = hit ? 0 : std::max<SimTime>(1, std::llround(p.load_time_us / scale));
            t.infer = std::max<SimTime>(1, std::llround(p.infer_time_us / scale));
            clock::time_point ready = clock::now();
            if (!hit) {
                ready = std::max(ready, copy_free[g]) + std::chrono::microseconds(t.load);
                copy_free[g] = ready;
            }
            t.due = std::max(ready, compute_free[g]) + std::chrono::microseconds(t.infer);
            compute_free[g] = t.due;
            q[g].push_back(t);
        }
        void on_complete(int, int, SimTime) override {}
        bool done(int gpu) override {
            const auto& d = q[static_cast<std::size_t>(gpu)];
            return d.empty() || clock::now() >= d.front().due;
        }
        void retire(int gpu) override {
            auto& d = q[static_cast<std::size_t>(gpu)];
            if (!d.empty()) d.pop_front();
        }
        bool measured(int gpu, SimTime* l, SimTime* i) override {
            const auto& d = q[static_cast<std::size_t>(gpu)];
            if (d.empty()) return false;
            *l = d.front().load;
            *i = d.front().infer;
            return true;
        }
    };
    try {
        std::istringstream in(catalog_csv);
        const Catalog cat = parse_catalog_csv(in, "catalog");
        std::vector<Request> reqs = gpufaas::capi::make_requests(*c, cat, trace_csv);
        auto* h = new SimHandle();
        for (const Request& r : reqs) h->model_idx.push_back(cat.index_of(r.model_id));
        Timed dev;
        const std::size_t G = static_cast<std::size_t>(std::max(c->gpu_count, 1));
        dev.cat = &cat;
        dev.q.assign(G, {});
        dev.copy_free.assign(G, std::chrono::steady_clock::now());
        dev.compute_free.assign(G, std::chrono::steady_clock::now());
        dev.scale = time_scale;
        const auto t0 = std::chrono::steady_clock::now();
        h->result = run_live(gpufaas::capi::to_sim_config(*c), cat, std::move(reqs), time_scale, &dev, dev, nullptr,
                             ema_alpha);
        h->run_ns = std::chrono::duration<double, std::nano>(std::chrono::steady_clock::now() - t0).count();
        h->report_json = report_to_json(h->result.report).dump();
        return h;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

int gfx_sim_azure_convert(const char* in_path, const char* out_path, int top_k, int max_minutes,
                          int64_t* rows_read, int64_t* rows_kept) {
    try {
        std::ifstream in(in_path);
        if (!in) throw std::runtime_error(std::string("cannot open '") + in_path + "'");
        AzureIngest opts;
        opts.top_k = top_k;
        opts.max_minutes = max_minutes;
        const TraceMatrix t = parse_azure_trace_csv(in, in_path, opts);
        save_trace(t, out_path);
        if (rows_read) *rows_read = opts.rows_read;
        if (rows_kept) *rows_kept = static_cast<int64_t>(t.functions.size());
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

int64_t gfx_sim_num_decisions(void* hp) { return static_cast<SimHandle*>(hp)->result.decisions.size(); }
int64_t gfx_sim_num_requests(void* hp) { return static_cast<SimHandle*>(hp)->result.requests.size(); }
double gfx_sim_run_ns(void* hp) { return static_cast<SimHandle*>(hp)->run_ns; }

void gfx_sim_get_decisions(void* hp, int32_t* ints, int64_t* times) {
    const auto& ds = static_cast<SimHandle*>(hp)->result.decisions;
    for (std::size_t i = 0; i < ds.size(); ++i) {
        const Decision& d = ds[i];
        int32_t* o = ints + 7 * i;
        o[0] = static_cast<int32_t>(d.kind);
        o[1] = d.request_id;
        o[2] = d.gpu_id;
        o[3] = d.from_local_queue;
        o[4] = d.false_miss;
        o[5] = d.skip_count;
        o[6] = static_cast<int32_t>(d.evicted.size());
        times[3 * i] = d.completion_us;
        times[3 * i + 1] = d.load_us;
        times[3 * i + 2] = d.infer_us;
    }
}

void gfx_sim_get_requests(void* hp, int32_t* model_idx, int64_t* arrival, int64_t* dispatched,
                          int64_t* completed, int32_t* skip) {
    auto* h = static_cast<SimHandle*>(hp);
    const auto& rs = h->result.requests;
    for (std::size_t i = 0; i < rs.size(); ++i) {
        model_idx[i] = h->model_idx[i];
        arrival[i] = rs[i].arrival_us;
        dispatched[i] = rs[i].dispatched_at_us;
        completed[i] = rs[i].completed_at_us;
        skip[i] = rs[i].skip_count;
    }
}

uint64_t gfx_sim_decision_digest(void* hp) {
    std::uint64_t h = kBasis;
    for (const Decision& d : static_cast<SimHandle*>(hp)->result.decisions) {
        h = fnv_v<int32_t>(h, static_cast<int32_t>(d.kind));
        h = fnv_v<int32_t>(h, d.request_id);
        h = fnv_v<int32_t>(h, d.gpu_id);
        h = fnv_v<int32_t>(h, d.from_local_queue);
        h = fnv_v<int32_t>(h, d.false_miss);
        h = fnv_v<int32_t>(h, d.skip_count);
        h = fnv_v<int64_t>(h, d.completion_us);
        h = fnv_v<int64_t>(h, d.load_us);
        h = fnv_v<int64_t>(h, d.infer_us);
        h = fnv_v<int32_t>(h, static_cast<int32_t>(d.evicted.size()));
        for (const std::string& s : d.evicted) h = fnv(h, s.c_str(), s.size() + 1);
    }
    return h;
}

uint64_t gfx_sim_request_digest(void* hp) {
    std::uint64_t h = kBasis;
    for (const Request& r : static_cast<SimHandle*>(hp)->result.requests) {
        h = fnv_v<int64_t>(h, r.dispatched_at_us);
        h = fnv_v<int64_t>(h, r.completed_at_us);
        h = fnv_v<int32_t>(h, r.skip_count);
    }
    return h;
}

uint64_t gfx_sim_log_digest(void* hp) {
    const std::string& s = static_cast<SimHandle*>(hp)->log;
    return fnv(kBasis, s.data(), s.size());
}
int64_t gfx_sim_log_size(void* hp) { return static_cast<SimHandle*>(hp)->log.size(); }
const char* gfx_sim_log(void* hp) { return static_cast<SimHandle*>(hp)->log.c_str(); }
const char* gfx_sim_report_json(void* hp) { return static_cast<SimHandle*>(hp)->report_json.c_str(); }
void gfx_sim_free(void* hp) { delete static_cast<SimHandle*>(hp); }

}  // extern "C"
