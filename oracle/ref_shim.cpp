// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI shim over the UNMODIFIED reference simulator (arXiv 2303.05601,
// /root/reference/proj). It is compiled in place against the reference's own
// headers and sources by oracle/Makefile into oracle/_ref/libgpufaas_ref.so;
// nothing from the reference is copied into this repository.
//
// Exposed to tests/ and bench.py (reference arm / cpu_baseline) through
// ctypes. The ABI (ref_sim_*) mirrors oracle/gpufaas_oracle.h (orc_sim_*) and
// the product's gfx_sim_* entry points so all three can be compared
// field-by-field with the same canonical digests (see oracle/gpufaas_oracle.h
// for the digest definitions).

#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "gpufaas/engine.hpp"                    // proj/include/gpufaas/engine.hpp:61-63 run_stream
#include "support/reference_scheduler.hpp"       // proj/tests/support/reference_scheduler.hpp:14

using namespace gpufaas;

namespace {

thread_local std::string g_err;

struct SimCfg {  // identical layout in oracle/gpufaas_oracle.h and include/gpufaas_b200.h
    int32_t gpu_count;
    int32_t policy;          // 0 lb, 1 lalb, 2 lalbo3
    int32_t o3_limit;
    int32_t working_set;
    int32_t per_minute_total;
    int32_t duration_minutes;
    int32_t use_synthetic_trace;
    int32_t syn_function_count;
    int32_t syn_minutes;
    int32_t syn_draws_per_minute;
    int32_t debug_checks;
    int32_t log_events;      // 0 none, 1 log, 2 log + caches
    int32_t use_reference_scheduler;  // plug tests/support ReferenceScheduler in
    int32_t pipeline;                 // product/oracle extension; the reference has no such mode
    double capacity_mb;
    double syn_zipf_exponent;
    uint64_t seed;
    uint64_t syn_seed;
};

struct Handle {
    SimResult result;
    std::vector<int> model_idx;  // per request, index into the catalog
    std::string log;
    std::string report_json;
    double run_ns = 0;
};

uint64_t fnv_bytes(uint64_t h, const void* p, size_t n) {
    const unsigned char* b = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) {
        h ^= b[i];
        h *= 1099511628211ULL;
    }
    return h;
}
template <typename T>
uint64_t fnv_val(uint64_t h, T v) { return fnv_bytes(h, &v, sizeof v); }
constexpr uint64_t kFnvBasis = 14695981039346656037ULL;

Policy to_policy(int p) {
    if (p == 0) return Policy::LB;
    if (p == 1) return Policy::LALB;
    return Policy::LALBO3;
}

SimConfig to_config(const SimCfg& c) {
    if (c.pipeline) throw std::runtime_error("the reference has no pipelined-GPU mode");
    SimConfig cfg;
    cfg.gpu_count = c.gpu_count;
    cfg.capacity_mb = c.capacity_mb;
    cfg.scheduler.policy = to_policy(c.policy);
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
    return cfg;
}

Handle* finish(const SimCfg& c, const SimConfig& cfg, const Catalog& cat, std::vector<Request> reqs) {
    auto* h = new Handle();
    h->model_idx.reserve(reqs.size());
    for (const Request& r : reqs) {
        int idx = -1;
        for (size_t i = 0; i < cat.profiles().size(); ++i)
            if (cat.profiles()[i].model_id == r.model_id) idx = static_cast<int>(i);
        h->model_idx.push_back(idx);
    }
    std::ostringstream log;
    EventLogger logger(log, c.log_events == 2);
    gpufaas::testing::ReferenceScheduler* ref = nullptr;
    if (c.use_reference_scheduler) ref = new gpufaas::testing::ReferenceScheduler(cfg.scheduler);
    auto t0 = std::chrono::steady_clock::now();
    h->result = run_stream(cfg, cat, std::move(reqs), c.log_events ? &logger : nullptr, ref);
    auto t1 = std::chrono::steady_clock::now();
    h->run_ns = std::chrono::duration<double, std::nano>(t1 - t0).count();
    delete ref;
    h->log = log.str();
    h->report_json = report_to_json(h->result.report).dump();
    return h;
}

}  // namespace

extern "C" {

const char* ref_sim_last_error() { return g_err.c_str(); }

// Mirrors run(cfg, catalog, trace, logger) (proj/src/engine.cpp:175-179).
void* ref_sim_run(const char* catalog_csv, const char* trace_csv, const SimCfg* c) {
    try {
        std::istringstream cin_(catalog_csv);
        Catalog cat = parse_catalog_csv(cin_, "catalog");
        SimConfig cfg = to_config(*c);
        TraceMatrix trace;
        if (trace_csv && !c->use_synthetic_trace) {
            std::istringstream tin(trace_csv);
            trace = parse_trace_csv(tin, "trace");
        } else {
            trace = make_synthetic_trace(cfg.synthetic);
        }
        std::vector<Request> reqs = synthesize_workload(trace, cfg.workload, cat);
        return finish(*c, cfg, cat, std::move(reqs));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

// Mirrors run_stream(cfg, catalog, requests) (proj/src/engine.cpp:100-173).
void* ref_sim_run_stream(const char* catalog_csv, const SimCfg* c, int n, const int32_t* model_idx,
                         const int64_t* arrival_us) {
    try {
        std::istringstream cin_(catalog_csv);
        Catalog cat = parse_catalog_csv(cin_, "catalog");
        SimConfig cfg = to_config(*c);
        std::vector<Request> reqs(static_cast<size_t>(n));
        for (int i = 0; i < n; ++i) {
            reqs[i].request_id = i;
            reqs[i].model_id = cat.profiles().at(static_cast<size_t>(model_idx[i])).model_id;
            reqs[i].arrival_us = arrival_us[i];
        }
        return finish(*c, cfg, cat, std::move(reqs));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

int64_t ref_sim_num_decisions(void* hp) { return static_cast<Handle*>(hp)->result.decisions.size(); }
int64_t ref_sim_num_requests(void* hp) { return static_cast<Handle*>(hp)->result.requests.size(); }
double ref_sim_run_ns(void* hp) { return static_cast<Handle*>(hp)->run_ns; }

// ints: [kind, request_id, gpu_id, from_local, false_miss, skip_count, n_evicted] x n
// times: [completion_us, load_us, infer_us] x n
void ref_sim_get_decisions(void* hp, int32_t* ints, int64_t* times) {
    const auto& ds = static_cast<Handle*>(hp)->result.decisions;
    for (size_t i = 0; i < ds.size(); ++i) {
        const Decision& d = ds[i];
        int32_t* o = ints + 7 * i;
        o[0] = static_cast<int32_t>(d.kind);
        o[1] = d.request_id;
        o[2] = d.gpu_id;
        o[3] = d.from_local_queue;
        o[4] = d.false_miss;
        o[5] = d.skip_count;
        o[6] = static_cast<int32_t>(d.evicted.size());
        times[3 * i + 0] = d.completion_us;
        times[3 * i + 1] = d.load_us;
        times[3 * i + 2] = d.infer_us;
    }
}

void ref_sim_get_requests(void* hp, int32_t* model_idx, int64_t* arrival, int64_t* dispatched,
                          int64_t* completed, int32_t* skip) {
    auto* h = static_cast<Handle*>(hp);
    const auto& rs = h->result.requests;
    for (size_t i = 0; i < rs.size(); ++i) {
        model_idx[i] = h->model_idx[i];
        arrival[i] = rs[i].arrival_us;
        dispatched[i] = rs[i].dispatched_at_us;
        completed[i] = rs[i].completed_at_us;
        skip[i] = rs[i].skip_count;
    }
}

// Canonical digests (definition: oracle/gpufaas_oracle.h).
uint64_t ref_sim_decision_digest(void* hp) {
    uint64_t h = kFnvBasis;
    for (const Decision& d : static_cast<Handle*>(hp)->result.decisions) {
        h = fnv_val<int32_t>(h, static_cast<int32_t>(d.kind));
        h = fnv_val<int32_t>(h, d.request_id);
        h = fnv_val<int32_t>(h, d.gpu_id);
        h = fnv_val<int32_t>(h, d.from_local_queue);
        h = fnv_val<int32_t>(h, d.false_miss);
        h = fnv_val<int32_t>(h, d.skip_count);
        h = fnv_val<int64_t>(h, d.completion_us);
        h = fnv_val<int64_t>(h, d.load_us);
        h = fnv_val<int64_t>(h, d.infer_us);
        h = fnv_val<int32_t>(h, static_cast<int32_t>(d.evicted.size()));
        for (const std::string& s : d.evicted) h = fnv_bytes(h, s.c_str(), s.size() + 1);
    }
    return h;
}

uint64_t ref_sim_request_digest(void* hp) {
    uint64_t h = kFnvBasis;
    for (const Request& r : static_cast<Handle*>(hp)->result.requests) {
        h = fnv_val<int64_t>(h, r.dispatched_at_us);
        h = fnv_val<int64_t>(h, r.completed_at_us);
        h = fnv_val<int32_t>(h, r.skip_count);
    }
    return h;
}

uint64_t ref_sim_log_digest(void* hp) {
    const std::string& s = static_cast<Handle*>(hp)->log;
    return fnv_bytes(kFnvBasis, s.data(), s.size());
}

int64_t ref_sim_log_size(void* hp) { return static_cast<Handle*>(hp)->log.size(); }
const char* ref_sim_log(void* hp) { return static_cast<Handle*>(hp)->log.c_str(); }
const char* ref_sim_report_json(void* hp) { return static_cast<Handle*>(hp)->report_json.c_str(); }
void ref_sim_free(void* hp) { delete static_cast<Handle*>(hp); }

// Reference synthetic trace as CSV (proj/src/trace.cpp:156-192, :113 trace_to_csv)
// and catalog round-trip (proj/src/catalog.cpp:113-125). Returned strings live
// until the next call on the same thread.
const char* ref_synthetic_trace_csv(int function_count, int minutes, int draws, double zipf,
                                    uint64_t seed) {
    static thread_local std::string s;
    SyntheticTraceParams p;
    p.function_count = function_count;
    p.minutes = minutes;
    p.draws_per_minute = draws;
    p.zipf_exponent = zipf;
    p.seed = seed;
    s = trace_to_csv(make_synthetic_trace(p));
    return s.c_str();
}

}  // extern "C"
