#pragma once
// Shared by the C-ABI translation units: error-class mapping, the canonical
// decision digest (same definition as oracle/gpufaas_oracle.h) and percentiles.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "common.cuh"
#include "gpufaas/engine.hpp"
#include "gpufaas_b200.h"

namespace gpufaas::capi {
SimConfig to_sim_config(const gfx_sim_config& c);
std::vector<Request> make_requests(const gfx_sim_config& c, const Catalog& cat, const char* trace_csv);

// Runs f, mapping exceptions to the C-ABI status codes; the message goes to err.
template <typename F>
int guarded_call(std::string& err, F&& f) {
    try {
        f();
        return GFX_OK;
    } catch (const gfx::CudaError& e) {
        err = e.what();
        return GFX_ERR_CUDA;
    } catch (const std::logic_error& e) {
        err = e.what();
        // std::invalid_argument derives from logic_error but is a caller error.
        return dynamic_cast<const std::invalid_argument*>(&e) ? GFX_ERR_DOMAIN : GFX_ERR_INTERNAL;
    } catch (const std::exception& e) {
        err = e.what();
        return GFX_ERR_DOMAIN;
    }
}

// FNV-1a over every Decision field (canonical digest shared with the oracle and the reference shim).
inline uint64_t decision_digest(const std::vector<Decision>& decisions) {
    uint64_t h = 14695981039346656037ULL;
    auto fnv = [&](const void* p, size_t len) {
        const unsigned char* c = static_cast<const unsigned char*>(p);
        for (size_t i = 0; i < len; ++i) {
            h ^= c[i];
            h *= 1099511628211ULL;
        }
    };
    for (const Decision& d : decisions) {
        const int32_t a[6] = {static_cast<int32_t>(d.kind), d.request_id, d.gpu_id, d.from_local_queue,
                              d.false_miss, d.skip_count};
        fnv(a, sizeof a);
        fnv(&d.completion_us, 8);
        fnv(&d.load_us, 8);
        fnv(&d.infer_us, 8);
        const int32_t ne = static_cast<int32_t>(d.evicted.size());
        fnv(&ne, 4);
        for (const std::string& s : d.evicted) fnv(s.c_str(), s.size() + 1);
    }
    return h;
}

// Nearest-rank percentile.
inline double percentile(std::vector<double> v, double q) {
    if (v.empty()) return 0.0;
    std::sort(v.begin(), v.end());
    size_t rank = static_cast<size_t>(std::ceil(q / 100.0 * static_cast<double>(v.size())));
    rank = std::clamp<size_t>(rank, 1, v.size());
    return v[rank - 1];
}

}  // namespace gpufaas::capi
