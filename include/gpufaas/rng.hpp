#pragma once
// Deterministic random source for trace and workload synthesis. Only raw
// mt19937_64 output is consumed (never <random> distributions, whose results
// are implementation-defined) — the contract of
// proj/include/gpufaas/rng.hpp:11-30, so request streams match the reference.

#include <cstdint>
#include <random>

namespace gpufaas {

class Rng {
public:
    explicit Rng(std::uint64_t seed) : engine_(seed) {}

    std::uint64_t next_u64() { return engine_(); }

    // [0, n) by plain modulo of one raw draw.
    std::int64_t uniform_below(std::int64_t n) {
        const std::uint64_t raw = engine_();
        return static_cast<std::int64_t>(raw % static_cast<std::uint64_t>(n));
    }

    // [0, 1) from the top 53 bits of one raw draw.
    double uniform01() {
        const std::uint64_t top53 = engine_() >> 11;
        return static_cast<double>(top53) * 0x1.0p-53;
    }

private:
    std::mt19937_64 engine_;
};

}  // namespace gpufaas
