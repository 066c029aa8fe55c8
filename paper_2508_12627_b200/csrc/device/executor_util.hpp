// Internal helpers shared by the executor's translation units (runtime.cpp,
// program.cpp, launch.cpp, contractor.cpp, lattice.cpp). Not installed.
#pragma once

#include <bit>
#include <cstdint>
#include <vector>

#include "executor.hpp"

namespace ustats::dev {

inline std::uint32_t bit(int id) { return 1u << id; }

inline std::vector<int> ids_of(std::uint32_t mask) {
    std::vector<int> v;
    for (std::uint32_t r = mask; r; r &= r - 1) v.push_back(std::countr_zero(r));
    return v;
}

inline std::uint64_t ipow(long long n, int e) {
    std::uint64_t v = 1;
    while (e-- > 0) v *= static_cast<std::uint64_t>(n);
    return v;
}

inline std::uint32_t ids_of_views(const std::vector<View>& vs) {
    std::uint32_t m = 0;
    for (const View& v : vs) m |= v.ids;
    return m;
}

// Every view an op reads (operands, stream factors, fused-epilogue weights).
template <class F>
void for_each_read(const Op& op, F&& f) {
    for (const View& v : op.factors) f(v);
    for (const View& v : op.fa) f(v);
    for (const View& v : op.fb) f(v);
    for (const Op::Epi& e : op.epis)
        for (const View& v : e.w) f(v);
}

}  // namespace ustats::dev
