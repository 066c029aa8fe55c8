// Elimination-order selection (proj/include/ustats/ordering.hpp:10-37).
#pragma once

#include <cstdint>
#include <vector>

#include "ustats/config.hpp"
#include "ustats/notation.hpp"

// the public C++ API is exported from libustats_b200.so (built -fvisibility=hidden)
#pragma GCC visibility push(default)
namespace ustats {

struct EliminationOrder {
    std::vector<int> order;
    int predicted_width = 0;
    std::uint64_t predicted_peak_entries = 0;
};

int simulate_elimination_width(const EinsumNotation& notation, const std::vector<int>& order);

EliminationOrder optimize_order(const EinsumNotation& notation, int extent,
                                OrderStrategy strategy = OrderStrategy::Auto,
                                const Config& config = {});

/// Every width-optimal elimination order of the notation's graph (used by the
/// cross-term planner to pick the one that shares most work). Capped at `limit`.
std::vector<std::vector<int>> optimal_orders(const EinsumNotation& notation, int width,
                                             std::size_t limit);

}  // namespace ustats
#pragma GCC visibility pop
