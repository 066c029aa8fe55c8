// Treewidth and elimination orders (proj/include/ustats/treewidth.hpp:12-40).
#pragma once

#include <vector>

#include "ustats/config.hpp"
#include "ustats/graph.hpp"

// the public C++ API is exported from libustats_b200.so (built -fvisibility=hidden)
#pragma GCC visibility push(default)
namespace ustats {

struct TreewidthResult {
    int width = 0;
    std::vector<int> order;
};

TreewidthResult treewidth_exact(const SimpleGraph& g, const Config& config = {});

enum class EliminationHeuristic { MinDegree, MinFill };
TreewidthResult treewidth_upper(const SimpleGraph& g,
                                EliminationHeuristic heuristic = EliminationHeuristic::MinFill);
int degeneracy(const SimpleGraph& g);
int max_treewidth_by_edges(int e);

}  // namespace ustats
#pragma GCC visibility pop
