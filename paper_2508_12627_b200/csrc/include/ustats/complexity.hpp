// Cost anatomy of a signature's lattice evaluation
// (proj/include/ustats/complexity.hpp:19-51): survivor count, the exact
// treewidth histogram of the survivors' quotient graphs, and the exact
// (arbitrary-precision) FLOP estimate K * sum_w count_w * n^(w+1).
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include "ustats/config.hpp"
#include "ustats/notation.hpp"

// the public C++ API is exported from libustats_b200.so (built -fvisibility=hidden)
#pragma GCC visibility push(default)
namespace ustats {

struct ComplexityReport {
    std::vector<IndexTuple> signature;  // canonical 0-based tuples
    int index_count = 0;
    int extent = 0;
    int graph_vertices = 0;
    int graph_edges = 0;
    int treewidth_lower = 0;             // degeneracy
    int treewidth_upper = 0;             // min over the MinFill / MinDegree heuristics
    std::optional<int> treewidth_exact;  // when m <= exact_treewidth_bound
    std::uint64_t bell_count = 0;
    std::uint64_t sparsified_count = 0;
    std::map<int, std::uint64_t> count_by_width;
    int max_quotient_width = 0;
    std::string flops_estimate;          // decimal, exact past 2^64
};

ComplexityReport complexity_report(const std::vector<IndexTuple>& signature, int extent, const Config& config = {});

// ((1,2),(2,3),...,(m-1,m)), 1-based (complexity.cpp chain_signature).
std::vector<IndexTuple> chain_signature(int m);

}  // namespace ustats
#pragma GCC visibility pop
