// Index graphs for contraction planning (proj/include/ustats/graph.hpp:12-72).
#pragma once

#include <map>
#include <vector>

#include "ustats/notation.hpp"

// the public C++ API is exported from libustats_b200.so (built -fvisibility=hidden)
#pragma GCC visibility push(default)
namespace ustats {

class SetPartition;

class SimpleGraph {
  public:
    SimpleGraph() = default;
    static SimpleGraph from_edges(int n, const std::vector<std::pair<int, int>>& edges);
    static SimpleGraph on_vertices(const std::vector<int>& ids);
    static SimpleGraph complete(int n);

    void add_vertex(int v);
    void add_edge(int u, int v);
    bool has_vertex(int v) const;
    bool has_edge(int u, int v) const;
    int vertex_count() const { return static_cast<int>(adj_.size()); }
    int edge_count() const;
    int degree(int v) const;
    std::vector<int> vertices() const;
    const std::vector<int>& neighbors(int v) const;
    std::vector<std::pair<int, int>> edges() const;
    bool operator==(const SimpleGraph& o) const { return adj_ == o.adj_; }

  private:
    std::map<int, std::vector<int>> adj_;
};

SimpleGraph decomposition_graph(const EinsumNotation& notation);
SimpleGraph decomposition_graph(const std::vector<IndexTuple>& signature);
SimpleGraph eliminate_vertex(const SimpleGraph& g, int v);
SimpleGraph quotient_graph(const SimpleGraph& g, const SetPartition& partition);

}  // namespace ustats
#pragma GCC visibility pop
