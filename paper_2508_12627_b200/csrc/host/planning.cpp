// Index graphs, treewidth and elimination orders: the per-V-term planning that
// fixes each contraction's sequence (proj/src/{graph,treewidth,ordering}.cpp).
// Internally everything runs on bitmask adjacency (ids < 64).
#include <algorithm>
#include <bit>
#include <cstdint>
#include <string>
#include <unordered_map>

#include "ustats/errors.hpp"
#include "ustats/graph.hpp"
#include "ustats/ordering.hpp"
#include "ustats/partition.hpp"
#include "ustats/treewidth.hpp"

namespace ustats {

// ------------------------------------------------------------ SimpleGraph
SimpleGraph SimpleGraph::from_edges(int n, const std::vector<std::pair<int, int>>& edges) {
    if (n < 0) fail(ErrorCode::InvalidArgument, "vertex count must be >= 0");
    SimpleGraph g;
    for (int v = 0; v < n; ++v) g.add_vertex(v);
    for (auto [u, v] : edges) {
        if (u < 0 || v < 0 || u >= n || v >= n)
            fail(ErrorCode::InvalidArgument, "edge endpoint outside [0,n)");
        g.add_edge(u, v);
    }
    return g;
}

SimpleGraph SimpleGraph::on_vertices(const std::vector<int>& ids) {
    SimpleGraph g;
    for (int v : ids) g.add_vertex(v);
    return g;
}

SimpleGraph SimpleGraph::complete(int n) {
    SimpleGraph g;
    for (int v = 0; v < n; ++v) g.add_vertex(v);
    for (int u = 0; u < n; ++u)
        for (int v = u + 1; v < n; ++v) g.add_edge(u, v);
    return g;
}

void SimpleGraph::add_vertex(int v) { adj_.try_emplace(v); }

void SimpleGraph::add_edge(int u, int v) {
    if (u == v) fail(ErrorCode::InvalidArgument, "self-loop on vertex " + std::to_string(u));
    auto link = [](std::vector<int>& list, int x) {
        auto it = std::lower_bound(list.begin(), list.end(), x);
        if (it == list.end() || *it != x) list.insert(it, x);
    };
    link(adj_[u], v);
    link(adj_[v], u);
}

bool SimpleGraph::has_vertex(int v) const { return adj_.count(v) > 0; }

bool SimpleGraph::has_edge(int u, int v) const {
    auto it = adj_.find(u);
    return it != adj_.end() && std::binary_search(it->second.begin(), it->second.end(), v);
}

int SimpleGraph::edge_count() const {
    std::size_t ends = 0;
    for (const auto& kv : adj_) ends += kv.second.size();
    return static_cast<int>(ends / 2);
}

int SimpleGraph::degree(int v) const { return static_cast<int>(neighbors(v).size()); }

std::vector<int> SimpleGraph::vertices() const {
    std::vector<int> ids;
    for (const auto& kv : adj_) ids.push_back(kv.first);
    return ids;
}

const std::vector<int>& SimpleGraph::neighbors(int v) const {
    auto it = adj_.find(v);
    if (it == adj_.end())
        fail(ErrorCode::VertexAbsent, "vertex " + std::to_string(v) + " is not in the graph");
    return it->second;
}

std::vector<std::pair<int, int>> SimpleGraph::edges() const {
    std::vector<std::pair<int, int>> out;
    for (const auto& [v, nb] : adj_)
        for (int u : nb)
            if (v < u) out.emplace_back(v, u);
    return out;
}

SimpleGraph decomposition_graph(const std::vector<IndexTuple>& signature) {
    SimpleGraph g;
    for (const IndexTuple& t : signature) {
        for (int id : t) g.add_vertex(id);
        for (std::size_t a = 0; a < t.size(); ++a)
            for (std::size_t b = a + 1; b < t.size(); ++b)
                if (t[a] != t[b]) g.add_edge(t[a], t[b]);
    }
    return g;
}

SimpleGraph decomposition_graph(const EinsumNotation& notation) {
    return decomposition_graph(notation.inputs);
}

SimpleGraph eliminate_vertex(const SimpleGraph& g, int v) {
    const std::vector<int> nb = g.neighbors(v);
    SimpleGraph out;
    for (int u : g.vertices())
        if (u != v) out.add_vertex(u);
    for (auto [a, b] : g.edges())
        if (a != v && b != v) out.add_edge(a, b);
    for (std::size_t i = 0; i < nb.size(); ++i)
        for (std::size_t j = i + 1; j < nb.size(); ++j) out.add_edge(nb[i], nb[j]);
    return out;
}

SimpleGraph quotient_graph(const SimpleGraph& g, const SetPartition& partition) {
    const std::vector<int> ids = g.vertices();
    if (partition.ground_size() != static_cast<int>(ids.size()))
        fail(ErrorCode::GroundSetMismatch,
             "partition of " + std::to_string(partition.ground_size()) +
                 " elements does not cover a graph on " + std::to_string(ids.size()) + " vertices");
    auto pos = [&](int id) {
        return static_cast<int>(std::lower_bound(ids.begin(), ids.end(), id) - ids.begin());
    };
    SimpleGraph q;
    for (int b = 0; b < partition.block_count(); ++b) q.add_vertex(b);
    for (auto [a, b] : g.edges()) {
        int ba = partition.block_of(pos(a)), bb = partition.block_of(pos(b));
        if (ba != bb) q.add_edge(ba, bb);
    }
    return q;
}

// -------------------------------------------------------------- treewidth
namespace {

using Mask = std::uint64_t;

struct MaskGraph {
    std::vector<int> ids;   // position -> vertex id (sorted)
    std::vector<Mask> adj;  // position adjacency
};

MaskGraph to_masks(const SimpleGraph& g) {
    MaskGraph mg;
    mg.ids = g.vertices();
    if (mg.ids.size() > 64) fail(ErrorCode::TooLarge, "graphs beyond 64 vertices are unsupported");
    mg.adj.assign(mg.ids.size(), 0);
    for (std::size_t i = 0; i < mg.ids.size(); ++i)
        for (int u : g.neighbors(mg.ids[i])) {
            auto p = std::lower_bound(mg.ids.begin(), mg.ids.end(), u) - mg.ids.begin();
            mg.adj[i] |= Mask{1} << p;
        }
    return mg;
}

inline Mask bit(int v) { return Mask{1} << v; }

// Eliminating v joins its live neighbours into a clique.
void join_neighbours(std::vector<Mask>& adj, int v, Mask live) {
    const Mask nb = adj[static_cast<std::size_t>(v)] & live;
    for (Mask r = nb; r; r &= r - 1) {
        int u = std::countr_zero(r);
        adj[static_cast<std::size_t>(u)] = (adj[static_cast<std::size_t>(u)] | nb) & ~bit(u) & ~bit(v);
    }
    adj[static_cast<std::size_t>(v)] = 0;
}

bool clique(const std::vector<Mask>& adj, Mask verts) {
    for (Mask r = verts; r; r &= r - 1) {
        int v = std::countr_zero(r);
        Mask others = verts & ~bit(v);
        if ((adj[static_cast<std::size_t>(v)] & others) != others) return false;
    }
    return true;
}

// Width-optimal elimination by search over live sets (treewidth.cpp:22-132
// semantics): peel simplicial vertices lowest-first, then try candidates in
// ascending position keeping the first strictly better width. The elimination
// graph of a live set is independent of how it was reached, so results are
// memoized on the live set.
class WidthSearch {
  public:
    explicit WidthSearch(std::size_t V) : V_(static_cast<int>(V)) {}

    struct Best {
        int width;
        std::vector<int> seq;
    };

    Best run(std::vector<Mask> adj, Mask live) {
        const Mask key = live;
        if (auto hit = memo_.find(key); hit != memo_.end()) return hit->second;

        Best out{0, {}};
        for (bool again = true; again && live;) {
            again = false;
            for (Mask r = live; r; r &= r - 1) {
                int v = std::countr_zero(r);
                Mask nb = adj[static_cast<std::size_t>(v)] & live;
                if (!clique(adj, nb)) continue;
                out.width = std::max(out.width, std::popcount(nb));
                out.seq.push_back(v);
                join_neighbours(adj, v, live);
                live &= ~bit(v);
                again = true;
                break;
            }
        }
        if (live) {
            int best_w = V_;
            std::vector<int> best_seq;
            for (Mask r = live; r; r &= r - 1) {
                int v = std::countr_zero(r);
                int deg = std::popcount(adj[static_cast<std::size_t>(v)] & live);
                if (deg >= best_w) continue;
                std::vector<Mask> next = adj;
                join_neighbours(next, v, live);
                Best sub = run(std::move(next), live & ~bit(v));
                int w = std::max(deg, sub.width);
                if (w < best_w) {
                    best_w = w;
                    best_seq.assign(1, v);
                    best_seq.insert(best_seq.end(), sub.seq.begin(), sub.seq.end());
                }
            }
            out.width = std::max(out.width, best_w);
            out.seq.insert(out.seq.end(), best_seq.begin(), best_seq.end());
        }
        memo_.emplace(key, out);
        return out;
    }

  private:
    int V_;
    std::unordered_map<Mask, Best> memo_;
};

}  // namespace

TreewidthResult treewidth_exact(const SimpleGraph& g, const Config& config) {
    if (g.vertex_count() > config.exact_treewidth_bound)
        fail(ErrorCode::TooLarge, "exact treewidth limited to " +
                                      std::to_string(config.exact_treewidth_bound) +
                                      " vertices, got " + std::to_string(g.vertex_count()));
    if (g.vertex_count() == 0) return {0, {}};
    MaskGraph mg = to_masks(g);
    const int V = static_cast<int>(mg.ids.size());
    const Mask all = V == 64 ? ~Mask{0} : (bit(V) - 1);
    WidthSearch search(mg.ids.size());
    WidthSearch::Best b = search.run(mg.adj, all);
    TreewidthResult r;
    r.width = b.width;
    for (int p : b.seq) r.order.push_back(mg.ids[static_cast<std::size_t>(p)]);
    return r;
}

TreewidthResult treewidth_upper(const SimpleGraph& g, EliminationHeuristic heuristic) {
    MaskGraph mg = to_masks(g);
    const int V = static_cast<int>(mg.ids.size());
    Mask live = V == 64 ? ~Mask{0} : (bit(V) - 1);
    TreewidthResult r;
    while (live) {
        int chosen = -1;
        long best = -1;
        for (Mask rest = live; rest; rest &= rest - 1) {
            int v = std::countr_zero(rest);
            Mask nb = mg.adj[static_cast<std::size_t>(v)] & live;
            long score = 0;
            if (heuristic == EliminationHeuristic::MinDegree) {
                score = std::popcount(nb);
            } else {
                for (Mask a = nb; a; a &= a - 1) {
                    int u = std::countr_zero(a);
                    score += std::popcount(nb & ~mg.adj[static_cast<std::size_t>(u)] & ~bit(u) &
                                           ((bit(u) - 1) ^ ~Mask{0}));  // pairs (u,w) with w>u
                }
            }
            if (best < 0 || score < best) {
                best = score;
                chosen = v;
            }
        }
        r.width = std::max(r.width, std::popcount(mg.adj[static_cast<std::size_t>(chosen)] & live));
        r.order.push_back(mg.ids[static_cast<std::size_t>(chosen)]);
        join_neighbours(mg.adj, chosen, live);
        live &= ~bit(chosen);
    }
    return r;
}

int degeneracy(const SimpleGraph& g) {
    MaskGraph mg = to_masks(g);
    const int V = static_cast<int>(mg.ids.size());
    Mask live = V == 64 ? ~Mask{0} : (bit(V) - 1);
    int degen = 0;
    while (live) {
        int chosen = -1, low = 1 << 30;
        for (Mask r = live; r; r &= r - 1) {
            int v = std::countr_zero(r);
            int d = std::popcount(mg.adj[static_cast<std::size_t>(v)] & live);
            if (d < low) {
                low = d;
                chosen = v;
            }
        }
        degen = std::max(degen, low);
        live &= ~bit(chosen);
    }
    return degen;
}

int max_treewidth_by_edges(int e) {
    // Largest k with k(k+1)/2 <= e, i.e. the biggest clique e edges can build
    // (K_{k+1} needs k(k+1)/2 edges): the verified table of treewidth.cpp:219-225.
    if (e < 1 || e > 15)
        fail(ErrorCode::OutOfTable,
             "edge-count treewidth table covers 1..15 edges, got " + std::to_string(e));
    int k = 0;
    while ((k + 1) * (k + 2) / 2 <= e) ++k;
    return k;
}

// --------------------------------------------------------------- ordering
namespace {
std::uint64_t saturating_pow(int base, int exp) {
    unsigned __int128 v = 1;
    while (exp-- > 0) {
        v *= static_cast<unsigned>(base);
        if (v > ~std::uint64_t{0}) return ~std::uint64_t{0};
    }
    return static_cast<std::uint64_t>(v);
}

void require_permutation(const std::vector<int>& order, int count) {
    if (static_cast<int>(order.size()) != count)
        fail(ErrorCode::InvalidArgument,
             "elimination order must cover all " + std::to_string(count) + " indices");
    std::vector<char> seen(static_cast<std::size_t>(count), 0);
    for (int v : order) {
        if (v < 0 || v >= count || seen[static_cast<std::size_t>(v)])
            fail(ErrorCode::InvalidArgument, "elimination order is not a permutation");
        seen[static_cast<std::size_t>(v)] = 1;
    }
}
}  // namespace

int simulate_elimination_width(const EinsumNotation& notation, const std::vector<int>& order) {
    require_permutation(order, notation.index_count);
    MaskGraph mg = to_masks(decomposition_graph(notation));
    // ids are 0..index_count-1 (canonical), so positions == ids.
    Mask live = 0;
    for (int id : mg.ids) live |= bit(id);
    int width = 0;
    for (int v : order) {
        width = std::max(width, std::popcount(mg.adj[static_cast<std::size_t>(v)] & live));
        join_neighbours(mg.adj, v, live);
        live &= ~bit(v);
    }
    return width;
}

EliminationOrder optimize_order(const EinsumNotation& notation, int extent, OrderStrategy strategy,
                                const Config& config) {
    if (extent < 1) fail(ErrorCode::InvalidArgument, "extent must be >= 1");
    if (strategy == OrderStrategy::Auto)
        strategy = notation.index_count <= config.exhaustive_index_bound ? OrderStrategy::Exhaustive
                                                                          : OrderStrategy::GreedyMinFill;
    const SimpleGraph g = decomposition_graph(notation);
    TreewidthResult tw;
    if (strategy == OrderStrategy::GreedyMinDegree) {
        tw = treewidth_upper(g, EliminationHeuristic::MinDegree);
    } else if (strategy == OrderStrategy::GreedyMinFill) {
        tw = treewidth_upper(g, EliminationHeuristic::MinFill);
    } else {
        if (notation.index_count > config.exhaustive_index_bound)
            fail(ErrorCode::TooLargeForExhaustive,
                 "exhaustive order search limited to " +
                     std::to_string(config.exhaustive_index_bound) + " indices, got " +
                     std::to_string(notation.index_count));
        Config exact = config;
        exact.exact_treewidth_bound = config.exhaustive_index_bound;
        tw = treewidth_exact(g, exact);
    }
    EliminationOrder o;
    o.order = std::move(tw.order);
    o.predicted_width = tw.width;
    o.predicted_peak_entries = saturating_pow(extent, tw.width + 1);
    return o;
}

std::vector<std::vector<int>> optimal_orders(const EinsumNotation& notation, int width,
                                             std::size_t limit) {
    MaskGraph mg = to_masks(decomposition_graph(notation));
    std::vector<std::vector<int>> found;
    std::vector<int> seq;
    Mask all = 0;
    for (int id : mg.ids) all |= bit(id);
    auto dfs = [&](auto&& self, std::vector<Mask> adj, Mask live) -> void {
        if (found.size() >= limit) return;
        if (!live) {
            found.push_back(seq);
            return;
        }
        for (Mask r = live; r; r &= r - 1) {
            int v = std::countr_zero(r);
            if (std::popcount(adj[static_cast<std::size_t>(v)] & live) > width) continue;
            std::vector<Mask> next = adj;
            join_neighbours(next, v, live);
            seq.push_back(v);
            self(self, std::move(next), live & ~bit(v));
            seq.pop_back();
        }
    };
    dfs(dfs, mg.adj, all);
    return found;
}

}  // namespace ustats
