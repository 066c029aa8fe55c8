// C-ABI driver over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/).
// TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
// reference/cpu_baseline arm load it as the checker; the product never does.
//
// Entry points mirror the reference's public API (engine.hpp:58-65,
// einsum.hpp:41-43, bruteforce.hpp:20-36) over caller-owned row-major f64
// tensors, so Python can drive the reference exactly as a user would.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include <cmath>
#include <memory>
#include <span>

#include "ustats/complexity.hpp"
#include "ustats/dcov.hpp"
#include "ustats/motifs.hpp"
#include "ustats/ustats.hpp"

namespace {

thread_local std::string g_err;

struct Problem {
    int m = 0;
    std::vector<ustats::IndexTuple> sig0;  // 0-based
    std::vector<const double*> data;
    int n = 0;
};

Problem make_problem(int m, int K, const int* tuple_len, const int* tuple_idx,
                     const double* const* factors, int n) {
    Problem p;
    p.m = m;
    p.n = n;
    int off = 0;
    for (int k = 0; k < K; ++k) {
        ustats::IndexTuple t(tuple_idx + off, tuple_idx + off + tuple_len[k]);
        off += tuple_len[k];
        p.sig0.push_back(t);
        p.data.push_back(factors[k]);
    }
    return p;
}

// MDKernel whose component k reads factor k at its picks (row-major, extent n):
// the "factors over data matrices/vectors" form (motifs.cpp:16-29 precedent).
ustats::MDKernel kernel_of(const Problem& p) {
    ustats::MDKernel k;
    k.arity = p.m;
    k.name = "tensor-backed";
    for (std::size_t c = 0; c < p.sig0.size(); ++c) {
        ustats::IndexTuple one;
        for (int s : p.sig0[c]) one.push_back(s + 1);
        k.signature.push_back(one);
        const double* d = p.data[c];
        const std::uint64_t n = static_cast<std::uint64_t>(p.n);
        k.components.push_back([d, n](const ustats::Sample&, std::span<const int> idx) {
            std::uint64_t off = 0;
            for (int i : idx) off = off * n + static_cast<std::uint64_t>(i);
            return d[off];
        });
    }
    return k;
}

ustats::Config config_of(int threads, std::uint64_t cap) {
    ustats::Config c;
    c.threads = threads;
    if (cap) c.memory_cap_entries = cap;
    return c;
}

int status_of(const std::exception& e) {
    g_err = e.what();
    if (auto* ue = dynamic_cast<const ustats::Error*>(&e)) return 1 + static_cast<int>(ue->code());
    return 100;
}

void export_stats(const ustats::RunStats& rs, double* stats) {
    if (!stats) return;
    stats[0] = rs.tensorize_seconds;
    stats[1] = rs.contract_seconds;
    stats[2] = static_cast<double>(rs.einsum_calls);
    stats[3] = static_cast<double>(rs.partitions_enumerated);
    stats[4] = static_cast<double>(rs.partitions_evaluated);
    stats[5] = static_cast<double>(rs.multiply_adds);
    stats[6] = static_cast<double>(rs.peak_intermediate_entries);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ustats::u_statistic (engine.cpp:173-193) on a tensor-backed kernel.
// stats (7 doubles): tensorize_s, contract_s, einsum_calls, enumerated, evaluated, madds, peak.
int ref_u_statistic(int m, int K, const int* tuple_len, const int* tuple_idx,
                    const double* const* factors, int n, int threads, std::uint64_t cap,
                    double* u_out, double* stats) {
    try {
        Problem p = make_problem(m, K, tuple_len, tuple_idx, factors, n);
        ustats::RunStats rs;
        *u_out = ustats::u_statistic(kernel_of(p), ustats::Sample::indices_only(n),
                                     config_of(threads, cap), &rs);
        export_stats(rs, stats);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

int ref_v_statistic(int m, int K, const int* tuple_len, const int* tuple_idx,
                    const double* const* factors, int n, int threads, std::uint64_t cap,
                    double* v_out, double* stats) {
    try {
        Problem p = make_problem(m, K, tuple_len, tuple_idx, factors, n);
        ustats::RunStats rs;
        *v_out = ustats::v_statistic(kernel_of(p), ustats::Sample::indices_only(n),
                                     config_of(threads, cap), &rs);
        export_stats(rs, stats);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

int ref_u_statistic_unsparsified(int m, int K, const int* tuple_len, const int* tuple_idx,
                                 const double* const* factors, int n, int threads,
                                 std::uint64_t cap, double* u_out, double* stats) {
    try {
        Problem p = make_problem(m, K, tuple_len, tuple_idx, factors, n);
        ustats::RunStats rs;
        *u_out = ustats::u_statistic_unsparsified(kernel_of(p), ustats::Sample::indices_only(n),
                                                  config_of(threads, cap), &rs);
        export_stats(rs, stats);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

int ref_restricted_v(int m, int K, const int* tuple_len, const int* tuple_idx,
                     const double* const* factors, int n, const int* rgs, int threads,
                     double* v_out) {
    try {
        Problem p = make_problem(m, K, tuple_len, tuple_idx, factors, n);
        ustats::SetPartition part(std::vector<int>(rgs, rgs + m));
        *v_out = ustats::restricted_v(kernel_of(p), ustats::Sample::indices_only(n), part,
                                      config_of(threads, 0));
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// Literal U over injective tuples (bruteforce.cpp:57-72), long-double accumulation.
int ref_u_brute_force(int m, int K, const int* tuple_len, const int* tuple_idx,
                      const double* const* factors, int n, double* u_out) {
    try {
        Problem p = make_problem(m, K, tuple_len, tuple_idx, factors, n);
        ustats::Config c;
        c.brute_force_term_cap = ~std::uint64_t{0};
        *u_out = ustats::u_brute_force(ustats::flatten(kernel_of(p)), m,
                                       ustats::Sample::indices_only(n), c);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// Per-survivor terms exactly as lattice_combination computes them
// (engine.cpp:67-73): sparsify each factor (tensor.cpp:54-76), stream survivors
// (partition.cpp:214-234), einsum the induced notation, weight by mu.
// rgs_out: max_terms*m ints; mu_out, v_out: max_terms each. Returns count via *count.
int ref_u_terms(int m, int K, const int* tuple_len, const int* tuple_idx,
                const double* const* factors, int n, int threads, std::uint64_t cap,
                int max_terms, int* count, int* rgs_out, long long* mu_out, double* v_out,
                double* madds_out) {
    try {
        Problem p = make_problem(m, K, tuple_len, tuple_idx, factors, n);
        ustats::Config cfg = config_of(threads, cap);
        std::vector<ustats::DenseTensor> tensors;
        for (std::size_t k = 0; k < p.sig0.size(); ++k) {
            ustats::DenseTensor t(static_cast<int>(p.sig0[k].size()), n, cfg);
            std::memcpy(t.data.data(), p.data[k], t.data.size() * sizeof(double));
            tensors.push_back(ustats::sparsify(t));
        }
        ustats::SparsifiedPartitionStream stream(m, p.sig0);
        ustats::SetPartition part;
        int c = 0;
        while (stream.next(part)) {
            if (c >= max_terms) {
                g_err = "too many terms";
                return 99;
            }
            ustats::EinsumNotation notation(ustats::induced_signature(p.sig0, part));
            ustats::ExecStats es;
            double v = ustats::einsum(tensors, notation, cfg, nullptr, &es).scalar();
            for (int i = 0; i < m; ++i) rgs_out[c * m + i] = part.rgs()[i];
            mu_out[c] = ustats::mobius_coefficient(part);
            v_out[c] = v;
            if (madds_out) madds_out[c] = static_cast<double>(es.multiply_adds);
            ++c;
        }
        *count = c;
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// ustats::einsum (einsum.hpp:41-43) on a raw notation; out has n^|output| entries.
int ref_einsum(int K, const int* tuple_len, const int* tuple_idx, const double* const* tensors,
               int n, int out_len, const int* out_idx, int threads, double* out,
               double* madds_out) {
    try {
        std::vector<ustats::IndexTuple> raw;
        std::vector<ustats::DenseTensor> ts;
        int off = 0;
        ustats::Config cfg = config_of(threads, 0);
        for (int k = 0; k < K; ++k) {
            raw.emplace_back(tuple_idx + off, tuple_idx + off + tuple_len[k]);
            off += tuple_len[k];
            ustats::DenseTensor t(tuple_len[k], n, cfg);
            std::memcpy(t.data.data(), tensors[k], t.data.size() * sizeof(double));
            ts.push_back(std::move(t));
        }
        ustats::EinsumNotation notation(raw, ustats::IndexTuple(out_idx, out_idx + out_len));
        ustats::ExecStats es;
        ustats::DenseTensor r = ustats::einsum(ts, notation, cfg, nullptr, &es);
        std::memcpy(out, r.data.data(), r.data.size() * sizeof(double));
        if (madds_out) *madds_out = static_cast<double>(es.multiply_adds);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// optimize_order (ordering.cpp:48-86) for a notation: writes the order and width.
int ref_optimize_order(int K, const int* tuple_len, const int* tuple_idx, int* order_out,
                       int* width_out) {
    try {
        std::vector<ustats::IndexTuple> raw;
        int off = 0;
        for (int k = 0; k < K; ++k) {
            raw.emplace_back(tuple_idx + off, tuple_idx + off + tuple_len[k]);
            off += tuple_len[k];
        }
        ustats::EinsumNotation notation(raw);
        ustats::EliminationOrder o = ustats::optimize_order(notation, 2);
        for (std::size_t i = 0; i < o.order.size(); ++i) order_out[i] = o.order[i];
        *width_out = o.predicted_width;
        return static_cast<int>(o.order.size()) >= 0 ? 0 : 1;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// complexity_report (complexity.cpp:73-127): ints[8] = index_count, extent,
// graph_vertices, graph_edges, treewidth_lower, treewidth_upper,
// treewidth_exact (-1 absent), max_quotient_width; counts[2] = bell,
// sparsified; hist[16] by width; flops decimal into buf[cap].
int ref_complexity_report(int K, const int* tuple_len, const int* tuple_idx, int extent, int* ints,
                          std::uint64_t* counts, std::uint64_t* hist, char* buf, int cap) {
    try {
        std::vector<ustats::IndexTuple> raw;
        int off = 0;
        for (int k = 0; k < K; ++k) {
            raw.emplace_back(tuple_idx + off, tuple_idx + off + tuple_len[k]);
            off += tuple_len[k];
        }
        auto r = ustats::complexity_report(raw, extent);
        ints[0] = r.index_count;
        ints[1] = r.extent;
        ints[2] = r.graph_vertices;
        ints[3] = r.graph_edges;
        ints[4] = r.treewidth_lower;
        ints[5] = r.treewidth_upper;
        ints[6] = r.treewidth_exact ? *r.treewidth_exact : -1;
        ints[7] = r.max_quotient_width;
        counts[0] = r.bell_count;
        counts[1] = r.sparsified_count;
        for (int w = 0; w < 16; ++w) hist[w] = 0;
        for (const auto& [w, c] : r.count_by_width)
            if (w >= 0 && w < 16) hist[w] = c;
        std::snprintf(buf, static_cast<std::size_t>(cap), "%s", r.flops_estimate.c_str());
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// dcov_squared (dcov.cpp:35-87) on row-major paired samples.
int ref_dcov_squared(const double* x, int dx, const double* y, int dy, int n, int threads, double* out) {
    try {
        std::vector<ustats::Observation> xs(static_cast<std::size_t>(n)), ys(static_cast<std::size_t>(n));
        for (int i = 0; i < n; ++i) {
            xs[static_cast<std::size_t>(i)].assign(x + static_cast<std::size_t>(i) * dx, x + static_cast<std::size_t>(i + 1) * dx);
            ys[static_cast<std::size_t>(i)].assign(y + static_cast<std::size_t>(i) * dy, y + static_cast<std::size_t>(i + 1) * dy);
        }
        ustats::Sample sx(std::move(xs)), sy(std::move(ys));
        *out = ustats::dcov_squared(sx, sy, config_of(threads, 0));
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// hoif_tau (hoif.cpp:74-100) with truncation_phi(k) on rows [A, Y, Z...].
int ref_hoif_tau(int m, int k, const double* data, int n, int d, int threads, double* out) {
    try {
        std::vector<ustats::Observation> rows(static_cast<std::size_t>(n));
        for (int i = 0; i < n; ++i)
            rows[static_cast<std::size_t>(i)].assign(data + static_cast<std::size_t>(i) * d,
                                                     data + static_cast<std::size_t>(i + 1) * d);
        ustats::Sample s(std::move(rows));
        *out = ustats::hoif_tau(m, ustats::truncation_phi(k), s, config_of(threads, 0));
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

// motif_count (motifs.cpp:53-69) on the graph over vertices 0..n-1.
int ref_motif_count(int n, int edge_count, const int* edges, const char* id, int threads, long long* out) {
    try {
        ustats::SimpleGraph g;
        for (int v = 0; v < n; ++v) g.add_vertex(v);
        for (int e = 0; e < edge_count; ++e) g.add_edge(edges[2 * e], edges[2 * e + 1]);
        *out = ustats::motif_count(g, ustats::motif_by_id(id), config_of(threads, 0));
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Data kernels through the reference's OWN tensorize path (engine.cpp:108-136):
// the components are std::function callbacks evaluated per entry on the sample,
// exactly how a reference user states the BASELINE kernels. Specs as in
// us_u_statistic_data: rbf:<shape>:<h>, proj:<m>:<kmax>, hoif:<j>:<k>, prod2.
namespace {

std::vector<std::string> split_spec(const std::string& s) {
    std::vector<std::string> out;
    std::string cur;
    for (char c : s) {
        if (c == ':') {
            out.push_back(cur);
            cur.clear();
        } else {
            cur += c;
        }
    }
    out.push_back(cur);
    return out;
}

}  // namespace

extern "C" int ref_u_statistic_data(const char* spec_c, const double* data, int n, int d, int threads,
                                    std::uint64_t cap, double* u_out, double* stats) {
    try {
        const std::string spec(spec_c);
        const auto p = split_spec(spec);
        std::vector<ustats::Observation> rows(static_cast<std::size_t>(n));
        for (int i = 0; i < n; ++i) rows[static_cast<std::size_t>(i)].assign(data + i * d, data + (i + 1) * d);
        ustats::Sample sample(std::move(rows));
        ustats::MDKernel k;
        if (p[0] == "prod2") {
            k = ustats::prod2_kernel();
        } else if (p[0] == "hoif") {
            k = ustats::hoif_kernel(std::stoi(p[1]), ustats::truncation_phi(std::stoi(p[2])));
        } else if (p[0] == "rbf") {
            const std::string shape = p[1];
            const double scale = 0.5 / (std::stod(p[2]) * std::stod(p[2]));
            auto rbf = [scale](const ustats::Sample& s, std::span<const int> idx) {
                const auto& a = s.points[static_cast<std::size_t>(idx[0])];
                const auto& b = s.points[static_cast<std::size_t>(idx[1])];
                double acc = 0.0;
                for (std::size_t c = 0; c < a.size(); ++c) {
                    const double t = a[c] - b[c];
                    acc += t * t;
                }
                return std::exp(-scale * acc);
            };
            std::vector<ustats::IndexTuple> sig;
            int m = 0;
            if (shape == "k4tail") {
                m = 6;
                sig = {{1, 2}, {1, 3}, {1, 4}, {2, 3}, {2, 4}, {3, 4}, {4, 5}, {5, 6}};
            } else {
                m = std::stoi(shape.substr(5));
                for (int i = 1; i < m; ++i) sig.push_back({i, i + 1});
                if (shape[1] == 'y') sig.push_back({m, 1});
            }
            k.arity = m;
            k.signature = sig;
            k.components.assign(sig.size(), rbf);
            k.name = spec;
        } else if (p[0] == "proj") {
            const int m = std::stoi(p[1]), kmax = std::stoi(p[2]);
            const int c = d - 2, F = c * kmax;
            // user-side kernel setup: features, Omega = (Z'Z/n)^-1, W = Z Omega
            std::vector<double> Z(static_cast<std::size_t>(n) * F), G(static_cast<std::size_t>(F) * F, 0.0);
            for (int i = 0; i < n; ++i)
                for (int cc = 0; cc < c; ++cc)
                    for (int kk = 1; kk <= kmax; ++kk)
                        Z[static_cast<std::size_t>(i) * F + cc * kmax + kk - 1] = std::cos(M_PI * kk * data[i * d + cc]);
            for (int i = 0; i < n; ++i)
                for (int a = 0; a < F; ++a)
                    for (int b = 0; b < F; ++b)
                        G[static_cast<std::size_t>(a) * F + b] +=
                            Z[static_cast<std::size_t>(i) * F + a] * Z[static_cast<std::size_t>(i) * F + b];
            for (double& g : G) g /= n;
            // Gauss-Jordan inverse
            std::vector<double> inv(static_cast<std::size_t>(F) * F, 0.0);
            for (int i = 0; i < F; ++i) inv[static_cast<std::size_t>(i) * F + i] = 1.0;
            for (int col = 0; col < F; ++col) {
                const double piv = G[static_cast<std::size_t>(col) * F + col];
                for (int j = 0; j < F; ++j) {
                    G[static_cast<std::size_t>(col) * F + j] /= piv;
                    inv[static_cast<std::size_t>(col) * F + j] /= piv;
                }
                for (int r = 0; r < F; ++r) {
                    if (r == col) continue;
                    const double f = G[static_cast<std::size_t>(r) * F + col];
                    for (int j = 0; j < F; ++j) {
                        G[static_cast<std::size_t>(r) * F + j] -= f * G[static_cast<std::size_t>(col) * F + j];
                        inv[static_cast<std::size_t>(r) * F + j] -= f * inv[static_cast<std::size_t>(col) * F + j];
                    }
                }
            }
            auto W = std::make_shared<std::vector<double>>(static_cast<std::size_t>(n) * F, 0.0);
            for (int i = 0; i < n; ++i)
                for (int a = 0; a < F; ++a) {
                    double s = 0;
                    for (int b = 0; b < F; ++b)
                        s += Z[static_cast<std::size_t>(i) * F + b] * inv[static_cast<std::size_t>(b) * F + a];
                    (*W)[static_cast<std::size_t>(i) * F + a] = s;
                }
            auto Zs = std::make_shared<std::vector<double>>(std::move(Z));
            auto proj = [W, Zs, F](const ustats::Sample&, std::span<const int> idx) {
                const double* w = W->data() + static_cast<std::size_t>(idx[0]) * F;
                const double* z = Zs->data() + static_cast<std::size_t>(idx[1]) * F;
                double s = 0;
                for (int a = 0; a < F; ++a) s += w[a] * z[a];
                return s;
            };
            const int rc = d - 2, ec = d - 1;
            k.arity = m;
            k.signature.push_back({1});
            k.components.push_back([rc](const ustats::Sample& s, std::span<const int> idx) {
                return s.points[static_cast<std::size_t>(idx[0])][static_cast<std::size_t>(rc)];
            });
            for (int i = 1; i < m; ++i) {
                k.signature.push_back({i, i + 1});
                k.components.push_back(proj);
            }
            k.signature.push_back({m});
            k.components.push_back([ec](const ustats::Sample& s, std::span<const int> idx) {
                return s.points[static_cast<std::size_t>(idx[0])][static_cast<std::size_t>(ec)];
            });
            k.name = spec;
        } else {
            g_err = "unknown spec";
            return 99;
        }
        ustats::RunStats rs;
        *u_out = ustats::u_statistic(k, sample, config_of(threads, cap), &rs);
        export_stats(rs, stats);
        return 0;
    } catch (const std::exception& e) {
        return status_of(e);
    }
}
