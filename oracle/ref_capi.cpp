// C-ABI driver over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/).
// TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
// reference/cpu_baseline arm load it as the checker; the product never does.
//
// Entry points mirror the reference's public API (engine.hpp:58-65,
// einsum.hpp:41-43, bruteforce.hpp:20-36) over caller-owned row-major f64
// tensors, so Python can drive the reference exactly as a user would.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

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

}  // extern "C"
