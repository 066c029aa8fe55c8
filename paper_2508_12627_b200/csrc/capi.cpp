// extern "C" boundary (include/ustats_b200.h): decodes plain arguments into
// the host API types, runs the engine, and maps exceptions to status codes.
#include "../../include/ustats_b200.h"

#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "device/executor.hpp"
#include "device/tensorize.hpp"
#include "ustats/ustats.hpp"
#include "ustats/complexity.hpp"

namespace ustats::dev {
double combine_terms(const std::vector<double>& terms);
}

namespace {

thread_local std::string g_error;

int fail_status(const std::exception& e) {
    g_error = e.what();
    if (const auto* ue = dynamic_cast<const ustats::Error*>(&e)) return 1 + static_cast<int>(ue->code());
    return 1 + static_cast<int>(ustats::ErrorCode::InvalidArgument);
}

template <typename F>
int guarded(F&& body) {
    try {
        body();
        return 0;
    } catch (const std::exception& e) {
        return fail_status(e);
    } catch (...) {
        g_error = "unknown failure";
        return 1 + static_cast<int>(ustats::ErrorCode::InvalidArgument);
    }
}

ustats::Config to_config(const us_config* c) {
    ustats::Config cfg;
    if (!c) return cfg;
    if (c->memory_cap_entries) cfg.memory_cap_entries = c->memory_cap_entries;
    cfg.threads = c->threads;
    if (c->strategy < 0 || c->strategy > 3)
        ustats::fail(ustats::ErrorCode::InvalidArgument, "unknown order strategy");
    cfg.strategy = static_cast<ustats::OrderStrategy>(c->strategy);
    if (c->exhaustive_index_bound) cfg.exhaustive_index_bound = c->exhaustive_index_bound;
    if (c->exact_treewidth_bound) cfg.exact_treewidth_bound = c->exact_treewidth_bound;
    cfg.device.device = c->device;
    cfg.device.rank = c->rank;
    cfg.device.world_size = c->world_size < 1 ? 1 : c->world_size;
    if (cfg.device.rank < 0 || cfg.device.rank >= cfg.device.world_size)
        ustats::fail(ustats::ErrorCode::InvalidArgument, "rank outside [0, world_size)");
    cfg.device.share_subexpressions = c->flags & 1;
    cfg.device.fuse_epilogues = c->flags & 2;
    cfg.device.exploit_symmetry = c->flags & 4;
    cfg.device.reorder_for_sharing = c->flags & 8;
    cfg.device.donate_inputs = c->flags & 16;
    cfg.device.shard_rows = c->flags & 32;
    cfg.device.serial_launch = c->flags & 64;
    cfg.device.fp64_emulation = !(c->flags & 128);
    cfg.device.graph_replay = !(c->flags & 256);
    cfg.device.emulate_world = c->emulate_world;
    cfg.device.memory_budget_bytes = c->memory_budget_bytes;
    if (c->oz_slices != 0 && (c->oz_slices < 4 || c->oz_slices > 7))
        ustats::fail(ustats::ErrorCode::InvalidArgument, "oz_slices must be 0 (auto) or 4..7");
    cfg.device.oz_slices = c->oz_slices;
    if (c->oz_max_k < 0 || (c->oz_max_k > 0 && c->oz_max_k < 64))
        ustats::fail(ustats::ErrorCode::InvalidArgument, "oz_max_k must be 0 (auto) or >= 64");
    cfg.device.oz_max_k = c->oz_max_k;
    if (c->oz_min_dim < 0 || (c->oz_min_dim > 0 && c->oz_min_dim < 128))
        ustats::fail(ustats::ErrorCode::InvalidArgument, "oz_min_dim must be 0 (1024) or >= 128");
    cfg.device.oz_min_dim = c->oz_min_dim;
    return cfg;
}

std::vector<ustats::IndexTuple> decode(int32_t K, const int32_t* len, const int32_t* idx) {
    if (K < 1) ustats::fail(ustats::ErrorCode::InvalidArgument, "need at least one component");
    std::vector<ustats::IndexTuple> sig;
    int off = 0;
    for (int k = 0; k < K; ++k) {
        if (len[k] < 0) ustats::fail(ustats::ErrorCode::InvalidArgument, "negative tuple length");
        sig.emplace_back(idx + off, idx + off + len[k]);
        off += len[k];
    }
    return sig;
}

// MDKernel::validate (kernel.cpp:10-37) on the 0-based encoding.
void validate_signature(int m, const std::vector<ustats::IndexTuple>& sig) {
    if (m < 1) ustats::fail(ustats::ErrorCode::InvalidArgument, "kernel arity must be >= 1");
    std::vector<char> covered(static_cast<std::size_t>(m), 0);
    for (const auto& t : sig) {
        if (t.empty()) ustats::fail(ustats::ErrorCode::InvalidArgument, "signature tuples must be non-empty");
        std::vector<char> here(static_cast<std::size_t>(m), 0);
        for (int s : t) {
            if (s < 0 || s >= m)
                ustats::fail(ustats::ErrorCode::InvalidArgument,
                             "signature slot " + std::to_string(s + 1) + " outside 1.." + std::to_string(m));
            if (here[static_cast<std::size_t>(s)])
                ustats::fail(ustats::ErrorCode::InvalidArgument,
                             "signature slot " + std::to_string(s + 1) + " repeated within one tuple");
            here[static_cast<std::size_t>(s)] = covered[static_cast<std::size_t>(s)] = 1;
        }
    }
    for (int s = 0; s < m; ++s)
        if (!covered[static_cast<std::size_t>(s)])
            ustats::fail(ustats::ErrorCode::InvalidArgument,
                         "argument slot " + std::to_string(s + 1) + " appears in no signature tuple");
}

void export_stats(const ustats::RunStats& rs, us_stats* s) {
    if (!s) return;
    s->tensorize_seconds = rs.tensorize_seconds;
    s->contract_seconds = rs.contract_seconds;
    s->einsum_calls = rs.einsum_calls;
    s->partitions_enumerated = rs.partitions_enumerated;
    s->partitions_evaluated = rs.partitions_evaluated;
    s->multiply_adds = rs.multiply_adds;
    s->peak_intermediate_entries = rs.peak_intermediate_entries;
    s->executed_gemm_macs = rs.executed_gemm_macs;
    s->executed_stream_entries = rs.executed_stream_entries;
    s->gemm_launches = rs.gemm_launches;
    s->stream_launches = rs.stream_launches;
    s->shared_hits = rs.shared_hits;
    s->kernel_launches = 0;
    s->emulated_gemm_macs = 0;
    s->int8_tensor_ops = 0;
    s->oz_slices = 0;
}

void export_dev(const ustats::dev::StatisticResult& r, int rank, us_stats* s) {
    if (!s) return;
    ustats::RunStats rs;
    rs.tensorize_seconds = r.upload_seconds;
    rs.contract_seconds = r.contract_seconds;
    std::uint64_t mine = 0;
    for (int o : r.owner) mine += o == rank;
    rs.einsum_calls = mine;
    rs.partitions_enumerated = r.enumerated;
    rs.partitions_evaluated = mine;
    rs.multiply_adds = r.stats.ref_madds;
    rs.peak_intermediate_entries = r.stats.ref_peak;
    rs.executed_gemm_macs = r.stats.gemm_macs;
    rs.executed_stream_entries = r.stats.stream_entries;
    rs.gemm_launches = r.stats.gemm_launches;
    rs.stream_launches = r.stats.stream_launches;
    rs.shared_hits = r.stats.shared_hits;
    export_stats(rs, s);
    s->kernel_launches = r.stats.kernel_launches;
    s->emulated_gemm_macs = r.stats.emulated_macs;
    s->int8_tensor_ops = r.stats.int8_ops;
    s->oz_slices = r.stats.oz_slices;
}

ustats::dev::StatisticResult run_lattice(int32_t m, int32_t K, const int32_t* tuple_len,
                                         const int32_t* tuple_idx, const double* const* factors, int64_t n,
                                         int32_t on_device, const us_config* cfg,
                                         ustats::dev::LatticeMode mode) {
    ustats::Config config = to_config(cfg);
    auto sig = decode(K, tuple_len, tuple_idx);
    validate_signature(m, sig);
    if (n < 1) ustats::fail(ustats::ErrorCode::InvalidArgument, "sample is empty");
    if (n < m)
        ustats::fail(ustats::ErrorCode::SampleTooSmall,
                     "need at least " + std::to_string(m) + " observations, have " + std::to_string(n));
    std::vector<const double*> ptrs(factors, factors + K);
    return ustats::dev::lattice_statistic(ptrs, on_device != 0, sig, m, n, mode, config);
}

std::vector<ustats::DenseTensor> host_tensors(const std::vector<ustats::IndexTuple>& sig,
                                              const double* const* data, int64_t n,
                                              const ustats::Config& config) {
    std::vector<ustats::DenseTensor> ts;
    for (std::size_t k = 0; k < sig.size(); ++k) {
        ustats::DenseTensor t(static_cast<int>(sig[k].size()), static_cast<int>(n), config);
        std::memcpy(t.data.data(), data[k], t.data.size() * sizeof(double));
        ts.push_back(std::move(t));
    }
    return ts;
}

}  // namespace

extern "C" {

const char* us_version(void) { return "ustats_b200 0.1 (sm_100a)"; }
const char* us_last_error(void) { return g_error.c_str(); }

void us_config_default(us_config* cfg) {
    std::memset(cfg, 0, sizeof(*cfg));
    cfg->device = -1;
    cfg->world_size = 1;
    cfg->flags = US_FLAGS_DEFAULT;
}

int us_u_statistic(int32_t m, int32_t K, const int32_t* tuple_len, const int32_t* tuple_idx,
                   const double* const* factors, int64_t n, int32_t on_device, const us_config* cfg,
                   double* u_out, us_stats* stats) {
    return guarded([&] {
        auto r = run_lattice(m, K, tuple_len, tuple_idx, factors, n, on_device, cfg,
                             ustats::dev::LatticeMode::Sparsified);
        *u_out = r.value;
        export_dev(r, cfg ? cfg->rank : 0, stats);
    });
}

int us_u_terms(int32_t m, int32_t K, const int32_t* tuple_len, const int32_t* tuple_idx,
               const double* const* factors, int64_t n, int32_t on_device, const us_config* cfg,
               int32_t max_terms, int32_t* count, int32_t* rgs_out, int64_t* mu_out, double* v_out,
               int32_t* owner_out, double* u_out, us_stats* stats) {
    return guarded([&] {
        auto r = run_lattice(m, K, tuple_len, tuple_idx, factors, n, on_device, cfg,
                             ustats::dev::LatticeMode::Sparsified);
        const int T = static_cast<int>(r.v.size());
        *count = T;
        if (T > max_terms) ustats::fail(ustats::ErrorCode::TooManyTerms, "term buffer too small");
        for (int t = 0; t < T; ++t) {
            for (int i = 0; i < m; ++i) rgs_out[t * m + i] = r.rgs[static_cast<std::size_t>(t)][static_cast<std::size_t>(i)];
            mu_out[t] = r.mu[static_cast<std::size_t>(t)];
            v_out[t] = r.v[static_cast<std::size_t>(t)];
            if (owner_out) owner_out[t] = r.owner[static_cast<std::size_t>(t)];
        }
        if (u_out) *u_out = r.value;
        export_dev(r, cfg ? cfg->rank : 0, stats);
    });
}

int us_u_statistic_data(const char* kernel, const double* data, int64_t n, int32_t d, int32_t on_device,
                        const us_config* cfg, double* u_out, us_stats* stats) {
    return guarded([&] {
        ustats::Config config = to_config(cfg);
        if (!kernel) ustats::fail(ustats::ErrorCode::InvalidArgument, "null kernel spec");
        if (n < 1 || d < 1) ustats::fail(ustats::ErrorCode::InvalidArgument, "data must be a non-empty n x d array");
        double tz = 0;
        auto r = ustats::dev::u_statistic_data(kernel, data, n, d, on_device != 0, config, &tz);
        *u_out = r.value;
        export_dev(r, cfg ? cfg->rank : 0, stats);
        if (stats) stats->tensorize_seconds = tz;
    });
}

int us_dcov_squared(const double* x, int32_t dx, const double* y, int32_t dy, int64_t n, int32_t on_device,
                    const us_config* cfg, double* out, us_stats* stats) {
    return guarded([&] {
        if (!x || !y || !out) ustats::fail(ustats::ErrorCode::InvalidArgument, "null argument");
        auto r = ustats::dev::dcov_squared(x, dx, y, dy, n, on_device != 0, to_config(cfg));
        *out = r.value;
        export_dev(r, cfg ? cfg->rank : 0, stats);
    });
}

int us_hoif_tau(int32_t m, int32_t k, const double* data, int64_t n, int32_t d, int32_t on_device, const us_config* cfg,
                double* tau_out, us_stats* stats) {
    return guarded([&] {
        if (!data || !tau_out) ustats::fail(ustats::ErrorCode::InvalidArgument, "null argument");
        auto r = ustats::dev::hoif_tau_data(m, k, data, n, d, on_device != 0, to_config(cfg));
        *tau_out = r.value;
        export_dev(r, cfg ? cfg->rank : 0, stats);
    });
}

int us_motif_count(int64_t n, int64_t edge_count, const int32_t* edges, const char* motif_id, const us_config* cfg,
                   int64_t* count, us_stats* stats) {
    return guarded([&] {
        if (!motif_id || !count || (edge_count > 0 && !edges) || edge_count < 0)
            ustats::fail(ustats::ErrorCode::InvalidArgument, "null argument");
        long long c = 0;
        auto r = ustats::dev::motif_count(n, edges, edge_count, motif_id, to_config(cfg), &c);
        *count = c;
        export_dev(r, cfg ? cfg->rank : 0, stats);
    });
}

int us_u_statistic_batch(int32_t S, const int32_t* m, const int32_t* K, const int32_t* tuple_len,
                         const int32_t* tuple_idx, const double* const* factors, int64_t n, int32_t on_device,
                         const us_config* cfg, double* u_out, us_stats* stats) {
    return guarded([&] {
        ustats::Config config = to_config(cfg);
        if (S < 1) ustats::fail(ustats::ErrorCode::InvalidArgument, "need at least one statistic");
        if (n < 1) ustats::fail(ustats::ErrorCode::InvalidArgument, "sample is empty");
        std::vector<ustats::dev::StatisticSpec> specs;
        int comp = 0, idx = 0;
        for (int s = 0; s < S; ++s) {
            ustats::dev::StatisticSpec sp;
            sp.m = m[s];
            for (int k = 0; k < K[s]; ++k) {
                sp.sig.emplace_back(tuple_idx + idx, tuple_idx + idx + tuple_len[comp]);
                idx += tuple_len[comp];
                sp.inputs.push_back(factors[comp]);
                ++comp;
            }
            validate_signature(sp.m, sp.sig);
            if (n < sp.m)
                ustats::fail(ustats::ErrorCode::SampleTooSmall,
                             "need at least " + std::to_string(sp.m) + " observations, have " + std::to_string(n));
            specs.push_back(std::move(sp));
        }
        auto res = ustats::dev::lattice_batch(specs, on_device != 0, n, ustats::dev::LatticeMode::Sparsified, config);
        for (int s = 0; s < S; ++s) u_out[s] = res[static_cast<std::size_t>(s)].value;
        if (stats) export_dev(res[0], cfg ? cfg->rank : 0, stats);
    });
}

int us_u_statistic_unsparsified(int32_t m, int32_t K, const int32_t* tuple_len, const int32_t* tuple_idx,
                                const double* const* factors, int64_t n, int32_t on_device,
                                const us_config* cfg, double* u_out, us_stats* stats) {
    return guarded([&] {
        auto r = run_lattice(m, K, tuple_len, tuple_idx, factors, n, on_device, cfg,
                             ustats::dev::LatticeMode::Unsparsified);
        *u_out = r.value;
        export_dev(r, cfg ? cfg->rank : 0, stats);
    });
}

int us_v_statistic(int32_t m, int32_t K, const int32_t* tuple_len, const int32_t* tuple_idx,
                   const double* const* factors, int64_t n, const us_config* cfg, double* v_out,
                   us_stats* stats) {
    return guarded([&] {
        ustats::Config config = to_config(cfg);
        auto sig = decode(K, tuple_len, tuple_idx);
        validate_signature(m, sig);
        if (n < 1) ustats::fail(ustats::ErrorCode::InvalidArgument, "sample is empty");
        auto ts = host_tensors(sig, factors, n, config);
        ustats::EinsumNotation notation(sig);
        ustats::ExecStats es;
        ustats::RunStats rs;
        *v_out = ustats::einsum(ts, notation, config, nullptr, &es).scalar();
        rs.einsum_calls = 1;
        rs.multiply_adds = es.multiply_adds;
        rs.peak_intermediate_entries = es.peak_intermediate_entries;
        export_stats(rs, stats);
    });
}

int us_restricted_v(int32_t m, int32_t K, const int32_t* tuple_len, const int32_t* tuple_idx,
                    const double* const* factors, int64_t n, const int32_t* rgs, const us_config* cfg,
                    double* v_out, us_stats* stats) {
    return guarded([&] {
        ustats::Config config = to_config(cfg);
        auto sig = decode(K, tuple_len, tuple_idx);
        validate_signature(m, sig);
        ustats::SetPartition part(std::vector<int>(rgs, rgs + m));
        auto ts = host_tensors(sig, factors, n, config);
        ustats::EinsumNotation notation(ustats::induced_signature(sig, part));
        ustats::ExecStats es;
        *v_out = ustats::einsum(ts, notation, config, nullptr, &es).scalar();
        ustats::RunStats rs;
        rs.einsum_calls = 1;
        rs.multiply_adds = es.multiply_adds;
        rs.peak_intermediate_entries = es.peak_intermediate_entries;
        export_stats(rs, stats);
    });
}

int us_einsum(int32_t K, const int32_t* tuple_len, const int32_t* tuple_idx, const double* const* tensors,
              int64_t n, int32_t out_len, const int32_t* out_idx, const int32_t* order, int32_t order_len,
              const us_config* cfg, double* out, uint64_t* multiply_adds, uint64_t* peak_entries,
              int32_t* steps) {
    return guarded([&] {
        ustats::Config config = to_config(cfg);
        if (K < 1) ustats::fail(ustats::ErrorCode::InvalidNotation, "a notation needs at least one input tuple");
        std::vector<ustats::IndexTuple> raw;
        int off = 0;
        for (int k = 0; k < K; ++k) {
            raw.emplace_back(tuple_idx + off, tuple_idx + off + tuple_len[k]);
            off += tuple_len[k];
        }
        ustats::EinsumNotation notation =
            ustats::validate_notation(raw, ustats::IndexTuple(out_idx, out_idx + out_len));
        std::vector<ustats::DenseTensor> ts;
        for (int k = 0; k < K; ++k) {
            ustats::DenseTensor t(tuple_len[k], static_cast<int>(n), config);
            std::memcpy(t.data.data(), tensors[k], t.data.size() * sizeof(double));
            ts.push_back(std::move(t));
        }
        ustats::EliminationOrder eo;
        const ustats::EliminationOrder* eop = nullptr;
        if (order) {
            eo.order.assign(order, order + order_len);
            eop = &eo;
        }
        ustats::ExecStats es;
        ustats::DenseTensor r = ustats::einsum(ts, notation, config, eop, &es);
        std::memcpy(out, r.data.data(), r.data.size() * sizeof(double));
        if (multiply_adds) *multiply_adds = es.multiply_adds;
        if (peak_entries) *peak_entries = es.peak_intermediate_entries;
        if (steps) *steps = es.steps;
    });
}

int us_eliminate_index(int32_t K, const int32_t* tuple_len, const int32_t* tuple_idx,
                       const double* const* tensors, int64_t n, int32_t index, const us_config* cfg,
                       double* out, uint64_t out_cap, int32_t* out_tuple, int32_t* out_tuple_len) {
    return guarded([&] {
        ustats::Config config = to_config(cfg);
        if (K < 1) ustats::fail(ustats::ErrorCode::ShapeMismatch, "need one tuple per tensor");
        std::vector<ustats::IndexTuple> tuples;
        std::vector<ustats::DenseTensor> ts;
        int off = 0;
        for (int k = 0; k < K; ++k) {
            tuples.emplace_back(tuple_idx + off, tuple_idx + off + tuple_len[k]);
            off += tuple_len[k];
            ustats::DenseTensor t(tuple_len[k], static_cast<int>(n), config);
            std::memcpy(t.data.data(), tensors[k], t.data.size() * sizeof(double));
            ts.push_back(std::move(t));
        }
        auto [r, tuple] = ustats::eliminate_index(ts, tuples, index, config);
        if (r.data.size() > out_cap) ustats::fail(ustats::ErrorCode::InvalidArgument, "output buffer too small");
        std::memcpy(out, r.data.data(), r.data.size() * sizeof(double));
        for (std::size_t i = 0; i < tuple.size(); ++i) out_tuple[i] = tuple[i];
        *out_tuple_len = static_cast<int32_t>(tuple.size());
    });
}

double us_combine_terms(int32_t count, const int64_t* mu, const double* v) {
    std::vector<double> terms(static_cast<std::size_t>(count < 0 ? 0 : count));
    for (std::size_t t = 0; t < terms.size(); ++t) terms[t] = static_cast<double>(mu[t]) * v[t];
    return ustats::dev::combine_terms(terms);
}

uint64_t us_bell_number(int32_t m) {
    try {
        return ustats::bell_number(m);
    } catch (const std::exception& e) {
        g_error = e.what();
        return 0;
    }
}

int us_survivors(int32_t m, int32_t K, const int32_t* tuple_len, const int32_t* tuple_idx, int32_t max_terms,
                 int32_t* count, int32_t* rgs_out, int64_t* mu_out, uint64_t* enumerated) {
    return guarded([&] {
        auto sig = decode(K, tuple_len, tuple_idx);
        ustats::SparsifiedPartitionStream s(m, sig);
        ustats::SetPartition p;
        int c = 0;
        while (s.next(p)) {
            if (c < max_terms) {
                for (int i = 0; i < m; ++i) rgs_out[c * m + i] = p.rgs()[static_cast<std::size_t>(i)];
                mu_out[c] = ustats::mobius_coefficient(p);
            }
            ++c;
        }
        *count = c;
        if (enumerated) *enumerated = s.enumerated();
        if (c > max_terms) ustats::fail(ustats::ErrorCode::TooManyTerms, "term buffer too small");
    });
}

int us_optimize_order(int32_t K, const int32_t* tuple_len, const int32_t* tuple_idx, int32_t strategy,
                      int32_t* order_out, int32_t* index_count, int32_t* width_out) {
    return guarded([&] {
        std::vector<ustats::IndexTuple> raw;
        int off = 0;
        for (int k = 0; k < K; ++k) {
            raw.emplace_back(tuple_idx + off, tuple_idx + off + tuple_len[k]);
            off += tuple_len[k];
        }
        ustats::EinsumNotation notation(raw);
        if (strategy < 0 || strategy > 3) ustats::fail(ustats::ErrorCode::InvalidArgument, "unknown strategy");
        auto o = ustats::optimize_order(notation, 2, static_cast<ustats::OrderStrategy>(strategy));
        for (std::size_t i = 0; i < o.order.size(); ++i) order_out[i] = o.order[i];
        *index_count = notation.index_count;
        *width_out = o.predicted_width;
    });
}

int us_complexity_report(int32_t K, const int32_t* tuple_len, const int32_t* tuple_idx, int32_t extent,
                         const us_config* cfg, us_complexity* out, char* flops, int32_t cap) {
    return guarded([&] {
        if (K < 0 || (K > 0 && (!tuple_len || !tuple_idx)) || !out)
            ustats::fail(ustats::ErrorCode::InvalidArgument, "null argument");
        std::vector<ustats::IndexTuple> raw;
        int off = 0;
        for (int k = 0; k < K; ++k) {
            raw.emplace_back(tuple_idx + off, tuple_idx + off + tuple_len[k]);
            off += tuple_len[k];
        }
        const auto r = ustats::complexity_report(raw, extent, to_config(cfg));
        us_complexity c{};
        c.index_count = r.index_count;
        c.extent = r.extent;
        c.graph_vertices = r.graph_vertices;
        c.graph_edges = r.graph_edges;
        c.treewidth_lower = r.treewidth_lower;
        c.treewidth_upper = r.treewidth_upper;
        c.treewidth_exact = r.treewidth_exact ? *r.treewidth_exact : -1;
        c.max_quotient_width = r.max_quotient_width;
        c.bell_count = r.bell_count;
        c.sparsified_count = r.sparsified_count;
        for (const auto& [w, count] : r.count_by_width)
            if (w >= 0 && w < 16) c.count_by_width[w] = count;
        *out = c;
        if (flops && cap > 0) {
            if (static_cast<int32_t>(r.flops_estimate.size()) >= cap)
                ustats::fail(ustats::ErrorCode::InvalidArgument, "flops buffer too small");
            std::copy(r.flops_estimate.begin(), r.flops_estimate.end(), flops);
            flops[r.flops_estimate.size()] = '\0';
        }
    });
}

int us_treewidth(int32_t n, int32_t edge_count, const int32_t* edges, int32_t* width_out, int32_t* order_out) {
    return guarded([&] {
        std::vector<std::pair<int, int>> es;
        for (int i = 0; i < edge_count; ++i) es.emplace_back(edges[2 * i], edges[2 * i + 1]);
        auto g = ustats::SimpleGraph::from_edges(n, es);
        ustats::Config c;
        c.exact_treewidth_bound = std::max(c.exact_treewidth_bound, g.vertex_count());
        auto r = ustats::treewidth_exact(g, c);
        *width_out = r.width;
        for (std::size_t i = 0; i < r.order.size(); ++i) order_out[i] = r.order[i];
    });
}

int us_plan_terms(int32_t m, int32_t K, const int32_t* tuple_len, const int32_t* tuple_idx, int64_t n,
                  int32_t world_size, int32_t max_terms, int32_t* count, int32_t* owner_out, double* cost_out) {
    return guarded([&] {
        auto sig = decode(K, tuple_len, tuple_idx);
        validate_signature(m, sig);
        ustats::Config config;
        config.device.world_size = world_size < 1 ? 1 : world_size;
        auto plan = ustats::dev::plan_terms(sig, m, n, ustats::dev::LatticeMode::Sparsified, config);
        const int T = static_cast<int>(plan.owner.size());
        *count = T;
        if (T > max_terms) ustats::fail(ustats::ErrorCode::TooManyTerms, "term buffer too small");
        for (int t = 0; t < T; ++t) {
            owner_out[t] = plan.owner[static_cast<std::size_t>(t)];
            if (cost_out) cost_out[t] = plan.cost[static_cast<std::size_t>(t)];
        }
    });
}

int us_plan_summary(int32_t m, int32_t K, const int32_t* tuple_len, const int32_t* tuple_idx, int64_t n,
                    const us_config* cfg, int32_t inputs_symmetric, char* text, uint64_t cap, uint64_t* totals) {
    return guarded([&] {
        auto sig = decode(K, tuple_len, tuple_idx);
        validate_signature(m, sig);
        ustats::Config config = to_config(cfg);
        ustats::dev::Program::Totals t;
        std::string s = ustats::dev::plan_summary(sig, m, n, config, inputs_symmetric != 0, &t);
        if (text && cap) {
            const std::size_t k = std::min<std::size_t>(s.size(), cap - 1);
            std::memcpy(text, s.data(), k);
            text[k] = 0;
        }
        if (totals) {
            totals[0] = t.gemms;
            totals[1] = t.gemm_macs;
            totals[2] = t.streams;
            totals[3] = t.stream_entries;
            totals[4] = t.fused;
            totals[5] = t.symmetric;
            totals[6] = t.peak_entries;
        }
    });
}

int us_nccl_unique_id(void* id_out) {
    return guarded([&] { ustats::dev::Runtime::nccl_unique_id(id_out); });
}

int us_nccl_init(int32_t device, int32_t rank, int32_t world_size, const void* id) {
    return guarded([&] { ustats::dev::Runtime::get(device).nccl_init(rank, world_size, id); });
}

int us_device_count(int32_t* count) {
    return guarded([&] {
        int c = 0;
        ustats::dev::check_cuda(cudaGetDeviceCount(&c), "cudaGetDeviceCount");
        *count = c;
    });
}

int us_device_synchronize(int32_t device) {
    return guarded([&] { ustats::dev::Runtime::get(device).sync(); });
}

int us_dgemm(int32_t method, int32_t slices, int32_t symmetric, int64_t m, int64_t n, int64_t k, const double* a,
             const double* b, double* c, double* ms_out) {
    return guarded([&] {
        using namespace ustats::dev;
        if (m < 1 || n < 1 || k < 1 || !a || !b || !c) ustats::fail(ustats::ErrorCode::InvalidArgument, "bad GEMM shape");
        if (symmetric && m != n) ustats::fail(ustats::ErrorCode::InvalidArgument, "symmetric GEMM needs m = n");
        Runtime& rt = Runtime::get(-1);
        cudaStream_t s = rt.main_stream();
        rt.set_stream(s);
        Buf da = rt.allocate(1, m * k), db = rt.allocate(1, n * k), dc = rt.allocate(1, m * n);
        check_cuda(cudaMemcpyAsync(da->ptr, a, sizeof(double) * m * k, cudaMemcpyHostToDevice, s), "H2D");
        check_cuda(cudaMemcpyAsync(db->ptr, b, sizeof(double) * n * k, cudaMemcpyHostToDevice, s), "H2D");
        check_cuda(cudaMemsetAsync(dc->ptr, 0, sizeof(double) * m * n, s), "memset");
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        int8_t *sa = nullptr, *sb = nullptr;
        int *ea = nullptr, *eb = nullptr;
        if (method == 1) {
            if (slices < 4 || slices > kOzMaxSlices) ustats::fail(ustats::ErrorCode::InvalidArgument, "slices must be 4..7");
            const std::size_t abytes = ozaki_slice_bytes(m, k, 128), bbytes = ozaki_slice_bytes(n, k, 128);
            check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&sa), abytes * slices, s), "alloc");
            check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&sb), bbytes * slices, s), "alloc");
            check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&ea), sizeof(int) * m, s), "alloc");
            check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&eb), sizeof(int) * n, s), "alloc");
            cudaEventRecord(e0, s);
            ozaki_split(da->ptr, m, k, k, 1, 128, slices, sa, ea, s);
            ozaki_split(db->ptr, n, k, k, 1, 128, slices, sb, eb, s);
            OzakiArgs p;
            p.a = sa;
            p.b = sb;
            p.a_slice = static_cast<long long>(abytes);
            p.b_slice = static_cast<long long>(bbytes);
            p.a_exp = ea;
            p.b_exp = eb;
            p.m = m;
            p.n = n;
            p.mpad = (m + 127) / 128 * 128;
            p.npad = (n + 127) / 128 * 128;
            p.kpad = (k + 63) / 64 * 64;
            p.slices = slices;
            p.symmetric = symmetric ? 1 : 0;
            p.epis.count = 1;
            p.epis.d[0].mode = kEpiStore;
            p.epis.d[0].out = dc->ptr;
            double* work = nullptr;
            check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&work), ozaki_work_entries() * sizeof(double), s), "alloc");
            p.work = work;
            const int launched = launch_ozaki_gemm(p, s);
            cudaFreeAsync(work, s);
            if (launched < 0)
                ustats::fail(ustats::ErrorCode::InvalidArgument, "Ozaki GEMM: slices * k * 128^2 must stay below 2^31");
            cudaEventRecord(e1, s);
        } else {
            GemmArgs g;
            g.a.nf = g.b.nf = 1;
            g.a.nr = g.b.nr = 1;
            g.a.ptr[0] = da->ptr;
            g.b.ptr[0] = db->ptr;
            g.a.rstride[0][0] = k;
            g.b.rstride[0][0] = k;
            g.a.kstride[0] = g.b.kstride[0] = 1;
            g.n = k;
            g.rows = m;
            g.cols = n;
            g.a_kmajor = g.b_kmajor = 1;
            g.symmetric_out = symmetric ? 1 : 0;
            EpiSet e;
            e.count = 1;
            e.d[0].mode = kEpiStore;
            e.d[0].out = dc->ptr;
            cudaEventRecord(e0, s);
            // the TMA-fed DMMA kernel (the executor's gather fallback assumes every
            // extent equals n, as in a U-statistic; it is not exposed here)
            if (launch_gemm_multi(g, e, s) < 0)
                ustats::fail(ustats::ErrorCode::InvalidArgument, "dmma test GEMM needs an even k (16-byte aligned rows)");
            cudaEventRecord(e1, s);
        }
        check_cuda(cudaGetLastError(), "dgemm launch");
        check_cuda(cudaMemcpyAsync(c, dc->ptr, sizeof(double) * m * n, cudaMemcpyDeviceToHost, s), "D2H");
        check_cuda(cudaStreamSynchronize(s), "sync");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms_out) *ms_out = ms;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        if (sa) cudaFree(sa);
        if (sb) cudaFree(sb);
        if (ea) cudaFree(ea);
        if (eb) cudaFree(eb);
    });
}

int us_graph_replays(int32_t device, uint64_t* count_out) {
    return guarded([&] { *count_out = ustats::dev::graph_replays(ustats::dev::Runtime::get(device).device()); });
}

int us_device_stream(int32_t device, void** stream_out) {
    return guarded([&] { *stream_out = static_cast<void*>(ustats::dev::Runtime::get(device).stream()); });
}

int us_profile(int32_t device, int32_t enable, int32_t reset, double* ms_out, uint64_t* groups_out) {
    return guarded([&] {
        auto& rt = ustats::dev::Runtime::get(device);
        auto p = rt.collect(reset != 0);
        rt.profile_enable(enable != 0);
        for (int i = 0; i < 3; ++i) {
            if (ms_out) ms_out[i] = p.ms[i];
            if (groups_out) groups_out[i] = p.groups[i];
        }
    });
}

}  // extern "C"
