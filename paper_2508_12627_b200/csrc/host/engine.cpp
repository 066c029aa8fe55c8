// Statistic entry points and tensor-level einsum of the host API
// (proj/src/engine.cpp:108-211, proj/src/einsum.cpp:380-486 boundaries).
// Tensorization stays on the host (caller callbacks); everything after it is
// the device executor's.
#include "ustats/engine.hpp"

#include <chrono>
#include <cmath>
#include <exception>
#include <set>
#include <string>

#include "../device/executor.hpp"
#include "ustats/errors.hpp"

namespace ustats {

namespace {
using Clock = std::chrono::steady_clock;
double since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

void merge(RunStats& rs, const dev::DevStats& ds, std::uint64_t calls) {
    rs.einsum_calls += calls;
    rs.multiply_adds += ds.ref_madds;
    rs.peak_intermediate_entries = std::max(rs.peak_intermediate_entries, ds.ref_peak);
    rs.executed_gemm_macs += ds.gemm_macs;
    rs.executed_stream_entries += ds.stream_entries;
    rs.gemm_launches += ds.gemm_launches;
    rs.stream_launches += ds.stream_launches;
    rs.shared_hits += ds.shared_hits;
}

std::vector<const double*> data_of(std::span<const DenseTensor> ts) {
    std::vector<const double*> p;
    for (const DenseTensor& t : ts) p.push_back(t.data.data());
    return p;
}

double lattice(std::span<const DenseTensor> tensors, const std::vector<IndexTuple>& zero_sig, int m,
               dev::LatticeMode mode, const Config& config, RunStats& rs, std::vector<double>* terms) {
    const int n = tensors.empty() ? 1 : tensors[0].extent;
    for (std::size_t k = 0; k < tensors.size(); ++k) {
        if (tensors[k].extent != n) fail(ErrorCode::ShapeMismatch, "tensors disagree on extent");
        if (tensors[k].order != static_cast<int>(zero_sig[k].size()))
            fail(ErrorCode::ShapeMismatch, "tensor order does not match its signature tuple");
    }
    dev::StatisticResult r =
        dev::lattice_statistic(data_of(tensors), false, zero_sig, m, n, mode, config);
    rs.tensorize_seconds += r.upload_seconds;  // sparsify is tensorize time (engine.cpp:184-186)
    rs.contract_seconds += r.contract_seconds;
    std::uint64_t mine = 0;
    for (int o : r.owner) mine += o == config.device.rank;
    merge(rs, r.stats, mine);
    rs.partitions_enumerated += r.enumerated;
    rs.partitions_evaluated += mine;
    if (terms) *terms = r.terms;
    return r.value;
}

void check_sample(const MDKernel& kernel, const Sample& sample) {
    if (sample.size() < kernel.arity)
        fail(ErrorCode::SampleTooSmall, "need at least " + std::to_string(kernel.arity) +
                                            " observations, have " + std::to_string(sample.size()));
}

double single_contraction(const std::vector<DenseTensor>& tensors, const EinsumNotation& notation,
                          const Config& config, RunStats& rs) {
    const auto t0 = Clock::now();
    std::vector<const double*> ptrs;
    std::vector<int> orders;
    for (const DenseTensor& t : tensors) {
        ptrs.push_back(t.data.data());
        orders.push_back(t.order);
    }
    dev::DevStats ds;
    std::vector<double> out =
        dev::contract_host(ptrs, orders, tensors.empty() ? 1 : tensors[0].extent, notation, nullptr, config, &ds);
    rs.contract_seconds += since(t0);
    merge(rs, ds, 1);
    return out.at(0);
}
}  // namespace

std::vector<DenseTensor> tensorize(const MDKernel& kernel, const Sample& sample, const Config& config,
                                   RunStats* stats) {
    kernel.validate();
    const int n = sample.size();
    if (n < 1) fail(ErrorCode::InvalidArgument, "sample is empty");
    const auto t0 = Clock::now();
    std::vector<DenseTensor> out;
    for (std::size_t k = 0; k < kernel.signature.size(); ++k) {
        auto entry = [&, k](std::span<const int> alpha) {
            double v = 0.0;
            try {
                v = kernel.components[k](sample, alpha);
            } catch (const std::exception& e) {
                fail(ErrorCode::ComponentEvaluationError,
                     "component " + std::to_string(k) + " failed: " + e.what());
            }
            if (config.strict_nonfinite && !std::isfinite(v))
                fail(ErrorCode::ComponentEvaluationError,
                     "component " + std::to_string(k) + " returned a non-finite value");
            return v;
        };
        out.push_back(tensor_from_function(static_cast<int>(kernel.signature[k].size()), n, entry, config));
    }
    if (stats) stats->tensorize_seconds += since(t0);
    return out;
}

double v_statistic(const MDKernel& kernel, const Sample& sample, const Config& config, RunStats* stats) {
    RunStats local;
    RunStats& rs = stats ? *stats : local;
    std::vector<DenseTensor> tensors = tensorize(kernel, sample, config, &rs);
    return single_contraction(tensors, EinsumNotation(kernel.zero_based_signature()), config, rs);
}

double restricted_v(const MDKernel& kernel, const Sample& sample, const SetPartition& partition,
                    const Config& config, RunStats* stats) {
    kernel.validate();
    if (partition.ground_size() != kernel.arity)
        fail(ErrorCode::GroundSetMismatch, "partition ground set has " +
                                               std::to_string(partition.ground_size()) +
                                               " elements, kernel arity is " + std::to_string(kernel.arity));
    RunStats local;
    RunStats& rs = stats ? *stats : local;
    std::vector<DenseTensor> tensors = tensorize(kernel, sample, config, &rs);
    return single_contraction(
        tensors, EinsumNotation(induced_signature(kernel.zero_based_signature(), partition)), config, rs);
}

double u_statistic(const MDKernel& kernel, const Sample& sample, const Config& config, RunStats* stats) {
    kernel.validate();
    check_sample(kernel, sample);
    RunStats local;
    RunStats& rs = stats ? *stats : local;
    std::vector<DenseTensor> tensors = tensorize(kernel, sample, config, &rs);
    return lattice(tensors, kernel.zero_based_signature(), kernel.arity, dev::LatticeMode::Sparsified, config,
                   rs, nullptr);
}

double u_statistic_unsparsified(const MDKernel& kernel, const Sample& sample, const Config& config,
                                RunStats* stats) {
    kernel.validate();
    check_sample(kernel, sample);
    RunStats local;
    RunStats& rs = stats ? *stats : local;
    std::vector<DenseTensor> tensors = tensorize(kernel, sample, config, &rs);
    return lattice(tensors, kernel.zero_based_signature(), kernel.arity, dev::LatticeMode::Unsparsified,
                   config, rs, nullptr);
}

double u_statistic_tensors(std::span<const DenseTensor> tensors, const std::vector<IndexTuple>& zero_sig,
                           int arity, const Config& config, RunStats* stats, std::vector<double>* terms) {
    if (tensors.size() != zero_sig.size())
        fail(ErrorCode::ShapeMismatch, "need one tensor per signature tuple");
    const int n = tensors.empty() ? 0 : tensors[0].extent;
    if (n < arity)
        fail(ErrorCode::SampleTooSmall,
             "need at least " + std::to_string(arity) + " observations, have " + std::to_string(n));
    RunStats local;
    RunStats& rs = stats ? *stats : local;
    return lattice(tensors, zero_sig, arity, dev::LatticeMode::Sparsified, config, rs, terms);
}

// ------------------------------------------------------------------ einsum
DenseTensor einsum(std::span<const DenseTensor> tensors, const EinsumNotation& notation, const Config& config,
                   const EliminationOrder* order, ExecStats* stats) {
    const std::size_t K = notation.inputs.size();
    if (tensors.size() != K)
        fail(ErrorCode::ShapeMismatch, "notation expects " + std::to_string(K) + " tensors, got " +
                                           std::to_string(tensors.size()));
    if (K == 0) fail(ErrorCode::InvalidNotation, "notation has no inputs");
    const int n = tensors[0].extent;
    for (std::size_t k = 0; k < K; ++k) {
        if (tensors[k].order != static_cast<int>(notation.inputs[k].size()))
            fail(ErrorCode::ShapeMismatch, "tensor " + std::to_string(k) + " has order " +
                                               std::to_string(tensors[k].order) + " but its tuple has " +
                                               std::to_string(notation.inputs[k].size()) + " indices");
        if (tensors[k].extent != n) fail(ErrorCode::ShapeMismatch, "tensors disagree on extent");
    }
    if (order) {
        if (static_cast<int>(order->order.size()) != notation.index_count)
            fail(ErrorCode::InvalidArgument, "elimination order must cover all indices");
        std::vector<char> seen(static_cast<std::size_t>(notation.index_count), 0);
        for (int v : order->order) {
            if (v < 0 || v >= notation.index_count || seen[static_cast<std::size_t>(v)])
                fail(ErrorCode::InvalidArgument, "elimination order is not a permutation");
            seen[static_cast<std::size_t>(v)] = 1;
        }
    }
    std::vector<const double*> ptrs;
    std::vector<int> orders;
    for (const DenseTensor& t : tensors) {
        ptrs.push_back(t.data.data());
        orders.push_back(t.order);
    }
    dev::DevStats ds;
    std::vector<double> host = dev::contract_host(ptrs, orders, n, notation, order, config, &ds);
    if (stats) {
        stats->multiply_adds += ds.ref_madds;
        stats->peak_intermediate_entries = std::max(stats->peak_intermediate_entries, ds.ref_peak);
        stats->steps += ds.steps;
    }
    DenseTensor out(static_cast<int>(notation.output.size()), n, config);
    out.data = std::move(host);
    return out;
}

std::pair<DenseTensor, IndexTuple> eliminate_index(std::span<const DenseTensor> tensors,
                                                   const std::vector<IndexTuple>& tuples, int index,
                                                   const Config& config, ExecStats* stats) {
    if (tensors.size() != tuples.size() || tensors.empty())
        fail(ErrorCode::ShapeMismatch, "need one tuple per tensor");
    const int n = tensors[0].extent;
    for (std::size_t k = 0; k < tensors.size(); ++k) {
        if (tensors[k].extent != n) fail(ErrorCode::ShapeMismatch, "tensors disagree on extent");
        if (tensors[k].order != static_cast<int>(tuples[k].size()))
            fail(ErrorCode::ShapeMismatch, "tensor order does not match its tuple");
        if (std::find(tuples[k].begin(), tuples[k].end(), index) == tuples[k].end())
            fail(ErrorCode::IndexAbsent, "tuple " + std::to_string(k) + " lacks index " + std::to_string(index));
        for (int id : tuples[k])
            if (id < 0 || id >= dev::kMaxIds)
                fail(ErrorCode::InvalidArgument, "index outside the device executor's range");
    }
    std::vector<const double*> ptrs;
    for (const DenseTensor& t : tensors) ptrs.push_back(t.data.data());
    dev::DevStats ds;
    IndexTuple tuple;
    std::vector<double> host = dev::eliminate_host(ptrs, tuples, n, index, config, &ds, &tuple);
    DenseTensor result(static_cast<int>(tuple.size()), n, config);
    result.data = std::move(host);
    if (stats) {
        stats->multiply_adds += ds.ref_madds;
        stats->peak_intermediate_entries = std::max(stats->peak_intermediate_entries, ds.ref_peak);
        stats->steps += ds.steps;
    }
    return {std::move(result), std::move(tuple)};
}

}  // namespace ustats
