// hoif_tau and its chain kernels (proj/src/hoif.cpp:10-100 boundary). The two
// distinct component matrices (middle, last) are tensorized once on the host
// (caller callbacks); every chain order 2..m is one StatisticSpec of a single
// device batch, so the orders share their sub-contractions (the reference
// evaluates them in m - 1 independent u_statistic calls, hoif.cpp:84-86).
#include "ustats/hoif.hpp"

#include <algorithm>
#include <string>
#include <utility>

#include "../device/executor.hpp"
#include "ustats/errors.hpp"

namespace ustats {

namespace {

const Observation& point(const Sample& s, int i) {
    const Observation& o = s.points[static_cast<std::size_t>(i)];
    if (o.size() < 2)
        fail(ErrorCode::InvalidArgument, "observation " + std::to_string(i) + " needs at least the A and Y coordinates");
    return o;
}

double basis_dot(const PhiFn& phi, const Observation& x, const Observation& y) {
    const std::vector<double> u = phi(HoifObservation::z(x)), v = phi(HoifObservation::z(y));
    if (u.size() != v.size()) fail(ErrorCode::InvalidArgument, "basis expansions disagree in length");
    double s = 0.0;
    for (std::size_t c = 0; c < u.size(); ++c) s += u[c] * v[c];  // coordinate order
    return s;
}

}  // namespace

PhiFn truncation_phi(int k) {
    if (k < 1) fail(ErrorCode::InvalidArgument, "basis size must be >= 1");
    return [k](std::span<const double> z) {
        if (static_cast<int>(z.size()) < k)
            fail(ErrorCode::InvalidArgument, "covariate block has " + std::to_string(z.size()) +
                                                 " coordinates, basis asks for " + std::to_string(k));
        return std::vector<double>(z.begin(), z.begin() + k);
    };
}

MDKernel hoif_kernel(int j, PhiFn phi) {
    if (j < 2) fail(ErrorCode::InvalidArgument, "sequential kernel needs order >= 2");
    MDKernel kernel;
    kernel.arity = j;
    kernel.name = "hoif:" + std::to_string(j);
    for (int i = 1; i < j; ++i) kernel.signature.push_back({i, i + 1});
    ComponentFn middle = [phi](const Sample& s, std::span<const int> idx) {
        const Observation& x = point(s, idx[0]);
        const Observation& y = point(s, idx[1]);
        return HoifObservation::a(x) * basis_dot(phi, x, y) * HoifObservation::a(y);
    };
    ComponentFn last = [phi](const Sample& s, std::span<const int> idx) {
        const Observation& x = point(s, idx[0]);
        const Observation& y = point(s, idx[1]);
        return HoifObservation::a(x) * basis_dot(phi, x, y) * HoifObservation::y(y);
    };
    kernel.components.assign(static_cast<std::size_t>(j - 2), middle);
    kernel.components.push_back(last);
    return kernel;
}

double hoif_tau(int m, const PhiFn& phi, const Sample& sample, const Config& config, RunStats* stats) {
    if (m < 2) fail(ErrorCode::InvalidArgument, "statistic order must be >= 2");
    const int n = sample.size();
    if (n < m) fail(ErrorCode::SampleTooSmall, "need at least " + std::to_string(m) + " observations, have " + std::to_string(n));
    // the distinct components once: [middle, last] (order 3) or [last] (order 2)
    RunStats local;
    RunStats& rs = stats ? *stats : local;
    const std::vector<DenseTensor> mats = tensorize(hoif_kernel(m > 2 ? 3 : 2, phi), sample, config, &rs);
    const double* last = mats.back().data.data();
    const double* middle = m > 2 ? mats.front().data.data() : nullptr;
    std::vector<dev::StatisticSpec> specs;
    for (int order = 2; order <= m; ++order) {
        dev::StatisticSpec sp;
        sp.m = order;
        for (int i = 0; i + 1 < order; ++i) {
            sp.sig.push_back({i, i + 1});
            sp.inputs.push_back(i + 2 < order ? middle : last);
        }
        specs.push_back(std::move(sp));
    }
    std::vector<dev::StatisticResult> res = dev::lattice_batch(specs, false, n, dev::LatticeMode::Sparsified, config);
    std::vector<double> u(static_cast<std::size_t>(m + 1), 0.0);
    for (int order = 2; order <= m; ++order) {
        const dev::StatisticResult& r = res[static_cast<std::size_t>(order - 2)];
        u[static_cast<std::size_t>(order)] = r.value;
        rs.multiply_adds += r.stats.ref_madds;
        rs.peak_intermediate_entries = std::max(rs.peak_intermediate_entries, r.stats.ref_peak);
        rs.partitions_enumerated += r.enumerated;
        rs.partitions_evaluated += r.rgs.size();
        rs.einsum_calls += r.rgs.size();
    }
    // the batch's device work is carried by its first statistic
    rs.contract_seconds += res[0].contract_seconds;
    rs.executed_gemm_macs += res[0].stats.gemm_macs;
    rs.executed_stream_entries += res[0].stats.stream_entries;
    rs.gemm_launches += res[0].stats.gemm_launches;
    rs.stream_launches += res[0].stats.stream_launches;
    rs.shared_hits += res[0].stats.shared_hits;
    return dev::hoif_combine(m, n, u);
}

}  // namespace ustats
