// Data-level entry: parse a kernel spec, tensorize its components on the
// device from the raw sample, evaluate the U-statistic (engine.cpp:173-193
// with tensorize, engine.cpp:108-136, moved to the GPU).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <map>
#include <memory>
#include <mutex>
#include <string>

#include "executor.hpp"
#include "kernels.hpp"
#include "tensorize.hpp"
#include "ustats/errors.hpp"
#include "ustats/partition.hpp"
#include "ustats/tensor.hpp"

namespace ustats::dev {

namespace {

std::vector<std::string> split(const std::string& s, char sep) {
    std::vector<std::string> out;
    std::string cur;
    for (char ch : s) {
        if (ch == sep) {
            out.push_back(cur);
            cur.clear();
        } else {
            cur += ch;
        }
    }
    out.push_back(cur);
    return out;
}

int to_int(const std::string& s, const std::string& spec) {
    try {
        std::size_t used = 0;
        const int v = std::stoi(s, &used);
        if (used != s.size()) throw std::invalid_argument(s);
        return v;
    } catch (const std::exception&) {
        fail(ErrorCode::InvalidArgument, "bad number '" + s + "' in kernel spec '" + spec + "'");
    }
}

double to_double(const std::string& s, const std::string& spec) {
    try {
        std::size_t used = 0;
        const double v = std::stod(s, &used);
        if (used != s.size()) throw std::invalid_argument(s);
        return v;
    } catch (const std::exception&) {
        fail(ErrorCode::InvalidArgument, "bad number '" + s + "' in kernel spec '" + spec + "'");
    }
}

// Cholesky G = R R^T (lower R) and M = R^{-T}, so Z G^{-1} Z^T = (Z M)(Z M)^T.
std::vector<double> inverse_cholesky_transpose(const std::vector<double>& G, int F) {
    std::vector<double> R(static_cast<std::size_t>(F * F), 0.0);
    for (int i = 0; i < F; ++i)
        for (int j = 0; j <= i; ++j) {
            long double s = G[static_cast<std::size_t>(i * F + j)];
            for (int k = 0; k < j; ++k) s -= static_cast<long double>(R[static_cast<std::size_t>(i * F + k)]) * R[static_cast<std::size_t>(j * F + k)];
            if (i == j) {
                if (s <= 0) fail(ErrorCode::InvalidArgument, "feature Gram matrix is not positive definite");
                R[static_cast<std::size_t>(i * F + i)] = static_cast<double>(std::sqrt(s));
            } else {
                R[static_cast<std::size_t>(i * F + j)] = static_cast<double>(s / R[static_cast<std::size_t>(j * F + j)]);
            }
        }
    // Rinv (lower) by forward substitution; M = Rinv^T
    std::vector<double> Rinv(static_cast<std::size_t>(F * F), 0.0);
    for (int c = 0; c < F; ++c)
        for (int i = c; i < F; ++i) {
            long double s = (i == c) ? 1.0L : 0.0L;
            for (int k = c; k < i; ++k) s -= static_cast<long double>(R[static_cast<std::size_t>(i * F + k)]) * Rinv[static_cast<std::size_t>(k * F + c)];
            Rinv[static_cast<std::size_t>(i * F + c)] = static_cast<double>(s / R[static_cast<std::size_t>(i * F + i)]);
        }
    std::vector<double> M(static_cast<std::size_t>(F * F), 0.0);
    for (int i = 0; i < F; ++i)
        for (int j = 0; j < F; ++j) M[static_cast<std::size_t>(i * F + j)] = Rinv[static_cast<std::size_t>(j * F + i)];
    return M;
}

}  // namespace

DataKernel parse_data_kernel(const std::string& spec, int d) {
    DataKernel k;
    const auto parts = split(spec, ':');
    const std::string& kind = parts[0];
    if (kind == "prod2" && parts.size() == 1) {
        if (d < 1) fail(ErrorCode::InvalidArgument, "prod2 needs at least one coordinate");
        k.m = 2;
        k.sig = {{0}, {1}};
        k.recipe = {"col:0", "col:0"};
        return k;
    }
    if (kind == "hoif" && parts.size() == 3) {  // hoif.cpp:50-72
        const int j = to_int(parts[1], spec), kk = to_int(parts[2], spec);
        if (j < 2) fail(ErrorCode::InvalidArgument, "sequential kernel needs order >= 2");
        if (kk < 1) fail(ErrorCode::InvalidArgument, "basis size must be >= 1");
        if (d < 2 + kk) fail(ErrorCode::InvalidArgument, "covariate block shorter than the basis");
        k.m = j;
        for (int i = 0; i + 1 < j; ++i) {
            k.sig.push_back({i, i + 1});
            k.recipe.push_back(i + 2 < j ? "gram:0:0:2:" + std::to_string(kk) : "gram:0:1:2:" + std::to_string(kk));
        }
        return k;
    }
    if (kind == "rbf" && parts.size() == 3) {
        const std::string& shape = parts[1];
        const double h = to_double(parts[2], spec);
        if (!(h > 0)) fail(ErrorCode::InvalidArgument, "RBF bandwidth must be positive");
        const std::string rec = "rbf:" + parts[2];
        if (shape.rfind("chain", 0) == 0 || shape.rfind("cycle", 0) == 0) {
            const int m = to_int(shape.substr(5), spec);
            if (m < 2) fail(ErrorCode::InvalidArgument, "shape needs m >= 2");
            k.m = m;
            for (int i = 0; i + 1 < m; ++i) k.sig.push_back({i, i + 1});
            if (shape[1] == 'y') k.sig.push_back({m - 1, 0});
        } else if (shape == "k4tail") {  // BASELINE C4
            k.m = 6;
            k.sig = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}, {3, 4}, {4, 5}};
        } else {
            fail(ErrorCode::InvalidArgument, "unknown RBF shape '" + shape + "' (chain<m> | cycle<m> | k4tail)");
        }
        k.recipe.assign(k.sig.size(), rec);
        return k;
    }
    if (kind == "proj" && parts.size() == 3) {  // BASELINE C3 / C5: r B ... B e
        const int m = to_int(parts[1], spec), kmax = to_int(parts[2], spec);
        if (m < 2 || kmax < 1) fail(ErrorCode::InvalidArgument, "proj needs m >= 2 and kmax >= 1");
        if (d < 3) fail(ErrorCode::InvalidArgument, "proj needs data columns [u_1..u_c, r, e] with c >= 1");
        k.m = m;
        k.sig.push_back({0});
        k.recipe.push_back("col:" + std::to_string(d - 2));
        for (int i = 0; i + 1 < m; ++i) {
            k.sig.push_back({i, i + 1});
            k.recipe.push_back("proj:" + std::to_string(d - 2) + ":" + std::to_string(kmax));
        }
        k.sig.push_back({m - 1});
        k.recipe.push_back("col:" + std::to_string(d - 1));
        return k;
    }
    fail(ErrorCode::InvalidArgument,
         "unknown kernel spec '" + spec + "' (prod2 | hoif:<j>:<k> | rbf:<shape>:<h> | proj:<m>:<kmax>)");
}

namespace {

// Replay cache of the data API (small n): the whole evaluation of a repeated
// call -- sample upload, tensorization, every kernel of the cached plan, the
// D2H of the terms -- is captured once as a CUDA graph and launched as one
// node chain afterwards (a bootstrap loop calls u_statistic thousands of
// times on the same buffers; the evaluation is launch-bound there). Keyed by
// the spec, the shape, the data pointer and the config; dropped when the plan
// cache evicts (the graph refers to the plan's term slots).
struct ReplayEntry {
    int calls = 0;
    bool dead = false;
    std::uint64_t generation = 0, used = 0;
    std::unique_ptr<GraphCapture> cap;
    StatisticResult result;  // everything but the term values
};
constexpr long long kReplayMaxN = 4096;
constexpr std::size_t kReplayEntries = 8;
std::map<std::string, ReplayEntry>& replay_cache(int device) {
    static auto* all = new std::map<int, std::map<std::string, ReplayEntry>>();  // under the device mutex
    return (*all)[device];
}

std::atomic<std::uint64_t> g_replays[64];

bool host_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

StatisticResult recombine(const ReplayEntry& e) {
    StatisticResult r = e.result;
    const GraphCapture& c = *e.cap;
    for (std::size_t t = 0; t < c.T; ++t) r.v[t] = c.host_v[t];
    for (const auto& [dup, src] : c.alias) r.v[dup] = r.v[src];
    for (std::size_t t = 0; t < c.T; ++t) r.terms[t] = static_cast<double>(r.mu[t]) * r.v[t];
    r.value = combine_terms(r.terms);
    return r;
}

StatisticResult u_statistic_data_once(const DataKernel& k, const double* data, long long n, int d, bool on_device,
                                      const Config& config, double* tensorize_seconds);

}  // namespace

std::uint64_t graph_replays(int device) { return g_replays[static_cast<unsigned>(device) & 63].load(); }

StatisticResult u_statistic_data(const std::string& spec, const double* data, long long n, int d, bool on_device,
                                 const Config& config, double* tensorize_seconds) {
    const DataKernel k = parse_data_kernel(spec, d);
    if (n < k.m)
        fail(ErrorCode::SampleTooSmall,
             "need at least " + std::to_string(k.m) + " observations, have " + std::to_string(n));
    for (std::size_t c = 0; c < k.sig.size(); ++c)
        checked_entry_count(static_cast<int>(k.sig[c].size()), static_cast<int>(n), config);
    Runtime& rt = Runtime::get(config.device.device);
    std::lock_guard<std::recursive_mutex> lock(device_mutex(rt.device()));
    const DeviceConfig& dc = config.device;
    const bool eligible = dc.graph_replay && n <= kReplayMaxN && !dc.shard_rows && dc.world_size <= 1 &&
                          !rt.profiling() && k.m <= 10 && (on_device || host_pinned(data));
    if (!eligible) return u_statistic_data_once(k, data, n, d, on_device, config, tensorize_seconds);

    auto& cache = replay_cache(rt.device());
    static std::atomic<std::uint64_t> clock{0};
    const std::string key = spec + "|" + std::to_string(n) + "x" + std::to_string(d) + "|" +
                            std::to_string(reinterpret_cast<std::uintptr_t>(data)) + (on_device ? "d|" : "h|") +
                            config_key(config);
    auto it = cache.find(key);
    if (it == cache.end()) {
        while (cache.size() >= kReplayEntries) {
            auto lru = cache.begin();
            for (auto j = cache.begin(); j != cache.end(); ++j)
                if (j->second.used < lru->second.used) lru = j;
            cache.erase(lru);
        }
        it = cache.emplace(key, ReplayEntry{}).first;
    }
    ReplayEntry& e = it->second;
    e.used = ++clock;
    if (e.cap && e.generation != plan_generation(rt.device())) {  // the plan it was captured from is gone
        e.cap.reset();
        e.calls = 0;
    }
    if (e.cap && e.cap->exec) {
        check_cuda(cudaGraphLaunch(e.cap->exec, rt.main_stream()), "cudaGraphLaunch");
        rt.sync();
        ++g_replays[static_cast<unsigned>(rt.device()) & 63];
        if (tensorize_seconds) *tensorize_seconds = 0.0;
        return recombine(e);
    }
    if (e.dead || e.calls < 1) {  // first call: records and caches the plan
        ++e.calls;
        return u_statistic_data_once(k, data, n, d, on_device, config, tensorize_seconds);
    }
    // second call with the same arguments: capture it
    auto cap = std::make_unique<GraphCapture>();
    cap->capacity = static_cast<std::size_t>(bell_number(k.m));
    check_cuda(cudaMallocHost(reinterpret_cast<void**>(&cap->host_v), sizeof(double) * cap->capacity), "cudaMallocHost");
    rt.set_stream(rt.main_stream());
    check_cuda(cudaStreamBeginCapture(rt.main_stream(), cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
    active_capture() = cap.get();
    try {
        StatisticResult r = u_statistic_data_once(k, data, n, d, on_device, config, tensorize_seconds);
        if (!cap->launched) fail(ErrorCode::CudaError, "graph capture did not complete");
        e.generation = plan_generation(rt.device());
        e.result = r;
        e.cap = std::move(cap);
        return r;
    } catch (...) {
        // not capturable (an allocation that had to synchronize, a missing plan ...):
        // discard the capture and evaluate the plain way from now on
        active_capture() = nullptr;
        cudaGraph_t g = nullptr;
        cudaStreamEndCapture(rt.main_stream(), &g);
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
        e.dead = true;
    }
    return u_statistic_data_once(k, data, n, d, on_device, config, tensorize_seconds);
}

namespace {

StatisticResult u_statistic_data_once(const DataKernel& k, const double* data, long long n, int d, bool on_device,
                                      const Config& config, double* tensorize_seconds) {
    Runtime& rt = Runtime::get(config.device.device);
    cudaStream_t s = rt.main_stream();
    rt.set_stream(s);
    const auto t0 = std::chrono::steady_clock::now();

    // the sample on the device (n x d doubles: the only H2D of the call)
    Buf sample;
    const double* x = data;
    if (!on_device) {
        sample = rt.allocate(1, n * d);
        check_cuda(cudaMemcpyAsync(sample->ptr, data, static_cast<std::size_t>(n * d) * sizeof(double),
                                   cudaMemcpyHostToDevice, s),
                   "upload sample");
        x = sample->ptr;
    }
    std::map<std::string, Buf> built;
    std::uint64_t launches = 0;
    for (const std::string& rec : k.recipe) {
        if (built.count(rec)) continue;
        const auto p = split(rec, ':');
        Buf b;
        if (p[0] == "col") {
            b = rt.allocate(1, n);
            launch_column(x, n, d, std::stoi(p[1]), b->ptr, s);
            ++launches;
        } else if (p[0] == "gram") {
            b = rt.allocate(2, n);
            launch_scaled_gram(x, n, d, std::stoi(p[1]), std::stoi(p[2]), std::stoi(p[3]), std::stoi(p[4]), b->ptr, s);
            ++launches;
        } else if (p[0] == "rbf") {
            b = rt.allocate(2, n);
            launch_rbf(x, n, d, std::stod(p[1]), b->ptr, s, /*zero_diag=*/true);  // sparsified as it is written
            ++launches;
        } else {  // proj: B = Z (Z^T Z / n)^{-1} Z^T as the symmetric product (Z M)(Z M)^T
            const int ncols = std::stoi(p[1]), kmax = std::stoi(p[2]);
            const int F = ncols * kmax;
            Buf z = rt.allocate(1, n * F), y = rt.allocate(1, n * F), g = rt.allocate(1, static_cast<long long>(F) * F);
            launch_cosine_features(x, n, d, ncols, kmax, z->ptr, s);
            const long long gram_scratch = thin_gram_scratch_entries(n, F);
            Buf gp = gram_scratch ? rt.allocate(1, gram_scratch) : nullptr;
            launch_thin_gram(z->ptr, n, F, g->ptr, gp ? gp->ptr : nullptr, s);
            std::vector<double> G(static_cast<std::size_t>(F * F));
            check_cuda(cudaMemcpyAsync(G.data(), g->ptr, G.size() * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
            check_cuda(cudaStreamSynchronize(s), "sync");
            const std::vector<double> M = inverse_cholesky_transpose(G, F);
            check_cuda(cudaMemcpyAsync(g->ptr, M.data(), M.size() * sizeof(double), cudaMemcpyHostToDevice, s), "H2D");
            launch_times_small(z->ptr, n, F, g->ptr, y->ptr, s);
            b = rt.allocate(2, n);
            GemmArgs a;
            a.a.nf = a.b.nf = 1;
            a.a.nr = a.b.nr = 1;
            a.a.ptr[0] = a.b.ptr[0] = y->ptr;
            a.a.rstride[0][0] = a.b.rstride[0][0] = F;
            a.a.kstride[0] = a.b.kstride[0] = 1;
            a.n = F;
            a.rows = a.cols = n;
            a.symmetric_out = 1;
            EpiSet e;
            e.count = 1;
            e.d[0].mode = kEpiStore;
            e.d[0].out = b->ptr;
            launches += gram_scratch ? 4 : 3;  // features, thin Gram (+ its finalizer), Z M
            const int gl = launch_gemm_multi(a, e, s);
            launches += gl > 0 ? static_cast<std::uint64_t>(gl) : 1;
            if (gl < 0) {  // operands not TMA-eligible (odd F): plain product
                a.symmetric_out = 0;
                a.mode = kEpiStore;
                a.out = b->ptr;
                launch_gemm(a, s);
            }
            check_cuda(cudaStreamSynchronize(s), "sync");  // z, y, g freed at scope exit
        }
        check_cuda(cudaGetLastError(), "tensorize");
        built[rec] = b;
    }
    // no sync here: the tensorization kernels run while the host plans the
    // statistic (tensorize_seconds is the host time to build and enqueue them)
    if (tensorize_seconds)
        *tensorize_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();

    StatisticSpec spec_in;
    spec_in.m = k.m;
    spec_in.sig = k.sig;
    for (const std::string& rec : k.recipe) {
        spec_in.inputs.push_back(built[rec]->ptr);
        // RBF entries are computed once per unordered pair and mirrored; the
        // projection is a mirrored symmetric GEMM: both bitwise symmetric
        spec_in.symmetric.push_back(rec.rfind("rbf", 0) == 0 || rec.rfind("proj", 0) == 0);
        spec_in.sparsified.push_back(rec.rfind("rbf", 0) == 0);
    }
    Config cfg = config;
    cfg.device.donate_inputs = true;  // our own tensors: sparsify in place
    // under a graph capture the tensors and the sample are released inside it
    // (every allocation of a replayed graph must be freed by the graph)
    if (GraphCapture* cap = active_capture())
        cap->before_sync = [&] {
            built.clear();
            sample.reset();
        };
    auto res = lattice_batch({spec_in}, true, n, LatticeMode::Sparsified, cfg);
    res[0].stats.kernel_launches += launches;
    return res[0];
}

}  // namespace

}  // namespace ustats::dev

// ------------------------------------------------------------ drivers
namespace ustats::dev {

namespace {

// Folds the per-statistic results of one shared batch into one report: the
// device work is the batch's (carried by the first), lattice counters add up.
StatisticResult merged(std::vector<StatisticResult>& parts, double value) {
    StatisticResult r = parts[0];
    r.value = value;
    for (std::size_t q = 1; q < parts.size(); ++q) {
        r.enumerated += parts[q].enumerated;
        r.owner.insert(r.owner.end(), parts[q].owner.begin(), parts[q].owner.end());
        r.stats.ref_madds += parts[q].stats.ref_madds;
        r.stats.ref_peak = std::max(r.stats.ref_peak, parts[q].stats.ref_peak);
    }
    return r;
}

}  // namespace

StatisticResult dcov_squared(const double* x, int dx, const double* y, int dy, long long n, bool on_device,
                             const Config& config) {
    if (dx < 1 || dy < 1) fail(ErrorCode::InvalidArgument, "observations need at least one coordinate");
    if (n < 4) fail(ErrorCode::SampleTooSmall, "need at least 4 paired observations, have " + std::to_string(n));
    checked_entry_count(2, static_cast<int>(n), config);
    Runtime& rt = Runtime::get(config.device.device);
    cudaStream_t s = rt.main_stream();
    rt.set_stream(s);
    Buf xs, ys;
    const double* xd = x;
    const double* yd = y;
    if (!on_device) {
        xs = rt.allocate(1, n * dx);
        ys = rt.allocate(1, n * dy);
        check_cuda(cudaMemcpyAsync(xs->ptr, x, static_cast<std::size_t>(n * dx) * sizeof(double),
                                   cudaMemcpyHostToDevice, s), "upload x");
        check_cuda(cudaMemcpyAsync(ys->ptr, y, static_cast<std::size_t>(n * dy) * sizeof(double),
                                   cudaMemcpyHostToDevice, s), "upload y");
        xd = xs->ptr;
        yd = ys->ptr;
    }
    Buf d1 = rt.allocate(2, n), d2 = rt.allocate(2, n);
    launch_distance(xd, n, dx, 0, dx, d1->ptr, s);
    launch_distance(yd, n, dy, 0, dy, d2->ptr, s);
    check_cuda(cudaGetLastError(), "distance");
    // dcov.cpp:74-77: ((1,2),(3,4)), ((1,2),(1,2)), ((1,2),(1,3)), ((1,2),(2,3)), components (d1, d2)
    const std::vector<std::pair<int, std::vector<IndexTuple>>> shapes = {
        {4, {{0, 1}, {2, 3}}}, {2, {{0, 1}, {0, 1}}}, {3, {{0, 1}, {0, 2}}}, {3, {{0, 1}, {1, 2}}}};
    std::vector<StatisticSpec> specs;
    for (const auto& [m, sig] : shapes) {
        StatisticSpec sp;
        sp.m = m;
        sp.sig = sig;
        sp.inputs = {d1->ptr, d2->ptr};
        sp.symmetric = {1, 1};
        specs.push_back(std::move(sp));
    }
    Config cfg = config;
    cfg.device.donate_inputs = true;
    auto res = lattice_batch(specs, true, n, LatticeMode::Sparsified, cfg);
    // dcov.cpp:79-85, in long double
    const long double nn = static_cast<long double>(n);
    long double c = static_cast<long double>(res[0].value) + (nn - 2) * (nn - 3) * static_cast<long double>(res[1].value) -
                    (nn - 3) * static_cast<long double>(res[2].value) - (nn - 3) * static_cast<long double>(res[3].value);
    c /= nn * (nn - 1) * (nn - 2) * (nn - 3);
    StatisticResult r = merged(res, static_cast<double>(c));
    r.stats.kernel_launches += 2;
    return r;
}

double hoif_combine(int m, long long n, const std::vector<double>& u) {
    auto binom = [](int a, int b) {
        std::uint64_t v = 1;
        for (int i = 0; i < b; ++i) v = v * static_cast<std::uint64_t>(a - i) / static_cast<std::uint64_t>(i + 1);
        return v;
    };
    long double tau = 0.0L;
    for (int j = 2; j <= m; ++j) {
        const double sign = j % 2 == 0 ? 1.0 : -1.0;
        for (int l = 0; l + 2 <= j; ++l) {
            long double w = 1.0L;  // (n - l)! / n!
            for (int i = 0; i < l; ++i) w /= static_cast<long double>(n - i);
            tau += sign * static_cast<long double>(binom(j - 2, l)) * w *
                   static_cast<long double>(u[static_cast<std::size_t>(l + 2)]);
        }
    }
    return static_cast<double>(tau);
}

StatisticResult hoif_tau_data(int m, int k, const double* data, long long n, int d, bool on_device,
                              const Config& config) {
    if (m < 2) fail(ErrorCode::InvalidArgument, "statistic order must be >= 2");
    if (k < 1) fail(ErrorCode::InvalidArgument, "basis size must be >= 1");
    if (d < 2 + k) fail(ErrorCode::InvalidArgument, "covariate block shorter than the basis");
    if (n < m)
        fail(ErrorCode::SampleTooSmall, "need at least " + std::to_string(m) + " observations, have " + std::to_string(n));
    checked_entry_count(2, static_cast<int>(n), config);
    Runtime& rt = Runtime::get(config.device.device);
    cudaStream_t s = rt.main_stream();
    rt.set_stream(s);
    Buf sample;
    const double* x = data;
    if (!on_device) {
        sample = rt.allocate(1, n * d);
        check_cuda(cudaMemcpyAsync(sample->ptr, data, static_cast<std::size_t>(n * d) * sizeof(double),
                                   cudaMemcpyHostToDevice, s),
                   "upload sample");
        x = sample->ptr;
    }
    // A_x phi(Z_x).phi(Z_y) A_y (middle) and A_x phi(Z_x).phi(Z_y) Y_y (last)
    Buf last = rt.allocate(2, n), middle;
    launch_scaled_gram(x, n, d, 0, 1, 2, k, last->ptr, s);
    std::uint64_t launches = 1;
    if (m > 2) {
        middle = rt.allocate(2, n);
        launch_scaled_gram(x, n, d, 0, 0, 2, k, middle->ptr, s);
        ++launches;
    }
    check_cuda(cudaGetLastError(), "tensorize");
    std::vector<StatisticSpec> specs;
    for (int order = 2; order <= m; ++order) {
        StatisticSpec sp;
        sp.m = order;
        for (int i = 0; i + 1 < order; ++i) {
            sp.sig.push_back({i, i + 1});
            const bool mid = i + 2 < order;
            sp.inputs.push_back(mid ? middle->ptr : last->ptr);
            sp.symmetric.push_back(0);  // probed: (A_x dot) A_y and (A_y dot) A_x may differ in the last bit
        }
        specs.push_back(std::move(sp));
    }
    Config cfg = config;
    cfg.device.donate_inputs = true;
    auto res = lattice_batch(specs, true, n, LatticeMode::Sparsified, cfg);
    std::vector<double> u(static_cast<std::size_t>(m + 1), 0.0);
    for (int order = 2; order <= m; ++order) u[static_cast<std::size_t>(order)] = res[static_cast<std::size_t>(order - 2)].value;
    StatisticResult r = merged(res, hoif_combine(m, n, u));
    r.stats.kernel_launches += launches;
    return r;
}

const std::vector<MotifSpec>& motif_catalog() {
    // induced patterns on 3-4 vertices (motifs.hpp:33-36): edges that must be
    // present / absent, automorphism counts
    static const std::vector<MotifSpec> cat = {
        {"r1", 3, 2, {{1, 2}, {2, 3}}, {{1, 3}}},                                  // path P3
        {"r2", 3, 6, {{1, 2}, {1, 3}, {2, 3}}, {}},                                // triangle
        {"r3", 4, 6, {{1, 2}, {1, 3}, {1, 4}}, {{2, 3}, {2, 4}, {3, 4}}},          // 3-star
        {"r4", 4, 2, {{1, 2}, {2, 3}, {3, 4}}, {{1, 3}, {1, 4}, {2, 4}}},          // path P4
        {"r5", 4, 2, {{1, 2}, {1, 3}, {2, 3}, {3, 4}}, {{1, 4}, {2, 4}}},          // tailed triangle
        {"r6", 4, 8, {{1, 2}, {2, 3}, {3, 4}, {1, 4}}, {{1, 3}, {2, 4}}},          // 4-cycle
        {"r7", 4, 4, {{1, 2}, {1, 3}, {1, 4}, {2, 3}, {2, 4}}, {{3, 4}}},          // diamond
        {"r8", 4, 24, {{1, 2}, {1, 3}, {1, 4}, {2, 3}, {2, 4}, {3, 4}}, {}},       // K4
    };
    return cat;
}

StatisticResult motif_count(long long n, const int* edges, long long edge_count, const std::string& id,
                            const Config& config, long long* count) {
    const MotifSpec* spec = nullptr;
    for (const MotifSpec& m : motif_catalog())
        if (id == m.id) spec = &m;
    if (!spec) fail(ErrorCode::InvalidArgument, "unknown motif id '" + id + "' (expected r1..r8)");
    if (n < 0) fail(ErrorCode::InvalidArgument, "vertex count must be non-negative");
    for (long long e = 0; e < edge_count; ++e) {
        const int u = edges[2 * e], v = edges[2 * e + 1];
        if (u < 0 || v < 0 || u >= n || v >= n)
            fail(ErrorCode::InvalidArgument, "graph vertex ids must be contiguous 0..n-1");
        if (u == v) fail(ErrorCode::InvalidArgument, "self-loop on vertex " + std::to_string(u));
    }
    StatisticResult r;
    *count = 0;
    if (n < spec->order) return r;  // motifs.cpp:59
    checked_entry_count(2, static_cast<int>(n), config);
    Runtime& rt = Runtime::get(config.device.device);
    cudaStream_t s = rt.main_stream();
    rt.set_stream(s);
    int* de = nullptr;
    if (edge_count > 0) {
        check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&de), static_cast<std::size_t>(edge_count) * 2 * sizeof(int), s),
                   "alloc edges");
        check_cuda(cudaMemcpyAsync(de, edges, static_cast<std::size_t>(edge_count) * 2 * sizeof(int),
                                   cudaMemcpyHostToDevice, s), "upload edges");
    }
    Buf a = rt.allocate(2, n), b = rt.allocate(2, n);
    launch_adjacency(de, edge_count, n, a->ptr, b->ptr, s);
    check_cuda(cudaGetLastError(), "adjacency");
    if (de) cudaFreeAsync(de, s);
    StatisticSpec sp;
    sp.m = spec->order;
    for (const auto& [u, v] : spec->present) {
        sp.sig.push_back({u - 1, v - 1});
        sp.inputs.push_back(a->ptr);
        sp.symmetric.push_back(1);
    }
    for (const auto& [u, v] : spec->absent) {
        sp.sig.push_back({u - 1, v - 1});
        sp.inputs.push_back(b->ptr);
        sp.symmetric.push_back(1);
    }
    Config cfg = config;
    cfg.device.donate_inputs = true;
    auto res = lattice_batch({sp}, true, n, LatticeMode::Sparsified, cfg);
    r = res[0];
    r.stats.kernel_launches += edge_count > 0 ? 2 : 1;
    const double scaled = r.value / static_cast<double>(spec->automorphisms);
    const double rounded = std::nearbyint(scaled);
    if (std::abs(scaled - rounded) > 1e-6)
        fail(ErrorCode::NonIntegerResult, "count " + std::to_string(scaled) + " is not an integer");
    *count = static_cast<long long>(rounded);
    return r;
}

}  // namespace ustats::dev
