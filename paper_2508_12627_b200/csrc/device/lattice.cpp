// Statistic drivers (executor.hpp): lattice of V-terms, term plans,
// cross-term program recording, plan cache, combination.
#include "executor.hpp"

#include <dlfcn.h>

#include <algorithm>
#include <bit>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>

#include "executor_util.hpp"
#include "ustats/errors.hpp"
#include "ustats/partition.hpp"
#include "ustats/tensor.hpp"

namespace ustats::dev {

// ------------------------------------------------------- statistic drivers
namespace {

using Clock = std::chrono::steady_clock;

double pairwise(const double* x, std::size_t count) {
    if (count == 0) return 0.0;
    if (count <= 4) {
        double acc = x[0];
        for (std::size_t i = 1; i < count; ++i) acc += x[i];
        return acc;
    }
    const std::size_t half = count / 2;
    return pairwise(x, half) + pairwise(x + half, count - half);
}

// Lone ids (one occurrence) are marginalized before the ordered loop, so
// orders that differ only in their positions are the same plan.
std::vector<std::vector<int>> candidate_orders(const EinsumNotation& nt, const EliminationOrder& ref,
                                               std::size_t limit) {
    std::vector<int> occ(static_cast<std::size_t>(nt.index_count), 0);
    for (const auto& t : nt.inputs) {
        std::uint32_t seen = 0;
        for (int id : t)
            if (!(seen & bit(id))) {
                seen |= bit(id);
                ++occ[static_cast<std::size_t>(id)];
            }
    }
    auto project = [&](const std::vector<int>& o) {
        std::vector<int> p;
        for (int id : o)
            if (occ[static_cast<std::size_t>(id)] > 1) p.push_back(id);
        return p;
    };
    std::vector<std::vector<int>> out{ref.order};
    std::vector<std::vector<int>> seen{project(ref.order)};
    for (auto& o : optimal_orders(nt, ref.predicted_width, limit)) {
        auto p = project(o);
        if (std::find(seen.begin(), seen.end(), p) != seen.end()) continue;
        seen.push_back(p);
        out.push_back(std::move(o));
    }
    return out;
}

}  // namespace

double combine_terms(const std::vector<double>& terms) {
    constexpr std::size_t kChunk = 512;  // engine.cpp:51
    double total = 0.0;
    for (std::size_t at = 0; at < terms.size(); at += kChunk)
        total += pairwise(terms.data() + at, std::min(kChunk, terms.size() - at));
    return total;
}

TermPlan plan_terms(const std::vector<IndexTuple>& zero_sig, int m, long long n, LatticeMode mode,
                    const Config& config) {
    TermPlan plan;
    std::vector<SetPartition> parts;
    {
        SetPartition p;
        if (mode == LatticeMode::Sparsified) {
            SparsifiedPartitionStream s(m, zero_sig);
            while (s.next(p)) parts.push_back(p);
            plan.enumerated = s.enumerated();
        } else {
            PartitionStream s(m);
            while (s.next(p)) parts.push_back(p);
            plan.enumerated = bell_number(m);
        }
    }
    for (const SetPartition& p : parts) {
        plan.rgs.push_back(p.rgs());
        plan.mu.push_back(mobius_coefficient(p));
        plan.notation.emplace_back(induced_signature(zero_sig, p));
        plan.order.push_back(optimize_order(plan.notation.back(), static_cast<int>(n), config.strategy, config));
        plan.cost.push_back(static_cast<double>(plan.order.back().predicted_peak_entries));
    }
    const std::size_t T = parts.size();
    plan.owner.assign(T, 0);
    const int W = std::max(1, config.device.world_size);
    if (W > 1) {
        std::vector<std::size_t> idx(T);
        std::iota(idx.begin(), idx.end(), 0);
        std::stable_sort(idx.begin(), idx.end(), [&](std::size_t a, std::size_t b) { return plan.cost[a] > plan.cost[b]; });
        std::vector<double> load(static_cast<std::size_t>(W), 0.0);
        for (std::size_t t : idx) {
            auto w = static_cast<std::size_t>(std::min_element(load.begin(), load.end()) - load.begin());
            plan.owner[t] = static_cast<int>(w);
            load[w] += plan.cost[t];
        }
    }
    return plan;
}

// Records every owned term into one Program: the reference order is walked
// once for the reference-rule counters; the recorded order is the
// width-optimal one that adds the least new work given earlier terms.
void record_terms(Program& prog, const TermPlan& plan, const std::vector<int>& inputs, int rank, double* d_v,
                  DevStats* counters) {
    const Config& cfg = prog.config();
    const bool reorder = cfg.device.reorder_for_sharing && cfg.device.share_subexpressions;
    for (std::size_t t = 0; t < plan.rgs.size(); ++t) {
        if (plan.owner[t] != rank) continue;
        const EinsumNotation& nt = plan.notation[t];
        const EliminationOrder& ref = plan.order[t];
        EliminationOrder best = ref;
        if (reorder) {
            double best_cost = -1.0;
            for (const auto& cand : candidate_orders(nt, ref, 2048)) {
                Program::Mark mk = prog.mark();
                EliminationOrder o = ref;
                o.order = cand;
                Contractor(prog, nullptr).run(inputs, nt, o, d_v + t);
                const double c = prog.cost_since(mk);
                if (std::getenv("USTATS_ORDER_DEBUG")) {
                    std::fprintf(stderr, "[order] term %zu cand", t);
                    for (int id : cand) std::fprintf(stderr, " %d", id);
                    std::fprintf(stderr, " cost %.4g\n", c);
                }
                prog.rollback(mk);
                if (best_cost < 0 || c < best_cost * (1 - 1e-12)) {
                    best_cost = c;
                    best = o;
                }
            }
        }
        if (best.order == ref.order) {
            Contractor(prog, counters).run(inputs, nt, ref, d_v + t);
        } else {
            Program::Mark mk = prog.mark();
            Contractor(prog, counters).run(inputs, nt, ref, d_v + t);  // counters + cap checks
            prog.rollback(mk);
            Contractor(prog, nullptr).run(inputs, nt, best, d_v + t);
        }
    }
}

namespace {
// Host matrices at least this big are uploaded in row panels on the copy
// stream so the first (symmetric) GEMM starts on the panels that landed.
constexpr long long kChunkMinN = 2048;
constexpr int kUploadPanels = 16;
}  // namespace

// ------------------------------------------------------------ plan cache
// Recording a statistic (term plans, candidate orders, the cross-term
// program, fusion, the memory-bounded schedule) is pure host work that
// depends only on the signatures, the extent, the inputs' orders / symmetry /
// aliasing and the config; the cache keeps the optimized program per device
// (LRU, 16 entries) so repeated evaluations go straight to launching.
struct PlanEntry {
    Config config;  // the program refers to this copy
    std::vector<TermPlan> plans;
    std::vector<DevStats> counters;  // per statistic: reference-rule counters
    DevStats recorded;               // record-time device counters (shared hits, ...)
    std::unique_ptr<Program> prog;
    Buf v;                           // term slots the program's reductions write
    std::size_t T = 0;
    std::vector<std::pair<std::size_t, std::size_t>> alias;
    std::uint64_t used = 0;
};

namespace {

constexpr std::size_t kPlanCacheEntries = 16;

struct PlanCache {
    std::mutex mu;
    std::map<std::string, std::unique_ptr<PlanEntry>> entries;
    std::uint64_t clock = 0;
};

PlanCache& plan_cache(int device) {
    static auto* caches = new std::map<int, PlanCache>();  // leaked on purpose: no teardown-order issues
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    return (*caches)[device];
}

std::string plan_key(const std::vector<StatisticSpec>& specs, const std::vector<std::vector<int>>& slot,
                     const std::vector<Buf>& uniq, long long n, LatticeMode mode, const Config& c, double budget) {
    std::string k = std::to_string(n) + "|" + std::to_string(static_cast<int>(mode)) + "|" +
                    std::to_string(static_cast<long long>(budget / 8.589934592e9)) + "|" + config_key(c) + "|";
    for (const Buf& b : uniq) k += std::to_string(b->order) + (b->symmetric ? "s" : "g");
    for (std::size_t q = 0; q < specs.size(); ++q) {
        k += "|" + std::to_string(specs[q].m) + ":";
        for (std::size_t f = 0; f < specs[q].sig.size(); ++f) {
            k += std::to_string(slot[q][f]) + "(";
            for (int i : specs[q].sig[f]) k += std::to_string(i) + ",";
            k += ")";
        }
    }
    return k;
}

std::uint64_t g_plan_generation[64] = {};

PlanEntry* find_plan(int device, const std::string& key) {
    if (std::getenv("USTATS_NO_PLAN_CACHE")) return nullptr;
    PlanCache& pc = plan_cache(device);
    std::lock_guard<std::mutex> lock(pc.mu);
    auto it = pc.entries.find(key);
    if (it == pc.entries.end()) return nullptr;
    it->second->used = ++pc.clock;
    return it->second.get();
}

PlanEntry* store_plan(int device, const std::string& key, std::unique_ptr<PlanEntry> e) {
    PlanCache& pc = plan_cache(device);
    std::lock_guard<std::mutex> lock(pc.mu);
    e->used = ++pc.clock;
    while (pc.entries.size() >= kPlanCacheEntries) {
        auto lru = pc.entries.begin();
        for (auto it = pc.entries.begin(); it != pc.entries.end(); ++it)
            if (it->second->used < lru->second->used) lru = it;
        pc.entries.erase(lru);
        ++g_plan_generation[static_cast<unsigned>(device) & 63];  // captured graphs refer to evicted term slots
    }
    PlanEntry* raw = e.get();
    pc.entries[key] = std::move(e);
    return raw;
}

}  // namespace

// One evaluation at a time per device: a cached Program (its buffers, term
// slots and launch order) and the Runtime's current stream / profiling state
// are shared, and ctypes releases the GIL during the call, so two host
// threads evaluating on one device are serialized here (different devices
// run concurrently).
GraphCapture::~GraphCapture() {
    if (exec) cudaGraphExecDestroy(exec);
    if (host_v) cudaFreeHost(host_v);
}

GraphCapture*& active_capture() {
    thread_local GraphCapture* cap = nullptr;
    return cap;
}

std::recursive_mutex& device_mutex(int device) {
    static std::mutex table_mu;
    static std::map<int, std::unique_ptr<std::recursive_mutex>> per_device;
    std::lock_guard<std::mutex> lock(table_mu);
    auto& slot = per_device[device];
    if (!slot) slot = std::make_unique<std::recursive_mutex>();
    return *slot;
}

std::uint64_t plan_generation(int device) { return g_plan_generation[static_cast<unsigned>(device) & 63]; }

std::string config_key(const Config& c) {
    const DeviceConfig& d = c.device;
    return std::to_string(c.memory_cap_entries) + "," + std::to_string(static_cast<int>(c.strategy)) + "," +
           std::to_string(c.exhaustive_index_bound) + "," + std::to_string(c.exact_treewidth_bound) + "|" +
           std::to_string(d.share_subexpressions) + std::to_string(d.fuse_epilogues) +
           std::to_string(d.exploit_symmetry) + std::to_string(d.reorder_for_sharing) +
           std::to_string(d.serial_launch) + std::to_string(d.shard_rows) + std::to_string(d.fp64_emulation) + "," +
           std::to_string(d.rank) + "," + std::to_string(d.world_size) + "," + std::to_string(d.emulate_world) + "," +
           std::to_string(d.memory_budget_bytes) + "," + std::to_string(d.oz_slices) + "," +
           std::to_string(d.oz_max_k) + "," + std::to_string(d.oz_min_dim);
}

std::vector<StatisticResult> lattice_batch(const std::vector<StatisticSpec>& specs, bool inputs_on_device,
                                           long long n, LatticeMode mode, const Config& config) {
    std::lock_guard<std::recursive_mutex> lock(device_mutex(Runtime::get(config.device.device).device()));
    return lattice_batch_impl(specs, inputs_on_device, n, mode, config, true);
}

std::vector<StatisticResult> lattice_batch_impl(const std::vector<StatisticSpec>& specs, bool inputs_on_device,
                                                long long n, LatticeMode mode, const Config& config, bool speculate) {
    std::vector<StatisticResult> out(specs.size());
    Runtime& rt = Runtime::get(config.device.device);
    const auto t_up = Clock::now();

    // Upload each distinct factor of every statistic once; sparsify on device
    // (tensor.cpp:54-76) and probe matrices for bitwise symmetry.
    std::map<const double*, Buf> by_ptr;
    std::vector<std::vector<Buf>> tensors(specs.size());
    std::vector<std::pair<Buf, int*>> probes;
    std::vector<std::tuple<Buf, int*, std::pair<const void*, long long>>> speculative;
    std::vector<std::pair<std::pair<const void*, long long>, int>> probe_keys;
    std::size_t total_factors = 0;
    for (const auto& sp : specs) total_factors += sp.sig.size();
    int* flags = nullptr;
    DevStats upload_stats;
    // probe flags only when some matrix input is not symmetric by construction
    // (device-tensorized components are: no allocation, events or frees then)
    bool may_probe = false;
    for (const auto& sp : specs)
        for (std::size_t k = 0; k < sp.sig.size(); ++k)
            may_probe |= sp.sig[k].size() == 2 && !(k < sp.symmetric.size() && sp.symmetric[k]);
    if (config.device.exploit_symmetry && may_probe)
        check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&flags), sizeof(int) * total_factors + 4, rt.stream()),
                   "alloc flags");
    for (std::size_t q = 0; q < specs.size(); ++q) tensors[q].assign(specs[q].sig.size(), nullptr);
    // Small host inputs go first: H2D copies share the copy engines in issue
    // order, so a vector queued behind a matrix's panels would hold the
    // main stream until the whole matrix landed.
    for (int pass = 0; pass < 2; ++pass)
    for (std::size_t q = 0; q < specs.size(); ++q) {
        const StatisticSpec& sp = specs[q];
        for (std::size_t k = 0; k < sp.sig.size(); ++k) {
            const int order = static_cast<int>(sp.sig[k].size());
            const bool big = !inputs_on_device && order == 2 && n >= kChunkMinN;
            if (pass == 0 && big) continue;
            if (pass == 1 && !big) continue;
            checked_entry_count(order, static_cast<int>(n), config);
            auto hit = by_ptr.find(sp.inputs[k]);
            if (hit != by_ptr.end() && hit->second->order == order) {
                tensors[q][k] = hit->second;
                continue;
            }
            Buf b;
            const bool panels = !inputs_on_device && order == 2 && n >= kChunkMinN;
            if (inputs_on_device && config.device.donate_inputs) {
                b = rt.borrow(sp.inputs[k], order, n);  // sparsified in place: the caller donated it
            } else if (panels) {
                // row panels on the copy stream, each sparsified as it lands
                b = rt.allocate(order, n);
                cudaEvent_t allocated;
                check_cuda(cudaEventCreateWithFlags(&allocated, cudaEventDisableTiming), "event");
                check_cuda(cudaEventRecord(allocated, rt.main_stream()), "event");
                check_cuda(cudaStreamWaitEvent(rt.copy_stream(), allocated, 0), "wait");
                cudaEventDestroy(allocated);
                const long long step = ((n + kUploadPanels - 1) / kUploadPanels + 127) / 128 * 128;
                for (long long r0 = 0; r0 < n; r0 += step) {
                    const long long r1 = std::min(n, r0 + step);
                    check_cuda(cudaMemcpyAsync(b->ptr + r0 * n, sp.inputs[k] + r0 * n,
                                               static_cast<std::size_t>((r1 - r0) * n) * sizeof(double),
                                               cudaMemcpyHostToDevice, rt.copy_stream()),
                               "upload panel");
                    // the copy stream carries copies only (a kernel there would wait
                    // for an SM held by the GEMM and stall the next copy); the panel
                    // is sparsified on the high-priority prep stream
                    cudaEvent_t landed, ev;
                    check_cuda(cudaEventCreateWithFlags(&landed, cudaEventDisableTiming), "event");
                    check_cuda(cudaEventRecord(landed, rt.copy_stream()), "event");
                    check_cuda(cudaStreamWaitEvent(rt.prep_stream(), landed, 0), "wait");
                    cudaEventDestroy(landed);
                    if (mode == LatticeMode::Sparsified)
                        upload_stats.kernel_launches +=
                            static_cast<std::uint64_t>(launch_zero_diagonal_rows(b->ptr, n, r0, r1, rt.prep_stream()));
                    check_cuda(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
                    check_cuda(cudaEventRecord(ev, rt.prep_stream()), "event");
                    b->ready.emplace_back(r1, ev);
                }
            } else {
                b = rt.allocate(order, n);
                check_cuda(cudaMemcpyAsync(b->ptr, sp.inputs[k], b->entries() * sizeof(double),
                                           inputs_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                           rt.stream()),
                           "upload");
            }
            rt.begin(Runtime::kOther);
            if (mode == LatticeMode::Sparsified && !panels && !(k < sp.sparsified.size() && sp.sparsified[k]))
                upload_stats.kernel_launches += static_cast<std::uint64_t>(launch_sparsify(b->ptr, order, n, rt.stream()));
            if (order == 2 && k < sp.symmetric.size() && sp.symmetric[k]) {
                b->symmetric = config.device.exploit_symmetry;  // known by construction: no probe
            } else if (flags && order == 2) {
                int* f = flags + probes.size();
                const auto key = std::make_pair(static_cast<const void*>(sp.inputs[k]), n);
                auto seen = rt.symmetry_seen.find(key);
                if (std::getenv("USTATS_TRACE"))
                    std::fprintf(stderr, "[trace] input %p n=%lld panels=%d seen=%d sym=%d\n", static_cast<const void*>(sp.inputs[k]),
                                 n, panels ? 1 : 0, seen != rt.symmetry_seen.end() ? 1 : 0,
                                 seen != rt.symmetry_seen.end() && seen->second ? 1 : 0);
                if (panels && speculate && seen != rt.symmetry_seen.end() && seen->second) {
                    // speculate (the same host matrix was symmetric last time):
                    // plan now, verify with a probe queued behind the upload
                    b->symmetric = true;
                    upload_stats.kernel_launches +=
                        static_cast<std::uint64_t>(launch_symmetry_check(b->ptr, n, f, rt.prep_stream()));
                    speculative.emplace_back(b, f, key);
                } else {
                    if (panels) check_cuda(cudaStreamWaitEvent(rt.stream(), b->ready.back().second, 0), "wait upload");
                    upload_stats.kernel_launches +=
                        static_cast<std::uint64_t>(launch_symmetry_check(b->ptr, n, f, rt.stream()));
                    probes.emplace_back(b, f);
                    if (!inputs_on_device) probe_keys.emplace_back(key, static_cast<int>(probes.size()) - 1);
                }
            }
            rt.end(Runtime::kOther);
            by_ptr[sp.inputs[k]] = b;
            tensors[q][k] = b;
        }
    }
    if (!probes.empty()) {
        std::vector<int> host(probes.size());
        check_cuda(cudaMemcpyAsync(host.data(), flags, sizeof(int) * probes.size(), cudaMemcpyDeviceToHost, rt.stream()),
                   "flags");
        check_cuda(cudaStreamSynchronize(rt.main_stream()), "sync");
        for (std::size_t i = 0; i < probes.size(); ++i) probes[i].first->symmetric = host[i] == 0;
        for (const auto& [key, idx] : probe_keys) rt.symmetry_seen[key] = host[static_cast<std::size_t>(idx)] == 0;
    }
    // no sync: the copies / sparsify kernels are stream-ordered before the
    // program, whose host-side planning overlaps them
    const double enqueue_s = std::chrono::duration<double>(Clock::now() - t_up).count();
    const double upload_s = enqueue_s;
    const bool trace = std::getenv("USTATS_TRACE") != nullptr;

    const auto t0 = Clock::now();
    // The schedule counts the distinct inputs as live from the start, so the
    // budget is the memory available now PLUS those inputs (every one of them
    // is device-resident by now: uploaded, donated or caller-owned), minus a
    // reserve for the small pool allocations (epilogue partials, stream
    // scratch, term slots) the schedule does not itemize.
    double budget = static_cast<double>(config.device.memory_budget_bytes);
    if (budget <= 0) {
        double inputs = 0;
        std::vector<const DeviceBuffer*> seen;
        for (const auto& ts : tensors)
            for (const Buf& b : ts)
                if (std::find(seen.begin(), seen.end(), b.get()) == seen.end()) {
                    seen.push_back(b.get());
                    inputs += 8.0 * static_cast<double>(b->entries());
                }
        const double n2 = 8.0 * static_cast<double>(n) * static_cast<double>(n);
        if (n2 * 6 > 0.5 * rt.free_bytes()) rt.refresh_free_bytes();  // a program that needs most of the device
        budget = rt.free_bytes() + inputs - 1.5 * 1073741824.0;
    }
    // distinct inputs in first-use order, and each factor's position among them
    std::vector<Buf> uniq;
    std::vector<std::vector<int>> slot(specs.size());
    for (std::size_t q = 0; q < specs.size(); ++q)
        for (const Buf& b : tensors[q]) {
            auto it = std::find(uniq.begin(), uniq.end(), b);
            slot[q].push_back(static_cast<int>(it - uniq.begin()));
            if (it == uniq.end()) uniq.push_back(b);
        }
    const std::string key = plan_key(specs, slot, uniq, n, mode, config, budget);
    PlanEntry* entry = find_plan(rt.device(), key);
    const bool hit = entry != nullptr;
    GraphCapture* cap = active_capture();
    if (cap && (!hit || flags || config.device.shard_rows))  // recording allocates persistent state: never inside a capture
        fail(ErrorCode::CudaError, "graph capture needs a cached single-GPU plan with inputs symmetric by construction");
    if (!hit) {
        // Record every statistic into one program (sub-contractions shared
        // across them), optimize it, and keep it: a later call with the same
        // signatures, extent, input structure and config re-executes it.
        auto e = std::make_unique<PlanEntry>();
        e->config = config;
        std::size_t T = 0;
        for (const auto& sp : specs) {
            e->plans.push_back(plan_terms(sp.sig, sp.m, n, mode, e->config));
            if (config.device.shard_rows) e->plans.back().owner.assign(e->plans.back().owner.size(), 0);
            T += e->plans.back().rgs.size();
        }
        e->T = T;
        e->v = rt.allocate(1, static_cast<long long>(std::max<std::size_t>(T, 1)));
        e->counters.resize(specs.size());
        e->prog = std::make_unique<Program>(&rt, n, e->config, &e->recorded);
        std::size_t at = 0;
        for (std::size_t q = 0; q < specs.size(); ++q) {
            std::vector<int> ids;
            for (const Buf& b : tensors[q]) ids.push_back(e->prog->add_input(b));
            record_terms(*e->prog, e->plans[q], ids, config.device.shard_rows ? 0 : config.device.rank,
                         e->v->ptr + at, &e->counters[q]);
            at += e->plans[q].rgs.size();
        }
        e->prog->optimize(budget);
        for (const auto& [dup, src] : e->prog->term_aliases())
            e->alias.emplace_back(static_cast<std::size_t>(dup - e->v->ptr), static_cast<std::size_t>(src - e->v->ptr));
        e->prog->release_buffers();
        entry = store_plan(rt.device(), key, std::move(e));
    }
    const std::vector<TermPlan>& plans = entry->plans;
    const std::size_t T = entry->T;
    double* d_v = entry->v->ptr;
    const std::vector<std::pair<std::size_t, std::size_t>>& term_alias = entry->alias;
    for (std::size_t q = 0; q < specs.size(); ++q) out[q].stats = entry->counters[q];
    check_cuda(cudaMemsetAsync(d_v, 0, sizeof(double) * std::max<std::size_t>(T, 1), rt.stream()), "memset");
    DevStats shared = entry->recorded;  // record-time counters; execute adds the launches
    const double plan_s = std::chrono::duration<double>(Clock::now() - t0).count();
    {
        Program& prog = *entry->prog;
        prog.set_stats(&shared);
        prog.rebind_inputs(uniq);
        try {
            prog.execute();
        } catch (...) {
            prog.release_buffers();
            throw;
        }
        prog.release_buffers();
        prog.set_stats(nullptr);
        if (trace)
            std::fprintf(stderr, "[trace] upload-enqueue %.3f ms, upload-sync %.3f ms, plan %.3f ms (%s), launch done %.3f ms\n",
                         enqueue_s * 1e3, upload_s * 1e3, plan_s * 1e3, hit ? "cached" : "recorded",
                         std::chrono::duration<double>(Clock::now() - t0).count() * 1e3);
    }
    // row sharding: every term value is a sum of per-rank partials
    if (config.device.shard_rows && config.device.emulate_world <= 1 && rt.has_comm()) rt.allreduce_sum(d_v, T);
    std::vector<double> v(T, 0.0);
    if (cap && T > cap->capacity) fail(ErrorCode::CudaError, "graph capture: term buffer too small");
    double* host_v = cap ? cap->host_v : v.data();  // a captured copy lands in the capture's pinned buffer
    if (T) check_cuda(cudaMemcpyAsync(host_v, d_v, sizeof(double) * T, cudaMemcpyDeviceToHost, rt.stream()), "D2H");
    std::vector<int> spec_flags(speculative.size(), 0);
    for (std::size_t i = 0; i < speculative.size(); ++i)  // in prep-stream order: after the probe itself
        check_cuda(cudaMemcpyAsync(&spec_flags[i], std::get<1>(speculative[i]), sizeof(int), cudaMemcpyDeviceToHost,
                                   rt.prep_stream()),
                   "D2H flag");
    if (flags) {
        cudaEvent_t probed;
        check_cuda(cudaEventCreateWithFlags(&probed, cudaEventDisableTiming), "event");
        check_cuda(cudaEventRecord(probed, rt.prep_stream()), "event");
        check_cuda(cudaStreamWaitEvent(rt.main_stream(), probed, 0), "wait");
        cudaEventDestroy(probed);
        cudaFreeAsync(flags, rt.main_stream());
    }
    tensors.clear();
    by_ptr.clear();
    probes.clear();
    if (cap) {
        // everything of this evaluation is enqueued: close the capture where the
        // evaluation would synchronize, and run the graph once for this call
        if (cap->before_sync) cap->before_sync();
        cap->T = T;
        cap->alias = term_alias;
        cudaGraph_t graph = nullptr;
        check_cuda(cudaStreamEndCapture(rt.main_stream(), &graph), "cudaStreamEndCapture");
        active_capture() = nullptr;
        const cudaError_t inst = cudaGraphInstantiate(&cap->exec, graph, 0);
        cudaGraphDestroy(graph);
        check_cuda(inst, "cudaGraphInstantiate");
        check_cuda(cudaGraphLaunch(cap->exec, rt.main_stream()), "cudaGraphLaunch");
        cap->launched = true;
    }
    rt.sync();
    if (cap)
        for (std::size_t t = 0; t < T; ++t) v[t] = cap->host_v[t];
    bool mispredicted = false;
    for (std::size_t i = 0; i < speculative.size(); ++i)
        if (spec_flags[i] != 0) {
            rt.symmetry_seen[std::get<2>(speculative[i])] = false;
            mispredicted = true;
        }
    speculative.clear();
    if (mispredicted)  // the host matrix changed and is no longer symmetric: redo without speculation
        return lattice_batch_impl(specs, inputs_on_device, n, mode, config, false);
    for (const auto& [dup, src] : term_alias) v[dup] = v[src];
    const double contract_s = std::chrono::duration<double>(Clock::now() - t0).count();
    if (trace) std::fprintf(stderr, "[trace] contract total %.3f ms\n", contract_s * 1e3);

    std::size_t at = 0;
    for (std::size_t q = 0; q < specs.size(); ++q) {
        StatisticResult& res = out[q];
        const TermPlan& plan = plans[q];
        const std::size_t Tq = plan.rgs.size();
        res.enumerated = plan.enumerated;
        res.owner = plan.owner;
        res.mu = plan.mu;
        res.rgs = plan.rgs;
        res.v.assign(v.begin() + static_cast<std::ptrdiff_t>(at), v.begin() + static_cast<std::ptrdiff_t>(at + Tq));
        res.terms.resize(Tq);
        for (std::size_t t = 0; t < Tq; ++t) res.terms[t] = static_cast<double>(res.mu[t]) * res.v[t];
        res.value = combine_terms(res.terms);
        at += Tq;
        // device work of the shared program is reported once, on the first statistic
        if (q == 0) {
            res.stats.gemm_macs = shared.gemm_macs;
            res.stats.stream_entries = shared.stream_entries;
            res.stats.gemm_launches = shared.gemm_launches;
            res.stats.stream_launches = shared.stream_launches;
            res.stats.shared_hits = shared.shared_hits;
            res.stats.kernel_launches = shared.kernel_launches + upload_stats.kernel_launches;
            res.stats.fused_epilogues = shared.fused_epilogues;
            res.stats.symmetric_gemms = shared.symmetric_gemms;
            res.stats.emulated_macs = shared.emulated_macs;
            res.stats.int8_ops = shared.int8_ops;
            res.stats.oz_slices = shared.oz_slices;
        }
        res.upload_seconds = upload_s;
        res.contract_seconds = contract_s;
        res.plan_seconds = plan_s;
    }
    return out;
}

StatisticResult lattice_statistic(const std::vector<const double*>& inputs, bool inputs_on_device,
                                  const std::vector<IndexTuple>& zero_sig, int m, long long n, LatticeMode mode,
                                  const Config& config) {
    return lattice_batch({StatisticSpec{inputs, zero_sig, m}}, inputs_on_device, n, mode, config)[0];
}

namespace {
std::vector<Buf> upload_all(Runtime& rt, const std::vector<const double*>& inputs, const std::vector<int>& orders,
                            long long n) {
    std::map<std::pair<const double*, int>, Buf> by_ptr;
    std::vector<Buf> tensors;
    for (std::size_t k = 0; k < inputs.size(); ++k) {
        auto key = std::make_pair(inputs[k], orders[k]);
        auto hit = by_ptr.find(key);
        if (hit != by_ptr.end()) {
            tensors.push_back(hit->second);
            continue;
        }
        Buf b = rt.allocate(orders[k], n);
        check_cuda(cudaMemcpyAsync(b->ptr, inputs[k], b->entries() * sizeof(double), cudaMemcpyHostToDevice, rt.stream()),
                   "upload");
        by_ptr[key] = b;
        tensors.push_back(b);
    }
    return tensors;
}

std::vector<double> download(Runtime& rt, const Buf& out) {
    std::vector<double> host(out->entries());
    check_cuda(cudaMemcpyAsync(host.data(), out->ptr, host.size() * sizeof(double), cudaMemcpyDeviceToHost, rt.stream()),
               "D2H");
    rt.sync();
    return host;
}
}  // namespace

std::vector<double> contract_host(const std::vector<const double*>& inputs, const std::vector<int>& orders, long long n,
                                  const EinsumNotation& notation, const EliminationOrder* order, const Config& config,
                                  DevStats* stats) {
    Runtime& rt = Runtime::get(config.device.device);
    std::vector<Buf> tensors = upload_all(rt, inputs, orders, n);
    EliminationOrder chosen;
    if (!order) {
        chosen = optimize_order(notation, static_cast<int>(n), config.strategy, config);
        order = &chosen;
    }
    Buf out;
    {
        Program prog(&rt, n, config, stats);
        std::vector<int> ids;
        for (const Buf& b : tensors) ids.push_back(prog.add_input(b));
        const int res = Contractor(prog, stats).run(ids, notation, *order, nullptr);
        prog.keep(res);
        prog.optimize();
        prog.execute();
        out = prog.take(res);
    }
    return download(rt, out);
}

std::vector<double> eliminate_host(const std::vector<const double*>& inputs, const std::vector<IndexTuple>& tuples,
                                   long long n, int index, const Config& config, DevStats* stats,
                                   IndexTuple* result_tuple) {
    Runtime& rt = Runtime::get(config.device.device);
    std::vector<int> orders;
    for (const auto& t : tuples) orders.push_back(static_cast<int>(t.size()));
    std::vector<Buf> tensors = upload_all(rt, inputs, orders, n);
    Buf out;
    {
        Program prog(&rt, n, config, stats);
        std::vector<int> ids;
        for (const Buf& b : tensors) ids.push_back(prog.add_input(b));
        const int res = Contractor(prog, stats).eliminate_single(ids, tuples, index, result_tuple);
        prog.keep(res);
        prog.optimize();
        prog.execute();
        out = prog.take(res);
    }
    return download(rt, out);
}

std::string plan_summary(const std::vector<IndexTuple>& zero_sig, int m, long long n, const Config& config,
                         bool inputs_symmetric, Program::Totals* totals) {
    TermPlan plan = plan_terms(zero_sig, m, n, LatticeMode::Sparsified, config);
    if (config.device.shard_rows) plan.owner.assign(plan.owner.size(), 0);  // every rank records every term
    DevStats stats;
    Program prog(nullptr, n, config, &stats);
    // Declared-symmetric inputs: every order-2 factor is the same matrix (the
    // BASELINE configs alias one matrix); other factors are distinct.
    std::vector<int> ids;
    int shared_matrix = -1;
    for (const IndexTuple& t : zero_sig) {
        const int order = static_cast<int>(t.size());
        if (inputs_symmetric && order == 2) {
            if (shared_matrix < 0) shared_matrix = prog.add_symbolic_input(2, true);
            ids.push_back(shared_matrix);
        } else {
            ids.push_back(prog.add_symbolic_input(order, false));
        }
    }
    std::vector<double> dummy(plan.rgs.size() + 1);
    record_terms(prog, plan, ids, 0, dummy.data(), &stats);
    const double budget = config.device.memory_budget_bytes ? static_cast<double>(config.device.memory_budget_bytes)
                                                             : 179.0 * 1024 * 1024 * 1024;
    prog.optimize(budget);
    if (totals) *totals = prog.totals();
    std::string head = "terms=" + std::to_string(plan.rgs.size()) + " shared_hits=" + std::to_string(stats.shared_hits) +
                       " ref_madds=" + std::to_string(stats.ref_madds) + "\n";
    std::string tail;
    const int W = config.device.world_size;
    if (config.device.shard_rows && W > 1) {  // the row-sharding plan this rank would run
        prog.plan_shards(W);
        tail = "-- shard plan\n" + prog.shard_dump(config.device.rank);
    }
    return head + prog.dump() + tail;
}

}  // namespace ustats::dev
