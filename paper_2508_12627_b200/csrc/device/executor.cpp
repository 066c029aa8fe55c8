// Device executor (see executor.hpp). Host C++; launches the sm_100a kernels
// of stream_kernels.cu and gemm_f64.cu on one stream per device.
#include "executor.hpp"

#include <algorithm>
#include <bit>
#include <chrono>
#include <cstring>
#include <mutex>
#include <numeric>
#include <unordered_map>

#include "ustats/errors.hpp"
#include "ustats/partition.hpp"
#include "ustats/tensor.hpp"

namespace ustats::dev {

void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        fail(ErrorCode::CudaError, std::string(what) + ": " + cudaGetErrorString(e));
}

// ---------------------------------------------------------------- Runtime
DeviceBuffer::~DeviceBuffer() {
    if (ptr && !borrowed && rt) cudaFreeAsync(ptr, rt->stream());
}

std::uint64_t DeviceBuffer::entries() const {
    std::uint64_t e = 1;
    for (int i = 0; i < order; ++i) e *= static_cast<std::uint64_t>(n);
    return e;
}

Runtime& Runtime::get(int device) {
    static std::mutex mu;
    static std::map<int, std::unique_ptr<Runtime>> all;
    std::lock_guard<std::mutex> lock(mu);
    if (device < 0) check_cuda(cudaGetDevice(&device), "cudaGetDevice");
    auto& slot = all[device];
    if (!slot) slot.reset(new Runtime(device));
    check_cuda(cudaSetDevice(device), "cudaSetDevice");
    return *slot;
}

Runtime::Runtime(int device) : device_(device) {
    check_cuda(cudaSetDevice(device), "cudaSetDevice");
    check_cuda(cudaDeviceGetAttribute(&sm_count_, cudaDevAttrMultiProcessorCount, device),
               "cudaDeviceGetAttribute");
    check_cuda(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "cudaStreamCreate");
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        std::uint64_t keep = ~std::uint64_t{0};
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
}

Runtime::~Runtime() {}

Buf Runtime::allocate(int order, long long n) {
    auto b = std::make_shared<DeviceBuffer>();
    b->order = order;
    b->n = n;
    b->rt = this;
    b->uid = next_uid_++;
    void* p = nullptr;
    check_cuda(cudaMallocAsync(&p, std::max<std::uint64_t>(b->entries(), 1) * sizeof(double), stream_),
               "cudaMallocAsync");
    b->ptr = static_cast<double*>(p);
    return b;
}

Buf Runtime::borrow(const double* ptr, int order, long long n) {
    auto b = std::make_shared<DeviceBuffer>();
    b->ptr = const_cast<double*>(ptr);
    b->order = order;
    b->n = n;
    b->borrowed = true;
    b->rt = this;
    b->uid = next_uid_++;
    return b;
}

double* Runtime::scratch(std::size_t entries) {
    void* p = nullptr;
    check_cuda(cudaMallocAsync(&p, std::max<std::size_t>(entries, 1) * sizeof(double), stream_),
               "cudaMallocAsync(scratch)");
    return static_cast<double*>(p);
}

void Runtime::release(double* p) {
    if (p) cudaFreeAsync(p, stream_);
}

void Runtime::sync() { check_cuda(cudaStreamSynchronize(stream_), "cudaStreamSynchronize"); }

void Runtime::begin(Kind k) {
    if (!profiling_) return;
    while (pool_.size() < 2) {
        cudaEvent_t e;
        check_cuda(cudaEventCreate(&e), "cudaEventCreate");
        pool_.push_back(e);
    }
    Mark m{k, pool_.back(), nullptr};
    pool_.pop_back();
    m.b = pool_.back();
    pool_.pop_back();
    cudaEventRecord(m.a, stream_);
    marks_.push_back(m);
}

void Runtime::end(Kind k) {
    if (!profiling_ || marks_.empty()) return;
    (void)k;
    cudaEventRecord(marks_.back().b, stream_);
}

Runtime::Profile Runtime::collect(bool reset) {
    sync();
    for (const Mark& m : marks_) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, m.a, m.b) == cudaSuccess) {
            totals_.ms[m.kind] += ms;
            totals_.groups[m.kind] += 1;
        }
        pool_.push_back(m.a);
        pool_.push_back(m.b);
    }
    marks_.clear();
    Profile p = totals_;
    if (reset) totals_ = Profile{};
    return p;
}

// ------------------------------------------------------------- Contractor
namespace {
inline std::uint32_t bit(int id) { return 1u << id; }

std::vector<int> ids_of(std::uint32_t mask) {
    std::vector<int> v;
    for (std::uint32_t r = mask; r; r &= r - 1) v.push_back(std::countr_zero(r));
    return v;
}
}  // namespace

std::uint64_t Contractor::pw(int e) const {
    std::uint64_t v = 1;
    while (e-- > 0) v *= static_cast<std::uint64_t>(n_);
    return v;
}

void Contractor::ref_count_alloc(int order) {
    checked_entry_count(order, static_cast<int>(n_), config_);
}

void Contractor::ref_owned(int order) {
    if (stats_) stats_->ref_peak = std::max(stats_->ref_peak, pw(order));
}

Contractor::View Contractor::view_of(const Buf& b, const IndexTuple& tuple) const {
    View v;
    v.buf = b;
    long long s = 1;
    for (std::size_t p = tuple.size(); p-- > 0;) {
        if (tuple[p] >= kMaxIds) fail(ErrorCode::InvalidArgument, "too many indices for the device executor");
        v.stride[static_cast<std::size_t>(tuple[p])] += s;
        v.ids |= bit(tuple[p]);
        s *= n_;
    }
    return v;
}

Contractor::View Contractor::output_view(const Buf& b, const std::vector<int>& layout) const {
    return view_of(b, layout);
}

Contractor::Slot Contractor::slot_of(const Buf& b, const IndexTuple& tuple) {
    Slot s;
    s.factors.push_back(view_of(b, tuple));
    s.ids = s.factors[0].ids;
    IndexTuple distinct;
    for (int id : tuple)
        if (std::find(distinct.begin(), distinct.end(), id) == distinct.end()) distinct.push_back(id);
    if (distinct.size() != tuple.size()) {  // extract_diagonal (einsum.cpp:183-206): a strided view here
        ref_count_alloc(static_cast<int>(distinct.size()));
        ref_owned(static_cast<int>(distinct.size()));
        s.owned = true;
    }
    s.tuple = distinct;
    return s;
}

// Keeps at most `limit` factors by materializing the product of the leading
// ones over their joint ids (rare: very long fold chains).
std::vector<Contractor::View> Contractor::limit_factors(std::vector<View> fs, std::size_t limit) {
    while (fs.size() > limit) {
        const std::size_t take = std::min<std::size_t>(kMaxFactors, fs.size() - limit + 1);
        std::vector<View> head(fs.begin(), fs.begin() + static_cast<std::ptrdiff_t>(take));
        std::uint32_t ids = 0;
        for (const View& v : head) ids |= v.ids;
        std::vector<int> layout = ids_of(ids);
        Buf b = stream_to_buffer(head, layout, 0, nullptr);
        fs.erase(fs.begin(), fs.begin() + static_cast<std::ptrdiff_t>(take));
        fs.insert(fs.begin(), output_view(b, layout));
    }
    return fs;
}

Buf Contractor::stream_to_buffer(std::vector<View> factors, const std::vector<int>& out_ids,
                                 std::uint32_t sum_ids, double* out_ptr) {
    factors = limit_factors(std::move(factors), kMaxFactors);
    std::vector<int> sums = ids_of(sum_ids);
    // Innermost summed dim: the one most factors read with unit stride
    // (symmetric matrices can be read in either orientation).
    auto unit = [&](const View& v, int id) {
        if (!(v.ids & bit(id))) return false;
        if (v.stride[static_cast<std::size_t>(id)] == 1) return true;
        return v.buf->symmetric && std::popcount(v.ids) == 2;
    };
    if (!sums.empty()) {
        int best = sums.back(), best_score = -1;
        for (int id : sums) {
            int score = 0;
            for (const View& v : factors) score += unit(v, id) ? (v.buf->order >= 2 ? 4 : 1) : 0;
            if (score > best_score) {
                best_score = score;
                best = id;
            }
        }
        sums.erase(std::find(sums.begin(), sums.end(), best));
        sums.push_back(best);
    }
    int fast = -1;
    if (!sums.empty()) {
        int cs = 0, co = 0;
        for (const View& v : factors) {
            if (v.buf->symmetric) continue;
            cs += v.stride[static_cast<std::size_t>(sums.back())] == 1 && (v.ids & bit(sums.back()));
            if (!out_ids.empty())
                co += v.stride[static_cast<std::size_t>(out_ids.back())] == 1 && (v.ids & bit(out_ids.back()));
        }
        fast = (out_ids.empty() || cs >= co) ? sums.back() : out_ids.back();
    } else if (!out_ids.empty()) {
        fast = out_ids.back();
    }
    if (fast >= 0)
        for (View& v : factors) {
            if (!v.buf->symmetric || std::popcount(v.ids) != 2 || !(v.ids & bit(fast))) continue;
            if (v.stride[static_cast<std::size_t>(fast)] == 1) continue;
            const int other = std::countr_zero(v.ids & ~bit(fast));
            std::swap(v.stride[static_cast<std::size_t>(fast)], v.stride[static_cast<std::size_t>(other)]);
        }

    StreamArgs a;
    a.nf = static_cast<int>(factors.size());
    a.n_out = static_cast<int>(out_ids.size());
    a.n_sum = static_cast<int>(sums.size());
    a.n = n_;
    if (a.n_out + a.n_sum > kMaxDims)
        fail(ErrorCode::InvalidArgument, "contraction step spans too many indices for the stream kernel");
    std::vector<int> dims = out_ids;
    dims.insert(dims.end(), sums.begin(), sums.end());
    for (int f = 0; f < a.nf; ++f) {
        a.ptr[f] = factors[static_cast<std::size_t>(f)].buf->ptr;
        for (std::size_t d = 0; d < dims.size(); ++d)
            a.stride[f][d] = factors[static_cast<std::size_t>(f)].stride[static_cast<std::size_t>(dims[d])];
    }
    Buf result;
    if (out_ptr) {
        a.out = out_ptr;
    } else {
        result = rt_.allocate(static_cast<int>(out_ids.size()), n_);
        a.out = result->ptr;
    }
    const std::size_t scratch_n = stream_scratch_entries(a, rt_.sm_count());
    double* scratch = scratch_n ? rt_.scratch(scratch_n) : nullptr;
    rt_.begin(Runtime::kStream);
    const int launched = launch_stream(a, scratch, scratch_n, rt_.sm_count(), rt_.stream());
    rt_.end(Runtime::kStream);
    check_cuda(cudaGetLastError(), "stream kernel launch");
    if (stats_) stats_->kernel_launches += static_cast<std::uint64_t>(launched);
    rt_.release(scratch);
    if (stats_) {
        stats_->stream_entries += pw(a.n_out + a.n_sum) * static_cast<std::uint64_t>(a.nf);
        ++stats_->stream_launches;
    }
    return result;
}

Buf Contractor::gemm_to_buffer(std::vector<View> fa, std::vector<View> fb, const std::vector<int>& ra,
                               const std::vector<int>& rb, int e) {
    // Multi-factor (Hadamard / scaled / Khatri-Rao) operands are formed once
    // by a stream kernel into a k-major buffer (rows..., e): O(rows*n) traffic
    // against O(rows*cols*n) DMMA work, and the GEMM then runs the TMA path.
    auto flatten = [&](std::vector<View>& fs, const std::vector<int>& rows) {
        if (fs.size() <= 1) return;
        std::vector<int> layout = rows;
        layout.push_back(e);
        Buf m = stream_to_buffer(fs, layout, 0, nullptr);
        fs = {output_view(m, layout)};
    };
    flatten(fa, ra);
    flatten(fb, rb);
    fa = limit_factors(std::move(fa), kMaxGemmFactors);
    fb = limit_factors(std::move(fb), kMaxGemmFactors);
    // Orient symmetric factors so the inner (k) index is their fast axis.
    for (auto* side : {&fa, &fb})
        for (View& v : *side) {
            if (!v.buf->symmetric || std::popcount(v.ids) != 2 || !(v.ids & bit(e))) continue;
            if (v.stride[static_cast<std::size_t>(e)] == 1) continue;
            const int other = std::countr_zero(v.ids & ~bit(e));
            std::swap(v.stride[static_cast<std::size_t>(e)], v.stride[static_cast<std::size_t>(other)]);
        }
    auto fill = [&](GemmSide& side, const std::vector<View>& fs, const std::vector<int>& rows) {
        side.nf = static_cast<int>(fs.size());
        side.nr = static_cast<int>(rows.size());
        for (int f = 0; f < side.nf; ++f) {
            const View& v = fs[static_cast<std::size_t>(f)];
            side.ptr[f] = v.buf->ptr;
            side.kstride[f] = v.stride[static_cast<std::size_t>(e)];
            for (int d = 0; d < side.nr; ++d)
                side.rstride[f][d] = v.stride[static_cast<std::size_t>(rows[static_cast<std::size_t>(d)])];
        }
    };
    // k-major loads when the biggest factor is contiguous along k.
    auto kmajor = [&](const std::vector<View>& fs, const std::vector<int>& rows) {
        const View* big = &fs[0];
        for (const View& v : fs)
            if (v.buf->order > big->buf->order) big = &v;
        if (big->stride[static_cast<std::size_t>(e)] == 1) return 1;
        if (!rows.empty() && big->stride[static_cast<std::size_t>(rows.back())] == 1) return 0;
        return 1;
    };
    GemmArgs g;
    fill(g.a, fa, ra);
    fill(g.b, fb, rb);
    g.n = n_;
    g.rows = static_cast<long long>(pw(static_cast<int>(ra.size())));
    g.cols = static_cast<long long>(pw(static_cast<int>(rb.size())));
    g.a_kmajor = kmajor(fa, ra);
    g.b_kmajor = kmajor(fb, rb);
    g.mode = kEpiStore;
    Buf out = rt_.allocate(static_cast<int>(ra.size() + rb.size()), n_);
    g.out = out->ptr;
    rt_.begin(Runtime::kGemm);
    const int launched = launch_gemm(g, rt_.stream());
    rt_.end(Runtime::kGemm);
    check_cuda(cudaGetLastError(), "gemm launch");
    if (stats_) stats_->kernel_launches += static_cast<std::uint64_t>(launched);
    if (stats_) {
        stats_->gemm_macs += static_cast<std::uint64_t>(g.rows) * static_cast<std::uint64_t>(g.cols) *
                             static_cast<std::uint64_t>(n_);
        ++stats_->gemm_launches;
    }
    return out;
}

// Lazy marginalization: the sum is recorded on the slot and formed by the
// kernel that finally consumes (or materializes) it.
Contractor::Slot Contractor::marginalize(const Slot& s, std::uint32_t summed) {
    const int kept = std::popcount(s.ids & ~summed);
    ref_count_alloc(kept);
    if (stats_) stats_->ref_madds += pw(std::popcount(s.ids));
    ref_owned(kept);
    Slot r = s;
    r.ids = s.ids & ~summed;
    r.owned = true;
    IndexTuple t;
    for (int id : s.tuple)
        if (!(summed & bit(id))) t.push_back(id);
    r.tuple = t;
    // pending sums are the ids present in factors but not in the slot
    return r;
}

namespace {
std::uint32_t pending_of(const Contractor::Slot& s) {
    std::uint32_t all = 0;
    for (const auto& v : s.factors) all |= v.ids;
    return all & ~s.ids;
}
}  // namespace

Contractor::Slot Contractor::gemm_step(const Slot& a, const Slot& b, int e) {
    std::vector<int> ra, rb;
    for (int id : ids_of(a.ids))
        if (id != e) ra.push_back(id);
    for (int id : ids_of(b.ids))
        if (id != e) rb.push_back(id);
    ref_count_alloc(std::popcount(a.ids));
    ref_count_alloc(std::popcount(b.ids));
    ref_count_alloc(static_cast<int>(ra.size() + rb.size()));
    if (stats_) stats_->ref_madds += pw(static_cast<int>(ra.size())) * pw(1) * pw(static_cast<int>(rb.size()));
    ref_owned(static_cast<int>(ra.size() + rb.size()));

    auto operand = [&](const Slot& s) {
        if (!pending_of(s)) return s.factors;
        std::vector<int> layout = ids_of(s.ids);
        Buf m = stream_to_buffer(s.factors, layout, pending_of(s), nullptr);
        return std::vector<View>{output_view(m, layout)};
    };
    std::vector<int> layout = ra;
    layout.insert(layout.end(), rb.begin(), rb.end());
    Buf out;
    if (ra.size() <= static_cast<std::size_t>(kMaxRowDims) && rb.size() <= static_cast<std::size_t>(kMaxRowDims)) {
        out = gemm_to_buffer(operand(a), operand(b), ra, rb, e);
    } else {
        std::vector<View> all = operand(a);
        std::vector<View> fb = operand(b);
        all.insert(all.end(), fb.begin(), fb.end());
        out = stream_to_buffer(all, layout, bit(e), nullptr);
    }
    Slot r;
    r.factors.push_back(output_view(out, layout));
    r.ids = r.factors[0].ids;
    r.owned = true;
    std::vector<int> t = ra;
    t.insert(t.end(), rb.begin(), rb.end());
    r.tuple = t;
    return r;
}

Contractor::Slot Contractor::generic_step(const std::vector<Slot>& parts, int e) {
    std::uint32_t uni = 0;
    for (const Slot& p : parts) uni |= p.ids;
    uni &= ~bit(e);
    const int out_order = std::popcount(uni);
    ref_count_alloc(out_order);
    if (stats_) stats_->ref_madds += pw(out_order) * pw(1) * parts.size();
    ref_owned(out_order);

    // Khatri-Rao lowering: operands meeting only at e -> (rows of all but the
    // widest) x (rows of the widest) DMMA GEMM.
    bool disjoint = true;
    std::uint32_t seen = 0;
    for (const Slot& p : parts) {
        std::uint32_t rest = p.ids & ~bit(e);
        if (rest & seen) disjoint = false;
        seen |= rest;
    }
    std::vector<View> fa, fb;
    std::size_t widest = 0;
    for (std::size_t i = 1; i < parts.size(); ++i)
        if (std::popcount(parts[i].ids) >= std::popcount(parts[widest].ids)) widest = i;
    std::uint32_t rows_mask = 0;
    for (std::size_t i = 0; i < parts.size(); ++i) {
        std::vector<View> fs = parts[i].factors;
        if (pending_of(parts[i])) {
            std::vector<int> layout = ids_of(parts[i].ids);
            Buf m = stream_to_buffer(fs, layout, pending_of(parts[i]), nullptr);
            fs = {output_view(m, layout)};
        }
        if (i == widest) {
            fb.insert(fb.end(), fs.begin(), fs.end());
        } else {
            fa.insert(fa.end(), fs.begin(), fs.end());
            rows_mask |= parts[i].ids & ~bit(e);
        }
    }
    const std::vector<int> ra = ids_of(rows_mask);
    const std::vector<int> rb = ids_of(parts[widest].ids & ~bit(e));
    std::vector<int> layout = ra;
    layout.insert(layout.end(), rb.begin(), rb.end());
    Buf out;
    if (disjoint && !ra.empty() && !rb.empty() && ra.size() <= static_cast<std::size_t>(kMaxRowDims) &&
        rb.size() <= static_cast<std::size_t>(kMaxRowDims)) {
        out = gemm_to_buffer(fa, fb, ra, rb, e);
    } else {
        layout = ids_of(uni);
        std::vector<View> all = fa;
        all.insert(all.end(), fb.begin(), fb.end());
        out = stream_to_buffer(all, layout, bit(e), nullptr);
    }
    Slot r;
    r.factors.push_back(output_view(out, layout));
    r.ids = uni;
    r.owned = true;
    r.tuple = ids_of(uni);
    return r;
}

// eliminate_one (einsum.cpp:310-366): same operand collection, fold rule and
// dispatch; folds are lazy (factor lists concatenate).
void Contractor::eliminate_one(std::vector<Slot>& slots, int e) {
    std::vector<Slot> parts;
    for (auto it = slots.begin(); it != slots.end();) {
        if (it->ids & bit(e)) {
            parts.push_back(std::move(*it));
            it = slots.erase(it);
        } else {
            ++it;
        }
    }
    if (parts.empty()) return;
    if (stats_) ++stats_->steps;

    for (bool folded = true; folded && parts.size() > 1;) {
        folded = false;
        for (std::size_t i = 0; i < parts.size() && !folded; ++i)
            for (std::size_t j = 0; j < parts.size(); ++j) {
                if (i == j) continue;
                if (std::popcount(parts[i].ids) > std::popcount(parts[j].ids)) continue;
                if ((parts[i].ids & ~parts[j].ids) != 0) continue;
                if (!parts[j].owned) {
                    ref_owned(std::popcount(parts[j].ids));
                    parts[j].owned = true;
                }
                if (stats_) stats_->ref_madds += pw(std::popcount(parts[j].ids));
                Slot src = parts[i];
                if (pending_of(src)) {  // a pending sum must not leak into the target's space
                    std::vector<int> layout = ids_of(src.ids);
                    Buf m = stream_to_buffer(src.factors, layout, pending_of(src), nullptr);
                    src.factors = {output_view(m, layout)};
                }
                parts[j].factors.insert(parts[j].factors.end(), src.factors.begin(), src.factors.end());
                parts.erase(parts.begin() + static_cast<std::ptrdiff_t>(i));
                folded = true;
                break;
            }
    }

    Slot result;
    if (parts.size() == 1) {
        result = marginalize(parts[0], bit(e));
    } else if (parts.size() == 2 && std::popcount(parts[0].ids & parts[1].ids) == 1) {
        result = gemm_step(parts[0], parts[1], e);
    } else {
        result = generic_step(parts, e);
    }
    slots.push_back(std::move(result));
}

Buf Contractor::run(const std::vector<Buf>& inputs, const EinsumNotation& notation,
                    const EliminationOrder& order, double* scalar_out) {
    const std::size_t K = notation.inputs.size();
    if (inputs.size() != K)
        fail(ErrorCode::ShapeMismatch, "notation expects " + std::to_string(K) + " tensors, got " +
                                           std::to_string(inputs.size()));
    for (std::size_t k = 0; k < K; ++k)
        if (inputs[k]->order != static_cast<int>(notation.inputs[k].size()))
            fail(ErrorCode::ShapeMismatch, "tensor " + std::to_string(k) + " has order " +
                                               std::to_string(inputs[k]->order) + " but its tuple has " +
                                               std::to_string(notation.inputs[k].size()) + " indices");
    if (notation.index_count > kMaxIds)
        fail(ErrorCode::InvalidArgument, "device executor supports at most 16 indices per notation");

    std::vector<Slot> slots;
    for (std::size_t k = 0; k < K; ++k) slots.push_back(slot_of(inputs[k], notation.inputs[k]));

    // lone-index marginalization pre-pass (einsum.cpp:433-443)
    std::vector<int> occ(static_cast<std::size_t>(notation.index_count), 0);
    for (const Slot& s : slots)
        for (int id : ids_of(s.ids)) ++occ[static_cast<std::size_t>(id)];
    for (Slot& s : slots) {
        std::uint32_t lonely = 0;
        for (int id : ids_of(s.ids))
            if (occ[static_cast<std::size_t>(id)] == 1 && !notation.index_in_output(id)) lonely |= bit(id);
        if (lonely) s = marginalize(s, lonely);
    }

    for (int e : order.order) {
        if (notation.index_in_output(e)) continue;
        eliminate_one(slots, e);
    }

    // assembly (einsum.cpp:466-485): product of the surviving slots. Pending
    // sums of all but the widest slot are formed first so the final kernel
    // iterates one slot's space only.
    const int out_order = static_cast<int>(notation.output.size());
    ref_count_alloc(out_order);
    if (stats_) stats_->ref_madds += pw(out_order) * slots.size();
    std::size_t widest = 0;
    for (std::size_t i = 0; i < slots.size(); ++i)
        if (std::popcount(pending_of(slots[i])) > std::popcount(pending_of(slots[widest]))) widest = i;
    std::vector<View> all;
    std::uint32_t sum_ids = 0;
    for (std::size_t i = 0; i < slots.size(); ++i) {
        std::uint32_t pend = pending_of(slots[i]);
        if (pend && i != widest) {
            std::vector<int> layout = ids_of(slots[i].ids);
            Buf m = stream_to_buffer(slots[i].factors, layout, pend, nullptr);
            all.push_back(output_view(m, layout));
        } else {
            all.insert(all.end(), slots[i].factors.begin(), slots[i].factors.end());
            sum_ids |= pend;
        }
    }
    std::vector<int> out_ids(notation.output.begin(), notation.output.end());
    if (out_ids.empty() && scalar_out) {
        stream_to_buffer(all, out_ids, sum_ids, scalar_out);
        return nullptr;
    }
    return stream_to_buffer(all, out_ids, sum_ids, nullptr);
}

Buf Contractor::eliminate_single(const std::vector<Buf>& inputs, const std::vector<IndexTuple>& tuples,
                                 int index, IndexTuple* result_tuple) {
    std::vector<Slot> slots;
    for (std::size_t k = 0; k < inputs.size(); ++k) slots.push_back(slot_of(inputs[k], tuples[k]));
    eliminate_one(slots, index);
    const Slot& r = slots.back();
    std::vector<int> asc = ids_of(r.ids);
    if (result_tuple) *result_tuple = asc;
    return stream_to_buffer(r.factors, asc, pending_of(r), nullptr);
}

// ------------------------------------------------------- statistic drivers
namespace {

using Clock = std::chrono::steady_clock;

// Fixed-shape pairwise tree in term order (engine.cpp:25-34).
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
    const std::size_t T = parts.size();
    for (std::size_t t = 0; t < T; ++t) {
        plan.rgs.push_back(parts[t].rgs());
        plan.mu.push_back(mobius_coefficient(parts[t]));
        plan.notation.emplace_back(induced_signature(zero_sig, parts[t]));
        plan.order.push_back(optimize_order(plan.notation.back(), static_cast<int>(n), config.strategy, config));
        plan.cost.push_back(static_cast<double>(plan.order.back().predicted_peak_entries));
    }
    // LPT: heaviest term first onto the least-loaded rank (ties: lowest rank).
    plan.owner.assign(T, 0);
    const int W = std::max(1, config.device.world_size);
    if (W > 1) {
        std::vector<std::size_t> idx(T);
        std::iota(idx.begin(), idx.end(), 0);
        std::stable_sort(idx.begin(), idx.end(),
                         [&](std::size_t a, std::size_t b) { return plan.cost[a] > plan.cost[b]; });
        std::vector<double> load(static_cast<std::size_t>(W), 0.0);
        for (std::size_t t : idx) {
            auto w = static_cast<std::size_t>(std::min_element(load.begin(), load.end()) - load.begin());
            plan.owner[t] = static_cast<int>(w);
            load[w] += plan.cost[t];
        }
    }
    return plan;
}

StatisticResult lattice_statistic(const std::vector<const double*>& inputs, bool inputs_on_device,
                                  const std::vector<IndexTuple>& zero_sig, int m, long long n,
                                  LatticeMode mode, const Config& config) {
    StatisticResult res;
    Runtime& rt = Runtime::get(config.device.device);
    const auto t_up = Clock::now();

    // Upload each distinct factor once; sparsify on device (tensor.cpp:54-76).
    std::map<const double*, Buf> by_ptr;
    std::vector<Buf> tensors;
    std::vector<std::pair<Buf, int*>> probes;
    int* flags = nullptr;
    if (config.device.exploit_symmetry) check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&flags), sizeof(int) * zero_sig.size() + 4, rt.stream()), "alloc flags");
    for (std::size_t k = 0; k < zero_sig.size(); ++k) {
        const int order = static_cast<int>(zero_sig[k].size());
        checked_entry_count(order, static_cast<int>(n), config);
        auto hit = by_ptr.find(inputs[k]);
        if (hit != by_ptr.end() && hit->second->order == order) {
            tensors.push_back(hit->second);
            continue;
        }
        Buf b = rt.allocate(order, n);
        check_cuda(cudaMemcpyAsync(b->ptr, inputs[k], b->entries() * sizeof(double),
                                   inputs_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                   rt.stream()),
                   "upload");
        rt.begin(Runtime::kOther);
        if (mode == LatticeMode::Sparsified)
            res.stats.kernel_launches += static_cast<std::uint64_t>(launch_sparsify(b->ptr, order, n, rt.stream()));
        if (flags && order == 2) {
            int* f = flags + probes.size();
            res.stats.kernel_launches += static_cast<std::uint64_t>(launch_symmetry_check(b->ptr, n, f, rt.stream()));
            probes.emplace_back(b, f);
        }
        rt.end(Runtime::kOther);
        by_ptr[inputs[k]] = b;
        tensors.push_back(b);
    }
    if (!probes.empty()) {
        std::vector<int> host(probes.size());
        check_cuda(cudaMemcpyAsync(host.data(), flags, sizeof(int) * probes.size(), cudaMemcpyDeviceToHost,
                                   rt.stream()),
                   "flags");
        rt.sync();
        for (std::size_t i = 0; i < probes.size(); ++i) probes[i].first->symmetric = host[i] == 0;
    }
    if (flags) cudaFreeAsync(flags, rt.stream());
    rt.sync();
    res.upload_seconds = std::chrono::duration<double>(Clock::now() - t_up).count();

    const auto t0 = Clock::now();
    TermPlan plan = plan_terms(zero_sig, m, n, mode, config);
    const std::size_t T = plan.rgs.size();
    res.enumerated = plan.enumerated;
    res.owner = plan.owner;

    double* d_v = rt.scratch(std::max<std::size_t>(T, 1));
    check_cuda(cudaMemsetAsync(d_v, 0, sizeof(double) * std::max<std::size_t>(T, 1), rt.stream()), "memset");
    for (std::size_t t = 0; t < T; ++t) {
        if (res.owner[t] != config.device.rank) continue;
        Contractor c(rt, n, config, &res.stats);
        c.run(tensors, plan.notation[t], plan.order[t], d_v + t);
    }
    res.v.assign(T, 0.0);
    if (T) check_cuda(cudaMemcpyAsync(res.v.data(), d_v, sizeof(double) * T, cudaMemcpyDeviceToHost, rt.stream()), "D2H");
    rt.release(d_v);
    tensors.clear();
    by_ptr.clear();
    probes.clear();
    rt.sync();
    res.contract_seconds = std::chrono::duration<double>(Clock::now() - t0).count();

    res.terms.resize(T);
    res.mu.resize(T);
    res.rgs.resize(T);
    for (std::size_t t = 0; t < T; ++t) {
        res.mu[t] = plan.mu[t];
        res.rgs[t] = plan.rgs[t];
        res.terms[t] = static_cast<double>(res.mu[t]) * res.v[t];
    }
    res.value = combine_terms(res.terms);
    return res;
}

std::vector<double> contract_host(const std::vector<const double*>& inputs, const std::vector<int>& orders,
                                  long long n, const EinsumNotation& notation, const EliminationOrder* order,
                                  const Config& config, DevStats* stats) {
    Runtime& rt = Runtime::get(config.device.device);
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
        check_cuda(cudaMemcpyAsync(b->ptr, inputs[k], b->entries() * sizeof(double), cudaMemcpyHostToDevice,
                                   rt.stream()),
                   "upload");
        by_ptr[key] = b;
        tensors.push_back(b);
    }
    EliminationOrder chosen;
    if (!order) {
        chosen = optimize_order(notation, static_cast<int>(n), config.strategy, config);
        order = &chosen;
    }
    Contractor c(rt, n, config, stats);
    Buf out = c.run(tensors, notation, *order, nullptr);
    std::vector<double> host(out->entries());
    check_cuda(cudaMemcpyAsync(host.data(), out->ptr, host.size() * sizeof(double), cudaMemcpyDeviceToHost,
                               rt.stream()),
               "D2H");
    out.reset();
    tensors.clear();
    by_ptr.clear();
    rt.sync();
    return host;
}

}  // namespace ustats::dev
