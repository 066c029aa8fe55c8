// Contractor (executor.hpp): records one einsum with the reference's
// elimination walk (proj/src/einsum.cpp:310-486).
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
#include <mutex>
#include <numeric>
#include <string>

#include "executor_util.hpp"
#include "ustats/errors.hpp"
#include "ustats/partition.hpp"
#include "ustats/tensor.hpp"

namespace ustats::dev {

// -------------------------------------------------------------- Contractor
std::uint64_t Contractor::pw(int e) const { return ipow(p_.n(), e); }

void Contractor::cap(int order) {
    if (count_) checked_entry_count(order, static_cast<int>(p_.n()), p_.config());
}

void Contractor::owned(int order) {
    if (count_) count_->ref_peak = std::max(count_->ref_peak, pw(order));
}

Contractor::Slot Contractor::slot_of(int buf, const IndexTuple& tuple) {
    Slot s;
    s.factors.push_back(p_.view_of(buf, tuple));
    s.ids = s.factors[0].ids;
    std::uint32_t seen = 0;
    bool repeat = false;
    for (int id : tuple) {
        if (seen & bit(id)) repeat = true;
        seen |= bit(id);
    }
    if (repeat) {  // extract_diagonal (einsum.cpp:183-206): a strided view here
        cap(std::popcount(seen));
        owned(std::popcount(seen));
        s.owned = true;
    }
    return s;
}

std::vector<View> Contractor::formed(const Slot& s) {
    const std::uint32_t pend = ids_of_views(s.factors) & ~s.ids;
    if (!pend) return s.factors;
    std::vector<int> layout = ids_of(s.ids);
    int b = p_.stream(s.factors, layout, pend, nullptr);
    return {p_.view_of(b, layout)};
}

void Contractor::settle(Slot& s) {
    const std::uint32_t pend = ids_of_views(s.factors) & ~s.ids;
    if (!pend) return;
    std::vector<int> layout = ids_of(s.ids);
    const int b = p_.lookup_stream(s.factors, layout, pend);
    if (b < 0) return;
    s.factors = {p_.view_of(b, layout)};
}

Contractor::Slot Contractor::marginalize(const Slot& s, std::uint32_t summed) {
    const int kept = std::popcount(s.ids & ~summed);
    cap(kept);
    if (count_) count_->ref_madds += pw(std::popcount(s.ids));
    owned(kept);
    Slot r = s;
    r.ids = s.ids & ~summed;
    r.owned = true;
    return r;
}

Contractor::Slot Contractor::gemm_step(const Slot& a, const Slot& b, int e) {
    std::vector<int> ra, rb;
    for (int id : ids_of(a.ids))
        if (id != e) ra.push_back(id);
    for (int id : ids_of(b.ids))
        if (id != e) rb.push_back(id);
    cap(std::popcount(a.ids));
    cap(std::popcount(b.ids));
    cap(static_cast<int>(ra.size() + rb.size()));
    if (count_) count_->ref_madds += pw(static_cast<int>(ra.size())) * pw(1) * pw(static_cast<int>(rb.size()));
    owned(static_cast<int>(ra.size() + rb.size()));
    Slot r;
    r.owned = true;
    r.ids = (a.ids | b.ids) & ~bit(e);
    std::vector<View> fa = formed(a), fb = formed(b);
    if (ra.size() <= static_cast<std::size_t>(kMaxRowDims) && rb.size() <= static_cast<std::size_t>(kMaxRowDims)) {
        std::vector<int> layout;
        int buf = p_.gemm(fa, fb, ra, rb, e, &layout);
        r.factors.push_back(p_.view_of(buf, layout));
    } else {
        fa.insert(fa.end(), fb.begin(), fb.end());
        std::vector<int> layout = ids_of(r.ids);
        int buf = p_.stream(fa, layout, bit(e), nullptr);
        r.factors.push_back(p_.view_of(buf, layout));
    }
    return r;
}

Contractor::Slot Contractor::generic_step(const std::vector<Slot>& parts, int e) {
    std::uint32_t uni = 0;
    for (const Slot& p : parts) uni |= p.ids;
    uni &= ~bit(e);
    const int out_order = std::popcount(uni);
    cap(out_order);
    if (count_) count_->ref_madds += pw(out_order) * pw(1) * parts.size();
    owned(out_order);

    bool disjoint = true;
    std::uint32_t seen = 0;
    for (const Slot& p : parts) {
        const std::uint32_t rest = p.ids & ~bit(e);
        if (rest & seen) disjoint = false;
        seen |= rest;
    }
    std::size_t widest = 0;
    for (std::size_t i = 1; i < parts.size(); ++i)
        if (std::popcount(parts[i].ids) >= std::popcount(parts[widest].ids)) widest = i;
    std::vector<View> fa, fb;
    std::uint32_t rows = 0;
    for (std::size_t i = 0; i < parts.size(); ++i) {
        std::vector<View> fs = formed(parts[i]);
        if (i == widest) {
            fb.insert(fb.end(), fs.begin(), fs.end());
        } else {
            fa.insert(fa.end(), fs.begin(), fs.end());
            rows |= parts[i].ids & ~bit(e);
        }
    }
    const std::vector<int> ra = ids_of(rows), rb = ids_of(parts[widest].ids & ~bit(e));
    Slot r;
    r.owned = true;
    r.ids = uni;
    if (disjoint && !ra.empty() && !rb.empty() && ra.size() <= static_cast<std::size_t>(kMaxRowDims) &&
        rb.size() <= static_cast<std::size_t>(kMaxRowDims)) {
        std::vector<int> layout;
        int buf = p_.gemm(fa, fb, ra, rb, e, &layout);
        r.factors.push_back(p_.view_of(buf, layout));
    } else {
        fa.insert(fa.end(), fb.begin(), fb.end());
        std::vector<int> layout = ids_of(uni);
        int buf = p_.stream(fa, layout, bit(e), nullptr);
        r.factors.push_back(p_.view_of(buf, layout));
    }
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
    if (count_) ++count_->steps;
    for (Slot& p : parts) settle(p);

    for (bool folded = true; folded && parts.size() > 1;) {
        folded = false;
        for (std::size_t i = 0; i < parts.size() && !folded; ++i)
            for (std::size_t j = 0; j < parts.size(); ++j) {
                if (i == j) continue;
                if (std::popcount(parts[i].ids) > std::popcount(parts[j].ids)) continue;
                if ((parts[i].ids & ~parts[j].ids) != 0) continue;
                if (!parts[j].owned) {
                    owned(std::popcount(parts[j].ids));
                    parts[j].owned = true;
                }
                if (count_) count_->ref_madds += pw(std::popcount(parts[j].ids));
                std::vector<View> src = formed(parts[i]);  // a pending sum must not leak into the target
                settle(parts[j]);  // the target's own pending sum may be the op just formed
                parts[j].factors.insert(parts[j].factors.end(), src.begin(), src.end());
                parts.erase(parts.begin() + static_cast<std::ptrdiff_t>(i));
                folded = true;
                break;
            }
    }

    Slot result;
    if (parts.size() == 1) result = marginalize(parts[0], bit(e));
    else if (parts.size() == 2 && std::popcount(parts[0].ids & parts[1].ids) == 1) result = gemm_step(parts[0], parts[1], e);
    else result = generic_step(parts, e);
    slots.push_back(std::move(result));
}

int Contractor::run(const std::vector<int>& inputs, const EinsumNotation& notation, const EliminationOrder& order,
                    double* scalar_out) {
    const std::size_t K = notation.inputs.size();
    if (inputs.size() != K)
        fail(ErrorCode::ShapeMismatch,
             "notation expects " + std::to_string(K) + " tensors, got " + std::to_string(inputs.size()));
    for (std::size_t k = 0; k < K; ++k)
        if (p_.buf(inputs[k]).order != static_cast<int>(notation.inputs[k].size()))
            fail(ErrorCode::ShapeMismatch, "tensor " + std::to_string(k) + " has order " +
                                               std::to_string(p_.buf(inputs[k]).order) + " but its tuple has " +
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

    // assembly (einsum.cpp:466-485): one kernel over the widest slot's
    // pending sums; other pending sums are formed first.
    const int out_order = static_cast<int>(notation.output.size());
    cap(out_order);
    if (count_) count_->ref_madds += pw(out_order) * slots.size();
    for (Slot& s : slots) settle(s);
    std::size_t widest = 0;
    auto pend = [&](const Slot& s) { return ids_of_views(s.factors) & ~s.ids; };
    for (std::size_t i = 0; i < slots.size(); ++i)
        if (std::popcount(pend(slots[i])) > std::popcount(pend(slots[widest]))) widest = i;
    std::vector<View> all;
    std::uint32_t sum_ids = 0;
    for (std::size_t i = 0; i < slots.size(); ++i) {
        if (i != widest) {
            std::vector<View> f = formed(slots[i]);
            all.insert(all.end(), f.begin(), f.end());
        } else {
            all.insert(all.end(), slots[i].factors.begin(), slots[i].factors.end());
            sum_ids |= pend(slots[i]);
        }
    }
    std::vector<int> out_ids(notation.output.begin(), notation.output.end());
    return p_.stream(all, out_ids, sum_ids, out_ids.empty() ? scalar_out : nullptr);
}

int Contractor::eliminate_single(const std::vector<int>& inputs, const std::vector<IndexTuple>& tuples, int index,
                                 IndexTuple* result_tuple) {
    std::vector<Slot> slots;
    for (std::size_t k = 0; k < inputs.size(); ++k) slots.push_back(slot_of(inputs[k], tuples[k]));
    eliminate_one(slots, index);
    const Slot& r = slots.back();
    std::vector<int> asc = ids_of(r.ids);
    if (result_tuple) *result_tuple = asc;
    return p_.stream(r.factors, asc, ids_of_views(r.factors) & ~r.ids, nullptr);
}

}  // namespace ustats::dev
