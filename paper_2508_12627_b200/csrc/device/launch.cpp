// Program execution (executor.hpp): kernel launch per op, the two-stream
// schedule, row-sharded lockstep execution, plan reuse.
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

void Program::run_sweep(const Op& op) {
    SweepArgs a;
    a.x = ptr(op.factors[0].buf);
    a.xr = n_;
    a.cols = n_;
    a.r0 = 0;
    a.r1 = n_;
    if (slice_world_ > 1) {
        a.r0 = row_lo(slice_rank_);
        a.r1 = row_lo(slice_rank_ + 1);
        a.accumulate = 1;
        if (a.r1 <= a.r0) return;
    }
    const int blocks = sweep_blocks(a.r1 - a.r0, rt_->sm_count());
    std::size_t scalars = 0;
    for (const Op::Epi& e : op.epis) scalars += e.mode == kEpiSumAll;
    double* scratch = scalars ? rt_->scratch(scalars * static_cast<std::size_t>(blocks)) : nullptr;
    std::size_t at = 0;
    for (const Op::Epi& e : op.epis) {
        SweepOut& o = a.o[a.count++];
        o.mode = e.mode == kEpiSumAll ? kSweepAll : kSweepRow;
        o.power = e.self_power;
        for (const View& v : e.w) {
            const auto [wr, wc] = sweep_strides(v, e.row_id, e.col_id);
            if (wc != 0 || o.nrow >= 4) fail(ErrorCode::InvalidArgument, "executor: sweep weight is not a row weight");
            o.rowv[o.nrow] = ptr(v.buf);
            o.rows_stride[o.nrow++] = wr;
        }
        if (e.ext) {
            o.out = e.ext;
        } else {
            SymBuf& b = bufs_[static_cast<std::size_t>(e.out)];
            if (!b.real) {
                b.real = rt_->allocate(b.order, n_);
                if (slice_world_ > 1)
                    check_cuda(cudaMemsetAsync(b.real->ptr, 0, b.real->entries() * sizeof(double), rt_->stream()),
                               "memset");
            }
            o.out = b.real->ptr;
        }
        if (o.mode == kSweepAll) {
            o.partial = scratch + at;
            at += static_cast<std::size_t>(blocks);
        }
    }
    rt_->begin(Runtime::kStream);
    const int launched = launch_sweep(a, rt_->sm_count(), rt_->stream());
    rt_->end(Runtime::kStream);
    check_cuda(cudaGetLastError(), "sweep launch");
    rt_->release(scratch);
    if (stats_) {
        stats_->stream_entries += ipow(n_, 2);
        ++stats_->stream_launches;
        stats_->kernel_launches += static_cast<std::uint64_t>(launched);
    }
}

double* Program::ptr(int buf) const {
    const SymBuf& b = bufs_[static_cast<std::size_t>(buf)];
    if (!b.real) fail(ErrorCode::InvalidArgument, "executor: operand buffer b" + std::to_string(buf) + " not materialized");
    return b.real->ptr;
}

void Program::run_stream(const Op& op, double* out) {
    std::vector<View> factors = op.factors;
    std::vector<int> sums = ids_of(op.sum);
    const std::vector<int>& out_ids = op.out_ids;
    auto unit = [&](const View& v, int id) {
        if (!(v.ids & bit(id))) return false;
        if (v.stride[static_cast<std::size_t>(id)] == 1) return true;
        return bufs_[static_cast<std::size_t>(v.buf)].symmetric && std::popcount(v.ids) == 2;
    };
    if (!sums.empty()) {
        int best = sums.back(), best_score = -1;
        for (int id : sums) {
            int score = 0;
            for (const View& v : factors)
                score += unit(v, id) ? (bufs_[static_cast<std::size_t>(v.buf)].order >= 2 ? 4 : 1) : 0;
            if (score > best_score) {
                best_score = score;
                best = id;
            }
        }
        sums.erase(std::find(sums.begin(), sums.end(), best));
        sums.push_back(best);
    }
    // row sharding of a reduction to a scalar: the planned id is sliced (dim 0)
    const int shard_id = (slice_world_ > 1 && step_) ? step_->shard_id : -1;
    if (shard_id >= 0 && out_ids.empty() && sums.size() > 1 && sums.front() != shard_id) {
        sums.erase(std::find(sums.begin(), sums.end(), shard_id));
        sums.insert(sums.begin(), shard_id);
    }
    // The output dim along which the big non-symmetric operand is contiguous
    // may not be the layout's last (C4: b9{1:1024 2:1 3:n^2} summed over 1
    // into (2,3)): iterate it fastest, one thread per output, writing through
    // output strides, instead of reading that operand with a stride of n.
    std::vector<int> ord = out_ids;
    int moved = -1;
    if (!sums.empty() && out_ids.size() >= 2 && slice_world_ == 1) {
        auto weight = [&](const View& v, int id) -> long long {
            const SymBuf& b = bufs_[static_cast<std::size_t>(v.buf)];
            if (b.symmetric || !(v.ids & bit(id)) || v.stride[static_cast<std::size_t>(id)] != 1) return 0;
            return b.order >= 3 ? 16 : b.order == 2 ? 4 : 1;
        };
        long long on_sum = 0, best = 0;
        for (const View& v : factors) on_sum += weight(v, sums.back());
        for (int id : out_ids) {
            long long w = 0;
            for (const View& v : factors) w += weight(v, id);
            if (w > best) {
                best = w;
                moved = id;
            }
        }
        if (moved == out_ids.back() || best <= on_sum) moved = -1;
        if (moved >= 0) {
            ord.erase(std::find(ord.begin(), ord.end(), moved));
            ord.push_back(moved);
        }
    }
    int fast = -1;
    if (moved >= 0) {
        fast = moved;
    } else if (!sums.empty()) {
        int cs = 0, co = 0;
        for (const View& v : factors) {
            if (bufs_[static_cast<std::size_t>(v.buf)].symmetric) continue;
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
            if (!bufs_[static_cast<std::size_t>(v.buf)].symmetric || std::popcount(v.ids) != 2 || !(v.ids & bit(fast)))
                continue;
            if (v.stride[static_cast<std::size_t>(fast)] == 1) continue;
            const int other = std::countr_zero(v.ids & ~bit(fast));
            std::swap(v.stride[static_cast<std::size_t>(fast)], v.stride[static_cast<std::size_t>(other)]);
        }
    // a row-sharded symmetric matrix read through its transpose: read it by
    // rows along the sliced id (this rank holds only those rows)
    if (shard_id >= 0)
        for (View& v : factors) {
            const SymBuf& sb = bufs_[static_cast<std::size_t>(v.buf)];
            if (sb.input || !sb.symmetric || sb.order != 2 || std::popcount(v.ids) != 2 || !(v.ids & bit(shard_id)))
                continue;
            if (v.stride[static_cast<std::size_t>(shard_id)] >= n_) continue;
            const int other = std::countr_zero(v.ids & ~bit(shard_id));
            std::swap(v.stride[static_cast<std::size_t>(shard_id)], v.stride[static_cast<std::size_t>(other)]);
        }
    StreamArgs a;
    a.nf = static_cast<int>(factors.size());
    a.n_out = static_cast<int>(out_ids.size());
    a.n_sum = static_cast<int>(sums.size());
    a.n = n_;
    std::vector<int> dims = ord;
    dims.insert(dims.end(), sums.begin(), sums.end());
    for (int f = 0; f < a.nf; ++f) {
        a.ptr[f] = ptr(factors[static_cast<std::size_t>(f)].buf);
        for (std::size_t d = 0; d < dims.size(); ++d)
            a.stride[f][d] = factors[static_cast<std::size_t>(f)].stride[static_cast<std::size_t>(dims[d])];
    }
    a.out = out;
    if (moved >= 0) {
        a.permuted_out = 1;
        for (std::size_t d = 0; d < ord.size(); ++d) {
            const auto k = static_cast<std::size_t>(std::find(out_ids.begin(), out_ids.end(), ord[d]) - out_ids.begin());
            a.ostride[d] = static_cast<long long>(ipow(n_, static_cast<int>(out_ids.size() - 1 - k)));
        }
    }
    if (slice_world_ > 1) {
        // row sharding: this rank covers [lo, hi) of iteration dim 0 (an output
        // dim -> disjoint rows of the zeroed output; a summed dim -> a partial
        // sum); every rank accumulates, the all-reduce / lockstep adds them up
        a.accumulate = 1;
        if (dims.empty()) {
            if (slice_rank_ != 0) return;
        } else {
            const long long lo = row_lo(slice_rank_), hi = row_lo(slice_rank_ + 1);
            if (hi <= lo) return;
            a.n0 = hi - lo;
            for (int f = 0; f < a.nf; ++f) a.ptr[f] += lo * a.stride[f][0];
            if (a.n_out >= 1) a.out += lo * static_cast<long long>(ipow(n_, a.n_out - 1));
        }
    }
    const std::size_t scratch_n = stream_scratch_entries(a, rt_->sm_count());
    double* scratch = scratch_n ? rt_->scratch(scratch_n) : nullptr;
    rt_->begin(Runtime::kStream);
    const int launched = launch_stream(a, scratch, scratch_n, rt_->sm_count(), rt_->stream());
    rt_->end(Runtime::kStream);
    check_cuda(cudaGetLastError(), "stream kernel launch");
    rt_->release(scratch);
    if (stats_) {
        stats_->stream_entries += ipow(n_, a.n_out + a.n_sum) * static_cast<std::uint64_t>(a.nf);
        ++stats_->stream_launches;
        stats_->kernel_launches += static_cast<std::uint64_t>(launched);
    }
}

// FP64 emulation on the INT8 tensor cores (gemm_ozaki.cu) for large plain
// products whose K keeps every digit diagonal exact in int32.
// Smallest rows / cols / K of an emulated GEMM: below 1024, DMMA is as fast and
// needs no digit pass, and per-tile drains outweigh the MMA savings (C4's
// Khatri-Rao GEMMs, K = 1024: 297 -> 216 ms per evaluation). Config.oz_min_dim
// lowers it (tests pin the emulated path at sizes the CPU reference reaches).
long long oz_min_dim(const DeviceConfig& dc) { return dc.oz_min_dim > 0 ? dc.oz_min_dim : 1024; }
constexpr double kOzDigitCap = 6.5 * 1073741824.0;  // digit bytes per operand per K chunk (C4: 4 GiB split its
                                                    // K = 1024 GEMMs in two, 112 -> 158 ms per evaluation; C5:
                                                    // four chunks of 16384, 6.0 GiB per operand)
constexpr double kOzDigitCapLong = 8.25 * 1073741824.0;  // where the schedule has room (Op::long_chunks): C5 runs
                                                         // three chunks of 21888 (8.02 GiB per operand) there

// Error-bound guard. With S balanced 8-bit slices, truncation and the dropped
// products t + u >= S bound every entry's error by (S + 2) 2^{2-8S} K
// max|A_i| max|B_j| (gemm_ozaki.cu). The FP64 dot product the emulation
// replaces has the classical worst-case bound gamma_K = K u / (1 - K u),
// u = 2^-53, over the same K max|A_i| max|B_j|. The guard takes the fewest
// slices whose bound does not exceed gamma_K, so the emulated product is never
// less accurate, worst case, than the DMMA product it replaces (S = 6 for every
// K >= 1024, S = 7 below); a forced Config.oz_slices overrides it (tests).
int oz_guard_slices(long long K) {
    const double u = std::ldexp(1.0, -53), gamma = static_cast<double>(K) * u / (1.0 - static_cast<double>(K) * u);
    for (int S = 4; S <= kOzMaxSlices; ++S)
        if ((S + 2) * std::ldexp(1.0, 2 - 8 * S) <= gamma) return S;
    return kOzMaxSlices;
}

OzPlan oz_plan(long long K, long long rows, long long cols, bool same_operand, const DeviceConfig& dc,
               bool long_chunks) {
    OzPlan p;
    p.slices = dc.oz_slices > 0 ? dc.oz_slices : oz_guard_slices(K);
    // the products of K * 128^2 one int32 accumulator sums must stay below 2^31: S on the top
    // diagonal, S - 1 since the kernels split it over two accumulators (S > 4, gemm_ozaki.cu)
    const long long per_acc = p.slices > 4 ? p.slices - 1 : p.slices;
    const long long exact = ((1ll << 31) - 1) / (per_acc * 128 * 128) / 64 * 64;
    const long long max_k = dc.oz_max_k > 0 ? std::min<long long>(dc.oz_max_k / 64 * 64, exact) : exact;
    // fewest chunks whose digit panels stay within kOzDigitCap per operand (C5:
    // 65536 rows x 65536 K would need 24 GiB of digits per operand; 4, 6, 8 and
    // 12 chunks measured within 2% of each other there)
    const long long rows_pad = (std::max(rows, cols) + 127) / 128 * 128;
    double cap = long_chunks ? kOzDigitCapLong : kOzDigitCap;
    if (const char* e = std::getenv("USTATS_OZ_DIGIT_CAP_GB")) cap = std::atof(e) * 1073741824.0;
    const long long cap_k = std::max<long long>(64, static_cast<long long>(cap / (static_cast<double>(rows_pad) * p.slices)) / 64 * 64);
    const long long limit = std::min(max_k, cap_k);
    p.nchunks = (K + limit - 1) / limit;
    p.kc = ((K + p.nchunks - 1) / p.nchunks + 63) / 64 * 64;  // chunk starts stay 512-byte aligned
    while (p.kc > limit) {
        ++p.nchunks;
        p.kc = ((K + p.nchunks - 1) / p.nchunks + 63) / 64 * 64;
    }
    p.a_bytes = ozaki_slice_bytes(rows, p.kc, 128) * static_cast<std::size_t>(p.slices);
    p.b_bytes = same_operand ? 0 : ozaki_slice_bytes(cols, p.kc, 128) * static_cast<std::size_t>(p.slices);
    p.scratch_bytes = p.a_bytes + p.b_bytes + ozaki_work_entries() * sizeof(double) +
                      sizeof(int) * static_cast<std::size_t>(rows + cols) + (std::size_t{96} << 20);  // + tail partials
    return p;
}

// A single-factor operand whose row digits flatten to one stride (a
// materialized Khatri-Rao operand of n^2 rows is one): its row stride, or -1.
long long flat_row_stride(const GemmSide& s, long long n) {
    if (s.nf != 1) return -1;
    for (int d = s.nr - 1; d > 0; --d)
        if (s.rstride[0][d - 1] != s.rstride[0][d] * n) return -1;
    return s.rstride[0][s.nr - 1];
}

// A lazy operand (a product of factors: a Khatri-Rao / Hadamard operand the
// optimizer left unmaterialized, Program::lazy_operands) is digitized
// straight from its factors (ozaki_split_lazy).
bool lazy_side(const GemmSide& s) { return s.nf >= 2 && s.nf <= kMaxGemmFactors && s.nr <= kMaxRowDims; }

bool Program::emulated_eligible(const GemmArgs& g) const {
    if (!config_.device.fp64_emulation) return false;
    const long long lo = oz_min_dim(config_.device);
    if (g.n < lo || g.rows < lo || g.cols < lo) return false;
    return (flat_row_stride(g.a, n_) >= 0 || lazy_side(g.a)) && (flat_row_stride(g.b, n_) >= 0 || lazy_side(g.b));
}

// The transient device bytes an op needs while it runs, beyond its outputs:
// the emulated GEMM's digit panels for one K chunk (the memory-bounded
// schedule adds them at the op, so they are planned, not found at run time).
std::size_t Program::op_scratch_bytes(const Op& op) const {
    if (!op.gemm || !config_.device.fp64_emulation) return 0;
    const long long rows = static_cast<long long>(ipow(n_, static_cast<int>(op.ra.size())));
    const long long cols = static_cast<long long>(ipow(n_, static_cast<int>(op.rb.size())));
    const long long lo = oz_min_dim(config_.device);
    if (n_ < lo || rows < lo || cols < lo) return 0;
    const bool same = op.fa.size() == 1 && op.fb.size() == 1 && op.fa[0].buf == op.fb[0].buf && rows == cols;
    return oz_plan(n_, rows, cols, same, config_.device, op.long_chunks).scratch_bytes;
}

// Digits of both operands, the product (straight into a plain store's output,
// else into scratch), then the fused epilogues over the stored product.
// K beyond the exact int32 bound (C5: K = 65536) runs as equal K chunks (oz_plan),
// each digitized on its own (per-chunk row exponents) and accumulated into the
// outputs in chunk order: every epilogue is linear in C.
// The canonical description of a GEMM operand (factor buffers and their row /
// K strides, a symmetric matrix read K-contiguous as run_gemm reads it): two
// GEMMs with the same key digitize the same values.
std::string Program::operand_key(const std::vector<View>& fs, const std::vector<int>& rows, int e) const {
    std::vector<std::string> parts;
    for (View v : fs) {
        if (bufs_[static_cast<std::size_t>(v.buf)].symmetric && std::popcount(v.ids) == 2 && (v.ids & bit(e)) &&
            v.stride[static_cast<std::size_t>(e)] != 1) {
            const int other = std::countr_zero(v.ids & ~bit(e));
            std::swap(v.stride[static_cast<std::size_t>(e)], v.stride[static_cast<std::size_t>(other)]);
        }
        std::string k = "b" + std::to_string(v.buf) + ":";
        for (int id : rows) k += std::to_string(v.stride[static_cast<std::size_t>(id)]) + ",";
        k += "k" + std::to_string(v.stride[static_cast<std::size_t>(e)]);
        parts.push_back(k);
    }
    std::sort(parts.begin(), parts.end());
    std::string key = std::to_string(rows.size()) + "|";
    for (const auto& p : parts) key += p + ";";
    return key;
}

// How many emulated single-chunk GEMMs read each operand (single-GPU runs).
void Program::plan_digit_reuse() {
    digit_uses_.clear();
    const long long lo = oz_min_dim(config_.device);
    if (!config_.device.fp64_emulation || n_ < lo) return;
    for (std::size_t i : schedule_) {
        const Op& op = ops_[i];
        if (op.dead || !op.gemm) continue;
        const long long rows = static_cast<long long>(ipow(n_, static_cast<int>(op.ra.size())));
        const long long cols = static_cast<long long>(ipow(n_, static_cast<int>(op.rb.size())));
        if (rows < lo || cols < lo) continue;
        if (oz_plan(n_, rows, cols, false, config_.device).nchunks != 1) continue;
        const std::string ka = operand_key(op.fa, op.ra, op.e), kb = operand_key(op.fb, op.rb, op.e);
        ++digit_uses_[ka];
        if (kb != ka) ++digit_uses_[kb];
    }
}

void Program::drop_digits() {
    for (auto& [key, c] : digits_) {
        rt_->raw_free(c.d, c.bytes);
        rt_->release(reinterpret_cast<double*>(c.e));
    }
    digits_.clear();
}

int Program::run_emulated(const GemmArgs& g, const EpiSet& set) {
    cudaStream_t s = rt_->stream();
    // one set of digits when both operands are the same matrix view (A A^T)
    const long long ars = flat_row_stride(g.a, n_), brs = flat_row_stride(g.b, n_);
    const bool same = ars >= 0 && brs >= 0 && g.a.ptr[0] == g.b.ptr[0] && g.rows == g.cols && ars == brs &&
                      g.a.kstride[0] == g.b.kstride[0];
    const OzPlan oz = oz_plan(g.n, g.rows, g.cols, same, config_.device, cur_long_chunks_);
    const int S = oz.slices;
    const long long kc = oz.kc;
    if (oz.nchunks > 1)  // a consumer of C^2 is not linear in C: the caller runs it on DMMA
        for (int q = 0; q < set.count; ++q)
            if (set.d[q].self_power != 1) return -1;
    // digit reuse across GEMMs (one K chunk, whole operands, memory to spare)
    const bool reuse = oz.nchunks == 1 && slice_world_ == 1 && block_rows_.first < 0 && g.tile_count < 0 &&
                       !key_a_.empty() && budget_ > 0 && (same || key_a_ != key_b_);
    auto cached = [&](const std::string& key) -> CachedDigits* {
        auto it = digits_.find(key);
        return (reuse && it != digits_.end()) ? &it->second : nullptr;
    };
    CachedDigits* ca = cached(key_a_);
    CachedDigits* cb = same ? nullptr : cached(key_b_);
    // digit panels: slabs the schedule planned for (op_scratch_bytes); the
    // choice of engine depends only on the plan, never on a failed allocation,
    // so row-sharded ranks always agree on it
    int8_t* da = ca ? ca->d : static_cast<int8_t*>(rt_->raw_alloc(oz.a_bytes));
    int8_t* db = same ? da : cb ? cb->d : static_cast<int8_t*>(rt_->raw_alloc(oz.b_bytes));
    int* ea = ca ? ca->e : static_cast<int*>(rt_->raw_alloc(sizeof(int) * static_cast<std::size_t>(g.rows), false));
    int* eb = same ? ea : cb ? cb->e : static_cast<int*>(rt_->raw_alloc(sizeof(int) * static_cast<std::size_t>(g.cols), false));
    double* work = static_cast<double*>(rt_->raw_alloc(ozaki_work_entries() * sizeof(double), false));
    const bool sym = g.symmetric_out && g.rows == g.cols;
    int launched = 0;
    long long tiles = 0;
    auto split = [&](const double* x, long long rows, long long k, long long rs, long long ks, int8_t* out, int* exps,
                     const std::vector<int>* panels) {
        const int l = ozaki_split(x, rows, k, rs, ks, 128, S, out, exps, s, panels);
        if (l < 0) fail(ErrorCode::CudaError, "executor: Ozaki digit split failed");
        check_cuda(cudaPeekAtLastError(), "Ozaki digit split launch");
        launched += l;
    };
    auto split_lazy = [&](const GemmSide& side, long long rows, long long k0, long long k, int8_t* out, int* exps) {
        const int l = ozaki_split_lazy(side, n_, rows, k0, k, S, out, exps, s);
        if (l < 0) fail(ErrorCode::CudaError, "executor: lazy Ozaki digit split failed");
        check_cuda(cudaPeekAtLastError(), "lazy Ozaki digit split launch");
        launched += l;
    };
    const bool lazy_a = ars < 0, lazy_b = brs < 0;
    for (long long k0 = 0; k0 < g.n; k0 += kc) {
        const long long k = std::min(kc, g.n - k0);
        const double* xa = g.a.ptr[0] + k0 * g.a.kstride[0];
        const double* xb = g.b.ptr[0] + k0 * g.b.kstride[0];
        OzakiArgs p;
        p.a = da;
        p.b = db;
        // slice stride of this chunk's digit layout (a shorter last chunk packs tighter)
        p.a_slice = static_cast<long long>(ozaki_slice_bytes(g.rows, k, 128));
        p.b_slice = static_cast<long long>(ozaki_slice_bytes(g.cols, k, 128));
        p.a_exp = ea;
        p.b_exp = eb;
        p.m = g.rows;
        p.n = g.cols;
        p.mpad = (g.rows + 127) / 128 * 128;
        p.npad = (g.cols + 127) / 128 * 128;
        p.kpad = (k + 63) / 64 * 64;
        p.slices = S;
        p.symmetric = sym ? 1 : 0;
        p.accumulate = k0 == 0 ? g.accumulate : 1;
        p.epis = set;  // the same fused consumers (and partial slots) as the DMMA kernel's
        if (g.tile_count >= 0) {  // row sharding: this rank's range of the (same) tile list
            p.tile_begin = g.tile_begin;
            p.tile_count = g.tile_count;
        }
        tiles = p.tile_count >= 0 ? p.tile_count : ozaki_tile_count(p);
        p.work = work;
        // digits: all panels, or under row sharding only the panels this rank's tiles read
        if (ca || cb) {  // reused digits for one side (one chunk: k0 == 0)
            if (!ca) {
                if (lazy_a) split_lazy(g.a, g.rows, k0, k, da, ea);
                else split(xa, g.rows, k, ars, g.a.kstride[0], da, ea, nullptr);
            }
            if (!cb && !same) {
                if (lazy_b) split_lazy(g.b, g.cols, k0, k, db, eb);
                else split(xb, g.cols, k, brs, g.b.kstride[0], db, eb, nullptr);
            }
        } else if (lazy_a || lazy_b) {
            if (lazy_a) split_lazy(g.a, g.rows, k0, k, da, ea);
            else split(xa, g.rows, k, ars, g.a.kstride[0], da, ea, nullptr);
            if (lazy_b) split_lazy(g.b, g.cols, k0, k, db, eb);
            else split(xb, g.cols, k, brs, g.b.kstride[0], db, eb, nullptr);
        } else if (g.tile_count >= 0) {
            std::vector<int> pa, pb;
            ozaki_tile_panels(p, &pa, &pb);
            if (same) {
                std::vector<int> u(pa);
                u.insert(u.end(), pb.begin(), pb.end());
                std::sort(u.begin(), u.end());
                u.erase(std::unique(u.begin(), u.end()), u.end());
                split(xa, g.rows, k, ars, g.a.kstride[0], da, ea, &u);
            } else {
                split(xa, g.rows, k, ars, g.a.kstride[0], da, ea, &pa);
                split(xb, g.cols, k, brs, g.b.kstride[0], db, eb, &pb);
            }
        } else {
            split(xa, g.rows, k, ars, g.a.kstride[0], da, ea, nullptr);
            if (!same) split(xb, g.cols, k, brs, g.b.kstride[0], db, eb, nullptr);
        }
        const int l = launch_ozaki_gemm(p, s);
        if (l < 0) fail(ErrorCode::CudaError, "executor: emulated GEMM launch failed");
        check_cuda(cudaPeekAtLastError(), "emulated GEMM launch");
        launched += l;
    }
    if (stats_) {
        const std::uint64_t tile = 128ull * 128ull * static_cast<std::uint64_t>((g.n + 63) / 64 * 64);
        const std::uint64_t products = static_cast<std::uint64_t>(S * (S + 1) / 2);
        stats_->int8_ops += 2 * static_cast<std::uint64_t>(tiles) * tile * products;
        const std::uint64_t full = static_cast<std::uint64_t>(g.rows) * static_cast<std::uint64_t>(g.cols) *
                                   static_cast<std::uint64_t>(g.n);
        const std::uint64_t tm = static_cast<std::uint64_t>((g.rows + 127) / 128);
        stats_->emulated_macs += sym ? full / (tm * tm) * (tm * (tm + 1) / 2) : full;  // as gemm_macs counts it
        stats_->oz_slices = static_cast<std::uint64_t>(S);
    }
    // keep or release each side's digits: a later GEMM reading the same
    // operand reuses them while the schedule's headroom covers them
    auto settle = [&](const std::string& key, CachedDigits* hit, int8_t* d, int* e, std::size_t bytes, long long rows) {
        if (hit) {
            if (--hit->uses <= 0) {
                rt_->raw_free(hit->d, hit->bytes);
                rt_->release(reinterpret_cast<double*>(hit->e));
                digits_.erase(key);
            }
            return;
        }
        auto u = digit_uses_.find(key);
        double held = 0;
        for (const auto& [k2, c] : digits_) held += static_cast<double>(c.bytes);
        const bool keep = reuse && u != digit_uses_.end() && u->second > 1 &&
                          budget_ - sched_peak_ >= 2.0 * (held + static_cast<double>(bytes)) + 2e9;
        if (keep) {
            digits_[key] = CachedDigits{d, e, bytes, rows, u->second - 1};
            return;
        }
        rt_->raw_free(d, bytes);
        rt_->release(reinterpret_cast<double*>(e));
    };
    settle(key_a_, ca, da, ea, oz.a_bytes, g.rows);
    if (!same) settle(key_b_, cb, db, eb, oz.b_bytes, g.cols);
    rt_->release(work);
    return launched;
}

void Program::run_gemm(const Op& op, double* out) {
    std::vector<View> fa = op.fa, fb = op.fb;
    const int e = op.e;
    for (auto* side : {&fa, &fb})
        for (View& v : *side) {
            if (!bufs_[static_cast<std::size_t>(v.buf)].symmetric || std::popcount(v.ids) != 2 || !(v.ids & bit(e)))
                continue;
            if (v.stride[static_cast<std::size_t>(e)] == 1) continue;
            const int other = std::countr_zero(v.ids & ~bit(e));
            std::swap(v.stride[static_cast<std::size_t>(e)], v.stride[static_cast<std::size_t>(other)]);
        }
    auto fill = [&](GemmSide& side, const std::vector<View>& fs, const std::vector<int>& rows) {
        side.nf = static_cast<int>(fs.size());
        side.nr = static_cast<int>(rows.size());
        for (int f = 0; f < side.nf; ++f) {
            const View& v = fs[static_cast<std::size_t>(f)];
            side.ptr[f] = ptr(v.buf);
            side.kstride[f] = v.stride[static_cast<std::size_t>(e)];
            for (int d = 0; d < side.nr; ++d)
                side.rstride[f][d] = v.stride[static_cast<std::size_t>(rows[static_cast<std::size_t>(d)])];
        }
    };
    auto kmajor = [&](const std::vector<View>& fs, const std::vector<int>& rows) {
        const View& big = fs[0];
        if (big.stride[static_cast<std::size_t>(e)] == 1) return 1;
        if (!rows.empty() && big.stride[static_cast<std::size_t>(rows.back())] == 1) return 0;
        return 1;
    };
    key_a_ = operand_key(op.fa, op.ra, op.e);
    key_b_ = operand_key(op.fb, op.rb, op.e);
    cur_long_chunks_ = op.long_chunks && slice_world_ == 1 && block_rows_.first < 0;
    GemmArgs g;
    fill(g.a, fa, op.ra);
    fill(g.b, fb, op.rb);
    g.n = n_;
    g.rows = static_cast<long long>(ipow(n_, static_cast<int>(op.ra.size())));
    g.cols = static_cast<long long>(ipow(n_, static_cast<int>(op.rb.size())));
    g.a_kmajor = kmajor(fa, op.ra);
    g.b_kmajor = kmajor(fb, op.rb);
    g.symmetric_out = op.symmetric_out ? 1 : 0;
    g.mode = kEpiStore;
    g.out = out;
    int launched = -1;
    double* scratch = nullptr;
    // Row sharding (shard.cpp): this rank's row panel [lo, hi) of the row id
    // over every column, or one block of a symmetric product (run_tri_gemm,
    // `out` is then the block's own rows x cols buffer). Operand pointers are
    // offset, so every engine sees a smaller plain GEMM.
    long long row_off = 0;  // first row of the panel (flattened rows: times n^(|ra| - 1))
    if (block_rows_.first >= 0) {
        for (int f = 0; f < g.a.nf; ++f) g.a.ptr[f] += block_rows_.first * g.a.rstride[f][0];
        for (int f = 0; f < g.b.nf; ++f) g.b.ptr[f] += block_cols_.first * g.b.rstride[f][0];
        g.rows = block_rows_.second - block_rows_.first;
        g.cols = block_cols_.second - block_cols_.first;
    } else if (slice_world_ > 1) {
        const long long lo = row_lo(slice_rank_), hi = row_lo(slice_rank_ + 1);
        if (hi <= lo) return;
        const long long inner = static_cast<long long>(ipow(n_, static_cast<int>(op.ra.size()) - 1));
        for (int f = 0; f < g.a.nf; ++f) g.a.ptr[f] += lo * g.a.rstride[f][0];
        row_off = lo * inner;
        g.rows = (hi - lo) * inner;
        if (g.out) g.out += row_off * g.cols;
        out = g.out;
        g.symmetric_out = 0;
        g.accumulate = 1;
    }
    const bool multi_path = !op.epis.empty() || (g.symmetric_out && gemm_tma_eligible(g, nullptr, nullptr));
    if (multi_path) {
        EpiSet set;
        std::size_t part_total = 0;
        if (op.store) {
            EpiDesc& d = set.d[set.count++];
            d.mode = kEpiStore;
            d.out = out;
        }
        if (op.epis.size() + (op.store ? 1 : 0) > static_cast<std::size_t>(kMaxEpilogues))
            fail(ErrorCode::InvalidArgument, "executor: too many fused epilogues");
        for (const Op::Epi& e : op.epis) {
            EpiDesc& d = set.d[set.count++];
            d.mode = e.mode;
            d.self_power = e.self_power;
            d.transpose = e.transpose ? 1 : 0;
            d.nw = static_cast<int>(e.w.size());
            for (int f = 0; f < d.nw; ++f) {
                const View& v = e.w[static_cast<std::size_t>(f)];
                d.wptr[f] = ptr(v.buf);
                d.wr[f] = v.stride[static_cast<std::size_t>(e.row_id)];
                d.wc[f] = v.stride[static_cast<std::size_t>(e.col_id)];
                d.wptr[f] += row_off * d.wr[f];  // a row panel reads its rows of the weights
                // a symmetric matrix reads the same transposed: make the column stride unit
                if (bufs_[static_cast<std::size_t>(v.buf)].symmetric && d.wr[f] == 1 && d.wc[f] == n_) {
                    d.wr[f] = n_;
                    d.wc[f] = 1;
                }
            }
            // weights with a unit row stride go first so the kernel picks row-fastest order
            // only when no weight prefers columns
            for (int f = 1; f < d.nw; ++f)
                if (d.wc[f] == 1 && d.wc[0] != 1) {
                    std::swap(d.wptr[0], d.wptr[f]);
                    std::swap(d.wr[0], d.wr[f]);
                    std::swap(d.wc[0], d.wc[f]);
                }
            if (e.ext) {
                d.out = e.ext;
            } else {
                SymBuf& b = bufs_[static_cast<std::size_t>(e.out)];
                if (!b.real) {
                    b.real = rt_->allocate(b.order, n_);
                    if (slice_world_ > 1)
                        check_cuda(cudaMemsetAsync(b.real->ptr, 0, b.real->entries() * sizeof(double), rt_->stream()),
                                   "memset");
                }
                d.out = b.real->ptr;
            }
            // a row panel's row-indexed outputs start at its first row
            if (d.mode == kEpiSumCols || (d.mode == kEpiStore && !d.transpose)) d.out += row_off * (d.mode == kEpiStore ? g.cols : 1);
            part_total += gemm_epi_partial_entries(g, d.mode);
        }
        scratch = part_total ? rt_->scratch(part_total) : nullptr;
        if (scratch && slice_world_ > 1)  // tiles of other ranks leave their partial slots at zero
            check_cuda(cudaMemsetAsync(scratch, 0, part_total * sizeof(double), rt_->stream()), "memset");
        std::size_t at = 0;
        for (int q = 0; q < set.count; ++q) {
            set.d[q].partial = scratch + at;
            at += gemm_epi_partial_entries(g, set.d[q].mode);
        }
        // A symmetric product of an input still being uploaded in row panels:
        // launch the column-ordered tile triangle in pieces, each as soon as
        // the panels it reads have landed (upload/compute overlap).
        const DeviceBuffer* src = bufs_[static_cast<std::size_t>(fa[0].buf)].real.get();
        const bool chunked = slice_world_ == 1 && block_rows_.first < 0 && g.symmetric_out && g.rows == g.cols &&
                             fa[0].buf == fb[0].buf && src && src->ready.size() > 1;
        rt_->begin(Runtime::kGemm);
        if (emulated_eligible(g)) {
            // the emulated GEMM digitizes whole operands: an input still arriving
            // in panels is waited for (its upload then overlaps only the split)
            if (chunked) check_cuda(cudaStreamWaitEvent(rt_->stream(), src->ready.back().second, 0), "wait upload");
            launched = run_emulated(g, set);
            if (launched < 0) launched = launch_gemm_multi(g, set, rt_->stream());
        } else if (!chunked) {
            launched = launch_gemm_multi(g, set, rt_->stream());
        } else {
            // Pieces run concurrently on the chunk streams (a piece smaller than
            // one wave must not serialize the next); reductions land in
            // per-piece slots combined in piece order afterwards; stores are
            // disjoint tiles accumulated into the zeroed output.
            cudaStream_t main = rt_->stream();
            for (int q = 0; q < set.count; ++q)
                if (set.d[q].mode == kEpiStore)
                    check_cuda(cudaMemsetAsync(set.d[q].out, 0, static_cast<std::size_t>(g.rows * g.cols) * sizeof(double),
                                               main),
                               "memset");
            const long long tiles_n = (g.rows + 127) / 128;
            std::vector<std::pair<long long, cudaEvent_t>> pieces;
            long long prev = 0;
            for (const auto& [rows_ready, ev] : src->ready) {
                const long long k = rows_ready >= g.rows ? tiles_n : rows_ready / 128;
                if (k > prev) {
                    pieces.emplace_back(k, ev);
                    prev = k;
                }
            }
            const int C = static_cast<int>(pieces.size());
            auto out_len = [&](int mode) -> long long {
                return mode == kEpiSumAll ? 1 : mode == kEpiSumCols ? g.rows : mode == kEpiSumRows ? g.cols : 0;
            };
            // slots of epilogue q: [q][piece][len_q]
            std::vector<std::size_t> base(static_cast<std::size_t>(set.count) + 1, 0);
            for (int q = 0; q < set.count; ++q)
                base[static_cast<std::size_t>(q) + 1] =
                    base[static_cast<std::size_t>(q)] + static_cast<std::size_t>(out_len(set.d[q].mode)) * C;
            const std::size_t slot_total = base.back();
            double* slots = slot_total ? rt_->scratch(slot_total) : nullptr;
            double* parts = part_total ? rt_->scratch(part_total * static_cast<std::size_t>(C)) : nullptr;
            if (slots) check_cuda(cudaMemsetAsync(slots, 0, slot_total * sizeof(double), main), "memset");
            if (parts) check_cuda(cudaMemsetAsync(parts, 0, part_total * C * sizeof(double), main), "memset");
            cudaEvent_t start;
            check_cuda(cudaEventCreateWithFlags(&start, cudaEventDisableTiming), "event");
            check_cuda(cudaEventRecord(start, main), "event");
            std::vector<cudaEvent_t> finished;
            long long lo = 0;
            launched = 0;
            for (int c = 0; c < C; ++c) {
                cudaStream_t cs = rt_->chunk_stream(c);
                check_cuda(cudaStreamWaitEvent(cs, start, 0), "wait");
                check_cuda(cudaStreamWaitEvent(cs, pieces[static_cast<std::size_t>(c)].second, 0), "wait panel");
                EpiSet piece = set;
                std::size_t po = 0;
                for (int q = 0; q < piece.count; ++q) {
                    EpiDesc& d = piece.d[q];
                    const long long len = out_len(d.mode);
                    if (len > 0) d.out = slots + base[static_cast<std::size_t>(q)] + static_cast<std::size_t>(c * len);
                    d.partial = parts ? parts + static_cast<std::size_t>(c) * part_total + po : nullptr;
                    po += gemm_epi_partial_entries(g, d.mode);
                }
                const long long k = pieces[static_cast<std::size_t>(c)].first;
                GemmArgs gc = g;
                gc.tri_colmajor = 1;
                gc.tile_begin = lo * (lo + 1) / 2;
                gc.tile_count = k * (k + 1) / 2 - gc.tile_begin;
                gc.accumulate = 1;  // stores: disjoint tiles into the zeroed output; slots are zeroed
                const int l = launch_gemm_multi(gc, piece, cs);
                if (l < 0) {
                    launched = -1;
                    break;
                }
                launched += l;
                cudaEvent_t done;
                check_cuda(cudaEventCreateWithFlags(&done, cudaEventDisableTiming), "event");
                check_cuda(cudaEventRecord(done, cs), "event");
                finished.push_back(done);
                lo = k;
            }
            for (cudaEvent_t e : finished) {
                check_cuda(cudaStreamWaitEvent(main, e, 0), "wait piece");
                cudaEventDestroy(e);
            }
            cudaEventDestroy(start);
            for (int q = 0; q < set.count && launched >= 0; ++q) {
                const long long len = out_len(set.d[q].mode);
                if (len > 0)
                    launched += launch_sum_slices(slots + base[static_cast<std::size_t>(q)], C, len, set.d[q].out, 0, main);
            }
            rt_->release(slots);
            rt_->release(parts);
        }
        rt_->end(Runtime::kGemm);
        if (launched < 0) fail(ErrorCode::InvalidArgument, "executor: fused GEMM lost TMA eligibility");
    } else if (emulated_eligible(g)) {  // a plain product (e.g. a Khatri-Rao GEMM) on the INT8 tensor cores
        EpiSet set;
        set.count = 1;
        set.d[0].mode = kEpiStore;
        set.d[0].out = out;
        g.symmetric_out = 0;
        rt_->begin(Runtime::kGemm);
        launched = run_emulated(g, set);
        if (launched < 0) launched = launch_gemm(g, rt_->stream());
        rt_->end(Runtime::kGemm);
    } else {
        g.symmetric_out = 0;
        rt_->begin(Runtime::kGemm);
        launched = launch_gemm(g, rt_->stream());
        rt_->end(Runtime::kGemm);
    }
    check_cuda(cudaGetLastError(), "gemm launch");
    rt_->release(scratch);
    if (stats_) {
        const bool tri = g.symmetric_out && g.rows == g.cols && gemm_tma_eligible(g, nullptr, nullptr);
        const long long tm = (g.rows + 127) / 128;
        const std::uint64_t full = static_cast<std::uint64_t>(g.rows) * static_cast<std::uint64_t>(g.cols) *
                                   static_cast<std::uint64_t>(n_);
        const std::uint64_t macs = tri ? full / static_cast<std::uint64_t>(tm * tm) *
                                             static_cast<std::uint64_t>(tm * (tm + 1) / 2)
                                       : full;
        stats_->gemm_macs += macs;
        ++stats_->gemm_launches;
        stats_->kernel_launches += static_cast<std::uint64_t>(launched);
        if (tri) ++stats_->symmetric_gemms;
    }
}

void Program::launch(Op& op) {
    if (op.sweep) {
        run_sweep(op);
        return;
    }
    double* out = op.ext;
    if (!out && (!op.gemm || op.store)) {
        SymBuf& b = bufs_[static_cast<std::size_t>(op.out)];
        if (!b.real) {
            b.real = rt_->allocate(b.order, n_);
            if (slice_world_ > 1)
                check_cuda(cudaMemsetAsync(b.real->ptr, 0, b.real->entries() * sizeof(double), rt_->stream()), "memset");
        }
        b.real->symmetric = b.symmetric;
        out = b.real->ptr;
    }
    if (op.gemm && step_ && step_->tri && slice_world_ > 1) run_tri_gemm(op, out, shard_emulate_);
    else if (op.gemm) run_gemm(op, out);
    else run_stream(op, out);
}

// Launches the schedule. GEMMs and ops that allocate order>=2 tensors stay
// on the main stream in schedule order (the memory bound assumes that);
// reductions to vectors / scalars go to a side stream so they fill the SMs a
// GEMM's last wave leaves idle. Cross-stream reads wait on the producer's
// event; a buffer is freed on the stream of its last reader after the other
// stream's readers are done.
void Program::execute() {
    const DeviceConfig& dc = config_.device;
    const int emulate = dc.shard_rows && dc.emulate_world > 1 ? dc.emulate_world : 0;
    const int world = emulate ? emulate : (dc.shard_rows ? std::max(1, dc.world_size) : 1);
    if (world > 1) {
        if (!emulate && !rt_->has_comm()) fail(ErrorCode::CollectiveError, "row sharding needs us_nccl_init first");
        execute_sharded(world, emulate != 0);
        return;
    }
    plan_digit_reuse();
    struct DropDigits {  // cached digits never outlive one execution
        Program* p;
        ~DropDigits() { p->drop_digits(); }
    } drop_guard{this};
    bool has_gemm = false;
    for (std::size_t i : schedule_) has_gemm |= ops_[i].gemm;
    const bool multi =
        has_gemm && !config_.device.serial_launch && (budget_ <= 0 || sched_peak_ <= 0.7 * budget_);
    // only reductions over at most an n^2 space go to the side stream: heavier
    // bandwidth ops running under a GEMM steal its SMs mid-wave (C4: -3%)
    auto side_ok = [&](const Op& op) {
        if (op.sweep) {
            for (const Op::Epi& e : op.epis)
                if (e.mode == kEpiStore) return false;
            return true;
        }
        if (op.gemm || (!op.ext && bufs_[static_cast<std::size_t>(op.out)].order >= 2)) return false;
        const int dims = static_cast<int>(op.out_ids.size()) + std::popcount(op.sum);
        return dims <= 2;
    };
    cudaStream_t streams[2] = {rt_->main_stream(), multi ? rt_->side_stream() : rt_->main_stream()};
    const std::size_t N = ops_.size();
    if (multi && !launch_ordered_) {
        launch_ordered_ = true;  // a cached program re-executes in the same order
        // Side-stream reductions are launched right after the next GEMM, so the
        // GEMM takes the whole GPU first and they fill its last wave; a main-
        // stream op that reads a deferred op's output flushes the queue first.
        std::vector<std::size_t> order, deferred;
        std::vector<char> pending_out(bufs_.size(), 0);
        auto flush = [&] {
            for (std::size_t d : deferred) {
                order.push_back(d);
                const Op& o = ops_[d];
                if (!o.ext && o.out >= 0) pending_out[static_cast<std::size_t>(o.out)] = 0;
                for (const Op::Epi& e : o.epis)
                    if (!e.ext && e.out >= 0) pending_out[static_cast<std::size_t>(e.out)] = 0;
            }
            deferred.clear();
        };
        for (std::size_t i : schedule_) {
            const Op& op = ops_[i];
            if (side_ok(op)) {
                deferred.push_back(i);
                if (!op.ext && op.out >= 0) pending_out[static_cast<std::size_t>(op.out)] = 1;
                for (const Op::Epi& e : op.epis)
                    if (!e.ext && e.out >= 0) pending_out[static_cast<std::size_t>(e.out)] = 1;
                continue;
            }
            bool needs = false;
            for_each_read(op, [&](const View& v) { needs |= pending_out[static_cast<std::size_t>(v.buf)] != 0; });
            if (needs) flush();
            order.push_back(i);
            if (op.gemm) flush();
        }
        flush();
        schedule_ = order;
        for (SymBuf& b : bufs_) b.last_use = -1;
        for (std::size_t pos = 0; pos < schedule_.size(); ++pos)
            for_each_read(ops_[schedule_[pos]],
                          [&](const View& v) { bufs_[static_cast<std::size_t>(v.buf)].last_use = static_cast<int>(pos); });
    }
    if (multi) {
        // inputs were prepared (uploaded, sparsified, probed) on the main
        // stream: the side stream starts behind that work
        cudaEvent_t inputs_ready;
        check_cuda(cudaEventCreateWithFlags(&inputs_ready, cudaEventDisableTiming), "event");
        check_cuda(cudaEventRecord(inputs_ready, rt_->main_stream()), "event");
        check_cuda(cudaStreamWaitEvent(rt_->side_stream(), inputs_ready, 0), "wait");
        cudaEventDestroy(inputs_ready);
    }
    std::vector<cudaEvent_t> done(N, nullptr);
    std::vector<int> on(N, 0), producer(bufs_.size(), -1);
    std::vector<std::array<int, 2>> readers(bufs_.size(), {-1, -1});
    std::vector<std::pair<int, int>> upload_waited;
    for (std::size_t pos = 0; pos < schedule_.size(); ++pos) {
        const std::size_t i = schedule_[pos];
        Op& op = ops_[i];
        const int si = (multi && side_ok(op)) ? 1 : 0;
        on[i] = si;
        cudaStream_t s = streams[si];
        if (multi)
            for_each_read(op, [&](const View& v) {
                const int p = producer[static_cast<std::size_t>(v.buf)];
                if (p >= 0 && on[static_cast<std::size_t>(p)] != si) check_cuda(cudaStreamWaitEvent(s, done[static_cast<std::size_t>(p)], 0), "wait");
            });
        // inputs still uploading in panels: every reader except the panel-aware
        // symmetric GEMM waits for the whole upload (once per stream)
        for_each_read(op, [&](const View& v) {
            const SymBuf& b = bufs_[static_cast<std::size_t>(v.buf)];
            if (!b.input || !b.real || b.real->ready.empty()) return;
            const bool panel_aware = op.gemm && op.symmetric_out && op.fa.size() == 1 && op.fb.size() == 1 &&
                                     op.fa[0].buf == op.fb[0].buf && (!op.epis.empty() || op.symmetric_out);
            if (panel_aware) return;
            const auto key = std::make_pair(v.buf, si);
            if (std::find(upload_waited.begin(), upload_waited.end(), key) != upload_waited.end()) return;
            upload_waited.push_back(key);
            check_cuda(cudaStreamWaitEvent(s, b.real->ready.back().second, 0), "wait upload");
        });
        rt_->set_stream(s);
        launch(op);
        if (!op.ext && op.out >= 0) producer[static_cast<std::size_t>(op.out)] = static_cast<int>(i);
        for (const Op::Epi& e : op.epis)
            if (!e.ext && e.out >= 0) producer[static_cast<std::size_t>(e.out)] = static_cast<int>(i);
        if (multi) {
            check_cuda(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming), "cudaEventCreate");
            check_cuda(cudaEventRecord(done[i], s), "cudaEventRecord");
        }
        for_each_read(op, [&](const View& v) { readers[static_cast<std::size_t>(v.buf)][si] = static_cast<int>(i); });
        for_each_read(op, [&](const View& v) {
            SymBuf& b = bufs_[static_cast<std::size_t>(v.buf)];
            if (b.input || b.last_use != static_cast<int>(pos) || !b.real || b.real.use_count() != 1 || keep_.count(v.buf))
                return;
            const int other = readers[static_cast<std::size_t>(v.buf)][1 - si];
            if (multi && other >= 0) check_cuda(cudaStreamWaitEvent(s, done[static_cast<std::size_t>(other)], 0), "wait");
            b.real.reset();
        });
    }
    if (multi) {
        cudaEvent_t side_done;
        check_cuda(cudaEventCreateWithFlags(&side_done, cudaEventDisableTiming), "cudaEventCreate");
        check_cuda(cudaEventRecord(side_done, streams[1]), "cudaEventRecord");
        check_cuda(cudaStreamWaitEvent(streams[0], side_done, 0), "wait");
        cudaEventDestroy(side_done);
        for (cudaEvent_t e : done)
            if (e) cudaEventDestroy(e);
    }
    rt_->set_stream(streams[0]);
}

Buf Program::take(int buf) { return bufs_[static_cast<std::size_t>(buf)].real; }

std::vector<Buf> Program::inputs() const {
    std::vector<Buf> out;
    for (const SymBuf& b : bufs_)
        if (b.input) out.push_back(b.real);
    return out;
}

void Program::rebind_inputs(const std::vector<Buf>& reals) {
    std::size_t k = 0;
    for (SymBuf& b : bufs_) {
        if (!b.input) continue;
        if (k >= reals.size()) fail(ErrorCode::InvalidArgument, "executor: cached plan input count mismatch");
        b.real = reals[k++];
    }
    if (k != reals.size()) fail(ErrorCode::InvalidArgument, "executor: cached plan input count mismatch");
}

void Program::release_buffers() {
    for (SymBuf& b : bufs_) b.real.reset();
}

}  // namespace ustats::dev
