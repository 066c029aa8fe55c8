// Program recording and optimization (executor.hpp): content-addressed
// ops, symmetry tracking, epilogue and sweep fusion, memory-bounded schedule.
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

// ----------------------------------------------------------------- Program
int Program::add_input(const Buf& real) {
    for (std::size_t i = 0; i < bufs_.size(); ++i)
        if (bufs_[i].input && bufs_[i].real == real) return static_cast<int>(i);
    SymBuf b;
    b.order = real->order;
    b.symmetric = real->symmetric;
    b.input = true;
    b.real = real;
    b.content = static_cast<int>(bufs_.size());
    bufs_.push_back(b);
    return b.content;
}

int Program::add_symbolic_input(int order, bool symmetric) {
    SymBuf b;
    b.order = order;
    b.symmetric = symmetric && order == 2;
    b.input = true;
    b.content = static_cast<int>(bufs_.size());
    bufs_.push_back(b);
    return b.content;
}

Program::Totals Program::totals() const {
    Totals t;
    t.peak_entries = static_cast<std::uint64_t>(sched_peak_ / 8.0);
    for (const Op& op : ops_) {
        if (op.dead) continue;
        if (op.gemm) {
            ++t.gemms;
            const std::uint64_t tm = (ipow(n_, static_cast<int>(op.ra.size())) + 127) / 128;
            std::uint64_t macs = ipow(n_, static_cast<int>(op.ra.size() + op.rb.size()) + 1);
            const bool tri = op.symmetric_out && op.ra.size() == 1 && op.rb.size() == 1;
            if (tri) {
                macs = macs / (tm * tm) * (tm * (tm + 1) / 2);
                ++t.symmetric;
            }
            t.gemm_macs += macs;
            t.fused += op.epis.size();
        } else if (op.sweep) {
            ++t.streams;
            t.stream_entries += ipow(n_, 2);
            t.fused += op.epis.size();
        } else {
            ++t.streams;
            t.stream_entries += ipow(n_, static_cast<int>(op.out_ids.size()) + std::popcount(op.sum)) *
                                static_cast<std::uint64_t>(op.factors.size());
        }
    }
    return t;
}

std::string Program::dump() const {
    static const char* modes[] = {"store", "sum_all", "sum_cols", "sum_rows"};
    std::string out;
    auto vs = [&](const std::vector<View>& v) {
        std::string s;
        for (const View& x : v) {
            s += " b" + std::to_string(x.buf) + "{";
            for (int id : ids_of(x.ids)) s += std::to_string(id) + ":" + std::to_string(x.stride[static_cast<std::size_t>(id)]) + " ";
            s += "}";
        }
        return s;
    };
    for (std::size_t i = 0; i < ops_.size(); ++i) {
        const Op& op = ops_[i];
        if (op.dead) continue;
        std::string line = std::to_string(i) + ": ";
        if (op.gemm) {
            line += "GEMM rows=" + std::to_string(op.ra.size()) + " cols=" + std::to_string(op.rb.size()) + " e=" +
                    std::to_string(op.e) + " A:" + vs(op.fa) + " B:" + vs(op.fb) + (op.symmetric_out ? " SYM" : "") +
                    (op.store ? " store" : " nostore");
            for (const Op::Epi& e : op.epis)
                line += std::string(" | epi ") + modes[e.mode] + " pow=" + std::to_string(e.self_power) +
                        (e.w.empty() ? "" : " W:" + vs(e.w)) + (e.ext ? " -> term" : " -> b" + std::to_string(e.out));
        } else if (op.sweep) {
            line += "SWEEP X:" + vs(op.factors);
            for (const Op::Epi& e : op.epis)
                line += std::string(" | ") + modes[e.mode] + " pow=" + std::to_string(e.self_power) +
                        (e.w.empty() ? "" : " W:" + vs(e.w)) + (e.ext ? " -> term" : " -> b" + std::to_string(e.out));
            out += line + "\n";
            continue;
        } else {
            line += "STREAM out=[";
            for (int id : op.out_ids) line += std::to_string(id) + " ";
            line += "] sum=[";
            for (int id : ids_of(op.sum)) line += std::to_string(id) + " ";
            line += "]" + vs(op.factors);
        }
        line += op.ext ? " -> term" : " -> b" + std::to_string(op.out);
        out += line + "\n";
    }
    return out;
}

int Program::new_buf(int order, bool symmetric) {
    SymBuf b;
    b.order = order;
    b.symmetric = symmetric;
    b.content = static_cast<int>(bufs_.size());
    bufs_.push_back(b);
    return b.content;
}

View Program::view_of(int buf, const IndexTuple& layout) const {
    View v;
    v.buf = buf;
    long long s = 1;
    for (std::size_t p = layout.size(); p-- > 0;) {
        if (layout[p] < 0 || layout[p] >= kMaxIds)
            fail(ErrorCode::InvalidArgument, "too many indices for the device executor");
        v.stride[static_cast<std::size_t>(layout[p])] += s;
        v.ids |= bit(layout[p]);
        s *= n_;
    }
    return v;
}

// Canonical descriptor of a factor over an ordered list of local dims:
// content id + stride per dim. A symmetric matrix reads the same either way,
// so both orientations map to one descriptor.
std::string Program::desc(const View& v, const std::vector<int>& dims) const {
    std::vector<long long> s;
    for (int d : dims) s.push_back(v.stride[static_cast<std::size_t>(d)]);
    const SymBuf& b = bufs_[static_cast<std::size_t>(v.buf)];
    if (b.symmetric && std::popcount(v.ids) == 2) {
        std::vector<long long> t = s;
        for (long long& x : t) x = x == 1 ? n_ : (x == n_ ? 1 : x);
        if (n_ > 1 && t > s) s = t;
    }
    std::string out = "b" + std::to_string(b.content) + "[";
    for (long long x : s) out += std::to_string(x) + ",";
    return out + "]";
}

// Canonical content key of a stream op: factor descriptors over (out dims,
// summed dims), minimised over the order of the summed dims.
std::string Program::stream_key(const std::vector<View>& factors, const std::vector<int>& out_ids,
                                std::uint32_t sum) const {
    std::vector<int> sums = ids_of(sum);
    std::sort(sums.begin(), sums.end());
    std::string best;
    do {
        std::vector<int> dims = out_ids;
        dims.insert(dims.end(), sums.begin(), sums.end());
        std::vector<std::string> ds;
        for (const View& v : factors) ds.push_back(desc(v, dims));
        std::sort(ds.begin(), ds.end());
        std::string k = "S" + std::to_string(out_ids.size()) + ":";
        for (auto& d : ds) k += d;
        if (best.empty() || k < best) best = k;
    } while (std::next_permutation(sums.begin(), sums.end()));
    return best;
}

// A full-matrix view of a symmetric matrix that is a known power B^p of a
// symmetric base (a symmetric input is its own base, p = 1).
bool Program::power_of(const View& v, int* base, int* pw) const {
    const SymBuf& b = bufs_[static_cast<std::size_t>(v.buf)];
    if (b.order != 2 || !b.symmetric || std::popcount(v.ids) != 2) return false;
    const int i = std::countr_zero(v.ids), j = 31 - std::countl_zero(v.ids);
    const long long si = v.stride[static_cast<std::size_t>(i)], sj = v.stride[static_cast<std::size_t>(j)];
    if (!((si == 1 && sj == n_) || (si == n_ && sj == 1))) return false;
    *base = b.power_base >= 0 ? b.power_base : b.content;
    *pw = b.power_base >= 0 ? b.power : 1;
    return true;
}

int Program::lookup_stream(const std::vector<View>& factors, const std::vector<int>& out_ids,
                           std::uint32_t sum) const {
    if (!sharing() || factors.size() > static_cast<std::size_t>(kMaxFactors)) return -1;
    if (static_cast<int>(out_ids.size()) + std::popcount(sum) > kMaxDims) return -1;
    auto hit = memo_.find(stream_key(factors, out_ids, sum));
    return hit == memo_.end() ? -1 : hit->second;
}

int Program::stream(std::vector<View> factors, const std::vector<int>& out_ids, std::uint32_t sum, double* ext) {
    // keep within the kernel's factor budget: form the product of the leading
    // factors over their own ids first
    while (factors.size() > static_cast<std::size_t>(kMaxFactors)) {
        std::vector<View> head(factors.begin(), factors.begin() + kMaxFactors);
        std::vector<int> layout = ids_of(ids_of_views(head));
        int b = stream(head, layout, 0, nullptr);
        factors.erase(factors.begin(), factors.begin() + kMaxFactors);
        factors.insert(factors.begin(), view_of(b, layout));
    }
    if (static_cast<int>(out_ids.size()) + std::popcount(sum) > kMaxDims)
        fail(ErrorCode::InvalidArgument, "contraction step spans too many indices for the stream kernel");
    std::string key;
    if (sharing()) {
        key = stream_key(factors, out_ids, sum);
        if (ext) {
            key = "X" + key;
            auto hit = term_memo_.find(key);
            if (hit != term_memo_.end()) {
                if (stats_) ++stats_->shared_hits;
                aliases_.emplace_back(ext, hit->second);
                return -1;
            }
        } else {
            auto hit = memo_.find(key);
            if (hit != memo_.end()) {
                if (stats_) ++stats_->shared_hits;
                return hit->second;
            }
        }
    }
    // B^p scaled along one axis by a vector: remember it (see SymBuf)
    int sc_base = -1, sc_pow = 0, sc_w = -1, sc_axis = -1;
    if (!ext && sum == 0 && out_ids.size() == 2 && factors.size() >= 2) {
        // one matrix factor B^p and vectors that all run along one output index
        int mats = 0, b = -1, p = 0, wid = -1;
        bool ok = true;
        for (const View& v : factors) {
            int vb = -1, vp = 0;
            if (power_of(v, &vb, &vp)) {
                ++mats;
                b = vb;
                p = vp;
            } else if (bufs_[static_cast<std::size_t>(v.buf)].order == 1 && std::popcount(v.ids) == 1 &&
                       (wid < 0 || wid == std::countr_zero(v.ids))) {
                wid = std::countr_zero(v.ids);
            } else {
                ok = false;
            }
        }
        const auto pos = wid >= 0 ? std::find(out_ids.begin(), out_ids.end(), wid) - out_ids.begin() : 2;
        if (ok && mats == 1 && pos <= 1) {
            sc_base = b;
            sc_pow = p;
            sc_w = wid;
            sc_axis = static_cast<int>(pos);
        }
    }
    Op op;
    op.factors = std::move(factors);
    op.out_ids = out_ids;
    op.sum = sum;
    op.ext = ext;
    if (!ext) {
        op.out = new_buf(static_cast<int>(out_ids.size()), false);
        SymBuf& ob = bufs_[static_cast<std::size_t>(op.out)];
        ob.scaled_base = sc_base;
        ob.scaled_power = sc_pow;
        ob.scaled_w = sc_w;
        ob.scaled_axis = sc_axis;
    }
    ops_.push_back(op);
    if (!key.empty()) {
        if (ext) term_memo_[key] = ext;
        else memo_[key] = op.out;
        memo_log_.push_back(key);
    }
    return op.out;
}

int Program::gemm(std::vector<View> fa, std::vector<View> fb, const std::vector<int>& ra_in,
                  const std::vector<int>& rb_in, int e, std::vector<int>* layout) {
    std::vector<int> ra = ra_in, rb = rb_in;
    // A diagonal weight (factors over the contracted index alone) can sit on
    // either operand; put it on a canonical side so that X D Y and (Y D X)^T
    // lower to the same operands and share one GEMM (C5: B D (B o B) and
    // (B o B) D B).
    {
        std::vector<View> diag, ka0, kb0;
        for (const View& v : fa) (v.ids == bit(e) ? diag : ka0).push_back(v);
        for (const View& v : fb) (v.ids == bit(e) ? diag : kb0).push_back(v);
        if (!diag.empty() && !ka0.empty() && !kb0.empty()) {
            auto side_key = [&](const std::vector<View>& fs, const std::vector<int>& rows) {
                std::vector<int> d = rows;
                d.push_back(e);
                std::vector<std::string> ks;
                for (const View& v : fs) ks.push_back(desc(v, d));
                std::sort(ks.begin(), ks.end());
                std::string k;
                for (const auto& x : ks) k += x + ";";
                return k;
            };
            const bool to_b = side_key(kb0, rb) > side_key(ka0, ra);
            (to_b ? kb0 : ka0).insert((to_b ? kb0 : ka0).end(), diag.begin(), diag.end());
            fa = std::move(ka0);
            fb = std::move(kb0);
        }
    }
    // Multi-factor (Hadamard / scaled / Khatri-Rao) operands are formed once,
    // k-major (rows..., e): O(rows*n) traffic against O(rows*cols*n) DMMA work.
    auto lower = [&](std::vector<View>& fs, const std::vector<int>& rows) {
        if (fs.size() <= 1) return;
        std::vector<int> lay = rows;
        lay.push_back(e);
        int b = stream(fs, lay, 0, nullptr);
        fs = {view_of(b, lay)};
    };
    lower(fa, ra);
    lower(fb, rb);
    std::vector<int> da = ra, db = rb;
    da.push_back(e);
    db.push_back(e);
    std::string ka = desc(fa[0], da), kb = desc(fb[0], db);
    if (kb < ka) {
        std::swap(fa, fb);
        std::swap(ra, rb);
        std::swap(ka, kb);
    }
    *layout = ra;
    layout->insert(layout->end(), rb.begin(), rb.end());
    std::string key = "G" + std::to_string(ra.size()) + "." + std::to_string(rb.size()) + ":" + ka + "|" + kb;
    if (sharing()) {
        auto hit = memo_.find(key);
        if (hit != memo_.end()) {
            if (stats_) ++stats_->shared_hits;
            return hit->second;
        }
    }
    bool sym = ka == kb && ra.size() == 1 && rb.size() == 1 && config_.device.exploit_symmetry;
    // B^p * B^q = B^(p+q) for a symmetric B: symmetric although the operands
    // differ (C5: B * B^2), so only its upper tiles are computed
    int out_base = -1, out_power = 0;
    // B^p D_w with w on the contracted index: A * (B^p D_w)^T = B^p D_w B^p
    auto scaled_on_e = [&](const View& v, int* base, int* pw) {
        const SymBuf& b = bufs_[static_cast<std::size_t>(v.buf)];
        if (b.scaled_base < 0 || std::popcount(v.ids) != 2 || !(v.ids & bit(e))) return false;
        if (v.stride[static_cast<std::size_t>(e)] != (b.scaled_axis == 0 ? n_ : 1)) return false;
        *base = b.scaled_base;
        *pw = b.scaled_power;
        return true;
    };
    if (ra.size() == 1 && rb.size() == 1 && fa.size() == 1 && fb.size() == 1 && config_.device.exploit_symmetry) {
        int ba = -1, pa = 0, bb = -1, pb = 0;
        if (power_of(fa[0], &ba, &pa) && power_of(fb[0], &bb, &pb) && ba == bb) {
            sym = true;
            out_base = ba;
            out_power = pa + pb;
        } else if ((power_of(fa[0], &ba, &pa) && scaled_on_e(fb[0], &bb, &pb) && ba == bb && pa == pb) ||
                   (scaled_on_e(fa[0], &ba, &pa) && power_of(fb[0], &bb, &pb) && ba == bb && pa == pb)) {
            sym = true;  // B^p D B^p
        }
    }
    Op op;
    op.gemm = true;
    op.fa = std::move(fa);
    op.fb = std::move(fb);
    op.ra = ra;
    op.rb = rb;
    op.e = e;
    op.symmetric_out = sym;
    op.out = new_buf(static_cast<int>(ra.size() + rb.size()), sym);
    bufs_[static_cast<std::size_t>(op.out)].power_base = out_base;
    bufs_[static_cast<std::size_t>(op.out)].power = out_power;
    ops_.push_back(op);
    if (sharing()) {
        memo_[key] = op.out;
        memo_log_.push_back(key);
    }
    return op.out;
}

void Program::rollback(const Mark& m) {
    for (std::size_t i = m.log; i < memo_log_.size(); ++i) {
        if (memo_log_[i][0] == 'X') term_memo_.erase(memo_log_[i]);
        else memo_.erase(memo_log_[i]);
    }
    memo_log_.resize(m.log);
    aliases_.resize(m.aliases);
    ops_.resize(m.ops);
    bufs_.resize(m.bufs);
}

double Program::cost_since(const Mark& m) const {
    // 1 streamed entry ~ 23 DMMA MACs on B200 (8 B at 6.5 TB/s vs 18.6 TMAC/s)
    double c = 0.0;
    for (std::size_t i = m.ops; i < ops_.size(); ++i) {
        const Op& op = ops_[i];
        if (op.gemm) {
            // a symmetric product computes only its upper tiles
            c += static_cast<double>(ipow(n_, static_cast<int>(op.ra.size() + op.rb.size()) + 1)) *
                 (op.symmetric_out ? 0.5 : 1.0);
        } else {
            const int dims = static_cast<int>(op.out_ids.size()) + std::popcount(op.sum);
            c += 23.0 * static_cast<double>(ipow(n_, dims)) * static_cast<double>(op.factors.size());
        }
    }
    return c;
}

// Host mirror of gemm_tma_eligible for one operand view: a single strided
// matrix with a unit stride along rows or k and an even other stride.
bool Program::tma_plain(const View& v, const std::vector<int>& rows, int e) const {
    if (rows.size() != 1) return false;
    const long long rs = v.stride[static_cast<std::size_t>(rows[0])], ks = v.stride[static_cast<std::size_t>(e)];
    const bool sym = bufs_[static_cast<std::size_t>(v.buf)].symmetric;
    auto ok = [](long long unit, long long other) { return unit == 1 && other > 0 && other % 2 == 0; };
    return ok(ks, rs) || ok(rs, ks) || (sym && (ok(rs, ks) || ok(ks, rs)));
}

// Multi-consumer epilogue fusion. A stream op S that reads the output of a
// GEMM G (once, or twice -> self_power 2), iterates exactly over G's
// (row, col) space, and whose other factors do not depend on G, becomes an
// epilogue of G: Hadamard with its weights, then a fixed-order reduction to a
// scalar / row vector / column vector, or an elementwise store. G keeps
// storing its product only if something else still reads it.
void Program::fuse_epilogues() {
    if (n_ % 2 != 0) return;  // TMA operands need even strides
    const std::size_t N = ops_.size();
    std::vector<int> producer(bufs_.size(), -1);
    for (std::size_t i = 0; i < N; ++i)
        if (!ops_[i].dead && !ops_[i].ext && ops_[i].out >= 0) producer[static_cast<std::size_t>(ops_[i].out)] = static_cast<int>(i);
    const std::size_t words = (N + 63) / 64;
    std::vector<std::uint64_t> deps(N * words, 0);
    auto dep_has = [&](std::size_t i, std::size_t j) { return (deps[i * words + j / 64] >> (j % 64)) & 1; };
    auto closure = [&] {
        std::fill(deps.begin(), deps.end(), 0);
        for (std::size_t i = 0; i < N; ++i) {
            if (ops_[i].dead) continue;
            for_each_read(ops_[i], [&](const View& v) {
                const int p = producer[static_cast<std::size_t>(v.buf)];
                if (p < 0) return;
                const auto pp = static_cast<std::size_t>(p);
                for (std::size_t w = 0; w < words; ++w) deps[i * words + w] |= deps[pp * words + w];
                deps[i * words + pp / 64] |= std::uint64_t{1} << (pp % 64);
            });
        }
    };
    closure();
    for (std::size_t gi = 0; gi < N; ++gi) {
        Op& g = ops_[gi];
        if (g.dead || !g.gemm || g.ra.size() != 1 || g.rb.size() != 1) continue;
        if (g.fa.size() != 1 || g.fb.size() != 1 || !tma_plain(g.fa[0], g.ra, g.e) || !tma_plain(g.fb[0], g.rb, g.e))
            continue;
        const int gb = g.out;
        // one descriptor slot stays free for the plain store of the product
        for (std::size_t si = gi + 1; si < N && g.epis.size() + 1 < static_cast<std::size_t>(kMaxEpilogues); ++si) {
            Op& s = ops_[si];
            if (s.dead || s.gemm) continue;
            std::vector<View> mine, rest;
            for (const View& v : s.factors) (v.buf == gb ? mine : rest).push_back(v);
            if (mine.empty() || mine.size() > 2 || rest.size() > static_cast<std::size_t>(kMaxEpiW)) continue;
            // Epilogue weights are read while the SM's DMMA pipe idles (one CTA
            // per SM): only vector / scalar weights are cheap enough there
            // (measured: matrix weights cost more than the stream pass they save).
            bool light = true;
            for (const View& w : rest) light &= bufs_[static_cast<std::size_t>(w.buf)].order <= 1;
            if (!light) continue;
            int x = -1, y = -1;
            for (int id : ids_of(mine[0].ids)) {
                if (mine[0].stride[static_cast<std::size_t>(id)] == n_) x = id;
                if (mine[0].stride[static_cast<std::size_t>(id)] == 1) y = id;
            }
            if (x < 0 || y < 0 || x == y || std::popcount(mine[0].ids) != 2) continue;
            bool consistent = true;
            for (const View& v : mine) {
                const bool same = v.stride[static_cast<std::size_t>(x)] == n_ && v.stride[static_cast<std::size_t>(y)] == 1;
                const bool flip = v.stride[static_cast<std::size_t>(x)] == 1 && v.stride[static_cast<std::size_t>(y)] == n_;
                if (!(same || (flip && g.symmetric_out)) || std::popcount(v.ids) != 2) consistent = false;
            }
            if (!consistent) continue;
            const std::uint32_t space = bit(x) | bit(y);
            std::uint32_t iter = s.sum;
            for (int id : s.out_ids) iter |= bit(id);
            if (iter != space || (ids_of_views(rest) & ~space)) continue;
            // the weights must exist before G runs and must not depend on G
            bool acyclic = true;
            for (const View& w : rest) {
                const int p = producer[static_cast<std::size_t>(w.buf)];
                if (w.buf == gb || (p >= 0 && (static_cast<std::size_t>(p) == gi || dep_has(static_cast<std::size_t>(p), gi))))
                    acyclic = false;
            }
            if (!acyclic) continue;
            Op::Epi e;
            if (s.out_ids.empty()) e.mode = kEpiSumAll;
            else if (s.out_ids.size() == 1 && s.out_ids[0] == x) e.mode = kEpiSumCols;
            else if (s.out_ids.size() == 1 && s.out_ids[0] == y) e.mode = kEpiSumRows;
            else if (s.out_ids.size() == 2 && s.out_ids[0] == x && s.out_ids[1] == y) e.mode = kEpiStore;
            else if (s.out_ids.size() == 2 && s.out_ids[0] == y && s.out_ids[1] == x) {
                e.mode = kEpiStore;
                e.transpose = true;
            } else continue;
            e.w = rest;
            e.self_power = static_cast<int>(mine.size());
            e.row_id = x;
            e.col_id = y;
            e.out = s.out;
            e.ext = s.ext;
            g.epis.push_back(std::move(e));
            s.dead = true;
            if (!s.ext && s.out >= 0) producer[static_cast<std::size_t>(s.out)] = static_cast<int>(gi);
            if (stats_) ++stats_->fused_epilogues;
            closure();
        }
    }
    // a GEMM stores its product only while something still reads it
    std::vector<int> reads(bufs_.size(), 0);
    for (const Op& op : ops_)
        if (!op.dead) for_each_read(op, [&](const View& v) { ++reads[static_cast<std::size_t>(v.buf)]; });
    for (Op& op : ops_) {
        if (op.dead || !op.gemm) continue;
        op.store = reads[static_cast<std::size_t>(op.out)] > 0 || keep_.count(op.out);
        if (!op.store && op.epis.empty()) op.dead = true;
    }
}

// Sweep fusion. Reductions over a 2-index space that each stream the same
// n x n matrix X and otherwise read only row weights (vectors or scalars
// indexed by X's row) are merged into one pass over X that forms the row
// power sums S_p = sum_C X^p (p <= 4); each reduction becomes a consumer
// scaling S_p by its row weights into a scalar or a row vector (C2: sum A^4
// and the row sums of A^2). X is read row-major (a symmetric X in either
// orientation). Only mutually independent consumers share a sweep.
void Program::fuse_sweeps() {
    struct Cand {
        std::size_t op;
        Op::Epi epi;
    };
    // candidates: live stream ops over two indices reading an order-2 buffer X
    auto candidates = [&] {
        std::map<int, std::vector<Cand>> by_x;
        for (std::size_t i = 0; i < ops_.size(); ++i) {
            const Op& s = ops_[i];
            if (s.dead || s.gemm || s.sweep) continue;
            std::uint32_t space = s.sum;
            for (int id : s.out_ids) space |= bit(id);
            if (std::popcount(space) != 2) continue;
            const int a = std::countr_zero(space), b = 31 - std::countl_zero(space);
            std::map<int, int> count;  // X: the order-2 buffer over exactly {a, b} read most often
            for (const View& v : s.factors)
                if (v.ids == space && bufs_[static_cast<std::size_t>(v.buf)].order == 2) ++count[v.buf];
            int xb = -1, best = 0;
            for (const auto& [buf, c] : count)
                if (c > best) {
                    best = c;
                    xb = buf;
                }
            if (xb < 0 || best > 4) continue;
            const bool xsym = bufs_[static_cast<std::size_t>(xb)].symmetric;
            const View* x0 = nullptr;
            for (const View& v : s.factors)
                if (v.buf == xb && v.ids == space) {
                    x0 = &v;
                    break;
                }
            // the sweep's row index: the output index of a row reduction, the
            // first output index of a store, else X's leading index
            int R, mode;
            if (s.out_ids.empty()) {
                mode = kEpiSumAll;
                R = x0->stride[static_cast<std::size_t>(a)] == n_ ? a : b;
            } else if (s.out_ids.size() == 1) {
                mode = kEpiSumCols;
                R = s.out_ids[0];
            } else {
                continue;  // elementwise outputs stay stream ops
            }
            const int Cc = R == a ? b : a;
            bool ok = true;
            int power = 0;
            std::vector<View> w;
            for (const View& v : s.factors) {
                if (v.buf == xb && v.ids == space) {
                    const long long sr = v.stride[static_cast<std::size_t>(R)], sc = v.stride[static_cast<std::size_t>(Cc)];
                    if (!((sr == n_ && sc == 1) || (xsym && sr == 1 && sc == n_))) ok = false;
                    ++power;
                } else {
                    if (v.ids & ~space) ok = false;
                    w.push_back(v);
                }
            }
            int nrow = 0, ncol = 0;
            for (const View& v : w) {
                if (!ok) break;
                const auto [wr, wc] = sweep_strides(v, R, Cc);
                if (wc != 0 && wc != 1) ok = false;
                nrow += wc == 0;
                ncol += wc == 1;
            }
            if (!ok || nrow > 4 || ncol > 0) continue;  // row weights only: consumers share the power sums
            Op::Epi e;
            e.mode = mode;
            e.w = std::move(w);
            e.self_power = power;
            e.row_id = R;
            e.col_id = Cc;
            e.out = s.out;
            e.ext = s.ext;
            by_x[xb].push_back({i, std::move(e)});
        }
        return by_x;
    };
    for (bool merged = true; merged;) {
        merged = false;
        // transitive producers over the current (possibly already swept) program
        const std::size_t N = ops_.size();
        std::vector<int> producer(bufs_.size(), -1);
        for (std::size_t i = 0; i < N; ++i) {
            const Op& op = ops_[i];
            if (op.dead) continue;
            if (!op.ext && op.out >= 0 && (!op.gemm || op.store)) producer[static_cast<std::size_t>(op.out)] = static_cast<int>(i);
            for (const Op::Epi& e : op.epis)
                if (!e.ext && e.out >= 0) producer[static_cast<std::size_t>(e.out)] = static_cast<int>(i);
        }
        const std::size_t words = (N + 63) / 64;
        std::vector<std::uint64_t> deps(N * words, 0);
        std::vector<char> state(N, 0);
        auto close = [&](auto&& self, std::size_t i) -> void {
            if (state[i] == 2) return;
            state[i] = 1;
            for_each_read(ops_[i], [&](const View& v) {
                const int p = producer[static_cast<std::size_t>(v.buf)];
                if (p < 0 || static_cast<std::size_t>(p) == i) return;
                const auto pp = static_cast<std::size_t>(p);
                if (state[pp] != 2) self(self, pp);
                for (std::size_t w = 0; w < words; ++w) deps[i * words + w] |= deps[pp * words + w];
                deps[i * words + pp / 64] |= std::uint64_t{1} << (pp % 64);
            });
            state[i] = 2;
        };
        for (std::size_t i = 0; i < N; ++i)
            if (!ops_[i].dead) close(close, i);
        auto depends = [&](std::size_t i, std::size_t j) { return (deps[i * words + j / 64] >> (j % 64)) & 1; };
        // Matrix weights tie their buffers' lifetimes to the sweep: allowed
        // only while X plus every such weight stays a small share of the
        // memory budget (C3: 2 GiB matrices yes; C5: 32 GiB ones no)
        const double mat = 8.0 * static_cast<double>(n_) * static_cast<double>(n_);
        const double room = budget_ > 0 ? 0.25 * budget_ : 0.25 * 179.0 * 1073741824.0;
        for (auto& [xb, cands] : candidates()) {
            if (cands.size() < 2) continue;
            std::vector<Cand> group;
            std::vector<int> mats;

            for (Cand& c : cands) {
                if (group.size() >= static_cast<std::size_t>(kMaxSweep)) break;
                bool indep = true;
                for (const Cand& g : group)
                    if (depends(c.op, g.op) || depends(g.op, c.op)) indep = false;
                if (!indep) continue;
                std::vector<int> m2 = mats;
                for (const View& v : c.epi.w)
                    if (bufs_[static_cast<std::size_t>(v.buf)].order >= 2 &&
                        std::find(m2.begin(), m2.end(), v.buf) == m2.end())
                        m2.push_back(v.buf);
                if (!m2.empty() && mat * static_cast<double>(m2.size() + 1) > room) continue;
                mats = std::move(m2);
                group.push_back(std::move(c));
            }
            if (group.size() < 2) continue;
            Op sw;
            sw.sweep = true;
            View xv;
            xv.buf = xb;
            xv.ids = bit(0) | bit(1);  // positional: 0 = row, 1 = column
            xv.stride[0] = n_;
            xv.stride[1] = 1;
            sw.factors = {xv};
            for (Cand& c : group) {
                sw.epis.push_back(std::move(c.epi));
                ops_[c.op].dead = true;
            }
            if (stats_) stats_->fused_epilogues += group.size();
            ops_.push_back(std::move(sw));
            merged = true;
            break;  // recompute dependencies with the new sweep in place
        }
    }
}

// (row stride, column stride) of a sweep weight; a symmetric matrix read
// column-major is read row-major instead. Column stride 0 = a row weight,
// 1 = a column stream; anything else cannot join a sweep.
std::pair<long long, long long> Program::sweep_strides(const View& v, int row_id, int col_id) const {
    long long wr = v.ids & bit(row_id) ? v.stride[static_cast<std::size_t>(row_id)] : 0;
    long long wc = v.ids & bit(col_id) ? v.stride[static_cast<std::size_t>(col_id)] : 0;
    if (bufs_[static_cast<std::size_t>(v.buf)].symmetric && wr == 1 && wc == n_) {
        wr = n_;
        wc = 1;
    }
    return {wr, wc};
}


// Memory-bounded scheduling. Ops that allocate no tensor of order >= 2 run
// eagerly as soon as their inputs exist (they only free memory); the order in
// which the "big" producers (GEMM products, materialized Hadamard operands)
// run is searched depth-first, cheapest resulting live set first, pruning any
// branch whose peak (inputs + live intermediates) exceeds the budget. Shared
// sub-contractions make the naive recording order hold many n^2 products at
// once (C5: 412 GB); the search finds orders that fit one B200.
void Program::make_schedule(double budget) {
    const std::size_t N = ops_.size();
    for (Op& op : ops_) op.long_chunks = false;  // decided at the end, from this schedule's slack
    std::vector<std::vector<int>> reads(N), outs(N);
    std::vector<int> consumers(bufs_.size(), 0);
    for (std::size_t i = 0; i < N; ++i) {
        const Op& op = ops_[i];
        if (op.dead) continue;
        for_each_read(op, [&](const View& v) {
            if (std::find(reads[i].begin(), reads[i].end(), v.buf) == reads[i].end()) reads[i].push_back(v.buf);
        });
        for (int b : reads[i]) ++consumers[static_cast<std::size_t>(b)];
        if (!op.ext && op.out >= 0 && (!op.gemm || op.store)) outs[i].push_back(op.out);
        for (const Op::Epi& e : op.epis)
            if (!e.ext && e.out >= 0) outs[i].push_back(e.out);
    }
    auto size = [&](int b) { return 8.0 * static_cast<double>(ipow(n_, bufs_[static_cast<std::size_t>(b)].order)); };
    // transient bytes while the op runs (emulated-GEMM digit panels): counted
    // at the op, after its outputs are allocated and before its inputs are freed
    std::vector<double> scratch(N, 0.0);
    for (std::size_t i = 0; i < N; ++i)
        if (!ops_[i].dead) scratch[i] = static_cast<double>(op_scratch_bytes(ops_[i]));
    std::vector<char> big(N, 0);
    for (std::size_t i = 0; i < N; ++i)
        for (int b : outs[i]) big[i] |= bufs_[static_cast<std::size_t>(b)].order >= 2;

    struct State {
        std::vector<char> exec, avail;
        std::vector<int> left;
        double live = 0, peak = 0;
        std::vector<std::size_t> order;
    };
    State s0;
    s0.exec.assign(N, 0);
    s0.avail.assign(bufs_.size(), 0);
    s0.left = consumers;
    for (std::size_t b = 0; b < bufs_.size(); ++b)
        if (bufs_[b].input) {
            s0.avail[b] = 1;
            s0.live += size(static_cast<int>(b));
        }
    s0.peak = s0.live;
    std::size_t live_ops = 0;
    for (const Op& op : ops_) live_ops += !op.dead;

    auto ready = [&](const State& st, std::size_t i) {
        if (ops_[i].dead || st.exec[i]) return false;
        for (int b : reads[i])
            if (!st.avail[static_cast<std::size_t>(b)]) return false;
        return true;
    };
    auto run = [&](State& st, std::size_t i) {
        st.exec[i] = 1;
        st.order.push_back(i);
        for (int b : outs[i]) {
            st.avail[static_cast<std::size_t>(b)] = 1;
            st.live += size(b);
        }
        st.peak = std::max(st.peak, st.live + scratch[i]);
        for (int b : reads[i])
            if (--st.left[static_cast<std::size_t>(b)] == 0 && !bufs_[static_cast<std::size_t>(b)].input && !keep_.count(b))
                st.live -= size(b);
    };
    auto drain = [&](State& st) {  // every ready op that allocates nothing big
        for (bool again = true; again;) {
            again = false;
            for (std::size_t i = 0; i < N; ++i)
                if (!big[i] && ready(st, i)) {
                    run(st, i);
                    again = true;
                }
        }
    };
    std::size_t nodes = 0;
    const std::size_t node_limit = 20000;
    bool found = false;
    State best;
    auto dfs = [&](auto&& self, State st) -> void {
        if (found || ++nodes > node_limit) return;
        drain(st);
        if (st.order.size() == live_ops) {
            found = true;
            best = std::move(st);
            return;
        }
        std::vector<std::pair<double, State>> next, idle;
        for (std::size_t i = 0; i < N; ++i) {
            if (!big[i] || !ready(st, i)) continue;
            State t = st;
            run(t, i);
            // a product read by exactly one other op (a materialized GEMM
            // operand) is consumed at once: the pair is one scheduling step
            for (int b : outs[i]) {
                if (consumers[static_cast<std::size_t>(b)] != 1) continue;
                for (std::size_t j = 0; j < N; ++j)
                    if (std::find(reads[j].begin(), reads[j].end(), b) != reads[j].end() && ready(t, j)) run(t, j);
            }
            drain(t);
            if (budget > 0 && t.peak > budget) continue;
            // products nobody can consume yet only hold memory: try them last
            bool useful = false;
            for (int b : outs[i]) useful |= t.left[static_cast<std::size_t>(b)] < consumers[static_cast<std::size_t>(b)];
            (useful ? next : idle).emplace_back(t.live, std::move(t));
        }
        std::stable_sort(idle.begin(), idle.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
        std::stable_sort(next.begin(), next.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
        for (auto& nx : idle) next.push_back(std::move(nx));
        for (auto& nx : next) {
            self(self, std::move(nx.second));
            if (found) return;
        }
    };
    dfs(dfs, s0);
    if (std::getenv("USTATS_SCHED_DEBUG"))
        std::fprintf(stderr, "[sched] ops=%zu nodes=%zu found=%d budget=%.1f GiB inputs=%.1f GiB\n", live_ops, nodes,
                     found ? 1 : 0, budget / 1073741824.0, s0.live / 1073741824.0);
    if (!found) {  // no order within budget: least-growth greedy (may exceed the budget)
        State st = s0;
        while (st.order.size() < live_ops) {
            drain(st);
            if (st.order.size() == live_ops) break;
            long pick = -1;
            double pick_live = 0;
            for (std::size_t i = 0; i < N; ++i) {
                if (!big[i] || !ready(st, i)) continue;
                State t = st;
                run(t, i);
                drain(t);
                if (pick < 0 || t.live < pick_live) {
                    pick = static_cast<long>(i);
                    pick_live = t.live;
                }
            }
            if (pick < 0) fail(ErrorCode::InvalidArgument, "executor: dependency cycle in the device program");
            run(st, static_cast<std::size_t>(pick));
            if (std::getenv("USTATS_SCHED_DEBUG"))
                std::fprintf(stderr, "[sched] greedy big op %ld live %.1f GiB peak %.1f GiB\n", pick, st.live / 1073741824.0,
                             st.peak / 1073741824.0);
        }
        best = std::move(st);
    }
    schedule_ = best.order;
    sched_peak_ = best.peak;
    sched_fits_ = found;
    // Fewer, longer K chunks for the emulated GEMMs whose place in this order
    // leaves room for the larger digit panels (C5: 3 chunks of 21888 need
    // 2 x 8.02 GiB where 4 chunks of 16384 need 2 x 6 GiB; each chunk less saves
    // a read-modify-write pass over the outputs and a drain per tile). Decided
    // per op from the live set at that op, with 2 GiB to spare; the schedule's
    // peak never rises above the budget.
    if (found && budget > 0 && rt_ && !config_.device.shard_rows) {
        State st = s0;
        for (std::size_t i : best.order) {
            Op& op = ops_[i];
            double live_with_outputs = st.live;
            for (int b : outs[i]) live_with_outputs += size(b);
            if (op.gemm && !op.dead && scratch[i] > 0) {
                op.long_chunks = true;
                const double longer = static_cast<double>(op_scratch_bytes(op));
                if (longer <= scratch[i] || live_with_outputs + longer + 2.0 * 1073741824.0 > budget) op.long_chunks = false;
                else scratch[i] = longer;
            }
            run(st, i);
        }
        sched_peak_ = std::max(sched_peak_, st.peak);
    }
}

// Lazy GEMM operands. A multi-factor operand is recorded as an elementwise
// stream op forming it k-major (Program::gemm's `lower`); when that product
// is read only as a whole operand of GEMMs that run emulated, it is never
// materialized: the op is dropped and each GEMM reads the factors directly,
// their digits formed straight from them (ozaki_split_lazy). C4: its two
// n^3 Khatri-Rao operands (8.6 GB each in FP64) are written, read for the
// row exponents and read again for the digits no more.
void Program::lazy_operands() {
    const std::uint64_t lo = config_.device.oz_min_dim > 0 ? static_cast<std::uint64_t>(config_.device.oz_min_dim) : 1024;
    if (!config_.device.fp64_emulation || static_cast<std::uint64_t>(n_) < lo) return;
    std::vector<int> readers(bufs_.size(), 0);
    for (const Op& op : ops_)
        if (!op.dead) for_each_read(op, [&](const View& v) { ++readers[static_cast<std::size_t>(v.buf)]; });
    auto flat_rows = [&](const View& v, const std::vector<int>& rows) {
        for (std::size_t d = 1; d < rows.size(); ++d)
            if (v.stride[static_cast<std::size_t>(rows[d - 1])] != v.stride[static_cast<std::size_t>(rows[d])] * n_)
                return false;
        return true;
    };
    for (Op& s : ops_) {
        if (s.dead || s.gemm || s.sweep || s.ext || s.sum != 0 || s.out < 0 || keep_.count(s.out)) continue;
        if (s.factors.size() < 2 || s.factors.size() > static_cast<std::size_t>(kMaxGemmFactors)) continue;
        // order >= 3 only: an n^3 Khatri-Rao operand from n^2 factors (forming
        // an n^2 Hadamard product once is cheaper than re-forming it per K chunk
        // and per operand side: C5's B o B measured 21.2 -> 25.1 s lazy)
        const int b = s.out, order = static_cast<int>(s.out_ids.size());
        if (order < 3) continue;
        // every reader: a GEMM holding b as the single view of one operand, emulated by size
        std::vector<std::pair<Op*, bool>> uses;  // (gemm, on side a)
        bool ok = true;
        int seen = 0;
        for (Op& g : ops_) {
            if (g.dead) continue;
            int here = 0;
            for_each_read(g, [&](const View& v) { here += v.buf == b; });
            if (!here) continue;
            seen += here;
            const bool on_a = g.gemm && g.fa.size() == 1 && g.fa[0].buf == b;
            const bool on_b = g.gemm && g.fb.size() == 1 && g.fb[0].buf == b;
            const std::uint64_t rows = ipow(n_, static_cast<int>(g.ra.size())), cols = ipow(n_, static_cast<int>(g.rb.size()));
            // fused epilogues need plain TMA operands on the DMMA path (row panels
            // too short for the INT8 path fall back to it): plain stores only
            if (here != 1 || !(on_a || on_b) || rows < lo || cols < lo || !g.epis.empty()) {
                ok = false;
                break;
            }
            // the other operand must be a plain matrix view (or itself lazy)
            const std::vector<View>& other = on_a ? g.fb : g.fa;
            if (other.size() == 1 && !flat_rows(other[0], on_a ? g.rb : g.ra)) {
                ok = false;
                break;
            }
            uses.emplace_back(&g, on_a);
        }
        if (!ok || uses.empty() || seen != readers[static_cast<std::size_t>(b)]) continue;
        // compose each use: GEMM id -> axis of b -> the stream op's id
        std::vector<std::vector<View>> composed;
        for (auto& [g, on_a] : uses) {
            const View& v = on_a ? g->fa[0] : g->fb[0];
            std::vector<int> axis_src(static_cast<std::size_t>(order), -1);  // axis -> GEMM id
            for (int id : ids_of(v.ids)) {
                const long long st = v.stride[static_cast<std::size_t>(id)];
                int a = -1;
                for (int x = 0; x < order; ++x)
                    if (st == static_cast<long long>(ipow(n_, order - 1 - x))) a = x;
                if (a < 0 || axis_src[static_cast<std::size_t>(a)] >= 0) {
                    ok = false;
                    break;
                }
                axis_src[static_cast<std::size_t>(a)] = id;
            }
            if (!ok) break;
            for (int x = 0; x < order; ++x) ok &= axis_src[static_cast<std::size_t>(x)] >= 0;
            if (!ok) break;
            std::vector<View> fs;
            for (const View& f : s.factors) {
                View c;
                c.buf = f.buf;
                for (int x = 0; x < order; ++x) {
                    const int sid = s.out_ids[static_cast<std::size_t>(x)], gid = axis_src[static_cast<std::size_t>(x)];
                    if (!(f.ids & bit(sid))) continue;
                    c.ids |= bit(gid);
                    c.stride[static_cast<std::size_t>(gid)] = f.stride[static_cast<std::size_t>(sid)];
                }
                fs.push_back(c);
            }
            composed.push_back(std::move(fs));
        }
        if (!ok) continue;
        for (std::size_t u = 0; u < uses.size(); ++u) (uses[u].second ? uses[u].first->fa : uses[u].first->fb) = composed[u];
        s.dead = true;
    }
}

void Program::optimize(double budget_bytes) {
    budget_ = budget_bytes;
    if (config_.device.fuse_epilogues) fuse_epilogues();
    lazy_operands();
    make_schedule(budget_bytes);
    if (config_.device.fuse_epilogues) {
        // sweeps tie their consumers' operands together; keep them only if
        // the memory-bounded schedule stays well inside the budget or does
        // not get a higher peak (C5 at n = 65536 reverts, C3/C4 keep them)
        const std::vector<Op> before = ops_;
        const std::vector<std::size_t> sched = schedule_;
        const double peak = sched_peak_;
        const bool fits = sched_fits_;
        const std::uint64_t fused = stats_ ? stats_->fused_epilogues : 0;
        fuse_sweeps();
        if (ops_.size() != before.size()) {
            make_schedule(budget_bytes);
            const double roomy = 0.6 * (budget_bytes > 0 ? budget_bytes : 179.0 * 1073741824.0);
            if (sched_peak_ > std::max(peak * 1.0001 + 1.0, roomy)) {
                ops_ = before;
                schedule_ = sched;
                sched_peak_ = peak;
                sched_fits_ = fits;
                if (stats_) stats_->fused_epilogues = fused;
            }
        }
    }
    // a program that cannot fit the device fails here, typed, before anything
    // is launched (the reference throws MemoryCapExceeded before allocating,
    // tensor.cpp:9-23); plan-only programs (no runtime) just report the peak
    if (rt_ && budget_bytes > 0 && !sched_fits_ && sched_peak_ > budget_bytes)
        fail(ErrorCode::MemoryCapExceeded,
             "device program needs " + std::to_string(static_cast<long long>(sched_peak_ / 1048576.0)) +
                 " MiB at its peak (inputs, live intermediates and GEMM digit scratch) but the device budget is " +
                 std::to_string(static_cast<long long>(budget_bytes / 1048576.0)) + " MiB");
    for (SymBuf& b : bufs_) b.last_use = -1;
    for (std::size_t pos = 0; pos < schedule_.size(); ++pos)
        for_each_read(ops_[schedule_[pos]],
                      [&](const View& v) { bufs_[static_cast<std::size_t>(v.buf)].last_use = static_cast<int>(pos); });
    // every operand is an input or produced earlier in the schedule
    std::vector<char> have(bufs_.size(), 0);
    for (std::size_t b = 0; b < bufs_.size(); ++b) have[b] = bufs_[b].input;
    for (std::size_t i : schedule_) {
        const Op& op = ops_[i];
        for_each_read(op, [&](const View& v) {
            if (!have[static_cast<std::size_t>(v.buf)])
                fail(ErrorCode::InvalidArgument, "executor: op " + std::to_string(i) + " reads b" + std::to_string(v.buf) +
                                                     " before it is produced");
        });
        if (!op.ext && op.out >= 0 && (!op.gemm || op.store)) have[static_cast<std::size_t>(op.out)] = 1;
        for (const Op::Epi& e : op.epis)
            if (!e.ext && e.out >= 0) have[static_cast<std::size_t>(e.out)] = 1;
    }
}

}  // namespace ustats::dev
