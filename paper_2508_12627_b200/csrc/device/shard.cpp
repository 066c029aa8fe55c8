// Row-sharded execution over W ranks (executor.hpp, ShardStep): the plan is
// pure host work, identical on every rank (it depends only on the recorded
// program and W), so every rank enqueues the same collectives in the same
// order. North star: "the outermost summed index is row-sharded ... each GPU
// emits partial sums combined by a single NCCL all-reduce"; the reference's
// own unit of independence is the V-term (engine.cpp:67-96), combined once
// (engine.cpp:100). Here the shared cross-term program is split instead:
//
//   * every rank owns rows [lo_r, hi_r) of dim 0 of every intermediate;
//   * an op whose output has rows computes only its own rows (stream ops:
//     iteration dim 0 sliced; GEMMs: a row panel of the output, or for a
//     symmetric product stored whole, the blocks (r, r + d), d <= W / 2, of
//     the block triangle, whose transposes go to their row owners);
//   * a reduction to a scalar (or a vector over a non-row index) yields a
//     per-rank partial; the term slots stay partial until the one all-reduce;
//   * a buffer read in a way its distribution cannot serve is first
//     all-gathered (row slabs) or all-reduced (partials: vectors / scalars);
//     a cheap stream op whose output would need gathering and whose inputs
//     are all replicated is computed replicated instead.
#include <algorithm>
#include <bit>
#include <cstdio>
#include <set>
#include <sstream>

#include "executor.hpp"
#include "executor_util.hpp"
#include "ustats/errors.hpp"

namespace ustats::dev {

// The pieces of a symmetric product rank r computes: rows are always its own
// (the row operand is row-local), columns a block R_b: the diagonal block
// (symmetric itself), the blocks R_{r+d}, 0 < d < W/2, and for even W the
// block pair {x, x + W/2} split in halves (x: columns of the first half of
// R_{x+W/2}; x + W/2: its second-half rows against R_x). Every piece's
// transpose belongs to the owner of its columns. Each rank computes W/2
// block units: balanced.
std::vector<TriPiece> Program::tri_pieces(int r) const {
    const int W = std::max(1, shard_planned_world_);
    std::vector<TriPiece> out;
    const long long lo = row_lo(r), hi = row_lo(r + 1);
    out.push_back({lo, hi, lo, hi, r});
    for (int d = 1; 2 * d < W; ++d) {
        const int b = (r + d) % W;
        out.push_back({lo, hi, row_lo(b), row_lo(b + 1), b});
    }
    if (W % 2 == 0 && W > 1) {
        const int b = (r + W / 2) % W;
        if (r < W / 2) {
            const long long c0 = row_lo(b), c1 = row_lo(b + 1), mid = (c0 + (c1 - c0) / 2) & ~1LL;
            out.push_back({lo, hi, c0, mid, b});
        } else {
            const long long mid = (lo + (hi - lo) / 2) & ~1LL;
            out.push_back({mid, hi, row_lo(b), row_lo(b + 1), b});
        }
    }
    return out;
}

namespace {

const char* mode_name(int m) { return m == ShardStep::Repl ? "repl" : m == ShardStep::Rows ? "rows" : "part"; }
const char* coll_name(int k) {
    return k == ShardCollective::Gather ? "gather" : k == ShardCollective::Reduce ? "reduce" : "exchange";
}

}  // namespace

void Program::plan_shards(int world) {
    shard_planned_world_ = world;
    const std::size_t B = bufs_.size();
    std::set<int> force_repl;  // stream outputs produced replicated (their readers need every row)
    for (int pass = 0; pass < 4; ++pass) {
        std::vector<int> dist(B, -1);
        for (std::size_t b = 0; b < B; ++b)
            if (bufs_[b].input) dist[b] = ShardStep::Repl;
        shard_.assign(schedule_.size(), ShardStep{});
        std::set<int> gathered;
        std::vector<int> producer(B, -1);

        // a view of buffer b reads only the rows of dim 0 the op's slice of `id` owns
        auto aligned = [&](const View& v, int id) {
            const int d = dist[static_cast<std::size_t>(v.buf)];
            if (d == ShardStep::Repl) return true;
            if (d != ShardStep::Rows || id < 0 || !(v.ids & bit(id))) return false;
            const SymBuf& sb = bufs_[static_cast<std::size_t>(v.buf)];
            if (sb.order == 0) return false;
            const long long top = static_cast<long long>(ipow(n_, sb.order - 1));
            if (v.stride[static_cast<std::size_t>(id)] >= top) return true;
            return sb.symmetric && sb.order == 2 && std::popcount(v.ids) == 2;  // read through the transpose
        };
        auto bytes_of = [&](int b) { return 8.0 * static_cast<double>(ipow(n_, bufs_[static_cast<std::size_t>(b)].order)); };

        for (std::size_t pos = 0; pos < schedule_.size(); ++pos) {
            const Op& op = ops_[schedule_[pos]];
            ShardStep& st = shard_[pos];
            auto need_repl = [&](int b) {
                int& d = dist[static_cast<std::size_t>(b)];
                if (d == ShardStep::Repl) return;
                for (const ShardCollective& c : st.before)
                    if (c.buf == b) return;
                if (d == ShardStep::Rows) {
                    st.before.push_back({ShardCollective::Gather, b});
                    gathered.insert(b);
                } else {
                    st.before.push_back({ShardCollective::Reduce, b});
                }
                d = ShardStep::Repl;
            };
            auto settle = [&](const View& v, int id) {
                if (!aligned(v, id)) need_repl(v.buf);
            };
            auto set_out = [&](int b, int mode) {
                if (b >= 0) {
                    dist[static_cast<std::size_t>(b)] = mode;
                    producer[static_cast<std::size_t>(b)] = static_cast<int>(pos);
                }
            };
            if (op.sweep) {
                const int rid = op.epis.empty() ? -1 : op.epis[0].row_id;
                st.mode = ShardStep::Rows;
                st.shard_id = rid;
                settle(op.factors[0], rid);
                for (const Op::Epi& e : op.epis)
                    for (const View& v : e.w) settle(v, rid);
                for (const Op::Epi& e : op.epis)
                    if (!e.ext) set_out(e.out, e.mode == kEpiSumAll ? ShardStep::Part : ShardStep::Rows);
                continue;
            }
            if (!op.gemm) {
                if (!op.out_ids.empty()) {
                    const int id = op.out_ids[0];
                    bool all_repl = true;
                    for (const View& v : op.factors) all_repl &= dist[static_cast<std::size_t>(v.buf)] == ShardStep::Repl;
                    if (!op.ext && all_repl && force_repl.count(op.out)) {
                        st.mode = ShardStep::Repl;
                        set_out(op.out, ShardStep::Repl);
                        continue;
                    }
                    st.mode = ShardStep::Rows;
                    st.shard_id = id;
                    for (const View& v : op.factors) settle(v, id);
                    set_out(op.ext ? -1 : op.out, ShardStep::Rows);
                    continue;
                }
                // a reduction to a scalar: slice the summed id that needs the fewest gathers
                const std::vector<int> sums = ids_of(op.sum);
                int best = sums.empty() ? -1 : sums[0];
                double best_cost = -1;
                for (int id : sums) {
                    double cost = 0;
                    for (const View& v : op.factors)
                        if (!aligned(v, id)) cost += dist[static_cast<std::size_t>(v.buf)] == ShardStep::Repl ? 0 : bytes_of(v.buf);
                    if (best_cost < 0 || cost < best_cost) {
                        best_cost = cost;
                        best = id;
                    }
                }
                st.mode = ShardStep::Part;
                st.shard_id = best;
                for (const View& v : op.factors) settle(v, best);
                set_out(op.ext ? -1 : op.out, ShardStep::Part);
                continue;
            }
            // GEMM: out[ra, rb] = sum_e fa fb (+ fused consumers)
            const bool plain = op.epis.empty() && op.store;
            const bool square = op.ra.size() == 1 && op.rb.size() == 1;
            auto side_ok = [&](const std::vector<View>& row_side, int rid, const std::vector<View>& col_side) {
                for (const View& v : row_side)
                    if (!aligned(v, rid)) return false;
                for (const View& v : col_side)
                    if (dist[static_cast<std::size_t>(v.buf)] != ShardStep::Repl) return false;
                return true;
            };
            bool tstore = false;  // a fused transposed store writes columns, not rows: run it whole
            for (const Op::Epi& e : op.epis) tstore |= e.mode == kEpiStore && e.transpose && !e.ext;
            if (tstore || op.ra.empty()) {
                st.mode = ShardStep::Repl;
                for_each_read(op, [&](const View& v) { need_repl(v.buf); });
                if (op.store && !op.ext) set_out(op.out, ShardStep::Repl);
                for (const Op::Epi& e : op.epis)
                    if (!e.ext) set_out(e.out, ShardStep::Repl);
                continue;
            }
            st.mode = ShardStep::Rows;
            st.shard_id = op.ra[0];
            if (op.symmetric_out && plain && square) {
                // a symmetric product: the operands may trade places (equal values)
                if (!side_ok(op.fa, op.ra[0], op.fb) && side_ok(op.fb, op.rb[0], op.fa)) {
                    st.swap = true;
                    st.shard_id = op.rb[0];
                }
                st.tri = true;
            }
            const std::vector<View>& rows_side = st.swap ? op.fb : op.fa;
            const std::vector<View>& cols_side = st.swap ? op.fa : op.fb;
            for (const View& v : rows_side) settle(v, st.shard_id);
            for (const View& v : cols_side) need_repl(v.buf);
            for (const Op::Epi& e : op.epis)
                for (const View& v : e.w) settle(v, e.row_id);
            if (op.store && !op.ext) {
                set_out(op.out, ShardStep::Rows);
                if (st.tri && world > 1) st.after.push_back({ShardCollective::Exchange, op.out});
            }
            for (const Op::Epi& e : op.epis) {
                if (e.ext) continue;
                const bool row_local = e.mode == kEpiSumCols || (e.mode == kEpiStore && !e.transpose);
                set_out(e.out, row_local ? ShardStep::Rows : ShardStep::Part);
            }
        }
        shard_dist_ = dist;
        // gathered outputs of replicable stream ops: produce them replicated next pass
        bool changed = false;
        for (int b : gathered) {
            const int p = producer[static_cast<std::size_t>(b)];
            if (p < 0 || force_repl.count(b)) continue;
            const Op& op = ops_[schedule_[static_cast<std::size_t>(p)]];
            if (op.gemm || op.sweep || op.out_ids.empty()) continue;
            force_repl.insert(b);
            changed = true;
        }
        if (!changed) break;
    }
    // bytes each rank receives per evaluation
    shard_bytes_[0] = shard_bytes_[1] = shard_bytes_[2] = 0;
    const double W = world;
    for (std::size_t pos = 0; pos < shard_.size(); ++pos) {
        for (const auto* list : {&shard_[pos].before, &shard_[pos].after})
            for (const ShardCollective& c : *list) {
                const double bytes = 8.0 * static_cast<double>(ipow(n_, bufs_[static_cast<std::size_t>(c.buf)].order));
                if (c.kind == ShardCollective::Gather) shard_bytes_[0] += bytes * (W - 1) / W;
                else if (c.kind == ShardCollective::Reduce) shard_bytes_[1] += 2.0 * bytes * (W - 1) / W;  // ring
                else {  // the transposed pieces rank 0 receives
                    double got = 0;
                    for (int a = 1; a < world; ++a)
                        for (const TriPiece& q : tri_pieces(a))
                            if (q.col_owner == 0) got += 8.0 * static_cast<double>((q.r1 - q.r0) * (q.c1 - q.c0));
                    shard_bytes_[2] += got;
                }
            }
    }
}

std::string Program::shard_dump(int rank) const {
    std::ostringstream o;
    const int W = shard_planned_world_;
    o << "world=" << W << " rank=" << rank << " n=" << n_ << " gather_bytes=" << shard_bytes_[0]
      << " reduce_bytes=" << shard_bytes_[1] << " exchange_bytes=" << shard_bytes_[2] << "\n";
    for (std::size_t pos = 0; pos < shard_.size(); ++pos) {
        const ShardStep& st = shard_[pos];
        const Op& op = ops_[schedule_[pos]];
        o << pos << " op" << schedule_[pos] << " " << (op.gemm ? "gemm" : op.sweep ? "sweep" : "stream") << " "
          << mode_name(st.mode)
          << " id=" << st.shard_id;
        if (st.swap) o << " swap";
        auto ord = [&](int b) { return bufs_[static_cast<std::size_t>(b)].order; };
        for (const ShardCollective& c : st.before) o << " pre:" << coll_name(c.kind) << ":b" << c.buf << ":o" << ord(c.buf);
        for (const ShardCollective& c : st.after) o << " post:" << coll_name(c.kind) << ":b" << c.buf << ":o" << ord(c.buf);
        if (st.mode != ShardStep::Repl) {
            if (st.tri) {
                o << " pieces=";
                for (const TriPiece& q : tri_pieces(rank))
                    o << "[" << q.r0 << "," << q.r1 << ")x[" << q.c0 << "," << q.c1 << ")->" << q.col_owner;
            } else {
                o << " rows=[" << row_lo(rank) << "," << row_lo(rank + 1) << ")";
            }
        }
        o << "\n";
    }
    return o.str();
}

// ------------------------------------------------------------- execution

void Program::run_collective(const ShardCollective& c, bool emulate) {
    SymBuf& sb = bufs_[static_cast<std::size_t>(c.buf)];
    if (!sb.real) fail(ErrorCode::InvalidArgument, "shard: collective on an unmaterialized buffer");
    if (emulate) return;  // virtual ranks share one buffer: its rows / partials are already complete
    if (c.kind == ShardCollective::Reduce) {
        rt_->allreduce_sum(sb.real->ptr, sb.real->entries());
    } else if (c.kind == ShardCollective::Gather) {
        const long long row = static_cast<long long>(ipow(n_, sb.order - 1));
        std::vector<std::pair<long long, long long>> slabs;
        for (int r = 0; r < shard_planned_world_; ++r) slabs.emplace_back(row_lo(r) * row, (row_lo(r + 1) - row_lo(r)) * row);
        rt_->allgather_rows(sb.real->ptr, slabs);
    }
    // Exchange runs inside run_tri_gemm (it needs the block temporaries)
}

// A symmetric product as pieces of the block triangle (tri_pieces): rank r
// computes each piece into a temporary, stores it at C[rows, cols] (its own
// rows) and sends its transpose to the owner of the columns, which stores it
// at C[cols, rows]. Virtual ranks (emulate) store the transpose directly.
void Program::run_tri_gemm(const Op& op, double* out, bool emulate) {
    const ShardStep* saved = step_;
    const int W = shard_planned_world_, me = slice_rank_;
    cudaStream_t s = rt_->stream();
    struct Pending {
        int peer;
        double* buf;
        long long r0, r1, c0, c1;  // where it lands: C[r0:r1, c0:c1]
    };
    std::vector<Pending> sends, recvs;
    auto bytes = [](long long r, long long c) { return sizeof(double) * static_cast<std::size_t>(r * c); };
    for (const TriPiece& q : tri_pieces(me)) {
        const long long rows = q.r1 - q.r0, cols = q.c1 - q.c0;
        if (rows <= 0 || cols <= 0) continue;
        double* t = static_cast<double*>(rt_->raw_alloc(bytes(rows, cols)));
        Op blk = op;
        if (saved->swap) {
            std::swap(blk.fa, blk.fb);
            std::swap(blk.ra, blk.rb);
        }
        blk.symmetric_out = op.symmetric_out && q.r0 == q.c0 && q.r1 == q.c1;  // a diagonal block
        block_rows_ = {q.r0, q.r1};
        block_cols_ = {q.c0, q.c1};
        step_ = nullptr;
        try {
            run_gemm(blk, t);
        } catch (...) {
            step_ = saved;
            block_rows_ = block_cols_ = {-1, -1};
            throw;
        }
        step_ = saved;
        block_rows_ = block_cols_ = {-1, -1};
        check_cuda(cudaMemcpy2DAsync(out + q.r0 * n_ + q.c0, sizeof(double) * n_, t, sizeof(double) * cols,
                                     sizeof(double) * cols, rows, cudaMemcpyDeviceToDevice, s),
                   "store piece");
        if (q.col_owner != me || (q.r0 != q.c0 || q.r1 != q.c1)) {
            if (emulate || q.col_owner == me) {
                launch_transpose(t, rows, cols, cols, out + q.c0 * n_ + q.r0, n_, s);
            } else {
                double* tt = static_cast<double*>(rt_->raw_alloc(bytes(rows, cols)));
                launch_transpose(t, rows, cols, cols, tt, rows, s);
                sends.push_back({q.col_owner, tt, q.c0, q.c1, q.r0, q.r1});
            }
        }
        rt_->raw_free(t, bytes(rows, cols));
    }
    if (!emulate) {
        // pieces of other ranks whose transposes land in this rank's rows
        for (int a = 0; a < W; ++a) {
            if (a == me) continue;
            for (const TriPiece& q : tri_pieces(a))
                if (q.col_owner == me && q.r1 > q.r0 && q.c1 > q.c0)
                    recvs.push_back({a, static_cast<double*>(rt_->raw_alloc(bytes(q.c1 - q.c0, q.r1 - q.r0))), q.c0, q.c1,
                                     q.r0, q.r1});
        }
        std::vector<Runtime::P2P> ops;
        for (const Pending& p : sends)
            ops.push_back({true, p.peer, p.buf, static_cast<std::size_t>((p.r1 - p.r0) * (p.c1 - p.c0))});
        for (const Pending& p : recvs)
            ops.push_back({false, p.peer, p.buf, static_cast<std::size_t>((p.r1 - p.r0) * (p.c1 - p.c0))});
        rt_->sendrecv(ops);
        for (const Pending& p : recvs) {
            const long long cols = p.c1 - p.c0;
            check_cuda(cudaMemcpy2DAsync(out + p.r0 * n_ + p.c0, sizeof(double) * n_, p.buf, sizeof(double) * cols,
                                         sizeof(double) * cols, p.r1 - p.r0, cudaMemcpyDeviceToDevice, s),
                       "store received piece");
            rt_->raw_free(p.buf, bytes(p.r1 - p.r0, cols));
        }
        for (const Pending& p : sends) rt_->raw_free(p.buf, bytes(p.r1 - p.r0, p.c1 - p.c0));
    }
}

void Program::execute_sharded(int world, bool emulate) {
    const DeviceConfig& dc = config_.device;
    shard_emulate_ = emulate;
    if (shard_planned_world_ != world || shard_.size() != schedule_.size()) plan_shards(world);
    rt_->set_stream(rt_->main_stream());
    for (const SymBuf& b : bufs_)
        if (b.input && b.real && !b.real->ready.empty())
            check_cuda(cudaStreamWaitEvent(rt_->main_stream(), b.real->ready.back().second, 0), "wait upload");
    for (std::size_t pos = 0; pos < schedule_.size(); ++pos) {
        Op& op = ops_[schedule_[pos]];
        const ShardStep& st = shard_[pos];
        slice_world_ = world;
        for (const ShardCollective& c : st.before) run_collective(c, emulate);
        step_ = &st;
        if (st.mode == ShardStep::Repl) {
            slice_world_ = 1;  // the whole op on every rank (once when emulated)
            slice_rank_ = 0;
            step_ = nullptr;
            launch(op);
        } else {
            for (int r = (emulate ? 0 : dc.rank); r < (emulate ? world : dc.rank + 1); ++r) {
                slice_rank_ = r;
                launch(op);
            }
        }
        step_ = nullptr;
        slice_world_ = world;
        for_each_read(op, [&](const View& v) {
            SymBuf& b = bufs_[static_cast<std::size_t>(v.buf)];
            if (!b.input && b.last_use == static_cast<int>(pos) && b.real && b.real.use_count() == 1 &&
                !keep_.count(v.buf))
                b.real.reset();
        });
    }
    slice_world_ = 1;
    slice_rank_ = 0;
}

}  // namespace ustats::dev
