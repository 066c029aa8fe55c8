// Device executor. Each V-term's notation is *recorded* into a Program with
// the reference's elimination semantics (proj/src/einsum.cpp:310-486), then
// the whole statistic's Program is optimized and launched:
//   * lazy folds / marginalizations: a fold (fold_into, einsum.cpp:134-147)
//     appends a factor view; a marginalization records a pending sum; both are
//     formed inside whichever kernel consumes the slot;
//   * every materialized intermediate is content-addressed: an op whose
//     canonical form (kind, operand buffers' content ids and the stride
//     pattern over its local dims) was already recorded — in this V-term or
//     an earlier one — is not recorded again (the reference recomputes every
//     sub-contraction of every V-term);
//   * among the width-optimal elimination orders of a V-term, the one whose
//     new work (DMMA MACs + streamed entries) is smallest given what earlier
//     terms already produced is chosen;
//   * a reduction that is the only consumer of a GEMM output is fused into
//     the GEMM epilogue (Hadamard with its other factors, the GEMM output
//     itself when it appears twice, fixed-order reduction to a scalar or
//     vector); a GEMM whose two operands are the same content is symmetric
//     and only its upper tiles are computed.
// Reference-rule counters (ExecStats semantics, einsum.cpp:146-484) are
// tallied on a counting walk of the reference's own order.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include <cuda_runtime.h>

#include <functional>
#include <mutex>

#include "kernels.hpp"
#include "ustats/config.hpp"
#include "ustats/notation.hpp"
#include "ustats/ordering.hpp"

namespace ustats::dev {

constexpr int kMaxIds = 16;

void check_cuda(cudaError_t e, const char* what);

class Runtime;

struct DeviceBuffer {
    double* ptr = nullptr;
    int order = 0;
    long long n = 1;
    bool symmetric = false;
    bool borrowed = false;
    bool slab = false;  // from the runtime's slab cache (returned there, not freed)
    Runtime* rt = nullptr;
    // chunked upload in flight: rows [0, first) are usable once `second` completes
    std::vector<std::pair<long long, cudaEvent_t>> ready;
    ~DeviceBuffer();
    std::uint64_t entries() const;
};
using Buf = std::shared_ptr<DeviceBuffer>;

class Runtime {
  public:
    static Runtime& get(int device);
    ~Runtime();

    cudaStream_t stream() const { return cur_; }  // where allocations / launches go now
    cudaStream_t main_stream() const { return stream_; }
    // the auxiliary streams note that they were handed out: sync() waits only
    // for those (eight cudaStreamSynchronize calls per evaluation otherwise)
    cudaStream_t side_stream() { used_ |= 1; return side_; }
    cudaStream_t copy_stream() { used_ |= 2; return copy_; }
    cudaStream_t prep_stream() { used_ |= 4; return prep_; }
    // Device memory available to this engine: free memory when the runtime was
    // created (the stream-ordered pool then recycles it). cudaMemGetInfo can
    // stall for tens of ms, so it is re-queried only for programs that need
    // most of the device (refresh_free_bytes).
    double free_bytes() const { return free_bytes_; }
    void refresh_free_bytes();
    void agree_free_bytes();  // row sharding: every rank plans with the communicator's minimum
    static constexpr int kChunkStreams = 4;
    cudaStream_t chunk_stream(int i) { used_ |= 8; return chunk_[i % kChunkStreams]; }
    // bitwise-symmetry results of host inputs seen before (speculation key)
    std::map<std::pair<const void*, long long>, bool> symmetry_seen;
    void set_stream(cudaStream_t s) { cur_ = s; }
    int device() const { return device_; }
    int sm_count() const { return sm_count_; }

    Buf allocate(int order, long long n);
    Buf borrow(const double* ptr, int order, long long n);
    double* scratch(std::size_t entries);
    void release(double* p);
    void sync();          // end of an evaluation: waits for the main stream and every auxiliary stream it used
    void wait_streams();  // the same wait in the middle of one (keeps the used-stream notes)

    // Large buffers (>= kSlabMin: n^2 intermediates, Ozaki digit panels) come
    // from a cache of exact-size slabs instead of the stream-ordered pool: a
    // 32 GiB request then never fails on a pool fragmented by smaller blocks,
    // and a program that repeats (the plan cache) reuses the same slabs. A
    // returned slab carries the event of its release, which its next user's
    // stream waits on. reclaim() hands every idle slab and the pool's unused
    // blocks back to the driver (after a sync) when an allocation fails.
    static constexpr std::size_t kSlabMin = std::size_t{1} << 30;
    // slab (>= kSlabMin and slab_ok) or pool, retrying once after reclaim();
    // MemoryCapExceeded when even that fails
    void* raw_alloc(std::size_t bytes, bool slab_ok = true);
    void raw_free(void* p, std::size_t bytes);     // stream-ordered on the current stream
    void reclaim();
    double idle_slab_bytes() const;

    // NCCL communicator for row sharding (libnccl resolved at run time, so
    // the library has no link-time NCCL dependency and shares the process's copy).
    void nccl_init(int rank, int world, const void* unique_id);
    static void nccl_unique_id(void* out128);
    bool has_comm() const { return comm_ != nullptr; }
    int comm_world() const { return comm_world_; }
    void allreduce_sum(double* p, std::size_t count);
    // row sharding: every rank's slab (offset, entries) to every rank, in place
    void allgather_rows(double* p, const std::vector<std::pair<long long, long long>>& slabs);
    struct P2P {
        bool send = true;
        int peer = 0;
        double* buf = nullptr;
        std::size_t count = 0;
    };
    void sendrecv(const std::vector<P2P>& ops);  // one NCCL group

    enum Kind { kGemm = 0, kStream = 1, kOther = 2 };
    struct Profile {
        double ms[3] = {0, 0, 0};
        std::uint64_t groups[3] = {0, 0, 0};
    };
    void profile_enable(bool on) { profiling_ = on; }
    bool profiling() const { return profiling_; }
    void begin(Kind k);
    void end(Kind k);
    Profile collect(bool reset);

  private:
    explicit Runtime(int device);
    int device_ = 0;
    int sm_count_ = 148;
    cudaStream_t stream_ = nullptr;
    cudaStream_t side_ = nullptr;  // second stream: bandwidth ops overlap GEMM tails
    cudaStream_t copy_ = nullptr;  // chunked host->device uploads (copies only: never waits for an SM)
    cudaStream_t prep_ = nullptr;  // per-panel sparsify / probe kernels behind the copies (high priority)
    cudaStream_t chunk_[kChunkStreams] = {};  // concurrent per-panel GEMM pieces
    cudaStream_t cur_ = nullptr;
    unsigned used_ = 0;  // auxiliary streams handed out since the last sync (bit 0 side, 1 copy, 2 prep, 3 chunk)
    void* comm_ = nullptr;
    int comm_world_ = 1;
    double free_bytes_ = 0;
    bool profiling_ = false;
    std::vector<cudaEvent_t> pool_;
    struct Slab {
        void* ptr = nullptr;
        std::size_t bytes = 0;
        cudaEvent_t freed = nullptr;
    };
    std::vector<Slab> idle_;
    void* slab_get(std::size_t bytes);
    void slab_put(void* p, std::size_t bytes);
    struct Mark {
        Kind kind;
        cudaEvent_t a, b;
    };
    std::vector<Mark> marks_;
    Profile totals_;
};

struct DevStats {
    std::uint64_t ref_madds = 0;
    std::uint64_t ref_peak = 0;
    int steps = 0;
    std::uint64_t gemm_macs = 0;
    std::uint64_t stream_entries = 0;
    std::uint64_t gemm_launches = 0;
    std::uint64_t stream_launches = 0;
    std::uint64_t shared_hits = 0;
    std::uint64_t kernel_launches = 0;
    std::uint64_t emulated_macs = 0;  // FP64 MACs of GEMMs run on the INT8 tensor cores
    std::uint64_t int8_ops = 0;       // INT8 tensor-core ops those issued
    std::uint64_t fused_epilogues = 0;
    std::uint64_t symmetric_gemms = 0;
    std::uint64_t oz_slices = 0;      // digit slices the last emulated GEMM used (0 = none ran)
};

// Emulated-GEMM plan of one product (launch.cpp): digit slices (error-bound
// guard or Config.oz_slices), K chunking, and the digit scratch it needs.
struct OzPlan {
    int slices = 6;
    long long nchunks = 1, kc = 0;
    std::size_t a_bytes = 0, b_bytes = 0, scratch_bytes = 0;
};
int oz_guard_slices(long long K);
// long_chunks: the op's place in the schedule leaves room for bigger digit panels (fewer K chunks)
OzPlan oz_plan(long long K, long long rows, long long cols, bool same_operand, const DeviceConfig& dc,
               bool long_chunks = false);

// ------------------------------------------------------------------ Program
struct View {
    int buf = -1;
    std::array<long long, kMaxIds> stride{};
    std::uint32_t ids = 0;
};

struct SymBuf {
    int order = 0;
    bool symmetric = false;
    // a known power of a symmetric matrix: base content id (-1 = none) and
    // exponent; products of powers of one base commute, so they are symmetric
    int power_base = -1;
    int power = 0;
    // B^p scaled by vectors along one axis (row or column), i.e. B^p D or
    // D B^p for a diagonal D: B^p D B^p is symmetric
    int scaled_base = -1, scaled_power = 0, scaled_w = -1, scaled_axis = -1;
    bool input = false;
    Buf real;
    int content = -1;
    int last_use = -1;
};

struct Op {
    bool gemm = false;
    // stream: out[out_ids] = sum_{sum} prod factors
    std::vector<View> factors;
    std::vector<int> out_ids;
    std::uint32_t sum = 0;
    // gemm: out[ra, rb] = sum_e prod(fa) prod(fb)   (fa, fb single views after lowering)
    std::vector<View> fa, fb;
    std::vector<int> ra, rb;
    int e = -1;
    // fused consumers of the product (multi-epilogue); `store` also writes it to `out`
    struct Epi {
        int mode = kEpiStore;
        std::vector<View> w;     // weights over (row_id, col_id) of the consumer's ids
        int self_power = 1;
        int row_id = -1, col_id = -1;
        bool transpose = false;  // Store: the consumer wants (col, row) layout
        int out = -1;
        double* ext = nullptr;
    };
    std::vector<Epi> epis;
    bool store = true;
    bool symmetric_out = false;
    // emulated GEMM: the schedule leaves room at this op for the larger digit
    // panels (fewer K chunks; make_schedule decides from the live set)
    bool long_chunks = false;
    // sweep: one pass over the matrix factors[0] (row-major view) feeding the
    // consumers in `epis` (row_id = the matrix's row index)
    bool sweep = false;
    // destination: a program buffer, or an external device pointer
    int out = -1;
    double* ext = nullptr;
    bool dead = false;
};

// Row-sharded execution plan (shard.cpp): every rank owns rows [lo_r, hi_r)
// of dim 0 of every intermediate; buffers are replicated (every rank holds
// all of it), row-sharded (each rank its rows) or partial (each rank holds a
// summand). Collectives appear only where an op needs a buffer in a state
// it is not in: all-gather of row slabs, all-reduce of a partial (vectors and
// scalars only), and the transpose exchange of a symmetric product computed
// as triangle blocks. The term vector is partial until ONE final all-reduce.
struct ShardCollective {
    enum Kind : int { Gather = 0, Reduce = 1, Exchange = 2 } kind = Gather;
    int buf = -1;
};
struct ShardStep {
    enum Mode : int { Repl = 0, Rows = 1, Part = 2 } mode = Repl;
    int shard_id = -1;    // iteration id sliced by rows (stream: placed first; gemm: the row id)
    bool swap = false;    // gemm: operands swapped (symmetric product; the row side is op.fb)
    bool tri = false;     // gemm: symmetric product as blocks (r, r + d), d <= W / 2, then exchanged
    std::vector<ShardCollective> before, after;
};

struct TriPiece {
    long long r0 = 0, r1 = 0, c0 = 0, c1 = 0;  // C[r0:r1, c0:c1], rows owned by the computing rank
    int col_owner = 0;                          // owner of rows [c0, c1): receives the transpose
};

class Program {
  public:
    Program(Runtime* rt, long long n, const Config& config, DevStats* stats)
        : rt_(rt), n_(n), config_(config), stats_(stats) {}  // rt == nullptr: plan only

    // Plan-only inputs (no device memory): order and symmetry of a factor.
    int add_symbolic_input(int order, bool symmetric);
    std::string dump() const;
    struct Totals {
        std::uint64_t gemms = 0, gemm_macs = 0, streams = 0, stream_entries = 0, fused = 0, symmetric = 0;
        std::uint64_t peak_entries = 0;  // live intermediates + inputs, simulated over the schedule
    };
    Totals totals() const;

    int add_input(const Buf& real);
    long long n() const { return n_; }
    const SymBuf& buf(int id) const { return bufs_[static_cast<std::size_t>(id)]; }
    const Config& config() const { return config_; }
    bool sharing() const { return config_.device.share_subexpressions; }

    View view_of(int buf, const IndexTuple& layout) const;

    // Records out[out_ids] = sum_{sum} prod(factors). With `ext`, writes there
    // and returns -1 (a repeat of an earlier term's op becomes a term alias);
    // else returns the (possibly shared) buffer.
    int stream(std::vector<View> factors, const std::vector<int>& out_ids, std::uint32_t sum, double* ext);
    // The buffer an identical earlier stream op produced, or -1 (records nothing).
    int lookup_stream(const std::vector<View>& factors, const std::vector<int>& out_ids, std::uint32_t sum) const;
    // Records a GEMM; returns the buffer and the caller-side layout (ids).
    int gemm(std::vector<View> fa, std::vector<View> fb, const std::vector<int>& ra, const std::vector<int>& rb,
             int e, std::vector<int>* layout);

    struct Mark {
        std::size_t ops = 0, bufs = 0, log = 0, aliases = 0;
    };
    Mark mark() const { return {ops_.size(), bufs_.size(), memo_log_.size(), aliases_.size()}; }
    // Terms whose final reduction repeats an earlier term's (same canonical
    // op): (duplicate slot, source slot); the host copies the value after
    // the D2H instead of launching the reduction again.
    const std::vector<std::pair<double*, double*>>& term_aliases() const { return aliases_; }
    void rollback(const Mark& m);
    double cost_since(const Mark& m) const;

    void keep(int buf) { keep_[buf] = true; }  // a result the caller takes after execute()
    void optimize(double budget_bytes = 0);  // fusion, memory-bounded schedule, last uses
    double scheduled_peak_bytes() const { return sched_peak_; }
    void execute();   // launches every live op in order
    Buf take(int buf);  // result buffer (allocated during execute)
    // Plan reuse: the distinct inputs in first-use order; rebinding new device
    // buffers with the same orders / symmetry / aliasing re-executes the plan.
    std::vector<Buf> inputs() const;
    void rebind_inputs(const std::vector<Buf>& reals);
    void release_buffers();  // drop every device reference after a run
    void set_stats(DevStats* stats) { stats_ = stats; }
    // Plans row-sharded execution over `world` ranks (host only, identical on
    // every rank); dump(): one line per scheduled op plus the collective bytes.
    void plan_shards(int world);
    std::string shard_dump(int rank) const;
    // rows [lo, hi) of dim 0 that rank r owns (every buffer, every op)
    long long row_lo(int r) const {
        const int W = std::max(1, shard_planned_world_);
        return r >= W ? n_ : (n_ * r / W) & ~1LL;
    }
    // the pieces of a symmetric product rank r computes (shard.cpp)
    std::vector<TriPiece> tri_pieces(int r) const;

  private:
    std::string desc(const View& v, const std::vector<int>& dims) const;
    bool power_of(const View& v, int* base, int* pw) const;
    int new_buf(int order, bool symmetric);
    void fuse_epilogues();
    void lazy_operands();
    void fuse_sweeps();
    void run_sweep(const Op& op);
    bool emulated_eligible(const GemmArgs& g) const;
    std::size_t op_scratch_bytes(const Op& op) const;
    int run_emulated(const GemmArgs& g, const EpiSet& set);
    std::pair<long long, long long> sweep_strides(const View& v, int row_id, int col_id) const;
    bool tma_plain(const View& v, const std::vector<int>& rows, int e) const;
    void launch(Op& op);
    void execute_sharded(int world, bool emulate);
    // Digits of an emulated GEMM operand kept for the next GEMM that reads the
    // same operand (one K chunk, single-GPU execution; C4: its Khatri-Rao
    // operand feeds three GEMMs): key -> buffers and the uses still to come
    struct CachedDigits {
        int8_t* d = nullptr;
        int* e = nullptr;
        std::size_t bytes = 0;
        long long rows = 0;
        int uses = 0;
    };
    std::map<std::string, CachedDigits> digits_;
    std::map<std::string, int> digit_uses_;
    std::string key_a_, key_b_;  // operand keys of the GEMM being launched (run_gemm -> run_emulated)
    bool cur_long_chunks_ = false;  // the GEMM being launched may use the larger digit panels
    std::string operand_key(const std::vector<View>& fs, const std::vector<int>& rows, int e) const;
    void plan_digit_reuse();
    void drop_digits();
    void run_collective(const ShardCollective& c, bool emulate);
    void run_tri_gemm(const Op& op, double* out, bool emulate);
    const ShardStep* step_ = nullptr;      // the current op's shard step (row sharding)
    bool shard_emulate_ = false;           // virtual ranks on one device (collectives are no-ops)
    // a block of a GEMM (run_tri_gemm): rows [first, second) of its row id, columns of its column id
    std::pair<long long, long long> block_rows_{-1, -1}, block_cols_{-1, -1};
    std::vector<ShardStep> shard_;         // per schedule position
    std::vector<int> shard_dist_;          // per buffer: final ShardStep::Mode after the plan
    int shard_planned_world_ = 0;
    double shard_bytes_[3] = {0, 0, 0};    // per rank and evaluation: gather / reduce / exchange bytes received
    void run_stream(const Op& op, double* out);
    void run_gemm(const Op& op, double* out);
    double* ptr(int buf) const;

    Runtime* rt_;
    long long n_;
    const Config& config_;
    DevStats* stats_;
    std::vector<SymBuf> bufs_;
    std::vector<Op> ops_;
    std::unordered_map<std::string, int> memo_;
    std::vector<std::string> memo_log_;
    std::string stream_key(const std::vector<View>& factors, const std::vector<int>& out_ids, std::uint32_t sum) const;
    std::map<std::string, double*> term_memo_;  // canonical key of a term-final op -> its slot
    std::vector<std::pair<double*, double*>> aliases_;
    std::map<int, bool> keep_;
    std::vector<std::size_t> schedule_;  // execution order of live ops (memory-aware)
    int slice_rank_ = 0, slice_world_ = 1;  // row sharding: the slice launch() computes
    double sched_peak_ = 0;
    bool sched_fits_ = true;
    double budget_ = 0;
    bool launch_ordered_ = false;
    void make_schedule(double budget_bytes);
};

// Records one notation into a Program with the reference's elimination walk.
// With `count`, also tallies the reference-rule counters and checks the
// memory cap on the reference plan's intermediates.
class Contractor {
  public:
    Contractor(Program& prog, DevStats* count) : p_(prog), count_(count) {}

    // Records the einsum; returns the result buffer (order |output|), or -1
    // when `scalar_out` receives the scalar.
    int run(const std::vector<int>& inputs, const EinsumNotation& notation, const EliminationOrder& order,
            double* scalar_out);
    int eliminate_single(const std::vector<int>& inputs, const std::vector<IndexTuple>& tuples, int index,
                         IndexTuple* result_tuple);

    struct Slot {
        std::uint32_t ids = 0;
        std::vector<View> factors;
        bool owned = false;
    };

  private:
    Slot slot_of(int buf, const IndexTuple& tuple);
    void eliminate_one(std::vector<Slot>& slots, int e);
    Slot marginalize(const Slot& s, std::uint32_t summed);
    Slot gemm_step(const Slot& a, const Slot& b, int e);
    Slot generic_step(const std::vector<Slot>& parts, int e);
    std::vector<View> formed(const Slot& s);  // factors with pending sums formed
    void settle(Slot& s);                     // pending sums an earlier op already formed
    void cap(int order);
    void owned(int order);
    std::uint64_t pw(int e) const;

    Program& p_;
    DevStats* count_;
};

// -------------------------------------------------------- statistic drivers
struct StatisticResult {
    double value = 0.0;
    std::vector<double> terms;
    std::vector<std::vector<int>> rgs;
    std::vector<long long> mu;
    std::vector<double> v;
    std::vector<int> owner;
    DevStats stats;
    std::uint64_t enumerated = 0;
    double upload_seconds = 0.0;
    double contract_seconds = 0.0;
    double plan_seconds = 0.0;
};

enum class LatticeMode { Sparsified, Unsparsified };

struct TermPlan {
    std::vector<std::vector<int>> rgs;
    std::vector<long long> mu;
    std::vector<EinsumNotation> notation;
    std::vector<EliminationOrder> order;
    std::vector<double> cost;
    std::vector<int> owner;
    std::uint64_t enumerated = 0;
};
TermPlan plan_terms(const std::vector<IndexTuple>& zero_sig, int m, long long n, LatticeMode mode,
                    const Config& config);

// Several U-statistics over factors of one extent in ONE program: aliased
// factor pointers are uploaded once and sub-contractions are shared across
// the statistics (e.g. hoif_tau's chain orders 2..m, hoif.cpp:84-86).
struct StatisticSpec {
    std::vector<const double*> inputs;
    std::vector<IndexTuple> sig;
    int m = 0;
    // per input: symmetric by construction (device-built kernels), so the
    // bitwise symmetry probe is skipped; empty = probe every matrix
    std::vector<char> symmetric;
    // per input: already sparsified by its device tensorizer (repeated-index
    // entries written as zero): the separate sparsify pass is skipped
    std::vector<char> sparsified;
};
// Graph replay of a small cached evaluation (data_kernels.cpp). While a
// capture is active on this thread, lattice_batch_impl requires a cached plan,
// copies the term values into the capture's pinned buffer and, where it would
// synchronize, releases the caller's device buffers (before_sync), ends the
// capture, instantiates the graph and launches it once; the evaluation then
// finishes as usual. Later calls launch the graph and recombine the terms.
struct GraphCapture {
    cudaGraphExec_t exec = nullptr;
    double* host_v = nullptr;  // pinned, capacity doubles
    std::size_t capacity = 0, T = 0;
    std::vector<std::pair<std::size_t, std::size_t>> alias;  // (duplicate term, source term)
    std::function<void()> before_sync;
    bool launched = false;
    ~GraphCapture();
};
GraphCapture*& active_capture();                // thread-local; nullptr = none
std::recursive_mutex& device_mutex(int device);  // one evaluation at a time per device
std::uint64_t plan_generation(int device);       // bumps whenever a cached plan is evicted
std::string config_key(const Config& c);
std::uint64_t graph_replays(int device);          // evaluations served by a replayed graph

std::vector<StatisticResult> lattice_batch(const std::vector<StatisticSpec>& specs, bool inputs_on_device,
                                           long long n, LatticeMode mode, const Config& config);
std::vector<StatisticResult> lattice_batch_impl(const std::vector<StatisticSpec>& specs, bool inputs_on_device,
                                                long long n, LatticeMode mode, const Config& config, bool speculate);

StatisticResult lattice_statistic(const std::vector<const double*>& inputs, bool inputs_on_device,
                                  const std::vector<IndexTuple>& zero_sig, int m, long long n,
                                  LatticeMode mode, const Config& config);

std::vector<double> contract_host(const std::vector<const double*>& inputs, const std::vector<int>& orders,
                                  long long n, const EinsumNotation& notation, const EliminationOrder* order,
                                  const Config& config, DevStats* stats);

std::vector<double> eliminate_host(const std::vector<const double*>& inputs, const std::vector<IndexTuple>& tuples,
                                   long long n, int index, const Config& config, DevStats* stats,
                                   IndexTuple* result_tuple);

double combine_terms(const std::vector<double>& terms);

// hoif_tau's combination of the chain statistics u[2..m] (hoif.cpp:88-97):
// sum_j (-1)^j sum_l C(j-2, l) (n-l)!/n! u[l+2], accumulated in long double.
double hoif_combine(int m, long long n, const std::vector<double>& u);
// hoif_tau with the truncation basis phi(z) = z[0..k) on a sample [A, Y, Z...]
// (n x d, row-major, host or device): both component matrices tensorized on
// the device, the chain orders 2..m in one program.
StatisticResult hoif_tau_data(int m, int k, const double* data, long long n, int d, bool on_device,
                              const Config& config);

// Plan-only view of a statistic (no GPU): the optimized Program's ops and totals.
std::string plan_summary(const std::vector<IndexTuple>& zero_sig, int m, long long n, const Config& config,
                         bool inputs_symmetric, Program::Totals* totals);

}  // namespace ustats::dev
