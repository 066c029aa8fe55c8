// Device executor (see executor.hpp).
#include "executor.hpp"

#include <dlfcn.h>

#include <algorithm>
#include <bit>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>

#include "ustats/errors.hpp"
#include "ustats/partition.hpp"
#include "ustats/tensor.hpp"

namespace ustats::dev {

void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(ErrorCode::CudaError, std::string(what) + ": " + cudaGetErrorString(e));
}

// ---------------------------------------------------------------- Runtime
DeviceBuffer::~DeviceBuffer() {
    for (auto& r : ready) cudaEventDestroy(r.second);
    if (ptr && !borrowed && rt) {
        cudaFreeAsync(ptr, rt->stream());
        if (std::getenv("USTATS_SCHED_DEBUG") && entries() * 8 > (1ull << 30))
            std::fprintf(stderr, "[free] %.2f GiB\n", entries() * 8 / 1073741824.0);
    }
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
    check_cuda(cudaDeviceGetAttribute(&sm_count_, cudaDevAttrMultiProcessorCount, device), "cudaDeviceGetAttribute");
    // the main stream (GEMMs) outranks the side stream (reductions filling
    // the GEMM's tail): pending GEMM CTAs get freed SMs first
    int lo_prio = 0, hi_prio = 0;
    check_cuda(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio), "cudaDeviceGetStreamPriorityRange");
    check_cuda(cudaStreamCreateWithPriority(&stream_, cudaStreamNonBlocking, hi_prio), "cudaStreamCreate");
    check_cuda(cudaStreamCreateWithPriority(&side_, cudaStreamNonBlocking, lo_prio), "cudaStreamCreate");
    check_cuda(cudaStreamCreateWithFlags(&copy_, cudaStreamNonBlocking), "cudaStreamCreate");
    check_cuda(cudaStreamCreateWithPriority(&prep_, cudaStreamNonBlocking, hi_prio), "cudaStreamCreate");
    for (auto& c : chunk_) check_cuda(cudaStreamCreateWithPriority(&c, cudaStreamNonBlocking, hi_prio), "cudaStreamCreate");
    cur_ = stream_;
    refresh_free_bytes();
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        std::uint64_t keep = ~std::uint64_t{0};
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
}

Runtime::~Runtime() {}

void Runtime::refresh_free_bytes() {
    std::size_t free_b = 0, total_b = 0;
    check_cuda(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
    double pooled = 0;  // freed blocks our stream-ordered pool keeps for reuse
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device_) == cudaSuccess) {
        std::uint64_t reserved = 0, used = 0;
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
        pooled = static_cast<double>(reserved > used ? reserved - used : 0);
    }
    free_bytes_ = static_cast<double>(free_b) + pooled;
    agree_free_bytes();
}

Buf Runtime::allocate(int order, long long n) {
    auto b = std::make_shared<DeviceBuffer>();
    b->order = order;
    b->n = n;
    b->rt = this;
    void* p = nullptr;
    const std::size_t bytes = std::max<std::uint64_t>(b->entries(), 1) * sizeof(double);
    const cudaError_t e = cudaMallocAsync(&p, bytes, cur_);
    if (e != cudaSuccess || std::getenv("USTATS_SCHED_DEBUG")) {
        std::size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        if (e != cudaSuccess || bytes > (1ull << 30))
            std::fprintf(stderr, "[alloc] %.2f GiB -> %s (free %.2f / %.2f GiB)\n", bytes / 1073741824.0,
                         cudaGetErrorString(e), fr / 1073741824.0, tot / 1073741824.0);
    }
    check_cuda(e, "cudaMallocAsync");
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
    return b;
}

double* Runtime::scratch(std::size_t entries) {
    void* p = nullptr;
    check_cuda(cudaMallocAsync(&p, std::max<std::size_t>(entries, 1) * sizeof(double), cur_), "cudaMallocAsync");
    return static_cast<double*>(p);
}

void Runtime::release(double* p) {
    if (p) cudaFreeAsync(p, cur_);
}

void Runtime::sync() {
    for (auto& c : chunk_) check_cuda(cudaStreamSynchronize(c), "cudaStreamSynchronize");
    check_cuda(cudaStreamSynchronize(copy_), "cudaStreamSynchronize");
    check_cuda(cudaStreamSynchronize(prep_), "cudaStreamSynchronize");
    check_cuda(cudaStreamSynchronize(side_), "cudaStreamSynchronize");
    check_cuda(cudaStreamSynchronize(stream_), "cudaStreamSynchronize");
}

// ------------------------------------------------------------------- NCCL
namespace {
struct NcclApi {
    using GetId = int (*)(void*);
    using Init = int (*)(void**, int, std::array<char, 128>, int);
    using AllReduce = int (*)(const void*, void*, std::size_t, int, int, void*, cudaStream_t);
    using ErrStr = const char* (*)(int);
    GetId get_id = nullptr;
    Init init = nullptr;
    AllReduce all_reduce = nullptr;
    ErrStr err = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's copy (torch) if loaded
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) return;
        api.get_id = reinterpret_cast<NcclApi::GetId>(dlsym(h, "ncclGetUniqueId"));
        api.init = reinterpret_cast<NcclApi::Init>(dlsym(h, "ncclCommInitRank"));
        api.all_reduce = reinterpret_cast<NcclApi::AllReduce>(dlsym(h, "ncclAllReduce"));
        api.err = reinterpret_cast<NcclApi::ErrStr>(dlsym(h, "ncclGetErrorString"));
    });
    if (!api.get_id || !api.init || !api.all_reduce) fail(ErrorCode::CollectiveError, "libnccl.so.2 not available");
    return api;
}

void nccl_check(int r, const char* what) {
    if (r != 0)
        fail(ErrorCode::CollectiveError,
             std::string(what) + ": " + (nccl().err ? nccl().err(r) : ("nccl error " + std::to_string(r)).c_str()));
}
}  // namespace

void Runtime::nccl_unique_id(void* out128) { nccl_check(nccl().get_id(out128), "ncclGetUniqueId"); }

void Runtime::nccl_init(int rank, int world, const void* unique_id) {
    std::array<char, 128> id{};
    std::memcpy(id.data(), unique_id, 128);
    void* comm = nullptr;
    check_cuda(cudaSetDevice(device_), "cudaSetDevice");
    nccl_check(nccl().init(&comm, world, id, rank), "ncclCommInitRank");
    comm_ = comm;
    comm_world_ = world;
    agree_free_bytes();
}

// Row-sharded ranks must record identical programs (the same collectives in
// the same order), and the memory-bounded schedule depends on the budget:
// every rank plans with the smallest free memory of the communicator.
void Runtime::agree_free_bytes() {
    if (!comm_ || comm_world_ <= 1) return;
    constexpr int kNcclFloat64 = 8, kNcclMin = 3;  // nccl.h enum values
    double* d = nullptr;
    check_cuda(cudaMalloc(reinterpret_cast<void**>(&d), sizeof(double)), "cudaMalloc");
    check_cuda(cudaMemcpy(d, &free_bytes_, sizeof(double), cudaMemcpyHostToDevice), "H2D");
    nccl_check(nccl().all_reduce(d, d, 1, kNcclFloat64, kNcclMin, comm_, stream_), "ncclAllReduce(min)");
    check_cuda(cudaStreamSynchronize(stream_), "sync");
    check_cuda(cudaMemcpy(&free_bytes_, d, sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    cudaFree(d);
}

void Runtime::allreduce_sum(double* p, std::size_t count) {
    if (!comm_ || comm_world_ <= 1 || count == 0) return;
    constexpr int kNcclFloat64 = 8, kNcclSum = 0;  // nccl.h enum values
    nccl_check(nccl().all_reduce(p, p, count, kNcclFloat64, kNcclSum, comm_, cur_), "ncclAllReduce");
}

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
    cudaEventRecord(m.a, cur_);
    marks_.push_back(m);
}

void Runtime::end(Kind) {
    if (!profiling_ || marks_.empty()) return;
    cudaEventRecord(marks_.back().b, cur_);
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

// ----------------------------------------------------------------- helpers
namespace {
inline std::uint32_t bit(int id) { return 1u << id; }

std::vector<int> ids_of(std::uint32_t mask) {
    std::vector<int> v;
    for (std::uint32_t r = mask; r; r &= r - 1) v.push_back(std::countr_zero(r));
    return v;
}

std::uint64_t ipow(long long n, int e) {
    std::uint64_t v = 1;
    while (e-- > 0) v *= static_cast<std::uint64_t>(n);
    return v;
}

std::uint32_t ids_of_views(const std::vector<View>& vs) {
    std::uint32_t m = 0;
    for (const View& v : vs) m |= v.ids;
    return m;
}

// Every view an op reads (operands, stream factors, fused-epilogue weights).
template <class F>
void for_each_read(const Op& op, F&& f) {
    for (const View& v : op.factors) f(v);
    for (const View& v : op.fa) f(v);
    for (const View& v : op.fb) f(v);
    for (const Op::Epi& e : op.epis)
        for (const View& v : e.w) f(v);
}
}  // namespace

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

void Program::run_sweep(const Op& op) {
    SweepArgs a;
    a.x = ptr(op.factors[0].buf);
    a.xr = n_;
    a.cols = n_;
    a.r0 = 0;
    a.r1 = n_;
    if (slice_world_ > 1) {
        a.r0 = n_ * slice_rank_ / slice_world_;
        a.r1 = n_ * (slice_rank_ + 1) / slice_world_;
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

// Memory-bounded scheduling. Ops that allocate no tensor of order >= 2 run
// eagerly as soon as their inputs exist (they only free memory); the order in
// which the "big" producers (GEMM products, materialized Hadamard operands)
// run is searched depth-first, cheapest resulting live set first, pruning any
// branch whose peak (inputs + live intermediates) exceeds the budget. Shared
// sub-contractions make the naive recording order hold many n^2 products at
// once (C5: 412 GB); the search finds orders that fit one B200.
void Program::make_schedule(double budget) {
    const std::size_t N = ops_.size();
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
        st.peak = std::max(st.peak, st.live);
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
}

void Program::optimize(double budget_bytes) {
    budget_ = budget_bytes;
    if (config_.device.fuse_epilogues) fuse_epilogues();
    make_schedule(budget_bytes);
    if (config_.device.fuse_epilogues) {
        // sweeps tie their consumers' operands together; keep them only if
        // the memory-bounded schedule stays well inside the budget or does
        // not get a higher peak (C5 at n = 65536 reverts, C3/C4 keep them)
        const std::vector<Op> before = ops_;
        const std::vector<std::size_t> sched = schedule_;
        const double peak = sched_peak_;
        const std::uint64_t fused = stats_ ? stats_->fused_epilogues : 0;
        fuse_sweeps();
        if (ops_.size() != before.size()) {
            make_schedule(budget_bytes);
            const double roomy = 0.6 * (budget_bytes > 0 ? budget_bytes : 179.0 * 1073741824.0);
            if (sched_peak_ > std::max(peak * 1.0001 + 1.0, roomy)) {
                ops_ = before;
                schedule_ = sched;
                sched_peak_ = peak;
                if (stats_) stats_->fused_epilogues = fused;
            }
        }
    }
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
            const long long lo = n_ * slice_rank_ / slice_world_, hi = n_ * (slice_rank_ + 1) / slice_world_;
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
    const bool multi_path = !op.epis.empty() || (op.symmetric_out && gemm_tma_eligible(g, nullptr, nullptr));
    if (slice_world_ > 1) {
        // row sharding: a contiguous range of the tile list per rank
        const bool tri = multi_path && op.symmetric_out && g.rows == g.cols;
        const long long total = gemm_tile_total(g, tri);
        g.tile_begin = total * slice_rank_ / slice_world_;
        g.tile_count = total * (slice_rank_ + 1) / slice_world_ - g.tile_begin;
        g.accumulate = 1;
        if (g.tile_count <= 0) return;
    }
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
        const bool chunked = slice_world_ == 1 && op.symmetric_out && g.rows == g.cols && fa[0].buf == fb[0].buf &&
                             src && src->ready.size() > 1;
        rt_->begin(Runtime::kGemm);
        if (!chunked) {
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
    } else {
        g.symmetric_out = 0;
        rt_->begin(Runtime::kGemm);
        launched = launch_gemm(g, rt_->stream());
        rt_->end(Runtime::kGemm);
    }
    check_cuda(cudaGetLastError(), "gemm launch");
    rt_->release(scratch);
    if (stats_) {
        const bool tri = op.symmetric_out && g.rows == g.cols && gemm_tma_eligible(g, nullptr, nullptr);
        const long long tm = (g.rows + 127) / 128;
        const std::uint64_t full = static_cast<std::uint64_t>(g.rows) * static_cast<std::uint64_t>(g.cols) *
                                   static_cast<std::uint64_t>(n_);
        std::uint64_t macs = tri ? full / static_cast<std::uint64_t>(tm * tm) *
                                       static_cast<std::uint64_t>(tm * (tm + 1) / 2)
                                 : full;
        if (slice_world_ > 1 && g.tile_count >= 0) {
            const long long total = gemm_tile_total(g, tri);
            macs = static_cast<std::uint64_t>(static_cast<double>(macs) * static_cast<double>(g.tile_count) /
                                              static_cast<double>(total));
        }
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
    if (op.gemm) run_gemm(op, out);
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
        // Row sharding: each op runs as a slice per rank into zeroed outputs;
        // with NCCL one all-reduce per materialized output completes it, in
        // emulation the virtual ranks' slices accumulate on this device.
        const bool collective = !emulate && rt_->has_comm();
        if (!emulate && !collective) fail(ErrorCode::CollectiveError, "row sharding needs us_nccl_init first");
        rt_->set_stream(rt_->main_stream());
        for (const SymBuf& b : bufs_)
            if (b.input && b.real && !b.real->ready.empty())
                check_cuda(cudaStreamWaitEvent(rt_->main_stream(), b.real->ready.back().second, 0), "wait upload");
        slice_world_ = world;
        for (std::size_t pos = 0; pos < schedule_.size(); ++pos) {
            Op& op = ops_[schedule_[pos]];
            for (int r = (emulate ? 0 : dc.rank); r < (emulate ? world : dc.rank + 1); ++r) {
                slice_rank_ = r;
                launch(op);
            }
            if (collective) {
                auto reduce = [&](int b) {
                    SymBuf& sb = bufs_[static_cast<std::size_t>(b)];
                    if (sb.real) rt_->allreduce_sum(sb.real->ptr, sb.real->entries());
                };
                if (!op.ext && op.out >= 0 && (!op.gemm || op.store)) reduce(op.out);
                for (const Op::Epi& e : op.epis)
                    if (!e.ext && e.out >= 0) reduce(e.out);
            }
            for_each_read(op, [&](const View& v) {
                SymBuf& b = bufs_[static_cast<std::size_t>(v.buf)];
                if (!b.input && b.last_use == static_cast<int>(pos) && b.real && b.real.use_count() == 1 &&
                    !keep_.count(v.buf))
                    b.real.reset();
            });
        }
        slice_world_ = 1;
        slice_rank_ = 0;
        return;
    }
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
    cudaStream_t streams[2] = {rt_->main_stream(), rt_->side_stream()};
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
    const DeviceConfig& d = c.device;
    std::string k = std::to_string(n) + "|" + std::to_string(static_cast<int>(mode)) + "|" +
                    std::to_string(static_cast<long long>(budget / 8.589934592e9)) + "|" +
                    std::to_string(c.memory_cap_entries) + "," + std::to_string(static_cast<int>(c.strategy)) + "," +
                    std::to_string(c.exhaustive_index_bound) + "," + std::to_string(c.exact_treewidth_bound) + "|" +
                    std::to_string(d.share_subexpressions) + std::to_string(d.fuse_epilogues) +
                    std::to_string(d.exploit_symmetry) + std::to_string(d.reorder_for_sharing) +
                    std::to_string(d.serial_launch) + std::to_string(d.shard_rows) + "," + std::to_string(d.rank) + "," +
                    std::to_string(d.world_size) + "," + std::to_string(d.emulate_world) + "," +
                    std::to_string(d.memory_budget_bytes) + "|";
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
    }
    PlanEntry* raw = e.get();
    pc.entries[key] = std::move(e);
    return raw;
}

}  // namespace

std::vector<StatisticResult> lattice_batch(const std::vector<StatisticSpec>& specs, bool inputs_on_device,
                                           long long n, LatticeMode mode, const Config& config) {
    return lattice_batch_impl(specs, inputs_on_device, n, mode, config, true);
}

std::vector<StatisticResult> lattice_batch_impl(const std::vector<StatisticSpec>& specs, bool inputs_on_device,
                                                long long n, LatticeMode mode, const Config& config, bool speculate) {
    std::vector<StatisticResult> out(specs.size());
    Runtime& rt = Runtime::get(config.device.device);
    {
        // re-measure free memory only when this call's footprint is a large
        // share of the device (n^2 matrices of several GiB)
        const double n2 = 8.0 * static_cast<double>(n) * static_cast<double>(n);
        if (n2 * 6 > 0.5 * rt.free_bytes()) rt.refresh_free_bytes();
    }
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
    if (config.device.exploit_symmetry)
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
            if (mode == LatticeMode::Sparsified && !panels)
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
    double budget = static_cast<double>(config.device.memory_budget_bytes);
    if (budget <= 0) budget = 0.94 * rt.free_bytes() - 2.0e9;  // inputs included: they came out of it
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
    if (T) check_cuda(cudaMemcpyAsync(v.data(), d_v, sizeof(double) * T, cudaMemcpyDeviceToHost, rt.stream()), "D2H");
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
    rt.sync();
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
    return head + prog.dump();
}

}  // namespace ustats::dev
