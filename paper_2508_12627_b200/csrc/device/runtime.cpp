// Device runtime (executor.hpp): streams, stream-ordered allocation, the
// NCCL communicator for row sharding, event profiling.
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

void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(ErrorCode::CudaError, std::string(what) + ": " + cudaGetErrorString(e));
}

// ---------------------------------------------------------------- Runtime
DeviceBuffer::~DeviceBuffer() {
    for (auto& r : ready) cudaEventDestroy(r.second);
    if (ptr && !borrowed && rt) {
        if (std::getenv("USTATS_SCHED_DEBUG") && entries() * 8 > (1ull << 30))
            std::fprintf(stderr, "[free] %.2f GiB\n", entries() * 8 / 1073741824.0);
        rt->raw_free(ptr, std::max<std::uint64_t>(entries(), 1) * sizeof(double));
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

Runtime::~Runtime() {}  // process teardown: the driver reclaims device memory

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
    free_bytes_ = static_cast<double>(free_b) + pooled + idle_slab_bytes();
    agree_free_bytes();
}

Buf Runtime::allocate(int order, long long n) {
    auto b = std::make_shared<DeviceBuffer>();
    b->order = order;
    b->n = n;
    b->rt = this;
    const std::size_t bytes = std::max<std::uint64_t>(b->entries(), 1) * sizeof(double);
    b->ptr = static_cast<double*>(raw_alloc(bytes));
    b->slab = bytes >= kSlabMin;
    return b;
}

void* Runtime::slab_get(std::size_t bytes) {
    for (std::size_t i = 0; i < idle_.size(); ++i)
        if (idle_[i].bytes == bytes) {
            Slab s = idle_[i];
            idle_.erase(idle_.begin() + static_cast<std::ptrdiff_t>(i));
            check_cuda(cudaStreamWaitEvent(cur_, s.freed, 0), "wait slab release");
            cudaEventDestroy(s.freed);
            return s.ptr;
        }
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
        cudaGetLastError();  // the allocation error only
        return nullptr;
    }
    return p;
}

void Runtime::slab_put(void* p, std::size_t bytes) {
    Slab s{p, bytes, nullptr};
    if (cudaEventCreateWithFlags(&s.freed, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventRecord(s.freed, cur_) != cudaSuccess) {
        cudaGetLastError();
        cudaStreamSynchronize(cur_);
        if (s.freed) cudaEventDestroy(s.freed);
        cudaFree(p);
        return;
    }
    idle_.push_back(s);
}

double Runtime::idle_slab_bytes() const {
    double t = 0;
    for (const Slab& s : idle_) t += static_cast<double>(s.bytes);
    return t;
}

void Runtime::reclaim() {
    wait_streams();  // this runtime's streams only: every pending user of an idle slab has finished
    for (Slab& s : idle_) {
        cudaEventDestroy(s.freed);
        cudaFree(s.ptr);
    }
    idle_.clear();
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device_) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
}

void* Runtime::raw_alloc(std::size_t bytes, bool slab_ok) {
    bytes = std::max<std::size_t>(bytes, 8);
    auto attempt = [&]() -> void* {
        if (slab_ok && bytes >= kSlabMin) return slab_get(bytes);
        void* p = nullptr;
        const cudaError_t e = cudaMallocAsync(&p, bytes, cur_);
        if (e == cudaErrorMemoryAllocation) {
            cudaGetLastError();  // clears exactly this allocation error
            return nullptr;
        }
        check_cuda(e, "cudaMallocAsync");
        return p;
    };
    void* p = attempt();
    if (!p) {
        reclaim();
        p = attempt();
    }
    if (!p || std::getenv("USTATS_SCHED_DEBUG")) {
        std::size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        if (!p || bytes > (1ull << 30))
            std::fprintf(stderr, "[alloc] %.2f GiB -> %s (free %.2f / %.2f GiB)\n", bytes / 1073741824.0,
                         p ? "ok" : "out of memory", fr / 1073741824.0, tot / 1073741824.0);
    }
    if (!p)
        fail(ErrorCode::MemoryCapExceeded, "device allocation of " + std::to_string(bytes) +
                                               " bytes failed after reclaiming idle memory (the memory-bounded "
                                               "schedule exceeded the device)");
    return p;
}

void Runtime::raw_free(void* p, std::size_t bytes) {
    if (!p) return;
    if (std::max<std::size_t>(bytes, 8) >= kSlabMin) slab_put(p, std::max<std::size_t>(bytes, 8));
    else cudaFreeAsync(p, cur_);
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
    return static_cast<double*>(raw_alloc(std::max<std::size_t>(entries, 1) * sizeof(double), false));
}

void Runtime::release(double* p) {
    if (p) cudaFreeAsync(p, cur_);
}

void Runtime::sync() {
    wait_streams();
    used_ = 0;  // the evaluation is over: the next one notes its own streams
}

void Runtime::wait_streams() {
    const unsigned used = used_;
    if (used & 8)
        for (auto& c : chunk_) check_cuda(cudaStreamSynchronize(c), "cudaStreamSynchronize");
    if (used & 2) check_cuda(cudaStreamSynchronize(copy_), "cudaStreamSynchronize");
    if (used & 4) check_cuda(cudaStreamSynchronize(prep_), "cudaStreamSynchronize");
    if (used & 1) check_cuda(cudaStreamSynchronize(side_), "cudaStreamSynchronize");
    check_cuda(cudaStreamSynchronize(stream_), "cudaStreamSynchronize");
}

// ------------------------------------------------------------------- NCCL
namespace {
struct NcclApi {
    using GetId = int (*)(void*);
    using Init = int (*)(void**, int, std::array<char, 128>, int);
    using AllReduce = int (*)(const void*, void*, std::size_t, int, int, void*, cudaStream_t);
    using ErrStr = const char* (*)(int);
    using Bcast = int (*)(const void*, void*, std::size_t, int, int, void*, cudaStream_t);
    using P2POp = int (*)(const void*, std::size_t, int, int, void*, cudaStream_t);  // ncclSend / ncclRecv
    using Group = int (*)();
    GetId get_id = nullptr;
    Init init = nullptr;
    AllReduce all_reduce = nullptr;
    ErrStr err = nullptr;
    Bcast bcast = nullptr;
    P2POp send = nullptr, recv = nullptr;
    Group group_start = nullptr, group_end = nullptr;
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
        api.bcast = reinterpret_cast<NcclApi::Bcast>(dlsym(h, "ncclBroadcast"));
        api.send = reinterpret_cast<NcclApi::P2POp>(dlsym(h, "ncclSend"));
        api.recv = reinterpret_cast<NcclApi::P2POp>(dlsym(h, "ncclRecv"));
        api.group_start = reinterpret_cast<NcclApi::Group>(dlsym(h, "ncclGroupStart"));
        api.group_end = reinterpret_cast<NcclApi::Group>(dlsym(h, "ncclGroupEnd"));
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

// Row slabs [off_r, off_r + len_r) of every rank to every rank, in place:
// one broadcast per rank inside one NCCL group (slabs may differ in size).
void Runtime::allgather_rows(double* p, const std::vector<std::pair<long long, long long>>& slabs) {
    if (!comm_ || comm_world_ <= 1) return;
    const NcclApi& api = nccl();
    if (!api.bcast || !api.group_start || !api.group_end) fail(ErrorCode::CollectiveError, "ncclBroadcast not available");
    constexpr int kNcclFloat64 = 8;
    nccl_check(api.group_start(), "ncclGroupStart");
    for (std::size_t r = 0; r < slabs.size(); ++r)
        if (slabs[r].second > 0)
            nccl_check(api.bcast(p + slabs[r].first, p + slabs[r].first, static_cast<std::size_t>(slabs[r].second),
                                 kNcclFloat64, static_cast<int>(r), comm_, cur_),
                       "ncclBroadcast");
    nccl_check(api.group_end(), "ncclGroupEnd");
}

void Runtime::sendrecv(const std::vector<P2P>& ops) {
    if (!comm_ || comm_world_ <= 1 || ops.empty()) return;
    const NcclApi& api = nccl();
    if (!api.send || !api.recv || !api.group_start || !api.group_end)
        fail(ErrorCode::CollectiveError, "ncclSend / ncclRecv not available");
    constexpr int kNcclFloat64 = 8;
    nccl_check(api.group_start(), "ncclGroupStart");
    for (const P2P& o : ops)
        nccl_check((o.send ? api.send : api.recv)(o.buf, o.count, kNcclFloat64, o.peer, comm_, cur_),
                   o.send ? "ncclSend" : "ncclRecv");
    nccl_check(api.group_end(), "ncclGroupEnd");
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

}  // namespace ustats::dev
