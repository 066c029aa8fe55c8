// Device executor: runs one einsum notation over device-resident tensors with
// the reference's elimination semantics (proj/src/einsum.cpp:310-486) lowered
// to two kernel families:
//   * lazy Hadamard folds — a fold (fold_into, einsum.cpp:134-147) just
//     appends a factor view to the target slot; nothing is materialized;
//   * a "stream" kernel for every marginalization / generic step / assembly
//     (the lazy product is formed on the fly while reducing);
//   * the DMMA GEMM for two-operand steps and for K-way steps whose operands
//     only share the eliminated index (Khatri-Rao rows).
// Reference-rule counters (ExecStats semantics) are tallied symbolically along
// the same walk so RunStats.multiply_adds matches the reference plan, while
// executed DMMA MACs and streamed entries are tallied separately.
#pragma once

#include <array>
#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include <cuda_runtime.h>

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
    bool symmetric = false;  // order 2 and bitwise equal to its transpose
    bool borrowed = false;   // caller memory: never freed, never written
    Runtime* rt = nullptr;
    std::uint64_t uid = 0;   // stable identity for cross-term sharing keys
    ~DeviceBuffer();
    std::uint64_t entries() const;
};
using Buf = std::shared_ptr<DeviceBuffer>;

class Runtime {
  public:
    static Runtime& get(int device);  // -1: current device
    ~Runtime();

    cudaStream_t stream() const { return stream_; }
    int device() const { return device_; }
    int sm_count() const { return sm_count_; }

    Buf allocate(int order, long long n);
    Buf borrow(const double* ptr, int order, long long n);
    double* scratch(std::size_t entries);
    void release(double* p);
    void sync();

    // Kernel-class timing with CUDA events on the engine stream (bench
    // roofline evidence). Cheap: two event records per timed launch group.
    enum Kind { kGemm = 0, kStream = 1, kOther = 2 };
    struct Profile {
        double ms[3] = {0, 0, 0};
        std::uint64_t groups[3] = {0, 0, 0};
    };
    void profile_enable(bool on) { profiling_ = on; }
    void begin(Kind k);
    void end(Kind k);
    Profile collect(bool reset);  // synchronizes the stream

  private:
    explicit Runtime(int device);
    int device_ = 0;
    int sm_count_ = 148;
    cudaStream_t stream_ = nullptr;
    std::uint64_t next_uid_ = 1;
    bool profiling_ = false;
    std::vector<cudaEvent_t> pool_;
    struct Mark {
        Kind kind;
        cudaEvent_t a, b;
    };
    std::vector<Mark> marks_;
    Profile totals_;
    friend struct DeviceBuffer;
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
};

// Content-addressed cache of intermediates shared across V-terms of one
// statistic evaluation (reference: SPEC.md:469 — no deduplication).
class ShareCache {
  public:
    Buf find(const std::string& key) const {
        auto it = map_.find(key);
        return it == map_.end() ? nullptr : it->second;
    }
    void put(const std::string& key, Buf b) { map_[key] = std::move(b); }
    void clear() { map_.clear(); }

  private:
    std::map<std::string, Buf> map_;
};

class Contractor {
  public:
    Contractor(Runtime& rt, long long n, const Config& config, DevStats* stats,
               ShareCache* cache = nullptr)
        : rt_(rt), n_(n), config_(config), stats_(stats), cache_(cache) {}

    // Full einsum. Returns the output buffer (order |output|); when
    // `scalar_out` is given and the output is a scalar, writes it there
    // (device pointer) and returns null.
    Buf run(const std::vector<Buf>& inputs, const EinsumNotation& notation,
            const EliminationOrder& order, double* scalar_out = nullptr);

    // One elimination step in isolation (einsum.hpp:49-52); result ids ascending.
    Buf eliminate_single(const std::vector<Buf>& inputs, const std::vector<IndexTuple>& tuples,
                         int index, IndexTuple* result_tuple);

    struct View {
        Buf buf;
        std::array<long long, kMaxIds> stride{};
        std::uint32_t ids = 0;
    };
    struct Slot {
        std::uint32_t ids = 0;
        std::vector<View> factors;
        bool owned = false;
        IndexTuple tuple;  // the reference's tuple order (for counting only)
    };

  private:
    View view_of(const Buf& b, const IndexTuple& tuple) const;
    Slot slot_of(const Buf& b, const IndexTuple& tuple);
    void eliminate_one(std::vector<Slot>& slots, int e);
    Slot marginalize(const Slot& s, std::uint32_t summed);
    Slot gemm_step(const Slot& a, const Slot& b, int e);
    Slot generic_step(const std::vector<Slot>& parts, int e);

    // Kernel-level primitives
    Buf stream_to_buffer(std::vector<View> factors, const std::vector<int>& out_ids,
                         std::uint32_t sum_ids, double* out_ptr);
    Buf gemm_to_buffer(std::vector<View> fa, std::vector<View> fb, const std::vector<int>& ra,
                       const std::vector<int>& rb, int e);
    std::vector<View> limit_factors(std::vector<View> fs, std::size_t limit);
    View output_view(const Buf& b, const std::vector<int>& ids_in_layout) const;

    void ref_count_alloc(int order);  // cap check on a reference-plan intermediate
    void ref_owned(int order);        // peak bookkeeping (make_owned)
    std::uint64_t pw(int e) const;

    Runtime& rt_;
    long long n_;
    const Config& config_;
    DevStats* stats_;
    ShareCache* cache_;
};

// Device-side U/V statistic drivers over tensor inputs (host or device memory).
struct StatisticResult {
    double value = 0.0;
    std::vector<double> terms;          // mu * V per evaluated partition (enumeration order)
    std::vector<std::vector<int>> rgs;  // the partitions
    std::vector<long long> mu;
    std::vector<double> v;              // raw V per partition (0 for terms owned by other ranks)
    std::vector<int> owner;             // rank that evaluated each term
    DevStats stats;
    std::uint64_t enumerated = 0;
    double upload_seconds = 0.0;
    double contract_seconds = 0.0;
};

enum class LatticeMode { Sparsified, Unsparsified };

// Host-only planning of one statistic: the evaluated partitions in
// enumeration order, their induced notations and elimination orders, and the
// LPT assignment of terms to ranks (term sharding; no GPU needed).
struct TermPlan {
    std::vector<std::vector<int>> rgs;
    std::vector<long long> mu;
    std::vector<EinsumNotation> notation;
    std::vector<EliminationOrder> order;
    std::vector<double> cost;   // relative work estimate (n^(width+1) per term)
    std::vector<int> owner;
    std::uint64_t enumerated = 0;
};
TermPlan plan_terms(const std::vector<IndexTuple>& zero_sig, int m, long long n, LatticeMode mode,
                    const Config& config);

// `inputs[k]` points at factor k (row-major, n^|sig[k]| entries) in host memory
// (inputs_on_device = false) or device memory. Aliased pointers are uploaded
// and sparsified once.
StatisticResult lattice_statistic(const std::vector<const double*>& inputs, bool inputs_on_device,
                                  const std::vector<IndexTuple>& zero_sig, int m, long long n,
                                  LatticeMode mode, const Config& config);

// Single contraction (v_statistic / restricted_v / einsum) over host tensors.
std::vector<double> contract_host(const std::vector<const double*>& inputs,
                                  const std::vector<int>& orders, long long n,
                                  const EinsumNotation& notation, const EliminationOrder* order,
                                  const Config& config, DevStats* stats);

}  // namespace ustats::dev
