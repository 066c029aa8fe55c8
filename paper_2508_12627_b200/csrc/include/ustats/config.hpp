// Engine knobs. The host fields mirror the reference Config
// (proj/include/ustats/config.hpp:17-44) field for field; `device` is the
// B200 section (which GPU, how the V-terms are shared across ranks, and which
// plan rewrites are enabled).
#pragma once

#include <cstdint>

// the public C++ API is exported from libustats_b200.so (built -fvisibility=hidden)
#pragma GCC visibility push(default)
namespace ustats {

enum class OrderStrategy { Auto, GreedyMinDegree, GreedyMinFill, Exhaustive };

struct DeviceConfig {
    int device = -1;               ///< CUDA device ordinal; -1 = current device
    int rank = 0;                  ///< this process's share of the V-terms (term sharding)
    int world_size = 1;            ///< number of ranks the V-terms are spread over
    bool share_subexpressions = true;  ///< hash-cons identical GEMMs/reductions across V-terms
    bool fuse_epilogues = true;        ///< fold+marginalize consumers into GEMM epilogues
    bool exploit_symmetry = true;      ///< detect bitwise-symmetric matrices, read either orientation
    bool reorder_for_sharing = true;   ///< choose among equal-width orders to maximize sharing
    bool donate_inputs = false;        ///< device inputs may be sparsified in place (no copy)
    bool serial_launch = false;        ///< one stream only (no GEMM/reduction overlap)
    /// Large FP64 GEMMs (K <= 19000) run as Ozaki digit splitting on the INT8
    /// tcgen05 tensor cores (7 digits: ~1e-12 relative to the row-scale
    /// product) instead of DMMA; false = DMMA everywhere.
    bool fp64_emulation = true;
    /// Multi-GPU scheme: false = V-terms sharded over ranks (LPT, one all-reduce
    /// of the term vector); true = every op row-sharded over ranks (GEMM tile
    /// ranges / leading-index slices, one all-reduce per materialized output).
    bool shard_rows = false;
    /// Row sharding over `emulate_world` virtual ranks on this one device, op
    /// by op in lockstep (tests the decomposition without NCCL). 0 = off.
    int emulate_world = 0;
    /// Device-memory budget for inputs + live intermediates of one statistic's
    /// program (0 = free device memory at execution; plan-only: 179 GiB).
    std::uint64_t memory_budget_bytes = 0;
    /// Digit slices of the emulated FP64 GEMM (0 = the error-bound guard's
    /// choice, see gemm_ozaki.cu / DESIGN.md 2.3a; 4..7 forces a count).
    int oz_slices = 0;
    /// Longest K an emulated GEMM runs in one pass (0 = the int32-exact bound,
    /// 21000); longer K runs as equal K chunks summed in FP64 (tests lower it
    /// to exercise the chunked path at small n).
    long long oz_max_k = 0;
    /// Smallest rows / cols / K of a GEMM that runs emulated (0 = 1024: below,
    /// DMMA is as fast and needs no digit pass). Tests lower it so the emulated
    /// and lazy-operand paths run at sizes the CPU reference reaches.
    int oz_min_dim = 0;
    /// Replay repeated small data-API evaluations (same spec, shape, buffers
    /// and config, n <= 4096) as one captured CUDA graph.
    bool graph_replay = true;
};

struct Config {
    std::uint64_t memory_cap_entries = std::uint64_t{1} << 31;
    int threads = 0;
    OrderStrategy strategy = OrderStrategy::Auto;
    int exhaustive_index_bound = 12;
    int exact_treewidth_bound = 10;
    std::uint64_t brute_force_term_cap = 10'000'000;
    bool strict_nonfinite = false;
    DeviceConfig device;

    int effective_threads() const;
};

}  // namespace ustats
#pragma GCC visibility pop
