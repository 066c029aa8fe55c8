// Statistic entry points (proj/include/ustats/engine.hpp:17-65). Tensorization
// runs on the host (caller callbacks); sparsification, the V-term contractions
// and their reduction run on the B200; the Möbius combination runs on the host
// in enumeration order (bit-for-bit the reference's pairwise tree).
#pragma once

#include <cstdint>
#include <vector>

#include "ustats/config.hpp"
#include "ustats/einsum.hpp"
#include "ustats/kernel.hpp"
#include "ustats/partition.hpp"
#include "ustats/tensor.hpp"

// the public C++ API is exported from libustats_b200.so (built -fvisibility=hidden)
#pragma GCC visibility push(default)
namespace ustats {

struct RunStats {
    double tensorize_seconds = 0.0;
    double contract_seconds = 0.0;
    std::uint64_t einsum_calls = 0;
    std::uint64_t partitions_enumerated = 0;
    std::uint64_t partitions_evaluated = 0;
    std::uint64_t multiply_adds = 0;              ///< reference-plan count
    std::uint64_t peak_intermediate_entries = 0;
    // B200 additions
    std::uint64_t executed_gemm_macs = 0;         ///< DMMA multiply-adds actually issued
    std::uint64_t executed_stream_entries = 0;    ///< factor entries read by bandwidth kernels
    std::uint64_t gemm_launches = 0;
    std::uint64_t stream_launches = 0;
    std::uint64_t shared_hits = 0;                ///< sub-contractions reused across V-terms
};

std::vector<DenseTensor> tensorize(const MDKernel& kernel, const Sample& sample,
                                   const Config& config = {}, RunStats* stats = nullptr);
double v_statistic(const MDKernel& kernel, const Sample& sample, const Config& config = {},
                   RunStats* stats = nullptr);
double restricted_v(const MDKernel& kernel, const Sample& sample, const SetPartition& partition,
                    const Config& config = {}, RunStats* stats = nullptr);
double u_statistic(const MDKernel& kernel, const Sample& sample, const Config& config = {},
                   RunStats* stats = nullptr);
double u_statistic_unsparsified(const MDKernel& kernel, const Sample& sample,
                                const Config& config = {}, RunStats* stats = nullptr);

/// Tensor-level U-statistic (engine.cpp:182-192 after tensorize): `tensors[k]`
/// is component k materialized over [0,n)^|sig[k]| (unsparsified), `zero_sig`
/// the 0-based signature. Optional `terms` receives mu*V per survivor in
/// enumeration order (only this rank's terms are non-zero when sharded).
double u_statistic_tensors(std::span<const DenseTensor> tensors,
                           const std::vector<IndexTuple>& zero_sig, int arity,
                           const Config& config = {}, RunStats* stats = nullptr,
                           std::vector<double>* terms = nullptr);

}  // namespace ustats
#pragma GCC visibility pop
