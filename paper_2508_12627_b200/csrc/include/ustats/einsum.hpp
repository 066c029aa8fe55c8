// Tensor-level contraction on the B200 (proj/include/ustats/einsum.hpp:13-52).
// The notation is planned on the host (same elimination sequence as the
// reference) and executed by the device executor's kernels; results return
// to the host as DenseTensor.
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "ustats/config.hpp"
#include "ustats/notation.hpp"
#include "ustats/ordering.hpp"
#include "ustats/tensor.hpp"

// the public C++ API is exported from libustats_b200.so (built -fvisibility=hidden)
#pragma GCC visibility push(default)
namespace ustats {

struct ExecStats {
    std::uint64_t multiply_adds = 0;             ///< reference-plan counting rules
    std::uint64_t peak_intermediate_entries = 0;
    int steps = 0;
};

DenseTensor einsum(std::span<const DenseTensor> tensors, const EinsumNotation& notation,
                   const Config& config = {}, const EliminationOrder* order = nullptr,
                   ExecStats* stats = nullptr);

std::pair<DenseTensor, IndexTuple> eliminate_index(std::span<const DenseTensor> tensors,
                                                   const std::vector<IndexTuple>& tuples,
                                                   int index, const Config& config = {},
                                                   ExecStats* stats = nullptr);

}  // namespace ustats
#pragma GCC visibility pop
