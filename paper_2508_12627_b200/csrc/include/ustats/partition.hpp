// Set-partition lattice of the slots {0..m-1}: restricted-growth streaming,
// Möbius weights and the sparsification survivor filter. Host-side planning;
// semantics follow proj/include/ustats/partition.hpp:14-121.
#pragma once

#include <cstdint>
#include <vector>

#include "ustats/notation.hpp"

// the public C++ API is exported from libustats_b200.so (built -fvisibility=hidden)
#pragma GCC visibility push(default)
namespace ustats {

class SetPartition {
  public:
    SetPartition() = default;
    explicit SetPartition(std::vector<int> rgs);
    static SetPartition finest(int m);
    static SetPartition coarsest(int m);
    static SetPartition from_blocks(int m, const std::vector<std::vector<int>>& blocks);

    int ground_size() const { return static_cast<int>(rgs_.size()); }
    int block_count() const { return blocks_; }
    int block_of(int element) const { return rgs_[element]; }
    const std::vector<int>& rgs() const { return rgs_; }
    std::vector<std::vector<int>> blocks() const;
    bool operator==(const SetPartition& other) const { return rgs_ == other.rgs_; }

  private:
    std::vector<int> rgs_;
    int blocks_ = 0;
};

/// Lexicographic restricted-growth order, coarsest (00..0) first, finest last.
class PartitionStream {
  public:
    explicit PartitionStream(int m);
    bool next(SetPartition& out);
    std::size_t next_chunk(std::vector<SetPartition>& chunk, std::size_t max_count);

  private:
    std::vector<int> word_;
    bool started_ = false;
    bool done_ = false;
};

std::uint64_t bell_number(int m);
std::int64_t mobius_coefficient(const SetPartition& partition);
bool is_refinement(const SetPartition& fine, const SetPartition& coarse);
std::int64_t mobius_pair(const SetPartition& fine, const SetPartition& coarse);
bool passes_sparsification(const SetPartition& partition, const std::vector<IndexTuple>& signature);

class SparsifiedPartitionStream {
  public:
    SparsifiedPartitionStream(int m, const std::vector<IndexTuple>& signature);
    bool next(SetPartition& out);
    std::size_t next_chunk(std::vector<SetPartition>& chunk, std::size_t max_count);
    std::uint64_t enumerated() const { return enumerated_; }

  private:
    PartitionStream all_;
    std::vector<std::uint32_t> clash_;  // clash_[a]: bitmask of b>a that co-occur with a
    std::uint64_t enumerated_ = 0;
};

std::vector<IndexTuple> induced_signature(const std::vector<IndexTuple>& signature,
                                          const SetPartition& partition);

}  // namespace ustats
#pragma GCC visibility pop
