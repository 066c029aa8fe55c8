// Einsum notation: canonical (first-appearance) index ids, duplicate-free
// output. Semantics follow proj/include/ustats/notation.hpp:12-36.
#pragma once

#include <string>
#include <vector>

// the public C++ API is exported from libustats_b200.so (built -fvisibility=hidden)
#pragma GCC visibility push(default)
namespace ustats {

using IndexTuple = std::vector<int>;

struct EinsumNotation {
    std::vector<IndexTuple> inputs;
    IndexTuple output;
    int index_count = 0;

    EinsumNotation() = default;
    EinsumNotation(std::vector<IndexTuple> raw_inputs, IndexTuple raw_output = {});

    bool index_in_output(int index) const;
    std::string to_string() const;
};

EinsumNotation validate_notation(const std::vector<IndexTuple>& raw_inputs,
                                 const IndexTuple& raw_output = {});

}  // namespace ustats
#pragma GCC visibility pop
