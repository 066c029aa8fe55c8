// Multiplicatively decomposable kernels (proj/include/ustats/kernel.hpp:14-57).
#pragma once

#include <functional>
#include <span>
#include <string>
#include <vector>

#include "ustats/notation.hpp"

// the public C++ API is exported from libustats_b200.so (built -fvisibility=hidden)
#pragma GCC visibility push(default)
namespace ustats {

using Observation = std::vector<double>;

struct Sample {
    std::vector<Observation> points;
    Sample() = default;
    explicit Sample(std::vector<Observation> pts) : points(std::move(pts)) {}
    static Sample indices_only(int n) { return Sample(std::vector<Observation>(n)); }
    int size() const { return static_cast<int>(points.size()); }
};

using ComponentFn = std::function<double(const Sample&, std::span<const int>)>;

struct MDKernel {
    int arity = 0;
    std::vector<IndexTuple> signature;  ///< 1-based slots
    std::vector<ComponentFn> components;
    std::string name;

    void validate() const;
    std::vector<IndexTuple> zero_based_signature() const;
    double evaluate(const Sample& sample, std::span<const int> indices) const;
};

MDKernel prod2_kernel();

}  // namespace ustats
#pragma GCC visibility pop
