// Errors, config, notation, tensor and kernel basics of the host layer.
// Behaviour mirrors proj/src/{errors,config,notation,tensor,kernel}.cpp.
#include <algorithm>
#include <cmath>
#include <thread>
#include <unordered_map>

#include "ustats/config.hpp"
#include "ustats/errors.hpp"
#include "ustats/kernel.hpp"
#include "ustats/notation.hpp"
#include "ustats/tensor.hpp"

namespace ustats {

// ---------------------------------------------------------------- errors
const char* error_code_name(ErrorCode code) {
    static const char* const names[] = {
        "InvalidNotation",   "InvalidOutput",      "ShapeMismatch",
        "MemoryCapExceeded", "IndexAbsent",        "TooLargeForExhaustive",
        "OrderTooLarge",     "NotRefinement",      "GroundSetMismatch",
        "VertexAbsent",      "TooLarge",           "OutOfTable",
        "SampleTooSmall",    "TooManyTerms",       "NonIntegerResult",
        "ComponentEvaluationError", "InvalidArgument", "CudaError",
        "CollectiveError"};
    auto i = static_cast<std::size_t>(code);
    return i < sizeof(names) / sizeof(names[0]) ? names[i] : "UnknownError";
}

void fail(ErrorCode code, const std::string& message) { throw Error(code, message); }

// ---------------------------------------------------------------- config
int Config::effective_threads() const {
    if (threads > 0) return threads;
    const unsigned hw = std::thread::hardware_concurrency();
    return hw ? static_cast<int>(hw) : 1;
}

// -------------------------------------------------------------- notation
// (notation.cpp:10-45) ids renumbered by first appearance across inputs.
EinsumNotation validate_notation(const std::vector<IndexTuple>& raw_inputs,
                                 const IndexTuple& raw_output) {
    if (raw_inputs.empty())
        fail(ErrorCode::InvalidNotation, "a notation needs at least one input tuple");
    std::unordered_map<int, int> rename;
    EinsumNotation out;
    for (const IndexTuple& raw : raw_inputs) {
        if (raw.empty()) fail(ErrorCode::InvalidNotation, "input tuples must be non-empty");
        IndexTuple t;
        t.reserve(raw.size());
        for (int id : raw) {
            if (id < 0) fail(ErrorCode::InvalidNotation, "indices must be non-negative");
            auto it = rename.find(id);
            if (it == rename.end()) it = rename.emplace(id, static_cast<int>(rename.size())).first;
            t.push_back(it->second);
        }
        out.inputs.push_back(std::move(t));
    }
    out.index_count = static_cast<int>(rename.size());
    std::vector<char> used(static_cast<std::size_t>(out.index_count), 0);
    for (int id : raw_output) {
        auto it = rename.find(id);
        if (it == rename.end())
            fail(ErrorCode::InvalidOutput,
                 "output index " + std::to_string(id) + " appears in no input tuple");
        if (used[static_cast<std::size_t>(it->second)])
            fail(ErrorCode::InvalidOutput, "output index " + std::to_string(id) + " is repeated");
        used[static_cast<std::size_t>(it->second)] = 1;
        out.output.push_back(it->second);
    }
    return out;
}

EinsumNotation::EinsumNotation(std::vector<IndexTuple> raw_inputs, IndexTuple raw_output) {
    *this = validate_notation(raw_inputs, raw_output);
}

bool EinsumNotation::index_in_output(int index) const {
    return std::find(output.begin(), output.end(), index) != output.end();
}

std::string EinsumNotation::to_string() const {
    auto render = [](const IndexTuple& t) {
        std::string s = "(";
        for (std::size_t i = 0; i < t.size(); ++i) s += (i ? "," : "") + std::to_string(t[i]);
        return s + ")";
    };
    std::string s = "(";
    for (std::size_t k = 0; k < inputs.size(); ++k) s += (k ? "," : "") + render(inputs[k]);
    return s + ")->" + render(output);
}

// ---------------------------------------------------------------- tensor
// (tensor.cpp:9-26) the cap is checked before any allocation.
std::uint64_t checked_entry_count(int order, int extent, const Config& config) {
    if (order < 0) fail(ErrorCode::InvalidArgument, "tensor order must be >= 0");
    if (extent < 1) fail(ErrorCode::InvalidArgument, "tensor extent must be >= 1");
    std::uint64_t entries = 1;
    for (int i = 0; i < order; ++i) {
        if (entries > config.memory_cap_entries / static_cast<std::uint64_t>(extent))
            fail(ErrorCode::MemoryCapExceeded,
                 "tensor of order " + std::to_string(order) + " at extent " +
                     std::to_string(extent) + " exceeds the cap of " +
                     std::to_string(config.memory_cap_entries) + " entries");
        entries *= static_cast<std::uint64_t>(extent);
    }
    if (entries > config.memory_cap_entries)
        fail(ErrorCode::MemoryCapExceeded, "tensor exceeds the entry cap");
    return entries;
}

DenseTensor::DenseTensor(int order_, int extent_, const Config& config)
    : order(order_), extent(extent_), data(checked_entry_count(order_, extent_, config), 0.0) {}

std::uint64_t DenseTensor::offset_of(std::span<const int> index) const {
    std::uint64_t flat = 0;
    for (int a = 0; a < order; ++a)
        flat = flat * static_cast<std::uint64_t>(extent) + static_cast<std::uint64_t>(index[a]);
    return flat;
}

bool next_multi_index(std::span<int> index, int extent) {
    for (std::size_t a = index.size(); a-- > 0;) {
        if (++index[a] < extent) return true;
        index[a] = 0;
    }
    return false;
}

DenseTensor tensor_from_function(int order, int extent,
                                 const std::function<double(std::span<const int>)>& fn,
                                 const Config& config) {
    DenseTensor t(order, extent, config);
    std::vector<int> idx(static_cast<std::size_t>(order), 0);
    std::uint64_t flat = 0;
    do {
        t.data[flat++] = fn(idx);
    } while (next_multi_index(idx, extent));
    return t;
}

DenseTensor sparsify(const DenseTensor& t) {
    DenseTensor out = t;
    if (t.order < 2) return out;
    std::vector<int> idx(static_cast<std::size_t>(t.order), 0);
    std::uint64_t flat = 0;
    do {
        bool repeat = false;
        for (int a = 0; a < t.order && !repeat; ++a)
            for (int b = a + 1; b < t.order && !repeat; ++b) repeat = idx[a] == idx[b];
        if (repeat) out.data[flat] = 0.0;
        ++flat;
    } while (next_multi_index(idx, t.extent));
    return out;
}

// ---------------------------------------------------------------- kernel
// (kernel.cpp:10-60)
void MDKernel::validate() const {
    if (arity < 1) fail(ErrorCode::InvalidArgument, "kernel arity must be >= 1");
    if (signature.empty()) fail(ErrorCode::InvalidArgument, "kernel needs at least one component");
    if (signature.size() != components.size())
        fail(ErrorCode::InvalidArgument, "kernel needs one component per signature tuple");
    std::vector<char> covered(static_cast<std::size_t>(arity), 0);
    for (const IndexTuple& tuple : signature) {
        if (tuple.empty()) fail(ErrorCode::InvalidArgument, "signature tuples must be non-empty");
        std::vector<char> here(static_cast<std::size_t>(arity), 0);
        for (int slot : tuple) {
            if (slot < 1 || slot > arity)
                fail(ErrorCode::InvalidArgument, "signature slot " + std::to_string(slot) +
                                                     " outside 1.." + std::to_string(arity));
            auto s = static_cast<std::size_t>(slot - 1);
            if (here[s])
                fail(ErrorCode::InvalidArgument,
                     "signature slot " + std::to_string(slot) + " repeated within one tuple");
            here[s] = covered[s] = 1;
        }
    }
    for (int s = 0; s < arity; ++s)
        if (!covered[static_cast<std::size_t>(s)])
            fail(ErrorCode::InvalidArgument,
                 "argument slot " + std::to_string(s + 1) + " appears in no signature tuple");
}

std::vector<IndexTuple> MDKernel::zero_based_signature() const {
    std::vector<IndexTuple> z = signature;
    for (IndexTuple& t : z)
        for (int& s : t) --s;
    return z;
}

double MDKernel::evaluate(const Sample& sample, std::span<const int> indices) const {
    double prod = 1.0;
    std::vector<int> picks;
    for (std::size_t k = 0; k < signature.size(); ++k) {
        picks.clear();
        for (int slot : signature[k]) picks.push_back(indices[static_cast<std::size_t>(slot - 1)]);
        prod *= components[k](sample, picks);
    }
    return prod;
}

MDKernel prod2_kernel() {
    auto x0 = [](const Sample& s, std::span<const int> idx) {
        const Observation& o = s.points[static_cast<std::size_t>(idx[0])];
        if (o.empty()) fail(ErrorCode::InvalidArgument, "prod2 needs at least one coordinate");
        return o[0];
    };
    MDKernel k;
    k.arity = 2;
    k.signature = {{1}, {2}};
    k.components = {x0, x0};
    k.name = "prod2";
    return k;
}

}  // namespace ustats
