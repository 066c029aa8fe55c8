// Device tensorization kernels (tensorize.cu) and the data-kernel front end
// (data_kernels.cpp).
#pragma once

#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "ustats/config.hpp"
#include "ustats/notation.hpp"

namespace ustats::dev {

// zero_diag: write the sparsified matrix directly (zero diagonal, tensor.cpp:54-76)
void launch_rbf(const double* x, long long n, int d, double bandwidth, double* out, cudaStream_t s,
                bool zero_diag = false);
// Euclidean distance matrix over sample columns [c0, c0 + dc) (row stride d).
void launch_distance(const double* x, long long n, int d, int c0, int dc, double* out, cudaStream_t s);
// Adjacency indicator a and co-indicator b (zero diagonal) of an edge list
// (count pairs of vertex ids in [0, n), no self-loops).
void launch_adjacency(const int* edges, long long count, long long n, double* a, double* b, cudaStream_t s);
void launch_scaled_gram(const double* x, long long n, int d, int col_left, int col_right, int z0, int k, double* out,
                        cudaStream_t s);
void launch_column(const double* x, long long n, int d, int c, double* out, cudaStream_t s);
void launch_cosine_features(const double* x, long long n, int d, int ncols, int kmax, double* z, cudaStream_t s);
// G = Z^T Z / n; `partial` holds thin_gram_scratch_entries(n, F) doubles (0: none needed).
long long thin_gram_scratch_entries(long long n, int F);
void launch_thin_gram(const double* z, long long n, int F, double* g, double* partial, cudaStream_t s);
void launch_times_small(const double* z, long long n, int F, const double* M, double* y, cudaStream_t s);

struct StatisticResult;

// Parsed data kernel: component k reads slots sig[k] and is built by recipe[k].
struct DataKernel {
    int m = 0;
    std::vector<IndexTuple> sig;   // 0-based
    std::vector<std::string> recipe;  // canonical component recipe (equal strings = same tensor)
};

// Kernel specs (the binding's prod2 / hoif:<j>:<k>, plus the BASELINE
// workloads): "prod2", "hoif:<j>:<k>", "rbf:<shape>:<bandwidth>" with shape
// chain<m> | cycle<m> | k4tail, "proj:<m>:<kmax>" (cosine-feature projection
// chain r B..B e over data columns [u_1..u_c, r, e]).
DataKernel parse_data_kernel(const std::string& spec, int d);

// Tensorizes on the device from the sample and evaluates the U-statistic.
StatisticResult u_statistic_data(const std::string& spec, const double* data, long long n, int d, bool on_device,
                                 const Config& config, double* tensorize_seconds);

// dcov_squared (dcov.cpp:35-87): four U-statistics over the two distance
// matrices, evaluated as one shared device program.
StatisticResult dcov_squared(const double* x, int dx, const double* y, int dy, long long n, bool on_device,
                             const Config& config);

// motif_count (motifs.cpp:53-69): the ordered indicator-product U-statistic
// over the graph's adjacency / co-adjacency, divided by the automorphisms.
struct MotifSpec {
    const char* id;
    int order;
    int automorphisms;
    std::vector<std::pair<int, int>> present, absent;  // 1-based pairs
};
const std::vector<MotifSpec>& motif_catalog();
StatisticResult motif_count(long long n, const int* edges, long long edge_count, const std::string& id,
                            const Config& config, long long* count);

}  // namespace ustats::dev
