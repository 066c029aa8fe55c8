// Device-side tensorization: the kernel components of the
// BASELINE workloads and of the binding's kernel specs are materialized on
// the GPU from the raw sample (n x d, row-major) instead of n^|A_k|
// std::function calls on the host (engine.cpp:108-136, tensor.cpp:42-52).
#include <cmath>

#include "kernels.hpp"
#include "tensorize.hpp"

namespace ustats::dev {

namespace {

// A_ij = exp(-scale * sum_c (x_ic - x_jc)^2). The squared differences are
// summed in coordinate order, so A is bitwise symmetric.
__global__ void rbf(const double* __restrict__ x, long long n, int d, double scale, double* __restrict__ out,
                    int zero_diag) {
    const long long j = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    const long long i = blockIdx.y;
    if (j >= n) return;
    const double* xi = x + i * d;
    const double* xj = x + j * d;
    double s = 0.0;
    for (int c = 0; c < d; ++c) {
        const double t = xi[c] - xj[c];
        s += t * t;
    }
    out[i * n + j] = (zero_diag && i == j) ? 0.0 : exp(-scale * s);
}

// Symmetric tiled pair kernels: one 32x32 tile pair (ti <= tj) per block,
// sample rows staged in shared memory, the entry evaluated once per
// unordered pair and written to both (i, j) and (j, i) with coalesced stores
// (the transpose goes through a padded smem tile). The squared distance is
// summed per coordinate in order, as the reference's per-entry callbacks do,
// so the matrix is bitwise symmetric.
//   kind 0: exp(-scale * s)   (RBF)
//   kind 1: sqrt(s)           (Euclidean distance, dcov.cpp:24-31)
constexpr int kPairTile = 32, kPairMaxDim = 64;
template <int KIND>
__global__ void pair_sym(const double* __restrict__ x, long long n, int d, int c0, int dc, double scale,
                         double* __restrict__ out, int zero_diag) {
    const int ti = blockIdx.y, tj = blockIdx.x;
    if (ti > tj) return;
    __shared__ double xi[kPairTile][kPairMaxDim + 1], xj[kPairTile][kPairMaxDim + 1];
    __shared__ double t[kPairTile][kPairTile + 1];
    const long long i0 = static_cast<long long>(ti) * kPairTile, j0 = static_cast<long long>(tj) * kPairTile;
    const int tid = threadIdx.y * kPairTile + threadIdx.x;
    for (int e = tid; e < kPairTile * dc; e += kPairTile * 8) {
        const int r = e / dc, c = e - r * dc;
        xi[r][c] = i0 + r < n ? x[(i0 + r) * d + c0 + c] : 0.0;
        xj[r][c] = j0 + r < n ? x[(j0 + r) * d + c0 + c] : 0.0;
    }
    __syncthreads();
    const int cj = threadIdx.x;
#pragma unroll
    for (int k = 0; k < kPairTile / 8; ++k) {
        const int ri = threadIdx.y + 8 * k;
        double s = 0.0;
        for (int c = 0; c < dc; ++c) {
            const double u = xi[ri][c] - xj[cj][c];
            s += u * u;
        }
        double v = KIND == 0 ? exp(-scale * s) : sqrt(s);
        if (zero_diag && ti == tj && ri == cj) v = 0.0;  // sparsified on the fly (tensor.cpp:54-76)
        t[ri][cj] = v;
        if (i0 + ri < n && j0 + cj < n) out[(i0 + ri) * n + j0 + cj] = v;
    }
    if (ti == tj) return;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kPairTile / 8; ++k) {
        const int rj = threadIdx.y + 8 * k;  // row j0 + rj of the mirror tile
        if (j0 + rj < n && i0 + cj < n) out[(j0 + rj) * n + i0 + cj] = t[cj][rj];
    }
}

// Register-blocked form for narrow samples (dc <= 32): 64x64 tile pairs
// (ti <= tj), each thread a 4x4 block (4 + 4 shared loads per coordinate for
// 16 entries), the entry written to (i, j) and — for off-diagonal tiles — to
// (j, i), each as 32-byte row segments. Same per-entry arithmetic (squared
// differences summed per coordinate in order), so the matrix is identical to
// pair_sym's and bitwise symmetric.
constexpr int kBlkTile = 64, kBlkDim = 32;
template <int KIND>
__global__ void __launch_bounds__(256) pair_sym_blocked(const double* __restrict__ x, long long n, int d, int c0,
                                                        int dc, double scale, double* __restrict__ out, int zero_diag) {
    const int ti = blockIdx.y, tj = blockIdx.x;
    if (ti > tj) return;
    // coordinate-major point blocks; reused afterwards as the transposed 64 x 64 tile
    __shared__ double buf[2 * kBlkDim * (kBlkTile + 1)];
    static_assert(2 * kBlkDim >= kBlkTile, "the transposed tile fits the point blocks");
    auto xi = reinterpret_cast<double(*)[kBlkTile + 1]>(buf);
    auto xj = reinterpret_cast<double(*)[kBlkTile + 1]>(buf + kBlkDim * (kBlkTile + 1));
    const long long i0 = static_cast<long long>(ti) * kBlkTile, j0 = static_cast<long long>(tj) * kBlkTile;
    const int tid = threadIdx.x;
    for (int e = tid; e < kBlkTile * dc; e += 256) {
        const int r = e / dc, c = e - r * dc;
        xi[c][r] = i0 + r < n ? x[(i0 + r) * d + c0 + c] : 0.0;
        xj[c][r] = j0 + r < n ? x[(j0 + r) * d + c0 + c] : 0.0;
    }
    __syncthreads();
    const int ty = tid >> 4, tx = tid & 15;
    double s[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) s[a][b] = 0.0;
    for (int c = 0; c < dc; ++c) {
        double u[4], v[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) u[a] = xi[c][ty * 4 + a];
#pragma unroll
        for (int b = 0; b < 4; ++b) v[b] = xj[c][tx * 4 + b];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const double t = u[a] - v[b];
                s[a][b] += t * t;
            }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) s[a][b] = KIND == 0 ? exp(-scale * s[a][b]) : sqrt(s[a][b]);
    if (zero_diag && ti == tj && ty == tx) {  // sparsified on the fly (tensor.cpp:54-76)
#pragma unroll
        for (int a = 0; a < 4; ++a) s[a][a] = 0.0;
    }
    const long long ib = i0 + ty * 4, jb = j0 + tx * 4;
    const bool full = i0 + kBlkTile <= n && j0 + kBlkTile <= n && (n & 1) == 0;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        if (full) {
            double2* o = reinterpret_cast<double2*>(out + (ib + a) * n + jb);
            o[0] = make_double2(s[a][0], s[a][1]);
            o[1] = make_double2(s[a][2], s[a][3]);
        } else if (ib + a < n) {
            for (int b = 0; b < 4; ++b)
                if (jb + b < n) out[(ib + a) * n + jb + b] = s[a][b];
        }
    }
    if (ti == tj) return;
    if (full) {  // the mirrored block through shared memory: a warp writes 512 contiguous bytes of a row
        __syncthreads();  // every thread is done with the point blocks
        auto tr = reinterpret_cast<double(*)[kBlkTile + 1]>(buf);  // tr[j][i]
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) tr[tx * 4 + b][ty * 4 + a] = s[a][b];
        __syncthreads();
        for (int e = tid; e < kBlkTile * kBlkTile / 2; e += 256) {
            const int j = e / (kBlkTile / 2), i = 2 * (e % (kBlkTile / 2));
            *reinterpret_cast<double2*>(out + (j0 + j) * n + i0 + i) = make_double2(tr[j][i], tr[j][i + 1]);
        }
        return;
    }
#pragma unroll
    for (int b = 0; b < 4; ++b)
        if (jb + b < n)
            for (int a = 0; a < 4; ++a)
                if (ib + a < n) out[(jb + b) * n + ib + a] = s[a][b];
}

// Euclidean distances over columns [c0, c0 + dc) (fallback for wide samples).
__global__ void distance(const double* __restrict__ x, long long n, int d, int c0, int dc, double* __restrict__ out) {
    const long long j = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    const long long i = blockIdx.y;
    if (j >= n) return;
    double s = 0.0;
    for (int c = 0; c < dc; ++c) {
        const double u = x[i * d + c0 + c] - x[j * d + c0 + c];
        s += u * u;
    }
    out[i * n + j] = sqrt(s);
}

// Graph indicators (motifs.cpp:11-31): A[u][v] = A[v][u] = 1 per edge over a
// zeroed matrix; the co-indicator B = 1 - A off the diagonal, 0 on it.
__global__ void scatter_edges(const int* __restrict__ edges, long long count, long long n, double* __restrict__ a) {
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < count;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long u = edges[2 * e], v = edges[2 * e + 1];
        a[u * n + v] = 1.0;
        a[v * n + u] = 1.0;
    }
}

__global__ void co_indicator(const double* __restrict__ a, long long n, double* __restrict__ b) {
    const long long total = n * n;
    for (long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; q < total;
         q += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long i = q / n, j = q - i * n;
        b[q] = i == j ? 0.0 : 1.0 - a[q];
    }
}

// out_ij = left_i * (sum_c z_ic z_jc) * right_j   (hoif.cpp:50-72 components)
__global__ void scaled_gram(const double* __restrict__ x, long long n, int d, int col_left, int col_right, int z0,
                            int k, double* __restrict__ out) {
    const long long j = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    const long long i = blockIdx.y;
    if (j >= n) return;
    const double* xi = x + i * d;
    const double* xj = x + j * d;
    double dot = 0.0;
    for (int c = 0; c < k; ++c) dot += xi[z0 + c] * xj[z0 + c];
    const double l = col_left >= 0 ? xi[col_left] : 1.0;
    const double r = col_right >= 0 ? xj[col_right] : 1.0;
    out[i * n + j] = (l * dot) * r;
}

__global__ void column(const double* __restrict__ x, long long n, int d, int c, double* __restrict__ out) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i < n) out[i] = x[i * d + c];
}

// Z_i,(c*kmax + k-1) = cos(pi * k * u_ic), k = 1..kmax, for columns c < ncols.
__global__ void cosine_features(const double* __restrict__ x, long long n, int d, int ncols, int kmax,
                                double* __restrict__ z) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const int F = ncols * kmax;
    for (int c = 0; c < ncols; ++c) {
        const double u = x[i * d + c];
        for (int k = 1; k <= kmax; ++k) z[i * F + c * kmax + (k - 1)] = cos(M_PI * k * u);
    }
}

// G = Z^T Z / n for a thin Z (n x F). Each block takes a contiguous range of
// rows, stages 32-row tiles of Z in shared memory with coalesced loads and
// accumulates its F x F partial Gram in registers (thread t: entries
// t, t + 256, ...; rows in order); gram_finalize then sums the block partials
// in block order. Fixed order throughout: deterministic, and G is bitwise
// symmetric (entry (f, h) and (h, f) add the same products in the same order).
constexpr int kGramRows = 32, kGramMaxF = 64, kGramPerThread = kGramMaxF * kGramMaxF / 256;
__global__ void __launch_bounds__(256) thin_gram_partial(const double* __restrict__ z, long long n, int F,
                                                         double* __restrict__ partial) {
    __shared__ double tile[kGramRows][kGramMaxF + 1];
    const long long B = gridDim.x;
    const long long lo = n * blockIdx.x / B, hi = n * (blockIdx.x + 1) / B;
    double acc[kGramPerThread];
#pragma unroll
    for (int q = 0; q < kGramPerThread; ++q) acc[q] = 0.0;
    for (long long r0 = lo; r0 < hi; r0 += kGramRows) {
        const int rows = static_cast<int>(hi - r0 < kGramRows ? hi - r0 : kGramRows);
        __syncthreads();
        for (int e = threadIdx.x; e < rows * F; e += 256) tile[e / F][e % F] = z[r0 * F + e];
        __syncthreads();
#pragma unroll
        for (int q = 0; q < kGramPerThread; ++q) {
            const int e = threadIdx.x + 256 * q;
            if (e < F * F) {
                const int f = e / F, h = e % F;
                double s = acc[q];
                for (int r = 0; r < rows; ++r) s += tile[r][f] * tile[r][h];
                acc[q] = s;
            }
        }
    }
#pragma unroll
    for (int q = 0; q < kGramPerThread; ++q) {
        const int e = threadIdx.x + 256 * q;
        if (e < F * F) partial[static_cast<long long>(blockIdx.x) * F * F + e] = acc[q];
    }
}
__global__ void gram_finalize(const double* __restrict__ partial, int blocks, int F, long long n, double* __restrict__ g) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= F * F) return;
    double s = 0.0;
    for (int b = 0; b < blocks; ++b) s += partial[static_cast<long long>(b) * F * F + e];
    g[e] = s / static_cast<double>(n);
}

// Fallback for wide feature sets (F > 64): one block per (f, g) pair,
// fixed-order strided sums + tree (deterministic).
__global__ void thin_gram(const double* __restrict__ z, long long n, int F, double* __restrict__ g) {
    __shared__ double red[256];
    const int f = blockIdx.x, h = blockIdx.y;
    double s = 0.0;
    for (long long i = threadIdx.x; i < n; i += blockDim.x) s += z[i * F + f] * z[i * F + h];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) g[f * F + h] = red[0] / static_cast<double>(n);
}

// Y = Z M (n x F times a small dense F x F): a thread per output entry, the
// F products summed in order (lanes along the output row: M reads coalesce,
// the Z row is a warp-wide broadcast).
__global__ void times_small(const double* __restrict__ z, long long n, int F, const double* __restrict__ M,
                            double* __restrict__ y) {
    const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (e >= n * F) return;
    const long long i = e / F;
    const int c = static_cast<int>(e - i * F);
    double s = 0.0;
    for (int r = 0; r < F; ++r) s += __ldg(z + i * F + r) * __ldg(M + r * F + c);
    y[e] = s;
}

}  // namespace

void launch_rbf(const double* x, long long n, int d, double bandwidth, double* out, cudaStream_t s, bool zero_diag) {
    const double scale = 0.5 / (bandwidth * bandwidth);
    if (d <= kBlkDim) {
        const unsigned T = static_cast<unsigned>((n + kBlkTile - 1) / kBlkTile);
        pair_sym_blocked<0><<<dim3(T, T), 256, 0, s>>>(x, n, d, 0, d, scale, out, zero_diag ? 1 : 0);
        return;
    }
    if (d <= kPairMaxDim) {
        const unsigned T = static_cast<unsigned>((n + kPairTile - 1) / kPairTile);
        pair_sym<0><<<dim3(T, T), dim3(kPairTile, 8), 0, s>>>(x, n, d, 0, d, scale, out, zero_diag ? 1 : 0);
        return;
    }
    rbf<<<dim3(static_cast<unsigned>((n + 255) / 256), static_cast<unsigned>(n)), 256, 0, s>>>(x, n, d, scale, out,
                                                                                                  zero_diag ? 1 : 0);
}

void launch_distance(const double* x, long long n, int d, int c0, int dc, double* out, cudaStream_t s) {
    if (dc <= kBlkDim) {
        const unsigned T = static_cast<unsigned>((n + kBlkTile - 1) / kBlkTile);
        pair_sym_blocked<1><<<dim3(T, T), 256, 0, s>>>(x, n, d, c0, dc, 0.0, out, 0);
        return;
    }
    if (dc <= kPairMaxDim) {
        const unsigned T = static_cast<unsigned>((n + kPairTile - 1) / kPairTile);
        pair_sym<1><<<dim3(T, T), dim3(kPairTile, 8), 0, s>>>(x, n, d, c0, dc, 0.0, out, 0);
        return;
    }
    distance<<<dim3(static_cast<unsigned>((n + 255) / 256), static_cast<unsigned>(n)), 256, 0, s>>>(x, n, d, c0, dc,
                                                                                                  out);
}

void launch_adjacency(const int* edges, long long count, long long n, double* a, double* b, cudaStream_t s) {
    cudaMemsetAsync(a, 0, static_cast<std::size_t>(n * n) * sizeof(double), s);
    if (count > 0) {
        long long blocks = (count + 255) / 256;
        if (blocks > 148 * 16) blocks = 148 * 16;
        scatter_edges<<<static_cast<unsigned>(blocks), 256, 0, s>>>(edges, count, n, a);
    }
    long long blocks = (n * n + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    co_indicator<<<static_cast<unsigned>(blocks), 256, 0, s>>>(a, n, b);
}

void launch_scaled_gram(const double* x, long long n, int d, int col_left, int col_right, int z0, int k, double* out,
                        cudaStream_t s) {
    scaled_gram<<<dim3(static_cast<unsigned>((n + 255) / 256), static_cast<unsigned>(n)), 256, 0, s>>>(
        x, n, d, col_left, col_right, z0, k, out);
}

void launch_column(const double* x, long long n, int d, int c, double* out, cudaStream_t s) {
    column<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(x, n, d, c, out);
}

void launch_cosine_features(const double* x, long long n, int d, int ncols, int kmax, double* z, cudaStream_t s) {
    cosine_features<<<static_cast<unsigned>((n + 127) / 128), 128, 0, s>>>(x, n, d, ncols, kmax, z);
}

long long thin_gram_scratch_entries(long long n, int F) {
    if (F > kGramMaxF) return 0;
    long long blocks = (n + 4 * kGramRows - 1) / (4 * kGramRows);  // at least 128 rows per block
    if (blocks > 296) blocks = 296;
    return blocks * F * F;
}

void launch_thin_gram(const double* z, long long n, int F, double* g, double* partial, cudaStream_t s) {
    if (F <= kGramMaxF) {
        const int blocks = static_cast<int>(thin_gram_scratch_entries(n, F) / (static_cast<long long>(F) * F));
        thin_gram_partial<<<static_cast<unsigned>(blocks), 256, 0, s>>>(z, n, F, partial);
        gram_finalize<<<static_cast<unsigned>((F * F + 255) / 256), 256, 0, s>>>(partial, blocks, F, n, g);
        return;
    }
    thin_gram<<<dim3(static_cast<unsigned>(F), static_cast<unsigned>(F)), 256, 0, s>>>(z, n, F, g);
}

void launch_times_small(const double* z, long long n, int F, const double* M, double* y, cudaStream_t s) {
    times_small<<<static_cast<unsigned>((n * F + 255) / 256), 256, 0, s>>>(z, n, F, M, y);
}

}  // namespace ustats::dev
