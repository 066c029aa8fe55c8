// Argument blocks and launchers of the sm_100a kernels. Shared by the .cu
// kernel files and the host-side executor (plain C++: no CUDA types beyond
// cudaStream_t leak into the planner).
#pragma once

#include <cstdint>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include <cuda_runtime.h>

namespace ustats::dev {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel):
// function attributes are per device, so a process-wide flag would leave the
// kernel unconfigured on a second GPU.
inline void set_max_smem_once(const void* func, int bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, int> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    int& have = done[{dev, func}];
    if (have < bytes) {
        cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        have = bytes;
    }
}

constexpr int kMaxDims = 12;         // iteration dims of one stream (bandwidth) kernel
constexpr int kMaxFactors = 8;       // factors multiplied inside one kernel
constexpr int kMaxGemmFactors = 6;   // factors per GEMM operand (prologue product)
constexpr int kMaxRowDims = 3;       // ids folded into one GEMM row / column index

// Multi-consumer matrix sweep: ONE pass over a matrix X (row-major view,
// X(R, C) = x[R * xr + C]) feeding several reductions that would each have
// streamed X again. Per row the kernel forms the power sums
// S_p(R) = sum_C X(R,C)^p (p = 1..4); consumer q scales S_{power_q} by its
// row weights f_q(R) = prod_i rowv_i[R * rs_i]:
//   kSweepAll: out[0] (+)= sum_R f_q(R) S_p(R)   (block partials, then in order)
//   kSweepRow: out[R] (+)= f_q(R) S_p(R)
constexpr int kMaxSweep = 16;
enum SweepMode : int { kSweepAll = 0, kSweepRow = 1 };
struct SweepOut {
    int mode = kSweepAll;
    int power = 1;
    int nrow = 0;
    const double* rowv[4] = {};
    long long rows_stride[4] = {};
    double* out = nullptr;
    double* partial = nullptr;  // kSweepAll: one slot per block
};
struct SweepArgs {
    const double* x = nullptr;
    long long xr = 0;           // row stride of X (column stride 1)
    long long cols = 0;
    long long r0 = 0, r1 = 0;   // rows [r0, r1) (a rank's slice under row sharding)
    int accumulate = 0;
    int count = 0;
    SweepOut o[kMaxSweep];
};
// Blocks a sweep over `rows` rows launches (= partial slots per kSweepAll consumer).
int sweep_blocks(long long rows, int sm_count);
int launch_sweep(const SweepArgs& a, int sm_count, cudaStream_t s);

// Broadcast-product-reduce ("stream") kernel:
//   out[o] = scale * sum_{s} prod_f F_f[ sum_d digit_d * stride[f][d] ]
// iteration dims [0, n_out) are the output (row-major, last fastest),
// [n_out, n_out + n_sum) are summed (last fastest). Every dim has extent n.
struct StreamArgs {
    int nf = 0;
    int n_out = 0;
    int n_sum = 0;
    long long n = 1;
    const double* ptr[kMaxFactors] = {};
    long long stride[kMaxFactors][kMaxDims] = {};
    double* out = nullptr;
    double scale = 1.0;
    long long n0 = 0;      // extent of iteration dim 0 (0 = n): a rank's slice in row sharding
    int accumulate = 0;    // out += result (outputs pre-zeroed; slices of all ranks add up)
    // permuted outputs: the output dims are iterated in an order other than
    // the buffer's layout; output dim d sits at out[sum_d digit_d * ostride[d]]
    int permuted_out = 0;
    long long ostride[kMaxDims] = {};
    // mult[0]: multiplicity of factor 0 (1..4): identical views of one tensor
    // merged by launch_stream into one load raised to a power (paired kernels only)
    int mult[kMaxFactors] = {1, 1, 1, 1, 1, 1, 1, 1};
};

// One GEMM operand: value(r, k) = prod_f ptr_f[ off_f(r) + kstride_f * k ]
// with off_f(r) = sum over the nr row digits of r (base n, row-major) times rstride.
struct GemmSide {
    int nf = 0;
    int nr = 1;
    const double* ptr[kMaxGemmFactors] = {};
    long long rstride[kMaxGemmFactors][kMaxRowDims] = {};
    long long kstride[kMaxGemmFactors] = {};
};

enum EpilogueMode : int {
    kEpiStore = 0,      // out[r * cols + c] = scale * C * W (symmetric_out: mirrored too)
    kEpiSumAll = 1,     // partial[block] = sum_{r,c} C * W      (then finalize; symmetric_out:
                        //   upper tiles only, off-diagonal tiles counted twice)
    kEpiSumCols = 2,    // partial[tile_n][r] = sum_c C * W     (then finalize -> out[r])
    kEpiSumRows = 3,    // partial[tile_m][c] = sum_r C * W     (then finalize -> out[c])
};

// Epilogue factors W(r, c) = prod_g ptr_g[ roff_g(r) + coff_g(c) ].
struct EpilogueSide {
    int nf = 0;
    const double* ptr[kMaxGemmFactors] = {};
    long long rstride[kMaxGemmFactors][kMaxRowDims] = {};
    long long cstride[kMaxGemmFactors][kMaxRowDims] = {};
};

struct GemmArgs {
    GemmSide a;          // rows x k
    GemmSide b;          // cols x k (described by its column digits)
    EpilogueSide w;
    long long n = 1;     // extent of every id, including k
    long long rows = 0;
    long long cols = 0;
    int mode = kEpiStore;
    double* out = nullptr;      // store target, or finalize target
    double* partial = nullptr;  // scratch for reduce modes
    double scale = 1.0;
    int a_kmajor = 1;           // loader orientation hints (coalescing)
    int b_kmajor = 1;
    int symmetric_out = 0;      // rows==cols and C symmetric: compute upper tiles only
    int self_power = 1;         // epilogue value = C^self_power * W (2: the consumer read C twice)
    int tri_colmajor = 0;       // symmetric tile list ordered by column (tiles of row panels <= tn first)
    long long tile_begin = 0;   // row sharding: this rank's contiguous range of the tile list
    long long tile_count = -1;  // -1 = every tile
    int accumulate = 0;         // outputs += (pre-zeroed), see StreamArgs::accumulate
};

// Number of CTA tiles of a GEMM launch (upper triangle when symmetric_out and square).
long long gemm_tile_total(const GemmArgs& a, bool tma_symmetric);

// Multi-consumer epilogues of the TMA GEMM: every consumer of a GEMM output
// that iterates exactly over its (row, col) space runs on the accumulator tile
// staged in shared memory. Weights W(r,c) = prod_f wptr[f][r*wr[f] + c*wc[f]].
constexpr int kMaxEpiW = 4;
constexpr int kMaxEpilogues = 40;
struct EpiDesc {
    int mode = kEpiStore;
    int self_power = 1;
    int nw = 0;
    int transpose = 0;          // Store: write out[C * rows + R] instead of out[R * cols + C]
    const double* wptr[kMaxEpiW] = {};
    long long wr[kMaxEpiW] = {};
    long long wc[kMaxEpiW] = {};
    double* out = nullptr;      // Store: rows x cols matrix; reductions: finalize target
    double* partial = nullptr;  // reduction scratch (gemm_epi_partial_entries)
};
struct EpiSet {
    int count = 0;
    EpiDesc d[kMaxEpilogues];
};

// ------------------------------------------------------------- launchers
// Launchers return the number of kernels they enqueued.
int launch_stream(const StreamArgs& a, double* scratch, std::size_t scratch_entries,
                  int sm_count, cudaStream_t s);
std::size_t stream_scratch_entries(const StreamArgs& a, int sm_count);

// TMA-fed kernel when both operands are single plain strided matrices
// (gemm_tma.cu), otherwise the lazy-product gather kernel (gemm_f64.cu).
int launch_gemm(const GemmArgs& a, cudaStream_t s);
bool gemm_tma_eligible(const GemmArgs& a, int* a_kmajor, int* b_kmajor);
// Multi-epilogue TMA GEMM (a.mode/a.w/a.out ignored; symmetric_out computes
// upper tiles and mirrors every epilogue). Returns kernels launched, or -1
// if the operands are not TMA-eligible.
int launch_gemm_multi(const GemmArgs& a, const EpiSet& epis, cudaStream_t s);
// The fixed-order finalizers of the reduction epilogues of `epis` after a
// launch of `blocks` 128 x 128 tiles over a rows x cols product.
int launch_epilogue_finalize(long long rows, long long cols, const EpiSet& epis, long long blocks, int accumulate,
                             cudaStream_t s);
std::size_t gemm_epi_partial_entries(const GemmArgs& a, int mode);
std::size_t gemm_partial_entries(const GemmArgs& a);

// Zero every entry of an order-`order` tensor whose multi-index repeats a
// coordinate (tensor.cpp:54-76), in place.
int launch_sparsify(double* data, int order, long long n, cudaStream_t s);
// out[i] (+)= sum_{c < C} slices[c * len + i], c in order (deterministic
// combine of per-chunk reductions).
int launch_sum_slices(const double* slices, int C, long long len, double* out, int accumulate, cudaStream_t s);
// Zeroes the diagonal entries of rows [r0, r1) of an n x n matrix (a panel
// of a chunked upload).
int launch_zero_diagonal_rows(double* data, long long n, long long r0, long long r1, cudaStream_t s);
// dst[c * dst_pitch + r] = src[r * src_pitch + c] for r < rows, c < cols.
int launch_transpose(const double* src, long long rows, long long cols, long long src_pitch, double* dst,
                     long long dst_pitch, cudaStream_t s);
// flag[0] = 0 if the n x n matrix is bitwise symmetric, else 1.
int launch_symmetry_check(const double* data, long long n, int* flag, cudaStream_t s);

// FP64 GEMM by Ozaki splitting on the INT8 tensor cores (gemm_ozaki.cu):
// C (m x n, row stride ldc) = A B^T with A m x k and B n x k given as
// pre-split digit slices (ozaki_split: tiled K-major int8, row exponents).
constexpr int kOzMaxSlices = 7;
struct OzakiArgs {
    const int8_t* a = nullptr;   // slices of A: tiles of 128 rows x 64 bytes
    const int8_t* b = nullptr;   // slices of B: tiles of 128 rows x 64 bytes (may alias A)
    long long a_slice = 0, b_slice = 0;  // bytes between consecutive slices
    const int* a_exp = nullptr;
    const int* b_exp = nullptr;
    long long m = 0, n = 0, mpad = 0, npad = 0, kpad = 0;
    int slices = 7;
    int symmetric = 0;           // B = A: upper tiles only, mirrored epilogues
    int accumulate = 0;          // epilogue outputs += (pre-zeroed)
    long long tile_begin = 0;    // row sharding: this launch covers tiles [tile_begin, tile_begin + tile_count)
    long long tile_count = -1;   // -1: to the end of the tile list
    int prefetch = 0;            // k-tiles ahead the producer warms L2 (set by launch_ozaki_gemm)
    int group2 = 0;              // CTA-pair kernel, non-symmetric: pair rows per tile group (0 = default)
    int sym_group2 = 0;          // CTA-pair kernel, symmetric: pair rows per row group (0 = column groups)
    long long pairs = 0;         // CTA-pair kernel: pair tiles of the launch (clusters loop over them)
    unsigned long long* wave_ctr = nullptr;  // CTA-pair kernel: wave-barrier counters [tile start, pass 1] (null: none)
    int resync = 0;              // CTA-pair kernel: also meet before pass 1
    double* work = nullptr;      // 128 x 128 doubles per SM (ozaki_work_entries): the high-diagonal partial
    // last partial wave split along K (set by launch_ozaki_gemm): launch-relative
    // tiles >= tail_from run as tail_split CTAs each over a K range; the last
    // one to finish sums the partial tiles (in chunk order) and runs the epilogues
    long long tail_from = 0;
    int tail_split = 1;
    double* tail_part = nullptr;
    unsigned* tail_count = nullptr;
    EpiSet epis;                 // fused consumers of the product tile (a plain store is one of them)
};
std::size_t ozaki_slice_bytes(long long rows, long long k, int tile_rows);
// Digits of a rows x k operand (row stride rs, k stride ks) for tile_rows = 128;
// with `panels`, only those 128-row panels are written.
int ozaki_split(const double* x, long long rows, long long k, long long rs, long long ks, int tile_rows, int slices,
                int8_t* out, int* exps, cudaStream_t s, const std::vector<int>* panels = nullptr);
// Digits of a lazy operand (GemmSide: a product of factors, rows in base n)
// over K columns [k0, k0 + k), formed from the factors without an FP64 copy.
int ozaki_split_lazy(const GemmSide& side, long long n, long long rows, long long k0, long long k, int slices,
                     int8_t* out, int* exps, cudaStream_t s);
long long ozaki_tile_count(const OzakiArgs& p);
// The 128-row panels of A and of B that the tiles [tile_begin, tile_begin + tile_count) read.
void ozaki_tile_panels(const OzakiArgs& p, std::vector<int>* a_panels, std::vector<int>* b_panels);
std::size_t ozaki_work_entries();  // doubles of OzakiArgs::work
// Launches the emulated GEMM with its fused epilogues and their finalizers.
int launch_ozaki_gemm(const OzakiArgs& p, cudaStream_t s);

}  // namespace ustats::dev
