// FP64 tensor-core GEMM for the executor's pairwise contractions
// (replaces gemm_step + permuted_copy + Eigen, proj/src/einsum.cpp:116-130,
// 209-259, and the Khatri-Rao form of generic_step, 263-301).
//
// sm_100a has no tcgen05 kind::f64, so the FP64 tensor pipe is reached with
// warp-level mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4). Structure:
//   * 128x128 CTA tile, 8 warps as 2x4, 64x32 warp tile = 8x4 DMMA tiles,
//     64 FP64 accumulators per thread;
//   * operands are *lazy products*: each element is the product of up to 6
//     strided factor reads (Hadamard folds, diagonal scalings, Khatri-Rao
//     rows) formed once on the global->shared path, so folded operands are
//     never materialized;
//   * register-staged double buffering: tile k+1 is in flight from L2/HBM
//     while the DMMAs of tile k run; one barrier per k-tile;
//   * shared tiles are k-major (pitch 18) or m-major (pitch 136) to match the
//     coalesced direction of the dominant factor; both pitches make the
//     fragment reads 2-wavefront (conflict-free for 256 B);
//   * fused epilogues: Hadamard with W(r,c) and a fixed-order reduction to a
//     scalar, a row vector or a column vector (fold + marginalize consumers of
//     the product never see HBM).
#include "kernels.hpp"

namespace ustats::dev {

namespace {

constexpr int BM = 128, BN = 128, BKT = 16, THREADS = 256;
constexpr int PK = BKT + 2;    // k-major pitch (doubles)
constexpr int PM = BM + 8;     // m-major pitch (doubles)
constexpr int TILE = (BM * PK > BKT * PM) ? BM * PK : BKT * PM;
constexpr int GROUP_M = 8;

struct Smem {
    double a[2][TILE];
    double b[2][TILE];
    long long aoff[kMaxGemmFactors][BM];
    long long boff[kMaxGemmFactors][BN];
    long long woff_r[kMaxGemmFactors][BM];
    long long woff_c[kMaxGemmFactors][BN];
    double red[4][BM];
};

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// Offsets of one operand's factors for the tile's BM (or BN) rows; -1 marks
// rows past the end.
__device__ void row_offsets(const GemmSide& s, long long n, long long limit, long long first,
                            long long (*off)[BM]) {
    for (int i = threadIdx.x; i < s.nf * BM; i += THREADS) {
        const int f = i / BM, r = i % BM;
        long long g = first + r;
        long long o = -1;
        if (g < limit) {
            o = 0;
            for (int d = s.nr - 1; d >= 0; --d) {
                const long long q = g / n;
                o += (g - q * n) * s.rstride[f][d];
                g = q;
            }
        }
        off[f][r] = o;
    }
}

__device__ void epi_offsets(const EpilogueSide& w, int nr, int nc, long long n, long long rows,
                            long long cols, long long r0, long long c0, long long (*roff)[BM],
                            long long (*coff)[BN]) {
    for (int i = threadIdx.x; i < w.nf * BM; i += THREADS) {
        const int f = i / BM, r = i % BM;
        long long g = r0 + r, o = 0;
        if (g < rows)
            for (int d = nr - 1; d >= 0; --d) {
                const long long q = g / n;
                o += (g - q * n) * w.rstride[f][d];
                g = q;
            }
        roff[f][r] = o;
    }
    for (int i = threadIdx.x; i < w.nf * BN; i += THREADS) {
        const int f = i / BN, c = i % BN;
        long long g = c0 + c, o = 0;
        if (g < cols)
            for (int d = nc - 1; d >= 0; --d) {
                const long long q = g / n;
                o += (g - q * n) * w.cstride[f][d];
                g = q;
            }
        coff[f][c] = o;
    }
}

// Gathers 8 product values of one operand's k-tile into registers.
template <bool KMAJOR>
__device__ __forceinline__ void gather(const GemmSide& s, const long long (*off)[BM], long long n,
                                       long long k0, double (&v)[8]) {
    const int tid = threadIdx.x;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        int r, kl;
        if (KMAJOR) {
            kl = tid & 15;
            r = (tid >> 4) + 16 * i;
        } else {
            r = tid & 127;
            kl = (tid >> 7) + 2 * i;
        }
        const long long k = k0 + kl;
        double x = 0.0;
        if (k < n && off[0][r] >= 0) {
            x = __ldg(s.ptr[0] + off[0][r] + s.kstride[0] * k);
#pragma unroll
            for (int f = 1; f < kMaxGemmFactors; ++f)
                if (f < s.nf) x *= __ldg(s.ptr[f] + off[f][r] + s.kstride[f] * k);
        }
        v[i] = x;
    }
}

template <bool KMAJOR>
__device__ __forceinline__ void stash(double* tile, const double (&v)[8]) {
    const int tid = threadIdx.x;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        if (KMAJOR)
            tile[((tid >> 4) + 16 * i) * PK + (tid & 15)] = v[i];
        else
            tile[((tid >> 7) + 2 * i) * PM + (tid & 127)] = v[i];
    }
}

template <bool KMAJOR>
__device__ __forceinline__ double frag(const double* tile, int row, int k) {
    return KMAJOR ? tile[row * PK + k] : tile[k * PM + row];
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <bool AK, bool BK>
__global__ void __launch_bounds__(THREADS, 1) gemm_f64_kernel(GemmArgs p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw);

    const long long tiles_m = (p.rows + BM - 1) / BM, tiles_n = (p.cols + BN - 1) / BN;
    const long long bid = p.tile_begin + blockIdx.x;
    const long long width = GROUP_M * tiles_n;
    const long long group = bid / width, first_m = group * GROUP_M;
    const long long gsz = (tiles_m - first_m) < GROUP_M ? (tiles_m - first_m) : GROUP_M;
    const long long tm = first_m + (bid % width) % gsz;
    const long long tn = (bid % width) / gsz;
    const long long r0 = tm * BM, c0 = tn * BN;

    row_offsets(p.a, p.n, p.rows, r0, sm.aoff);
    row_offsets(p.b, p.n, p.cols, c0, sm.boff);
    if (p.w.nf) epi_offsets(p.w, p.a.nr, p.b.nr, p.n, p.rows, p.cols, r0, c0, sm.woff_r, sm.woff_c);
    __syncthreads();

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wm = warp >> 2, wn = warp & 3;
    const int g = lane >> 2, t = lane & 3;

    double acc[8][4][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    const long long KT = (p.n + BKT - 1) / BKT;
    double va[8], vb[8];
    gather<AK>(p.a, sm.aoff, p.n, 0, va);
    gather<BK>(p.b, sm.boff, p.n, 0, vb);
    stash<AK>(sm.a[0], va);
    stash<BK>(sm.b[0], vb);
    __syncthreads();

    for (long long kt = 0; kt < KT; ++kt) {
        const int cur = static_cast<int>(kt & 1);
        const bool more = kt + 1 < KT;
        if (more) {
            gather<AK>(p.a, sm.aoff, p.n, (kt + 1) * BKT, va);
            gather<BK>(p.b, sm.boff, p.n, (kt + 1) * BKT, vb);
        }
        const double* ta = sm.a[cur];
        const double* tb = sm.b[cur];
#pragma unroll
        for (int ks = 0; ks < BKT / 4; ++ks) {
            double af[8], bf[4];
#pragma unroll
            for (int mi = 0; mi < 8; ++mi) af[mi] = frag<AK>(ta, wm * 64 + mi * 8 + g, ks * 4 + t);
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) bf[ni] = frag<BK>(tb, wn * 32 + ni * 8 + g, ks * 4 + t);
#pragma unroll
            for (int mi = 0; mi < 8; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
        }
        if (more) {
            stash<AK>(sm.a[cur ^ 1], va);
            stash<BK>(sm.b[cur ^ 1], vb);
        }
        __syncthreads();
    }

    // ---------------------------------------------------------- epilogue
    auto cpow = [&](double c) { return p.self_power == 2 ? c * c : c; };
    auto weight = [&](int rl, int cl) {
        double w = p.scale;
        for (int f = 0; f < p.w.nf; ++f) w *= __ldg(p.w.ptr[f] + sm.woff_r[f][rl] + sm.woff_c[f][cl]);
        return w;
    };

    if (p.mode == kEpiStore) {
#pragma unroll
        for (int mi = 0; mi < 8; ++mi) {
            const int rl = wm * 64 + mi * 8 + g;
            const long long r = r0 + rl;
            if (r >= p.rows) continue;
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) {
                const int cl = wn * 32 + ni * 8 + 2 * t;
                const long long c = c0 + cl;
                double* dst = p.out + r * p.cols + c;
                const double v0 = cpow(acc[mi][ni][0]) * weight(rl, cl);
                if (c + 1 < p.cols) {
                    const double v1 = cpow(acc[mi][ni][1]) * weight(rl, cl + 1);
                    if (p.accumulate) {
                        dst[0] += v0;
                        dst[1] += v1;
                    } else if ((reinterpret_cast<unsigned long long>(dst) & 15) == 0) {
                        *reinterpret_cast<double2*>(dst) = make_double2(v0, v1);
                    } else {
                        dst[0] = v0;
                        dst[1] = v1;
                    }
                } else if (c < p.cols) {
                    dst[0] = p.accumulate ? dst[0] + v0 : v0;
                }
            }
        }
        return;
    }

    // reductions: masked values contribute 0 (acc is 0 there, weights finite)
    auto val = [&](int mi, int ni, int h) {
        const int rl = wm * 64 + mi * 8 + g, cl = wn * 32 + ni * 8 + 2 * t + h;
        if (r0 + rl >= p.rows || c0 + cl >= p.cols) return 0.0;
        return cpow(acc[mi][ni][h]) * weight(rl, cl);
    };

    if (p.mode == kEpiSumAll) {
        double s = 0.0;
#pragma unroll
        for (int mi = 0; mi < 8; ++mi)
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) s += val(mi, ni, 0) + val(mi, ni, 1);
        s = warp_sum(s);
        if (lane == 0) sm.red[0][warp] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
            double tot = 0.0;
            for (int w = 0; w < THREADS / 32; ++w) tot += sm.red[0][w];
            p.partial[blockIdx.x] = tot;
        }
        return;
    }

    if (p.mode == kEpiSumCols) {  // out[r] = sum_c
#pragma unroll
        for (int mi = 0; mi < 8; ++mi) {
            double s = 0.0;
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) s += val(mi, ni, 0) + val(mi, ni, 1);
            s += __shfl_xor_sync(0xffffffffu, s, 1);
            s += __shfl_xor_sync(0xffffffffu, s, 2);
            if (t == 0) sm.red[wn][wm * 64 + mi * 8 + g] = s;
        }
        __syncthreads();
        for (int rl = threadIdx.x; rl < BM; rl += THREADS) {
            const long long r = r0 + rl;
            if (r < p.rows)
                p.partial[tn * p.rows + r] = ((sm.red[0][rl] + sm.red[1][rl]) + sm.red[2][rl]) + sm.red[3][rl];
        }
        return;
    }

    // kEpiSumRows: out[c] = sum_r
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            double s = 0.0;
#pragma unroll
            for (int mi = 0; mi < 8; ++mi) s += val(mi, ni, h);
            s += __shfl_xor_sync(0xffffffffu, s, 4);
            s += __shfl_xor_sync(0xffffffffu, s, 8);
            s += __shfl_xor_sync(0xffffffffu, s, 16);
            if (g == 0) sm.red[wm][wn * 32 + ni * 8 + 2 * t + h] = s;
        }
    }
    __syncthreads();
    for (int cl = threadIdx.x; cl < BN; cl += THREADS) {
        const long long c = c0 + cl;
        if (c < p.cols) p.partial[tm * p.cols + c] = sm.red[0][cl] + sm.red[1][cl];
    }
}

__global__ void gemm_finalize_scalar(const double* partial, long long P, double* out, int accumulate) {
    __shared__ double red[32];
    double acc = 0.0;
    for (long long i = threadIdx.x; i < P; i += blockDim.x) acc += partial[i];
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        v = warp_sum(v);
        if (threadIdx.x == 0) out[0] = (accumulate ? out[0] : 0.0) + v;
    }
}

__global__ void gemm_finalize_vector(const double* partial, long long P, long long len, double* out, int accumulate) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= len) return;
    double acc = 0.0;
    for (long long q = 0; q < P; ++q) acc += partial[q * len + i];
    out[i] = (accumulate ? out[i] : 0.0) + acc;
}

template <bool AK, bool BK>
void launch_variant(const GemmArgs& a, cudaStream_t s) {
    set_max_smem_once(reinterpret_cast<const void*>(gemm_f64_kernel<AK, BK>), static_cast<int>(sizeof(Smem)));
    const long long total = ((a.rows + BM - 1) / BM) * ((a.cols + BN - 1) / BN);
    const long long tiles = a.tile_count < 0 ? total - a.tile_begin : a.tile_count;
    if (tiles > 0) gemm_f64_kernel<AK, BK><<<static_cast<unsigned>(tiles), THREADS, sizeof(Smem), s>>>(a);
}

}  // namespace

std::size_t gemm_partial_entries(const GemmArgs& a) {
    const long long tm = (a.rows + BM - 1) / BM, tn = (a.cols + BN - 1) / BN;
    switch (a.mode) {
        case kEpiSumAll: return static_cast<std::size_t>(tm * tn);
        case kEpiSumCols: return static_cast<std::size_t>(tn * a.rows);
        case kEpiSumRows: return static_cast<std::size_t>(tm * a.cols);
        default: return 0;
    }
}

// gemm_tma.cu: plain-store TMA launch (1) or -1 when not eligible / a reduction
long long launch_gemm_tma(const GemmArgs& a, cudaStream_t s);

int launch_gemm(const GemmArgs& a, cudaStream_t s) {
    const long long launched = launch_gemm_tma(a, s);
    if (launched > 0) {
        // shared finalize below
    } else if (a.a_kmajor) {
        if (a.b_kmajor) launch_variant<true, true>(a, s);
        else launch_variant<true, false>(a, s);
    } else {
        if (a.b_kmajor) launch_variant<false, true>(a, s);
        else launch_variant<false, false>(a, s);
    }
    const long long tm = (a.rows + BM - 1) / BM, tn = (a.cols + BN - 1) / BN;
    if (a.mode == kEpiSumAll) {
        const long long blocks = a.tile_count < 0 ? tm * tn - a.tile_begin : a.tile_count;
        gemm_finalize_scalar<<<1, 1024, 0, s>>>(a.partial, blocks, a.out, a.accumulate);
    } else if (a.mode == kEpiSumCols) {
        gemm_finalize_vector<<<static_cast<unsigned>((a.rows + 255) / 256), 256, 0, s>>>(a.partial, tn, a.rows, a.out,
                                                                                         a.accumulate);
    } else if (a.mode == kEpiSumRows) {
        gemm_finalize_vector<<<static_cast<unsigned>((a.cols + 255) / 256), 256, 0, s>>>(a.partial, tm, a.cols, a.out,
                                                                                         a.accumulate);
    } else {
        return 1;
    }
    return 2;
}

}  // namespace ustats::dev
