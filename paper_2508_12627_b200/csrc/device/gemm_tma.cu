// FP64 tensor-core GEMM fed by TMA — the executor's hot kernel for every
// two-operand contraction whose operands are plain strided matrices (the
// reference's gemm_step, proj/src/einsum.cpp:209-259, which transposes both
// operands into scratch copies and calls Eigen; here the transposes are TMA
// box orientations and nothing is copied).
//
// sm_100a has no tcgen05 kind::f64, so the math is warp-level
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4). Data movement is Blackwell-native:
//   * one thread issues cp.async.bulk.tensor (TMA) boxes into a 4-stage
//     shared-memory ring with 128B swizzle; completion is tracked by
//     mbarrier transaction counts (full[s]); consumers release a stage by
//     arriving on empty[s]; the refill for k-tile kt+4 is issued as soon as
//     all 8 warps have drained stage kt%4 — no block-wide barrier in the loop;
//   * operand tiles are k-major (box 16k x 128 rows) or row-major-along-m
//     (8 boxes of 16m x 16k) depending on which global stride is unit, so
//     transposed reads cost nothing;
//   * 128x128 CTA tile, 8 warps as 2x4, 64x32 warp tile (8x4 DMMA tiles,
//     64 FP64 accumulators per thread), grouped rasterization for L2 reuse;
//   * epilogues shared with the gather kernel (store / fused Hadamard +
//     fixed-order reductions).
#include <cuda.h>

#include <mutex>

#include "kernels.hpp"

namespace ustats::dev {

namespace {

constexpr int BM = 128, BN = 128, BK = 16, STAGES = 4, THREADS = 256;
constexpr int TILE_DOUBLES = BM * BK;              // 2048 doubles = 16 KiB
constexpr unsigned STAGE_BYTES = 2u * TILE_DOUBLES * 8u;
constexpr int GROUP_M = 8;

struct alignas(1024) TmaSmem {
    double a[STAGES][TILE_DOUBLES];
    double b[STAGES][TILE_DOUBLES];
    unsigned long long full[STAGES];
    unsigned long long empty[STAGES];
    long long woff_r[kMaxGemmFactors][BM];
    long long woff_c[kMaxGemmFactors][BN];
    double red[4][BM];
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// Element (row m, k) of a swizzled operand tile.
//  k-major: 128 rows x 128 B; 16-byte chunk index (k/2) XOR (m%8).
//  m-major: 8 boxes of [16 k-rows x 128 B]; chunk ((m%16)/2) XOR (k%8).
template <bool KMAJOR>
__device__ __forceinline__ double tile_at(const double* tile, int m, int k) {
    if (KMAJOR) {
        const int chunk = (k >> 1) ^ (m & 7);
        return tile[m * 16 + chunk * 2 + (k & 1)];
    } else {
        const int chunk = ((m & 15) >> 1) ^ (k & 7);
        return tile[(m >> 4) * 256 + k * 16 + chunk * 2 + (m & 1)];
    }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

struct TmaArgs {
    GemmArgs g;
    int a_kmajor, b_kmajor;
};

template <bool AK, bool BKM>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_tma_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                    TmaArgs args) {
    const GemmArgs& p = args.g;
    extern __shared__ unsigned char smem_raw[];
    TmaSmem& sm = *reinterpret_cast<TmaSmem*>(
        (reinterpret_cast<unsigned long long>(smem_raw) + 1023ull) & ~1023ull);

    const long long tiles_m = (p.rows + BM - 1) / BM, tiles_n = (p.cols + BN - 1) / BN;
    const long long bid = blockIdx.x;
    long long tm, tn;
    if (p.symmetric_out) {
        // upper-triangular tiles, row by row: row tm holds tiles tm..tiles_n-1
        long long rest = bid;
        tm = 0;
        while (rest >= tiles_n - tm) {
            rest -= tiles_n - tm;
            ++tm;
        }
        tn = tm + rest;
    } else {
        const long long width = GROUP_M * tiles_n;
        const long long group = bid / width, first_m = group * GROUP_M;
        const long long gsz = (tiles_m - first_m) < GROUP_M ? (tiles_m - first_m) : GROUP_M;
        tm = first_m + (bid % width) % gsz;
        tn = (bid % width) / gsz;
    }
    const bool mirror = p.symmetric_out && tm != tn;
    const int r0 = static_cast<int>(tm * BM), c0 = static_cast<int>(tn * BN);
    const int KT = static_cast<int>((p.n + BK - 1) / BK);

    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], THREADS / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    auto issue = [&](int kt, int s) {
        mbar_expect_tx(&sm.full[s], STAGE_BYTES);
        const int k0 = kt * BK;
        if (AK) {
            tma_load_2d(sm.a[s], &map_a, k0, r0, &sm.full[s]);
        } else {
#pragma unroll
            for (int q = 0; q < BM / 16; ++q) tma_load_2d(sm.a[s] + q * 256, &map_a, r0 + 16 * q, k0, &sm.full[s]);
        }
        if (BKM) {
            tma_load_2d(sm.b[s], &map_b, k0, c0, &sm.full[s]);
        } else {
#pragma unroll
            for (int q = 0; q < BN / 16; ++q) tma_load_2d(sm.b[s] + q * 256, &map_b, c0 + 16 * q, k0, &sm.full[s]);
        }
    };

    if (tid == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<unsigned long long>(&map_a)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<unsigned long long>(&map_b)) : "memory");
        for (int kt = 0; kt < STAGES && kt < KT; ++kt) issue(kt, kt);
    }
    // epilogue offsets can be computed while the first stages land
    if (p.w.nf) {
        for (int i = tid; i < p.w.nf * BM; i += THREADS) {
            const int f = i / BM, r = i % BM;
            long long g = r0 + r, o = 0;
            if (g < p.rows)
                for (int d = p.a.nr - 1; d >= 0; --d) {
                    const long long q = g / p.n;
                    o += (g - q * p.n) * p.w.rstride[f][d];
                    g = q;
                }
            sm.woff_r[f][r] = o;
        }
        for (int i = tid; i < p.w.nf * BN; i += THREADS) {
            const int f = i / BN, c = i % BN;
            long long g = c0 + c, o = 0;
            if (g < p.cols)
                for (int d = p.b.nr - 1; d >= 0; --d) {
                    const long long q = g / p.n;
                    o += (g - q * p.n) * p.w.cstride[f][d];
                    g = q;
                }
            sm.woff_c[f][c] = o;
        }
    }

    const int warp = tid >> 5, lane = tid & 31;
    const int wm = warp >> 2, wn = warp & 3;
    const int g = lane >> 2, t = lane & 3;

    double acc[8][4][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (int kt = 0; kt < KT; ++kt) {
        const int s = kt % STAGES;
        const unsigned ph = static_cast<unsigned>((kt / STAGES) & 1);
        mbar_wait(&sm.full[s], ph);
        const double* ta = sm.a[s];
        const double* tb = sm.b[s];
#pragma unroll
        for (int ks = 0; ks < BK / 4; ++ks) {
            double af[8], bf[4];
#pragma unroll
            for (int mi = 0; mi < 8; ++mi) af[mi] = tile_at<AK>(ta, wm * 64 + mi * 8 + g, ks * 4 + t);
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) bf[ni] = tile_at<BKM>(tb, wn * 32 + ni * 8 + g, ks * 4 + t);
#pragma unroll
            for (int mi = 0; mi < 8; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[s]);
        if (tid == 0 && kt + STAGES < KT) {
            mbar_wait(&sm.empty[s], ph);
            issue(kt + STAGES, s);
        }
    }
    __syncthreads();  // epilogue offsets visible

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
                    if ((reinterpret_cast<unsigned long long>(dst) & 15) == 0)
                        *reinterpret_cast<double2*>(dst) = make_double2(v0, v1);
                    else {
                        dst[0] = v0;
                        dst[1] = v1;
                    }
                    if (mirror) {
                        p.out[c * p.cols + r] = v0;
                        p.out[(c + 1) * p.cols + r] = v1;
                    }
                } else if (c < p.cols) {
                    dst[0] = v0;
                    if (mirror) p.out[c * p.cols + r] = v0;
                }
            }
        }
        return;
    }

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
        if (tid == 0) {
            double tot = 0.0;
            for (int w = 0; w < THREADS / 32; ++w) tot += sm.red[0][w];
            p.partial[blockIdx.x] = mirror ? 2.0 * tot : tot;
        }
        return;
    }

    if (p.mode == kEpiSumCols) {
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
        for (int rl = tid; rl < BM; rl += THREADS) {
            const long long r = r0 + rl;
            if (r < p.rows)
                p.partial[tn * p.rows + r] = ((sm.red[0][rl] + sm.red[1][rl]) + sm.red[2][rl]) + sm.red[3][rl];
        }
        return;
    }

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
    for (int cl = tid; cl < BN; cl += THREADS) {
        const long long c = c0 + cl;
        if (c < p.cols) p.partial[tm * p.cols + c] = sm.red[0][cl] + sm.red[1][cl];
    }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encoder() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    return fn;
}

// A plain operand: one factor whose row digits flatten to a single stride.
bool plain(const GemmSide& s, long long n, long long& rs, long long& ks) {
    if (s.nf != 1) return false;
    rs = s.rstride[0][s.nr - 1];
    for (int d = s.nr - 1; d > 0; --d)
        if (s.rstride[0][d - 1] != s.rstride[0][d] * n) return false;
    ks = s.kstride[0];
    return true;
}

bool encode(CUtensorMap* map, const double* ptr, bool kmajor, long long rows, long long K, long long rs,
            long long ks) {
    EncodeFn fn = encoder();
    if (!fn) return false;
    cuuint64_t dims[2], strides[1];
    cuuint32_t box[2], estr[2] = {1, 1};
    if (kmajor) {
        dims[0] = static_cast<cuuint64_t>(K);
        dims[1] = static_cast<cuuint64_t>(rows);
        strides[0] = static_cast<cuuint64_t>(rs) * 8;
        box[0] = BK;
        box[1] = BM;
    } else {
        dims[0] = static_cast<cuuint64_t>(rows);
        dims[1] = static_cast<cuuint64_t>(K);
        strides[0] = static_cast<cuuint64_t>(ks) * 8;
        box[0] = 16;
        box[1] = BK;
    }
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(ptr), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <bool AK, bool BKM>
long long launch_tma(const CUtensorMap& ma, const CUtensorMap& mb, const TmaArgs& args, cudaStream_t s) {
    static std::once_flag once;
    const int bytes = static_cast<int>(sizeof(TmaSmem)) + 1024;
    std::call_once(once, [&] {
        cudaFuncSetAttribute(gemm_tma_kernel<AK, BKM>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    });
    const long long tm = (args.g.rows + BM - 1) / BM, tn = (args.g.cols + BN - 1) / BN;
    const long long tiles = args.g.symmetric_out ? tm * (tm + 1) / 2 : tm * tn;
    gemm_tma_kernel<AK, BKM><<<static_cast<unsigned>(tiles), THREADS, bytes, s>>>(ma, mb, args);
    return tiles;
}

}  // namespace

bool gemm_tma_eligible(const GemmArgs& a, int* a_kmajor_out, int* b_kmajor_out) {
    int ak_local = 1, bk_local = 1;
    int* a_kmajor = a_kmajor_out ? a_kmajor_out : &ak_local;
    int* b_kmajor = b_kmajor_out ? b_kmajor_out : &bk_local;
    long long ars, aks, brs, bks;
    if (!plain(a.a, a.n, ars, aks) || !plain(a.b, a.n, brs, bks)) return false;
    if (a.rows >= (1ll << 31) || a.cols >= (1ll << 31) || a.n >= (1ll << 31)) return false;
    auto layout = [](const double* ptr, long long rs, long long ks, int* km) {
        if ((reinterpret_cast<unsigned long long>(ptr) & 15) != 0) return false;
        if (ks == 1 && rs > 0 && (rs % 2) == 0) {
            *km = 1;
            return true;
        }
        if (rs == 1 && ks > 0 && (ks % 2) == 0) {
            *km = 0;
            return true;
        }
        return false;
    };
    return layout(a.a.ptr[0], ars, aks, a_kmajor) && layout(a.b.ptr[0], brs, bks, b_kmajor) && encoder() != nullptr;
}

long long launch_gemm_tma(const GemmArgs& in, cudaStream_t s) {
    int ak = 1, bk = 1;
    if (!gemm_tma_eligible(in, &ak, &bk)) return -1;
    GemmArgs a = in;
    // upper tiles only for symmetric store / full reductions with square output
    if (a.symmetric_out && !(a.rows == a.cols && (a.mode == kEpiStore || a.mode == kEpiSumAll))) a.symmetric_out = 0;
    long long ars, aks, brs, bks;
    plain(a.a, a.n, ars, aks);
    plain(a.b, a.n, brs, bks);
    CUtensorMap ma, mb;
    if (!encode(&ma, a.a.ptr[0], ak, a.rows, a.n, ars, aks) || !encode(&mb, a.b.ptr[0], bk, a.cols, a.n, brs, bks))
        return -1;
    TmaArgs args{a, ak, bk};
    if (ak) return bk ? launch_tma<true, true>(ma, mb, args, s) : launch_tma<true, false>(ma, mb, args, s);
    return bk ? launch_tma<false, true>(ma, mb, args, s) : launch_tma<false, false>(ma, mb, args, s);
}

}  // namespace ustats::dev
