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

#include <cmath>
#include <mutex>

#include "epilogue.cuh"
#include "kernels.hpp"

namespace ustats::dev {

namespace {

constexpr int BM = 128, BN = 128, BK = 16, STAGES = 4, THREADS = 256;
constexpr int TILE_DOUBLES = BM * BK;              // 2048 doubles = 16 KiB
constexpr unsigned STAGE_BYTES = 2u * TILE_DOUBLES * 8u;
constexpr int GROUP_M = 8;
constexpr int TP = BN + 1;                          // staged accumulator tile pitch (odd: conflict-free columns)

struct alignas(1024) TmaSmem {
    union {
        struct {
            double a[STAGES][TILE_DOUBLES];
            double b[STAGES][TILE_DOUBLES];
        } st;
        double tile[BM * TP];
    } u;
    unsigned long long full[STAGES];
    unsigned long long empty[STAGES];
    double red[THREADS / 32];
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
    long long rows, cols, n;
    long long tile_begin;  // row sharding: first tile of this rank's range
    int symmetric;
    int colmajor;          // symmetric list ordered by column: tile (tm <= tn) at tn(tn+1)/2 + tm
    int accumulate;        // outputs += (pre-zeroed)
    // Split-K tail (the last, partial wave): phase 1 computes K-slices of the
    // leftover tiles into kpart, phase 2 sums the slices in order and runs the
    // epilogues; phase 0 is the ordinary full-K tile.
    int phase;
    int ksplit;
    long long slot_base;   // reduction-partial slot of this launch's first tile
    double* kpart;
    EpiSet epis;
};

template <bool AK, bool BKM>
__global__ void __launch_bounds__(THREADS, 1)
    gemm_tma_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                    const __grid_constant__ TmaArgs p) {
    extern __shared__ unsigned char smem_raw[];
    TmaSmem& sm = *reinterpret_cast<TmaSmem*>(
        (reinterpret_cast<unsigned long long>(smem_raw) + 1023ull) & ~1023ull);

    const long long tiles_m = (p.rows + BM - 1) / BM, tiles_n = (p.cols + BN - 1) / BN;
    const long long local = p.phase == 1 ? blockIdx.x / p.ksplit : blockIdx.x;
    const int slice = p.phase == 1 ? static_cast<int>(blockIdx.x % p.ksplit) : 0;
    const long long bid = p.tile_begin + local;
    long long tm, tn;
    if (p.symmetric && p.colmajor) {
        // column by column: column tn holds tiles 0..tn (panels <= tn)
        tn = static_cast<long long>((sqrt(8.0 * static_cast<double>(bid) + 1.0) - 1.0) * 0.5);
        while (tn * (tn + 1) / 2 > bid) --tn;
        while ((tn + 1) * (tn + 2) / 2 <= bid) ++tn;
        tm = bid - tn * (tn + 1) / 2;
    } else if (p.symmetric) {
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
    const bool mirror = p.symmetric && tm != tn;
    const int r0 = static_cast<int>(tm * BM), c0 = static_cast<int>(tn * BN);
    const int KT = static_cast<int>((p.n + BK - 1) / BK);
    const int kt0 = p.phase == 1 ? static_cast<int>(static_cast<long long>(KT) * slice / p.ksplit) : 0;
    const int kt1 = p.phase == 1 ? static_cast<int>(static_cast<long long>(KT) * (slice + 1) / p.ksplit) : KT;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    double* tile = sm.u.tile;

    if (p.phase != 2) {
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
                tma_load_2d(sm.u.st.a[s], &map_a, k0, r0, &sm.full[s]);
            } else {
#pragma unroll
                for (int q = 0; q < BM / 16; ++q) tma_load_2d(sm.u.st.a[s] + q * 256, &map_a, r0 + 16 * q, k0, &sm.full[s]);
            }
            if (BKM) {
                tma_load_2d(sm.u.st.b[s], &map_b, k0, c0, &sm.full[s]);
            } else {
#pragma unroll
                for (int q = 0; q < BN / 16; ++q) tma_load_2d(sm.u.st.b[s] + q * 256, &map_b, c0 + 16 * q, k0, &sm.full[s]);
            }
        };

        if (tid == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<unsigned long long>(&map_a)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<unsigned long long>(&map_b)) : "memory");
            for (int j = 0; j < STAGES && kt0 + j < kt1; ++j) issue(kt0 + j, j);
        }

        const int wm = warp >> 2, wn = warp & 3;
        const int g = lane >> 2, t = lane & 3;

        double acc[8][4][2];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

        for (int j = 0; j < kt1 - kt0; ++j) {
            const int s = j % STAGES;
            const unsigned ph = static_cast<unsigned>((j / STAGES) & 1);
            mbar_wait(&sm.full[s], ph);
            const double* ta = sm.u.st.a[s];
            const double* tb = sm.u.st.b[s];
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
            if (tid == 0 && kt0 + j + STAGES < kt1) {
                mbar_wait(&sm.empty[s], ph);
                issue(kt0 + j + STAGES, s);
            }
        }

        if (p.phase == 1) {  // a K-slice of a tail tile: raw accumulators out, no epilogue
            double* dst = p.kpart + static_cast<long long>(blockIdx.x) * (BM * BN);
#pragma unroll
            for (int mi = 0; mi < 8; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) {
                    const int r = wm * 64 + mi * 8 + g, c = wn * 32 + ni * 8 + 2 * t;
                    *reinterpret_cast<double2*>(dst + r * BN + c) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
                }
            return;
        }
        __syncthreads();  // every stage consumed: the ring becomes the accumulator tile
#pragma unroll
        for (int mi = 0; mi < 8; ++mi)
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) {
                const int r = wm * 64 + mi * 8 + g, c = wn * 32 + ni * 8 + 2 * t;
                tile[r * TP + c] = acc[mi][ni][0];
                tile[r * TP + c + 1] = acc[mi][ni][1];
            }
    } else {
        // phase 2: the tile is the in-order sum of its K-slices
        const double* src = p.kpart + static_cast<long long>(blockIdx.x) * p.ksplit * (BM * BN);
        for (int i = tid; i < BM * BN; i += THREADS) {
            double v = 0.0;
            for (int sl = 0; sl < p.ksplit; ++sl) v += src[static_cast<long long>(sl) * (BM * BN) + i];
            tile[(i >> 7) * TP + (i & 127)] = v;
        }
    }
    __syncthreads();
    const long long slot = p.slot_base + blockIdx.x;

    epi::apply<THREADS>(p.epis, p.rows, p.cols, p.accumulate, tile, r0, c0, tm, tn, mirror, slot, sm.red, tid,
                        [] { __syncthreads(); });
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
void launch_tma(const CUtensorMap& ma, const CUtensorMap& mb, const TmaArgs& args, long long grid, cudaStream_t s) {
    const int bytes = static_cast<int>(sizeof(TmaSmem)) + 1024;
    set_max_smem_once(reinterpret_cast<const void*>(gemm_tma_kernel<AK, BKM>), bytes);
    if (grid > 0) gemm_tma_kernel<AK, BKM><<<static_cast<unsigned>(grid), THREADS, bytes, s>>>(ma, mb, args);
}

int sm_count_cached() {
    static int sms = 0;
    static std::once_flag once;
    std::call_once(once, [] {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    });
    return sms;
}

__global__ void epi_finalize_scalar(const double* partial, long long P, double* out, int accumulate) {
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

__global__ void epi_finalize_vector(const double* partial, long long P, long long len, double* out, int accumulate) {
    const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (i >= len) return;
    double acc = 0.0;
    for (long long q = 0; q < P; ++q) acc += partial[q * len + i];
    out[i] = (accumulate ? out[i] : 0.0) + acc;
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

std::size_t gemm_epi_partial_entries(const GemmArgs& a, int mode) {
    const long long tm = (a.rows + BM - 1) / BM, tn = (a.cols + BN - 1) / BN;
    switch (mode) {
        case kEpiSumAll: return static_cast<std::size_t>(tm * tn);
        case kEpiSumCols: return static_cast<std::size_t>(tn * a.rows);
        case kEpiSumRows: return static_cast<std::size_t>(tm * a.cols);
        default: return 0;
    }
}

int launch_gemm_multi(const GemmArgs& a, const EpiSet& epis, cudaStream_t s) {
    int ak = 1, bk = 1;
    if (!gemm_tma_eligible(a, &ak, &bk) || epis.count < 1 || epis.count > kMaxEpilogues) return -1;
    long long ars, aks, brs, bks;
    plain(a.a, a.n, ars, aks);
    plain(a.b, a.n, brs, bks);
    CUtensorMap ma, mb;
    if (!encode(&ma, a.a.ptr[0], ak, a.rows, a.n, ars, aks) || !encode(&mb, a.b.ptr[0], bk, a.cols, a.n, brs, bks))
        return -1;
    TmaArgs args;
    args.rows = a.rows;
    args.cols = a.cols;
    args.n = a.n;
    args.tile_begin = a.tile_begin;
    args.symmetric = (a.symmetric_out && a.rows == a.cols) ? 1 : 0;
    args.colmajor = a.tri_colmajor;
    args.accumulate = a.accumulate;
    args.phase = 0;
    args.ksplit = 1;
    args.slot_base = 0;
    args.kpart = nullptr;
    args.epis = epis;
    const long long tm_ = (a.rows + BM - 1) / BM, tn_ = (a.cols + BN - 1) / BN;
    const long long total = args.symmetric ? tm_ * (tm_ + 1) / 2 : tm_ * tn_;
    const long long blocks = a.tile_count < 0 ? total - a.tile_begin : a.tile_count;
    if (blocks <= 0) return 0;
    auto go = [&](const TmaArgs& t, long long grid) {
        if (ak) {
            if (bk) launch_tma<true, true>(ma, mb, t, grid, s);
            else launch_tma<true, false>(ma, mb, t, grid, s);
        } else {
            if (bk) launch_tma<false, true>(ma, mb, t, grid, s);
            else launch_tma<false, false>(ma, mb, t, grid, s);
        }
    };
    // The last wave of a multi-wave grid is partial (C2: 2080 tiles = 14.05
    // waves of 148): its tiles are split along K over the idle SMs and
    // re-assembled, so the tail costs ~1/S of a tile instead of a whole tile.
    const int sms = sm_count_cached();
    const long long tail = blocks % sms;
    const int KT = static_cast<int>((a.n + BK - 1) / BK);
    // K-split factor of the tail: the one that finishes it soonest, in units
    // of a full tile (ceil(tail*S / sms) / S), with at least 4 k-tiles per
    // slice and at most 256 MiB of slice partials; used only if it beats
    // running the tail unsplit (row-sharded C2 on 8 GPUs: 260 tiles per rank
    // = 148 + 112, S = 5 -> 1.8 instead of 2 tile times)
    int S = 1;
    if (tail > 0) {
        double best = 1.0;
        for (int c = 2; c <= KT / 4 && c <= 64; ++c) {
            if (static_cast<double>(tail) * c * BM * BN * 8.0 > 268435456.0) break;
            const double t = std::ceil(static_cast<double>(tail) * c / sms) / c;
            if (t < best * 0.95) {
                best = t;
                S = c;
            }
        }
    }
    int launched_kernels = 0;
    if (tail > 0 && S >= 2) {
        go(args, blocks - tail);
        double* kpart = nullptr;
        const std::size_t kbytes = static_cast<std::size_t>(tail) * S * BM * BN * sizeof(double);
        if (cudaMallocAsync(reinterpret_cast<void**>(&kpart), kbytes, s) != cudaSuccess) return -1;
        TmaArgs t1 = args;
        t1.tile_begin = a.tile_begin + blocks - tail;
        t1.phase = 1;
        t1.ksplit = S;
        t1.kpart = kpart;
        go(t1, tail * S);
        TmaArgs t2 = t1;
        t2.phase = 2;
        t2.slot_base = blocks - tail;
        go(t2, tail);
        cudaFreeAsync(kpart, s);
        launched_kernels = 3;
    } else {
        go(args, blocks);
        launched_kernels = 1;
    }
    int launched = launched_kernels + launch_epilogue_finalize(a.rows, a.cols, epis, blocks, a.accumulate, s);
    return launched;
}

int launch_epilogue_finalize(long long rows, long long cols, const EpiSet& epis, long long blocks, int accumulate,
                             cudaStream_t s) {
    const long long tm = (rows + BM - 1) / BM, tn = (cols + BN - 1) / BN;
    int launched = 0;
    for (int q = 0; q < epis.count; ++q) {
        const EpiDesc& d = epis.d[q];
        if (d.mode == kEpiSumAll) {
            epi_finalize_scalar<<<1, 1024, 0, s>>>(d.partial, blocks, d.out, accumulate);
        } else if (d.mode == kEpiSumCols) {
            epi_finalize_vector<<<static_cast<unsigned>((rows + 255) / 256), 256, 0, s>>>(d.partial, tn, rows, d.out,
                                                                                        accumulate);
        } else if (d.mode == kEpiSumRows) {
            epi_finalize_vector<<<static_cast<unsigned>((cols + 255) / 256), 256, 0, s>>>(d.partial, tm, cols, d.out,
                                                                                        accumulate);
        } else {
            continue;
        }
        ++launched;
    }
    return launched;
}

// Single-epilogue entry used by launch_gemm: plain store, or one fused
// epilogue whose weights fit the multi-epilogue form.
long long launch_gemm_tma(const GemmArgs& in, cudaStream_t s) {
    int ak = 1, bk = 1;
    if (!gemm_tma_eligible(in, &ak, &bk)) return -1;
    if (in.w.nf > kMaxEpiW || (in.w.nf > 0 && (in.a.nr != 1 || in.b.nr != 1))) return -1;
    if (in.mode != kEpiStore) return -1;  // reductions go through launch_gemm_multi
    EpiSet e;
    e.count = 1;
    EpiDesc& d = e.d[0];
    d.mode = kEpiStore;
    d.self_power = in.self_power;
    d.nw = in.w.nf;
    for (int f = 0; f < d.nw; ++f) {
        d.wptr[f] = in.w.ptr[f];
        d.wr[f] = in.w.rstride[f][0];
        d.wc[f] = in.w.cstride[f][0];
    }
    d.out = in.out;
    GemmArgs a = in;
    if (a.symmetric_out && a.rows != a.cols) a.symmetric_out = 0;
    const int k = launch_gemm_multi(a, e, s);
    return k >= 0 ? 1 : -1;
}

long long gemm_tile_total(const GemmArgs& a, bool tma_symmetric) {
    const long long tm = (a.rows + BM - 1) / BM, tn = (a.cols + BN - 1) / BN;
    return (tma_symmetric && a.rows == a.cols) ? tm * (tm + 1) / 2 : tm * tn;
}

}  // namespace ustats::dev
