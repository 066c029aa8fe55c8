// FP64 GEMM emulated on the 5th-generation INT8 tensor cores (tcgen05.mma
// kind::i8, accumulators in TMEM) — the Ozaki splitting scheme:
//
//   every row x of an operand is scaled by a power of two 2^-e (e = the
//   exponent of the row's largest |x|, so |x 2^-e| < 1) and cut into S signed
//   7-bit digits, x 2^-e = sum_{t<S} 2^{-7(t+1)} x_t, x_t in [-127, 127]
//   (each digit is an exact subtraction: no rounding);
//   C = A B^T = 2^{eA_i + eB_j} sum_{t+u<S} 2^{-7(t+u+2)} (A_t B_u^T)
//
// Each digit product A_t B_u^T is an exact int8 x int8 -> int32 tensor-core
// GEMM; products of one diagonal d = t+u share a TMEM accumulator (exact while
// (d+1) K 127^2 < 2^31). The dropped products (t+u >= S) bound the error by
// ~2^{-7S} K max|A_i| max|B_j| per entry: S = 7 keeps it below 1e-14 of the
// row-scale product. The FP64 result is assembled from the S int32 diagonals
// in a fixed order, so it is deterministic (and bitwise symmetric for A B^T
// with B = A).
//
// Operand digits live in global memory pre-tiled in the tensor core's K-major
// "core matrix" layout (tiles of TH rows x 64 bytes: four 16-byte K chunks,
// each TH rows x 16 B), so each stage is a handful of 1-D bulk copies.
#include <cstdint>
#include <cstdio>

#include "kernels.hpp"

namespace ustats::dev {

namespace {

constexpr int OZ_BM = 128, OZ_BN = 64, OZ_BK = 64;  // tile rows, tile cols, K bytes per stage
constexpr int OZ_STAGES = 2;
constexpr int OZ_THREADS = 128;

__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ unsigned long long umma_desc(unsigned smem_addr, unsigned lbo, unsigned sbo) {
    unsigned long long d = 0;
    d |= static_cast<unsigned long long>((smem_addr >> 4) & 0x3FFF);
    d |= static_cast<unsigned long long>((lbo >> 4) & 0x3FFF) << 16;
    d |= static_cast<unsigned long long>((sbo >> 4) & 0x3FFF) << 32;
    d |= 1ull << 46;  // descriptor version (sm_100); no swizzle, base offset 0
    return d;
}

__device__ __forceinline__ void bar_init(unsigned long long* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count));
}
__device__ __forceinline__ void bar_expect(unsigned long long* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(unsigned long long* b, unsigned parity) {
    asm volatile(
        "{\n.reg .pred p;\nOZW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra OZW_%=;\n}\n" ::"r"(
            su32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
        "l"(reinterpret_cast<unsigned long long>(src)), "r"(bytes), "r"(su32(bar))
        : "memory");
}

struct OzSmem {
    int8_t a[OZ_STAGES][kOzMaxSlices][OZ_BM * OZ_BK];  // 8 KiB per slice
    int8_t b[OZ_STAGES][kOzMaxSlices][OZ_BN * OZ_BK];  // 4 KiB per slice
    unsigned long long full[OZ_STAGES], empty[OZ_STAGES], done;
    unsigned tmem;
};

// One 128 x 64 output tile per CTA. Warp 0 lane 0 streams the digit tiles,
// warp 1 lane 0 issues the MMAs, all four warps assemble the FP64 tile.
__global__ void __launch_bounds__(OZ_THREADS, 1) ozaki_gemm_kernel(OzakiArgs p) {
    extern __shared__ unsigned char oz_raw[];
    OzSmem& sm = *reinterpret_cast<OzSmem*>((reinterpret_cast<unsigned long long>(oz_raw) + 1023) & ~1023ull);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int S = p.slices;
    const long long tiles_n = p.npad / OZ_BN;
    long long tm, tn;
    if (p.symmetric) {  // upper tiles (by 128-row blocks) in column order
        // tile t of the column-ordered list of (tm, tn) with 128 tm < 64 (tn + 1)
        long long t = blockIdx.x, col = 0;
        for (;; ++col) {
            const long long h = (64 * (col + 1) + OZ_BM - 1) / OZ_BM;  // row tiles touching the upper part
            if (t < h) break;
            t -= h;
        }
        tm = t;
        tn = col;
    } else {
        tm = blockIdx.x / tiles_n;
        tn = blockIdx.x % tiles_n;
    }
    const long long kt_count = p.kpad / OZ_BK;
    const int8_t* abase = p.a + tm * kt_count * (OZ_BM * OZ_BK);
    const int8_t* bbase = p.b + tn * kt_count * (OZ_BN * OZ_BK);

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&sm.tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 32) {
        for (int s = 0; s < OZ_STAGES; ++s) {
            bar_init(&sm.full[s], 1);
            bar_init(&sm.empty[s], 1);
        }
        bar_init(&sm.done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const unsigned tmem = sm.tmem;

    if (tid == 0) {  // producer
        const unsigned bytes = static_cast<unsigned>(S) * (OZ_BM + OZ_BN) * OZ_BK;
        for (long long kt = 0; kt < kt_count; ++kt) {
            const int s = static_cast<int>(kt % OZ_STAGES);
            if (kt >= OZ_STAGES) bar_wait(&sm.empty[s], static_cast<unsigned>(((kt / OZ_STAGES) - 1) & 1));
            bar_expect(&sm.full[s], bytes);
            for (int t = 0; t < S; ++t) {
                bulk_load(sm.a[s][t], abase + t * p.a_slice + kt * (OZ_BM * OZ_BK), OZ_BM * OZ_BK, &sm.full[s]);
                bulk_load(sm.b[s][t], bbase + t * p.b_slice + kt * (OZ_BN * OZ_BK), OZ_BN * OZ_BK, &sm.full[s]);
            }
        }
    } else if (tid == 32) {  // MMA issuer
        // kind::i8, int32 accumulate, signed A and B, both K-major, N = 64, M = 128
        const unsigned idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((OZ_BN >> 3) << 17) | ((OZ_BM >> 4) << 24);
        for (long long kt = 0; kt < kt_count; ++kt) {
            const int s = static_cast<int>(kt % OZ_STAGES);
            bar_wait(&sm.full[s], static_cast<unsigned>((kt / OZ_STAGES) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;");
            for (int t = 0; t < S; ++t)
                for (int u = 0; t + u < S; ++u) {
                    const unsigned acc = tmem + static_cast<unsigned>((t + u) * OZ_BN);
                    for (int ks = 0; ks < OZ_BK / 32; ++ks) {
                        // 32 K bytes = two 16-byte chunks: chunk stride = rows x 16 B
                        const unsigned long long da =
                            umma_desc(su32(sm.a[s][t]) + ks * 2 * OZ_BM * 16, OZ_BM * 16, 128);
                        const unsigned long long db =
                            umma_desc(su32(sm.b[s][u]) + ks * 2 * OZ_BN * 16, OZ_BN * 16, 128);
                        const unsigned accumulate = (kt > 0 || ks > 0 || t > 0) ? 1u : 0u;  // first product of diagonal t+u: t = 0
                        asm volatile(
                            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(acc),
                            "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
                    }
                }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                su32(&sm.empty[s])));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&sm.done)));
    }
    __syncwarp();
    bar_wait(&sm.done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");

    // epilogue: thread = one row of the tile (TMEM lane), 16 columns at a time
    const long long row = tm * OZ_BM + warp * 32 + lane;
    const bool row_ok = row < p.m;
    const int ea = row_ok ? p.a_exp[row] : 0;
    for (int c0 = 0; c0 < OZ_BN; c0 += 16) {
        double v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = 0.0;
        for (int d = S - 1; d >= 0; --d) {  // smallest contributions first
            unsigned r[16];
            const unsigned addr = tmem + (static_cast<unsigned>(warp * 32) << 16) + static_cast<unsigned>(d * OZ_BN + c0);
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                  "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                : "r"(addr));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            const double scale = ldexp(1.0, -7 * (d + 2));
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] += static_cast<double>(static_cast<int>(r[j])) * scale;
        }
        if (!row_ok) continue;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const long long col = tn * OZ_BN + c0 + j;
            if (col >= p.n) continue;
            const double x = ldexp(v[j], ea + p.b_exp[col]);
            if (p.symmetric && col < row) continue;  // lower part: written by the mirror of (col, row)
            p.c[row * p.ldc + col] = x;
            if (p.symmetric && col != row) p.c[col * p.ldc + row] = x;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// Row exponents: e_i with max_k |x_ik| < 2^e_i (0 for an all-zero row).
__global__ void oz_row_exponents(const double* __restrict__ x, long long rows, long long k, long long rs, long long ks,
                                 int* __restrict__ exps) {
    const long long r = blockIdx.x * static_cast<long long>(blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    double mx = 0.0;
    for (long long c = lane; c < k; c += 32) mx = fmax(mx, fabs(x[r * rs + c * ks]));
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) {
        int e = 0;
        if (mx > 0.0) frexp(mx, &e);  // mx = f 2^e, f in [0.5, 1): |x| 2^-e < 1
        exps[r] = e;
    }
}

// Digits into the tiled core-matrix layout: thread = (row, 16-byte K chunk).
__global__ void oz_split(const double* __restrict__ x, long long rows, long long k, long long rs, long long ks,
                         const int* __restrict__ exps, int th, long long rows_pad, long long kpad, int slices,
                         long long slice_bytes, int8_t* __restrict__ out) {
    const long long chunks = kpad / 16;
    const long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (g >= rows_pad * chunks) return;
    const long long r = g % rows_pad, ch = g / rows_pad;  // consecutive threads: consecutive rows
    const long long kt = ch / (OZ_BK / 16), cin = ch % (OZ_BK / 16);
    const long long rt = r / th, rin = r % th;
    const long long off = (rt * (kpad / OZ_BK) + kt) * (th * OZ_BK) + cin * (th * 16) + rin * 16;
    double v[16];
    const int e = r < rows ? exps[r] : 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const long long c = ch * 16 + j;
        v[j] = (r < rows && c < k) ? ldexp(x[r * rs + c * ks], -e) : 0.0;
    }
    for (int t = 0; t < slices; ++t) {
        unsigned w[4] = {0, 0, 0, 0};
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const double y = v[j] * 128.0;       // exact (power of two)
            const double dgt = trunc(y);         // in [-127, 127]
            v[j] = y - dgt;                      // exact
            const unsigned byte = static_cast<unsigned>(static_cast<int>(dgt)) & 0xFFu;
            w[j >> 2] |= byte << ((j & 3) * 8);
        }
        *reinterpret_cast<uint4*>(out + t * slice_bytes + off) = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

}  // namespace

std::size_t ozaki_slice_bytes(long long rows, long long k, int tile_rows) {
    const long long rp = (rows + tile_rows - 1) / tile_rows * tile_rows;
    const long long kp = (k + OZ_BK - 1) / OZ_BK * OZ_BK;
    return static_cast<std::size_t>(rp * kp);
}

int ozaki_split(const double* x, long long rows, long long k, long long rs, long long ks, int tile_rows, int slices,
                int8_t* out, int* exps, cudaStream_t s) {
    if (slices < 1 || slices > kOzMaxSlices) return -1;
    const long long rp = (rows + tile_rows - 1) / tile_rows * tile_rows;
    const long long kp = (k + OZ_BK - 1) / OZ_BK * OZ_BK;
    oz_row_exponents<<<static_cast<unsigned>((rows + 7) / 8), 256, 0, s>>>(x, rows, k, rs, ks, exps);
    const long long threads = rp * (kp / 16);
    oz_split<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, s>>>(x, rows, k, rs, ks, exps, tile_rows, rp, kp,
                                                                        slices, rp * kp, out);
    return 2;
}

long long ozaki_tile_count(const OzakiArgs& p) {
    const long long tiles_n = p.npad / 64;
    if (!p.symmetric) return (p.mpad / 128) * tiles_n;
    long long total = 0;
    for (long long col = 0; col < tiles_n; ++col) total += (64 * (col + 1) + 127) / 128;
    return total;
}

int launch_ozaki_gemm(const OzakiArgs& p, cudaStream_t s) {
    if (p.slices < 1 || p.slices > kOzMaxSlices || p.kpad % OZ_BK != 0) return -1;
    const int bytes = static_cast<int>(sizeof(OzSmem)) + 1024;
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(ozaki_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        configured = true;
    }
    const long long tiles = ozaki_tile_count(p);
    if (tiles <= 0) return 0;
    ozaki_gemm_kernel<<<static_cast<unsigned>(tiles), OZ_THREADS, bytes, s>>>(p);
    return 1;
}

}  // namespace ustats::dev
