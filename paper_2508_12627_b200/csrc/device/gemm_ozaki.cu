// FP64 GEMM emulated on the 5th-generation INT8 tensor cores (tcgen05.mma
// kind::i8, accumulators in TMEM) — the Ozaki splitting scheme:
//
//   every row x of an operand is scaled by a power of two 2^-e (e = the
//   exponent of the row's largest |x|, so |x 2^-e| < 1), truncated to the
//   integer m = trunc(x 2^{8S-2-e}) (|m| < 2^{8S-2}) and written in balanced
//   base 256: m = sum_{t<S} 256^{S-1-t} x_t, x_t in [-128, 127] (every digit
//   exact: the signed int8 range is used in full, 8 bits per slice);
//   C = A B^T = 2^{eA_i + eB_j} sum_{t+u<S} 2^{-8(t+u)-12} (A_t B_u^T)
//
// Each digit product A_t B_u^T is an exact int8 x int8 -> int32 tensor-core
// GEMM; products of one diagonal d = t+u share a TMEM accumulator (exact while
// S K 128^2 < 2^31). Truncation and the dropped products (t+u >= S) bound the
// error by ~(S + 2) 2^{2-8S} K max|A_i| max|B_j| per entry: S = 6 (21 products,
// 46 bits) keeps it near 1e-13 of the row-scale product. The FP64 result is
// assembled from the S int32 diagonals in a fixed order, so it is
// deterministic (and bitwise symmetric for A B^T with B = A).
//
// Operand digits live in global memory pre-tiled in the tensor core's K-major
// "core matrix" layout (tiles of TH rows x 64 bytes: four 16-byte K chunks,
// each TH rows x 16 B), so each stage is a handful of 1-D bulk copies.
#include <cuda.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <map>
#include <mutex>
#include <type_traits>
#include <vector>

#include "epilogue.cuh"
#include "kernels.hpp"

namespace ustats::dev {

namespace {

constexpr int OZ_BM = 128, OZ_BN = 128;   // output tile
constexpr int OZ_BK = 64;                  // K bytes per tile of the global digit layout
constexpr int OZ_SK = 64;                  // K bytes per pipeline stage (two MMA k-steps)
constexpr int OZ_STAGES = 2;
constexpr int OZ_THREADS = 320;            // warps 0-3 and 6-9 epilogue, 4 producer, 5 MMA issuer
constexpr int OZ_EPI = 256;                // epilogue threads: two per tile row (TMEM lane), 64 columns each
constexpr int OZ_TILE_STAGE = OZ_BM * OZ_SK;  // 8 KiB per operand slice per stage
constexpr int kOzWorkSlots = 256;             // per-SM scratch slots (see ozaki_work_entries)

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
__device__ __forceinline__ void bar_arrive(unsigned long long* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
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
// Asynchronous TMEM load (no wait): pair with tmem_wait_ld, which also pins
// the loaded registers after the wait.
__device__ __forceinline__ void tmem_ld16_async(unsigned addr, unsigned* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(addr));
}
template <int N>
__device__ __forceinline__ void tmem_wait_ld(unsigned (&r)[N][16]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
        for (int j = 0; j < 16; ++j) asm volatile("" : "+r"(r[i][j]));
}

struct OzSmem {
    union {
        struct {
            int8_t a[OZ_STAGES][kOzMaxSlices][OZ_TILE_STAGE];
            int8_t b[OZ_STAGES][kOzMaxSlices][OZ_TILE_STAGE];
        } st;
        double tile[epi::BM * epi::TP];  // the FP64 product tile once every MMA has read its operands
    } u;
    unsigned long long full[OZ_STAGES], empty[OZ_STAGES], done[2], drained;
    unsigned long long full1[8], empty1[8];  // pass 1's deeper ring (oz_p1_stages)
    double red[OZ_EPI / 32];
    int bexp[OZ_BN];       // column exponents of the tile
    double bscale[OZ_BN];  // 2^bexp (0 for padding columns) while every |bexp| <= 511
    int bwide;             // some column exponent outside [-511, 511]
    int last;              // K-split tail tile: this CTA sums the partials
    unsigned tmem;
};

// One 128 x 128 output tile per CTA, in two passes over K so that the digit
// diagonals fit TMEM at N = 128 (the full-rate MMA shape): pass 0 sums the
// high diagonals d = P..S-1 (slices 0..S-1), pass 1 the low ones d = 0..P-1
// (slices 0..P-1, P = oz_pass_split(S)), each into <= 4 int32 accumulators of
// 128 columns. Between
// the passes the epilogue warps drain pass 0 into the output tile (FP64,
// before the row/column exponents); pass 1 adds to it.
// Tile order: square groups of OZ_GROUP x OZ_GROUP tiles (upper groups only
// when symmetric), column-major inside a group, so one wave of CTAs streams a
// bounded set of A and B panels that mostly stay L2-resident across the wave
// (measured on C2: 16 > 12, 20, 24 > 8, 32).
constexpr long long OZ_GROUP = 16;
__host__ __device__ __forceinline__ void oz_tile_of(const OzakiArgs& p, long long bid, long long* tm, long long* tn) {
    const long long T_m = p.mpad / OZ_BM, T_n = p.npad / OZ_BN;
    if (!p.symmetric) {  // groups of OZ_GROUP row tiles x all column tiles, column-major inside: O(1)
        const long long width = OZ_GROUP * T_n;
        const long long g = bid / width, m0 = g * OZ_GROUP;
        const long long gsz = (T_m - m0) < OZ_GROUP ? (T_m - m0) : OZ_GROUP;
        const long long rem = bid - g * width;
        *tm = m0 + rem % gsz;
        *tn = rem / gsz;
        return;
    }
    // symmetric (T_m == T_n): column group J holds J full OZ_GROUP x w groups
    // above its diagonal group (w (w + 1) / 2 tiles), w = its width; whole
    // groups are skipped in O(1), so a tile lookup costs O(T / OZ_GROUP)
    // (C5, T = 512: 32 steps instead of ~8k column steps per CTA)
    const long long gn = (T_n + OZ_GROUP - 1) / OZ_GROUP;
    for (long long J = 0; J < gn; ++J) {
        const long long n0 = J * OZ_GROUP, w = (n0 + OZ_GROUP < T_n) ? OZ_GROUP : T_n - n0;
        const long long above = J * OZ_GROUP * w, col_total = above + w * (w + 1) / 2;
        if (bid >= col_total) {
            bid -= col_total;
            continue;
        }
        if (bid < above) {  // full group I = bid / (OZ_GROUP w), column-major inside
            const long long I = bid / (OZ_GROUP * w), r = bid - I * OZ_GROUP * w;
            *tm = I * OZ_GROUP + r % OZ_GROUP;
            *tn = n0 + r / OZ_GROUP;
            return;
        }
        bid -= above;  // diagonal group: column c holds rows n0..c
        for (long long c = n0; c < n0 + w; ++c) {
            const long long h = c + 1 - n0;
            if (bid < h) {
                *tm = n0 + bid;
                *tn = c;
                return;
            }
            bid -= h;
        }
    }
    *tm = 0;
    *tn = 0;
}

// Diagonals of pass 1 (the rest, at most 4, go to pass 0). Pass 0 loads all S
// slices, pass 1 only P: the fewer accumulators pass 0 takes, the fewer bytes
// per k, the more MMAs per staged byte in pass 0.
#ifndef OZ_PASS0_ACC
#define OZ_PASS0_ACC 3
#endif
__host__ __device__ constexpr int oz_pass_split(int S) { return S <= 4 ? S : S - OZ_PASS0_ACC; }
static_assert(oz_pass_split(7) <= 4 && 7 - oz_pass_split(7) <= 4, "TMEM holds 4 accumulators of 128 columns");
// Pass 0 of S > 4 slices holds three diagonals, which leaves one 128-column
// accumulator of TMEM spare: the top diagonal d = S - 1 (S products per k, the
// most of any) is split over two accumulators -- products t < oz_top_half(S)
// into its own, the rest into the spare one -- and the two are added in FP64
// when pass 0 drains. No int32 accumulator then sums more than S - 1 products,
// so K up to (2^31 - 1) / ((S - 1) 128^2) stays exact (S = 6: 26176 instead of
// 21824: C5's K = 65536 can run as 3 chunks instead of 4 where memory allows).
__host__ __device__ constexpr bool oz_top_split(int S, int D0, int D1) { return S > 4 && D1 == S && D1 - D0 == OZ_PASS0_ACC; }
__host__ __device__ constexpr int oz_top_half(int S) { return (S + 1) / 2; }

// Issued by the whole MMA warp: every operand is warp-uniform (one base
// descriptor plus compile-time offsets), so the descriptors stay in uniform
// registers and each MMA is one elected UTCIMMA (no per-MMA waterfall loop).
template <int S, int D0, int D1, int SLOT0>
__device__ __forceinline__ void oz_issue_stage(unsigned tmem, unsigned long long desc0, unsigned idesc, bool first0) {
    // diagonals [D0, D1) of the digit products, accumulators at (d - D0) * 128 columns;
    // two 32-byte k-steps per stage: the second starts two 16-byte chunks (2 x 2048 B) further
    constexpr unsigned b_off = OZ_STAGES * kOzMaxSlices * OZ_TILE_STAGE;  // sm.u.st.b after sm.u.st.a
#pragma unroll
    for (int ks = 0; ks < OZ_SK / 32; ++ks) {
        const bool first = first0 && ks == 0;
#pragma unroll
        for (int d = D0; d < D1; ++d)
#pragma unroll
            for (int t = 0; t <= d; ++t) {
                const int u = d - t;
                if (t >= S || u >= S) continue;
                const unsigned a_off = (SLOT0 + t) * OZ_TILE_STAGE + ks * 2 * OZ_BM * 16;
                const unsigned bo = b_off + (SLOT0 + u) * OZ_TILE_STAGE + ks * 2 * OZ_BN * 16;
                const bool spare = oz_top_split(S, D0, D1) && d == S - 1 && t >= oz_top_half(S);
                const unsigned acc = tmem + static_cast<unsigned>((spare ? OZ_PASS0_ACC : d - D0) * OZ_BN);
                const unsigned accumulate = (first && (t == 0 || (spare && t == oz_top_half(S)))) ? 0u : 1u;
                asm volatile(
                    "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
                    "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(acc),
                    "l"(desc0 + (a_off >> 4)), "l"(desc0 + (bo >> 4)), "r"(idesc), "r"(accumulate));
            }
    }
}

// Pass 1 stages only `split` slices, so its ring reuses the flat slot array
// (OZ_STAGES x kOzMaxSlices slots per operand) as OZ_STAGES x kOzMaxSlices /
// split smaller stages: stage q starts at slot q * split. Deeper lookahead
// where pass 1 has the fewest MMAs per byte (measured: split 3 of S = 6 beats
// 2 and 4).
__host__ __device__ constexpr int oz_p1_stages(int split) {
    return OZ_STAGES * kOzMaxSlices / split < 8 ? OZ_STAGES * kOzMaxSlices / split : 8;
}
__host__ __device__ constexpr int oz_p1_slot(int split, int q) { return q * split; }
template <int S, int SPLIT, int Q = 0>
__device__ __forceinline__ void oz_issue_p1(int q, unsigned tmem, unsigned long long desc0, unsigned idesc, bool first) {
    if (q == Q) oz_issue_stage<S, 0, SPLIT, oz_p1_slot(SPLIT, Q)>(tmem, desc0, idesc, first);
    else if constexpr (Q + 1 < oz_p1_stages(SPLIT)) oz_issue_p1<S, SPLIT, Q + 1>(q, tmem, desc0, idesc, first);
}

__device__ __forceinline__ void oz_commit(unsigned long long* bar) {
    asm volatile(
        "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(su32(bar)));
}

constexpr int kOzNoColumn = 1 << 30;  // padding column of the tile
// K-split of the last partial wave: more chunks shorten it but lengthen the
// summing of the partial tiles that follows
constexpr int kOzMaxTailSplit = 8;

// v 2^e: one exact multiply while 2^e is a normal double; ldexp (out of line:
// inlined, its range handling costs ~60 instructions per value) otherwise
__device__ __noinline__ double oz_scale_slow(double v, int e) { return ldexp(v, e); }
__device__ __forceinline__ double oz_scale(double v, int e) {
    if (e >= -1022 && e <= 1023) return v * __longlong_as_double(static_cast<long long>(e + 1023) << 52);
    return oz_scale_slow(v, e);
}

// Adds the diagonals [D0, D1) of columns c0..c0+15 (this thread's TMEM lane) to
// v, smallest contributions first: all loads in flight, one wait.
// TOP: the top diagonal's second accumulator (oz_top_split) sits after the
// D1 - D0 regular ones; both halves are exact integers, added in FP64.
template <int D0, int D1, bool TOP = false>
__device__ __forceinline__ void oz_drain(unsigned lane_base, int c0, double (&v)[16], bool add) {
    constexpr int NA = D1 - D0 + (TOP ? 1 : 0);
    unsigned r[NA][16];
#pragma unroll
    for (int a = 0; a < NA; ++a) tmem_ld16_async(lane_base + static_cast<unsigned>(a * OZ_BN + c0), r[a]);
    tmem_wait_ld(r);
    if (!add)
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = 0.0;
#pragma unroll
    for (int d = D1 - 1; d >= D0; --d) {
        const double scale = __longlong_as_double(static_cast<long long>(1023 - 8 * d - 12) << 52);  // 2^{-8d-12}
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            double x = static_cast<double>(static_cast<int>(r[d - D0][j]));
            if (TOP && d == D1 - 1) x += static_cast<double>(static_cast<int>(r[NA - 1][j]));
            v[j] += x * scale;
        }
    }
}

template <int S>
__global__ void __launch_bounds__(OZ_THREADS, 1) ozaki_gemm_kernel(OzakiArgs p) {
    // no swizzle: 16-byte alignment is all the descriptors and bulk copies need, and
    // addressing the struct straight off the shared array keeps every access in .shared
    extern __shared__ __align__(128) unsigned char oz_raw[];
    OzSmem& sm = *reinterpret_cast<OzSmem*>(oz_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr int split = oz_pass_split(S);  // diagonals of pass 1: [0, split); pass 0: [split, S)
    long long rel = blockIdx.x, tm, tn;  // tile index inside this launch
    int chunk = 0;
    const bool tail = p.tail_split > 1 && rel >= p.tail_from;
    if (tail) {  // one K range of a tile of the last partial wave
        const long long q = rel - p.tail_from;
        rel = p.tail_from + q / p.tail_split;
        chunk = static_cast<int>(q % p.tail_split);
    }
    oz_tile_of(p, p.tile_begin + rel, &tm, &tn);
    const long long ktiles = p.kpad / OZ_BK;
    const long long kb = tail ? chunk * ktiles / p.tail_split : 0;
    const long long ksteps = (tail ? (chunk + 1) * ktiles / p.tail_split : ktiles) - kb;  // OZ_SK == OZ_BK
    const long long tile_bytes = OZ_BM * OZ_BK;  // one 128-row x 64-byte tile of the global layout
    const int8_t* abase = p.a + (tm * ktiles + kb) * tile_bytes;
    const int8_t* bbase = p.b + (tn * ktiles + kb) * tile_bytes;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&sm.tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 128) {
        for (int s = 0; s < OZ_STAGES; ++s) {
            bar_init(&sm.full[s], 1);
            bar_init(&sm.empty[s], 1);
        }
        for (int q = 0; q < oz_p1_stages(split); ++q) {
            bar_init(&sm.full1[q], 1);
            bar_init(&sm.empty1[q], 1);
        }
        bar_init(&sm.done[0], 1);
        bar_init(&sm.done[1], 1);
        bar_init(&sm.drained, OZ_EPI / 32);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const unsigned tmem = sm.tmem;

    if (tid == 128) {  // producer: pass 0 through the 2-stage ring, then pass 1 through its deeper one
        auto load_stage = [&](long long k, int ns, int slot0, unsigned long long* bar) {
            bar_expect(bar, static_cast<unsigned>(2 * ns * OZ_TILE_STAGE));
            // stage k = global k-tile k (four 16-byte chunks, contiguous)
            const long long off = k * tile_bytes;
            for (int t = 0; t < ns; ++t) {
                bulk_load(sm.u.st.a[0][0] + (slot0 + t) * OZ_TILE_STAGE, abase + t * p.a_slice + off, OZ_TILE_STAGE, bar);
                bulk_load(sm.u.st.b[0][0] + (slot0 + t) * OZ_TILE_STAGE, bbase + t * p.b_slice + off, OZ_TILE_STAGE, bar);
            }
            // warm L2 a few k-tiles ahead
            if (p.prefetch > 0 && k + p.prefetch < ksteps) {
                const long long poff = off + p.prefetch * tile_bytes;
                for (int t = 0; t < ns; ++t) {
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                                     reinterpret_cast<unsigned long long>(abase + t * p.a_slice + poff)),
                                 "r"(static_cast<unsigned>(OZ_TILE_STAGE))
                                 : "memory");
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                                     reinterpret_cast<unsigned long long>(bbase + t * p.b_slice + poff)),
                                 "r"(static_cast<unsigned>(OZ_TILE_STAGE))
                                 : "memory");
                }
            }
        };
        if constexpr (split < S) {
#pragma unroll 1
            for (long long k = 0; k < ksteps; ++k) {
                const int s = static_cast<int>(k % OZ_STAGES);
                if (k >= OZ_STAGES) bar_wait(&sm.empty[s], static_cast<unsigned>(((k / OZ_STAGES) - 1) & 1));
                load_stage(k, S, s * kOzMaxSlices, &sm.full[s]);
            }
            bar_wait(&sm.done[0], 0);  // every pass-0 MMA has read its operands: the slots are free
        }
        constexpr int P1 = oz_p1_stages(split);
#pragma unroll 1
        for (long long k = 0; k < ksteps; ++k) {
            const int q = static_cast<int>(k % P1);
            if (k >= P1) bar_wait(&sm.empty1[q], static_cast<unsigned>(((k / P1) - 1) & 1));
            load_stage(k, split, oz_p1_slot(split, q), &sm.full1[q]);
        }
    } else if (warp == 5) {  // MMA warp: the loop runs warp-wide, one elected lane issues
        // kind::i8, int32 accumulate, signed A and B, both K-major, N = 128, M = 128
        const unsigned idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((OZ_BN >> 3) << 17) | ((OZ_BM >> 4) << 24);
        // a[0][0]; every other slice / stage / operand tile at a constant offset (K-major core matrices:
        // leading-byte offset = one 16-byte K chunk of 128 rows, stride-byte offset = 8 rows x 16 B)
        const unsigned long long desc0 = umma_desc(su32(sm.u.st.a[0][0]), OZ_BM * 16, 128);
        static_assert(OZ_BM == OZ_BN, "one descriptor template for both operands");
        if constexpr (split < S) {
#pragma unroll 1
            for (long long k = 0; k < ksteps; ++k) {
                const int s = static_cast<int>(k % OZ_STAGES);
                bar_wait(&sm.full[s], static_cast<unsigned>((k / OZ_STAGES) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;");
                if (s == 0) oz_issue_stage<S, split, S, 0>(tmem, desc0, idesc, k == 0);
                else oz_issue_stage<S, split, S, kOzMaxSlices>(tmem, desc0, idesc, k == 0);
                oz_commit(&sm.empty[s]);
            }
            oz_commit(&sm.done[0]);
            bar_wait(&sm.drained, 0);  // pass 0 read out of TMEM
            asm volatile("tcgen05.fence::after_thread_sync;");
        }
        constexpr int P1 = oz_p1_stages(split);
#pragma unroll 1
        for (long long k = 0; k < ksteps; ++k) {
            const int q = static_cast<int>(k % P1);
            bar_wait(&sm.full1[q], static_cast<unsigned>((k / P1) & 1));
            asm volatile("tcgen05.fence::after_thread_sync;");
            oz_issue_p1<S, split>(q, tmem, desc0, idesc, k == 0);
            oz_commit(&sm.empty1[q]);
        }
        oz_commit(&sm.done[1]);
    } else if (warp < 4 || warp >= 6) {  // epilogue warps: thread = one row of the tile (TMEM lane), half its columns
        // a warp reaches only the TMEM lanes 32 (warp % 4) .. +31: warps 0-3 take columns 0-63 of
        // their lanes, warps 6-9 (lane quarters 2, 3, 0, 1) columns 64-127
        const int quarter = warp & 3, half = warp >= 6 ? 1 : 0;
        const int et = half * 128 + quarter * 32 + lane;  // epilogue thread index, warp-aligned
        const int rt = quarter * 32 + lane;               // row inside the tile
        const int cb = half * (OZ_BN / 2);                // first column of this thread's half
        const long long row = tm * OZ_BM + rt;
        const bool row_ok = row < p.m;
        auto sync_epi = [] { asm volatile("bar.sync 1, 256;" ::: "memory"); };
        static_assert(OZ_EPI == 256, "named barrier count");
        if (et == 0) sm.bwide = 0;
        sync_epi();
        if (et < OZ_BN) {
            const int rt = et;
            const long long col = tn * OZ_BN + rt;
            const int eb = col < p.n ? p.b_exp[col] : kOzNoColumn;
            sm.bexp[rt] = eb;
            const bool pad = eb == kOzNoColumn, narrow = eb >= -511 && eb <= 511;
            sm.bscale[rt] = (pad || !narrow) ? 0.0 : __longlong_as_double(static_cast<long long>(eb + 1023) << 52);
            if (!pad && !narrow) sm.bwide = 1;
        }
        sync_epi();
        const int ea = row_ok ? p.a_exp[row] : 0;
        const bool narrow = !sm.bwide && ea >= -511 && ea <= 511;
        const double sa = row_ok ? __longlong_as_double(static_cast<long long>(ea + 1023) << 52) : 0.0;
        // one CTA per SM at a time (shared memory and TMEM say so): the scratch
        // of the high-diagonal partial is per SM, L2-resident, column-major so a
        // warp's 32 rows of one column are one coalesced 256-byte access
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        if (smid >= static_cast<unsigned>(kOzWorkSlots)) __trap();
        double* work = p.work + static_cast<long long>(smid) * (OZ_BM * OZ_BN) + rt;
        const unsigned lane_base = tmem + (static_cast<unsigned>(quarter * 32) << 16);
        if constexpr (split < S) {  // pass 0: high diagonals into the scratch
            bar_wait(&sm.done[0], 0);
            asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll 1
            for (int c0 = cb; c0 < cb + OZ_BN / 2; c0 += 16) {
                double v[16];
                oz_drain<split, S, oz_top_split(S, split, S)>(lane_base, c0, v, false);
#pragma unroll
                for (int j = 0; j < 16; ++j) work[(c0 + j) * OZ_BM] = v[j];
            }
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) bar_arrive(&sm.drained);
        }
        // the high-diagonal partial comes back from L2 two 16-column chunks ahead
        // of its use (the first two while pass 1 still runs: this thread wrote them)
        double h0[16], h1[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            h0[j] = split < S ? work[(cb + j) * OZ_BM] : 0.0;
            h1[j] = split < S ? work[(cb + 16 + j) * OZ_BM] : 0.0;
        }
        bar_wait(&sm.done[1], 0);
        asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll 1
        for (int c0 = cb; c0 < cb + OZ_BN / 2; c0 += 16) {
            double v[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                v[j] = h0[j];
                h0[j] = h1[j];
                if (c0 + 32 < cb + OZ_BN / 2) h1[j] = split < S ? work[(c0 + 32 + j) * OZ_BM] : 0.0;
            }
            oz_drain<0, split>(lane_base, c0, v, true);
            // the product tile in shared memory (every MMA has completed: the ring is free);
            // exact power-of-two scaling: (v 2^ea) 2^eb, branch-free while both |e| <= 511
            if (narrow)
#pragma unroll
                for (int j = 0; j < 16; ++j) sm.u.tile[rt * epi::TP + c0 + j] = (v[j] * sa) * sm.bscale[c0 + j];
            else
                for (int j = 0; j < 16; ++j) {
                    const int eb = sm.bexp[c0 + j];
                    sm.u.tile[rt * epi::TP + c0 + j] = (row_ok && eb != kOzNoColumn) ? oz_scale(v[j], ea + eb) : 0.0;
                }
        }
        // the fused consumers of the tile (plain store, Hadamard + reductions), as in the DMMA kernel
        sync_epi();
        bool apply = true;
        if (tail) {  // partial tile out; the last of the tile's chunks sums them in chunk order
            const long long t = rel - p.tail_from;
            double* part = p.tail_part + (t * p.tail_split + chunk) * (OZ_BM * OZ_BN);
            for (int i = et; i < OZ_BM * OZ_BN; i += OZ_EPI) part[i] = sm.u.tile[(i >> 7) * epi::TP + (i & 127)];
            __threadfence();
            sync_epi();
            if (et == 0) {
                const unsigned done_before = atomicAdd(&p.tail_count[t], 1u);
                sm.last = done_before == static_cast<unsigned>(p.tail_split - 1);
            }
            sync_epi();
            apply = sm.last;
            if (apply) {
                __threadfence();
                // 16-byte loads, 4 x kOzMaxTailSplit of them in flight per thread
                const double2* p0 = reinterpret_cast<const double2*>(p.tail_part + t * p.tail_split * (OZ_BM * OZ_BN));
                constexpr int H = OZ_BM * OZ_BN / 2;  // double2 per partial tile
#pragma unroll 1
                for (int i0 = et; i0 < H; i0 += 4 * OZ_EPI) {
                    double2 acc[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) acc[u] = make_double2(0.0, 0.0);
#pragma unroll
                    for (int c = 0; c < kOzMaxTailSplit; ++c)
                        if (c < p.tail_split)
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const double2 v = __ldcg(p0 + c * H + i0 + u * OZ_EPI);
                                acc[u].x += v.x;
                                acc[u].y += v.y;
                            }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int i = 2 * (i0 + u * OZ_EPI);
                        sm.u.tile[(i >> 7) * epi::TP + (i & 127)] = acc[u].x;
                        sm.u.tile[((i + 1) >> 7) * epi::TP + ((i + 1) & 127)] = acc[u].y;
                    }
                }
                if (et == 0) p.tail_count[t] = 0;  // reusable counters
                sync_epi();
            }
        }
        if (apply)
            epi::apply<OZ_EPI>(p.epis, p.m, p.n, p.accumulate, sm.u.tile, tm * OZ_BM, tn * OZ_BN, tm, tn,
                               p.symmetric && tm != tn, rel, sm.red, et, sync_epi);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ---------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): two SMs of one TPC compute a 256 x 128
// output pair tile with M = 256 MMAs issued by the even CTA. Each CTA stages
// its own 128 rows of A and HALF of B (64 of the 128 columns): the B bytes per
// SM halve, so L2 -> SM traffic per int8 op drops by a third against the
// single-SM kernel, whose 128 x 128 tiles pin it at the L2 throughput cap
// (C2: 11.7 TB/s of TMA reads, tensor pipe 76%). Same two passes over K, same
// per-CTA TMEM accumulators (128 lanes x 128 columns per diagonal), same
// epilogue. Both CTAs stage through 3-D tensor maps over the digit layout
// (one TMA per slice and operand: A box 128 rows, B box 64 rows x four 16-byte
// K columns) with the cta_group::2 form, whose transaction bytes land on the
// even CTA's barrier: the MMA issuer waits on one barrier per stage.
constexpr int OZ2_SLOTS = 18;                  // digit slots per operand in the ring
constexpr int OZ2_A = OZ_BM * OZ_SK;           // 8 KiB: 128 rows x 64 B of one slice
constexpr int OZ2_B = (OZ_BN / 2) * OZ_SK;     // 4 KiB: this CTA's 64 columns of one slice
constexpr long long OZ2_GROUP = OZ_GROUP / 2;  // pair rows per tile group (16 tile rows)
__host__ __device__ constexpr int oz2_stages(int per_stage) {
    return OZ2_SLOTS / per_stage < 8 ? OZ2_SLOTS / per_stage : 8;
}

struct Oz2Smem {
    union {
        struct {
            int8_t a[OZ2_SLOTS][OZ2_A];
            int8_t b[OZ2_SLOTS][OZ2_B];
        } st;
        double tile[epi::BM * epi::TP];
    } u;
    unsigned long long full[8], empty[8], full1[8], empty1[8], done[2], drained, tmem_free, epi_done;
    double red[OZ_EPI / 32];
    int bexp[OZ_BN];
    double bscale[OZ_BN];
    int bwide;
    unsigned tmem;
};

// Pair tiles: pair row pm covers tile rows 2 pm, 2 pm + 1. Symmetric: every
// pair whose first tile is on or above the diagonal (2 pm <= tn); the odd tile
// of a diagonal pair (2 pm + 1 > tn) is computed and dropped.
__host__ __device__ __forceinline__ long long oz2_pair_count(const OzakiArgs& p) {
    const long long T_m = p.mpad / OZ_BM, T_n = p.npad / OZ_BN, P_m = (T_m + 1) / 2;
    if (!p.symmetric) return P_m * T_n;
    long long c = 0;
    for (long long tn = 0; tn < T_n; ++tn) c += tn / 2 + 1;
    return c;
}
__host__ __device__ __forceinline__ void oz2_pair_of(const OzakiArgs& p, long long bid, long long* pm, long long* tn) {
    const long long T_m = p.mpad / OZ_BM, T_n = p.npad / OZ_BN, P_m = (T_m + 1) / 2;
    if (!p.symmetric) {  // groups of G pair rows x all columns, column-major inside
        const long long G = p.group2 > 0 ? p.group2 : OZ2_GROUP;
        const long long width = G * T_n;
        const long long g = bid / width, m0 = g * G;
        const long long gsz = (P_m - m0) < G ? (P_m - m0) : G;
        const long long rem = bid - g * width;
        *pm = m0 + rem % gsz;
        *tn = rem / gsz;
        return;
    }
    if (p.sym_group2 > 0) {
        // groups of G pair rows x their columns (tn >= 2 pm), column-major
        // inside: the group's A panels stay in L2 while the B panels stream by
        const long long G = p.sym_group2;
        for (long long m0 = 0; m0 < P_m; m0 += G) {
            const long long gsz = (P_m - m0) < G ? (P_m - m0) : G;
            long long total = 0;
            for (long long q = m0; q < m0 + gsz; ++q) total += T_n - 2 * q;
            if (bid >= total) {
                bid -= total;
                continue;
            }
            long long c = 2 * m0;
            for (; c < 2 * (m0 + gsz - 1); ++c) {  // the ramp: pair rows m0 .. c / 2
                const long long h = c / 2 - m0 + 1;
                if (bid < h) {
                    *pm = m0 + bid;
                    *tn = c;
                    return;
                }
                bid -= h;
            }
            *pm = m0 + bid % gsz;
            *tn = c + bid / gsz;
            return;
        }
        *pm = 0;
        *tn = 0;
        return;
    }
    // column groups of OZ_GROUP columns: the pair-row groups fully above the
    // diagonal block first (column-major inside), then the diagonal block
    const long long gn = (T_n + OZ_GROUP - 1) / OZ_GROUP;
    for (long long J = 0; J < gn; ++J) {
        const long long n0 = J * OZ_GROUP, w = (n0 + OZ_GROUP < T_n) ? OZ_GROUP : T_n - n0;
        const long long above = (n0 / 2) * w;  // pair rows 0 .. n0/2 - 1
        long long diag = 0;
        for (long long c = n0; c < n0 + w; ++c) diag += c / 2 - n0 / 2 + 1;
        if (bid >= above + diag) {
            bid -= above + diag;
            continue;
        }
        if (bid < above) {
            const long long I = bid / (OZ2_GROUP * w), r = bid - I * OZ2_GROUP * w;
            *pm = I * OZ2_GROUP + r % OZ2_GROUP;
            *tn = n0 + r / OZ2_GROUP;
            return;
        }
        bid -= above;
        for (long long c = n0; c < n0 + w; ++c) {
            const long long h = c / 2 - n0 / 2 + 1;
            if (bid < h) {
                *pm = n0 / 2 + bid;
                *tn = c;
                return;
            }
            bid -= h;
        }
    }
    *pm = 0;
    *tn = 0;
}

__device__ __forceinline__ unsigned oz2_cta_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void oz2_cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on the even CTA's copy of barrier b (its own copy when called there)
__device__ __forceinline__ void oz2_arrive_leader(unsigned long long* b) {
    unsigned remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(su32(b)));
    // default (cta-scope) semantics, as CUTLASS's 2-SM pipelines use: a
    // cluster-scope release / acquire emits an L1 invalidate (CCTL.IVALL) per
    // stage on the MMA issuer's critical path
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
__device__ __forceinline__ void oz2_wait_cluster(unsigned long long* b, unsigned parity) { bar_wait(b, parity); }
// tcgen05.commit to the barrier at the same offset in both CTAs of the pair
__device__ __forceinline__ void oz2_commit(unsigned long long* bar) {
    asm volatile(
        "{\n.reg .pred e;\n.reg .b16 m;\nmov.b16 m, 3;\nelect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n}\n" ::"r"(
            su32(bar)));
}

// One stage of diagonals [D0, D1) from slots SLOT0.. (M = 256 over the pair, N = 128).
template <int S, int D0, int D1, int SLOT0>
__device__ __forceinline__ void oz2_issue_stage(unsigned tmem, unsigned long long desc_a, unsigned long long desc_b,
                                                unsigned idesc, bool first0) {
#pragma unroll
    for (int ks = 0; ks < OZ_SK / 32; ++ks) {
        const bool first = first0 && ks == 0;
#pragma unroll
        for (int d = D0; d < D1; ++d)
#pragma unroll
            for (int t = 0; t <= d; ++t) {
                const int u = d - t;
                if (t >= S || u >= S) continue;
                // 32-byte k-step = two 16-byte core-matrix columns (A: 128 rows, B: 64 rows each)
                const unsigned a_off = (SLOT0 + t) * OZ2_A + ks * 2 * OZ_BM * 16;
                const unsigned b_off = (SLOT0 + u) * OZ2_B + ks * 2 * (OZ_BN / 2) * 16;
                const bool spare = oz_top_split(S, D0, D1) && d == S - 1 && t >= oz_top_half(S);
                const unsigned acc = tmem + static_cast<unsigned>((spare ? OZ_PASS0_ACC : d - D0) * OZ_BN);
                const unsigned accumulate = (first && (t == 0 || (spare && t == oz_top_half(S)))) ? 0u : 1u;
                asm volatile(
                    "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
                    "@e tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(acc),
                    "l"(desc_a + (a_off >> 4)), "l"(desc_b + (b_off >> 4)), "r"(idesc), "r"(accumulate));
            }
    }
}
// stage q of a ring of NST stages of NS slots each (compile-time slot base)
template <int S, int D0, int D1, int NS, int NST, int Q = 0>
__device__ __forceinline__ void oz2_issue(int q, unsigned tmem, unsigned long long da, unsigned long long db,
                                          unsigned idesc, bool first) {
    if (q == Q) oz2_issue_stage<S, D0, D1, Q * NS>(tmem, da, db, idesc, first);
    else if constexpr (Q + 1 < NST) oz2_issue<S, D0, D1, NS, NST, Q + 1>(q, tmem, da, db, idesc, first);
}

// 3-D view of a digit buffer: (64 rows x 16 B as 128 8-byte words, 2 row
// halves, K columns of every tile of every panel of every slice): a
// (128, 2 or 1, 4) box is one tile's slice, all of it (A) or one half (B)
__device__ __forceinline__ void oz2_tma(void* dst, const CUtensorMap* map, int half, int col, unsigned leader_bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
        "%4}], [%5];" ::"r"(su32(dst)),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(0), "r"(half), "r"(col), "r"(leader_bar)
        : "memory");
}
__device__ __forceinline__ unsigned oz2_leader_addr(const void* p) {
    unsigned remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(su32(p)));
    return remote;
}

// Persistent over pair tiles: cluster c runs tiles c, c + P, c + 2P, ...
// (P = gridDim.x / 2; a full grid runs one tile per cluster). Stage counters
// and barrier phases carry across tiles; the producer starts tile j + 1 only
// after its CTA's epilogue released the staging tile (epi_done), the MMA
// issuer only after both CTAs drained the accumulators (tmem_free). With
// p.lockstep the producers of every CTA meet at a wave barrier in global
// memory before each tile (bounded spin: a CTA that is not resident only
// delays the others by the timeout), so all tiles of a wave stream K in
// step and the digit panels they share are read from DRAM once.
template <int S>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(OZ_THREADS, 1)
    ozaki_gemm_2sm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                          const __grid_constant__ OzakiArgs p) {
    extern __shared__ __align__(128) unsigned char oz_raw[];
    Oz2Smem& sm = *reinterpret_cast<Oz2Smem*>(oz_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const unsigned rank = oz2_cta_rank();
    constexpr int split = oz_pass_split(S);  // pass 1: diagonals [0, split); pass 0: [split, S)
    constexpr int P0 = oz2_stages(S), P1 = oz2_stages(split);
    const long long T_m = p.mpad / OZ_BM, T_n = p.npad / OZ_BN;
    const long long ktiles = p.kpad / OZ_BK;
    const long long P = gridDim.x >> 1, cl = blockIdx.x >> 1, pairs = p.pairs;
    struct Tile {
        long long pm, tn, tm, tm_load;
        bool ok;
    };
    auto tile_at = [&](long long it) {
        Tile t;
        oz2_pair_of(p, p.tile_begin + it, &t.pm, &t.tn);
        t.tm = 2 * t.pm + rank;
        t.ok = t.tm < T_m && !(p.symmetric && t.tm > t.tn);
        t.tm_load = t.tm < T_m ? t.tm : T_m - 1;  // a missing odd panel: load any (its rows are dropped)
        return t;
    };

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&sm.tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    if (tid == 128) {
        for (int s = 0; s < 8; ++s) {
            bar_init(&sm.full[s], 1);
            bar_init(&sm.empty[s], 1);
            bar_init(&sm.full1[s], 1);
            bar_init(&sm.empty1[s], 1);
        }
        bar_init(&sm.done[0], 1);
        bar_init(&sm.done[1], 1);
        bar_init(&sm.drained, 2 * OZ_EPI / 32);
        bar_init(&sm.tmem_free, 2 * OZ_EPI / 32);
        bar_init(&sm.epi_done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    oz2_cluster_sync();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const unsigned tmem = sm.tmem;

    if (tid == 128) {  // producer (both CTAs): own A panel, own half of the B panel, bytes counted on the even CTA
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<unsigned long long>(&map_a)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<unsigned long long>(&map_b)) : "memory");
        const long long a_sl = T_m * ktiles * 4, b_sl = T_n * ktiles * 4;
        long long g0 = 0, g1 = 0, target = 0, target1 = 0;
        int j = 0;
        // bounded spin until *ctr reaches `want` (globaltimer ns)
        auto wave_wait = [&](unsigned long long* ctr, long long want) {
            atomicAdd(ctr, 1ull);
            unsigned long long t0, now, seen;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
            do {
                asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(seen) : "l"(ctr) : "memory");
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
            } while (seen < static_cast<unsigned long long>(want) && now - t0 < 200000ull);
        };
        for (long long it = cl; it < pairs; it += P, ++j) {
            const Tile t = tile_at(it);
            // column coordinate of (slice, panel, k-tile k): ((slice * panels + panel) * ktiles + k) * 4
            const long long acol0 = t.tm_load * ktiles * 4, bcol0 = t.tn * ktiles * 4;
            auto load_stage = [&](long long k, int ns, int slot0, unsigned long long* bar) {
                if (rank == 0) bar_expect(bar, static_cast<unsigned>(2 * ns * (OZ2_A + OZ2_B)));  // both CTAs' bytes
                const unsigned lb = oz2_leader_addr(bar);
                for (int q = 0; q < ns; ++q) {
                    oz2_tma(sm.u.st.a[slot0 + q], &map_a, 0, static_cast<int>(acol0 + q * a_sl + k * 4), lb);
                    oz2_tma(sm.u.st.b[slot0 + q], &map_b, static_cast<int>(rank),
                            static_cast<int>(bcol0 + q * b_sl + k * 4), lb);
                }
            };
            if (j > 0) {
                bar_wait(&sm.epi_done, static_cast<unsigned>((j - 1) & 1));  // the staging tile is free again
                if (p.wave_ctr) {  // wave barrier: every CTA that runs iteration j
                    const long long here = pairs - static_cast<long long>(j) * P;
                    target += 2 * (here < P ? here : P);
                    wave_wait(p.wave_ctr, target);
                }
            }
            if constexpr (split < S) {
#pragma unroll 1
                for (long long k = 0; k < ktiles; ++k, ++g0) {
                    const int s = static_cast<int>(g0 % P0);
                    if (g0 >= P0) bar_wait(&sm.empty[s], static_cast<unsigned>(((g0 / P0) - 1) & 1));
                    load_stage(k, S, s * S, &sm.full[s]);
                }
                bar_wait(&sm.done[0], static_cast<unsigned>(j & 1));  // every pass-0 MMA has read its operands
                if (p.wave_ctr && p.resync) {  // re-align the wave before pass 1 re-streams K
                    const long long here = pairs - static_cast<long long>(j) * P;
                    target1 += 2 * (here < P ? here : P);
                    wave_wait(p.wave_ctr + 1, target1);
                }
            }
#pragma unroll 1
            for (long long k = 0; k < ktiles; ++k, ++g1) {
                const int q = static_cast<int>(g1 % P1);
                if (g1 >= P1) bar_wait(&sm.empty1[q], static_cast<unsigned>(((g1 / P1) - 1) & 1));
                load_stage(k, split, q * split, &sm.full1[q]);
            }
        }
    } else if (warp == 5 && rank == 0) {  // MMA issuer (even CTA): kind::i8, s32 accumulators, M = 256, N = 128
        const unsigned idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((OZ_BN >> 3) << 17) | (((2 * OZ_BM) >> 4) << 24);
        const unsigned long long da = umma_desc(su32(sm.u.st.a[0]), OZ_BM * 16, 128);
        const unsigned long long db = umma_desc(su32(sm.u.st.b[0]), (OZ_BN / 2) * 16, 128);
        long long g0 = 0, g1 = 0;
        int j = 0;
        for (long long it = cl; it < pairs; it += P, ++j) {
            if (j > 0) {  // both CTAs have read the previous tile's accumulators
                oz2_wait_cluster(&sm.tmem_free, static_cast<unsigned>((j - 1) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;");
            }
            if constexpr (split < S) {
#pragma unroll 1
                for (long long k = 0; k < ktiles; ++k, ++g0) {
                    const int s = static_cast<int>(g0 % P0);
                    oz2_wait_cluster(&sm.full[s], static_cast<unsigned>((g0 / P0) & 1));
                    asm volatile("tcgen05.fence::after_thread_sync;");
                    oz2_issue<S, split, S, S, P0>(s, tmem, da, db, idesc, k == 0);
                    oz2_commit(&sm.empty[s]);
                }
                oz2_commit(&sm.done[0]);
                oz2_wait_cluster(&sm.drained, static_cast<unsigned>(j & 1));  // both CTAs read pass 0 out of TMEM
                asm volatile("tcgen05.fence::after_thread_sync;");
            }
#pragma unroll 1
            for (long long k = 0; k < ktiles; ++k, ++g1) {
                const int q = static_cast<int>(g1 % P1);
                oz2_wait_cluster(&sm.full1[q], static_cast<unsigned>((g1 / P1) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;");
                oz2_issue<S, 0, split, split, P1>(q, tmem, da, db, idesc, k == 0);
                oz2_commit(&sm.empty1[q]);
            }
            oz2_commit(&sm.done[1]);
        }
    } else if (warp < 4 || warp >= 6) {  // epilogue warps (both CTAs): as in ozaki_gemm_kernel
        const int quarter = warp & 3, half = warp >= 6 ? 1 : 0;
        const int et = half * 128 + quarter * 32 + lane;
        const int rt = quarter * 32 + lane;
        const int cb = half * (OZ_BN / 2);
        auto sync_epi = [] { asm volatile("bar.sync 1, 256;" ::: "memory"); };
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        if (smid >= static_cast<unsigned>(kOzWorkSlots)) __trap();
        double* work = p.work + static_cast<long long>(smid) * (OZ_BM * OZ_BN) + rt;
        const unsigned lane_base = tmem + (static_cast<unsigned>(quarter * 32) << 16);
        int j = 0;
        for (long long it = cl; it < pairs; it += P, ++j) {
            const Tile t = tile_at(it);
            const long long row = t.tm * OZ_BM + rt;
            const bool row_ok = t.ok && row < p.m;
            if (et == 0) sm.bwide = 0;
            sync_epi();
            if (et < OZ_BN) {
                const long long col = t.tn * OZ_BN + et;
                const int eb = col < p.n ? p.b_exp[col] : kOzNoColumn;
                sm.bexp[et] = eb;
                const bool pad = eb == kOzNoColumn, narrow = eb >= -511 && eb <= 511;
                sm.bscale[et] = (pad || !narrow) ? 0.0 : __longlong_as_double(static_cast<long long>(eb + 1023) << 52);
                if (!pad && !narrow) sm.bwide = 1;
            }
            sync_epi();
            const int ea = row_ok ? p.a_exp[row] : 0;
            const bool narrow = !sm.bwide && ea >= -511 && ea <= 511;
            const double sa = row_ok ? __longlong_as_double(static_cast<long long>(ea + 1023) << 52) : 0.0;
            if constexpr (split < S) {
                bar_wait(&sm.done[0], static_cast<unsigned>(j & 1));
                asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll 1
                for (int c0 = cb; c0 < cb + OZ_BN / 2; c0 += 16) {
                    double v[16];
                    oz_drain<split, S, oz_top_split(S, split, S)>(lane_base, c0, v, false);
#pragma unroll
                    for (int q = 0; q < 16; ++q) work[(c0 + q) * OZ_BM] = v[q];
                }
                asm volatile("tcgen05.fence::before_thread_sync;");
                __syncwarp();
                if (lane == 0) oz2_arrive_leader(&sm.drained);
            }
            double h0[16], h1[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                h0[q] = split < S ? work[(cb + q) * OZ_BM] : 0.0;
                h1[q] = split < S ? work[(cb + 16 + q) * OZ_BM] : 0.0;
            }
            bar_wait(&sm.done[1], static_cast<unsigned>(j & 1));
            asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll 1
            for (int c0 = cb; c0 < cb + OZ_BN / 2; c0 += 16) {
                double v[16];
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    v[q] = h0[q];
                    h0[q] = h1[q];
                    if (c0 + 32 < cb + OZ_BN / 2) h1[q] = split < S ? work[(c0 + 32 + q) * OZ_BM] : 0.0;
                }
                oz_drain<0, split>(lane_base, c0, v, true);
                if (narrow)
#pragma unroll
                    for (int q = 0; q < 16; ++q) sm.u.tile[rt * epi::TP + c0 + q] = (v[q] * sa) * sm.bscale[c0 + q];
                else
                    for (int q = 0; q < 16; ++q) {
                        const int eb = sm.bexp[c0 + q];
                        sm.u.tile[rt * epi::TP + c0 + q] = (row_ok && eb != kOzNoColumn) ? oz_scale(v[q], ea + eb) : 0.0;
                    }
            }
            // the accumulators are read: the next tile's MMAs may overwrite them
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) oz2_arrive_leader(&sm.tmem_free);
            sync_epi();
            if (t.ok) {
                // dense slot of the tile: the finalizers sum ozaki_tile_count slots
                const long long slot = p.symmetric ? t.tn * (t.tn + 1) / 2 + t.tm : t.tm * T_n + t.tn;
                epi::apply<OZ_EPI>(p.epis, p.m, p.n, p.accumulate, sm.u.tile, t.tm * OZ_BM, t.tn * OZ_BN, t.tm, t.tn,
                                   p.symmetric && t.tm != t.tn, slot, sm.red, et, sync_epi);
            }
            sync_epi();  // every epilogue thread is done with the staging tile
            if (et == 0) bar_arrive(&sm.epi_done);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    oz2_cluster_sync();  // no CTA leaves while its pair may still signal its barriers or use its TMEM
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// Row exponents: e_i with max_k |x_ik| < 2^e_i (0 for an all-zero row).
__global__ void oz_row_exponents(const double* __restrict__ x, long long rows, long long k, long long rs, long long ks,
                                 int* __restrict__ exps, const int* __restrict__ panels) {
    long long r = blockIdx.x * static_cast<long long>(blockDim.x / 32) + (threadIdx.x >> 5);
    if (panels) r = static_cast<long long>(panels[r / OZ_BM]) * OZ_BM + r % OZ_BM;  // rows of the listed panels
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

// Digits into the tiled core-matrix layout, one (th x 64) tile per block:
// the FP64 tile is staged in shared memory with coalesced row reads, each
// thread turns one (row, 16-element chunk) into S 16-byte digit words, and
// every slice tile (th x 64 bytes, contiguous) is written coalesced.
// |x| 2^-e < 1, so m = trunc(x 2^{8S-2-e}) satisfies |m| < 2^{8S-2}: its S
// balanced base-256 digits (low byte as a signed int8, subtract, shift) fit
// int8, the top one in [-64, 64].
// x 2^sh as two exact power-of-two multiplies (each factor a normal double)
__device__ __forceinline__ double oz_pow2_mul(double x, int sh) {
    const int a = sh / 2, b = sh - a;
    return x * __longlong_as_double(static_cast<long long>(a + 1023) << 52) *
           __longlong_as_double(static_cast<long long>(b + 1023) << 52);
}

// The S digit words of 16 consecutive values of one row (exponent e) to
// out[t * slice_bytes], t = 0 (most significant) .. S-1.
// Balanced base-256 digits without a per-digit carry chain: with
// C = sum_t 128 * 256^t, m + C is non-negative (|m| < 2^{8S-2} < C) and its
// plain bytes u_t satisfy m = sum_t (u_t - 128) 256^t, so the balanced digit
// is u_t - 128 = u_t ^ 0x80 as an int8 (the representation with digits in
// [-128, 127] is unique: the same digits the carry chain produced). One
// 64-bit add and xor per value; the bytes are gathered into the slice words
// with byte permutes (three per word).
__device__ __forceinline__ void oz_digits16(const double (&xv)[16], int e, int slices, long long slice_bytes,
                                            int8_t* __restrict__ out) {
    const unsigned long long C = 0x8080808080808080ull >> (8 * (8 - slices));
    unsigned lo[16], hi[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const long long m = static_cast<long long>(oz_pow2_mul(xv[j], 8 * slices - 2 - e));
        const unsigned long long u = (static_cast<unsigned long long>(m) + C) ^ C;
        lo[j] = static_cast<unsigned>(u);
        hi[j] = static_cast<unsigned>(u >> 32);
    }
    for (int t = 0; t < slices; ++t) {
        const int b = slices - 1 - t;  // byte of u holding digit t
        const unsigned sel = static_cast<unsigned>(b & 3) | (static_cast<unsigned>(4 + (b & 3)) << 4);
        unsigned w[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            const unsigned p01 = b < 4 ? __byte_perm(lo[4 * g], lo[4 * g + 1], sel) : __byte_perm(hi[4 * g], hi[4 * g + 1], sel);
            const unsigned p23 = b < 4 ? __byte_perm(lo[4 * g + 2], lo[4 * g + 3], sel)
                                       : __byte_perm(hi[4 * g + 2], hi[4 * g + 3], sel);
            w[g] = __byte_perm(p01, p23, 0x5410);
        }
        *reinterpret_cast<uint4*>(out + t * slice_bytes) = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

// k-contiguous rows with 16-byte aligned starts: a thread per (row, 16-value
// chunk) reads its 128 bytes straight from global memory (8 vector loads in
// flight), lanes along rows so every slice word store of a warp is 512
// contiguous bytes. Block: 128 rows x 2 chunks; grid (panels, kpad / 32).
__global__ void __launch_bounds__(256) oz_split_rows(const double* __restrict__ x, long long rows, long long k,
                                                     long long rs, const int* __restrict__ exps, long long kpad,
                                                     int slices, long long slice_bytes, int8_t* __restrict__ out,
                                                     const int* __restrict__ panels) {
    const int rr = threadIdx.x & 127;
    const long long rt = panels ? panels[blockIdx.x] : blockIdx.x;
    const long long R = rt * OZ_BM + rr;
    const long long c0 = (static_cast<long long>(blockIdx.y) * 2 + (threadIdx.x >> 7)) * 16;
    double xv[16];
    if (R < rows && c0 + 16 <= k) {
        const double2* src = reinterpret_cast<const double2*>(x + R * rs + c0);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const double2 v = __ldg(src + j);
            xv[2 * j] = v.x;
            xv[2 * j + 1] = v.y;
        }
    } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) xv[j] = (R < rows && c0 + j < k) ? x[R * rs + c0 + j] : 0.0;
    }
    const int e = R < rows ? exps[R] : 0;
    const long long kt = c0 / OZ_BK, cin = (c0 % OZ_BK) / 16;
    const long long off = (rt * (kpad / OZ_BK) + kt) * (OZ_BM * OZ_BK) + cin * (OZ_BM * 16) + rr * 16;
    oz_digits16(xv, e, slices, slice_bytes, out + off);
}

// Lazy (Khatri-Rao / Hadamard) operands: value(r, k) = prod_f F_f[off_f(r) +
// kstride_f k], off_f(r) = sum_d digit_d(r) rstride_f[d] (r in base n, most
// significant digit first) -- the GEMM operand is never materialized in FP64;
// its digits are formed straight from the (L2-resident) factors.
struct OzLazy {
    int nf = 0, nr = 1;
    long long n = 1;
    const double* ptr[kMaxGemmFactors] = {};
    long long rstride[kMaxGemmFactors][kMaxRowDims] = {};
    long long kstride[kMaxGemmFactors] = {};
};
__device__ __forceinline__ void oz_lazy_bases(const OzLazy& z, long long r, long long k0, const double* (&base)[kMaxGemmFactors]) {
    long long off[kMaxGemmFactors];
#pragma unroll
    for (int f = 0; f < kMaxGemmFactors; ++f) off[f] = 0;
    long long rr = r;
    for (int d = z.nr - 1; d >= 0; --d) {
        const long long dig = rr % z.n;
        rr /= z.n;
#pragma unroll
        for (int f = 0; f < kMaxGemmFactors; ++f)
            if (f < z.nf) off[f] += dig * z.rstride[f][d];
    }
#pragma unroll
    for (int f = 0; f < kMaxGemmFactors; ++f)
        if (f < z.nf) base[f] = z.ptr[f] + off[f] + k0 * z.kstride[f];
}
// vec: every factor has unit K stride and 16-byte aligned rows (double2 loads)
template <int NF, bool VEC>
__global__ void oz_row_exponents_lazy(OzLazy z, long long rows, long long k0, long long k, int* __restrict__ exps) {
    const long long r = blockIdx.x * static_cast<long long>(blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    const double* base[kMaxGemmFactors];
    oz_lazy_bases(z, r, k0, base);
    double mx = 0.0;
    if constexpr (VEC) {
        for (long long c = 2 * lane; c + 1 < k; c += 64) {
            double2 v = make_double2(1.0, 1.0);
#pragma unroll
            for (int f = 0; f < NF; ++f) {
                const double2 w = __ldg(reinterpret_cast<const double2*>(base[f] + c));
                v.x *= w.x;
                v.y *= w.y;
            }
            mx = fmax(mx, fmax(fabs(v.x), fabs(v.y)));
        }
        if ((k & 1) && lane == 0) {
            double v = 1.0;
#pragma unroll
            for (int f = 0; f < NF; ++f) v *= __ldg(base[f] + (k - 1));
            mx = fmax(mx, fabs(v));
        }
    } else {
        for (long long c = lane; c < k; c += 32) {
            double v = 1.0;
#pragma unroll
            for (int f = 0; f < NF; ++f) v *= __ldg(base[f] + c * z.kstride[f]);
            mx = fmax(mx, fabs(v));
        }
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) {
        int e = 0;
        if (mx > 0.0) frexp(mx, &e);
        exps[r] = e;
    }
}
// a thread per (row, 16 values), rows across the warp (as oz_split_rows)
template <int NF, bool VEC>
__global__ void __launch_bounds__(256) oz_split_lazy(OzLazy z, long long rows, long long k0, long long k,
                                                     const int* __restrict__ exps, long long kpad, int slices,
                                                     long long slice_bytes, int8_t* __restrict__ out) {
    const int rr = threadIdx.x & 127;
    const long long rt = blockIdx.x;
    const long long R = rt * OZ_BM + rr;
    const long long c0 = (static_cast<long long>(blockIdx.y) * 2 + (threadIdx.x >> 7)) * 16;
    double xv[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) xv[j] = 0.0;
    if (R < rows) {
        const double* base[kMaxGemmFactors];
        oz_lazy_bases(z, R, k0, base);
        if (VEC && c0 + 16 <= k) {
#pragma unroll
            for (int j = 0; j < 16; ++j) xv[j] = 1.0;
#pragma unroll
            for (int f = 0; f < NF; ++f) {
                const double2* src = reinterpret_cast<const double2*>(base[f] + c0);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const double2 w = __ldg(src + j);
                    xv[2 * j] *= w.x;
                    xv[2 * j + 1] *= w.y;
                }
            }
        } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) xv[j] = c0 + j < k ? 1.0 : 0.0;
#pragma unroll
            for (int f = 0; f < NF; ++f) {
                const long long ks = z.kstride[f];
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (c0 + j < k) xv[j] *= __ldg(base[f] + (c0 + j) * ks);
            }
        }
    }
    const int e = R < rows ? exps[R] : 0;
    const long long kt = c0 / OZ_BK, cin = (c0 % OZ_BK) / 16;
    const long long off = (rt * (kpad / OZ_BK) + kt) * (OZ_BM * OZ_BK) + cin * (OZ_BM * 16) + rr * 16;
    oz_digits16(xv, e, slices, slice_bytes, out + off);
}

// Unit-K-stride factors (VEC): the block's 128 rows x 32 values are formed
// with lanes along K (a half warp reads one row's 256 contiguous bytes of
// every factor as double2, so a warp instruction touches 2 lines instead of
// the 32 a row-per-lane read does: the row-per-lane form ran at the L1
// wavefront rate, 1.2-1.7 TB/s of digits) and staged as FP64 products in
// shared memory (pitch 33: conflict-free for the row-per-lane digit phase,
// which is unchanged: 512-byte coalesced slice stores per warp).
template <int NF>
__global__ void __launch_bounds__(256) oz_split_lazy_tiled(OzLazy z, long long rows, long long k0, long long k,
                                                           const int* __restrict__ exps, long long kpad, int slices,
                                                           long long slice_bytes, int8_t* __restrict__ out) {
    constexpr int P = 33;
    __shared__ double tile[OZ_BM * P];
    __shared__ long long offs[NF][OZ_BM];
    const long long rt = blockIdx.x;
    const long long cb = static_cast<long long>(blockIdx.y) * 32;  // first K value of the block
    if (threadIdx.x < OZ_BM) {
        const long long R = rt * OZ_BM + threadIdx.x;
        const double* base[kMaxGemmFactors];
        if (R < rows) oz_lazy_bases(z, R, k0, base);
#pragma unroll
        for (int f = 0; f < NF; ++f) offs[f][threadIdx.x] = R < rows ? base[f] - z.ptr[f] : 0;
    }
    __syncthreads();
    const int kp2 = threadIdx.x & 15;  // K pair within the 32 values
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int rr = (threadIdx.x >> 4) + 16 * i;
        const long long c = cb + 2 * kp2;
        double2 v = make_double2(0.0, 0.0);
        if (rt * OZ_BM + rr < rows && c < k) {
            if (c + 1 < k) {
                v = make_double2(1.0, 1.0);
#pragma unroll
                for (int f = 0; f < NF; ++f) {
                    const double2 w = __ldg(reinterpret_cast<const double2*>(z.ptr[f] + offs[f][rr] + c));
                    v.x *= w.x;
                    v.y *= w.y;
                }
            } else {  // odd K: the last value alone
                v.x = 1.0;
#pragma unroll
                for (int f = 0; f < NF; ++f) v.x *= __ldg(z.ptr[f] + offs[f][rr] + c);
            }
        }
        tile[rr * P + 2 * kp2] = v.x;
        tile[rr * P + 2 * kp2 + 1] = v.y;
    }
    __syncthreads();
    const int rr = threadIdx.x & 127;
    const int half = threadIdx.x >> 7;
    const long long R = rt * OZ_BM + rr;
    const long long c0 = cb + half * 16;
    double xv[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) xv[j] = tile[rr * P + half * 16 + j];
    const int e = R < rows ? exps[R] : 0;
    const long long kt = c0 / OZ_BK, cin = (c0 % OZ_BK) / 16;
    const long long off = (rt * (kpad / OZ_BK) + kt) * (OZ_BM * OZ_BK) + cin * (OZ_BM * 16) + rr * 16;
    oz_digits16(xv, e, slices, slice_bytes, out + off);
}

constexpr int OZ_SPLIT_THREADS = 256;
__global__ void __launch_bounds__(OZ_SPLIT_THREADS) oz_split(const double* __restrict__ x, long long rows, long long k,
                                                            long long rs, long long ks, const int* __restrict__ exps,
                                                            int th, long long kpad, int slices, long long slice_bytes,
                                                            int8_t* __restrict__ out, const int* __restrict__ panels) {
    extern __shared__ double tilebuf[];  // th x (OZ_BK + 1) doubles
    const long long kt_count = kpad / OZ_BK;
    const long long pi = blockIdx.x / kt_count, kt = blockIdx.x % kt_count;
    const long long rt = panels ? panels[pi] : pi;
    const long long r0 = rt * th, k0 = kt * OZ_BK;
    const int tid = threadIdx.x;
    constexpr int P = OZ_BK + 1;
    if (ks == 1) {  // k-contiguous rows: lanes along k
        for (int i = tid; i < th * OZ_BK; i += OZ_SPLIT_THREADS) {
            const int rr = i / OZ_BK, cc = i % OZ_BK;
            const long long R = r0 + rr, C = k0 + cc;
            tilebuf[rr * P + cc] = (R < rows && C < k) ? x[R * rs + C] : 0.0;
        }
    } else {  // row-contiguous (m-major) operand: lanes along rows
        for (int i = tid; i < th * OZ_BK; i += OZ_SPLIT_THREADS) {
            const int cc = i / th, rr = i % th;
            const long long R = r0 + rr, C = k0 + cc;
            tilebuf[rr * P + cc] = (R < rows && C < k) ? x[R * rs + C * ks] : 0.0;
        }
    }
    __syncthreads();
    const long long tile_off = (rt * kt_count + kt) * (static_cast<long long>(th) * OZ_BK);
    for (int item = tid; item < th * (OZ_BK / 16); item += OZ_SPLIT_THREADS) {
        const int rr = item % th, cin = item / th;  // consecutive threads: consecutive rows of one chunk
        const long long R = r0 + rr;
        const int e = R < rows ? exps[R] : 0;
        double xv[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) xv[j] = tilebuf[rr * P + cin * 16 + j];
        oz_digits16(xv, e, slices, slice_bytes, out + tile_off + cin * (th * 16) + rr * 16);
    }
}

}  // namespace

std::size_t ozaki_slice_bytes(long long rows, long long k, int tile_rows) {
    const long long rp = (rows + tile_rows - 1) / tile_rows * tile_rows;
    const long long kp = (k + OZ_BK - 1) / OZ_BK * OZ_BK;
    return static_cast<std::size_t>(rp * kp);
}

int ozaki_split(const double* x, long long rows, long long k, long long rs, long long ks, int tile_rows, int slices,
                int8_t* out, int* exps, cudaStream_t s, const std::vector<int>* panels) {
    if (slices < 1 || slices > kOzMaxSlices || tile_rows != OZ_BM) return -1;
    const long long rp = (rows + tile_rows - 1) / tile_rows * tile_rows;
    const long long kp = (k + OZ_BK - 1) / OZ_BK * OZ_BK;
    int* dpanels = nullptr;
    long long npanels = rp / tile_rows;
    if (panels) {  // only these 128-row panels (a row-sharded rank's tiles read no others)
        npanels = static_cast<long long>(panels->size());
        if (npanels == 0) return 0;
        if (cudaMallocAsync(reinterpret_cast<void**>(&dpanels), sizeof(int) * panels->size(), s) != cudaSuccess) {
            cudaGetLastError();
            return -1;
        }
        cudaMemcpyAsync(dpanels, panels->data(), sizeof(int) * panels->size(), cudaMemcpyHostToDevice, s);
    }
    const long long exp_rows = panels ? npanels * tile_rows : rows;
    oz_row_exponents<<<static_cast<unsigned>((exp_rows + 7) / 8), 256, 0, s>>>(x, rows, k, rs, ks, exps, dpanels);
    const int smem = tile_rows * (OZ_BK + 1) * static_cast<int>(sizeof(double));
    set_max_smem_once(reinterpret_cast<const void*>(oz_split), smem);
    if (ks == 1 && rs % 2 == 0 && reinterpret_cast<std::uintptr_t>(x) % 16 == 0)
        oz_split_rows<<<dim3(static_cast<unsigned>(npanels), static_cast<unsigned>(kp / 32)), 256, 0, s>>>(
            x, rows, k, rs, exps, kp, slices, rp * kp, out, dpanels);
    else
        oz_split<<<static_cast<unsigned>(npanels * (kp / OZ_BK)), OZ_SPLIT_THREADS, smem, s>>>(
            x, rows, k, rs, ks, exps, tile_rows, kp, slices, rp * kp, out, dpanels);
    if (dpanels) cudaFreeAsync(dpanels, s);
    return 2;
}

int ozaki_split_lazy(const GemmSide& side, long long n, long long rows, long long k0, long long k, int slices,
                     int8_t* out, int* exps, cudaStream_t s) {
    if (slices < 1 || slices > kOzMaxSlices || side.nf < 1 || side.nf > kMaxGemmFactors || side.nr > kMaxRowDims)
        return -1;
    OzLazy z;
    z.nf = side.nf;
    z.nr = side.nr;
    z.n = n;
    for (int f = 0; f < side.nf; ++f) {
        z.ptr[f] = side.ptr[f];
        z.kstride[f] = side.kstride[f];
        for (int d = 0; d < side.nr; ++d) z.rstride[f][d] = side.rstride[f][d];
    }
    const long long rp = (rows + OZ_BM - 1) / OZ_BM * OZ_BM;
    const long long kp = (k + OZ_BK - 1) / OZ_BK * OZ_BK;
    // unit K strides, even row offsets and 16-byte aligned bases: double2 loads
    bool vec = true;
    for (int f = 0; f < z.nf; ++f) {
        vec &= z.kstride[f] == 1 && (reinterpret_cast<std::uintptr_t>(z.ptr[f] + k0) & 15) == 0;
        for (int d = 0; d < z.nr; ++d) vec &= (z.rstride[f][d] & 1) == 0;
    }
    const dim3 eg(static_cast<unsigned>((rows + 7) / 8)), sg(static_cast<unsigned>(rp / OZ_BM), static_cast<unsigned>(kp / 32));
    auto go = [&](auto nf) {
        constexpr int NF = decltype(nf)::value;
        if (vec) {
            oz_row_exponents_lazy<NF, true><<<eg, 256, 0, s>>>(z, rows, k0, k, exps);
            oz_split_lazy_tiled<NF><<<sg, 256, 0, s>>>(z, rows, k0, k, exps, kp, slices, rp * kp, out);
        } else {
            oz_row_exponents_lazy<NF, false><<<eg, 256, 0, s>>>(z, rows, k0, k, exps);
            oz_split_lazy<NF, false><<<sg, 256, 0, s>>>(z, rows, k0, k, exps, kp, slices, rp * kp, out);
        }
    };
    switch (z.nf) {
        case 2: go(std::integral_constant<int, 2>{}); break;
        case 3: go(std::integral_constant<int, 3>{}); break;
        case 4: go(std::integral_constant<int, 4>{}); break;
        case 5: go(std::integral_constant<int, 5>{}); break;
        case 6: go(std::integral_constant<int, 6>{}); break;
        default: return -1;
    }
    return 2;
}

void ozaki_tile_panels(const OzakiArgs& p, std::vector<int>* a_panels, std::vector<int>* b_panels) {
    const long long total = ozaki_tile_count(p);
    const long long end = p.tile_count < 0 ? total : p.tile_begin + p.tile_count;
    std::vector<char> ma(static_cast<std::size_t>(p.mpad / OZ_BM), 0), mb(static_cast<std::size_t>(p.npad / OZ_BN), 0);
    for (long long b = p.tile_begin; b < end; ++b) {
        long long tm = 0, tn = 0;
        oz_tile_of(p, b, &tm, &tn);
        ma[static_cast<std::size_t>(tm)] = 1;
        mb[static_cast<std::size_t>(tn)] = 1;
    }
    a_panels->clear();
    b_panels->clear();
    for (std::size_t i = 0; i < ma.size(); ++i)
        if (ma[i]) a_panels->push_back(static_cast<int>(i));
    for (std::size_t i = 0; i < mb.size(); ++i)
        if (mb[i]) b_panels->push_back(static_cast<int>(i));
}

// The per-SM high-diagonal scratch is indexed by %smid, which PTX bounds only
// by %nsmid (not by the enabled SM count): kOzWorkSlots covers every SM id a
// Blackwell part exposes, and the kernel traps on anything beyond it.
std::size_t ozaki_work_entries() { return static_cast<std::size_t>(kOzWorkSlots) * OZ_BM * OZ_BN; }

namespace {
long long ozaki_sm_count() {  // per device (function attributes and SM counts are per device)
    static std::mutex mu;
    static std::map<int, int> by_dev;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    int& v = by_dev[dev];
    if (!v) {
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        if (v <= 0) v = 148;
    }
    return v;
}
}  // namespace

long long ozaki_tile_count(const OzakiArgs& p) {
    const long long tiles_m = p.mpad / OZ_BM, tiles_n = p.npad / OZ_BN;
    return p.symmetric ? tiles_n * (tiles_n + 1) / 2 : tiles_m * tiles_n;
}

template <int S>
void launch_oz(const OzakiArgs& p, long long tiles, cudaStream_t s) {
    const int bytes = static_cast<int>(sizeof(OzSmem));
    set_max_smem_once(reinterpret_cast<const void*>(ozaki_gemm_kernel<S>), bytes);
    ozaki_gemm_kernel<S><<<static_cast<unsigned>(tiles), OZ_THREADS, bytes, s>>>(p);
}

using OzEncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
OzEncodeFn oz_encoder() {
    static OzEncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<OzEncodeFn>(f);
    });
    return fn;
}
// digits of `slices` slices of `panels` 128-row panels x ktiles tiles as
// (16 B, 128 rows, 4 * ktiles * panels * slices K columns); box rows = box_rows
bool oz2_encode(CUtensorMap* map, const int8_t* base, long long panels, long long ktiles, int slices, int box_rows) {
    OzEncodeFn fn = oz_encoder();
    if (!fn) return false;
    // 8-byte elements: the innermost box run is 64 rows x 16 B = 1 KiB contiguous
    // (a 16-byte innermost run measured 1.8x slower: TMA moves short rows poorly)
    const cuuint64_t dims[3] = {128, 2, static_cast<cuuint64_t>(4 * ktiles * panels * slices)};
    const cuuint64_t strides[2] = {64 * 16, 128 * 16};
    const cuuint32_t box[3] = {128, static_cast<cuuint32_t>(box_rows / 64), 4}, estr[3] = {1, 1, 1};
    return fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<int8_t*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int S>
bool launch_oz2(const OzakiArgs& p, long long clusters, cudaStream_t s) {
    CUtensorMap ma, mb;
    const long long ktiles = p.kpad / OZ_BK;
    if (!oz2_encode(&ma, p.a, p.mpad / OZ_BM, ktiles, p.slices, OZ_BM) ||
        !oz2_encode(&mb, p.b, p.npad / OZ_BN, ktiles, p.slices, OZ_BN / 2))
        return false;
    const int bytes = static_cast<int>(sizeof(Oz2Smem));
    set_max_smem_once(reinterpret_cast<const void*>(ozaki_gemm_2sm_kernel<S>), bytes);
    ozaki_gemm_2sm_kernel<S><<<static_cast<unsigned>(2 * clusters), OZ_THREADS, bytes, s>>>(ma, mb, p);
    return true;
}

// The CTA-pair kernel (default; USTATS_OZ_2SM=0 selects the single-SM one):
// whole launches only (a row-sharded tile range keeps the single-SM tile list).
bool oz2_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("USTATS_OZ_2SM");
        return !(e && e[0] == '0');
    }();
    return on;
}

int launch_ozaki_gemm(const OzakiArgs& in, cudaStream_t s) {
    if (in.kpad % OZ_BK != 0) return -1;
    // int32 accumulators exact: at most S products each, S - 1 with the split top diagonal (S > 4)
    if (static_cast<long long>(in.slices > 4 ? in.slices - 1 : in.slices) * in.kpad * 128 * 128 >= (1ll << 31)) return -1;
    if (oz2_enabled() && in.tile_count < 0 && in.tile_begin == 0 && in.mpad >= 2 * OZ_BM) {
        OzakiArgs p = in;
        p.prefetch = 0;
        p.tail_split = 1;
        // row groups of 2 pair rows (4 tile rows): their A digit panels stay
        // L2-resident while the B panels stream past (C5, n = 65536: 25.1 ->
        // 22.9 s per evaluation; less DRAM traffic, so higher clocks under the
        // power cap; profiles/r02_l2_grouping.log)
        p.group2 = 2;
        p.sym_group2 = 2;
        const long long pairs = oz2_pair_count(p);
        p.pairs = pairs;
        // persistent: one cluster per SM pair looping over the pair tiles;
        // long-K launches also keep their waves in lock step (wave barrier)
        const long long ktiles = p.kpad / OZ_BK;
        int persist = 1, lockstep = ktiles >= 64 ? 1 : 0;
        if (const char* e = std::getenv("USTATS_OZ2_PERSIST")) persist = std::atoi(e);
        if (const char* e = std::getenv("USTATS_OZ2_LOCKSTEP")) lockstep = std::atoi(e);
        if (lockstep && persist) p.group2 = p.sym_group2 = 8;  // square waves: fewest distinct panels
        if (const char* e = std::getenv("USTATS_OZ2_GROUP")) p.group2 = std::atoi(e);
        if (const char* e = std::getenv("USTATS_OZ2_SYMG")) p.sym_group2 = std::atoi(e);
        const long long slots = ozaki_sm_count() / 2;
        const long long clusters = persist ? std::min(pairs, slots) : pairs;
        if (persist && lockstep && pairs > clusters) {
            if (cudaPeekAtLastError() != cudaSuccess) return -1;
            if (cudaMallocAsync(reinterpret_cast<void**>(&p.wave_ctr), 2 * sizeof(unsigned long long), s) != cudaSuccess) {
                cudaGetLastError();  // exactly this allocation error: run without the wave barrier
                p.wave_ctr = nullptr;
            } else {
                cudaMemsetAsync(p.wave_ctr, 0, 2 * sizeof(unsigned long long), s);
            }
            if (const char* e = std::getenv("USTATS_OZ2_RESYNC")) p.resync = std::atoi(e);
        }
        bool ok = false;
        switch (p.slices) {
            case 4: ok = launch_oz2<4>(p, clusters, s); break;
            case 5: ok = launch_oz2<5>(p, clusters, s); break;
            case 6: ok = launch_oz2<6>(p, clusters, s); break;
            case 7: ok = launch_oz2<7>(p, clusters, s); break;
            default: return -1;
        }
        if (p.wave_ctr) cudaFreeAsync(p.wave_ctr, s);
        if (ok) return 1 + launch_epilogue_finalize(p.m, p.n, p.epis, ozaki_tile_count(p), p.accumulate, s);
        // no tensor-map encoder: the single-SM kernel below
    }
    OzakiArgs p = in;
    // warming L2 k-tiles ahead of the bulk copies (p.prefetch > 0) paid with the
    // 2-stage ring of the first version (C2 +2%); with pass 1 on its deeper ring
    // it no longer does (C2 -0.5%, C3 -9%), so it is off
    p.prefetch = 0;
    const long long total = ozaki_tile_count(p);
    const long long tiles = p.tile_count < 0 ? total - p.tile_begin : p.tile_count;
    if (tiles <= 0) return 0;
    // one CTA per SM: a last wave at most half full runs its tiles split along K
    // over the SMs the full waves leave idle (C2: 2080 tiles = 14 x 148 + 8)
    const long long sms = ozaki_sm_count();
    const long long rem = tiles % sms, ktiles = p.kpad / OZ_BK;
    long long grid = tiles;
    p.tail_split = 1;
    if (rem > 0 && 2 * rem <= sms) {
        const long long split = std::min({sms / rem, ktiles / 4, static_cast<long long>(kOzMaxTailSplit)});
        if (split >= 2) {
            const std::size_t part = static_cast<std::size_t>(rem * split) * OZ_BM * OZ_BN * sizeof(double);
            if (cudaPeekAtLastError() != cudaSuccess) return -1;  // an earlier launch failed: report, never mask it
            const cudaError_t e1 = cudaMallocAsync(reinterpret_cast<void**>(&p.tail_part), part, s);
            const cudaError_t e2 =
                e1 == cudaSuccess ? cudaMallocAsync(reinterpret_cast<void**>(&p.tail_count), sizeof(unsigned) * rem, s)
                                  : cudaSuccess;
            if (e1 == cudaSuccess && e2 == cudaSuccess) {
                cudaMemsetAsync(p.tail_count, 0, sizeof(unsigned) * rem, s);
                p.tail_split = static_cast<int>(split);
                p.tail_from = tiles - rem;
                grid = p.tail_from + rem * split;
            } else {
                // no room for the partial tiles: the tail runs unsplit (same result, later)
                if ((e1 != cudaSuccess && e1 != cudaErrorMemoryAllocation) ||
                    (e2 != cudaSuccess && e2 != cudaErrorMemoryAllocation))
                    return -1;
                cudaGetLastError();  // exactly the allocation error just returned
                if (e1 == cudaSuccess) cudaFreeAsync(p.tail_part, s);
                p.tail_part = nullptr;
                p.tail_count = nullptr;
            }
        }
    }
    switch (p.slices) {
        case 4: launch_oz<4>(p, grid, s); break;
        case 5: launch_oz<5>(p, grid, s); break;
        case 6: launch_oz<6>(p, grid, s); break;
        case 7: launch_oz<7>(p, grid, s); break;
        default: return -1;
    }
    if (p.tail_split > 1) {
        cudaFreeAsync(p.tail_part, s);
        cudaFreeAsync(p.tail_count, s);
    }
    return 1 + launch_epilogue_finalize(p.m, p.n, p.epis, tiles, p.accumulate, s);
}

}  // namespace ustats::dev
