// The fused GEMM epilogues (EpiDesc / EpiSet, kernels.hpp) over a 128 x 128
// FP64 product tile staged in shared memory (pitch TP), shared by the DMMA
// TMA kernel (gemm_tma.cu, 256 threads) and the INT8-emulated kernel
// (gemm_ozaki.cu, 256 epilogue threads). NT threads of the calling group take part;
// `sync()` must synchronize exactly them. Fixed-order reductions: every
// scalar partial is a warp tree then an in-order sum over the NT/32 warps.
#pragma once

#include "kernels.hpp"

namespace ustats::dev::epi {

constexpr int BM = 128, BN = 128, TP = BN + 1;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <int NT, class Sync>
__device__ __forceinline__ void apply(const EpiSet& epis, long long rows, long long cols, int accumulate,
                                      const double* tile, long long r0, long long c0, long long tm, long long tn,
                                      bool mirror, long long slot, double* red, int tid, Sync sync) {
    const int warp = tid >> 5, lane = tid & 31;
    for (int q = 0; q < epis.count; ++q) {
        const EpiDesc& d = epis.d[q];
        auto W = [&](long long R, long long C) {
            double w = 1.0;
            for (int f = 0; f < d.nw; ++f) w *= __ldg(d.wptr[f] + R * d.wr[f] + C * d.wc[f]);
            return w;
        };
        auto P = [&](double x) { return d.self_power == 2 ? x * x : x; };
        // element order: column-fastest unless the first weight is column-major
        const bool cfast = !(d.nw > 0 && d.wr[0] == 1 && d.wc[0] != 1);
        if (d.mode == kEpiStore && d.nw == 0 && !d.transpose) {  // plain store: a warp per row, lanes along it
            for (int r = warp; r < BM; r += NT / 32) {
                const long long R = r0 + r;
                if (R >= rows) break;
                double* o = d.out + R * cols + c0;
#pragma unroll 4
                for (int c = lane; c < BN; c += 32)
                    if (c0 + c < cols) {
                        const double v = P(tile[r * TP + c]);
                        o[c] = accumulate ? o[c] + v : v;
                    }
            }
            if (mirror)  // out[C][R] = tile[R][C]: a warp per tile column, lanes down it
                for (int c = warp; c < BN; c += NT / 32) {
                    const long long C = c0 + c;
                    if (C >= cols) break;
                    double* o = d.out + C * cols + r0;
#pragma unroll 4
                    for (int r = lane; r < BM; r += 32)
                        if (r0 + r < rows) {
                            const double v = P(tile[r * TP + c]);
                            o[r] = accumulate ? o[r] + v : v;
                        }
                }
        } else if (d.mode == kEpiSumAll) {
            // a warp per line of the tile, lanes along it (columns when the first weight is
            // row-major, else rows, so weight loads coalesce); per-line weight bases hoisted
            double s = 0.0;
            auto lines = [&](bool transposed) {  // transposed: the mirror tile, weights at (C, R)
                for (int l = warp; l < BM; l += NT / 32) {
                    // line l: a tile row (cfast) or a tile column; position q along it
                    const double* base[kMaxEpiW];
                    long long step[kMaxEpiW];
                    const long long L = (cfast ? r0 : c0) + l;
                    if (L >= (cfast ? rows : cols)) break;
                    for (int f = 0; f < d.nw; ++f) {
                        // weight index (R, C) or, mirrored, (C, R)
                        const long long sl = transposed ? (cfast ? d.wc[f] : d.wr[f]) : (cfast ? d.wr[f] : d.wc[f]);
                        const long long sq = transposed ? (cfast ? d.wr[f] : d.wc[f]) : (cfast ? d.wc[f] : d.wr[f]);
                        base[f] = d.wptr[f] + L * sl + (cfast ? c0 : r0) * sq;
                        step[f] = sq;
                    }
                    const long long qn = (cfast ? cols - c0 : rows - r0) < BN ? (cfast ? cols - c0 : rows - r0) : BN;
                    for (int q = lane; q < qn; q += 32) {
                        const int r = cfast ? l : q, c = cfast ? q : l;
                        double w = P(tile[r * TP + c]);
                        for (int f = 0; f < d.nw; ++f) w *= __ldg(base[f] + q * step[f]);
                        s += w;
                    }
                }
            };
            lines(false);
            if (mirror) lines(true);
            s = warp_sum(s);
            if (lane == 0) red[warp] = s;
            sync();
            if (tid == 0) {
                double tot = 0.0;
                for (int w = 0; w < NT / 32; ++w) tot += red[w];
                d.partial[slot] = tot;
            }
            sync();
        } else if (d.mode == kEpiStore || d.mode == kEpiSumAll) {
            double s = 0.0;
            for (int i = tid; i < BM * BN; i += NT) {
                const int r = cfast ? (i >> 7) : (i & 127), c = cfast ? (i & 127) : (i >> 7);
                const long long R = r0 + r, C = c0 + c;
                if (R >= rows || C >= cols) continue;
                const double v = P(tile[r * TP + c]) * W(R, C);
                if (d.mode == kEpiStore) {
                    double& o = d.out[d.transpose ? C * rows + R : R * cols + C];
                    o = accumulate ? o + v : v;
                } else {
                    s += v;
                }
            }
            if (mirror)  // the transposed tile (C, R): same values, weights at (C, R)
                for (int i = tid; i < BM * BN; i += NT) {
                    const int c = cfast ? (i >> 7) : (i & 127), r = cfast ? (i & 127) : (i >> 7);
                    const long long R = r0 + r, C = c0 + c;
                    if (R >= rows || C >= cols) continue;
                    const double v = P(tile[r * TP + c]) * W(C, R);
                    if (d.mode == kEpiStore) {
                        double& o = d.out[d.transpose ? R * rows + C : C * cols + R];
                        o = accumulate ? o + v : v;
                    } else {
                        s += v;
                    }
                }
            if (d.mode == kEpiSumAll) {
                s = warp_sum(s);
                if (lane == 0) red[warp] = s;
                sync();
                if (tid == 0) {
                    double tot = 0.0;
                    for (int w = 0; w < NT / 32; ++w) tot += red[w];
                    d.partial[slot] = tot;
                }
                sync();
            }
        } else if (d.mode == kEpiSumCols) {  // out[R] = sum_C
            for (int r = warp; r < BM; r += NT / 32) {
                const long long R = r0 + r;
                double s = 0.0;
                for (int c = lane; c < BN; c += 32) {
                    const long long C = c0 + c;
                    if (R < rows && C < cols) s += P(tile[r * TP + c]) * W(R, C);
                }
                s = warp_sum(s);
                if (lane == 0 && R < rows) d.partial[tn * rows + R] = s;
            }
            if (mirror)
                for (int c = warp; c < BN; c += NT / 32) {
                    const long long C = c0 + c;
                    double s = 0.0;
                    for (int r = lane; r < BM; r += 32) {
                        const long long R = r0 + r;
                        if (R < rows && C < cols) s += P(tile[r * TP + c]) * W(C, R);
                    }
                    s = warp_sum(s);
                    if (lane == 0 && C < rows) d.partial[tm * rows + C] = s;
                }
        } else {  // kEpiSumRows: out[C] = sum_R
            if (tid < BN) {
                const int c = tid;
                const long long C = c0 + c;
                double s = 0.0;
                for (int r = 0; r < BM; ++r) {
                    const long long R = r0 + r;
                    if (R < rows && C < cols) s += P(tile[r * TP + c]) * W(R, C);
                }
                if (C < cols) d.partial[tm * cols + C] = s;
            }
            if (mirror && tid >= NT - BM) {
                const int r = tid - (NT - BM);
                const long long R = r0 + r;
                double s = 0.0;
                for (int c = 0; c < BN; ++c) {
                    const long long C = c0 + c;
                    if (R < rows && C < cols) s += P(tile[r * TP + c]) * W(C, R);
                }
                if (R < cols) d.partial[tn * cols + R] = s;
            }
        }
    }
}

}  // namespace ustats::dev::epi
