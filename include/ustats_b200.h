/*
 * ustats_b200 — C-ABI of the B200 exact-U-statistic engine.
 *
 * Drop-in boundary for the reference's FFI on this path: the pybind11 module
 * `_ustats` (proj/python/ustats_py.cpp:68-174) and the C++ entry points it
 * wraps (proj/include/ustats/engine.hpp:32-65, einsum.hpp:41-52). Every
 * function is `extern "C"`, takes plain pointers and sizes, never throws, and
 * returns 0 on success or 1 + the reference ErrorCode value
 * (proj/include/ustats/errors.hpp:10-28; CudaError = 18, CollectiveError = 19)
 * with the message in us_last_error() (thread-local).
 *
 * Problem encoding shared by the statistic calls (the tensor-backed form of
 * MDKernel, kernel.hpp:39-54, after tensorize):
 *   m          kernel arity
 *   K          number of components
 *   tuple_len  K entries: |signature[k]|
 *   tuple_idx  concatenated 0-based slots of signature[k]
 *   factors    K pointers: component k materialized over [0,n)^|sig[k]|,
 *              row-major f64, NOT sparsified (the engine sparsifies on device).
 *              Equal pointers denote the same tensor and are uploaded once.
 *   n          sample size (shared extent)
 *   on_device  0: factors are host memory; 1: CUDA device memory (read-only)
 */
#ifndef USTATS_B200_H
#define USTATS_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define US_API __attribute__((visibility("default")))
#else
#define US_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Config (proj/include/ustats/config.hpp:17-44) plus the device section. */
typedef struct us_config {
    uint64_t memory_cap_entries; /* 0 = reference default 2^31 */
    int32_t threads;             /* host threads for tensorization (0 = hw) */
    int32_t strategy;            /* OrderStrategy: 0 Auto, 1 MinDegree, 2 MinFill, 3 Exhaustive */
    int32_t exhaustive_index_bound; /* 0 = 12 */
    int32_t exact_treewidth_bound;  /* 0 = 10 */
    int32_t device;              /* CUDA ordinal, -1 = current */
    int32_t rank;                /* term-sharding rank */
    int32_t world_size;          /* term-sharding world size (1 = all terms here) */
    int32_t flags;               /* bit0 share, bit1 fuse epilogues, bit2 symmetry, bit3 reorder,
                                    bit4 donate device inputs (sparsified in place, no copy),
                                    bit5 row sharding across ranks (else V-term sharding),
                                    bit6 serial launch (one stream),
                                    bit7 exact DMMA only (no INT8 tensor-core emulation of
                                    large FP64 GEMMs),
                                    bit8 no CUDA-graph replay of repeated small data-API calls;
                                    US_FLAGS_DEFAULT = 0xF */
    int32_t emulate_world;       /* row sharding over this many virtual ranks on one device (tests) */
    uint64_t memory_budget_bytes; /* device bytes the memory-bounded schedule may plan for (0 = free memory) */
    int32_t oz_slices;           /* emulated-GEMM digit slices (0 = error-bound guard; 4..7 forced) */
    int32_t oz_min_dim;          /* smallest rows / cols / K of an emulated GEMM (0 = 1024; tests lower it to
                                    pin the emulated path against the reference at sizes its CPU run reaches) */
    int64_t oz_max_k;            /* longest emulated K per pass (0 = 21000, the int32-exact bound) */
} us_config;

#define US_FLAGS_DEFAULT 0xF

/* RunStats (engine.hpp:17-25) + device counters. */
typedef struct us_stats {
    double tensorize_seconds;       /* upload + on-device sparsify */
    double contract_seconds;
    uint64_t einsum_calls;
    uint64_t partitions_enumerated;
    uint64_t partitions_evaluated;
    uint64_t multiply_adds;         /* reference-plan counting rules */
    uint64_t peak_intermediate_entries;
    uint64_t executed_gemm_macs;    /* DMMA multiply-adds issued */
    uint64_t executed_stream_entries;
    uint64_t gemm_launches;
    uint64_t stream_launches;
    uint64_t shared_hits;
    uint64_t kernel_launches;       /* every kernel this call enqueued */
    uint64_t emulated_gemm_macs;    /* FP64 multiply-adds done on the INT8 tensor cores (Ozaki) */
    uint64_t int8_tensor_ops;       /* INT8 tensor-core operations those issued (2 per MAC) */
    uint64_t oz_slices;             /* digit slices of the emulated GEMMs (error-bound guard; 0 = none ran) */
} us_stats;

US_API const char* us_version(void);
US_API const char* us_last_error(void);
US_API void us_config_default(us_config* cfg);

/* u_statistic after tensorize (engine.cpp:173-193; ustats_py.cpp:92-101). */
US_API int us_u_statistic(int32_t m, int32_t K, const int32_t* tuple_len, const int32_t* tuple_idx,
                   const double* const* factors, int64_t n, int32_t on_device,
                   const us_config* cfg, double* u_out, us_stats* stats);

/* Same evaluation, also returning every survivor in enumeration order:
 * rgs_out[t*m + i], mu_out[t], v_out[t] (raw V; 0 when owned by another rank),
 * owner_out[t] (rank). Capacity max_terms; *count receives the survivor count.
 * lattice_combination per-term values (engine.cpp:67-73). */
US_API int us_u_terms(int32_t m, int32_t K, const int32_t* tuple_len, const int32_t* tuple_idx,
               const double* const* factors, int64_t n, int32_t on_device, const us_config* cfg,
               int32_t max_terms, int32_t* count, int32_t* rgs_out, int64_t* mu_out, double* v_out,
               int32_t* owner_out, double* u_out, us_stats* stats);

/* Data-level u_statistic (engine.cpp:173-193 including tensorize, and
 * _ustats.u_statistic(kernel, data), ustats_py.cpp:92-101): the kernel spec's
 * components are tensorized ON THE DEVICE from the sample (n rows x d columns,
 * row-major; host or device memory), so only the sample crosses PCIe.
 * Specs: "prod2", "hoif:<j>:<k>" (hoif.cpp:50-72), "rbf:<shape>:<h>"
 * (exp(-|x_i-x_j|^2/(2h^2)); shape chain<m> | cycle<m> | k4tail) and
 * "proj:<m>:<kmax>" (r B..B e chain, B = Z(Z'Z/n)^-1 Z' of cosine features
 * cos(pi k u), k=1..kmax, of the first d-2 columns; r, e the last two).
 * stats->tensorize_seconds is the device tensorization time. */
US_API int us_u_statistic_data(const char* kernel, const double* data, int64_t n, int32_t d, int32_t on_device,
                               const us_config* cfg, double* u_out, us_stats* stats);

/* Several U-statistics over factors of one extent n, evaluated as ONE device
 * program (factors uploaded once, sub-contractions shared across statistics;
 * e.g. hoif_tau's chain orders, hoif.cpp:74-100). Statistic s has arity m[s]
 * and K[s] components; tuple_len / tuple_idx / factors are the per-statistic
 * encodings concatenated in statistic order. u_out receives S values. */
/* Callers of the path (SURVEY 8b "callers to keep working"), evaluated on the
 * device end to end:
 * us_dcov_squared: dcov_squared (dcov.hpp:22-23) of paired samples x (n x dx)
 *   and y (n x dy), row-major, host or device; the four U-statistics share one
 *   program. SampleTooSmall below 4 pairs.
 * us_motif_count: motif_count (motifs.hpp:47-48) of motif id "r1".."r8" in the
 *   graph on vertices 0..n-1 given by edge_count (u, v) pairs (host int32);
 *   NonIntegerResult when the scaled count is not integral. */
/* hoif_tau (hoif.hpp:44-48, hoif.cpp:74-100) with the truncation basis
 * phi(z) = z[0..k) (truncation_phi, hoif.cpp:37-47) on a sample of n rows
 * [A, Y, Z_1..Z_{d-2}] (row-major, host or device): the two component
 * matrices are tensorized on the device, the chain orders 2..m run as one
 * program, and the alternating-sign combination accumulates in long double.
 * InvalidArgument for m < 2, k < 1 or d < 2 + k; SampleTooSmall for n < m. */
US_API int us_hoif_tau(int32_t m, int32_t k, const double* data, int64_t n, int32_t d, int32_t on_device,
                       const us_config* cfg, double* tau_out, us_stats* stats);

US_API int us_dcov_squared(const double* x, int32_t dx, const double* y, int32_t dy, int64_t n,
                           int32_t on_device, const us_config* cfg, double* out, us_stats* stats);
US_API int us_motif_count(int64_t n, int64_t edge_count, const int32_t* edges, const char* motif_id,
                          const us_config* cfg, int64_t* count, us_stats* stats);

US_API int us_u_statistic_batch(int32_t S, const int32_t* m, const int32_t* K, const int32_t* tuple_len,
                                const int32_t* tuple_idx, const double* const* factors, int64_t n,
                                int32_t on_device, const us_config* cfg, double* u_out, us_stats* stats);

/* u_statistic_unsparsified (engine.cpp:195-211): every lattice partition. */
US_API int us_u_statistic_unsparsified(int32_t m, int32_t K, const int32_t* tuple_len,
                                const int32_t* tuple_idx, const double* const* factors, int64_t n,
                                int32_t on_device, const us_config* cfg, double* u_out,
                                us_stats* stats);

/* v_statistic (engine.cpp:138-151): one contraction of the raw signature. */
US_API int us_v_statistic(int32_t m, int32_t K, const int32_t* tuple_len, const int32_t* tuple_idx,
                   const double* const* factors, int64_t n, const us_config* cfg, double* v_out,
                   us_stats* stats);

/* restricted_v (engine.cpp:153-171): contraction of the induced signature of rgs. */
US_API int us_restricted_v(int32_t m, int32_t K, const int32_t* tuple_len, const int32_t* tuple_idx,
                    const double* const* factors, int64_t n, const int32_t* rgs,
                    const us_config* cfg, double* v_out, us_stats* stats);

/* einsum (einsum.hpp:41-43; ustats_py.cpp:73-90): tensors[k] has order
 * tuple_len[k] over extent n (host memory); output tuple out_idx[0..out_len);
 * `order` (nullable, order_len entries) an explicit elimination order over
 * the canonical ids. out receives n^out_len entries. */
US_API int us_einsum(int32_t K, const int32_t* tuple_len, const int32_t* tuple_idx,
              const double* const* tensors, int64_t n, int32_t out_len, const int32_t* out_idx,
              const int32_t* order, int32_t order_len, const us_config* cfg, double* out,
              uint64_t* multiply_adds, uint64_t* peak_entries, int32_t* steps);

/* eliminate_index (einsum.hpp:49-52): result over the ascending union of the
 * other ids, written to out (capacity out_cap entries) and out_tuple. */
US_API int us_eliminate_index(int32_t K, const int32_t* tuple_len, const int32_t* tuple_idx,
                       const double* const* tensors, int64_t n, int32_t index,
                       const us_config* cfg, double* out, uint64_t out_cap, int32_t* out_tuple,
                       int32_t* out_tuple_len);

/* The reference's combination of per-term values (engine.cpp:47-104):
 * term_t = mu_t * v_t, pairwise tree per 512-term chunk, chunks summed in order.
 * Pure host arithmetic; bit-identical to the reference given identical v. */
US_API double us_combine_terms(int32_t count, const int64_t* mu, const double* v);

/* Host-side lattice/planning helpers (no GPU needed). us_survivors always
 * sets *count to the full survivor count; when it exceeds max_terms it
 * returns TooManyTerms after writing the first max_terms. */
US_API uint64_t us_bell_number(int32_t m);
US_API int us_survivors(int32_t m, int32_t K, const int32_t* tuple_len, const int32_t* tuple_idx,
                 int32_t max_terms, int32_t* count, int32_t* rgs_out, int64_t* mu_out,
                 uint64_t* enumerated);
US_API int us_optimize_order(int32_t K, const int32_t* tuple_len, const int32_t* tuple_idx,
                      int32_t strategy, int32_t* order_out, int32_t* index_count,
                      int32_t* width_out);
US_API int us_treewidth(int32_t n, int32_t edge_count, const int32_t* edges, int32_t* width_out,
                 int32_t* order_out);

/* complexity_report (proj/include/ustats/complexity.hpp:46-47, host only):
 * lattice sizes, the survivors' exact quotient-treewidth histogram and the
 * exact decimal FLOP estimate K * sum_w count_w * n^(w+1) (into flops[0..cap),
 * NUL-terminated). Tuples may be 0- or 1-based (canonicalized as
 * validate_notation does). treewidth_exact is -1 when m exceeds
 * cfg->exact_treewidth_bound. */
typedef struct us_complexity {
    int32_t index_count, extent, graph_vertices, graph_edges;
    int32_t treewidth_lower, treewidth_upper, treewidth_exact, max_quotient_width;
    uint64_t bell_count, sparsified_count;
    uint64_t count_by_width[16]; /* [w] = survivors whose quotient has treewidth w */
} us_complexity;
US_API int us_complexity_report(int32_t K, const int32_t* tuple_len, const int32_t* tuple_idx,
                                int32_t extent, const us_config* cfg, us_complexity* out,
                                char* flops, int32_t cap);

/* Term sharding plan (host only): for the sparsified lattice of the
 * signature at extent n over world_size ranks, owner_out[t] receives the rank
 * that evaluates survivor t (LPT on n^(width+1)), cost_out[t] its estimate. */
US_API int us_plan_terms(int32_t m, int32_t K, const int32_t* tuple_len, const int32_t* tuple_idx,
                         int64_t n, int32_t world_size, int32_t max_terms, int32_t* count,
                         int32_t* owner_out, double* cost_out);

/* Plan inspection (host only): the optimized device program for the
 * sparsified lattice of a signature at extent n — one line per kernel
 * (GEMM / stream, operands, fused epilogue) into text[0..cap) — and totals[7]
 * = {gemms, gemm_macs, streams, stream_entries, fused_epilogues,
 * symmetric_gemms, peak_entries (inputs + live intermediates over the schedule)}. inputs_symmetric != 0 treats every order-2 factor as the
 * same bitwise-symmetric matrix (the BASELINE configs). */
US_API int us_plan_summary(int32_t m, int32_t K, const int32_t* tuple_len, const int32_t* tuple_idx,
                           int64_t n, const us_config* cfg, int32_t inputs_symmetric, char* text,
                           uint64_t cap, uint64_t* totals);

/* Multi-GPU row sharding: rank 0 creates an NCCL unique id (128 bytes),
 * the caller broadcasts it (e.g. torch.distributed), every rank calls
 * us_nccl_init; then us_u_* with flags bit5 and cfg->rank/world_size. */
US_API int us_nccl_unique_id(void* id_out);
US_API int us_nccl_init(int32_t device, int32_t rank, int32_t world_size, const void* id);

/* Device plumbing. */
US_API int us_device_count(int32_t* count);
US_API int us_device_synchronize(int32_t device);
/* FP64 GEMM C = A B^T (A m x k, B n x k, C m x n; row-major host buffers)
 * on the device: method 0 = DMMA (mma.sync f64, TMA-fed), 1 = Ozaki
 * splitting on the INT8 tcgen05 tensor cores with `slices` balanced 8-bit
 * digits (4..7, slices * k * 128^2 < 2^31; method 0 needs an even k); symmetric != 0 asserts B = A (upper
 * tiles, mirrored). ms_out
 * (optional) receives the device time of the GEMM itself. */
US_API int us_dgemm(int32_t method, int32_t slices, int32_t symmetric, int64_t m, int64_t n, int64_t k,
                    const double* a, const double* b, double* c, double* ms_out);
/* The engine's CUDA stream on `device` (cudaStream_t as void*), so callers can
 * order their own work / record events against it. */
US_API int us_device_stream(int32_t device, void** stream_out);
/* How many evaluations on `device` ran as a replayed CUDA graph so far
 * (us_u_statistic_data on repeated small problems; flags bit8 turns it off). */
US_API int us_graph_replays(int32_t device, uint64_t* count_out);
/* Kernel-class timing (CUDA events on the engine stream): enable != 0 turns it
 * on; ms_out[3] / groups_out[3] receive accumulated milliseconds and launch
 * groups for {GEMM, stream, other}; reset != 0 clears the totals after reading.
 * Synchronizes the engine stream. */
US_API int us_profile(int32_t device, int32_t enable, int32_t reset, double* ms_out,
                      uint64_t* groups_out);

#ifdef __cplusplus
}
#endif

#endif /* USTATS_B200_H */
