// INT8 tcgen05 issue-rate probe: one CTA per SM, one thread issuing
// tcgen05.mma.cta_group::1.kind::i8 (M=128, N=256, K=32) back to back on
// resident shared-memory operands, int32 accumulators in TMEM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ unsigned long long desc(unsigned a, unsigned lbo, unsigned sbo) {
    return (unsigned long long)((a >> 4) & 0x3FFF) | ((unsigned long long)((lbo >> 4) & 0x3FFF) << 16) |
           ((unsigned long long)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

// RANDOM: eight distinct A and B operand tiles of uniformly random int8 digits
// (the data a real digit GEMM feeds the tensor cores), rotated MMA to MMA, so
// the operand buses and multipliers toggle as they do under load; otherwise
// one resident tile of small constants (pure issue rate, little switching).
template <int N, bool RANDOM = false>
__global__ void peak(int iters, int* sink) {
    constexpr int T = RANDOM ? 8 : 1;
    extern __shared__ __align__(1024) int8_t smem[];
    int8_t* a = smem;
    int8_t* b = smem + T * 128 * 32;
    __shared__ unsigned tmem;
    __shared__ __align__(8) unsigned long long bar;
    if (RANDOM) {
        for (int i = threadIdx.x; i < T * (128 + N) * 32; i += blockDim.x) {
            unsigned h = (unsigned)i * 2654435761u + blockIdx.x * 40503u;
            h ^= h >> 15; h *= 2246822519u; h ^= h >> 13;
            smem[i] = (int8_t)(h & 0xFF);
        }
    } else {
        for (int i = threadIdx.x; i < 128 * 32; i += blockDim.x) a[i] = (int8_t)(i & 7);
        for (int i = threadIdx.x; i < N * 32; i += blockDim.x) b[i] = (int8_t)(i & 3);
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const unsigned idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((128 >> 4) << 24);
    if (threadIdx.x == 0) {
        const unsigned long long da = desc(su32(a), 128 * 16, 128), db = desc(su32(b), N * 16, 128);
        for (int i = 0; i < iters; ++i) {
            const unsigned acc = tmem + (unsigned)((i & 1) * N);
            // descriptor start addresses are in 16-byte units: step to the next tile
            const unsigned long long ta = da + (unsigned long long)((i % T) * (128 * 32 / 16));
            const unsigned long long tb = db + (unsigned long long)(((i / 3) % T) * (N * 32 / 16));
            // random data: restart the accumulation every 512 MMAs (int32 stays exact)
            const int accumulate = RANDOM ? ((i & 511) > 1 ? 1 : 0) : (i > 1 ? 1 : 0);
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(acc),
                         "l"(ta), "l"(tb), "r"(idesc), "r"(accumulate));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    }
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    unsigned v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem + ((threadIdx.x / 32 * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    if (threadIdx.x == 0) sink[blockIdx.x] = (int)v;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N, bool RANDOM = false>
void run(int blocks, int iters) {
    int* sink;
    cudaMalloc(&sink, blocks * sizeof(int));
    const int bytes = (RANDOM ? 8 : 1) * (128 + N) * 32;
    cudaFuncSetAttribute(peak<N, RANDOM>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    peak<N, RANDOM><<<blocks, 128, bytes>>>(100, sink);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    peak<N, RANDOM><<<blocks, 128, bytes>>>(iters, sink);
    cudaEventRecord(e1);
    cudaError_t e = cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = 2.0 * 128 * N * 32 * (double)iters * blocks;
    printf("N=%d%s blocks=%d iters=%d: %.3f ms, %.1f TOPS (%s)\n", N, RANDOM ? " random-digits" : "", blocks, iters, ms, ops / ms / 1e9, cudaGetErrorString(e));
    cudaFree(sink);
}

// i8_peak            -> burst: one launch per shape
// i8_peak sustained  -> N=256 launched back to back for ~4 s (clocks settle
//                       under the power cap; nvidia-smi samples them)
// i8_peak random     -> the same with random int8 operands rotated MMA to MMA
int main(int argc, char** argv) {
    if (argc > 1 && argv[1][0] == 'r') {  // random digits, back to back for ~4 s
        for (int r = 0; r < 300; ++r) run<256, true>(148, 200000);
        return 0;
    }
    if (argc > 1) {
        for (int r = 0; r < 300; ++r) run<256>(148, 200000);
        return 0;
    }
    run<256>(148, 200000);
    run<128>(148, 200000);
    run<64>(148, 200000);
    return 0;
}
