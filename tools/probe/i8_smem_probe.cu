// Does a concurrent bulk-copy stream into shared memory slow tcgen05 INT8 MMAs,
// and does N = 256 suffer less than N = 128? One CTA per SM: lane 0 of warp 0
// issues `iters` MMAs (M=128, K=32) on resident operands; with COPY, lane 0 of
// warp 1 keeps a 4 x 16 KiB ring of cp.async.bulk global->shared copies
// (L2-resident source) running until the MMAs finish.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ unsigned long long desc(unsigned a, unsigned lbo, unsigned sbo) {
    return (unsigned long long)((a >> 4) & 0x3FFF) | ((unsigned long long)((lbo >> 4) & 0x3FFF) << 16) |
           ((unsigned long long)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
__device__ __forceinline__ bool try_wait(unsigned long long* b, unsigned parity) {
    unsigned ok;
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(su32(b)), "r"(parity) : "memory");
    return ok;
}

template <int N, bool COPY>
__global__ void probe(int iters, const int8_t* src, unsigned long long* copied, int* sink) {
    extern __shared__ __align__(1024) unsigned char sm[];
    int8_t* a = reinterpret_cast<int8_t*>(sm);              // 128 x 32
    int8_t* b = a + 128 * 32;                                // N x 32
    unsigned char* ring = sm + 128 * 32 + N * 32;            // 4 x 16 KiB
    __shared__ unsigned tmem;
    __shared__ __align__(8) unsigned long long bar, cbar[4];
    __shared__ volatile int done;
    for (int i = threadIdx.x; i < 128 * 32; i += blockDim.x) a[i] = (int8_t)((i * 37) & 0xFF);
    for (int i = threadIdx.x; i < N * 32; i += blockDim.x) b[i] = (int8_t)((i * 91) & 0xFF);
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tmem)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        done = 0;
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        for (int q = 0; q < 4; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&cbar[q])));
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
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(acc),
                         "l"(da), "l"(db), "r"(idesc), "r"(i > 1 ? 1 : 0));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
        while (!try_wait(&bar, 0)) {}
        done = 1;
    } else if (COPY && threadIdx.x == 32) {
        unsigned long long n = 0;
        const int8_t* s = src + (blockIdx.x % 16) * (256 << 10);
        long long it = 0;
        for (;; ++it) {
            const int q = (int)(it & 3);
            if (it >= 4) while (!try_wait(&cbar[q], (unsigned)(((it >> 2) - 1) & 1))) {}
            if (done) break;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&cbar[q])), "r"(16384u) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             su32(ring + q * 16384)),
                         "l"(reinterpret_cast<unsigned long long>(s + (it % 16) * 16384)), "r"(16384u), "r"(su32(&cbar[q]))
                         : "memory");
            n += 16384;
        }
        // drain the copies still in flight (issued at it-3 .. it-1)
        for (long long j = it - 3; j < it; ++j)
            if (j >= 0) while (!try_wait(&cbar[j & 3], (unsigned)((j >> 2) & 1))) {}
        atomicAdd(copied, n);
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    unsigned v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem + ((threadIdx.x / 32 * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    if (threadIdx.x == 0) sink[blockIdx.x] = (int)v;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N, bool COPY>
void run(int iters, const int8_t* src, unsigned long long* copied, int* sink) {
    const int smem = 128 * 32 + N * 32 + 4 * 16384;
    cudaFuncSetAttribute(probe<N, COPY>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    probe<N, COPY><<<148, 128, smem>>>(1000, src, copied, sink);
    cudaDeviceSynchronize();
    cudaMemset(copied, 0, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<N, COPY><<<148, 128, smem>>>(iters, src, copied, sink);
    cudaEventRecord(e1);
    cudaError_t e = cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long c = 0;
    cudaMemcpy(&c, copied, 8, cudaMemcpyDeviceToHost);
    const double ops = 2.0 * 128 * N * 32 * (double)iters * 148;
    const double cyc = ms * 1e-3 * 1.965e9;
    printf("N=%d copy=%d: %.3f ms, %.1f TOPS, copy %.2f TB/s (%.1f B/clk/SM), MMA smem reads %.1f B/clk/SM (%s)\n", N,
           (int)COPY, ms, ops / ms / 1e9, c / (ms * 1e-3) / 1e12, c / 148.0 / cyc,
           (128.0 * 32 + N * 32) * iters / cyc, cudaGetErrorString(e));
}

int main() {
    int8_t* src;
    unsigned long long* copied;
    int* sink;
    cudaMalloc(&src, 16 << 20);
    cudaMemset(src, 1, 16 << 20);
    cudaMalloc(&copied, 8);
    cudaMalloc(&sink, 148 * sizeof(int));
    for (int rep = 0; rep < 2; ++rep) {
        run<128, false>(200000, src, copied, sink);
        run<128, true>(200000, src, copied, sink);
        run<256, false>(100000, src, copied, sink);
        run<256, true>(100000, src, copied, sink);
    }
    return 0;
}
