// Microbenchmark: sustained FP64 tensor-core (DMMA) throughput on sm_100a via mma.sync.
#include <cstdio>
#include <cuda_runtime.h>

template <int ACC>
__global__ void dmma_loop(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
    double c[ACC][2];
#pragma unroll
    for (int i = 0; i < ACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ACC; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.0) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
    double c[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) c[i] = fma(a, b, c[i]);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += c[i];
    if (s == 12345.0) out[0] = s;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out; cudaMalloc(&out, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 20000;
    for (int warps = 4; warps <= 16; warps *= 2) {
        for (int bps = 1; bps <= 2; ++bps) {
            int blocks = sms * bps;
            dmma_loop<8><<<blocks, warps * 32>>>(out, 100);
            cudaEventRecord(e0);
            dmma_loop<8><<<blocks, warps * 32>>>(out, iters);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double flops = 2.0 * 256.0 * 8 * iters * (double)blocks * warps;
            printf("DMMA m8n8k4 warps/blk=%d blk/SM=%d: %.2f TFLOP/s\n", warps, bps, flops / ms / 1e9);
        }
    }
    {
        int blocks = sms * 4;
        dfma_loop<<<blocks, 256>>>(out, 100);
        cudaEventRecord(e0);
        dfma_loop<<<blocks, 256>>>(out, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 16 * iters * (double)blocks * 256;
        printf("DFMA: %.2f TFLOP/s\n", flops / ms / 1e9);
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
