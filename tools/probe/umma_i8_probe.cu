// Probe: one 128x64 (M x N) int8 x int8 -> int32 tile over K = 64 with
// tcgen05.mma kind::i8, operands in shared memory in the K-major no-swizzle
// core-matrix layout, accumulator in TMEM, read back with tcgen05.ld.
// Usage: umma_i8_probe [lbo sbo]   (bytes)
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

constexpr int M = 128, N = 64, K = 64;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ unsigned long long make_desc(const void* smem, unsigned lbo, unsigned sbo) {
    unsigned long long d = 0;
    d |= (unsigned long long)((smem_u32(smem) >> 4) & 0x3FFF);
    d |= (unsigned long long)((lbo >> 4) & 0x3FFF) << 16;
    d |= (unsigned long long)((sbo >> 4) & 0x3FFF) << 32;
    d |= 1ull << 46;  // version (sm100)
    // base offset 0, lbo mode 0, layout type 0 (no swizzle)
    return d;
}

__global__ void probe(const int8_t* a, const int8_t* b, int* out, unsigned lbo, unsigned sbo, unsigned idesc) {
    __shared__ __align__(1024) int8_t sa[M * K];
    __shared__ __align__(1024) int8_t sb[N * K];
    __shared__ unsigned tmem_base;
    __shared__ __align__(8) unsigned long long bar;
    const int tid = threadIdx.x;
    // K-major no-swizzle core-matrix layout: chunk c = k/16 (16 bytes); within a
    // chunk, rows are contiguous at 16-byte pitch: byte (c * rows + r) * 16 + k%16
    for (int i = tid; i < M * K; i += blockDim.x) {
        const int r = i / K, k = i % K;
        sa[((k / 16) * M + r) * 16 + k % 16] = a[i];
    }
    for (int i = tid; i < N * K; i += blockDim.x) {
        const int r = i / K, k = i % K;
        sb[((k / 16) * N + r) * 16 + k % 16] = b[i];
    }
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");  // generic smem writes -> async proxy (UMMA)
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const unsigned tmem = tmem_base;
    if (tid == 0) {
        for (int ks = 0; ks < K / 32; ++ks) {
            // K = 32 bytes per instruction = 2 core-matrix chunks of 16 bytes
            const unsigned long long da = make_desc(sa + ks * 2 * M * 16, lbo, sbo);
            const unsigned long long db = make_desc(sb + ks * 2 * N * 16, lbo == 0 ? 0 : lbo * N / M, sbo);
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                "l"(da), "l"(db), "r"(idesc), "r"(ks));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    }
    // wait for the MMAs
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(smem_u32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    // warp w reads TMEM lanes 32w..32w+31; thread = one row, 16 columns at a time
    const int warp = tid / 32, lane = tid % 32;
    for (int c0 = 0; c0 < N; c0 += 16) {
        unsigned v[16];
        const unsigned addr = tmem + ((unsigned)(warp * 32) << 16) + c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(addr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int j = 0; j < 16; ++j) out[(warp * 32 + lane) * N + c0 + j] = (int)v[j];
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

int main(int argc, char** argv) {
    unsigned lbo = argc > 1 ? atoi(argv[1]) : M * 16;
    unsigned sbo = argc > 2 ? atoi(argv[2]) : 128;
    // instruction descriptor: c_format S32 (2) bits 4-5, a/b signed (1) bits 7-9 / 10-12,
    // K-major both, n_dim = N>>3 bits 17-22, m_dim = M>>4 bits 24-28
    unsigned idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((unsigned)(N >> 3) << 17) | ((unsigned)(M >> 4) << 24);
    std::vector<int8_t> a(M * K), b(N * K);
    srand(1);
    for (auto& x : a) x = (int8_t)(rand() % 255 - 127);
    for (auto& x : b) x = (int8_t)(rand() % 255 - 127);
    std::vector<int> ref(M * N, 0), got(M * N, 0);
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < N; ++j) {
            int s = 0;
            for (int k = 0; k < K; ++k) s += a[i * K + k] * b[j * K + k];
            ref[i * N + j] = s;
        }
    int8_t *da, *db;
    int* dout;
    cudaMalloc(&da, a.size());
    cudaMalloc(&db, b.size());
    cudaMalloc(&dout, got.size() * 4);
    cudaMemcpy(da, a.data(), a.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(db, b.data(), b.size(), cudaMemcpyHostToDevice);
    cudaMemset(dout, 0, got.size() * 4);
    probe<<<1, 128>>>(da, db, dout, lbo, sbo, idesc);
    cudaError_t e = cudaDeviceSynchronize();
    printf("lbo %u sbo %u: %s\n", lbo, sbo, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    cudaMemcpy(got.data(), dout, got.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < M * N; ++i) bad += got[i] != ref[i];
    printf("mismatches %d / %d; got[0]=%d ref[0]=%d got[1]=%d ref[1]=%d got[N]=%d ref[N]=%d\n", bad, M * N, got[0], ref[0],
           got[1], ref[1], got[N], ref[N]);
    return bad != 0;
}
