// umma_bench.cu -- tcgen05.mma kind::i8 issue-rate probe for the conv MAC
// layouts (mac_umma.cu): operands resident in shared memory, one CTA per SM,
// one thread issuing R rounds of 16 MMAs (M = 128, N = 256 or 128, K = 32),
// commit + wait per round.  Reports cycles per MMA against the 128 x N / 256
// floor.  Modes:
//   0  no-swizzle, B windows shifted by 7 - j rows (the production pattern)
//   1  no-swizzle, B windows aligned (start on an 8-row core-matrix boundary)
//   2  like 0 with N = 128
//   3  SWIZZLE_128B, 128-byte rows (K = 128 per row, 4 k-steps of 32 bytes)
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 umma_bench.cu -o umma_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

typedef unsigned long long u64;
typedef unsigned int u32;

__device__ __forceinline__ u32 saddr(const void* p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ u64 sdesc(u32 a, u32 lbo, u32 sbo, u32 layout) {
    return (u64)((a >> 4) & 0x3fffu) | ((u64)((lbo >> 4) & 0x3fffu) << 16) | ((u64)((sbo >> 4) & 0x3fffu) << 32) |
           (1ull << 46) | ((u64)layout << 61);
}
__device__ __forceinline__ void mma(u32 d, u64 a, u64 b, u32 idesc, u32 acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc)
                 : "memory");
}

__global__ void __launch_bounds__(128, 1) bench(int mode, int rounds, u64* cycles) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ u64 bar;
    __shared__ u32 tslot;
    for (int i = threadIdx.x; i < 200 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(i, 3 * i, 0, 7);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(saddr(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const u32 tmem = tslot;
    const int N = mode == 2 ? 128 : 256;
    const u32 idesc = (2u << 4) | ((u32)(N >> 3) << 17) | ((128u >> 4) << 24);
    if (threadIdx.x == 0) {
        const u32 A = saddr(sm), B = A + 32768;
        long long t0 = clock64();
        u32 phase = 0;
        for (int r = 0; r < rounds; r++) {
            for (int nb = 0; nb < 2; nb++)
                for (int j = 0; j < 8; j++) {
                    u64 ad, bd;
                    if (mode == 3) {        // 128-byte swizzled rows: k-step j%4 at +32 j bytes
                        ad = sdesc(A + (j & 3) * 32, 16, 1024, 2);
                        bd = sdesc(B + (j & 3) * 32 + nb * 32768, 16, 1024, 2);
                    } else {
                        ad = sdesc(A + j * 4096, 2048, 128, 0);
                        const int shift = mode == 1 ? 0 : 7 - j;
                        bd = sdesc(B + (nb * 256 + shift) * 16, 8320, 128, 0);
                    }
                    mma(tmem + nb * 256, ad, bd, idesc, (r | j) ? 1u : 0u);
                }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(&bar)));
            u32 done = 0;
            while (!done)
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                             : "=r"(done) : "r"(saddr(&bar)), "r"(phase));
            phase ^= 1;
        }
        cycles[blockIdx.x] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
    u64* d;
    cudaMalloc(&d, 148 * sizeof(u64));
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const int rounds = 2000;
    for (int mode = 0; mode < 4; mode++) {
        bench<<<148, 128, 200 * 1024>>>(mode, 10, d);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        bench<<<148, 128, 200 * 1024>>>(mode, rounds, d);
        cudaEventRecord(b);
        cudaError_t e = cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        u64 h[148];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        const int N = mode == 2 ? 128 : 256;
        const double per = (double)h[0] / (rounds * 16.0);
        const double tops = 148.0 * rounds * 16 * 128.0 * N * 32 * 2 / (ms * 1e-3) / 1e12;
        printf("mode %d (%s): %.1f cycles/MMA (floor %d), %.0f int8 TOP/s, %.3f ms\n", mode, cudaGetErrorString(e), per,
               128 * N / 256, tops, ms);
    }
    return 0;
}
