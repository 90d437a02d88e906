// Microbenchmark: legacy warp-level integer MMA (mma.sync m16n8k32 u8) on sm_100a.
#include <cstdio>
#include <cstdint>
__global__ void k(int* out, int iters, uint32_t seed) {
    uint32_t a0 = seed ^ threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
    int c[8][4] = {};
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int t = 0; t < 8; t++) {
            asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+r"(c[t][0]), "+r"(c[t][1]), "+r"(c[t][2]), "+r"(c[t][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0 + t), "r"(b1));
        }
    }
    int r = 0;
#pragma unroll
    for (int t = 0; t < 8; t++) r += c[t][0] + c[t][1] + c[t][2] + c[t][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
int main() {
    int* out;
    cudaMalloc(&out, 148 * 64 * 1024 * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 2048;
    for (int wpb : {4, 8, 16}) {
        const int blocks = 148 * 4, tpb = 32 * wpb;
        for (int rep = 0; rep < 3; rep++) {
            cudaEventRecord(e0);
            k<<<blocks, tpb>>>(out, iters, 1234u);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double ops = 2.0 * blocks * wpb * (double)iters * 8 * 16 * 8 * 32;
            if (rep == 2) printf("warps/block %d: %.3f ms  %.1f TOPS (int8 dense)  err=%s\n", wpb, ms, ops / ms / 1e9,
                                 cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
