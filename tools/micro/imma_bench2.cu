// IMMA throughput with the conv-MAC access pattern: 15 diagonal accumulators,
// 8 A planes x 8 B planes per k-step (acc[i+j] += A_i B_j), 16 warps/CTA.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ void imma(int* d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
template <int MODE>
__global__ void __launch_bounds__(512, 1) k(int* out, int iters, uint32_t seed) {
    extern __shared__ uint4 sm[];
    const int tid = threadIdx.x;
    for (int i = tid; i < 1024; i += blockDim.x) sm[i] = make_uint4(seed ^ i, i * 3, i * 5, i * 7);
    __syncthreads();
    int acc[15][4] = {};
    uint32_t b0[8], b1[8];
#pragma unroll
    for (int j = 0; j < 8; j++) { b0[j] = seed * (j + 1) ^ tid; b1[j] = b0[j] * 3; }
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 8; i++) {
            uint4 a = MODE ? sm[(tid + i * 32 + it) & 1023] : make_uint4(seed + i, seed * 3, seed * 5, seed * 7);
#pragma unroll
            for (int j = 0; j < 8; j++) imma(acc[i + j], a.x, a.y, a.z, a.w, b0[j], b1[j]);
        }
    }
    int r = 0;
#pragma unroll
    for (int s = 0; s < 15; s++) r += acc[s][0] ^ acc[s][1] ^ acc[s][2] ^ acc[s][3];
    out[blockIdx.x * blockDim.x + tid] = r;
}
int main() {
    int* out; cudaMalloc(&out, 148 * 4 * 512 * 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 256;
    cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
    cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
    for (int mode = 0; mode < 2; mode++) for (int cfg = 0; cfg < 4; cfg++) {
        const int wpb = cfg < 2 ? 8 : 16;
        const int blocks = 148 * (cfg == 0 ? 2 : cfg == 1 ? 4 : cfg == 2 ? 1 : 2), tpb = 32 * wpb;
        for (int rep = 0; rep < 3; rep++) {
            cudaEventRecord(e0);
            if (mode) k<1><<<blocks, tpb, 16384>>>(out, iters, 77u); else k<0><<<blocks, tpb, 16384>>>(out, iters, 77u);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double ops = 2.0 * blocks * wpb * (double)iters * 64 * 16 * 8 * 32;
            if (rep == 2) printf("mode %d (A %s) warps/block %d blocks/SM %d: %.1f TOPS\n", mode, mode ? "LDS.128" : "const", wpb, blocks / 148, ops / ms / 1e9);
        }
    }
    return 0;
}
