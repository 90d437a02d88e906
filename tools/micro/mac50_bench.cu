// Microbenchmark: exact multiply-accumulate of 50-bit residues.
//   mode 0: Acc4 (32-bit halves, 4-word carry chain: 2 IMAD.WIDE + 4 IMAD + 3 IADD)
//   mode 1: 25-bit halves, three 64-bit accumulators (4 IMAD.WIDE, no carries)
// Both feed two accumulators from one shared operand u (the key-switch pattern
// u * k0, u * k1).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2402_01296_b200/csrc tools/micro/mac50_bench.cu
#include <atomic>
#include <cstdio>
#include "common.cuh"
std::atomic<unsigned long long> bcn::g_launches{0};

struct Acc50 {
    u64 L, M, H;
    __device__ __forceinline__ void zero() { L = M = H = 0ull; }
    __device__ __forceinline__ void mac(u32 a0, u32 a1, u32 b0, u32 b1) {
        asm("mad.wide.u32 %0, %3, %5, %0;\n\t"
            "mad.wide.u32 %1, %3, %6, %1;\n\t"
            "mad.wide.u32 %1, %4, %5, %1;\n\t"
            "mad.wide.u32 %2, %4, %6, %2;"
            : "+l"(L), "+l"(M), "+l"(H)
            : "r"(a0), "r"(a1), "r"(b0), "r"(b1));
    }
};
__device__ __forceinline__ void split25(u64 a, u32& a0, u32& a1) {
    a0 = (u32)a & 0x1ffffffu;
    a1 = (u32)(a >> 25);
}

template <int MODE>
__global__ void k(u64* out, const u64* in, int iters) {
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    u64 kk0[4], kk1[4];
#pragma unroll
    for (int o = 0; o < 4; o++) { kk0[o] = in[(tid + 37 * o + 1) & 1023]; kk1[o] = in[(tid + 91 * o + 5) & 1023]; }
    u64 u = in[tid & 1023];
    Acc4 x0, x1;
    Acc50 y0, y1;
    x0.zero(); x1.zero(); y0.zero(); y1.zero();
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int o = 0; o < 4; o++) {
            const u64 uu = u + o;
            if (MODE == 0) {
                x0.mac(uu, kk0[o]);
                x1.mac(uu, kk1[o]);
            } else {
                u32 u0, u1, a0, a1, b0, b1;
                split25(uu, u0, u1);
                split25(kk0[o], a0, a1);
                split25(kk1[o], b0, b1);
                y0.mac(u0, u1, a0, a1);
                y1.mac(u0, u1, b0, b1);
            }
        }
        u = (u * 3 + 1) & ((1ull << 50) - 1);
#pragma unroll
        for (int o = 0; o < 4; o++) { kk0[o] ^= u; kk1[o] += u; kk0[o] &= (1ull << 50) - 1; kk1[o] &= (1ull << 50) - 1; }
    }
    out[tid] = MODE == 0 ? x0.hi ^ x0.lo ^ x1.hi ^ x1.lo : y0.L ^ y0.M ^ y0.H ^ y1.L ^ y1.M ^ y1.H;
}

int main() {
    u64 *in, *out;
    cudaMalloc(&in, 1024 * 8);
    cudaMalloc(&out, 148 * 8 * 256 * 8);
    cudaMemset(in, 0x11, 1024 * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096, blocks = 148 * 8, tpb = 256;
    for (int mode = 0; mode < 2; mode++) {
        float ms = 0;
        for (int rep = 0; rep < 3; rep++) {
            cudaEventRecord(e0);
            if (mode == 0) k<0><<<blocks, tpb>>>(out, in, iters);
            else k<1><<<blocks, tpb>>>(out, in, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
        }
        const double macs = (double)blocks * tpb * iters * 8;   // 4 (u, k0, k1) triples = 8 products
        printf("mode %d (%s): %.3f ms, %.1f G MAC/s, %.2f MAC/clk/SM\n", mode, mode ? "25-bit halves" : "Acc4", ms,
               macs / ms / 1e6, macs / (ms * 1e-3) / 1.965e9 / 148);
    }
    return 0;
}
