// Microbenchmark: u128 multiply-accumulate flavours (Acc128.mac_nr vs Acc4).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2402_01296_b200/csrc tools/micro/mac_bench.cu
#include <cstdio>
#include "common.cuh"
std::atomic<unsigned long long> bcn::g_launches{0};

template <int MODE>
__global__ void k(u64* out, const u64* in, int iters) {
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    u64 a = in[tid & 1023], b[8];
#pragma unroll
    for (int o = 0; o < 8; o++) b[o] = in[(tid + 37 * o + 1) & 1023];
    Acc128 x[8];
    Acc4 y[8];
#pragma unroll
    for (int o = 0; o < 8; o++) { x[o].zero(); y[o].zero(); }
    const u64 q = 0x1fffffffffe00001ull;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int o = 0; o < 8; o++) {
            if (MODE == 0) x[o].mac_nr(a, b[o]);
            else y[o].mac((u32)a, (u32)(a >> 32), (u32)b[o], (u32)(b[o] >> 32));
        }
        a = a * 3 + 1;   // keep the operand changing
        a &= 0x0fffffffffffffffull;
        if ((i & 7) == 7) {
#pragma unroll
            for (int o = 0; o < 8; o++) { if (MODE == 0) x[o].fold(q); else y[o].fold_hi(q, 8); }
        }
    }
    u64 r = 0;
#pragma unroll
    for (int o = 0; o < 8; o++) r ^= MODE == 0 ? x[o].hi ^ x[o].lo : y[o].hi ^ y[o].lo;
    out[tid] = r;
}

int main() {
    u64 *in, *out;
    cudaMalloc(&in, 1024 * 8);
    cudaMalloc(&out, 148 * 4 * 1024 * 8 * 8);
    cudaMemset(in, 0x11, 1024 * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096, blocks = 148 * 8, tpb = 256;
    for (int mode = 0; mode < 2; mode++) {
        for (int rep = 0; rep < 3; rep++) {
            cudaEventRecord(e0);
            if (mode == 0) k<0><<<blocks, tpb>>>(out, in, iters);
            else k<1><<<blocks, tpb>>>(out, in, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double macs = (double)blocks * tpb * iters * 8;
            if (rep == 2) printf("mode %d (%s): %.3f ms, %.1f G MAC/s, %.1f SMSP-cycles per warp-MAC\n", mode,
                                 mode ? "Acc4" : "Acc128.mac_nr", ms, macs / ms / 1e6,
                                 (ms * 1e-3 * 1.965e9 * 592) / (macs / 32));
        }
    }
    return 0;
}
