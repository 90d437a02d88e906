// Microbenchmark: NTT butterfly throughput on the integer (IMAD) pipe vs the
// FP64 pipe, and both at once (warp-split).  Register-resident radix-16
// passes, no memory traffic in the loop.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2402_01296_b200/csrc tools/micro/bfly_bench.cu
#include <atomic>
#include <cstdio>
#include "common.cuh"
std::atomic<unsigned long long> bcn::g_launches{0};

static constexpr double MAGIC = 6755399441055744.0;   // 1.5 * 2^52: rint by add/subtract

// a*w mod q (signed, |r| < ~2q) for exact integers |a| < 2^53, 0 <= w < q < 2^50, wq = w/q
__device__ __forceinline__ double fmod_mul(double a, double w, double wq, double q) {
    const double hi = __dmul_rn(a, w);
    const double lo = __fma_rn(a, w, -hi);
    const double qt = __dadd_rn(__fma_rn(a, wq, MAGIC), -MAGIC);
    return __dadd_rn(__fma_rn(-qt, q, hi), lo);
}

// value reduction into (-q/2 - eps, q/2 + eps)
__device__ __forceinline__ double fred(double a, double qinv, double q) {
    const double qt = __dadd_rn(__fma_rn(a, qinv, MAGIC), -MAGIC);
    return __fma_rn(-qt, q, a);
}

template <int MODE>
__global__ void __launch_bounds__(256) k(u64* out, const ulonglong2* tw, int iters) {
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    const int warp = threadIdx.x >> 5;
    const bool use_fp = MODE == 1 || (MODE == 2 && (warp & 1)) || (MODE == 3 && (warp % 3 == 2));
    const u64 q = 0x3ffffffffe40001ull & ((1ull << 50) - 1);   // any odd < 2^50 (throughput only)
    if (!use_fp) {
        u64 x[16];
#pragma unroll
        for (int i = 0; i < 16; i++) x[i] = (tid * 7919ull + i * 104729ull) % q;
        const u64 q2 = 2 * q;
        for (int it = 0; it < iters; it++) {
#pragma unroll
            for (int ls = 0; ls < 4; ls++) {
                const int h = 8 >> ls;
#pragma unroll
                for (int kk = 0; kk < 16; kk++) {
                    if (kk & h) continue;
                    const ulonglong2 w = tw[((it & 7) << 4) + (1 << ls) + (kk >> (4 - ls))];
                    u64 u = x[kk];
                    if ((ls & 1) == 0) u = csub(u, 4 * q);
                    const u64 v = shoup_lazy(x[kk + h], w.x, w.y, q);
                    x[kk] = u + v;
                    x[kk + h] = u - v + q2;
                }
            }
        }
        u64 r = 0;
#pragma unroll
        for (int i = 0; i < 16; i++) r ^= x[i];
        out[tid] = r;
    } else {
        double x[16];
        const double qd = (double)q, qinv = 1.0 / qd;
#pragma unroll
        for (int i = 0; i < 16; i++) x[i] = (double)((tid * 7919ull + i * 104729ull) % q);
        const double2* twd = reinterpret_cast<const double2*>(tw);
        for (int it = 0; it < iters; it++) {
#pragma unroll
            for (int ls = 0; ls < 4; ls++) {
                const int h = 8 >> ls;
#pragma unroll
                for (int kk = 0; kk < 16; kk++) {
                    if (kk & h) continue;
                    const double2 w = twd[((it & 7) << 4) + (1 << ls) + (kk >> (4 - ls))];
                    const double u = x[kk];
                    const double v = fmod_mul(x[kk + h], w.x, w.y, qd);
                    x[kk] = __dadd_rn(u, v);
                    x[kk + h] = __dadd_rn(u, -v);
                }
            }
#pragma unroll
            for (int i = 0; i < 16; i++) x[i] = fred(x[i], qinv, qd);   // one reduction per 4 stages
        }
        u64 r = 0;
#pragma unroll
        for (int i = 0; i < 16; i++) r ^= (u64)(long long)x[i];
        out[tid] = r;
    }
}

int main() {
    u64* out;
    ulonglong2* tw;
    cudaMalloc(&out, 148ull * 16 * 256 * 8);
    cudaMalloc(&tw, 256 * 16);
    cudaMemset(tw, 0x11, 256 * 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 2048, tpb = 256;
    const char* names[] = {"int (IMAD)", "fp64 (DFMA)", "split 1:1", "split 2:1 int:fp"};
    for (int blocks_per_sm : {4, 8}) {
        const int blocks = 148 * blocks_per_sm;
        for (int mode = 0; mode < 4; mode++) {
            float ms = 0;
            for (int rep = 0; rep < 3; rep++) {
                cudaEventRecord(e0);
                if (mode == 0) k<0><<<blocks, tpb>>>(out, tw, iters);
                else if (mode == 1) k<1><<<blocks, tpb>>>(out, tw, iters);
                else if (mode == 2) k<2><<<blocks, tpb>>>(out, tw, iters);
                else k<3><<<blocks, tpb>>>(out, tw, iters);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
            }
            const double bf = (double)blocks * tpb * iters * 32;   // 4 stages x 8 butterflies
            printf("%d CTA/SM  %-18s %.3f ms  %.1f G bfly/s  %.2f bfly/clk/SM\n", blocks_per_sm, names[mode], ms,
                   bf / ms / 1e6, bf / (ms * 1e-3) / 1.965e9 / 148);
        }
    }
    cudaError_t e = cudaGetLastError();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
