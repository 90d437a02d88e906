// Store-pattern probe: 4 GiB written as 16-byte stores per lane, varying how one
// warp instruction's 512 bytes are laid out.  nvcc -arch=sm_100a -O3 -o store_bench store_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
// mode 0: 512 B contiguous per instruction, warps stream contiguous 32 KB tiles
// mode 1: 8 rows x 64 B, rows 1 KB apart (tile = 32 rows x 1 KB contiguous 32 KB), 16 instr per 8 KB... 
// mode 2: 4 rows x 128 B, rows 1 KB apart
// mode 3: 8 rows x 64 B, rows 256 KB apart (slot-major staging: row stride = K * 1 KB)
// mode 4: 4 rows x 128 B, rows 256 KB apart
__global__ void __launch_bounds__(512, 2) k(u64* S, int mode, long long tiles) {
    const int lane = threadIdx.x & 31;
    const long long warp = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long tile = warp; tile < tiles; tile += nw) {       // tile = 32 rows x 128 words
        // slot-major address of (row r, col c): mode >= 3: ((nblk * 32 + r) * 256 + k) * 128 + c with tile = nblk * 256 + k
        const long long nblk = tile >> 8, kk = tile & 255;
#pragma unroll 4
        for (int i = 0; i < 64; i++) {                            // 64 instr x 512 B = 32 KB
            long long off;
            if (mode == 0) off = tile * 4096 + i * 64 + lane * 2;
            else if (mode == 1 || mode == 3) {
                const int r = (i & 3) * 8 + (lane >> 2), c = (i >> 2) * 8 + (lane & 3) * 2;
                off = mode == 1 ? tile * 4096 + r * 128 + c : ((nblk * 32 + r) * 256 + kk) * 128 + c;
            } else {
                const int r = (i & 7) * 4 + (lane >> 3), c = (i >> 3) * 16 + (lane & 7) * 2;
                off = mode == 2 ? tile * 4096 + r * 128 + c : ((nblk * 32 + r) * 256 + kk) * 128 + c;
            }
            *reinterpret_cast<ulonglong2*>(S + off) = make_ulonglong2(tile, i);
        }
    }
}
int main() {
    const long long tiles = 131072;                               // x 32 KB = 4 GiB
    u64* S;
    cudaMalloc(&S, tiles * 32768);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int mode = 0; mode < 5; mode++)
        for (int grid : {296, 1184, 8192}) {
            k<<<grid, 512>>>(S, mode, tiles);
            cudaEventRecord(a);
            for (int r = 0; r < 3; r++) k<<<grid, 512>>>(S, mode, tiles);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("mode %d grid %5d: %.3f ms  %.0f GB/s\n", mode, grid, ms / 3, tiles * 32768.0 / (ms / 3) / 1e6);
        }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
