// mac_umma.cu -- the conv-layer MAC (out_o = sum_k pt_{o,k} (x) B'_k, the
// lazy-ModDown terms staged slot-major by slot_major_ks_kernel) on the
// 5th-generation tensor cores: tcgen05.mma kind::i8 with the accumulators in
// TMEM.  Same arithmetic as mac_imma.cu (byte planes, fifteen exact int32
// partials D_s = sum_{i+j=s} P_i C_j, one REDC), different mapping:
//
//   D[col][(o, s)] += sum_k  C_j[col][k] * W_j[(o, s)][k]        j = 0..7
//
// * M = 128 ciphertext columns (64 slot sets x 2 components) of one slot;
//   A = byte plane j of their words, built in shared memory by the producer
//   warps (one PRMT byte-transpose per 4 words).
// * N = 16 outputs x 16 rows s; B = a shifted window over the plaintext
//   planes: output o owns 16 rows of 32 term-bytes, plane i at row 7 + i and
//   zeros elsewhere, so the window that starts 7 - j rows into the strip has
//   plane s - j at row s (zero when s - j is outside 0..7, including the
//   reads that run into the next strip's leading zero rows).  The MMA then
//   lands D_s of output o directly in TMEM column 16 o + s: every partial of
//   one output word sits in ONE thread's lane, so the epilogue is per-thread
//   (tcgen05.ld, recombine, REDC, store) with no shuffles.
// * Half of the N rows are zero (8 of every 16 per j), the price of that
//   epilogue; at 128 x 256 x 32 per instruction the tensor core still does
//   about 4x the useful byte products of mma.sync IMMA per SM cycle.
//
// Warp roles (persistent, one CTA per SM):
//   warp 4      bulk-copy issuer (one lane): the chunk's 32 x 128 staged words
//               (one contiguous 32 KB run of S) and its plane strips, by
//               cp.async.bulk into a 2-deep raw ring (mbarrier complete_tx)
//   warps 0-3   transposers, one thread per column: raw words -> byte planes
//               (A) and plane rows -> strips (B) in a 3-deep stage ring,
//               fence.proxy.async, arrive on full[stage]
//   warp 5      MMA issuer (one lane) + TMEM allocation (512 columns = two
//               256-column accumulators, one per 16-output block)
//   warps 6-13  epilogue: warp w reads TMEM lanes 32 (w % 4).. (its 32
//               columns), outputs 8 ((w - 6) / 4) .. + 7 of the block
// Work item = (slot, block of 32 outputs).  The accumulator of output block
// half nb is released as soon as its epilogue has read it, so the next item's
// MMAs into it overlap the drain of the other half.
#include <cstdio>
#include <cstdlib>
#include "common.cuh"
#include "ops.cuh"

namespace bcn {

typedef unsigned char u8;

#ifndef UM_ST
#define UM_ST 3                                   // plane stages (transposers -> MMA)
#endif
#ifndef UM_RS
#define UM_RS 2                                   // raw stages (bulk copy -> transposers)
#endif
#ifndef UM_PAIR_MAXO
#define UM_PAIR_MAXO 32                           // widest output count stored as slot pairs
#endif
#ifndef UM_TR
#define UM_TR 4                                   // transposer warps: one thread per column (8: per column and k-half, no gain; 4 leaves the epilogue registers for slot pairs)
#endif
#define UM_W_COPY UM_TR                           // bulk-copy issuer warp
#define UM_W_MMA (UM_TR + 1)                      // MMA issuer warp (also owns TMEM)
#define UM_W_EPI (UM_TR + 2)                      // first of the epilogue warps
#define UM_EPI 8                                  // epilogue warps (2 per TMEM lane quarter)
#define UM_THREADS ((UM_W_EPI + UM_EPI) * 32)     // 14 warps: <= 4 per sub-core, 128 registers
constexpr int UM_COLS = 128;                      // M: ciphertext columns per item
constexpr int UM_APLANE = UM_COLS * 32;           // bytes of one A plane (128 rows x 32 k)
constexpr int UM_ABYTES = 8 * UM_APLANE;
constexpr int UM_BROWS = 32 * 16 + 8;             // 32 output strips + the tail window overrun
constexpr int UM_BHALF = UM_BROWS * 16;           // one 16-byte k-half of all rows
constexpr int UM_SBYTES = UM_ABYTES + 2 * UM_BHALF;
constexpr int UM_RBYTES = UM_COLS * 32 * 8 + 32 * 256;   // raw chunk: 32 x 128 words + 32 outputs' planes
constexpr size_t UM_SMEM = (size_t)UM_ST * UM_SBYTES + (size_t)UM_RS * UM_RBYTES + 128;

// ---------------------------------------------------------------- packing
// planes[((b * nch + c) * opad + o) * 256 + kh * 128 + i * 16 + kb]
//   = byte i of pt[o][32 c + 16 kh + kb] at slot b (0 past n_terms / short plaintexts):
// the 128 bytes of one (output, k-half) are exactly its strip rows 7..14.
__global__ void pack_planes_umma_kernel(u8* __restrict__ planes, const u64* const* __restrict__ pts, int n_out,
                                        int n_terms, int opad, int nch, int logn, const int* __restrict__ tlimbs) {
    const int N = 1 << logn;
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    const int t = blockIdx.y;
    const int o = blockIdx.z / nch, c = blockIdx.z % nch;
    const long long b = (long long)t * N + n;
    u32 w[2][8][4];                                       // [kh][plane][4-byte group]
#pragma unroll
    for (int h = 0; h < 2; h++)
#pragma unroll
        for (int i = 0; i < 8; i++)
#pragma unroll
            for (int d = 0; d < 4; d++) w[h][i][d] = 0u;
#pragma unroll
    for (int kk = 0; kk < 32; kk++) {
        const int k = c * 32 + kk;
        const bool live = o < n_out && k < n_terms && (!tlimbs || t < tlimbs[k]);
        const u64 v = live ? __ldg(pts[(size_t)o * n_terms + k] + b) : 0ull;
        const int h = kk >> 4, d = (kk & 15) >> 2, sh = (kk & 3) * 8;
#pragma unroll
        for (int i = 0; i < 8; i++) w[h][i][d] |= (u32)((v >> (8 * i)) & 0xffull) << sh;
    }
    uint4* dst = reinterpret_cast<uint4*>(planes + ((b * nch + c) * opad + o) * 256);
#pragma unroll
    for (int h = 0; h < 2; h++)
#pragma unroll
        for (int i = 0; i < 8; i++) dst[h * 8 + i] = make_uint4(w[h][i][0], w[h][i][1], w[h][i][2], w[h][i][3]);
}

cudaError_t pack_planes_umma_op(u8* planes, const u64* const* pts_dev, int n_out, int n_terms, int opad, int nch,
                                int nl, int logn, cudaStream_t st, const int* tlimbs_dev) {
    const int N = 1 << logn;
    const int tpb = N < 128 ? N : 128;
    dim3 grid((N + tpb - 1) / tpb, nl, opad * nch);
    pack_planes_umma_kernel<<<grid, tpb, 0, st>>>(planes, pts_dev, n_out, n_terms, opad, nch, logn, tlimbs_dev);
    return launched();
}

// ---------------------------------------------------------------- tcgen05 helpers
// shared-memory matrix descriptor, K-major, no swizzle: rows of 16 bytes
// (8-row core matrices SBO apart), the two 16-byte k-halves LBO apart
__device__ __forceinline__ u64 umma_sdesc(u32 saddr, u32 lbo, u32 sbo) {
    return (u64)((saddr >> 4) & 0x3fffu) | ((u64)((lbo >> 4) & 0x3fffu) << 16) |
           ((u64)((sbo >> 4) & 0x3fffu) << 32) | (1ull << 46);   // version 1 (sm_100), layout SWIZZLE_NONE
}
// instruction descriptor: D s32, A/B u8, both K-major, N = 256, M = 128
constexpr u32 UM_IDESC = (2u << 4) | ((256u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void umma_i8(u32 tmem_d, u64 adesc, u64 bdesc, u32 accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(UM_IDESC), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit(u64* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(u64* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
// bounded wait: a protocol bug traps (launch error) instead of hanging the GPU
__device__ __forceinline__ void um_wait(u64* bar, u32 parity) {
    for (u32 spin = 0;; spin++) {
        u32 done;
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
        if (done) return;
        if (spin > (1u << 24)) __trap();
    }
}
// 16 consecutive TMEM columns of this thread's lane
__device__ __forceinline__ void tmem_ld16(u32 taddr, u32 (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// bytes j of four k-consecutive words -> b[j] = {w0.bj, w1.bj, w2.bj, w3.bj}
__device__ __forceinline__ void bytes_by_plane(const u64 v[4], u32 b[8]) {
#pragma unroll
    for (int h = 0; h < 2; h++) {
        const u32 x0 = (u32)(v[0] >> (32 * h)), x1 = (u32)(v[1] >> (32 * h));
        const u32 x2 = (u32)(v[2] >> (32 * h)), x3 = (u32)(v[3] >> (32 * h));
        const u32 p01l = __byte_perm(x0, x1, 0x5140), p01h = __byte_perm(x0, x1, 0x7362);
        const u32 p23l = __byte_perm(x2, x3, 0x5140), p23h = __byte_perm(x2, x3, 0x7362);
        b[4 * h + 0] = __byte_perm(p01l, p23l, 0x5410);
        b[4 * h + 1] = __byte_perm(p01l, p23l, 0x7632);
        b[4 * h + 2] = __byte_perm(p01h, p23h, 0x5410);
        b[4 * h + 3] = __byte_perm(p01h, p23h, 0x7632);
    }
}

// the prime constants the epilogue needs, held in registers for a whole item
struct RedcK {
    u64 q, qinv_neg, floor264, r1, r1_shoup;
};
__device__ __forceinline__ RedcK redc_consts(const PrimeInfo* __restrict__ pr, int prime) {
    const PrimeInfo& P = pr[prime];
    return RedcK{__ldg(&P.q), __ldg(&P.qinv_neg), __ldg(&P.pad[2]), __ldg(&P.r1), __ldg(&P.r1_shoup)};
}

// value = sum_s 2^(8s) D_s (D_s < 2^31) -> REDC(value) in [0, q)
__device__ __forceinline__ u64 partials_redc(const u32 (&d)[16], const RedcK& P) {
    const u64 q = P.q;
    auto quad = [&](int s0, int cnt) {
        u64 v = 0;
#pragma unroll
        for (int e = 0; e < 4; e++)
            if (e < cnt) v += (u64)d[s0 + e] << (8 * e);
        return v;
    };
    const u64 A = quad(0, 4), B = quad(4, 4), C = quad(8, 4), D = quad(12, 3);
    const u64 bl = B << 32, cl = C + (D << 32);
    const u64 lo = A + bl;
    const u64 hi = (B >> 32) + (lo < A ? 1ull : 0ull);
    const u64 h = (D >> 32) + (cl < C ? 1ull : 0ull);
    u64 l = cl - umulhi(cl, P.floor264) * q;
    l = l >= q ? l - q : l;
    const u64 hr = shoup(h, P.r1, P.r1_shoup, q);
    const u64 xh = hi + l + hr;
    const u64 mq = lo * P.qinv_neg;
    u64 r = xh + umulhi(mq, q) + (lo != 0ull ? 1ull : 0ull);
    r = csub(r, 2 * q);
    return csub(r, q);
}

// ---------------------------------------------------------------- kernel
#ifdef BCN_UMMA_PROF      // experiments: per-role wait/busy cycles of CTA 0, printed at exit
#define UM_TIMED(acc, stmt) do { const long long _t = clock64(); stmt; acc += clock64() - _t; } while (0)
#else
#define UM_TIMED(acc, stmt) stmt
#endif
// S[(bl * n_terms + k) * 128 + col]: the staged words of slot bl (bl = tl N + n);
// out[o * ostride + g * 2 LN + c * LN + t N + n], g = g0 + col / 2, c = col % 2
__global__ void __launch_bounds__(UM_THREADS, 1)
    mac_umma_kernel(u64* __restrict__ out, long long ostride, int n_out, int n_terms, const u8* __restrict__ planes,
                    const u64* __restrict__ S, int g0, int gcnt, int t0, int tcnt, int opad, int nch, int nlimb,
                    int logn, Limbs limbs, const PrimeInfo* __restrict__ pr, int accumulate, int dbg, int nplanes) {
    extern __shared__ __align__(1024) unsigned char um_smem[];
    unsigned char* raw = um_smem + (size_t)UM_ST * UM_SBYTES;                  // [UM_RS] raw chunk images
    u64* bars = reinterpret_cast<u64*>(raw + (size_t)UM_RS * UM_RBYTES);
    u64* full = bars;                         // [UM_ST]  transposers -> MMA
    u64* empty = full + UM_ST;                // [UM_ST]  MMA commit -> transposers
    u64* rfull = empty + UM_ST;               // [UM_RS]  bulk copies landed -> transposers
    u64* rempty = rfull + UM_RS;              // [UM_RS]  transposers -> copy issuer
    u64* accf = rempty + UM_RS;               // [2]      MMA commit -> epilogue
    u64* acce = accf + 2;                     // [2]      epilogue -> MMA
    u32* tmem_slot = reinterpret_cast<u32*>(acce + 2);

    const int N = 1 << logn;
    const long long LN = (long long)nlimb << logn;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nob = (opad + 31) >> 5;
    const long long items = (long long)tcnt * N * nob;

    // zero the B strips once: only plane rows 7..14 are ever rewritten
    for (int x = threadIdx.x; x < UM_ST * 2 * UM_BHALF / 16; x += blockDim.x) {
        const int st = x / (2 * UM_BHALF / 16), r = x % (2 * UM_BHALF / 16);
        reinterpret_cast<uint4*>(um_smem + (size_t)st * UM_SBYTES + UM_ABYTES)[r] = make_uint4(0, 0, 0, 0);
    }
    fence_async_smem();
    if (threadIdx.x == 0) {
        for (int s = 0; s < UM_ST; s++) {
            mbar_init(&full[s], UM_TR * 32);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < UM_RS; s++) {
            mbar_init(&rfull[s], 1);
            mbar_init(&rempty[s], UM_TR * 32);
        }
        for (int s = 0; s < 2; s++) {
            mbar_init(&accf[s], 1);
            mbar_init(&acce[s], UM_EPI * 32);
        }
        fence_barrier_init();
    }
    if (warp == UM_W_MMA) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const u32 tmem = *tmem_slot;
    long long tw = 0, tw2 = 0;
    const long long tstart = clock64();
    // items strided over the CTAs: at any moment the GPU streams adjacent slots,
    // i.e. one contiguous region of S (a contiguous run per CTA is 2x slower)
    const long long i_hi = items;
    // item sequence of this CTA: items strided over the CTAs; with one item per
    // slot (<= 32 outputs) in pairs of adjacent slots, so the epilogue can hold a
    // pair's words and store them as 16-byte runs (half the store requests of
    // the 32-lines-per-instruction 8-byte stores)
    const bool paired = nob == 1 && opad <= UM_PAIR_MAXO && !(dbg & 16);
#ifndef UM_ALT
#define UM_ALT 1
#endif
    const bool alt = UM_ALT && nob == 1 && opad <= 16;       // every item has ONE 16-output block
    auto item_at = [&](long long k) -> long long {
        return paired ? 2 * ((long long)blockIdx.x + (k >> 1) * gridDim.x) + (k & 1)
                      : (long long)blockIdx.x + k * gridDim.x;
    };

    if (warp == UM_W_COPY) {
        // ------------------------------------------------ bulk-copy issuer (one lane)
        if (lane == 0) {
            u32 it = 0;
            for (long long kk = 0, item = item_at(0); item < i_hi; item = item_at(++kk)) {
                const long long bl = item / nob;
                const int ob = (int)(item - bl * nob);
                const int nbo = min(2, (opad - ob * 32) >> 4);
                const long long b = bl + (long long)t0 * N;
                for (int c = 0; c < nch; c++, it++) {
                    const int rs = it % UM_RS;
                    UM_TIMED(tw, um_wait(&rempty[rs], ((it / UM_RS) & 1) ^ 1));
                    const int kmax = min(32, n_terms - c * 32);
                    const u32 sb = (u32)kmax * UM_COLS * 8, pb = (u32)nbo * 16 * 256;
                    unsigned char* dst = raw + (size_t)rs * UM_RBYTES;
                    mbar_expect_tx(&rfull[rs], sb + pb);
#ifndef UM_SPLIT
#define UM_SPLIT 1
#endif
#pragma unroll
                    for (int sp = 0; sp < UM_SPLIT; sp++)    // UM_SPLIT concurrent bulk copies per chunk
                        bulk_load(dst + sp * (sb / UM_SPLIT),
                                  reinterpret_cast<const unsigned char*>(S + (bl * n_terms + c * 32) * UM_COLS) +
                                      sp * (sb / UM_SPLIT),
                                  sb / UM_SPLIT, &rfull[rs]);
                    bulk_load(dst + UM_COLS * 32 * 8, planes + ((b * nch + c) * opad + ob * 32) * 256, pb, &rfull[rs]);
                }
            }
        }
    } else if (warp < UM_TR) {
        // ------------------------------------------------ transposers: raw words -> byte planes
        // thread = one column; per k-half it reads 16 words (lanes: 32 consecutive
        // columns, conflict-free) and writes one 16-byte core-matrix row per plane
        // (lanes: 512 contiguous bytes, conflict-free)
        const int col = threadIdx.x & (UM_COLS - 1);     // 0 .. 127
        constexpr int KH = UM_TR * 32 / UM_COLS;         // k-halves per thread's column split: 1 or 2 threads
        const int kh0 = (UM_TR == 8) ? (threadIdx.x >> 7) : 0;
        u32 it = 0;
        for (long long kk = 0, item = item_at(0); item < i_hi; item = item_at(++kk)) {
            const long long bl = item / nob;
            const int ob = (int)(item - bl * nob);
            const int nbo = min(2, (opad - ob * 32) >> 4);
            for (int c = 0; c < nch; c++, it++) {
                const int rs = it % UM_RS, stage = it % UM_ST;
                UM_TIMED(tw, um_wait(&rfull[rs], (it / UM_RS) & 1));
                UM_TIMED(tw2, um_wait(&empty[stage], ((it / UM_ST) & 1) ^ 1));
                const u64* rw = reinterpret_cast<const u64*>(raw + (size_t)rs * UM_RBYTES);
                const uint4* rp = reinterpret_cast<const uint4*>(raw + (size_t)rs * UM_RBYTES + UM_COLS * 32 * 8);
                u8* As = um_smem + (size_t)stage * UM_SBYTES;
                u8* Bs = As + UM_ABYTES;
#pragma unroll
                for (int kx = 0; kx < 2 / KH; kx++) {
                    const int kh = kh0 + kx;
                    u32 pl[8][4];
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        u64 v[4];
#pragma unroll
                        for (int r = 0; r < 4; r++) v[r] = rw[(kh * 16 + q * 4 + r) * UM_COLS + col];
                        u32 bp[8];
                        bytes_by_plane(v, bp);
#pragma unroll
                        for (int j = 0; j < 8; j++) pl[j][q] = bp[j];
                    }
                    u8* dst = As + kh * (UM_COLS * 16) + (col >> 3) * 128 + (col & 7) * 16;
#pragma unroll
                    for (int j = 0; j < 8; j++)
                        *reinterpret_cast<uint4*>(dst + j * UM_APLANE) = make_uint4(pl[j][0], pl[j][1], pl[j][2], pl[j][3]);
                }
                // B: piece (output, k-half, plane) -> its strip row 7 + plane
                for (int p = threadIdx.x; p < nbo * 256; p += UM_TR * 32) {
                    const int o = p >> 4, kh = (p >> 3) & 1, i = p & 7;
                    *reinterpret_cast<uint4*>(Bs + kh * UM_BHALF + (o * 16 + 7 + i) * 16) = rp[p];
                }
                fence_async_smem();
                mbar_arrive(&full[stage]);
                mbar_arrive(&rempty[rs]);
            }
        }
    } else if (warp == UM_W_MMA) {
        // ------------------------------------------------ MMA issuer
        u32 it = 0, use[2] = {0, 0};
        for (long long kk = 0, item = item_at(0); item < i_hi; item = item_at(++kk)) {
            const int ob = (int)(item % nob);
            const int nbo = min(2, (opad - ob * 32) >> 4);
            for (int c = 0; c < nch; c++, it++) {
                const int stage = it % UM_ST;
                UM_TIMED(tw, um_wait(&full[stage], (it / UM_ST) & 1));
                tc_fence_after();
                if (lane == 0) {
                    const u32 a0 = smem_addr(um_smem + (size_t)stage * UM_SBYTES);
                    const u32 b0 = a0 + UM_ABYTES;
                    for (int nb = 0; nb < nbo; nb++) {
                        // one 16-output block per item: items alternate between the two TMEM
                        // accumulators, so the next item's MMAs run while this one drains
                        const int ai = alt ? (int)(kk & 1) : nb;
                        if (c == 0) {
                            UM_TIMED(tw2, um_wait(&acce[ai], (use[ai] & 1) ^ 1));
                            tc_fence_after();
                        }
#pragma unroll
                        for (int j = 0; j < 8; j++) {             // byte planes of the staged words
                            if (j >= nplanes) break;              // every prime < 2^56: byte 7 is zero
                            const u64 ad = umma_sdesc(a0 + j * UM_APLANE, UM_COLS * 16, 128);
                            const u64 bd = umma_sdesc(b0 + (nb * 256 + 7 - j) * 16, UM_BHALF, 128);
                            if (!(dbg & 4)) umma_i8(tmem + ai * 256, ad, bd, (c > 0 || j > 0) ? 1u : 0u);
                        }
                        if (c == nch - 1) umma_commit(&accf[ai]);
                    }
                    umma_commit(&empty[stage]);
                }
                __syncwarp();
            }
            if (alt) use[kk & 1]++;
            else
                for (int nb = 0; nb < nbo; nb++) use[nb]++;
        }
    } else {
        // ------------------------------------------------ epilogue
        const int e = warp - UM_W_EPI;                   // 0 .. 7
        const int quarter = warp & 3;                    // TMEM lanes this warp may read
        const int ohalf = e >> 2;                        // outputs 8 ohalf .. + 7 of each 16-block
        const int col = quarter * 32 + lane;
        const bool live_col = col < 2 * gcnt;
        u32 use[2] = {0, 0};
        u64 hold[16];                                    // paired mode: the even slot's words [nb][og][x]
#pragma unroll
        for (int x = 0; x < 16; x++) hold[x] = 0;
        for (long long kk = 0, item = item_at(0); item < i_hi; item = item_at(++kk)) {
            const long long bl = item / nob;
            const int ob = (int)(item - bl * nob);
            const int nbo = min(2, (opad - ob * 32) >> 4);
            const long long b = bl + (long long)t0 * N;  // t N + n
            const RedcK P = redc_consts(pr, limbs.prime[(int)(b >> logn)]);
            u64* obase = out + (long long)(g0 + (col >> 1)) * 2 * LN + (col & 1) * LN + b;
            for (int nb = 0; nb < nbo; nb++) {
                const int ai = alt ? (int)(kk & 1) : nb;
                UM_TIMED(tw, um_wait(&accf[ai], use[ai] & 1));
                tc_fence_after();
                // two groups of four outputs: four TMEM loads in flight per wait, four
                // independent recombine+REDC chains; the accumulator is released as
                // soon as the last group is in registers
#pragma unroll 1
                for (int og = 0; og < 2; og++) {
                    u32 d[4][16];
                    const bool hold_it = paired && (kk & 1) == 0;     // even slot of a pair: keep
                    const bool pair_st = paired && (kk & 1) == 1;     // odd slot: store both
#pragma unroll
                    for (int x = 0; x < 4; x++)
                        tmem_ld16(tmem + ((u32)(quarter * 32) << 16) + ai * 256 + (ohalf * 8 + og * 4 + x) * 16, d[x]);
                    tmem_wait_ld();
                    if (og == 1) {
                        tc_fence_before();
                        mbar_arrive(&acce[ai]);
                    }
                    u64 r[4];                            // branch-free: four interleaved chains
#pragma unroll
                    for (int x = 0; x < 4; x++) r[x] = partials_redc(d[x], P);
#pragma unroll
                    for (int x = 0; x < 4; x++) {
                        const int o = ob * 32 + nb * 16 + ohalf * 8 + og * 4 + x;
                        if (hold_it) {                            // static register indices
                            if (nb == 0) { if (og == 0) hold[x] = r[x]; else hold[4 + x] = r[x]; }
                            else { if (og == 0) hold[8 + x] = r[x]; else hold[12 + x] = r[x]; }
                        } else if (live_col && o < n_out && !(dbg & 1)) {
                            u64* po = obase + (long long)o * ostride;
                            if (pair_st) {                        // slots b - 1, b: one 16-byte store
                                ulonglong2* pp = reinterpret_cast<ulonglong2*>(po - 1);
                                const u64 h = nb == 0 ? (og == 0 ? hold[x] : hold[4 + x])
                                                      : (og == 0 ? hold[8 + x] : hold[12 + x]);
                                ulonglong2 v = make_ulonglong2(h, r[x]);
                                if (accumulate) {
                                    const ulonglong2 a = *pp;
                                    v.x = add_mod(v.x, a.x, P.q);
                                    v.y = add_mod(v.y, a.y, P.q);
                                }
                                *pp = v;
                            } else {
                                const u64 v = accumulate ? add_mod(r[x], *po, P.q) : r[x];
                                if (!(dbg & 8) || v == 12345ull) *po = v;
                            }
                        }
                    }
                }
                use[ai]++;
            }
        }
    }
#ifdef BCN_UMMA_PROF
    if (blockIdx.x == 0 && lane == 0 && (warp == 0 || warp == UM_W_COPY || warp == UM_W_MMA || warp == UM_W_EPI))
        printf("umma role %d: total %lld wait %lld wait2 %lld\n", warp, clock64() - tstart, tw, tw2);
#endif
    (void)tw;
    (void)tw2;
    (void)tstart;
    tc_fence_before();
    __syncthreads();
    if (warp == UM_W_MMA)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

size_t mac_umma_smem() { return UM_SMEM; }

cudaError_t mac_umma_op(u64* out, long long out_stride, int n_out, int n_terms, const u8* planes, const u64* S,
                        int g0, int gcnt, int t0, int tcnt, int opad, int nlimb, int logn, const Limbs& limbs,
                        const PrimeInfo* pr, int accumulate, cudaStream_t st, int nplanes) {
    if (gcnt <= 0 || n_terms <= 0 || n_out <= 0) return cudaSuccess;
    if (gcnt > UM_COLS / 2 || nplanes < 7 || nplanes > 8) return cudaErrorInvalidValue;
    const int nch = (n_terms + 31) / 32;
    static unsigned long long smem_cfg = 0;
    unsigned long long smem_bit = 0;
    if (first_on_device(&smem_cfg, &smem_bit)) {
        cudaError_t ae = cudaSuccess;
        BCN_SMEM_ATTR(ae, (mac_umma_kernel), (int)UM_SMEM);
        if (ae != cudaSuccess) return ae;
        smem_cfg |= smem_bit;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long items = (long long)tcnt * (1LL << logn) * ((opad + 31) / 32);
    const int grid = (int)std::min<long long>(items, sms);
    static const int dbg = getenv("BCN_UMMA_DBG") ? atoi(getenv("BCN_UMMA_DBG")) : 0;   // experiments only
    mac_umma_kernel<<<grid, UM_THREADS, UM_SMEM, st>>>(out, out_stride, n_out, n_terms, planes, S, g0, gcnt, t0, tcnt,
                                                       opad, nch, nlimb, logn, limbs, pr, accumulate, dbg, nplanes);
    return launched();
}

}  // namespace bcn
