// mac_imma.cu -- multi-output ciphertext x plaintext MAC (the conv-layer
// linear combination out_o = sum_k ct_k (x) pt_{o,k}) on the integer tensor
// cores.
//
// For one coefficient slot b = (limb t, coefficient n) the op is a small
// matrix product over Z: D[o][gc] = sum_k P[o][k] * C[k][gc] with P the
// (Montgomery) plaintext words, C the ciphertext words of all slot sets and
// components (gc = 2g + c), every entry < q < 2^61.  Splitting both operands
// into bytes, P = sum_i 2^(8i) P_i and C = sum_j 2^(8j) C_j, gives
//     D = sum_s 2^(8s) D_s,   D_s = sum_{i+j=s} P_i C_j   (s = 0..14),
// fifteen u8 x u8 -> s32 matrix products with exact int32 accumulation
// (<= 8 pairs x 256 terms x 255^2 < 2^31).  Each D_s is computed on the
// tensor cores with mma.sync m16n8k32 (IMMA); the epilogue recombines the
// fifteen partials into the 128-bit value, reduces it mod q (one REDC, which
// also strips the Montgomery factor of P) and writes the canonical word.
// Bit-exact with the CUDA-core kernel (mac_multi_op) by construction.
//
// Operands:
//  * P is constant per layer, so it is packed ONCE (pack_planes_kernel) into
//    byte planes laid out exactly as the A fragments want them:
//      planes[((b * nch + c) * 8 + i) * opad * 32 + o * 32 + kperm(kk)]
//    = byte i of pt[o][32c + kk] at slot b  (zero-padded to opad rows and
//    nch * 32 terms), where kperm interleaves k so that a thread's two A
//    registers (k = 4tq.. and 16 + 4tq..) are one 8-byte load.
//  * C is the fresh rotated ciphertexts: each CTA gathers the words of its
//    slot (one word per (k, gc), cp.async 8 B) into shared memory, and every
//    thread byte-transposes its four k-consecutive words into the eight B
//    fragments (j = 0..7) with 16 PRMTs.
// One CTA = one slot b x one block of up to 32 slot-set columns x one block
// of up to 32 outputs; warp w owns M-tile (16 outputs) x N-tile (8 columns)
// and keeps its 15 partial accumulators (60 registers) over the whole term
// loop, which runs in chunks of 32 terms through a 3-stage cp.async ring.
#include "common.cuh"
#include "ops.cuh"

namespace bcn {

typedef unsigned char u8;

// one thread per (o, chunk c, limb t, coefficient n); n fastest -> the 32
// plaintext reads of a warp are coalesced.  Within a plane, each 16-row
// M-tile is stored in mma.m16n8k32 A-fragment order: the 16 bytes a lane
// (gq, tq) needs -- {row gq, row gq+8} x {k 4tq.., k 16+4tq..} -- are one
// contiguous LDS.128 in the MAC kernel:
//   offset(o, kk) = (o/16)*512 + ((o%8)*4 + (kk%16)/4)*16 + ((kk/16)*2 + (o%16)/8)*4 + kk%4
__global__ void pack_planes_kernel(u8* __restrict__ planes, const u64* const* __restrict__ pts, int n_out,
                                   int n_terms, int opad, int nch, int logn, const int* __restrict__ tlimbs) {
    const int N = 1 << logn;
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    const int t = blockIdx.y;
    const int o = blockIdx.z / nch, c = blockIdx.z % nch;
    const long long b = (long long)t * N + n;
    u32 w[8][8];                                          // [plane i][hi * 4 + tq]
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
        for (int d = 0; d < 8; d++) w[i][d] = 0u;
#pragma unroll
    for (int kk = 0; kk < 32; kk++) {
        const int k = c * 32 + kk;
        const bool live = o < n_out && k < n_terms && (!tlimbs || t < tlimbs[k]);   // short plaintexts: 0 above
        const u64 v = live ? __ldg(pts[(size_t)o * n_terms + k] + b) : 0ull;
        const int d = (kk >> 4) * 4 + ((kk & 15) >> 2), sh = (kk & 3) * 8;
#pragma unroll
        for (int i = 0; i < 8; i++) w[i][d] |= (u32)((v >> (8 * i)) & 0xffull) << sh;
    }
    const int m = o >> 4, g = o & 7, half = (o >> 3) & 1;
    u8* base = planes + ((b * nch + c) * 8) * (long long)opad * 32 + (long long)m * 512 + g * 64 + half * 4;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        u32* p = reinterpret_cast<u32*>(base + (long long)i * opad * 32);
#pragma unroll
        for (int d = 0; d < 8; d++) p[((d & 3) * 16 + (d >> 2) * 8) / 4] = w[i][d];   // tq*16 + hi*8
    }
}

cudaError_t pack_planes_op(u8* planes, const u64* const* pts_dev, int n_out, int n_terms, int opad, int nch, int nl,
                           int logn, cudaStream_t st, const int* tlimbs_dev) {
    const int N = 1 << logn;
    const int tpb = N < 128 ? N : 128;
    dim3 grid((N + tpb - 1) / tpb, nl, opad * nch);
    pack_planes_kernel<<<grid, tpb, 0, st>>>(planes, pts_dev, n_out, n_terms, opad, nch, logn, tlimbs_dev);
    return launched();
}

// ------------------------------------- fused key switch + slot-major staging
// Conv layer with lazy ModDown: term k is the source ciphertext x_k rotated
// by g_k (g_k = 1: x_k itself).  Instead of materialising rot_k(x_k) (one
// ModDown per rotation) the MAC runs on the extended basis over
//   B'_k,c = sum_j sigma_k(U_k,j) (x) key_k,j,c  +  [c = 0] P sigma_k(c0_k)   (g_k != 1)
//   B'_k,c = P x_k,c  on q_0..q_l, 0 on p_*                                   (g_k = 1)
// so that ModDown(B'_k) = rot_k(x_k) exactly in value, and the conv outputs
// need one merged ModDown+rescale each.  This kernel computes B'_k for a
// block of slot sets and extended limbs and writes it slot-major
// (S[(tl N + n) K + k][64]) for mac_imma_kernel; the key inner product never
// touches HBM.  One CTA = (32 coefficients, limb, term).  Under X -> X^g an
// aligned 32-block is the image of one aligned 32-block, so the gathers stay
// inside one 256-byte segment.
// a staged word congruent to acc mod q, in [0, 2^52): ND <= 2 (|acc| < 1.9q, the
// P sigma(c0) term included): acc + 2q; else fred to [-q/2, q/2] then + q
template <int ND>
__device__ __forceinline__ u64 fstage(double acc, double stage_c, double qinv, double q) {
    const double y = ND <= 2 ? acc : fred(acc, qinv, q);
    return (u64)__double_as_longlong(__dadd_rn(y, stage_c)) & ((1ull << 52) - 1);
}

#ifndef BCN_SMKS_MINB
#define BCN_SMKS_MINB 4
#endif
#ifndef BCN_SMKS_UNROLL
#define BCN_SMKS_UNROLL 2
#endif
constexpr int kSmksUnroll = BCN_SMKS_UNROLL;    // (#pragma arguments are not macro-expanded)
#ifndef BCN_SMKS_FP64_BOTH
#define BCN_SMKS_FP64_BOTH 1      // both components on the FP64 pipe (0: component 1 on IMAD; A/B 108.9 vs 111.0 ms)
#endif
template <int ND>    // digits (1..4); 0: any count, key words re-read from L1
__global__ void __launch_bounds__(256, BCN_SMKS_MINB) slot_major_ks_kernel(u64* __restrict__ S, const KsTerms T, int g0, int gcnt,
                                                            int t0, int nq, int next, int ndig, int logn,
                                                            int spitch, long long kds, long long kcs, Limbs ext,
                                                            const PrimeInfo* __restrict__ pr,
                                                            const u64* __restrict__ pmod,
                                                            const double2* __restrict__ fq) {
    __shared__ u64 tile[128][33];
    const int N = 1 << logn;
    const int n0 = blockIdx.x * 32, tl = blockIdx.y, k = blockIdx.z;
    const int t = t0 + tl;
    const int ncol = 2 * gcnt;
    const int kt = ext.prime[t];
    const PrimeInfo& P = pr[kt];
    const u64 q = P.q;
    const u32 g = T.g[k];
    const long long LNs = (long long)nq * N;                      // source ct: [G][2][nq][N]
    // lane = coefficient, warp = a strided set of slot sets (both components:
    // one set of U loads feeds the two key products); the permutation, the
    // key words and the P multiplier are per lane only
    const int nn = threadIdx.x & 31, w0 = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int n = n0 + nn;
    const u64* src = T.src[k] + (long long)t * N;
    const bool qlimb = t < nq;
    const u64 pw = qlimb ? pmod[2 * t] : 0ull, pwp = qlimb ? pmod[2 * t + 1] : 0ull;
    if (g == 1u) {
#pragma unroll 4
        for (int col = w0; col < ncol; col += nw) {
            const int gs = g0 + (col >> 1), c = col & 1;
            tile[col][nn] = qlimb ? shoup(__ldg(src + (long long)gs * 2 * LNs + c * LNs + n), pw, pwp, q) : 0ull;
        }
    } else {
        const int sn = (int)automorph_src((u32)n, g, logn);
        constexpr int KD = ND > 0 ? ND : 1;
        u64 k0[KD], k1[KD];
        const u64* kp = T.key[k] + (long long)kt * N + n;
        if constexpr (ND > 0) {
#pragma unroll
            for (int j = 0; j < ND; j++) { k0[j] = __ldg(kp + j * kds); k1[j] = __ldg(kp + j * kds + kcs); }
        }
        const int nd = ND > 0 ? ND : ndig;
        const long long dstr = (long long)next * N;
        const u64* Ub = T.U[k] + (long long)t * N + sn;
        if constexpr (ND > 0) {
            if (fq) {
                // component 0 on the FP64 pipe, component 1 on the IMAD pipe: the two
                // inner products of one set of U words run on different units.  The
                // key words are Montgomery (k 2^64): REDC once per thread to k, then
                // {k, k/q} as doubles (companion from fl(1/q): |a w/q - qt| <= 0.75).
                const double2 f = fq[kt];
                double kd[ND], kq[ND];
#pragma unroll
                for (int j = 0; j < ND; j++) {
                    kd[j] = fload(redc(0ull, k0[j], q, P.qinv_neg));
                    kq[j] = __dmul_rn(kd[j], f.y);
                }
                // staged words need only be < 2^56 and congruent mod q (the tensor-core
                // epilogues reduce any such sum): ND <= 2 sums stay in (-1.9q, 1.9q), so the
                // word is acc + 2q read off the mantissa of acc + (2^52 + 2q)
                const double stage_c = ND <= 2 ? __dadd_rn(4503599627370496.0, __dadd_rn(f.x, f.x))
                                               : __dadd_rn(4503599627370496.0, f.x);
#if BCN_SMKS_FP64_BOTH
                // component 1 on the FP64 pipe as well: the converted U words feed both sums
                double kd1[ND], kq1[ND];
#pragma unroll
                for (int j = 0; j < ND; j++) {
                    kd1[j] = fload(redc(0ull, k1[j], q, P.qinv_neg));
                    kq1[j] = __dmul_rn(kd1[j], f.y);
                }
#endif
                // P sigma(c0) joins component 0's FP64 sum as one more two-product term
                // (|sum| < (ND + 1) 0.63 q < 2^53: exact), so no 64-bit Shoup product;
                // the operand pointers advance by constant strides (no per-slot-set
                // 64-bit index products)
                const double pd = qlimb ? fload(pw) : 0.0, pq = __dmul_rn(pd, f.y);
                const long long ustep = (long long)nw * nd * dstr, cstep = (long long)nw * 2 * LNs;
                const u64* Up = Ub + (long long)(g0 + w0) * nd * dstr;
                const u64* Cp = src + (long long)(g0 + w0) * 2 * LNs + sn;
#pragma unroll kSmksUnroll
                for (int gi = w0; gi < gcnt; gi += nw, Up += ustep, Cp += cstep) {
                    double acc = qlimb ? fmm(fload(__ldg(Cp)), pd, pq, f.x) : 0.0;
#if BCN_SMKS_FP64_BOTH
                    double acc1 = 0.0;
#pragma unroll
                    for (int j = 0; j < ND; j++) {
                        const double ud = fload(__ldg(Up + j * dstr));
                        acc = __dadd_rn(acc, fmm(ud, kd[j], kq[j], f.x));
                        acc1 = __dadd_rn(acc1, fmm(ud, kd1[j], kq1[j], f.x));
                    }
                    tile[2 * gi][nn] = fstage<ND>(acc, stage_c, f.y, f.x);
                    tile[2 * gi + 1][nn] = fstage<ND>(acc1, stage_c, f.y, f.x);
#else
                    Acc4 a1;
                    a1.zero();
#pragma unroll
                    for (int j = 0; j < ND; j++) {
                        const u64 u = __ldg(Up + j * dstr);
                        acc = __dadd_rn(acc, fmm(fload(u), kd[j], kq[j], f.x));
                        a1.mac(u, k1[j]);
                    }
                    tile[2 * gi][nn] = fcanon(acc, f.y, f.x);
                    tile[2 * gi + 1][nn] = a1.reduce(q, P.qinv_neg, P.pad[2]);
#endif
                }
            }
        }
#pragma unroll 2
        for (int gi = w0; gi < gcnt && !(ND > 0 && fq); gi += nw) {
            const int gs = g0 + gi;
            const u64* Up = Ub + (long long)gs * nd * dstr;
            Acc4 a0, a1;
            a0.zero();
            a1.zero();
            if constexpr (ND > 0) {
#pragma unroll
                for (int j = 0; j < ND; j++) {
                    const u64 u = __ldg(Up + j * dstr);
                    a0.mac(u, k0[j]);
                    a1.mac(u, k1[j]);
                }
            } else {
                for (int j = 0; j < nd; j++) {
                    const u64 u = __ldg(Up + j * dstr);
                    a0.mac(u, __ldg(kp + j * kds));
                    a1.mac(u, __ldg(kp + j * kds + kcs));
                }
            }
            u64 v0 = a0.reduce(q, P.qinv_neg, P.pad[2]);
            if (qlimb) v0 = add_mod(v0, shoup(__ldg(src + (long long)gs * 2 * LNs + sn), pw, pwp, q), q);
            tile[2 * gi][nn] = v0;
            tile[2 * gi + 1][nn] = a1.reduce(q, P.qinv_neg, P.pad[2]);
        }
    }
    __syncthreads();
    u64* dst = S + (((long long)tl * N + n0) * T.n + k) * spitch;
    for (int r = w0; r < 32; r += nw)                      // row r: this slot's run of ncol words
        for (int col = nn; col < ncol; col += 32) dst[(long long)r * T.n * spitch + col] = tile[col][r];
}

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int K> __device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(K) : "memory");
}

// ---- source-shared form: every U word crosses L2 once, not once per rotation ----
// ncu on the kernel above (conv2: 16 sources x 16 rotations, 64 slot sets, one
// limb): 6.4 GB of L2 reads (each U word gathered by all 16 rotations of its
// source) + 4.3 GB of staged writes per launch, ~5 TB/s through L2 whatever
// the occupancy or the loads in flight (a warp-per-term variant with 12 loads
// in flight per thread and half the instructions measured 2.27 vs 2.02 ms).
// So the work is regrouped by SOURCE block: a CTA takes 32 source coefficients m of one limb and a run of
// <= 16 consecutive terms over the same (src, U), loads the block's U digits and
// c0 for every slot set into shared memory once (cp.async), and each warp then
// evaluates whole terms from that tile: lane = m, output coefficient n =
// sigma_g^-1(m) (X -> X^g maps the aligned 32-block of m onto ONE aligned
// 32-block of n, permuted), keys gathered at n, staged words into the warp's
// private tile at row n % 32 and flushed as 16-byte stores (__syncwarp only).
// Bank conflicts: within the block lane -> n % 32 is brev5(c + g brev5(lane)),
// which keeps each aligned group of 8 lanes inside one aligned group of 8 rows,
// so the 16-byte tile stores (8 lanes per wavefront) never collide.
struct KsGroups {
    int n;
    unsigned short start[BCN_IMMA_TERMS];
    unsigned char count[BCN_IMMA_TERMS];
};
// Work split inside the CTA: by SLOT SET, not by term.  Warp w owns 4 slot sets
// of the CTA's 32 and walks the run's terms: its U digits (as doubles) and the
// rotation-independent P c0 product stay in registers for all <= 16 rotations,
// so per (slot set, rotation) only the 2 ND key products remain (30 FP64
// instructions at ND = 2 instead of 39 + 3 conversions).  The run's key words
// are converted once per CTA -- warp w converts rotations w and w + 8 into
// {k, k/q} doubles in shared memory, indexed by the SOURCE coefficient -- with
// one __syncthreads; after it warps never wait on each other.
constexpr int KS3_TP = 10;                                     // out tile pitch (u64): 8 columns + pad
template <int ND> constexpr size_t ks3_smem_bytes() {
    return (size_t)16 * ND * 4 * 256 + (size_t)8 * 32 * KS3_TP * 8 + 16 * 32 + 16 * 4;
}
template <int ND>
__global__ void __launch_bounds__(256, 3)
    slot_major_ks3_kernel(u64* __restrict__ S, const KsTerms T, const KsGroups GR, int g0, int gcnt, int nsplit, int t0,
                          int nq, int next, int logn, int spitch, long long kds, long long kcs, Limbs ext,
                          const PrimeInfo* __restrict__ pr, const u64* __restrict__ pmod,
                          const double2* __restrict__ fq, int nat_gtot) {
    extern __shared__ __align__(16) unsigned char ks3_smem[];
    double(*kfp)[ND][4][32] = reinterpret_cast<double(*)[ND][4][32]>(ks3_smem);          // [16 terms]: kd, kq, kd1, kq1
    u64(*tiles)[32][KS3_TP] = reinterpret_cast<u64(*)[32][KS3_TP]>(ks3_smem + (size_t)16 * ND * 4 * 256);   // [8 warps]
    unsigned char(*nrow_s)[32] =
        reinterpret_cast<unsigned char(*)[32]>(ks3_smem + (size_t)16 * ND * 4 * 256 + (size_t)8 * 32 * KS3_TP * 8);
    int* nblk_s = reinterpret_cast<int*>(nrow_s + 16);
    const int N = 1 << logn;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int m0 = blockIdx.x * 32, tl = blockIdx.y / nsplit, half = blockIdx.y - tl * nsplit, t = t0 + tl;
    const int kfirst = GR.start[blockIdx.z], kcount = GR.count[blockIdx.z];
    const int kt = ext.prime[t];
    const PrimeInfo& P = pr[kt];
    const u64 q = P.q;
    const long long LNs = (long long)nq * N;
    const bool qlimb = t < nq;
    const long long dstr = (long long)next * N;
    const long long ustep = (long long)ND * dstr, cstep = 2 * LNs;
    const double2 f = fq[kt];
    const int gs0 = half * 32 + w * 4;                         // this warp's slot sets gs0 .. gs0 + 3
    // ---- this thread's operands, once (12 loads in flight), before the key conversion's own loads
    const u64* U0 = nullptr;                                   // the run's ModUp: its first rotation term's
    for (int ki = 0; ki < kcount && !U0; ki++)
        if (T.g[kfirst + ki] != 1u) U0 = T.U[kfirst + ki];
    u64 uw[4][ND], cw[4];
    {
        const u64* Up = U0 ? U0 + (long long)t * N + m0 + lane + (long long)g0 * ustep : nullptr;
        const u64* Cp = T.src[kfirst] + (long long)t * N + m0 + lane + (long long)g0 * cstep;
#pragma unroll
        for (int b = 0; b < 4; b++) {
            const long long gs = gs0 + b < gcnt ? gs0 + b : 0;
            cw[b] = qlimb ? __ldg(Cp + gs * cstep) : 0ull;
#pragma unroll
            for (int j = 0; j < ND; j++) uw[b][j] = Up ? __ldg(Up + gs * ustep + j * dstr) : 0ull;
        }
    }
    // ---- the run's keys: rotation r's words at n = sigma_r^-1(m), as doubles, by warps r % 8
    for (int r = w; r < kcount; r += 8) {
        const int k = kfirst + r;
        const u32 g = T.g[k];
        u32 ginv = g;                                          // g^-1 mod 2^32 (Newton; g g = 1 mod 8)
#pragma unroll
        for (int i = 0; i < 4; i++) ginv *= 2u - g * ginv;
        const int n = g == 1u ? m0 + lane : (int)automorph_src((u32)(m0 + lane), ginv & ((2u << logn) - 1u), logn);
        nrow_s[r][lane] = (unsigned char)(n & 31);
        if (lane == 0) nblk_s[r] = n & ~31;
        if (g != 1u) {
            const u64* kp = T.key[k] + (long long)kt * N + n;
            u64 kw[ND][2];
#pragma unroll
            for (int j = 0; j < ND; j++) { kw[j][0] = __ldg(kp + j * kds); kw[j][1] = __ldg(kp + j * kds + kcs); }
#pragma unroll
            for (int j = 0; j < ND; j++)
#pragma unroll
                for (int c = 0; c < 2; c++) {                  // Montgomery key word -> {k, k/q}
                    const double kd = fload(redc(0ull, kw[j][c], q, P.qinv_neg));
                    kfp[r][j][2 * c][lane] = kd;
                    kfp[r][j][2 * c + 1][lane] = __dmul_rn(kd, f.y);
                }
        }
    }
    const u64 pw = qlimb ? pmod[2 * t] : 0ull;
    const double pd = qlimb ? fload(pw) : 0.0, pq = __dmul_rn(pd, f.y);
    const double stage_c = ND <= 2 ? __dadd_rn(4503599627370496.0, __dadd_rn(f.x, f.x))
                                   : __dadd_rn(4503599627370496.0, f.x);
    double ud[4][ND], a0[4];
#pragma unroll
    for (int b = 0; b < 4; b++) {
        a0[b] = qlimb ? fmm(fload(cw[b]), pd, pq, f.x) : 0.0;  // P c0: the same for every rotation
#pragma unroll
        for (int j = 0; j < ND; j++) ud[b][j] = fload(uw[b][j]);
    }
    __syncthreads();
    if (gs0 >= gcnt) return;
    u64(*tw)[KS3_TP] = tiles[w];
    const int fr = lane >> 2, fp = lane & 3;                   // flush: 8 rows x four 16-byte pieces per instruction
    const long long rstride = (long long)T.n * spitch;
    for (int r = 0; r < kcount; r++) {
        const int k = kfirst + r;
        const u32 g = T.g[k];
        const int nrow = nrow_s[r][lane];
        u64 v0[4], v1[4];
        if (g == 1u) {                                         // P x (both components); c1 from HBM
            const u64* c1p = T.src[k] + (long long)t * N + m0 + lane + LNs + (long long)g0 * cstep;
#pragma unroll
            for (int b = 0; b < 4; b++) {
                const long long gs = gs0 + b < gcnt ? gs0 + b : 0;
                const double a1 = qlimb ? fmm(fload(__ldg(c1p + gs * cstep)), pd, pq, f.x) : 0.0;
                v0[b] = nat_gtot ? fcanon(a0[b], f.y, f.x) : fstage<ND>(a0[b], stage_c, f.y, f.x);
                v1[b] = nat_gtot ? fcanon(a1, f.y, f.x) : fstage<ND>(a1, stage_c, f.y, f.x);
            }
        } else {
            double kd[ND], kq[ND], kd1[ND], kq1[ND];
#pragma unroll
            for (int j = 0; j < ND; j++) {
                kd[j] = kfp[r][j][0][lane];
                kq[j] = kfp[r][j][1][lane];
                kd1[j] = kfp[r][j][2][lane];
                kq1[j] = kfp[r][j][3][lane];
            }
#pragma unroll
            for (int b = 0; b < 4; b++) {
                double acc = a0[b], acc1 = 0.0;
#pragma unroll
                for (int j = 0; j < ND; j++) {
                    acc = __dadd_rn(acc, fmm(ud[b][j], kd[j], kq[j], f.x));
                    acc1 = __dadd_rn(acc1, fmm(ud[b][j], kd1[j], kq1[j], f.x));
                }
                v0[b] = nat_gtot ? fcanon(acc, f.y, f.x) : fstage<ND>(acc, stage_c, f.y, f.x);
                v1[b] = nat_gtot ? fcanon(acc1, f.y, f.x) : fstage<ND>(acc1, stage_c, f.y, f.x);
            }
        }
        if (nat_gtot) {
            // natural layout (hoisted multi-rotation key switch): out[term][slot set][component][limb][n],
            // canonical residues; the lanes' n are a permutation of one aligned 32-block
            const int n = nblk_s[r] + nrow;
#pragma unroll
            for (int b = 0; b < 4; b++) {
                if (gs0 + b >= gcnt) break;
                u64* o = S + ((((long long)k * nat_gtot + g0 + gs0 + b) * 2) * next + t) * (long long)N + n;
                o[0] = v0[b];
                o[(long long)next * N] = v1[b];
            }
            continue;
        }
#pragma unroll
        for (int b = 0; b < 4; b++) {
            const bool live = gs0 + b < gcnt;
            *reinterpret_cast<ulonglong2*>(&tw[nrow][2 * b]) = make_ulonglong2(live ? v0[b] : 0ull, live ? v1[b] : 0ull);
        }
        __syncwarp();
        u64* dst = S + (((long long)tl * N + nblk_s[r]) * T.n + k) * spitch + gs0 * 2 + 2 * fp;
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const int rr = i * 8 + fr;
            const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(&tw[rr][2 * fp]);
            *reinterpret_cast<ulonglong2*>(dst + (long long)rr * rstride) = v;
        }
        __syncwarp();
    }
}

template <int ND>
static cudaError_t ks3_launch(u64* S, const KsTerms& T, const KsGroups& GR, int g0, int gcnt, int t0, int tcnt, int nq,
                              int next, int logn, int spitch, long long kds, long long kcs, const Limbs& ext,
                              const PrimeInfo* pr, const u64* pmod, const double2* fq, cudaStream_t st,
                              int nat_gtot = 0) {
    const size_t smem = ks3_smem_bytes<ND>();
    static unsigned long long cfg = 0;
    unsigned long long bit = 0;
    if (first_on_device(&cfg, &bit)) {
        cudaError_t ae = cudaSuccess;
        BCN_SMEM_ATTR(ae, (slot_major_ks3_kernel<ND>), (int)smem);
        if (ae != cudaSuccess) return ae;
        cfg |= bit;
    }
    const int nsplit = (gcnt + 31) / 32;
    dim3 grid((1 << logn) / 32, tcnt * nsplit, GR.n);
    slot_major_ks3_kernel<ND><<<grid, 256, smem, st>>>(S, T, GR, g0, gcnt, nsplit, t0, nq, next, logn, spitch, kds, kcs,
                                                       ext, pr, pmod, fq, nat_gtot);
    return launched();
}

// B'_k = sum_j sigma_k(U_j) (x) key_k,j + [c = 0] P sigma_k(c0) for <= 16 rotations k of ONE source, written in
// the natural layout out[k][G][2][next][N] (canonical): the source's U digits cross L2 once for all the rotations
// (bcn_rotate_hoisted_many).  Every T.src / T.U must be the same source; G in blocks of 64.
cudaError_t ks_inner_multi_op(u64* out, const KsTerms& T, int G, int nq, int next, int ndig, int logn, long long kds,
                              long long kcs, const Limbs& ext, const PrimeInfo* pr, const u64* pmod,
                              const double2* fq, cudaStream_t st) {
    if (!fq || ndig < 1 || ndig > 3 || T.n < 1 || T.n > 16) return cudaErrorInvalidValue;
    KsGroups GR;
    GR.n = 1;
    GR.start[0] = 0;
    GR.count[0] = (unsigned char)T.n;
    for (int g0 = 0; g0 < G; g0 += 64) {
        const int gcnt = G - g0 < 64 ? G - g0 : 64;
        cudaError_t e;
        switch (ndig) {
            case 1: e = ks3_launch<1>(out, T, GR, g0, gcnt, 0, next, nq, next, logn, 128, kds, kcs, ext, pr, pmod, fq, st, G); break;
            case 2: e = ks3_launch<2>(out, T, GR, g0, gcnt, 0, next, nq, next, logn, 128, kds, kcs, ext, pr, pmod, fq, st, G); break;
            default: e = ks3_launch<3>(out, T, GR, g0, gcnt, 0, next, nq, next, logn, 128, kds, kcs, ext, pr, pmod, fq, st, G);
        }
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t slot_major_ks_op(u64* S, const KsTerms& T, int g0, int gcnt, int t0, int tcnt, int nq, int next, int ndig,
                             int logn, int spitch, long long kds, long long kcs, const Limbs& ext, const PrimeInfo* pr,
                             const u64* pmod, cudaStream_t st, const double2* fq) {
    if (2 * gcnt > spitch || spitch > 128) return cudaErrorInvalidValue;
    if (ndig > 12) fq = nullptr;
    const int N = 1 << logn;
    static const bool shared_form = !(getenv("BCN_SMKS_SHARED") && getenv("BCN_SMKS_SHARED")[0] == '0');
    if (shared_form && fq && ndig >= 1 && ndig <= 3 && gcnt <= 64 && spitch >= 8 * ((gcnt + 3) / 4)) {
        // runs of consecutive terms over the same source (<= 16 per CTA)
        KsGroups GR;
        GR.n = 0;
        for (int k = 0; k < T.n;) {
            const u64* gu = T.g[k] == 1u ? nullptr : T.U[k];   // the run's ModUp (identity terms carry none)
            int c = 1;
            while (k + c < T.n && c < 16 && T.src[k + c] == T.src[k]) {
                if (T.g[k + c] != 1u) {
                    if (gu && T.U[k + c] != gu) break;
                    gu = T.U[k + c];
                }
                c++;
            }
            GR.start[GR.n] = (unsigned short)k;
            GR.count[GR.n] = (unsigned char)c;
            GR.n++;
            k += c;
        }
        switch (ndig) {
            case 1: return ks3_launch<1>(S, T, GR, g0, gcnt, t0, tcnt, nq, next, logn, spitch, kds, kcs, ext, pr, pmod, fq, st);
            case 2: return ks3_launch<2>(S, T, GR, g0, gcnt, t0, tcnt, nq, next, logn, spitch, kds, kcs, ext, pr, pmod, fq, st);
            default: return ks3_launch<3>(S, T, GR, g0, gcnt, t0, tcnt, nq, next, logn, spitch, kds, kcs, ext, pr, pmod, fq, st);
        }
    }
    dim3 grid(N / 32, tcnt, T.n);
    switch (ndig) {
#define BCN_SMK(D) case D: slot_major_ks_kernel<D><<<grid, 256, 0, st>>>(S, T, g0, gcnt, t0, nq, next, ndig, logn, \
                                                   spitch, kds, kcs, ext, pr, pmod, fq); break;
        BCN_SMK(1) BCN_SMK(2) BCN_SMK(3) BCN_SMK(4)
#undef BCN_SMK
        default:
            slot_major_ks_kernel<0><<<grid, 256, 0, st>>>(S, T, g0, gcnt, t0, nq, next, ndig, logn, spitch, kds, kcs, ext, pr,
                                                          pmod, fq);
    }
    return launched();
}

// -------------------------------------------------- slot-major transpose
// S[((tl * N + n) * K + k) * 64 + col] = ct_k[g0 + col/2][col%2][t0 + tl][n]
// for col < 2 * gcnt: every slot's K x 64 word matrix becomes one contiguous
// run, so the MAC kernel streams it instead of gathering 8-byte words.  One
// CTA = (k, limb, 32 coefficients): 64 coalesced 256-byte row reads, 32
// coalesced 512-byte row writes through a padded SMEM tile.
__global__ void __launch_bounds__(256) slot_major_kernel(u64* __restrict__ S, const MacImma m, int g0, int gcnt,
                                                         int t0, int nlimb, int logn, int spitch) {
    __shared__ u64 tile[128][33];
    const int N = 1 << logn;
    const long long LN = (long long)nlimb << logn;
    const int n0 = blockIdx.x * 32, tl = blockIdx.y, k = blockIdx.z;
    const int ncol = 2 * gcnt;
    const u64* src = m.ct[k] + (long long)(t0 + tl) * N + n0;
    for (int x = threadIdx.x; x < ncol * 32; x += blockDim.x) {
        const int col = x >> 5, nn = x & 31;
        tile[col][nn] = __ldg(src + (long long)(g0 + (col >> 1)) * 2 * LN + (col & 1) * LN + nn);
    }
    __syncthreads();
    u64* dst = S + (((long long)tl * N + n0) * m.n_terms + k) * spitch;
    const int lane = threadIdx.x & 31;
    for (int r = threadIdx.x >> 5; r < 32; r += blockDim.x >> 5)
        for (int col = lane; col < ncol; col += 32) dst[(long long)r * m.n_terms * spitch + col] = tile[col][r];
}

// ---------------------------------------------------------------- kernel
#define IM_BP 66          // B tile row pitch in words (2-way = conflict-optimal LDS.64)
#define IM_GC 64          // max slot-set columns per CTA (32 slot sets x 2 components)

#ifndef IM_ST
#define IM_ST 3           // pipeline stages
#endif

__device__ __forceinline__ void imma(int* d, u32 a0, u32 a1, u32 a2, u32 a3, u32 b0, u32 b1) {
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// bytes j of four k-consecutive words -> b[j] = {w0.bj, w1.bj, w2.bj, w3.bj}
__device__ __forceinline__ void transpose4(const u64 v[4], u32 b[8]) {
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

__global__ void __launch_bounds__(512, 1)
    mac_imma_kernel(u64* __restrict__ out, long long ostride, const MacImma m, const u8* __restrict__ planes,
                    const u64* __restrict__ S, int g0, int gcnt, int t0, int opad, int nch, int nlimb, int logn,
                    Limbs limbs, const PrimeInfo* __restrict__ pr, int accumulate) {
    extern __shared__ __align__(128) unsigned char im_smem[];
    const int N = 1 << logn;
    const long long LN = (long long)nlimb << logn;
    const long long bl = blockIdx.x;                     // slot within the limb block
    const long long b = bl + (long long)t0 * N;          // slot: t * N + n
    const int t = (int)(b >> logn), n = (int)(b & (N - 1));
    const int ngc = 2 * gcnt;                            // columns in this CTA (<= 64)
    const int o0 = blockIdx.z * 32;
    const int MT = (opad - o0) >= 32 ? 2 : 1;            // M-tiles of 16 outputs
    const int NT = (ngc + 7) >> 3;
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int warp = tid >> 5, lane = tid & 31, gq = lane >> 2, tq = lane & 3;
    const int mt = MT == 2 ? (warp & 1) : 0, nt = MT == 2 ? (warp >> 1) : warp;
    constexpr int ABYTES = 8 * 32 * 32;                  // 8 planes x 32 rows x 32 bytes
    constexpr int BBYTES = 32 * IM_BP * 8;
    constexpr int SBYTES = ABYTES + BBYTES;              // one pipeline stage
    const int arow = MT * 16;                            // A rows this CTA reads per plane
    const int lg_pieces = MT == 2 ? 6 : 5;               // log2(16-byte pieces per plane)
    const long long coff = (long long)t * N + n;
    const int nwarps = nthr >> 5;

    auto load_chunk = [&](int c, int stage) {
        u8* As = im_smem + stage * SBYTES;
        u64* Bs = reinterpret_cast<u64*>(As + ABYTES);
        // A: 8 planes x arow rows x 32 bytes, contiguous per plane
        const u8* asrc = planes + ((b * nch + c) * 8) * (long long)opad * 32 + (long long)o0 * 32;
        for (int x = tid; x < (8 << lg_pieces); x += nthr) {
            const int i = x >> lg_pieces, r = x & ((1 << lg_pieces) - 1);
            cp_async16(As + i * 32 * 32 + r * 16, asrc + (long long)i * opad * 32 + r * 16);
        }
        // B: rows k < n_terms of this slot's contiguous K x 64 block (A rows are zero past it)
        const int kmax = min(32, m.n_terms - c * 32);
        const u64* bsrc = S + (bl * m.n_terms + c * 32) * 64;
        const int pieces = ngc >> 1;                     // 16-byte pieces per row (<= 32)
        for (int kk = warp; kk < kmax; kk += nwarps)      // a row per warp, a piece per lane
            if (lane < pieces) cp_async16(Bs + kk * IM_BP + 2 * lane, bsrc + kk * 64 + 2 * lane);
        cp_async_commit();
    };
    (void)arow;
    (void)LN;

    int acc[15][4];
#pragma unroll
    for (int s = 0; s < 15; s++) acc[s][0] = acc[s][1] = acc[s][2] = acc[s][3] = 0;

    // IM_ST-stage cp.async ring: chunks c+1 .. c+IM_ST-1 load while c multiplies
    for (int c = 0; c < IM_ST - 1; c++) {
        if (c < nch) load_chunk(c, c);
        else cp_async_commit();
    }
    const bool active = warp < MT * NT;
    for (int c = 0; c < nch; c++) {
        const int stage = c % IM_ST;
        cp_async_wait<IM_ST - 2>();
        __syncthreads();
        if (active) {
            const u8* Ab = im_smem + stage * SBYTES;
            const u64* Bs = reinterpret_cast<const u64*>(Ab + ABYTES);
            const int col = nt * 8 + gq;
            u64 v[8];
#pragma unroll
            for (int r = 0; r < 4; r++) {
                v[r] = Bs[(4 * tq + r) * IM_BP + col];
                v[4 + r] = Bs[(16 + 4 * tq + r) * IM_BP + col];
            }
            u32 b0[8], b1[8];
            transpose4(v, b0);
            transpose4(v + 4, b1);
            const u8* As = Ab + mt * 512 + (gq * 4 + tq) * 16;   // fragment-ordered M-tile
#pragma unroll
            for (int i = 0; i < 8; i++) {
                const uint4 a = *reinterpret_cast<const uint4*>(As + i * 32 * 32);
#pragma unroll
                for (int j = 0; j < 8; j++) imma(acc[i + j], a.x, a.y, a.z, a.w, b0[j], b1[j]);
            }
        }
        __syncthreads();                                 // stage consumed
        if (c + IM_ST - 1 < nch) load_chunk(c + IM_ST - 1, (c + IM_ST - 1) % IM_ST);
        else cp_async_commit();
    }
    if (!active) return;

    // epilogue: value = sum_s 2^(8s) D_s = V_lo + 2^64 V_hi; result = REDC(value)
    const PrimeInfo& P = pr[limbs.prime[t]];
    const u64 q = P.q;
#pragma unroll
    for (int e = 0; e < 4; e++) {
        const int o = o0 + mt * 16 + gq + 8 * (e >> 1);
        const int col = nt * 8 + 2 * tq + (e & 1);
        if (o >= m.n_out || col >= ngc) continue;
        // partials D_s < 2^31: four consecutive ones fit a 64-bit word (< 2^56)
        auto quad = [&](int s0, int cnt) {
            u64 v = 0;
#pragma unroll
            for (int d = 0; d < 4; d++)
                if (d < cnt) v += (u64)(u32)acc[s0 + d][e] << (8 * d);
            return v;
        };
        const u64 A = quad(0, 4), B = quad(4, 4), C = quad(8, 4), D = quad(12, 3);
        // V_lo = A + 2^32 B (< 2^89), V_hi = C + 2^32 D (< 2^81)
        const u64 bl = B << 32, cl = C + (D << 32);
        const u64 lo = A + bl;
        u64 hi = (B >> 32) + (lo < A ? 1ull : 0ull);
        const u64 h = (D >> 32) + (cl < C ? 1ull : 0ull); // V_hi = 2^64 h + cl, h < 2^17
        u64 l = cl - umulhi(cl, P.pad[2]) * q;           // cl mod q
        l = l >= q ? l - q : l;
        const u64 hr = shoup(h, P.r1, P.r1_shoup, q);    // h 2^64 mod q
        const u64 xl = lo;
        const u64 xh = hi + l + hr;                      // < 2^25 + 2q < 3q
        const u64 mq = xl * P.qinv_neg;
        u64 r = xh + umulhi(mq, q) + (xl != 0ull ? 1ull : 0ull);   // < 4q
        r = csub(r, 2 * q);
        r = csub(r, q);
        const int g = g0 + (col >> 1), cc = col & 1;
        u64* po = out + (long long)o * ostride + (long long)g * 2 * LN + cc * LN + coff;
        if (accumulate) r = add_mod(r, *po, q);
        *po = r;
    }
}

size_t mac_imma_smem() { return IM_ST * (8 * 32 * 32 + 32 * IM_BP * 8); }

cudaError_t slot_major_op(u64* S, const MacImma& m, int g0, int gcnt, int t0, int tcnt, int nlimb, int logn,
                          cudaStream_t st, int spitch) {
    const int N = 1 << logn;
    if (2 * gcnt > spitch || spitch > 128) return cudaErrorInvalidValue;
    dim3 grid(N / 32, tcnt, m.n_terms);
    slot_major_kernel<<<grid, 256, 0, st>>>(S, m, g0, gcnt, t0, nlimb, logn, spitch);
    return launched();
}

cudaError_t mac_imma_op(u64* out, long long out_stride, const MacImma& m, const u8* planes, const u64* S, int g0,
                        int gcnt, int t0, int tcnt, int opad, int nlimb, int logn, const Limbs& limbs,
                        const PrimeInfo* pr, int accumulate, cudaStream_t st) {
    const int N = 1 << logn;
    if (gcnt <= 0 || m.n_terms <= 0 || m.n_out <= 0) return cudaSuccess;
    const int nch = (m.n_terms + 31) / 32;
    const size_t smem = mac_imma_smem();
    static unsigned long long smem_cfg = 0;
    unsigned long long smem_bit = 0;
    if (first_on_device(&smem_cfg, &smem_bit)) {
        cudaError_t ae = cudaSuccess;
        BCN_SMEM_ATTR(ae, (mac_imma_kernel), (int)smem);
        if (ae != cudaSuccess) return ae;
        smem_cfg |= smem_bit;
    }
    const int oblocks = (opad + 31) / 32;
    const int mt = opad >= 32 ? 2 : 1;
    const int threads = 32 * mt * ((2 * gcnt + 7) / 8);
    dim3 grid((unsigned)((long long)tcnt * N), 1, oblocks);
    mac_imma_kernel<<<grid, threads, smem, st>>>(out, out_stride, m, planes, S, g0, gcnt, t0, opad, nch, nlimb, logn,
                                                 limbs, pr, accumulate);
    return launched();
}

}  // namespace bcn
