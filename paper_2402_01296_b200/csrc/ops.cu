// ops.cu -- HBM-streaming RNS kernels: modular add/sub/mul (K3), fused
// ct x pt multiply-accumulate (K4), tensor square (K6), automorphism (K8),
// ModUp / inner-product / ModDown pieces of hybrid key switching (K7) and
// the rescale lift/combine (K5).  All are one pass over their operands with
// every output written once; constants (Shoup pairs, Montgomery base-
// conversion tables) are tiny and broadcast through L1.
#include "common.cuh"
#include "ops.cuh"

namespace bcn {

static inline int blocks_for(long long n, int tpb) {
    long long b = (n + tpb - 1) / tpb;
    return (int)(b > 2147483647LL ? 2147483647LL : b);
}

// --------------------------------------------------------------- binary
// out[p][t][n] = a[p][t][n] (op) b[p][t][n]; strides in words, 0 = broadcast.
template <int OP>
__global__ void binary_kernel(u64* __restrict__ out, long long os, const u64* __restrict__ a, long long as,
                              const u64* __restrict__ b, long long bs, int nlimb, int logn, Limbs limbs,
                              const PrimeInfo* __restrict__ pr, long long total) {
    // grid (N / blockDim, limb, poly): no per-element division
    const int N = 1 << logn;
    const int n = blockIdx.x * blockDim.x + threadIdx.x, t = blockIdx.y;
    const long long p = blockIdx.z;
    if (n < N) {
        const PrimeInfo& P = pr[limbs.prime[t]];
        const u64 x = a[p * as + (long long)t * N + n];
        const u64 y = b[p * bs + (long long)t * N + n];
        u64 r;
        if (OP == 0) r = add_mod(x, y, P.q);
        else if (OP == 1) r = sub_mod(x, y, P.q);
        else r = mont_mul(x, y, P.q, P.qinv_neg);   // y in Montgomery form
        out[p * os + (long long)t * N + n] = r;
    }
    (void)nlimb;
    (void)total;
}

cudaError_t binary_op(int op, u64* out, long long os, const u64* a, long long as, const u64* b, long long bs,
                      int npoly, int nlimb, int logn, const Limbs& limbs, const PrimeInfo* pr, cudaStream_t st) {
    long long total = (long long)npoly * nlimb << logn;
    if (total == 0) return cudaSuccess;
    if (npoly > 65535) return cudaErrorInvalidValue;
    const int N = 1 << logn, tpb = N < 256 ? N : 256;
    const dim3 nb(N / tpb, nlimb, npoly);
    if (op == 0) binary_kernel<0><<<nb, tpb, 0, st>>>(out, os, a, as, b, bs, nlimb, logn, limbs, pr, total);
    else if (op == 1) binary_kernel<1><<<nb, tpb, 0, st>>>(out, os, a, as, b, bs, nlimb, logn, limbs, pr, total);
    else binary_kernel<2><<<nb, tpb, 0, st>>>(out, os, a, as, b, bs, nlimb, logn, limbs, pr, total);
    return launched();
}

// out = to_mont(a) (in place allowed)
__global__ void to_mont_kernel(u64* out, const u64* a, int nlimb, int logn, Limbs limbs,
                               const PrimeInfo* __restrict__ pr, long long total) {
    const int N = 1 << logn;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int t = (int)((idx >> logn) % nlimb);
        (void)N;
        out[idx] = to_mont(a[idx], pr[limbs.prime[t]]);
    }
}

cudaError_t to_mont_op(u64* out, const u64* a, int npoly, int nlimb, int logn, const Limbs& limbs,
                       const PrimeInfo* pr, cudaStream_t st) {
    long long total = (long long)npoly * nlimb << logn;
    if (!total) return cudaSuccess;
    to_mont_kernel<<<blocks_for(total, 256), 256, 0, st>>>(out, a, nlimb, logn, limbs, pr, total);
    return launched();
}

// ------------------------------------------------------------------ MAC
// out[g] = sum_{t in group g} ct[t] (x) pt_mont[t]   (2 polys per ct)
// ct: [T][2][L][N] stride ct_stride; pt: [T][L][N] stride pt_stride;
// out: [G][2][L][N].  Lazy u128 accumulation, one REDC per output word.
__global__ void mac_kernel(u64* __restrict__ out, const u64* __restrict__ ct, long long ct_stride,
                           const u64* __restrict__ pt, long long pt_stride, int n_items, int group,
                           int nlimb, int logn, Limbs limbs, const PrimeInfo* __restrict__ pr) {
    const int N = 1 << logn;
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    const int t = blockIdx.y;
    const int gidx = blockIdx.z;
    const PrimeInfo& P = pr[limbs.prime[t]];
    const u64 q = P.q;
    Acc128 a0, a1;
    a0.zero(); a1.zero();
    const int start = gidx * group;
    const int end = min(start + group, n_items);
    for (int k = start; k < end; k++) {
        const u64 p = __ldg(pt + (long long)k * pt_stride + (long long)t * N + n);
        const u64* c = ct + (long long)k * ct_stride + (long long)t * N + n;
        a0.mac(__ldg(c), p, q);
        a1.mac(__ldg(c + (long long)nlimb * N), p, q);
    }
    u64* o = out + (long long)gidx * 2 * nlimb * N + (long long)t * N + n;
    o[0] = a0.reduce(q, P.qinv_neg);
    o[(long long)nlimb * N] = a1.reduce(q, P.qinv_neg);
}

cudaError_t mac_op(u64* out, const u64* ct, long long ct_stride, const u64* pt, long long pt_stride,
                   int n_items, int group, int nlimb, int logn, const Limbs& limbs, const PrimeInfo* pr,
                   cudaStream_t st) {
    const int N = 1 << logn;
    const int ngroups = (n_items + group - 1) / group;
    if (!ngroups) return cudaSuccess;
    int tpb = N < 256 ? N : 256;
    dim3 grid((N + tpb - 1) / tpb, nlimb, ngroups);
    mac_kernel<<<grid, tpb, 0, st>>>(out, ct, ct_stride, pt, pt_stride, n_items, group, nlimb, logn, limbs, pr);
    return launched();
}

// ------------------------------------------- linear combination MAC (K4)
// out[g][c] (+)= REDC( sum_t ct_t[g][c] * pt_t[g|0] ): the conv-tap / FC-
// diagonal sum of the ciphertext branch in one pass -- every rotated input
// and plaintext read once, u128 lazy accumulation, one REDC per word.
__global__ void __launch_bounds__(256) mac_terms_kernel(u64* __restrict__ out, const MacTerms terms, int nlimb,
                                                        int logn, Limbs limbs, const PrimeInfo* __restrict__ pr,
                                                        int accumulate, long long total) {
    // grid (N / blockDim, limb, slot set)
    const int N = 1 << logn;
    const long long LN = (long long)nlimb << logn;
    const int n = blockIdx.x * blockDim.x + threadIdx.x, t = blockIdx.y;
    const long long g = blockIdx.z;
    if (n < N) {
        const long long off = (long long)t * N + n;
        const PrimeInfo& P = pr[limbs.prime[t]];
        const u64 q = P.q;
        Acc4 a0, a1;
        a0.zero(); a1.zero();
        const long long cbase = g * 2 * LN + off;
        const long long pbase = g * LN + off;
        for (int k = 0; k < terms.n; k++) {
            const u64 p = __ldg(terms.pt[k] + (terms.pt_batched[k] ? pbase : off));
            const u64* c = terms.ct[k] + cbase;
            a0.mac(__ldg(c), p);
            a1.mac(__ldg(c + LN), p);
            if ((k & 31) == 31) { a0.fold_hi(q, P.pad[2]); a1.fold_hi(q, P.pad[2]); }
        }
        u64 r0 = a0.reduce(q, P.qinv_neg, P.pad[2]), r1 = a1.reduce(q, P.qinv_neg, P.pad[2]);
        u64* o = out + cbase;
        if (accumulate) {
            r0 = add_mod(r0, o[0], q);
            r1 = add_mod(r1, o[LN], q);
        }
        o[0] = r0;
        o[LN] = r1;
    }
    (void)total;
}

cudaError_t mac_terms_op(u64* out, const MacTerms& terms, int G, int nlimb, int logn, const Limbs& limbs,
                         const PrimeInfo* pr, int accumulate, cudaStream_t st) {
    long long total = (long long)G * nlimb << logn;
    if (!total || terms.n <= 0) return cudaSuccess;
    if (G > 65535) return cudaErrorInvalidValue;
    const int N = 1 << logn, tpb = N < 256 ? N : 256;
    mac_terms_kernel<<<dim3(N / tpb, nlimb, G), tpb, 0, st>>>(out, terms, nlimb, logn, limbs, pr, accumulate, total);
    return launched();
}

// ----------------------------------------- multi-output linear combination
// out[o][g][c][t][n] (+)= REDC(sum_k ct_k[g][c][t][n] * pt[o][k][t][n]).
// blockIdx.x = slot set g (fastest), so the G CTAs that multiply the same
// plaintext slice by different ciphertexts run back to back and the
// plaintexts come from L2; each ct word is loaded once per output tile.
template <int OT>
__global__ void __launch_bounds__(256, 2) mac_multi_kernel(u64* __restrict__ out, long long ostride, const MacMulti m,
                                                        int nlimb, int logn, Limbs limbs,
                                                        const PrimeInfo* __restrict__ pr, int accumulate) {
    const int N = 1 << logn;
    const long long LN = (long long)nlimb << logn;
    const long long g = blockIdx.x;
    const int n = blockIdx.y * blockDim.x + threadIdx.x;
    const int t = blockIdx.z;
    if (n >= N) return;
    const PrimeInfo& P = pr[limbs.prime[t]];
    const u64 q = P.q, qn = P.qinv_neg;
    const long long off = (long long)t * N + n;
    const long long cbase = g * 2 * LN + off;
    Acc128 a0[OT], a1[OT];
#pragma unroll
    for (int o = 0; o < OT; o++) { a0[o].zero(); a1[o].zero(); }
    // register double buffer: term k+1's words are in flight while term k multiplies
    u64 nc0 = __ldg(m.ct[0] + cbase), nc1 = __ldg(m.ct[0] + cbase + LN), np_[OT];
#pragma unroll
    for (int o = 0; o < OT; o++) np_[o] = o < m.n_out ? __ldg(m.pt[o][0] + off) : 0ull;
    for (int k = 0; k < m.n_terms; k++) {
        const u64 c0 = nc0, c1 = nc1;
        u64 p[OT];
#pragma unroll
        for (int o = 0; o < OT; o++) p[o] = np_[o];
        if (k + 1 < m.n_terms) {
            nc0 = __ldg(m.ct[k + 1] + cbase);
            nc1 = __ldg(m.ct[k + 1] + cbase + LN);
#pragma unroll
            for (int o = 0; o < OT; o++) np_[o] = o < m.n_out ? __ldg(m.pt[o][k + 1] + off) : 0ull;
        }
#pragma unroll
        for (int o = 0; o < OT; o++) {
            a0[o].mac_nr(c0, p[o]);
            a1[o].mac_nr(c1, p[o]);
        }
        if (k % 7 == 6) {
#pragma unroll
            for (int o = 0; o < OT; o++) { a0[o].fold(q); a1[o].fold(q); }
        }
    }
#pragma unroll
    for (int o = 0; o < OT; o++) {
        if (o >= m.n_out) break;
        a0[o].fold(q);
        a1[o].fold(q);
        u64* po = out + o * ostride + cbase;
        u64 r0 = a0[o].reduce(q, qn), r1 = a1[o].reduce(q, qn);
        if (accumulate) { r0 = add_mod(r0, po[0], q); r1 = add_mod(r1, po[LN], q); }
        po[0] = r0;
        po[LN] = r1;
    }
}

// Staged variant for N >= 128 (the production path).  CTA = (slot set g,
// 128-coefficient block, limb t), 256 threads: threads 0-127 own component 0,
// 128-255 component 1, one coefficient each, OT output accumulators.  Per
// term k, thread 0 issues 1-KiB bulk async copies (TMA engine) of the two
// ct slices and the OT plaintext slices into an S-deep shared-memory ring
// (completion on one mbarrier per stage), so the loads of term k+S overlap
// the multiplies of term k without holding prefetch registers.  The MAC is
// exact u128 (Acc4: 4 IMAD.WIDE + carry add, no per-term reduction); the high
// half is Barrett-folded every 32 terms and one REDC finishes each output.
#define MM_NB 128
template <int OT, int S, bool FULL>
__global__ void __launch_bounds__(2 * MM_NB, 2)
    mac_multi_tma_kernel(u64* __restrict__ out, long long ostride, const MacMulti m, int nlimb, int logn, Limbs limbs,
                         const PrimeInfo* __restrict__ pr, int accumulate) {
    extern __shared__ __align__(128) u64 ring[];     // [S][2 + OT][MM_NB]
    __shared__ __align__(8) u64 full[S];
    const int N = 1 << logn;
    const long long LN = (long long)nlimb << logn;
    const long long g = blockIdx.x;
    const int n0 = blockIdx.y * MM_NB;
    const int t = blockIdx.z;
    const int tid = threadIdx.x, comp = tid / MM_NB, n = tid % MM_NB;
    const int n_out = m.n_out, nt = m.n_terms;
    const long long off = (long long)t * N + n0;
    const long long cbase = g * 2 * LN + off;
    constexpr int SW = (2 + OT) * MM_NB;             // words per stage
    const u32 bytes = (u32)((2 + n_out) * MM_NB * sizeof(u64));
    if (tid == 0) {
        for (int s = 0; s < S; s++) mbar_init(&full[s], 1);
        fence_barrier_init();
    }
    __syncthreads();
    // the 2 + n_out copies of a stage are spread over the 8 warps (lane 0 of
    // warp w issues copies w, w + 8, ...); warp 0 also arms the barrier.  A
    // copy may land before the arm: tx-count may dip below zero, and the
    // phase cannot complete before warp 0's arrival.
    const int warp = tid >> 5;
    auto issue = [&](int k) {
        const int s = k % S;
        u64* dst = ring + s * SW;
        if (warp == 0) mbar_expect_tx(&full[s], bytes);
        for (int c = warp; c < 2 + n_out; c += 2 * MM_NB / 32) {
            const u64* src = c < 2 ? m.ct[k] + cbase + c * LN : m.pt[c - 2][k] + off;
            bulk_load(dst + c * MM_NB, src, MM_NB * 8, &full[s]);
        }
    };
    if ((tid & 31) == 0)
        for (int k = 0; k < S && k < nt; k++) issue(k);
    const PrimeInfo& P = pr[limbs.prime[t]];
    Acc4 acc[OT];
#pragma unroll
    for (int o = 0; o < OT; o++) acc[o].zero();
    for (int k = 0; k < nt; k++) {
        const int s = k % S;
        mbar_wait(&full[s], (u32)((k / S) & 1));
        const u64* st = ring + s * SW;
        const u64 c = st[comp * MM_NB + n];
        const u32 c0 = (u32)c, c1 = (u32)(c >> 32);
#pragma unroll
        for (int o = 0; o < OT; o++) {
            if (FULL || o < n_out) {
                const u64 p = st[(2 + o) * MM_NB + n];
                acc[o].mac(c0, c1, (u32)p, (u32)(p >> 32));
            }
        }
        if ((k & 31) == 31) {
#pragma unroll
            for (int o = 0; o < OT; o++) acc[o].fold_hi(P.q, P.pad[2]);
        }
        __syncthreads();                             // stage s fully consumed
        if ((tid & 31) == 0 && k + S < nt) issue(k + S);
    }
    const u64 q = P.q;
    u64* po = out + cbase + (long long)comp * LN + n;
#pragma unroll
    for (int o = 0; o < OT; o++) {
        if (FULL || o < n_out) {
            u64 r = acc[o].reduce(q, P.qinv_neg, P.pad[2]);
            if (accumulate) r = add_mod(r, po[o * ostride], q);
            po[o * ostride] = r;
        }
    }
}

template <int OT, int S, bool FULL>
static cudaError_t launch_mac_multi_tma(u64* out, long long out_stride, const MacMulti& m, int G, int nlimb, int logn,
                                        const Limbs& limbs, const PrimeInfo* pr, int accumulate, cudaStream_t st) {
    const size_t smem = (size_t)S * (2 + OT) * MM_NB * sizeof(u64);
    static unsigned long long smem_cfg = 0;
    unsigned long long smem_bit = 0;
    if (first_on_device(&smem_cfg, &smem_bit)) {
        cudaError_t ae = cudaSuccess;
        BCN_SMEM_ATTR(ae, (mac_multi_tma_kernel<OT, S, FULL>), (int)smem);
        if (ae != cudaSuccess) return ae;
        smem_cfg |= smem_bit;
    }
    dim3 grid(G, (1 << logn) / MM_NB, nlimb);
    mac_multi_tma_kernel<OT, S, FULL>
        <<<grid, 2 * MM_NB, smem, st>>>(out, out_stride, m, nlimb, logn, limbs, pr, accumulate);
    return launched();
}

cudaError_t mac_multi_op(u64* out, long long out_stride, const MacMulti& m, int G, int nlimb, int logn,
                         const Limbs& limbs, const PrimeInfo* pr, int accumulate, cudaStream_t st) {
    const int N = 1 << logn;
    if (G <= 0 || m.n_terms <= 0 || m.n_out <= 0) return cudaSuccess;
    if (N >= MM_NB) {
        const int no = m.n_out;
        if (no == BCN_MAC_OUT)
            return launch_mac_multi_tma<BCN_MAC_OUT, 6, true>(out, out_stride, m, G, nlimb, logn, limbs, pr, accumulate, st);
        if (no == 8) return launch_mac_multi_tma<8, 8, true>(out, out_stride, m, G, nlimb, logn, limbs, pr, accumulate, st);
        if (no < 8) return launch_mac_multi_tma<8, 8, false>(out, out_stride, m, G, nlimb, logn, limbs, pr, accumulate, st);
        return launch_mac_multi_tma<BCN_MAC_OUT, 6, false>(out, out_stride, m, G, nlimb, logn, limbs, pr, accumulate, st);
    }
    const int tpb = N < 256 ? N : 256;
    dim3 grid(G, (N + tpb - 1) / tpb, nlimb);
    if (m.n_out <= 4) mac_multi_kernel<4><<<grid, tpb, 0, st>>>(out, out_stride, m, nlimb, logn, limbs, pr, accumulate);
    else mac_multi_kernel<BCN_MAC_OUT><<<grid, tpb, 0, st>>>(out, out_stride, m, nlimb, logn, limbs, pr, accumulate);
    return launched();
}

// ---------------------------------------------------------- tensor (K6)
// d0 = a0 b0, d1 = a0 b1 + a1 b0, d2 = a1 b1 for G ciphertext pairs.
// a, b: [G][2][L][N] with strides; d: [G][3][L][N]
__global__ void tensor_kernel(u64* __restrict__ d, const u64* __restrict__ a, long long as,
                              const u64* __restrict__ b, long long bs, int nlimb, int logn, Limbs limbs,
                              const PrimeInfo* __restrict__ pr, long long total, const double2* __restrict__ fq) {
    // grid (N / blockDim, limb, slot set)
    const int N = 1 << logn;
    const long long LN = (long long)nlimb * N;
    const int n = blockIdx.x * blockDim.x + threadIdx.x, t = blockIdx.y;
    const long long g = blockIdx.z;
    if (n < N) {
        const long long off = (long long)t * N + n;
        const PrimeInfo& P = pr[limbs.prime[t]];
        const u64 q = P.q;
        u64* o = d + g * 3 * LN + off;
        if (fq) {                                    // FP64 pipe: plain products, exact two-product fmm
            const double2 f = fq[limbs.prime[t]];
            const double a0 = fload(a[g * as + off]), a1 = fload(a[g * as + LN + off]);
            const double b0 = fload(b[g * bs + off]), b1 = fload(b[g * bs + LN + off]);
            const double b0q = __dmul_rn(b0, f.y), b1q = __dmul_rn(b1, f.y);   // |a (b/q - bq)| <= 0.25
            o[0] = fcanon_small(fmm(a0, b0, b0q, f.x), f.x);
            o[LN] = fcanon(__dadd_rn(fmm(a0, b1, b1q, f.x), fmm(a1, b0, b0q, f.x)), f.y, f.x);
            o[2 * LN] = fcanon_small(fmm(a1, b1, b1q, f.x), f.x);
            return;
        }
        const u64 a0 = a[g * as + off], a1 = a[g * as + LN + off];
        const u64 b0 = to_mont(b[g * bs + off], P), b1 = to_mont(b[g * bs + LN + off], P);
        o[0] = mont_mul(a0, b0, q, P.qinv_neg);
        Acc128 acc; acc.zero();
        acc.mac(a0, b1, q);
        acc.mac(a1, b0, q);
        o[LN] = acc.reduce(q, P.qinv_neg);
        o[2 * LN] = mont_mul(a1, b1, q, P.qinv_neg);
    }
    (void)total;
}

cudaError_t tensor_op(u64* d, const u64* a, long long as, const u64* b, long long bs, int G, int nlimb,
                      int logn, const Limbs& limbs, const PrimeInfo* pr, cudaStream_t st, const double2* fq) {
    long long total = (long long)G * nlimb << logn;
    if (!total) return cudaSuccess;
    if (G > 65535) return cudaErrorInvalidValue;
    const int N = 1 << logn, tpb = N < 256 ? N : 256;
    tensor_kernel<<<dim3(N / tpb, nlimb, G), tpb, 0, st>>>(d, a, as, b, bs, nlimb, logn, limbs, pr, total, fq);
    return launched();
}

// ----------------------------------------------------- automorphism (K8)
__global__ void automorph_kernel(u64* __restrict__ out, long long os, const u64* __restrict__ in, long long is,
                                 int nlimb, int logn, u32 g, long long total) {
    const int N = 1 << logn;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int n = (int)(idx & (N - 1));
        const long long rest = idx >> logn;
        const int t = (int)(rest % nlimb);
        const long long p = rest / nlimb;
        out[p * os + (long long)t * N + n] = in[p * is + (long long)t * N + automorph_src(n, g, logn)];
    }
}

cudaError_t automorph_op(u64* out, long long os, const u64* in, long long is, int npoly, int nlimb, int logn,
                         u32 g, cudaStream_t st) {
    long long total = (long long)npoly * nlimb << logn;
    if (!total) return cudaSuccess;
    automorph_kernel<<<blocks_for(total, 256), 256, 0, st>>>(out, os, in, is, nlimb, logn, g, total);
    return launched();
}

// ---------------------------------------------------------- ModUp (K7)
// For digit j (grid.z) of poly p (grid.y): y_i = [x_i * hatinv_i]_{q_i} for
// the digit's limbs, then U[p][j][t] = REDC(sum_i y_i * hat_m[i][t]) for
// every extended limb t outside the digit (coefficient domain; NTT'd by the
// caller), and U[p][j][t] = x_ntt[t] (already NTT domain) inside it.
template <int A>     // A >= digit size, compile time: y[] stays in registers (0: runtime, local array)
__global__ void modup_kernel(u64* __restrict__ U, const u64* __restrict__ xc, long long xc_stride,
                             const u64* __restrict__ xn, long long x_stride, int nq, int next, int alpha, int ndig,
                             int logn,
                             Limbs ext, const PrimeInfo* __restrict__ pr, const ConvTable* __restrict__ tab,
                             const __grid_constant__ FConvSet fc, int use_fp) {
    constexpr int YA = A > 0 ? A : BCN_MAX_ALPHA;
    const int N = 1 << logn;
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    const long long p = blockIdx.y;
    const int j = blockIdx.z;
    const ConvTable& T = tab[j];
    const int i0 = j * alpha;
    const int na = T.n_src;
    u64 y[YA];
    const u64* xcp = xc + p * xc_stride + n;
    const u64* xnp = xn + p * x_stride + n;
    u64* Up = U + (p * ndig + j) * (long long)next * N + n;
#pragma unroll
    for (int i = 0; i < YA; i++) {
        if (i < na) {
            const PrimeInfo& P = pr[ext.prime[i0 + i]];
            y[i] = shoup(__ldg(xcp + (long long)(i0 + i) * N), T.hatinv[i], T.hatinv_p[i], P.q);
            Up[(long long)(i0 + i) * N] = __ldg(xnp + (long long)(i0 + i) * N);
        } else {
            y[i] = 0ull;
        }
    }
    if (use_fp) {                                      // FP64 pipe (every basis prime in (2^49, 2^50))
        double yd[YA];
#pragma unroll
        for (int i = 0; i < YA; i++) yd[i] = fload(y[i]);
        const FConv& F = fc.d[j];
        for (int t = 0; t < next; t++) {
            if (t >= i0 && t < i0 + na) continue;
            const double2 f = F.fq[t];
            double acc = 0.0;
#pragma unroll
            for (int i = 0; i < YA; i++)
                if (i < na) acc = __dadd_rn(acc, fmm(yd[i], F.h[i][t].x, F.h[i][t].y, f.x));
            Up[(long long)t * N] = fcanon(acc, f.y, f.x);
        }
        return;
    }
    for (int t = 0; t < next; t++) {
        if (t >= i0 && t < i0 + na) continue;
        const PrimeInfo& P = pr[ext.prime[t]];
        Acc4 acc; acc.zero();                          // na <= 16 products
#pragma unroll
        for (int i = 0; i < YA; i++)
            if (i < na) acc.mac(y[i], T.hat_m[i * BCN_MAX_LIMBS + t]);
        Up[(long long)t * N] = acc.reduce(P.q, P.qinv_neg, P.pad[2]);
    }
    (void)nq;
}

// FP64 form: two coefficients per thread (n, n + blockDim) share every
// constant-bank load of the conversion table (the kernel is issue-bound)
template <int A>
__global__ void modup_fp_kernel(u64* __restrict__ U, const u64* __restrict__ xc, long long xc_stride,
                                const u64* __restrict__ xn, long long x_stride, int next, int alpha, int ndig, int logn,
                                Limbs ext, const PrimeInfo* __restrict__ pr, const ConvTable* __restrict__ tab,
                                const __grid_constant__ FConvSet fc) {
    constexpr int YA = A;
    const int N = 1 << logn;
    const int n = blockIdx.x * 2 * blockDim.x + threadIdx.x;   // and n + blockDim.x (N >= 2 blockDim)
    const long long p = blockIdx.y;
    const int j = blockIdx.z;
    const ConvTable& T = tab[j];
    const int i0 = j * alpha;
    const int na = T.n_src;
    const u64* xcp = xc + p * xc_stride + n;
    const u64* xnp = xn + p * x_stride + n;
    u64* Up = U + (p * ndig + j) * (long long)next * N + n;
    const int h = blockDim.x;
    double y0[YA], y1[YA];
#pragma unroll
    for (int i = 0; i < YA; i++) {
        if (i < na) {
            const PrimeInfo& P = pr[ext.prime[i0 + i]];
            const long long o = (long long)(i0 + i) * N;
            y0[i] = fload(shoup(__ldg(xcp + o), T.hatinv[i], T.hatinv_p[i], P.q));
            y1[i] = fload(shoup(__ldg(xcp + o + h), T.hatinv[i], T.hatinv_p[i], P.q));
            Up[o] = __ldg(xnp + o);
            Up[o + h] = __ldg(xnp + o + h);
        } else {
            y0[i] = y1[i] = 0.0;
        }
    }
    const FConv& F = fc.d[j];
    for (int t = 0; t < next; t++) {
        if (t >= i0 && t < i0 + na) continue;
        const double2 f = F.fq[t];
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int i = 0; i < YA; i++)
            if (i < na) {
                const double2 hh = F.h[i][t];
                a0 = __dadd_rn(a0, fmm(y0[i], hh.x, hh.y, f.x));
                a1 = __dadd_rn(a1, fmm(y1[i], hh.x, hh.y, f.x));
            }
        Up[(long long)t * N] = fcanon(a0, f.y, f.x);
        Up[(long long)t * N + h] = fcanon(a1, f.y, f.x);
    }
}

cudaError_t modup_op(u64* U, const u64* xc, long long xc_stride, const u64* xn, long long x_stride, int npoly, int nq,
                     int next, int alpha, int ndig, int logn, const Limbs& ext, const PrimeInfo* pr,
                     const ConvTable* tab, cudaStream_t st, const FConvSet* fcp) {
    const int N = 1 << logn;
    int tpb = N < 256 ? N : 256;
    dim3 grid((N + tpb - 1) / tpb, npoly, ndig);
    static FConvSet none;
    const int use_fp = fcp && alpha <= BCN_FC_SRC && next <= BCN_FC_TGT && ndig <= 3;
    const FConvSet& fc = use_fp ? *fcp : none;
    if (use_fp && N >= 512 && alpha >= 1) {
        const dim3 g2(N / 512, npoly, ndig);
        switch (alpha) {
#define BCN_MF(AA) case AA: modup_fp_kernel<AA><<<g2, 256, 0, st>>>(U, xc, xc_stride, xn, x_stride, next, alpha, ndig, \
                                                                    logn, ext, pr, tab, *fcp); return launched();
            BCN_MF(1) BCN_MF(2) BCN_MF(3) BCN_MF(4) BCN_MF(5) BCN_MF(6) BCN_MF(7) BCN_MF(8)
#undef BCN_MF
            default: break;
        }
    }
    switch (alpha) {
#define BCN_MU(AA) case AA: modup_kernel<AA><<<grid, tpb, 0, st>>>(U, xc, xc_stride, xn, x_stride, nq, next, alpha, \
                                                                  ndig, logn, ext, pr, tab, fc, use_fp); break;
        BCN_MU(1) BCN_MU(2) BCN_MU(3) BCN_MU(4) BCN_MU(5) BCN_MU(6) BCN_MU(7) BCN_MU(8)
#undef BCN_MU
        default:
            modup_kernel<0><<<grid, tpb, 0, st>>>(U, xc, xc_stride, xn, x_stride, nq, next, alpha, ndig, logn, ext, pr,
                                                  tab, fc, 0);
    }
    return launched();
}

// ------------------------------------------- key inner product (K7, K8)
// A[p][c][t][n] = REDC( sum_j U[p][j][t][perm_g(n)] * key[j][c][kt(t)][n] )
// One CTA = one aligned block of BLK output positions of one limb and poly.
// Under X -> X^g an aligned block of the bit-reversed NTT domain is the
// image of one aligned source block, so the gather is staged through smem
// with coalesced loads.
template <int BLK>
__global__ void __launch_bounds__(256) inner_kernel(u64* __restrict__ A, const u64* __restrict__ U, int next,
                                                    int ndig, int logn, u32 g, const u64* __restrict__ key,
                                                    long long key_digit_stride, long long key_comp_stride,
                                                    Limbs ext, Limbs keyl, const PrimeInfo* __restrict__ pr, int t0) {
    extern __shared__ u64 sm[];
    const int N = 1 << logn;
    const int logb = __ffs(BLK) - 1;
    const int blk = blockIdx.x;
    const int t = t0 + blockIdx.y;
    const long long p = blockIdx.z;
    const PrimeInfo& P = pr[ext.prime[t]];
    const u64 q = P.q;
    const int dst0 = blk * BLK;
    const int src_blk = (g == 1u) ? blk : (int)(automorph_src((u32)dst0, g, logn) >> logb);
    for (int j = 0; j < ndig; j++) {
        const u64* src = U + ((p * ndig + j) * (long long)next + t) * N + (long long)src_blk * BLK;
        for (int i = threadIdx.x; i < BLK; i += blockDim.x) sm[j * BLK + i] = src[i];
    }
    __syncthreads();
    const int kt = keyl.prime[t];
    for (int i = threadIdx.x; i < BLK; i += blockDim.x) {
        const int n = dst0 + i;
        const int s = (g == 1u) ? i : (int)(automorph_src((u32)n, g, logn) & (BLK - 1));
        Acc4 a0, a1;                                   // ndig <= 32 products
        a0.zero(); a1.zero();
        for (int j = 0; j < ndig; j++) {
            const u64 u = sm[j * BLK + s];
            const u64* kp = key + j * key_digit_stride + (long long)kt * N + n;
            a0.mac(u, __ldg(kp));
            a1.mac(u, __ldg(kp + key_comp_stride));
        }
        u64* o = A + (p * 2 * next + t) * (long long)N + n;
        o[0] = a0.reduce(q, P.qinv_neg, P.pad[2]);
        o[(long long)next * N] = a1.reduce(q, P.qinv_neg, P.pad[2]);
    }
}

// inner_fp: the key-switch inner product on the FP64 pipe (basis primes below
// 2^50): a thread owns (coefficient, limb) for SS polynomials' worth of slot
// sets, the 2 ND key words are converted to {k, k/q} doubles once, the SS x ND
// digit words are loaded together (under X -> X^g the gather index is computed
// once), and each product is one fmm.  ~65 instead of ~120 instructions per
// output pair at ND = 3; the integer form re-read the key words per slot set.
template <int ND>
__global__ void __launch_bounds__(256, 3) inner_fp_kernel(u64* __restrict__ A, const u64* __restrict__ U, int npoly,
                                                          int next, int logn, u32 g, const u64* __restrict__ key,
                                                          long long kds, long long kcs, Limbs ext, Limbs keyl,
                                                          const PrimeInfo* __restrict__ pr,
                                                          const double2* __restrict__ fq, int t0) {
    constexpr int SS = 4;
    const int N = 1 << logn;
    const int n = blockIdx.x * 256 + threadIdx.x;
    const int t = t0 + blockIdx.y;
    const long long p0 = (long long)blockIdx.z * SS;
    const int kt = keyl.prime[t];
    const PrimeInfo& P = pr[ext.prime[t]];
    const u64 q = P.q;
    const double2 f = fq[ext.prime[t]];
    const int sn = g == 1u ? n : (int)automorph_src((u32)n, g, logn);
    int live = npoly - (int)p0;
    live = live > SS ? SS : live;
    const long long dstr = (long long)next * N, ustep = (long long)ND * dstr;
    const u64* Up = U + (p0 * ND * next + t) * (long long)N + sn;
    u64 uw[SS][ND];
#pragma unroll
    for (int s = 0; s < SS; s++) {
        const long long so = s < live ? s : 0;
#pragma unroll
        for (int j = 0; j < ND; j++) uw[s][j] = __ldg(Up + so * ustep + j * dstr);
    }
    double kd[ND], kq[ND], kd1[ND], kq1[ND];
    const u64* kp = key + (long long)kt * N + n;
#pragma unroll
    for (int j = 0; j < ND; j++) {
        kd[j] = fload(redc(0ull, __ldg(kp + j * kds), q, P.qinv_neg));
        kq[j] = __dmul_rn(kd[j], f.y);
        kd1[j] = fload(redc(0ull, __ldg(kp + j * kds + kcs), q, P.qinv_neg));
        kq1[j] = __dmul_rn(kd1[j], f.y);
    }
#pragma unroll
    for (int s = 0; s < SS; s++) {
        if (s >= live) break;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int j = 0; j < ND; j++) {
            const double ud = fload(uw[s][j]);
            a0 = __dadd_rn(a0, fmm(ud, kd[j], kq[j], f.x));
            a1 = __dadd_rn(a1, fmm(ud, kd1[j], kq1[j], f.x));
        }
        u64* o = A + ((p0 + s) * 2 * next + t) * (long long)N + n;
        o[0] = fcanon(a0, f.y, f.x);
        o[(long long)next * N] = fcanon(a1, f.y, f.x);
    }
}

cudaError_t inner_op(u64* A, const u64* U, int npoly, int next, int ndig, int logn, u32 g, const u64* key,
                     long long key_digit_stride, long long key_comp_stride, const Limbs& ext, const Limbs& keyl,
                     const PrimeInfo* pr, cudaStream_t st, int t0, int tcnt, const double2* fq) {
    const int N = 1 << logn;
    if (tcnt < 0) tcnt = next - t0;
    if (tcnt <= 0) return cudaSuccess;
    static const bool fp_off = getenv("BCN_INNER_FP64") && getenv("BCN_INNER_FP64")[0] == '0';
    if (fq && !fp_off && N >= 256 && ndig >= 1 && ndig <= 4) {
        dim3 grid(N / 256, tcnt, (npoly + 3) / 4);
        switch (ndig) {
#define BCN_IFP(D) case D: inner_fp_kernel<D><<<grid, 256, 0, st>>>(A, U, npoly, next, logn, g, key, key_digit_stride, \
                                                                  key_comp_stride, ext, keyl, pr, fq, t0); break;
            BCN_IFP(1) BCN_IFP(2) BCN_IFP(3) BCN_IFP(4)
#undef BCN_IFP
        }
        return launched();
    }
    if (N >= 1024) {
        constexpr int BLK = 1024;
        size_t smem = (size_t)ndig * BLK * sizeof(u64);
        static unsigned long long smem_cfg = 0;
    unsigned long long smem_bit = 0;
    if (first_on_device(&smem_cfg, &smem_bit)) {
        cudaError_t ae = cudaSuccess;
        BCN_SMEM_ATTR(ae, (inner_kernel<BLK>), 200 * 1024);
        if (ae != cudaSuccess) return ae;
        smem_cfg |= smem_bit;
    }
        dim3 grid(N / BLK, tcnt, npoly);
        inner_kernel<BLK><<<grid, 256, smem, st>>>(A, U, next, ndig, logn, g, key, key_digit_stride,
                                                   key_comp_stride, ext, keyl, pr, t0);
    } else {
        // small rings: one block covers the whole polynomial
        size_t smem = (size_t)ndig * N * sizeof(u64);
        dim3 grid(1, tcnt, npoly);
        switch (N) {
#define BCN_SMALL(NN) case NN: inner_kernel<NN><<<grid, 256, smem, st>>>(A, U, next, ndig, logn, g, key, \
                        key_digit_stride, key_comp_stride, ext, keyl, pr, t0); break;
            BCN_SMALL(8) BCN_SMALL(16) BCN_SMALL(32) BCN_SMALL(64) BCN_SMALL(128) BCN_SMALL(256) BCN_SMALL(512)
#undef BCN_SMALL
            default: return cudaErrorInvalidValue;
        }
    }
    return launched();
}

// ---------------------------------------------------------------- plaintext-branch conv (float64)
// The plaintext branch's 3x3 convolutions (layers.py:329-346) over the whole batch: cuDNN's float64
// implicit-GEMM takes 2.5-3.1 ms per layer for 4,096 32x32 images; the direct form -- a thread per
// output pixel with all (<= 32) output channels in registers, the weights in shared memory -- is
// bound by the 0.5 GB it writes.  x [B][C][H][W], w [O][C][kh][kw], out [B][O][OH][OW].
template <int OB>
__global__ void __launch_bounds__(128) plain_conv_kernel(const double* __restrict__ x, const double* __restrict__ w,
                                                         const double* __restrict__ b, double* __restrict__ out,
                                                         int B, int C, int H, int W, int O, int kh, int kw, int sh,
                                                         int sw, int ph, int pw, int OH, int OW) {
    extern __shared__ double wsm[];                         // [C kh kw][OB] of this output block
    const int o0 = blockIdx.y * OB;
    const int K = C * kh * kw;
    for (int i = threadIdx.x; i < K * OB; i += blockDim.x) {
        const int k = i / OB, o = i - k * OB;
        wsm[i] = o0 + o < O ? w[(long long)(o0 + o) * K + k] : 0.0;
    }
    __syncthreads();
    const long long pix = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long npix = (long long)B * OH * OW;
    if (pix >= npix) return;
    const int ow = (int)(pix % OW), oh = (int)((pix / OW) % OH);
    const long long bi = pix / ((long long)OW * OH);
    double acc[OB];
#pragma unroll
    for (int o = 0; o < OB; o++) acc[o] = (b && o0 + o < O) ? b[o0 + o] : 0.0;
    const double* xb = x + bi * C * H * W;
    for (int c = 0; c < C; c++)
        for (int di = 0; di < kh; di++) {
            const int ih = oh * sh - ph + di;
            if (ih < 0 || ih >= H) continue;
            for (int dj = 0; dj < kw; dj++) {
                const int iw = ow * sw - pw + dj;
                if (iw < 0 || iw >= W) continue;
                const double v = __ldg(xb + ((long long)c * H + ih) * W + iw);
                const double* wk = wsm + ((c * kh + di) * kw + dj) * OB;
#pragma unroll
                for (int o = 0; o < OB; o++) acc[o] = __fma_rn(v, wk[o], acc[o]);
            }
        }
    double* ob = out + (bi * O + o0) * OH * OW + (long long)oh * OW + ow;
#pragma unroll
    for (int o = 0; o < OB; o++)
        if (o0 + o < O) ob[(long long)o * OH * OW] = acc[o];
}

cudaError_t plain_conv_op(const double* x, const double* w, const double* b, double* out, int B, int C, int H, int W,
                          int O, int kh, int kw, int sh, int sw, int ph, int pw, cudaStream_t st) {
    const int OH = (H + 2 * ph - kh) / sh + 1, OW = (W + 2 * pw - kw) / sw + 1;
    if (OH <= 0 || OW <= 0 || B <= 0) return cudaErrorInvalidValue;
    constexpr int OB = 16;
    const size_t smem = (size_t)C * kh * kw * OB * sizeof(double);
    if (smem > 48 * 1024) return cudaErrorInvalidValue;
    const long long npix = (long long)B * OH * OW;
    dim3 grid((unsigned)((npix + 127) / 128), (O + OB - 1) / OB);
    plain_conv_kernel<OB><<<grid, 128, smem, st>>>(x, w, b, out, B, C, H, W, O, kh, kw, sh, sw, ph, pw, OH, OW);
    return launched();
}

// ------------------------------- lazy-ModDown rotation sum (K7 + K4 + K8)
// For every output word (g, ext limb t, n) and every term k:
//   a_c = REDC( sum_j sigma_gk(U_k,j)[n] * key_k[j][c][t][n] )      (c = 0, 1)
//   B_c += a_c * pt_k[t][n],   C0 += sigma_gk(c0_k)[n] * pt_k[t][n]  (t <= l)
// The ModDown of B happens ONCE for the whole sum (caller), instead of once
// per rotation.  One CTA = one aligned source/destination block of BLK words
// of one limb of one slot set; blockIdx.x is the slot set, so the G CTAs that
// read the same key slice run back to back and share it through L2.
template <int BLK>
__global__ void __launch_bounds__(BLK < 1024 ? BLK : 1024) rotsum_kernel(
        u64* __restrict__ B, u64* __restrict__ C0, const RotTerms T, long long c0_gstride, int nq, int next,
        int ndig, int logn, long long kds, long long kcs, Limbs ext, const PrimeInfo* __restrict__ pr,
        int acc_flags, long long c0_ostride) {
    const int accumulate = acc_flags & 1;             // add onto B
    const int c0_acc = (acc_flags >> 1) & 1;          // add onto C0
    // one thread per output word; term k+1's staging words, key words and
    // multiplier are loaded into registers while term k is being multiplied
    constexpr int MAXD = 3;
    extern __shared__ u64 sm[];
    const int N = 1 << logn;
    const int logb = __ffs(BLK) - 1;
    const long long p = blockIdx.x;
    const int blk = blockIdx.y;
    const int t = blockIdx.z;
    const int kt = ext.prime[t];
    const PrimeInfo& P = pr[kt];
    const u64 q = P.q, qn = P.qinv_neg, one_m = P.r1;
    const bool has_c0 = t < nq;
    const int dst0 = blk * BLK;
    const int tid = threadIdx.x;
    const int n = dst0 + tid;
    const int nd = ndig < MAXD ? ndig : MAXD;
    const u64 inv1 = P.pad[2];
    Acc4 b0, b1, cc;
    b0.zero(); b1.zero(); cc.zero();
    // loop-invariant offsets (words): only the term's base pointers and its
    // source block change from term to term
    // (32-bit: every operand of one launch is < 2^32 words, checked by the launcher)
    const u32 dstr = (u32)next * (u32)N;                                // digit stride of U
    const u32 uoff = (((u32)p * ndig) * (u32)next + t) * (u32)N + tid;
    const u32 coff = (u32)(p * c0_gstride) + (u32)t * N + tid;
    const u32 koff = (u32)kt * N + n;
    const u32 poff_b = ((u32)p * next + t) * (u32)N + n, poff_1 = (u32)t * N + n;
    u64 su[MAXD + 1], kv0[MAXD], kv1[MAXD], w = one_m;
    int s_next = 0;
    auto fetch = [&](int k) {
        const u32 g = T.g[k];
        const int sblk = (int)(automorph_src((u32)dst0, g, logn) >> logb);
        const u32 so = (u32)sblk * BLK;
        const u64* Uk = T.U[k] + uoff + so;
#pragma unroll
        for (int j = 0; j < MAXD; j++)
            if (j < nd) su[j] = __ldg(Uk + j * dstr);
        su[MAXD] = has_c0 ? __ldg(T.c0[k] + coff + so) : 0ull;
        const u64* kp = T.key[k] + koff;
#pragma unroll
        for (int j = 0; j < MAXD; j++)
            if (j < nd) { kv0[j] = __ldg(kp + j * kds); kv1[j] = __ldg(kp + j * kds + kcs); }
        const u64* pk = T.pt[k];
        w = pk ? __ldg(pk + (T.pt_batched[k] ? poff_b : poff_1)) : one_m;
        s_next = (int)(automorph_src((u32)n, g, logn) & (BLK - 1));
    };
    fetch(0);
    int np = 0;                                       // products in b0/b1 since the last fold
    for (int k = 0; k < T.n; k++) {
        __syncthreads();
#pragma unroll
        for (int j = 0; j < MAXD; j++)
            if (j < nd) sm[j * BLK + tid] = su[j];
        for (int j = MAXD; j < ndig; j++) {           // (rare) more digits than prefetch slots
            const int sblk = (int)(automorph_src((u32)dst0, T.g[k], logn) >> logb);
            sm[j * BLK + tid] = __ldg(T.U[k] + uoff + (u32)sblk * BLK + (u32)j * dstr);
        }
        if (has_c0) sm[ndig * BLK + tid] = su[MAXD];
        const u64 wk = w;
        const int s = s_next;
        __syncthreads();
        if (T.fused[k]) {
            // multiplier folded into the key (or absent): products go straight
            // into the output sums -- ndig MACs per component, no REDC
            if (np + ndig > 32) { b0.fold_hi(q, inv1); b1.fold_hi(q, inv1); np = 0; }
#pragma unroll
            for (int j = 0; j < MAXD; j++) {
                if (j < nd) {
                    const u64 u = sm[j * BLK + s];
                    b0.mac(u, kv0[j]);
                    b1.mac(u, kv1[j]);
                }
            }
            for (int j = MAXD; j < ndig; j++) {
                const u64 u = sm[j * BLK + s];
                const u64* kp = T.key[k] + koff;
                b0.mac(u, __ldg(kp + j * kds));
                b1.mac(u, __ldg(kp + j * kds + kcs));
            }
            np += ndig;
        } else {
            Acc4 a0, a1;                               // ndig <= 32 products
            a0.zero(); a1.zero();
#pragma unroll
            for (int j = 0; j < MAXD; j++) {
                if (j < nd) {
                    const u64 u = sm[j * BLK + s];
                    a0.mac(u, kv0[j]);
                    a1.mac(u, kv1[j]);
                }
            }
            for (int j = MAXD; j < ndig; j++) {
                const u64 u = sm[j * BLK + s];
                const u64* kp = T.key[k] + koff;
                a0.mac(u, __ldg(kp + j * kds));
                a1.mac(u, __ldg(kp + j * kds + kcs));
            }
            if (np + 1 > 32) { b0.fold_hi(q, inv1); b1.fold_hi(q, inv1); np = 0; }
            b0.mac(a0.reduce(q, qn, inv1), wk);
            b1.mac(a1.reduce(q, qn, inv1), wk);
            np += 1;
        }
        if (has_c0) cc.mac(sm[ndig * BLK + s], wk);
        if ((k & 31) == 31) cc.fold_hi(q, inv1);
        if (k + 1 < T.n) fetch(k + 1);   // other warps hide this latency
    }
    u64* o0 = B + (p * 2 * next + t) * (long long)N + n;
    u64* o1 = o0 + (long long)next * N;
    u64 r0 = b0.reduce(q, qn, inv1), r1 = b1.reduce(q, qn, inv1);
    if (accumulate) { r0 = add_mod(r0, *o0, q); r1 = add_mod(r1, *o1, q); }
    *o0 = r0;
    *o1 = r1;
    if (has_c0) {
        u64* oc = C0 + p * c0_ostride + (long long)t * N + n;
        u64 rc = cc.reduce(q, qn, inv1);
        if (c0_acc) rc = add_mod(rc, *oc, q);
        *oc = rc;
    }
}

__global__ void premul_key_kernel(u64* __restrict__ out, const u64* __restrict__ key, const u64* __restrict__ pt,
                                  int next, int logn, long long kds, long long kcs, Limbs ext,
                                  const PrimeInfo* __restrict__ pr) {
    const int N = 1 << logn;
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    const int t = blockIdx.y, jc = blockIdx.z, j = jc >> 1, c = jc & 1;
    if (n >= N) return;
    const int kt = ext.prime[t];
    const PrimeInfo& P = pr[kt];
    const long long o = j * kds + c * kcs + (long long)kt * N + n;
    out[o] = mont_mul(__ldg(key + o), __ldg(pt + (long long)t * N + n), P.q, P.qinv_neg);
}

cudaError_t premul_key_op(u64* out, const u64* key, const u64* pt, int ndig, int next, int logn, long long kds,
                          long long kcs, const Limbs& ext, const PrimeInfo* pr, cudaStream_t st) {
    const int N = 1 << logn;
    const int tpb = N < 256 ? N : 256;
    dim3 grid((N + tpb - 1) / tpb, next, 2 * ndig);
    premul_key_kernel<<<grid, tpb, 0, st>>>(out, key, pt, next, logn, kds, kcs, ext, pr);
    return launched();
}

// Direct-gather rotation sum: one thread per output word (slot set, limb,
// coefficient).  Under X -> X^g an aligned 32-block of the bit-reversed NTT
// domain is the image of one aligned 32-block (tests/test_oracle.py), so the
// 32 gathers of a warp hit one 256-byte run -- coalesced without the SMEM
// staging and the two barriers per term of rotsum_kernel.
#ifndef BCN_RS2_MINB
#define BCN_RS2_MINB 6
#endif
template <int ND>    // digits (1..4); 0: runtime count
__global__ void __launch_bounds__(256, BCN_RS2_MINB) rotsum2_kernel(
        u64* __restrict__ B, u64* __restrict__ C0, const RotTerms T, long long c0_gstride, int nq, int next,
        int ndig, int logn, long long kds, long long kcs, Limbs ext, const PrimeInfo* __restrict__ pr,
        int acc_flags, long long c0_ostride) {
    const int N = 1 << logn;
    const int n = blockIdx.x * 256 + threadIdx.x;
    const int t = blockIdx.y;
    const long long p = blockIdx.z;
    const int kt = ext.prime[t];
    const PrimeInfo& P = pr[kt];
    const u64 q = P.q, qn = P.qinv_neg, one_m = P.r1, inv1 = P.pad[2];
    const bool has_c0 = t < nq;
    const int nd = ND > 0 ? ND : ndig;
    // 32-bit word offsets (the launcher checks every operand stays below 2^32 words)
    const u32 dstr = (u32)next * (u32)N;
    const u32 uoff = ((u32)p * nd * next + t) * (u32)N;
    const u32 coff = (u32)(p * c0_gstride) + (u32)t * N;
    const u32 koff = (u32)kt * N + n;
    const u32 poff_b = ((u32)p * next + t) * (u32)N + n, poff_1 = (u32)t * N + n;
    const u32 kds32 = (u32)kds, kcs32 = (u32)kcs;
    Acc4 b0, b1, cc;
    b0.zero(); b1.zero(); cc.zero();
    int np = 0;                                       // products in b0/b1 since the last fold
    for (int k = 0; k < T.n; k++) {
        const u32 sn = automorph_src((u32)n, T.g[k], logn);
        const u64* Uk = T.U[k] + (uoff + sn);
        const u64* kp = T.key[k] + koff;
        const u64* pk = T.pt[k];
        const u64 w = pk ? __ldg(pk + (T.pt_batched[k] ? poff_b : poff_1)) : one_m;
        if (T.fused[k]) {
            if (np + nd > 32) { b0.fold_hi(q, inv1); b1.fold_hi(q, inv1); np = 0; }
#pragma unroll
            for (int j = 0; j < (ND > 0 ? ND : 1); j++) {
                if (ND == 0) break;
                const u64 u = __ldg(Uk + j * dstr);
                b0.mac(u, __ldg(kp + j * kds32));
                b1.mac(u, __ldg(kp + j * kds32 + kcs32));
            }
            if (ND == 0)
                for (int j = 0; j < nd; j++) {
                    const u64 u = __ldg(Uk + (u32)j * dstr);
                    b0.mac(u, __ldg(kp + (u32)j * kds32));
                    b1.mac(u, __ldg(kp + (u32)j * kds32 + kcs32));
                }
            np += nd;
        } else {
            Acc4 a0, a1;
            a0.zero(); a1.zero();
            for (int j = 0; j < nd; j++) {
                const u64 u = __ldg(Uk + (u32)j * dstr);
                a0.mac(u, __ldg(kp + (u32)j * kds32));
                a1.mac(u, __ldg(kp + (u32)j * kds32 + kcs32));
            }
            if (np + 1 > 32) { b0.fold_hi(q, inv1); b1.fold_hi(q, inv1); np = 0; }
            b0.mac(a0.reduce(q, qn, inv1), w);
            b1.mac(a1.reduce(q, qn, inv1), w);
            np += 1;
        }
        if (has_c0) {
            cc.mac(__ldg(T.c0[k] + (coff + sn)), w);
            if ((k & 31) == 31) cc.fold_hi(q, inv1);
        }
    }
    const int accumulate = acc_flags & 1, c0_acc = (acc_flags >> 1) & 1;
    u64* o0 = B + (p * 2 * next + t) * (long long)N + n;
    u64* o1 = o0 + (long long)next * N;
    u64 r0 = b0.reduce(q, qn, inv1), r1 = b1.reduce(q, qn, inv1);
    if (accumulate) { r0 = add_mod(r0, *o0, q); r1 = add_mod(r1, *o1, q); }
    *o0 = r0;
    *o1 = r1;
    if (has_c0) {
        u64* oc = C0 + p * c0_ostride + (long long)t * N + n;
        u64 rc = cc.reduce(q, qn, inv1);
        if (c0_acc) rc = add_mod(rc, *oc, q);
        *oc = rc;
    }
}

// rotsum3: rotsum2 for the common case -- every term's key already carries its
// multiplier (fused, bcn_premul_key) and no plaintext is batched per slot set.
// Straight-line term loop: the per-term state is the Galois element and four
// pointers from the parameter bank, the block coordinates are hoisted, and
// the high halves fold every 32 / ND terms at a uniform counter instead of a
// per-term check (ISA: ~90 instead of ~210 instructions per term at ND = 2).
#ifndef BCN_RS3_MINB
#define BCN_RS3_MINB 6
#endif
template <int ND>
__global__ void __launch_bounds__(256, BCN_RS3_MINB) rotsum3_kernel(
        u64* __restrict__ B, u64* __restrict__ C0, const RotTerms T, long long c0_gstride, int nq, int next,
        int logn, long long kds, long long kcs, Limbs ext, const PrimeInfo* __restrict__ pr, int acc_flags,
        long long c0_ostride) {
    constexpr int FOLD = 32 / ND;
    const int N = 1 << logn;
    const int n = blockIdx.x * 256 + threadIdx.x;
    const int t = blockIdx.y;
    const long long p = blockIdx.z;
    const int kt = ext.prime[t];
    const PrimeInfo& P = pr[kt];
    const u64 q = P.q, qn = P.qinv_neg, one_m = P.r1, inv1 = P.pad[2];
    const bool has_c0 = t < nq;
    const u32 dstr = (u32)next * (u32)N;
    const u32 uoff = ((u32)p * ND * next + t) * (u32)N;
    const u32 coff = (u32)(p * c0_gstride) + (u32)t * N;
    const u32 koff = (u32)kt * N + n;
    const u32 poff = (u32)t * N + n;
    const u32 kds32 = (u32)kds, kcs32 = (u32)kcs;
    Acc4 b0, b1, cc;
    b0.zero(); b1.zero(); cc.zero();
    int kf = 0;
    for (int k = 0; k < T.n; k++) {
        const u32 sn = automorph_src((u32)n, T.g[k], logn);
        const u64* __restrict__ Uk = T.U[k] + (uoff + sn);
        const u64* __restrict__ kp = T.key[k] + koff;
#pragma unroll
        for (int j = 0; j < ND; j++) {
            const u64 u = __ldg(Uk + j * dstr);
            b0.mac(u, __ldg(kp + j * kds32));
            b1.mac(u, __ldg(kp + j * kds32 + kcs32));
        }
        if (has_c0) {
            const u64* pk = T.pt[k];
            const u64 w = pk ? __ldg(pk + poff) : one_m;
            cc.mac(__ldg(T.c0[k] + (coff + sn)), w);
            if ((k & 31) == 31) cc.fold_hi(q, inv1);
        }
        if (++kf == FOLD) { b0.fold_hi(q, inv1); b1.fold_hi(q, inv1); kf = 0; }
    }
    const int accumulate = acc_flags & 1, c0_acc = (acc_flags >> 1) & 1;
    u64* o0 = B + (p * 2 * next + t) * (long long)N + n;
    u64* o1 = o0 + (long long)next * N;
    u64 r0 = b0.reduce(q, qn, inv1), r1 = b1.reduce(q, qn, inv1);
    if (accumulate) { r0 = add_mod(r0, *o0, q); r1 = add_mod(r1, *o1, q); }
    *o0 = r0;
    *o1 = r1;
    if (has_c0) {
        u64* oc = C0 + p * c0_ostride + (long long)t * N + n;
        u64 rc = cc.reduce(q, qn, inv1);
        if (c0_acc) rc = add_mod(rc, *oc, q);
        *oc = rc;
    }
}

// rotsum4: rotsum3 on the FP64 pipe (every basis prime below 2^50).  The
// integer form spends ~125 instructions per (term, output pair) -- u128 MACs on
// the 32-bit IMAD datapath, the automorphism index and five key / plaintext
// words re-read by every slot set.  Here a thread owns (coefficient, limb) for
// SS slot sets: the term's index and its key / plaintext words (Montgomery ->
// {w, w/q} doubles) are paid once per SS slot sets, the SS x (ND + 1) operand
// loads go out together, and each product is one fmm (6 FP64 instructions);
// the sums stay exact integers in doubles, folded to [-q/2, q/2] every 4 terms
// (|sum| <= 0.5 q + 4 (ND <= 4 products) 0.61 q... kept below 2^53 by FOLD).
#ifndef BCN_RS4_SS
#define BCN_RS4_SS 4
#endif
#ifndef BCN_RS4_MINB
#define BCN_RS4_MINB 3
#endif
template <int ND>
__global__ void __launch_bounds__(256, BCN_RS4_MINB) rotsum4_kernel(
        u64* __restrict__ B, u64* __restrict__ C0, const RotTerms T, long long c0_gstride, int G, int nq, int next,
        int logn, long long kds, long long kcs, Limbs ext, const PrimeInfo* __restrict__ pr,
        const double2* __restrict__ fq, int acc_flags, long long c0_ostride) {
    constexpr int SS = BCN_RS4_SS;
    constexpr int FOLD = ND <= 2 ? 4 : 2;          // products per sum between folds: FOLD * ND <= 8 (8 x 0.61 q + q/2 < 2^53 / q)
    const int N = 1 << logn;
    const int n = blockIdx.x * 256 + threadIdx.x;
    const int t = blockIdx.y;
    const long long p0 = (long long)blockIdx.z * SS;
    const int kt = ext.prime[t];
    const PrimeInfo& P = pr[kt];
    const u64 q = P.q, qn = P.qinv_neg, one_m = P.r1;
    const double2 f = fq[kt];
    const bool has_c0 = t < nq;
    const long long dstr = (long long)next * N;
    const long long ustep = (long long)ND * dstr;                 // per slot set
    const long long uoff = (p0 * ND * next + t) * (long long)N;
    const long long coff = p0 * c0_gstride + (long long)t * N;
    const long long koff = (long long)kt * N + n;
    const long long poff = (long long)t * N + n;
    int live = G - (int)p0;
    live = live > SS ? SS : live;
    double b0[SS], b1[SS], cc[SS];
#pragma unroll
    for (int s = 0; s < SS; s++) b0[s] = b1[s] = cc[s] = 0.0;
    int kf = 0;
    for (int k = 0; k < T.n; k++) {
        const long long sn = automorph_src((u32)n, T.g[k], logn);
        const u64* __restrict__ Uk = T.U[k] + (uoff + sn);
        const u64* __restrict__ Ck = T.c0[k] + (coff + sn);
        const u64* __restrict__ kp = T.key[k] + koff;
        u64 uw[SS][ND], cw[SS], k0[ND], k1[ND];
#pragma unroll
        for (int j = 0; j < ND; j++) { k0[j] = __ldg(kp + j * kds); k1[j] = __ldg(kp + j * kds + kcs); }
        const u64* pk = T.pt[k];
        const u64 w = has_c0 && pk ? __ldg(pk + poff) : one_m;
#pragma unroll
        for (int s = 0; s < SS; s++) {                            // a slot set past G re-reads the first one
            const long long so = s < live ? s : 0;
#pragma unroll
            for (int j = 0; j < ND; j++) uw[s][j] = __ldg(Uk + so * ustep + j * dstr);
            cw[s] = has_c0 ? __ldg(Ck + so * c0_gstride) : 0ull;
        }
        double kd[ND], kq[ND], kd1[ND], kq1[ND];
#pragma unroll
        for (int j = 0; j < ND; j++) {
            kd[j] = fload(redc(0ull, k0[j], q, qn));
            kq[j] = __dmul_rn(kd[j], f.y);
            kd1[j] = fload(redc(0ull, k1[j], q, qn));
            kq1[j] = __dmul_rn(kd1[j], f.y);
        }
        const double wd = fload(redc(0ull, w, q, qn)), wq = __dmul_rn(wd, f.y);
#pragma unroll
        for (int s = 0; s < SS; s++) {
#pragma unroll
            for (int j = 0; j < ND; j++) {
                const double ud = fload(uw[s][j]);
                b0[s] = __dadd_rn(b0[s], fmm(ud, kd[j], kq[j], f.x));
                b1[s] = __dadd_rn(b1[s], fmm(ud, kd1[j], kq1[j], f.x));
            }
            if (has_c0) cc[s] = __dadd_rn(cc[s], fmm(fload(cw[s]), wd, wq, f.x));
        }
        if (++kf == FOLD) {
#pragma unroll
            for (int s = 0; s < SS; s++) {
                b0[s] = fred(b0[s], f.y, f.x);
                b1[s] = fred(b1[s], f.y, f.x);
            }
            kf = 0;
        }
        if ((k & 7) == 7) {
#pragma unroll
            for (int s = 0; s < SS; s++) cc[s] = fred(cc[s], f.y, f.x);
        }
    }
    const int accumulate = acc_flags & 1, c0_acc = (acc_flags >> 1) & 1;
#pragma unroll
    for (int s = 0; s < SS; s++) {
        if (s >= live) break;
        const long long p = p0 + s;
        u64* o0 = B + (p * 2 * next + t) * (long long)N + n;
        u64* o1 = o0 + (long long)next * N;
        u64 r0 = fcanon(b0[s], f.y, f.x), r1 = fcanon(b1[s], f.y, f.x);
        if (accumulate) { r0 = add_mod(r0, *o0, q); r1 = add_mod(r1, *o1, q); }
        *o0 = r0;
        *o1 = r1;
        if (has_c0) {
            u64* oc = C0 + p * c0_ostride + (long long)t * N + n;
            u64 rc = fcanon(cc[s], f.y, f.x);
            if (c0_acc) rc = add_mod(rc, *oc, q);
            *oc = rc;
        }
    }
}

cudaError_t rotsum_op(u64* B, u64* C0, const RotTerms& terms, long long c0_gstride, int G, int nq, int next,
                      int ndig, int logn, long long kds, long long kcs, const Limbs& ext, const PrimeInfo* pr,
                      int accumulate, cudaStream_t st, long long c0_ostride, int c0_accumulate, const double2* fq) {
    const int N = 1 << logn;
    if (terms.n <= 0 || G <= 0) return cudaSuccess;
    if (c0_ostride < 0) c0_ostride = (long long)nq * N;
    if (c0_accumulate < 0) c0_accumulate = accumulate;
    const int flags = (accumulate ? 1 : 0) | (c0_accumulate ? 2 : 0);
    if ((long long)G * (ndig + 2) * next * N >= (1LL << 32) || (long long)G * c0_gstride >= (1LL << 32) ||
        2LL * kds >= (1LL << 32))
        return cudaErrorInvalidValue;                 // kernel offsets are 32-bit
    if (N >= 256 && !getenv("BCN_ROTSUM_STAGED")) {
        dim3 grid(N / 256, next, G);
        static const bool rs3_off = getenv("BCN_ROTSUM3") && getenv("BCN_ROTSUM3")[0] == '0';
        bool simple = !rs3_off && ndig >= 1 && ndig <= 4;
        for (int k = 0; k < terms.n && simple; k++) simple = terms.fused[k] && !terms.pt_batched[k];
        static const bool rs4_off = getenv("BCN_ROTSUM4") && getenv("BCN_ROTSUM4")[0] == '0';
        if (simple && fq && !rs4_off) {
            dim3 grid4(N / 256, next, (G + BCN_RS4_SS - 1) / BCN_RS4_SS);
            switch (ndig) {
#define BCN_RS4(D) case D: rotsum4_kernel<D><<<grid4, 256, 0, st>>>(B, C0, terms, c0_gstride, G, nq, next, logn, kds, \
                                                                  kcs, ext, pr, fq, flags, c0_ostride); break;
                BCN_RS4(1) BCN_RS4(2) BCN_RS4(3) BCN_RS4(4)
#undef BCN_RS4
            }
            return launched();
        }
        if (simple) {
            switch (ndig) {
#define BCN_RS3(D) case D: rotsum3_kernel<D><<<grid, 256, 0, st>>>(B, C0, terms, c0_gstride, nq, next, logn, kds, kcs, \
                                                                 ext, pr, flags, c0_ostride); break;
                BCN_RS3(1) BCN_RS3(2) BCN_RS3(3) BCN_RS3(4)
#undef BCN_RS3
            }
            return launched();
        }
        switch (ndig) {
#define BCN_RS2(D) case D: rotsum2_kernel<D><<<grid, 256, 0, st>>>(B, C0, terms, c0_gstride, nq, next, ndig, logn, \
                                                                 kds, kcs, ext, pr, flags, c0_ostride); break;
            BCN_RS2(1) BCN_RS2(2) BCN_RS2(3) BCN_RS2(4)
#undef BCN_RS2
            default:
                rotsum2_kernel<0><<<grid, 256, 0, st>>>(B, C0, terms, c0_gstride, nq, next, ndig, logn, kds, kcs, ext,
                                                        pr, flags, c0_ostride);
        }
        return launched();
    }
    if ((long long)G * (ndig + 2) * next * N >= (1LL << 32) || (long long)G * c0_gstride >= (1LL << 32))
        return cudaErrorInvalidValue;                 // kernel offsets are 32-bit
    if (N >= 1024) {
        constexpr int BLK = 1024;
        const size_t smem = (size_t)(ndig + 1) * BLK * sizeof(u64);
        static unsigned long long smem_cfg = 0;
    unsigned long long smem_bit = 0;
    if (first_on_device(&smem_cfg, &smem_bit)) {
        cudaError_t ae = cudaSuccess;
        BCN_SMEM_ATTR(ae, (rotsum_kernel<BLK>), 200 * 1024);
        if (ae != cudaSuccess) return ae;
        smem_cfg |= smem_bit;
    }
        dim3 grid(G, N / BLK, next);
        rotsum_kernel<BLK><<<grid, BLK, smem, st>>>(B, C0, terms, c0_gstride, nq, next, ndig, logn, kds, kcs, ext, pr,
                                                    flags, c0_ostride);
    } else {
        const size_t smem = (size_t)(ndig + 1) * N * sizeof(u64);
        dim3 grid(G, 1, next);
        switch (N) {
#define BCN_RS(NN) case NN: rotsum_kernel<NN><<<grid, NN, smem, st>>>(B, C0, terms, c0_gstride, \
                        nq, next, ndig, logn, kds, kcs, ext, pr, flags, c0_ostride); break;
            BCN_RS(8) BCN_RS(16) BCN_RS(32) BCN_RS(64) BCN_RS(128) BCN_RS(256) BCN_RS(512)
#undef BCN_RS
            default: return cudaErrorInvalidValue;
        }
    }
    return launched();
}

// dst[p][n] += src[p][n] * w mod q  (merged ModDown + rescale: Y_top = B_top + P C_top)
__global__ void axpy_limb_kernel(u64* __restrict__ dst, long long ds, const u64* __restrict__ src, long long ss,
                                 u64 w, u64 wp, u64 q, int logn, long long total) {
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long p = idx >> logn;
        const int n = (int)(idx & ((1 << logn) - 1));
        u64* d = dst + p * ds + n;
        *d = add_mod(*d, shoup(src[p * ss + n], w, wp, q), q);
    }
}

cudaError_t axpy_limb_op(u64* dst, long long ds, const u64* src, long long ss, int npoly, u64 w, u64 wp, u64 q,
                         int logn, cudaStream_t st) {
    const long long total = (long long)npoly << logn;
    if (!total) return cudaSuccess;
    axpy_limb_kernel<<<blocks_for(total, 256), 256, 0, st>>>(dst, ds, src, ss, w, wp, q, logn, total);
    return launched();
}

// out[p][i] = (B[p][i] - Z[p][i]) * pq_i + C[(p/2)][(p%2)][i] * ql_i for i < nout (staged merged ModDown+rescale)
__global__ void mdr_combine_kernel(u64* __restrict__ out, const u64* __restrict__ B, long long bps,
                                   const u64* __restrict__ Z, const u64* __restrict__ C, long long cps, int add_c1,
                                   int nout, int logn, Limbs ql, const PrimeInfo* __restrict__ pr,
                                   const u64* __restrict__ pqinv, const u64* __restrict__ qlinv, long long total) {
    const int N = 1 << logn;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int n = (int)(idx & (N - 1));
        const long long rest = idx >> logn;
        const int i = (int)(rest % nout);
        const long long p = rest / nout;
        const u64 q = pr[ql.prime[i]].q;
        u64 r = shoup(B[p * bps + (long long)i * N + n] + q - Z[(p * nout + i) * N + n], pqinv[2 * i],
                      pqinv[2 * i + 1], q);
        const int comp = (int)(p & 1);
        if (C && (comp == 0 || add_c1))
            r = add_mod(r, shoup(C[(p >> 1) * cps + (long long)comp * (nout + 1) * N + (long long)i * N + n],
                                 qlinv[2 * i], qlinv[2 * i + 1], q), q);
        out[(p * nout + i) * N + n] = r;
    }
}

cudaError_t mdr_combine_op(u64* out, const u64* B, long long bps, const u64* Z, const u64* C, long long cps,
                           int add_c1, int npoly, int nout, int logn, const Limbs& ql, const PrimeInfo* pr,
                           const u64* pqinv, const u64* qlinv, cudaStream_t st) {
    const long long total = (long long)npoly * nout << logn;
    if (!total) return cudaSuccess;
    mdr_combine_kernel<<<blocks_for(total, 256), 256, 0, st>>>(out, B, bps, Z, C, cps, add_c1, nout, logn, ql, pr,
                                                              pqinv, qlinv, total);
    return launched();
}

// -------------------------------------------------------- ModDown (K7)
// Z[p][i] = REDC(sum_k [xP_k * phatinv_k]_{p_k} * phat_m[k][i]) for i <= level
// (coefficient domain), from the INTT'd special limbs of A.
template <int KK>    // source count at compile time: y[] in registers (0: runtime count, local array)
__global__ void moddown_conv_kernel(u64* __restrict__ Z, const u64* __restrict__ A, long long a_stride,
                                    int nq, int K, int logn, Limbs ext, const PrimeInfo* __restrict__ pr,
                                    const ConvTable* __restrict__ tab, const __grid_constant__ FConv fc, int use_fp) {
    constexpr int YK = KK > 0 ? KK : BCN_MAX_ALPHA;
    const int N = 1 << logn;
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    const long long p = blockIdx.y;
    const ConvTable& T = *tab;
    const int nk = KK > 0 ? KK : K;
    u64 y[YK];
    const u64* ap = A + p * a_stride + (long long)nq * N + n;
#pragma unroll
    for (int k = 0; k < YK; k++) {
        if (k < nk) {
            const PrimeInfo& P = pr[ext.prime[nq + k]];
            y[k] = shoup(__ldg(ap + (long long)k * N), T.hatinv[k], T.hatinv_p[k], P.q);
        }
    }
    u64* zp = Z + p * (long long)nq * N + n;
    if (use_fp) {                                      // FP64 pipe (every basis prime in (2^49, 2^50))
        double yd[YK];
#pragma unroll
        for (int k = 0; k < YK; k++) yd[k] = k < nk ? fload(y[k]) : 0.0;
        for (int i = 0; i < nq; i++) {
            const double2 f = fc.fq[i];
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < YK; k++)
                if (k < nk) acc = __dadd_rn(acc, fmm(yd[k], fc.h[k][i].x, fc.h[k][i].y, f.x));
            zp[(long long)i * N] = fcanon(acc, f.y, f.x);
        }
        return;
    }
    for (int i = 0; i < nq; i++) {
        const PrimeInfo& P = pr[ext.prime[i]];
        Acc4 acc; acc.zero();                          // K <= 16 products
#pragma unroll
        for (int k = 0; k < YK; k++)
            if (k < nk) acc.mac(y[k], T.hat_m[k * BCN_MAX_LIMBS + i]);
        zp[(long long)i * N] = acc.reduce(P.q, P.qinv_neg, P.pad[2]);
    }
}

// FP64 form, two coefficients per thread (see modup_fp_kernel)
template <int KK>
__global__ void moddown_conv_fp_kernel(u64* __restrict__ Z, const u64* __restrict__ A, long long a_stride, int nq,
                                       int logn, Limbs ext, const PrimeInfo* __restrict__ pr,
                                       const ConvTable* __restrict__ tab, const __grid_constant__ FConv fc) {
    const int N = 1 << logn;
    const int n = blockIdx.x * 2 * blockDim.x + threadIdx.x;   // and n + blockDim.x
    const int h = blockDim.x;
    const long long p = blockIdx.y;
    const ConvTable& T = *tab;
    double y0[KK], y1[KK];
    const u64* ap = A + p * a_stride + (long long)nq * N + n;
#pragma unroll
    for (int k = 0; k < KK; k++) {
        const PrimeInfo& P = pr[ext.prime[nq + k]];
        y0[k] = fload(shoup(__ldg(ap + (long long)k * N), T.hatinv[k], T.hatinv_p[k], P.q));
        y1[k] = fload(shoup(__ldg(ap + (long long)k * N + h), T.hatinv[k], T.hatinv_p[k], P.q));
    }
    u64* zp = Z + p * (long long)nq * N + n;
    for (int i = 0; i < nq; i++) {
        const double2 f = fc.fq[i];
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int k = 0; k < KK; k++) {
            const double2 hh = fc.h[k][i];
            a0 = __dadd_rn(a0, fmm(y0[k], hh.x, hh.y, f.x));
            a1 = __dadd_rn(a1, fmm(y1[k], hh.x, hh.y, f.x));
        }
        zp[(long long)i * N] = fcanon(a0, f.y, f.x);
        zp[(long long)i * N + h] = fcanon(a1, f.y, f.x);
    }
}

cudaError_t moddown_conv_op(u64* Z, const u64* A, long long a_stride, int npoly, int nq, int K, int logn,
                            const Limbs& ext, const PrimeInfo* pr, const ConvTable* tab, cudaStream_t st,
                            const FConv* fcp) {
    const int N = 1 << logn;
    int tpb = N < 256 ? N : 256;
    dim3 grid((N + tpb - 1) / tpb, npoly);
    static FConv none;
    const int use_fp = fcp && K <= BCN_FC_SRC && nq <= BCN_FC_TGT;
    const FConv& fc = use_fp ? *fcp : none;
    if (use_fp && N >= 512) {
        const dim3 g2(N / 512, npoly);
        switch (K) {
#define BCN_MF(KV) case KV: moddown_conv_fp_kernel<KV><<<g2, 256, 0, st>>>(Z, A, a_stride, nq, logn, ext, pr, tab, \
                                                                           *fcp); return launched();
            BCN_MF(1) BCN_MF(2) BCN_MF(3) BCN_MF(4) BCN_MF(5) BCN_MF(6) BCN_MF(7) BCN_MF(8)
#undef BCN_MF
            default: break;
        }
    }
    switch (K) {
#define BCN_MC(KV) case KV: moddown_conv_kernel<KV><<<grid, tpb, 0, st>>>(Z, A, a_stride, nq, K, logn, ext, pr, tab, fc, use_fp); break;
        BCN_MC(1) BCN_MC(2) BCN_MC(3) BCN_MC(4) BCN_MC(5) BCN_MC(6) BCN_MC(7) BCN_MC(8) BCN_MC(9)
#undef BCN_MC
        default: moddown_conv_kernel<0><<<grid, tpb, 0, st>>>(Z, A, a_stride, nq, K, logn, ext, pr, tab, fc, 0);
    }
    return launched();
}

// out[p][c][i] = addend[p][c][i] + (A[p][c][i] - Z[p][c][i]) * P^-1   (c = 0, 1)
// addend (optional, stride as) is permuted by X -> X^g when g != 1 and
// only applied to component 0 when add_c1 == 0.
__global__ void moddown_combine_kernel(u64* __restrict__ out, long long os, const u64* __restrict__ A,
                                       int next, const u64* __restrict__ Z, const u64* __restrict__ addend,
                                       long long as, int add_c1, u32 g, int nq, int logn, Limbs ql,
                                       const PrimeInfo* __restrict__ pr, const u64* __restrict__ pinv,
                                       long long total) {
    const int N = 1 << logn;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int n = (int)(idx & (N - 1));
        long long rest = idx >> logn;
        const int i = (int)(rest % nq);
        rest /= nq;
        const int c = (int)(rest & 1);
        const long long p = rest >> 1;
        const PrimeInfo& P = pr[ql.prime[i]];
        const u64 q = P.q;
        const u64 a = A[(p * 2 + c) * next * (long long)N + (long long)i * N + n];
        const u64 z = Z[(p * 2 + c) * nq * (long long)N + (long long)i * N + n];
        u64 r = shoup(a + q - z, pinv[2 * i], pinv[2 * i + 1], q);
        if (addend && (c == 0 || add_c1)) {
            const int src = (g == 1u) ? n : (int)automorph_src((u32)n, g, logn);
            r = add_mod(r, addend[p * as + (long long)c * nq * N + (long long)i * N + src], q);
        }
        out[p * os + (long long)c * nq * N + (long long)i * N + n] = r;
    }
}

cudaError_t moddown_combine_op(u64* out, long long os, const u64* A, int next, const u64* Z, const u64* addend,
                               long long as, int add_c1, u32 g, int npoly, int nq, int logn, const Limbs& ql,
                               const PrimeInfo* pr, const u64* pinv, cudaStream_t st) {
    long long total = (long long)npoly * 2 * nq << logn;
    if (!total) return cudaSuccess;
    moddown_combine_kernel<<<blocks_for(total, 256), 256, 0, st>>>(out, os, A, next, Z, addend, as, add_c1, g,
                                                                   nq, logn, ql, pr, pinv, total);
    return launched();
}

// ---------------------------------------------------------- rescale (K5)
// W[p][i] = centred(top[p]) mod q_i, i < nq (coefficient domain)
__global__ void rescale_lift_kernel(u64* __restrict__ W, const u64* __restrict__ top, int nq, u64 qtop,
                                    int logn, Limbs ql, const PrimeInfo* __restrict__ pr, long long total) {
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int n = (int)(idx & ((1 << logn) - 1));
        long long rest = idx >> logn;
        const int i = (int)(rest % nq);
        const long long p = rest / nq;
        const u64 q = pr[ql.prime[i]].q;
        const u64 v = top[(p << logn) + n];
        u64 r = v % q;
        if (v > (qtop >> 1)) r = sub_mod(r, qtop % q, q);   // v - qtop
        W[idx] = r;
    }
}

cudaError_t rescale_lift_op(u64* W, const u64* top, int npoly, int nq, u64 qtop, int logn, const Limbs& ql,
                            const PrimeInfo* pr, cudaStream_t st) {
    long long total = (long long)npoly * nq << logn;
    if (!total) return cudaSuccess;
    rescale_lift_kernel<<<blocks_for(total, 256), 256, 0, st>>>(W, top, nq, qtop, logn, ql, pr, total);
    return launched();
}

// out[p][i] = (c[p][i] - W[p][i]) * q_top^-1
__global__ void rescale_combine_kernel(u64* __restrict__ out, long long os, const u64* __restrict__ c,
                                       long long cs, const u64* __restrict__ W, int nq, int logn, Limbs ql,
                                       const PrimeInfo* __restrict__ pr, const u64* __restrict__ qinv,
                                       long long total) {
    const int N = 1 << logn;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int n = (int)(idx & (N - 1));
        long long rest = idx >> logn;
        const int i = (int)(rest % nq);
        const long long p = rest / nq;
        const u64 q = pr[ql.prime[i]].q;
        const u64 a = c[p * cs + (long long)i * N + n];
        out[p * os + (long long)i * N + n] = shoup(a + q - W[idx], qinv[2 * i], qinv[2 * i + 1], q);
    }
}

cudaError_t rescale_combine_op(u64* out, long long os, const u64* c, long long cs, const u64* W, int npoly,
                               int nq, int logn, const Limbs& ql, const PrimeInfo* pr, const u64* qinv,
                               cudaStream_t st) {
    long long total = (long long)npoly * nq << logn;
    if (!total) return cudaSuccess;
    rescale_combine_kernel<<<blocks_for(total, 256), 256, 0, st>>>(out, os, c, cs, W, nq, logn, ql, pr, qinv,
                                                                   total);
    return launched();
}

// gather one limb of every poly: dst[p][n] = src[p * stride + off + n]
__global__ void gather_limb_kernel(u64* __restrict__ dst, const u64* __restrict__ src, long long stride,
                                   long long off, int logn, long long total) {
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long p = idx >> logn;
        dst[idx] = src[p * stride + off + (idx & ((1 << logn) - 1))];
    }
}

cudaError_t gather_limb_op(u64* dst, const u64* src, long long stride, long long off, int npoly, int logn,
                           cudaStream_t st) {
    long long total = (long long)npoly << logn;
    if (!total) return cudaSuccess;
    gather_limb_kernel<<<blocks_for(total, 256), 256, 0, st>>>(dst, src, stride, off, logn, total);
    return launched();
}

// copy limbs [0, nlimb) of each poly between differently-strided buffers
// grid (words / (2 blockDim), poly): 16-byte moves, no per-element division
__global__ void copy_limbs_kernel(u64* __restrict__ dst, long long ds, const u64* __restrict__ src, long long ss,
                                  long long per_poly, long long total) {
    const long long p = blockIdx.y;
    const long long o = 2 * ((long long)blockIdx.x * blockDim.x + threadIdx.x);
    if (o < per_poly) {
        const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(src + p * ss + o);
        *reinterpret_cast<ulonglong2*>(dst + p * ds + o) = v;
    }
    (void)total;
}
__global__ void copy_limbs_scalar_kernel(u64* __restrict__ dst, long long ds, const u64* __restrict__ src,
                                         long long ss, long long per_poly) {
    const long long p = blockIdx.y;
    const long long o = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (o < per_poly) dst[p * ds + o] = src[p * ss + o];
}

cudaError_t copy_limbs_op(u64* dst, long long ds, const u64* src, long long ss, int npoly, long long per_poly,
                          cudaStream_t st) {
    long long total = (long long)npoly * per_poly;
    if (!total) return cudaSuccess;
    if (npoly > 65535) return cudaErrorInvalidValue;
    const bool vec = per_poly % 2 == 0 && ds % 2 == 0 && ss % 2 == 0 && ((uintptr_t)dst & 15) == 0 &&
                     ((uintptr_t)src & 15) == 0;
    if (vec)
        copy_limbs_kernel<<<dim3((unsigned)((per_poly / 2 + 255) / 256), npoly), 256, 0, st>>>(dst, ds, src, ss, per_poly,
                                                                                           total);
    else
        copy_limbs_scalar_kernel<<<dim3((unsigned)((per_poly + 255) / 256), npoly), 256, 0, st>>>(dst, ds, src, ss,
                                                                                               per_poly);
    return launched();
}

}  // namespace bcn
