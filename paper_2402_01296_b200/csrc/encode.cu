// encode.cu -- canonical embedding (K9), encryption randomness (K10),
// decryption (K11) and switching-key generation.
//
// The special FFT runs in float64 with every add/sub/mul spelled with the
// _rn intrinsics (and -fmad=false), in exactly the order oracle/ckks.py
// uses, so GPU and oracle produce the same coefficient bits.  Randomness is
// Philox4x32-10 keyed by (seed) with counters (n, limb | domain << 16, id):
// the same stream the oracle reads.
#include "common.cuh"
#include "ops.cuh"

namespace bcn {

// ---------------------------------------------------------------- encode
// out[p][t][i] = round(scale * m_i) (+ e_i) mod q_t, coefficient domain.
__global__ void encode_kernel(u64* __restrict__ out, long long os, const double* __restrict__ vals, int vlen,
                              long long vs, double scale, int logn, Limbs limbs, const PrimeInfo* __restrict__ pr,
                              FftTab ft, int add_err, u64 seed, u64 id_base, const u64* __restrict__ id_dev,
                              i64* __restrict__ raw) {
    extern __shared__ double fsm[];
    const int N = 1 << logn, S = N >> 1, M = N << 1, logs = logn - 1;
    if (id_dev) id_base = *id_dev;   // graph replays: the encryption counter lives in device memory
    double* xr = fsm;
    double* xi = fsm + S;
    const int p = blockIdx.x;
    const double* v = vals + (long long)p * vs;
    for (int j = threadIdx.x; j < S; j += blockDim.x) {
        xr[j] = j < vlen ? v[j] : 0.0;
        xi[j] = 0.0;
    }
    __syncthreads();
    for (int len = S; len >= 2; len >>= 1) {
        const int h = len >> 1, lenq = len << 2, lgh = __ffs(h) - 1;
        for (int pr_ = threadIdx.x; pr_ < (S >> 1); pr_ += blockDim.x) {
            const int blk = pr_ >> lgh, jj = pr_ & (h - 1);      // h, lenq: powers of two
            const int i1 = blk * len + jj, i2 = i1 + h;
            const int idx = (lenq - (ft.rot[jj] & (lenq - 1))) << (logn + 1 - lgh - 3);   // M / lenq, M = 2N = 2^(logn+1), lenq = 8h
            const double tr = ft.re[idx], ti = ft.im[idx];
            const double ar = xr[i1], ai = xi[i1], cr = xr[i2], ci = xi[i2];
            const double ur = __dadd_rn(ar, cr), ui = __dadd_rn(ai, ci);
            const double dr = __dsub_rn(ar, cr), di = __dsub_rn(ai, ci);
            xr[i1] = ur;
            xi[i1] = ui;
            xr[i2] = __dsub_rn(__dmul_rn(dr, tr), __dmul_rn(di, ti));
            xi[i2] = __dadd_rn(__dmul_rn(dr, ti), __dmul_rn(di, tr));
        }
        __syncthreads();
    }
    const double invS = 1.0 / (double)S;
    u64* o = out + (long long)p * os;
    for (int i = threadIdx.x; i < S; i += blockDim.x) {
        const int src = logs > 0 ? (int)brev_bits((u32)i, logs) : 0;
        const double wr = __dmul_rn(xr[src], invS), wi = __dmul_rn(xi[src], invS);
        i64 cr = (i64)rint(__dmul_rn(wr, scale));
        i64 ci = (i64)rint(__dmul_rn(wi, scale));
        if (raw) {                                   // the integer coefficients only (encode_rot_kernel finishes)
            raw[(long long)p * N + i] = cr;
            raw[(long long)p * N + i + S] = ci;
            continue;
        }
        if (add_err) {
            cr += cbd21(draw(seed, 2u /*DOM_ENC_E*/, 0u, id_base + p, (u32)i));
            ci += cbd21(draw(seed, 2u, 0u, id_base + p, (u32)(i + S)));
        }
        for (int t = 0; t < limbs.n; t++) {
            const PrimeInfo& P = pr[limbs.prime[t]];
            o[(long long)t * N + i] = signed_to_residue_fast(cr, P.q, P.pad[2]);
            o[(long long)t * N + i + S] = signed_to_residue_fast(ci, P.q, P.pad[2]);
        }
    }
}

cudaError_t encode_op(u64* out, long long os, const double* vals, int vlen, long long vs, int nplain, double scale,
                      int logn, const Limbs& limbs, const PrimeInfo* pr, const FftTab& ft, int add_err, u64 seed,
                      u64 id_base, cudaStream_t st, const u64* id_dev, i64* raw) {
    if (!nplain) return cudaSuccess;
    const int N = 1 << logn;
    const size_t smem = (size_t)N * sizeof(double);
    static unsigned long long smem_cfg = 0;
    unsigned long long smem_bit = 0;
    if (first_on_device(&smem_cfg, &smem_bit)) {
        cudaError_t ae = cudaSuccess;
        BCN_SMEM_ATTR(ae, (encode_kernel), 200 * 1024);
        if (ae != cudaSuccess) return ae;
        smem_cfg |= smem_bit;
    }
    // threads per plaintext: a stage is N/4 butterflies behind one barrier, each with two table loads from
    // L2, so the fewer butterflies per thread the shorter the chain (BCN_FFT_TPB: 512 was the default before)
    static const int tpb_max = getenv("BCN_FFT_TPB") ? atoi(getenv("BCN_FFT_TPB")) : 1024;
    int tpb = N / 4 < tpb_max ? (N / 4 < 32 ? 32 : N / 4) : tpb_max;
    encode_kernel<<<nplain, tpb, smem, st>>>(out, os, vals, vlen, vs, scale, logn, limbs, pr, ft, add_err, seed,
                                             id_base, id_dev, raw);
    return launched();
}

// Fresh encryptions of rotated copies of the same plaintexts: the plaintext of rot_r(x) is the
// automorphism X -> X^g (g = 5^r) of the plaintext of x, an exact signed permutation of its integer
// coefficients -- out[i] = +-m[i g^-1 mod 2N] -- so the canonical embedding runs once per plaintext and
// each copy adds its own fresh error and reduces:
//   out[(c G + p)][t][i] = (sigma_gc(m_p)[i] + e_{id + c G + p}[i]) mod q_t     (coefficient domain)
struct RotCopies {
    int n;
    u32 ginv[32];                      // g^-1 mod 2N per copy (1: the plaintext itself)
};
__global__ void __launch_bounds__(256) encode_rot_kernel(u64* __restrict__ out, long long os,
                                                         const i64* __restrict__ raw, int G, int logn, Limbs limbs,
                                                         const PrimeInfo* __restrict__ pr, RotCopies rc, u64 seed,
                                                         u64 id_base) {
    const int N = 1 << logn;
    const int i = blockIdx.x * 256 + threadIdx.x;
    if (i >= N) return;
    const int c = blockIdx.y, p = blockIdx.z;
    const u32 j = ((u32)i * rc.ginv[c]) & (u32)(2 * N - 1);
    const i64 m = j < (u32)N ? raw[(long long)p * N + j] : -raw[(long long)p * N + (j - N)];
    const long long row = (long long)c * G + p;
    const i64 v = m + cbd21(draw(seed, 2u /*DOM_ENC_E*/, 0u, id_base + (u64)row, (u32)i));
    u64* o = out + row * os + i;
    for (int t = 0; t < limbs.n; t++) {
        const PrimeInfo& P = pr[limbs.prime[t]];
        o[(long long)t * N] = signed_to_residue_fast(v, P.q, P.pad[2]);
    }
}

cudaError_t encode_rot_op(u64* out, long long os, const i64* raw, int G, int logn, const Limbs& limbs,
                          const PrimeInfo* pr, int n_copies, const u32* ginv, u64 seed, u64 id_base, cudaStream_t st) {
    if (n_copies < 1 || n_copies > 32 || G > 65535) return cudaErrorInvalidValue;
    RotCopies rc;
    rc.n = n_copies;
    for (int c = 0; c < n_copies; c++) rc.ginv[c] = ginv[c];
    const int N = 1 << logn;
    dim3 grid((N + 255) / 256, n_copies, G);
    encode_rot_kernel<<<grid, 256, 0, st>>>(out, os, raw, G, logn, limbs, pr, rc, seed, id_base);
    return launched();
}

// ---------------------------------------------------------------- decode
// poly: [npoly][k][N] coefficient residues mod q0 (and q1); out: [npoly][nout]
__device__ __forceinline__ double crt_value(u64 x0, u64 x1, int k, const PrimeInfo& P0, const PrimeInfo& P1,
                                            u64 q0inv, u64 q0inv_p) {
    const u64 q0 = P0.q;
    if (k == 1) {
        i64 m = x0 > (q0 >> 1) ? (i64)x0 - (i64)q0 : (i64)x0;
        return __ll2double_rn(m);
    }
    const u64 q1 = P1.q;
    const u64 x0r = x0 % q1;
    const u64 y = shoup(sub_mod(x1, x0r, q1), q0inv, q0inv_p, q1);
    // m = x0 + q0 * y  (u128)
    u64 lo = q0 * y, hi = umulhi(q0, y);
    u64 nlo = lo + x0;
    hi += (nlo < lo);
    lo = nlo;
    // Q = q0 q1; centre: m > (Q-1)/2 -> m - Q
    const u64 Qlo = q0 * q1, Qhi = umulhi(q0, q1);
    // half = (Q - 1) >> 1 ; Q odd
    const u64 hlo = ((Qlo - 1) >> 1) | (Qhi << 63), hhi = Qhi >> 1;
    if (hi > hhi || (hi == hhi && lo > hlo)) {
        const u64 blo = lo - Qlo;
        hi = hi - Qhi - (lo < Qlo);
        lo = blo;
    }
    const bool fits = (hi == 0 && (lo >> 63) == 0) || (hi == ~0ull && (lo >> 63) == 1);
    if (fits) return __ll2double_rn((i64)lo);
    return __dadd_rn(__dmul_rn(__ll2double_rn((i64)hi), 18446744073709551616.0), __ull2double_rn(lo));
}

__global__ void decode_kernel(double* __restrict__ out, int nout, const u64* __restrict__ poly, long long ps, int k,
                              double scale, int logn, const PrimeInfo* __restrict__ pr, FftTab ft, u64 q0inv,
                              u64 q0inv_p) {
    extern __shared__ double fsm[];
    const int N = 1 << logn, S = N >> 1, M = N << 1, logs = logn - 1;
    double* xr = fsm;
    double* xi = fsm + S;
    const int p = blockIdx.x;
    const u64* P = poly + (long long)p * ps;
    const PrimeInfo P0 = pr[0], P1 = pr[1];
    for (int i = threadIdx.x; i < S; i += blockDim.x) {
        const int dst = logs > 0 ? (int)brev_bits((u32)i, logs) : 0;   // bit-reversed load
        const double mr = crt_value(P[i], k > 1 ? P[N + i] : 0ull, k, P0, P1, q0inv, q0inv_p);
        const double mi = crt_value(P[i + S], k > 1 ? P[N + i + S] : 0ull, k, P0, P1, q0inv, q0inv_p);
        xr[dst] = __ddiv_rn(mr, scale);
        xi[dst] = __ddiv_rn(mi, scale);
    }
    __syncthreads();
    for (int len = 2; len <= S; len <<= 1) {
        const int h = len >> 1, lenq = len << 2, lgh = __ffs(h) - 1;
        for (int pr_ = threadIdx.x; pr_ < (S >> 1); pr_ += blockDim.x) {
            const int blk = pr_ >> lgh, jj = pr_ & (h - 1);      // h, lenq: powers of two
            const int i1 = blk * len + jj, i2 = i1 + h;
            const int idx = (ft.rot[jj] & (lenq - 1)) << (logn + 1 - lgh - 3);   // M / lenq, M = 2N = 2^(logn+1), lenq = 8h
            const double tr = ft.re[idx], ti = ft.im[idx];
            const double ur = xr[i1], ui = xi[i1], cr = xr[i2], ci = xi[i2];
            const double vr = __dsub_rn(__dmul_rn(cr, tr), __dmul_rn(ci, ti));
            const double vi = __dadd_rn(__dmul_rn(cr, ti), __dmul_rn(ci, tr));
            xr[i1] = __dadd_rn(ur, vr);
            xi[i1] = __dadd_rn(ui, vi);
            xr[i2] = __dsub_rn(ur, vr);
            xi[i2] = __dsub_rn(ui, vi);
        }
        __syncthreads();
    }
    for (int j = threadIdx.x; j < nout; j += blockDim.x) out[(long long)p * nout + j] = xr[j];
}

cudaError_t decode_op(double* out, int nout, const u64* poly, long long ps, int k, int npoly, double scale, int logn,
                      const PrimeInfo* pr, const FftTab& ft, u64 q0inv_mod_q1, u64 q0inv_p, cudaStream_t st) {
    if (!npoly) return cudaSuccess;
    const int N = 1 << logn;
    const size_t smem = (size_t)N * sizeof(double);
    static unsigned long long smem_cfg = 0;
    unsigned long long smem_bit = 0;
    if (first_on_device(&smem_cfg, &smem_bit)) {
        cudaError_t ae = cudaSuccess;
        BCN_SMEM_ATTR(ae, (decode_kernel), 200 * 1024);
        if (ae != cudaSuccess) return ae;
        smem_cfg |= smem_bit;
    }
    // threads per plaintext: a stage is N/4 butterflies behind one barrier, each with two table loads from
    // L2, so the fewer butterflies per thread the shorter the chain (BCN_FFT_TPB: 512 was the default before)
    static const int tpb_max = getenv("BCN_FFT_TPB") ? atoi(getenv("BCN_FFT_TPB")) : 1024;
    int tpb = N / 4 < tpb_max ? (N / 4 < 32 ? 32 : N / 4) : tpb_max;
    decode_kernel<<<npoly, tpb, smem, st>>>(out, nout, poly, ps, k, scale, logn, pr, ft, q0inv_mod_q1, q0inv_p);
    return launched();
}

// ------------------------------------------------------------- sampling
__global__ void sample_uniform_kernel(u64* __restrict__ out, long long os, int nlimb, int logn, Limbs limbs,
                                      const PrimeInfo* __restrict__ pr, u64 seed, u32 domain, u64 id_base,
                                      u64 id_step, long long total) {
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int n = (int)(idx & ((1 << logn) - 1));
        long long rest = idx >> logn;
        const int t = (int)(rest % nlimb);
        const long long p = rest / nlimb;
        const int pi = limbs.prime[t];
        out[p * os + ((long long)t << logn) + n] =
            uniform_mod(draw(seed, domain, (u32)pi, id_base + (u64)p * id_step, (u32)n), pr[pi]);
    }
}

cudaError_t sample_uniform_op(u64* out, long long os, int npoly, int nlimb, int logn, const Limbs& limbs,
                              const PrimeInfo* pr, u64 seed, u32 domain, u64 id_base, u64 id_step, cudaStream_t st) {
    long long total = (long long)npoly * nlimb << logn;
    if (!total) return cudaSuccess;
    long long nb = (total + 255) / 256;
    sample_uniform_kernel<<<(int)(nb > 1048576 ? 1048576 : nb), 256, 0, st>>>(out, os, nlimb, logn, limbs, pr, seed,
                                                                               domain, id_base, id_step, total);
    return launched();
}

__global__ void sample_small_kernel(u64* __restrict__ out, long long os, int nlimb, int logn, Limbs limbs,
                                    const PrimeInfo* __restrict__ pr, u64 seed, u32 domain, u64 id_base,
                                    u64 id_step, int ternary, long long total) {
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int n = (int)(idx & ((1 << logn) - 1));
        const long long p = idx >> logn;
        const uint4 o = draw(seed, domain, 0u, id_base + (u64)p * id_step, (u32)n);
        const i64 v = ternary ? (i64)(o.x % 3u) - 1 : cbd21(o);
        for (int t = 0; t < nlimb; t++)
            out[p * os + ((long long)t << logn) + n] = signed_to_residue_fast(v, pr[limbs.prime[t]].q,
                                                                                pr[limbs.prime[t]].pad[2]);
    }
}

cudaError_t sample_small_op(u64* out, long long os, int npoly, int nlimb, int logn, const Limbs& limbs,
                            const PrimeInfo* pr, u64 seed, u32 domain, u64 id_base, u64 id_step, int ternary,
                            cudaStream_t st) {
    long long total = (long long)npoly << logn;
    if (!total) return cudaSuccess;
    sample_small_kernel<<<(int)((total + 255) / 256), 256, 0, st>>>(out, os, nlimb, logn, limbs, pr, seed, domain,
                                                                    id_base, id_step, ternary, total);
    return launched();
}

// ct: [G][2][L][N]; c0 holds NTT(m + e) on entry.  c1 = a, c0 -= a s.
__global__ void __launch_bounds__(256) encrypt_combine_kernel(u64* __restrict__ ct, int nlimb, int logn, Limbs limbs,
                                                              const PrimeInfo* __restrict__ pr,
                                                              const u64* __restrict__ s_mont, u64 seed, u64 id_base,
                                                              u64 g_off, const u64* __restrict__ id_dev) {
    // grid (N / 256, limb, slot set): no 64-bit index division per word, the prime's constants per block
    const int N = 1 << logn;
    if (id_dev) id_base = *id_dev;
    const int n = blockIdx.x * 256 + threadIdx.x;
    if (n >= N) return;
    const int t = blockIdx.y;
    const long long g = blockIdx.z;
    const int pi = limbs.prime[t];
    const PrimeInfo& P = pr[pi];
    const u64 a = uniform_mod(draw(seed, 1u /*DOM_ENC_A*/, (u32)pi, id_base + g_off + (u64)g, (u32)n), P);
    u64* c0 = ct + g * 2 * nlimb * (long long)N + (long long)t * N + n;
    const u64 as = mont_mul(a, s_mont[(long long)pi * N + n], P.q, P.qinv_neg);
    c0[0] = sub_mod(c0[0], as, P.q);
    c0[(long long)nlimb * N] = a;
}

cudaError_t encrypt_combine_op(u64* ct, int G, int nlimb, int logn, const Limbs& limbs, const PrimeInfo* pr,
                               const u64* s_mont, u64 seed, u64 id_base, cudaStream_t st, const u64* id_dev) {
    if (G <= 0 || nlimb <= 0) return cudaSuccess;
    const int N = 1 << logn;
    for (int g0 = 0; g0 < G; g0 += 65535) {                 // grid.z limit
        const int gc = G - g0 < 65535 ? G - g0 : 65535;
        dim3 grid((N + 255) / 256, nlimb, gc);
        encrypt_combine_kernel<<<grid, 256, 0, st>>>(ct + (size_t)g0 * 2 * nlimb * N, nlimb, logn, limbs, pr, s_mont,
                                                     seed, id_base, (u64)g0, id_dev);
    }
    return launched();
}

// one digit of a switching key over the full basis (nbasis limbs, prime t = t):
//   a = U(DOM_KSK_A, kid), b = -a s + e + [d0 <= t < d1] (P mod q_t) s'_t ;
// both stored in Montgomery form.
__global__ void ksk_digit_kernel(u64* __restrict__ b_out, u64* __restrict__ a_out, const u64* __restrict__ e_ntt,
                                 const u64* __restrict__ s_mont, const u64* __restrict__ sprime, int nbasis, int d0,
                                 int d1, int logn, const PrimeInfo* __restrict__ pr, const u64* __restrict__ pmod,
                                 u64 seed, u64 kid, long long total) {
    const int N = 1 << logn;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int n = (int)(idx & (N - 1));
        const int t = (int)(idx >> logn);
        const PrimeInfo& P = pr[t];
        const u64 q = P.q;
        const u64 a = uniform_mod(draw(seed, 4u /*DOM_KSK_A*/, (u32)t, kid, (u32)n), P);
        u64 b = sub_mod(e_ntt[idx], mont_mul(a, s_mont[idx], q, P.qinv_neg), q);
        if (t >= d0 && t < d1) b = add_mod(b, shoup(sprime[idx], pmod[2 * t], pmod[2 * t + 1], q), q);
        b_out[idx] = to_mont(b, P);
        a_out[idx] = to_mont(a, P);
    }
    (void)nbasis;
}

cudaError_t ksk_digit_op(u64* b_out, u64* a_out, const u64* e_ntt, const u64* s_mont, const u64* sprime,
                         int nbasis, int d0, int d1, int logn, const PrimeInfo* pr, const u64* pmod, u64 seed,
                         u64 kid, cudaStream_t st) {
    long long total = (long long)nbasis << logn;
    ksk_digit_kernel<<<(int)((total + 255) / 256), 256, 0, st>>>(b_out, a_out, e_ntt, s_mont, sprime, nbasis, d0, d1,
                                                                 logn, pr, pmod, seed, kid, total);
    return launched();
}

// m = c0 + c1 s on limbs 0..k-1 (NTT domain), out: [npoly][k][N]
__global__ void decrypt_core_kernel(u64* __restrict__ out, const u64* __restrict__ ct, long long cs, int nlimb_ct,
                                    int k, int logn, const PrimeInfo* __restrict__ pr,
                                    const u64* __restrict__ s_mont, long long total) {
    const int N = 1 << logn;
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int n = (int)(idx & (N - 1));
        long long rest = idx >> logn;
        const int t = (int)(rest % k);
        const long long p = rest / k;
        const PrimeInfo& P = pr[t];
        const u64* c = ct + p * cs + (long long)t * N + n;
        const u64 v = mont_mul(c[(long long)nlimb_ct * N], s_mont[(long long)t * N + n], P.q, P.qinv_neg);
        out[idx] = add_mod(c[0], v, P.q);
    }
}

cudaError_t decrypt_core_op(u64* out, const u64* ct, long long cs, int nlimb_ct, int k, int npoly, int logn,
                            const PrimeInfo* pr, const u64* s_mont, long long s_stride, cudaStream_t st) {
    (void)s_stride;
    long long total = (long long)npoly * k << logn;
    if (!total) return cudaSuccess;
    decrypt_core_kernel<<<(int)((total + 255) / 256), 256, 0, st>>>(out, ct, cs, nlimb_ct, k, logn, pr, s_mont,
                                                                    total);
    return launched();
}

__global__ void from_mont_kernel(u64* out, const u64* in, long long per_limb, int nlimb, Limbs limbs,
                                 const PrimeInfo* __restrict__ pr, long long total) {
    for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int t = (int)((idx / per_limb) % nlimb);
        const PrimeInfo& P = pr[limbs.prime[t]];
        out[idx] = redc(0ull, in[idx], P.q, P.qinv_neg);
    }
}

cudaError_t from_mont_op(u64* out, const u64* in, long long per_limb, int nlimb, int npoly, const Limbs& limbs,
                         const PrimeInfo* pr, cudaStream_t st) {
    long long total = (long long)npoly * nlimb * per_limb;
    if (!total) return cudaSuccess;
    from_mont_kernel<<<(int)((total + 255) / 256), 256, 0, st>>>(out, in, per_limb, nlimb, limbs, pr, total);
    return launched();
}

}  // namespace bcn
