/*
 * ckks_oracle.c -- CPU restatement of the RNS-CKKS integer primitives.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links or calls
 * this file; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs load it, as the checker or the timed CPU baseline.
 *
 * Why it exists: the reference (pkg/src/bibranch/sim.py:1-12) simulates CKKS
 * semantics on float64 slot vectors and holds no lattice arithmetic
 * (SPEC.md:18).  The ciphertext-level parity source therefore has to be
 * written here: every function below is the plain, exact (unsigned __int128)
 * form of the algorithm the CUDA kernels compute with lazy reductions and
 * Montgomery/Shoup tricks.  All outputs are canonical residues in [0, q).
 *
 * The scheme-level composition (encode, keygen, encrypt, key switch,
 * rescale, ...) lives in oracle/ckks.py; this file only holds the loops that
 * would be too slow in numpy.  Bit-exactness contract: DESIGN.md section 3.
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>
#include <stdlib.h>

typedef unsigned __int128 u128;

static inline uint64_t mulmod(uint64_t a, uint64_t b, uint64_t q) {
    return (uint64_t)(((u128)a * b) % q);
}

uint64_t orc_powmod(uint64_t a, uint64_t e, uint64_t q) {
    uint64_t r = 1 % q;
    a %= q;
    while (e) {
        if (e & 1) r = mulmod(r, a, q);
        a = mulmod(a, a, q);
        e >>= 1;
    }
    return r;
}

/* Deterministic Miller-Rabin for 64-bit integers (bases = first 12 primes). */
int orc_is_prime(uint64_t n) {
    static const uint64_t bases[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return 0;
    for (int i = 0; i < 12; i++) {
        if (n == bases[i]) return 1;
        if (n % bases[i] == 0) return 0;
    }
    uint64_t d = n - 1;
    int s = 0;
    while ((d & 1) == 0) { d >>= 1; s++; }
    for (int i = 0; i < 12; i++) {
        uint64_t x = orc_powmod(bases[i], d, n);
        if (x == 1 || x == n - 1) continue;
        int comp = 1;
        for (int r = 1; r < s; r++) {
            x = mulmod(x, x, n);
            if (x == n - 1) { comp = 0; break; }
        }
        if (comp) return 0;
    }
    return 1;
}

static inline uint32_t brev(uint32_t x, int bits) {
    uint32_t r = 0;
    for (int i = 0; i < bits; i++) { r = (r << 1) | (x & 1); x >>= 1; }
    return r;
}

static int ilog2(size_t n) { int b = 0; while (((size_t)1 << b) < n) b++; return b; }

/* W[k] = psi^brev(k), Winv[k] = psi^-brev(k), k < N. */
void orc_ntt_tables(size_t N, uint64_t q, uint64_t psi, uint64_t *W, uint64_t *Winv) {
    int lg = ilog2(N);
    uint64_t psi_inv = orc_powmod(psi, q - 2, q);
    uint64_t p = 1, pi = 1;
    uint64_t *pw = (uint64_t *)malloc(N * sizeof(uint64_t));
    uint64_t *pwi = (uint64_t *)malloc(N * sizeof(uint64_t));
    for (size_t k = 0; k < N; k++) {
        pw[k] = p; pwi[k] = pi;
        p = mulmod(p, psi, q); pi = mulmod(pi, psi_inv, q);
    }
    for (size_t k = 0; k < N; k++) {
        W[k] = pw[brev((uint32_t)k, lg)];
        Winv[k] = pwi[brev((uint32_t)k, lg)];
    }
    free(pw); free(pwi);
}

/* Forward negacyclic NTT (Cooley-Tukey, natural in -> bit-reversed out):
 * a[k] <- sum_j a_j psi^{(2 brev(k) + 1) j}.  `count` independent polys. */
void orc_ntt_fwd(uint64_t *a, size_t count, size_t N, uint64_t q, const uint64_t *W) {
    #pragma omp parallel for schedule(static)
    for (size_t c = 0; c < count; c++) {
        uint64_t *x = a + c * N;
        size_t t = N;
        for (size_t m = 1; m < N; m <<= 1) {
            t >>= 1;
            for (size_t i = 0; i < m; i++) {
                uint64_t w = W[m + i];
                size_t j0 = 2 * i * t;
                for (size_t j = j0; j < j0 + t; j++) {
                    uint64_t u = x[j];
                    uint64_t v = mulmod(x[j + t], w, q);
                    uint64_t s = u + v; if (s >= q) s -= q;
                    uint64_t d = u >= v ? u - v : u + q - v;
                    x[j] = s; x[j + t] = d;
                }
            }
        }
    }
}

/* Inverse (Gentleman-Sande, bit-reversed in -> natural out), times N^-1. */
void orc_ntt_inv(uint64_t *a, size_t count, size_t N, uint64_t q, const uint64_t *Winv, uint64_t n_inv) {
    #pragma omp parallel for schedule(static)
    for (size_t c = 0; c < count; c++) {
        uint64_t *x = a + c * N;
        size_t t = 1;
        for (size_t m = N; m > 1; m >>= 1) {
            size_t h = m >> 1;
            for (size_t i = 0; i < h; i++) {
                uint64_t w = Winv[h + i];
                size_t j0 = 2 * i * t;
                for (size_t j = j0; j < j0 + t; j++) {
                    uint64_t u = x[j], v = x[j + t];
                    uint64_t s = u + v; if (s >= q) s -= q;
                    uint64_t d = u >= v ? u - v : u + q - v;
                    x[j] = s; x[j + t] = mulmod(d, w, q);
                }
            }
            t <<= 1;
        }
        for (size_t j = 0; j < N; j++) x[j] = mulmod(x[j], n_inv, q);
    }
}

void orc_mul_vec(const uint64_t *a, const uint64_t *b, uint64_t *out, size_t n, uint64_t q) {
    #pragma omp parallel for schedule(static)
    for (size_t i = 0; i < n; i++) out[i] = mulmod(a[i], b[i], q);
}

void orc_mul_scalar(const uint64_t *a, uint64_t s, uint64_t *out, size_t n, uint64_t q) {
    #pragma omp parallel for schedule(static)
    for (size_t i = 0; i < n; i++) out[i] = mulmod(a[i], s, q);
}

/* out = sum_t a_t * b_t mod q over T terms, each of n words (a: T x n, b: T x n). */
void orc_mac(const uint64_t *a, const uint64_t *b, uint64_t *out, size_t T, size_t n, uint64_t q) {
    #pragma omp parallel for schedule(static)
    for (size_t i = 0; i < n; i++) {
        uint64_t acc = 0;
        for (size_t t = 0; t < T; t++) {
            acc += mulmod(a[t * n + i], b[t * n + i], q);
            if (acc >= q) acc -= q;
        }
        out[i] = acc;
    }
}

/* ---- Philox4x32-10 (Salmon et al., SC'11), counter-based PRNG ---- */
void orc_philox(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; r++) {
        if (r) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        c0 = hi1 ^ c1 ^ k0;
        c1 = lo1;
        c2 = hi0 ^ c3 ^ k1;
        c3 = lo0;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Counter layout shared with the CUDA samplers:
 *   ctr = (n, limb | domain << 16, id_lo, id_hi), key = (seed_lo, seed_hi). */
static inline void draw(uint64_t seed, uint32_t domain, uint32_t limb, uint64_t id, uint32_t n, uint32_t o[4]) {
    uint32_t ctr[4] = {n, limb | (domain << 16), (uint32_t)id, (uint32_t)(id >> 32)};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    orc_philox(ctr, key, o);
}

/* uniform residue: ((o1:o0) * 2^64 + (o3:o2)) mod q */
void orc_sample_uniform(uint64_t *out, size_t N, uint64_t q, uint64_t seed,
                        uint32_t domain, uint32_t limb, uint64_t id) {
    #pragma omp parallel for schedule(static)
    for (size_t n = 0; n < N; n++) {
        uint32_t o[4];
        draw(seed, domain, limb, id, (uint32_t)n, o);
        uint64_t x = ((uint64_t)o[1] << 32) | o[0];
        uint64_t y = ((uint64_t)o[3] << 32) | o[2];
        out[n] = (uint64_t)((((u128)x << 64) | y) % q);
    }
}

/* centred binomial, eta = 21: popcount(o0 & M) - popcount(o1 & M) */
void orc_sample_cbd(int64_t *out, size_t N, uint64_t seed, uint32_t domain, uint64_t id) {
    for (size_t n = 0; n < N; n++) {
        uint32_t o[4];
        draw(seed, domain, 0, id, (uint32_t)n, o);
        out[n] = (int64_t)__builtin_popcount(o[0] & 0x1FFFFFu) - (int64_t)__builtin_popcount(o[1] & 0x1FFFFFu);
    }
}

/* uniform ternary: (o0 mod 3) - 1 */
void orc_sample_ternary(int64_t *out, size_t N, uint64_t seed, uint32_t domain, uint64_t id) {
    for (size_t n = 0; n < N; n++) {
        uint32_t o[4];
        draw(seed, domain, 0, id, (uint32_t)n, o);
        out[n] = (int64_t)(o[0] % 3u) - 1;
    }
}

/* Fast (approximate) RNS base conversion, coefficient domain.
 * in: n_src x N residues of x modulo src_q[i]; out: n_dst x N with
 *   out_t = sum_i [x_i * (Qs/q_i)^-1]_{q_i} * (Qs/q_i)  mod dst_q[t]
 * -- the exact integer sum reduced mod t (no overflow correction). */
void orc_base_conv(const uint64_t *in, size_t n_src, const uint64_t *src_q,
                   uint64_t *out, size_t n_dst, const uint64_t *dst_q, size_t N) {
    uint64_t *hat_inv = (uint64_t *)malloc(n_src * sizeof(uint64_t));
    uint64_t *hat_mod = (uint64_t *)malloc(n_src * n_dst * sizeof(uint64_t));
    for (size_t i = 0; i < n_src; i++) {
        uint64_t qi = src_q[i], prod = 1;
        for (size_t k = 0; k < n_src; k++) if (k != i) prod = mulmod(prod, src_q[k] % qi, qi);
        hat_inv[i] = orc_powmod(prod, qi - 2, qi);
        for (size_t t = 0; t < n_dst; t++) {
            uint64_t qt = dst_q[t], pm = 1;
            for (size_t k = 0; k < n_src; k++) if (k != i) pm = mulmod(pm, src_q[k] % qt, qt);
            hat_mod[i * n_dst + t] = pm;
        }
    }
    #pragma omp parallel for schedule(static)
    for (size_t n = 0; n < N; n++) {
        uint64_t y[64];
        for (size_t i = 0; i < n_src; i++) y[i] = mulmod(in[i * N + n], hat_inv[i], src_q[i]);
        for (size_t t = 0; t < n_dst; t++) {
            uint64_t qt = dst_q[t];
            u128 acc = 0;
            for (size_t i = 0; i < n_src; i++) acc += (u128)y[i] * hat_mod[i * n_dst + t];
            out[t * N + n] = (uint64_t)(acc % qt);
        }
    }
    free(hat_inv); free(hat_mod);
}

/* Automorphism X -> X^g on the bit-reversed NTT domain: pure permutation
 *   out[k] = in[pi(k)],  2 brev(pi(k)) + 1 = g (2 brev(k) + 1) mod 2N. */
void orc_automorph_ntt(const uint64_t *in, uint64_t *out, size_t count, size_t N, uint64_t g) {
    int lg = ilog2(N);
    uint64_t M = 2 * N;
    #pragma omp parallel for schedule(static)
    for (size_t c = 0; c < count; c++) {
        for (size_t k = 0; k < N; k++) {
            uint64_t e = (2 * (uint64_t)brev((uint32_t)k, lg) + 1) * g % M;
            size_t src = brev((uint32_t)((e - 1) >> 1), lg);
            out[c * N + k] = in[c * N + src];
        }
    }
}

/* Automorphism in the coefficient domain: X^i -> X^{ig mod 2N}, with the
 * negacyclic sign when ig mod 2N >= N. */
void orc_automorph_coef(const uint64_t *in, uint64_t *out, size_t N, uint64_t g, uint64_t q) {
    uint64_t M = 2 * N;
    for (size_t i = 0; i < N; i++) {
        uint64_t e = (uint64_t)i * g % M;
        uint64_t v = in[i];
        if (e >= N) { e -= N; v = v ? q - v : 0; }
        out[e] = v;
    }
}
