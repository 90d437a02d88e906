// common.cuh -- shared device helpers for the sm_100a RNS-CKKS engine.
//
// Word type: u64 residues, primes q < 2^61 (4q < 2^63 for Harvey lazy
// butterflies).  Three modular-multiply flavours, chosen per operand kind:
//   * Shoup   -- constant operand w with companion w' = floor(w 2^64 / q)
//                (NTT twiddles, q_l^-1, P^-1, base-conversion scalars);
//   * Montgomery REDC -- stored operands kept as x*2^64 mod q (switching
//                keys, plaintext multipliers, the secret key);
//   * u128 lazy accumulation of several products followed by ONE REDC.
// Every value written back to HBM is canonical ([0, q)) so ciphertexts are
// comparable bit for bit with oracle/ckks.py.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

typedef unsigned long long u64;
typedef long long i64;
typedef unsigned int u32;

#define BCN_MAX_LIMBS 64

struct PrimeInfo {
    u64 q;          // modulus
    u64 qinv_neg;   // -q^-1 mod 2^64      (Montgomery)
    u64 r2;         // 2^128 mod q         (to-Montgomery)
    u64 r1;         // 2^64 mod q
    u64 r1_shoup;   // floor(r1 * 2^64 / q)
    u64 pad[3];
};

// limb t of a buffer lives modulo prime[t] (index into the context's basis)
struct Limbs {
    int n;
    short prime[BCN_MAX_LIMBS];
};

__device__ __forceinline__ u64 umulhi(u64 a, u64 b) { return __umul64hi(a, b); }

// a*w mod q in [0, 2q) for any 64-bit a; w < q, wp = floor(w 2^64 / q)
__device__ __forceinline__ u64 shoup_lazy(u64 a, u64 w, u64 wp, u64 q) {
    return a * w - umulhi(a, wp) * q;
}
__device__ __forceinline__ u64 shoup(u64 a, u64 w, u64 wp, u64 q) {
    u64 r = shoup_lazy(a, w, wp, q);
    return r >= q ? r - q : r;
}

// (hi:lo) * 2^-64 mod q for hi < q; result canonical
__device__ __forceinline__ u64 redc(u64 hi, u64 lo, u64 q, u64 qinv_neg) {
    u64 m = lo * qinv_neg;
    u64 r = hi + umulhi(m, q) + (lo != 0ull ? 1ull : 0ull);
    return r >= q ? r - q : r;
}

// a * b_mont * 2^-64 mod q  (b_mont = b 2^64 mod q  ->  a*b mod q)
__device__ __forceinline__ u64 mont_mul(u64 a, u64 b, u64 q, u64 qinv_neg) {
    return redc(umulhi(a, b), a * b, q, qinv_neg);
}

__device__ __forceinline__ u64 to_mont(u64 a, const PrimeInfo& p) {
    return mont_mul(a, p.r2, p.q, p.qinv_neg);
}

// lazy u128 accumulator: keeps hi < q so REDC applies at the end
struct Acc128 {
    u64 hi, lo;
    __device__ __forceinline__ void zero() { hi = 0; lo = 0; }
    __device__ __forceinline__ void mac(u64 a, u64 b, u64 q) {
        u64 pl = a * b, ph = umulhi(a, b);
        u64 nl = lo + pl;
        hi += ph + (nl < lo ? 1ull : 0ull);
        lo = nl;
        if (hi >= q) hi -= q;
    }
    // unreduced MAC: a, b < q < 2^61 adds floor(ab / 2^64) + carry <= q/8 to hi,
    // so up to 7 of these may follow a state with hi < q before fold() (hi < 2q -> < q)
    __device__ __forceinline__ void mac_nr(u64 a, u64 b) {
        u64 pl = a * b, ph = umulhi(a, b);
        u64 nl = lo + pl;
        hi += ph + (nl < lo ? 1ull : 0ull);
        lo = nl;
    }
    __device__ __forceinline__ void fold(u64 q) {
        const u64 t = hi - q;
        hi = (i64)t < 0 ? hi : t;
    }
    __device__ __forceinline__ u64 reduce(u64 q, u64 qinv_neg) const { return redc(hi, lo, q, qinv_neg); }
};

// x - m if x >= m else x, for x < 2m < 2^64 and m < 2^63 (sign-bit select)
__device__ __forceinline__ u64 csub(u64 x, u64 m) {
    const u64 t = x - m;
    return (i64)t < 0 ? x : t;
}

__device__ __forceinline__ u64 add_mod(u64 a, u64 b, u64 q) { u64 s = a + b; return s >= q ? s - q : s; }
__device__ __forceinline__ u64 sub_mod(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }
__device__ __forceinline__ u64 neg_mod(u64 a, u64 q) { return a ? q - a : 0ull; }

__device__ __forceinline__ u32 brev_bits(u32 x, int bits) { return __brev(x) >> (32 - bits); }

// NTT-domain automorphism X -> X^g: out[p] = in[perm(p)]
__device__ __forceinline__ u32 automorph_src(u32 p, u32 g, int logn) {
    u32 M = 2u << logn;
    u32 k = brev_bits(p, logn);
    u32 e = (u32)(((unsigned long long)g * (2u * k + 1u)) & (M - 1u));
    return brev_bits((e - 1u) >> 1, logn);
}

// ---- Philox4x32-10 (counter layout: DESIGN.md 3.4) ----
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; r++) {
        if (r) { k.x += 0x9E3779B9u; k.y += 0xBB67AE85u; }
        u32 lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        u32 lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        uint4 n;
        n.x = hi1 ^ c.y ^ k.x;
        n.y = lo1;
        n.z = hi0 ^ c.w ^ k.y;
        n.w = lo0;
        c = n;
    }
    return c;
}

__device__ __forceinline__ uint4 draw(u64 seed, u32 domain, u32 limb, u64 id, u32 n) {
    uint4 c = make_uint4(n, limb | (domain << 16), (u32)id, (u32)(id >> 32));
    uint2 k = make_uint2((u32)seed, (u32)(seed >> 32));
    return philox4x32_10(c, k);
}

// ((o1:o0) * 2^64 + (o3:o2)) mod q  ==  x*(2^64 mod q) + y  mod q
__device__ __forceinline__ u64 uniform_mod(uint4 o, const PrimeInfo& p) {
    u64 x = ((u64)o.y << 32) | o.x;
    u64 y = ((u64)o.w << 32) | o.z;
    u64 q = p.q;
    u64 xr = x % q;  // cold path (keygen / encrypt only)
    u64 t = shoup(xr, p.r1, p.r1_shoup, q);
    u64 yr = y % q;
    return add_mod(t, yr, q);
}

__device__ __forceinline__ i64 cbd21(uint4 o) {
    return (i64)__popc(o.x & 0x1FFFFFu) - (i64)__popc(o.y & 0x1FFFFFu);
}

__device__ __forceinline__ u64 signed_to_residue(i64 v, u64 q) {
    i64 r = v % (i64)q;
    return r < 0 ? (u64)(r + (i64)q) : (u64)r;
}

#define BCN_CHECK_LAUNCH() do { cudaError_t _e = cudaGetLastError(); if (_e != cudaSuccess) return _e; } while (0)

// Every launcher in this library launches exactly one kernel and returns
// through launched(): the count is exported as bcn_launch_count() so the
// bench can report how many of OUR kernels ran in its timed region.
#include <atomic>
namespace bcn {
extern std::atomic<unsigned long long> g_launches;
}
static inline cudaError_t launched() {
    bcn::g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}
