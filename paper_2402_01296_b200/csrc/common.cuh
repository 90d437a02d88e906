// common.cuh -- shared device helpers for the sm_100a RNS-CKKS engine.
//
// Word type: u64 residues, primes q < 2^61 (4q < 2^63 for Harvey lazy
// butterflies).  Three modular-multiply flavours, chosen per operand kind:
//   * Shoup   -- constant operand w with companion w' = floor(w 2^64 / q)
//                (NTT twiddles, q_l^-1, P^-1, base-conversion scalars);
//   * Montgomery REDC -- stored operands kept as x*2^64 mod q (switching
//                keys, plaintext multipliers, the secret key);
//   * u128 lazy accumulation of several products followed by ONE REDC;
//   * FP64 (primes q < 2^50): exact integers in doubles, a*w mod q by the
//     FMA two-product and a rounded quotient (fmm / fred below) -- on the
//     FP64 pipe, which the integer kernels leave idle (NTT butterflies,
//     base conversions, the Mul_CC tensor product).
// Every value written back to HBM is canonical ([0, q)) so ciphertexts are
// comparable bit for bit with oracle/ckks.py, whichever flavour produced them.
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
    u64 pad[3];     // [0] n^-1, [1] its Shoup companion, [2] floor(2^64 / q)
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

// ((o1:o0) * 2^64 + (o3:o2)) mod q  ==  x*(2^64 mod q) + y  mod q; the two
// 64-bit reductions are Shoup multiplies by 1 (pad[2] = floor(2^64 / q)):
// exact for any 64-bit word, the same residues as x % q
__device__ __forceinline__ u64 uniform_mod(uint4 o, const PrimeInfo& p) {
    u64 x = ((u64)o.y << 32) | o.x;
    u64 y = ((u64)o.w << 32) | o.z;
    u64 q = p.q;
    u64 xr = shoup(x, 1ull, p.pad[2], q);
    u64 t = shoup(xr, p.r1, p.r1_shoup, q);
    u64 yr = shoup(y, 1ull, p.pad[2], q);
    return add_mod(t, yr, q);
}

__device__ __forceinline__ i64 cbd21(uint4 o) {
    return (i64)__popc(o.x & 0x1FFFFFu) - (i64)__popc(o.y & 0x1FFFFFu);
}

__device__ __forceinline__ u64 signed_to_residue(i64 v, u64 q) {
    i64 r = v % (i64)q;
    return r < 0 ? (u64)(r + (i64)q) : (u64)r;
}
// the same without a 64-bit division: |v| mod q by a Shoup multiply by 1
// (inv1 = floor(2^64 / q)), then the sign
__device__ __forceinline__ u64 signed_to_residue_fast(i64 v, u64 q, u64 inv1) {
    const u64 a = v < 0 ? (u64)0 - (u64)v : (u64)v;
    const u64 r = shoup(a, 1ull, inv1, q);
    return v < 0 ? neg_mod(r, q) : r;
}

// ---- exact u128 multiply-accumulate (4 x 32-bit words, no reduction) ----
// acc += a*b for a, b < 2^61: four IMAD.WIDE.U32 (a0b0 and a1b1 straight into
// the aligned word pairs, the two cross products summed into one 64-bit word
// first) plus a 3-word carry add.  Products are < 2^122, so 32 of them fit
// on top of a state whose high half is < q before fold_hi() must run.
struct Acc4 {
    u64 lo, hi;            // kept as aligned register pairs: no moves between MACs
    __device__ __forceinline__ void zero() { lo = hi = 0ull; }
    __device__ __forceinline__ void mac(u32 a0, u32 a1, u32 b0, u32 b1) {
        u64 x;
        asm("mul.wide.u32 %0, %1, %2;\n\tmad.wide.u32 %0, %3, %4, %0;" : "=l"(x) : "r"(a0), "r"(b1), "r"(a1), "r"(b0));
        asm("{\n\t.reg .u32 w0, w1, w2, w3, x0, x1;\n\t"
            "mov.b64 {w0, w1}, %0;\n\t"
            "mov.b64 {w2, w3}, %1;\n\t"
            "mov.b64 {x0, x1}, %6;\n\t"
            "mad.lo.cc.u32 w0, %2, %4, w0;\n\t"
            "madc.hi.cc.u32 w1, %2, %4, w1;\n\t"
            "madc.lo.cc.u32 w2, %3, %5, w2;\n\t"
            "madc.hi.u32 w3, %3, %5, w3;\n\t"
            "add.cc.u32 w1, w1, x0;\n\t"
            "addc.cc.u32 w2, w2, x1;\n\t"
            "addc.u32 w3, w3, 0;\n\t"
            "mov.b64 %0, {w0, w1};\n\t"
            "mov.b64 %1, {w2, w3};\n\t}"
            : "+l"(lo), "+l"(hi)
            : "r"(a0), "r"(a1), "r"(b0), "r"(b1), "l"(x));
    }
    __device__ __forceinline__ void mac(u64 a, u64 b) { mac((u32)a, (u32)(a >> 32), (u32)b, (u32)(b >> 32)); }
    // high half -> [0, q) (value changes by a multiple of q 2^64); inv1 = floor(2^64 / q)
    __device__ __forceinline__ void fold_hi(u64 q, u64 inv1) {
        u64 h = hi - umulhi(hi, inv1) * q;
        hi = h >= q ? h - q : h;
    }
    // REDC of the (folded) value: sum a*b * 2^-64 mod q
    __device__ __forceinline__ u64 reduce(u64 q, u64 qinv_neg, u64 inv1) {
        fold_hi(q, inv1);
        return redc(hi, lo, q, qinv_neg);
    }
};

// ---- FP64 modular arithmetic for primes q < 2^50 ----
// Residues are exact integers held in doubles.  fmm(a, w, w/q): a*w mod q
// with |result| <= 0.61 q for |a| < 2q (the quotient a*w/q must stay below
// 2^51 for the add-1.5*2^52 rounding); fred(x): x mod q into [-q/2, q/2]
// (+2^-50 q) for any exact |x| < 2^53.
static constexpr double FMAGIC = 6755399441055744.0;   // 1.5 * 2^52

__device__ __forceinline__ double fmm(double a, double w, double wq, double q) {
    const double hi = __dmul_rn(a, w);
    const double lo = __fma_rn(a, w, -hi);
    const double qt = __dadd_rn(__fma_rn(a, wq, FMAGIC), -FMAGIC);
    return __dadd_rn(__fma_rn(-qt, q, hi), lo);
}
__device__ __forceinline__ double fred(double x, double qinv, double q) {
    const double qt = __dadd_rn(__fma_rn(x, qinv, FMAGIC), -FMAGIC);
    return __fma_rn(-qt, q, x);
}
// |x| < q  ->  [0, q) as u64 (bits of x + 2^52 carry x in the low mantissa)
__device__ __forceinline__ u64 fcanon_small(double x, double q) {
    const double y = x < 0.0 ? __dadd_rn(x, q) : x;
    return (u64)__double_as_longlong(__dadd_rn(y, 4503599627370496.0)) & ((1ull << 52) - 1);
}
__device__ __forceinline__ u64 fcanon(double x, double qinv, double q) { return fcanon_small(fred(x, qinv, q), q); }
// canonical u64 < 2^52 -> exact double
__device__ __forceinline__ double fload(u64 v) {
    return __dadd_rn(__longlong_as_double((long long)(v | 0x4330000000000000ull)), -4503599627370496.0);
}

// ---- bulk async copies (TMA engine, 1-D) completing on an mbarrier ----
__device__ __forceinline__ u32 smem_addr(const void* p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(u64* bar, u32 count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n\tfence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(u64* bar, u32 bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, u32 bytes, u64* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}
// L2 prefetch of a contiguous range by the TMA engine (no registers, no completion)
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, u32 bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(u64* bar, u32 parity) {
    u32 done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
    } while (!done);
}

#define BCN_CHECK_LAUNCH() do { cudaError_t _e = cudaGetLastError(); if (_e != cudaSuccess) return _e; } while (0)

// Every launcher in this library launches exactly one kernel and returns
// through launched(): the count is exported as bcn_launch_count() so the
// bench can report how many of OUR kernels ran in its timed region.
#include <atomic>
namespace bcn {
extern std::atomic<unsigned long long> g_launches;
}
// Kernel attributes (max dynamic SMEM) are per device: `mask` (a static at
// the call site) records the devices already configured, so a second
// context on another device in the same process configures its own.
static inline bool first_on_device(unsigned long long* mask, unsigned long long* bit) {
    int d = 0;
    cudaGetDevice(&d);
    *bit = 1ull << (d & 63);
    return (*mask & *bit) == 0;
}
#define BCN_SMEM_ATTR(err, fn, bytes) \
    do { if ((err) == cudaSuccess) (err) = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(bytes)); } while (0)

static inline cudaError_t launched() {
    bcn::g_launches.fetch_add(1, std::memory_order_relaxed);
    return cudaGetLastError();
}
