// ntt_mac_rescale.cu -- BASELINE config 2 as ONE pass:
//
//     Y_g = Rescale( sum_{t < group} NTT(ct_{g,t}) (.) pt_{g,t} )
//
// for ciphertexts given in the coefficient domain, plaintexts in the NTT
// domain, and the output in the NTT domain one level down.  This is the
// RNS form of one packed conv output channel (the reference's
// conv_accumulate, pkg/src/bibranch/layers.py:149-172: a sum of plaintext
// products followed by one rescale, sim.py:221-248).  The unfused engine
// needs an NTT launch, a MAC launch and a rescale (INTT of the top limb,
// lift, NTT, combine); here every ciphertext word is read once from HBM,
// transformed in shared memory, multiplied and accumulated on chip, and only
// the rescaled output is written.
//
// Two word widths share this code (template on W):
//   * W = u32 -- the 32-bit-limb variant: primes q < 2^30 (Harvey's lazy
//     [0, 4q) butterflies need 4q < 2^32), Delta = 2^30 = the reference's
//     default scale (pkg/src/bibranch/cli.py:66).  Half the HBM bytes of the
//     u64 engine, native 32-bit IMAD (umulhi.u32 / mul.wide.u32) instead of
//     the 4-IMAD 64-bit products.  Own context (bcn32_ctx: u32 twiddles).
//   * W = u64 -- BASELINE config 2's own ~60-bit primes, on the main
//     context's tables (bcn_ntt_mac_rescale).
//
// Layout: a thread-block cluster per output group, one CTA per (component,
// RNS limb) (cluster size 2 nlimb <= 16).  A CTA keeps the running sum of its
// limb in shared memory (N words, each thread owning the words its last NTT
// pass leaves in its registers, so the MAC needs no barrier) and a 2-deep
// ring of bulk-copied (TMA engine, cp.async.bulk) input limb-polys, so the
// next term's HBM read overlaps the current term's butterflies; each NTT runs
// in place in its ring slot.  The two components' CTAs of one limb read the
// same plaintext words (the second read is an L2 hit).  Rescale: the
// top-limb CTAs inverse-transform their sums in place; after one cluster
// barrier every other CTA reads them over DSMEM as the first pass of its
// forward NTT (centred lift into its own prime on the fly), and writes
// (acc - NTT(lift)) * q_top^-1.
//
// Ordering / conventions are those of ntt.cu (the contract with
// oracle/ckks_oracle.c): forward output index k holds a(psi^(2 brev(k)+1)),
// twiddles {w, floor(w 2^bits / q)} in bit-reversed order, the inverse table
// slot 0 holds {w1 n^-1, shoup}.  Plaintexts are in Montgomery form
// (pt 2^bits mod q).  Every output word is canonical.
#include <cooperative_groups.h>

#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "ops.cuh"
#include "../../include/bcn.h"

namespace cg = cooperative_groups;

namespace bcn {

template <class W> struct Ar;

template <> struct Ar<u32> {
    typedef uint2 TW;
    __device__ static __forceinline__ u32 shoup_lazy(u32 a, u32 w, u32 wp, u32 q) { return a * w - __umulhi(a, wp) * q; }
    // a * b_mont * 2^-32 mod q, canonical (a, b < q < 2^30)
    __device__ static __forceinline__ u32 mont(u32 a, u32 b, u32 q, u32 qneg) {
        const u64 t = (u64)a * b;
        const u32 m = (u32)t * qneg;
        const u32 r = (u32)((t + (u64)m * q) >> 32);
        return r >= q ? r - q : r;
    }
};

template <> struct Ar<u64> {
    typedef ulonglong2 TW;
    __device__ static __forceinline__ u64 shoup_lazy(u64 a, u64 w, u64 wp, u64 q) { return a * w - __umul64hi(a, wp) * q; }
    __device__ static __forceinline__ u64 mont(u64 a, u64 b, u64 q, u64 qneg) { return mont_mul(a, b, q, qneg); }
};

// x - m if x >= m else x, for x < 2m, m <= 2^(bits-1): the wrapped difference
// is larger than x exactly when x < m (one IADD + one VIMNMX for u32)
template <class W> __device__ __forceinline__ W csubw(W x, W m) { return min(x, (W)(x - m)); }
template <class W> __device__ __forceinline__ W shoupw(W a, W w, W wp, W q) { return csubw<W>(Ar<W>::shoup_lazy(a, w, wp, q), q); }

template <int LOGN> struct NmrCfg {
    static constexpr int LOGE = 4;
    static constexpr int N = 1 << LOGN;
    static constexpr int E = 1 << LOGE;
    static constexpr int T = N / E;
    static constexpr int R0 = (LOGN % LOGE) ? (LOGN % LOGE) : LOGE;
};

// SMEM layout: one pad word per 32 (index j lives at j + j / 32).  For every
// pass of the E = 16 schedule the address is affine in the unrolled element
// index (immediate offsets from one per-thread base: no per-access ALU), and
// the 32 lanes of a warp hit 32 distinct banks with 4-byte words: runs of 32
// consecutive columns (strides >= 32), stride-16 runs in the last pass, and
// in the stride-16 pass the two half-warps take block rows 2 apart (bits 4
// and 5 of the block index swapped, blk()), which the padding puts 16 banks
// apart.
template <int LOGN> __device__ __forceinline__ int sw(int j) { return j + (j >> 5); }
template <int LOGN> struct Pad { static constexpr int NP = (1 << LOGN) + ((1 << LOGN) >> 5); };
// padded address of element base + k TL as (per-thread base) + (compile-time offset)
template <int TL, int BS>
__device__ __forceinline__ int pad_at(int pbase, int base, int k) {
    if constexpr (TL % 32 == 0) return pbase + k * TL + ((k * TL) >> 5);
    else if constexpr (TL == 16) return pbase + 16 * k + (k >> 1);      // base % 32 < 16
    else if constexpr (TL == 1 && BS == 16) return pbase + k;           // base % 16 == 0
    else return (base + k * TL) + ((base + k * TL) >> 5);
}
// block index of thread slot b in a pass with element stride TL
template <int TL> __device__ __forceinline__ int blk(int b) {
    if constexpr (TL == 16) return (b & ~0x30) | ((b & 0x10) << 1) | ((b & 0x20) >> 1);
    else return b;
}

struct NoHook { __device__ void operator()() const {} };

template <class W, int LOGN, int S0, int R, bool FIRST, bool LAST, class Ld, class Hook = NoHook>
__device__ __forceinline__ void fpass(W* x, W* sm, const typename Ar<W>::TW* __restrict__ Wt, W q, int tid, Ld ld,
                                      Hook hook = Hook()) {
    using C = NmrCfg<LOGN>;
    constexpr int BS = 1 << R, NB = C::E / BS, TL = C::N >> (S0 + R);
    const W q2 = 2 * q;
#pragma unroll
    for (int i = 0; i < NB; i++) {
        const int b = blk<TL>(tid + i * C::T);
        const int base = (b / TL) * (C::N >> S0) + (b % TL);
        const int pbase = base + (base >> 5);
#pragma unroll
        for (int k = 0; k < BS; k++)
            x[i * BS + k] = FIRST ? ld(base + k * TL) : sm[pad_at<TL, BS>(pbase, base, k)];
    }
    if (FIRST) {
        __syncthreads();
        hook();                                         // every thread is past its previous use of SMEM
    }
#pragma unroll
    for (int i = 0; i < NB; i++) {
        const int b = blk<TL>(tid + i * C::T);
        const int gi = b / TL;
        const int base = gi * (C::N >> S0) + (b % TL);
        const int pbase = base + (base >> 5);
#pragma unroll
        for (int ls = 0; ls < R; ls++) {
            const int h = BS >> (ls + 1);
            const int s = S0 + ls;
            const typename Ar<W>::TW* __restrict__ ws = Wt + (1 << s) + (gi << ls);   // + compile-time offsets
#pragma unroll
            for (int k = 0; k < BS; k++) {
                if (k & h) continue;
                const typename Ar<W>::TW w = ws[k >> (R - ls)];
                W u = x[i * BS + k];
                if (!(FIRST && ls == 0)) u = csubw<W>(u, q2);
                const W v = Ar<W>::shoup_lazy(x[i * BS + k + h], w.x, w.y, q);
                x[i * BS + k] = u + v;
                x[i * BS + k + h] = u - v + q2;
            }
        }
#pragma unroll
        for (int k = 0; k < BS; k++) {
            if (LAST) x[i * BS + k] = csubw<W>(csubw<W>(x[i * BS + k], q2), q);
            else sm[pad_at<TL, BS>(pbase, base, k)] = x[i * BS + k];
        }
    }
}

template <class W, int LOGN, int S0, class Hook2>
__device__ __forceinline__ void frest(W* x, W* sm, const typename Ar<W>::TW* __restrict__ Wt, W q, int tid,
                                      Hook2 last_hook) {
    using C = NmrCfg<LOGN>;
    if constexpr (S0 < LOGN) {
        __syncthreads();
        if constexpr (S0 + C::LOGE >= LOGN) last_hook();
        fpass<W, LOGN, S0, C::LOGE, false, (S0 + C::LOGE >= LOGN)>(x, sm, Wt, q, tid, [](int) { return W(0); });
        frest<W, LOGN, S0 + C::LOGE>(x, sm, Wt, q, tid, last_hook);
    }
}

// full forward NTT: input via ld(j), result canonical in x (no trailing
// barrier); hook() runs on every thread right after the first barrier,
// last_hook() right before the last pass (e.g. to issue the loads the code
// after the transform consumes)
template <class W, int LOGN, class Ld, class Hook = NoHook, class Hook2 = NoHook>
__device__ __forceinline__ void fwd_ntt(W* x, W* sm, const typename Ar<W>::TW* __restrict__ Wt, W q, int tid, Ld ld,
                                        Hook hook = Hook(), Hook2 last_hook = Hook2()) {
    using C = NmrCfg<LOGN>;
    fpass<W, LOGN, 0, C::R0, true, (C::R0 >= LOGN)>(x, sm, Wt, q, tid, ld, hook);
    frest<W, LOGN, C::R0>(x, sm, Wt, q, tid, last_hook);
}

// the words the last forward pass leaves in x[e] of thread tid
template <int LOGN> struct Own {
    using C = NmrCfg<LOGN>;
    static constexpr int BS = 1 << ((C::R0 >= LOGN) ? C::R0 : C::LOGE);
    static constexpr int NB = C::E / BS;
    __device__ static __forceinline__ int word(int tid, int e) { return (tid + (e / BS) * C::T) * BS + (e % BS); }
};

// x[i BS .. i BS + BS) <-> consecutive words: 16-byte vector accesses
template <class W, int LOGN>
__device__ __forceinline__ void load_own(W* x, const W* __restrict__ src, int tid) {
    using O = Own<LOGN>;
    constexpr int PER = 16 / sizeof(W);
#pragma unroll
    for (int i = 0; i < O::NB; i++) {
        const uint4* s = reinterpret_cast<const uint4*>(src + O::word(tid, i * O::BS));
#pragma unroll
        for (int v = 0; v < O::BS / PER; v++) {
            const uint4 r = __ldg(s + v);
            memcpy(&x[i * O::BS + v * PER], &r, 16);
        }
    }
}
template <class W, int LOGN>
__device__ __forceinline__ void store_own(W* dst, const W* x, int tid) {
    using O = Own<LOGN>;
    constexpr int PER = 16 / sizeof(W);
#pragma unroll
    for (int i = 0; i < O::NB; i++) {
        uint4* d = reinterpret_cast<uint4*>(dst + O::word(tid, i * O::BS));
#pragma unroll
        for (int v = 0; v < O::BS / PER; v++) {
            uint4 r;
            memcpy(&r, &x[i * O::BS + v * PER], 16);
            d[v] = r;
        }
    }
}

// ---- inverse (Gentleman-Sande) in place on the swizzled array `a`; the last
// stage folds N^-1; output canonical in `a` (swizzled).  Ends with a barrier.
template <class W, int LOGN, int S0, int R, bool LAST, bool GIN = false, bool GOUT = false>
__device__ __forceinline__ void ipass(W* x, W* a, const typename Ar<W>::TW* __restrict__ Wi, W q, W ninv, W ninv_p,
                                      W wn, W wn_p, int tid, const W* __restrict__ gin = nullptr,
                                      W* __restrict__ gout = nullptr) {
    using C = NmrCfg<LOGN>;
    constexpr int BS = 1 << R, NB = C::E / BS, TL = C::N >> (S0 + R);
    const W q2 = 2 * q;
#pragma unroll
    for (int i = 0; i < NB; i++) {
        const int b = blk<TL>(tid + i * C::T);
        const int gi = b / TL;
        const int base = gi * (C::N >> S0) + (b % TL);
        const int pbase = base + (base >> 5);
        if constexpr (GIN) {                            // first pass straight from HBM: contiguous 16-word runs
            static_assert(TL == 1 && BS == 16, "global input needs a contiguous first pass");
            constexpr int PER = 16 / sizeof(W);
#pragma unroll
            for (int v = 0; v < BS / PER; v++) {
                const uint4 r = __ldg(reinterpret_cast<const uint4*>(gin + base) + v);
                memcpy(&x[i * BS + v * PER], &r, 16);
            }
        } else {
#pragma unroll
            for (int k = 0; k < BS; k++) x[i * BS + k] = a[pad_at<TL, BS>(pbase, base, k)];
        }
#pragma unroll
        for (int ls = R - 1; ls >= 0; ls--) {
            const int h = BS >> (ls + 1);
            const int s = S0 + ls;
            const typename Ar<W>::TW* __restrict__ ws = Wi + (1 << s) + (gi << ls);
#pragma unroll
            for (int k = 0; k < BS; k++) {
                if (k & h) continue;
                const W u = x[i * BS + k], v = x[i * BS + k + h];
                if (LAST && s == 0) {
                    x[i * BS + k] = shoupw<W>(u + v, ninv, ninv_p, q);
                    x[i * BS + k + h] = shoupw<W>(u - v + q2, wn, wn_p, q);
                } else {
                    const typename Ar<W>::TW w = ws[k >> (R - ls)];
                    x[i * BS + k] = csubw<W>(u + v, q2);
                    x[i * BS + k + h] = Ar<W>::shoup_lazy(u - v + q2, w.x, w.y, q);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < BS; k++) {
            if constexpr (GOUT) gout[base + k * TL] = x[i * BS + k];   // last pass straight to HBM (coalesced)
            else a[pad_at<TL, BS>(pbase, base, k)] = x[i * BS + k];
        }
    }
    if constexpr (!GOUT) __syncthreads();
}

template <class W, int LOGN, int S0, bool GIN = false>
__device__ __forceinline__ void irest(W* x, W* a, const typename Ar<W>::TW* __restrict__ Wi, W q, W ninv, W ninv_p,
                                      W wn, W wn_p, int tid, const W* gin = nullptr) {
    using C = NmrCfg<LOGN>;
    if constexpr (S0 >= C::R0) {
        ipass<W, LOGN, S0, C::LOGE, false, GIN>(x, a, Wi, q, ninv, ninv_p, wn, wn_p, tid, gin);
        irest<W, LOGN, S0 - C::LOGE>(x, a, Wi, q, ninv, ninv_p, wn, wn_p, tid);
    }
}

// inverse NTT: in place on the padded SMEM array `a`, or (GIO) from gio in HBM
// back to gio, with `a` as the exchange buffer
template <class W, int LOGN, bool GIO = false>
__device__ __forceinline__ void inv_ntt_smem(W* x, W* a, const typename Ar<W>::TW* __restrict__ Wi, W q, W ninv,
                                             W ninv_p, W wn, W wn_p, int tid, W* gio = nullptr) {
    using C = NmrCfg<LOGN>;
    static_assert(!GIO || LOGN - C::LOGE >= C::R0, "global in/out needs at least two passes");
    irest<W, LOGN, LOGN - C::LOGE, GIO>(x, a, Wi, q, ninv, ninv_p, wn, wn_p, tid, gio);
    ipass<W, LOGN, 0, C::R0, true, false, GIO>(x, a, Wi, q, ninv, ninv_p, wn, wn_p, tid, nullptr, gio);
}

// ---- the fused kernel --------------------------------------------------
// Cluster = 2 nlimb CTAs: rank = component * nlimb + limb.  SMEM per CTA:
// ring[2][33 N / 32] (bulk-copied ciphertext limb-polys; each NTT runs in
// place in its slot, padded) | 2 mbarriers: 66 KiB (u32) / 132 KiB (u64) at
// N = 8192.  The running sum lives in registers: the words the last NTT pass
// leaves in a thread are the words it accumulates, and its plaintext words
// (16 consecutive) come straight from HBM/L2 with 16-byte loads issued
// before the last pass.
#ifndef NMR_MINB32
#define NMR_MINB32 2
#endif
template <class W, int LOGN> struct NmrOcc { static constexpr int MINB = (sizeof(W) == 4 && LOGN <= 13) ? NMR_MINB32 : 1; };

template <class W, int LOGN>
__global__ void __launch_bounds__(NmrCfg<LOGN>::T, (NmrOcc<W, LOGN>::MINB)) ntt_mac_rescale_kernel(NmrArgs<W> a) {
    using C = NmrCfg<LOGN>;
    using O = Own<LOGN>;
    extern __shared__ __align__(16) unsigned char smraw[];
    constexpr int NP = Pad<LOGN>::NP;                  // padded slot (the in-place NTT writes j + j / 32)
    W* ring = reinterpret_cast<W*>(smraw);
    u64* bar = reinterpret_cast<u64*>(ring + 2 * NP);  // [0], [1] ring slots
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int comp = rank / a.nlimb, t = rank - comp * a.nlimb;
    const int g = blockIdx.y;                           // output group
    const int top = a.nlimb - 1;
    const int tid = threadIdx.x;
    const W q = a.k.q[t];
    const typename Ar<W>::TW* Wt = reinterpret_cast<const typename Ar<W>::TW*>(a.tw) + (size_t)t * 2 * C::N;
    const int k0 = g * a.group;
    const int nterm = min(a.group, a.n_items - k0);
    constexpr u32 BYTES = C::N * sizeof(W);
    auto src_of = [&](int s) { return a.ct + (((size_t)(k0 + s) * 2 + comp) * a.nlimb + t) * C::N; };
    auto pt_of = [&](int s) { return a.pt + ((size_t)(k0 + s) * a.nlimb + t) * C::N; };
    if (tid == 0) {
        for (int i = 0; i < 2; i++) mbar_init(&bar[i], 1);
        fence_barrier_init();
        for (int s = 0; s < 2 && s < nterm; s++) {
            mbar_expect_tx(&bar[s], BYTES);
            bulk_load(ring + s * NP, src_of(s), BYTES, &bar[s]);
        }
    }
    W x[C::E];
    W p[C::E];
    W acc[C::E];
#pragma unroll
    for (int e = 0; e < C::E; e++) acc[e] = 0;
    __syncthreads();                                    // mbarrier init visible before any wait
    const W qneg = a.k.qneg[t];
    for (int s = 0; s < nterm; s++) {
        const int slot = s & 1;
        mbar_wait(&bar[slot], (u32)((s >> 1) & 1));
        W* in = ring + slot * NP;
        // the plaintext words this thread multiplies (its 16 output words, 4 x 16-byte
        // loads) are issued right before the last pass, whose butterflies hide them
        fwd_ntt<W, LOGN>(x, in, Wt, q, tid, [&](int j) { return in[j]; }, NoHook(),
                         [&]() { load_own<W, LOGN>(p, pt_of(s), tid); });
        __syncthreads();                                // every thread is done with ring[slot]
        if (tid == 0 && s + 2 < nterm) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&bar[slot], BYTES);
            bulk_load(in, src_of(s + 2), BYTES, &bar[slot]);
        }
#pragma unroll
        for (int e = 0; e < C::E; e++) acc[e] = csubw<W>(acc[e] + Ar<W>::mont(x[e], p[e], q, qneg), q);
    }
    __syncthreads();                                    // ring free
    // ---- rescale by q_top: the top limb's sums go through SMEM (ring slot 0)
    W* sums = ring;
    if (t == top) {
#pragma unroll
        for (int e = 0; e < C::E; e++) sums[sw<LOGN>(O::word(tid, e))] = acc[e];
        __syncthreads();
        inv_ntt_smem<W, LOGN>(x, sums, Wt + C::N, q, a.k.ninv[t], a.k.ninv_p[t], a.k.wn[t], a.k.wn_p[t], tid);
    }
    cluster.sync();                                     // the top limb's INTT is visible cluster-wide
    if (t != top) {
        const W* rs = cluster.map_shared_rank(sums, comp * a.nlimb + top);
        const W qt = a.k.q[top], half = qt >> 1;
        const W inv1 = a.k.inv1[t], qlm = a.k.qlmod[t];
        const W qli = a.k.qlinv[t], qlip = a.k.qlinv_p[t];
        fwd_ntt<W, LOGN>(x, ring + NP, Wt, q, tid, [&](int j) {
            const W v = rs[sw<LOGN>(j)];
            const W r = shoupw<W>(v, W(1), inv1, q);                   // v mod q_t
            return v > half ? (r >= qlm ? r - qlm : r + q - qlm) : r;  // centred lift: v - q_top
        });
#pragma unroll
        for (int e = 0; e < C::E; e++) x[e] = shoupw<W>(acc[e] + q - x[e], qli, qlip, q);
        store_own<W, LOGN>(a.out + (((size_t)g * 2 + comp) * (a.nlimb - 1) + t) * C::N, x, tid);
    }
    cluster.sync();                                     // peers are done reading the top limb's SMEM
}

template <class W, int LOGN>
static size_t nmr_smem() { return (size_t)2 * Pad<LOGN>::NP * sizeof(W) + 16; }

template <class W, int LOGN>
static cudaError_t nmr_launch_t(const NmrArgs<W>& a, int n_groups, cudaStream_t st) {
    using C = NmrCfg<LOGN>;
    const size_t smem = nmr_smem<W, LOGN>();
    static unsigned long long cfg = 0;
    unsigned long long bit = 0;
    if (first_on_device(&cfg, &bit)) {
        cudaError_t e = cudaSuccess;
        BCN_SMEM_ATTR(e, (ntt_mac_rescale_kernel<W, LOGN>), smem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(ntt_mac_rescale_kernel<W, LOGN>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        cfg |= bit;
    }
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(2 * a.nlimb, n_groups);
    lc.blockDim = dim3(C::T);
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2 * a.nlimb;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&lc, ntt_mac_rescale_kernel<W, LOGN>, a);
    if (e != cudaSuccess) return e;
    return launched();
}

template <class W>
cudaError_t ntt_mac_rescale_launch(const NmrArgs<W>& a, int logn, cudaStream_t st) {
    const int n_groups = (a.n_items + a.group - 1) / a.group;
    if (n_groups <= 0) return cudaSuccess;
    switch (logn) {
        case 10: return nmr_launch_t<W, 10>(a, n_groups, st);
        case 11: return nmr_launch_t<W, 11>(a, n_groups, st);
        case 12: return nmr_launch_t<W, 12>(a, n_groups, st);
        case 13: return nmr_launch_t<W, 13>(a, n_groups, st);
        case 14:
            if constexpr (sizeof(W) == 4) return nmr_launch_t<W, 14>(a, n_groups, st);
            return cudaErrorInvalidValue;               // u64 at 2^14: 3 N words exceed 227 KiB of SMEM
        default: return cudaErrorInvalidValue;
    }
}

// ---- plain batched NTT / INTT of the 32-bit variant (one CTA per limb-poly)
template <class W, int LOGN, bool INV>
__global__ void __launch_bounds__(NmrCfg<LOGN>::T) ntt_w_kernel(W* data, const typename Ar<W>::TW* tw,
                                                              NmrConst<W> k, int nlimb) {
    using C = NmrCfg<LOGN>;
    extern __shared__ __align__(16) unsigned char smraw[];
    W* sm = reinterpret_cast<W*>(smraw);
    const int t = blockIdx.x, poly = blockIdx.y, tid = threadIdx.x;
    W* g = data + ((size_t)poly * nlimb + t) * C::N;
    const typename Ar<W>::TW* Wt = tw + (size_t)t * 2 * C::N;
    const W q = k.q[t];
    W x[C::E];
    if constexpr (!INV) {
        fwd_ntt<W, LOGN>(x, sm, Wt, q, tid, [&](int j) { return g[j]; });
        store_own<W, LOGN>(g, x, tid);
    } else {
        inv_ntt_smem<W, LOGN, true>(x, sm, Wt + C::N, q, k.ninv[t], k.ninv_p[t], k.wn[t], k.wn_p[t], tid, g);
    }
}

template <class W, int LOGN>
static cudaError_t ntt_w_launch_t(bool inv, W* data, const typename Ar<W>::TW* tw, const NmrConst<W>& k, int nlimb,
                                  int npoly, cudaStream_t st) {
    using C = NmrCfg<LOGN>;
    const size_t smem = (size_t)Pad<LOGN>::NP * sizeof(W);
    static unsigned long long cfg = 0;
    unsigned long long bit = 0;
    if (first_on_device(&cfg, &bit)) {
        cudaError_t e = cudaSuccess;
        BCN_SMEM_ATTR(e, (ntt_w_kernel<W, LOGN, false>), smem);
        BCN_SMEM_ATTR(e, (ntt_w_kernel<W, LOGN, true>), smem);
        if (e != cudaSuccess) return e;
        cfg |= bit;
    }
    dim3 grid(nlimb, npoly);
    if (inv) ntt_w_kernel<W, LOGN, true><<<grid, C::T, smem, st>>>(data, tw, k, nlimb);
    else ntt_w_kernel<W, LOGN, false><<<grid, C::T, smem, st>>>(data, tw, k, nlimb);
    return launched();
}

template <class W>
static cudaError_t ntt_w_launch(bool inv, int logn, W* data, const typename Ar<W>::TW* tw, const NmrConst<W>& k,
                                int nlimb, int npoly, cudaStream_t st) {
    if (npoly <= 0) return cudaSuccess;
    switch (logn) {
        case 10: return ntt_w_launch_t<W, 10>(inv, data, tw, k, nlimb, npoly, st);
        case 11: return ntt_w_launch_t<W, 11>(inv, data, tw, k, nlimb, npoly, st);
        case 12: return ntt_w_launch_t<W, 12>(inv, data, tw, k, nlimb, npoly, st);
        case 13: return ntt_w_launch_t<W, 13>(inv, data, tw, k, nlimb, npoly, st);
        case 14: return ntt_w_launch_t<W, 14>(inv, data, tw, k, nlimb, npoly, st);
        default: return cudaErrorInvalidValue;
    }
}

// u32 -> Montgomery form (x 2^32 mod q), elementwise over [npoly][nlimb][N]
__global__ void to_mont32_kernel(u32* out, const u32* in, NmrConst<u32> k, int nlimb, int N, size_t total) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
        const int t = (int)((i / N) % nlimb);
        out[i] = (u32)((((u64)in[i]) << 32) % k.q[t]);
    }
}

// host-side instantiations used by api.cu (u64 path on the main context)
template cudaError_t ntt_mac_rescale_launch<u64>(const NmrArgs<u64>&, int, cudaStream_t);

}  // namespace bcn

// ====================================================================
// bcn32_*: the 32-bit-limb context (primes q < 2^30, q = 1 mod 2N)
// ====================================================================
using namespace bcn;

struct bcn32_ctx {
    int device = 0, logn = 0, N = 0, nlimb = 0;
    std::vector<u32> q;
    NmrConst<u32> k{};
    uint2* tw = nullptr;
};

namespace {
thread_local std::string g_err32;
int fail32(int code, const std::string& m) { g_err32 = m; return code; }
int cuda_fail32(cudaError_t e) { g_err32 = std::string("CUDA: ") + cudaGetErrorString(e); return BCN_ERR_CUDA; }

u64 pw32(u64 a, u64 e, u64 m) { u64 r = 1; a %= m; while (e) { if (e & 1) r = r * a % m; a = a * a % m; e >>= 1; } return r; }
u32 brev32(u32 x, int bits) { u32 r = 0; for (int i = 0; i < bits; i++) { r = (r << 1) | (x & 1); x >>= 1; } return r; }
u32 shoup32(u64 w, u64 q) { return (u32)((w << 32) / q); }
bool prime32(u64 n) {
    if (n < 2) return false;
    for (u64 d = 2; d * d <= n; d++) if (n % d == 0) return false;
    return true;
}
}  // namespace

extern "C" {

const char* bcn32_last_error(void) { return g_err32.c_str(); }

int bcn32_ctx_create(bcn32_ctx** out, int logn, int nlimb, const uint32_t* q, int device) {
    if (!out) return fail32(BCN_ERR_PARAM, "null output pointer");
    if (logn < 10 || logn > 14) return fail32(BCN_ERR_PARAM, "logn must be in [10, 14]");
    if (nlimb < 2 || nlimb > 8) return fail32(BCN_ERR_PARAM, "nlimb must be in [2, 8] (one cluster CTA per limb)");
    const u64 N = 1ull << logn;
    bcn32_ctx* c = new bcn32_ctx();
    c->device = device; c->logn = logn; c->N = (int)N; c->nlimb = nlimb;
    for (int i = 0; i < nlimb; i++) {
        const u64 qi = q[i];
        if (qi >= (1ull << 30) || qi % (2 * N) != 1 || !prime32(qi)) {
            delete c;
            return fail32(BCN_ERR_PARAM, "prime " + std::to_string(qi) + " is not a prime < 2^30 with q = 1 mod 2N");
        }
        for (int j = 0; j < i; j++) if (q[j] == q[i]) { delete c; return fail32(BCN_ERR_PARAM, "duplicate prime"); }
        c->q.push_back((u32)qi);
    }
    std::vector<uint2> tw((size_t)nlimb * 2 * N);
    const u64 qt = q[nlimb - 1];
    for (int i = 0; i < nlimb; i++) {
        const u64 qi = q[i];
        u64 x = 2, psi = 0;                                    // first x^((q-1)/2N) with psi^N = -1
        for (;; x++) { psi = pw32(x, (qi - 1) / (2 * N), qi); if (pw32(psi, N, qi) == qi - 1) break; }
        const u64 psi_inv = pw32(psi, qi - 2, qi), ninv = pw32(N % qi, qi - 2, qi);
        std::vector<u64> pw(N), pwi(N);
        u64 a = 1, b = 1;
        for (u64 kk = 0; kk < N; kk++) { pw[kk] = a; pwi[kk] = b; a = a * psi % qi; b = b * psi_inv % qi; }
        uint2* F = &tw[(size_t)i * 2 * N];
        uint2* I = F + N;
        for (u64 kk = 0; kk < N; kk++) {
            const u64 w = pw[brev32((u32)kk, logn)], wi = pwi[brev32((u32)kk, logn)];
            F[kk] = make_uint2((u32)w, shoup32(w, qi));
            I[kk] = make_uint2((u32)wi, shoup32(wi, qi));
        }
        const u64 wn = I[1].x * ninv % qi;
        I[0] = make_uint2((u32)wn, shoup32(wn, qi));
        u32 inv = 1;                                           // Newton: q^-1 mod 2^32
        for (int it = 0; it < 6; it++) inv *= 2 - (u32)qi * inv;
        c->k.q[i] = (u32)qi;
        c->k.qneg[i] = (u32)0 - inv;
        c->k.ninv[i] = (u32)ninv; c->k.ninv_p[i] = shoup32(ninv, qi);
        c->k.wn[i] = (u32)wn; c->k.wn_p[i] = shoup32(wn, qi);
        c->k.inv1[i] = shoup32(1, qi);
        if (i < nlimb - 1) {
            const u64 li = pw32(qt % qi, qi - 2, qi);
            c->k.qlinv[i] = (u32)li; c->k.qlinv_p[i] = shoup32(li, qi);
            c->k.qlmod[i] = (u32)(qt % qi);
        }
    }
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaMalloc((void**)&c->tw, sizeof(uint2) * tw.size());
    if (e == cudaSuccess) e = cudaMemcpy(c->tw, tw.data(), sizeof(uint2) * tw.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) { cudaFree(c->tw); delete c; return cuda_fail32(e); }
    *out = c;
    return BCN_OK;
}

int bcn32_ctx_destroy(bcn32_ctx* c) {
    if (!c) return BCN_OK;
    cudaFree(c->tw);
    delete c;
    return BCN_OK;
}

int bcn32_ntt_fwd(bcn32_ctx* c, uint32_t* data, int npoly, void* stream) {
    if (!c || !data) return fail32(BCN_ERR_PARAM, "null argument");
    cudaError_t e = ntt_w_launch<u32>(false, c->logn, data, c->tw, c->k, c->nlimb, npoly, (cudaStream_t)stream);
    return e == cudaSuccess ? BCN_OK : cuda_fail32(e);
}

int bcn32_ntt_inv(bcn32_ctx* c, uint32_t* data, int npoly, void* stream) {
    if (!c || !data) return fail32(BCN_ERR_PARAM, "null argument");
    cudaError_t e = ntt_w_launch<u32>(true, c->logn, data, c->tw, c->k, c->nlimb, npoly, (cudaStream_t)stream);
    return e == cudaSuccess ? BCN_OK : cuda_fail32(e);
}

int bcn32_to_montgomery(bcn32_ctx* c, uint32_t* out, const uint32_t* in, int npoly, void* stream) {
    if (!c || !out || !in) return fail32(BCN_ERR_PARAM, "null argument");
    const size_t total = (size_t)npoly * c->nlimb * c->N;
    if (!total) return BCN_OK;
    to_mont32_kernel<<<(unsigned)std::min<size_t>((total + 255) / 256, 148 * 16), 256, 0, (cudaStream_t)stream>>>(
        out, in, c->k, c->nlimb, c->N, total);
    cudaError_t e = launched();
    return e == cudaSuccess ? BCN_OK : cuda_fail32(e);
}

int bcn32_ntt_mac_rescale(bcn32_ctx* c, uint32_t* out, const uint32_t* ct, const uint32_t* pt_mont, int n_items,
                          int group, void* stream) {
    if (!c || !out || !ct || !pt_mont) return fail32(BCN_ERR_PARAM, "null argument");
    if (n_items < 0 || group < 1) return fail32(BCN_ERR_PARAM, "bad n_items / group");
    NmrArgs<u32> a;
    a.ct = ct; a.pt = pt_mont; a.out = out; a.tw = c->tw;
    a.n_items = n_items; a.group = group; a.nlimb = c->nlimb; a.k = c->k;
    cudaError_t e = ntt_mac_rescale_launch<u32>(a, c->logn, (cudaStream_t)stream);
    return e == cudaSuccess ? BCN_OK : cuda_fail32(e);
}

}  // extern "C"
