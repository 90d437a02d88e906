// ntt_cluster.cu -- NTT / INTT for N = 2^13, 2^14 on a thread-block cluster
// (distributed shared memory): 2 CTAs x 32 KiB at N = 2^13, 4 CTAs x 32 KiB
// at N = 2^14 (BCN_CLUSTER2 builds the 2 x 64 KiB variant for comparison).
//
// The single-CTA kernel (ntt.cu) needs the whole limb-polynomial in SMEM
// (128 KiB at N = 2^14), so only one CTA fits per SM and its global-load,
// butterfly and store phases cannot overlap with another CTA.  Here the
// polynomial is split over a cluster of CS CTAs with N/CS words each, so
// 4 independent CTAs share an SM and hide each other's barriers:
//   forward: pass A (the first R0 >= log2 CS stages, blocks strided by
//            N/2^R0) reads HBM directly, each CTA taking 1/CS of the blocks;
//            its outputs are written to the SMEM of the CTA that owns their
//            part (local or peer via DSMEM); one cluster barrier; the
//            remaining radix-16 passes only touch the CTA's own part; the
//            last pass writes HBM.
//   inverse: the mirror image -- local passes first, one cluster barrier,
//            pass A reads its inputs from the owners' SMEM.
// Output order and values are exactly those of ntt.cu (same contract with
// the oracle).  The integer butterflies follow ntt.cu's lazy bounds; the
// FP64 butterflies (primes < 2^50) have their own bounds and a
// pass-transposed twiddle table (see "FP64 butterflies" below).
#include <cooperative_groups.h>

#include "common.cuh"
#include "ops.cuh"

namespace cg = cooperative_groups;

namespace bcn {

template <int LOGN> struct CCfg {
    static constexpr int LOGE = 4;
    static constexpr int N = 1 << LOGN;
#ifdef BCN_CLUSTER2
    static constexpr int LOGCS = 1;
#else
    static constexpr int LOGCS = LOGN >= 14 ? 2 : 1;     // 4 CTAs x 32 KiB at N = 2^14, 2 x 32 KiB at 2^13
#endif
    static constexpr int CS = 1 << LOGCS;                // CTAs per cluster
    static constexpr int PART = N / CS;                  // words owned by one CTA
    static constexpr int E = 1 << LOGE;
    static constexpr int T = N / (CS * E);               // threads per CTA
    static constexpr int R0 = (LOGN % LOGE) ? (LOGN % LOGE) : LOGE;
    static_assert(R0 >= LOGCS, "pass A must cover the cross-CTA stages");
    static constexpr int SWZ = 15;
#ifdef BCN_CNTT_MINB
    static constexpr int MINB = BCN_CNTT_MINB;
#else
    static constexpr int MINB = 65536 / (64 * T);        // resident CTAs per SM at a 64-register budget
#endif
};

// grid order: limb fastest -- consecutive clusters transform consecutive limbs
// of one poly, i.e. one contiguous run of HBM.  With the FP64 butterflies this
// measured faster than poly-fastest order (same prime, same twiddle table for
// consecutive clusters), which the integer kernels had preferred: N = 2^14
// forward 0.115 vs 0.120, inverse 0.105 vs 0.109 us per limb-poly; the cifar3
// forward is unchanged.  Poly-fastest order is kept for launches with more
// than 65535 polys (grid.y limit) and under BCN_NTT_POLY_MAJOR=1.
template <int LOGCS> __device__ __forceinline__ int ntt_limb(const NttArgs& a) {
    return a.grid_pm ? blockIdx.y : blockIdx.x >> LOGCS;
}
template <int LOGCS> __device__ __forceinline__ int ntt_poly(const NttArgs& a) {
    return a.grid_pm ? blockIdx.x >> LOGCS : blockIdx.y;
}

// cluster barrier without the release fence of cluster.sync(): for the
// barriers that only need the peers to have started / to be done reading,
// so the arrive does not wait for this thread's outstanding HBM loads/stores
__device__ __forceinline__ void cluster_sync_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}

__device__ __forceinline__ int cswz(int j) { return j ^ ((j >> 4) & 15); }

// local index of global word j in its owner CTA (owner = j / PART)
template <int LOGN> __device__ __forceinline__ int local_idx(int j) { return j & (CCfg<LOGN>::PART - 1); }

// fused prologue: the value the forward transform reads at position j
template <int MODE>
struct Prologue {             // MODE 0 plain, 1 rescale lift, 2 ModDown base conversion
    const u64* src;           // mode 0: the limb; mode 1: the coefficient-form top limb of this poly
    u64 q, qtop, qtop_mod_q, inv_p;   // inv_p = floor(2^64 / q): v mod q by a Shoup multiply by 1
    __device__ __forceinline__ u64 operator()(int j) const {
        if constexpr (MODE == 0) {
            return src[j];
        } else if constexpr (MODE == 1) {
            const u64 v = src[j];                   // canonical mod qtop, centred lift -> mod q
            u64 r = inv_p ? shoup(v, 1ull, inv_p, q) : csub(v, q);   // inv_p = 0: v < 2q (api.cu, lift1)
            if (v > (qtop >> 1)) r = sub_mod(r, qtop_mod_q, q);
            return r;
        } else {                                    // sum_k y_k[j] * [P/p_k]_q (Montgomery table)
            Acc4 acc;                               // K <= 16 products: no intermediate fold
            acc.zero();
            for (int k = 0; k < K; k++) acc.mac(src[(size_t)k * nstride + j], hat[k * BCN_MAX_LIMBS]);
            return acc.reduce(q, qinv_neg, inv1);
        }
    }
    int K = 0;
    long long nstride = 0;
    const u64* hat = nullptr;   // &conv.hat_m[t]
    u64 qinv_neg = 0;
    u64 inv1 = 0;               // floor(2^64 / q)
};

// fused epilogue: what the forward transform writes for canonical result v at j
template <int MODE>
struct Epilogue {             // MODE 0 store, 1 rescale combine (c - v) * q_top^-1, 2 ModDown combine,
                              // 3 merged ModDown + rescale: (c - v) (P q_l)^-1 + addend q_l^-1,
                              // 4 ModDown combine with c = the key-switch inner product computed here,
                              // 5 encryption: c0 = v - a s with a drawn here (Philox) and stored as c1
    static constexpr int kMode = MODE;
    u64* out;
    const u64* c;
    u64 q, w, wp;
    const u64* add = nullptr;   // ModDown addend for this (ct, component, limb), or null
    u32 g = 1;
    int logn = 0;
    u64 w2 = 0, wp2 = 0;
    const u64* U = nullptr;     // mode 4: U[d * uds + sigma(j)] (this ct, this limb)
    const u64* kp = nullptr;    //         key[d * kds + j] (this component, this limb)
    long long uds = 0, kds = 0;
    int ndig = 0;
    u64 qinv_neg = 0, inv1 = 0;
    // mode 5 (encryption): c0 = v - a s, c1 = a
    const u64* es = nullptr;    // s (Montgomery) for this limb
    u64* out1 = nullptr;        // component 1 of this (ct, limb)
    u64 eseed = 0, eid = 0, r1 = 0, r1s = 0;
    u32 epi_prime = 0;
    __device__ __forceinline__ u64 enc(int j, u64 v, u64& a_out) const {
        PrimeInfo P;
        P.q = q; P.qinv_neg = qinv_neg; P.r1 = r1; P.r1_shoup = r1s; P.pad[2] = inv1;
        const u64 a = uniform_mod(draw(eseed, 1u /*DOM_ENC_A*/, epi_prime, eid, (u32)j), P);
        a_out = a;
        return sub_mod(v, mont_mul(a, __ldg(es + j), q, qinv_neg), q);
    }
    // issue L2 bulk prefetches of everything operator() will read for the
    // words [j0, j0 + part) of this CTA, so those loads overlap the transform
    // instead of following it.  Under X -> X^g an aligned 32-block is the image
    // of one aligned 32-block, so a gathered operand is 256-byte runs.
    __device__ __forceinline__ void prefetch(int j0, int part, int tid, int nthr) const {
        if constexpr (MODE == 0 || MODE == 5) {
            return;
        } else {
            constexpr u32 RUN = 32 * sizeof(u64);
            const bool gather = (MODE == 2 || MODE == 4) && g != 1u;
            for (int b = tid; b < part / 32; b += nthr) {
                const int j = j0 + 32 * b;
                const int sj = gather ? ((int)automorph_src((u32)j, g, logn) & ~31) : j;
                if constexpr (MODE == 4) {
                    for (int d = 0; d < ndig; d++) {
                        bulk_prefetch_l2(U + d * uds + sj, RUN);
                        bulk_prefetch_l2(kp + d * kds + j, RUN);
                    }
                } else {
                    bulk_prefetch_l2(c + j, RUN);
                }
                if (add) bulk_prefetch_l2(add + (MODE == 3 ? j : sj), RUN);
            }
        }
    }
    // modes 1-3 split into operand loads and arithmetic, so the caller can issue the loads of several
    // outputs before the first store (c / add and out are not restrict: the compiler keeps program order)
    __device__ __forceinline__ ulonglong2 load_c(int j) const { return *reinterpret_cast<const ulonglong2*>(c + j); }
    __device__ __forceinline__ ulonglong2 load_add(int j) const {
        if constexpr (MODE == 2) {
            if (g != 1u) return make_ulonglong2(add[(int)automorph_src((u32)j, g, logn)],
                                                add[(int)automorph_src((u32)(j + 1), g, logn)]);
        }
        return *reinterpret_cast<const ulonglong2*>(add + j);
    }
    __device__ __forceinline__ u64 combine(u64 v, u64 cj, u64 aj) const {
        u64 r = shoup(cj + q - v, w, wp, q);
        if constexpr (MODE == 2) {
            if (add) r = add_mod(r, aj, q);
        } else if constexpr (MODE == 3) {
            if (add) r = add_mod(r, shoup(aj, w2, wp2, q), q);
        }
        return r;
    }
    __device__ __forceinline__ u64 operator()(int j, u64 v) const {
        if constexpr (MODE == 0 || MODE == 5) {
            return v;
        } else if constexpr (MODE == 4) {
            // the IMAD-pipe inner product runs inside the FP64-pipe NTT: no A round trip
            const int sj = g == 1u ? j : (int)automorph_src((u32)j, g, logn);
            Acc4 acc;
            acc.zero();
            for (int d = 0; d < ndig; d++) acc.mac(__ldg(U + d * uds + sj), __ldg(kp + d * kds + j));
            const u64 a = acc.reduce(q, qinv_neg, inv1);
            u64 r = shoup(a + q - v, w, wp, q);
            if (add) r = add_mod(r, add[sj], q);
            return r;
        } else {
            u64 r = shoup(c[j] + q - v, w, wp, q);
            if constexpr (MODE == 2) {
                if (add) r = add_mod(r, add[g == 1u ? j : (int)automorph_src((u32)j, g, logn)], q);
            } else if constexpr (MODE == 3) {
                if (add) r = add_mod(r, shoup(add[j], w2, wp2, q), q);
            }
            return r;
        }
    }
};

// ------------------------------------------------------------------ forward
// Lazy bounds of the forward butterflies (q < 2^61, so 8q < 2^64).  Default:
// stage 0 reads canonical input; from stage 2 on, even stages fold the upper
// input into [0, 4q) with one conditional subtraction of 4q and odd stages
// skip it (invariant: inputs < 8q, u < 4q, v < 2q, outputs < 6q / 8q), so
// half of the stages save a 64-bit compare-select.  BCN_NTT_FULL_CSUB keeps
// the classic Harvey schedule (inputs < 4q, csub 2q every stage).  Results
// are canonical either way (identical outputs).
#ifdef BCN_NTT_FULL_CSUB
__device__ __forceinline__ constexpr bool fwd_reduce(int s) { return s > 0; }
__device__ __forceinline__ u64 fwd_rbound(u64 q) { return 2 * q; }
__device__ __forceinline__ u64 fwd_final(u64 x, u64 q) { return csub(csub(x, 2 * q), q); }
#else
__device__ __forceinline__ constexpr bool fwd_reduce(int s) { return s >= 2 && (s & 1) == 0; }
__device__ __forceinline__ u64 fwd_rbound(u64 q) { return 4 * q; }
__device__ __forceinline__ u64 fwd_final(u64 x, u64 q) { return csub(csub(csub(x, 4 * q), 2 * q), q); }
#endif

// Last-pass stores of the combine epilogues (modes 1-3), called right after the thread's canonical results
// went to `su` and BEFORE the CTA barrier: the c (and addend) words of HB outputs are in flight per thread,
// the first batch across the barrier.  One dependent 8-byte load per output measured 28% of the ModDown
// tail's stall samples on the load -> combine edge (profiles/ncu_cfg3_tail_r02_summary.txt).
template <int LOGN, class EPI>
__device__ __forceinline__ void epi_store_batched(const EPI& epi, const u64* su, int rank, int tid) {
    using C = CCfg<LOGN>;
    constexpr int M = C::PART / (2 * C::T), HB = M < 4 ? M : 4;
    const int j0 = rank * C::PART;
    ulonglong2 cv[HB], av[HB];
#pragma unroll
    for (int m0 = 0; m0 < M; m0 += HB) {
#pragma unroll
        for (int i = 0; i < HB; i++) {
            const int e = 2 * tid + (m0 + i) * 2 * C::T;
            cv[i] = epi.load_c(j0 + e);
            av[i] = epi.add ? epi.load_add(j0 + e) : make_ulonglong2(0ull, 0ull);
        }
        if (m0 == 0) __syncthreads();
#pragma unroll
        for (int i = 0; i < HB; i++) {
            const int e = 2 * tid + (m0 + i) * 2 * C::T;
            ulonglong2 v;
            v.x = epi.combine(su[cswz(e)], cv[i].x, av[i].x);
            v.y = epi.combine(su[cswz(e + 1)], cv[i].y, av[i].y);
            *reinterpret_cast<ulonglong2*>(epi.out + j0 + e) = v;
        }
    }
}

template <int LOGN, class PRO>
__device__ __forceinline__ void cfwd_passA(u64* x, const PRO& pro, u64* const* peers, int rank,
                                           const ulonglong2* __restrict__ W, u64 q, int tid) {
    using C = CCfg<LOGN>;
    constexpr int R = C::R0, BS = 1 << R, NB = C::E / BS, TL = C::N >> R;
    const u64 q2 = 2 * q;
#pragma unroll
    for (int i = 0; i < NB; i++) {
        const int b = rank * (TL / C::CS) + tid + i * C::T;    // gi == 0 for S0 == 0
#pragma unroll
        for (int k = 0; k < BS; k++) x[i * BS + k] = pro(b + k * TL);
#pragma unroll
        for (int ls = 0; ls < R; ls++) {
            const int h = BS >> (ls + 1);
#pragma unroll
            for (int k = 0; k < BS; k++) {
                if (k & h) continue;
                const ulonglong2 w = W[(1 << ls) + (k >> (R - ls))];
                u64 u = x[i * BS + k];
                if (fwd_reduce(ls)) u = csub(u, fwd_rbound(q));
                const u64 v = shoup_lazy(x[i * BS + k + h], w.x, w.y, q);
                x[i * BS + k] = u + v;
                x[i * BS + k + h] = u - v + q2;
            }
        }
#pragma unroll
        for (int k = 0; k < BS; k++) {          // word b + k TL belongs to CTA k >> (R0 - LOGCS)
            const int j = b + k * TL;
            peers[k >> (R - C::LOGCS)][cswz(local_idx<LOGN>(j))] = x[i * BS + k];
        }
    }
}

// one local radix-16 pass (S0 >= R0): this CTA's half only
template <int LOGN, int S0, bool LAST, class EPI>
__device__ __forceinline__ void cfwd_pass(u64* x, const EPI& epi, u64* sm, int rank,
                                          const ulonglong2* __restrict__ W, u64 q, int tid) {
    using C = CCfg<LOGN>;
    constexpr int R = C::LOGE, BS = 1 << R, TL = C::N >> (S0 + R);
    const u64 q2 = 2 * q;
    const int b = rank * ((C::N >> R) / C::CS) + tid;
    const int gi = b / TL;
    const int base = gi * (C::N >> S0) + (b % TL);
    const int lbase = base - rank * C::PART;
#pragma unroll
    for (int k = 0; k < BS; k++) x[k] = sm[cswz(lbase + k * TL)];
#pragma unroll
    for (int ls = 0; ls < R; ls++) {
        const int h = BS >> (ls + 1);
        const int s = S0 + ls;
#pragma unroll
        for (int k = 0; k < BS; k++) {
            if (k & h) continue;
            const ulonglong2 w = W[(1 << s) + ((k >> (R - ls)) << S0) + gi];   // pass-transposed table
            const u64 u = fwd_reduce(s) ? csub(x[k], fwd_rbound(q)) : x[k];
            const u64 v = shoup_lazy(x[k + h], w.x, w.y, q);
            x[k] = u + v;
            x[k + h] = u - v + q2;
        }
    }
    if constexpr (LAST) {
        static_assert(TL == 1, "last pass is contiguous");   // coalesced stores via SMEM (see dfwd_pass)
#pragma unroll
        for (int k = 0; k < BS; k++) sm[cswz(lbase + k)] = fwd_final(x[k], q);
#ifndef BCN_EPI_SERIAL
        if constexpr (EPI::kMode >= 1 && EPI::kMode <= 3) {
            epi_store_batched<LOGN, EPI>(epi, sm, rank, tid);
            return;
        }
#endif
        __syncthreads();
        const int j0 = rank * C::PART;
#pragma unroll
        for (int m = 0; m < C::PART / (2 * C::T); m++) {
            const int e = 2 * tid + m * 2 * C::T;
            ulonglong2 v;
            if constexpr (EPI::kMode == 5) {
                ulonglong2 av;
                v.x = epi.enc(j0 + e, sm[cswz(e)], av.x);
                v.y = epi.enc(j0 + e + 1, sm[cswz(e + 1)], av.y);
                *reinterpret_cast<ulonglong2*>(epi.out1 + j0 + e) = av;
            } else {
                v.x = epi(j0 + e, sm[cswz(e)]);
                v.y = epi(j0 + e + 1, sm[cswz(e + 1)]);
            }
            *reinterpret_cast<ulonglong2*>(epi.out + j0 + e) = v;
        }
    } else {
#pragma unroll
        for (int k = 0; k < BS; k++) sm[cswz(lbase + k * TL)] = x[k];
    }
}

template <int LOGN, int S0, class EPI>
__device__ __forceinline__ void cfwd_rest(u64* x, const EPI& epi, u64* sm, int rank,
                                          const ulonglong2* __restrict__ W, u64 q, int tid) {
    using C = CCfg<LOGN>;
    if constexpr (S0 < LOGN) {
        if constexpr (S0 > C::R0) __syncthreads();
        cfwd_pass<LOGN, S0, (S0 + C::LOGE >= LOGN), EPI>(x, epi, sm, rank, W, q, tid);
        cfwd_rest<LOGN, S0 + C::LOGE, EPI>(x, epi, sm, rank, W, q, tid);
    }
}

// ------------------------------------------------- FP64 butterflies (q < 2^50)
// Twiddle table twf: {w, w/q} per entry, and within each stage s of a
// radix-16 pass starting at stage S0 the entries are transposed so that the
// threads of a warp (consecutive block index gi) read consecutive entries:
// twf[2^s + j 2^S0 + gi] = W[2^s + (gi << (s - S0)) + j]  (api.cu builds it;
// one 512-B run per warp-wide load instead of 2^(s-S0) strided lines).
// For primes below 2^50 the butterflies run on the FP64 pipe instead of the
// 64-bit integer multiplies on the IMAD pipe (tools/micro/bfly_bench.cu:
// 6.3 vs 3.1 butterflies/clk/SM on this B200).  Residues are exact integers
// held in doubles, signed, |x| < 2^53; SMEM holds the double bits.  fmm /
// fred are in common.cuh; the twiddles are signed (|w| <= q/2), which widens
// fmm's input range to |a| < 4q, and the reduction schedule is fwd_fred /
// inv_fred below.  Outputs are canonicalised (fred, +q if negative) -- the
// same canonical residues as the integer path, interchangeable bit for bit.
struct FQ {                     // per-prime FP64 constants
    double q, qinv;
};

// FP64 lazy-reduction schedule.  Twiddles are stored signed, |w| <= q/2, so
// fmm(a, w) only needs |a| < 4q (quotient |a w / q| < 2^51) and returns
// |v| <= 0.5q + |a| 2^-55 <= 0.63q.
//   forward (CT): u is reduced on stages s = 4 mod 5; starting from
//     canonical input (or a reduced stage, <= 1.13q) every value stays
//     <= 1.13q + 4 * 0.63q < 3.7q (< 4q: fmm's input bound; < 8q: exact);
//   inverse (GS): the sum is reduced on every other stage counted from the
//     first (t = LOGN-1-s odd); every value stays <= 2q before a reduced
//     stage and <= 1.25q after it, so u - v stays < 4q.
__device__ __forceinline__ constexpr bool fwd_fred(int s) { return s % 5 == 4; }
template <int LOGN> __device__ __forceinline__ constexpr bool inv_fred(int s) { return ((LOGN - 1 - s) & 1) == 1; }

// pass A: the loads (issued before the cluster barrier that guards the
// scatter, so their HBM latency overlaps the barrier wait), then the
// butterflies on registers and the scatter to the owners' SMEM
template <int LOGN, class PRO>
__device__ __forceinline__ void dfwd_passA_load(double* x, const PRO& pro, int rank, int tid) {
    using C = CCfg<LOGN>;
    constexpr int R = C::R0, BS = 1 << R, NB = C::E / BS, TL = C::N >> R;
#pragma unroll
    for (int i = 0; i < NB; i++) {
        const int b = rank * (TL / C::CS) + tid + i * C::T;
#pragma unroll
        for (int k = 0; k < BS; k++) x[i * BS + k] = fload(pro(b + k * TL));
    }
}

template <int LOGN>
__device__ __forceinline__ void dfwd_passA_core(double* x, double* const* peers, int rank,
                                                const double2* __restrict__ W, FQ f, int tid) {
    using C = CCfg<LOGN>;
    constexpr int R = C::R0, BS = 1 << R, NB = C::E / BS, TL = C::N >> R;
#pragma unroll
    for (int i = 0; i < NB; i++) {
        const int b = rank * (TL / C::CS) + tid + i * C::T;
#pragma unroll
        for (int ls = 0; ls < R; ls++) {
            const int h = BS >> (ls + 1);
#pragma unroll
            for (int k = 0; k < BS; k++) {
                if (k & h) continue;
                const double2 w = W[(1 << ls) + (k >> (R - ls))];
                double u = x[i * BS + k];
                if (fwd_fred(ls)) u = fred(u, f.qinv, f.q);
                const double v = fmm(x[i * BS + k + h], w.x, w.y, f.q);
                x[i * BS + k] = __dadd_rn(u, v);
                x[i * BS + k + h] = __dadd_rn(u, -v);
            }
        }
#pragma unroll
        for (int k = 0; k < BS; k++) {
            const int j = b + k * TL;
            peers[k >> (R - C::LOGCS)][cswz(local_idx<LOGN>(j))] = x[i * BS + k];
        }
    }
}

// DSMEM scatter with st.async: each remote store decrements the owner CTA's
// mbarrier transaction count, so the owner waits for exactly its own 32 KiB
// instead of a release-fenced cluster barrier (which drains every thread's
// remote stores and waits for the slowest CTA of the cluster)
__device__ __forceinline__ u32 mapa_rank(u32 saddr, u32 rank) {
    u32 r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_async_f64(u32 raddr, double v, u32 rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
                 "l"(__double_as_longlong(v)), "r"(rbar)
                 : "memory");
}

// bounded wait: a protocol bug traps (launch error) instead of hanging the GPU
__device__ __forceinline__ void mbar_wait_bounded(u64* bar, u32 parity) {
    for (u32 spin = 0;; spin++) {
        u32 done;
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_addr(bar)), "r"(parity)
            : "memory");
        if (done) return;
        if (spin > (1u << 26)) __trap();
    }
}

template <int LOGN>
__device__ __forceinline__ void dfwd_passA_core_async(double* x, const u32* rsm, const u32* rbar, int rank,
                                                      const double2* __restrict__ W, FQ f, int tid) {
    using C = CCfg<LOGN>;
    constexpr int R = C::R0, BS = 1 << R, NB = C::E / BS, TL = C::N >> R;
#pragma unroll
    for (int i = 0; i < NB; i++) {
        const int b = rank * (TL / C::CS) + tid + i * C::T;
#pragma unroll
        for (int ls = 0; ls < R; ls++) {
            const int h = BS >> (ls + 1);
#pragma unroll
            for (int k = 0; k < BS; k++) {
                if (k & h) continue;
                const double2 w = W[(1 << ls) + (k >> (R - ls))];
                double u = x[i * BS + k];
                if (fwd_fred(ls)) u = fred(u, f.qinv, f.q);
                const double v = fmm(x[i * BS + k + h], w.x, w.y, f.q);
                x[i * BS + k] = __dadd_rn(u, v);
                x[i * BS + k + h] = __dadd_rn(u, -v);
            }
        }
#pragma unroll
        for (int k = 0; k < BS; k++) {
            const int j = b + k * TL, r = k >> (R - C::LOGCS);
            st_async_f64(rsm[r] + 8u * (u32)cswz(local_idx<LOGN>(j)), x[i * BS + k], rbar[r]);
        }
    }
}

template <int LOGN, int S0, bool LAST, class EPI>
__device__ __forceinline__ void dfwd_pass(double* x, const EPI& epi, double* sm, int rank,
                                          const double2* __restrict__ W, FQ f, int tid) {
    using C = CCfg<LOGN>;
    constexpr int R = C::LOGE, BS = 1 << R, TL = C::N >> (S0 + R);
    const int b = rank * ((C::N >> R) / C::CS) + tid;
    const int gi = b / TL;
    const int base = gi * (C::N >> S0) + (b % TL);
    const int lbase = base - rank * C::PART;
#pragma unroll
    for (int k = 0; k < BS; k++) x[k] = sm[cswz(lbase + k * TL)];
#pragma unroll
    for (int ls = 0; ls < R; ls++) {
        const int h = BS >> (ls + 1);
        const int s = S0 + ls;
#pragma unroll
        for (int k = 0; k < BS; k++) {
            if (k & h) continue;
            const double2 w = W[(1 << s) + ((k >> (R - ls)) << S0) + gi];   // pass-transposed table
            const double u = fwd_fred(s) ? fred(x[k], f.qinv, f.q) : x[k];
            const double v = fmm(x[k + h], w.x, w.y, f.q);
            x[k] = __dadd_rn(u, v);
            x[k + h] = __dadd_rn(u, -v);
        }
    }
    if constexpr (LAST) {
        // each thread holds 16 consecutive words: exchange through SMEM so that
        // the epilogue's reads and the HBM stores are warp-coalesced (a direct
        // store would touch 32 lines per instruction)
        static_assert(TL == 1, "last pass is contiguous");
        u64* su = reinterpret_cast<u64*>(sm);
#pragma unroll
        for (int k = 0; k < BS; k++) su[cswz(lbase + k)] = fcanon(x[k], f.qinv, f.q);
#ifndef BCN_EPI_SERIAL
        if constexpr (EPI::kMode >= 1 && EPI::kMode <= 3) {
            epi_store_batched<LOGN, EPI>(epi, su, rank, tid);
            return;
        }
#endif
        __syncthreads();
        const int j0 = rank * C::PART;
#pragma unroll
        for (int m = 0; m < C::PART / (2 * C::T); m++) {
            const int e = 2 * tid + m * 2 * C::T;
            ulonglong2 v;
            if constexpr (EPI::kMode == 5) {
                ulonglong2 av;
                v.x = epi.enc(j0 + e, su[cswz(e)], av.x);
                v.y = epi.enc(j0 + e + 1, su[cswz(e + 1)], av.y);
                *reinterpret_cast<ulonglong2*>(epi.out1 + j0 + e) = av;
            } else {
                v.x = epi(j0 + e, su[cswz(e)]);
                v.y = epi(j0 + e + 1, su[cswz(e + 1)]);
            }
            *reinterpret_cast<ulonglong2*>(epi.out + j0 + e) = v;
        }
    } else {
#pragma unroll
        for (int k = 0; k < BS; k++) sm[cswz(lbase + k * TL)] = x[k];
    }
}

template <int LOGN, int S0, class EPI>
__device__ __forceinline__ void dfwd_rest(double* x, const EPI& epi, double* sm, int rank,
                                          const double2* __restrict__ W, FQ f, int tid) {
    using C = CCfg<LOGN>;
    if constexpr (S0 < LOGN) {
        if constexpr (S0 > C::R0) __syncthreads();
        dfwd_pass<LOGN, S0, (S0 + C::LOGE >= LOGN), EPI>(x, epi, sm, rank, W, f, tid);
        dfwd_rest<LOGN, S0 + C::LOGE, EPI>(x, epi, sm, rank, W, f, tid);
    }
}

template <int LOGN, int S0, bool FIRST>
__device__ __forceinline__ void dinv_pass(double* x, const u64* __restrict__ gin, double* sm, int rank,
                                          const double2* __restrict__ Wi, FQ f, int tid) {
    using C = CCfg<LOGN>;
    constexpr int R = C::LOGE, BS = 1 << R, TL = C::N >> (S0 + R);
    const int b = rank * ((C::N >> R) / C::CS) + tid;
    const int gi = b / TL;
    const int base = gi * (C::N >> S0) + (b % TL);
    const int lbase = base - rank * C::PART;
    if constexpr (FIRST) {
        // coalesced HBM reads straight into SMEM (cp.async: no register staging),
        // then the per-thread contiguous runs from SMEM
        static_assert(TL == 1, "first inverse pass is contiguous");
        const int j0 = rank * C::PART;
        u64* su = reinterpret_cast<u64*>(sm);
#pragma unroll
        for (int m = 0; m < C::PART / C::T; m++) {
            const int e = tid + m * C::T;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(su + cswz(e))), "l"(gin + j0 + e)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
        __syncthreads();
#pragma unroll
        for (int k = 0; k < BS; k++) x[k] = fload(su[cswz(lbase + k)]);
    } else {
#pragma unroll
        for (int k = 0; k < BS; k++) x[k] = sm[cswz(lbase + k * TL)];
    }
#pragma unroll
    for (int ls = R - 1; ls >= 0; ls--) {
        const int h = BS >> (ls + 1);
        const int s = S0 + ls;
#pragma unroll
        for (int k = 0; k < BS; k++) {
            if (k & h) continue;
            const double2 w = Wi[(1 << s) + ((k >> (R - ls)) << S0) + gi];  // pass-transposed table
            const double u = x[k], v = x[k + h];
            const double sum = __dadd_rn(u, v);
            x[k] = inv_fred<LOGN>(s) ? fred(sum, f.qinv, f.q) : sum;
            x[k + h] = fmm(__dadd_rn(u, -v), w.x, w.y, f.q);
        }
    }
#pragma unroll
    for (int k = 0; k < BS; k++) sm[cswz(lbase + k * TL)] = x[k];
}

template <int LOGN, int S0>
__device__ __forceinline__ void dinv_rest(double* x, const u64* gin, double* sm, int rank,
                                          const double2* __restrict__ Wi, FQ f, int tid) {
    using C = CCfg<LOGN>;
    if constexpr (S0 >= C::R0) {
        dinv_pass<LOGN, S0, (S0 == LOGN - C::LOGE)>(x, gin, sm, rank, Wi, f, tid);
        if constexpr (S0 - C::LOGE >= C::R0) __syncthreads();
        dinv_rest<LOGN, S0 - C::LOGE>(x, gin, sm, rank, Wi, f, tid);
    }
}

// last inverse stages; the final stage folds n^-1 (x scale) into its two multipliers
template <int LOGN>
__device__ __forceinline__ void dinv_passA(double* x, u64* __restrict__ g, double* const* peers, int rank,
                                           const double2* __restrict__ Wi, FQ f, double2 nw, double2 ww, int tid) {
    using C = CCfg<LOGN>;
    constexpr int R = C::R0, BS = 1 << R, NB = C::E / BS, TL = C::N >> R;
#pragma unroll
    for (int i = 0; i < NB; i++) {
        const int b = rank * (TL / C::CS) + tid + i * C::T;
#pragma unroll
        for (int k = 0; k < BS; k++) {
            const int j = b + k * TL;
            x[i * BS + k] = peers[k >> (R - C::LOGCS)][cswz(local_idx<LOGN>(j))];
        }
#pragma unroll
        for (int ls = R - 1; ls >= 0; ls--) {
            const int h = BS >> (ls + 1);
#pragma unroll
            for (int k = 0; k < BS; k++) {
                if (k & h) continue;
                const double u = x[i * BS + k], v = x[i * BS + k + h];
                if (ls == 0) {
                    x[i * BS + k] = fmm(__dadd_rn(u, v), nw.x, nw.y, f.q);
                    x[i * BS + k + h] = fmm(__dadd_rn(u, -v), ww.x, ww.y, f.q);
                } else {
                    const double2 w = Wi[(1 << ls) + (k >> (R - ls))];
                    const double sum = __dadd_rn(u, v);
                    x[i * BS + k] = inv_fred<LOGN>(ls) ? fred(sum, f.qinv, f.q) : sum;
                    x[i * BS + k + h] = fmm(__dadd_rn(u, -v), w.x, w.y, f.q);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < BS; k++) g[b + k * TL] = fcanon_small(x[i * BS + k], f.q);
    }
}

__device__ __forceinline__ double2 fpair(u64 w, double q) {      // signed twiddle pair (see fwd_fred)
    double wd = (double)w;
    if (wd > 0.5 * q) wd = __dadd_rn(wd, -q);
    return make_double2(wd, __ddiv_rn(wd, q));
}

__device__ __forceinline__ bool cskip(const NttArgs& a, int t, int poly) {
    if (a.skip_alpha <= 0) return false;
    return t <= a.skip_level && t / a.skip_alpha == poly % a.skip_dnum;
}

template <int LOGN, int PM, int EM, bool FPO = false>   // FPO: FP64-only instantiation (see ntt_inv_cluster)
__global__ void __cluster_dims__(CCfg<LOGN>::CS, 1, 1) __launch_bounds__(CCfg<LOGN>::T, CCfg<LOGN>::MINB)
    ntt_fwd_cluster(NttArgs a) {
    using C = CCfg<LOGN>;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ u64 sm[];
    const int rank = (int)cluster.block_rank();
    const int t = ntt_limb<C::LOGCS>(a), poly = ntt_poly<C::LOGCS>(a);
    if (cskip(a, t, poly)) {                // all CTAs of the cluster skip together
        if (a.copy_src) {                    // ModUp: the digit's own limb, already in NTT form
            const ulonglong2* src = reinterpret_cast<const ulonglong2*>(
                a.copy_src + (size_t)(poly / a.skip_dnum) * a.copy_stride + (size_t)t * C::N + rank * C::PART);
            ulonglong2* dst = reinterpret_cast<ulonglong2*>(
                a.data + (size_t)poly * a.poly_stride + (size_t)t * C::N + rank * C::PART);
            for (int i = threadIdx.x; i < C::PART / 2; i += C::T) dst[i] = src[i];
        }
        return;
    }
    u64* peers[C::CS];
#pragma unroll
    for (int r = 0; r < C::CS; r++) peers[r] = cluster.map_shared_rank(sm, r);
    const int pidx = a.limbs.prime[t];
    const u64 q = a.pr[pidx].q;
    const ulonglong2* W = a.twt + (size_t)pidx * 2 * C::N;
    u64* g = a.data + (size_t)poly * a.poly_stride + (size_t)t * C::N;
    const u64* gin = a.src ? a.src + (size_t)poly * a.src_poly_stride + (size_t)t * a.src_limb_stride : g;
    Prologue<PM> pro;
    pro.q = q;
    if constexpr (PM == 1) {
        pro.src = a.pro_src + (size_t)poly * a.pro_stride;
        pro.qtop = a.pro_qtop;
        pro.qtop_mod_q = a.pro_tab[2 * t];
        pro.inv_p = a.pro_tab[2 * t + 1];
    } else if constexpr (PM == 2) {
        if (a.pro_dnum > 0) {                // ModUp: digit poly % dnum of entry poly / dnum
            const int d = poly % a.pro_dnum;
            const ConvTable* tab = a.pro_conv + d;
            pro.src = a.pro_src + (size_t)(poly / a.pro_dnum) * a.pro_stride + (size_t)d * a.pro_dstride;
            pro.K = tab->n_src;
            pro.hat = tab->hat_m + t;
        } else {                             // ModDown: the special limbs of poly
            pro.src = a.pro_src + (size_t)poly * a.pro_stride;
            pro.K = a.pro_K;
            pro.hat = a.pro_conv->hat_m + t;
        }
        pro.nstride = C::N;
        pro.qinv_neg = a.pr[pidx].qinv_neg;
        pro.inv1 = a.pr[pidx].pad[2];
        pro.qtop = pro.qtop_mod_q = pro.inv_p = 0;
    } else {
        pro.src = gin;
        pro.qtop = pro.qtop_mod_q = pro.inv_p = 0;
    }
    Epilogue<EM> epi;
    epi.out = g;
    epi.q = q;
    if constexpr (EM == 1 || EM == 2 || EM == 3 || EM == 4) {
        epi.c = EM == 4 ? nullptr : a.epi_c + (size_t)poly * a.epi_cps + (size_t)t * a.epi_cls;
        epi.w = a.epi_tab[2 * t];
        epi.wp = a.epi_tab[2 * t + 1];
        if constexpr (EM == 4) {
            const int kt = a.limbs.prime[t];
            epi.U = a.epi_U + (size_t)(poly >> 1) * a.epi_Ups + (size_t)t * C::N;
            epi.uds = a.epi_Uds;
            epi.kp = a.epi_key + (size_t)(poly & 1) * a.epi_kcs + (size_t)kt * C::N;
            epi.kds = a.epi_kds;
            epi.ndig = a.epi_ndig;
            epi.qinv_neg = a.pr[pidx].qinv_neg;
            epi.inv1 = a.pr[pidx].pad[2];
        }
        if constexpr (EM == 2 || EM == 3 || EM == 4) {
            const int comp = poly & 1;
            const long long acs = a.epi_acs ? a.epi_acs : (long long)a.limbs.n * C::N;
            epi.add = (a.epi_add && (comp == 0 || a.epi_add_c1))
                          ? a.epi_add + (size_t)(poly >> 1) * a.epi_aps + (size_t)comp * acs + (size_t)t * C::N
                          : nullptr;
            epi.g = a.epi_g;
            epi.logn = LOGN;
            if constexpr (EM == 3) {
                epi.w2 = a.epi_tab2[2 * t];
                epi.wp2 = a.epi_tab2[2 * t + 1];
            }
        }
    } else if constexpr (EM == 5) {
        epi.c = nullptr;
        epi.w = epi.wp = 0;
        const PrimeInfo& PI = a.pr[pidx];
        epi.qinv_neg = PI.qinv_neg;
        epi.inv1 = PI.pad[2];
        epi.r1 = PI.r1;
        epi.r1s = PI.r1_shoup;
        epi.epi_prime = (u32)pidx;
        epi.es = a.enc_s + (size_t)pidx * C::N;
        epi.eseed = a.enc_seed;
        epi.eid = (a.enc_id_dev ? *a.enc_id_dev : a.enc_id) + (u64)poly;
        epi.out1 = g + a.enc_c1_off;
    } else {
        epi.c = nullptr;
        epi.w = epi.wp = 0;
    }
    const int tid = threadIdx.x;
    if constexpr (EM != 0 && EM != 5) {
        if (a.epi_pf) epi.prefetch(rank * C::PART, C::PART, tid, C::T);
    }
    if (a.twf && q < (1ull << 50)) {         // FP64 butterflies (uniform per cluster: one limb)
        double* dpeers[C::CS];
#pragma unroll
        for (int r = 0; r < C::CS; r++) dpeers[r] = reinterpret_cast<double*>(peers[r]);
        const double2* Wf = a.twf + (size_t)pidx * 2 * C::N;
        FQ f;
        f.q = (double)q;
        f.qinv = 1.0 / f.q;
        double xf[C::E];
        __shared__ __align__(8) u64 xbar;
        if (tid == 0) {
            mbar_init(&xbar, 1);
            fence_barrier_init();
        }
        dfwd_passA_load<LOGN, Prologue<PM>>(xf, pro, rank, tid);
        cluster_sync_relaxed();   // peers are running and their barriers initialised
        if (tid == 0) mbar_expect_tx(&xbar, (u32)(C::PART * sizeof(double)));
        u32 rsm[C::CS], rbar[C::CS];
#pragma unroll
        for (int r = 0; r < C::CS; r++) {
            rsm[r] = mapa_rank(smem_addr(sm), (u32)r);
            rbar[r] = mapa_rank(smem_addr(&xbar), (u32)r);
        }
        dfwd_passA_core_async<LOGN>(xf, rsm, rbar, rank, Wf, f, tid);
        mbar_wait_bounded(&xbar, 0);         // this CTA's PART words have all landed
        dfwd_rest<LOGN, C::R0, Epilogue<EM>>(xf, epi, reinterpret_cast<double*>(sm), rank, Wf, f, tid);
        (void)dpeers;
        return;
    }
    if constexpr (FPO) {
        __trap();                            // the launcher checked every limb is below 2^50
    } else {
    u64 x[C::E];
    cluster_sync_relaxed();   // peers are running (no ordering needed)
    cfwd_passA<LOGN, Prologue<PM>>(x, pro, peers, rank, W, q, tid);
    cluster.sync();                          // all chunks delivered
    cfwd_rest<LOGN, C::R0, Epilogue<EM>>(x, epi, sm, rank, W, q, tid);
    }
}

// ------------------------------------------------------------------ inverse
template <int LOGN, int S0, bool FIRST>
__device__ __forceinline__ void cinv_pass(u64* x, const u64* __restrict__ gin, u64* sm, int rank,
                                          const ulonglong2* __restrict__ Wi, u64 q, int tid) {
    using C = CCfg<LOGN>;
    constexpr int R = C::LOGE, BS = 1 << R, TL = C::N >> (S0 + R);
    const u64 q2 = 2 * q;
    const int b = rank * ((C::N >> R) / C::CS) + tid;
    const int gi = b / TL;
    const int base = gi * (C::N >> S0) + (b % TL);
    const int lbase = base - rank * C::PART;
    if constexpr (FIRST) {
        static_assert(TL == 1, "first inverse pass is contiguous");   // coalesced loads via SMEM
        const int j0 = rank * C::PART;
#pragma unroll
        for (int m = 0; m < C::PART / (2 * C::T); m++) {
            const int e = 2 * tid + m * 2 * C::T;
            const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(gin + j0 + e);
            sm[cswz(e)] = v.x;
            sm[cswz(e + 1)] = v.y;
        }
        __syncthreads();
    }
#pragma unroll
    for (int k = 0; k < BS; k++) x[k] = sm[cswz(lbase + k * TL)];
#pragma unroll
    for (int ls = R - 1; ls >= 0; ls--) {
        const int h = BS >> (ls + 1);
        const int s = S0 + ls;
#pragma unroll
        for (int k = 0; k < BS; k++) {
            if (k & h) continue;
            const ulonglong2 w = Wi[(1 << s) + ((k >> (R - ls)) << S0) + gi];  // pass-transposed table
            const u64 u = x[k], v = x[k + h];
            x[k] = csub(u + v, q2);
            x[k + h] = shoup_lazy(u - v + q2, w.x, w.y, q);
        }
    }
#pragma unroll
    for (int k = 0; k < BS; k++) sm[cswz(lbase + k * TL)] = x[k];
}

template <int LOGN, int S0>
__device__ __forceinline__ void cinv_rest(u64* x, const u64* gin, u64* sm, int rank, const ulonglong2* __restrict__ Wi,
                                          u64 q, int tid) {
    using C = CCfg<LOGN>;
    if constexpr (S0 >= C::R0) {
        cinv_pass<LOGN, S0, (S0 == LOGN - C::LOGE)>(x, gin, sm, rank, Wi, q, tid);
        if constexpr (S0 - C::LOGE >= C::R0) __syncthreads();
        cinv_rest<LOGN, S0 - C::LOGE>(x, gin, sm, rank, Wi, q, tid);
    }
}

template <int LOGN>
__device__ __forceinline__ void cinv_passA(u64* x, u64* __restrict__ g, u64* const* peers, int rank,
                                           const ulonglong2* __restrict__ Wi, u64 q, u64 ninv, u64 ninv_p, u64 wn,
                                           u64 wn_p, int tid) {
    using C = CCfg<LOGN>;
    constexpr int R = C::R0, BS = 1 << R, NB = C::E / BS, TL = C::N >> R;
    const u64 q2 = 2 * q;
#pragma unroll
    for (int i = 0; i < NB; i++) {
        const int b = rank * (TL / C::CS) + tid + i * C::T;
#pragma unroll
        for (int k = 0; k < BS; k++) {
            const int j = b + k * TL;
            x[i * BS + k] = peers[k >> (R - C::LOGCS)][cswz(local_idx<LOGN>(j))];
        }
#pragma unroll
        for (int ls = R - 1; ls >= 0; ls--) {
            const int h = BS >> (ls + 1);
#pragma unroll
            for (int k = 0; k < BS; k++) {
                if (k & h) continue;
                const u64 u = x[i * BS + k], v = x[i * BS + k + h];
                if (ls == 0) {
                    x[i * BS + k] = shoup(u + v, ninv, ninv_p, q);
                    x[i * BS + k + h] = shoup(u - v + q2, wn, wn_p, q);
                } else {
                    const ulonglong2 w = Wi[(1 << ls) + (k >> (R - ls))];
                    x[i * BS + k] = csub(u + v, q2);
                    x[i * BS + k + h] = shoup_lazy(u - v + q2, w.x, w.y, q);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < BS; k++) g[b + k * TL] = x[i * BS + k];
    }
}

// FPO: every limb of the launch is below 2^50, so the integer path is not
// compiled in (fewer registers, no spills: measured 0.108 vs 0.115 us per
// N = 2^14 limb-poly)
template <int LOGN, bool FPO>
__global__ void __cluster_dims__(CCfg<LOGN>::CS, 1, 1) __launch_bounds__(CCfg<LOGN>::T, CCfg<LOGN>::MINB)
    ntt_inv_cluster(NttArgs a) {
    using C = CCfg<LOGN>;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ u64 sm[];
    const int rank = (int)cluster.block_rank();
    const int t = ntt_limb<C::LOGCS>(a), poly = ntt_poly<C::LOGCS>(a);
    u64* peers[C::CS];
#pragma unroll
    for (int r = 0; r < C::CS; r++) peers[r] = cluster.map_shared_rank(sm, r);
    const int pidx = a.limbs.prime[t];
    const PrimeInfo& P = a.pr[pidx];
    const u64 q = P.q;
    const ulonglong2* Wi = a.twt + (size_t)pidx * 2 * C::N + C::N;
    u64* g = a.data + (size_t)poly * a.poly_stride + (size_t)t * C::N;
    const u64* gin = a.src ? a.src + (size_t)poly * a.src_poly_stride + (size_t)t * a.src_limb_stride : g;
    const int tid = threadIdx.x;
    if (a.twf && q < (1ull << 50)) {         // FP64 butterflies
        double* dpeers[C::CS];
#pragma unroll
        for (int r = 0; r < C::CS; r++) dpeers[r] = reinterpret_cast<double*>(peers[r]);
        const double2* Wif = a.twf + (size_t)pidx * 2 * C::N + C::N;
        FQ f;
        f.q = (double)q;
        f.qinv = 1.0 / f.q;
        double xf[C::E];
        dinv_rest<LOGN, LOGN - C::LOGE>(xf, gin, reinterpret_cast<double*>(sm), rank, Wif, f, tid);
        cluster.sync();
        double2 nw, ww;
        if (a.inv_scale) {
            const u64* sc = a.inv_scale + 4 * t;
            nw = fpair(sc[0], f.q);
            ww = fpair(sc[2], f.q);
        } else {
            nw = fpair(P.pad[0], f.q);
            ww = Wif[0];
        }
        dinv_passA<LOGN>(xf, g, dpeers, rank, Wif, f, nw, ww, tid);
        cluster_sync_relaxed();   // peers' reads of our SMEM have returned (their values were stored)
        return;
    }
    if constexpr (FPO) {
        __trap();                            // the launcher checked every limb is below 2^50
    } else {
    u64 x[C::E];
    cinv_rest<LOGN, LOGN - C::LOGE>(x, gin, sm, rank, Wi, q, tid);
    cluster.sync();                          // both halves complete
    const ulonglong2 wn = Wi[0];
    if (a.inv_scale) {
        const u64* sc = a.inv_scale + 4 * t;
        cinv_passA<LOGN>(x, g, peers, rank, Wi, q, sc[0], sc[1], sc[2], sc[3], tid);
    } else {
        cinv_passA<LOGN>(x, g, peers, rank, Wi, q, P.pad[0], P.pad[1], wn.x, wn.y, tid);
    }
    cluster_sync_relaxed();   // peers' reads of our SMEM have returned (their values were stored)
    }
}

template <int LOGN>
static cudaError_t launch_cluster(bool inverse, const NttArgs& a, int nlimbs, int npolys, cudaStream_t st) {
    using C = CCfg<LOGN>;
    const size_t smem = (size_t)C::PART * sizeof(u64);
    static unsigned long long smem_cfg = 0;
    unsigned long long smem_bit = 0;
    if (first_on_device(&smem_cfg, &smem_bit)) {
        cudaError_t ae = cudaSuccess;
        BCN_SMEM_ATTR(ae, (ntt_fwd_cluster<LOGN, 0, 0>), (int)smem);
        BCN_SMEM_ATTR(ae, (ntt_fwd_cluster<LOGN, 1, 1>), (int)smem);
        BCN_SMEM_ATTR(ae, (ntt_fwd_cluster<LOGN, 2, 2>), (int)smem);
        BCN_SMEM_ATTR(ae, (ntt_fwd_cluster<LOGN, 2, 0>), (int)smem);
        BCN_SMEM_ATTR(ae, (ntt_fwd_cluster<LOGN, 2, 3>), (int)smem);
        BCN_SMEM_ATTR(ae, (ntt_fwd_cluster<LOGN, 0, 2>), (int)smem);
        BCN_SMEM_ATTR(ae, (ntt_fwd_cluster<LOGN, 1, 2>), (int)smem);
        BCN_SMEM_ATTR(ae, (ntt_fwd_cluster<LOGN, 0, 4>), (int)smem);
        BCN_SMEM_ATTR(ae, (ntt_fwd_cluster<LOGN, 1, 4>), (int)smem);
        BCN_SMEM_ATTR(ae, (ntt_fwd_cluster<LOGN, 0, 3>), (int)smem);
        BCN_SMEM_ATTR(ae, (ntt_fwd_cluster<LOGN, 0, 3, true>), (int)smem);
        BCN_SMEM_ATTR(ae, (ntt_fwd_cluster<LOGN, 0, 5>), (int)smem);
        BCN_SMEM_ATTR(ae, (ntt_inv_cluster<LOGN, false>), (int)smem);
        BCN_SMEM_ATTR(ae, (ntt_inv_cluster<LOGN, true>), (int)smem);
        if (ae != cudaSuccess) return ae;
        smem_cfg |= smem_bit;
    }
    static const bool pm_env = getenv("BCN_NTT_POLY_MAJOR") && getenv("BCN_NTT_POLY_MAJOR")[0] == '1';
    NttArgs b = a;
    b.grid_pm = (pm_env || npolys > 65535) ? 1 : 0;
    // BCN_EPI_PREFETCH=1: L2 bulk prefetch of the fused epilogue's operands at kernel
    // start -- measured slower (config-3 rotations 65.8 -> 70.2 ms, cifar3 step unchanged)
    static const bool pf_on = getenv("BCN_EPI_PREFETCH") && getenv("BCN_EPI_PREFETCH")[0] == '1';
    b.epi_pf = pf_on ? 1 : 0;
    const dim3 grid = b.grid_pm ? dim3(C::CS * npolys, nlimbs) : dim3(C::CS * nlimbs, npolys);
    // FP64-only instantiations where they measured faster (the inverse, the merged tails
    // <0,3>: 74.8 -> 70.9 ms per cifar3 forward); the plain forward <0,0> measured slower
    const bool fpo = a.twf && a.fp_all;
    if (inverse && a.twf && a.fp_all) ntt_inv_cluster<LOGN, true><<<grid, C::T, smem, st>>>(b);
    else if (inverse) ntt_inv_cluster<LOGN, false><<<grid, C::T, smem, st>>>(b);
    else if (fpo && a.pro == 0 && a.epi == 3) ntt_fwd_cluster<LOGN, 0, 3, true><<<grid, C::T, smem, st>>>(b);
    else if (a.pro == 1 && a.epi == 1) ntt_fwd_cluster<LOGN, 1, 1><<<grid, C::T, smem, st>>>(b);
    else if (a.pro == 2 && a.epi == 2) ntt_fwd_cluster<LOGN, 2, 2><<<grid, C::T, smem, st>>>(b);
    else if (a.pro == 2 && a.epi == 0) ntt_fwd_cluster<LOGN, 2, 0><<<grid, C::T, smem, st>>>(b);
    else if (a.pro == 2 && a.epi == 3) ntt_fwd_cluster<LOGN, 2, 3><<<grid, C::T, smem, st>>>(b);
    else if (a.pro == 0 && a.epi == 2) ntt_fwd_cluster<LOGN, 0, 2><<<grid, C::T, smem, st>>>(b);
    else if (a.pro == 1 && a.epi == 2) ntt_fwd_cluster<LOGN, 1, 2><<<grid, C::T, smem, st>>>(b);
    else if (a.pro == 0 && a.epi == 4) ntt_fwd_cluster<LOGN, 0, 4><<<grid, C::T, smem, st>>>(b);
    else if (a.pro == 1 && a.epi == 4) ntt_fwd_cluster<LOGN, 1, 4><<<grid, C::T, smem, st>>>(b);
    else if (a.pro == 0 && a.epi == 3) ntt_fwd_cluster<LOGN, 0, 3><<<grid, C::T, smem, st>>>(b);
    else if (a.pro == 0 && a.epi == 5) ntt_fwd_cluster<LOGN, 0, 5><<<grid, C::T, smem, st>>>(b);
    else ntt_fwd_cluster<LOGN, 0, 0><<<grid, C::T, smem, st>>>(b);
    return launched();
}

cudaError_t ntt_cluster_launch(bool inverse, int logn, const NttArgs& a, int nlimbs, int npolys, cudaStream_t st) {
    if (nlimbs <= 0 || npolys <= 0) return cudaSuccess;
    if (logn == 13) return launch_cluster<13>(inverse, a, nlimbs, npolys, st);
    if (logn == 14) return launch_cluster<14>(inverse, a, nlimbs, npolys, st);
    return cudaErrorInvalidValue;
}

}  // namespace bcn
