// ntt.cu -- batched negacyclic NTT / INTT over RNS limbs (K1/K2).
//
// One CTA transforms one limb-polynomial (N <= 2^14 u64 words = 128 KiB,
// staged in shared memory).  Each thread owns E = 2^LOGE words; a pass
// performs LOGE Cooley-Tukey (forward) or Gentleman-Sande (inverse) stages
// entirely in registers on blocks of E words spaced t_last apart, so the
// 13/14 stages cost 3 shared-memory round trips instead of 13/14.  Twiddles
// {w, floor(w 2^64/q)} are interleaved 16-byte pairs (one LDG.128 each) and
// stay L2-resident across the batch.  Harvey lazy butterflies keep values in
// [0, 4q) (forward) / [0, 2q) (inverse); outputs are canonical.
//
// Ordering (the contract with oracle/ckks_oracle.c): forward output index k
// holds a(psi^(2 brev(k) + 1)); the inverse takes that order back to
// coefficients and folds N^-1 into its final stage.
#include <cstdlib>

#include <vector>

#include "common.cuh"
#include "ops.cuh"

namespace bcn {

template <int LOGN> struct NttCfg {
    static constexpr int LOGE = LOGN >= 14 ? 4 : (LOGN >= 10 ? 3 : (LOGN >= 8 ? 2 : 1));
    static constexpr int N = 1 << LOGN;
    static constexpr int E = 1 << LOGE;
    static constexpr int T = N / E;
    static constexpr int R0 = (LOGN % LOGE) ? (LOGN % LOGE) : LOGE;
    static constexpr int SWZ = E >= 8 ? 15 : E - 1;   // conflict-free for every pass (tools/swizzle_check)
};

template <int LOGE, int SWZ>
__device__ __forceinline__ int swz(int j) { return j ^ ((j >> LOGE) & SWZ); }

// ---------------------------------------------------------------- forward
template <int LOGN, int S0, int R, bool FIRST, bool LAST>
__device__ __forceinline__ void fwd_pass(u64* x, u64* __restrict__ g, u64* sm,
                                         const ulonglong2* __restrict__ W, u64 q, int tid) {
    using C = NttCfg<LOGN>;
    constexpr int BS = 1 << R;               // block size
    constexpr int NB = C::E / BS;            // blocks per thread
    constexpr int TL = C::N >> (S0 + R);     // element stride inside a block
    const u64 q2 = 2 * q;
#pragma unroll
    for (int i = 0; i < NB; i++) {
        const int b = tid + i * C::T;
        const int gi = b / TL;
        const int base = gi * (C::N >> S0) + (b % TL);
#pragma unroll
        for (int k = 0; k < BS; k++) {
            const int j = base + k * TL;
            x[i * BS + k] = FIRST ? g[j] : sm[swz<C::LOGE, C::SWZ>(j)];
        }
#pragma unroll
        for (int ls = 0; ls < R; ls++) {
            constexpr int dummy = 0; (void)dummy;
            const int h = BS >> (ls + 1);
            const int s = S0 + ls;
#pragma unroll
            for (int k = 0; k < BS; k++) {
                if (k & h) continue;
                const ulonglong2 w = W[(1 << s) + (gi << ls) + (k >> (R - ls))];
                u64 u = x[i * BS + k];
                if (!(FIRST && ls == 0)) u = csub(u, q2);   // canonical input needs no fold
                const u64 v = shoup_lazy(x[i * BS + k + h], w.x, w.y, q);
                x[i * BS + k] = u + v;
                x[i * BS + k + h] = u - v + q2;
            }
        }
        if constexpr (LAST && TL == 1) {
            // final pass: a thread owns BS consecutive words -> 16-byte stores
#pragma unroll
            for (int k = 0; k < BS; k += 2) {
                ulonglong2 v;
                v.x = csub(csub(x[i * BS + k], q2), q);
                v.y = csub(csub(x[i * BS + k + 1], q2), q);
                *reinterpret_cast<ulonglong2*>(g + base + k) = v;
            }
        } else {
#pragma unroll
            for (int k = 0; k < BS; k++) {
                const int j = base + k * TL;
                u64 v = x[i * BS + k];
                if (LAST) v = csub(csub(v, q2), q);
                sm[swz<C::LOGE, C::SWZ>(j)] = v;
            }
        }
    }
}

template <int LOGN, int S0>
__device__ __forceinline__ void fwd_rest(u64* x, u64* g, u64* sm, const ulonglong2* __restrict__ W, u64 q, int tid) {
    using C = NttCfg<LOGN>;
    if constexpr (S0 < LOGN) {
        __syncthreads();
        fwd_pass<LOGN, S0, C::LOGE, false, (S0 + C::LOGE >= LOGN)>(x, g, sm, W, q, tid);
        fwd_rest<LOGN, S0 + C::LOGE>(x, g, sm, W, q, tid);
    }
}

__device__ __forceinline__ bool skip_limb(const NttArgs& a, int t, int poly) {
    if (a.skip_alpha <= 0) return false;
    const int d = poly % a.skip_dnum;
    return t <= a.skip_level && t / a.skip_alpha == d;
}

template <int LOGN>
__global__ void __launch_bounds__(NttCfg<LOGN>::T) ntt_fwd_kernel(NttArgs a) {
    using C = NttCfg<LOGN>;
    extern __shared__ u64 sm[];
    const int t = blockIdx.x, poly = blockIdx.y;
    if (skip_limb(a, t, poly)) return;
    const int pidx = a.limbs.prime[t];
    const u64 q = a.pr[pidx].q;
    const ulonglong2* W = a.tw + (size_t)pidx * 2 * C::N;
    u64* g = a.data + (size_t)poly * a.poly_stride + (size_t)t * C::N;
    const u64* gin = a.src ? a.src + (size_t)poly * a.src_poly_stride + (size_t)t * a.src_limb_stride : g;
    u64 x[C::E];
    const int tid = threadIdx.x;
    fwd_pass<LOGN, 0, C::R0, true, (C::R0 >= LOGN)>(x, const_cast<u64*>(gin), sm, W, q, tid);
    fwd_rest<LOGN, C::R0>(x, g, sm, W, q, tid);
}

// ---------------------------------------------------------------- inverse
template <int LOGN, int S0, int R, bool LAST, bool FIRST = false>
__device__ __forceinline__ void inv_pass(u64* x, u64* __restrict__ g, const u64* __restrict__ gin, u64* sm,
                                         const ulonglong2* __restrict__ Wi, u64 q,
                                         u64 ninv, u64 ninv_p, u64 wn, u64 wn_p, int tid) {
    using C = NttCfg<LOGN>;
    constexpr int BS = 1 << R;
    constexpr int NB = C::E / BS;
    constexpr int TL = C::N >> (S0 + R);
    const u64 q2 = 2 * q;
#pragma unroll
    for (int i = 0; i < NB; i++) {
        const int b = tid + i * C::T;
        const int gi = b / TL;
        const int base = gi * (C::N >> S0) + (b % TL);
        if constexpr (FIRST && TL == 1) {
#pragma unroll
            for (int k = 0; k < BS; k += 2) {
                const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(gin + base + k);
                x[i * BS + k] = v.x;
                x[i * BS + k + 1] = v.y;
            }
        } else {
#pragma unroll
            for (int k = 0; k < BS; k++) x[i * BS + k] = sm[swz<C::LOGE, C::SWZ>(base + k * TL)];
        }
#pragma unroll
        for (int ls = R - 1; ls >= 0; ls--) {
            const int h = BS >> (ls + 1);
            const int s = S0 + ls;
#pragma unroll
            for (int k = 0; k < BS; k++) {
                if (k & h) continue;
                const u64 u = x[i * BS + k], v = x[i * BS + k + h];
                if (LAST && s == 0) {
                    // final stage: fold N^-1 (x[k] *= n^-1, x[k+h] *= w n^-1)
                    x[i * BS + k] = shoup(u + v, ninv, ninv_p, q);
                    x[i * BS + k + h] = shoup(u - v + q2, wn, wn_p, q);
                } else {
                    const ulonglong2 w = Wi[(1 << s) + (gi << ls) + (k >> (R - ls))];
                    x[i * BS + k] = csub(u + v, q2);
                    x[i * BS + k + h] = shoup_lazy(u - v + q2, w.x, w.y, q);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < BS; k++) {
            const int j = base + k * TL;
            if (LAST) g[j] = x[i * BS + k];
            else sm[swz<C::LOGE, C::SWZ>(j)] = x[i * BS + k];
        }
    }
}

template <int LOGN, int S0>
__device__ __forceinline__ void inv_rest(u64* x, u64* g, const u64* gin, u64* sm, const ulonglong2* __restrict__ Wi,
                                         u64 q, u64 ninv, u64 ninv_p, u64 wn, u64 wn_p, int tid) {
    using C = NttCfg<LOGN>;
    if constexpr (S0 >= C::R0) {
        inv_pass<LOGN, S0, C::LOGE, false, (S0 == LOGN - C::LOGE)>(x, g, gin, sm, Wi, q, ninv, ninv_p, wn, wn_p,
                                                                    tid);
        __syncthreads();
        inv_rest<LOGN, S0 - C::LOGE>(x, g, gin, sm, Wi, q, ninv, ninv_p, wn, wn_p, tid);
    }
}

template <int LOGN>
__global__ void __launch_bounds__(NttCfg<LOGN>::T) ntt_inv_kernel(NttArgs a) {
    using C = NttCfg<LOGN>;
    extern __shared__ u64 sm[];
    const int t = blockIdx.x, poly = blockIdx.y;
    const int pidx = a.limbs.prime[t];
    const PrimeInfo& P = a.pr[pidx];
    const u64 q = P.q;
    const ulonglong2* Wi = a.tw + (size_t)pidx * 2 * C::N + C::N;
    u64* g = a.data + (size_t)poly * a.poly_stride + (size_t)t * C::N;
    const u64* gin = a.src ? a.src + (size_t)poly * a.src_poly_stride + (size_t)t * a.src_limb_stride : g;
    const int tid = threadIdx.x;
    u64 x[C::E];
    u64 ninv = P.pad[0], ninv_p = P.pad[1];
    ulonglong2 wn = Wi[0];   // slot 0 of the inverse table holds {w1 n^-1, shoup}
    if (a.inv_scale) {       // per-limb extra factor folded into the final stage (ModDown)
        const u64* sc = a.inv_scale + 4 * t;
        ninv = sc[0]; ninv_p = sc[1]; wn.x = sc[2]; wn.y = sc[3];
    }
    inv_rest<LOGN, LOGN - C::LOGE>(x, g, gin, sm, Wi, q, ninv, ninv_p, wn.x, wn.y, tid);
    inv_pass<LOGN, 0, C::R0, true>(x, g, gin, sm, Wi, q, ninv, ninv_p, wn.x, wn.y, tid);
}

template <int LOGN>
static cudaError_t launch_one(bool inverse, const NttArgs& a, int nlimbs, int npolys, cudaStream_t st) {
    using C = NttCfg<LOGN>;
    const size_t smem = (size_t)C::N * sizeof(u64);
    static unsigned long long smem_cfg = 0;
    unsigned long long smem_bit = 0;
    if (first_on_device(&smem_cfg, &smem_bit)) {
        cudaError_t ae = cudaSuccess;
        BCN_SMEM_ATTR(ae, (ntt_fwd_kernel<LOGN>), (int)smem);
        BCN_SMEM_ATTR(ae, (ntt_inv_kernel<LOGN>), (int)smem);
        if (ae != cudaSuccess) return ae;
        smem_cfg |= smem_bit;
    }
    dim3 grid(nlimbs, npolys);
    if (inverse) ntt_inv_kernel<LOGN><<<grid, C::T, smem, st>>>(a);
    else ntt_fwd_kernel<LOGN><<<grid, C::T, smem, st>>>(a);
    return launched();
}

static int cluster_mode() {
    static int mode = -1;
    if (mode < 0) {
        const char* e = getenv("BCN_NTT_CLUSTER");
        mode = (e && e[0] == '0') ? 0 : 1;
    }
    return mode;
}

static cudaError_t ntt_launch_impl(bool inverse, int logn, const NttArgs& a, int nlimbs, int npolys,
                                   cudaStream_t st) {
    // fused prologue / epilogue / copy forms exist only in the cluster kernels
    const bool fused = a.pro || a.epi || a.copy_src || a.inv_scale;
    if ((logn == 13 || logn == 14) && (cluster_mode() || fused))
        return ntt_cluster_launch(inverse, logn, a, nlimbs, npolys, st);
    switch (logn) {
        case 3: return launch_one<3>(inverse, a, nlimbs, npolys, st);
        case 4: return launch_one<4>(inverse, a, nlimbs, npolys, st);
        case 5: return launch_one<5>(inverse, a, nlimbs, npolys, st);
        case 6: return launch_one<6>(inverse, a, nlimbs, npolys, st);
        case 7: return launch_one<7>(inverse, a, nlimbs, npolys, st);
        case 8: return launch_one<8>(inverse, a, nlimbs, npolys, st);
        case 9: return launch_one<9>(inverse, a, nlimbs, npolys, st);
        case 10: return launch_one<10>(inverse, a, nlimbs, npolys, st);
        case 11: return launch_one<11>(inverse, a, nlimbs, npolys, st);
        case 12: return launch_one<12>(inverse, a, nlimbs, npolys, st);
        case 13: return launch_one<13>(inverse, a, nlimbs, npolys, st);
        case 14: return launch_one<14>(inverse, a, nlimbs, npolys, st);
        default: return cudaErrorInvalidValue;
    }
}

// ---- in-step NTT timing (bcn_ntt_timing): a CUDA event pair around every
// NTT launch on its own stream, so bench.py can report the byte-weighted
// roofline fraction of all NTT launches of a real forward step.  Classes:
// 0 plain forward, 1 plain inverse, 2 fused forward, 3 fused inverse
// (fused = prologue / epilogue / out-of-place forms), 4 the forward NTT of an
// encryption with the combine c0 = v - a s, c1 = a in its epilogue (epilogue 5).  Algorithmic bytes:
// ntt_algorithmic_bytes() below (16 B per coefficient plus the fused
// operands); the 16-B-only count is kept alongside for comparison.
struct NttTimer {
    bool on = false;
    std::vector<cudaEvent_t> ev;     // 2 per record
    std::vector<int> cls;
    std::vector<unsigned long long> bytes;
    size_t used = 0;
};
static NttTimer g_ntt_timer;

// Algorithmic bytes of one launch (distinct inputs read once,
// outputs written once): 16 B per coefficient of every limb-poly transformed,
// plus the operands a fused prologue / epilogue reads -- the rescale lift's
// top limb (once per poly), the combine inputs c / A / B, the ModDown addend
// sigma(c0), the K special limbs converted in prologue 2, epilogue 4's U
// digits (shared by the two components of a ciphertext).  Key words and
// twiddles are excluded (L2-resident, amortised over the batch).
static unsigned long long ntt_algorithmic_bytes(bool inverse, int logn, const NttArgs& a, int nlimbs, int npolys) {
    const unsigned long long unit = 8ull << logn, nl = (unsigned long long)nlimbs, np = (unsigned long long)npolys;
    unsigned long long b = 2 * unit * nl * np;
    if (inverse) return b;
    if (a.pro == 1) b += unit * np;
    if (a.pro == 2 && a.pro_dnum == 0) b += unit * np * (unsigned long long)a.pro_K;
    if (a.epi == 1) b += unit * nl * np;
    if (a.epi == 2 || a.epi == 3) b += unit * nl * np;
    if (a.epi == 4) b += unit * nl * (np / 2) * (unsigned long long)a.epi_ndig;
    if (a.epi == 5) b += unit * nl * np;                        // the second component written (the key s is L2-resident)
    if ((a.epi == 2 || a.epi == 3 || a.epi == 4) && a.epi_add) b += unit * nl * (a.epi_add_c1 ? np : (np + 1) / 2);
    return b;
}

cudaError_t ntt_launch(bool inverse, int logn, const NttArgs& a, int nlimbs, int npolys, cudaStream_t st) {
    if (nlimbs <= 0 || npolys <= 0) return cudaSuccess;
    NttTimer& T = g_ntt_timer;
    if (!T.on) return ntt_launch_impl(inverse, logn, a, nlimbs, npolys, st);
    if (T.used == T.cls.size()) {
        cudaEvent_t e0, e1;
        cudaError_t e = cudaEventCreate(&e0);
        if (e == cudaSuccess) e = cudaEventCreate(&e1);
        if (e != cudaSuccess) return e;
        T.ev.push_back(e0);
        T.ev.push_back(e1);
        T.cls.push_back(0);
        T.bytes.push_back(0);
    }
    const size_t i = T.used++;
    const bool fused = a.pro || a.epi || a.copy_src || a.inv_scale || a.src;
    T.cls[i] = a.epi == 5 ? 4 : (fused ? 2 : 0) + (inverse ? 1 : 0);
    T.bytes[i] = ntt_algorithmic_bytes(inverse, logn, a, nlimbs, npolys);
    cudaEventRecord(T.ev[2 * i], st);
    cudaError_t e = ntt_launch_impl(inverse, logn, a, nlimbs, npolys, st);
    cudaEventRecord(T.ev[2 * i + 1], st);
    return e;
}

}  // namespace bcn

extern "C" int bcn_ntt_timing(int enable) {
    bcn::g_ntt_timer.on = enable != 0;
    if (enable) bcn::g_ntt_timer.used = 0;
    return 0;
}

extern "C" int bcn_ntt_timing_read(double* ms, uint64_t* bytes, uint64_t* launches) {
    bcn::NttTimer& T = bcn::g_ntt_timer;
    for (int k = 0; k < 5; k++) { ms[k] = 0.0; bytes[k] = 0; launches[k] = 0; }
    for (size_t i = 0; i < T.used; i++) {
        if (cudaEventSynchronize(T.ev[2 * i + 1]) != cudaSuccess) return 4;
        float t = 0.f;
        if (cudaEventElapsedTime(&t, T.ev[2 * i], T.ev[2 * i + 1]) != cudaSuccess) return 4;
        ms[T.cls[i]] += t;
        bytes[T.cls[i]] += T.bytes[i];
        launches[T.cls[i]] += 1;
    }
    return 0;
}
