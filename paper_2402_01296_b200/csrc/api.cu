// api.cu -- the C ABI of libbcn.so (include/bcn.h): context, tables, keys,
// scratch arena and the composition of kernels into HE operations.  This is
// the native runtime behind paper_2402_01296_b200/sim.py; it never touches
// host data on the hot path and never falls back to the CPU.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../../include/bcn.h"
#include "common.cuh"
#include "ops.cuh"


using namespace bcn;
typedef unsigned __int128 u128;

std::atomic<unsigned long long> bcn::g_launches{0};

static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}
#define CUDA_TRY(x)                                                                           \
    do {                                                                                      \
        cudaError_t _e = (x);                                                                 \
        if (_e != cudaSuccess) return fail(BCN_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(_e)); \
    } while (0)

// ------------------------------------------------------------ host math
static u64 mulmod_h(u64 a, u64 b, u64 q) { return (u64)((u128)a * b % q); }
static u64 powmod_h(u64 a, u64 e, u64 q) {
    u64 r = 1 % q;
    a %= q;
    while (e) {
        if (e & 1) r = mulmod_h(r, a, q);
        a = mulmod_h(a, a, q);
        e >>= 1;
    }
    return r;
}
static u64 inv_h(u64 a, u64 q) { return powmod_h(a, q - 2, q); }
static u64 shoup_h(u64 w, u64 q) { return (u64)(((u128)w << 64) / q); }
static u64 mont_h(u64 a, u64 q) { return (u64)(((u128)(a % q) << 64) % q); }

static u64 primitive_root_2n(u64 q, u64 N) {
    u64 e = (q - 1) / (2 * N);
    for (u64 x = 2;; x++) {
        u64 g = powmod_h(x, e, q);
        if (powmod_h(g, N, q) == q - 1) return g;
    }
}

static u32 brev_h(u32 x, int bits) {
    u32 r = 0;
    for (int i = 0; i < bits; i++) { r = (r << 1) | (x & 1); x >>= 1; }
    return r;
}

// ------------------------------------------------------------- context
struct LevelTables {
    ConvTable* modup = nullptr;     // [ndig]
    ConvTable* moddown = nullptr;   // [1]
    u64* pinv = nullptr;            // [2 * (level+1)] Shoup pairs of P^-1 mod q_i
    u64* qlinv = nullptr;           // [2 * level] Shoup pairs of q_level^-1 mod q_i
    u64* qtopmod = nullptr;         // [level] q_level mod q_i (fused rescale lift)
    u64* lift1 = nullptr;           // [2 (level+1)] {0, floor(2^64 / q_i)}: plain lift prologue (K = 1 ModDown)
    u64* upscale = nullptr;         // [4 (level+1)] ModUp INTT constants {n^-1 h_i, sh, w1 n^-1 h_i, sh}
    // merged ModDown + rescale (P' = q_level * P, sources {q_level, p_0..p_{K-1}}, targets q_0..q_{level-1})
    ConvTable* mdr = nullptr;       // [1]
    FConvSet fc_up;                 // FP64 conversion constants (kernel parameters), see ops.cuh
    FConv fc_down, fc_mdr;
    u64* mdr_scale = nullptr;       // [4 (K+1)] INTT constants with (P'/s)^-1 folded in
    u64* pqinv = nullptr;           // [2 level] Shoup pairs of (P q_level)^-1 mod q_i
    int ndig = 0;
};

struct bcn_ctx {
    int device = 0;
    int logn = 0, N = 0, L = 0, nq = 0, K = 0, dnum = 0, alpha = 0, nbasis = 0;
    u64 seed = 0;
    std::vector<u64> primes;
    std::vector<PrimeInfo> hpr;
    std::vector<u64> wn_host;     // per prime: w1 n^-1 (inverse-table entry 0), for folded INTT scales
    std::vector<u64> pmod_host;   // [2 nq] Shoup pairs of P mod q_i
    PrimeInfo* pr = nullptr;
    ulonglong2* tw = nullptr;
    ulonglong2* twt = nullptr;    // tw in the cluster NTT's pass-transposed layout
    double2* twf = nullptr;       // FP64 twiddles {w, w/q} (pass-transposed layout)
    double2* fq = nullptr;        // per prime {q, 1/q} (FP64 base conversions)
    bool fp_conv = false;         // every basis prime in (2^49, 2^50): base conversions on the FP64 pipe
    bool fp_ntt = true;           // BCN_NTT_FP64=0: integer butterflies for every prime
    double* ksi_re = nullptr;
    double* ksi_im = nullptr;
    int* rot = nullptr;
    u64* s_ntt = nullptr;    // canonical
    u64* s_mont = nullptr;   // Montgomery
    u64* pmod = nullptr;     // Shoup pairs of P mod q_i (i < nq)
    std::map<int, LevelTables> lt;
    std::map<u64, u64*> keys;
    u64* scratch = nullptr;
    size_t scratch_bytes = 0;
    u64* scratch2 = nullptr;
    size_t scratch2_bytes = 0;
    void* ptr_dev = nullptr;  // device copy of a host pointer table (plane packing)
    size_t ptr_cap = 0;
    int frozen = 0;           // > 0 while a captured CUDA graph holds pointers into the arenas (bcn_ctx_freeze)
    size_t table_bytes = 0, key_bytes = 0;
    u64 q0inv_q1 = 0, q0inv_q1_p = 0;
    u64* md_scale = nullptr;  // [4K] {n^-1 h_k, shoup, w1 n^-1 h_k, shoup}: ModDown INTT outputs y_k directly

    size_t key_words() const { return (size_t)dnum * 2 * nbasis * N; }
};

static cudaError_t dmalloc(void** p, size_t bytes, size_t* acc) {
    cudaError_t e = cudaMalloc(p, bytes);
    if (e == cudaSuccess && acc) *acc += bytes;
    return e;
}

static const char* kFrozen = "context arenas are frozen by a captured CUDA graph (bcn_ctx_freeze): "
                             "this call needs a larger arena; use another context";

static u64* scratch_get(bcn_ctx* c, size_t words, int* err) {
    size_t bytes = words * sizeof(u64);
    if (bytes > c->scratch_bytes) {
        if (c->frozen) { *err = fail(BCN_ERR_USAGE, kFrozen); return nullptr; }
        if (c->scratch) cudaFree(c->scratch);   // synchronising: in-flight users are done
        c->scratch = nullptr;
        size_t nb = bytes + bytes / 4;
        if (cudaMalloc(&c->scratch, nb) != cudaSuccess) {
            c->scratch_bytes = 0;
            *err = fail(BCN_ERR_CUDA, "scratch allocation of " + std::to_string(nb) + " bytes failed");
            return nullptr;
        }
        c->scratch_bytes = nb;
    }
    return c->scratch;
}

// second arena for operands that live alongside scratch (slot-major MAC staging)
static u64* scratch2_get(bcn_ctx* c, size_t words, int* err) {
    size_t bytes = words * sizeof(u64);
    if (bytes > c->scratch2_bytes) {
        if (c->frozen) { *err = fail(BCN_ERR_USAGE, kFrozen); return nullptr; }
        if (c->scratch2) cudaFree(c->scratch2);
        c->scratch2 = nullptr;
        if (cudaMalloc(&c->scratch2, bytes) != cudaSuccess) {
            c->scratch2_bytes = 0;
            *err = fail(BCN_ERR_CUDA, "scratch allocation of " + std::to_string(bytes) + " bytes failed");
            return nullptr;
        }
        c->scratch2_bytes = bytes;
    }
    return c->scratch2;
}

static Limbs limbs_range(int prime0, int n) {
    Limbs l;
    l.n = n;
    for (int i = 0; i < n && i < BCN_MAX_LIMBS; i++) l.prime[i] = (short)(prime0 + i);
    return l;
}

// extended basis at level l: q_0..q_l, p_0..p_{K-1}
static Limbs limbs_ext(const bcn_ctx* c, int level) {
    Limbs l;
    l.n = level + 1 + c->K;
    for (int t = 0; t <= level; t++) l.prime[t] = (short)t;
    for (int k = 0; k < c->K; k++) l.prime[level + 1 + k] = (short)(c->nq + k);
    return l;
}

static int ndig_at(const bcn_ctx* c, int level) { return (level + c->alpha) / c->alpha; }

static NttArgs ntt_args(const bcn_ctx* c, u64* data, long long poly_stride, const Limbs& l) {
    NttArgs a;
    a.data = data;
    a.poly_stride = poly_stride;
    a.digit_stride = 0;
    a.limbs = l;
    a.tw = c->tw;
    a.twt = c->twt;
    a.twf = c->fp_ntt ? c->twf : nullptr;
    a.fp_all = 1;
    for (int i = 0; i < l.n; i++) a.fp_all &= c->primes[l.prime[i]] < (1ull << 50) ? 1 : 0;
    a.pr = c->pr;
    a.skip_alpha = 0;
    a.skip_dnum = 1;
    a.skip_level = 0;
    a.grid_pm = 0;
    a.src = nullptr;
    a.src_poly_stride = 0;
    a.src_limb_stride = 0;
    a.pro = 0;
    a.pro_src = nullptr;
    a.pro_stride = 0;
    a.pro_qtop = 0;
    a.pro_tab = nullptr;
    a.epi = 0;
    a.epi_c = nullptr;
    a.epi_cps = a.epi_cls = 0;
    a.epi_tab = nullptr;
    a.pro_conv = nullptr;
    a.pro_K = 0;
    a.epi_add = nullptr;
    a.epi_aps = 0;
    a.epi_add_c1 = 0;
    a.epi_g = 1;
    a.inv_scale = nullptr;
    a.pro_dnum = 0;
    a.pro_dstride = 0;
    a.copy_src = nullptr;
    a.copy_stride = 0;
    a.epi_tab2 = nullptr;
    a.epi_acs = 0;
    a.enc_s = nullptr;
    a.enc_seed = a.enc_id = 0;
    a.enc_id_dev = nullptr;
    a.enc_c1_off = 0;
    return a;
}

static bool getenv_flag_on(const char* name) {
    const char* v = getenv(name);
    return v && v[0] == '1';
}

static bool getenv_flag_off(const char* name) {
    const char* e = getenv(name);
    return e && e[0] == '0';
}

// out-of-place transform: read limb t of poly p at src + p*src_ps + t*src_ls, write dst (packed)
static cudaError_t ntt_run_src(const bcn_ctx* c, bool inv, u64* dst, long long dst_ps, const u64* src, long long src_ps,
                               long long src_ls, const Limbs& l, int npoly, cudaStream_t st) {
    NttArgs a = ntt_args(c, dst, dst_ps, l);
    a.src = src;
    a.src_poly_stride = src_ps;
    a.src_limb_stride = src_ls;
    return ntt_launch(inv, c->logn, a, l.n, npoly, st);
}

static cudaError_t ntt_run(const bcn_ctx* c, bool inv, u64* data, long long poly_stride, const Limbs& l, int npoly,
                           cudaStream_t st) {
    NttArgs a = ntt_args(c, data, poly_stride, l);
    return ntt_launch(inv, c->logn, a, l.n, npoly, st);
}

static int build_level(bcn_ctx* c, int level, LevelTables** out) {
    auto it = c->lt.find(level);
    if (it != c->lt.end()) { *out = &it->second; return BCN_OK; }
    LevelTables T;
    const int ndig = ndig_at(c, level);
    T.ndig = ndig;
    const Limbs ext = limbs_ext(c, level);
    std::vector<ConvTable> up(ndig);
    for (int j = 0; j < ndig; j++) {
        ConvTable& t = up[j];
        memset(&t, 0, sizeof(t));
        const int i0 = j * c->alpha, i1 = std::min((j + 1) * c->alpha, level + 1);
        t.n_src = i1 - i0;
        for (int i = i0; i < i1; i++) {
            const u64 qi = c->primes[i];
            u64 prod = 1;
            for (int k = i0; k < i1; k++) if (k != i) prod = mulmod_h(prod, c->primes[k] % qi, qi);
            const u64 hinv = inv_h(prod, qi);
            t.hatinv[i - i0] = hinv;
            t.hatinv_p[i - i0] = shoup_h(hinv, qi);
            for (int e = 0; e < ext.n; e++) {
                const u64 qt = c->primes[ext.prime[e]];
                u64 pm = 1;
                for (int k = i0; k < i1; k++) if (k != i) pm = mulmod_h(pm, c->primes[k] % qt, qt);
                t.hat_m[(i - i0) * BCN_MAX_LIMBS + e] = mont_h(pm, qt);
                if (j < 3 && i - i0 < BCN_FC_SRC && e < BCN_FC_TGT) {
                    T.fc_up.d[j].h[i - i0][e] = make_double2((double)pm, (double)pm / (double)qt);
                    T.fc_up.d[j].fq[e] = make_double2((double)qt, 1.0 / (double)qt);
                }
            }
        }
    }
    ConvTable down;
    memset(&down, 0, sizeof(down));
    down.n_src = c->K;
    for (int k = 0; k < c->K; k++) {
        const u64 pk = c->primes[c->nq + k];
        u64 prod = 1;
        for (int k2 = 0; k2 < c->K; k2++) if (k2 != k) prod = mulmod_h(prod, c->primes[c->nq + k2] % pk, pk);
        const u64 hinv = inv_h(prod, pk);
        down.hatinv[k] = hinv;
        down.hatinv_p[k] = shoup_h(hinv, pk);
        for (int i = 0; i <= level; i++) {
            const u64 qi = c->primes[i];
            u64 pm = 1;
            for (int k2 = 0; k2 < c->K; k2++) if (k2 != k) pm = mulmod_h(pm, c->primes[c->nq + k2] % qi, qi);
            down.hat_m[k * BCN_MAX_LIMBS + i] = mont_h(pm, qi);
            if (k < BCN_FC_SRC && i < BCN_FC_TGT) {
                T.fc_down.h[k][i] = make_double2((double)pm, (double)pm / (double)qi);
                T.fc_down.fq[i] = make_double2((double)qi, 1.0 / (double)qi);
            }
        }
    }
    std::vector<u64> pinv(2 * (level + 1)), qlinv(2 * std::max(level, 1));
    for (int i = 0; i <= level; i++) {
        const u64 qi = c->primes[i];
        u64 P = 1;
        for (int k = 0; k < c->K; k++) P = mulmod_h(P, c->primes[c->nq + k] % qi, qi);
        const u64 v = inv_h(P, qi);
        pinv[2 * i] = v;
        pinv[2 * i + 1] = shoup_h(v, qi);
    }
    for (int i = 0; i < level; i++) {
        const u64 qi = c->primes[i];
        const u64 v = inv_h(c->primes[level] % qi, qi);
        qlinv[2 * i] = v;
        qlinv[2 * i + 1] = shoup_h(v, qi);
    }
    CUDA_TRY(dmalloc((void**)&T.modup, sizeof(ConvTable) * ndig, &c->table_bytes));
    CUDA_TRY(dmalloc((void**)&T.moddown, sizeof(ConvTable), &c->table_bytes));
    CUDA_TRY(dmalloc((void**)&T.pinv, sizeof(u64) * pinv.size(), &c->table_bytes));
    CUDA_TRY(dmalloc((void**)&T.qlinv, sizeof(u64) * qlinv.size(), &c->table_bytes));
    std::vector<u64> qtm(2 * std::max(level, 1));
    for (int i = 0; i < level; i++) {
        qtm[2 * i] = c->primes[level] % c->primes[i];
        qtm[2 * i + 1] = (u64)(((u128)1 << 64) / c->primes[i]);   // Shoup companion of 1
    }
    if (level >= 1) {
        // sources s = {q_level, p_0..p_{K-1}} (prime indices), P' = prod s
        const int ns = c->K + 1;
        std::vector<int> sp(ns);
        sp[0] = level;
        for (int k = 0; k < c->K; k++) sp[1 + k] = c->nq + k;
        ConvTable m;
        memset(&m, 0, sizeof(m));
        m.n_src = ns;
        std::vector<u64> msc(4 * ns);
        for (int a = 0; a < ns; a++) {
            const u64 sa = c->primes[sp[a]];
            u64 prod = 1;
            for (int b = 0; b < ns; b++) if (b != a) prod = mulmod_h(prod, c->primes[sp[b]] % sa, sa);
            const u64 hinv = inv_h(prod, sa);
            m.hatinv[a] = hinv;
            m.hatinv_p[a] = shoup_h(hinv, sa);
            for (int i = 0; i < level; i++) {
                const u64 qi = c->primes[i];
                u64 pm = 1;
                for (int b = 0; b < ns; b++) if (b != a) pm = mulmod_h(pm, c->primes[sp[b]] % qi, qi);
                m.hat_m[a * BCN_MAX_LIMBS + i] = mont_h(pm, qi);
                if (a < BCN_FC_SRC && i < BCN_FC_TGT) {
                    T.fc_mdr.h[a][i] = make_double2((double)pm, (double)pm / (double)qi);
                    T.fc_mdr.fq[i] = make_double2((double)qi, 1.0 / (double)qi);
                }
            }
            const u64 x = mulmod_h(c->hpr[sp[a]].pad[0], hinv, sa), y = mulmod_h(c->wn_host[sp[a]], hinv, sa);
            msc[4 * a] = x; msc[4 * a + 1] = shoup_h(x, sa);
            msc[4 * a + 2] = y; msc[4 * a + 3] = shoup_h(y, sa);
        }
        std::vector<u64> pq(2 * level);
        for (int i = 0; i < level; i++) {
            const u64 qi = c->primes[i];
            u64 v = c->primes[level] % qi;
            for (int k = 0; k < c->K; k++) v = mulmod_h(v, c->primes[c->nq + k] % qi, qi);
            const u64 vi = inv_h(v, qi);
            pq[2 * i] = vi;
            pq[2 * i + 1] = shoup_h(vi, qi);
        }
        CUDA_TRY(dmalloc((void**)&T.mdr, sizeof(ConvTable), &c->table_bytes));
        CUDA_TRY(cudaMemcpy(T.mdr, &m, sizeof(ConvTable), cudaMemcpyHostToDevice));
        CUDA_TRY(dmalloc((void**)&T.mdr_scale, sizeof(u64) * msc.size(), &c->table_bytes));
        CUDA_TRY(cudaMemcpy(T.mdr_scale, msc.data(), sizeof(u64) * msc.size(), cudaMemcpyHostToDevice));
        CUDA_TRY(dmalloc((void**)&T.pqinv, sizeof(u64) * pq.size(), &c->table_bytes));
        CUDA_TRY(cudaMemcpy(T.pqinv, pq.data(), sizeof(u64) * pq.size(), cudaMemcpyHostToDevice));
    }
    std::vector<u64> ups(4 * (level + 1));
    for (int j = 0; j < ndig; j++) {
        const int i0 = j * c->alpha;
        for (int i = i0; i < i0 + up[j].n_src; i++) {
            const u64 qi = c->primes[i];
            const u64 h = up[j].hatinv[i - i0];
            const u64 a = mulmod_h(c->hpr[i].pad[0], h, qi), b = mulmod_h(c->wn_host[i], h, qi);
            ups[4 * i] = a; ups[4 * i + 1] = shoup_h(a, qi);
            ups[4 * i + 2] = b; ups[4 * i + 3] = shoup_h(b, qi);
        }
    }
    CUDA_TRY(dmalloc((void**)&T.upscale, sizeof(u64) * ups.size(), &c->table_bytes));
    CUDA_TRY(cudaMemcpy(T.upscale, ups.data(), sizeof(u64) * ups.size(), cudaMemcpyHostToDevice));
    CUDA_TRY(dmalloc((void**)&T.qtopmod, sizeof(u64) * qtm.size(), &c->table_bytes));
    CUDA_TRY(cudaMemcpy(T.qtopmod, qtm.data(), sizeof(u64) * qtm.size(), cudaMemcpyHostToDevice));
    {
        std::vector<u64> l1(2 * (level + 1));
        for (int i = 0; i <= level; i++) {
            l1[2 * i] = 0;
            // 0: one conditional subtraction reduces a residue of the (single) special prime mod q_i
            l1[2 * i + 1] = (c->K == 1 && c->primes[c->nq] < 2 * c->primes[i] && !getenv_flag_off("BCN_LIFT_CSUB"))
                                ? 0ull : (u64)(((u128)1 << 64) / c->primes[i]);
        }
        CUDA_TRY(dmalloc((void**)&T.lift1, sizeof(u64) * l1.size(), &c->table_bytes));
        CUDA_TRY(cudaMemcpy(T.lift1, l1.data(), sizeof(u64) * l1.size(), cudaMemcpyHostToDevice));
    }
    CUDA_TRY(cudaMemcpy(T.modup, up.data(), sizeof(ConvTable) * ndig, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(T.moddown, &down, sizeof(ConvTable), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(T.pinv, pinv.data(), sizeof(u64) * pinv.size(), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(T.qlinv, qlinv.data(), sizeof(u64) * qlinv.size(), cudaMemcpyHostToDevice));
    c->lt[level] = T;
    *out = &c->lt[level];
    return BCN_OK;
}


// rescale by q_level of npoly polys: in (poly stride in_ps, level+1 limbs) -> out
// (poly stride level*N).  N = 2^13 / 2^14: INTT of the top limb + ONE fused
// cluster NTT whose prologue does the centred lift and whose epilogue does
// (c - x) * q_level^-1 (no intermediate in HBM); other N: the staged kernels.
static cudaError_t rescale_tail(const bcn_ctx* c, u64* out, const u64* in, long long in_ps, int npoly, int level,
                                u64* top, u64* W, const LevelTables* T, cudaStream_t st) {
    const long long N = c->N;
    cudaError_t e = ntt_run_src(c, true, top, N, in + (size_t)level * N, in_ps, N, limbs_range(level, 1), npoly, st);
    if (e != cudaSuccess) return e;
    Limbs ql = limbs_range(0, level);
    if ((c->logn == 13 || c->logn == 14) && !getenv_flag_off("BCN_FUSED_RESCALE")) {
        NttArgs a = ntt_args(c, out, (long long)level * N, ql);
        a.pro = 1;
        a.pro_src = top;
        a.pro_stride = N;
        a.pro_qtop = c->primes[level];
        a.pro_tab = T->qtopmod;
        a.epi = 1;
        a.epi_c = in;
        a.epi_cps = in_ps;
        a.epi_cls = N;
        a.epi_tab = T->qlinv;
        return ntt_launch(false, c->logn, a, level, npoly, st);
    }
    e = rescale_lift_op(W, top, npoly, level, c->primes[level], c->logn, ql, c->pr, st);
    if (e != cudaSuccess) return e;
    e = ntt_run(c, false, W, (long long)level * N, ql, npoly, st);
    if (e != cudaSuccess) return e;
    return rescale_combine_op(out, (long long)level * N, in, in_ps, W, npoly, level, c->logn, ql, c->pr, T->qlinv, st);
}

static int check_level(const bcn_ctx* c, int level) {
    if (level < 0 || level > c->L) return fail(BCN_ERR_PARAM, "level " + std::to_string(level) + " outside [0, " + std::to_string(c->L) + "]");
    return BCN_OK;
}

static FftTab fft_tab(const bcn_ctx* c) {
    FftTab f;
    f.re = c->ksi_re;
    f.im = c->ksi_im;
    f.rot = c->rot;
    return f;
}

extern "C" {

const char* bcn_last_error(void) { return g_err.c_str(); }
int bcn_version(void) { return 1; }

int bcn_plain_conv2d(const double* x, const double* w, const double* bias, double* out, int B, int C, int H, int W,
                     int O, int kh, int kw, int sh, int sw, int ph, int pw, void* stream) {
    if (B < 1 || C < 1 || O < 1 || kh < 1 || kw < 1 || sh < 1 || sw < 1 || ph < 0 || pw < 0)
        return fail(BCN_ERR_PARAM, "bad conv2d shape");
    if ((size_t)C * kh * kw * 16 * sizeof(double) > 48 * 1024)
        return fail(BCN_ERR_CAPACITY, "conv2d weights exceed the shared-memory tile (C kh kw <= 384)");
    CUDA_TRY(plain_conv_op(x, w, bias, out, B, C, H, W, O, kh, kw, sh, sw, ph, pw, (cudaStream_t)stream));
    return BCN_OK;
}

int bcn_launch_count(uint64_t* out) {
    *out = g_launches.load(std::memory_order_relaxed);
    return BCN_OK;
}

int bcn_ctx_create(bcn_ctx** out, int logn, int max_level, const uint64_t* q, int n_special, const uint64_t* p,
                   int dnum, uint64_t seed, int device) {
    if (!out) return fail(BCN_ERR_PARAM, "null output pointer");
    if (logn < 3 || logn > 14) return fail(BCN_ERR_PARAM, "logn must be in [3, 14]");
    if (max_level < 0 || n_special < 1 || dnum < 1) return fail(BCN_ERR_PARAM, "bad level / special / dnum");
    const int nq = max_level + 1, nb = nq + n_special;
    if (nb > BCN_MAX_LIMBS) return fail(BCN_ERR_PARAM, "too many primes");
    const int alpha = (nq + dnum - 1) / dnum;
    if (alpha > BCN_MAX_ALPHA || n_special > BCN_MAX_ALPHA) return fail(BCN_ERR_PARAM, "digit too wide");
    const u64 N = 1ull << logn;
    std::unique_ptr<bcn_ctx> c(new bcn_ctx());
    c->device = device;
    CUDA_TRY(cudaSetDevice(device));
    c->logn = logn; c->N = (int)N; c->L = max_level; c->nq = nq; c->K = n_special;
    c->dnum = dnum; c->alpha = alpha; c->nbasis = nb; c->seed = seed;
    for (int i = 0; i < nq; i++) c->primes.push_back(q[i]);
    for (int k = 0; k < n_special; k++) c->primes.push_back(p[k]);
    for (int i = 0; i < nb; i++) {
        const u64 qi = c->primes[i];
        if (qi >= (1ull << 61) || qi % (2 * N) != 1) return fail(BCN_ERR_PARAM, "prime " + std::to_string(qi) + " is not < 2^61 and 1 mod 2N");
        for (int j = 0; j < i; j++) if (c->primes[j] == qi) return fail(BCN_ERR_PARAM, "duplicate prime");
    }
    // prime info + twiddles
    c->hpr.resize(nb);
    std::vector<ulonglong2> tw((size_t)nb * 2 * N);
    std::vector<u64> pw(N), pwi(N);
    for (int i = 0; i < nb; i++) {
        const u64 qi = c->primes[i];
        PrimeInfo& P = c->hpr[i];
        memset(&P, 0, sizeof(P));
        P.q = qi;
        u64 inv = 1;   // Newton: q^-1 mod 2^64
        for (int it = 0; it < 7; it++) inv *= 2 - qi * inv;
        P.qinv_neg = (u64)0 - inv;
        P.r1 = (u64)(((u128)1 << 64) % qi);
        P.r1_shoup = shoup_h(P.r1, qi);
        P.r2 = mulmod_h(P.r1, P.r1, qi);
        const u64 ninv = inv_h(N % qi, qi);
        P.pad[0] = ninv;
        P.pad[1] = shoup_h(ninv, qi);
        P.pad[2] = shoup_h(1, qi);      // floor(2^64 / q): Barrett reduction of a 64-bit word
        const u64 psi = primitive_root_2n(qi, N), psi_inv = inv_h(psi, qi);
        u64 a = 1, b = 1;
        for (u64 k = 0; k < N; k++) { pw[k] = a; pwi[k] = b; a = mulmod_h(a, psi, qi); b = mulmod_h(b, psi_inv, qi); }
        ulonglong2* F = &tw[(size_t)i * 2 * N];
        ulonglong2* I = F + N;
        for (u64 k = 0; k < N; k++) {
            const u64 w = pw[brev_h((u32)k, logn)], wi = pwi[brev_h((u32)k, logn)];
            F[k] = make_ulonglong2(w, shoup_h(w, qi));
            I[k] = make_ulonglong2(wi, shoup_h(wi, qi));
        }
        const u64 wn = mulmod_h(I[1].x, ninv, qi);
        I[0] = make_ulonglong2(wn, shoup_h(wn, qi));
        c->wn_host.push_back(wn);
    }
    CUDA_TRY(dmalloc((void**)&c->pr, sizeof(PrimeInfo) * nb, &c->table_bytes));
    CUDA_TRY(cudaMemcpy(c->pr, c->hpr.data(), sizeof(PrimeInfo) * nb, cudaMemcpyHostToDevice));
    CUDA_TRY(dmalloc((void**)&c->tw, sizeof(ulonglong2) * tw.size(), &c->table_bytes));
    CUDA_TRY(cudaMemcpy(c->tw, tw.data(), sizeof(ulonglong2) * tw.size(), cudaMemcpyHostToDevice));
    {   // FP64 companions: {w, w/q} (correctly rounded division of exact doubles; only primes < 2^50 use them)
        // layout: pass-transposed for the cluster NTT's radix-16 passes (ntt_cluster.cu):
        // entry 2^s + (gi << ls) + j of stage s = S0 + ls lives at 2^s + j 2^S0 + gi
        std::vector<double2> twf(tw.size());
        std::vector<ulonglong2> twt(tw.size());
        const int R0 = (logn % 4) ? (logn % 4) : 4;
        auto pos = [&](u64 k) -> u64 {
            if (k == 0 || (logn != 13 && logn != 14)) return k;
            int s = 63 - __builtin_clzll(k);
            const int S0 = s < R0 ? 0 : R0 + 4 * ((s - R0) / 4), ls = s - S0;
            const u64 r = k - (1ull << s), gi = r >> ls, j = r & ((1ull << ls) - 1);
            return (1ull << s) + (j << S0) + gi;
        };
        for (int i = 0; i < nb; i++) {
            const double qd = (double)c->primes[i];
            for (int half = 0; half < 2; half++)
                for (u64 k = 0; k < (u64)N; k++) {
                    const ulonglong2 e = tw[(size_t)i * 2 * N + (size_t)half * N + k];
                    const double w = e.x > c->primes[i] / 2 ? (double)e.x - qd : (double)e.x;   // signed, |w| <= q/2
                    twf[(size_t)i * 2 * N + (size_t)half * N + pos(k)] = make_double2(w, w / qd);
                    twt[(size_t)i * 2 * N + (size_t)half * N + pos(k)] = e;
                }
        }
        CUDA_TRY(dmalloc((void**)&c->twt, sizeof(ulonglong2) * twt.size(), &c->table_bytes));
        CUDA_TRY(cudaMemcpy(c->twt, twt.data(), sizeof(ulonglong2) * twt.size(), cudaMemcpyHostToDevice));
        CUDA_TRY(dmalloc((void**)&c->twf, sizeof(double2) * twf.size(), &c->table_bytes));
        CUDA_TRY(cudaMemcpy(c->twf, twf.data(), sizeof(double2) * twf.size(), cudaMemcpyHostToDevice));
        c->fp_ntt = !getenv_flag_off("BCN_NTT_FP64");
        std::vector<double2> fq(nb);
        bool band = true;
        for (int i = 0; i < nb; i++) {
            fq[i] = make_double2((double)c->primes[i], 1.0 / (double)c->primes[i]);
            band &= c->primes[i] > (1ull << 49) && c->primes[i] < (1ull << 50);
        }
        CUDA_TRY(dmalloc((void**)&c->fq, sizeof(double2) * nb, &c->table_bytes));
        CUDA_TRY(cudaMemcpy(c->fq, fq.data(), sizeof(double2) * nb, cudaMemcpyHostToDevice));
        c->fp_conv = band && !getenv_flag_off("BCN_CONV_FP64");
    }
    // canonical-embedding tables: ksi[k] = exp(2 pi i k / M) as computed by numpy on the host
    // are uploaded by the Python layer through bcn_ctx_set_fft (see below); rot[j] = 5^j mod M here.
    const u64 M = 2 * N, S = N / 2;
    std::vector<int> rot(S);
    u64 v = 1;
    for (u64 j = 0; j < S; j++) { rot[j] = (int)v; v = v * 5 % M; }
    CUDA_TRY(dmalloc((void**)&c->rot, sizeof(int) * S, &c->table_bytes));
    CUDA_TRY(cudaMemcpy(c->rot, rot.data(), sizeof(int) * S, cudaMemcpyHostToDevice));
    CUDA_TRY(dmalloc((void**)&c->ksi_re, sizeof(double) * (M + 1), &c->table_bytes));
    CUDA_TRY(dmalloc((void**)&c->ksi_im, sizeof(double) * (M + 1), &c->table_bytes));
    // P mod q_i (Shoup pairs)
    std::vector<u64> pmod(2 * nq);
    for (int i = 0; i < nq; i++) {
        const u64 qi = c->primes[i];
        u64 P = 1;
        for (int k = 0; k < n_special; k++) P = mulmod_h(P, c->primes[nq + k] % qi, qi);
        pmod[2 * i] = P;
        pmod[2 * i + 1] = shoup_h(P, qi);
    }
    c->pmod_host = pmod;
    CUDA_TRY(dmalloc((void**)&c->pmod, sizeof(u64) * pmod.size(), &c->table_bytes));
    CUDA_TRY(cudaMemcpy(c->pmod, pmod.data(), sizeof(u64) * pmod.size(), cudaMemcpyHostToDevice));
    {
        std::vector<u64> ms(4 * n_special);
        for (int k = 0; k < n_special; k++) {
            const u64 pk = c->primes[nq + k];
            u64 prod = 1;
            for (int k2 = 0; k2 < n_special; k2++) if (k2 != k) prod = mulmod_h(prod, c->primes[nq + k2] % pk, pk);
            const u64 h = inv_h(prod, pk);                                 // (P/p_k)^-1 mod p_k
            const u64 a = mulmod_h(c->hpr[nq + k].pad[0], h, pk);          // n^-1 h
            const u64 b = mulmod_h(tw[(size_t)(nq + k) * 2 * N + N + 1].x, a, pk);   // w1 n^-1 h
            ms[4 * k] = a; ms[4 * k + 1] = shoup_h(a, pk);
            ms[4 * k + 2] = b; ms[4 * k + 3] = shoup_h(b, pk);
        }
        CUDA_TRY(dmalloc((void**)&c->md_scale, sizeof(u64) * ms.size(), &c->table_bytes));
        CUDA_TRY(cudaMemcpy(c->md_scale, ms.data(), sizeof(u64) * ms.size(), cudaMemcpyHostToDevice));
    }
    if (nq >= 2) {
        c->q0inv_q1 = inv_h(c->primes[0] % c->primes[1], c->primes[1]);
        c->q0inv_q1_p = shoup_h(c->q0inv_q1, c->primes[1]);
    }
    // secret key: ternary (DOM_SECRET = 3, id 0) -> all basis limbs -> NTT
    CUDA_TRY(dmalloc((void**)&c->s_ntt, sizeof(u64) * nb * N, &c->key_bytes));
    CUDA_TRY(dmalloc((void**)&c->s_mont, sizeof(u64) * nb * N, &c->key_bytes));
    Limbs all = limbs_range(0, nb);
    CUDA_TRY(sample_small_op(c->s_ntt, (long long)nb * N, 1, nb, logn, all, c->pr, seed, 3u, 0, 0, 1, 0));
    CUDA_TRY(ntt_run(c.get(), false, c->s_ntt, (long long)nb * N, all, 1, 0));
    CUDA_TRY(to_mont_op(c->s_mont, c->s_ntt, 1, nb, logn, all, c->pr, 0));
    CUDA_TRY(cudaDeviceSynchronize());
    *out = c.release();
    return BCN_OK;
}

// ksi table upload (float64[M+1] each): see paper_2402_01296_b200/params.py
int bcn_ctx_set_fft(bcn_ctx* c, const double* re, const double* im) {
    if (!c) return fail(BCN_ERR_PARAM, "null context");
    const size_t M = 2 * (size_t)c->N;
    CUDA_TRY(cudaMemcpy(c->ksi_re, re, sizeof(double) * (M + 1), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(c->ksi_im, im, sizeof(double) * (M + 1), cudaMemcpyHostToDevice));
    return BCN_OK;
}

int bcn_ctx_destroy(bcn_ctx* c) {
    if (!c) return BCN_OK;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    for (auto& kv : c->lt) {
        cudaFree(kv.second.modup); cudaFree(kv.second.moddown);
        cudaFree(kv.second.pinv); cudaFree(kv.second.qlinv);
        cudaFree(kv.second.qtopmod); cudaFree(kv.second.lift1); cudaFree(kv.second.upscale);
        cudaFree(kv.second.mdr); cudaFree(kv.second.mdr_scale); cudaFree(kv.second.pqinv);
    }
    for (auto& kv : c->keys) cudaFree(kv.second);
    cudaFree(c->pr); cudaFree(c->tw); cudaFree(c->twt); cudaFree(c->twf); cudaFree(c->fq); cudaFree(c->ksi_re); cudaFree(c->ksi_im); cudaFree(c->rot);
    cudaFree(c->s_ntt); cudaFree(c->s_mont); cudaFree(c->pmod); cudaFree(c->md_scale);
    if (c->scratch) cudaFree(c->scratch);
    if (c->ptr_dev) cudaFree(c->ptr_dev);
    if (c->scratch2) cudaFree(c->scratch2);
    delete c;
    return BCN_OK;
}

int bcn_ctx_memory(bcn_ctx* c, uint64_t* bytes) {
    *bytes = c->table_bytes + c->key_bytes + c->scratch_bytes + c->scratch2_bytes;
    return BCN_OK;
}

int bcn_ctx_freeze(bcn_ctx* c, int delta) {
    if (c->frozen + delta < 0) return fail(BCN_ERR_USAGE, "bcn_ctx_freeze: unbalanced release");
    c->frozen += delta;
    return BCN_OK;
}

int bcn_ctx_trim(bcn_ctx* c) {
    if (c->frozen) return fail(BCN_ERR_USAGE, kFrozen);
    if (c->scratch || c->scratch2) cudaDeviceSynchronize();
    if (c->scratch) cudaFree(c->scratch);
    if (c->scratch2) cudaFree(c->scratch2);
    c->scratch = nullptr;
    c->scratch_bytes = 0;
    c->scratch2 = nullptr;
    c->scratch2_bytes = 0;
    return BCN_OK;
}

// ------------------------------------------------------------------ NTT
int bcn_ntt_fwd(bcn_ctx* c, uint64_t* data, int npoly, int nlimb, int prime0, void* stream) {
    if (prime0 < 0 || prime0 + nlimb > c->nbasis) return fail(BCN_ERR_PARAM, "limb range outside basis");
    CUDA_TRY(ntt_run(c, false, (u64*)data, (long long)nlimb * c->N, limbs_range(prime0, nlimb), npoly, (cudaStream_t)stream));
    return BCN_OK;
}

int bcn_ntt_inv(bcn_ctx* c, uint64_t* data, int npoly, int nlimb, int prime0, void* stream) {
    if (prime0 < 0 || prime0 + nlimb > c->nbasis) return fail(BCN_ERR_PARAM, "limb range outside basis");
    CUDA_TRY(ntt_run(c, true, (u64*)data, (long long)nlimb * c->N, limbs_range(prime0, nlimb), npoly, (cudaStream_t)stream));
    return BCN_OK;
}

// --------------------------------------------------------------- encode
int bcn_encode(bcn_ctx* c, const double* vals, int vlen, int vstride, int nplain, double scale, int level,
               int montgomery, uint64_t* out, void* stream) {
    int e = check_level(c, level);
    if (e) return e;
    if (vlen > c->N / 2) return fail(BCN_ERR_CAPACITY, "vector exceeds slot count");
    cudaStream_t st = (cudaStream_t)stream;
    const int nl = level + 1;
    Limbs l = limbs_range(0, nl);
    CUDA_TRY(encode_op((u64*)out, (long long)nl * c->N, vals, vlen, vstride, nplain, scale, c->logn, l, c->pr,
                       fft_tab(c), 0, 0, 0, st));
    CUDA_TRY(ntt_run(c, false, (u64*)out, (long long)nl * c->N, l, nplain, st));
    if (montgomery) CUDA_TRY(to_mont_op((u64*)out, (u64*)out, nplain, nl, c->logn, l, c->pr, st));
    return BCN_OK;
}

// encode over the extended basis q_0..q_level, p_0..p_{K-1} (multipliers of lazy-ModDown sums)
int bcn_encode_ext(bcn_ctx* c, const double* vals, int vlen, int vstride, int nplain, double scale, int level,
                   uint64_t* out, void* stream) {
    int e = check_level(c, level);
    if (e) return e;
    if (vlen > c->N / 2) return fail(BCN_ERR_CAPACITY, "vector exceeds slot count");
    cudaStream_t st = (cudaStream_t)stream;
    Limbs l = limbs_ext(c, level);
    const long long ps = (long long)l.n * c->N;
    CUDA_TRY(encode_op((u64*)out, ps, vals, vlen, vstride, nplain, scale, c->logn, l, c->pr, fft_tab(c), 0, 0, 0, st));
    CUDA_TRY(ntt_run(c, false, (u64*)out, ps, l, nplain, st));
    CUDA_TRY(to_mont_op((u64*)out, (u64*)out, nplain, l.n, c->logn, l, c->pr, st));
    return BCN_OK;
}

static int encrypt_impl(bcn_ctx* c, const double* vals, int vlen, int vstride, int G, int level, double scale,
                        uint64_t counter0, const uint64_t* counter_dev, uint64_t* ct, void* stream) {
    int e = check_level(c, level);
    if (e) return e;
    if (vlen > c->N / 2) return fail(BCN_ERR_CAPACITY, "vector exceeds slot count");
    cudaStream_t st = (cudaStream_t)stream;
    const int nl = level + 1;
    Limbs l = limbs_range(0, nl);
    const long long cs = 2LL * nl * c->N;
    CUDA_TRY(encode_op((u64*)ct, cs, vals, vlen, vstride, G, scale, c->logn, l, c->pr, fft_tab(c), 1, c->seed,
                       counter0, st, (const u64*)counter_dev));
    if ((c->logn == 13 || c->logn == 14) && !getenv_flag_off("BCN_FUSED_ENCRYPT")) {
        // c0 = NTT(m + e) - a s and c1 = a in the NTT's epilogue (epilogue 5): the Philox draws and the
        // IMAD-pipe products run beside the FP64-pipe butterflies of the other resident clusters, and c0
        // is not read and written once more
        NttArgs a = ntt_args(c, (u64*)ct, cs, l);
        a.epi = 5;
        a.enc_s = c->s_mont;
        a.enc_seed = c->seed;
        a.enc_id = counter0;
        a.enc_id_dev = (const u64*)counter_dev;
        a.enc_c1_off = (long long)nl * c->N;
        CUDA_TRY(ntt_launch(false, c->logn, a, l.n, G, st));
        return BCN_OK;
    }
    CUDA_TRY(ntt_run(c, false, (u64*)ct, cs, l, G, st));
    CUDA_TRY(encrypt_combine_op((u64*)ct, G, nl, c->logn, l, c->pr, c->s_mont, c->seed, counter0, st,
                                (const u64*)counter_dev));
    return BCN_OK;
}

// ct: [(n_gal) x G][2][level+1][N]; copy c (Galois element gal[c], 1 = the plaintext itself) of row p is a
// fresh encryption (id counter0 + c G + p) of sigma_gal[c](encode(vals[p])), i.e. of the slots rotated by
// the r with 5^r = gal[c]: one canonical embedding per row instead of one per copy
int bcn_encrypt_rotated(bcn_ctx* c, const double* vals, int vlen, int vstride, int G, int level, double scale,
                        uint64_t counter0, int n_gal, const uint64_t* gal, uint64_t* ct, void* stream) {
    int e = check_level(c, level);
    if (e) return e;
    if (vlen > c->N / 2) return fail(BCN_ERR_CAPACITY, "vector exceeds slot count");
    if (n_gal < 1 || n_gal > 32) return fail(BCN_ERR_PARAM, "1..32 copies per plaintext");
    if (G < 1 || G > 65535) return fail(BCN_ERR_PARAM, "1..65535 plaintexts per call");
    cudaStream_t st = (cudaStream_t)stream;
    const int nl = level + 1;
    Limbs l = limbs_range(0, nl);
    const long long cs = 2LL * nl * c->N;
    u32 ginv[32];
    for (int k = 0; k < n_gal; k++) {
        if ((gal[k] & 1) == 0) return fail(BCN_ERR_PARAM, "Galois elements must be odd");
        u32 g = (u32)gal[k], x = g;
        for (int it = 0; it < 5; it++) x *= 2u - g * x;          // g^-1 mod 2^32
        ginv[k] = x & (u32)(2 * c->N - 1);
    }
    int err = 0;
    i64* raw = (i64*)scratch_get(c, (size_t)G * c->N, &err);
    if (!raw) return err;
    CUDA_TRY(encode_op(nullptr, 0, vals, vlen, vstride, G, scale, c->logn, l, c->pr, fft_tab(c), 0, c->seed, 0, st,
                       nullptr, raw));
    CUDA_TRY(encode_rot_op((u64*)ct, cs, raw, G, c->logn, l, c->pr, n_gal, ginv, c->seed, counter0, st));
    const int rows = n_gal * G;
    if ((c->logn == 13 || c->logn == 14) && !getenv_flag_off("BCN_FUSED_ENCRYPT")) {
        NttArgs a = ntt_args(c, (u64*)ct, cs, l);
        a.epi = 5;
        a.enc_s = c->s_mont;
        a.enc_seed = c->seed;
        a.enc_id = counter0;
        a.enc_c1_off = (long long)nl * c->N;
        CUDA_TRY(ntt_launch(false, c->logn, a, l.n, rows, st));
        return BCN_OK;
    }
    CUDA_TRY(ntt_run(c, false, (u64*)ct, cs, l, rows, st));
    CUDA_TRY(encrypt_combine_op((u64*)ct, rows, nl, c->logn, l, c->pr, c->s_mont, c->seed, counter0, st, nullptr));
    return BCN_OK;
}

int bcn_encrypt(bcn_ctx* c, const double* vals, int vlen, int vstride, int G, int level, double scale,
                uint64_t counter0, uint64_t* ct, void* stream) {
    return encrypt_impl(c, vals, vlen, vstride, G, level, scale, counter0, nullptr, ct, stream);
}

int bcn_encrypt_devctr(bcn_ctx* c, const double* vals, int vlen, int vstride, int G, int level, double scale,
                       const uint64_t* counter_dev, uint64_t* ct, void* stream) {
    return encrypt_impl(c, vals, vlen, vstride, G, level, scale, 0, counter_dev, ct, stream);
}

static int decrypt_poly_impl(bcn_ctx* c, const uint64_t* ct, int ct_nlimb, int G, int level, u64* out,
                             cudaStream_t st) {
    const int k = level >= 1 ? 2 : 1;
    CUDA_TRY(decrypt_core_op(out, (const u64*)ct, 2LL * ct_nlimb * c->N, ct_nlimb, k, G, c->logn, c->pr, c->s_mont,
                             0, st));
    CUDA_TRY(ntt_run(c, true, out, (long long)k * c->N, limbs_range(0, k), G, st));
    return BCN_OK;
}

int bcn_decrypt_poly(bcn_ctx* c, const uint64_t* ct, int ct_nlimb, int G, int level, uint64_t* out, void* stream) {
    int e = check_level(c, level);
    if (e) return e;
    return decrypt_poly_impl(c, ct, ct_nlimb, G, level, (u64*)out, (cudaStream_t)stream);
}

int bcn_decrypt(bcn_ctx* c, const uint64_t* ct, int ct_nlimb, int G, int level, double scale, double* out, int nout,
                void* stream) {
    int e = check_level(c, level);
    if (e) return e;
    if (nout > c->N / 2) return fail(BCN_ERR_PARAM, "nout exceeds slot count");
    cudaStream_t st = (cudaStream_t)stream;
    const int k = level >= 1 ? 2 : 1;
    int err = 0;
    u64* tmp = scratch_get(c, (size_t)G * k * c->N, &err);
    if (!tmp) return err;
    e = decrypt_poly_impl(c, ct, ct_nlimb, G, level, tmp, st);
    if (e) return e;
    CUDA_TRY(decode_op(out, nout, tmp, (long long)k * c->N, k, G, scale, c->logn, c->pr, fft_tab(c), c->q0inv_q1,
                       c->q0inv_q1_p, st));
    return BCN_OK;
}

// ------------------------------------------------------------ add / sub
int bcn_add(bcn_ctx* c, uint64_t* out, const uint64_t* a, int a_nlimb, const uint64_t* b, int b_nlimb,
            int b_is_plain, int b_batch, int G, int level, void* stream) {
    int e = check_level(c, level);
    if (e) return e;
    if (a_nlimb < level + 1 || b_nlimb < level + 1) return fail(BCN_ERR_PARAM, "operand has too few limbs");
    cudaStream_t st = (cudaStream_t)stream;
    const int nl = level + 1;
    const long long N = c->N;
    Limbs l = limbs_range(0, nl);
    if (!b_is_plain) {
        CUDA_TRY(binary_op(0, (u64*)out, nl * N, (const u64*)a, a_nlimb * N, (const u64*)b, b_nlimb * N, 2 * G, nl,
                           c->logn, l, c->pr, st));
    } else {
        const long long bs = (b_batch == 1) ? 0 : (long long)b_nlimb * N;
        CUDA_TRY(binary_op(0, (u64*)out, 2 * nl * N, (const u64*)a, 2 * a_nlimb * N, (const u64*)b, bs, G, nl,
                           c->logn, l, c->pr, st));
        if ((const u64*)out != (const u64*)a || a_nlimb != nl)
            CUDA_TRY(copy_limbs_op((u64*)out + nl * N, 2 * nl * N, (const u64*)a + a_nlimb * N, 2 * a_nlimb * N, G,
                                   nl * N, st));
    }
    return BCN_OK;
}

int bcn_sub(bcn_ctx* c, uint64_t* out, const uint64_t* a, int a_nlimb, const uint64_t* b, int b_nlimb, int G,
            int level, void* stream) {
    int e = check_level(c, level);
    if (e) return e;
    const int nl = level + 1;
    const long long N = c->N;
    CUDA_TRY(binary_op(1, (u64*)out, nl * N, (const u64*)a, a_nlimb * N, (const u64*)b, b_nlimb * N, 2 * G, nl,
                       c->logn, limbs_range(0, nl), c->pr, (cudaStream_t)stream));
    return BCN_OK;
}

// -------------------------------------------------------------- rescale
static int rescale_impl(bcn_ctx* c, u64* out, const u64* in, int in_nlimb, int G, int level, cudaStream_t st) {
    if (level < 1) return fail(BCN_ERR_DEPTH, "multiplicative depth exhausted: level is 0");
    LevelTables* T;
    int e = build_level(c, level, &T);
    if (e) return e;
    const long long N = c->N;
    const int npoly = 2 * G;
    int err = 0;
    u64* top = scratch_get(c, (size_t)npoly * N * (1 + level), &err);
    if (!top) return err;
    u64* W = top + (size_t)npoly * N;
    CUDA_TRY(rescale_tail(c, out, in, (long long)in_nlimb * N, npoly, level, top, W, T, st));
    return BCN_OK;
}

int bcn_rescale(bcn_ctx* c, uint64_t* out, const uint64_t* in, int in_nlimb, int G, int level, void* stream) {
    int e = check_level(c, level);
    if (e) return e;
    return rescale_impl(c, (u64*)out, (const u64*)in, in_nlimb, G, level, (cudaStream_t)stream);
}

// ----------------------------------------------------------- mul plain
static int mul_plain_impl(bcn_ctx* c, u64* out, const u64* ct, int ct_nlimb, const u64* pt, int pt_batch, int G,
                          int level, bool rescale, cudaStream_t st) {
    int e = check_level(c, level);
    if (e) return e;
    if (rescale && level < 1) return fail(BCN_ERR_DEPTH, "multiplicative depth exhausted: level is 0");
    const int nl = level + 1;
    const long long N = c->N;
    Limbs l = limbs_range(0, nl);
    const long long ps = (pt_batch == 1) ? 0 : nl * N;
    // product on c0 and c1: treat as 2 polys per ct sharing the ct's plaintext
    u64* prod = out;
    int err = 0;
    if (rescale) {
        prod = scratch_get(c, (size_t)G * 2 * nl * N + (size_t)2 * G * N * (1 + level), &err);
        if (!prod) return err;
    }
    for (int comp = 0; comp < 2; comp++)
        CUDA_TRY(binary_op(2, prod + comp * nl * N, 2 * nl * N, ct + comp * (long long)ct_nlimb * N,
                           2LL * ct_nlimb * N, pt, ps, G, nl, c->logn, l, c->pr, st));
    if (!rescale) return BCN_OK;
    // rescale needs its own scratch: place the product after it by re-running with an offset arena
    LevelTables* T;
    e = build_level(c, level, &T);
    if (e) return e;
    const int npoly = 2 * G;
    u64* top = prod + (size_t)G * 2 * nl * N;
    u64* W = top + (size_t)npoly * N;
    CUDA_TRY(rescale_tail(c, out, prod, nl * N, npoly, level, top, W, T, st));
    return BCN_OK;
}

int bcn_mul_plain(bcn_ctx* c, uint64_t* out, const uint64_t* ct, int ct_nlimb, const uint64_t* pt_mont,
                  int pt_batch, int G, int level, void* stream) {
    return mul_plain_impl(c, (u64*)out, (const u64*)ct, ct_nlimb, (const u64*)pt_mont, pt_batch, G, level, true,
                          (cudaStream_t)stream);
}

int bcn_mul_plain_norescale(bcn_ctx* c, uint64_t* out, const uint64_t* ct, int ct_nlimb, const uint64_t* pt_mont,
                            int pt_batch, int G, int level, void* stream) {
    return mul_plain_impl(c, (u64*)out, (const u64*)ct, ct_nlimb, (const u64*)pt_mont, pt_batch, G, level, false,
                          (cudaStream_t)stream);
}

static int mac_terms_impl(bcn_ctx* c, uint64_t* out, int n_terms, const uint64_t* const* cts,
                          const uint64_t* const* pts, const int* pt_batched, int G, int level, int rescale,
                          int accumulate, void* stream);

int bcn_mac_terms(bcn_ctx* c, uint64_t* out, int n_terms, const uint64_t* const* cts, const uint64_t* const* pts,
                  const int* pt_batched, int G, int level, int rescale, void* stream) {
    return mac_terms_impl(c, out, n_terms, cts, pts, pt_batched, G, level, rescale, 0, stream);
}

int bcn_mac_multi(bcn_ctx* c, uint64_t* out, int n_out, int n_terms, const uint64_t* const* cts,
                  const uint64_t* const* pts, int G, int level, int rescale, void* stream) {
    int e = check_level(c, level);
    if (e) return e;
    if (n_out < 1 || n_terms < 1) return fail(BCN_ERR_PARAM, "no outputs / terms");
    if (rescale && level < 1) return fail(BCN_ERR_DEPTH, "multiplicative depth exhausted: level is 0");
    cudaStream_t st = (cudaStream_t)stream;
    const int nl = level + 1;
    const long long N = c->N;
    const long long cw = (long long)G * 2 * nl * N;   // one output batch
    Limbs l = limbs_range(0, nl);
    u64* acc = (u64*)out;
    int err = 0;
    if (rescale) {
        acc = scratch_get(c, (size_t)n_out * cw + (size_t)2 * n_out * G * N * (1 + level), &err);
        if (!acc) return err;
    }
    MacMulti M;
    for (int o0 = 0; o0 < n_out; o0 += BCN_MAC_OUT) {
        M.n_out = std::min(BCN_MAC_OUT, n_out - o0);
        for (int k0 = 0; k0 < n_terms; k0 += BCN_MULTI_TERMS) {
            M.n_terms = std::min(BCN_MULTI_TERMS, n_terms - k0);
            for (int k = 0; k < M.n_terms; k++) {
                M.ct[k] = (const u64*)cts[k0 + k];
                for (int o = 0; o < M.n_out; o++) M.pt[o][k] = (const u64*)pts[(size_t)(o0 + o) * n_terms + k0 + k];
            }
            CUDA_TRY(mac_multi_op(acc + o0 * cw, cw, M, G, nl, c->logn, l, c->pr, k0 > 0, st));
        }
    }
    if (!rescale) return BCN_OK;
    LevelTables* LT;
    e = build_level(c, level, &LT);
    if (e) return e;
    const int npoly = 2 * n_out * G;
    u64* top = acc + (size_t)n_out * cw;
    u64* W = top + (size_t)npoly * N;
    CUDA_TRY(rescale_tail(c, (u64*)out, acc, nl * N, npoly, level, top, W, LT, st));
    return BCN_OK;
}

// ---- tensor-core multi-output MAC (mac_imma.cu) ----
static int imma_gblock() {
    const char* v = getenv("BCN_IMMA_GB");
    const int g = v ? atoi(v) : 16;
    return g >= 1 && g <= 32 ? g : 16;
}

static int planes_geometry(int n_out, int n_terms, int* opad, int* nch) {
    if (n_out < 1 || n_terms < 1) return fail(BCN_ERR_PARAM, "no outputs / terms");
    if (n_terms > BCN_IMMA_TERMS) return fail(BCN_ERR_PARAM, "more than 256 terms per plane pack");
    *opad = n_out <= 16 ? 16 : (n_out + 31) / 32 * 32;
    *nch = (n_terms + 31) / 32;
    return BCN_OK;
}

int bcn_planes_bytes(bcn_ctx* c, int n_out, int n_terms, int level, uint64_t* bytes) {
    int e = check_level(c, level);
    if (e) return e;
    int opad, nch;
    e = planes_geometry(n_out, n_terms, &opad, &nch);
    if (e) return e;
    *bytes = (uint64_t)(level + 1) * c->N * nch * 8 * opad * 32;
    return BCN_OK;
}

int bcn_pack_planes(bcn_ctx* c, uint8_t* planes, int n_out, int n_terms, const uint64_t* const* pts, int level,
                    void* stream) {
    return bcn_pack_planes_layout(c, planes, n_out, n_terms, pts, level, BCN_PLANES_IMMA, stream);
}

int bcn_pack_planes_layout(bcn_ctx* c, uint8_t* planes, int n_out, int n_terms, const uint64_t* const* pts,
                           int level, int layout, void* stream) {
    if (layout != BCN_PLANES_IMMA && layout != BCN_PLANES_TCGEN05) return fail(BCN_ERR_PARAM, "unknown planes layout");
    int e = check_level(c, level);
    if (e) return e;
    int opad, nch;
    e = planes_geometry(n_out, n_terms, &opad, &nch);
    if (e) return e;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t np = (size_t)n_out * n_terms;
    if (np > c->ptr_cap) {
        if (c->frozen) return fail(BCN_ERR_USAGE, kFrozen);
        if (c->ptr_dev) cudaFree(c->ptr_dev);
        c->ptr_dev = nullptr;
        c->ptr_cap = 0;
        if (cudaMalloc(&c->ptr_dev, np * sizeof(u64*)) != cudaSuccess) return fail(BCN_ERR_CUDA, "pointer table");
        c->ptr_cap = np;
    }
    CUDA_TRY(cudaMemcpyAsync(c->ptr_dev, pts, np * sizeof(u64*), cudaMemcpyHostToDevice, st));
    if (layout == BCN_PLANES_TCGEN05)
        CUDA_TRY(pack_planes_umma_op(planes, (const u64* const*)c->ptr_dev, n_out, n_terms, opad, nch, level + 1,
                                     c->logn, st));
    else
        CUDA_TRY(pack_planes_op(planes, (const u64* const*)c->ptr_dev, n_out, n_terms, opad, nch, level + 1,
                                c->logn, st));
    CUDA_TRY(cudaStreamSynchronize(st));          // the host pointer table may go away after return
    return BCN_OK;
}

// extended-basis planes (conv with lazy ModDown): term k's plaintexts have
// term_limbs[k] limbs (level+1+K for rotation terms, level+1 for identity
// terms, whose special limbs multiply zeros); packed over level+1+K limbs
int bcn_planes_ext_bytes(bcn_ctx* c, int n_out, int n_terms, int level, uint64_t* bytes) {
    int e = check_level(c, level);
    if (e) return e;
    int opad, nch;
    e = planes_geometry(n_out, n_terms, &opad, &nch);
    if (e) return e;
    *bytes = (uint64_t)(level + 1 + c->K) * c->N * nch * 8 * opad * 32;
    return BCN_OK;
}

int bcn_pack_planes_ext(bcn_ctx* c, uint8_t* planes, int n_out, int n_terms, const uint64_t* const* pts,
                        const int* term_limbs, int level, int layout, void* stream) {
    if (layout != BCN_PLANES_IMMA && layout != BCN_PLANES_TCGEN05) return fail(BCN_ERR_PARAM, "unknown plane layout");
    int e = check_level(c, level);
    if (e) return e;
    int opad, nch;
    e = planes_geometry(n_out, n_terms, &opad, &nch);
    if (e) return e;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t np = (size_t)n_out * n_terms;
    const size_t bytes = np * sizeof(u64*) + (size_t)n_terms * sizeof(int);
    if (bytes > c->ptr_cap * sizeof(u64*)) {
        if (c->frozen) return fail(BCN_ERR_USAGE, kFrozen);
        if (c->ptr_dev) cudaFree(c->ptr_dev);
        c->ptr_dev = nullptr;
        c->ptr_cap = 0;
        if (cudaMalloc(&c->ptr_dev, bytes) != cudaSuccess) return fail(BCN_ERR_CUDA, "pointer table");
        c->ptr_cap = (bytes + sizeof(u64*) - 1) / sizeof(u64*);
    }
    std::vector<unsigned char> host(bytes);
    memcpy(host.data(), pts, np * sizeof(u64*));
    memcpy(host.data() + np * sizeof(u64*), term_limbs, (size_t)n_terms * sizeof(int));
    CUDA_TRY(cudaMemcpyAsync(c->ptr_dev, host.data(), bytes, cudaMemcpyHostToDevice, st));
    const int* tl = (const int*)((const unsigned char*)c->ptr_dev + np * sizeof(u64*));
    if (layout == BCN_PLANES_TCGEN05)
        CUDA_TRY(pack_planes_umma_op(planes, (const u64* const*)c->ptr_dev, n_out, n_terms, opad, nch,
                                     level + 1 + c->K, c->logn, st, tl));
    else
        CUDA_TRY(pack_planes_op(planes, (const u64* const*)c->ptr_dev, n_out, n_terms, opad, nch, level + 1 + c->K,
                                c->logn, st, tl));
    CUDA_TRY(cudaStreamSynchronize(st));
    return BCN_OK;
}

static int mdr_tail(bcn_ctx* c, u64* out, u64* B, const u64* C, int add_c1, int G, int level, const LevelTables* T,
                    u64* Z, cudaStream_t st, long long c_gstride = 0);
static u64* key_ptr(bcn_ctx* c, u64 id);

// ---- in-step timing of the conv operand path (bcn_conv_timing): a CUDA event
// pair around every staging launch (class 0: slot_major_ks3 / slot_major_ks /
// slot_major) and every tensor-core MAC launch (class 1: mac_umma / mac_imma),
// with the launch's algorithmic bytes, so bench.py can put both on the HBM roof.
struct ConvTimer {
    bool on = false;
    std::vector<cudaEvent_t> ev;
    std::vector<int> cls;
    std::vector<unsigned long long> bytes;
    size_t used = 0;
    int begin(int cls_, unsigned long long b, cudaStream_t st) {
        if (!on) return -1;
        if (used == cls.size()) {
            cudaEvent_t e0, e1;
            if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) return -1;
            ev.push_back(e0);
            ev.push_back(e1);
            cls.push_back(0);
            bytes.push_back(0);
        }
        const size_t i = used++;
        cls[i] = cls_;
        bytes[i] = b;
        cudaEventRecord(ev[2 * i], st);
        return (int)i;
    }
    void end(int i, cudaStream_t st) {
        if (i >= 0) cudaEventRecord(ev[2 * (size_t)i + 1], st);
    }
};
static ConvTimer g_conv_timer;

int bcn_conv_timing(int enable) {
    g_conv_timer.on = enable != 0;
    if (enable) g_conv_timer.used = 0;
    return BCN_OK;
}

int bcn_conv_timing_read(double* ms, uint64_t* bytes, uint64_t* launches) {
    ConvTimer& T = g_conv_timer;
    for (int k = 0; k < 2; k++) { ms[k] = 0.0; bytes[k] = 0; launches[k] = 0; }
    for (size_t i = 0; i < T.used; i++) {
        if (cudaEventSynchronize(T.ev[2 * i + 1]) != cudaSuccess) return fail(BCN_ERR_CUDA, "conv timing event");
        float t = 0.f;
        if (cudaEventElapsedTime(&t, T.ev[2 * i], T.ev[2 * i + 1]) != cudaSuccess)
            return fail(BCN_ERR_CUDA, "conv timing event");
        ms[T.cls[i]] += t;
        bytes[T.cls[i]] += T.bytes[i];
        launches[T.cls[i]] += 1;
    }
    return BCN_OK;
}

int bcn_conv_ks_mac(bcn_ctx* c, uint64_t* out, int n_out, int n_terms, const uint64_t* const* srcs,
                    const uint64_t* const* Us, const uint64_t* gal, const uint8_t* planes, int layout, int G,
                    int level, void* stream) {
    if (layout != BCN_PLANES_IMMA && layout != BCN_PLANES_TCGEN05) return fail(BCN_ERR_PARAM, "unknown plane layout");
    int e = check_level(c, level);
    if (e) return e;
    int opad, nch;
    e = planes_geometry(n_out, n_terms, &opad, &nch);
    if (e) return e;
    if (level < 1) return fail(BCN_ERR_DEPTH, "multiplicative depth exhausted: level is 0");
    cudaStream_t st = (cudaStream_t)stream;
    for (int k = 0; k < n_terms; k++) {
        if (gal[k] == 1) continue;
        if ((gal[k] & 1) == 0) return fail(BCN_ERR_PARAM, "Galois elements must be odd");
        if (!key_ptr(c, gal[k])) {
            e = bcn_keygen_galois(c, gal[k], stream);
            if (e) return e;
        }
    }
    LevelTables* T;
    e = build_level(c, level, &T);
    if (e) return e;
    const long long N = c->N;
    const int nl = level + 1, next = nl + c->K;
    Limbs ext = limbs_ext(c, level);
    KsTerms KT;
    KT.n = n_terms;
    MacImma M;
    M.n_terms = n_terms;
    M.n_out = n_out;
    for (int k = 0; k < n_terms; k++) {
        KT.src[k] = (const u64*)srcs[k];
        KT.U[k] = (const u64*)Us[k];
        KT.key[k] = gal[k] == 1 ? nullptr : key_ptr(c, gal[k]);
        KT.g[k] = (u32)gal[k];
        M.ct[k] = nullptr;
    }
    const long long cw = (long long)G * 2 * next * N;    // one output's extended-basis sum
    const bool fused = (c->logn == 13 || c->logn == 14) && !getenv_flag_off("BCN_FUSED_MODDOWN");
    int err = 0;
    (void)fused;
    u64* acc = scratch_get(c, (size_t)n_out * cw + (size_t)n_out * G * 2 * level * N, &err);
    if (!acc) return err;
    u64* Z = acc + (size_t)n_out * cw;
    // tcgen05: blocks of 64 slot sets (M = 128 columns); IMMA: blocks of IMMA_GB slot
    // sets (16 -> 8-warp CTAs, two resident per SM, so one CTA's pipeline fill
    // overlaps the other's MMAs)
    const bool tc05 = layout == BCN_PLANES_TCGEN05;
    const int spitch = tc05 ? 128 : 64;
    const size_t per_limb = (size_t)N * n_terms * spitch * sizeof(u64);
    static const size_t stage_bytes = (size_t)(getenv("BCN_STAGE_GB") ? atof(getenv("BCN_STAGE_GB")) : 4.0) * (1ull << 30);
    const int tcnt = (int)std::max<size_t>(1, std::min<size_t>(next, stage_bytes / per_limb));
    u64* S = scratch2_get(c, (size_t)tcnt * N * n_terms * spitch, &err);
    if (!S) return err;
    const int GB = tc05 ? 64 : imma_gblock();
    // every basis prime below 2^56: byte plane 7 of every staged word and plaintext is zero
    bool planes7 = !getenv_flag_off("BCN_UMMA_7PLANES");
    for (int t = 0; t < next && planes7; t++) planes7 = c->primes[ext.prime[t]] < (1ull << 56);
    for (int g0 = 0; g0 < G; g0 += GB) {
        const int gcnt = std::min(GB, G - g0);
        for (int t0 = 0; t0 < next; t0 += tcnt) {
            const int tc = std::min(tcnt, next - t0);
            // algorithmic bytes of the pair (per limb: each distinct source's U digits and c0 / c1 once, each
            // term's key words once, the staged words written and read once, the plaintext planes, the outputs)
            const unsigned long long wN = 8ull * (unsigned long long)N, cols = 2ull * (unsigned long long)gcnt;
            const unsigned long long staged = (unsigned long long)tc * wN * n_terms * cols;
            unsigned long long src_words = 0, key_words = 0;
            for (int k = 0; k < n_terms; k++) {
                const bool first = k == 0 || srcs[k] != srcs[k - 1];
                if (first) src_words += (unsigned long long)(T->ndig + 2) * gcnt;     // U digits + c0 + c1 (upper bound)
                if (gal[k] != 1) key_words += 2ull * T->ndig;
            }
            int ti = g_conv_timer.begin(0, (unsigned long long)tc * wN * (src_words + key_words) + staged, st);
            CUDA_TRY(slot_major_ks_op(S, KT, g0, gcnt, t0, tc, nl, next, T->ndig, c->logn, spitch,
                                      2LL * c->nbasis * N, (long long)c->nbasis * N, ext, c->pr, c->pmod, st,
                                      c->fp_conv ? c->fq : nullptr));
            g_conv_timer.end(ti, st);
            ti = g_conv_timer.begin(1, staged + (unsigned long long)tc * N * nch * opad * 256ull +
                                           (unsigned long long)tc * wN * n_out * cols, st);
            if (tc05)
                CUDA_TRY(mac_umma_op(acc, cw, n_out, n_terms, (const unsigned char*)planes, S, g0, gcnt, t0, tc, opad,
                                     next, c->logn, ext, c->pr, 0, st, planes7 ? 7 : 8));
            else
                CUDA_TRY(mac_imma_op(acc, cw, M, (const unsigned char*)planes, S, g0, gcnt, t0, tc, opad, next,
                                     c->logn, ext, c->pr, 0, st));
            g_conv_timer.end(ti, st);
        }
    }
    // the O x G extended-basis sums -> one merged ModDown + rescale each
    return mdr_tail(c, (u64*)out, acc, nullptr, 0, n_out * G, level, T, Z, st);
}

int bcn_mac_multi_planes(bcn_ctx* c, uint64_t* out, int n_out, int n_terms, const uint64_t* const* cts,
                         const uint8_t* planes, int G, int level, int rescale, void* stream) {
    return bcn_mac_multi_planes_layout(c, out, n_out, n_terms, cts, planes, G, level, rescale, BCN_PLANES_IMMA,
                                       stream);
}

int bcn_mac_multi_planes_layout(bcn_ctx* c, uint64_t* out, int n_out, int n_terms, const uint64_t* const* cts,
                                const uint8_t* planes, int G, int level, int rescale, int layout, void* stream) {
    if (layout != BCN_PLANES_IMMA && layout != BCN_PLANES_TCGEN05) return fail(BCN_ERR_PARAM, "unknown planes layout");
    int e = check_level(c, level);
    if (e) return e;
    int opad, nch;
    e = planes_geometry(n_out, n_terms, &opad, &nch);
    if (e) return e;
    if (rescale && level < 1) return fail(BCN_ERR_DEPTH, "multiplicative depth exhausted: level is 0");
    cudaStream_t st = (cudaStream_t)stream;
    const int nl = level + 1;
    const long long N = c->N;
    const long long cw = (long long)G * 2 * nl * N;
    Limbs l = limbs_range(0, nl);
    u64* acc = (u64*)out;
    int err = 0;
    if (rescale) {
        acc = scratch_get(c, (size_t)n_out * cw + (size_t)2 * n_out * G * N * (1 + level), &err);
        if (!acc) return err;
    }
    MacImma M;
    M.n_terms = n_terms;
    M.n_out = n_out;
    for (int k = 0; k < n_terms; k++) M.ct[k] = (const u64*)cts[k];
    // stage blocks of slot sets x tcnt limbs slot-major (<= ~4 GiB), then multiply:
    // tcgen05 blocks of 64 slot sets (M = 128 columns), IMMA blocks of IMMA_GB
    const bool tc05 = layout == BCN_PLANES_TCGEN05;
    const int spitch = tc05 ? 128 : 64;
    const size_t per_limb = (size_t)N * n_terms * spitch * sizeof(u64);
    const int tcnt = (int)std::max<size_t>(1, std::min<size_t>(nl, ((size_t)4 << 30) / per_limb));
    u64* S = scratch2_get(c, (size_t)tcnt * N * n_terms * spitch, &err);
    if (!S) return err;
    bool planes7 = !getenv_flag_off("BCN_UMMA_7PLANES");
    for (int t = 0; t < nl && planes7; t++) planes7 = c->primes[t] < (1ull << 56);
    const int GB = tc05 ? 64 : imma_gblock();
    for (int g0 = 0; g0 < G; g0 += GB) {
        const int gcnt = std::min(GB, G - g0);
        for (int t0 = 0; t0 < nl; t0 += tcnt) {
            const int tc = std::min(tcnt, nl - t0);
            const unsigned long long wN = 8ull * (unsigned long long)N, cols = 2ull * (unsigned long long)gcnt;
            const unsigned long long staged = (unsigned long long)tc * wN * n_terms * cols;
            int ti = g_conv_timer.begin(0, 2 * staged, st);           // a transposition: every word read and written
            CUDA_TRY(slot_major_op(S, M, g0, gcnt, t0, tc, nl, c->logn, st, spitch));
            g_conv_timer.end(ti, st);
            ti = g_conv_timer.begin(1, staged + (unsigned long long)tc * N * nch * opad * 256ull +
                                           (unsigned long long)tc * wN * n_out * cols, st);
            if (tc05)
                CUDA_TRY(mac_umma_op(acc, cw, n_out, n_terms, (const unsigned char*)planes, S, g0, gcnt, t0, tc, opad,
                                     nl, c->logn, l, c->pr, 0, st, planes7 ? 7 : 8));
            else
                CUDA_TRY(mac_imma_op(acc, cw, M, (const unsigned char*)planes, S, g0, gcnt, t0, tc, opad, nl,
                                     c->logn, l, c->pr, 0, st));
            g_conv_timer.end(ti, st);
        }
    }
    if (!rescale) return BCN_OK;
    LevelTables* LT;
    e = build_level(c, level, &LT);
    if (e) return e;
    const int npoly = 2 * n_out * G;
    u64* top = acc + (size_t)n_out * cw;
    u64* W = top + (size_t)npoly * N;
    CUDA_TRY(rescale_tail(c, (u64*)out, acc, nl * N, npoly, level, top, W, LT, st));
    return BCN_OK;
}

int bcn_mac_terms_acc(bcn_ctx* c, uint64_t* out, int n_terms, const uint64_t* const* cts, const uint64_t* const* pts,
                      const int* pt_batched, int G, int level, void* stream) {
    return mac_terms_impl(c, out, n_terms, cts, pts, pt_batched, G, level, 0, 1, stream);
}

static int mac_terms_impl(bcn_ctx* c, uint64_t* out, int n_terms, const uint64_t* const* cts,
                          const uint64_t* const* pts, const int* pt_batched, int G, int level, int rescale,
                          int accumulate, void* stream) {
    int e = check_level(c, level);
    if (e) return e;
    if (n_terms < 1) return fail(BCN_ERR_PARAM, "no terms");
    if (rescale && level < 1) return fail(BCN_ERR_DEPTH, "multiplicative depth exhausted: level is 0");
    cudaStream_t st = (cudaStream_t)stream;
    const int nl = level + 1;
    const long long N = c->N;
    Limbs l = limbs_range(0, nl);
    u64* acc = (u64*)out;
    int err = 0;
    if (rescale) {
        acc = scratch_get(c, (size_t)G * 2 * nl * N + (size_t)2 * G * N * (1 + level), &err);
        if (!acc) return err;
    }
    MacTerms T;
    for (int t0 = 0; t0 < n_terms; t0 += BCN_MAC_TERMS) {
        T.n = std::min(BCN_MAC_TERMS, n_terms - t0);
        for (int k = 0; k < T.n; k++) {
            T.ct[k] = (const u64*)cts[t0 + k];
            T.pt[k] = (const u64*)pts[t0 + k];
            T.pt_batched[k] = (unsigned char)(pt_batched[t0 + k] != 0);
        }
        CUDA_TRY(mac_terms_op(acc, T, G, nl, c->logn, l, c->pr, (t0 > 0) || accumulate, st));
    }
    if (!rescale) return BCN_OK;
    LevelTables* LT;
    e = build_level(c, level, &LT);
    if (e) return e;
    const int npoly = 2 * G;
    u64* top = acc + (size_t)G * 2 * nl * N;
    u64* W = top + (size_t)npoly * N;
    CUDA_TRY(rescale_tail(c, (u64*)out, acc, nl * N, npoly, level, top, W, LT, st));
    return BCN_OK;
}

int bcn_mac(bcn_ctx* c, uint64_t* out, const uint64_t* ct, const uint64_t* pt_mont, int n_items, int group,
            int nlimb, void* stream) {
    if (nlimb < 1 || nlimb > c->nbasis || group < 1) return fail(BCN_ERR_PARAM, "bad MAC shape");
    const long long N = c->N;
    CUDA_TRY(mac_op((u64*)out, (const u64*)ct, 2 * nlimb * N, (const u64*)pt_mont, nlimb * N, n_items, group, nlimb,
                    c->logn, limbs_range(0, nlimb), c->pr, (cudaStream_t)stream));
    return BCN_OK;
}

// config 2 in one pass: out[g] = Rescale(sum_t NTT(ct_t) (.) pt_t), the
// ciphertexts in the coefficient domain (ntt_mac_rescale.cu)
int bcn_ntt_mac_rescale(bcn_ctx* c, uint64_t* out, const uint64_t* ct, const uint64_t* pt_mont, int n_items,
                        int group, int nlimb, void* stream) {
    if (nlimb < 2 || nlimb > 8 || nlimb > c->nq || group < 1 || n_items < 0)
        return fail(BCN_ERR_PARAM, "bad fused MAC shape (2 <= nlimb <= min(8, max_level + 1))");
    if (c->logn < 10 || c->logn > 13) return fail(BCN_ERR_PARAM, "fused NTT+MAC+rescale needs 2^10 <= N <= 2^13 (u64)");
    NmrArgs<u64> a;
    a.ct = (const u64*)ct; a.pt = (const u64*)pt_mont; a.out = (u64*)out; a.tw = c->tw;
    a.n_items = n_items; a.group = group; a.nlimb = nlimb;
    memset(&a.k, 0, sizeof(a.k));
    const int top = nlimb - 1;
    const u64 qt = c->primes[top];
    for (int t = 0; t < nlimb; t++) {
        const PrimeInfo& P = c->hpr[t];
        const u64 qi = P.q;
        a.k.q[t] = qi;
        a.k.qneg[t] = P.qinv_neg;
        a.k.ninv[t] = P.pad[0];
        a.k.ninv_p[t] = P.pad[1];
        a.k.wn[t] = c->wn_host[t];
        a.k.wn_p[t] = shoup_h(c->wn_host[t], qi);
        a.k.inv1[t] = P.pad[2];
        if (t < top) {
            const u64 li = inv_h(qt % qi, qi);
            a.k.qlinv[t] = li;
            a.k.qlinv_p[t] = shoup_h(li, qi);
            a.k.qlmod[t] = qt % qi;
        }
    }
    CUDA_TRY(ntt_mac_rescale_launch<u64>(a, c->logn, (cudaStream_t)stream));
    return BCN_OK;
}

// -------------------------------------------------------- key switching
static u64* key_ptr(bcn_ctx* c, u64 id) {
    auto it = c->keys.find(id);
    return it == c->keys.end() ? nullptr : it->second;
}

static int gen_key(bcn_ctx* c, u64 key_id, const u64* sprime, cudaStream_t st) {
    const long long N = c->N;
    const int nb = c->nbasis;
    u64* key = nullptr;
    CUDA_TRY(dmalloc((void**)&key, sizeof(u64) * c->key_words(), &c->key_bytes));
    int err = 0;
    u64* e_ntt = scratch_get(c, (size_t)nb * N, &err);
    if (!e_ntt) { cudaFree(key); return err; }
    Limbs all = limbs_range(0, nb);
    for (int j = 0; j < c->dnum; j++) {
        const int d0 = j * c->alpha, d1 = std::min((j + 1) * c->alpha, c->nq);
        const u64 kid = key_id * 64 + j;
        u64* b = key + (size_t)j * 2 * nb * N;
        u64* a = b + (size_t)nb * N;
        if (d0 >= c->nq) {   // empty digit (dnum > needed): zero key
            CUDA_TRY(cudaMemsetAsync(b, 0, sizeof(u64) * 2 * nb * N, st));
            continue;
        }
        CUDA_TRY(sample_small_op(e_ntt, nb * N, 1, nb, c->logn, all, c->pr, c->seed, 5u, kid, 0, 0, st));
        CUDA_TRY(ntt_run(c, false, e_ntt, nb * N, all, 1, st));
        CUDA_TRY(ksk_digit_op(b, a, e_ntt, c->s_mont, sprime, nb, d0, d1, c->logn, c->pr, c->pmod, c->seed, kid, st));
    }
    c->keys[key_id] = key;
    return BCN_OK;
}

int bcn_keygen_relin(bcn_ctx* c, void* stream) {
    if (key_ptr(c, 2)) return BCN_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const long long N = c->N;
    const int nb = c->nbasis;
    u64* s2 = nullptr;
    CUDA_TRY(cudaMalloc(&s2, sizeof(u64) * nb * N));
    CUDA_TRY(binary_op(2, s2, 0, c->s_ntt, 0, c->s_mont, 0, 1, nb, c->logn, limbs_range(0, nb), c->pr, st));
    int e = gen_key(c, 2, s2, st);
    cudaStreamSynchronize(st);
    cudaFree(s2);
    return e;
}

int bcn_keygen_galois(bcn_ctx* c, uint64_t g, void* stream) {
    if (g == 1 || key_ptr(c, g)) return BCN_OK;
    if ((g & 1) == 0 || g >= 2ull * c->N) return fail(BCN_ERR_PARAM, "Galois element must be odd and < 2N");
    cudaStream_t st = (cudaStream_t)stream;
    const long long N = c->N;
    const int nb = c->nbasis;
    u64* sg = nullptr;
    CUDA_TRY(cudaMalloc(&sg, sizeof(u64) * nb * N));
    CUDA_TRY(automorph_op(sg, N, c->s_ntt, N, 1, nb, c->logn, (u32)g, st));
    int e = gen_key(c, g, sg, st);
    cudaStreamSynchronize(st);
    cudaFree(sg);
    return e;
}

int bcn_export_key(bcn_ctx* c, uint64_t key_id, uint64_t* out, void* stream) {
    u64* k = key_ptr(c, key_id);
    if (!k) return fail(BCN_ERR_USAGE, "no key with id " + std::to_string(key_id));
    CUDA_TRY(from_mont_op((u64*)out, k, c->N, c->nbasis, 2 * c->dnum, limbs_range(0, c->nbasis), c->pr,
                          (cudaStream_t)stream));
    return BCN_OK;
}

int bcn_export_secret(bcn_ctx* c, uint64_t* out, void* stream) {
    CUDA_TRY(cudaMemcpyAsync(out, c->s_ntt, sizeof(u64) * c->nbasis * c->N, cudaMemcpyDeviceToDevice,
                             (cudaStream_t)stream));
    return BCN_OK;
}

int bcn_modup_words(bcn_ctx* c, int G, int level, uint64_t* words) {
    int e = check_level(c, level);
    if (e) return e;
    *words = (u64)G * ndig_at(c, level) * (level + 1 + c->K) * c->N;
    return BCN_OK;
}

// U = ModUp(x) for x = poly 0 of each of G entries (stride x_stride), level l
static int modup_impl(bcn_ctx* c, u64* U, const u64* x, long long x_stride, int G, int level, u64* tmp,
                      cudaStream_t st) {
    LevelTables* T;
    int e = build_level(c, level, &T);
    if (e) return e;
    const long long N = c->N;
    const int nl = level + 1, next = nl + c->K, ndig = T->ndig;
    Limbs ql = limbs_range(0, nl);
    Limbs ext = limbs_ext(c, level);
    if ((c->logn == 13 || c->logn == 14) && getenv_flag_on("BCN_FUSED_MODUP")) {   // opt-in: measured no faster
        // INTT with hatinv_i folded into its last stage -> y_i; then ONE forward
        // NTT whose prologue base-converts each digit's y to the other limbs and
        // whose skipped (own-digit) CTAs copy the NTT-domain input limbs
        NttArgs ia = ntt_args(c, tmp, nl * N, ql);
        ia.src = x;
        ia.src_poly_stride = x_stride;
        ia.src_limb_stride = N;
        ia.inv_scale = T->upscale;
        CUDA_TRY(ntt_launch(true, c->logn, ia, nl, G, st));
        NttArgs a = ntt_args(c, U, (long long)next * N, ext);
        a.skip_alpha = c->alpha;
        a.skip_dnum = ndig;
        a.skip_level = level;
        a.copy_src = x;
        a.copy_stride = x_stride;
        a.pro = 2;
        a.pro_src = tmp;
        a.pro_stride = nl * N;
        a.pro_dnum = ndig;
        a.pro_dstride = (long long)c->alpha * N;
        a.pro_conv = T->modup;
        CUDA_TRY(ntt_launch(false, c->logn, a, next, G * ndig, st));
        return BCN_OK;
    }
    // coefficient-domain copy of x
    CUDA_TRY(ntt_run_src(c, true, tmp, nl * N, x, x_stride, N, ql, G, st));     // coefficient form of x
    CUDA_TRY(modup_op(U, tmp, nl * N, x, x_stride, G, nl, next, c->alpha, ndig, c->logn, ext, c->pr, T->modup, st,
                      c->fp_conv ? &T->fc_up : nullptr));
    NttArgs a = ntt_args(c, U, (long long)next * N, ext);
    a.skip_alpha = c->alpha;
    a.skip_dnum = ndig;
    a.skip_level = level;
    CUDA_TRY(ntt_launch(false, c->logn, a, next, G * ndig, st));
    return BCN_OK;
}

int bcn_modup(bcn_ctx* c, uint64_t* U, const uint64_t* ct, int ct_nlimb, int G, int level, void* stream) {
    int e = check_level(c, level);
    if (e) return e;
    const long long N = c->N;
    const int nl = level + 1;
    int err = 0;
    u64* tmp = scratch_get(c, (size_t)2 * G * nl * N, &err);
    if (!tmp) return err;
    return modup_impl(c, (u64*)U, (const u64*)ct + (long long)ct_nlimb * N, 2LL * ct_nlimb * N, G, level, tmp,
                      (cudaStream_t)stream);
}


// out (packed ct layout, poly stride nl*N for the 2G component polys) =
//   addend' + (A - conv_P->Q(INTT(A_P))) * P^-1 over the extended-basis pair A.
// N = 2^13 / 2^14: the INTT of the special limbs folds (P/p_k)^-1 into its last
// stage (outputs y_k), then ONE fused cluster NTT converts y -> q_t in its
// prologue and applies the combine + addend in its epilogue; other N: staged.
// fU / fkey (optional, fused form): A's q-limbs were not materialised; the NTT's
// epilogue computes them as the key-switch inner product sum_d sigma(U_d) key_d.
static int moddown_tail(bcn_ctx* c, u64* out, long long os, u64* A, int G, int level, const u64* addend,
                        long long as, int add_c1, u32 g, const LevelTables* T, u64* Z, cudaStream_t st,
                        const u64* fU = nullptr, const u64* fkey = nullptr) {
    const long long N = c->N;
    const int nl = level + 1, next = nl + c->K;
    Limbs ext = limbs_ext(c, level);
    Limbs pl;
    pl.n = c->K;
    for (int k = 0; k < c->K; k++) pl.prime[k] = (short)(c->nq + k);
    Limbs ql = limbs_range(0, nl);
    if ((c->logn == 13 || c->logn == 14) && os == 2LL * nl * N && !getenv_flag_off("BCN_FUSED_MODDOWN")) {
        const bool split = Z && !getenv_flag_off("BCN_SPLIT_CONV");
        NttArgs ia = ntt_args(c, A + (size_t)nl * N, (long long)next * N, pl);
        if (!split) ia.inv_scale = c->md_scale;
        CUDA_TRY(ntt_launch(true, c->logn, ia, c->K, 2 * G, st));
        NttArgs a = ntt_args(c, out, (long long)nl * N, ql);
        if (c->K == 1 && !getenv_flag_off("BCN_K1_LIFT")) {
            // one special prime: the conversion is y mod q_t (the hat factors are 1), so the
            // NTT's lift prologue reads the INTT'd special limb directly (no Z round trip);
            // qtop = ~0 disables the centring (the oracle's fast base conversion is not centred)
            a.pro = 1;
            a.pro_src = A + (size_t)nl * N;
            a.pro_stride = (long long)next * N;
            a.pro_qtop = ~0ull;
            a.pro_tab = T->lift1;
        } else if (split) {
            // base conversion once per coefficient (sources read once, in registers), then
            // a plain-prologue NTT with the fused combine: the prologue form re-reads the
            // sources for every output limb and stalls on their latency
            CUDA_TRY(moddown_conv_op(Z, A, (long long)next * N, 2 * G, nl, c->K, c->logn, ext, c->pr, T->moddown,
                                     st, c->fp_conv ? &T->fc_down : nullptr));
            a.src = Z;
            a.src_poly_stride = (long long)nl * N;
            a.src_limb_stride = N;
        } else {
            a.pro = 2;
            a.pro_src = A + (size_t)nl * N;
            a.pro_stride = (long long)next * N;
            a.pro_conv = T->moddown;
            a.pro_K = c->K;
        }
        a.epi = 2;
        a.epi_c = A;
        a.epi_cps = (long long)next * N;
        a.epi_cls = N;
        if (fU) {
            a.epi = 4;
            a.epi_U = fU;
            a.epi_Ups = (long long)T->ndig * next * N;
            a.epi_Uds = (long long)next * N;
            a.epi_key = fkey;
            a.epi_kds = 2LL * c->nbasis * N;
            a.epi_kcs = (long long)c->nbasis * N;
            a.epi_ndig = T->ndig;
        }
        a.epi_tab = T->pinv;
        a.epi_add = addend;
        a.epi_aps = as;
        a.epi_add_c1 = add_c1;
        a.epi_g = g;
        CUDA_TRY(ntt_launch(false, c->logn, a, nl, 2 * G, st));
        return BCN_OK;
    }
    CUDA_TRY(ntt_run(c, true, A + (size_t)nl * N, (long long)next * N, pl, 2 * G, st));
    CUDA_TRY(moddown_conv_op(Z, A, (long long)next * N, 2 * G, nl, c->K, c->logn, ext, c->pr, T->moddown, st, c->fp_conv ? &T->fc_down : nullptr));
    CUDA_TRY(ntt_run(c, false, Z, (long long)nl * N, ql, 2 * G, st));
    CUDA_TRY(moddown_combine_op(out, os, A, next, Z, addend, as, add_c1, g, G, nl, c->logn, ql, c->pr, T->pinv, st));
    return BCN_OK;
}

// out = addend (+ permuted c0) + ModDown(sum_j U_j (x) key_j)
static int keyswitch_tail(bcn_ctx* c, u64* out, long long os, const u64* U, int G, int level, u64 g, const u64* key,
                          const u64* addend, long long as, int add_c1, u64* tmp, cudaStream_t st) {
    LevelTables* T;
    int e = build_level(c, level, &T);
    if (e) return e;
    const long long N = c->N;
    const int nl = level + 1, next = nl + c->K, ndig = T->ndig;
    Limbs ext = limbs_ext(c, level);
    u64* A = tmp;                                   // [G][2][next][N]
    u64* Z = A + (size_t)G * 2 * next * N;          // [G][2][nl][N]
    if ((c->logn == 13 || c->logn == 14) && os == 2LL * nl * N && !getenv_flag_off("BCN_FUSED_MODDOWN") &&
        getenv_flag_on("BCN_FUSED_INNER")) {
        // BCN_FUSED_INNER=1: inner product of the special limbs only (the INTT needs them); the
        // q-limbs' inner products are computed by the ModDown NTT's epilogue (epilogue 4).  Off by
        // default since the combine epilogue batches its operand loads: materialising every limb and
        // combining in epilogue 2 measured relin 8.93 -> 8.31 ms, single rotations 70.6 -> 63.3 ms
        // (config 3, one box)
        CUDA_TRY(inner_op(A, U, G, next, ndig, c->logn, (u32)g, key, 2LL * c->nbasis * N, (long long)c->nbasis * N,
                          ext, ext, c->pr, st, nl, c->K, c->fp_conv ? c->fq : nullptr));
        return moddown_tail(c, out, os, A, G, level, addend, as, add_c1, (u32)g, T, Z, st, U, key);
    }
    CUDA_TRY(inner_op(A, U, G, next, ndig, c->logn, (u32)g, key, 2LL * c->nbasis * N, (long long)c->nbasis * N, ext,
                      ext, c->pr, st, 0, -1, c->fp_conv ? c->fq : nullptr));
    // INTT of the special limbs of both components
    return moddown_tail(c, out, os, A, G, level, addend, as, add_c1, (u32)g, T, Z, st);
}

static size_t tail_words(const bcn_ctx* c, int G, int level) {
    const int nl = level + 1, next = nl + c->K;
    return (size_t)G * 2 * next * c->N + (size_t)G * 2 * nl * c->N;
}

// out = C0 + ModDown(B) with B = sum_t pt_t sum_j sigma_t(U_t,j) key_t,j (lazy ModDown)
int bcn_premul_key(bcn_ctx* c, uint64_t* out, uint64_t g, const uint64_t* pt, int level, void* stream) {
    int e = check_level(c, level);
    if (e) return e;
    if (g == 1 || (g & 1) == 0) return fail(BCN_ERR_PARAM, "premultiplied keys need odd Galois elements != 1");
    if (!key_ptr(c, g)) {
        e = bcn_keygen_galois(c, g, stream);
        if (e) return e;
    }
    LevelTables* T;
    e = build_level(c, level, &T);
    if (e) return e;
    const long long N = c->N;
    CUDA_TRY(premul_key_op((u64*)out, key_ptr(c, g), (const u64*)pt, T->ndig, level + 1 + c->K, c->logn,
                           2LL * c->nbasis * N, (long long)c->nbasis * N, limbs_ext(c, level), c->pr,
                           (cudaStream_t)stream));
    return BCN_OK;
}

int bcn_rotsum(bcn_ctx* c, uint64_t* out, int n_terms, const uint64_t* const* U, const uint64_t* const* cts,
               const uint64_t* gal, const uint64_t* const* pts, const int* pt_batched, int G, int level,
               void* stream) {
    return bcn_rotsum_keys(c, out, n_terms, U, cts, gal, pts, pt_batched, nullptr, G, level, stream);
}

int bcn_rotsum_keys(bcn_ctx* c, uint64_t* out, int n_terms, const uint64_t* const* U, const uint64_t* const* cts,
                    const uint64_t* gal, const uint64_t* const* pts, const int* pt_batched,
                    const uint64_t* const* keys, int G, int level, void* stream) {
    int e = check_level(c, level);
    if (e) return e;
    if (n_terms < 1) return fail(BCN_ERR_PARAM, "no terms");
    cudaStream_t st = (cudaStream_t)stream;
    for (int k = 0; k < n_terms; k++) {
        if (gal[k] == 1 || (gal[k] & 1) == 0) return fail(BCN_ERR_PARAM, "rotation sum needs odd Galois elements != 1");
        if (!key_ptr(c, gal[k])) {
            e = bcn_keygen_galois(c, gal[k], stream);
            if (e) return e;
        }
    }
    LevelTables* T;
    e = build_level(c, level, &T);
    if (e) return e;
    const long long N = c->N;
    const int nl = level + 1, next = nl + c->K, ndig = T->ndig;
    Limbs ext = limbs_ext(c, level);
    int err = 0;
    u64* B = scratch_get(c, (size_t)G * 2 * next * N + (size_t)G * nl * N + (size_t)G * 2 * nl * N, &err);
    if (!B) return err;
    u64* C0 = B + (size_t)G * 2 * next * N;
    u64* Z = C0 + (size_t)G * nl * N;
    RotTerms R;
    for (int t0 = 0; t0 < n_terms; t0 += BCN_ROT_TERMS) {
        R.n = std::min(BCN_ROT_TERMS, n_terms - t0);
        for (int k = 0; k < R.n; k++) {
            R.U[k] = (const u64*)U[t0 + k];
            const u64* pk = keys ? (const u64*)keys[t0 + k] : nullptr;
            R.key[k] = pk ? pk : key_ptr(c, gal[t0 + k]);
            R.c0[k] = (const u64*)cts[t0 + k];
            R.pt[k] = (const u64*)pts[t0 + k];
            R.g[k] = (u32)gal[t0 + k];
            R.pt_batched[k] = (unsigned char)(pt_batched[t0 + k] != 0);
            if (pk && R.pt_batched[k]) return fail(BCN_ERR_PARAM, "premultiplied keys need a shared (unbatched) pt");
            R.fused[k] = (unsigned char)(pk != nullptr || R.pt[k] == nullptr);
        }
        CUDA_TRY(rotsum_op(B, C0, R, 2LL * nl * N, G, nl, next, ndig, c->logn, 2LL * c->nbasis * N,
                           (long long)c->nbasis * N, ext, c->pr, t0 > 0, st, -1, -1, c->fp_conv ? c->fq : nullptr));
    }
    return moddown_tail(c, (u64*)out, 2LL * nl * N, B, G, level, C0, (long long)nl * N, 0, 1u, T, Z, st);
}

// merged ModDown + rescale: out (level-1, [G][2][level][N]) =
// (B + P C) / (P q_level) for B [G][2][level+1+K][N] (consumed) and the
// optional addend C [G][2][level+1][N] (component 1 only when add_c1).
static int mdr_tail(bcn_ctx* c, u64* out, u64* B, const u64* C, int add_c1, int G, int level, const LevelTables* T,
                    u64* Z, cudaStream_t st, long long c_gstride) {
    const long long N = c->N;
    const int nl = level + 1, next = nl + c->K;
    if (c_gstride <= 0) c_gstride = 2LL * nl * N;       // addend: [G][2][nl][N] unless given
    Limbs sl;
    sl.n = c->K + 1;
    sl.prime[0] = (short)level;
    for (int k = 0; k < c->K; k++) sl.prime[1 + k] = (short)(c->nq + k);
    if (C) {   // Y_top = B_top + P C_top (component 0, and 1 when add_c1)
        const int npoly = add_c1 ? 2 * G : G;
        // polys of component 0 (and 1): B poly p = 2g + comp, C at g * c_gstride + comp * nl * N
        for (int comp = 0; comp < (add_c1 ? 2 : 1); comp++)
            CUDA_TRY(axpy_limb_op(B + (size_t)comp * next * N + (size_t)level * N, 2LL * next * N,
                                  C + (size_t)comp * nl * N + (size_t)level * N, c_gstride, G,
                                  c->pmod_host[2 * level], c->pmod_host[2 * level + 1], c->primes[level], c->logn,
                                  st));
        (void)npoly;
    }
    Limbs ql = limbs_range(0, level);
    if ((c->logn == 13 || c->logn == 14) && !getenv_flag_off("BCN_FUSED_MODDOWN")) {
        const bool split = Z && !getenv_flag_off("BCN_SPLIT_CONV");
        NttArgs ia = ntt_args(c, B + (size_t)level * N, (long long)next * N, sl);
        if (!split) ia.inv_scale = T->mdr_scale;
        CUDA_TRY(ntt_launch(true, c->logn, ia, sl.n, 2 * G, st));
        NttArgs a = ntt_args(c, out, (long long)level * N, ql);
        if (split) {   // conversion once per coefficient, then plain-prologue NTT + fused combine
            Limbs ext = limbs_ext(c, level);
            CUDA_TRY(moddown_conv_op(Z, B, (long long)next * N, 2 * G, level, sl.n, c->logn, ext, c->pr, T->mdr, st, c->fp_conv ? &T->fc_mdr : nullptr));
            a.src = Z;
            a.src_poly_stride = (long long)level * N;
            a.src_limb_stride = N;
        } else {
            a.pro = 2;
            a.pro_src = B + (size_t)level * N;
            a.pro_stride = (long long)next * N;
            a.pro_conv = T->mdr;
            a.pro_K = sl.n;
        }
        a.epi = 3;
        a.epi_c = B;
        a.epi_cps = (long long)next * N;
        a.epi_cls = N;
        a.epi_tab = T->pqinv;
        a.epi_tab2 = T->qlinv;
        a.epi_add = C;
        a.epi_aps = c_gstride;
        a.epi_acs = (long long)nl * N;
        a.epi_add_c1 = add_c1;
        CUDA_TRY(ntt_launch(false, c->logn, a, level, 2 * G, st));
        return BCN_OK;
    }
    CUDA_TRY(ntt_run(c, true, B + (size_t)level * N, (long long)next * N, sl, 2 * G, st));
    Limbs ext = limbs_ext(c, level);
    CUDA_TRY(moddown_conv_op(Z, B, (long long)next * N, 2 * G, level, sl.n, c->logn, ext, c->pr, T->mdr, st, c->fp_conv ? &T->fc_mdr : nullptr));
    CUDA_TRY(ntt_run(c, false, Z, (long long)level * N, ql, 2 * G, st));
    CUDA_TRY(mdr_combine_op(out, B, (long long)next * N, Z, C, c_gstride, add_c1, 2 * G, level, c->logn, ql, c->pr,
                            T->pqinv, T->qlinv, st));
    return BCN_OK;
}

int bcn_rotsum_rescale(bcn_ctx* c, uint64_t* out, int n_terms, const uint64_t* const* U, const uint64_t* const* cts,
                       const uint64_t* gal, const uint64_t* const* pts, const int* pt_batched,
                       const uint64_t* const* keys, int n_ct, const uint64_t* const* ct_cts,
                       const uint64_t* const* ct_pts, const int* ct_batched, int G, int level, void* stream) {
    int e = check_level(c, level);
    if (e) return e;
    if (n_terms < 1) return fail(BCN_ERR_PARAM, "no rotation terms");
    if (level < 1) return fail(BCN_ERR_DEPTH, "multiplicative depth exhausted: level is 0");
    cudaStream_t st = (cudaStream_t)stream;
    for (int k = 0; k < n_terms; k++) {
        if (gal[k] == 1 || (gal[k] & 1) == 0) return fail(BCN_ERR_PARAM, "rotation sum needs odd Galois elements != 1");
        if (!key_ptr(c, gal[k])) {
            e = bcn_keygen_galois(c, gal[k], stream);
            if (e) return e;
        }
    }
    LevelTables* T;
    e = build_level(c, level, &T);
    if (e) return e;
    const long long N = c->N;
    const int nl = level + 1, next = nl + c->K, ndig = T->ndig;
    Limbs ext = limbs_ext(c, level);
    int err = 0;
    u64* B = scratch_get(c, (size_t)G * 2 * next * N + (size_t)G * 2 * nl * N + (size_t)G * 2 * level * N, &err);
    if (!B) return err;
    u64* Cf = B + (size_t)G * 2 * next * N;
    u64* Z = Cf + (size_t)G * 2 * nl * N;
    if (n_ct > 0) {   // ct x pt terms -> both components of the addend
        MacTerms M;
        Limbs l = limbs_range(0, nl);
        for (int t0 = 0; t0 < n_ct; t0 += BCN_MAC_TERMS) {
            M.n = std::min(BCN_MAC_TERMS, n_ct - t0);
            for (int k = 0; k < M.n; k++) {
                M.ct[k] = (const u64*)ct_cts[t0 + k];
                M.pt[k] = (const u64*)ct_pts[t0 + k];
                M.pt_batched[k] = (unsigned char)(ct_batched[t0 + k] != 0);
            }
            CUDA_TRY(mac_terms_op(Cf, M, G, nl, c->logn, l, c->pr, t0 > 0, st));
        }
    }
    RotTerms R;
    for (int t0 = 0; t0 < n_terms; t0 += BCN_ROT_TERMS) {
        R.n = std::min(BCN_ROT_TERMS, n_terms - t0);
        for (int k = 0; k < R.n; k++) {
            const u64* pk = keys ? (const u64*)keys[t0 + k] : nullptr;
            R.key[k] = pk ? pk : key_ptr(c, gal[t0 + k]);
            R.U[k] = (const u64*)U[t0 + k];
            R.c0[k] = (const u64*)cts[t0 + k];
            R.pt[k] = (const u64*)pts[t0 + k];
            R.g[k] = (u32)gal[t0 + k];
            R.pt_batched[k] = (unsigned char)(pt_batched[t0 + k] != 0);
            if (pk && R.pt_batched[k]) return fail(BCN_ERR_PARAM, "premultiplied keys need a shared (unbatched) pt");
            R.fused[k] = (unsigned char)(pk != nullptr || R.pt[k] == nullptr);
        }
        CUDA_TRY(rotsum_op(B, Cf, R, 2LL * nl * N, G, nl, next, ndig, c->logn, 2LL * c->nbasis * N,
                           (long long)c->nbasis * N, ext, c->pr, t0 > 0, st, 2LL * nl * N, (t0 > 0) || (n_ct > 0),
                           c->fp_conv ? c->fq : nullptr));
    }
    return mdr_tail(c, (u64*)out, B, Cf, n_ct > 0, G, level, T, Z, st);
}

int bcn_rotate_hoisted(bcn_ctx* c, uint64_t* out, const uint64_t* ct, int ct_nlimb, const uint64_t* U, int G,
                       int level, uint64_t g, void* stream) {
    int e = check_level(c, level);
    if (e) return e;
    cudaStream_t st = (cudaStream_t)stream;
    const long long N = c->N;
    const int nl = level + 1;
    if (g == 1) {
        CUDA_TRY(copy_limbs_op((u64*)out, nl * N, (const u64*)ct, ct_nlimb * N, 2 * G, nl * N, st));
        return BCN_OK;
    }
    u64* key = key_ptr(c, g);
    if (!key) {
        e = bcn_keygen_galois(c, g, stream);
        if (e) return e;
        key = key_ptr(c, g);
    }
    int err = 0;
    u64* tmp = scratch_get(c, tail_words(c, G, level), &err);
    if (!tmp) return err;
    return keyswitch_tail(c, (u64*)out, 2LL * nl * N, (const u64*)U, G, level, g, key, (const u64*)ct,
                          2LL * ct_nlimb * N, 0, tmp, st);
}

// n_rot hoisted rotations of ONE source: out u64[n_rot][G][2][level+1][N].  Source-shared form: one FP64 kernel
// computes every rotation's key-switch inner products over all level+1+K limbs with the source's U digits (and
// P c0) in registers across <= 16 rotations (mac_imma.cu, slot_major_ks3's natural-layout mode), so U crosses L2
// once instead of once per rotation; the ModDown of ALL rotations is then one INTT launch and one NTT launch
// with the combine epilogue (ModDown(B + P sigma(c0)) = ModDown(B) + sigma(c0) exactly).
int bcn_rotate_hoisted_many(bcn_ctx* c, uint64_t* out, const uint64_t* ct, int ct_nlimb, const uint64_t* U, int G,
                            int level, int n_rot, const uint64_t* gal, void* stream) {
    int e = check_level(c, level);
    if (e) return e;
    if (n_rot < 1) return fail(BCN_ERR_PARAM, "no rotations");
    cudaStream_t st = (cudaStream_t)stream;
    const long long N = c->N;
    const int nl = level + 1, next = nl + c->K;
    LevelTables* T;
    e = build_level(c, level, &T);
    if (e) return e;
    bool shared = c->fp_conv && (c->logn == 13 || c->logn == 14) && T->ndig <= 3 && ct_nlimb == nl &&
                  !getenv_flag_off("BCN_ROT_MANY") && !getenv_flag_off("BCN_FUSED_MODDOWN");
    for (int k = 0; k < n_rot; k++) {
        if ((gal[k] & 1) == 0) return fail(BCN_ERR_PARAM, "Galois elements are odd");
        if (gal[k] == 1) shared = false;
    }
    const size_t ow = (size_t)G * 2 * nl * N;
    if (!shared) {
        for (int k = 0; k < n_rot; k++) {
            e = bcn_rotate_hoisted(c, out + k * ow, ct, ct_nlimb, U, G, level, gal[k], stream);
            if (e) return e;
        }
        return BCN_OK;
    }
    for (int k = 0; k < n_rot; k++)
        if (!key_ptr(c, gal[k])) {
            e = bcn_keygen_galois(c, gal[k], stream);
            if (e) return e;
        }
    const int chunk = std::min(n_rot, 16);
    int err = 0;
    u64* A = scratch_get(c, tail_words(c, chunk * G, level), &err);   // [chunk][G][2][next][N] (+ Z)
    if (!A) return err;
    u64* Z = A + (size_t)chunk * G * 2 * next * N;
    for (int k0 = 0; k0 < n_rot; k0 += chunk) {
        KsTerms KT;
        KT.n = std::min(chunk, n_rot - k0);
        for (int k = 0; k < KT.n; k++) {
            KT.src[k] = (const u64*)ct;
            KT.U[k] = (const u64*)U;
            KT.key[k] = key_ptr(c, gal[k0 + k]);
            KT.g[k] = (u32)gal[k0 + k];
        }
        CUDA_TRY(ks_inner_multi_op(A, KT, G, nl, next, T->ndig, c->logn, 2LL * c->nbasis * N,
                                   (long long)c->nbasis * N, limbs_ext(c, level), c->pr, c->pmod, c->fq, st));
        e = moddown_tail(c, (u64*)out + k0 * ow, 2LL * nl * N, A, KT.n * G, level, nullptr, 0, 0, 1u, T, Z, st);
        if (e) return e;
    }
    return BCN_OK;
}

int bcn_rotate(bcn_ctx* c, uint64_t* out, const uint64_t* ct, int ct_nlimb, int G, int level, uint64_t g,
               void* stream) {
    int e = check_level(c, level);
    if (e) return e;
    cudaStream_t st = (cudaStream_t)stream;
    const long long N = c->N;
    const int nl = level + 1;
    if (g == 1) return bcn_rotate_hoisted(c, out, ct, ct_nlimb, nullptr, G, level, g, stream);
    if (!key_ptr(c, g)) {
        e = bcn_keygen_galois(c, g, stream);
        if (e) return e;
    }
    LevelTables* T;
    e = build_level(c, level, &T);
    if (e) return e;
    const size_t uw = (size_t)G * T->ndig * (nl + c->K) * N;
    const size_t mw = (size_t)2 * G * nl * N;
    const size_t tw = tail_words(c, G, level);
    int err = 0;
    u64* base = scratch_get(c, uw + std::max(mw, tw), &err);
    if (!base) return err;
    u64* U = base;
    e = modup_impl(c, U, (const u64*)ct + (long long)ct_nlimb * N, 2LL * ct_nlimb * N, G, level, base + uw, st);
    if (e) return e;
    return keyswitch_tail(c, (u64*)out, 2LL * nl * N, U, G, level, g, key_ptr(c, g), (const u64*)ct,
                          2LL * ct_nlimb * N, 0, base + uw, st);
}

int bcn_mul_cc(bcn_ctx* c, uint64_t* out, const uint64_t* a, int a_nlimb, const uint64_t* b, int b_nlimb, int G,
               int level, int rescale, void* stream) {
    int e = check_level(c, level);
    if (e) return e;
    if (rescale && level < 1) return fail(BCN_ERR_DEPTH, "multiplicative depth exhausted: level is 0");
    cudaStream_t st = (cudaStream_t)stream;
    if (!key_ptr(c, 2)) {
        e = bcn_keygen_relin(c, stream);
        if (e) return e;
    }
    LevelTables* T;
    e = build_level(c, level, &T);
    if (e) return e;
    const long long N = c->N;
    const int nl = level + 1;
    const size_t dw = (size_t)G * 3 * nl * N;                 // d0, d1, d2
    const size_t uw = (size_t)G * T->ndig * (nl + c->K) * N;  // ModUp(d2)
    const size_t rw = (size_t)G * 2 * nl * N;                 // relinearised, pre-rescale
    const size_t mw = (size_t)2 * G * nl * N;
    const size_t tw = tail_words(c, G, level);
    int err = 0;
    u64* base = scratch_get(c, dw + uw + rw + std::max(mw, tw), &err);
    if (!base) return err;
    u64* d = base;
    u64* U = d + dw;
    u64* R = U + uw;
    u64* tmp = R + rw;
    CUDA_TRY(tensor_op(d, (const u64*)a, 2LL * a_nlimb * N, (const u64*)b, 2LL * b_nlimb * N, G, nl, c->logn,
                       limbs_range(0, nl), c->pr, st, c->fp_conv ? c->fq : nullptr));
    e = modup_impl(c, U, d + 2 * nl * N, 3LL * nl * N, G, level, tmp, st);
    if (e) return e;
    if (rescale && !getenv_flag_off("BCN_MERGED_RESCALE")) {
        // relinearise + rescale in one base conversion: (ModDown(A) + (d0, d1)) / q_l
        const int next = nl + c->K;
        u64* A = tmp;                                   // [G][2][next][N]
        u64* Z = A + (size_t)G * 2 * next * N;          // staged path only
        CUDA_TRY(inner_op(A, U, G, next, T->ndig, c->logn, 1u, key_ptr(c, 2), 2LL * c->nbasis * N,
                          (long long)c->nbasis * N, limbs_ext(c, level), limbs_ext(c, level), c->pr, st, 0, -1,
                          c->fp_conv ? c->fq : nullptr));
        return mdr_tail(c, (u64*)out, A, d, 1, G, level, T, Z, st, 3LL * nl * N);
    }
    u64* dst = rescale ? R : (u64*)out;
    e = keyswitch_tail(c, dst, 2LL * nl * N, U, G, level, 1, key_ptr(c, 2), d, 3LL * nl * N, 1, tmp, st);
    if (e) return e;
    if (!rescale) return BCN_OK;
    // rescale R -> out using the tail region as its scratch
    u64* top = tmp;
    u64* W = top + (size_t)2 * G * N;
    const int npoly = 2 * G;
    CUDA_TRY(rescale_tail(c, (u64*)out, R, nl * N, npoly, level, top, W, T, st));
    return BCN_OK;
}

// ----------------------------------------------------------- utilities
int bcn_sample_uniform(bcn_ctx* c, uint64_t* out, int npoly, int nlimb, int prime0, uint64_t seed, uint64_t id0,
                       void* stream) {
    if (prime0 < 0 || prime0 + nlimb > c->nbasis) return fail(BCN_ERR_PARAM, "limb range outside basis");
    CUDA_TRY(sample_uniform_op((u64*)out, (long long)nlimb * c->N, npoly, nlimb, c->logn, limbs_range(prime0, nlimb),
                               c->pr, seed, 6u /*DOM_DATA*/, id0, 1, (cudaStream_t)stream));
    return BCN_OK;
}

int bcn_to_montgomery(bcn_ctx* c, uint64_t* out, const uint64_t* in, int npoly, int nlimb, int prime0, void* stream) {
    if (prime0 < 0 || prime0 + nlimb > c->nbasis) return fail(BCN_ERR_PARAM, "limb range outside basis");
    CUDA_TRY(to_mont_op((u64*)out, (const u64*)in, npoly, nlimb, c->logn, limbs_range(prime0, nlimb), c->pr,
                        (cudaStream_t)stream));
    return BCN_OK;
}

int bcn_automorph(bcn_ctx* c, uint64_t* out, const uint64_t* in, int npoly, int nlimb, uint64_t g, void* stream) {
    const long long N = c->N;
    CUDA_TRY(automorph_op((u64*)out, nlimb * N, (const u64*)in, nlimb * N, npoly, nlimb, c->logn, (u32)g,
                          (cudaStream_t)stream));
    return BCN_OK;
}

}  // extern "C"
