// ops.cuh -- launcher declarations shared by the kernel files and api.cu
#pragma once
#include "common.cuh"

#define BCN_MAX_ALPHA 16

// Fast base conversion constants for one source set (a ModUp digit or the
// special primes): y_i = [x_i * hatinv_i]_{q_i}; out_t = sum_i y_i * hat_m[i][t]
// with hat_m in Montgomery form (hat * 2^64 mod q_t) so one REDC finishes.
struct ConvTable {
    int n_src;
    int pad;
    u64 hatinv[BCN_MAX_ALPHA];
    u64 hatinv_p[BCN_MAX_ALPHA];
    u64 hat_m[BCN_MAX_ALPHA * BCN_MAX_LIMBS];
};

// FP64 base-conversion constants passed BY VALUE as a kernel parameter: the
// kernel reads them from the constant bank (uniform LDC), not through the
// L1/LSU pipe that the per-thread data loads need (a global table read by
// every warp kept that pipe 77-87% busy).
#define BCN_FC_SRC 8
#define BCN_FC_TGT 24
struct FConv {
    double2 h[BCN_FC_SRC][BCN_FC_TGT];   // {hat_k mod t, that / t} per source k, target limb t
    double2 fq[BCN_FC_TGT];              // target {t, 1/t}
};
struct FConvSet {                        // one FConv per ModUp digit
    FConv d[3];
};

namespace bcn {

struct NttArgs {
    u64* data;
    long long poly_stride;   // words between consecutive batch polys (grid.y)
    long long digit_stride;  // unused unless skip_alpha > 0
    Limbs limbs;             // limb t (grid.x) -> prime index
    const ulonglong2* tw;    // [nprime][2][N] {w, w'}: forward then inverse
    const ulonglong2* twt;   // cluster NTT (logn 13/14): tw with the pass-transposed layout of twf
    const double2* twf;
    int fp_all;              // every limb of the launch is below 2^50 (FP64-only kernel variants)
    int epi_pf;              // cluster NTT: L2-prefetch the fused epilogue's operands at kernel start (set by the launcher)
    int grid_pm;             // cluster NTT grid order: 0 limb fastest (default), 1 poly fastest (set by the launcher)      // same layout, {w, w/q} in FP64 (cluster NTT, q < 2^50); nullptr: integer only
    const PrimeInfo* pr;
    int skip_alpha;          // ModUp: skip limb t of digit d when t/alpha == d and t <= skip_level
    int skip_dnum;
    int skip_level;
    const u64* src;          // out-of-place input (nullptr: in place); same limb layout
    long long src_poly_stride;
    long long src_limb_stride;   // words between limbs of one input poly (N when packed)
    // fused prologue / epilogue of the forward cluster NTT (ntt_cluster.cu)
    int pro;                 // 0: read input; 1: rescale lift of pro_src (one coef limb per poly)
    const u64* pro_src;
    long long pro_stride;
    u64 pro_qtop;            // lift: the dropped prime
    const u64* pro_tab;      // lift: [limb] q_top mod q_t
    int epi;                 // 0: store; 1: rescale combine out = (c - x) * q_top^-1;
                             // 2: ModDown combine out = (A - x) * P^-1 (+ addend)
    const u64* epi_c;        // c[poly * epi_cps + t * epi_cls + n]
    long long epi_cps, epi_cls;
    const u64* epi_tab;      // Shoup pairs per limb
    // ModDown: prologue 2 converts the INTT'd, pre-scaled special limbs
    // (y_k at pro_src + poly * pro_stride + k * N) to limb t; epilogue 2 adds
    // addend[(poly/2) * epi_aps + (poly%2) * nl * N + t * N + perm_g(n)] to
    // component 0 (and component 1 when epi_add_c1).
    const ConvTable* pro_conv;
    int pro_K;
    const u64* epi_add;
    long long epi_aps;
    int epi_add_c1;
    u32 epi_g;
    // inverse: per-limb replacement of the folded n^-1 constants
    // {n^-1 s_t, shoup, w1 n^-1 s_t, shoup} (s_t = hatinv of that special prime)
    const u64* inv_scale;
    // ModUp form of prologue 2: poly = entry * pro_dnum + digit; digit d converts
    // its own source limbs pro_src + entry * pro_stride + d * pro_dstride with
    // table pro_conv[d] (pro_K ignored).  0 = ModDown form.
    int pro_dnum;
    long long pro_dstride;
    // epilogue 3 (merged ModDown + rescale): out = (c - v) * epi_tab + addend * epi_tab2,
    // addend component stride epi_acs (0: limbs.n * N)
    const u64* epi_tab2;
    long long epi_acs;
    // epilogue 4 (fused key-switch inner product): c[j] of epilogue 2 is computed on the fly as
    // REDC(sum_d U[ct][d][t][sigma(j)] * key[d][comp][t][j]) (U: [G][ndig][next][N], key Montgomery)
    const u64* epi_U;
    long long epi_Ups, epi_Uds;
    const u64* epi_key;
    long long epi_kds, epi_kcs;
    int epi_ndig;
    // epilogue 5 (encryption): out = NTT(m + e) - a (x) s, and a written as component 1
    // (out + enc_c1_off): a = U(seed, DOM_ENC_A, prime, enc_id + poly [+ *enc_id_dev], n)
    const u64* enc_s;        // secret key, Montgomery, [nbasis][N]
    u64 enc_seed, enc_id;
    const u64* enc_id_dev;   // graph replays: the id base lives in device memory
    long long enc_c1_off;
    // skipped limbs (skip_alpha) copy copy_src[(poly / skip_dnum) * copy_stride + t * N + n]
    // instead of being left untouched (ModUp: the digit's own NTT-domain limbs)
    const u64* copy_src;
    long long copy_stride;
};

// fused NTT -> MAC -> rescale (ntt_mac_rescale.cu), word W = u32 or u64;
// per-limb constants (limb t = prime t of the chain q_0..q_{nlimb-1})
template <class W> struct NmrConst {
    W q[8], qneg[8], ninv[8], ninv_p[8], wn[8], wn_p[8];
    W qlinv[8], qlinv_p[8];   // q_top^-1 mod q_t (Shoup), t < top
    W qlmod[8];               // q_top mod q_t
    W inv1[8];                // floor(2^bits / q_t): reduction of any word by a Shoup multiply by 1
};
template <class W> struct NmrArgs {
    const W* ct;      // [n_items][2][nlimb][N], coefficient domain
    const W* pt;      // [n_items][nlimb][N], NTT domain, Montgomery
    W* out;           // [n_groups][2][nlimb-1][N], NTT domain
    const void* tw;   // {w, shoup} pairs of W; limb t at t * 2N (forward N entries, then inverse N entries)
    int n_items, group, nlimb;
    NmrConst<W> k;
};
template <class W> cudaError_t ntt_mac_rescale_launch(const NmrArgs<W>& a, int logn, cudaStream_t st);

cudaError_t ntt_launch(bool inverse, int logn, const NttArgs& a, int nlimbs, int npolys, cudaStream_t st);
cudaError_t ntt_cluster_launch(bool inverse, int logn, const NttArgs& a, int nlimbs, int npolys, cudaStream_t st);

cudaError_t binary_op(int op, u64* out, long long os, const u64* a, long long as, const u64* b, long long bs,
                      int npoly, int nlimb, int logn, const Limbs& limbs, const PrimeInfo* pr, cudaStream_t st);
cudaError_t to_mont_op(u64* out, const u64* a, int npoly, int nlimb, int logn, const Limbs& limbs,
                       const PrimeInfo* pr, cudaStream_t st);
cudaError_t mac_op(u64* out, const u64* ct, long long ct_stride, const u64* pt, long long pt_stride,
                   int n_items, int group, int nlimb, int logn, const Limbs& limbs, const PrimeInfo* pr,
                   cudaStream_t st);
// Linear combination sum_t ct_t (x) pt_t of up to BCN_MAC_TERMS terms, each
// ct_t a u64[G][2][nlimb][N] batch and pt_t a Montgomery u64[G or 1][nlimb][N].
#define BCN_MAC_TERMS 160
struct MacTerms {
    int n;
    const u64* ct[BCN_MAC_TERMS];
    const u64* pt[BCN_MAC_TERMS];
    unsigned char pt_batched[BCN_MAC_TERMS];
};
// Lazy-ModDown rotation sum: B = sum_t pt_t * sum_j sigma_t(U_t,j) (x) key_t,j over
// the extended basis and C0 = sum_t pt_t * sigma_t(c0_t) over q_0..q_l.
#define BCN_ROT_TERMS 96
struct RotTerms {
    int n;
    const u64* U[BCN_ROT_TERMS];     // [G][ndig][ext][N]
    const u64* key[BCN_ROT_TERMS];   // [dnum][2][nbasis][N] Montgomery
    const u64* c0[BCN_ROT_TERMS];    // component 0 of the source ct, [G] stride c0_gstride
    const u64* pt[BCN_ROT_TERMS];    // Montgomery, ext basis [G|1][ext][N]; null = 1
    u32 g[BCN_ROT_TERMS];
    unsigned char pt_batched[BCN_ROT_TERMS];
    // 1: key already carries the multiplier (pt (x) key, bcn_premul_key) or
    // there is none -- the digit products go straight into the output sums
    // (no per-term REDC and no second product); pt still multiplies c0
    unsigned char fused[BCN_ROT_TERMS];
};
// out[j][c][kt][n] = key[j][c][kt][n] (x) pt[t][n] over the extended limbs t of a level
cudaError_t premul_key_op(u64* out, const u64* key, const u64* pt, int ndig, int next, int logn,
                          long long kds, long long kcs, const Limbs& ext, const PrimeInfo* pr, cudaStream_t st);
// C0 output: slot set p at C0 + p * c0_ostride (nq limbs); c0_accumulate adds onto it
cudaError_t rotsum_op(u64* B, u64* C0, const RotTerms& terms, long long c0_gstride, int G, int nq, int next,
                      int ndig, int logn, long long key_digit_stride, long long key_comp_stride, const Limbs& ext,
                      const PrimeInfo* pr, int accumulate, cudaStream_t st, long long c0_ostride = -1,
                      int c0_accumulate = -1, const double2* fq = nullptr);
// plaintext-branch conv2d in float64 (direct form), x [B][C][H][W], w [O][C][kh][kw], out [B][O][OH][OW]
cudaError_t plain_conv_op(const double* x, const double* w, const double* b, double* out, int B, int C, int H, int W,
                          int O, int kh, int kw, int sh, int sw, int ph, int pw, cudaStream_t st);
// dst[p][n] = dst[p][n] + src[p][n] * w (mod q) on one limb (Shoup pair w, wp)
cudaError_t axpy_limb_op(u64* dst, long long ds, const u64* src, long long ss, int npoly, u64 w, u64 wp, u64 q,
                         int logn, cudaStream_t st);
// merged ModDown + rescale combine (staged form): out_i = (B_i - Z_i) * pq_i + C_i * ql_i
cudaError_t mdr_combine_op(u64* out, const u64* B, long long bps, const u64* Z, const u64* C, long long cps,
                           int add_c1, int npoly, int nout, int logn, const Limbs& ql, const PrimeInfo* pr,
                           const u64* pqinv, const u64* qlinv, cudaStream_t st);
// Multi-output linear combination out_o = sum_k ct_k (x) pt_{o,k} for a tile of
// up to BCN_MAC_OUT outputs sharing the same ct terms (conv output channels).
#define BCN_MAC_OUT 16
#define BCN_MULTI_TERMS 128
struct MacMulti {
    int n_terms;
    int n_out;
    const u64* ct[BCN_MULTI_TERMS];
    const u64* pt[BCN_MAC_OUT][BCN_MULTI_TERMS];
};
cudaError_t mac_multi_op(u64* out, long long out_stride, const MacMulti& m, int G, int nlimb, int logn,
                         const Limbs& limbs, const PrimeInfo* pr, int accumulate, cudaStream_t st);
// Tensor-core multi-output MAC (mac_imma.cu): ct words gathered per slot,
// plaintexts pre-packed into byte planes by pack_planes_op.
#define BCN_IMMA_TERMS 256
struct MacImma {
    int n_terms;
    int n_out;
    const u64* ct[BCN_IMMA_TERMS];
};
cudaError_t pack_planes_op(unsigned char* planes, const u64* const* pts_dev, int n_out, int n_terms, int opad,
                           int nch, int nl, int logn, cudaStream_t st, const int* tlimbs_dev = nullptr);
// conv terms with lazy ModDown (mac_imma.cu: slot_major_ks_kernel)
struct KsTerms {
    int n;
    const u64* src[BCN_IMMA_TERMS];   // source ct u64[G][2][level+1][N]
    const u64* U[BCN_IMMA_TERMS];     // its ModUp u64[G][ndig][ext][N] (g != 1)
    const u64* key[BCN_IMMA_TERMS];   // Galois key (g != 1)
    u32 g[BCN_IMMA_TERMS];            // 1: the source itself
};
cudaError_t slot_major_ks_op(u64* S, const KsTerms& T, int g0, int gcnt, int t0, int tcnt, int nq, int next, int ndig,
                             int logn, int spitch, long long kds, long long kcs, const Limbs& ext, const PrimeInfo* pr,
                             const u64* pmod, cudaStream_t st, const double2* fq = nullptr);
// <= 16 rotations of one source in the natural layout out[k][G][2][next][N] (mac_imma.cu, slot_major_ks3's other mode)
cudaError_t ks_inner_multi_op(u64* out, const KsTerms& T, int G, int nq, int next, int ndig, int logn, long long kds,
                              long long kcs, const Limbs& ext, const PrimeInfo* pr, const u64* pmod,
                              const double2* fq, cudaStream_t st);
// tcgen05 conv MAC (mac_umma.cu): planes in the strip layout, S with a 128-word pitch, gcnt <= 64
cudaError_t pack_planes_umma_op(unsigned char* planes, const u64* const* pts_dev, int n_out, int n_terms, int opad,
                                int nch, int nl, int logn, cudaStream_t st, const int* tlimbs_dev = nullptr);
cudaError_t mac_umma_op(u64* out, long long out_stride, int n_out, int n_terms, const unsigned char* planes,
                        const u64* S, int g0, int gcnt, int t0, int tcnt, int opad, int nlimb, int logn,
                        const Limbs& limbs, const PrimeInfo* pr, int accumulate, cudaStream_t st, int nplanes = 8);
// slot-major staging of a g-block x limb-block of the ct terms: S[(tl N + n) K + k][64]
cudaError_t slot_major_op(u64* S, const MacImma& m, int g0, int gcnt, int t0, int tcnt, int nlimb, int logn,
                          cudaStream_t st, int spitch = 64);
cudaError_t mac_imma_op(u64* out, long long out_stride, const MacImma& m, const unsigned char* planes, const u64* S,
                        int g0, int gcnt, int t0, int tcnt, int opad, int nlimb, int logn, const Limbs& limbs,
                        const PrimeInfo* pr, int accumulate, cudaStream_t st);
cudaError_t mac_terms_op(u64* out, const MacTerms& terms, int G, int nlimb, int logn, const Limbs& limbs,
                         const PrimeInfo* pr, int accumulate, cudaStream_t st);
cudaError_t tensor_op(u64* d, const u64* a, long long as, const u64* b, long long bs, int G, int nlimb,
                      int logn, const Limbs& limbs, const PrimeInfo* pr, cudaStream_t st, const double2* fq = nullptr);
cudaError_t automorph_op(u64* out, long long os, const u64* in, long long is, int npoly, int nlimb, int logn,
                         u32 g, cudaStream_t st);
cudaError_t modup_op(u64* U, const u64* xc, long long xc_stride, const u64* xn, long long x_stride, int npoly, int nq,
                     int next, int alpha, int ndig, int logn, const Limbs& ext, const PrimeInfo* pr,
                     const ConvTable* tab, cudaStream_t st, const FConvSet* fc = nullptr);
cudaError_t inner_op(u64* A, const u64* U, int npoly, int next, int ndig, int logn, u32 g, const u64* key,
                     long long key_digit_stride, long long key_comp_stride, const Limbs& ext, const Limbs& keyl,
                     const PrimeInfo* pr, cudaStream_t st, int t0 = 0, int tcnt = -1, const double2* fq = nullptr);
cudaError_t moddown_conv_op(u64* Z, const u64* A, long long a_stride, int npoly, int nq, int K, int logn,
                            const Limbs& ext, const PrimeInfo* pr, const ConvTable* tab, cudaStream_t st,
                            const FConv* fc = nullptr);
cudaError_t moddown_combine_op(u64* out, long long os, const u64* A, int next, const u64* Z, const u64* addend,
                               long long as, int add_c1, u32 g, int npoly, int nq, int logn, const Limbs& ql,
                               const PrimeInfo* pr, const u64* pinv, cudaStream_t st);
cudaError_t rescale_lift_op(u64* W, const u64* top, int npoly, int nq, u64 qtop, int logn, const Limbs& ql,
                            const PrimeInfo* pr, cudaStream_t st);
cudaError_t rescale_combine_op(u64* out, long long os, const u64* c, long long cs, const u64* W, int npoly,
                               int nq, int logn, const Limbs& ql, const PrimeInfo* pr, const u64* qinv,
                               cudaStream_t st);
cudaError_t gather_limb_op(u64* dst, const u64* src, long long stride, long long off, int npoly, int logn,
                           cudaStream_t st);
cudaError_t copy_limbs_op(u64* dst, long long ds, const u64* src, long long ss, int npoly, long long per_poly,
                          cudaStream_t st);

// encode.cu
struct FftTab {
    const double* re;
    const double* im;
    const int* rot;
};
cudaError_t encode_op(u64* out, long long os, const double* vals, int vlen, long long vs, int nplain, double scale,
                      int logn, const Limbs& limbs, const PrimeInfo* pr, const FftTab& ft, int add_err, u64 seed,
                      u64 id_base, cudaStream_t st, const u64* id_dev = nullptr, i64* raw = nullptr);
// rotated fresh copies from the integer coefficients `raw` [G][N] (encode_op(..., raw)): see encode.cu
cudaError_t encode_rot_op(u64* out, long long os, const i64* raw, int G, int logn, const Limbs& limbs,
                          const PrimeInfo* pr, int n_copies, const u32* ginv, u64 seed, u64 id_base, cudaStream_t st);
cudaError_t decode_op(double* out, int nout, const u64* poly, long long ps, int k, int npoly, double scale, int logn,
                      const PrimeInfo* pr, const FftTab& ft, u64 q0inv_mod_q1, u64 q0inv_p, cudaStream_t st);
cudaError_t sample_uniform_op(u64* out, long long os, int npoly, int nlimb, int logn, const Limbs& limbs,
                              const PrimeInfo* pr, u64 seed, u32 domain, u64 id_base, u64 id_step, cudaStream_t st);
cudaError_t sample_small_op(u64* out, long long os, int npoly, int nlimb, int logn, const Limbs& limbs,
                            const PrimeInfo* pr, u64 seed, u32 domain, u64 id_base, u64 id_step, int ternary,
                            cudaStream_t st);
cudaError_t encrypt_combine_op(u64* ct, int G, int nlimb, int logn, const Limbs& limbs, const PrimeInfo* pr,
                               const u64* s_mont, u64 seed, u64 id_base, cudaStream_t st,
                               const u64* id_dev = nullptr);
cudaError_t ksk_digit_op(u64* b_out, u64* a_out, const u64* e_ntt, const u64* s_mont, const u64* sprime,
                         int nbasis, int d0, int d1, int logn, const PrimeInfo* pr, const u64* pmod, u64 seed,
                         u64 kid, cudaStream_t st);
cudaError_t decrypt_core_op(u64* out, const u64* ct, long long cs, int nlimb_ct, int k, int npoly, int logn,
                            const PrimeInfo* pr, const u64* s_mont, long long s_stride, cudaStream_t st);
cudaError_t from_mont_op(u64* out, const u64* in, long long n_words_per_limb, int nlimb, int npoly,
                         const Limbs& limbs, const PrimeInfo* pr, cudaStream_t st);

}  // namespace bcn
