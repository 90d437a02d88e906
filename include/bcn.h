/*
 * bcn.h -- C ABI of libbcn.so, the sm_100a RNS-CKKS engine behind the
 * ciphertext branch of Bi-CryptoNets (arXiv 2402.01296).
 *
 * Boundary: the reference's only plugin seam is the
 * float64 slot-kernel module `ops` (pkg/src/bibranch/backend.py:12-27,
 * _slotops_cy.pyx:16-101).  Real ciphertexts are not slot arrays, so this
 * library sits one level up, behind the `bibranch.sim` API
 * (pkg/src/bibranch/sim.py:142-283); each entry point below names the
 * reference function whose semantics it realises.  The Python mirror
 * (paper_2402_01296_b200/sim.py) binds these with ctypes; INTEGRATION.md
 * shows the binding a maintainer adds to the reference.
 *
 * Conventions
 *  - All buffers are DEVICE pointers to u64 residues (canonical, [0, q))
 *    or float64, owned by the caller (torch).  The library owns only its
 *    tables, the secret key, switching keys and a scratch arena.
 *  - A ciphertext batch is u64[G][2][nlimb][N] in the bit-reversed NTT
 *    domain; limb t is modulo basis prime t (q_0..q_L, then p_0..p_{K-1}).
 *    A "level" l ciphertext uses limbs 0..l; `*_nlimb` arguments give the
 *    limb count of the buffer layout (>= level+1) so higher-level inputs
 *    are read in place (level = min semantics of sim.py:213).
 *  - Every call is asynchronous on `stream` (a cudaStream_t, may be NULL
 *    for the legacy stream).  One context must be used from one stream.
 *  - Return value: BCN_OK or an error code; bcn_last_error() gives a
 *    thread-local message.  Codes map onto the reference's exception
 *    classes (pkg/src/bibranch/errors.py:7-31) in the Python mirror.
 */
#ifndef BCN_H
#define BCN_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BCN_OK 0
#define BCN_ERR_PARAM 1      /* ParameterError / ShapeError       */
#define BCN_ERR_DEPTH 2      /* DepthBudgetError                  */
#define BCN_ERR_USAGE 3      /* UsageError                        */
#define BCN_ERR_CUDA 4       /* DeviceError (new)                 */
#define BCN_ERR_CAPACITY 5   /* CapacityError                     */

typedef struct bcn_ctx bcn_ctx;

const char *bcn_last_error(void);
int bcn_version(void);
/* number of kernels this library has launched in the process (bench evidence) */
int bcn_launch_count(uint64_t *out);

/* ---- plaintext branch (layers.py:329-346 conv_forward on clear tensors): float64
 * conv2d over the whole batch, direct form.  x f64[B][C][H][W], w f64[O][C][kh][kw],
 * bias f64[O] or NULL, out f64[B][O][OH][OW], OH = (H + 2 ph - kh) / sh + 1.
 * Sums in (c, di, dj) order with FMAs (float64 rounding only). */
int bcn_plain_conv2d(const double *x, const double *w, const double *bias, double *out, int B, int C, int H, int W,
                     int O, int kh, int kw, int sh, int sw, int ph, int pw, void *stream);

/* make_context (sim.py:142-169): ring degree N = 2^logn (8 <= N <= 16384),
 * ciphertext primes q[0..max_level], special primes p[0..n_special-1],
 * dnum key-switching digits, Philox seed for sk / keys / encryption. */
int bcn_ctx_create(bcn_ctx **out, int logn, int max_level, const uint64_t *q, int n_special,
                   const uint64_t *p, int dnum, uint64_t seed, int device);
/* upload the canonical-embedding table ksi[k] = exp(2 pi i k / 2N), k <= 2N
 * (host float64 arrays of 2N+1 entries each, computed by numpy on the host so
 * that engine and oracle share the same bits). Must be called once. */
int bcn_ctx_set_fft(bcn_ctx *ctx, const double *re, const double *im);
int bcn_ctx_destroy(bcn_ctx *ctx);
/* bytes of device memory held by tables + keys + scratch */
int bcn_ctx_memory(bcn_ctx *ctx, uint64_t *bytes);
/* drop the scratch arena (between workloads); BCN_ERR_USAGE while frozen */
int bcn_ctx_trim(bcn_ctx *ctx);
/* freeze (delta = +1) / release (delta = -1) the context's arenas.  A CUDA
 * graph captured over this context replays raw pointers into its scratch
 * arenas and pointer tables; while any graph holds the context (freeze count
 * > 0) a call that would grow or free an arena fails with BCN_ERR_USAGE
 * instead of moving memory under the graph.  No reference counterpart: the
 * reference has no device memory (graphs.py). */
int bcn_ctx_freeze(bcn_ctx *ctx, int delta);

/* ---- K1/K2: negacyclic NTT / INTT, in place.
 * data: u64[npoly][nlimb][N]; limb t is modulo basis prime (prime0 + t). */
int bcn_ntt_fwd(bcn_ctx *ctx, uint64_t *data, int npoly, int nlimb, int prime0, void *stream);
int bcn_ntt_inv(bcn_ctx *ctx, uint64_t *data, int npoly, int nlimb, int prime0, void *stream);
/* Measurement only (bench.py roofline): while enabled, every NTT/INTT launch
 * of every context is bracketed by a CUDA event pair on its stream.
 * bcn_ntt_timing(1) clears and starts recording, (0) stops.
 * bcn_ntt_timing_read syncs and fills 5 classes {plain fwd, plain inv,
 * fused fwd, fused inv, encryption NTT with the combine in its epilogue}:
 * summed launch ms, algorithmic bytes (16 B per coefficient + fused operands)
 * and launch counts.  Never used inside a CUDA-graph capture. */
int bcn_ntt_timing(int enable);
int bcn_ntt_timing_read(double *ms, uint64_t *bytes, uint64_t *launches);
/* The same for the conv operand path (bcn_conv_ks_mac / bcn_mac_multi_planes*):
 * 2 classes {slot-major staging (with the key-switch inner products when the
 * conv has them), tensor-core MAC}; bytes = each distinct source / key word
 * read once, the staged words written (class 0) and read (class 1) once, the
 * plaintext planes, the outputs. */
int bcn_conv_timing(int enable);
int bcn_conv_timing_read(double *ms, uint64_t *bytes, uint64_t *launches);

/* ---- K9: encode_plain (sim.py:172-181) + CKKS canonical embedding.
 * vals: f64[nplain][vstride] (first vlen used, rest zero).  out:
 * u64[nplain][level+1][N], NTT domain; montgomery != 0 stores x*2^64 mod q
 * (the form bcn_mul_plain expects for multipliers). */
int bcn_encode(bcn_ctx *ctx, const double *vals, int vlen, int vstride, int nplain, double scale, int level,
               int montgomery, uint64_t *out, void *stream);

/* encode over the extended basis q_0..q_level, p_0..p_{K-1}, Montgomery form:
 * out u64[nplain][level+1+K][N] (multipliers for bcn_rotsum) */
int bcn_encode_ext(bcn_ctx *ctx, const double *vals, int vlen, int vstride, int nplain, double scale, int level,
                   uint64_t *out, void *stream);

/* ---- K10: encrypt_vector (sim.py:184-189), secret-key RLWE.
 * ct_out: u64[G][2][level+1][N]; ciphertext g uses Philox id counter0 + g. */
int bcn_encrypt(bcn_ctx *ctx, const double *vals, int vlen, int vstride, int G, int level, double scale,
                uint64_t counter0, uint64_t *ct_out, void *stream);
/* Fresh encryptions of n_gal rotated copies of every row (the client holds the
 * plaintext: network.py's first conv reads he_rotate(x, r) of the fresh input,
 * sim.py:259-283): ct_out u64[n_gal][G][2][level+1][N]; copy c of row p is
 * Enc(sigma_gal[c](encode(vals[p]))) with Philox id counter0 + c G + p, where
 * sigma_g is X -> X^g on the integer plaintext (gal[c] = 5^r: slots rotated by
 * r; 1: the row itself).  One canonical embedding per row. */
int bcn_encrypt_rotated(bcn_ctx *ctx, const double *vals, int vlen, int vstride, int G, int level, double scale,
                        uint64_t counter0, int n_gal, const uint64_t *gal, uint64_t *ct_out, void *stream);

/* same, with the Philox id base read from DEVICE memory (*counter_dev) when the
 * kernels run -- lets a captured CUDA graph encrypt with fresh randomness on
 * every replay */
int bcn_encrypt_devctr(bcn_ctx *ctx, const double *vals, int vlen, int vstride, int G, int level, double scale,
                       const uint64_t *counter_dev, uint64_t *ct_out, void *stream);

/* ---- K11: decrypt_vector (sim.py:192-196): c0 + c1 s, INTT, CRT, FFT.
 * out: f64[G][nout] real slot values (nout <= N/2). */
int bcn_decrypt(bcn_ctx *ctx, const uint64_t *ct, int ct_nlimb, int G, int level, double scale, double *out,
                int nout, void *stream);
/* decrypted plaintext polynomial (coefficient domain, limbs 0..min(level,1)) */
int bcn_decrypt_poly(bcn_ctx *ctx, const uint64_t *ct, int ct_nlimb, int G, int level, uint64_t *out,
                     void *stream);

/* ---- K3: he_add (sim.py:208-218).  out = a + b (b_is_plain: b is a
 * u64[Gb][level+1][N] plaintext added to c0 only, Gb in {1, G}). */
int bcn_add(bcn_ctx *ctx, uint64_t *out, const uint64_t *a, int a_nlimb, const uint64_t *b, int b_nlimb,
            int b_is_plain, int b_batch, int G, int level, void *stream);
int bcn_sub(bcn_ctx *ctx, uint64_t *out, const uint64_t *a, int a_nlimb, const uint64_t *b, int b_nlimb,
            int G, int level, void *stream);

/* ---- K4+K5: he_mul ct x plain (sim.py:221-248): out(level-1) =
 * rescale(ct (x) pt); pt_mont: u64[Gp][level+1][N] Montgomery, Gp in {1, G}. */
int bcn_mul_plain(bcn_ctx *ctx, uint64_t *out, const uint64_t *ct, int ct_nlimb, const uint64_t *pt_mont,
                  int pt_batch, int G, int level, void *stream);
/* product without rescale (lazy-rescale accumulation), out at level */
int bcn_mul_plain_norescale(bcn_ctx *ctx, uint64_t *out, const uint64_t *ct, int ct_nlimb,
                            const uint64_t *pt_mont, int pt_batch, int G, int level, void *stream);
/* K4 fused linear combination -- the conv-tap / FC-diagonal sum of
 * conv_accumulate (layers.py:146-163) and fc_forward_multi (layers.py:275-314):
 * out = sum_t ct_t (x) pt_t over n_terms (cts / pts: HOST arrays of DEVICE
 * pointers; ct_t u64[G][2][level+1][N], pt_t Montgomery u64[G or 1][level+1][N]
 * per pt_batched[t]); rescale != 0 -> out u64[G][2][level][N] at level-1,
 * else out u64[G][2][level+1][N] unrescaled. */
int bcn_mac_terms(bcn_ctx *ctx, uint64_t *out, int n_terms, const uint64_t *const *cts, const uint64_t *const *pts,
                  const int *pt_batched, int G, int level, int rescale, void *stream);
/* multi-output form for conv layers (conv output channels share their rotated
 * inputs, network.py:220-228): out_o = sum_k ct_k (x) pt[o*n_terms + k] for
 * o < n_out; out u64[n_out][G][2][level or level+1][N] (rescaled or not). */
int bcn_mac_multi(bcn_ctx *ctx, uint64_t *out, int n_out, int n_terms, const uint64_t *const *cts,
                  const uint64_t *const *pts, int G, int level, int rescale, void *stream);
/* Tensor-core form of bcn_mac_multi (IMMA u8 byte-plane products, bit-exact
 * with it).  The plaintexts of a layer are packed once into byte planes
 * (bcn_planes_bytes bytes, device memory owned by the caller) and reused by
 * every call: pts as for bcn_mac_multi (n_terms <= 256). */
int bcn_planes_bytes(bcn_ctx *ctx, int n_out, int n_terms, int level, uint64_t *bytes);
int bcn_pack_planes(bcn_ctx *ctx, uint8_t *planes, int n_out, int n_terms, const uint64_t *const *pts, int level,
                    void *stream);
int bcn_mac_multi_planes(bcn_ctx *ctx, uint64_t *out, int n_out, int n_terms, const uint64_t *const *cts,
                         const uint8_t *planes, int G, int level, int rescale, void *stream);
/* the same with the byte planes in `layout` (BCN_PLANES_IMMA / BCN_PLANES_TCGEN05):
 * the tcgen05 layout runs the tensor-core MAC on tcgen05.mma with TMEM accumulators
 * (blocks of 64 slot sets); planes from bcn_pack_planes_layout with the same layout */
int bcn_pack_planes_layout(bcn_ctx *ctx, uint8_t *planes, int n_out, int n_terms, const uint64_t *const *pts,
                           int level, int layout, void *stream);
int bcn_mac_multi_planes_layout(bcn_ctx *ctx, uint64_t *out, int n_out, int n_terms, const uint64_t *const *cts,
                                const uint8_t *planes, int G, int level, int rescale, int layout, void *stream);
/* Conv layer with lazy ModDown: out[o] = Rescale(sum_k pt[o][k]
 * (x) rot_{g_k}(src_k)) with the key-switch inner products computed on the
 * fly into the tensor-core MAC over the extended basis and ONE merged
 * ModDown + rescale per output (no per-rotation ModDown).  srcs/Us: per term
 * the source ct u64[G][2][level+1][N] and its bcn_modup (ignored for g = 1);
 * planes: bcn_pack_planes_ext of the extended-basis plaintexts (rotation
 * terms from bcn_encode_ext, identity terms level+1 limbs), packed with the
 * same layout as passed here: BCN_PLANES_IMMA (mma.sync fragments, any G) or
 * BCN_PLANES_TCGEN05 (strip windows for tcgen05.mma kind::i8, 64 slot sets
 * per pass: for G >= 64).  Both give bit-identical results.
 * out u64[n_out][G][2][level][N] at level-1. */
#define BCN_PLANES_IMMA 0
#define BCN_PLANES_TCGEN05 1
int bcn_planes_ext_bytes(bcn_ctx *ctx, int n_out, int n_terms, int level, uint64_t *bytes);
int bcn_pack_planes_ext(bcn_ctx *ctx, uint8_t *planes, int n_out, int n_terms, const uint64_t *const *pts,
                        const int *term_limbs, int level, int layout, void *stream);
int bcn_conv_ks_mac(bcn_ctx *ctx, uint64_t *out, int n_out, int n_terms, const uint64_t *const *srcs,
                    const uint64_t *const *Us, const uint64_t *gal, const uint8_t *planes, int layout, int G,
                    int level, void *stream);
/* same, accumulating into an existing unrescaled out u64[G][2][level+1][N] */
int bcn_mac_terms_acc(bcn_ctx *ctx, uint64_t *out, int n_terms, const uint64_t *const *cts,
                      const uint64_t *const *pts, const int *pt_batched, int G, int level, void *stream);
/* K7+K8+K4 hoisted rotations with lazy ModDown: for terms t
 * = (U_t = bcn_modup of source ct_t, Galois element g_t, multiplier pt_t),
 *   out = sum_t pt_t (x) rotate_{g_t}(ct_t)
 * computed as (sum_t pt_t sigma(c0_t) + ModDown(B_0), ModDown(B_1)) with
 * B = sum_t pt_t * sum_j sigma(U_t,j) (x) key_t,j in the extended basis: one
 * ModDown for the whole sum.  pts: Montgomery, extended basis (bcn_encode_ext),
 * u64[G or 1][level+1+K][N], or NULL for the multiplier 1.  out is unrescaled,
 * u64[G][2][level+1][N]. */
int bcn_rotsum(bcn_ctx *ctx, uint64_t *out, int n_terms, const uint64_t *const *U, const uint64_t *const *cts,
               const uint64_t *gal, const uint64_t *const *pts, const int *pt_batched, int G, int level,
               void *stream);
/* same, with optional per-term key overrides keys[t] (NULL array or entry =
 * the context's Galois key): an override must be bcn_premul_key(g_t, pt_t),
 * i.e. the multiplier folded into the key, which saves the per-term REDC and
 * second product (pt_t must then be unbatched; it still multiplies c0). */
int bcn_rotsum_keys(bcn_ctx *ctx, uint64_t *out, int n_terms, const uint64_t *const *U, const uint64_t *const *cts,
                    const uint64_t *gal, const uint64_t *const *pts, const int *pt_batched,
                    const uint64_t *const *keys, int G, int level, void *stream);
/* Lazy rotation sum (as bcn_rotsum_keys) plus n_ct ciphertext x plaintext terms
 * (ct u64[G][2][level+1][N], Montgomery pt u64[G or 1][level+1][N]), evaluated
 * with ONE merged ModDown + rescale per component: the extended-basis sum B
 * and the q-basis sum C become (B + P C) / (P q_level) through a single base
 * conversion from {q_level, p_*}.  out u64[G][2][level][N]
 * at level-1 (multipliers encoded at q_level keep the scale). */
int bcn_rotsum_rescale(bcn_ctx *ctx, uint64_t *out, int n_terms, const uint64_t *const *U,
                       const uint64_t *const *cts, const uint64_t *gal, const uint64_t *const *pts,
                       const int *pt_batched, const uint64_t *const *keys, int n_ct, const uint64_t *const *ct_cts,
                       const uint64_t *const *ct_pts, const int *ct_batched, int G, int level, void *stream);
/* out u64[dnum][2][nbasis][N] (the Galois key layout) = key_g (x) pt over the
 * extended limbs of `level`; pt Montgomery u64[1][level+1+K][N]. */
int bcn_premul_key(bcn_ctx *ctx, uint64_t *out, uint64_t g, const uint64_t *pt, int level, void *stream);
/* K4 microbenchmark form: out[g] = sum_{t in [g*group, min((g+1)*group, n_items))} ct[t] (x) pt[t] */
int bcn_mac(bcn_ctx *ctx, uint64_t *out, const uint64_t *ct, const uint64_t *pt_mont, int n_items, int group,
            int nlimb, void *stream);

/* ---- K1+K4+K5 fused (BASELINE config 2 in ONE pass):
 * out[g] = Rescale( sum_{t < group} NTT(ct[g group + t]) (.) pt[g group + t] )
 * -- the RNS form of one packed conv output (conv_accumulate,
 * pkg/src/bibranch/layers.py:149-172: plaintext products summed, then one
 * rescale, sim.py:221-248).  ct: u64[n_items][2][nlimb][N] in the
 * COEFFICIENT domain (limb t mod q_t); pt_mont: u64[n_items][nlimb][N], NTT
 * domain, Montgomery; out: u64[ceil(n_items/group)][2][nlimb-1][N], NTT
 * domain.  2 <= nlimb <= 8, 2^10 <= N <= 2^13. */
int bcn_ntt_mac_rescale(bcn_ctx *ctx, uint64_t *out, const uint64_t *ct, const uint64_t *pt_mont, int n_items,
                        int group, int nlimb, void *stream);

/* ---- K5: rescale by q_level: in u64[G][2][in_nlimb][N] -> out u64[G][2][level][N] */
int bcn_rescale(bcn_ctx *ctx, uint64_t *out, const uint64_t *in, int in_nlimb, int G, int level, void *stream);

/* ---- K6+K7: he_mul ct x ct (square_act, layers.py:210-214): tensor,
 * relinearise, rescale.  out: u64[G][2][level][N]. */
int bcn_mul_cc(bcn_ctx *ctx, uint64_t *out, const uint64_t *a, int a_nlimb, const uint64_t *b, int b_nlimb,
               int G, int level, int rescale, void *stream);

/* ---- K7/K8: he_rotate (sim.py:251-256), hoisted form.
 * bcn_modup: U = ModUp(c1) -> u64[G][ndig][level+1+K][N] (size: bcn_modup_words)
 * bcn_rotate_hoisted: out = (sigma_g(c0) + KS0, KS1) using U and the Galois key of g
 * bcn_rotate: both in one call (scratch U).  g = 5^r mod 2N; g = 1 copies. */
int bcn_modup_words(bcn_ctx *ctx, int G, int level, uint64_t *words);
int bcn_modup(bcn_ctx *ctx, uint64_t *U, const uint64_t *ct, int ct_nlimb, int G, int level, void *stream);
int bcn_rotate_hoisted(bcn_ctx *ctx, uint64_t *out, const uint64_t *ct, int ct_nlimb, const uint64_t *U, int G,
                       int level, uint64_t g, void *stream);
int bcn_rotate(bcn_ctx *ctx, uint64_t *out, const uint64_t *ct, int ct_nlimb, int G, int level, uint64_t g,
               void *stream);
/* n_rot hoisted rotations of one source (the baby steps of fc_forward_multi, layers.py:283-330, and
 * BASELINE config 3's 14 rotations): out u64[n_rot][G][2][level+1][N], gal[k] = 5^r_k mod 2N.  Bit-identical to
 * n_rot bcn_rotate_hoisted calls; the source's U digits are read once for all rotations. */
int bcn_rotate_hoisted_many(bcn_ctx *ctx, uint64_t *out, const uint64_t *ct, int ct_nlimb, const uint64_t *U, int G,
                            int level, int n_rot, const uint64_t *gal, void *stream);

/* ---- switching keys (generated on device from the seed, cached) */
int bcn_keygen_relin(bcn_ctx *ctx, void *stream);
int bcn_keygen_galois(bcn_ctx *ctx, uint64_t g, void *stream);
/* canonical copy of a key: out u64[dnum][2][nbasis][N] (key_id: 2 = relin, g = Galois) */
int bcn_export_key(bcn_ctx *ctx, uint64_t key_id, uint64_t *out, void *stream);
/* canonical NTT-domain secret key over the full basis: u64[nbasis][N] */
int bcn_export_secret(bcn_ctx *ctx, uint64_t *out, void *stream);

/* ---- utilities for benches / parity tests */
int bcn_sample_uniform(bcn_ctx *ctx, uint64_t *out, int npoly, int nlimb, int prime0, uint64_t seed,
                       uint64_t id0, void *stream);
int bcn_to_montgomery(bcn_ctx *ctx, uint64_t *out, const uint64_t *in, int npoly, int nlimb, int prime0,
                      void *stream);
int bcn_automorph(bcn_ctx *ctx, uint64_t *out, const uint64_t *in, int npoly, int nlimb, uint64_t g, void *stream);

/* ==== 32-bit-limb variant ========================
 * Residues are u32 modulo primes q < 2^30 (q = 1 mod 2N), Delta = 2^30 -- the
 * reference's default scale (pkg/src/bibranch/cli.py:66) -- so every word is
 * half the HBM bytes of the u64 engine and every product a native 32-bit
 * multiply.  Own context: nlimb primes q[0..nlimb-1], 2 <= nlimb <= 8,
 * N = 2^logn, 2^10 <= N <= 2^14.  Same layouts and ordering as the u64
 * entry points above with uint32_t words; Montgomery form is x 2^32 mod q. */
typedef struct bcn32_ctx bcn32_ctx;
const char *bcn32_last_error(void);
int bcn32_ctx_create(bcn32_ctx **out, int logn, int nlimb, const uint32_t *q, int device);
int bcn32_ctx_destroy(bcn32_ctx *ctx);
/* in-place NTT / INTT of u32[npoly][nlimb][N] (limb t mod q_t) -- K1/K2 */
int bcn32_ntt_fwd(bcn32_ctx *ctx, uint32_t *data, int npoly, void *stream);
int bcn32_ntt_inv(bcn32_ctx *ctx, uint32_t *data, int npoly, void *stream);
/* out = in 2^32 mod q_t over u32[npoly][nlimb][N] */
int bcn32_to_montgomery(bcn32_ctx *ctx, uint32_t *out, const uint32_t *in, int npoly, void *stream);
/* bcn_ntt_mac_rescale with u32 words: ct u32[n_items][2][nlimb][N]
 * (coefficient domain), pt_mont u32[n_items][nlimb][N] (NTT domain,
 * Montgomery), out u32[ceil(n_items/group)][2][nlimb-1][N] (NTT domain) */
int bcn32_ntt_mac_rescale(bcn32_ctx *ctx, uint32_t *out, const uint32_t *ct, const uint32_t *pt_mont, int n_items,
                          int group, void *stream);

#ifdef __cplusplus
}
#endif
#endif
