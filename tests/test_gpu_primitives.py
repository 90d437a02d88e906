"""Ciphertext-level parity: every libbcn primitive against the CPU oracle,
bit for bit (canonical u64 residues), at sizes the oracle finishes quickly.
Called through the C ABI (paper_2402_01296_b200/engine.py -> libbcn.so)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle import ckks as O  # noqa: E402
from paper_2402_01296_b200.engine import Engine, to_numpy_u64  # noqa: E402
from paper_2402_01296_b200.params import make_params  # noqa: E402


def _pair(N, L, scale_bits=40, dnum=2, seed=7):
    hp = make_params(N, L, scale_bits, dnum=dnum, seed=seed)
    op = O.make_params(N, L, scale_bits, dnum=dnum, seed=seed)
    assert list(hp.q) == op.q and list(hp.p) == op.p
    return Engine(hp), O.Oracle(op), hp


def _ct_np(ct):
    a = to_numpy_u64(ct)
    return a[:, 0], a[:, 1]


def _assert_ct(gpu_ct, oct_list):
    c0, c1 = _ct_np(gpu_ct)
    for g, oc in enumerate(oct_list):
        np.testing.assert_array_equal(c0[g], oc.c0)
        np.testing.assert_array_equal(c1[g], oc.c1)


@pytest.mark.parametrize("logn", [3, 4, 6, 8, 9, 10, 11, 12, 13, 14])
def test_ntt_matches_oracle(logn):
    N = 1 << logn
    eng, orc, hp = _pair(N, 3, 30 if logn < 12 else 40, dnum=2)
    rng = np.random.default_rng(logn)
    basis = list(hp.q) + list(hp.p)
    x = np.stack([rng.integers(0, q, N, dtype=np.uint64) for q in basis])[None].repeat(3, 0)
    t = torch.from_numpy(x.view(np.int64).copy()).cuda()
    eng.ntt(t, 0)
    got = to_numpy_u64(t)
    exp = np.stack([O.ntt(x[i], basis) for i in range(3)])
    np.testing.assert_array_equal(got, exp)
    eng.ntt(t, 0, inverse=True)
    np.testing.assert_array_equal(to_numpy_u64(t), x)


@pytest.mark.parametrize("logn,bits", [(13, 50), (14, 50), (14, 49), (14, 45)])
def test_ntt_fp64_path_edges(logn, bits, monkeypatch):
    """Primes < 2^50 take the FP64 butterflies of the cluster NTT (primes of
    2^50 and above stay on the integer path): worst-case residues
    (all q-1, alternating 0 / q-1, a single spike) and uniform ones, forward
    and inverse, against the oracle; then the same data with BCN_NTT_FP64=0."""
    N = 1 << logn
    outs = []
    for fp in ("1", "0"):
        monkeypatch.setenv("BCN_NTT_FP64", fp)
        eng, orc, hp = _pair(N, 4, bits, dnum=2, seed=3)
        basis = list(hp.q) + list(hp.p)
        assert any(q < (1 << 50) for q in basis)
        rng = np.random.default_rng(bits)
        qs = np.array(basis, dtype=np.uint64)[:, None]
        alt = np.where(np.arange(N) % 2 == 0, 0, 1).astype(np.uint64)[None] * (qs - np.uint64(1))
        spike = np.zeros((len(basis), N), np.uint64)
        spike[:, N // 3] = (qs[:, 0] - np.uint64(1))
        x = np.stack([np.broadcast_to(qs - np.uint64(1), (len(basis), N)), alt, spike,
                      np.stack([rng.integers(0, q, N, dtype=np.uint64) for q in basis])])
        t = torch.from_numpy(x.view(np.int64).copy()).cuda()
        eng.ntt(t, 0)
        got = to_numpy_u64(t)
        exp = np.stack([O.ntt(x[i], basis) for i in range(len(x))])
        np.testing.assert_array_equal(got, exp)
        eng.ntt(t, 0, inverse=True)
        np.testing.assert_array_equal(to_numpy_u64(t), x)
        y = torch.from_numpy(exp.view(np.int64).copy()).cuda()
        eng.ntt(y, 0, inverse=True)
        np.testing.assert_array_equal(to_numpy_u64(y), x)
        outs.append(got)
    np.testing.assert_array_equal(outs[0], outs[1])


def test_secret_key_matches():
    eng, orc, hp = _pair(64, 4)
    np.testing.assert_array_equal(to_numpy_u64(eng.export_secret()), orc.keys.s_ntt)


def test_encode_matches():
    eng, orc, hp = _pair(256, 3)
    rng = np.random.default_rng(0)
    v = rng.standard_normal((2, 100))
    for lvl, scale in [(3, 2.0 ** 40), (1, float(hp.q[1]))]:
        pt = eng.encode(v, lvl, scale)
        got = to_numpy_u64(pt)
        for g in range(2):
            np.testing.assert_array_equal(got[g], orc.encode(v[g], lvl, scale))


@pytest.mark.parametrize("N", [16, 1024, 16384])
def test_encrypt_decrypt_matches(N):
    eng, orc, hp = _pair(N, 3)
    rng = np.random.default_rng(1)
    v = rng.standard_normal((2, N // 2))
    ct = eng.encrypt(v, counter=11)
    _assert_ct(ct, [orc.encrypt(v[0], 11), orc.encrypt(v[1], 12)])
    dec = eng.decrypt(ct, hp.max_level, hp.scale).cpu().numpy()
    for g in range(2):
        ref = orc.decrypt(orc.encrypt(v[g], 11 + g))
        np.testing.assert_allclose(dec[g], ref, rtol=0, atol=1e-12)
        assert np.abs(dec[g] - v[g]).max() < 1e-6


def _enc2(eng, orc, N, rng, counter=5):
    v = rng.standard_normal((2, N // 2))
    ct = eng.encrypt(v, counter=counter)
    oc = [orc.encrypt(v[0], counter), orc.encrypt(v[1], counter + 1)]
    return v, ct, oc


@pytest.mark.parametrize("N,L,level", [(1024, 3, 3), (8192, 4, 2), (16384, 4, 4)])
def test_encrypt_rotated_matches_oracle(N, L, level):
    """bcn_encrypt_rotated: every copy is the fresh encryption (its own id) of
    the automorphism of the row's plaintext -- bit-identical to the oracle's
    restatement, decrypting to np.roll(row, -r); the unrotated copy equals
    encrypt().  N >= 8192 runs the NTT with the fused encryption epilogue."""
    eng, orc, hp = _pair(N, L, 50 if N >= 8192 else 40, dnum=2)
    rng = np.random.default_rng(71)
    G, rots = 3, [1, 5, N // 2 - 3]
    v = rng.standard_normal((G, N // 2))
    cts = eng.encrypt_rotated(v, rots, level, counter=900)
    assert tuple(cts.shape) == (1 + len(rots), G, 2, level + 1, N)
    base = eng.encrypt(v, level, counter=900)
    assert torch.equal(cts[0], base)
    for c, r in enumerate([0] + rots):
        want = [orc.encrypt_rotated(v[g], r, 900 + c * G + g, level) if r else orc.encrypt(v[g], 900 + g, level)
                for g in range(G)]
        _assert_ct(cts[c], want)
        dec = eng.decrypt(cts[c], level, hp.scale).cpu().numpy()
        assert np.abs(dec - np.roll(v, -r, axis=1)).max() < 1e-6


@pytest.mark.parametrize("C,O,H,stride", [(3, 16, 32, 1), (16, 32, 32, 2), (1, 5, 28, 2), (5, 37, 9, 1)])
def test_plain_conv2d_matches_torch(C, O, H, stride, monkeypatch):
    """libbcn's direct float64 conv of the plaintext branch against cuDNN's
    (summation order differs: float64 rounding only), with and without bias,
    odd sizes and more than one 16-output block."""
    from paper_2402_01296_b200 import plainbranch as PB
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn((7, C, H, H + 3), dtype=torch.float64, device="cuda", generator=g)
    k = 5 if C == 1 else 3
    w = torch.randn((O, C, k, k), dtype=torch.float64, device="cuda", generator=g)
    b = torch.randn(O, dtype=torch.float64, device="cuda", generator=g)
    for bias in (b, None):
        got = PB.conv(x, w, bias, (stride, stride), (1, 1))
        monkeypatch.setenv("BCN_PLAIN_CONV", "0")
        want = PB.conv(x, w, bias, (stride, stride), (1, 1))
        monkeypatch.delenv("BCN_PLAIN_CONV")
        assert got.shape == want.shape
        assert (got - want).abs().max().item() < 1e-12 * max(1.0, want.abs().max().item())


def test_add_mulplain_rescale_match():
    N = 512
    eng, orc, hp = _pair(N, 4)
    rng = np.random.default_rng(2)
    v, ct, oc = _enc2(eng, orc, N, rng)
    w, ct2, oc2 = _enc2(eng, orc, N, rng, counter=9)
    L = hp.max_level
    _assert_ct(eng.add(ct, ct2, L), [orc.add_cc(oc[i], oc2[i]) for i in range(2)])
    p = rng.standard_normal(N // 2)
    pt = eng.encode(p, L, hp.scale)
    _assert_ct(eng.add_plain(ct, pt, L), [orc.add_plain(oc[i], p) for i in range(2)])
    ptm = eng.encode(p, L, float(hp.q[L]), montgomery=True)
    got = eng.mul_plain(ct, ptm, L)
    _assert_ct(got, [orc.mul_plain(oc[i], p) for i in range(2)])
    dec = eng.decrypt(got, L - 1, hp.scale).cpu().numpy()
    assert np.abs(dec[0] - v[0] * p).max() < 1e-6


@pytest.mark.parametrize("N,L,dnum", [(64, 4, 2), (2048, 5, 3), (16384, 6, 3)])
def test_square_relin_matches(N, L, dnum):
    eng, orc, hp = _pair(N, L, dnum=dnum)
    rng = np.random.default_rng(3)
    v, ct, oc = _enc2(eng, orc, N, rng)
    eng.keygen_relin()
    ok = orc.relin_key()
    key = to_numpy_u64(eng.export_key(O.RELIN_KEY_ID))
    for j in range(len(ok[0])):
        np.testing.assert_array_equal(key[j, 0], ok[0][j])
        np.testing.assert_array_equal(key[j, 1], ok[1][j])
    got = eng.mul_cc(ct, ct, L)
    _assert_ct(got, [orc.mul_cc(oc[i], oc[i]) for i in range(2)])
    dec = eng.decrypt(got, L - 1, hp.scale ** 2 / hp.q[L]).cpu().numpy()
    assert np.abs(dec[0] - v[0] ** 2).max() < 1e-5


@pytest.mark.parametrize("N,L,dnum", [(64, 3, 2), (4096, 5, 2), (16384, 4, 3)])
def test_rotate_matches(N, L, dnum):
    eng, orc, hp = _pair(N, L, dnum=dnum)
    rng = np.random.default_rng(4)
    v, ct, oc = _enc2(eng, orc, N, rng)
    for r in [1, 5, -1, N // 2 - 3]:
        got = eng.rotate(ct, r, L)
        _assert_ct(got, [orc.rotate(oc[i], r) for i in range(2)])
        dec = eng.decrypt(got, L, hp.scale).cpu().numpy()
        assert np.abs(dec[1] - np.roll(v[1], -r)).max() < 1e-6
    U = eng.modup(ct, L)
    for r in [2, 7]:
        _assert_ct(eng.rotate(ct, r, L, U=U), [orc.rotate(oc[i], r) for i in range(2)])


def test_rotate_at_lower_level_reads_in_place():
    N = 256
    eng, orc, hp = _pair(N, 4, dnum=2)
    rng = np.random.default_rng(5)
    v, ct, oc = _enc2(eng, orc, N, rng)
    p = rng.standard_normal(N // 2)
    m = eng.mul_plain(ct, eng.encode(p, 4, float(hp.q[4]), montgomery=True), 4)
    om = [orc.mul_plain(oc[i], p) for i in range(2)]
    got = eng.rotate(m, 3, 3)
    _assert_ct(got, [orc.rotate(om[i], 3) for i in range(2)])
    # level-2 view of a level-3 ciphertext (level = min on add, sim.py:213)
    got2 = eng.add(m, got, 2)
    exp = [orc.add_cc(O.Ct(om[i].c0[:3], om[i].c1[:3], 2, om[i].scale), orc.rotate(om[i], 3)) for i in range(2)]
    _assert_ct(got2, exp)


@pytest.mark.parametrize("N,L,dnum", [(64, 3, 2), (2048, 5, 3), (16384, 6, 3)])
def test_rotsum_lazy_moddown_matches(N, L, dnum):
    """Hoisted rotations with ONE ModDown for the whole sum (bcn_rotsum) == oracle."""
    eng, orc, hp = _pair(N, L, dnum=dnum)
    rng = np.random.default_rng(8)
    v, ct, oc = _enc2(eng, orc, N, rng)
    w, ct2, oc2 = _enc2(eng, orc, N, rng, counter=21)
    Ua, Ub = eng.modup(ct, L), eng.modup(ct2, L)
    from paper_2402_01296_b200.params import galois_element as ge
    p1, p2, p3 = rng.standard_normal((3, N // 2))
    ql = float(hp.q[L])
    terms = [(ct, Ua, ge(1, N), eng.encode_ext(p1, L, ql)), (ct, Ua, ge(5, N), eng.encode_ext(p2, L, ql)),
             (ct2, Ub, ge(3, N), eng.encode_ext(p3, L, ql))]
    got = eng.rotsum(terms, L)
    _assert_ct(got, [orc.rotsum([(oc[i], 1, p1), (oc[i], 5, p2), (oc2[i], 3, p3)], L) for i in range(2)])
    dec = eng.decrypt(eng.rescale(got, L), L - 1, hp.scale).cpu().numpy()[0]
    want = np.roll(v[0], -1) * p1 + np.roll(v[0], -5) * p2 + np.roll(w[0], -3) * p3
    assert np.abs(dec - want).max() < 1e-5
    unit = eng.rotsum([(ct, Ua, ge(2, N), None), (ct2, Ub, ge(7, N), None)], L)
    _assert_ct(unit, [orc.rotsum([(oc[i], 2, None), (oc2[i], 7, None)], L) for i in range(2)])
    # multipliers folded into the keys (bcn_premul_key): same ciphertext bit for bit
    keys = [eng.premul_key(t[2], t[3], L) for t in terms]
    _assert_ct(eng.rotsum(terms, L, keys=keys), [orc.rotsum([(oc[i], 1, p1), (oc[i], 5, p2), (oc2[i], 3, p3)], L)
                                                 for i in range(2)])
    mixed = terms + [(ct2, Ub, ge(7, N), None)]
    _assert_ct(eng.rotsum(mixed, L, keys=[keys[0], None, keys[2], None]),
               [orc.rotsum([(oc[i], 1, p1), (oc[i], 5, p2), (oc2[i], 3, p3), (oc2[i], 7, None)], L)
                for i in range(2)])


def test_mac_multi_matches_oracle_composition():
    """Multi-output conv MAC + batched rescale == per-output oracle sums + rescale."""
    N, L = 1024, 3
    eng, orc, hp = _pair(N, L)
    rng = np.random.default_rng(9)
    K, n_out = 11, 10            # > one output tile of 8
    vs = rng.standard_normal((K, N // 2))
    cts = [eng.encrypt(vs[k][None], counter=40 + k) for k in range(K)]
    octs = [orc.encrypt(vs[k], 40 + k) for k in range(K)]
    ws = rng.standard_normal((n_out, K, N // 2))
    ql = float(hp.q[L])
    pts = [[eng.encode(ws[o, k], L, ql, montgomery=True) for k in range(K)] for o in range(n_out)]
    got = eng.mac_multi(cts, pts, L, rescale=True)
    qs = list(hp.q[:L + 1])
    for o in range(n_out):
        acc0 = np.zeros((L + 1, N), dtype=np.uint64)
        acc1 = np.zeros_like(acc0)
        for k in range(K):
            pt = orc.encode(ws[o, k], L, ql)
            acc0 = O.add(acc0, O.mul(octs[k].c0, pt, qs), qs)
            acc1 = O.add(acc1, O.mul(octs[k].c1, pt, qs), qs)
        exp = orc.rescale(O.Ct(acc0, acc1, L, hp.scale * ql))
        _assert_ct(got[o], [exp])


def test_mac_matches():
    N = 1024
    eng, orc, hp = _pair(N, 3, 60)
    nl = 4
    rng = np.random.default_rng(6)
    basis = list(hp.q)
    T, group = 53, 25
    ct = np.stack([np.stack([np.stack([rng.integers(0, q, N, dtype=np.uint64) for q in basis])
                             for _ in range(2)]) for _ in range(T)])
    pt = np.stack([np.stack([rng.integers(0, q, N, dtype=np.uint64) for q in basis]) for _ in range(T)])
    tct = torch.from_numpy(ct.view(np.int64).copy()).cuda()
    tpt = eng.to_montgomery(torch.from_numpy(pt.view(np.int64).copy()).cuda())
    got = to_numpy_u64(eng.mac(tct, tpt, group))
    for g in range(3):
        lo, hi = g * group, min((g + 1) * group, T)
        for c in range(2):
            for i, q in enumerate(basis):
                exp = np.zeros(N, dtype=np.uint64)
                O.lib().orc_mac(O._p(np.ascontiguousarray(ct[lo:hi, c, i])), O._p(np.ascontiguousarray(pt[lo:hi, i])),
                                O._p(exp), hi - lo, N, q)
                np.testing.assert_array_equal(got[g, c, i], exp)


def test_mac_multi_planes_matches_oracle_composition():
    """Tensor-core (IMMA byte-plane) multi-output MAC + rescale == oracle sums + rescale."""
    N, L = 1024, 3
    eng, orc, hp = _pair(N, L)
    rng = np.random.default_rng(19)
    K, n_out = 13, 18            # two output blocks of 16 rows, one partial term chunk
    vs = rng.standard_normal((K, N // 2))
    cts = [eng.encrypt(vs[k][None], counter=80 + k) for k in range(K)]
    octs = [orc.encrypt(vs[k], 80 + k) for k in range(K)]
    ws = rng.standard_normal((n_out, K, N // 2))
    ql = float(hp.q[L])
    pts = [[eng.encode(ws[o, k], L, ql, montgomery=True) for k in range(K)] for o in range(n_out)]
    got = eng.mac_multi_planes(cts, eng.pack_planes(pts, L), n_out, L, rescale=True)
    qs = list(hp.q[:L + 1])
    for o in range(n_out):
        acc0 = np.zeros((L + 1, N), dtype=np.uint64)
        acc1 = np.zeros_like(acc0)
        for k in range(K):
            pt = orc.encode(ws[o, k], L, ql)
            acc0 = O.add(acc0, O.mul(octs[k].c0, pt, qs), qs)
            acc1 = O.add(acc1, O.mul(octs[k].c1, pt, qs), qs)
        exp = orc.rescale(O.Ct(acc0, acc1, L, hp.scale * ql))
        _assert_ct(got[o], [exp])


@pytest.mark.parametrize("layout", [0, 1], ids=["imma", "tcgen05"])
@pytest.mark.parametrize("n_out,K,G,extreme", [(5, 7, 3, False), (16, 33, 1, False), (40, 144, 33, False),
                                               (32, 256, 4, True), (16, 27, 70, False)])
def test_mac_multi_planes_bitexact(n_out, K, G, extreme, layout):
    """Tensor-core multi-output MAC (mma.sync IMMA and tcgen05 layouts) ==
    CUDA-core path bit for bit on uniform residues (60-bit primes: all eight
    bytes live), several output / slot-set blocks (G = 70: a partial second
    tcgen05 block), the 256-term maximum, and the all-(q-1) worst case of the
    int32 partials."""
    N, L = 4096, 2
    hp = make_params(N, L, 60, dnum=1, n_special=1)
    eng = Engine(hp)
    nl = L + 1
    cts = [eng.sample_uniform(2 * G, nl, 0, seed=1000 + k).view(G, 2, nl, N) for k in range(K)]
    pts = [[eng.to_montgomery(eng.sample_uniform(1, nl, 0, seed=5000 + 300 * o + k)) for k in range(K)]
           for o in range(n_out)]
    if extreme:
        for t in range(nl):
            qm1 = int(hp.q[t]) - 1
            qm1 = qm1 - (1 << 64) if qm1 >= (1 << 63) else qm1
            for c in cts:
                c[:, :, t, :] = qm1
            for row in pts:
                for p in row:
                    p[:, t, :] = qm1
    want = to_numpy_u64(eng.mac_multi(cts, pts, L, rescale=False))
    got = to_numpy_u64(eng.mac_multi_planes(cts, eng.pack_planes(pts, L, layout), n_out, L, rescale=False,
                                            layout=layout))
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("N,L", [(1024, 3), (8192, 3)])
def test_rotsum_rescale_merged_matches_oracle(N, L):
    """Rotation sum + ct x pt terms with ONE merged ModDown + rescale
    (bcn_rotsum_rescale; staged at N=1024, fused cluster NTT at N=8192) ==
    Oracle.rotsum_rescale bit for bit, with and without premultiplied keys;
    decrypts to the slot-wise expectation."""
    eng, orc, hp = _pair(N, L, dnum=2)
    rng = np.random.default_rng(31)
    v, ct, oc = _enc2(eng, orc, N, rng)
    w, ct2, oc2 = _enc2(eng, orc, N, rng, counter=41)
    Ua, Ub = eng.modup(ct, L), eng.modup(ct2, L)
    from paper_2402_01296_b200.params import galois_element as ge
    p1, p2, p3, p4 = rng.standard_normal((4, N // 2))
    ql = float(hp.q[L])
    terms = [(ct, Ua, ge(1, N), eng.encode_ext(p1, L, ql)), (ct2, Ub, ge(3, N), eng.encode_ext(p2, L, ql)),
             (ct, Ua, ge(9, N), None)]
    cterms = [(ct2, eng.encode(p3, L, ql, montgomery=True)), (ct, eng.encode(p4, L, ql, montgomery=True))]
    want = [orc.rotsum_rescale([(oc[i], 1, p1), (oc2[i], 3, p2), (oc[i], 9, None)],
                               [(oc2[i], p3), (oc[i], p4)], L) for i in range(2)]
    got = eng.rotsum_rescale(terms, L, ct_terms=cterms)
    _assert_ct(got, want)
    keys = [eng.premul_key(t[2], t[3], L) if t[3] is not None else None for t in terms]
    _assert_ct(eng.rotsum_rescale(terms, L, keys=keys, ct_terms=cterms), want)
    # without ct terms (addend on component 0 only)
    want0 = [orc.rotsum_rescale([(oc[i], 1, p1), (oc2[i], 3, p2)], [], L) for i in range(2)]
    _assert_ct(eng.rotsum_rescale(terms[:2], L), want0)
    scaled = eng.rotsum_rescale(terms[:2], L, ct_terms=cterms)     # every term carries a multiplier
    dec = eng.decrypt(scaled, L - 1, hp.scale).cpu().numpy()
    exp = np.roll(v, -1, axis=1) * p1 + np.roll(w, -3, axis=1) * p2 + w * p3 + v * p4
    assert np.abs(dec - exp).max() < 1e-4


@pytest.mark.parametrize("bits", [40, 50], ids=["int-staging", "fp64-staging"])
@pytest.mark.parametrize("layout", [0, 1], ids=["imma", "tcgen05"])
@pytest.mark.parametrize("N,L", [(1024, 3), (8192, 3)])
def test_conv_ks_mac_matches_oracle(N, L, layout, bits):
    """Conv layer with lazy ModDown (bcn_conv_ks_mac: key-switch inner products
    fused into the slot-major staging, tensor-core MAC over the extended
    basis, one merged ModDown+rescale per output) == Oracle.rotsum_rescale of
    each output bit for bit (identity taps enter as P*x, rotations as
    inner product + P*sigma(c0)).  At 50 bits every prime is in (2^49, 2^50)
    and the staging's component-0 inner products run on the FP64 pipe."""
    eng, orc, hp = _pair(N, L, bits, dnum=2)
    rng = np.random.default_rng(37)
    v, ct, oc = _enc2(eng, orc, N, rng)
    w, ct2, oc2 = _enc2(eng, orc, N, rng, counter=51)
    Ua, Ub = eng.modup(ct, L), eng.modup(ct2, L)
    from paper_2402_01296_b200.params import galois_element as ge
    ql = float(hp.q[L])
    taps = [(ct, Ua, 1, 0), (ct, Ua, 0, 0), (ct2, Ub, 3, 1), (ct2, Ub, 0, 1), (ct, Ua, 7, 0)]   # (src, U, r, which)
    n_out = 3
    vals = rng.standard_normal((n_out, len(taps), N // 2))
    pts = [[eng.encode_ext(vals[o, k], L, ql) if r else eng.encode(vals[o, k], L, ql, montgomery=True)
            for k, (_, _, r, _) in enumerate(taps)] for o in range(n_out)]
    planes = eng.pack_planes_ext(pts, L, layout)
    got = eng.conv_ks_mac([t[0] for t in taps], [t[1] if t[2] else None for t in taps],
                          [ge(t[2], N) if t[2] else 1 for t in taps], planes, n_out, L, layout)
    srcs = [oc, oc, oc2, oc2, oc]
    for o in range(n_out):
        want = [orc.rotsum_rescale([(srcs[k][i], r, vals[o, k]) for k, (_, _, r, _) in enumerate(taps) if r],
                                   [(srcs[k][i], vals[o, k]) for k, (_, _, r, _) in enumerate(taps) if not r], L)
                for i in range(2)]
        _assert_ct(got[o], want)
    dec = eng.decrypt(got[1], L - 1, hp.scale).cpu().numpy()
    x = [v, v, w, w, v]
    exp = sum(np.roll(x[k], -r, axis=1) * vals[1, k] for k, (_, _, r, _) in enumerate(taps))
    assert np.abs(dec - exp).max() < 1e-4


@pytest.mark.parametrize("level,dnum", [(5, 3), (3, 3), (1, 3), (4, 2)], ids=["3digits", "2digits", "1digit", "2digits-K3"])
def test_conv_ks_mac_source_shared_staging_edges(level, dnum):
    """The source-shared FP64 staging kernel (slot_major_ks3: runs of <= 16
    terms over one source, 4 slot sets per warp, 32 per CTA) against the oracle
    bit for bit on its edges: 1 / 2 / 3 key-switch digits, G = 37 slot sets (a
    second CTA half with a partial 4-block), a run of 19 rotations of one source
    (split 16 + 3), a run that starts with the identity tap, a lone identity
    term, and a source whose rotations are not consecutive."""
    N, L = 1024, 5
    eng, orc, hp = _pair(N, L, 50, dnum=dnum)
    rng = np.random.default_rng(53)
    G = 37
    from paper_2402_01296_b200.params import galois_element as ge
    vs = [rng.standard_normal((G, N // 2)) * 0.5 for _ in range(3)]
    xs = [eng.encrypt(v, level=level, counter=400 + 50 * i) for i, v in enumerate(vs)]
    Us = [eng.modup(x, level) for x in xs]
    check = [0, 3, 31, 32, 36]
    ocs = [{g: orc.encrypt(v[g], 400 + 50 * i + g, level) for g in check} for i, v in enumerate(vs)]
    taps = ([(0, r) for r in range(1, 20)] + [(1, 0), (1, 2), (1, 5)] + [(2, 0)] + [(0, 33), (1, 7)])
    ql = float(hp.q[level])
    n_out = 2
    vals = rng.standard_normal((n_out, len(taps), N // 2)) * 0.3
    pts = [[eng.encode_ext(vals[o, k], level, ql) if r else eng.encode(vals[o, k], level, ql, montgomery=True)
            for k, (_, r) in enumerate(taps)] for o in range(n_out)]
    got = eng.conv_ks_mac([xs[i] for i, _ in taps], [Us[i] if r else None for i, r in taps],
                          [ge(r, N) if r else 1 for _, r in taps], eng.pack_planes_ext(pts, level, 0), n_out, level, 0)
    got1 = eng.conv_ks_mac([xs[i] for i, _ in taps], [Us[i] if r else None for i, r in taps],
                           [ge(r, N) if r else 1 for _, r in taps], eng.pack_planes_ext(pts, level, 1), n_out, level, 1)
    assert torch.equal(got, got1)                       # IMMA (16-slot-set blocks) and tcgen05 (64) staging pitches
    c = to_numpy_u64(got.reshape(n_out * G, 2, level, N)).reshape(n_out, G, 2, level, N)
    for o in range(n_out):
        for g in check:
            want = orc.rotsum_rescale([(ocs[i][g], r, vals[o, k]) for k, (i, r) in enumerate(taps) if r],
                                      [(ocs[i][g], vals[o, k]) for k, (i, r) in enumerate(taps) if not r], level)
            np.testing.assert_array_equal(c[o, g, 0], want.c0)
            np.testing.assert_array_equal(c[o, g, 1], want.c1)


def test_conv_ks_mac_blocks_bitexact_vs_eager_path():
    """Lazy-ModDown conv over several output blocks (40 outputs: 32 + 8) and
    slot-set blocks (G = 20: 16 + 4), 60-bit primes with every byte live: the
    result equals the eager path (rotate with ModDown, then MAC, then rescale)
    to CKKS noise, and a rerun is bit-identical (deterministic)."""
    N, L = 2048, 3
    hp = make_params(N, L, 40, dnum=2)
    eng = Engine(hp)
    rng = np.random.default_rng(41)
    G, n_src, n_out = 20, 3, 40
    from paper_2402_01296_b200.params import galois_element as ge
    xs = [eng.encrypt(rng.standard_normal((G, N // 2)) * 0.5, counter=200 + 30 * i) for i in range(n_src)]
    Us = [eng.modup(x, L) for x in xs]
    rots = [0, 1, 5, 31]
    taps = [(i, r) for i in range(n_src) for r in rots]
    ql = float(hp.q[L])
    vals = rng.standard_normal((n_out, len(taps), N // 2)) * 0.3
    pts = [[eng.encode_ext(vals[o, k], L, ql) if r else eng.encode(vals[o, k], L, ql, montgomery=True)
            for k, (_, r) in enumerate(taps)] for o in range(n_out)]
    planes = eng.pack_planes_ext(pts, L)
    args = ([xs[i] for i, _ in taps], [Us[i] if r else None for i, r in taps], [ge(r, N) if r else 1 for _, r in taps],
            planes, n_out, L)
    got = eng.conv_ks_mac(*args)
    again = eng.conv_ks_mac(*args)
    assert torch.equal(got, again)
    dec = eng.decrypt(got.reshape(n_out * G, 2, L, N), L - 1, hp.scale).cpu().numpy().reshape(n_out, G, -1)
    xv = [eng.decrypt(x, L, hp.scale).cpu().numpy() for x in xs]
    for o in (0, 17, 39):
        want = sum(np.roll(xv[i], -r, axis=1) * vals[o, k] for k, (i, r) in enumerate(taps))
        assert np.abs(dec[o] - want).max() < 1e-3


@pytest.mark.parametrize("n_out,rots", [(40, [0, 1, 5, 31]), (16, [0, 1, 2, 3, 4, 5, 6, 7, 9, 11, 13, 17, 19, 23])])
def test_conv_ks_mac_tcgen05_bitexact_vs_imma(n_out, rots):
    """The tcgen05.mma kind::i8 conv MAC (TMEM accumulators, strip-window
    planes, 64 slot sets per pass) is bit-identical to the mma.sync IMMA one:
    G = 70 (one full 64-set pass + a 6-set remainder), 40 outputs (a 32 block
    + a 16-row half block) or 16, 12 terms (one 32-term chunk) or 42 terms
    (two chunks, second partial), 60-bit primes with every byte live."""
    N, L = 2048, 3
    hp = make_params(N, L, 60, dnum=2)
    eng = Engine(hp)
    rng = np.random.default_rng(43)
    G, n_src = 70, 3
    from paper_2402_01296_b200.params import galois_element as ge
    xs = [eng.encrypt(rng.standard_normal((G, N // 2)) * 0.5, counter=300 + 30 * i) for i in range(n_src)]
    Us = [eng.modup(x, L) for x in xs]
    taps = [(i, r) for i in range(n_src) for r in rots]
    ql = float(hp.q[L])
    vals = rng.standard_normal((n_out, len(taps), N // 2)) * 0.3
    pts = [[eng.encode_ext(vals[o, k], L, ql) if r else eng.encode(vals[o, k], L, ql, montgomery=True)
            for k, (_, r) in enumerate(taps)] for o in range(n_out)]
    args = ([xs[i] for i, _ in taps], [Us[i] if r else None for i, r in taps], [ge(r, N) if r else 1 for _, r in taps])
    ref = eng.conv_ks_mac(*args, eng.pack_planes_ext(pts, L, 0), n_out, L, 0)
    got = eng.conv_ks_mac(*args, eng.pack_planes_ext(pts, L, 1), n_out, L, 1)
    assert torch.equal(got, ref)


@pytest.mark.parametrize("N,L,dnum", [(2048, 5, 3), (8192, 6, 2), (16384, 8, 3)])
def test_fp64_base_conversions_match_oracle(N, L, dnum, monkeypatch):
    """All primes in (2^49, 2^50) (the default 50-bit chains): ModUp, ModDown
    and the merged ModDown+rescale base conversions run on the FP64 pipe.
    Rotation, square+relinearise and the merged rotation sum against the
    oracle, and against the integer conversions (BCN_CONV_FP64=0)."""
    from paper_2402_01296_b200.params import galois_element as ge
    outs = []
    for fp in ("1", "0"):
        monkeypatch.setenv("BCN_CONV_FP64", fp)
        eng, orc, hp = _pair(N, L, 50, dnum=dnum, seed=5)
        assert all((1 << 49) < q < (1 << 50) for q in list(hp.q) + list(hp.p))
        rng = np.random.default_rng(17)
        v, ct, oc = _enc2(eng, orc, N, rng)
        rot = eng.rotate(ct, 3, L)
        _assert_ct(rot, [orc.rotate(oc[i], 3) for i in range(2)])
        eng.keygen_relin()
        sq = eng.mul_cc(ct, ct, L)
        _assert_ct(sq, [orc.mul_cc(oc[i], oc[i]) for i in range(2)])
        p1 = rng.standard_normal(N // 2)
        ql = float(hp.q[L])
        U = eng.modup(ct, L)
        terms = [(ct, U, ge(1, N), eng.encode_ext(p1, L, ql)), (ct, U, ge(7, N), None)]
        rs = eng.rotsum_rescale(terms, L)
        want = [orc.rotsum_rescale([(oc[i], 1, p1), (oc[i], 7, None)], [], L) for i in range(2)]
        _assert_ct(rs, want)
        # premultiplied keys: every term fused
        rs2 = eng.rotsum_rescale(terms, L, keys=[eng.premul_key(terms[0][2], terms[0][3], L), None])
        _assert_ct(rs2, want)
        vals = rng.standard_normal((13, N // 2))
        many = [(ct, U, ge(r, N), eng.encode_ext(vals[r - 1], L, ql)) for r in range(1, 14)]
        rs3 = eng.rotsum(many, L, keys=[eng.premul_key(t[2], t[3], L) for t in many])
        if N <= 8192:        # 13 fused terms
            _assert_ct(rs3, [orc.rotsum([(oc[i], r, vals[r - 1]) for r in range(1, 14)], L) for i in range(2)])
        outs.append([to_numpy_u64(x) for x in (rot, sq, rs, rs2, rs3)])
    for a, b in zip(*outs):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("level,dnum", [(5, 3), (3, 3), (1, 3)], ids=["3digits", "2digits", "1digit"])
def test_rotsum_fp64_slot_set_groups(level, dnum):
    """rotsum4 / inner_fp own 4 slot sets per thread: G = 6 (a full group and a
    partial one), 21 premultiplied-key terms over two sources (folds of the
    exact double sums every 4 / 2 terms and of the c0 sum every 8), 1-3 digits,
    against the oracle at slot sets 0, 3, 4, 5; eager hoisted rotation and
    square + relinearise (inner_fp, identity and gathered) at the same G."""
    N, L = 1024, 5
    eng, orc, hp = _pair(N, L, 50, dnum=dnum, seed=9)
    from paper_2402_01296_b200.params import galois_element as ge
    rng = np.random.default_rng(61)
    G, check = 6, [0, 3, 4, 5]
    vs = [rng.standard_normal((G, N // 2)) * 0.5 for _ in range(2)]
    xs = [eng.encrypt(v, level=level, counter=700 + 20 * i) for i, v in enumerate(vs)]
    ocs = [{g: orc.encrypt(v[g], 700 + 20 * i + g, level) for g in check} for i, v in enumerate(vs)]
    Us = [eng.modup(x, level) for x in xs]
    ql = float(hp.q[level])
    taps = [(i, r) for i in range(2) for r in range(1, 11)] + [(0, 77)]
    vals = rng.standard_normal((len(taps), N // 2)) * 0.4
    terms = [(xs[i], Us[i], ge(r, N), eng.encode_ext(vals[k], level, ql)) for k, (i, r) in enumerate(taps)]
    got = eng.rotsum(terms, level, keys=[eng.premul_key(t[2], t[3], level) for t in terms])
    c = to_numpy_u64(got)
    for g in check:
        want = orc.rotsum([(ocs[i][g], r, vals[k]) for k, (i, r) in enumerate(taps)], level)
        np.testing.assert_array_equal(c[g, 0], want.c0)
        np.testing.assert_array_equal(c[g, 1], want.c1)
    rot = to_numpy_u64(eng.rotate(xs[0], 5, level))
    eng.keygen_relin()
    sq = to_numpy_u64(eng.mul_cc(xs[1], xs[1], level))
    for g in check:
        wr, ws = orc.rotate(ocs[0][g], 5), orc.mul_cc(ocs[1][g], ocs[1][g])
        np.testing.assert_array_equal(rot[g, 0], wr.c0)
        np.testing.assert_array_equal(rot[g, 1], wr.c1)
        np.testing.assert_array_equal(sq[g, 0], ws.c0)
        np.testing.assert_array_equal(sq[g, 1], ws.c1)


@pytest.mark.parametrize("N,L,dnum", [(8192, 7, 2), (16384, 7, 2)])
def test_single_special_prime_moddown_matches_oracle(N, L, dnum, monkeypatch):
    """K = 1 special prime (BASELINE config 3): the ModDown conversion is
    y mod q_t, read straight from the INTT'd special limb by the NTT's lift
    prologue.  Rotation and square+relinearise against the oracle, and
    against the base-conversion kernel path (BCN_K1_LIFT=0)."""
    outs = []
    for lift in ("1", "0"):
        monkeypatch.setenv("BCN_K1_LIFT", lift)
        hp = make_params(N, L, 50, dnum=dnum, n_special=1, seed=13)
        op = O.make_params(N, L, 50, dnum=dnum, n_special=1, seed=13)
        assert list(hp.q) == op.q and list(hp.p) == op.p and len(hp.p) == 1
        eng, orc = Engine(hp), O.Oracle(op)
        rng = np.random.default_rng(23)
        v, ct, oc = _enc2(eng, orc, N, rng)
        rot = eng.rotate(ct, 9, L)
        _assert_ct(rot, [orc.rotate(oc[i], 9) for i in range(2)])
        eng.keygen_relin()
        sq = eng.mul_cc(ct, ct, L)
        _assert_ct(sq, [orc.mul_cc(oc[i], oc[i]) for i in range(2)])
        outs.append([to_numpy_u64(rot), to_numpy_u64(sq)])
    for a, b in zip(*outs):
        np.testing.assert_array_equal(a, b)


# ------------------------------------------------- BASELINE configs 2 and 3 at their real shapes
def _worst_cases(basis, N, rng):
    qs = np.array(basis, dtype=np.uint64)[:, None]
    alt = np.where(np.arange(N) % 2 == 0, 0, 1).astype(np.uint64)[None] * (qs - np.uint64(1))
    spike = np.zeros((len(basis), N), np.uint64)
    spike[:, N // 3] = (qs[:, 0] - np.uint64(1))
    top = np.broadcast_to(qs - np.uint64(1), (len(basis), N))
    uni = np.stack([rng.integers(0, q, N, dtype=np.uint64) for q in basis])
    near = np.stack([q - np.uint64(1) - rng.integers(0, 4, N, dtype=np.uint64) for q in basis])
    return np.stack([top, alt, spike, uni, near])


@pytest.mark.parametrize("logn", [13, 14])
def test_ntt_60bit_cluster_matches_oracle(logn):
    """BASELINE config 2's NTT: ~60-bit primes (all >= 2^50, so the integer
    Shoup/Harvey butterflies of the cluster kernel, with lazy reduction up to
    4q < 2^62) at N = 8192 and 16384 -- worst-case residues (all q-1, q-1
    alternating with 0, a spike, near-q noise) and uniform ones, forward and
    inverse, bit for bit against the oracle."""
    N = 1 << logn
    eng, orc, hp = _pair(N, 3, 60, dnum=1)
    basis = list(hp.q) + list(hp.p)
    assert all(q >= (1 << 59) for q in basis)
    x = _worst_cases(basis, N, np.random.default_rng(logn))
    t = torch.from_numpy(x.view(np.int64).copy()).cuda()
    eng.ntt(t, 0)
    got = to_numpy_u64(t)
    exp = np.stack([O.ntt(x[i], basis) for i in range(len(x))])
    np.testing.assert_array_equal(got, exp)
    y = torch.from_numpy(exp.view(np.int64).copy()).cuda()
    eng.ntt(y, 0, inverse=True)
    np.testing.assert_array_equal(to_numpy_u64(y), x)


def test_config2_mac_matches_oracle():
    """BASELINE config 2's MAC at its real shape: N = 8192, 4 limbs of ~60-bit
    primes, Y_g = sum_{t<25} ct_{25g+t} (x) pt_{25g+t}; 60 ciphertexts -> groups
    of 25, 25 and a ragged last group of 10; all-(q-1) operands in one group."""
    N, limbs, n_ct, group = 8192, 4, 60, 25
    hp = make_params(N, limbs - 1, 60, dnum=1, n_special=1)
    eng = Engine(hp)
    q = list(hp.q)
    cts = eng.sample_uniform(n_ct * 2, limbs, 0, seed=1, id0=0).view(n_ct, 2, limbs, N)
    pts = eng.sample_uniform(n_ct, limbs, 0, seed=2, id0=0)
    qcol = torch.from_numpy((np.array(q, dtype=np.uint64) - np.uint64(1)).view(np.int64)).cuda()[:, None]
    cts[25:50] = qcol                                 # worst case: every operand q-1 in group 1
    pts[25:50] = qcol
    got = to_numpy_u64(eng.mac(cts, eng.to_montgomery(pts), group))
    c_np, p_np = to_numpy_u64(cts), to_numpy_u64(pts)
    assert got.shape == (3, 2, limbs, N)
    for g in range(3):
        for comp in range(2):
            acc = np.zeros((limbs, N), np.uint64)
            for k in range(g * group, min(n_ct, (g + 1) * group)):
                acc = O.add(acc, O.mul(c_np[k, comp], p_np[k], q), q)
            np.testing.assert_array_equal(got[g, comp], acc)


@pytest.mark.parametrize("fused_inner", ["0", "1"])
def test_config3_relin_no_rescale_and_rotation_match_oracle(fused_inner, monkeypatch):
    """BASELINE config 3 at its real shape: N = 16384, 8 limbs of 50-bit
    primes, K = 1 special prime, dnum = 2.  Stage A: ct x ct + relinearise
    WITHOUT rescale (mul_cc(rescale=False)); stage B: a hoisted rotation by
    +-2^k of the result -- both bit for bit against the oracle, with the q-limb
    inner products materialised (default) and inside the ModDown NTT's
    epilogue (BCN_FUSED_INNER=1)."""
    monkeypatch.setenv("BCN_FUSED_INNER", fused_inner)
    N, L = 16384, 7
    hp = make_params(N, L, 50, dnum=2, n_special=1, seed=5)
    op = O.make_params(N, L, 50, dnum=2, n_special=1, seed=5)
    assert list(hp.q) == op.q and list(hp.p) == op.p and hp.K == 1
    eng, orc = Engine(hp), O.Oracle(op)
    rng = np.random.default_rng(3)
    v = rng.standard_normal((2, N // 2)) * 0.5
    ct = eng.encrypt(v, counter=21)
    oc = [orc.encrypt(v[0], 21), orc.encrypt(v[1], 22)]
    sq = eng.mul_cc(ct, ct, L, rescale=False)
    osq = [orc.mul_cc(o, o, rescale=False) for o in oc]
    _assert_ct(sq, osq)
    U = eng.modup(sq, L)
    for r in (1, -64):
        _assert_ct(eng.rotate(sq, r, L, U=U), [orc.rotate(o, r) for o in osq])


@pytest.mark.parametrize("N,L,dnum,K,G,nrot", [(16384, 7, 2, 1, 3, 14), (8192, 5, 3, 2, 5, 18), (16384, 4, 3, 5, 66, 3)])
def test_rotate_many_matches_oracle_and_single_rotations(N, L, dnum, K, G, nrot, monkeypatch):
    """bcn_rotate_hoisted_many (source-shared inner products, one batched ModDown):
    config 3's 14 rotations by +-2^k at its real shape (K = 1, dnum = 2), more than 16
    rotations (two runs), ragged slot-set counts (G = 3, 5, 66: a partial warp quad and
    a second block of 64), K = 2 / 5 special primes (the split base conversion) -- bit
    for bit against one bcn_rotate_hoisted per rotation, against the oracle for the
    first slot sets, and against the fallback (BCN_ROT_MANY=0)."""
    hp = make_params(N, L, 50, dnum=dnum, n_special=K, seed=5)
    op = O.make_params(N, L, 50, dnum=dnum, n_special=K, seed=5)
    assert list(hp.q) == op.q and list(hp.p) == op.p and hp.K == K
    eng, orc = Engine(hp), O.Oracle(op)
    rng = np.random.default_rng(3)
    v = rng.standard_normal((G, N // 2)) * 0.5
    ct = eng.encrypt(v, counter=21)
    rots = [s * (1 << k) for k in range(7) for s in (1, -1)]
    rots = (rots + [3, 5, 7, N // 2 - 1])[:nrot]
    U = eng.modup(ct, L)
    got = eng.rotate_many(ct, rots, L, U=U)
    assert got.shape == (nrot, G, 2, L + 1, N)
    for k, r in enumerate(rots):
        assert torch.equal(got[k], eng.rotate(ct, r, L, U=U)), (k, r)
    n_or = 2 if N == 16384 and nrot > 3 else 1
    oc = [orc.encrypt(v[i], 21 + i) for i in range(n_or)]
    for k in (0, nrot - 1):
        _assert_ct(got[k][:n_or], [orc.rotate(o, rots[k]) for o in oc])
    monkeypatch.setenv("BCN_ROT_MANY", "0")
    assert torch.equal(got, eng.rotate_many(ct, rots, L, U=U))


def test_encryption_ids_are_partitioned_by_rank(monkeypatch):
    """Every rank derives the same keys from the shared seed, so two ranks must
    never draw the same Philox encryption randomness: rank r's ids start at
    1 + (r << 40).  Equal plaintexts on ranks 0 and 1 give different c1 (the
    uniform `a`) and both decrypt correctly."""
    from paper_2402_01296_b200.engine import counter_base

    N = 1024
    hp = make_params(N, 2, 40, dnum=1)
    v = np.random.default_rng(0).standard_normal((1, N // 2))
    cts = []
    for rank in (0, 1):
        monkeypatch.setenv("RANK", str(rank))
        eng = Engine(hp)
        assert eng._counter == counter_base(rank)
        ct = eng.encrypt(v)
        cts.append(to_numpy_u64(ct)[0])
        assert np.abs(eng.decrypt(ct, hp.max_level, hp.scale).cpu().numpy()[0] - v[0]).max() < 1e-6
    assert not np.array_equal(cts[0][1], cts[1][1])
    assert not np.array_equal(cts[0][0], cts[1][0])


def test_context_freeze_blocks_arena_moves():
    """bcn_ctx_freeze: while a captured graph holds a context, a call that would
    grow or free its scratch arena raises UsageError instead of moving memory."""
    from paper_2402_01296_b200.errors import UsageError

    eng, orc, hp = _pair(1024, 3, 40, dnum=2)
    rng = np.random.default_rng(0)
    ct = eng.encrypt(rng.standard_normal((1, 512)), counter=3)
    eng.mul_cc(ct, ct, hp.max_level)                    # sizes the arena for G = 1
    eng.freeze(+1)
    eng.mul_cc(ct, ct, hp.max_level)                    # fits: fine
    big = eng.encrypt(rng.standard_normal((64, 512)), counter=10)
    with pytest.raises(UsageError):
        eng.mul_cc(big, big, hp.max_level)              # would grow the arena
    with pytest.raises(UsageError):
        eng.trim()
    eng.freeze(-1)
    eng.mul_cc(big, big, hp.max_level)
    eng.trim()
