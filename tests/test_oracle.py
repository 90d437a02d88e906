"""CPU pins of the RNS-CKKS oracle (oracle/): published known-answer vectors,
naive ground truths, and the reference's slot semantics.  No GPU needed."""

import numpy as np
import pytest

from oracle import ckks as O
from paper_2402_01296_b200 import params as P


# Random123 philox4x32-10 known-answer vectors (kat_vectors, Salmon et al.)
KAT = [
    ([0, 0, 0, 0], [0, 0], [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]),
    ([0xffffffff] * 4, [0xffffffff] * 2, [0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd]),
    ([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344], [0xa4093822, 0x299f31d0],
     [0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1]),
]


@pytest.mark.parametrize("ctr,key,out", KAT)
def test_philox_known_answers(ctr, key, out):
    assert O.philox4x32(ctr, key) == out


def test_primes_match_engine_params():
    for N, L, bits in [(8, 1, 30), (1024, 5, 40), (8192, 10, 50), (16384, 14, 50), (8192, 3, 60)]:
        hp = P.make_params(N, L, bits, dnum=3)
        op = O.make_params(N, L, bits, dnum=3)
        assert list(hp.q) == op.q and list(hp.p) == op.p
        for q in op.q + op.p:
            assert q % (2 * N) == 1 and q < (1 << 61) and O.is_prime(q)
        assert len(set(op.q + op.p)) == len(op.q + op.p)


def test_engine_fft_table_is_the_oracle_table():
    re, im = P.fft_table(512)
    ft = O.fft_tables(512)
    assert np.array_equal(re, ft.re) and np.array_equal(im, ft.im)


@pytest.mark.parametrize("N", [8, 16, 32])
def test_ntt_product_is_negacyclic_convolution(N):
    q = O.ntt_primes(40, 1, N)[0]
    rng = np.random.default_rng(N)
    a = rng.integers(0, q, N, dtype=np.uint64)
    b = rng.integers(0, q, N, dtype=np.uint64)
    c = O.intt(O.mul(O.ntt(a[None], [q]), O.ntt(b[None], [q]), [q]), [q])[0]
    assert np.array_equal(c, O.negacyclic_mul_naive(a, b, q))


def test_ntt_evaluation_order():
    N = 16
    q = O.ntt_primes(30, 1, N)[0]
    psi = O.tables(N, q).psi
    rng = np.random.default_rng(0)
    a = rng.integers(0, q, N, dtype=np.uint64)
    A = O.ntt(a[None], [q])[0]
    for k in range(N):
        e = 2 * int(format(k, "04b")[::-1], 2) + 1
        assert int(A[k]) == sum(int(a[j]) * pow(psi, e * j, q) for j in range(N)) % q


def test_automorphism_ntt_matches_coefficient_form():
    N = 64
    q = O.ntt_primes(40, 1, N)[0]
    rng = np.random.default_rng(1)
    a = rng.integers(0, q, N, dtype=np.uint64)
    for r in (1, 3, 17):
        g = O.galois_elt(r, N)
        coef = np.empty_like(a)
        O.lib().orc_automorph_coef(O._p(a), O._p(coef), N, g, q)
        assert np.array_equal(O.automorph_ntt(O.ntt(a[None], [q]), g)[0], O.ntt(coef[None], [q])[0])


def test_automorphism_maps_aligned_blocks_to_aligned_blocks():
    # the engine's inner-product kernel stages one source block per destination block
    from_ = O.automorph_ntt
    N = 4096
    idx = np.arange(N, dtype=np.uint64)
    for r in (1, 2, 100, 2047):
        perm = from_(idx[None], O.galois_elt(r, N))[0].astype(np.int64)
        for blk in (32, 256, 1024):
            src = perm.reshape(-1, blk) // blk
            assert (src == src[:, :1]).all()


def test_special_fft_matches_definition_and_roundtrips():
    N = 64
    ft = O.fft_tables(N)
    rng = np.random.default_rng(2)
    v = rng.standard_normal(N // 2)
    wr, wi = O.special_ifft(v, np.zeros(N // 2), ft)
    zeta = np.exp(1j * np.pi / N)
    z = [sum((wr[i] + 1j * wi[i]) * zeta ** (i * int(ft.rot[j])) for i in range(N // 2)) for j in range(N // 2)]
    assert np.abs(np.array(z) - v).max() < 1e-12
    coef = O.encode_coeffs(v, N, 2.0 ** 40)
    assert np.abs(O.decode_coeffs(coef.astype(np.float64), N, 2.0 ** 40) - v).max() < 1e-10


@pytest.fixture(scope="module")
def orc():
    return O.Oracle(O.make_params(64, 4, 40, dnum=2, seed=3))


def test_oracle_semantics_follow_reference_sim(orc):
    """sim.py:184-283 slot semantics: add, Mul_PC / Mul_CC with level-1,
    left rotation == np.roll(x, -r), right for r < 0 (test_sim.py:144-158)."""
    rng = np.random.default_rng(4)
    x, y = rng.standard_normal((2, 32))
    cx, cy = orc.encrypt(x, 1), orc.encrypt(y, 2)
    assert cx.level == 4
    tol = 1e-7
    assert np.abs(orc.decrypt(orc.add_cc(cx, cy))[:32] - (x + y)).max() < tol
    m = orc.mul_plain(cx, y)
    assert m.level == 3 and np.abs(orc.decrypt(m)[:32] - x * y).max() < tol
    s = orc.mul_cc(cx, cy)
    assert s.level == 3 and np.abs(orc.decrypt(s)[:32] - x * y).max() < tol
    for r in (1, -1, 5, 31, 32):
        assert np.abs(orc.decrypt(orc.rotate(cx, r))[:32] - np.roll(x, -r)).max() < tol
    assert np.abs(orc.decrypt(orc.rotate(cx, 0))[:32] - x).max() < tol


def test_oracle_fc_4_to_2_matches_reference_pin(orc):
    """pkg/tests/test_layers.py:78-88: x=[1,2,3,4], W=arange(8).reshape(4,2) ->
    [40, 50] through n1+n2-1 = 5 rotate-multiplies by generalised diagonals."""
    S = 32
    x = np.zeros(S)
    x[:4] = [1, 2, 3, 4]
    W = np.arange(8.0).reshape(4, 2)
    ct = orc.encrypt(x, 7)
    acc = None
    t = np.arange(2)
    for d in range(3, -2, -1):
        q = t + d
        ok = (q >= 0) & (q < 4)
        vec = np.zeros(S)
        vec[t[ok]] = W[q[ok], t[ok]]
        term = orc.rotate_mul(ct, d, vec)
        acc = term if acc is None else orc.add_cc(acc, term)
    assert acc.level == 3
    assert np.abs(orc.decrypt(acc)[:2] - np.array([40.0, 50.0])).max() < 1e-6


def test_merged_moddown_rescale_equals_separate_evaluation(orc):
    """rotsum_rescale (ONE base conversion from {q_l, P}) decrypts to the same
    slots as rescale(rotsum + ct terms) (ModDown, then rescale), to CKKS noise."""
    rng = np.random.default_rng(12)
    x, y, p1, p2, p3 = rng.standard_normal((5, 32))
    cx, cy = orc.encrypt(x, 21), orc.encrypt(y, 22)
    L = cx.level
    merged = orc.rotsum_rescale([(cx, 1, p1), (cy, 5, p2)], [(cy, p3)], L)
    assert merged.level == L - 1
    want = np.roll(x, -1) * p1 + np.roll(y, -5) * p2 + y * p3
    assert np.abs(orc.decrypt(merged)[:32] - want).max() < 1e-6
    sep = orc.add_cc(orc.add_cc(orc.rotate_mul(cx, 1, p1), orc.rotate_mul(cy, 5, p2)), orc.mul_plain(cy, p3))
    assert np.abs(orc.decrypt(merged)[:32] - orc.decrypt(sep)[:32]).max() < 1e-6


def test_hoisted_rotation_equals_fresh_modup(orc):
    rng = np.random.default_rng(5)
    ct = orc.encrypt(rng.standard_normal(32), 9)
    a = orc.rotate(ct, 3)
    orc.rotate(ct, 1, modup_key="k")
    b = orc.rotate(ct, 3, modup_key="k")
    assert np.array_equal(a.c0, b.c0) and np.array_equal(a.c1, b.c1)


def test_depth_exhaustion_is_exact():
    o = O.Oracle(O.make_params(16, 2, 30, dnum=1))
    ct = o.encrypt([1.5], 1)
    ct = o.mul_plain(o.mul_plain(ct, [1.0]), [1.0])
    assert ct.level == 0
    with pytest.raises(AssertionError):
        o.rescale(ct)


@pytest.mark.parametrize("N,L,dnum,K", [(16384, 14, 3, None), (8192, 10, 3, None), (16384, 7, 2, 1)])
def test_default_chains_are_fp64_eligible(N, L, dnum, K):
    """The default chains (q0 and the specials at max(50, scale_bits) bits) put
    every prime in (2^49, 2^50): the condition under which the engine runs
    the NTT, the base conversions and the Mul_CC tensor product on the FP64
    pipe (csrc/api.cu fp_conv).  Primes stay distinct and 1 mod 2N."""
    from paper_2402_01296_b200.params import make_params
    hp = make_params(N, L, 50, dnum=dnum, n_special=K)
    op = O.make_params(N, L, 50, dnum=dnum, n_special=K)
    basis = list(hp.q) + list(hp.p)
    assert basis == op.q + op.p
    assert len(set(basis)) == len(basis)
    assert all((1 << 49) < q < (1 << 50) and q % (2 * N) == 1 for q in basis)
    # a scale above 2^50 keeps q0 / specials at least as wide as the rescale primes
    wide = make_params(N, 4, 55, dnum=dnum)
    assert all(q.bit_length() == 55 for q in list(wide.q) + list(wide.p))


@pytest.mark.parametrize("bits,L", [(30, 3), (60, 4)])
def test_ntt_mac_rescale_restatement_is_the_coefficient_definition(bits, L):
    """Pin of oracle.ntt_mac_rescale (config 2, 8(f) item 2) against its
    definition in the coefficient domain with the schoolbook negacyclic
    product: Y = round((sum_t ct_t * p_t) / q_top) per limb, i.e.
    (c_i - centred(c_top)) q_top^-1 mod q_i -- for 30-bit (32-bit-limb
    variant) and 60-bit (config 2) primes, a ragged last group."""
    N, n, group = 16, 5, 2
    primes = O.ntt_primes(bits, L, N)
    rng = np.random.default_rng(bits)
    cts = np.stack([np.stack([np.stack([rng.integers(0, q, N, dtype=np.uint64) for q in primes])
                              for _ in range(2)]) for _ in range(n)])
    pc = np.stack([np.stack([rng.integers(0, q, N, dtype=np.uint64) for q in primes]) for _ in range(n)])
    pts = np.stack([O.ntt(pc[k], primes) for k in range(n)])
    got = O.ntt_mac_rescale(cts, pts, primes, group)
    qt = primes[-1]
    for g, g0 in enumerate(range(0, n, group)):
        for comp in range(2):
            acc = [[0] * N for _ in primes]
            for k in range(g0, min(n, g0 + group)):
                for i, q in enumerate(primes):
                    prod = O.negacyclic_mul_naive(cts[k, comp, i], pc[k, i], q)
                    acc[i] = [(a + int(b)) % q for a, b in zip(acc[i], prod)]
            top = [v - qt if v > qt // 2 else v for v in acc[-1]]
            want = np.stack([np.array([((acc[i][j] - top[j]) * pow(qt, -1, q)) % q for j in range(N)],
                                      dtype=np.uint64) for i, q in enumerate(primes[:-1])])
            np.testing.assert_array_equal(O.intt(got[g, comp], primes[:-1]), want)
