"""the 32-bit-limb variant (primes < 2^30, Delta = 2^30,
the reference's default scale, pkg/src/bibranch/cli.py:66) and BASELINE
config 2 as ONE fused NTT -> MAC -> rescale pass, in both word widths -- bit
for bit against the oracle (oracle/ckks.py: ntt / intt / ntt_mac_rescale),
through the C ABI (bcn32_* and bcn_ntt_mac_rescale in include/bcn.h)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from oracle import ckks as O  # noqa: E402
from paper_2402_01296_b200.engine import Engine, to_numpy_u64  # noqa: E402
from paper_2402_01296_b200.errors import ParameterError  # noqa: E402
from paper_2402_01296_b200.limb32 import Engine32, from_numpy_u32, primes32, to_numpy_u32  # noqa: E402
from paper_2402_01296_b200.params import make_params  # noqa: E402


def _worst(primes, N, rng, n):
    """n limb-poly sets (n, L, N): all q-1, q-1/0 alternating, a spike, uniform, near q."""
    qs = np.array(primes, dtype=np.uint64)[:, None]
    L = len(primes)
    cases = [np.broadcast_to(qs - np.uint64(1), (L, N)),
             np.where(np.arange(N) % 2 == 0, 0, 1).astype(np.uint64)[None] * (qs - np.uint64(1)),
             np.zeros((L, N), np.uint64)]
    cases[2][:, N // 3] = qs[:, 0] - np.uint64(1)
    while len(cases) < n:
        if len(cases) % 2:
            cases.append(np.stack([rng.integers(0, q, N, dtype=np.uint64) for q in primes]))
        else:
            cases.append(np.stack([q - np.uint64(1) - rng.integers(0, 4, N, dtype=np.uint64) for q in primes]))
    return np.stack([np.array(c, dtype=np.uint64) for c in cases[:n]])


@pytest.mark.parametrize("logn", [10, 12, 13, 14])
def test_ntt32_matches_oracle(logn):
    N = 1 << logn
    primes = primes32(N, 4)
    assert all((1 << 29) < q < (1 << 30) for q in primes)
    eng = Engine32(N, primes)
    x = _worst(primes, N, np.random.default_rng(logn), 6)
    t = from_numpy_u32(x, eng.device)
    eng.ntt(t)
    exp = np.stack([O.ntt(x[i], primes) for i in range(len(x))])
    np.testing.assert_array_equal(to_numpy_u32(t).astype(np.uint64), exp)
    eng.ntt(t, inverse=True)
    np.testing.assert_array_equal(to_numpy_u32(t).astype(np.uint64), x)


def _fused_case(primes, N, n_items, seed, worst_group=None):
    rng = np.random.default_rng(seed)
    L = len(primes)
    cts = np.stack([np.stack([np.stack([rng.integers(0, q, N, dtype=np.uint64) for q in primes])
                              for _ in range(2)]) for _ in range(n_items)])
    pts = np.stack([np.stack([rng.integers(0, q, N, dtype=np.uint64) for q in primes]) for _ in range(n_items)])
    if worst_group is not None:
        g0, g1 = worst_group
        qm = (np.array(primes, dtype=np.uint64) - np.uint64(1))[:, None]
        cts[g0:g1] = np.broadcast_to(qm, (L, N))
        pts[g0:g1] = np.broadcast_to(qm, (L, N))
    return cts, pts


@pytest.mark.parametrize("logn,nlimb,n_items,group", [(13, 4, 60, 25), (10, 2, 7, 3), (11, 8, 9, 4), (14, 3, 5, 5)])
def test_ntt_mac_rescale32_matches_oracle(logn, nlimb, n_items, group):
    """32-bit words: ragged last group, one all-(q-1) group, cluster sizes
    4 .. 16 CTAs (2 components x nlimb), N = 2^10 .. 2^14."""
    N = 1 << logn
    primes = primes32(N, nlimb)
    eng = Engine32(N, primes)
    cts, pts = _fused_case(primes, N, n_items, logn, worst_group=(group, min(n_items, 2 * group)))
    ct_d = from_numpy_u32(cts, eng.device)
    pt_d = eng.to_montgomery(from_numpy_u32(pts, eng.device))
    got = to_numpy_u32(eng.ntt_mac_rescale(ct_d, pt_d, group)).astype(np.uint64)
    exp = O.ntt_mac_rescale(cts, pts, primes, group)
    assert got.shape == exp.shape == (-(-n_items // group), 2, nlimb - 1, N)
    np.testing.assert_array_equal(got, exp)


def test_ntt_mac_rescale64_config2_matches_oracle():
    """BASELINE config 2's own parameters in the fused pass: N = 8192, 4 limbs
    of ~60-bit primes, groups of 25 with a ragged last group of 10 and an
    all-(q-1) group."""
    N, limbs, n_items, group = 8192, 4, 60, 25
    hp = make_params(N, limbs - 1, 60, dnum=1, n_special=1)
    eng = Engine(hp)
    primes = list(hp.q)
    assert all(q > (1 << 59) for q in primes)
    cts, pts = _fused_case(primes, N, n_items, 5, worst_group=(25, 50))
    ct_d = torch.from_numpy(cts.view(np.int64).copy()).cuda()
    pt_d = torch.from_numpy(pts.view(np.int64).copy()).cuda().view(n_items, limbs, N)
    got = to_numpy_u64(eng.ntt_mac_rescale(ct_d, eng.to_montgomery(pt_d), group))
    np.testing.assert_array_equal(got, O.ntt_mac_rescale(cts, pts, primes, group))


def test_ntt_mac_rescale_equals_unfused_engine():
    """The fused u64 pass equals the engine's own three-launch form
    (bcn_ntt_fwd, bcn_mac, bcn_rescale) on the same data."""
    N, limbs, n_items, group = 8192, 4, 50, 25
    hp = make_params(N, limbs - 1, 60, dnum=1, n_special=1)
    eng = Engine(hp)
    cts = eng.sample_uniform(n_items * 2, limbs, 0, seed=1).view(n_items, 2, limbs, N)
    pts = eng.to_montgomery(eng.sample_uniform(n_items, limbs, 0, seed=2))
    fused = eng.ntt_mac_rescale(cts, pts, group)
    x = cts.clone()
    eng.ntt(x.view(n_items * 2, limbs, N), 0)
    acc = eng.mac(x, pts, group)
    ref = eng.rescale(acc, limbs - 1)
    np.testing.assert_array_equal(to_numpy_u64(fused), to_numpy_u64(ref))


def test_limb32_rejects_bad_primes():
    with pytest.raises(ParameterError):
        Engine32(8192, [(1 << 31) - 1, 40961])          # not < 2^30 / not 1 mod 2N
    with pytest.raises(ParameterError):
        primes32(8192, 4, bits=31)
