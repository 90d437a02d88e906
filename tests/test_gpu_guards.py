"""Out-of-bounds write guards (the memcheck substitute: compute-sanitizer is
closed on this GPU pool, profiles/sanitizer_r02_closed.log).

Every output below is a view into the middle of a larger buffer whose
leading and trailing guard words hold a sentinel; after the call through
the C ABI, the guards must be untouched and the result must equal the same
call into a fresh tensor.  Covers the kernels with the riskiest indexing:
the cluster / DSMEM NTTs (N = 2^13, 2^14, fused ModDown tails), the
single-CTA NTTs, Mul_CC with the merged ModDown+rescale, hoisted rotation,
ModUp, the 32-bit-limb NTTs and both fused NTT->MAC->rescale kernels."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2402_01296_b200 import _lib  # noqa: E402
from paper_2402_01296_b200.engine import Engine  # noqa: E402
from paper_2402_01296_b200.limb32 import Engine32, primes32  # noqa: E402
from paper_2402_01296_b200.params import galois_element, make_params  # noqa: E402

SENT64 = -0x5A5A5A5A5A5A5A5B
SENT32 = -0x5A5A5A5B
GUARD = 4096


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _guarded(shape, dtype=torch.int64):
    n = int(np.prod(shape))
    sent = SENT64 if dtype == torch.int64 else SENT32
    buf = torch.full((n + 2 * GUARD,), sent, dtype=dtype, device="cuda")
    return buf, buf[GUARD:GUARD + n].view(shape)


def _check_guards(buf, dtype=torch.int64):
    sent = SENT64 if dtype == torch.int64 else SENT32
    torch.cuda.synchronize()
    assert bool((buf[:GUARD] == sent).all()), "write before the output buffer"
    assert bool((buf[-GUARD:] == sent).all()), "write past the output buffer"


@pytest.mark.parametrize("logn", [12, 13, 14])
def test_ntt_in_place_stays_in_bounds(logn):
    N = 1 << logn
    hp = make_params(N, 6, 50, dnum=3)
    eng = Engine(hp)
    x = eng.sample_uniform(5, 7, 0, seed=1)
    buf, view = _guarded(tuple(x.shape))
    view.copy_(x)
    for inv in (False, True):
        _lib.call("bcn_ntt_inv" if inv else "bcn_ntt_fwd", eng._h, view.data_ptr(), 5, 7, 0, _stream())
        _check_guards(buf)
    assert torch.equal(view, x)                      # forward then inverse is the identity


def test_mul_cc_rotate_modup_stay_in_bounds():
    N, L, G = 16384, 6, 3
    hp = make_params(N, L, 50, dnum=3)
    eng = Engine(hp)
    ct = eng.encrypt(np.random.default_rng(0).standard_normal((G, N // 2)) * 0.1, counter=5)
    eng.keygen_relin()
    ref = eng.mul_cc(ct, ct, L)
    buf, out = _guarded(tuple(ref.shape))
    _lib.call("bcn_mul_cc", eng._h, out.data_ptr(), ct.data_ptr(), ct.shape[2], ct.data_ptr(), ct.shape[2], G, L, 1,
              _stream())
    _check_guards(buf)
    assert torch.equal(out, ref)
    U = eng.modup(ct, L)
    ubuf, Ug = _guarded(tuple(U.shape))
    _lib.call("bcn_modup", eng._h, Ug.data_ptr(), ct.data_ptr(), ct.shape[2], G, L, _stream())
    _check_guards(ubuf)
    assert torch.equal(Ug, U)
    g = galois_element(7, N)
    eng.keygen_galois(g)
    ref = eng.rotate(ct, 7, L, U=U)
    rbuf, rout = _guarded(tuple(ref.shape))
    _lib.call("bcn_rotate_hoisted", eng._h, rout.data_ptr(), ct.data_ptr(), ct.shape[2], U.data_ptr(), G, L, g,
              _stream())
    _check_guards(rbuf)
    assert torch.equal(rout, ref)


def test_fused_ntt_mac_rescale_stays_in_bounds():
    N, limbs, n_items, group = 8192, 4, 53, 25
    hp = make_params(N, limbs - 1, 60, dnum=1, n_special=1)
    eng = Engine(hp)
    cts = eng.sample_uniform(n_items * 2, limbs, 0, seed=1).view(n_items, 2, limbs, N)
    pts = eng.to_montgomery(eng.sample_uniform(n_items, limbs, 0, seed=2))
    ref = eng.ntt_mac_rescale(cts, pts, group)
    buf, out = _guarded(tuple(ref.shape))
    _lib.call("bcn_ntt_mac_rescale", eng._h, out.data_ptr(), cts.data_ptr(), pts.data_ptr(), n_items, group, limbs,
              _stream())
    _check_guards(buf)
    assert torch.equal(out, ref)
    e32 = Engine32(N, primes32(N, limbs))
    c32 = e32.uniform((n_items, 2, limbs, N), seed=3)
    p32 = e32.to_montgomery(e32.uniform((n_items, limbs, N), seed=4))
    ref = e32.ntt_mac_rescale(c32, p32, group)
    buf, out = _guarded(tuple(ref.shape), torch.int32)
    _lib.call("bcn32_ntt_mac_rescale", e32._h, out.data_ptr(), c32.data_ptr(), p32.data_ptr(), n_items, group,
              _stream())
    _check_guards(buf, torch.int32)
    assert torch.equal(out, ref)
    x = e32.uniform((3, limbs, N), seed=5)
    buf, view = _guarded(tuple(x.shape), torch.int32)
    view.copy_(x)
    _lib.call("bcn32_ntt_fwd", e32._h, view.data_ptr(), 3, _stream())
    _lib.call("bcn32_ntt_inv", e32._h, view.data_ptr(), 3, _stream())
    _check_guards(buf, torch.int32)
    assert torch.equal(view, x)
