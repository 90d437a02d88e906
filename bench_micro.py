"""Primitive microbenchmarks (BASELINE configs 2 and 3) -- imported by bench.py.

Config 2: 4096 ciphertexts x 2 polys x 4 limbs (60-bit primes), N = 8192:
  forward NTT and INTT over all 32,768 limb-polys; MAC of ct_k (x) pt_k over
  groups of 25 consecutive pairs (164 outputs).
Config 3: 1024 ciphertexts, N = 16384, 8 limbs (50-bit), K = 1, dnum = 2:
  stage A square + relinearise (no rescale), stage B 14 rotations (+-2^k,
  k = 0..6) of every squared ciphertext, all outputs written.
Algorithmic bytes: inputs read once, outputs written once,
each distinct key read once per launch; twiddles excluded.
"""

from __future__ import annotations

import time

import torch

from paper_2402_01296_b200.engine import Engine
from paper_2402_01296_b200.params import make_params


def _events():
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def time_region(fn, steps: int, warmup: int) -> float:
    """Average ms per call, CUDA events on the current stream."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    s, e = _events()
    s.record()
    for _ in range(steps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / steps


def config2(steps=10, warmup=3, n_ct=4096, limbs=4, N=8192):
    hp = make_params(N, limbs - 1, 60, dnum=1, n_special=1)
    eng = Engine(hp)
    data = eng.sample_uniform(n_ct * 2, limbs, 0, seed=1, id0=0)          # (8192, 4, N)
    pts = eng.to_montgomery(eng.sample_uniform(n_ct, limbs, 0, seed=2, id0=0))
    words = data.numel()
    ntt_bytes = 2 * words * 8
    fwd_ms = time_region(lambda: eng.ntt(data, 0), steps, warmup)
    inv_ms = time_region(lambda: eng.ntt(data, 0, inverse=True), steps, warmup)
    cts = data.view(n_ct, 2, limbs, N)
    group = 25
    n_out = -(-n_ct // group)
    mac_bytes = (cts.numel() + pts.numel() + n_out * 2 * limbs * N) * 8
    mac_ms = time_region(lambda: eng.mac(cts, pts, group), steps, warmup)
    res = {
        "ntt": {"ms": fwd_ms, "bytes": ntt_bytes, "GBps": ntt_bytes / fwd_ms / 1e6},
        "intt": {"ms": inv_ms, "bytes": ntt_bytes, "GBps": ntt_bytes / inv_ms / 1e6},
        "mac": {"ms": mac_ms, "bytes": mac_bytes, "GBps": mac_bytes / mac_ms / 1e6},
        "limb_polys": words // N,
    }
    del eng, data, pts
    torch.cuda.empty_cache()
    return res


def config2_fused(steps=10, warmup=3, n_ct=4096, limbs=4, N=8192, group=25):
    """Config 2 as ONE pass (bcn_ntt_mac_rescale / bcn32_ntt_mac_rescale,
    SURVEY.md 8(f) item 2): coefficient-domain ciphertexts -> NTT -> (.) pt ->
    sum of 25 -> rescale, in u64 words (BASELINE's ~60-bit primes) and in the
    32-bit-limb variant (primes < 2^30).  Algorithmic bytes: every ciphertext
    and plaintext word read once, the rescaled outputs written once."""
    from paper_2402_01296_b200.limb32 import Engine32, primes32

    n_out = -(-n_ct // group)
    res = {}
    hp = make_params(N, limbs - 1, 60, dnum=1, n_special=1)
    eng = Engine(hp)
    cts = eng.sample_uniform(n_ct * 2, limbs, 0, seed=1, id0=0).view(n_ct, 2, limbs, N)
    pts = eng.to_montgomery(eng.sample_uniform(n_ct, limbs, 0, seed=2, id0=0))
    nbytes = (cts.numel() + pts.numel() + n_out * 2 * (limbs - 1) * N) * 8
    ms = time_region(lambda: eng.ntt_mac_rescale(cts, pts, group), steps, warmup)
    res["u64"] = {"ms": ms, "bytes": nbytes, "GBps": nbytes / ms / 1e6, "primes_bits": 60}
    del eng, cts, pts
    torch.cuda.empty_cache()
    e32 = Engine32(N, primes32(N, limbs))
    cts = e32.uniform((n_ct, 2, limbs, N), seed=1)
    pts = e32.to_montgomery(e32.uniform((n_ct, limbs, N), seed=2))
    nbytes = (cts.numel() + pts.numel() + n_out * 2 * (limbs - 1) * N) * 4
    ms = time_region(lambda: e32.ntt_mac_rescale(cts, pts, group), steps, warmup)
    res["u32"] = {"ms": ms, "bytes": nbytes, "GBps": nbytes / ms / 1e6, "primes_bits": 30}
    data = cts.view(n_ct * 2, limbs, N)
    nb = 2 * data.numel() * 4
    ms = time_region(lambda: e32.ntt(data), steps, warmup)
    res["u32_ntt"] = {"ms": ms, "bytes": nb, "GBps": nb / ms / 1e6}
    ms = time_region(lambda: e32.ntt(data, inverse=True), steps, warmup)
    res["u32_intt"] = {"ms": ms, "bytes": nb, "GBps": nb / ms / 1e6}
    del e32, cts, pts, data
    torch.cuda.empty_cache()
    return res


def ntt14(steps=10, warmup=3, npoly=128, limbs=12):
    """The workload's NTT: N = 2^14 cluster kernels (ntt_fwd_cluster<14,0,0> /
    ntt_inv_cluster<14>) over a ModDown-shaped batch of 128 polys x 12 limbs of
    cifar3's 50-bit primes; one launch each, in place."""
    hp = make_params(16384, 14, 50, dnum=3)
    eng = Engine(hp)
    data = eng.sample_uniform(npoly, limbs, 0, seed=1)
    nbytes = 2 * data.numel() * 8
    fwd_ms = time_region(lambda: eng.ntt(data, 0), steps, warmup)
    inv_ms = time_region(lambda: eng.ntt(data, 0, inverse=True), steps, warmup)
    res = {"fwd": {"ms": fwd_ms, "bytes": nbytes, "GBps": nbytes / fwd_ms / 1e6},
           "inv": {"ms": inv_ms, "bytes": nbytes, "GBps": nbytes / inv_ms / 1e6},
           "limb_polys": npoly * limbs}
    del eng, data
    torch.cuda.empty_cache()
    return res


def config3(steps=3, warmup=1, n_ct=1024, N=16384, limbs=8, batch=128, many=True):
    """Keyswitch microbench, processed in batches of `batch` ciphertexts."""
    hp = make_params(N, limbs - 1, 50, dnum=2, n_special=1)
    eng = Engine(hp)
    L = hp.max_level
    rots = [s * (1 << k) for k in range(7) for s in (1, -1)]
    eng.keygen_relin()
    from paper_2402_01296_b200.params import galois_element
    for r in rots:
        eng.keygen_galois(galois_element(r, N))
    cts = eng.sample_uniform(n_ct * 2, limbs, 0, seed=3).view(n_ct, 2, limbs, N)
    sq = torch.empty_like(cts)
    outs = torch.empty((len(rots), batch, 2, limbs, N), dtype=torch.int64, device=cts.device)
    ct_bytes = 2 * limbs * N * 8
    key_bytes = 2 * hp.dnum * (limbs + hp.K) * N * 8

    def stage_a():
        for b0 in range(0, n_ct, batch):
            eng.mul_cc(cts[b0:b0 + batch], cts[b0:b0 + batch], L, rescale=False, out=sq[b0:b0 + batch])

    def stage_b():
        for b0 in range(0, n_ct, batch):
            x = sq[b0:b0 + batch]
            U = eng.modup(x, L)
            if many:
                eng.rotate_many(x, rots, L, U=U, out=outs)
            else:
                for i, r in enumerate(rots):
                    eng.rotate(x, r, L, U=U, out=outs[i])

    a_ms = time_region(stage_a, steps, warmup)
    b_ms = time_region(stage_b, steps, warmup)
    a_bytes = n_ct * 2 * ct_bytes + key_bytes
    b_bytes = n_ct * (ct_bytes + len(rots) * ct_bytes) + len(rots) * key_bytes
    res = {
        "relin": {"ms": a_ms, "bytes": a_bytes, "GBps": a_bytes / a_ms / 1e6},
        "rotations": {"ms": b_ms, "bytes": b_bytes, "GBps": b_bytes / b_ms / 1e6},
    }
    del eng, cts, sq, outs
    torch.cuda.empty_cache()
    return res


if __name__ == "__main__":
    import json
    t0 = time.time()
    import sys
    if "fused" in sys.argv:
        print(json.dumps({"config2_fused": config2_fused()}, indent=1))
        raise SystemExit(0)
    print(json.dumps({"config2": config2()}, indent=1))
    print(json.dumps({"config3": config3()}, indent=1))
    print("wall", time.time() - t0)
