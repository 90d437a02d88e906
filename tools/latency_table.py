"""Measured per-op latency table for the reference's cost model (SURVEY
8(f) item 4): writes {scheme: {op: ms}} in the format of the reference's
BIBRANCH_LATENCY_TABLE override (costs.py:22-47), from CUDA-event timings of
the engine's ops at config-4 parameters (N = 2^14, level 10, Delta = 2^50):

  CKKS_B200          one ciphertext per call (latency)
  CKKS_B200_G128     per ciphertext, amortised over a batch of 128 slot sets

Add_PC = encode + add (the plaintext is input dependent); Mul_PC = Montgomery
multiply + rescale with a cached plaintext; Mul_CC = tensor + relinearisation
+ rescale; Rot = hoisted rotation (ModUp + key switch).
usage: python tools/latency_table.py [out.json]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2402_01296_b200.engine import Engine  # noqa: E402
from paper_2402_01296_b200.params import galois_element, make_params  # noqa: E402


def ms(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def table(eng, hp, G, level=10):
    rng = np.random.default_rng(0)
    S = hp.N // 2
    vals = rng.standard_normal((G, S)) * 0.1
    ct = eng.encrypt(vals, level=level)
    ql = float(hp.q[level])
    pt_m = eng.encode(vals[:1], level, ql, montgomery=True)
    g = galois_element(1, hp.N)
    eng.keygen_galois(g)
    eng.keygen_relin()
    t = {
        "Add_CC": ms(lambda: eng.add(ct, ct, level)),
        "Add_PC": ms(lambda: eng.add_plain(ct, eng.encode(vals, level, hp.scale), level)),
        "Mul_PC": ms(lambda: eng.mul_plain(ct, pt_m, level)),
        "Mul_CC": ms(lambda: eng.mul_cc(ct, ct, level)),
        "Rot": ms(lambda: eng.rotate(ct, 1, level)),
    }
    return {k: v / G for k, v in t.items()}


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join("profiles", "latency_table_b200.json")
    hp = make_params(1 << 14, 14, 50, dnum=3)
    eng = Engine(hp)
    res = {"CKKS_B200": table(eng, hp, 1), "CKKS_B200_G128": table(eng, hp, 128)}
    res["_note"] = ("ms per ciphertext op on one B200, N=2^14, level 10 (11 limbs), Delta=2^50, dnum=3, K=5; "
                    "CUDA events, 20 reps; use with BIBRANCH_LATENCY_TABLE=<this file> and scheme "
                    "CKKS_B200 (latency) or CKKS_B200_G128 (batched throughput)")
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
