"""Tiny driver for ncu captures: runs the config-2 NTT/INTT/MAC once each
after a warm-up (usage: python tools/prof_kernels.py [ntt|ks])."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2402_01296_b200.engine import Engine
from paper_2402_01296_b200.params import make_params

what = sys.argv[1] if len(sys.argv) > 1 else "ntt"
if what == "ntt":
    hp = make_params(8192, 3, 60, dnum=1, n_special=1)
    eng = Engine(hp)
    data = eng.sample_uniform(8192, 4, 0, seed=1)
    pts = eng.to_montgomery(eng.sample_uniform(4096, 4, 0, seed=2))
    for _ in range(2):
        eng.ntt(data, 0)
        eng.ntt(data, 0, inverse=True)
        eng.mac(data.view(4096, 2, 4, 8192), pts, 25)
    torch.cuda.synchronize()
else:
    hp = make_params(16384, 7, 50, dnum=2, n_special=1)
    eng = Engine(hp)
    L = hp.max_level
    cts = eng.sample_uniform(256, 8, 0, seed=3).view(128, 2, 8, 16384)
    for _ in range(2):
        sq = eng.mul_cc(cts, cts, L, rescale=False)
        U = eng.modup(sq, L)
        eng.rotate(sq, 1, L, U=U)
    torch.cuda.synchronize()
print("done")
