"""Mul_CC (square + relinearise + merged ModDown/rescale) at cifar3 square1's shape: 16 channels x 128 slot sets,
as 16 calls of 128 vs one call of 2048 (channel-batched).  usage: python tools/time_square_batch.py [level]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_01296_b200.engine import Engine  # noqa: E402
from paper_2402_01296_b200.params import make_params  # noqa: E402

lvl = int(sys.argv[1]) if len(sys.argv) > 1 else 10
hp = make_params(16384, 14, 50, dnum=3)
eng = Engine(hp)
eng.keygen_relin()
C, G = 16, 128
big = eng.sample_uniform(C * G * 2, lvl + 1, 0, seed=5).view(C * G, 2, lvl + 1, 16384)


def t(fn, n=3):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


def per_channel():
    return [eng.mul_cc(big[c * G:(c + 1) * G], big[c * G:(c + 1) * G], lvl) for c in range(C)]


def batched(k):
    return [eng.mul_cc(big[c * G:(c + k) * G], big[c * G:(c + k) * G], lvl) for c in range(0, C, k)]


print(f"level {lvl}: 16 x 128: {t(per_channel):.2f} ms")
for k in (2, 4, 8, 16):
    print(f"  {C // k} x {k * G}: {t(lambda: batched(k)):.2f} ms")
