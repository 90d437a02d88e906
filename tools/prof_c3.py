"""Config 3 (key switching) for ncu: keys generated and one warm-up pass
outside the NVTX range; then exactly one batch of 128 ciphertexts of stage A
(square + relinearise, no rescale) inside range "c3A/" and of stage B (ModUp
+ 14 hoisted rotations) inside "c3B/".  Use with
  ncu --nvtx --nvtx-include c3A/ --nvtx-include c3B/ ...
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2402_01296_b200.engine import Engine  # noqa: E402
from paper_2402_01296_b200.params import galois_element, make_params  # noqa: E402

N, limbs, batch = 16384, 8, 128
hp = make_params(N, limbs - 1, 50, dnum=2, n_special=1)
eng = Engine(hp)
L = hp.max_level
rots = [s * (1 << k) for k in range(7) for s in (1, -1)]
eng.keygen_relin()
for r in rots:
    eng.keygen_galois(galois_element(r, N))
cts = eng.sample_uniform(batch * 2, limbs, 0, seed=3).view(batch, 2, limbs, N)
sq = torch.empty_like(cts)
outs = torch.empty((len(rots), batch, 2, limbs, N), dtype=torch.int64, device=cts.device)


def stage_a():
    eng.mul_cc(cts, cts, L, rescale=False, out=sq)


def stage_b():
    U = eng.modup(sq, L)
    for i, r in enumerate(rots):
        eng.rotate(sq, r, L, U=U, out=outs[i])


stage_a()
stage_b()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("c3A")
stage_a()
torch.cuda.nvtx.range_pop()
torch.cuda.nvtx.range_push("c3B")
stage_b()
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("ok")
