"""One batch (128 ciphertexts) of config 3's 14 hoisted rotations through
bcn_rotate_hoisted_many, for an ncu launch list (tools: ncu --metrics gpu__time_duration.sum)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch
from paper_2402_01296_b200.engine import Engine
from paper_2402_01296_b200.params import make_params, galois_element

N, limbs, batch = 16384, 8, int(os.environ.get("CFG3_BATCH", "128"))
hp = make_params(N, limbs - 1, 50, dnum=2, n_special=1)
eng = Engine(hp)
L = hp.max_level
rots = [s * (1 << k) for k in range(7) for s in (1, -1)]
for r in rots:
    eng.keygen_galois(galois_element(r, N))
x = eng.sample_uniform(batch * 2, limbs, 0, seed=3).view(batch, 2, limbs, N)
outs = torch.empty((len(rots), batch, 2, limbs, N), dtype=torch.int64, device=x.device)
for it in range(3):
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("cfg3_batch")
    U = eng.modup(x, L)
    eng.rotate_many(x, rots, L, U=U, out=outs)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
print("done")
