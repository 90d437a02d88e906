"""One launch each of the config-2 fused pass (u32, u64) and the 32-bit NTT
at full size -- the target of `ncu --set full` captures (profiles/)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2402_01296_b200.engine import Engine  # noqa: E402
from paper_2402_01296_b200.limb32 import Engine32, primes32  # noqa: E402
from paper_2402_01296_b200.params import make_params  # noqa: E402

N, L, n, group = 8192, 4, 4096, 25
what = sys.argv[1] if len(sys.argv) > 1 else "all"
if what in ("all", "u32"):
    e = Engine32(N, primes32(N, L))
    cts = e.uniform((n, 2, L, N), seed=1)
    pts = e.to_montgomery(e.uniform((n, L, N), seed=2))
    e.ntt_mac_rescale(cts, pts, group)
    e.ntt(cts.view(2 * n, L, N))
    torch.cuda.synchronize()
    del cts, pts
if what in ("all", "u64"):
    hp = make_params(N, L - 1, 60, dnum=1, n_special=1)
    eng = Engine(hp)
    cts = eng.sample_uniform(n * 2, L, 0, seed=1).view(n, 2, L, N)
    pts = eng.to_montgomery(eng.sample_uniform(n, L, 0, seed=2))
    eng.ntt_mac_rescale(cts, pts, group)
    torch.cuda.synchronize()
print("ok")
