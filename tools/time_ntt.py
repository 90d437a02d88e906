"""Timing probe for NTT variants: plain forward / inverse at N = 2^14 over a
ModDown-shaped batch, and one cifar3 forward at G groups of 32 images.
usage: python tools/time_ntt.py [groups]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2402_01296_b200.engine import Engine  # noqa: E402
from paper_2402_01296_b200.params import make_params  # noqa: E402


def cuda_ms(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


hp = make_params(16384, 14, 50, dnum=3)
eng = Engine(hp)
data = eng.sample_uniform(128, 12, 0, seed=1)
n = 128 * 12
f = cuda_ms(lambda: eng.ntt(data, 0))
i = cuda_ms(lambda: eng.ntt(data, 0, inverse=True))
print(f"ntt14 fwd {f*1e3/n:.3f} us/limb-poly  inv {i*1e3/n:.3f} us/limb-poly  "
      f"(fwd {2*8*16384*n/f/1e6:.0f} GB/s)")
G = int(sys.argv[1]) if len(sys.argv) > 1 else 32
import bench  # noqa: E402
import paper_2402_01296_b200 as BCN  # noqa: E402
from paper_2402_01296_b200.archive import TensorArchive  # noqa: E402
bundle, weights = bench.cifar3_weights()
sens, full = bench.rank_inputs("cfg4", 32 * G, 0, 1)
w = TensorArchive(weights)
ctx = BCN.make_context(1 << 14, BCN.required_levels(bundle) + 1, 2.0 ** 50)
dev = torch.device("cuda", 0)
inp = (torch.as_tensor(sens, device=dev), torch.as_tensor(full, device=dev))
for k in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    BCN.forward_bicrypto(bundle.bi, inp, w, ctx, group_size=32).logits_ct.data
    torch.cuda.synchronize()
    print(f"cifar3 forward G={G}: {(time.perf_counter()-t0)*1e3:.1f} ms")
