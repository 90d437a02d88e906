"""cProfile of the host side of one cifar3 forward (G groups): where the
Python drop-in layer spends time while the GPU runs."""
import cProfile
import io
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2402_01296_b200 as BCN  # noqa: E402
from paper_2402_01296_b200.archive import TensorArchive  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 32
bundle, weights, sens, full = bench.cifar3_setup(32 * G)
w = TensorArchive(weights)
ctx = BCN.make_context(1 << 14, BCN.required_levels(bundle) + 1, 2.0 ** 50)
dev = torch.device("cuda", 0)
inp = (torch.as_tensor(sens, device=dev), torch.as_tensor(full, device=dev))
for _ in range(2):
    BCN.forward_bicrypto(bundle.bi, inp, w, ctx, group_size=32).logits_ct.data
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
BCN.forward_bicrypto(bundle.bi, inp, w, ctx, group_size=32).logits_ct.data
pr.disable()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue {1e3*(t1-t0):.1f} ms, until GPU done {1e3*(t2-t0):.1f} ms")
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25)
print(s.getvalue()[:6000])
