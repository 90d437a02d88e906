"""Experiment: the cfg4 forward (G = 128 slot sets, 4096 images) captured as one
CUDA graph (graphs.GraphedForward) vs eager; prints ms per forward and the
max logit error of the replay against reference_forward."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2402_01296_b200 as BCN  # noqa: E402
from paper_2402_01296_b200.archive import TensorArchive  # noqa: E402
from paper_2402_01296_b200.graphs import GraphedForward  # noqa: E402
from paper_2402_01296_b200.network import reference_forward  # noqa: E402

bundle, weights = bench.cifar3_weights()
sens, full = bench.rank_inputs("cfg4", 4096, 0, 1)
w = TensorArchive(weights)
ctx = BCN.make_context(1 << 14, BCN.required_levels(bundle) + 1, bench.SCALE)
dev = torch.device("cuda", 0)
inp = (torch.as_tensor(sens, device=dev), torch.as_tensor(full, device=dev))
for _ in range(2):
    BCN.forward_bicrypto(bundle.bi, inp, w, ctx, group_size=32).logits_ct.data
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(3):
    BCN.forward_bicrypto(bundle.bi, inp, w, ctx, group_size=32).logits_ct.data
e.record()
torch.cuda.synchronize()
print(f"eager {s.elapsed_time(e) / 3:.1f} ms/forward")
t0 = time.time()
g = GraphedForward(bundle.bi, w, ctx, tuple(inp[0].shape), tuple(inp[1].shape), strategy="bhw", group_size=32)
print(f"capture {time.time() - t0:.1f} s, mem {torch.cuda.max_memory_allocated() / 2**30:.1f} GiB")
out = g(*inp)
torch.cuda.synchronize()
s.record()
for _ in range(3):
    out = g(*inp)
e.record()
torch.cuda.synchronize()
print(f"graph {s.elapsed_time(e) / 3:.1f} ms/forward")
