"""Config 1: where a graph-replayed request's wall time goes -- device time of the replay alone
(CUDA events) against the host-to-host time of GraphedForward.__call__."""
import os
import sys
import time
import statistics

sys.path.insert(0, os.getcwd())
import torch

import paper_2402_01296_b200 as BCN
import synthetic
from paper_2402_01296_b200.archive import TensorArchive
from paper_2402_01296_b200.graphs import GraphedForward

bundle = BCN.get("cnn3")
w = TensorArchive(synthetic.weights_for(synthetic.tensor_shapes(bundle), 0.1, seed=1))
sens, full = synthetic.cfg1_inputs(1, seed=0)
ctx = BCN.make_context(8192, BCN.required_levels(bundle) + 1, 2.0 ** 50)
gf = GraphedForward(bundle.bi, w, ctx, sens.shape, full.shape, strategy="hw")
sens_h = torch.as_tensor(sens).pin_memory()
full_h = torch.as_tensor(full).pin_memory()
for _ in range(5):
    gf(sens_h, full_h)
wall, dev = [], []
for _ in range(30):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    gf(sens_h, full_h)
    wall.append(time.perf_counter() - t0)
for _ in range(30):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    gf.graph.replay()
    b.record()
    torch.cuda.synchronize()
    dev.append(a.elapsed_time(b))
print({"wall_ms": round(statistics.median(wall) * 1e3, 3), "replay_device_ms": round(statistics.median(dev), 3)})
gf.close()
