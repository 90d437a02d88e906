"""Probe: do two independent cifar3 forwards (own context, own CUDA stream,
own host thread) overlap on one GPU?  Compares one forward of 2G slot sets
with two concurrent forwards of G.  usage: python tools/two_stream_probe.py [G]"""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2402_01296_b200 as BCN  # noqa: E402
from paper_2402_01296_b200.archive import TensorArchive  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 64
bundle, weights = bench.cifar3_weights()
sens, full = bench.rank_inputs("cfg4", 32 * 2 * G, 0, 1)
w = TensorArchive(weights)
dev = torch.device("cuda", 0)
inp_all = (torch.as_tensor(sens, device=dev), torch.as_tensor(full, device=dev))
halves = [(inp_all[0][i * 32 * G:(i + 1) * 32 * G], inp_all[1][i * 32 * G:(i + 1) * 32 * G]) for i in range(2)]


def fwd(ctx, inp):
    return BCN.forward_bicrypto(bundle.bi, inp, w, ctx, group_size=32).logits_ct.data


ctx0 = BCN.make_context(1 << 14, BCN.required_levels(bundle) + 1, 2.0 ** 50)
for _ in range(2):
    fwd(ctx0, inp_all)
torch.cuda.synchronize()
t0 = time.perf_counter()
fwd(ctx0, inp_all)
torch.cuda.synchronize()
one = time.perf_counter() - t0
print(f"one context, {2 * G} slot sets: {one * 1e3:.1f} ms")
del ctx0
torch.cuda.empty_cache()

ctxs = [BCN.make_context(1 << 14, BCN.required_levels(bundle) + 1, 2.0 ** 50) for _ in range(2)]
streams = [torch.cuda.Stream() for _ in range(2)]


def worker(i, reps):
    with torch.cuda.stream(streams[i]):
        for _ in range(reps):
            fwd(ctxs[i], halves[i])
    streams[i].synchronize()


for i in range(2):
    worker(i, 2)
torch.cuda.synchronize()
t0 = time.perf_counter()
th = [threading.Thread(target=worker, args=(i, 1)) for i in range(2)]
for t in th:
    t.start()
for t in th:
    t.join()
torch.cuda.synchronize()
two = time.perf_counter() - t0
print(f"two contexts x {G} slot sets, concurrent streams: {two * 1e3:.1f} ms  ({one / two:.3f}x)")
t0 = time.perf_counter()
for i in range(2):
    worker(i, 1)
torch.cuda.synchronize()
print(f"two contexts x {G} slot sets, back to back: {(time.perf_counter() - t0) * 1e3:.1f} ms")
