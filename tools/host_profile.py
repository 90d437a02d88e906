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
bundle, weights = bench.cifar3_weights()
sens, full = bench.rank_inputs("cfg4", 32 * G, 0, 1)
w = TensorArchive(weights)
ctx = BCN.make_context(1 << 14, BCN.required_levels(bundle) + 1, bench.SCALE)
dev = torch.device("cuda", 0)
inp = (torch.as_tensor(sens, device=dev), torch.as_tensor(full, device=dev))
for _ in range(2):
    BCN.forward_bicrypto(bundle.bi, inp, w, ctx, group_size=32).logits_ct.data
torch.cuda.synchronize()
# host timeline per layer scope (perf_counter at scope entry / exit)
from paper_2402_01296_b200 import sim as _sim  # noqa: E402
_stamps = []
_enter, _exit = _sim._Scope.__enter__, _sim._Scope.__exit__


def _e(self):
    _stamps.append((self.name, "in", time.perf_counter()))
    return _enter(self)


def _x(self, *a):
    r = _exit(self, *a)
    _stamps.append((self.name, "out", time.perf_counter()))
    return r


_sim._Scope.__enter__, _sim._Scope.__exit__ = _e, _x
torch.cuda.synchronize()
tt = time.perf_counter()
BCN.forward_bicrypto(bundle.bi, inp, w, ctx, group_size=32).logits_ct.data
th = time.perf_counter()
torch.cuda.synchronize()
print(f"host timeline: enqueue done at {1e3 * (th - tt):.1f} ms, GPU done at {1e3 * (time.perf_counter() - tt):.1f} ms")
last = {}
for name, kind, ts in _stamps:
    if kind == "in":
        last[name] = ts
    else:
        print(f"  {name:18s} host {1e3 * (last[name] - tt):7.1f} -> {1e3 * (ts - tt):7.1f} ms ({1e3 * (ts - last[name]):6.1f})")
_sim._Scope.__enter__, _sim._Scope.__exit__ = _enter, _exit
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
