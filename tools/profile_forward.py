"""Per-kernel time breakdown of one cifar3 forward (torch.profiler / CUPTI;
nsys is not installed).  usage: python tools/profile_forward.py [groups]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
import paper_2402_01296_b200 as BCN  # noqa: E402
from paper_2402_01296_b200.archive import TensorArchive  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 8
bundle, weights = bench.cifar3_weights()
sens, full = bench.rank_inputs("cfg4", 32 * G, 0, 1)
w = TensorArchive(weights)
ctx = BCN.make_context(1 << 14, BCN.required_levels(bundle) + 1, 2.0 ** 50)
dev = torch.device("cuda", 0)
inp = (torch.as_tensor(sens, device=dev), torch.as_tensor(full, device=dev))
BCN.forward_bicrypto(bundle.bi, inp, w, ctx, group_size=32).logits_ct.data
torch.cuda.synchronize()
t0 = time.perf_counter()
BCN.forward_bicrypto(bundle.bi, inp, w, ctx, group_size=32).logits_ct.data
torch.cuda.synchronize()
wall = time.perf_counter() - t0
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    BCN.forward_bicrypto(bundle.bi, inp, w, ctx, group_size=32).logits_ct.data
    torch.cuda.synchronize()
ev = prof.key_averages()
rows = sorted([e for e in ev if e.device_time_total > 0], key=lambda e: -e.device_time_total)
tot = sum(e.device_time_total for e in rows if e.device_type.name == "CUDA" or True)
gpu_total = sum(e.self_device_time_total for e in ev)
print(f"G={G} wall {wall*1e3:.1f} ms; summed kernel time {gpu_total/1e3:.1f} ms")
for e in sorted(ev, key=lambda e: -e.self_device_time_total)[:25]:
    if e.self_device_time_total <= 0:
        continue
    print(f"{e.self_device_time_total/1e3:9.2f} ms {100*e.self_device_time_total/gpu_total:5.1f}%  n={e.count:6d}  {e.key[:90]}")
