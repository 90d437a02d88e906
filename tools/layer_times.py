"""Device time per layer scope of one cifar3 forward (BASELINE config 4) at
the bench's device batch (G slot sets, default 128 = 4096 images), from the
OpRecorder's optional CUDA-event timing (sim.OpRecorder.enable_timing).
usage: python tools/layer_times.py [G]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2402_01296_b200 as BCN  # noqa: E402
from paper_2402_01296_b200.archive import TensorArchive  # noqa: E402
from paper_2402_01296_b200.sim import OpRecorder  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 128
bundle, weights = bench.cifar3_weights()
sens, full = bench.rank_inputs("cfg4", 32 * G, 0, 1)
w = TensorArchive(weights)
dnum = int(os.environ["BCN_DNUM"]) if os.environ.get("BCN_DNUM") else None   # A/B of the key-switch digits
ctx = BCN.make_context(1 << 14, BCN.required_levels(bundle) + 1, bench.SCALE, dnum=dnum)
dev = torch.device("cuda", 0)
inp = (torch.as_tensor(sens, device=dev), torch.as_tensor(full, device=dev))
for _ in range(2):
    BCN.forward_bicrypto(bundle.bi, inp, w, ctx, group_size=32).logits_ct.data
torch.cuda.synchronize()
rec = OpRecorder()
rec.enable_timing()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
res = BCN.forward_bicrypto(bundle.bi, inp, w, ctx, group_size=32, rec=rec)
res.logits_ct.data
e.record()
torch.cuda.synchronize()
total = s.elapsed_time(e)
print(f"G={G}: forward {total:.1f} ms")
acc = 0.0
for name, ms in rec.layer_times():
    acc += ms
    print(f"  {ms:8.2f} ms {100 * ms / total:5.1f}%  {name}")
print(f"  {total - acc:8.2f} ms outside scopes (incl. lazy tails run at .data)")
