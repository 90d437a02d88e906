"""Log the shapes of the heavy engine calls of one cifar3 forward (G groups)."""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2402_01296_b200 as BCN  # noqa: E402
from paper_2402_01296_b200.archive import TensorArchive  # noqa: E402
from paper_2402_01296_b200.engine import Engine  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 4
log = collections.Counter()
for name in ("rotsum", "mac_terms", "mac_multi_planes", "modup", "rotate", "rescale", "mul_cc", "mac_terms_acc",
             "encode", "encode_ext", "encrypt", "rotsum_rescale", "conv_ks_mac", "add", "add_plain"):
    fn = getattr(Engine, name)

    def wrap(self, *a, _fn=fn, _name=name, **k):
        if _name == "rotsum":
            key = (len(a[0]), a[1], sum(t[3] is None for t in a[0]))
        elif _name in ("mac_terms", "mac_terms_acc"):
            key = (len(a[0] if _name == "mac_terms" else a[1]), a[1] if _name == "mac_terms" else a[2])
        elif _name == "mac_multi_planes":
            key = (len(a[0]), a[2], a[3])
        elif _name in ("encode", "encode_ext", "encrypt"):
            import traceback
            st = traceback.extract_stack(limit=6)
            key = (tuple(getattr(a[0], "shape", ())), "/".join(f"{f.name}" for f in st[-5:-1]))
        else:
            key = tuple(x for x in a[1:3] if isinstance(x, int))
        log[(_name,) + tuple(key)] += 1
        return _fn(self, *a, **k)
    setattr(Engine, name, wrap)

bundle, weights = bench.cifar3_weights()
sens, full = bench.rank_inputs("cfg4", 32 * G, 0, 1)
w = TensorArchive(weights)
ctx = BCN.make_context(1 << 14, BCN.required_levels(bundle) + 1, 2.0 ** 50)
dev = torch.device("cuda", 0)
inp = (torch.as_tensor(sens, device=dev), torch.as_tensor(full, device=dev))
BCN.forward_bicrypto(bundle.bi, inp, w, ctx, group_size=32).logits_ct.data
log.clear()
BCN.forward_bicrypto(bundle.bi, inp, w, ctx, group_size=32).logits_ct.data
torch.cuda.synchronize()
for k, v in sorted(log.items(), key=lambda kv: str(kv[0])):
    print(v, k)
