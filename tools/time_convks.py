"""A/B timing of the conv layer with lazy ModDown on the tensor cores
(bcn_conv_ks_mac: slot_major_ks + mac_umma + merged ModDown/rescale tails)
at cifar3 conv2's shape: 16 sources x 9 taps = 144 terms, 32 outputs,
level 11, G slot sets (default 128); conv1: PROF_SRC=3 PROF_OUT=16 PROF_LVL=14.  Prints ms per call (CUDA events)."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2402_01296_b200 import _lib  # noqa: E402
from paper_2402_01296_b200.engine import Engine  # noqa: E402
from paper_2402_01296_b200.params import galois_element as ge, make_params  # noqa: E402

G = int(os.environ.get("PROF_G", "128"))
hp = make_params(16384, 14, 50, dnum=3)
eng = Engine(hp)
lvl, O = int(os.environ.get("PROF_LVL", "11")), int(os.environ.get("PROF_OUT", "32"))   # conv1: 14, 16, 3 sources
nsrc = int(os.environ.get("PROF_SRC", "16"))
srcs = [eng.sample_uniform(2 * G, lvl + 1, 0, seed=9 + i).view(G, 2, lvl + 1, 16384) for i in range(nsrc)]
Us = [eng.modup(x, lvl) for x in srcs]
rots = [0, 1, 2, 16, 17, 18, 32, 33, 34]
if os.environ.get("PROF_ROTS"):   # packed conv2 (current): PROF_LVL=8 PROF_OUT=8 PROF_ROTS=16
    rots = [(i // 4) * 16 + (i % 4) for i in range(int(os.environ["PROF_ROTS"]))]
terms = [(srcs[c], Us[c], ge(r, 16384) if r else 1) for c in range(nsrc) for r in rots]
nb = ctypes.c_uint64()
_lib.call("bcn_planes_ext_bytes", eng._h, O, len(terms), lvl, ctypes.byref(nb))
planes = torch.randint(0, 256, (int(nb.value),), dtype=torch.uint8, device="cuda")


def run():
    return eng.conv_ks_mac([t[0] for t in terms], [t[1] if t[2] != 1 else None for t in terms],
                           [t[2] for t in terms], planes, O, lvl, 1)


out = run()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
REPS = int(os.environ.get("PROF_REPS", "3"))
for _ in range(REPS):
    out = run()
e.record()
torch.cuda.synchronize()
print(f"{os.environ.get('BCN_LIB', 'default')}: conv_ks_mac G={G} {s.elapsed_time(e) / max(REPS, 1):.3f} ms "
      f"checksum {int(out.view(-1)[::9973].sum())}")
