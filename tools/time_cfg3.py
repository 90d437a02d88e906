"""Config 3 (key-switch microbench) timing: the 14 hoisted rotations as one
bcn_rotate_hoisted_many call per batch against one bcn_rotate_hoisted per rotation."""
import os
import sys

sys.path.insert(0, os.getcwd())
import bench_micro

for many in (True, False, True):
    r = bench_micro.config3(many=many)
    print("many" if many else "separate", {k: round(v["ms"], 2) for k, v in r.items()}, flush=True)
