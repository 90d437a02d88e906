"""Config 1 single-image latency (bench.latency_cfg1: eager and CUDA-graph replay, host to host)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import bench

r = bench.latency_cfg1(reps=20)
print({k: (round(v * 1e3, 3) if k in ("value", "eager_value") else v) for k, v in r.items() if k in ("value", "eager_value", "max_abs_logit_err")})
