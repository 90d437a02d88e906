"""Throughput vs slot sets per device batch (G): images/s of steady-state
cifar3 forwards, and device memory high-water mark.  usage: g_sweep.py G..."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2402_01296_b200 as BCN  # noqa: E402
from paper_2402_01296_b200.archive import TensorArchive  # noqa: E402

for G in [int(a) for a in sys.argv[1:]]:
    bundle, weights = bench.cifar3_weights()
    sens, full = bench.rank_inputs("cfg4", 32 * G, 0, 1)
    w = TensorArchive(weights)
    ctx = BCN.make_context(1 << 14, BCN.required_levels(bundle) + 1, 2.0 ** 50)
    dev = torch.device("cuda", 0)
    inp = (torch.as_tensor(sens, device=dev), torch.as_tensor(full, device=dev))
    try:
        for k in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            BCN.forward_bicrypto(bundle.bi, inp, w, ctx, group_size=32).logits_ct.data
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        free, total = torch.cuda.mem_get_info()
        print(f"G={G}: {dt*1e3:.1f} ms, {32*G/dt:.0f} images/s, device used {(total-free)/2**30:.1f} GiB, "
              f"torch peak {torch.cuda.max_memory_allocated()/2**30:.1f} GiB", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"G={G}: failed: {e}", flush=True)
    del ctx, inp
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()
