"""Reference arm: the UNMODIFIED reference `forward_bicrypto`, timed on the
host cores -- TEST / BASELINE INFRASTRUCTURE ONLY (bench.py's `--impl
reference` arm and cpu_baseline leg, tests/).  The product never imports it.

The reference (pkg/src/bibranch, staged into oracle/_ref by
oracle/build_ref.sh) is a float64 *simulator* of CKKS semantics with no
cryptography (sim.py:1-12): this arm is "reference simulator, no
cryptography", timed exactly as the reference's own harness times a forward
(pkg/benchmarks/bench_slotops.py:68-96: one process per backend, perf_counter
around `forward_bicrypto`), made process-parallel over independent BHW slot
sets of 32 images (`multiprocessing.Pool(n_cores)`, one
thread per worker).

Workload: BASELINE config 4 -- the cifar3 bi-network declared with the
reference's own classes (layers.LayerSpec, network.NetworkSpec,
ConnectionSpec, IntegrationSpec), N = 2^14 (8192 slots = 32 x 16 x 16),
max_level = required_levels + 1 = 14 (catalog.py:286-346), the same seeded
synthetic images and N(0, 0.05) weights as the GPU arm (synthetic.py).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")
IMAGES_PER_SET = 32

_ST: dict = {}


def available() -> bool:
    return os.path.isfile(os.path.join(REF_DIR, "bibranch", "__init__.py"))


def load(backend: str = "python"):
    """Import the staged reference with a fixed slot-kernel backend
    (BIBRANCH_BACKEND is read once at import, backend.py:12-22)."""
    if not available():
        raise RuntimeError("oracle/_ref is missing: run oracle/build_ref.sh where /root/reference exists")
    os.environ["BIBRANCH_BACKEND"] = backend
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import bibranch as R
    return R


def cifar3_net(R):
    """BASELINE config-4 network in the reference's own classes:
    cipher conv3x3 p1 3->16, x^2, conv3x3 s2 p1 16->32, x^2, avgpool 2x2/2;
    the plain branch mirrors it with ReLU; connections after each conv
    activation; head n1 = 20, n2 = 10 (network.py:49-68, 304-343)."""
    from bibranch.layers import LayerSpec
    from bibranch.network import ConnectionSpec, IntegrationSpec, NetworkSpec

    def conv(prefix, cin, cout, stride):
        return LayerSpec("conv", kernel=(3, 3), stride=stride, padding=(1, 1), in_channels=cin, out_channels=cout,
                         weight=f"{prefix}.weight", bias=f"{prefix}.bias")

    def branch(prefix, act):
        return (conv(f"{prefix}conv1", 3, 16, (1, 1)), LayerSpec(act), conv(f"{prefix}conv2", 16, 32, (2, 2)),
                LayerSpec(act), LayerSpec("sumpool", kernel=(2, 2), stride=(2, 2), scale=0.25))

    head = IntegrationSpec(n1=20, n2=10, w_c1="head.w_c1", w_p1="head.w_p1", w_p1_prime="head.w_p1_prime",
                           b1="head.b1", b1_prime="head.b1_prime", w_c2="head.w_c2", w_p2="head.w_p2", b2="head.b2")
    return NetworkSpec("cifar3", (3, 32, 32), (3, 16, 16), branch("cipher.", "square"), branch("plain.", "relu"),
                       (ConnectionSpec(1, 2, "connect.1.w_crot"), ConnectionSpec(3, 4, "connect.2.w_crot")), head)


def setup(weights: dict, sens: np.ndarray, full: np.ndarray, backend: str = "python") -> None:
    """Build the reference objects once in the parent; forked workers inherit them."""
    R = load(backend)
    from bibranch.archive import TensorArchive
    net = cifar3_net(R)
    ctx = R.make_context(1 << 14, R.required_levels(net) + 1, 2.0 ** 30)
    _ST.update(R=R, net=net, w=TensorArchive(dict(weights)), ctx=ctx, sens=sens, full=full)


def _worker_init() -> None:
    for v in ("OMP_NUM_THREADS", "MKL_NUM_THREADS", "OPENBLAS_NUM_THREADS"):
        os.environ[v] = "1"
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except ImportError:   # pragma: no cover
        pass


def group_forward(g: int) -> np.ndarray:
    """One BHW slot set (32 images) through the reference's forward_bicrypto
    (network.py:388-448) and ForwardResult.decrypt_logits (network.py:363-368)."""
    R = _ST["R"]
    from bibranch.network import DecomposedInput
    n = _ST["sens"].shape[0]
    idx = [(g * IMAGES_PER_SET + i) % n for i in range(IMAGES_PER_SET)]
    dec = [DecomposedInput(_ST["sens"][i], _ST["full"][i], (0, 0, 16, 16)) for i in idx]
    res = R.forward_bicrypto(_ST["net"], dec, _ST["w"], _ST["ctx"], strategy="bhw")
    return res.decrypt_logits()


def time_forward(cores: int, steps: int, warmup: int) -> dict:
    """Each step: `cores` independent slot sets, one per worker process
    (fork; no CUDA in this process tree).  Returns wall-clock seconds per step."""
    import multiprocessing as mp

    per_step = []
    logits = None
    with mp.get_context("fork").Pool(cores, initializer=_worker_init) as pool:
        pool.map(group_forward, range(cores))          # import / first-touch, not counted as a step
        for i in range(warmup + steps):
            t0 = time.perf_counter()
            out = pool.map(group_forward, range(i * cores, (i + 1) * cores))
            dt = time.perf_counter() - t0
            if i >= warmup:
                per_step.append(dt)
                logits = out
    images = cores * IMAGES_PER_SET
    return {"images_per_step": images, "seconds_per_step": per_step,
            "images_per_s": images * len(per_step) / sum(per_step),
            "backend": _ST["R"].active_backend(), "logits_last_step": np.concatenate(logits)}
