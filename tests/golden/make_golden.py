"""Generate the golden fixtures under tests/golden/ by running the UNMODIFIED
reference package (/root/reference/pkg/src/bibranch) in this container.

Run: python tests/golden/make_golden.py    (needs /root/reference; the GPU box
does not have it, which is why the outputs are committed as small .npz files)

Each fixture holds the inputs, the weights, the reference's clear logits
(`reference_forward`, network.py:451-507), the reference simulator's logits
(`forward_bicrypto`, network.py:388-448) and its OpRecorder counts and
per-layer table (sim.py:47-108), which the GPU engine must reproduce as
integers.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg/src"
sys.path.insert(0, ROOT)
sys.path.insert(0, REF)
os.environ.setdefault("BIBRANCH_BACKEND", "python")

import bibranch as R  # noqa: E402  (the reference)
from bibranch import catalog as RC  # noqa: E402
from bibranch.archive import TensorArchive as RArchive  # noqa: E402
from bibranch.fixtures import digit_images, fixture_weights  # noqa: E402
from bibranch.layers import LayerSpec as RLayer  # noqa: E402
from bibranch.network import ConnectionSpec as RConn  # noqa: E402
from bibranch.network import DecomposedInput as RDec  # noqa: E402
from bibranch.network import IntegrationSpec as RHead  # noqa: E402
from bibranch.network import NetworkSpec as RNet  # noqa: E402

import synthetic  # noqa: E402
from paper_2402_01296_b200 import catalog as C  # noqa: E402


def _ref_cifar3() -> RNet:
    """BASELINE config-4 network declared with the reference's own classes."""
    def conv(prefix, cin, cout, stride):
        return RLayer("conv", kernel=(3, 3), stride=stride, padding=(1, 1), in_channels=cin, out_channels=cout,
                      weight=f"{prefix}.weight", bias=f"{prefix}.bias")

    def branch(prefix, act):
        return (conv(f"{prefix}conv1", 3, 16, (1, 1)), RLayer(act), conv(f"{prefix}conv2", 16, 32, (2, 2)),
                RLayer(act), RLayer("sumpool", kernel=(2, 2), stride=(2, 2), scale=0.25))

    head = RHead(n1=20, n2=10, w_c1="head.w_c1", w_p1="head.w_p1", w_p1_prime="head.w_p1_prime", b1="head.b1",
                 b1_prime="head.b1_prime", w_c2="head.w_c2", w_p2="head.w_p2", b2="head.b2")
    return RNet("cifar3", (3, 32, 32), (3, 16, 16), branch("cipher.", "square"), branch("plain.", "relu"),
                (RConn(1, 2, "connect.1.w_crot"), RConn(3, 4, "connect.2.w_crot")), head)


def _run(net, dec, weights, ctx, strategy):
    res = R.forward_bicrypto(net, dec, weights, ctx, strategy=strategy)
    return res.decrypt_logits(), res.recorder


def _pack(path, **kw):
    np.savez_compressed(path, **kw)
    print("wrote", path, os.path.getsize(path), "bytes")


def _weights_arrays(w) -> dict:
    return {f"w::{k}": np.asarray(w[k], dtype=np.float64) for k in w.names()}


def cnn3_fixture():
    bundle = RC.get("cnn3")
    w = fixture_weights("cnn3", seed=0)
    imgs, labels = digit_images(8, seed=2)
    dec = R.decompose_batch(imgs, noise_sigma=0.1, seed=5)
    ctx = R.make_context(**RC.default_context_params(bundle))
    ref = R.reference_forward(bundle.bi, dec, w)
    sim, rec = _run(bundle.bi, dec, w, ctx, "bhw")
    _, rec1 = _run(bundle.bi, dec[0], w, ctx, "hw")
    meta = {"counts_bhw": rec.snapshot(), "counts_hw": rec1.snapshot(), "layer_table": rec.layer_table(),
            "required_levels": [RC.required_levels(bundle.bi), RC.required_levels(bundle.backbone)]}
    _pack(os.path.join(HERE, "cnn3_fixture.npz"), sens=np.stack([d.sensitive for d in dec]),
          full=np.stack([d.plain_full for d in dec]), labels=labels, logits_ref=ref, logits_sim=sim,
          meta=json.dumps(meta), **_weights_arrays(w))


def cnn3_cfg1():
    bundle = C.get("cnn3")
    w = synthetic.weights_for(synthetic.tensor_shapes(bundle), 0.1, seed=1)
    sens, full = synthetic.cfg1_inputs(1, seed=0)
    dec = [RDec(sens[0], full[0], (7, 7, 14, 14))]
    rbundle = RC.get("cnn3")
    ctx = R.make_context(8192, RC.required_levels(rbundle) + 1, 2.0 ** 30)
    warch = RArchive(dict(w))
    ref = R.reference_forward(rbundle.bi, dec, warch)
    sim, rec = _run(rbundle.bi, dec, warch, ctx, "hw")
    meta = {"counts_hw": rec.snapshot(), "layer_table": rec.layer_table()}
    _pack(os.path.join(HERE, "cnn3_cfg1.npz"), sens=sens, full=full, logits_ref=ref, logits_sim=sim,
          meta=json.dumps(meta), **{f"w::{k}": v for k, v in w.items()})


def cifar3_cfg4(n=8):
    bundle = C.get("cifar3")
    w = synthetic.weights_for(synthetic.tensor_shapes(bundle), 0.05, seed=3)
    sens, full = synthetic.cfg4_inputs(n, seed=2)
    dec = [RDec(s, f, (0, 0, 16, 16)) for s, f in zip(sens, full)]
    net = _ref_cifar3()
    warch = RArchive(dict(w))
    ctx = R.make_context(1 << 14, 14, 2.0 ** 30)
    ref = R.reference_forward(net, dec, warch)
    sim, rec = _run(net, dec, warch, ctx, "bhw")
    meta = {"counts_bhw": rec.snapshot(), "layer_table": rec.layer_table()}
    _pack(os.path.join(HERE, "cifar3_cfg4.npz"), sens=sens, full=full, logits_ref=ref, logits_sim=sim,
          meta=json.dumps(meta), **{f"w::{k}": v for k, v in w.items()})


def cifar3_cfg4_sets(n_sets=2):
    """Two FULL slot sets (32 images each, 32 x 16 x 16 = 8192 slots) of config-4
    inputs: reference_forward over all 64 images, the simulator's
    forward_bicrypto run set by set (one ciphertext set holds 32 images)."""
    bundle = C.get("cifar3")
    w = synthetic.weights_for(synthetic.tensor_shapes(bundle), 0.05, seed=3)
    sens, full = synthetic.cfg4_inputs(32 * n_sets, seed=9)
    dec = [RDec(s, f, (0, 0, 16, 16)) for s, f in zip(sens, full)]
    net = _ref_cifar3()
    warch = RArchive(dict(w))
    ctx = R.make_context(1 << 14, 14, 2.0 ** 30)
    ref = R.reference_forward(net, dec, warch)
    sims, recs = [], []
    for g in range(n_sets):
        sim, rec = _run(net, dec[32 * g:32 * (g + 1)], warch, ctx, "bhw")
        sims.append(sim)
        recs.append(rec.snapshot())
    assert all(r == recs[0] for r in recs)
    meta = {"counts_bhw": recs[0]}
    _pack(os.path.join(HERE, "cifar3_cfg4_sets.npz"), sens=sens, full=full, logits_ref=ref,
          logits_sim=np.concatenate(sims), meta=json.dumps(meta), **{f"w::{k}": v for k, v in w.items()})


def cnn3_backbone():
    """The single-chain cnn3 run fully encrypted by the reference's
    forward_backbone (network.py:510-582) on one whole image (the reference's
    own test recipe, pkg/tests/test_network.py:247-256): counts (1952 HE ops),
    per-layer table, simulator logits and reference_backbone logits."""
    bundle = RC.get("cnn3")
    w = fixture_weights("cnn3", seed=0)
    imgs, _ = digit_images(8, seed=2)
    dec = R.decompose_batch(imgs, noise_sigma=0.1, seed=5)
    img = dec[0].plain_full.copy()
    r0, c0, hs, ws = dec[0].region
    img[:, r0:r0 + hs, c0:c0 + ws] = dec[0].sensitive
    ctx = R.make_context(**RC.default_context_params(bundle))
    res = R.forward_backbone(bundle.backbone, img[None], w, ctx, strategy="hw")
    ref = R.reference_backbone(bundle.backbone, img[None], w)
    meta = {"counts_hw": res.recorder.snapshot(), "layer_table": res.recorder.layer_table()}
    _pack(os.path.join(HERE, "cnn3_backbone.npz"), image=img, logits_ref=ref, logits_sim=res.decrypt_logits(),
          meta=json.dumps(meta), **_weights_arrays(w))


if __name__ == "__main__":
    which = sys.argv[1:] or ["cnn3_fixture", "cnn3_cfg1", "cifar3_cfg4", "cnn3_backbone"]
    for name in which:
        globals()[name]()
