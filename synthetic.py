"""Seeded synthetic workloads for BASELINE.json configs 1 and 4 (no datasets
exist in this image).  Shared by
bench.py, tests and tests/golden/make_golden.py.  Plain numpy only: the
product package, the oracle and the reference all read the same inputs.

  cfg1 (cnn3, 28x28x1): pixels randint(0,256)/255; sensitive = centre 14x14;
    plain_full = image + Laplace(0, 0.1) outside the centre, zero inside
    (D5: the reference itself only has Gaussian perturbation); weights
    N(0, 0.1) float32.
  cfg4 (cifar3, 32x32x3): pixels U[0,1); sensitive = a random 16x16 box per
    image (origin randint(0,17) per axis, D6); plain_full = Laplace(0, 0.1)
    perturbed image with that box zeroed; weights N(0, 0.05) float32.
"""

from __future__ import annotations

import numpy as np


def weights_for(names_shapes: dict, sigma: float, seed: int) -> dict:
    rng = np.random.default_rng(seed)
    return {k: rng.normal(0.0, sigma, size=s).astype(np.float32).astype(np.float64)
            for k, s in names_shapes.items()}


def tensor_shapes(bundle) -> dict:
    """Shape of every tensor the bi-branch spec references (catalog walk)."""
    from paper_2402_01296_b200 import catalog

    net = bundle.bi
    out = {}
    for spec in (*net.cipher_layers, *net.plain_layers):
        if spec.kind == "conv":
            kh, kw = spec.kernel
            out[spec.weight] = (spec.out_channels, spec.in_channels, kh, kw)
            if spec.bias:
                out[spec.bias] = (spec.out_channels,)
    for name, shp in catalog.crot_shapes(net).items():
        out[name] = shp
    sh = catalog.branch_shapes(net)
    n_c, n_p = sh["n_c"], sh["n_p"]
    h = net.head
    half, n2 = h.n1 // 2, h.n2
    out.update({h.w_c1: (n_c, half), h.w_p1: (n_p, half), h.w_p1_prime: (n_p, half), h.b1: (half,),
                h.b1_prime: (half,), h.w_c2: (half, n2), h.w_p2: (half, n2), h.b2: (n2,)})
    return out


def cfg1_inputs(n: int = 1, seed: int = 0):
    """-> sensitive (n,1,14,14), plain_full (n,1,28,28)."""
    rng = np.random.default_rng(seed)
    img = rng.integers(0, 256, size=(n, 1, 28, 28)).astype(np.float64) / 255.0
    noise = rng.laplace(0.0, 0.1, size=img.shape)
    sens = img[:, :, 7:21, 7:21].copy()
    full = img + noise
    full[:, :, 7:21, 7:21] = 0.0
    return sens, full


def cfg4_inputs(n: int, seed: int = 0):
    """-> sensitive (n,3,16,16), plain_full (n,3,32,32) with a random box per image."""
    rng = np.random.default_rng(seed)
    img = rng.random((n, 3, 32, 32))
    r0 = rng.integers(0, 17, size=n)
    c0 = rng.integers(0, 17, size=n)
    noise = rng.laplace(0.0, 0.1, size=img.shape)
    full = img + noise
    sens = np.empty((n, 3, 16, 16))
    for i in range(n):
        sens[i] = img[i, :, r0[i]:r0[i] + 16, c0[i]:c0[i] + 16]
        full[i, :, r0[i]:r0[i] + 16, c0[i]:c0[i] + 16] = 0.0
    return sens, full


def decomposed(sens, full, region=None):
    from paper_2402_01296_b200.network import DecomposedInput

    return [DecomposedInput(s, f, region or (0, 0, s.shape[-2], s.shape[-1])) for s, f in zip(sens, full)]


def cfg4_set_inputs(set_ids, seed: int = 500, per_set: int = 32):
    """Config-5 inputs: slot set s (32 images) drawn from its own seeded
    stream (seed, s), so any rank can produce exactly its shard of the fixed
    65,536-image job, independent of the world size."""
    sens, full = [], []
    for s in set_ids:
        a, b = cfg4_inputs(per_set, seed=(seed, int(s)))
        sens.append(a)
        full.append(b)
    if not sens:
        return np.zeros((0, 3, 16, 16)), np.zeros((0, 3, 32, 32))
    return np.concatenate(sens), np.concatenate(full)
