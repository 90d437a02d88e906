"""Plaintext branch of the bi-network on the device (torch float64).

The reference evaluates it in numpy on the host (layers.py:329-404,
network.py:261-282); here the same layer semantics run on the GPU beside the
ciphertext branch, so the connection features z and the head's cross terms
are produced in HBM and handed straight to the encode kernel -- no host round
trip on the hot path.  Values agree with the numpy reference to float64
rounding (summation order only).
"""

from __future__ import annotations

import os

import numpy as np
import torch
import torch.nn.functional as F

from .errors import ShapeError, UsageError

torch.backends.cudnn.deterministic = True


class WeightCache:
    """float64 device copies of archive tensors (converted once per archive)."""

    def __init__(self, weights, device):
        self.weights = weights
        self.device = device
        self._t: dict = {}

    def __getitem__(self, name: str) -> torch.Tensor:
        t = self._t.get(name)
        if t is None:
            t = torch.as_tensor(np.asarray(self.weights[name], dtype=np.float64), device=self.device)
            self._t[name] = t
        return t


_INDEX: dict = {}


def index_tensor(key, make, device) -> torch.Tensor:
    """Device copy of a static index vector (slot anchors), uploaded once --
    keeps host->device copies out of steady-state forwards and CUDA graphs."""
    k = (key, str(device))
    t = _INDEX.get(k)
    if t is None:
        t = torch.as_tensor(np.asarray(make(), dtype=np.int64), device=device)
        _INDEX[k] = t
    return t


def weight_cache(ctx, weights) -> "WeightCache":
    """One WeightCache per (context, archive): weights are uploaded once."""
    caches = ctx.__dict__.setdefault("_weight_caches", {})
    wc = caches.get(id(weights))
    if wc is None or wc.weights is not weights:
        wc = WeightCache(weights, ctx.engine.device)
        caches[id(weights)] = wc
    return wc


def to_device(x, device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=torch.float64)
    return torch.as_tensor(np.asarray(x, dtype=np.float64), device=device)


def conv(x: torch.Tensor, w: torch.Tensor, b, stride, padding) -> torch.Tensor:
    if x.shape[1] != w.shape[1]:
        raise ShapeError(f"conv expects {w.shape[1]} input channels, got {x.shape[1]}")
    O, C, kh, kw = w.shape
    if (x.is_cuda and x.dtype == torch.float64 and x.dim() == 4 and C * kh * kw <= 384
            and os.environ.get("BCN_PLAIN_CONV", "1") != "0"):
        # libbcn's direct float64 conv (cuDNN's implicit-GEMM dgemm: 2.5-3.1 ms per cifar3 layer at 4,096
        # images; this: bound by its output write)
        from . import _lib
        B, _, H, W = x.shape
        (sh, sw), (ph, pw) = tuple(stride), tuple(padding)
        oh, ow = (H + 2 * ph - kh) // sh + 1, (W + 2 * pw - kw) // sw + 1
        xc, wc = x.contiguous(), w.contiguous()
        bc = b.contiguous() if b is not None else None
        out = torch.empty((B, O, oh, ow), dtype=torch.float64, device=x.device)
        _lib.call("bcn_plain_conv2d", xc.data_ptr(), wc.data_ptr(), bc.data_ptr() if bc is not None else None,
                  out.data_ptr(), B, C, H, W, O, kh, kw, sh, sw, ph, pw,
                  torch.cuda.current_stream(x.device).cuda_stream)
        return out
    return F.conv2d(x, w, b, stride=tuple(stride), padding=tuple(padding))


def sum_pool(x: torch.Tensor, window, stride, scale: float) -> torch.Tensor:
    (kh, kw), (sh, sw) = window, stride
    H, W = x.shape[-2:]
    oh, ow = (H - kh) // sh + 1, (W - kw) // sw + 1
    out = torch.zeros(x.shape[:-2] + (oh, ow), dtype=x.dtype, device=x.device)
    for di in range(kh):
        for dj in range(kw):
            out += x[..., di:di + (oh - 1) * sh + 1:sh, dj:dj + (ow - 1) * sw + 1:sw]
    return out * scale


def layer(x: torch.Tensor, spec, W: WeightCache) -> torch.Tensor:
    k = spec.kind
    if k == "conv":
        return conv(x, W[spec.weight], W[spec.bias] if spec.bias else None, spec.stride, spec.padding)
    if k == "sumpool":
        return sum_pool(x, spec.kernel, spec.stride, spec.scale)
    if k == "fc":
        out = x.reshape(x.shape[0], -1) @ W[spec.weight]
        return out + W[spec.bias] if spec.bias else out
    if k == "square":
        return x * x
    if k == "relu":
        return torch.clamp_min(x, 0.0)
    raise UsageError(f"plain layer cannot evaluate kind {k!r}")


def channel_mix(y: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    if y.shape[-3] != w.shape[1]:
        raise ShapeError(f"channel mismatch: matrix maps {w.shape[1]} channels, tensor has {y.shape[-3]}")
    return torch.einsum("kc,...chw->...khw", w, y)


def head_act(x: torch.Tensor, kind: str) -> torch.Tensor:
    if kind == "square":
        return x * x
    if kind == "relu":
        return torch.clamp_min(x, 0.0)
    raise UsageError(f"unsupported head activation {kind!r}")
