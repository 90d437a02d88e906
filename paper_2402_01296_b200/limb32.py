"""32-bit-limb variant of the engine.

Residues are u32 modulo NTT primes q < 2^30 (q = 1 mod 2N), with
Delta = 2^30 -- the reference's default scale (pkg/src/bibranch/cli.py:66,
catalog.py:339-346).  Every word is half the HBM bytes of the u64 engine and
every modular product a native 32-bit multiply (`bcn32_*` in include/bcn.h,
csrc/ntt_mac_rescale.cu).  Buffers are int32 tensors holding the u32 bit
patterns, in the same layouts as the u64 engine:

  * limb-polys u32[npoly][nlimb][N] (limb t modulo q_t);
  * `ntt_mac_rescale`: config 2 in one pass -- ciphertexts (n_items, 2,
    nlimb, N) in the coefficient domain, plaintexts (n_items, nlimb, N) in
    the NTT domain (Montgomery form x 2^32 mod q), output (n_groups, 2,
    nlimb - 1, N) = Rescale(sum_group NTT(ct) (.) pt) in the NTT domain.

Why q < 2^30 rather than 2^31: the Harvey lazy butterflies keep values in
[0, 4q), which must fit a 32-bit word.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .errors import DeviceError, ParameterError
from .params import ntt_primes

SCALE_BITS = 30          # the reference's default scale 2^30 (cli.py:66)


def primes32(N: int, nlimb: int, bits: int = SCALE_BITS) -> list[int]:
    """The largest `nlimb` NTT primes below 2^bits (bits <= 30), descending --
    the same selection rule as the u64 chain (params.ntt_primes)."""
    if bits > 30:
        raise ParameterError("the 32-bit-limb variant needs primes below 2^30 (lazy butterflies use 4q < 2^32)")
    return ntt_primes(bits, nlimb, N)


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def to_numpy_u32(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint32)


def from_numpy_u32(a: np.ndarray, device) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32)).to(device)


class Engine32:
    """One bcn32 context: N = 2^logn, primes q_0..q_{nlimb-1} (< 2^30)."""

    def __init__(self, N: int, primes: list[int], device: int | None = None):
        if not torch.cuda.is_available():
            raise DeviceError("no CUDA device: the 32-bit-limb engine runs on the GPU only")
        lib = _lib.load()
        self.N = N
        self.logn = N.bit_length() - 1
        self.q = list(primes)
        self.nlimb = len(primes)
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        arr = (ctypes.c_uint32 * self.nlimb)(*self.q)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(lib.bcn32_ctx_create(ctypes.byref(h), self.logn, self.nlimb, arr, self.device.index),
                       "bcn32_ctx_create")
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib._lib is not None:
            _lib._lib.bcn32_ctx_destroy(h)
            self._h = None

    def _check(self, x: torch.Tensor, limbs_axis_len: int) -> None:
        if x.dtype != torch.int32 or not x.is_contiguous() or x.device != self.device:
            raise ParameterError("expected a contiguous int32 (u32 bit pattern) tensor on the context's device")
        if x.shape[-1] != self.N or limbs_axis_len != self.nlimb:
            raise ParameterError(f"expected (..., {self.nlimb}, {self.N}) limb-polys, got {tuple(x.shape)}")

    def ntt(self, data: torch.Tensor, inverse: bool = False) -> torch.Tensor:
        """In-place NTT / INTT of (npoly, nlimb, N) u32 limb-polys."""
        self._check(data, data.shape[-2])
        npoly = data.numel() // (self.nlimb * self.N)
        _lib.call("bcn32_ntt_inv" if inverse else "bcn32_ntt_fwd", self._h, data.data_ptr(), npoly, _stream())
        return data

    def to_montgomery(self, x: torch.Tensor) -> torch.Tensor:
        self._check(x, x.shape[-2])
        out = torch.empty_like(x)
        npoly = x.numel() // (self.nlimb * self.N)
        _lib.call("bcn32_to_montgomery", self._h, out.data_ptr(), x.data_ptr(), npoly, _stream())
        return out

    def ntt_mac_rescale(self, ct_coef: torch.Tensor, pt_mont: torch.Tensor, group: int) -> torch.Tensor:
        self._check(ct_coef, ct_coef.shape[-2])
        self._check(pt_mont, pt_mont.shape[-2])
        n_items = ct_coef.shape[0]
        if ct_coef.shape[1] != 2 or pt_mont.shape[0] != n_items:
            raise ParameterError("ct (n_items, 2, nlimb, N) and pt (n_items, nlimb, N) must pair up")
        ng = -(-n_items // group)
        out = torch.empty((ng, 2, self.nlimb - 1, self.N), dtype=torch.int32, device=self.device)
        _lib.call("bcn32_ntt_mac_rescale", self._h, out.data_ptr(), ct_coef.data_ptr(), pt_mont.data_ptr(),
                  n_items, group, _stream())
        return out

    def uniform(self, shape: tuple, seed: int) -> torch.Tensor:
        """Seeded uniform residues (numpy PCG64, per limb modulo q_t) for
        benchmarks and tests; shape (..., nlimb, N)."""
        rng = np.random.default_rng(seed)
        q = np.array(self.q, dtype=np.uint64)[:, None]
        a = (rng.integers(0, 1 << 62, size=shape, dtype=np.uint64) % q).astype(np.uint32)
        return from_numpy_u32(a, self.device)
