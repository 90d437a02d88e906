"""Device engine: one libbcn context per HeParams, with torch-owned buffers.

Every method is a thin, asynchronous call into libbcn.so on the current
torch CUDA stream; ciphertext batches are int64 tensors (u64 bit patterns)
of shape (G, 2, limbs, N) in the bit-reversed NTT domain.  No method falls
back to the host: a missing library or device raises DeviceError.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import _lib
from .errors import CapacityError, DeviceError, ParameterError
from .params import HeParams, fft_table, galois_element

RELIN_KEY_ID = 2
RANK_ID_SHIFT = 40      # encryption ids of rank r start at 1 + (r << 40)


def process_rank() -> int:
    """This process's rank in a multi-GPU job (torch.distributed if it is
    initialised, else the launcher's RANK variable, else 0)."""
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return int(dist.get_rank())
    except (ImportError, RuntimeError):
        pass
    return int(os.environ.get("RANK", "0") or 0)


def counter_base(rank: int) -> int:
    """First Philox encryption id of a rank.  Every rank derives the same keys
    from the shared seed, so the ids (the per-ciphertext randomness `a`, `e`)
    must not overlap across ranks: 2^40 ids per rank."""
    if rank < 0 or rank >= (1 << (64 - RANK_ID_SHIFT)):
        raise ParameterError(f"rank {rank} outside [0, 2^{64 - RANK_ID_SHIFT})")
    return 1 + (rank << RANK_ID_SHIFT)


def _ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


class Engine:
    def __init__(self, params: HeParams, device: int | None = None):
        if not torch.cuda.is_available():
            raise DeviceError("no CUDA device: the RNS-CKKS engine runs on the GPU only")
        lib = _lib.load()
        self.params = params
        self.N = params.N
        self.logn = params.logn
        self.L = params.max_level
        self.K = params.K
        self.nbasis = self.L + 1 + self.K
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        q = (ctypes.c_uint64 * len(params.q))(*params.q)
        p = (ctypes.c_uint64 * len(params.p))(*params.p)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(lib.bcn_ctx_create(ctypes.byref(h), self.logn, self.L, q, len(params.p), p,
                                          params.dnum, params.seed, self.device.index), "bcn_ctx_create")
        self._h = h
        re, im = fft_table(self.N)
        _lib.call("bcn_ctx_set_fft", h, re.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                  im.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
        self._counter = counter_base(process_rank())   # Philox id of the next encryption
        self.graph_counter: torch.Tensor | None = None   # device-side id base (CUDA-graph replays)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None and getattr(_lib, "_lib", None) is not None:
            try:
                _lib._lib.bcn_ctx_destroy(h)
            except Exception:
                pass
            self._h = None

    # ---------------------------------------------------------- helpers
    @property
    def handle(self):
        return self._h

    def empty_ct(self, G: int, level: int) -> torch.Tensor:
        return torch.empty((G, 2, level + 1, self.N), dtype=torch.int64, device=self.device)

    def _dev_f64(self, vals) -> torch.Tensor:
        if isinstance(vals, torch.Tensor):
            t = vals.to(device=self.device, dtype=torch.float64)
        else:
            t = torch.as_tensor(np.asarray(vals, dtype=np.float64), device=self.device)
        if t.dim() == 1:
            t = t[None]
        return t.contiguous()

    def _check_mag(self, vals, scale: float) -> None:
        # the canonical-embedding inverse is a contraction: |coef| <= scale * max|v|.
        # Checked on host data only: a device-side check would cost a sync per encode.
        if isinstance(vals, np.ndarray) and vals.size:
            m = float(np.abs(vals).max())
            if not np.isfinite(m):
                raise ParameterError("plaintext vector must contain only finite values")
            if m * scale >= 2.0 ** 62:
                raise ParameterError(f"value {m:.3g} at scale 2^{np.log2(scale):.1f} overflows 62-bit coefficients")

    def next_counter(self, n: int = 1) -> int:
        c = self._counter
        self._counter += n
        if (self._counter - 1) >> RANK_ID_SHIFT != (c - 1) >> RANK_ID_SHIFT:
            raise ParameterError("encryption id range of this rank exhausted")
        return c

    # ---------------------------------------------------------- K1 / K2
    def ntt(self, data: torch.Tensor, prime0: int = 0, inverse: bool = False) -> torch.Tensor:
        """In-place NTT of int64[npoly, nlimb, N] (limb t mod basis prime prime0+t)."""
        npoly, nlimb, N = data.shape
        assert N == self.N and data.is_contiguous()
        _lib.call("bcn_ntt_inv" if inverse else "bcn_ntt_fwd", self._h, _ptr(data), npoly, nlimb, prime0, _stream())
        return data

    # ---------------------------------------------------------- K9-K11
    def encode(self, vals, level: int, scale: float, montgomery: bool = False) -> torch.Tensor:
        self._check_mag(vals, scale)
        v = self._dev_f64(vals)
        if v.shape[1] > self.N // 2:
            raise CapacityError(f"vector of length {v.shape[1]} exceeds {self.N // 2} slots")
        out = torch.empty((v.shape[0], level + 1, self.N), dtype=torch.int64, device=self.device)
        _lib.call("bcn_encode", self._h, _ptr(v), v.shape[1], v.shape[1], v.shape[0], float(scale), level,
                  int(montgomery), _ptr(out), _stream())
        return out

    def encrypt(self, vals, level: int | None = None, scale: float | None = None,
                counter: int | None = None) -> torch.Tensor:
        level = self.L if level is None else level
        scale = self.params.scale if scale is None else scale
        self._check_mag(vals, scale)
        v = self._dev_f64(vals)
        if v.shape[1] > self.N // 2:
            raise CapacityError(f"vector of length {v.shape[1]} exceeds {self.N // 2} slots")
        G = v.shape[0]
        ct = self.empty_ct(G, level)
        if self.graph_counter is not None and counter is None:
            # CUDA-graph mode: the Philox id base is read from device memory at run time
            _lib.call("bcn_encrypt_devctr", self._h, _ptr(v), v.shape[1], v.shape[1], G, level, float(scale),
                      _ptr(self.graph_counter), _ptr(ct), _stream())
            return ct
        counter = self.next_counter(G) if counter is None else counter
        _lib.call("bcn_encrypt", self._h, _ptr(v), v.shape[1], v.shape[1], G, level, float(scale), counter,
                  _ptr(ct), _stream())
        return ct

    def encrypt_rotated(self, vals, rots, level: int | None = None, scale: float | None = None,
                        counter: int | None = None) -> torch.Tensor:
        """Fresh encryptions of every row and of its rotations by `rots` slots
        (np.roll(row, -r)): (1 + len(rots), G, 2, level+1, N).  The plaintext
        of a rotated row is the automorphism X -> X^(5^r) of the row's plaintext,
        so the canonical embedding runs once per row (bcn_encrypt_rotated); copy
        c of row p uses encryption id counter + c G + p, like encrypt() of the
        stacked rolled rows."""
        from .params import galois_element
        level = self.L if level is None else level
        scale = self.params.scale if scale is None else scale
        self._check_mag(vals, scale)
        v = self._dev_f64(vals)
        if v.shape[1] > self.N // 2:
            raise CapacityError(f"vector of length {v.shape[1]} exceeds {self.N // 2} slots")
        G, ncopy = v.shape[0], 1 + len(rots)
        gal = (ctypes.c_uint64 * ncopy)(1, *[galois_element(int(r), self.N) for r in rots])
        ct = self.empty_ct(ncopy * G, level)
        counter = self.next_counter(ncopy * G) if counter is None else counter
        _lib.call("bcn_encrypt_rotated", self._h, _ptr(v), v.shape[1], v.shape[1], G, level, float(scale), counter,
                  ncopy, gal, _ptr(ct), _stream())
        return ct.view(ncopy, G, 2, level + 1, self.N)

    def decrypt(self, ct: torch.Tensor, level: int, scale: float, nout: int | None = None) -> torch.Tensor:
        G, two, nl, N = ct.shape
        nout = self.N // 2 if nout is None else nout
        out = torch.empty((G, nout), dtype=torch.float64, device=self.device)
        _lib.call("bcn_decrypt", self._h, _ptr(ct), nl, G, level, float(scale), _ptr(out), nout, _stream())
        return out

    def decrypt_poly(self, ct: torch.Tensor, level: int) -> torch.Tensor:
        G, _, nl, N = ct.shape
        k = 2 if level >= 1 else 1
        out = torch.empty((G, k, N), dtype=torch.int64, device=self.device)
        _lib.call("bcn_decrypt_poly", self._h, _ptr(ct), nl, G, level, _ptr(out), _stream())
        return out

    # ---------------------------------------------------------- K3-K8
    def add(self, a: torch.Tensor, b: torch.Tensor, level: int) -> torch.Tensor:
        G = a.shape[0]
        out = self.empty_ct(G, level)
        _lib.call("bcn_add", self._h, _ptr(out), _ptr(a), a.shape[2], _ptr(b), b.shape[2], 0, G, G, level,
                  _stream())
        return out

    def add_plain(self, a: torch.Tensor, pt: torch.Tensor, level: int, inplace: bool = False) -> torch.Tensor:
        """a + pt on component 0.  inplace (the caller owns `a`, which has exactly
        level+1 limbs): component 0 is updated where it lies and component 1 is
        not copied."""
        G = a.shape[0]
        out = a if inplace and a.shape[2] == level + 1 and a.is_contiguous() else self.empty_ct(G, level)
        _lib.call("bcn_add", self._h, _ptr(out), _ptr(a), a.shape[2], _ptr(pt), pt.shape[1], 1, pt.shape[0], G,
                  level, _stream())
        return out

    def mul_plain(self, a: torch.Tensor, pt_mont: torch.Tensor, level: int, rescale: bool = True) -> torch.Tensor:
        G = a.shape[0]
        out = self.empty_ct(G, level - 1 if rescale else level)
        name = "bcn_mul_plain" if rescale else "bcn_mul_plain_norescale"
        _lib.call(name, self._h, _ptr(out), _ptr(a), a.shape[2], _ptr(pt_mont), pt_mont.shape[0], G, level,
                  _stream())
        return out

    def rescale(self, a: torch.Tensor, level: int) -> torch.Tensor:
        G = a.shape[0]
        out = self.empty_ct(G, level - 1)
        _lib.call("bcn_rescale", self._h, _ptr(out), _ptr(a), a.shape[2], G, level, _stream())
        return out

    def mul_cc(self, a: torch.Tensor, b: torch.Tensor, level: int, rescale: bool = True,
               out: torch.Tensor | None = None) -> torch.Tensor:
        G = a.shape[0]
        if out is None:
            out = self.empty_ct(G, level - 1 if rescale else level)
        _lib.call("bcn_mul_cc", self._h, _ptr(out), _ptr(a), a.shape[2], _ptr(b), b.shape[2], G, level,
                  int(rescale), _stream())
        return out

    def modup(self, a: torch.Tensor, level: int) -> torch.Tensor:
        G = a.shape[0]
        w = ctypes.c_uint64()
        _lib.call("bcn_modup_words", self._h, G, level, ctypes.byref(w))
        U = torch.empty(int(w.value), dtype=torch.int64, device=self.device)
        _lib.call("bcn_modup", self._h, _ptr(U), _ptr(a), a.shape[2], G, level, _stream())
        return U

    def rotate(self, a: torch.Tensor, r: int, level: int, U: torch.Tensor | None = None,
               out: torch.Tensor | None = None) -> torch.Tensor:
        G = a.shape[0]
        g = galois_element(r, self.N)
        if out is None:
            out = self.empty_ct(G, level)
        if U is None:
            _lib.call("bcn_rotate", self._h, _ptr(out), _ptr(a), a.shape[2], G, level, g, _stream())
        else:
            _lib.call("bcn_rotate_hoisted", self._h, _ptr(out), _ptr(a), a.shape[2], _ptr(U), G, level, g,
                      _stream())
        return out

    def rotate_many(self, a: torch.Tensor, rots, level: int, U: torch.Tensor | None = None,
                    out: torch.Tensor | None = None) -> torch.Tensor:
        """Hoisted rotations of one source by every r in `rots` (bcn_rotate_hoisted_many):
        out[k] = rotate(a, rots[k]), bit-identical to separate calls; U = modup(a) is
        read once for all of them."""
        G = a.shape[0]
        n = len(rots)
        if out is None:
            out = torch.empty((n, G, 2, level + 1, self.N), dtype=torch.int64, device=self.device)
        if U is None:
            U = self.modup(a, level)
        gal = (ctypes.c_uint64 * n)(*[galois_element(r, self.N) for r in rots])
        _lib.call("bcn_rotate_hoisted_many", self._h, _ptr(out), _ptr(a), a.shape[2], _ptr(U), G, level, n, gal,
                  _stream())
        return out

    def keygen_galois(self, g: int) -> None:
        _lib.call("bcn_keygen_galois", self._h, g, _stream())

    def keygen_relin(self) -> None:
        _lib.call("bcn_keygen_relin", self._h, _stream())

    def export_key(self, key_id: int) -> torch.Tensor:
        out = torch.empty((self.params.dnum, 2, self.nbasis, self.N), dtype=torch.int64, device=self.device)
        _lib.call("bcn_export_key", self._h, key_id, _ptr(out), _stream())
        return out

    def export_secret(self) -> torch.Tensor:
        out = torch.empty((self.nbasis, self.N), dtype=torch.int64, device=self.device)
        _lib.call("bcn_export_secret", self._h, _ptr(out), _stream())
        return out

    def encode_ext(self, vals, level: int, scale: float) -> torch.Tensor:
        """Montgomery multiplier over the extended basis (limbs q_0..q_level, p_*)."""
        self._check_mag(vals, scale)
        v = self._dev_f64(vals)
        if v.shape[1] > self.N // 2:
            raise CapacityError(f"vector of length {v.shape[1]} exceeds {self.N // 2} slots")
        out = torch.empty((v.shape[0], level + 1 + self.K, self.N), dtype=torch.int64, device=self.device)
        _lib.call("bcn_encode_ext", self._h, _ptr(v), v.shape[1], v.shape[1], v.shape[0], float(scale), level,
                  _ptr(out), _stream())
        return out

    def rotsum(self, terms, level: int, out: torch.Tensor | None = None, keys=None) -> torch.Tensor:
        """sum_t pt_t (x) rot_{g_t}(ct_t) with ONE ModDown (unrescaled, at `level`).
        terms: [(ct u64[G,2,level+1,N], U from modup(ct), g, pt_ext or None)];
        keys: optional per-term premul_key(g_t, pt_t, level) tensors (or None)."""
        G = terms[0][0].shape[0]
        n = len(terms)
        Us = (ctypes.c_uint64 * n)(*[t[1].data_ptr() for t in terms])
        cts = (ctypes.c_uint64 * n)(*[t[0].data_ptr() for t in terms])
        gal = (ctypes.c_uint64 * n)(*[int(t[2]) for t in terms])
        pts = (ctypes.c_uint64 * n)(*[0 if t[3] is None else t[3].data_ptr() for t in terms])
        bat = (ctypes.c_int * n)(*[int(t[3] is not None and t[3].shape[0] != 1) for t in terms])
        if out is None:
            out = self.empty_ct(G, level)
        if keys is None:
            _lib.call("bcn_rotsum", self._h, _ptr(out), n, Us, cts, gal, pts, bat, G, level, _stream())
        else:
            ks = (ctypes.c_uint64 * n)(*[0 if k is None else k.data_ptr() for k in keys])
            _lib.call("bcn_rotsum_keys", self._h, _ptr(out), n, Us, cts, gal, pts, bat, ks, G, level, _stream())
        return out

    PLANES_IMMA, PLANES_TCGEN05 = 0, 1

    def pack_planes_ext(self, pts, level: int, layout: int = 0) -> torch.Tensor:
        """Extended-basis byte planes of an O x K plaintext matrix for conv_ks_mac:
        column k holds level+1+K-limb (rotation) or level+1-limb (identity) plaintexts.
        layout: PLANES_IMMA (mma.sync, any G) or PLANES_TCGEN05 (tcgen05, G >= 64)."""
        O, K = len(pts), len(pts[0])
        nb = ctypes.c_uint64()
        _lib.call("bcn_planes_ext_bytes", self._h, O, K, level, ctypes.byref(nb))
        planes = torch.empty(int(nb.value), dtype=torch.uint8, device=self.device)
        p_arr = (ctypes.c_uint64 * (O * K))(*[p.data_ptr() for row in pts for p in row])
        limbs = (ctypes.c_int * K)(*[int(p.shape[1]) for p in pts[0]])
        _lib.call("bcn_pack_planes_ext", self._h, _ptr(planes), O, K, p_arr, limbs, level, int(layout), _stream())
        return planes

    def conv_ks_mac(self, srcs, Us, gals, planes: torch.Tensor, n_out: int, level: int,
                    layout: int = 0) -> torch.Tensor:
        """Conv outputs with lazy ModDown: out[o] = Rescale(sum_k pt[o][k] (x) rot_{g_k}(srcs[k]))
        -> u64[n_out, G, 2, level, N] at level-1 (g_k = 1: srcs[k] itself, Us[k] unused).
        layout: the one planes was packed with."""
        K = len(srcs)
        G = srcs[0].shape[0]
        s_arr = (ctypes.c_uint64 * K)(*[x.data_ptr() for x in srcs])
        u_arr = (ctypes.c_uint64 * K)(*[0 if u is None else u.data_ptr() for u in Us])
        g_arr = (ctypes.c_uint64 * K)(*[int(g) for g in gals])
        out = torch.empty((n_out, G, 2, level, self.N), dtype=torch.int64, device=self.device)
        _lib.call("bcn_conv_ks_mac", self._h, _ptr(out), n_out, K, s_arr, u_arr, g_arr, _ptr(planes), int(layout),
                  G, level, _stream())
        return out

    def rotsum_rescale(self, terms, level: int, keys=None, ct_terms=()) -> torch.Tensor:
        """Rescaled lazy sum: rotation terms as in rotsum plus (ct, pt) terms, with
        ONE merged ModDown + rescale per component -> u64[G,2,level,N] at level-1."""
        G = terms[0][0].shape[0]
        n = len(terms)
        Us = (ctypes.c_uint64 * n)(*[t[1].data_ptr() for t in terms])
        cts = (ctypes.c_uint64 * n)(*[t[0].data_ptr() for t in terms])
        gal = (ctypes.c_uint64 * n)(*[int(t[2]) for t in terms])
        pts = (ctypes.c_uint64 * n)(*[0 if t[3] is None else t[3].data_ptr() for t in terms])
        bat = (ctypes.c_int * n)(*[int(t[3] is not None and t[3].shape[0] != 1) for t in terms])
        ks = None if keys is None else (ctypes.c_uint64 * n)(*[0 if k is None else k.data_ptr() for k in keys])
        m = len(ct_terms)
        c_c = (ctypes.c_uint64 * max(m, 1))(*[t[0].data_ptr() for t in ct_terms])
        c_p = (ctypes.c_uint64 * max(m, 1))(*[t[1].data_ptr() for t in ct_terms])
        c_b = (ctypes.c_int * max(m, 1))(*[int(t[1].shape[0] != 1) for t in ct_terms])
        out = self.empty_ct(G, level - 1)
        _lib.call("bcn_rotsum_rescale", self._h, _ptr(out), n, Us, cts, gal, pts, bat, ks, m, c_c, c_p, c_b, G,
                  level, _stream())
        return out

    def premul_key(self, g: int, pt: torch.Tensor, level: int) -> torch.Tensor:
        """Galois key g with the (unbatched, ext-basis Montgomery) multiplier pt
        folded in, for rotsum(keys=...): u64[dnum,2,nbasis,N]."""
        out = torch.empty((self.params.dnum, 2, self.nbasis, self.N), dtype=torch.int64, device=self.device)
        _lib.call("bcn_premul_key", self._h, _ptr(out), int(g), _ptr(pt), level, _stream())
        return out

    def mac_multi(self, cts, pts, level: int, rescale: bool = True) -> torch.Tensor:
        """out[o] = sum_k cts[k] (x) pts[o][k]; cts: K tensors u64[G,2,level+1,N];
        pts: O lists of K Montgomery plaintexts u64[1,level+1,N] -> u64[O,G,2,l,N]."""
        O, K = len(pts), len(cts)
        G = cts[0].shape[0]
        c_arr = (ctypes.c_uint64 * K)(*[c.data_ptr() for c in cts])
        p_arr = (ctypes.c_uint64 * (O * K))(*[p.data_ptr() for row in pts for p in row])
        nl = level if rescale else level + 1
        out = torch.empty((O, G, 2, nl, self.N), dtype=torch.int64, device=self.device)
        _lib.call("bcn_mac_multi", self._h, _ptr(out), O, K, c_arr, p_arr, G, level, int(rescale), _stream())
        return out

    def pack_planes(self, pts, level: int, layout: int = 0) -> torch.Tensor:
        """Byte-plane pack of an O x K plaintext matrix (Montgomery u64[1,level+1,N]
        each) for mac_multi_planes; K <= 256.  Done once per layer.
        layout: 0 mma.sync IMMA, 1 tcgen05 (the MAC must use the same)."""
        O, K = len(pts), len(pts[0])
        nb = ctypes.c_uint64()
        _lib.call("bcn_planes_bytes", self._h, O, K, level, ctypes.byref(nb))
        planes = torch.empty(int(nb.value), dtype=torch.uint8, device=self.device)
        p_arr = (ctypes.c_uint64 * (O * K))(*[p.data_ptr() for row in pts for p in row])
        _lib.call("bcn_pack_planes_layout", self._h, _ptr(planes), O, K, p_arr, level, int(layout), _stream())
        return planes

    def mac_multi_planes(self, cts, planes: torch.Tensor, n_out: int, level: int, rescale: bool = True,
                         layout: int = 0) -> torch.Tensor:
        """Tensor-core mac_multi: out[o] = sum_k cts[k] (x) pt[o][k] with the
        plaintexts given as pack_planes(..., layout) output; bit-identical to
        mac_multi in either layout."""
        K = len(cts)
        G = cts[0].shape[0]
        c_arr = (ctypes.c_uint64 * K)(*[c.data_ptr() for c in cts])
        nl = level if rescale else level + 1
        out = torch.empty((n_out, G, 2, nl, self.N), dtype=torch.int64, device=self.device)
        _lib.call("bcn_mac_multi_planes_layout", self._h, _ptr(out), n_out, K, c_arr, _ptr(planes), G, level,
                  int(rescale), int(layout), _stream())
        return out

    def mac_terms_acc(self, out: torch.Tensor, terms, level: int) -> torch.Tensor:
        G = terms[0][0].shape[0]
        n = len(terms)
        cts = (ctypes.c_uint64 * n)(*[t[0].data_ptr() for t in terms])
        pts = (ctypes.c_uint64 * n)(*[t[1].data_ptr() for t in terms])
        bat = (ctypes.c_int * n)(*[int(t[1].shape[0] != 1) for t in terms])
        _lib.call("bcn_mac_terms_acc", self._h, _ptr(out), n, cts, pts, bat, G, level, _stream())
        return out

    def mac_terms(self, terms, level: int, rescale: bool = True, out: torch.Tensor | None = None) -> torch.Tensor:
        """sum_t ct_t (x) pt_t (one fused launch per 160 terms), optionally rescaled.
        terms: [(ct u64[G,2,>=level+1,N] with exactly level+1 limbs, pt_mont u64[G|1,level+1,N])]."""
        G = terms[0][0].shape[0]
        n = len(terms)
        cts = (ctypes.c_uint64 * n)(*[t[0].data_ptr() for t in terms])
        pts = (ctypes.c_uint64 * n)(*[t[1].data_ptr() for t in terms])
        bat = (ctypes.c_int * n)(*[int(t[1].shape[0] != 1) for t in terms])
        if out is None:
            out = self.empty_ct(G, level - 1 if rescale else level)
        _lib.call("bcn_mac_terms", self._h, _ptr(out), n, cts, pts, bat, G, level, int(rescale), _stream())
        return out

    def mac(self, ct: torch.Tensor, pt_mont: torch.Tensor, group: int) -> torch.Tensor:
        n_items, _, nl, N = ct.shape
        ng = -(-n_items // group)
        out = torch.empty((ng, 2, nl, N), dtype=torch.int64, device=self.device)
        _lib.call("bcn_mac", self._h, _ptr(out), _ptr(ct), _ptr(pt_mont), n_items, group, nl, _stream())
        return out

    def ntt_mac_rescale(self, ct_coef: torch.Tensor, pt_mont: torch.Tensor, group: int) -> torch.Tensor:
        """BASELINE config 2 in one pass (bcn_ntt_mac_rescale): ct_coef
        (n_items, 2, nlimb, N) in the coefficient domain, pt_mont
        (n_items, nlimb, N) NTT domain / Montgomery -> (n_groups, 2, nlimb-1, N)
        = Rescale(sum over each group of NTT(ct) * pt), NTT domain."""
        n_items, _, nl, N = ct_coef.shape
        ng = -(-n_items // group)
        out = torch.empty((ng, 2, nl - 1, N), dtype=torch.int64, device=self.device)
        _lib.call("bcn_ntt_mac_rescale", self._h, _ptr(out), _ptr(ct_coef), _ptr(pt_mont), n_items, group, nl,
                  _stream())
        return out

    def sample_uniform(self, npoly: int, nlimb: int, prime0: int = 0, seed: int = 0, id0: int = 0) -> torch.Tensor:
        out = torch.empty((npoly, nlimb, self.N), dtype=torch.int64, device=self.device)
        _lib.call("bcn_sample_uniform", self._h, _ptr(out), npoly, nlimb, prime0, seed, id0, _stream())
        return out

    def to_montgomery(self, x: torch.Tensor, prime0: int = 0) -> torch.Tensor:
        npoly, nlimb, N = x.shape
        out = torch.empty_like(x)
        _lib.call("bcn_to_montgomery", self._h, _ptr(out), _ptr(x), npoly, nlimb, prime0, _stream())
        return out

    def automorph(self, x: torch.Tensor, g: int) -> torch.Tensor:
        npoly, nlimb, N = x.shape
        out = torch.empty_like(x)
        _lib.call("bcn_automorph", self._h, _ptr(out), _ptr(x), npoly, nlimb, g, _stream())
        return out

    def freeze(self, delta: int) -> None:
        """+1: a CUDA graph now holds pointers into this context's arenas (growth /
        trim fail with UsageError until released); -1: release."""
        _lib.call("bcn_ctx_freeze", self._h, int(delta))

    def trim(self) -> None:
        _lib.call("bcn_ctx_trim", self._h)

    def memory_bytes(self) -> int:
        b = ctypes.c_uint64()
        _lib.call("bcn_ctx_memory", self._h, ctypes.byref(b))
        return int(b.value)


def to_numpy_u64(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy().view(np.uint64)
