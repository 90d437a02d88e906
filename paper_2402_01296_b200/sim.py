"""Drop-in for the reference's `bibranch.sim` (pkg/src/bibranch/sim.py), backed
by real RNS-CKKS on the GPU.

Same names, signatures, level algebra, recorder counts and exceptions as the
reference; what changes is what a Ciphertext *is*: a batch of G RLWE
ciphertexts (u64[G, 2, level+1, N], bit-reversed NTT domain) living in HBM,
produced and consumed only by libbcn.so kernels.  `Ciphertext.slots` is a
lazy, read-only decryption (sim.py:128-139 exposes the slots directly).

Execution choices that keep the reference's observable semantics:
  * Lazy linear combinations.  A Mul_PC / rotate-multiply / rotation result
    is returned as an unevaluated term list, logically at the reference's
    level (sim.py:248, 256, 282).  Adding such lists concatenates them, so
    a conv tap loop, an FC diagonal sum, a pooling window or a channel
    concatenation is evaluated by ONE fused kernel, ONE ModDown and ONE
    rescale per output instead of one per product.
  * Rotations are hoisted: ModUp(c1) is computed once per ciphertext and
    shared by all its rotations.  Rotations reused by several outputs
    (multi-channel convs) are materialised once and memoised per (ct, r).
The recorder still counts every reference call exactly (sim.py:209-283).
"""

from __future__ import annotations

import itertools
import os
from collections import OrderedDict
from typing import Union

import numpy as np

from .errors import CapacityError, DepthBudgetError, ParameterError, UsageError
from .params import HeParams, galois_element, make_params, scale_bits_for

# Table-1 CPU latencies of the paper, ms per op; kept for
# the cost model exactly as the reference exposes them (sim.py:26-30).
LATENCY_MS = {
    "BGV": {"Add_PC": 0.049, "Add_CC": 0.077, "Mul_PC": 2.055, "Mul_CC": 3.379},
    "CKKS": {"Add_PC": 0.039, "Add_CC": 0.077, "Mul_PC": 0.173, "Mul_CC": 0.390},
    "TFHE": {"Add_PC": 56.03, "Add_CC": 256.8, "Mul_PC": 1018.0, "Mul_CC": 1585.0},
}
SCHEMES = tuple(LATENCY_MS)
HE_OP_KEYS = ("Add_PC", "Add_CC", "Mul_PC", "Mul_CC")
COUNTER_KEYS = HE_OP_KEYS + ("Rot", "Act_C", "Mul_PC_mask")

PlainLike = Union[np.ndarray, list, tuple]

MAX_RING = 1 << 14

# device work actually issued (after hoisting / memoisation / lazy rescale);
# the recorder keeps the reference's logical counts separately.
STATS = {"modup": 0, "keyswitch": 0, "keyswitch_lazy": 0, "moddown": 0, "rescale": 0, "encode": 0,
         "encode_hit": 0, "mac_launch": 0, "plane_pack": 0, "key_fold": 0}


def _term_batch(term) -> int:
    return int((term[1]._data if term[0] == "rot" else term[1]).shape[0])


def reset_stats() -> None:
    for k in STATS:
        STATS[k] = 0


def _zeros() -> dict:
    return dict.fromkeys(COUNTER_KEYS, 0)


class OpRecorder:
    """Per-op counters with innermost-scope layer attribution (sim.py:47-108).

    Every bump lands in the totals and in exactly one bucket (the innermost
    open layer, else the unscoped remainder), so layer_table() always sums
    to the totals.  merge() folds another recorder in deterministically.
    """

    def __init__(self):
        self.counters = _zeros()
        self.per_layer: list[tuple[str, dict]] = []
        self._open: list[tuple[str, dict]] = []
        self._unscoped = _zeros()
        self._timing = False
        self._events: list[tuple[str, object, object]] = []

    def enable_timing(self, on: bool = True) -> None:
        """Device time per layer scope (no reference counterpart; tracing aid):
        every scope records a CUDA event pair on the current stream and an
        NVTX range, read back by layer_times().  Lazily evaluated terms run in
        the scope that first uses them, so a layer's time is the device work
        issued while it is open."""
        self._timing = on

    def bump(self, key: str, n: int = 1) -> None:
        self.counters[key] += n
        bucket = self._open[-1][1] if self._open else self._unscoped
        bucket[key] += n

    def layer(self, layer_id: str) -> "_Scope":
        return _Scope(self, layer_id)

    @property
    def current_layer(self) -> str | None:
        return self._open[-1][0] if self._open else None

    def merge(self, other: "OpRecorder") -> None:
        for k, v in other.counters.items():
            self.counters[k] += v
        for k, v in other._unscoped.items():
            self._unscoped[k] += v
        self.per_layer.extend((name, dict(d)) for name, d in other.per_layer)

    def layer_table(self) -> list[tuple[str, dict]]:
        rows = [(name, dict(d)) for name, d in self.per_layer]
        if any(self._unscoped.values()):
            rows.append(("(unscoped)", dict(self._unscoped)))
        return rows

    def snapshot(self) -> dict:
        return dict(self.counters)

    def layer_times(self) -> list[tuple[str, float]]:
        """(scope, device ms) in scope-exit order; synchronises the events."""
        out = []
        for name, e0, e1 in self._events:
            e1.synchronize()
            out.append((name, e0.elapsed_time(e1)))
        return out


class _Scope:
    __slots__ = ("rec", "name")

    def __init__(self, rec: OpRecorder, name: str):
        self.rec, self.name = rec, name

    def __enter__(self):
        self.rec._open.append((self.name, _zeros()))
        if self.rec._timing:
            import torch
            torch.cuda.nvtx.range_push(self.name)
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            self.rec._open[-1] = (self.name, self.rec._open[-1][1], ev)
        return self.rec

    def __exit__(self, *exc):
        entry = self.rec._open.pop()
        name, delta = entry[0], entry[1]
        self.rec.per_layer.append((name, delta))
        if len(entry) > 2:
            import torch
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            torch.cuda.nvtx.range_pop()
            self.rec._events.append((name, entry[2], ev))
        return False


class HeContext:
    """Scheme parameters plus the device engine (sim.py:111-125).

    poly_degree / slot_count / max_level / scale / scheme / latency_table /
    noise_model keep the reference's meaning; `he` holds the RNS chain.  The
    libbcn context is created on first use, so parameter validation works on
    a host without a GPU; the first HE op there raises DeviceError.
    """

    def __init__(self, poly_degree, max_level, scale, scheme, latency_table, noise_model, he: HeParams,
                 device=None):
        self.poly_degree = poly_degree
        self.slot_count = poly_degree // 2
        self.max_level = max_level
        self.scale = float(scale)
        self.scheme = scheme
        self.latency_table = latency_table
        self.noise_model = noise_model
        self.he = he
        self._device = device
        self._engine = None
        self._ids = itertools.count()
        self._pt_cache = OrderedDict()
        self._pt_bytes = 0
        self.pt_cache_budget = int(float(os.environ.get("BCN_PT_CACHE_GB", "40")) * 2 ** 30)

    def __repr__(self):
        return (f"HeContext(poly_degree={self.poly_degree}, slot_count={self.slot_count}, "
                f"max_level={self.max_level}, scale={self.scale}, scheme={self.scheme!r})")

    def fresh_id(self) -> str:
        return f"ct{next(self._ids)}"

    @property
    def engine(self):
        if self._engine is None:
            from .engine import Engine
            self._engine = Engine(self.he, self._device)
        return self._engine

    @property
    def delta(self) -> float:
        """CKKS encoding scale of fresh ciphertexts."""
        return self.he.scale

    def q(self, level: int) -> int:
        return self.he.q[level]


class KeyedPlain(np.ndarray):
    """A plain multiplier / addend that carries a cache key.

    Weight-derived vectors (conv taps, masks, FC diagonals) are identical on
    every forward; the engine encodes each (key, level, scale) once and keeps
    the NTT-domain plaintext in HBM (HeContext plaintext cache).  Results of
    arithmetic on a KeyedPlain are ordinary, un-keyed vectors."""

    def __new__(cls, arr, key):
        obj = np.asarray(arr, dtype=np.float64).view(cls)
        obj.bcn_key = key
        return obj

    def __array_finalize__(self, obj):
        self.bcn_key = None


class LazyPlain:
    """A keyed plain vector whose values are only built on a plaintext-cache
    miss (`np.asarray(x)` calls the builder): in steady state a weight-derived
    multiplier is looked up by key alone, and the host never recomputes it."""

    __slots__ = ("bcn_key", "_fn")

    def __init__(self, fn, key):
        self.bcn_key = key
        self._fn = fn

    def __array__(self, dtype=None, copy=None):
        a = np.asarray(self._fn(), dtype=np.float64)
        return a if dtype is None else a.astype(dtype, copy=False)


class Ciphertext:
    """Batch of G RNS-CKKS ciphertexts + logical level / scale / id.

    Immutable from the outside (attribute assignment raises, as for the
    reference's frozen dataclass).  Internally it is either materialised
    (`_data`, exactly level+1 limbs) or a lazy linear combination
    (`_terms`: (ct data, Montgomery plaintext) pairs at data level
    level+1): Mul_PC / rotate-multiply results and sums of them stay lazy
    until something else needs the value, then ONE fused MAC launch plus ONE
    rescale materialises the whole sum.
    """

    __slots__ = ("level", "scale", "id", "ctx", "batch", "_data", "_terms", "_scaled", "_data_scale",
                 "_modup", "_rot", "_slots", "_eager", "__weakref__")

    def __init__(self, data, level: int, scale: float, ctx: HeContext, *, terms=None, scaled=True,
                 data_scale=None, cid: str | None = None):
        s = object.__setattr__
        s(self, "level", level)
        s(self, "scale", float(scale))
        s(self, "id", cid or ctx.fresh_id())
        s(self, "ctx", ctx)
        s(self, "batch", int(data.shape[0]) if data is not None else _term_batch(terms[0]))
        s(self, "_data", data)
        s(self, "_terms", terms)
        s(self, "_scaled", scaled)
        s(self, "_eager", False)
        s(self, "_data_scale", float(scale) if data_scale is None else float(data_scale))
        s(self, "_modup", None)
        s(self, "_rot", {})
        s(self, "_slots", None)

    def __setattr__(self, name, value):
        raise AttributeError("Ciphertext is immutable")

    def __repr__(self):
        return f"Ciphertext(id={self.id!r}, level={self.level}, batch={self.batch})"

    @property
    def pending(self) -> bool:
        return self._terms is not None

    @property
    def data_level(self) -> int:
        return self.level + 1 if (self._terms is not None and self._scaled) else self.level

    def materialize(self) -> "Ciphertext":
        """Evaluate a lazy sum in place (value unchanged): rotation terms by ONE
        lazy-ModDown rotsum, plain-multiplier terms by ONE fused MAC, then one
        rescale if the terms carry multipliers."""
        if self._terms is None:
            return self
        eng = self.ctx.engine
        lvl = self.data_level
        rots = [t for t in self._terms if t[0] == "rot"]
        cts = [t for t in self._terms if t[0] == "ct"]
        out = None
        if rots:
            for t in rots:
                src = t[1]
                if src._modup is None:
                    object.__setattr__(src, "_modup", eng.modup(src._data, src.level))
                    STATS["modup"] += 1
            keys = [_premul_key(self.ctx, t[2], t[3], lvl) if _fold_keys() and t[3] is not None
                    and t[3].shape[0] == 1 else None for t in rots]
            if self._scaled and _merged_rescale():
                # ModDown and rescale in one base conversion
                out = eng.rotsum_rescale([(t[1]._data, t[1]._modup, t[2], t[3]) for t in rots], lvl,
                                         keys=keys if any(k is not None for k in keys) else None,
                                         ct_terms=[(t[1], t[2]) for t in cts])
                STATS["moddown"] += 1
                STATS["keyswitch_lazy"] += len(rots)
                STATS["rescale"] += 1
                STATS["mac_launch"] += 1 if cts else 0
                object.__setattr__(self, "_data", out)
                object.__setattr__(self, "_terms", None)
                object.__setattr__(self, "_data_scale", self.scale)
                return self
            out = eng.rotsum([(t[1]._data, t[1]._modup, t[2], t[3]) for t in rots], lvl,
                             keys=keys if any(k is not None for k in keys) else None)
            STATS["moddown"] += 1
            STATS["keyswitch_lazy"] += len(rots)
        if cts:
            if self._scaled:
                pairs = [(t[1], t[2]) for t in cts]
                out = eng.mac_terms(pairs, lvl, rescale=False) if out is None else eng.mac_terms_acc(out, pairs, lvl)
                STATS["mac_launch"] += 1
            else:
                for t in cts:
                    out = t[1] if out is None else eng.add(out, t[1], lvl)
        if self._scaled:
            out = eng.rescale(out, lvl)
            STATS["rescale"] += 1
        object.__setattr__(self, "_data", out)
        object.__setattr__(self, "_terms", None)
        object.__setattr__(self, "_data_scale", self.scale)
        return self

    @property
    def data(self):
        return self.materialize()._data

    @property
    def slots(self) -> np.ndarray:
        if self._slots is None:
            out = _decrypt(self)
            out.flags.writeable = False
            object.__setattr__(self, "_slots", out)
        return self._slots


# ------------------------------------------------------------- context

def make_context(poly_degree: int, max_level: int, scale: float, scheme: str = "CKKS",
                 noise_model: bool = False, *, dnum: int | None = None, seed: int = 0,
                 q0_bits: int | None = None, special_bits: int | None = None, device=None) -> HeContext:
    """Reference checks (sim.py:142-169) plus the RNS chain (params.py).

    Real CKKS noise replaces the optional fixed-point rounding model, so
    `noise_model` is accepted and has no further effect."""
    if poly_degree < 8 or poly_degree & (poly_degree - 1):
        raise ParameterError(f"poly_degree must be a power of two >= 8, got {poly_degree}")
    if poly_degree > MAX_RING:
        raise ParameterError(f"poly_degree {poly_degree} above the engine maximum {MAX_RING}")
    if max_level < 1:
        raise ParameterError(f"max_level must be >= 1, got {max_level}")
    if not scale > 0:
        raise ParameterError(f"scale must be positive, got {scale}")
    scheme = scheme.upper()
    if scheme not in LATENCY_MS:
        raise ParameterError(f"unknown scheme {scheme!r}; expected one of {SCHEMES}")
    table = dict(LATENCY_MS[scheme])
    table.setdefault("Rot", table["Mul_PC"])
    if dnum is None:
        dnum = min(3, max_level + 1)
    he = make_params(poly_degree, max_level, scale_bits_for(scale), q0_bits=q0_bits,
                     special_bits=special_bits, dnum=dnum, seed=seed)
    return HeContext(poly_degree, max_level, scale, scheme, table, noise_model, he, device)


def encode_plain(v: PlainLike, ctx: HeContext) -> np.ndarray:
    """Zero-pad a real vector (or a (G, n) batch) to the slot width."""
    arr = np.asarray(v, dtype=np.float64)
    if arr.ndim <= 1:
        arr = arr.ravel()
        if arr.size > ctx.slot_count:
            raise CapacityError(f"vector of length {arr.size} exceeds {ctx.slot_count} slots")
        out = np.zeros(ctx.slot_count)
        out[:arr.size] = arr
        return out
    arr = arr.reshape(arr.shape[0], -1)
    if arr.shape[1] > ctx.slot_count:
        raise CapacityError(f"vector of length {arr.shape[1]} exceeds {ctx.slot_count} slots")
    out = np.zeros((arr.shape[0], ctx.slot_count))
    out[:, :arr.shape[1]] = arr
    return out


def _as_plain_rows(v, ctx: HeContext):
    """Host or device plain vector(s) -> 2-D float64 (rows, n<=S)."""
    try:
        import torch
        if isinstance(v, torch.Tensor):
            t = v.to(torch.float64)
            t = t.reshape(1, -1) if t.dim() <= 1 else t.reshape(t.shape[0], -1)
            if t.shape[1] > ctx.slot_count:
                raise CapacityError(f"vector of length {t.shape[1]} exceeds {ctx.slot_count} slots")
            return t
    except ImportError:  # pragma: no cover
        pass
    arr = np.asarray(v, dtype=np.float64)
    arr = arr.reshape(1, -1) if arr.ndim <= 1 else arr.reshape(arr.shape[0], -1)
    if arr.shape[1] > ctx.slot_count:
        raise CapacityError(f"vector of length {arr.shape[1]} exceeds {ctx.slot_count} slots")
    return arr


def encrypt_vector(v: PlainLike, ctx: HeContext, *, level: int | None = None) -> Ciphertext:
    """Encrypt <= slot_count reals (zero-padded) at max_level (sim.py:184-189).
    A 2-D (G, n) input encrypts G independent slot sets in one batch.
    level (engine-internal, forward_bicrypto's prepaid level steps): encrypt
    at a lower level instead."""
    rows = _as_plain_rows(v, ctx)
    if isinstance(rows, np.ndarray):
        if not np.all(np.isfinite(rows)):
            raise ParameterError("plaintext vector must contain only finite values")
    else:
        import torch
        # (no host sync while a CUDA graph is being captured; graph inputs are checked at replay)
        if not torch.cuda.is_current_stream_capturing() and not bool(torch.isfinite(rows).all()):
            raise ParameterError("plaintext vector must contain only finite values")
    eng = ctx.engine
    lv = ctx.max_level if level is None else int(level)
    if not 0 <= lv <= ctx.max_level:
        raise ParameterError(f"level {lv} outside [0, {ctx.max_level}]")
    data = eng.encrypt(rows, lv, ctx.delta)
    return Ciphertext(data, lv, ctx.delta, ctx)


def _decrypt(c: Ciphertext) -> np.ndarray:
    c.materialize()
    out = c.ctx.engine.decrypt(c._data, c.level, c.scale).cpu().numpy()
    return out[0] if c.batch == 1 else out


def decrypt_vector(c: Ciphertext, ctx: HeContext) -> np.ndarray:
    """Decrypt and decode the slots (never consumes level; sim.py:192-196)."""
    if c.ctx is not ctx:
        raise UsageError("ciphertext does not belong to this context")
    return _decrypt(c).copy()


def _same_ctx(a: Ciphertext, b) -> bool:
    if isinstance(b, Ciphertext):
        if a.ctx is not b.ctx:
            raise UsageError("operands come from different contexts")
        return True
    return False


def _depth_error(rec: OpRecorder, ctx: HeContext) -> DepthBudgetError:
    layer = rec.current_layer
    where = f" in layer {layer!r}" if layer else ""
    return DepthBudgetError(f"multiplicative depth exhausted{where}: level is 0 (context max_level={ctx.max_level})")


def _check_scales(sa: float, sb: float) -> None:
    if abs(sa / sb - 1.0) > 1e-6:
        raise UsageError(f"ciphertext scales differ ({sa:.6g} vs {sb:.6g}); CKKS addition needs equal scales")


def _batch_of(a: Ciphertext, b: Ciphertext) -> None:
    if a.batch != b.batch:
        raise UsageError(f"ciphertext batches differ ({a.batch} vs {b.batch})")


def _inplace_adds() -> bool:
    return os.environ.get("BCN_INPLACE_ADD", "1") != "0"


def he_add_plain_many(cts: list, vecs, rec: OpRecorder, *, consume: bool = False) -> list:
    """[he_add(ct_c, vecs[c])] (one Add_PC per channel, sim.py:208-218) with all
    channels' input-dependent plaintexts encoded by ONE batched launch when
    the ciphertexts share level and scale (vecs: (C, G, S) slots)."""
    import torch
    if not cts:
        return []
    for c in cts:
        c.materialize()
    same = isinstance(vecs, torch.Tensor) and all(c.level == cts[0].level and c.scale == cts[0].scale
                                                 and c.batch == cts[0].batch for c in cts)
    if not same or len(cts) == 1:
        return [he_add(ct, vecs[c], rec, consume=consume) for c, ct in enumerate(cts)]
    ctx, lvl, G = cts[0].ctx, cts[0].level, cts[0].batch
    if tuple(vecs.shape[:2]) != (len(cts), G):
        raise UsageError(f"plain batch {tuple(vecs.shape[:2])} does not match ({len(cts)}, {G})")
    pts = ctx.engine.encode(vecs.reshape(len(cts) * G, -1), lvl, cts[0].scale)
    STATS["encode"] += 1
    out = []
    for c, ct in enumerate(cts):
        rec.bump("Add_PC")
        if consume and _inplace_adds() and ct._data.shape[2] == lvl + 1 and not ct._rot:
            data = ctx.engine.add_plain(_consume(ct), pts[c * G:(c + 1) * G], lvl, inplace=True)
        else:
            data = ctx.engine.add_plain(ct._data, pts[c * G:(c + 1) * G], lvl)
        out.append(Ciphertext(data, lvl, ct.scale, ctx))
    return out


def _encode(ctx: HeContext, plain, level: int, scale: float, montgomery: bool, batch: int, ext: bool = False):
    """Encode a plain vector; keyed (weight-derived) vectors are cached in HBM.
    ext=True: Montgomery multiplier over the extended basis (rotsum terms)."""
    key = getattr(plain, "bcn_key", None)
    if key is not None:
        k = (key, level, scale, montgomery, ext)
        hit = ctx._pt_cache.get(k)
        if hit is not None:
            ctx._pt_cache.move_to_end(k)
            STATS["encode_hit"] += 1
            return hit
    rows = _as_plain_rows(plain, ctx)
    if rows.shape[0] not in (1, batch):
        raise UsageError(f"plain batch {rows.shape[0]} does not match ciphertext batch {batch}")
    pt = ctx.engine.encode_ext(rows, level, scale) if ext else ctx.engine.encode(rows, level, scale,
                                                                                  montgomery=montgomery)
    STATS["encode"] += 1
    if key is not None:
        _cache_put(ctx, k, pt)
    return pt


def _entry_bytes(v) -> int:
    t = v[0] if isinstance(v, tuple) else v
    return t.numel() * t.element_size()


def _cache_put(ctx: HeContext, k, v) -> None:
    """LRU insert into the HBM plaintext cache (budget BCN_PT_CACHE_GB)."""
    ctx._pt_cache[k] = v
    ctx._pt_bytes += _entry_bytes(v)
    while ctx._pt_bytes > ctx.pt_cache_budget and len(ctx._pt_cache) > 1:
        _, old = ctx._pt_cache.popitem(last=False)
        ctx._pt_bytes -= _entry_bytes(old)


def _use_imma() -> bool:
    return os.environ.get("BCN_MAC_IMMA", "1") != "0"


def _merged_rescale() -> bool:
    return os.environ.get("BCN_MERGED_RESCALE", "1") != "0"


def _fold_keys() -> bool:
    return os.environ.get("BCN_FOLD_KEYS", "1") != "0"


def _premul_key(ctx: HeContext, g: int, pt, level: int):
    """Galois key with a constant multiplier folded in (rotsum), cached next
    to the plaintexts; the entry pins the plaintext object it was made from."""
    key = ("premul", int(g), id(pt), level)
    hit = ctx._pt_cache.get(key)
    if hit is not None and hit[1][0] is pt:
        ctx._pt_cache.move_to_end(key)
        return hit[0]
    k = ctx.engine.premul_key(g, pt, level)
    STATS["key_fold"] += 1
    _cache_put(ctx, key, (k, [pt]))
    return k


def _conv_layout(G: int) -> int:
    """Plane layout of the conv MAC: tcgen05.mma (M = 64 slot sets x 2
    components per pass) once there are enough slot sets to fill it, else
    mma.sync IMMA.  BCN_TCGEN05=0/1 forces either."""
    v = os.environ.get("BCN_TCGEN05", "auto")
    if v in ("0", "1"):
        return int(v)
    return 1 if G >= 64 else 0


def _planes_for(ctx: HeContext, pts: list, level: int, ext: bool = False, layout: int = 0):
    """Byte planes of an O x K plaintext matrix for the tensor-core MAC, packed
    once and cached next to the plaintexts.  The entry keeps the plaintext
    tensors alive and is only reused for the very same objects."""
    key = ("planes_ext" if ext else "planes", level, layout, tuple(id(p) for row in pts for p in row))
    hit = ctx._pt_cache.get(key)
    if hit is not None and all(a is b for a, b in zip(hit[1], (p for row in pts for p in row))):
        ctx._pt_cache.move_to_end(key)
        return hit[0]
    planes = ctx.engine.pack_planes_ext(pts, level, layout) if ext else ctx.engine.pack_planes(pts, level, layout)
    STATS["plane_pack"] += 1
    _cache_put(ctx, key, (planes, [p for row in pts for p in row]))
    return planes


def _consume(a: Ciphertext):
    """Take over a's buffer for an in-place update: `a` itself becomes unusable
    (any later read raises instead of seeing the modified words)."""
    d = a._data
    object.__setattr__(a, "_data", None)
    object.__setattr__(a, "_terms", None)
    object.__setattr__(a, "_modup", None)
    return d


def he_add(a: Ciphertext, b, rec: OpRecorder, *, consume: bool = False) -> Ciphertext:
    """Add_CC (level = min) or Add_PC (level kept), sim.py:208-218.
    consume (engine-internal, Add_PC only): the caller drops `a` -- a fresh
    layer output nothing else references -- so the sum is written into a's own
    buffer (no copy of component 1, no second ciphertext in HBM)."""
    ctx = a.ctx
    eng = ctx.engine
    if _same_ctx(a, b):
        rec.bump("Add_CC")
        _batch_of(a, b)
        level = min(a.level, b.level)
        if a.pending and b.pending and a.level == b.level and a._scaled == b._scaled:
            _check_scales(a._data_scale, b._data_scale)
            return Ciphertext(None, level, a.scale, ctx, terms=a._terms + b._terms, scaled=a._scaled,
                              data_scale=a._data_scale)
        if a.level == b.level and (a.pending != b.pending):
            lazy, done = (a, b) if a.pending else (b, a)
            if not lazy._scaled:        # rotation sum + a materialised ciphertext: still one ModDown
                _check_scales(lazy.scale, done.scale)
                return Ciphertext(None, level, a.scale, ctx, terms=lazy._terms + (("ct", done._data, None),),
                                  scaled=False)
        a.materialize()
        b.materialize()
        _check_scales(a.scale, b.scale)
        return Ciphertext(eng.add(a._data, b._data, level), level, a.scale, ctx)
    rec.bump("Add_PC")
    a.materialize()       # a lazy sum's scale Delta*q_l would overflow a 64-bit encoding
    pt = _encode(ctx, b, a.level, a.scale, False, a.batch)
    if consume and _inplace_adds() and a._data.shape[2] == a.level + 1 and not a._rot:
        return Ciphertext(eng.add_plain(_consume(a), pt, a.level, inplace=True), a.level, a.scale, ctx)
    return Ciphertext(eng.add_plain(a._data, pt, a.level), a.level, a.scale, ctx)


def _times_plain(x: Ciphertext, plain) -> Ciphertext:
    """x (materialised, at level l) times a multiplier encoded at scale q_l:
    a one-term lazy sum at logical level l-1 with the scale kept exactly."""
    ctx = x.ctx
    level = x.level
    ql = ctx.q(level)
    pt = _encode(ctx, plain, level, float(ql), True, x.batch)
    return Ciphertext(None, level - 1, x.scale, ctx, terms=(("ct", x._data, pt),), data_scale=x.scale * float(ql))


def _distributes(a: Ciphertext) -> bool:
    """An unscaled lazy sum whose terms all sit at its level (sum_pool's
    rotations + identity) can take a multiplier term by term."""
    if os.environ.get("BCN_DISTRIBUTE_MUL", "1") == "0":
        return False
    for t in a._terms:
        if t[0] == "ct" and t[1].shape[2] != a.level + 1:
            return False
        if t[0] == "rot" and t[1].level != a.level:
            return False
    return True


def _lazy_times_plain(a: Ciphertext, plain) -> Ciphertext:
    """(sum_t term_t) * plain as the scaled lazy sum sum_t term_t * plain: the
    rotations keep their deferred ModDown, which the later materialisation
    merges with the rescale (one base conversion)."""
    ctx = a.ctx
    level = a.level
    ql = float(ctx.q(level))
    has_ct = any(t[0] == "ct" for t in a._terms)
    has_rot = any(t[0] == "rot" for t in a._terms)
    pt = _encode(ctx, plain, level, ql, True, a.batch) if has_ct else None
    pt_ext = _encode(ctx, plain, level, ql, True, a.batch, ext=True) if has_rot else None
    terms = tuple(("ct", t[1], pt) if t[0] == "ct" else ("rot", t[1], t[2], pt_ext) for t in a._terms)
    return Ciphertext(None, level - 1, a.scale, ctx, terms=terms, data_scale=a.scale * ql)


def _rot_times_plain(c: Ciphertext, r: int, plain) -> Ciphertext:
    """rotate(c, r) * plain as a lazy rotation term (ModDown deferred to the sum)."""
    ctx = c.ctx
    level = c.level
    ql = ctx.q(level)
    pt = _encode(ctx, plain, level, float(ql), True, c.batch, ext=True)
    g = galois_element(r, ctx.poly_degree)
    return Ciphertext(None, level - 1, c.scale, ctx, terms=(("rot", c, g, pt),), data_scale=c.scale * float(ql))


def he_mul(a: Ciphertext, b, rec: OpRecorder, *, mask: bool = False) -> Ciphertext:
    """Slot-wise product, result level = min(levels) - 1 (sim.py:221-248).

    ct x plain: multiplier encoded at scale q_level, product rescaled by
    q_level (lazily), so the scale is kept exactly.  ct x ct: tensor product,
    relinearisation (hybrid key switch), rescale."""
    ctx = a.ctx
    is_cc = _same_ctx(a, b)
    lvl = min(a.level, b.level) if is_cc else a.level
    if lvl < 1:
        raise _depth_error(rec, ctx)
    if is_cc:
        rec.bump("Mul_CC")
    else:
        rec.bump("Mul_PC")
        if mask:
            rec.bump("Mul_PC_mask")
    if not is_cc and a.pending and not a._scaled and _distributes(a):
        return _lazy_times_plain(a, b)
    a.materialize()
    if not is_cc:
        return _times_plain(a, b)
    _batch_of(a, b)
    b.materialize()
    data = ctx.engine.mul_cc(a._data, b._data, lvl)
    STATS["modup"] += 1
    STATS["keyswitch"] += 1
    STATS["rescale"] += 1
    return Ciphertext(data, lvl - 1, (a.scale * b.scale) / ctx.q(lvl), ctx)


def he_square_many(cts: list, rec: OpRecorder) -> list:
    """[he_mul(c, c)] for the channels of one layer (one Mul_CC each, sim.py:221-248).
    Below BCN_CONV_TC_MIN_G slot sets (the single-image path, where every launch is a
    latency, not a throughput) channels that share level, scale and shape run as ONE
    Mul_CC call on the stacked batch: slot sets are independent, so every channel's
    ciphertext is bit-identical to its own call."""
    first = cts[0] if cts else None
    small = bool(cts) and small_batch(cts) and os.environ.get("BCN_BATCH_SQUARE", "1") != "0"
    if small:
        for c in cts:
            c.materialize()
        small = all(c.ctx is first.ctx and c.level == first.level and c.scale == first.scale
                    and c._data.shape == first._data.shape for c in cts)
    if not small:
        return [he_mul(c, c, rec) for c in cts]
    ctx, lvl, G = first.ctx, first.level, first.batch
    if lvl < 1:
        raise _depth_error(rec, ctx)
    import torch

    rec.bump("Mul_CC", len(cts))
    stacked = torch.cat([c._data for c in cts], 0)
    data = ctx.engine.mul_cc(stacked, stacked, lvl)
    STATS["modup"] += 1
    STATS["keyswitch"] += 1
    STATS["rescale"] += 1
    scale = (first.scale * first.scale) / ctx.q(lvl)
    return [Ciphertext(data[i * G:(i + 1) * G], lvl - 1, scale, ctx) for i in range(len(cts))]


def small_batch(cts: list) -> bool:
    """The single-image regime (fewer than BCN_CONV_TC_MIN_G slot sets): every launch is a
    latency, so per-channel work is worth stacking into one batch."""
    return (len(cts) > 1 and os.environ.get("BCN_BATCH_CHANNELS", "1") != "0"
            and cts[0].batch < int(os.environ.get("BCN_CONV_TC_MIN_G", "4")))


def stack_batch(cts: list):
    """The channels' ciphertexts as ONE ciphertext whose batch is their slot sets back to
    back (slot sets are independent, so any op on it is the op on every channel), or None
    when they do not share context, level, scale and shape."""
    import torch

    first = cts[0]
    for c in cts:
        c.materialize()
    if not all(c.ctx is first.ctx and c.level == first.level and c.scale == first.scale
               and c._data.shape == first._data.shape for c in cts):
        return None
    return Ciphertext(torch.cat([c._data for c in cts], 0), first.level, first.scale, first.ctx)


def split_batch(ct: Ciphertext, n: int, *, modup: bool = False) -> list:
    """Inverse of stack_batch: n ciphertexts viewing ct's slot sets.  modup: the ModUp of the
    whole stacked batch is computed once and each piece gets its slice (for pieces that are
    about to be rotated)."""
    ct.materialize()
    G = ct.batch // n
    outs = [Ciphertext(ct._data[i * G:(i + 1) * G], ct.level, ct.scale, ct.ctx) for i in range(n)]
    if modup:
        U = ct.ctx.engine.modup(ct._data, ct.level).view(ct.batch, -1)
        STATS["modup"] += 1
        for i, o in enumerate(outs):
            object.__setattr__(o, "_modup", U[i * G:(i + 1) * G])
    return outs


def he_mul_support_mask(a: Ciphertext, rec: OpRecorder, *, drop: bool = True) -> Ciphertext:
    """he_mul(a, mask, mask=True) for a 0/1 mask that is 1 on a's whole slot
    support (a conv layer's output mask: every tap pattern is already zero off
    the output grid, layers.py _tap_pattern): value-preserving, so it is
    realised as the level step alone -- the top RNS limb is discarded (an
    exact modulus switch of a CKKS ciphertext, scale unchanged) instead of a
    plaintext product and a rescale.  Same counts (Mul_PC, Mul_PC_mask) and
    level algebra as sim.py:221-248; the off-grid slots keep their CKKS noise
    instead of being zeroed, and no later layer reads them (their taps read
    input-grid anchors only).  drop=False: the level step was taken in advance
    (forward_bicrypto's prepaid levels) -- counts only."""
    rec.bump("Mul_PC")
    rec.bump("Mul_PC_mask")
    if not drop:                 # the level step was prepaid (forward_bicrypto encrypted lower)
        return a.materialize()
    if a.level < 1:
        raise _depth_error(rec, a.ctx)
    return he_drop_levels(a, 1, rec)


def he_drop_levels(a: Ciphertext, n: int, rec: OpRecorder) -> Ciphertext:
    """a at level - n with the same value and scale: the top n RNS limbs are
    discarded (an exact modulus switch of a CKKS ciphertext, no rescale).  The
    engine's stand-in for reference ops whose level step it realises without
    work (he_mul_support_mask, layers.flatten_packed); DepthBudgetError as
    he_mul would raise it."""
    ctx = a.ctx
    if a.level < n:
        raise _depth_error(rec, ctx)
    a.materialize()
    if n == 0:
        return a
    return Ciphertext(a._data[:, :, :a.level + 1 - n].contiguous(), a.level - n, a.scale, ctx)


def _rotated(c: Ciphertext, r: int) -> Ciphertext:
    """Memoised, hoisted rotation of a materialised ciphertext (r reduced)."""
    ctx = c.ctx
    c.materialize()
    hit = c._rot.get(r)
    if hit is not None:
        return hit
    eng = ctx.engine
    if r == 0:
        out = Ciphertext(c._data, c.level, c.scale, ctx)
    else:
        if c._modup is None:
            object.__setattr__(c, "_modup", eng.modup(c._data, c.level))
            STATS["modup"] += 1
        data = eng.rotate(c._data, r, c.level, U=c._modup)
        STATS["keyswitch"] += 1
        out = Ciphertext(data, c.level, c.scale, ctx)
    c._rot[r] = out
    return out


def _rotate_many(c: Ciphertext, rs) -> None:
    """Fill c's rotation memo for every r in rs with ONE bcn_rotate_hoisted_many call (the
    source's ModUp digits read once, every ModDown in one launch); each entry is bit-identical
    to what _rotated(c, r) would have computed."""
    c.materialize()
    rs = [r for r in dict.fromkeys(int(r) for r in rs) if r != 0 and r not in c._rot]
    if len(rs) < 2 or os.environ.get("BCN_ROT_MANY_BSGS", "1") == "0":
        return
    eng = c.ctx.engine
    if c._modup is None:
        object.__setattr__(c, "_modup", eng.modup(c._data, c.level))
        STATS["modup"] += 1
    data = eng.rotate_many(c._data, rs, c.level, U=c._modup)
    STATS["keyswitch"] += len(rs)
    for k, r in enumerate(rs):
        c._rot[r] = Ciphertext(data[k], c.level, c.scale, c.ctx)


def release(c: Ciphertext) -> None:
    """Drop the hoisting / memo buffers of a ciphertext (device memory)."""
    object.__setattr__(c, "_modup", None)
    c._rot.clear()


def he_rotate(c: Ciphertext, r: int, rec: OpRecorder) -> Ciphertext:
    """Left rotation by r slots (right for r < 0), level unchanged (sim.py:251-256).
    Unless the source is marked for reuse, the result is a lazy rotation term:
    sums of rotations (sum_pool, concat_flat) then share ONE ModDown."""
    rec.bump("Rot")
    r = int(r) % c.ctx.slot_count
    c.materialize()
    if r == 0 or c._eager or r in c._rot:
        src = _rotated(c, r)
        return Ciphertext(src._data, src.level, src.scale, c.ctx)
    g = galois_element(r, c.ctx.poly_degree)
    return Ciphertext(None, c.level, c.scale, c.ctx, terms=(("rot", c, g, None),), scaled=False)


def he_rotate_mul(c: Ciphertext, r: int, plain, rec: OpRecorder, *, mask: bool = False) -> Ciphertext:
    """he_mul(he_rotate(c, r), plain): one Rot + one Mul_PC, level - 1 (sim.py:259-283)."""
    if c.level < 1:
        raise _depth_error(rec, c.ctx)
    rec.bump("Rot")
    rec.bump("Mul_PC")
    if mask:
        rec.bump("Mul_PC_mask")
    r = int(r) % c.ctx.slot_count
    c.materialize()
    if r == 0 or c._eager or r in c._rot:
        return _times_plain(_rotated(c, r), plain)
    return _rot_times_plain(c, r, plain)


def linear_bsgs(parts, rec: OpRecorder) -> Ciphertext:
    """sum over parts and generalised diagonals d of rot_d(x) * v_d, by
    baby-step / giant-step (Halevi-Shoup): with D diagonals per part and
    b = ceil(sqrt(D)) baby steps,
        sum_d v_d rot_d(x) = sum_j rot_{R_j}( sum_i roll(v_{R_j+i}, R_j) * rot_i(x) ),
    R_j = d_min + j b.  Key switches per part: b - 1 hoisted baby rotations +
    ~D/b giant rotations, all giant rotations sharing ONE lazy ModDown, and one
    rescale -- instead of D key switches.  The caller bumps the reference's
    per-diagonal counts (layers.py:275-314); depth semantics are he_rotate_mul's.

    parts: [(x Ciphertext, [(d, vector, key)])]."""
    import math
    ctx = parts[0][0].ctx
    eng = ctx.engine
    S = ctx.slot_count
    x0 = parts[0][0]
    if x0.level < 1:
        raise _depth_error(rec, ctx)
    giants = []          # (baby-step terms of P_j, R_j)
    level = None
    for x, diags in parts:
        x.materialize()
        level = x.level if level is None else level
        if x.level != level:
            raise UsageError("FC blocks must share one level")
        mark_reused(x)
        dmin = min(d for d, _, _ in diags)
        D = max(d for d, _, _ in diags) - dmin + 1
        b = max(1, math.isqrt(D - 1) + 1) if D > 1 else 1
        by_d = {d: (v, key) for d, v, key in diags}
        ql = ctx.q(level)
        _rotate_many(x, [i % S for j in range(-(-D // b)) for i in range(b) if dmin + j * b + i in by_d])
        for j in range(-(-D // b)):
            R = dmin + j * b
            pairs = []
            for i in range(b):
                d = R + i
                if d not in by_d:
                    continue
                v, key = by_d[d]
                pv = KeyedPlain(np.roll(v, R % S), key + ("bsgs", R)) if key is not None else np.roll(v, R % S)
                pt = _encode(ctx, pv, level, float(ql), True, x.batch)
                pairs.append((_rotated(x, i % S)._data, pt))
            if pairs:
                giants.append((pairs, R % S))
    # every giant's partial sum into one buffer, the rotated ones first: ONE ModUp launch
    # sequence for all of them (a slot-set batch of n_rot x G) instead of one per giant
    import torch
    giants.sort(key=lambda t: t[1] == 0)
    n_rot = sum(1 for _, R in giants if R)
    G = x0.batch
    buf = torch.empty((len(giants), G, 2, level + 1, ctx.poly_degree), dtype=torch.int64, device=x0._data.device)
    for k, (pairs, _) in enumerate(giants):
        eng.mac_terms(pairs, level, rescale=False, out=buf[k])
        STATS["mac_launch"] += 1
    rot_terms = []
    out = None
    if n_rot:
        U = eng.modup(buf[:n_rot].view(n_rot * G, 2, level + 1, ctx.poly_degree), level).view(n_rot * G, -1)
        STATS["modup"] += n_rot
    for k, (_, R) in enumerate(giants):
        if R == 0:
            out = buf[k] if out is None else eng.add(out, buf[k], level)
        else:
            rot_terms.append((buf[k], U[k * G:(k + 1) * G], galois_element(R, ctx.poly_degree), None))
    if rot_terms:
        rs = eng.rotsum(rot_terms, level)
        STATS["moddown"] += 1
        STATS["keyswitch_lazy"] += len(rot_terms)
        out = rs if out is None else eng.add(out, rs, level)
    out = eng.rescale(out, level)
    STATS["rescale"] += 1
    return Ciphertext(out, level - 1, x0.scale, ctx)


def materialize_group(cts: list) -> None:
    """Evaluate several lazy sums that share their ciphertext terms (the output
    channels of one conv layer) with one multi-output MAC pass and one batched
    rescale; anything that does not fit that pattern is materialised alone."""
    lazy = [c for c in cts if c.pending]
    if len(lazy) > 1:
        first = lazy[0]
        ref = [id(t[1]) for t in first._terms] if all(t[0] == "ct" for t in first._terms) else None
        same = ref is not None and all(
            c._scaled and c.level == first.level and len(c._terms) == len(ref)
            and all(t[0] == "ct" and id(t[1]) == r and t[2].shape[0] == 1 for t, r in zip(c._terms, ref))
            for c in lazy)
        if same and first._scaled:
            eng = first.ctx.engine
            lvl = first.data_level
            cts_k = [t[1] for t in first._terms]
            pts_ok = [[t[2] for t in c._terms] for c in lazy]
            # fewer than BCN_CONV_TC_MIN_G slot sets fill 2 G of the tensor-core MAC's 32+ columns:
            # the CUDA-core multi-output MAC is faster there (config-1 latency 3.56 -> 2.86 ms)
            small = int(cts_k[0].shape[0]) < int(os.environ.get("BCN_CONV_TC_MIN_G", "4"))
            if _use_imma() and len(cts_k) <= 256 and not small:
                layout = _conv_layout(int(cts_k[0].shape[0]))
                out = eng.mac_multi_planes(cts_k, _planes_for(first.ctx, pts_ok, lvl, layout=layout), len(lazy), lvl,
                                           layout=layout)
            else:
                out = eng.mac_multi(cts_k, pts_ok, lvl)
            STATS["mac_launch"] += 1
            STATS["rescale"] += len(lazy)
            for c, d in zip(lazy, out):
                object.__setattr__(c, "_data", d)
                object.__setattr__(c, "_terms", None)
                object.__setattr__(c, "_data_scale", c.scale)
    for c in cts:
        c.materialize()


def lazy_conv_enabled() -> bool:
    return os.environ.get("BCN_LAZY_CONV", "1") != "0"


def materialize_conv(accs: list) -> bool:
    """Evaluate the output channels of a conv layer whose taps are lazy
    rotation terms ("rot", x, g, pt_ext) and identity terms ("ct", x, pt) over
    the same (source, rotation) list: key-switch inner products fused into the
    tensor-core MAC over the extended basis, then ONE merged ModDown+rescale
    per output (bcn_conv_ks_mac) -- no ModDown per rotation.
    Returns False (nothing done) when the sums do not have that shape."""
    lazy = [c for c in accs if c.pending]
    if len(lazy) != len(accs) or len(lazy) < 2:
        return False
    first = lazy[0]
    if not first._scaled or len(first._terms) > 256:
        return False
    if not any(t[0] == "rot" for t in first._terms):
        return False                       # no key switching at all: the multi-output MAC (materialize_group)

    def sig(t):
        return (id(t[1]), t[2]) if t[0] == "rot" else (id(t[1]), 1)

    ref = [sig(t) for t in first._terms]
    for c in lazy:
        if not c._scaled or c.level != first.level or len(c._terms) != len(ref):
            return False
        for t, r in zip(c._terms, ref):
            if sig(t) != r or (t[0] == "rot" and (t[3] is None or t[3].shape[0] != 1)) or \
                    (t[0] == "ct" and t[2].shape[0] != 1):
                return False
    ctx = first.ctx
    eng = ctx.engine
    lvl = first.data_level
    srcs, Us, gals = [], [], []
    for t in first._terms:
        if t[0] == "rot":
            src = t[1]
            if src.level != lvl:
                return False
            if src._modup is None:
                object.__setattr__(src, "_modup", eng.modup(src._data, src.level))
                STATS["modup"] += 1
            srcs.append(src._data)
            Us.append(src._modup)
            gals.append(int(t[2]))
        else:
            if t[1].shape[2] != lvl + 1:
                return False
            srcs.append(t[1])
            Us.append(None)
            gals.append(1)
    if int(srcs[0].shape[0]) < int(os.environ.get("BCN_CONV_TC_MIN_G", "4")):
        # a handful of slot sets (single-image latency) fills a tiny fraction of the
        # tensor-core tiles (M = 2G columns): one CUDA-core rotation sum per output is faster
        return False
    pts = [[t[3] if t[0] == "rot" else t[2] for t in c._terms] for c in lazy]
    layout = _conv_layout(int(srcs[0].shape[0]))
    out = eng.conv_ks_mac(srcs, Us, gals, _planes_for(ctx, pts, lvl, ext=True, layout=layout), len(lazy), lvl,
                          layout)
    STATS["mac_launch"] += 1
    STATS["moddown"] += len(lazy)
    STATS["keyswitch_lazy"] += sum(g != 1 for g in gals)
    STATS["rescale"] += len(lazy)
    for c, d in zip(lazy, out):
        object.__setattr__(c, "_data", d)
        object.__setattr__(c, "_terms", None)
        object.__setattr__(c, "_data_scale", c.scale)
    return True


def mark_reused(c: Ciphertext) -> None:
    """Rotations of c will be reused by several outputs (multi-channel conv):
    materialise and memoise them instead of deferring their ModDown."""
    object.__setattr__(c, "_eager", True)
