"""ctypes binding of libbcn.so (include/bcn.h).

The extension is mandatory: importing the engine without it raises
DeviceError -- there is no CPU or eager fallback anywhere in the product.
"""

from __future__ import annotations

import ctypes
import os

from .errors import (
    CapacityError,
    DepthBudgetError,
    DeviceError,
    ParameterError,
    UsageError,
)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BCN_LIB") or os.path.join(HERE, "libbcn.so")   # BCN_LIB: experiments only

BCN_OK, BCN_ERR_PARAM, BCN_ERR_DEPTH, BCN_ERR_USAGE, BCN_ERR_CUDA, BCN_ERR_CAPACITY = range(6)
_ERRORS = {
    BCN_ERR_PARAM: ParameterError,
    BCN_ERR_DEPTH: DepthBudgetError,
    BCN_ERR_USAGE: UsageError,
    BCN_ERR_CUDA: DeviceError,
    BCN_ERR_CAPACITY: CapacityError,
}

_P = ctypes.c_void_p
_I = ctypes.c_int
_U64 = ctypes.c_uint64
_D = ctypes.c_double

# name -> argtypes (all return int)
SIGNATURES = {
    "bcn_launch_count": [ctypes.POINTER(_U64)],
    "bcn_plain_conv2d": [_P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _I, _I, _I, _I, _P],
    "bcn_ctx_create": [ctypes.POINTER(_P), _I, _I, ctypes.POINTER(_U64), _I, ctypes.POINTER(_U64), _I, _U64, _I],
    "bcn_ctx_set_fft": [_P, ctypes.POINTER(_D), ctypes.POINTER(_D)],
    "bcn_ctx_destroy": [_P],
    "bcn_ctx_memory": [_P, ctypes.POINTER(_U64)],
    "bcn_ctx_trim": [_P],
    "bcn_ctx_freeze": [_P, _I],
    "bcn_ntt_fwd": [_P, _P, _I, _I, _I, _P],
    "bcn_ntt_inv": [_P, _P, _I, _I, _I, _P],
    "bcn_ntt_timing": [_I],
    "bcn_ntt_timing_read": [ctypes.POINTER(_D), ctypes.POINTER(_U64), ctypes.POINTER(_U64)],
    "bcn_conv_timing": [_I],
    "bcn_conv_timing_read": [ctypes.POINTER(_D), ctypes.POINTER(_U64), ctypes.POINTER(_U64)],
    "bcn_encode": [_P, _P, _I, _I, _I, _D, _I, _I, _P, _P],
    "bcn_encrypt": [_P, _P, _I, _I, _I, _I, _D, _U64, _P, _P],
    "bcn_encrypt_devctr": [_P, _P, _I, _I, _I, _I, _D, _P, _P, _P],
    "bcn_encrypt_rotated": [_P, _P, _I, _I, _I, _I, _D, _U64, _I, _P, _P, _P],
    "bcn_decrypt": [_P, _P, _I, _I, _I, _D, _P, _I, _P],
    "bcn_decrypt_poly": [_P, _P, _I, _I, _I, _P, _P],
    "bcn_add": [_P, _P, _P, _I, _P, _I, _I, _I, _I, _I, _P],
    "bcn_sub": [_P, _P, _P, _I, _P, _I, _I, _I, _P],
    "bcn_mul_plain": [_P, _P, _P, _I, _P, _I, _I, _I, _P],
    "bcn_mul_plain_norescale": [_P, _P, _P, _I, _P, _I, _I, _I, _P],
    "bcn_mac": [_P, _P, _P, _P, _I, _I, _I, _P],
    "bcn_mac_terms": [_P, _P, _I, ctypes.POINTER(_U64), ctypes.POINTER(_U64), ctypes.POINTER(_I), _I, _I, _I, _P],
    "bcn_mac_multi": [_P, _P, _I, _I, ctypes.POINTER(_U64), ctypes.POINTER(_U64), _I, _I, _I, _P],
    "bcn_planes_bytes": [_P, _I, _I, _I, ctypes.POINTER(_U64)],
    "bcn_pack_planes": [_P, _P, _I, _I, ctypes.POINTER(_U64), _I, _P],
    "bcn_mac_multi_planes": [_P, _P, _I, _I, ctypes.POINTER(_U64), _P, _I, _I, _I, _P],
    "bcn_pack_planes_layout": [_P, _P, _I, _I, ctypes.POINTER(_U64), _I, _I, _P],
    "bcn_mac_multi_planes_layout": [_P, _P, _I, _I, ctypes.POINTER(_U64), _P, _I, _I, _I, _I, _P],
    "bcn_mac_terms_acc": [_P, _P, _I, ctypes.POINTER(_U64), ctypes.POINTER(_U64), ctypes.POINTER(_I), _I, _I, _P],
    "bcn_rotsum": [_P, _P, _I, ctypes.POINTER(_U64), ctypes.POINTER(_U64), ctypes.POINTER(_U64),
                   ctypes.POINTER(_U64), ctypes.POINTER(_I), _I, _I, _P],
    "bcn_rotsum_keys": [_P, _P, _I, ctypes.POINTER(_U64), ctypes.POINTER(_U64), ctypes.POINTER(_U64),
                        ctypes.POINTER(_U64), ctypes.POINTER(_I), ctypes.POINTER(_U64), _I, _I, _P],
    "bcn_premul_key": [_P, _P, _U64, _P, _I, _P],
    "bcn_planes_ext_bytes": [_P, _I, _I, _I, ctypes.POINTER(_U64)],
    "bcn_pack_planes_ext": [_P, _P, _I, _I, ctypes.POINTER(_U64), ctypes.POINTER(_I), _I, _I, _P],
    "bcn_conv_ks_mac": [_P, _P, _I, _I, ctypes.POINTER(_U64), ctypes.POINTER(_U64), ctypes.POINTER(_U64), _P, _I,
                        _I, _I, _P],
    "bcn_rotsum_rescale": [_P, _P, _I, ctypes.POINTER(_U64), ctypes.POINTER(_U64), ctypes.POINTER(_U64),
                           ctypes.POINTER(_U64), ctypes.POINTER(_I), ctypes.POINTER(_U64), _I,
                           ctypes.POINTER(_U64), ctypes.POINTER(_U64), ctypes.POINTER(_I), _I, _I, _P],
    "bcn_encode_ext": [_P, _P, _I, _I, _I, _D, _I, _P, _P],
    "bcn_rescale": [_P, _P, _P, _I, _I, _I, _P],
    "bcn_mul_cc": [_P, _P, _P, _I, _P, _I, _I, _I, _I, _P],
    "bcn_modup_words": [_P, _I, _I, ctypes.POINTER(_U64)],
    "bcn_modup": [_P, _P, _P, _I, _I, _I, _P],
    "bcn_rotate_hoisted": [_P, _P, _P, _I, _P, _I, _I, _U64, _P],
    "bcn_rotate": [_P, _P, _P, _I, _I, _I, _U64, _P],
    "bcn_rotate_hoisted_many": [_P, _P, _P, _I, _P, _I, _I, _I, ctypes.POINTER(_U64), _P],
    "bcn_keygen_relin": [_P, _P],
    "bcn_keygen_galois": [_P, _U64, _P],
    "bcn_export_key": [_P, _U64, _P, _P],
    "bcn_export_secret": [_P, _P, _P],
    "bcn_sample_uniform": [_P, _P, _I, _I, _I, _U64, _U64, _P],
    "bcn_to_montgomery": [_P, _P, _P, _I, _I, _I, _P],
    "bcn_automorph": [_P, _P, _P, _I, _I, _U64, _P],
    "bcn_ntt_mac_rescale": [_P, _P, _P, _P, _I, _I, _I, _P],
    # 32-bit-limb variant (own context, bcn32_last_error)
    "bcn32_ctx_create": [ctypes.POINTER(_P), _I, _I, ctypes.POINTER(ctypes.c_uint32), _I],
    "bcn32_ctx_destroy": [_P],
    "bcn32_ntt_fwd": [_P, _P, _I, _P],
    "bcn32_ntt_inv": [_P, _P, _I, _P],
    "bcn32_to_montgomery": [_P, _P, _P, _I, _P],
    "bcn32_ntt_mac_rescale": [_P, _P, _P, _P, _I, _I, _P],
}

_lib = None


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError(
                f"libbcn.so not built at {LIB_PATH}; run __graft_entry__.build() "
                "(the engine has no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        lib.bcn_last_error.restype = ctypes.c_char_p
        lib.bcn_last_error.argtypes = []
        lib.bcn_version.restype = _I
        lib.bcn32_last_error.restype = ctypes.c_char_p
        lib.bcn32_last_error.argtypes = []
        for name, argt in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = _I
            fn.argtypes = argt
        _lib = lib
    return _lib


def exported_symbols() -> list[str]:
    return ["bcn_last_error", "bcn_version", "bcn32_last_error", *SIGNATURES]


def check(code: int, what: str = "") -> None:
    if code != BCN_OK:
        last = load().bcn32_last_error if what.startswith("bcn32_") else load().bcn_last_error
        msg = last().decode(errors="replace")
        raise _ERRORS.get(code, DeviceError)(f"{what}: {msg}" if what else msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def launch_count() -> int:
    v = ctypes.c_uint64()
    call("bcn_launch_count", ctypes.byref(v))
    return int(v.value)


NTT_CLASSES = ("plain_fwd", "plain_inv", "fused_fwd", "fused_inv", "encrypt_fwd")


def ntt_timing(enable: bool) -> None:
    """Bracket every NTT launch with CUDA events (measurement only, bcn.h)."""
    call("bcn_ntt_timing", int(bool(enable)))


def ntt_timing_read() -> dict:
    ms = (ctypes.c_double * 5)()
    nb = (_U64 * 5)()
    nl = (_U64 * 5)()
    call("bcn_ntt_timing_read", ms, nb, nl)
    return {c: {"ms": ms[i], "bytes": int(nb[i]), "launches": int(nl[i])} for i, c in enumerate(NTT_CLASSES)}


CONV_CLASSES = ("staging", "mac")


def conv_timing(enable: bool) -> None:
    """Bracket every conv staging / tensor-core MAC launch with CUDA events (measurement only, bcn.h)."""
    call("bcn_conv_timing", int(bool(enable)))


def conv_timing_read() -> dict:
    ms = (ctypes.c_double * 2)()
    nb = (_U64 * 2)()
    nl = (_U64 * 2)()
    call("bcn_conv_timing_read", ms, nb, nl)
    return {c: {"ms": ms[i], "bytes": int(nb[i]), "launches": int(nl[i])} for i, c in enumerate(CONV_CLASSES)}
