"""RNS-CKKS parameter selection.

The reference sizes the chain as max_level = required_levels(net) + 1
(pkg/src/bibranch/catalog.py:286-346) and carries a single float `scale`
(sim.py:111-121).  Here a level-l ciphertext has limbs q_0..q_l: q_0 is a
`q0_bits` prime, q_1..q_L are `scale_bits` primes (the rescale primes, so
Mul_PC keeps the scale exactly and Mul_CC keeps it to ~2^-30), and
K = ceil((L+1)/dnum) `special_bits` primes extend the basis for hybrid key
switching.  All primes are 1 mod 2N and < 2^61.  q_0 and the specials default
to max(50, scale_bits) bits: a ciphertext never drops below level 1, so
decryption always has q_0 q_1 (>= 2^99) of headroom, and P ~ each digit's
modulus keeps the key-switch noise near 2^18 against Delta = 2^50.  At
scale_bits <= 50 every prime is then below 2^50, which is what lets the
cluster NTT run all limbs on the FP64 pipe (csrc/ntt_cluster.cu).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

_MR_BASES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


def is_prime(n: int) -> bool:
    if n < 2:
        return False
    for b in _MR_BASES:
        if n % b == 0:
            return n == b
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for b in _MR_BASES:
        x = pow(b, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def ntt_primes(bits: int, count: int, N: int, exclude=()) -> list[int]:
    """The `count` largest primes below 2^bits that are 1 mod 2N."""
    if not 20 <= bits <= 60:
        raise ValueError(f"prime size {bits} bits outside [20, 60]")
    out, excl = [], set(exclude)
    step = 2 * N
    q = (1 << bits) - step + 1
    while len(out) < count:
        if q <= (1 << (bits - 1)):
            raise ValueError(f"not enough {bits}-bit primes = 1 mod {step}")
        if q not in excl and is_prime(q):
            out.append(q)
        q -= step
    return out


@dataclass(frozen=True)
class HeParams:
    N: int
    max_level: int
    scale_bits: int
    q0_bits: int = 50
    special_bits: int = 50
    dnum: int = 3
    n_special: int | None = None
    seed: int = 0
    q: tuple = field(default=(), compare=False)
    p: tuple = field(default=(), compare=False)

    @property
    def logn(self) -> int:
        return self.N.bit_length() - 1

    @property
    def alpha(self) -> int:
        return -(-(self.max_level + 1) // self.dnum)

    @property
    def K(self) -> int:
        return len(self.p)

    @property
    def scale(self) -> float:
        return float(2.0 ** self.scale_bits)


def make_params(N: int, max_level: int, scale_bits: int = 50, *, q0_bits: int | None = None,
                special_bits: int | None = None, dnum: int = 3, n_special: int | None = None,
                seed: int = 0) -> HeParams:
    q0_bits = max(50, scale_bits) if q0_bits is None else q0_bits
    special_bits = max(50, scale_bits) if special_bits is None else special_bits
    alpha = -(-(max_level + 1) // dnum)
    K = alpha if n_special is None else n_special
    q0 = ntt_primes(q0_bits, 1, N)
    qs = ntt_primes(scale_bits, max_level, N, exclude=q0) if max_level else []
    sp = ntt_primes(special_bits, K, N, exclude=q0 + qs)
    return HeParams(N=N, max_level=max_level, scale_bits=scale_bits, q0_bits=q0_bits,
                    special_bits=special_bits, dnum=dnum, n_special=n_special, seed=seed,
                    q=tuple(q0 + qs), p=tuple(sp))


def scale_bits_for(scale: float) -> int:
    """CKKS Delta from the reference's `scale` argument: the rescale primes
    are sized to log2(scale), clamped to [20, 58]; scales below 2^20 (the
    reference's unit tests use 1.0, which only feeds its optional rounding
    model, sim.py:244-247) get 2^40."""
    if scale < 2.0 ** 20:
        return 40
    return int(min(58, max(20, round(math.log2(scale)))))


def fft_table(N: int) -> tuple[np.ndarray, np.ndarray]:
    """ksi[k] = exp(2 pi i k / M), M = 2N, k = 0..M -- float64 via numpy
    (the same expression oracle/ckks.py evaluates, so both sides hold the
    same bits)."""
    M = 2 * N
    k = np.arange(M + 1, dtype=np.float64)
    ang = 2.0 * np.pi * k / M
    return np.ascontiguousarray(np.cos(ang)), np.ascontiguousarray(np.sin(ang))


def galois_element(r: int, N: int) -> int:
    """Left rotation by r slots <-> X -> X^(5^r mod 2N) (sim.py:251-256)."""
    return pow(5, r % (N // 2), 2 * N)
