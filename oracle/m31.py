"""TEST INFRASTRUCTURE ONLY. Vectorized F_p, p = 2^31 - 1, and keyed hashes.

Restates paper_2506_15961_b200/csrc/field.hpp in numpy (uint64 arrays holding
residues in [0, p)). Written independently of the product's field.py so the
two can check each other.
"""

from __future__ import annotations

import numpy as np

P = np.uint64(2147483647)
PI = 2147483647
GOLDEN = np.uint64(0x9E3779B97F4A7C15)
VAR_STEP = np.uint64(0xD1B54A32D192ED03)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)
S30, S27, S31, S33 = np.uint64(30), np.uint64(27), np.uint64(31), np.uint64(33)


def mix64(z: np.ndarray) -> np.ndarray:
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> S30)) * M1
        z = (z ^ (z >> S27)) * M2
    return z ^ (z >> S31)


def to_field(h: np.ndarray) -> np.ndarray:
    r = np.asarray(h, dtype=np.uint64) >> S33
    return np.where(r == P, np.uint64(0), r)


def fnv1a64(s: str) -> int:
    h = 0xCBF29CE484222325
    for b in s.encode():
        h = ((h ^ b) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def var_values(seed: int, prefix: str, n: int, witnesses: np.ndarray) -> np.ndarray:
    """(n, W) values of variables prefix.0..prefix.(n-1) at the given witnesses."""
    base = np.uint64((seed ^ fnv1a64("var:" + prefix)) & 0xFFFFFFFFFFFFFFFF)
    i = np.arange(1, n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        keys = mix64(base + i * VAR_STEP)
        w = np.asarray(witnesses, dtype=np.uint64) + np.uint64(1)
        return to_field(mix64(keys[:, None] + w[None, :] * GOLDEN))


def fn_key(seed: int, fn: str) -> np.uint64:
    return mix64(np.uint64((seed ^ fnv1a64("fn:" + fn)) & 0xFFFFFFFFFFFFFFFF))


def uf(seed: int, fn: str, x: np.ndarray) -> np.ndarray:
    k = fn_key(seed, fn)
    with np.errstate(over="ignore"):
        return to_field(mix64(k + np.asarray(x, dtype=np.uint64)))


def add(a, b):
    s = a + b
    return np.where(s >= P, s - P, s)


def sub(a, b):
    return np.where(a >= b, a - b, a + P - b)


def mul(a, b):
    return (a * b) % P   # a, b < 2^31 so the product fits in uint64


def inv(a):
    """Elementwise a^(p-2) (0 -> 0) by square-and-multiply."""
    a = np.asarray(a, dtype=np.uint64)
    result = np.ones_like(a)
    base = a.copy()
    e = PI - 2
    while e:
        if e & 1:
            result = mul(result, base)
        base = mul(base, base)
        e >>= 1
    return result


def const(q) -> np.uint64:
    """Residue of a rational (Fraction/int)."""
    from fractions import Fraction
    q = Fraction(q)
    return np.uint64((q.numerator % PI) * pow(q.denominator % PI, PI - 2, PI) % PI)


def total(xs, axis):
    """Sum mod p along an axis (values < 2^31, chunked to stay below 2^64)."""
    xs = np.asarray(xs, dtype=np.uint64)
    n = xs.shape[axis]
    out = None
    step = 1 << 30
    for lo in range(0, max(n, 1), step):
        part = np.take(xs, range(lo, min(n, lo + step)), axis=axis).sum(axis=axis, dtype=np.uint64) % P
        out = part if out is None else add(out, part)
    if out is None:
        shape = list(xs.shape)
        del shape[axis]
        return np.zeros(shape, dtype=np.uint64)
    return out
