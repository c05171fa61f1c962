"""Host-side definitions of the witness field and keyed hashes.

The field is F_p with p = 2^31 - 1. Everything here must agree bit-for-bit
with csrc/field.hpp (device) -- tests pin the two against each other and
against oracle/m31.py.

Keys:
  var key   = mix64(((seed ^ fnv1a64("var:" + prefix)) + (i + 1) * VAR_STEP) mod 2^64)
              for the variable "<prefix>.<i>"; prefixes follow the reference's
              symbol names ("v.<tid>", "ps.<shard>", stages.py:150 and :168);
  fn key    = mix64(seed ^ fnv1a64("fn:" + NAME))    NAME in EXP, RSQRT, SIGMOID.
Witness value of a variable at witness w: to_field(mix64(key + (w+1)*GOLDEN)).
Uninterpreted function: f(x) = to_field(mix64(fn_key + x)).
"""

from __future__ import annotations

from fractions import Fraction

P = (1 << 31) - 1
MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
FN_NAMES = ("EXP", "RSQRT", "SIGMOID")


def mix64(z: int) -> int:
    z &= MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def fnv1a64(s: str) -> int:
    h = 0xCBF29CE484222325
    for b in s.encode():
        h ^= b
        h = (h * 0x100000001B3) & MASK64
    return h


def to_field(h: int) -> int:
    r = h >> 33
    return 0 if r == P else r


VAR_STEP = 0xD1B54A32D192ED03


def var_key(seed: int, prefix: str, i: int) -> int:
    base = (seed & MASK64) ^ fnv1a64("var:" + prefix)
    return mix64((base + (i + 1) * VAR_STEP) & MASK64)


def fn_key(seed: int, fn: str) -> int:
    return mix64((seed & MASK64) ^ fnv1a64("fn:" + fn))


def fn_keys(seed: int) -> tuple[int, int, int]:
    return tuple(fn_key(seed, f) for f in FN_NAMES)  # type: ignore[return-value]


def witness_value(key: int, w: int) -> int:
    return to_field(mix64((key + (w + 1) * GOLDEN) & MASK64))


def uf_apply(key: int, x: int) -> int:
    return to_field(mix64((key + x) & MASK64))


def residue(q) -> int:
    """Image of a rational in F_p (denominator must be a unit mod p)."""
    q = Fraction(q)
    den = q.denominator % P
    if den == 0:
        raise ZeroDivisionError(f"denominator of {q} is divisible by p")
    return (q.numerator % P) * pow(den, P - 2, P) % P


def const_triple(q) -> tuple[int, int, int]:
    """(residue, exact numerator, exact denominator) for the C-ABI const table.

    Exact parts that do not fit in int64 are dropped (denominator 0 marks the
    constant inexact: its sign is then unknown to the compiler).
    """
    q = Fraction(q)
    lim = (1 << 63) - 1
    if abs(q.numerator) <= lim and q.denominator <= lim:
        return residue(q), q.numerator, q.denominator
    return residue(q), 0, 0
