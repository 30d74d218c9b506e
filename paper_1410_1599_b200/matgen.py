"""Seeded MP inputs (matgen.hpp:13-52 and the BASELINE configs' distributions).

All generators are integer code in libmpgpu's host part (mpgpu_gen); they produce
the same values on every platform:

  gen_random        matgen.hpp:45-52: x = RN_p((2k - 2^53) / 2^53), k = top53() (reference)
  gen_uniform_full  full-mantissa uniform [-1,1): x = (k - 2^p)/2^p, k = the top p+1 bits
                    of the concatenated top53() draws (first draw most significant); exact
  gen_scaled        BASELINE config 3: sign = next64()>>63, e = next64() % 41 - 20,
                    mantissa 2^(p-1) + (p-1 random bits from top53() draws); x = +-m/2^p * 2^e
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as _L
from .mpmm import EXP_ZERO, DomainError, Matrix, PrecisionContext

MASK64 = (1 << 64) - 1


class Prng64:
    """xorshift64* (matgen.hpp:13-42); seed 0 is remapped."""

    def __init__(self, seed: int):
        self.s = (seed & MASK64) or 0x9E3779B97F4A7C15

    def next64(self) -> int:
        x = self.s
        x ^= x >> 12
        x ^= (x << 25) & MASK64
        x ^= x >> 27
        self.s = x
        return (x * 2685821657736338717) & MASK64

    def top53(self) -> int:
        return self.next64() >> 11


def _gen(kind: int, rows: int, cols: int, seed: int, ctx: PrecisionContext) -> Matrix:
    out = Matrix(rows, cols, ctx)
    n = rows * cols
    rc = _L.lib.mpgpu_gen(kind, n, seed & MASK64, ctx.bits(), C.c_void_p(out.limbs.ctypes.data),
                          C.c_void_p(out.exp.ctypes.data), C.c_void_p(out.sign.ctypes.data), out.nlimbs)
    if rc:
        raise DomainError(f"mpgpu_gen failed ({rc})")
    return out


def gen_random(rows: int, cols: int, seed: int, ctx: PrecisionContext) -> Matrix:
    """matgen.hpp:45-52 (53-bit dyadic uniforms, exact products at p >= 128)."""
    return _gen(0, rows, cols, seed, ctx)


def gen_uniform_full(rows: int, cols: int, seed: int, ctx: PrecisionContext) -> Matrix:
    """Uniform [-1,1) with all p mantissa bits random (BASELINE configs 1, 2, 4, 5a)."""
    return _gen(1, rows, cols, seed, ctx)


def gen_scaled(rows: int, cols: int, seed: int, ctx: PrecisionContext) -> Matrix:
    """Mantissa in [1/2,1) fully random, exponent in [-20,20], random sign (config 3)."""
    return _gen(2, rows, cols, seed, ctx)


def from_ints(values, ctx: PrecisionContext, rows: int = None, cols: int = None) -> Matrix:
    """Exact small integers (|v| < 2^62) -> Matrix at ctx (mpfr_set_si; p >= 63 keeps
    them exact, smaller p rounds to nearest-even)."""
    v = np.asarray(values, dtype=np.int64)
    if rows is None:
        rows, cols = v.shape if v.ndim == 2 else (v.size, 1)
    v = v.reshape(-1)
    out = Matrix(rows, cols, ctx)
    L = out.nlimbs
    p = ctx.bits()
    for e, x in enumerate(v.tolist()):
        if x == 0:
            continue
        s = 1 if x < 0 else 0
        u = -x if x < 0 else x
        b = u.bit_length()
        ex = b
        if b > p:  # round to nearest even at p bits
            drop = b - p
            low = u & ((1 << drop) - 1)
            u >>= drop
            half = 1 << (drop - 1)
            if low > half or (low == half and (u & 1)):
                u += 1
                if u.bit_length() > p:
                    u >>= 1
                    ex += 1
            b = u.bit_length()
        mant = u << (32 * L - b)
        for k in range(L):
            out.limbs[k, e] = (mant >> (32 * k)) & 0xFFFFFFFF
        out.exp[e] = ex
        out.sign[e] = s
    return out


def to_fractions(x: Matrix):
    """Exact values as Python Fractions (tests / small cases)."""
    from fractions import Fraction
    L = x.nlimbs
    out = []
    for e in range(x.rows() * x.cols()):
        if x.exp[e] == EXP_ZERO:
            out.append(Fraction(0))
            continue
        m = 0
        for k in range(L - 1, -1, -1):
            m = (m << 32) | int(x.limbs[k, e])
        v = Fraction(m, 1 << (32 * L)) * (Fraction(2) ** int(x.exp[e]))
        out.append(-v if x.sign[e] else v)
    return out
