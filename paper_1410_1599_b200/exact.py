"""Exact host-side scalar arithmetic for the benchmark driver's closed-form inputs and
for decimal output (Python integers; no MPFR).

The benchmark operands and references (matgen.hpp:63-121) are correctly rounded
values of simple closed forms -- sqrt(k) times an integer, 1/q, integers -- with few
distinct values per matrix (a_ij depends on i+j, b_ij and c_ij on i).  They are
produced here exactly, one value per distinct entry, and scattered into SoA
matrices with numpy; the O(n^3) work stays on the device.

Values are (sign, M, e): x = (-1)^sign * M * 2^(e - p) with 2^(p-1) <= M < 2^p, i.e.
MPFR's convention x = 0.m * 2^e (precision.hpp:42-109); None is +0.
"""
from __future__ import annotations

import math
from fractions import Fraction
from typing import List, Optional, Sequence, Tuple

import numpy as np

from .mpmm import EXP_ZERO, Matrix, PrecisionContext

Value = Optional[Tuple[int, int, int]]


def _round_shift(u: int, drop: int, sticky: bool) -> Tuple[int, bool]:
    """RN-even of u / 2^drop (drop >= 1) with an extra sticky flag below u."""
    low = u & ((1 << drop) - 1)
    q = u >> drop
    half = 1 << (drop - 1)
    if low > half or (low == half and (sticky or (q & 1))):
        q += 1
    return q, False


def rn_scaled(num: int, sh: int, p: int, sticky: bool = False) -> Value:
    """RN_p(num * 2^sh) (num an integer; sticky: a nonzero fraction below num's LSB)."""
    if num == 0:
        return None
    s = 1 if num < 0 else 0
    u = -num if num < 0 else num
    b = u.bit_length()
    e = b + sh
    if b > p:
        M, _ = _round_shift(u, b - p, sticky)
        if M >> p:
            M >>= 1
            e += 1
    else:
        M = u << (p - b)
    return (s, M, e)


def rn_fraction(num: int, den: int, p: int) -> Value:
    """RN_p(num / den), den > 0."""
    if num == 0:
        return None
    s = 1 if num < 0 else 0
    u = -num if num < 0 else num
    e = u.bit_length() - den.bit_length()  # u/den in [2^(e-1), 2^(e+1))
    if (u >= (den << e)) if e >= 0 else ((u << -e) >= den):
        e += 1  # u/den in [2^(e-1), 2^e)
    sh = p - e
    q, r = divmod(u << sh, den) if sh >= 0 else divmod(u, den << -sh)
    if 2 * r > den or (2 * r == den and (q & 1)):
        q += 1
    if q >> p:
        q >>= 1
        e += 1
    return (s, q, e)


def rn_int(x: int, p: int) -> Value:
    """mpfr_set_si / set_ui at p bits."""
    return rn_scaled(x, 0, p)


def rn_sqrt_int(a: int, p: int) -> Value:
    """Correctly rounded sqrt of a nonnegative integer at p bits (mpfr_sqrt)."""
    if a == 0:
        return None
    k = max(0, (2 * p + 8 - a.bit_length()) // 2 + 1)
    t = a << (2 * k)
    r = math.isqrt(t)
    exact = r * r == t
    b = r.bit_length()
    if b > p:
        M, _ = _round_shift(r, b - p, not exact)
        e = b - k
        if M >> p:
            M >>= 1
            e += 1
        return (0, M, e)
    return rn_scaled(r, -k, p)


def mul_int(x: Value, c: int, p_x: int, p: int) -> Value:
    """RN_p(x * c) for an integer c (mpfr_mul_si / mul_ui)."""
    if x is None or c == 0:
        return None
    s, M, e = x
    v = rn_scaled(M * c, e - p_x, p)
    if v is None:
        return None
    return ((v[0] ^ s), v[1], v[2])


def to_fraction(x: Value, p: int) -> Fraction:
    if x is None:
        return Fraction(0)
    s, M, e = x
    v = Fraction(M) * (Fraction(2) ** (e - p))
    return -v if s else v


def values_to_matrix(vals: Sequence[Value], index: np.ndarray, rows: int, cols: int,
                     ctx: PrecisionContext) -> Matrix:
    """Matrix whose element t is vals[index[t]] (row-major)."""
    p = ctx.bits()
    out = Matrix(rows, cols, ctx)
    L = out.nlimbs
    K = len(vals)
    vl = np.zeros((L, K), np.uint32)
    ve = np.full(K, EXP_ZERO, np.int32)
    vs = np.zeros(K, np.uint8)
    for i, v in enumerate(vals):
        if v is None:
            continue
        s, M, e = v
        mant = M << (32 * L - p)
        for k in range(L):
            vl[k, i] = (mant >> (32 * k)) & 0xFFFFFFFF
        ve[i] = e
        vs[i] = s
    idx = np.asarray(index, np.int64).reshape(-1)
    out.limbs[:] = vl[:, idx]
    out.exp[:] = ve[idx]
    out.sign[:] = vs[idx]
    return out


def element(m: Matrix, t: int = 0) -> Value:
    """Element t of a host Matrix as a Value at m.bits()."""
    if m.exp[t] == EXP_ZERO:
        return None
    L = m.nlimbs
    mant = 0
    for k in range(L - 1, -1, -1):
        mant = (mant << 32) | int(m.limbs[k, t])
    p = m.bits()
    return (int(m.sign[t]), mant >> (32 * L - p), int(m.exp[t]))


def _floor_log10(v: Fraction) -> int:
    """floor(log10(v)) for v > 0, exactly."""
    est = int(math.floor((v.numerator.bit_length() - v.denominator.bit_length()) * 0.30102999566398120))
    k = est - 2
    while Fraction(10) ** (k + 1) <= v:
        k += 1
    while Fraction(10) ** k > v:
        k -= 1
    return k


def to_decimal(v: Fraction, digits: int, negative_zero: bool = False) -> str:
    """mpfr_asprintf("%.*Re", digits - 1, x) under RNDN (precision.hpp:293-300):
    d.ddde+XX with `digits` significant digits, round to nearest, ties to even."""
    if digits < 1:
        raise ValueError("to_decimal: need at least one digit")
    if v == 0:
        body = "0" + ("." + "0" * (digits - 1) if digits > 1 else "") + "e+00"
        return ("-" if negative_zero else "") + body
    sgn = "-" if v < 0 else ""
    a = -v if v < 0 else v
    k = _floor_log10(a)
    scaled = a / (Fraction(10) ** (k - digits + 1))
    q, r = divmod(scaled.numerator, scaled.denominator)
    if 2 * r > scaled.denominator or (2 * r == scaled.denominator and (q & 1)):
        q += 1
    if q == 10 ** digits:
        q //= 10
        k += 1
    ds = str(q)
    mant = ds[0] + ("." + ds[1:] if digits > 1 else "")
    ex = f"{abs(k):02d}"
    return f"{sgn}{mant}e{'-' if k < 0 else '+'}{ex}"


def matrix_scalar_decimal(m: Matrix, t: int, digits: int) -> str:
    x = element(m, t)
    return to_decimal(to_fraction(x, m.bits()), digits, negative_zero=(x is None and bool(m.sign[t])))
