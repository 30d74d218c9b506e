"""Text codec of the reference (precision.hpp:204-300, matrix.hpp:309-344) for golden-
file interchange with its tooling: hex-float scalars
`[-]0x1.<hex>p<exp>` that round-trip bit-exactly, and `mpmat <m> <n> <bits>` matrix
files.  Exact integer arithmetic on the host (exact.py); no MPFR.
"""
from __future__ import annotations

from fractions import Fraction
from typing import IO, Iterable

import numpy as np

from . import exact
from .mpmm import EXP_ZERO, DimensionError, Error, Matrix, PrecisionContext


class ParseError(Error):
    """mpmm::ParseError (errors.hpp:34-39): message and 0-based byte position."""

    def __init__(self, what: str, position: int):
        super().__init__(f"{what} (at position {position})")
        self.position = position


class IoError(Error):
    """mpmm::IoError (errors.hpp:46-48)"""


def _element_mz(m: Matrix, t: int):
    """(negative, M, k) with |x| = M * 2^k, M the full mantissa integer (MPFR's
    mpfr_get_z_2exp); None for zeros."""
    if m.exp[t] == EXP_ZERO:
        return None
    L = m.nlimbs
    mant = 0
    for q in range(L - 1, -1, -1):
        mant = (mant << 32) | int(m.limbs[q, t])
    p = m.bits()
    M = mant >> (32 * L - p)  # p-bit integer, MSB set
    return bool(m.sign[t]), M, int(m.exp[t]) - p


def to_hex(m: Matrix, t: int = 0) -> str:
    """precision.hpp:210-244: shortest canonical hex float, leading digit 1."""
    v = _element_mz(m, t)
    if v is None:  # is_negative() is mpfr_sgn < 0: both zeros print unsigned
        return "0x0p+0"
    neg, z, k = v
    bl = z.bit_length()
    shift = (4 - (bl - 1) % 4) % 4
    z <<= shift
    pexp = z.bit_length() - 1 + k - shift
    digits = format(z, "x")
    frac = digits[1:].rstrip("0")
    out = ("-" if neg else "") + "0x" + digits[0] + ("." + frac if frac else "")
    return out + "p" + ("-" if pexp < 0 else "+") + str(abs(pexp))


def from_hex(text: str, ctx: PrecisionContext):
    """precision.hpp:248-290: parse `sign? 0x hex (. hex)? p sign? dec`, round to nearest
    at ctx; ParseError at the offending byte.  Returns an exact.Value."""
    i = 0
    n = len(text)

    def fail(msg, pos):
        raise ParseError("hex-float: " + msg, pos)

    neg = False
    if i < n and text[i] in "+-":
        neg = text[i] == "-"
        i += 1
    if i >= n or text[i] != "0":
        fail("expected '0x'", i)
    i += 1
    if i >= n or text[i] not in "xX":
        fail("expected '0x'", i)
    i += 1
    hexd = "0123456789abcdefABCDEF"
    s0 = i
    while i < n and text[i] in hexd:
        i += 1
    if i == s0:
        fail("expected hex significand", i)
    intpart = text[s0:i]
    frac = ""
    if i < n and text[i] == ".":
        i += 1
        f0 = i
        while i < n and text[i] in hexd:
            i += 1
        if i == f0:
            fail("expected fraction digits after '.'", i)
        frac = text[f0:i]
    if i >= n or text[i] not in "pP":
        fail("expected 'p' exponent", i)
    i += 1
    esign = 1
    if i < n and text[i] in "+-":
        esign = -1 if text[i] == "-" else 1
        i += 1
    e0 = i
    while i < n and text[i].isdigit():
        i += 1
    if i == e0:
        fail("expected exponent digits", i)
    if i != n:
        fail("trailing characters", i)
    num = int(intpart + frac, 16)
    e2 = esign * int(text[e0:i]) - 4 * len(frac)
    p = ctx.bits()
    if num == 0:
        return None, neg
    return exact.rn_scaled(-num if neg else num, e2, p), neg


def scalar_matrix(values, ctx: PrecisionContext, rows: int, cols: int, neg_zero=None) -> Matrix:
    vals = list(values)
    m = exact.values_to_matrix(vals, np.arange(len(vals)), rows, cols, ctx)
    if neg_zero is not None:
        for t, nz in enumerate(neg_zero):
            if vals[t] is None and nz:
                m.sign[t] = 1
    return m


def write_matrix(out: IO[str], a: Matrix) -> None:
    """matrix.hpp:314-324"""
    try:
        out.write(f"mpmat {a.rows()} {a.cols()} {a.bits()}\n")
        for i in range(a.rows()):
            out.write(" ".join(to_hex(a, i * a.cols() + j) for j in range(a.cols())) + "\n")
    except OSError as e:
        raise IoError("write_matrix: stream failure") from e


def _tokens(src: IO[str]) -> Iterable[str]:
    for line in src:
        yield from line.split()


def read_matrix(src: IO[str]) -> Matrix:
    """matrix.hpp:326-344"""
    toks = _tokens(src)
    try:
        magic, m, n, bits = next(toks), next(toks), next(toks), next(toks)
        m, n, bits = int(m), int(n), int(bits)
    except (StopIteration, ValueError):
        raise IoError("read_matrix: bad header, expected 'mpmat <m> <n> <bits>'") from None
    if magic != "mpmat" or m < 0 or n < 0:
        raise IoError("read_matrix: bad header, expected 'mpmat <m> <n> <bits>'")
    if m == 0 or n == 0:
        raise DimensionError("read_matrix: zero dimension in header")
    ctx = PrecisionContext(bits)
    vals, negz = [], []
    for i in range(m):
        for j in range(n):
            try:
                tok = next(toks)
            except StopIteration:
                raise IoError(f"read_matrix: unexpected end of input at element ({i + 1},{j + 1})") from None
            v, neg = from_hex(tok, ctx)
            vals.append(v)
            negz.append(neg)
    return scalar_matrix(vals, ctx, m, n, negz)


def to_fraction(m: Matrix, t: int = 0) -> Fraction:
    v = _element_mz(m, t)
    if v is None:
        return Fraction(0)
    neg, M, k = v
    f = Fraction(M) * Fraction(2) ** k
    return -f if neg else f
