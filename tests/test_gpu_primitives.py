"""Device MP primitives (mp_arith.cuh) vs MPFR (precision.hpp:127-161):
add / sub / mul / div must be bit-identical to mpfr_* with MPFR_RNDN, including
the signs of zeros, on structured edge cases at every supported limb count."""
import numpy as np
import pytest

from mpgen import carry_patterns, structured_pairs, tie_cases

PRECS = [2, 17, 32, 33, 53, 64, 100, 128, 150, 200, 255, 256, 300, 512, 777, 1000, 1024]


def _mats(P, ctx, L, x, y):
    (xm, xe, xs), (ym, ye, ys) = x, y
    n = xe.size
    a = P.Matrix(n, 1, ctx, xm[-L:] if xm.shape[0] >= L else xm, xe, xs)
    b = P.Matrix(n, 1, ctx, ym[-L:] if ym.shape[0] >= L else ym, ye, ys)
    return a, b


@pytest.mark.gpu
@pytest.mark.parametrize("bits", PRECS)
def test_ops_match_mpfr(P, O, bits):
    ctx = P.PrecisionContext(bits)
    L = max(1, (bits + 31) // 32)
    rng = np.random.default_rng(1000 + bits)
    n = 20000 if bits <= 256 else 6000
    x, y = structured_pairs(rng, L, n, bits)
    a, b = _mats(P, ctx, L, x, y)
    for op in (0, 1, 2, 3):
        got = P.vec_op(op, a, b) if op != 3 else None
        if op == 3:  # division: drop zero divisors (SingularError path tested separately)
            keep = b.exp != P.EXP_ZERO
            a3 = P.Matrix(int(keep.sum()), 1, ctx, a.limbs[:, keep], a.exp[keep], a.sign[keep])
            b3 = P.Matrix(int(keep.sum()), 1, ctx, b.limbs[:, keep], b.exp[keep], b.sign[keep])
            got = P.vec_op(3, a3, b3)
            want = O.vec_op(3, a3, b3)
        else:
            want = O.vec_op(op, a, b)
        bad = ~((got.exp == want.exp) & (got.sign == want.sign) & np.all(got.limbs == want.limbs, axis=0))
        assert not bad.any(), f"op {op} bits {bits}: {int(bad.sum())} mismatches, first at {np.argmax(bad)}"


@pytest.mark.gpu
@pytest.mark.parametrize("bits", [64, 100, 128, 200, 256, 500, 512, 1000, 1024])
def test_mul_carry_extremes(P, O, bits):
    """Every pair of carry-saturating mantissas (all ones, one saturated limb at each position,
    alternating limbs, ...): the product's carry chains (mp_arith.cuh mul_eo_g, short and full
    product) against mpfr_mul, and the same operands through add / sub."""
    ctx = P.PrecisionContext(bits)
    L = max(1, (bits + 31) // 32)
    pat = carry_patterns(L, bits)
    npat = pat.shape[1]
    ia, ib = np.meshgrid(np.arange(npat), np.arange(npat), indexing="ij")
    xm, ym = pat[:, ia.ravel()], pat[:, ib.ravel()]
    n = xm.shape[1]
    rng = np.random.default_rng(bits)
    xe = rng.integers(-5, 5, size=n).astype(np.int64)
    ye = xe - rng.integers(0, 3, size=n)
    xs = rng.integers(0, 2, size=n).astype(np.uint8)
    ys = rng.integers(0, 2, size=n).astype(np.uint8)
    a, b = _mats(P, ctx, L, (xm, xe, xs), (ym, ye, ys))
    for op in (2, 0, 1):
        got, want = P.vec_op(op, a, b), O.vec_op(op, a, b)
        bad = ~((got.exp == want.exp) & (got.sign == want.sign) & np.all(got.limbs == want.limbs, axis=0))
        assert not bad.any(), f"op {op} bits {bits}: {int(bad.sum())} mismatches, first at {np.argmax(bad)}"


@pytest.mark.gpu
@pytest.mark.parametrize("bits", [53, 64, 128, 200, 256, 1024])
def test_ties_round_to_even(P, O, bits):
    ctx = P.PrecisionContext(bits)
    L = P.nlimbs_for(bits)
    x, y = tie_cases(L, bits)
    a, b = _mats(P, ctx, L, x, y)
    for op in (0, 1):
        got, want = P.vec_op(op, a, b), O.vec_op(op, a, b)
        assert P.identical(got, want)


@pytest.mark.gpu
def test_division_by_zero_is_singular(P):
    ctx = P.PrecisionContext(128)
    a = P.from_ints([1, 2], ctx)
    b = P.from_ints([1, 0], ctx)
    with pytest.raises(P.SingularError):
        P.vec_op(3, a, b)
