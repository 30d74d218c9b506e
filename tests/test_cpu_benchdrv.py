"""Host logic of the GPU benchmark driver (benchdrv.py / exact.py) against the compiled
reference: closed-form generators bit-identical, decimal formatting identical to
mpfr_asprintf("%.*Re"), CSV schema identical (bench.hpp:21-82)."""
import io
from fractions import Fraction

import numpy as np
import pytest

import oracle.oracle as O
import paper_1410_1599_b200 as P
from paper_1410_1599_b200 import benchdrv as B
from paper_1410_1599_b200 import exact as X

needs_ref = pytest.mark.skipif(not O.have_ref(), reason="compiled reference not built")


def same_values(a, b):
    """bit-identical values (zeros compare by sign too); limb counts may differ"""
    assert a.rows() == b.rows() and a.cols() == b.cols()
    fa, fb = P.to_fractions(a), P.to_fractions(b)
    assert fa == fb
    assert np.array_equal(a.exp, b.exp)


@needs_ref
@pytest.mark.parametrize("bits", [2, 24, 53, 100, 128, 256, 1000, 2048])
@pytest.mark.parametrize("m,l,n", [(1, 1, 1), (5, 7, 3), (17, 9, 12)])
def test_bench_pair_matches_reference(bits, m, l, n):
    a, b = B.gen_bench_pair(m, l, n, P.PrecisionContext(bits))
    ra, rb = O.gen_bench_pair(m, l, n, bits)
    same_values(a, ra)
    same_values(b, rb)


@needs_ref
@pytest.mark.parametrize("bits", [24, 128, 256, 512, 2048])
@pytest.mark.parametrize("m,l,n", [(1, 1, 1), (6, 11, 4), (13, 64, 2)])
def test_bench_reference_matches_reference(bits, m, l, n):
    c = B.bench_reference(m, l, n, P.PrecisionContext(bits))
    same_values(c, O.bench_reference(m, l, n, bits))


@pytest.mark.parametrize("i,l", [(1, 1), (3, 7), (1000, 1024), (4096, 4096)])
def test_bench_entry_closed_form(i, l):
    assert B.bench_entry_sum(i, l) == sum((i + k - 1) * (l - k + 1) for k in range(1, l + 1))


@needs_ref
@pytest.mark.parametrize("bits", [2, 53, 128, 333])
@pytest.mark.parametrize("n", [1, 2, 9])
def test_lotkin_matches_reference(bits, n):
    same_values(B.gen_lotkin(n, P.PrecisionContext(bits)), O.gen_lotkin(n, bits))


def _values_matrix(fracs, bits):
    vals = [X.rn_fraction(f.numerator, f.denominator, bits) if f else None for f in fracs]
    return X.values_to_matrix(vals, np.arange(len(vals)), len(vals), 1, P.PrecisionContext(bits))


@needs_ref
@pytest.mark.parametrize("digits", [1, 2, 3, 5, 41, 310, 619])
def test_to_decimal_matches_mpfr(digits):
    rng = np.random.default_rng(digits)
    fr = [Fraction(1, 8), Fraction(3, 8), Fraction(5, 2), Fraction(7, 2), Fraction(1, 16), Fraction(-15, 16),
          Fraction(0), Fraction(999999, 1000000), Fraction(-1, 3), Fraction(2) ** -1000, Fraction(2) ** 900]
    for _ in range(60):
        num = int(rng.integers(1, 1 << 62)) * (1 if rng.random() < 0.5 else -1)
        fr.append(Fraction(num, 1) * Fraction(2) ** int(rng.integers(-700, 300)))
    for bits in (53, 256, 2048):
        x = _values_matrix(fr, bits)
        want = O.to_decimal(x, digits)
        got = [X.matrix_scalar_decimal(x, t, digits) for t in range(len(fr))]
        assert got == want, (bits, digits)


def test_exact_rounding_helpers():
    p = 10
    assert X.to_fraction(X.rn_int(1023, p), p) == 1023
    assert X.to_fraction(X.rn_int(2047, p), p) == 2048  # tie -> even
    assert X.to_fraction(X.rn_int(2045, p), p) == 2044
    v = X.rn_sqrt_int(4, 53)
    assert X.to_fraction(v, 53) == 2
    r = X.rn_sqrt_int(2, 200)
    f = X.to_fraction(r, 200)
    assert abs(f * f - 2) < Fraction(1, 2 ** 195)
    assert X.to_fraction(X.rn_fraction(1, 3, 2), 2) == Fraction(3, 8)


@needs_ref
def test_csv_header_and_row_format():
    text = O.run_matmul(3, 3, 3, 24, 2, algos=("simple",))
    header = text.splitlines()[0]
    assert header == B.CSV_HEADER
    r = B.BenchRecord(command="lu", algorithm="columnwise", m=4, l=4, n=4, bits=128, n_min=32, seed=7,
                      wall_seconds=0.0004, max_rel_error="1.00e-30")
    assert r.to_csv_row() == "lu,columnwise,4,4,4,128,32,,,7,0.000,1.00e-30,,,"
    out = io.StringIO()
    B.print_csv(out, [r])
    assert out.getvalue().splitlines() == [B.CSV_HEADER, r.to_csv_row()]


def test_append_csv_header_once(tmp_path):
    p = tmp_path / "x.csv"
    r = B.BenchRecord(command="matmul", algorithm="block", m=1, l=1, n=1, bits=2, n_min=1)
    B.append_csv(str(p), [r])
    B.append_csv(str(p), [r, r])
    lines = p.read_text().splitlines()
    assert lines[0] == B.CSV_HEADER and lines.count(B.CSV_HEADER) == 1 and len(lines) == 4


def test_requests_validate():
    with pytest.raises(P.DomainError):
        B.run_lu(B.LURequest(matrix_kind="hilbert"))
    with pytest.raises(P.DomainError):
        B.run_lu(B.LURequest(alpha_lo=3, alpha_hi=2))
    with pytest.raises(P.DomainError):
        B.run_matmul(B.MatmulRequest(ref_bits_multiplier=0))


def test_error_digits():
    assert B.error_digits(128, False) == 3
    assert B.error_digits(128, True) == 41
    assert B.error_digits(2048, True) == 619
