"""Host-side product logic (CPU only): the C-ABI library loads and exports every
symbol include/mpgpu.h declares; the op model, recursion plan and input
generators equal the oracle / reference; Python-side validation mirrors the
reference's exception behaviour without touching a GPU."""
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def test_library_exports_every_declared_symbol(P):
    from paper_1410_1599_b200 import _lib
    hdr = (ROOT / "include" / "mpgpu.h").read_text()
    declared = set(re.findall(r"\b(mpgpu_[a-z_0-9]+)\s*\(", hdr))
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(_lib.lib, name), name
    assert declared == set(_lib.EXPORTED)


def test_no_cpu_fallback_in_product_path():
    # the product package must never import the oracle (the checker)
    for p in (ROOT / "paper_1410_1599_b200").rglob("*.py"):
        src = p.read_text()
        assert "from oracle" not in src and "import oracle" not in src, p


def test_count_fast_and_plan_match_oracle(P, O):
    rng = np.random.default_rng(5)
    for _ in range(300):
        m, l, n = (int(v) for v in rng.integers(1, 5000, 3))
        nm = int(rng.integers(1, 100))
        for alg in (P.Algorithm.simple, P.Algorithm.block, P.Algorithm.strassen, P.Algorithm.winograd):
            c = P.count_fast(alg, m, l, n, nm)
            assert (c.mul, c.addsub) == O.count_fast(int(alg), m, l, n, nm)
    if O.have_ref():
        for dims in [(1001, 777, 1537, 32), (4096, 4096, 4096, 512), (1024, 63, 1024, 32), (7, 9, 5, 1)]:
            mine = P.recursion_plan(*dims[:3], P.FastMMConfig(P.Algorithm.winograd, dims[3]))
            ref = O.recursion_plan(*dims)
            assert [(r.level, r.before.m, r.before.l, r.before.n, r.padded.m, r.padded.l, r.padded.n, int(r.base))
                    for r in mine] == [tuple(x) for x in ref]


def test_count_errors(P):
    with pytest.raises(P.DimensionError):
        P.count_simple(0, 1, 1)
    with pytest.raises(P.DimensionError):
        P.count_fast(P.Algorithm.strassen, 4, 4, 4, 0)
    with pytest.raises(P.DimensionError):
        P.recursion_plan(4, 4, 4, P.FastMMConfig(P.Algorithm.strassen, 0))


@pytest.mark.parametrize("bits", [2, 17, 32, 53, 64, 100, 128, 200, 256, 512, 1000, 1024])
def test_generators_match_oracle(P, O, bits):
    ctx = P.PrecisionContext(bits)
    assert P.identical(P.gen_random(9, 7, 42, ctx), O.gen_random(9, 7, 42, bits))
    assert P.identical(P.gen_uniform_full(9, 7, 43, ctx), O.gen_full(0, 9, 7, 43, bits))
    assert P.identical(P.gen_scaled(9, 7, 44, ctx), O.gen_full(1, 9, 7, 44, bits))
    if O.have_ref():
        assert P.identical(P.gen_random(9, 7, 42, ctx), O.gen_random(9, 7, 42, bits, "ref"))


def test_prng_python_mirror(P, O):
    r = P.Prng64(1)
    assert [r.next64() for _ in range(3)] == O.prng_stream(1, 3)


def test_from_ints_matches_mpfr_set_si(P, O):
    rng = np.random.default_rng(9)
    v = rng.integers(-(1 << 60), 1 << 60, 500)
    v[:5] = [0, 1, -1, (1 << 53) + 1, -(1 << 40) - 3]
    for bits in (2, 10, 53, 64, 128):
        assert P.identical(P.from_ints(v, P.PrecisionContext(bits), 500, 1), O.from_si(v, bits, 500, 1))


def test_precision_and_shape_validation(P):
    with pytest.raises(P.DomainError):
        P.PrecisionContext(1)
    with pytest.raises(P.DomainError):
        P.PrecisionContext((1 << 20) + 1)
    ctx = P.PrecisionContext(64)
    with pytest.raises(P.DimensionError):
        P.Matrix(0, 3, ctx)
    a = P.Matrix(2, 3, ctx)
    with pytest.raises(P.DimensionError):
        a.sub(1, 1, 2, 2)
    with pytest.raises(P.DimensionError):
        P.simple_mul(a, P.Matrix(2, 2, ctx), ctx)  # inner mismatch raises before any device work
    with pytest.raises(P.DomainError):
        P.add(a, P.Matrix(2, 3, P.PrecisionContext(128)))
    with pytest.raises(P.DimensionError):
        P.sub(a, P.Matrix(3, 2, ctx))
    with pytest.raises(P.DomainError):
        P.parse_algorithm("fast")


def test_pad_even_and_equal_values(P):
    ctx = P.PrecisionContext(64)
    a = P.from_ints([[1, 2, 3], [4, 5, 6], [7, 8, 9]], ctx)
    p = P.pad_even(a)
    assert (p.rows(), p.cols()) == (4, 4)
    assert P.equal_values(p.sub(0, 0, 3, 3), a)
    assert np.all(p.exp.reshape(4, 4)[3] == P.EXP_ZERO) and np.all(p.exp.reshape(4, 4)[:, 3] == P.EXP_ZERO)
    even = P.Matrix(4, 4, ctx)
    assert P.equal_values(P.pad_even(even), even)
    z1 = P.from_ints([0], ctx)
    z2 = z1.copy()
    z2.sign[:] = 1
    assert P.equal_values(z1, z2) and not P.identical(z1, z2)


def test_mpgpu_nlimbs(P):
    # wide formats above 1024 bits: 64, 128, 256, 288 limbs (mpgpu.h MPGPU_MAX_PREC = 9216)
    assert [P.nlimbs_for(b) for b in (1, 2, 32, 33, 64, 65, 128, 129, 256, 512, 1024, 1025, 2048, 2049, 8192,
                                      8650, 9216, 9217)] == \
        [0, 1, 1, 2, 2, 4, 4, 8, 8, 16, 32, 64, 64, 128, 256, 288, 288, 0]
