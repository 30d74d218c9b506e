"""Blocked LU (blocklu.hpp:121-146) and its solves on the GPU.

pivot-free: bit-exact against the compiled reference's lu_blocked / lu_solve and
the C restatement, every Schur kernel.  partial pivoting (extension): bit-exact
against the restatement (mp_oracle.c orc_lu_blocked), plus backward error.
"""
import numpy as np
import pytest

KERNELS = ["simple", "block", "strassen", "winograd"]


@pytest.mark.gpu
@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("n,K,n_min,bits", [(24, 8, 4, 256), (37, 8, 4, 128), (64, 16, 8, 256), (50, 12, 4, 512)])
def test_lu_pivot_free_matches_reference(P, O, kernel, n, K, n_min, bits):
    ctx = P.PrecisionContext(bits)
    a = P.gen_uniform_full(n, n, 100 + n, ctx)
    ops = P.OpCounter()
    f = P.lu_blocked(a, P.BlockLUConfig(K, P.Algorithm[kernel], n_min), ctx, ops)
    which = "ref" if O.have_ref() else "orc"
    want, _, wops = O.lu_blocked(O.OMat.of(a), K, kernel, n_min, which=which)
    assert P.identical(f.packed, want)
    assert (ops.mul, ops.addsub) == wops
    want2, _, _ = O.lu_blocked(O.OMat.of(a), K, kernel, n_min, which="orc")
    assert P.identical(f.packed, want2)


@pytest.mark.gpu
@pytest.mark.parametrize("kernel", ["block", "winograd"])
def test_lu_partial_pivoting_matches_restatement(P, O, kernel):
    ctx = P.PrecisionContext(256)
    n, K = 48, 16
    a = P.gen_uniform_full(n, n, 5, ctx)
    f = P.lu_blocked(a, P.BlockLUConfig(K, P.Algorithm[kernel], 8), ctx, pivoting=True)
    want, piv, _ = O.lu_blocked(O.OMat.of(a), K, kernel, 8, pivoting=True)
    assert np.array_equal(f.piv, piv)
    assert P.identical(f.packed, want)


@pytest.mark.gpu
def test_lu_solve_matches_reference(P, O):
    ctx = P.PrecisionContext(256)
    n = 40
    a = P.gen_uniform_full(n, n, 77, ctx)
    ones = P.from_ints(np.ones(n, np.int64), ctx)
    b = P.mat_vec_mul(a, ones, ctx)
    bw = O.mat_vec_mul(O.OMat.of(a), O.OMat.of(ones))
    assert P.identical(b, bw)
    f = P.lu_blocked(a, P.BlockLUConfig(8, P.Algorithm.winograd, 4), ctx)
    x = P.lu_solve(f, b, ctx)
    which = "ref" if O.have_ref() else "orc"
    xw = O.lu_solve(O.OMat.of(f.packed), O.OMat.of(b), which=which)
    assert P.identical(x, xw)
    # pivoted solve vs restatement
    fp = P.lu_blocked(a, P.BlockLUConfig(8, P.Algorithm.block, 4), ctx, pivoting=True)
    xp = P.lu_solve(fp, b, ctx)
    xpw = O.lu_solve(O.OMat.of(fp.packed), O.OMat.of(b), piv=fp.piv)
    assert P.identical(xp, xpw)
    err = np.max(np.abs(xp.to_float() - 1.0))
    assert err < 1e-60
    # column-oriented (non-replay) back substitution: within tolerance of the exact one
    xf = P.lu_solve(fp, b, ctx, exact=False)
    assert O.log2_max_abs_diff(O.OMat.of(xf), O.OMat.of(xpw)) < -240


@pytest.mark.gpu
def test_zero_pivot_reports_one_based_index(P):
    # test_blocklu.cpp:65-80
    ctx = P.PrecisionContext(64)
    with pytest.raises(P.SingularError) as e:
        P.lu_columnwise(P.from_ints([[0, 1], [1, 0]], ctx))
    assert e.value.pivot_index == 1
    with pytest.raises(P.SingularError) as e:
        P.lu_columnwise(P.from_ints([[1, 1], [1, 1]], ctx))
    assert e.value.pivot_index == 2
    with pytest.raises(P.DimensionError):
        P.lu_columnwise(P.Matrix(2, 3, ctx))
    # with pivoting the first matrix factors fine
    f = P.lu_blocked(P.from_ints([[0, 1], [1, 0]], ctx), P.BlockLUConfig(2, P.Algorithm.simple, 1), ctx,
                     pivoting=True)
    assert list(f.piv) == [1, 1]


@pytest.mark.gpu
def test_exact_integer_elimination_kernel_independent(P):
    # test_blocklu.cpp:116-126 (kExactA / kExactPacked)
    ctx = P.PrecisionContext(256)
    A = [[2, 1, 3, 1], [4, 3, 8, 3], [6, 4, 14, 6], [2, 3, 10, 9]]
    want = P.from_ints([[2, 1, 3, 1], [2, 1, 2, 1], [3, 1, 3, 2], [1, 2, 1, 4]], ctx)
    a = P.from_ints(A, ctx)
    assert P.equal_values(P.lu_columnwise(a).packed, want)
    for k in KERNELS:
        f = P.lu_blocked(a, P.BlockLUConfig(2, P.Algorithm[k], 1), ctx)
        assert P.equal_values(f.packed, want), k


@pytest.mark.gpu
def test_context_validation(P):
    ctx = P.PrecisionContext(128)
    a = P.gen_random(8, 8, 1, ctx)
    with pytest.raises(P.DomainError):
        P.lu_blocked(a, P.BlockLUConfig(4, P.Algorithm.simple, 4), P.PrecisionContext(256))
    with pytest.raises(P.DimensionError):
        P.lu_blocked(a, P.BlockLUConfig(0, P.Algorithm.simple, 4), ctx)


GOLD = __import__("pathlib").Path(__file__).resolve().parent / "golden"


@pytest.mark.gpu
@pytest.mark.parametrize("path", sorted(GOLD.glob("lu_*.npz")), ids=lambda p: p.stem)
def test_lu_matches_frozen_reference_fixture(P, path):
    d = np.load(path)

    def mat(p):
        r, c, bits = (int(v) for v in d[p + "_shape"])
        return P.Matrix(r, c, P.PrecisionContext(bits), d[p + "_limbs"], d[p + "_exp"], d[p + "_sign"])

    a, f, b, x = mat("a"), mat("f"), mat("b"), mat("x")
    ops = P.OpCounter()
    got = P.lu_blocked(a, P.BlockLUConfig(int(d["K"]), P.Algorithm[str(d["kernel"])], int(d["n_min"])), a.ctx(), ops)
    assert P.identical(got.packed, f)
    assert (ops.mul, ops.addsub) == tuple(int(v) for v in d["ops"])
    assert P.identical(P.mat_vec_mul(a, P.from_ints(np.ones(a.rows(), np.int64), a.ctx()), a.ctx()), b)
    assert P.identical(P.lu_solve(got, b, a.ctx()), x)
