"""BASELINE.json configurations at their full sizes, checked through size-independent
properties (the CPU oracle cannot replay a whole 1024^3 .. 4096^3 product in a test):

- exactness: the reference's own generator draws 53-bit dyadics, so at p >= 128 every
  product and sum of configs 2 / 4 is exact and all four algorithms must agree bit for
  bit -- and agree with the oracle on sampled rows;
- symmetry: RN is odd and commutes with scaling by powers of two, so
  C(-A, B) = -C(A, B) (as values; exact zeros are +0 either way) and
  C(2^s A, 2^t B) = 2^(s+t) C(A, B) bit-exactly, for every algorithm's operation DAG;
- sampled rows: row i of Block depends on row i of A only, so a few rows replay exactly
  on the CPU oracle;
- LU: the backward error ||PA - LU||_max / ||A||_max of the full n = 2048 factorisation
  (L U formed by the GPU GEMM) within c n 2^-p."""
import math

import numpy as np
import pytest

import oracle.oracle as O
import paper_1410_1599_b200 as P

pytestmark = pytest.mark.gpu


def rows_of(x, rows):
    cols = x.cols()
    idx = (np.asarray(rows)[:, None] * cols + np.arange(cols)[None, :]).reshape(-1)
    return P.Matrix(len(rows), cols, x.ctx(), x.limbs[:, idx], x.exp[idx], x.sign[idx])


def negated(x):
    return P.Matrix(x.rows(), x.cols(), x.ctx(), x.limbs, x.exp, x.sign ^ 1)


def scaled(x, s):
    e = np.where(x.exp == P.EXP_ZERO, x.exp, x.exp + s).astype(x.exp.dtype)
    return P.Matrix(x.rows(), x.cols(), x.ctx(), x.limbs, e, x.sign)


def gemm(algo, param, da, db, ctx, m, n):
    dc = P.DeviceMatrix(m, n, ctx)
    P.gemm_into(P.Algorithm[algo], param, da, db, dc)
    return dc.download()


ALGS = [("simple", 0), ("block", 64), ("strassen", 64), ("winograd", 64)]


def test_cfg2_reference_generator_all_algorithms_exact():
    n, bits = 1024, 256
    ctx = P.PrecisionContext(bits)
    a, b = P.gen_random(n, n, 1, ctx), P.gen_random(n, n, 2, ctx)
    da, db = a.to_device(), b.to_device()
    outs = {alg: gemm(alg, prm, da, db, ctx, n, n) for alg, prm in ALGS}
    for alg in ("block", "strassen", "winograd"):
        assert P.identical(outs[alg], outs["simple"]), alg
    rows = [0, 613, 1023]
    want, _ = O.gemm("simple", 0, O.OMat.of(rows_of(a, rows)), O.OMat.of(b))
    assert P.identical(rows_of(outs["simple"], rows), want)


@pytest.mark.parametrize("alg,prm", [("block", 64), ("winograd", 64), ("strassen", 64)])
def test_cfg2_full_mantissa_symmetries_and_sampled_rows(alg, prm):
    n, bits = 1024, 256
    ctx = P.PrecisionContext(bits)
    a, b = P.gen_uniform_full(n, n, 1, ctx), P.gen_uniform_full(n, n, 2, ctx)
    c = gemm(alg, prm, a.to_device(), b.to_device(), ctx, n, n)
    cn = gemm(alg, prm, negated(a).to_device(), b.to_device(), ctx, n, n)
    assert P.equal_values(cn, negated(c))
    cs = gemm(alg, prm, scaled(a, 7).to_device(), scaled(b, -3).to_device(), ctx, n, n)
    assert P.identical(cs, scaled(c, 4))
    if alg == "block":
        rows = [0, 511, 1023]
        want, _ = O.gemm("block", prm, O.OMat.of(rows_of(a, rows)), O.OMat.of(b))
        assert P.identical(rows_of(c, rows), want)


def test_cfg3_full_shape_odd_dims_symmetries_and_bound():
    m, l, n, bits = 1001, 777, 1537, 512
    ctx = P.PrecisionContext(bits)
    a, b = P.gen_scaled(m, l, 3, ctx), P.gen_scaled(l, n, 4, ctx)
    da, db = a.to_device(), b.to_device()
    c = gemm("winograd", 32, da, db, ctx, m, n)
    cn = gemm("winograd", 32, da, negated(b).to_device(), ctx, m, n)
    assert P.equal_values(cn, negated(c))
    # one sampled row against the oracle's exact-at-2p+64 product, north-star bound
    rows, hi = [777], 2 * bits + 64
    HL = (hi + 31) // 32

    def widen(x):
        return O.OMat(x.rows(), x.cols(), hi, np.vstack([np.zeros((HL - x.nlimbs, x.limbs.shape[1]), np.uint32),
                                                         x.limbs]), x.exp, x.sign)
    exact, _ = O.gemm("simple", 0, widen(rows_of(a, rows)), widen(b))
    d = O.log2_max_abs_diff(widen(rows_of(c, rows)), exact) - O.log2_max_abs(O.OMat.of(a)) - \
        O.log2_max_abs(O.OMat.of(b))
    assert d <= math.log2(4.0) + math.log2(7) * math.log2(max(m, l, n)) - bits


def test_cfg5_full_lu_backward_error():
    n, bits = 2048, 256
    ctx = P.PrecisionContext(bits)
    a = P.gen_uniform_full(n, n, 11, ctx)
    f = P.lu_blocked(a, P.BlockLUConfig(64, P.Algorithm.winograd, 32), ctx, pivoting=True)
    pk = f.packed
    idx = np.arange(n * n).reshape(n, n)
    lower, upper = np.tril(np.ones((n, n), bool), -1).reshape(-1), np.triu(np.ones((n, n), bool)).reshape(-1)
    Ll, Le, Ls = np.zeros_like(pk.limbs), np.full_like(pk.exp, P.EXP_ZERO), np.zeros_like(pk.sign)
    Ll[:, lower], Le[lower], Ls[lower] = pk.limbs[:, lower], pk.exp[lower], pk.sign[lower]
    diag = idx.diagonal()
    Ll[-1, diag] = 0x80000000  # unit diagonal: 0.5 * 2^1
    Le[diag] = 1
    Ul, Ue, Us = np.zeros_like(pk.limbs), np.full_like(pk.exp, P.EXP_ZERO), np.zeros_like(pk.sign)
    Ul[:, upper], Ue[upper], Us[upper] = pk.limbs[:, upper], pk.exp[upper], pk.sign[upper]
    Lm, Um = P.Matrix(n, n, ctx, Ll, Le, Ls), P.Matrix(n, n, ctx, Ul, Ue, Us)
    lu = gemm("block", 64, Lm.to_device(), Um.to_device(), ctx, n, n)
    perm = np.arange(n)
    for d, r in enumerate(f.piv):
        perm[[d, r]] = perm[[r, d]]
    pa = rows_of(a, perm)
    diff = P.sub(pa, lu)
    nz = diff.exp != P.EXP_ZERO
    log2_err = (int(diff.exp[nz].max()) if nz.any() else -10 ** 9) - int(a.exp[a.exp != P.EXP_ZERO].max())
    assert log2_err <= math.log2(4.0 * n) - bits + 2


def test_cfg4_full_size_reference_generator_exact_winograd_depth3_equals_block():
    """n = 4096 at 1024 bits, Winograd to depth 3 (n_min 512) vs Block 512: with the
    reference's 53-bit dyadic inputs both are exact, hence bit-identical."""
    n, bits = 4096, 1024
    ctx = P.PrecisionContext(bits)
    a, b = P.gen_random(n, n, 1, ctx), P.gen_random(n, n, 2, ctx)
    da, db = a.to_device(), b.to_device()
    dw, dbk = P.DeviceMatrix(n, n, ctx), P.DeviceMatrix(n, n, ctx)
    st = P.gemm_into(P.Algorithm.winograd, 512, da, db, dw)
    assert st.depth == 3
    P.gemm_into(P.Algorithm.block, 512, da, db, dbk)
    assert P.identical(dw.download(), dbk.download())
