"""Wide formats (64 / 128 / 256 / 288 limbs, 1025..9216 bits; the *_wide.cu kernels):
primitives bit-identical to MPFR on structured edge cases, every GEMM algorithm
bit-exact vs the restatement, LU / solve / inverse and the reference's run_lu on the
Lotkin matrix at the paper's 8192 / 8650 bits identical to the compiled reference."""
import numpy as np
import pytest

import oracle.oracle as O
from mpgen import structured_pairs, tie_cases

import paper_1410_1599_b200 as P
from paper_1410_1599_b200 import benchdrv as B

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(not O.have_ref(), reason="compiled reference not built")
WIDE = [1025, 2048, 3000, 4096, 8192, 8650, 9216]


def _mats(ctx, L, x, y):
    (xm, xe, xs), (ym, ye, ys) = x, y
    n = xe.size
    return (P.Matrix(n, 1, ctx, xm[-L:] if xm.shape[0] >= L else xm, xe, xs),
            P.Matrix(n, 1, ctx, ym[-L:] if ym.shape[0] >= L else ym, ye, ys))


@pytest.mark.parametrize("bits", WIDE)
def test_wide_ops_match_mpfr(bits):
    ctx = P.PrecisionContext(bits)
    L = (bits + 31) // 32
    rng = np.random.default_rng(7000 + bits)
    x, y = structured_pairs(rng, L, 600, bits)
    a, b = _mats(ctx, L, x, y)
    for op in (0, 1, 2, 3):
        if op == 3:
            keep = b.exp != P.EXP_ZERO
            a = P.Matrix(int(keep.sum()), 1, ctx, a.limbs[:, keep], a.exp[keep], a.sign[keep])
            b = P.Matrix(int(keep.sum()), 1, ctx, b.limbs[:, keep], b.exp[keep], b.sign[keep])
        got, want = P.vec_op(op, a, b), O.vec_op(op, a, b)
        bad = ~((got.exp == want.exp) & (got.sign == want.sign) & np.all(got.limbs == want.limbs, axis=0))
        assert not bad.any(), f"op {op} bits {bits}: {int(bad.sum())} mismatches, first at {np.argmax(bad)}"


@pytest.mark.parametrize("bits", [2048, 8192])
def test_wide_ties_round_to_even(bits):
    ctx = P.PrecisionContext(bits)
    x, y = tie_cases(P.nlimbs_for(bits), bits)
    a, b = _mats(ctx, P.nlimbs_for(bits), x, y)
    for op in (0, 1):
        assert P.identical(P.vec_op(op, a, b), O.vec_op(op, a, b))


@pytest.mark.parametrize("bits", [2048, 4096, 8650])
@pytest.mark.parametrize("alg,param", [("simple", 0), ("block", 3), ("strassen", 3), ("winograd", 2)])
def test_wide_gemm_bit_exact(bits, alg, param):
    ctx = P.PrecisionContext(bits)
    a = P.gen_uniform_full(11, 9, 1, ctx)
    b = P.gen_uniform_full(9, 13, 2, ctx)
    algo = P.Algorithm[alg]
    if algo == P.Algorithm.simple:
        c = P.simple_mul(a, b, ctx)
    elif algo == P.Algorithm.block:
        c = P.block_mul(a, b, param, ctx)
    else:
        c = P.fast_mul(a, b, P.FastMMConfig(algo, param), ctx).c
    want, _ = O.gemm(alg, param, O.OMat.of(a), O.OMat.of(b))
    assert P.identical(c, want)


@needs_ref
@pytest.mark.parametrize("bits,kernel", [(8192, "winograd"), (8650, "block"), (4096, "strassen")])
def test_wide_lu_and_solve_match_reference(bits, kernel):
    ctx = P.PrecisionContext(bits)
    n = 12
    a = P.gen_random(n, n, 3, ctx)
    f = P.lu_blocked(a, P.BlockLUConfig(4, P.Algorithm[kernel], 2), ctx)
    want, _, _ = O.lu_blocked(O.OMat.of(a), 4, kernel, 2, which="ref")
    assert P.identical(f.packed, want)
    x = P.from_ints(np.arange(n, dtype=np.int64), ctx, n, 1)
    bvec = P.mat_vec_mul(a, x, ctx)
    sol = P.lu_solve(f, bvec, ctx)
    assert P.identical(sol, O.lu_solve(want, O.OMat.of(bvec), which="ref"))


@needs_ref
@pytest.mark.parametrize("bits,kernel", [(8192, "winograd"), (8650, "winograd")])
def test_wide_run_lu_lotkin_rows_match_reference(bits, kernel):
    # the paper's ill-conditioned experiment at a small order
    out = B.run_lu(B.LURequest("lotkin", 10, bits, P.Algorithm[kernel], 2, 1, 2, 1, False))
    text, singular = O.run_lu("lotkin", 10, bits, kernel, 2, 1, 2)
    import io
    s = io.StringIO()
    B.print_csv(s, out.rows)

    def strip(t):
        return [",".join(f[:10] + ["T"] + f[11:]) if f[0] != "command" else ",".join(f)
                for f in (ln.split(",") for ln in t.strip().splitlines())]
    assert out.any_singular == singular
    assert strip(s.getvalue()) == strip(text)


@needs_ref
def test_wide_inverse_and_cond_one():
    ctx = P.PrecisionContext(2000)
    a = B.gen_lotkin(6, ctx)
    assert P.to_fractions(P.inverse(a, P.PrecisionContext(4096))) == P.to_fractions(O.inverse(a, 4096))
    assert P.to_fractions(P.cond_one(a)) == P.to_fractions(O.cond_one(a))
