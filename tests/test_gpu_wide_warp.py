"""Wide formats: the warp-cooperative kernels (wkern.cuh / wmp.cuh, default) against the
thread-per-element kernels (MPGPU_WIDE=thread) on the same inputs -- both are correctly
rounded replays of the reference's operation order, so every bit must agree; the MPFR
checks of test_gpu_wide.py pin the default path independently."""
import os

import numpy as np
import pytest

from mpgen import structured_pairs

import paper_1410_1599_b200 as P

pytestmark = pytest.mark.gpu


class _thread_kernels:
    def __enter__(self):
        os.environ["MPGPU_WIDE"] = "thread"

    def __exit__(self, *exc):
        os.environ.pop("MPGPU_WIDE", None)


def _both(fn):
    got = fn()
    with _thread_kernels():
        want = fn()
    return got, want


@pytest.mark.parametrize("bits", [2048, 4000, 8192, 8650, 9216])
def test_warp_ops_match_thread_ops(bits):
    ctx = P.PrecisionContext(bits)
    L = P.nlimbs_for(bits)
    rng = np.random.default_rng(91000 + bits)
    (xm, xe, xs), (ym, ye, ys) = structured_pairs(rng, L, 1500, bits)
    a = P.Matrix(xe.size, 1, ctx, xm, xe, xs)
    b = P.Matrix(ye.size, 1, ctx, ym, ye, ys)
    keep = b.exp != P.EXP_ZERO
    for op in (0, 1, 2, 3):
        aa, bb = a, b
        if op == 3:
            aa = P.Matrix(int(keep.sum()), 1, ctx, a.limbs[:, keep], a.exp[keep], a.sign[keep])
            bb = P.Matrix(int(keep.sum()), 1, ctx, b.limbs[:, keep], b.exp[keep], b.sign[keep])
        got, want = _both(lambda: P.vec_op(op, aa, bb))
        assert P.identical(got, want), f"op {op} at {bits} bits"


@pytest.mark.parametrize("bits,alg,param", [(4096, "block", 5), (8192, "simple", 0), (3000, "winograd", 4)])
def test_warp_gemm_matches_thread_gemm(bits, alg, param):
    ctx = P.PrecisionContext(bits)
    a = P.gen_scaled(19, 17, 3, ctx)
    b = P.gen_scaled(17, 21, 4, ctx)
    algo = P.Algorithm[alg]
    if algo == P.Algorithm.simple:
        got, want = _both(lambda: P.simple_mul(a, b, ctx))
    elif algo == P.Algorithm.block:
        got, want = _both(lambda: P.block_mul(a, b, param, ctx))
    else:
        got, want = _both(lambda: P.fast_mul(a, b, P.FastMMConfig(algo, param), ctx).c)
    assert P.identical(got, want)


@pytest.mark.parametrize("pivoting", [False, True])
@pytest.mark.parametrize("bits", [2048, 8650])
def test_warp_lu_and_solve_match_thread(bits, pivoting):
    ctx = P.PrecisionContext(bits)
    n = 26
    a = P.gen_uniform_full(n, n, 5, ctx)
    x = P.gen_uniform_full(n, 1, 6, ctx)
    b = P.mat_vec_mul(a, x, ctx)
    cfg = P.BlockLUConfig(8, P.Algorithm.winograd, 4)
    fw, ft = _both(lambda: P.lu_blocked(a, cfg, ctx, pivoting=pivoting))
    assert P.identical(fw.packed, ft.packed)
    if pivoting:
        assert np.array_equal(fw.piv, ft.piv)
    for exact in (True, False):
        xw, xt = _both(lambda: P.lu_solve(fw, b, ctx, exact=exact))
        assert P.identical(xw, xt)
