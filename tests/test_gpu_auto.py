"""Cutoff chosen per precision (MPGPU_AUTO_NMIN) and the depth-first top levels the driver uses
when a breadth-first level would not fit its scratch budget (run_gemm_chunked): both replay the
reference's operation DAG, so they must be bit-identical to the explicit / breadth-first runs."""
import os

import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("algo", ["strassen", "winograd"])
@pytest.mark.parametrize("bits,shape", [(256, (96, 80, 72)), (1024, (64, 64, 64)), (512, (37, 45, 29))])
def test_auto_nmin_is_the_chosen_explicit_cutoff(P, algo, bits, shape):
    m, l, n = shape
    ctx = P.PrecisionContext(bits)
    a, b = P.gen_uniform_full(m, l, 7, ctx), P.gen_uniform_full(l, n, 8, ctx)
    nm, d, _ = P.choose_n_min(P.Algorithm[algo], bits, m, l, n)
    st = P.Stats()
    auto = P.fast_mul(a, b, P.FastMMConfig(P.Algorithm[algo], P.AUTO_NMIN), ctx, stats=st)
    want = P.fast_mul(a, b, P.FastMMConfig(P.Algorithm[algo], nm), ctx)
    assert P.identical(auto.c, want.c) and st.depth == d
    assert (auto.ops.mul, auto.ops.addsub) == (want.ops.mul, want.ops.addsub)
    ref, ops = O.gemm(algo, nm, O.OMat.of(a), O.OMat.of(b))
    assert P.identical(auto.c, ref) and (auto.ops.mul, auto.ops.addsub) == ops


def test_auto_nmin_through_host_api_and_group(P):
    ctx = P.PrecisionContext(256)
    a, b = P.gen_uniform_full(64, 64, 1, ctx), P.gen_uniform_full(64, 64, 2, ctx)
    nm, _, _ = P.choose_n_min(P.Algorithm.winograd, 256, 64, 64, 64)
    want = P.Matrix(64, 64, ctx)
    P.gemm_host(P.Algorithm.winograd, nm, a, b, want, ctx)
    got = P.Matrix(64, 64, ctx)
    P.gemm_host(P.Algorithm.winograd, P.AUTO_NMIN, a, b, got, ctx)
    assert P.identical(got, want)
    got2 = P.Matrix(64, 64, ctx)
    P.DeviceGroup([0, 0]).gemm_host(P.Algorithm.winograd, P.AUTO_NMIN, a, b, got2, ctx)
    assert P.identical(got2, want)
    with pytest.raises(P.DomainError):
        P.gemm_host(P.Algorithm.block, P.AUTO_NMIN, a, b, got, ctx)


@pytest.mark.parametrize("algo", ["strassen", "winograd"])
@pytest.mark.parametrize("bits,shape,n_min", [(256, (128, 128, 128), 8), (512, (101, 77, 93), 6),
                                              (1024, (64, 64, 64), 4)])
def test_depth_first_top_levels_bit_exact(P, algo, bits, shape, n_min):
    m, l, n = shape
    ctx = P.PrecisionContext(bits)
    a, b = P.gen_uniform_full(m, l, 3, ctx), P.gen_uniform_full(l, n, 4, ctx)
    bfs = P.fast_mul(a, b, P.FastMMConfig(P.Algorithm[algo], n_min), ctx)
    os.environ["MPGPU_BFS_BUDGET_MB"] = "0"  # every level with >= 2 below it goes depth-first
    try:
        st = P.Stats()
        dfs = P.fast_mul(a, b, P.FastMMConfig(P.Algorithm[algo], n_min), ctx, stats=st)
    finally:
        del os.environ["MPGPU_BFS_BUDGET_MB"]
    assert P.identical(dfs.c, bfs.c)
    assert (dfs.ops.mul, dfs.ops.addsub) == (bfs.ops.mul, bfs.ops.addsub)
    assert st.leaf_madds == P.count_fast(P.Algorithm[algo], m, l, n, n_min).mul
    ref, _ = O.gemm(algo, n_min, O.OMat.of(a), O.OMat.of(b))
    assert P.identical(dfs.c, ref)
