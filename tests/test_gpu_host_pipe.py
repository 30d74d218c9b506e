"""Pipelined host GEMM (mpgpu_gemm_host, Winograd, even shapes >= 128^3): operands
uploaded by quadrant, the top level of fast_mul_rec (fastmm.hpp:174-198) unrolled so
m2 = a11 b11 and m3 = a12 b21 start on their own quadrants, output quadrants
downloaded as they complete.  Must be bit-identical to the device-resident path and
to the oracle (the same operation DAG per element)."""
import pytest

CASES = [
    # (m, l, n, bits, n_min, generator)
    (128, 128, 128, 256, 32, "uniform_full"),
    (192, 160, 224, 128, 16, "scaled"),
    (130, 134, 150, 256, 16, "random"),     # even top level, odd below (padding inside the subtrees)
    (256, 256, 256, 512, 64, "uniform_full"),
    (200, 200, 200, 64, 64, "scaled"),
    (128, 256, 160, 1024, 32, "uniform_full"),
    (256, 128, 128, 32, 8, "random"),
]


def _gen(P, kind):
    return {"uniform_full": P.gen_uniform_full, "scaled": P.gen_scaled, "random": P.gen_random}[kind]


@pytest.mark.gpu
@pytest.mark.parametrize("m,l,n,bits,n_min,kind", CASES)
def test_host_pipe_matches_device_path(P, m, l, n, bits, n_min, kind):
    ctx = P.PrecisionContext(bits)
    gen = _gen(P, kind)
    a, b = gen(m, l, 3, ctx), gen(l, n, 4, ctx)
    c = P.Matrix(m, n, ctx)
    st = P.gemm_host(P.Algorithm.winograd, n_min, a, b, c, ctx)
    want = P.fast_mul(a, b, P.FastMMConfig(P.Algorithm.winograd, n_min), ctx)
    assert P.identical(c, want.c), (m, l, n, bits, n_min, kind)
    assert (st.mul, st.addsub) == (want.ops.mul, want.ops.addsub)


@pytest.mark.gpu
def test_host_pipe_matches_oracle(P, O):
    ctx = P.PrecisionContext(128)
    a, b = P.gen_uniform_full(128, 128, 7, ctx), P.gen_uniform_full(128, 128, 8, ctx)
    c = P.Matrix(128, 128, ctx)
    st = P.gemm_host(P.Algorithm.winograd, 16, a, b, c, ctx)
    want, ops = O.gemm("winograd", 16, O.OMat.of(a), O.OMat.of(b))
    assert P.identical(c, want)
    assert (st.mul, st.addsub) == ops


@pytest.mark.gpu
def test_host_pipe_repeated_calls_stable(P):
    # back-to-back calls reuse the handle's streams and events: identical outputs every time
    ctx = P.PrecisionContext(256)
    a, b = P.gen_uniform_full(256, 256, 5, ctx), P.gen_uniform_full(256, 256, 6, ctx)
    first = P.Matrix(256, 256, ctx)
    P.gemm_host(P.Algorithm.winograd, 32, a, b, first, ctx)
    for _ in range(5):
        c = P.Matrix(256, 256, ctx)
        P.gemm_host(P.Algorithm.winograd, 32, a, b, c, ctx)
        assert P.identical(c, first)
