"""K1 leaf GEMM + K2/K3 fast-algorithm kernels through the C-ABI vs the oracle.

Bit-exact against the C restatement (oracle/mp_oracle.c) and the compiled
reference (oracle/_ref) for Simple (matrix.hpp:178-184), Block (matrix.hpp:225-233),
Strassen and Winograd (fastmm.hpp:244-255) -- the GPU replays the reference's
operation DAG, so results are identical element for element (signs of zeros too).
"""
import numpy as np
import pytest

ALGS = ["simple", "block", "strassen", "winograd"]


def _run(P, alg, param, a, b, ctx, ops=None):
    if alg == "simple":
        return P.simple_mul(a, b, ctx, ops)
    if alg == "block":
        return P.block_mul(a, b, param, ctx, ops)
    r = P.fast_mul(a, b, P.FastMMConfig(P.Algorithm[alg], param), ctx)
    if ops is not None:
        ops += r.ops
    return r.c


CASES = [
    # (m, l, n, bits, param)
    (16, 16, 16, 128, 4),
    (33, 17, 29, 128, 8),
    (64, 64, 64, 256, 16),
    (45, 63, 50, 256, 7),
    (24, 40, 31, 512, 5),
    (17, 19, 23, 1024, 4),
    (40, 40, 40, 53, 8),
    (21, 22, 23, 2, 3),
    (30, 30, 30, 200, 6),
    (65, 33, 66, 64, 16),
]


@pytest.mark.gpu
@pytest.mark.parametrize("m,l,n,bits,param", CASES)
@pytest.mark.parametrize("alg", ALGS)
def test_gemm_bit_exact_vs_oracle(P, O, alg, m, l, n, bits, param):
    ctx = P.PrecisionContext(bits)
    a = P.gen_uniform_full(m, l, 7 + m, ctx)
    b = P.gen_uniform_full(l, n, 9 + n, ctx)
    ops = P.OpCounter()
    c = _run(P, alg, param, a, b, ctx, ops)
    want, wops = O.gemm(alg, param, O.OMat.of(a), O.OMat.of(b))
    assert P.identical(c, want)
    assert (ops.mul, ops.addsub) == wops


@pytest.mark.gpu
@pytest.mark.parametrize("alg", ALGS)
def test_gemm_scaled_inputs_cfg3_shape_small(P, O, alg):
    # config 3's distribution (exponents in [-20,20], random signs) at odd dims
    ctx = P.PrecisionContext(512)
    a = P.gen_scaled(37, 29, 3, ctx)
    b = P.gen_scaled(29, 45, 4, ctx)
    c = _run(P, alg, 4, a, b, ctx)
    want, _ = O.gemm(alg, 4, O.OMat.of(a), O.OMat.of(b))
    assert P.identical(c, want)


@pytest.mark.gpu
@pytest.mark.parametrize("alg", ALGS)
def test_gemm_vs_compiled_reference(P, O, alg):
    if not O.have_ref():
        pytest.skip("oracle/_ref not built")
    ctx = P.PrecisionContext(256)
    a = P.gen_uniform_full(37, 41, 11, ctx)
    b = P.gen_uniform_full(41, 35, 12, ctx)
    c = _run(P, alg, 8, a, b, ctx)
    want, _ = O.gemm(alg, 8, O.OMat.of(a), O.OMat.of(b), which="ref")
    assert P.identical(c, want)


@pytest.mark.gpu
def test_exact_integer_inputs_all_algorithms_agree(P):
    # test_fastmm.cpp:130-149 style: integer inputs make every op exact
    ctx = P.PrecisionContext(256)
    rng = P.Prng64(31337)
    for _ in range(12):
        m, l, n = (1 + rng.next64() % 96 for _ in range(3))
        n_min = [1, 8, 32][rng.next64() % 3]
        A = np.array([(rng.next64() % 2049) - 1024 for _ in range(m * l)], np.int64).reshape(m, l)
        B = np.array([(rng.next64() % 2049) - 1024 for _ in range(l * n)], np.int64).reshape(l, n)
        a, b = P.from_ints(A, ctx), P.from_ints(B, ctx)
        exact = P.from_ints(A @ B, ctx)
        for alg in ALGS:
            c = _run(P, alg, n_min, a, b, ctx)
            assert P.equal_values(c, exact), (alg, m, l, n, n_min)


@pytest.mark.gpu
def test_winograd_2x2_trace(P):
    # test_fastmm.cpp:105-116
    ctx = P.PrecisionContext(64)
    a = P.from_ints([[1, 2], [3, 4]], ctx)
    b = P.from_ints([[5, 6], [7, 8]], ctx)
    tr = P.TopTrace()
    r = P.fast_mul(a, b, P.FastMMConfig(P.Algorithm.winograd, 1), ctx, tr)
    assert P.equal_values(r.c, P.from_ints([[19, 22], [43, 50]], ctx))
    vals = lambda ms: [int(m.to_float()[0, 0]) for m in ms]
    assert vals(tr.sums) == [7, 6, -2, -4, 1, 7, 2, 0]
    assert vals(tr.products) == [42, 5, 14, -4, 7, -32, 0]
    assert vals(tr.t) == [47, 43]
    assert (r.ops.mul, r.ops.addsub) == (7, 15)
    tr2 = P.TopTrace()
    r2 = P.fast_mul(a, b, P.FastMMConfig(P.Algorithm.strassen, 1), ctx, tr2)
    assert vals(tr2.products) == [65, 35, -2, 8, 24, 22, -30]
    assert tr2.sums == [] and (r2.ops.mul, r2.ops.addsub) == (7, 18)


@pytest.mark.gpu
def test_errors(P):
    ctx = P.PrecisionContext(64)
    a, b = P.Matrix(2, 3, ctx), P.Matrix(2, 2, ctx)
    with pytest.raises(P.DimensionError):
        P.fast_mul(a, b, P.FastMMConfig(P.Algorithm.strassen, 1), ctx)
    c = P.Matrix(3, 2, ctx)
    with pytest.raises(P.DomainError):
        P.fast_mul(a, c, P.FastMMConfig(P.Algorithm.simple, 1), ctx)
    with pytest.raises(P.DimensionError):
        P.fast_mul(a, c, P.FastMMConfig(P.Algorithm.strassen, 0), ctx)
    with pytest.raises(P.DimensionError):
        P.block_mul(a, c, 0, ctx)


@pytest.mark.gpu
def test_cfg1_all_four_bit_exact_and_reference_inputs(P, O):
    # BASELINE config 1: n=128 @128 bits, block 32, cutoff 32
    ctx = P.PrecisionContext(128)
    for gen in (P.gen_uniform_full, P.gen_random):
        a, b = gen(128, 128, 1, ctx), gen(128, 128, 2, ctx)
        for alg in ALGS:
            c = _run(P, alg, 32, a, b, ctx)
            want, _ = O.gemm(alg, 32, O.OMat.of(a), O.OMat.of(b))
            assert P.identical(c, want), alg


GOLD = __import__("pathlib").Path(__file__).resolve().parent / "golden"


@pytest.mark.gpu
@pytest.mark.parametrize("path", sorted(GOLD.glob("gemm_*.npz")), ids=lambda p: p.stem)
def test_gemm_matches_frozen_reference_fixture(P, path):
    d = np.load(path)

    def mat(p):
        r, c, bits = (int(v) for v in d[p + "_shape"])
        return P.Matrix(r, c, P.PrecisionContext(bits), d[p + "_limbs"], d[p + "_exp"], d[p + "_sign"])

    a, b, want = mat("a"), mat("b"), mat("c")
    ops = P.OpCounter()
    c = _run(P, str(d["alg"]), int(d["param"]), a, b, a.ctx(), ops)
    assert P.identical(c, want)
    assert (ops.mul, ops.addsub) == tuple(int(v) for v in d["ops"])


@pytest.mark.gpu
@pytest.mark.parametrize("alg,param", [("winograd", 8), ("block", 16), ("simple", 0)])
def test_gemm_host_buffers_path(P, O, alg, param):
    # mpgpu_gemm_host: the reference-facing call with host SoA buffers (bench e2e path)
    ctx = P.PrecisionContext(200)  # host limbs 7 < device limbs 8
    a, b = P.gen_uniform_full(40, 33, 1, ctx), P.gen_uniform_full(33, 29, 2, ctx)
    c = P.Matrix(40, 29, ctx)
    st = P.gemm_host(P.Algorithm[alg], param, a, b, c, ctx)
    want, ops = O.gemm(alg, param, O.OMat.of(a), O.OMat.of(b))
    assert P.identical(c, want)
    assert (st.mul, st.addsub) == ops


@pytest.mark.gpu
def test_randomized_shapes_precisions_algorithms(P, O):
    # seeded sweep over shapes (incl. 1-wide and odd), precisions and cutoffs
    rng = np.random.default_rng(20261020)
    for _ in range(40):
        m, l, n = (int(v) for v in rng.integers(1, 70, 3))
        bits = int(rng.choice([2, 24, 33, 64, 97, 128, 160, 256, 300, 512, 700, 1024]))
        alg = str(rng.choice(ALGS))
        param = int(rng.integers(1, 20))
        gen = [P.gen_uniform_full, P.gen_scaled, P.gen_random][int(rng.integers(0, 3))]
        ctx = P.PrecisionContext(bits)
        a, b = gen(m, l, int(rng.integers(1, 1 << 30)), ctx), gen(l, n, int(rng.integers(1, 1 << 30)), ctx)
        ops = P.OpCounter()
        c = _run(P, alg, param if alg != "simple" else 0, a, b, ctx, ops)
        want, wops = O.gemm(alg, param if alg != "simple" else 0, O.OMat.of(a), O.OMat.of(b))
        assert P.identical(c, want), (m, l, n, bits, alg, param)
        assert (ops.mul, ops.addsub) == wops


@pytest.mark.gpu
@pytest.mark.parametrize("alg", ["strassen", "winograd"])
def test_deep_recursion_more_leaves_than_grid_z(P, O, alg):
    # n_min 1 at n = 100: depth 7, 7^7 = 823543 leaves > 65535 (grid.z limit): the leaf
    # launch is split into batch chunks
    ctx = P.PrecisionContext(64)
    a = P.gen_uniform_full(100, 100, 3, ctx)
    b = P.gen_uniform_full(100, 100, 4, ctx)
    c = _run(P, alg, 1, a, b, ctx, P.OpCounter())
    want, _ = O.gemm(alg, 1, O.OMat.of(a), O.OMat.of(b))
    assert P.identical(c, want)


@pytest.mark.gpu
@pytest.mark.parametrize("bits", [256, 512, 1024])
@pytest.mark.parametrize("alg,param", [("simple", 0), ("block", 8), ("winograd", 16)])
def test_ragged_leaf_half_width_tiles(P, O, alg, param, bits):
    """32 x 25 x 49 (config 3's n_min-32 leaf shape): launch_gemm picks the half-width,
    double-height tile (it covers 32 x 56 outputs instead of 32 x 64) -- bit-exact."""
    ctx = P.PrecisionContext(bits)
    a = P.gen_scaled(32, 25, 21, ctx)
    b = P.gen_scaled(25, 49, 22, ctx)
    if alg == "simple":
        c = P.simple_mul(a, b, ctx)
    elif alg == "block":
        c = P.block_mul(a, b, param, ctx)
    else:
        c = P.fast_mul(a, b, P.FastMMConfig(P.Algorithm.winograd, param), ctx).c
    want, _ = O.gemm(alg, param, O.OMat.of(a), O.OMat.of(b))
    assert P.identical(c, want)


@pytest.mark.gpu
@pytest.mark.parametrize("alg,param", [("simple", 0), ("block", 5), ("strassen", 3), ("winograd", 3)])
@pytest.mark.parametrize("bits", [64, 256])
def test_zeros_signed_zeros_and_exact_cancellation(P, O, alg, param, bits):
    # sparse operands with +0 / -0 entries and rows that cancel exactly: the zero paths of the
    # primitives (RN(-0 + -0) = -0, RN(x - x) = +0) inside the leaf, the pre- and post-additions
    ctx = P.PrecisionContext(bits)
    rng = np.random.default_rng(bits + param)
    m, l, n = 23, 18, 21
    a = P.gen_uniform_full(m, l, 5, ctx)
    b = P.gen_uniform_full(l, n, 6, ctx)
    za = rng.random(m * l) < 0.4
    zb = rng.random(l * n) < 0.4
    for x, z in ((a, za), (b, zb)):
        x.limbs[:, z] = 0
        x.exp[z] = P.EXP_ZERO
        x.sign[z] = rng.integers(0, 2, int(z.sum())).astype(np.uint8)  # both zero signs
    # row 1 of A = -(row 0): exact cancellation in every product row pair of the Winograd sums
    a.limbs[:, l:2 * l] = a.limbs[:, 0:l]
    a.exp[l:2 * l] = a.exp[0:l]
    a.sign[l:2 * l] = 1 - a.sign[0:l]
    ops = P.OpCounter()
    c = _run(P, alg, param, a, b, ctx, ops)
    want, wops = O.gemm(alg, param, O.OMat.of(a), O.OMat.of(b))
    assert P.identical(c, want)  # signs of zeros included
    assert (ops.mul, ops.addsub) == wops
