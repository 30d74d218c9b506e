"""Pin the oracle before trusting it (CPU only).

1. The reference tests' own golden vectors / known answers (test_matgen.cpp,
   test_fastmm.cpp, test_blocklu.cpp, test_opmodel.cpp), checked on BOTH the C
   restatement (oracle/mp_oracle.c) and the compiled reference (oracle/_ref).
2. The restatement against the compiled reference on seeded inexact inputs
   (bit-exact), and against the frozen reference fixtures in tests/golden/.
"""
from pathlib import Path

import numpy as np
import pytest

GOLD = Path(__file__).resolve().parent / "golden"


def need_ref(O):
    if not O.have_ref():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")


def same(x, y):
    return (x.rows(), x.cols(), x.bits()) == (y.rows(), y.cols(), y.bits()) and np.array_equal(
        x.exp, y.exp) and np.array_equal(x.sign, y.sign) and np.array_equal(
            x.limbs[-min(x.nlimbs, y.nlimbs):], y.limbs[-min(x.nlimbs, y.nlimbs):])


def load(d, p, O):
    r, c, bits = (int(v) for v in d[p + "_shape"])
    return O.OMat(r, c, bits, d[p + "_limbs"], d[p + "_exp"], d[p + "_sign"])


# ---- 1. golden vectors from the reference's tests ---------------------------

@pytest.mark.parametrize("which", ["orc", "ref"])
def test_prng_golden_stream(O, which):
    if which == "ref":
        need_ref(O)
    # test_matgen.cpp:8-13
    assert O.prng_stream(1, 3, which) == [5180492295206395165, 12380297144915551517, 13389498078930870103]
    # test_matgen.cpp:15-18 (seed 0 remapped)
    assert O.prng_stream(0, 4, which) == O.prng_stream(0x9E3779B97F4A7C15, 4, which)


@pytest.mark.parametrize("which", ["orc", "ref"])
def test_frozen_uniforms(O, which):
    need_ref(O)  # to_hex is the reference's codec
    # test_matgen.cpp:20-26
    x = O.gen_random(3, 1, 1, 53, which)
    assert O.to_hex(x) == ["-0x1.c0d98da3b4994p-2", "0x1.5e7d354703cbp-2", "0x1.ce886c7f5b98cp-2"]


@pytest.mark.parametrize("which", ["orc", "ref"])
def test_two_by_two_traces(O, which):
    if which == "ref":
        need_ref(O)
    # test_fastmm.cpp:91-116
    a = O.from_si([1, 2, 3, 4], 64, 2, 2)
    b = O.from_si([5, 6, 7, 8], 64, 2, 2)
    c, sums, prods, t, _ = O.fast_mul_trace("winograd", 1, a, b, which)
    v = lambda ms: [O.to_double(m)[0, 0] for m in ms]
    assert v(sums) == [7, 6, -2, -4, 1, 7, 2, 0]
    assert v(prods) == [42, 5, 14, -4, 7, -32, 0]
    assert v(t) == [47, 43]
    assert O.to_double(c).ravel().tolist() == [19, 22, 43, 50]
    c, sums, prods, t, _ = O.fast_mul_trace("strassen", 1, a, b, which)
    assert v(prods) == [65, 35, -2, 8, 24, 22, -30] and sums == [] and t == []
    _, ops = O.gemm("winograd", 1, a, b)
    assert ops == (7, 15)
    _, ops = O.gemm("strassen", 1, a, b)
    assert ops == (7, 18)


@pytest.mark.parametrize("which", ["orc", "ref"])
def test_exact_lu_fixture(O, which):
    if which == "ref":
        need_ref(O)
    # test_blocklu.cpp:36-39 kExactA / kExactPacked, kernels x K = 2, n_min = 1
    A = O.from_si([2, 1, 3, 1, 4, 3, 8, 3, 6, 4, 14, 6, 2, 3, 10, 9], 256, 4, 4)
    want = O.from_si([2, 1, 3, 1, 2, 1, 2, 1, 3, 1, 3, 2, 1, 2, 1, 4], 256, 4, 4)
    for k in ["simple", "block", "strassen", "winograd"]:
        f, _, _ = O.lu_blocked(A, 2, k, 1, which=which)
        assert same(f, want), k


@pytest.mark.parametrize("which", ["orc", "ref"])
def test_zero_pivot_index(O, which):
    if which == "ref":
        need_ref(O)
    # test_blocklu.cpp:65-80 (lu_columnwise == blocked with K >= n)
    for vals, piv in (([0, 1, 1, 0], 1), ([1, 1, 1, 1], 2)):
        with pytest.raises(O.OracleError) as e:
            O.lu_blocked(O.from_si(vals, 64, 2, 2), 2, "simple", 1, which=which)
        assert e.value.rc == 3 and e.value.pivot == piv


def test_count_landmarks(O):
    # test_opmodel.cpp:7-31
    assert O.count_fast("simple", 512, 512, 512, 1) == (134217728, 133955584)
    assert O.count_fast("strassen", 512, 512, 512, 32)[0] == 78675968
    assert O.count_fast("strassen", 2, 2, 2, 1) == (7, 18)
    assert O.count_fast("winograd", 2, 2, 2, 1) == (7, 15)
    assert O.count_fast("strassen", 255, 255, 255, 32)[0] == 343 * 32768
    # cfg2 / cfg3 / cfg4 op counts
    assert O.count_fast("winograd", 1024, 1024, 1024, 64) == (629407744, 663502848)
    assert O.count_fast("winograd", 1001, 777, 1537, 32)[0] == 658834400
    assert O.count_fast("winograd", 4096, 4096, 4096, 512)[0] == 46036680704


def test_count_matches_reference(O):
    need_ref(O)
    rng = np.random.default_rng(3)
    for _ in range(200):
        m, l, n = (int(v) for v in rng.integers(1, 3000, 3))
        nm = int(rng.integers(1, 80))
        for alg in ("simple", "strassen", "winograd"):
            assert O.count_fast(alg, m, l, n, nm) == O.count_fast(alg, m, l, n, nm, "ref")


def test_recursion_plans(O):
    need_ref(O)
    # test_fastmm.cpp:66-89
    p = O.recursion_plan(64, 64, 64, 32)
    assert len(p) == 2 and p[0][4:7] == (64, 64, 64) and p[1][7] == 1 and p[1][1:4] == (32, 32, 32)
    assert len(O.recursion_plan(32, 32, 32, 32)) == 1
    r = O.recursion_plan(1024, 63, 1024, 32)
    assert len(r) == 2 and r[0][4:7] == (1024, 64, 1024) and r[1][1:4] == (512, 32, 512)
    d = O.recursion_plan(2048, 2048, 2048, 32)
    assert len(d) == 7 and d[-1][1:4] == (32, 32, 32)


# ---- 2. restatement vs compiled reference ------------------------------------

@pytest.mark.parametrize("alg,param", [("simple", 0), ("block", 7), ("strassen", 6), ("winograd", 6),
                                       ("winograd", 1)])
@pytest.mark.parametrize("bits", [53, 128, 256, 300])
def test_restatement_matches_reference_gemm(O, alg, param, bits):
    need_ref(O)
    a = O.gen_full(0, 23, 19, 5 + bits, bits)
    b = O.gen_full(0, 19, 27, 6 + bits, bits)
    c1, o1 = O.gemm(alg, param, a, b)
    c2, o2 = O.gemm(alg, param, a, b, which="ref")
    assert same(c1, c2) and o1 == o2


@pytest.mark.parametrize("kernel", ["simple", "block", "strassen", "winograd"])
def test_restatement_matches_reference_lu(O, kernel):
    need_ref(O)
    a = O.gen_full(0, 29, 29, 8, 256)
    f1, _, o1 = O.lu_blocked(a, 6, kernel, 3)
    f2, _, o2 = O.lu_blocked(a, 6, kernel, 3, which="ref")
    assert same(f1, f2) and o1 == o2
    ones = O.from_si(np.ones(29, np.int64), 256, 29, 1)
    b1, b2 = O.mat_vec_mul(a, ones), O.mat_vec_mul(a, ones, "ref")
    assert same(b1, b2)
    assert same(O.lu_solve(f1, b1), O.lu_solve(f2, b2, which="ref"))


def test_pivoting_restatement_is_a_factorisation(O):
    # P A = L U to working precision (the reference has no pivoting to compare to)
    n, bits = 24, 256
    a = O.gen_full(0, n, n, 17, bits)
    f, piv, _ = O.lu_blocked(a, 8, "block", 4, pivoting=True)
    Af = O.to_double(a)
    F = O.to_double(f)
    Lm = np.tril(F, -1) + np.eye(n)
    U = np.triu(F)
    PA = Af.copy()
    for d in range(n):
        PA[[d, piv[d]]] = PA[[piv[d], d]]
    assert np.max(np.abs(PA - Lm @ U)) < 1e-12
    assert np.all(np.abs(np.tril(F, -1)) <= 1.0)  # |multipliers| <= 1


@pytest.mark.parametrize("path", sorted(GOLD.glob("gemm_*.npz")), ids=lambda p: p.stem)
def test_restatement_matches_golden_gemm(O, path):
    d = np.load(path)
    a, b, c = load(d, "a", O), load(d, "b", O), load(d, "c", O)
    got, ops = O.gemm(str(d["alg"]), int(d["param"]), a, b)
    assert same(got, c) and ops == tuple(int(v) for v in d["ops"])


@pytest.mark.parametrize("path", sorted(GOLD.glob("lu_*.npz")), ids=lambda p: p.stem)
def test_restatement_matches_golden_lu(O, path):
    d = np.load(path)
    a, f, b, x = (load(d, p, O) for p in ("a", "f", "b", "x"))
    got, _, ops = O.lu_blocked(a, int(d["K"]), str(d["kernel"]), int(d["n_min"]))
    assert same(got, f) and ops == tuple(int(v) for v in d["ops"])
    assert same(O.lu_solve(f, b), x)
