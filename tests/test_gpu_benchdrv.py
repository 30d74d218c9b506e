"""GPU benchmark driver and device-side accuracy metrics vs the compiled reference:
max_rel_error / max_rel_error_solution / one_norm identical to the reference's
(matrix.hpp:237-279, blocklu.hpp:306-333), and run_matmul / run_lu CSV rows
identical to the reference's own run_matmul / run_lu except wall_seconds
(bench.hpp:117-249)."""
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import oracle.oracle as O
import paper_1410_1599_b200 as P
from paper_1410_1599_b200 import benchdrv as B

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(not O.have_ref(), reason="compiled reference not built")
ROOT = Path(__file__).resolve().parent.parent


def same_values(a, b):
    assert P.to_fractions(a) == P.to_fractions(b)


def _perturbed(x, seed, bits):
    """x at `bits` plus a few ulps of noise (an 'approximation' of x)."""
    ctx = P.PrecisionContext(bits)
    rng = np.random.default_rng(seed)
    y = P.Matrix(x.rows(), x.cols(), ctx)
    L, Lx = y.nlimbs, x.nlimbs
    # truncate x's mantissa to L limbs (most significant aligned), then flip low bits
    y.limbs[:] = x.limbs[Lx - L:]
    y.exp[:] = x.exp
    y.sign[:] = x.sign
    sh = 32 * L - bits
    noise = rng.integers(0, 1 << 12, size=y.exp.size, dtype=np.uint64).astype(np.uint32) << np.uint32(sh)
    nz = y.exp != P.EXP_ZERO
    y.limbs[0, nz] ^= noise[nz]
    y.limbs[0] &= np.uint32((0xFFFFFFFF << sh) & 0xFFFFFFFF)
    return y


@needs_ref
@pytest.mark.parametrize("bits,ref_bits", [(24, 48), (64, 128), (256, 512), (500, 1000), (1024, 2048), (256, 256)])
def test_max_rel_error_matches_reference(bits, ref_bits):
    ref = P.gen_uniform_full(9, 13, 5, P.PrecisionContext(ref_bits))
    ref.exp[[3, 40]] = P.EXP_ZERO  # zero references are skipped and counted
    ref.limbs[:, [3, 40]] = 0
    approx = _perturbed(ref, 7, bits)
    st = P.max_rel_error(approx, ref)
    want, skipped = O.max_rel_error(approx, ref)
    assert st.skipped_zero_refs == skipped == 2
    same_values(st.max, O.OMat(1, 1, ref_bits, want.limbs[:, :1], want.exp[:1], want.sign[:1]))
    same_values(st.min, O.OMat(1, 1, ref_bits, want.limbs[:, 1:], want.exp[1:], want.sign[1:]))


def test_max_rel_error_edge_cases():
    ctx = P.PrecisionContext(128)
    x = P.gen_uniform_full(4, 4, 1, ctx)
    st = P.max_rel_error(x, x)
    assert P.to_fractions(st.max) == [0] and P.to_fractions(st.min) == [0]
    z = P.Matrix(4, 4, ctx)
    with pytest.raises(P.UndefinedMetricError):
        P.max_rel_error(x, z)
    with pytest.raises(P.DimensionError):
        P.max_rel_error(x, P.Matrix(4, 5, ctx))
    with pytest.raises(P.DomainError):  # approximation wider than the reference
        P.max_rel_error(P.gen_uniform_full(4, 4, 1, P.PrecisionContext(512)), x)


@needs_ref
@pytest.mark.parametrize("bits", [53, 256, 1024])
def test_solution_error_matches_reference(bits):
    ctx = P.PrecisionContext(bits)
    xt = P.from_ints(np.arange(40, dtype=np.int64) - 3, ctx, 40, 1)  # one zero component
    xh = _perturbed(xt, 3, bits)
    xh.exp[3] = 10  # nonzero estimate of the zero component
    xh.limbs[:, 3] = 0
    xh.limbs[-1, 3] = 0x80000000
    se = P.max_rel_error_solution(xh, xt)
    want, zr = O.solution_error(xh, xt)
    assert se.zero_refs == zr == 1
    same_values(se.max_rel, O.OMat(1, 1, bits, want.limbs[:, :1], want.exp[:1], want.sign[:1]))
    same_values(se.max_zero_abs, O.OMat(1, 1, bits, want.limbs[:, 1:], want.exp[1:], want.sign[1:]))


@needs_ref
@pytest.mark.parametrize("bits", [24, 256, 1000])
@pytest.mark.parametrize("rows,cols", [(1, 1), (7, 5), (64, 33)])
def test_one_norm_matches_reference(bits, rows, cols):
    a = P.gen_uniform_full(rows, cols, rows + cols, P.PrecisionContext(bits))
    same_values(P.one_norm(a), O.one_norm(a))


def _strip_wall(text):
    out = []
    for line in text.strip().splitlines():
        f = line.split(",")
        if f[0] != "command":
            f[10] = "T"
        out.append(",".join(f))
    return out


def _csv(rows):
    import io
    s = io.StringIO()
    B.print_csv(s, rows)
    return s.getvalue()


@needs_ref
@pytest.mark.parametrize("m,l,n,bits,n_min,verbose", [(12, 10, 14, 128, 4, False), (20, 17, 9, 256, 3, True),
                                                     (16, 16, 16, 1024, 4, False), (9, 8, 10, 53, 2, True)])
def test_run_matmul_rows_match_reference(m, l, n, bits, n_min, verbose):
    rows = B.run_matmul(B.MatmulRequest(m=m, l=l, n=n, bits=bits, n_min=n_min, verbose=verbose))
    assert _strip_wall(_csv(rows)) == _strip_wall(O.run_matmul(m, l, n, bits, n_min, verbose=verbose))


@needs_ref
def test_run_matmul_ref_multiplier_one():
    rows = B.run_matmul(B.MatmulRequest(algos=[P.Algorithm.winograd], m=10, l=10, n=10, bits=200, n_min=4,
                                        ref_bits_multiplier=1))
    assert _strip_wall(_csv(rows)) == _strip_wall(O.run_matmul(10, 10, 10, 200, 4, algos=("winograd",),
                                                               ref_mult=1))


@needs_ref
@pytest.mark.parametrize("kind,n,bits,kernel,n_min,alo,ahi,verbose", [
    ("random", 24, 256, "winograd", 4, 1, 3, False),
    ("random", 17, 128, "block", 3, 1, 2, True),
    ("lotkin", 12, 128, "simple", 4, 1, 2, True),
    ("lotkin", 10, 24, "strassen", 2, 2, 3, False),
])
def test_run_lu_rows_match_reference(kind, n, bits, kernel, n_min, alo, ahi, verbose):
    out = B.run_lu(B.LURequest(kind, n, bits, P.parse_algorithm(kernel), n_min, alo, ahi, 1, verbose))
    text, singular = O.run_lu(kind, n, bits, kernel, n_min, alo, ahi, 1, verbose)
    assert out.any_singular == singular
    assert _strip_wall(_csv(out.rows)) == _strip_wall(text)


def test_cli_matmul_and_lu(tmp_path):
    env_py = sys.executable
    r = subprocess.run([env_py, "-m", "paper_1410_1599_b200.cli", "matmul", "--algo", "winograd", "--m", "8",
                        "--l", "8", "--n", "8", "--bits", "128", "--nmin", "2"], cwd=ROOT, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().splitlines()
    assert lines[0] == B.CSV_HEADER and lines[1].startswith("matmul,winograd,8,8,8,128,2,,,,")
    csvp = tmp_path / "lu.csv"
    r = subprocess.run([env_py, "-m", "paper_1410_1599_b200.cli", "lu", "--n", "8", "--bits", "64",
                        "--kernel", "block", "--alpha-sweep", "1..2", "--nmin", "2", "--csv", str(csvp)],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert csvp.read_text().splitlines()[0] == B.CSV_HEADER and len(csvp.read_text().splitlines()) == 4
    r = subprocess.run([env_py, "-m", "paper_1410_1599_b200.cli", "lu", "--alpha-sweep", "x"], cwd=ROOT,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 1


def test_wide_matrices_round_trip_and_limit():
    ctx = P.PrecisionContext(2048)
    a = P.gen_uniform_full(3, 3, 1, ctx)
    d = a.to_device()
    assert P.identical(d.download(), a)  # upload / download round trip at 64 limbs
    d.free()
    with pytest.raises(P.DomainError):  # above MPGPU_MAX_PREC (9216 bits)
        P.DeviceMatrix(2, 2, P.PrecisionContext(9217))
