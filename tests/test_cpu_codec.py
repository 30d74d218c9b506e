"""Host text codec (codec.py) and the CLI's host subcommands vs the compiled reference:
to_hex / from_hex (precision.hpp:204-290) bit-exact including rounding and parse-error
positions, mpmat files (matrix.hpp:309-344) identical in both directions, and the
opcount tables (opmodel.hpp:46-155) character for character."""
import io
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import oracle.oracle as O
import paper_1410_1599_b200 as P
from paper_1410_1599_b200 import benchdrv as B
from paper_1410_1599_b200 import codec

needs_ref = pytest.mark.skipif(not O.have_ref(), reason="compiled reference not built")
ROOT = Path(__file__).resolve().parent.parent


def _mixed(bits, n=40, seed=3):
    x = P.gen_scaled(n, 1, seed, P.PrecisionContext(bits))
    x.exp[:2] = P.EXP_ZERO
    x.limbs[:, :2] = 0
    x.sign[0] = 0
    x.sign[1] = 1  # -0
    return x


@needs_ref
@pytest.mark.parametrize("bits", [2, 24, 53, 64, 100, 256, 1024, 2048])
def test_to_hex_matches_reference(bits):
    x = _mixed(bits)
    assert [codec.to_hex(x, t) for t in range(x.rows())] == O.to_hex(x)


@needs_ref
@pytest.mark.parametrize("bits", [2, 10, 53, 128, 333])
def test_from_hex_rounds_like_mpfr(bits):
    texts = ["0x1p+0", "-0x0p+0", "0x0p+0", "0x1.8p-3", "0x1.fffffffffffffffffp+10", "-0x3.4p2", "0xABC.DEFp-100",
             "+0x1.000000000000000000000000000000001p+0", "0x1.8p+0", "0x1.4p+0", "0x2.8p0", "0X1P+5",
             "0x000.0001p+4", "0x7fffffffffffffffffffffffffffffffffffffffp-160"]
    for t in texts:
        v, neg = codec.from_hex(t, P.PrecisionContext(bits))
        mine = codec.scalar_matrix([v], P.PrecisionContext(bits), 1, 1, [neg])
        want, pos = O.from_hex(t, bits)
        assert pos is None
        assert P.to_fractions(mine) == P.to_fractions(want), t
        assert bool(mine.sign[0]) == bool(want.sign[0]), t


@needs_ref
def test_from_hex_parse_errors_at_the_same_position():
    for t in ["", "1p0", "0y1p0", "0x", "0xp0", "0x1.p0", "0x1", "0x1p", "0x1p+", "0x1p3z", " 0x1p0", "0x1.8q1"]:
        _, pos = O.from_hex(t, 53)
        with pytest.raises(codec.ParseError) as ei:
            codec.from_hex(t, P.PrecisionContext(53))
        assert ei.value.position == pos, t


@needs_ref
@pytest.mark.parametrize("bits", [24, 256, 1024])
def test_mpmat_files_both_directions(bits):
    x = _mixed(bits, 12, 5).reshaped(3, 4)
    s = io.StringIO()
    codec.write_matrix(s, x)
    assert s.getvalue() == O.write_matrix(x)
    back = codec.read_matrix(io.StringIO(s.getvalue()))
    assert P.equal_values(back, x)  # zeros print unsigned (mpfr_sgn), as in the reference
    ref_back = O.read_matrix(s.getvalue())
    assert P.to_fractions(back) == P.to_fractions(ref_back)


def test_read_matrix_errors():
    with pytest.raises(codec.IoError):
        codec.read_matrix(io.StringIO("matrix 1 1 53\n0x1p0\n"))
    with pytest.raises(P.DimensionError):
        codec.read_matrix(io.StringIO("mpmat 0 1 53\n"))
    with pytest.raises(codec.IoError):
        codec.read_matrix(io.StringIO("mpmat 1 2 53\n0x1p0\n"))
    with pytest.raises(codec.ParseError):
        codec.read_matrix(io.StringIO("mpmat 1 1 53\n1.0\n"))


@needs_ref
@pytest.mark.parametrize("fmt", ["table", "csv"])
def test_opcount_tables_match_reference(fmt):
    sizes = B.parse_sizes(["1..70", "100", "1000", "4096"])
    rows = B.ratio_table(sizes, 32)
    mine = B.format_ratio_table(rows) if fmt == "table" else B.format_ratio_csv(rows)
    assert mine == O.ratio_table([s[0] for s in sizes], 32, fmt)


def test_parse_sizes():
    assert [s[0] for s in B.parse_sizes(["1..9", "5"])] == [1, 2, 3, 4, 5, 7, 8, 9]
    with pytest.raises(P.DomainError):
        B.parse_sizes(["5..2"])


@needs_ref
@pytest.mark.parametrize("args,ref", [
    (["gen", "--kind", "lotkin", "--n", "5", "--bits", "100"], lambda: O.gen_lotkin(5, 100)),
    (["gen", "--kind", "random", "--m", "3", "--n", "4", "--bits", "64", "--seed", "9"],
     lambda: O.gen_random(3, 4, 9, 64, "ref")),
    (["gen", "--kind", "bench-a", "--m", "3", "--l", "5", "--bits", "256"], lambda: O.gen_bench_pair(3, 5, 1, 256)[0]),
    (["gen", "--kind", "bench-b", "--l", "4", "--n", "2", "--bits", "53"], lambda: O.gen_bench_pair(1, 4, 2, 53)[1]),
])
def test_cli_gen_matches_reference(args, ref):
    r = subprocess.run([sys.executable, "-m", "paper_1410_1599_b200.cli", *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert r.stdout == O.write_matrix(ref())


def test_cli_opcount_and_io_exit_code(tmp_path):
    r = subprocess.run([sys.executable, "-m", "paper_1410_1599_b200.cli", "opcount", "--sizes", "64,128",
                        "--format", "csv"], cwd=ROOT, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.startswith("m,l,n,n_min,")
    r = subprocess.run([sys.executable, "-m", "paper_1410_1599_b200.cli", "gen", "--out",
                        str(tmp_path / "no" / "such" / "dir.txt")], cwd=ROOT, capture_output=True, text=True,
                       timeout=120)
    assert r.returncode == 3
