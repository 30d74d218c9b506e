"""GPU drop-in for the reference CLI (mpmm_bench.cpp:66-240): `matmul` and `lu` run on
the GPU and print the reference's CSV; `opcount` (analytic ratios) and `gen` (matrix
text files) are host-side.  Same flags, same exit codes (1 error, 2 singular pivot in
the sweep, 3 I/O).

    python -m paper_1410_1599_b200.cli matmul --algo all --m 256 --l 256 --n 256 --bits 128 --nmin 32
    python -m paper_1410_1599_b200.cli lu --matrix random --n 128 --bits 256 --kernel winograd \\
        --alpha-sweep 1..10 --nmin 32 --seed 1 [--csv out.csv] [--verbose]
"""
from __future__ import annotations

import argparse
import sys

EXIT_ERROR, EXIT_SINGULAR, EXIT_IO = 1, 2, 3
KINDS = ["simple", "block", "strassen", "winograd"]


def _range(s: str):
    if ".." not in s:
        return None
    lo, hi = s.split("..", 1)
    return int(lo), int(hi)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="mpmm-bench-gpu",
                                 description="arbitrary-precision matrix multiplication and blocked LU benchmark "
                                             "(B200 path)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    mm = sub.add_parser("matmul", help="benchmark the multiplication algorithms")
    mm.add_argument("--algo", default="all", choices=KINDS + ["all"])
    mm.add_argument("--m", type=int, default=256)
    mm.add_argument("--l", type=int, default=256)
    mm.add_argument("--n", type=int, default=256)
    mm.add_argument("--bits", type=int, default=128)
    mm.add_argument("--nmin", type=int, default=32)
    mm.add_argument("--ref-bits-multiplier", type=int, default=2)
    mm.add_argument("--verbose", action="store_true")
    mm.add_argument("--csv", default="")
    lu = sub.add_parser("lu", help="benchmark column-wise vs blocked elimination")
    lu.add_argument("--matrix", default="random", choices=["random", "lotkin"])
    lu.add_argument("--n", type=int, default=128)
    lu.add_argument("--bits", type=int, default=256)
    lu.add_argument("--kernel", default="winograd", choices=KINDS)
    lu.add_argument("--alpha-sweep", default="1..10")
    lu.add_argument("--nmin", type=int, default=32)
    lu.add_argument("--seed", type=int, default=1)
    lu.add_argument("--verbose", action="store_true")
    lu.add_argument("--csv", default="")
    oc = sub.add_parser("opcount", help="analytic operation-count ratios")
    oc.add_argument("--sizes", required=True, help="sizes: integers and/or a..b ranges, comma-separated")
    oc.add_argument("--nmin", type=int, default=32)
    oc.add_argument("--format", default="table", choices=["table", "csv"])
    gn = sub.add_parser("gen", help="write a generated matrix as text")
    gn.add_argument("--kind", default="lotkin", choices=["bench-a", "bench-b", "random", "lotkin"])
    gn.add_argument("--m", type=int, default=4)
    gn.add_argument("--l", type=int, default=4)
    gn.add_argument("--n", type=int, default=4)
    gn.add_argument("--bits", type=int, default=128)
    gn.add_argument("--seed", type=int, default=1)
    gn.add_argument("--out", default="")
    a = ap.parse_args(argv)

    from . import benchdrv as B
    from .codec import IoError
    from .mpmm import Error, SingularError, parse_algorithm

    def emit(rows, path):
        if path:
            B.append_csv(path, rows)
        else:
            B.print_csv(sys.stdout, rows)

    try:
        if a.cmd == "opcount":
            rows = B.ratio_table(B.parse_sizes([t for t in a.sizes.split(",") if t]), a.nmin)
            sys.stdout.write(B.format_ratio_table(rows) if a.format == "table" else B.format_ratio_csv(rows))
            return 0
        if a.cmd == "gen":
            from . import codec
            from .matgen import gen_random
            from .mpmm import PrecisionContext
            ctx = PrecisionContext(a.bits)
            if a.kind == "bench-a":
                x = B.gen_bench_pair(a.m, a.l, 1, ctx)[0]
            elif a.kind == "bench-b":
                x = B.gen_bench_pair(1, a.l, a.n, ctx)[1]
            elif a.kind == "random":
                x = gen_random(a.m, a.n, a.seed, ctx)
            else:
                x = B.gen_lotkin(a.n, ctx)
            if not a.out:
                codec.write_matrix(sys.stdout, x)
                return 0
            try:
                with open(a.out, "w") as f:
                    codec.write_matrix(f, x)
            except OSError as e:
                raise IOError(f"cannot open output file: {a.out}") from e
            return 0
        if a.cmd == "matmul":
            algos = [parse_algorithm(k) for k in KINDS] if a.algo == "all" else [parse_algorithm(a.algo)]
            q = B.MatmulRequest(algos, a.m, a.l, a.n, a.bits, a.nmin, a.ref_bits_multiplier, a.verbose)
            emit(B.run_matmul(q), a.csv)
            return 0
        r = _range(a.alpha_sweep)
        if r is None:
            raise Error(f"bad --alpha-sweep value '{a.alpha_sweep}', expected a..b")
        q = B.LURequest(a.matrix, a.n, a.bits, parse_algorithm(a.kernel), a.nmin, r[0], r[1], a.seed, a.verbose)
        out = B.run_lu(q)
        emit(out.rows, a.csv)
        if out.any_singular:
            print("singular pivot encountered during the sweep", file=sys.stderr)
            return EXIT_SINGULAR
        return 0
    except SingularError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_SINGULAR
    except (IOError, OSError, IoError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_IO
    except Exception as e:  # noqa: BLE001 -- mirrors the reference's catch-all
        print(f"error: {e}", file=sys.stderr)
        return EXIT_ERROR

if __name__ == "__main__":
    sys.exit(main())
