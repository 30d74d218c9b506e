"""GPU drop-in for the reference CLI's `matmul` and `lu` subcommands
(mpmm_bench.cpp:66-79, 137-240): same flags, same CSV, same exit codes
(1 error, 2 singular pivot in the sweep, 3 I/O).

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
    a = ap.parse_args(argv)

    from . import benchdrv as B
    from .mpmm import Error, SingularError, parse_algorithm

    def emit(rows, path):
        if path:
            B.append_csv(path, rows)
        else:
            B.print_csv(sys.stdout, rows)

    try:
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
    except (IOError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_IO
    except Exception as e:  # noqa: BLE001 -- mirrors the reference's catch-all
        print(f"error: {e}", file=sys.stderr)
        return EXIT_ERROR


if __name__ == "__main__":
    sys.exit(main())
