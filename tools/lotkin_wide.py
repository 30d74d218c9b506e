"""The paper's ill-conditioned experiment on the GPU: run_lu on the
Lotkin matrix at 8192 / 8650 bits (wide formats), the reference's CSV rows.

    python tools/lotkin_wide.py [--n 256] [--bits 8192] [--kernel winograd] [--alpha 1..2]
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--bits", type=int, default=8192)
    ap.add_argument("--kernel", default="winograd")
    ap.add_argument("--alpha", default="1..2")
    ap.add_argument("--nmin", type=int, default=32)
    a = ap.parse_args()
    import paper_1410_1599_b200 as P
    from paper_1410_1599_b200 import benchdrv as B
    lo, hi = (int(x) for x in a.alpha.split(".."))
    t0 = time.perf_counter()
    out = B.run_lu(B.LURequest("lotkin", a.n, a.bits, P.Algorithm[a.kernel], a.nmin, lo, hi, 1, False))
    B.print_csv(sys.stdout, out.rows)
    print(f"# total wall {time.perf_counter() - t0:.1f} s", file=sys.stderr)


if __name__ == "__main__":
    main()
