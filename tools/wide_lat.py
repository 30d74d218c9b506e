"""Latency / throughput probe of the wide-format primitives (vec_op kernels): one
element (one warp: latency) and many elements (throughput), ops add, sub, mul, div.
Run under ncu for the per-launch times:  python tools/wide_lat.py [--bits 8192]"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bits", type=int, default=8192)
    ap.add_argument("--many", type=int, default=4096)
    a = ap.parse_args()
    import paper_1410_1599_b200 as P
    ctx = P.PrecisionContext(a.bits)
    for n in (1, a.many):
        x = P.gen_uniform_full(n, 1, 1, ctx)
        y = P.gen_uniform_full(n, 1, 2, ctx)
        for op in (0, 1, 2, 3):
            P.vec_op(op, x, y)


if __name__ == "__main__":
    main()
