"""Driver for ncu launch lists of the blocked LU: python tools/prof_lu.py [--n 1024] [--K 64] [--kernel block]"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--K", type=int, default=64)
    ap.add_argument("--kernel", default="block")
    ap.add_argument("--bits", type=int, default=256)
    ap.add_argument("--pivoting", type=int, default=1)
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--n-min", type=int, default=32)
    a = ap.parse_args()
    import paper_1410_1599_b200 as P
    ctx = P.PrecisionContext(a.bits)
    A = P.gen_uniform_full(a.n, a.n, 11, ctx)
    for _ in range(a.reps):
        st = P.Stats()
        P.lu_blocked(A, P.BlockLUConfig(a.K, P.Algorithm[a.kernel], a.n_min), ctx, pivoting=bool(a.pivoting), stats=st)
        print(f"lu n={a.n} K={a.K} n_min={a.n_min} {a.kernel}: {st.device_ms:.2f} ms (schur leaf {st.leaf_ms:.2f} ms)")


if __name__ == "__main__":
    main()
