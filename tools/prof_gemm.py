"""Small driver for ncu captures: runs one warm-up and one measured MP GEMM.

    python tools/prof_gemm.py [--algo winograd] [--n 1024] [--bits 256] [--n-min 64]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--algo", default="winograd")
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--bits", type=int, default=256)
    ap.add_argument("--n-min", type=int, default=64)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    import paper_1410_1599_b200 as P
    ctx = P.PrecisionContext(a.bits)
    A = P.gen_uniform_full(a.n, a.n, 1, ctx).to_device()
    B = P.gen_uniform_full(a.n, a.n, 2, ctx).to_device()
    C = P.DeviceMatrix(a.n, a.n, ctx)
    algo = P.Algorithm[a.algo]
    for _ in range(a.reps):
        st = P.gemm_into(algo, a.n_min if algo != P.Algorithm.simple else 0, A, B, C)
    print(f"{a.algo} n={a.n} bits={a.bits}: device {st.device_ms:.3f} ms, leaf {st.leaf_ms:.3f} ms")


if __name__ == "__main__":
    main()
