"""A/B timing of the leaf kernel: Winograd n=1024 (n_min 64) at several precisions,
min over repetitions of the leaf and whole-step device times.  Select a library
variant with MPGPU_LIB=paper_1410_1599_b200/_variants/<name>/libmpgpu.so.

    python tools/ab_leaf.py [--bits 256 512 1024] [--reps 5] [--tag name]
"""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bits", type=int, nargs="+", default=[256, 512, 1024])
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--shape", default=None, help="m,l,n (overrides --n)")
    ap.add_argument("--gen", default="uniform_full", choices=["uniform_full", "scaled"])
    ap.add_argument("--n-min", type=int, default=64)
    ap.add_argument("--algo", default="winograd")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--tag", default=os.environ.get("MPGPU_LIB", "default"))
    a = ap.parse_args()
    import paper_1410_1599_b200 as P
    algo = P.Algorithm[a.algo]
    for bits in a.bits:
        ctx = P.PrecisionContext(bits)
        m, l, n = (int(x) for x in a.shape.split(",")) if a.shape else (a.n, a.n, a.n)
        gen = P.gen_scaled if a.gen == "scaled" else P.gen_uniform_full
        A = gen(m, l, 1, ctx).to_device()
        B = gen(l, n, 2, ctx).to_device()
        C = P.DeviceMatrix(m, n, ctx)
        leaf, dev, pre, post = [], [], [], []
        for _ in range(a.reps + 1):
            st = P.gemm_into(algo, a.n_min if algo != P.Algorithm.simple else 0, A, B, C)
            leaf.append(st.leaf_ms)
            dev.append(st.device_ms)
            pre.append(st.preadd_ms)
            post.append(st.postadd_ms)
        print(json.dumps({"tag": a.tag, "algo": a.algo, "shape": [m, l, n], "n_min": a.n_min, "bits": bits,
                          "leaf_ms": min(leaf[1:]), "device_ms": min(dev[1:]), "preadd_ms": min(pre[1:]),
                          "postadd_ms": min(post[1:])}), flush=True)


if __name__ == "__main__":
    main()
