"""Wall time of mpgpu_lu_blocked_host (pinned buffers) vs upload + lu_blocked + download at
cfg5(a): n=2048 @256, Winograd Schur K=64, n_min 32, partial pivoting.

    python tools/lu_host_time.py [--n 2048] [--reps 4]
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2048)
    ap.add_argument("--bits", type=int, default=256)
    ap.add_argument("--reps", type=int, default=4)
    a = ap.parse_args()
    import torch
    import paper_1410_1599_b200 as P
    ctx = P.PrecisionContext(a.bits)
    A = P.gen_uniform_full(a.n, a.n, 11, ctx)

    def pinned(x):
        lim = torch.empty(x.limbs.shape, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
        ex = torch.empty(x.exp.shape, dtype=torch.int32, pin_memory=True).numpy()
        sg = torch.empty(x.sign.shape, dtype=torch.uint8, pin_memory=True).numpy()
        lim[:], ex[:], sg[:] = x.limbs, x.exp, x.sign
        return P.Matrix(x.rows(), x.cols(), x.ctx(), lim, ex, sg)

    src, work = pinned(A), pinned(A)
    cfg = P.BlockLUConfig(64, P.Algorithm.winograd, 32)
    for r in range(a.reps):
        work.limbs[:], work.exp[:], work.sign[:] = src.limbs, src.exp, src.sign
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        P.lu_blocked_host(work, cfg, ctx, pivoting=True, out=work)
        t1 = time.perf_counter()
        print(f"rep {r}: lu_blocked_host wall {1e3 * (t1 - t0):.2f} ms", flush=True)
    for r in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f = P.lu_blocked(src, cfg, ctx, pivoting=True)
        print(f"rep {r}: lu_blocked (upload, factor, download) wall {1e3 * (time.perf_counter() - t0):.2f} ms",
              flush=True)


if __name__ == "__main__":
    main()
