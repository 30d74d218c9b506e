"""Phase timeline of the pipelined host GEMM (MPGPU_PIPE_TRACE=1) at cfg2 and the wall
time of mpgpu_gemm_host with pinned buffers.

    MPGPU_PIPE_TRACE=1 python tools/pipe_trace.py [--n 1024] [--bits 256] [--n-min 64]
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--bits", type=int, default=256)
    ap.add_argument("--n-min", type=int, default=64)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import torch
    import paper_1410_1599_b200 as P
    ctx = P.PrecisionContext(a.bits)

    def pinned(x):
        lim = torch.empty(x.limbs.shape, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
        ex = torch.empty(x.exp.shape, dtype=torch.int32, pin_memory=True).numpy()
        sg = torch.empty(x.sign.shape, dtype=torch.uint8, pin_memory=True).numpy()
        lim[:] = x.limbs
        ex[:] = x.exp
        sg[:] = x.sign
        return P.Matrix(x.rows(), x.cols(), x.ctx(), lim, ex, sg)

    A = pinned(P.gen_uniform_full(a.n, a.n, 1, ctx))
    B = pinned(P.gen_uniform_full(a.n, a.n, 2, ctx))
    C = pinned(P.Matrix(a.n, a.n, ctx))
    for r in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        P.gemm_host(P.Algorithm.winograd, a.n_min, A, B, C, ctx)
        print(f"rep {r}: gemm_host wall {1e3 * (time.perf_counter() - t0):.3f} ms", file=sys.stderr, flush=True)


if __name__ == "__main__":
    main()
