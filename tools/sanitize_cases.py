"""Small cases for compute-sanitizer runs (memcheck / racecheck / synccheck): the leaf
GEMM (bulk-copy and edge tiles, Block fold, ragged half-width tiles), the fast algorithms,
the pivoted LU + both solves, and the wide (warp-per-value) kernels.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py

(compute-sanitizer is closed on this round's GPU pool; the same cases run plain as a quick
smoke of every kernel family.)"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import paper_1410_1599_b200 as P
    for bits in (256, 512):
        ctx = P.PrecisionContext(bits)
        a, b = P.gen_uniform_full(48, 40, 1, ctx), P.gen_uniform_full(40, 37, 2, ctx)
        P.simple_mul(a, b, ctx)
        P.block_mul(a, b, 8, ctx)
        P.fast_mul(a, b, P.FastMMConfig(P.Algorithm.winograd, 8), ctx)
        P.fast_mul(P.gen_scaled(32, 25, 3, ctx), P.gen_scaled(25, 49, 4, ctx),
                   P.FastMMConfig(P.Algorithm.strassen, 16), ctx)
        m = P.gen_uniform_full(40, 40, 5, ctx)
        x = P.gen_uniform_full(40, 1, 6, ctx)
        rhs = P.mat_vec_mul(m, x, ctx)
        f = P.lu_blocked(m, P.BlockLUConfig(8, P.Algorithm.winograd, 4), ctx, pivoting=True)
        P.lu_solve(f, rhs, ctx, exact=True)
        P.lu_solve(f, rhs, ctx, exact=False)
    for bits in (2048, 8192):
        ctx = P.PrecisionContext(bits)
        a, b = P.gen_uniform_full(9, 7, 1, ctx), P.gen_uniform_full(7, 11, 2, ctx)
        P.fast_mul(a, b, P.FastMMConfig(P.Algorithm.winograd, 2), ctx)
        P.block_mul(a, b, 3, ctx)
        m = P.gen_uniform_full(12, 12, 5, ctx)
        x = P.gen_uniform_full(12, 1, 6, ctx)
        rhs = P.mat_vec_mul(m, x, ctx)
        f = P.lu_blocked(m, P.BlockLUConfig(4, P.Algorithm.winograd, 2), ctx, pivoting=True)
        P.lu_solve(f, rhs, ctx, exact=True)
        P.vec_op(3, a, P.gen_uniform_full(9, 7, 3, ctx))
    print("sanitize cases done")


if __name__ == "__main__":
    main()
