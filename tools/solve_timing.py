import sys, time
sys.path.insert(0, '.')
import paper_1410_1599_b200 as P
import torch
ctx = P.PrecisionContext(256)
n = 2048
a = P.gen_uniform_full(n, n, 11, ctx)
f = P.lu_blocked(a, P.BlockLUConfig(64, P.Algorithm.winograd, 32), ctx, pivoting=True)
ones = P.gen_uniform_full(n, 1, 5, ctx)
for ex in (True, True, False):
    t0 = time.perf_counter(); x = P.lu_solve(f, ones, ctx, exact=ex); torch.cuda.synchronize()
    print("exact" if ex else "fast", round((time.perf_counter() - t0) * 1e3, 1), "ms")
