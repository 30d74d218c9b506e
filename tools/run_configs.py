"""Run every BASELINE.json config on one B200, time it, and check it.

    python tools/run_configs.py [--only 1,2,3,4,5] [--quick]

Checks (oracle = oracle/_ref or the C restatement, CPU):
  cfg1  n=128 @128: all four algorithms bit-exact vs the oracle, on full-mantissa and
        on the reference's own gen_random inputs
  cfg2  n=1024 @256: Block / Strassen / Winograd; sampled rows of Block bit-exact vs
        the oracle; Strassen / Winograd vs Block within the normwise bound
  cfg3  1001x777x1537 @512 (scaled inputs), Winograd n_min 32 / 64: sampled rows vs
        an oracle product at 2p+64 bits within the normwise bound
  cfg4  n=4096 @1024, Winograd n_min 512 (depth 3) and Block 512: sampled row of
        Block bit-exact vs the oracle; Winograd vs Block within the bound
  cfg5  LU n=2048 @256 with partial pivoting, inputs (a) uniform and (b) L*D*U:
        backward error ||PA - LU||_max / ||A||_max and the solve of A x = A*1
Prints one JSON line per measurement.
"""
from __future__ import annotations

import argparse
import json
import math
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_1410_1599_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402


def emit(**kw):
    print(json.dumps(kw), flush=True)


def timed(fn, reps=1):
    import torch
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return out, best


def rows_of(x, rows):
    cols = x.cols()
    idx = (np.asarray(rows)[:, None] * cols + np.arange(cols)[None, :]).reshape(-1)
    return P.Matrix(len(rows), cols, x.ctx(), x.limbs[:, idx], x.exp[idx], x.sign[idx])


def log2_norm_err(c, ref, a, b):
    """log2( max|C - ref| / (max|A| * max|B|) )"""
    d = O.log2_max_abs_diff(O.OMat.of(c), O.OMat.of(ref))
    return d - O.log2_max_abs(O.OMat.of(a)) - O.log2_max_abs(O.OMat.of(b))


def bound_log2(n, p, c=4.0):
    # north star: ||C_gpu - C_ref|| / (||A|| ||B||) <= c * n^{log2 7} * 2^-p
    return math.log2(c) + math.log2(7) * math.log2(n) - p


def gemm_dev(algo, param, da, db, ctx, m, n):
    dc = P.DeviceMatrix(m, n, ctx)
    st = P.gemm_into(algo, param, da, db, dc)
    return dc, st


def cfg1():
    ctx = P.PrecisionContext(128)
    for gname, gen in (("uniform_full", P.gen_uniform_full), ("ref_gen_random", P.gen_random)):
        a, b = gen(128, 128, 1, ctx), gen(128, 128, 2, ctx)
        da, db = a.to_device(), b.to_device()
        for algo, param in (("simple", 0), ("block", 32), ("strassen", 32), ("winograd", 32)):
            (dc, st), dt = timed(lambda: gemm_dev(P.Algorithm[algo], param, da, db, ctx, 128, 128), reps=3)
            c = dc.download()
            want, _ = O.gemm(algo, param, O.OMat.of(a), O.OMat.of(b))
            emit(cfg=1, inputs=gname, algo=algo, n=128, bits=128, ms=st.device_ms, wall_ms=dt * 1e3,
                 madd_per_s=128 ** 3 / (st.device_ms * 1e-3), bit_exact=bool(P.identical(c, want)))


def cfg2():
    n, bits = 1024, 256
    ctx = P.PrecisionContext(bits)
    a, b = P.gen_uniform_full(n, n, 1, ctx), P.gen_uniform_full(n, n, 2, ctx)
    da, db = a.to_device(), b.to_device()
    res = {}
    for algo in ("block", "strassen", "winograd"):
        (dc, st), _ = timed(lambda: gemm_dev(P.Algorithm[algo], 64, da, db, ctx, n, n))
        (dc, st), _ = timed(lambda: gemm_dev(P.Algorithm[algo], 64, da, db, ctx, n, n))
        res[algo] = dc.download()
        emit(cfg=2, algo=algo, n=n, bits=bits, n_min=64, ms=st.device_ms, leaf_ms=st.leaf_ms,
             madd_per_s=n ** 3 / (st.device_ms * 1e-3))
    rows = [0, 511, 1023]
    sub = rows_of(a, rows)
    want, _ = O.gemm("block", 64, O.OMat.of(sub), O.OMat.of(b))
    emit(cfg=2, check="block sampled rows vs oracle", rows=rows, bit_exact=bool(P.identical(rows_of(res["block"], rows), want)))
    for algo in ("strassen", "winograd"):
        e = log2_norm_err(res[algo], res["block"], a, b)
        emit(cfg=2, check=f"{algo} vs block normwise", log2_err=e, log2_bound=bound_log2(n, bits),
             ok=bool(e <= bound_log2(n, bits)))


def cfg3():
    m, l, n, bits = 1001, 777, 1537, 512
    ctx = P.PrecisionContext(bits)
    a, b = P.gen_scaled(m, l, 3, ctx), P.gen_scaled(l, n, 4, ctx)
    da, db = a.to_device(), b.to_device()
    rows = [0, 500, 1000]
    hi = 2 * bits + 64
    # oracle rows at 2p+64 bits: inputs are exact at hi precision (same values)
    sa, sb = rows_of(a, rows), b
    oa = O.OMat(len(rows), l, hi, np.vstack([np.zeros((34 - sa.nlimbs, sa.limbs.shape[1]), np.uint32), sa.limbs]),
                sa.exp, sa.sign)
    ob = O.OMat(l, n, hi, np.vstack([np.zeros((34 - sb.nlimbs, sb.limbs.shape[1]), np.uint32), sb.limbs]),
                sb.exp, sb.sign)
    exact_rows, _ = O.gemm("simple", 0, oa, ob)
    for n_min in (32, 64):
        (dc, st), _ = timed(lambda: gemm_dev(P.Algorithm.winograd, n_min, da, db, ctx, m, n))
        (dc, st), _ = timed(lambda: gemm_dev(P.Algorithm.winograd, n_min, da, db, ctx, m, n))
        c = dc.download()
        cr = rows_of(c, rows)
        # compare at hi precision: widen C's rows
        cw = O.OMat(len(rows), n, hi, np.vstack([np.zeros((34 - cr.nlimbs, cr.limbs.shape[1]), np.uint32), cr.limbs]),
                    cr.exp, cr.sign)
        d = O.log2_max_abs_diff(cw, exact_rows) - O.log2_max_abs(O.OMat.of(a)) - O.log2_max_abs(O.OMat.of(b))
        emit(cfg=3, algo="winograd", m=m, l=l, n=n, bits=bits, n_min=n_min, depth=st.depth, ms=st.device_ms,
             leaf_ms=st.leaf_ms, madd_per_s=m * l * n / (st.device_ms * 1e-3), leaf_madds=st.leaf_madds,
             log2_err_vs_exact_rows=d, log2_bound=bound_log2(max(m, l, n), bits), ok=bool(d <= bound_log2(max(m, l, n), bits)))


def cfg4(quick=False):
    n, bits = (2048, 1024) if quick else (4096, 1024)
    nmin = n // 8
    ctx = P.PrecisionContext(bits)
    a, b = P.gen_uniform_full(n, n, 1, ctx), P.gen_uniform_full(n, n, 2, ctx)
    da, db = a.to_device(), b.to_device()
    (dw, st), _ = timed(lambda: gemm_dev(P.Algorithm.winograd, nmin, da, db, ctx, n, n))
    emit(cfg=4, algo="winograd", n=n, bits=bits, n_min=nmin, depth=st.depth, ms=st.device_ms, leaf_ms=st.leaf_ms,
         preadd_ms=st.preadd_ms, postadd_ms=st.postadd_ms, madd_per_s=n ** 3 / (st.device_ms * 1e-3))
    cw = dw.download()
    dw.free()
    (dbk, st2), _ = timed(lambda: gemm_dev(P.Algorithm.block, nmin, da, db, ctx, n, n))
    emit(cfg=4, algo="block", n=n, bits=bits, n_min=nmin, ms=st2.device_ms, madd_per_s=n ** 3 / (st2.device_ms * 1e-3))
    cb = dbk.download()
    rows = [n - 1]
    want, _ = O.gemm("block", nmin, O.OMat.of(rows_of(a, rows)), O.OMat.of(b))
    emit(cfg=4, check="block sampled row vs oracle", rows=rows, bit_exact=bool(P.identical(rows_of(cb, rows), want)))
    e = log2_norm_err(cw, cb, a, b)
    emit(cfg=4, check="winograd vs block normwise", log2_err=e, log2_bound=bound_log2(n, bits), ok=bool(e <= bound_log2(n, bits)))


def ldu(n, ctx, seed):
    """A = RN(L * RN(D * U)): unit-triangular L, U with off-diagonals uniform [-1,1)
    (full mantissa), D_ii = 2^-round(199.32 i/(n-1)) (geometric 1 -> ~1e-60, exact
    powers of two so D*U is exact).  Built with the GPU Simple GEMM."""
    Lm = P.gen_uniform_full(n, n, seed, ctx)
    Um = P.gen_uniform_full(n, n, seed + 1, ctx)
    one = P.from_ints([1], ctx)
    E = np.arange(n * n).reshape(n, n)
    r, c = np.divmod(E, n)
    for M, keep in ((Lm, r > c), (Um, r < c)):
        flat = keep.reshape(-1)
        M.limbs[:, ~flat] = 0
        M.exp[~flat] = P.EXP_ZERO
        M.sign[~flat] = 0
        diag = (r == c).reshape(-1)
        M.limbs[:, diag] = one.limbs[:, :1]
        M.exp[diag] = one.exp[0]
        M.sign[diag] = 0
    # D * U: row i scaled by 2^-k_i (exact exponent shift)
    k = np.round(60 * math.log2(10) * np.arange(n) / (n - 1)).astype(np.int64)
    nz = Um.exp != P.EXP_ZERO
    Um.exp[nz] = (Um.exp.reshape(n, n) - k[:, None]).reshape(-1)[nz]
    return P.simple_mul(Lm, Um, ctx)


def cfg5(quick=False):
    n, bits = (512, 256) if quick else (2048, 256)
    ctx = P.PrecisionContext(bits)
    ones = P.from_ints(np.ones(n, np.int64), ctx)
    for inp in ("a_uniform", "b_LDU"):
        A = P.gen_uniform_full(n, n, 11, ctx) if inp == "a_uniform" else ldu(n, ctx, 21)
        bvec = P.mat_vec_mul(A, ones, ctx)
        for kernel, alpha in (("block", 1), ("block", 2), ("winograd", 2), ("winograd", 4), ("winograd", 8)):
            cfg = P.BlockLUConfig.with_alpha(alpha, 32, P.Algorithm[kernel])
            st = P.Stats()
            (f), dt = timed(lambda: P.lu_blocked(A, cfg, ctx, pivoting=True, stats=st))
            x, dts = timed(lambda: P.lu_solve(f, bvec, ctx, exact=False))
            # backward error of the factorisation: PA - L U with the GPU GEMM at p bits
            F = f.packed
            Lm, Um = F.copy(), F.copy()
            E = np.arange(n * n)
            r, c = np.divmod(E, n)
            for M, keep in ((Lm, r > c), (Um, r <= c)):
                M.limbs[:, ~keep] = 0
                M.exp[~keep] = P.EXP_ZERO
                M.sign[~keep] = 0
            diag = r == c
            Lm.limbs[:, diag] = ones.limbs[:, :1]
            Lm.exp[diag] = ones.exp[0]
            LU = P.simple_mul(Lm, Um, ctx)
            PA = A.copy().to_float()  # only for the permutation bookkeeping below
            perm = np.arange(n)
            for d in range(n):
                perm[[d, f.piv[d]]] = perm[[f.piv[d], d]]
            idx = (perm[:, None] * n + np.arange(n)[None, :]).reshape(-1)
            PAm = P.Matrix(n, n, ctx, A.limbs[:, idx], A.exp[idx], A.sign[idx])
            berr = O.log2_max_abs_diff(O.OMat.of(PAm), O.OMat.of(LU)) - O.log2_max_abs(O.OMat.of(A))
            xf = x.to_float().reshape(-1)
            extra = {}
            if kernel == "winograd" and alpha == 2:  # the reference's exact s-ascending replay
                xe, dte = timed(lambda: P.lu_solve(f, bvec, ctx, exact=True))
                extra = dict(exact_solve_wall_ms=dte * 1e3,
                             exact_vs_column_solve_max_abs_diff=float(np.max(np.abs(xe.to_float().reshape(-1) - xf))))
            emit(cfg=5, input=inp, n=n, bits=bits, kernel=kernel, alpha=alpha, K=cfg.block_size,
                 lu_ms=st.device_ms, lu_wall_ms=dt * 1e3, solve_wall_ms=dts * 1e3, solve="column-oriented",
                 schur_madds=st.mul, log2_backward_err=berr, log2_bound=math.log2(n) - bits + 8,
                 max_abs_x_minus_1=float(np.max(np.abs(xf - 1.0))), **extra)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="1,2,3,4,5")
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    want = {int(x) for x in args.only.split(",")}
    if 1 in want:
        cfg1()
    if 2 in want:
        cfg2()
    if 3 in want:
        cfg3()
    if 4 in want:
        cfg4(args.quick)
    if 5 in want:
        cfg5(args.quick)


if __name__ == "__main__":
    main()
