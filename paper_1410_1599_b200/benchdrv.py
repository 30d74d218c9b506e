"""The reference's benchmark drivers on the GPU path (bench.hpp:21-249; SURVEY.md §8f
rank 1): the same requests, the same 15-column CSV rows.

  run_matmul  bench.hpp:117-165 -- benchmark pair (matgen.hpp:63-78), each selected
              algorithm timed around the multiply call (host matrices in and out, as
              the reference's call), error against the closed-form product at
              bits * ref_bits_multiplier (matgen.hpp:84-105) on the device
  run_lu      bench.hpp:187-249 -- random or Lotkin system with x_true = 0..n-1, the
              column-wise solve, then lu_blocked + lu_solve per alpha; SINGULAR rows

Everything but wall_seconds is identical to the reference's row for the same request
(tests/test_gpu_benchdrv.py compares them with the compiled reference's own
run_matmul / run_lu).  The closed-form inputs are exact host integer arithmetic
(exact.py): one value per distinct entry; products, factorisations, solves and
error metrics run on the GPU.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import IO, List, Optional

import numpy as np

from . import exact
from .mpmm import (Algorithm, BlockLUConfig, DomainError, Matrix, OpCounter, PrecisionContext, SingularError,
                   algorithm_name, block_mul, count_simple, fast_mul, FastMMConfig, lu_blocked, lu_solve,
                   mat_vec_mul, max_rel_error, max_rel_error_solution, simple_mul, solve_columnwise)
from .matgen import from_ints, gen_random

CSV_HEADER = ("command,algorithm,m,l,n,bits,n_min,K,alpha,seed,wall_seconds,max_rel_error,min_rel_error,"
              "mul_count,addsub_count")


@dataclass
class BenchRecord:
    """bench.hpp:27-64: every column always emitted, inapplicable fields empty."""
    command: str = ""
    algorithm: str = ""
    m: Optional[int] = None
    l: Optional[int] = None
    n: Optional[int] = None
    bits: Optional[int] = None
    n_min: Optional[int] = None
    k: Optional[int] = None
    alpha: Optional[int] = None
    seed: Optional[int] = None
    wall_seconds: Optional[float] = None
    max_rel_error: str = ""
    min_rel_error: str = ""
    mul_count: Optional[int] = None
    addsub_count: Optional[int] = None

    def to_csv_row(self) -> str:
        def put(v):
            return "" if v is None else str(int(v))
        cols = [self.command, self.algorithm, put(self.m), put(self.l), put(self.n), put(self.bits),
                put(self.n_min), put(self.k), put(self.alpha), put(self.seed),
                "" if self.wall_seconds is None else f"{self.wall_seconds:.3f}",
                self.max_rel_error, self.min_rel_error, put(self.mul_count), put(self.addsub_count)]
        return ",".join(cols)


def print_csv(out: IO[str], rows: List[BenchRecord]) -> None:
    """bench.hpp:79-82"""
    out.write(CSV_HEADER + "\n")
    for r in rows:
        out.write(r.to_csv_row() + "\n")


def append_csv(path: str, rows: List[BenchRecord]) -> None:
    """bench.hpp:68-77: header only when the file is new or empty."""
    import os
    need_header = (not os.path.exists(path)) or os.path.getsize(path) == 0
    try:
        with open(path, "a") as f:
            if need_header:
                f.write(CSV_HEADER + "\n")
            for r in rows:
                f.write(r.to_csv_row() + "\n")
    except OSError as e:
        raise IOError(f"cannot open CSV file for append: {path}") from e


def _warm(fn) -> None:
    """Untimed warm-up of a GPU row on a small problem of the same precision and
    configuration: CUDA loads kernels lazily on first launch and the stream-ordered pool
    grows on first use -- one-time costs the reference's CPU rows do not have."""
    try:
        fn()
    except SingularError:
        pass


def _time_seconds(fn) -> float:
    """bench.hpp:87-94: monotonic wall time rounded to milliseconds."""
    t0 = time.perf_counter()
    fn()
    return round((time.perf_counter() - t0) * 1000.0) / 1000.0


def error_digits(bits: int, verbose: bool) -> int:
    """bench.hpp:96-99"""
    if not verbose:
        return 3
    return int(math.ceil(bits * 0.30102999566398120)) + 2


# ---------------------------------------------------------------------------
# closed-form generators (matgen.hpp:63-140), exact
# ---------------------------------------------------------------------------


def gen_bench_pair(m: int, l: int, n: int, ctx: PrecisionContext):
    """matgen.hpp:63-78: a_ij = RN(RN(sqrt 5) * (i+j+1)), b_ij = RN(RN(sqrt 3) * (l-i))."""
    p = ctx.bits()
    r5 = exact.rn_sqrt_int(5, p)
    r3 = exact.rn_sqrt_int(3, p)
    va = [exact.mul_int(r5, c, p, p) for c in range(0, m + l)]  # index i+j+1 in 1..m+l-1
    ia = (np.arange(m)[:, None] + np.arange(l)[None, :] + 1).reshape(-1)
    a = exact.values_to_matrix(va, ia, m, l, ctx)
    vb = [exact.mul_int(r3, l - i, p, p) for i in range(l)]
    ib = np.repeat(np.arange(l), n)
    b = exact.values_to_matrix(vb, ib, l, n, ctx)
    return a, b


def bench_entry_sum(i1: int, l: int) -> int:
    """sum_{k=1..l} (i+k-1)(l-k+1) for 1-based i (matgen.hpp:84-94), closed form."""
    s1 = l * (l - 1) // 2
    s2 = (l - 1) * l * (2 * l - 1) // 6
    return i1 * l * l + (l - i1) * s1 - s2


def bench_reference(m: int, l: int, n: int, ctx: PrecisionContext) -> Matrix:
    """matgen.hpp:84-105: c_ij = RN(RN(sqrt 15) * s_i) at ctx, constant along rows."""
    p = ctx.bits()
    r15 = exact.rn_sqrt_int(15, p)
    vals = [exact.mul_int(r15, bench_entry_sum(i + 1, l), p, p) for i in range(m)]
    return exact.values_to_matrix(vals, np.repeat(np.arange(m), n), m, n, ctx)


def gen_lotkin(n: int, ctx: PrecisionContext) -> Matrix:
    """matgen.hpp:107-121: first row ones, a_ij = RN(1/(i+j+1)) below."""
    p = ctx.bits()
    vals = [exact.rn_int(1, p)] + [exact.rn_fraction(1, q, p) for q in range(1, 2 * n)]
    idx = np.arange(n)[:, None] + np.arange(n)[None, :] + 1
    idx[0, :] = 0
    return exact.values_to_matrix(vals, idx.reshape(-1), n, n, ctx)


def gen_linear_system(a: Matrix, ctx: PrecisionContext):
    """matgen.hpp:131-141: x_true = RN(0..n-1), b = mat_vec_mul(a, x_true) (device)."""
    x = from_ints(np.arange(a.cols(), dtype=np.int64), ctx, a.cols(), 1)
    b = mat_vec_mul(a, x, ctx)
    return x, b


# ---------------------------------------------------------------------------
# drivers
# ---------------------------------------------------------------------------


@dataclass
class MatmulRequest:
    """bench.hpp:103-111"""
    algos: List[Algorithm] = field(default_factory=lambda: [Algorithm.simple, Algorithm.block,
                                                            Algorithm.strassen, Algorithm.winograd])
    m: int = 256
    l: int = 256
    n: int = 256
    bits: int = 128
    n_min: int = 32
    ref_bits_multiplier: int = 2
    verbose: bool = False


def run_matmul(q: MatmulRequest) -> List[BenchRecord]:
    """bench.hpp:117-165"""
    if q.ref_bits_multiplier < 1:
        raise DomainError("ref bits multiplier must be >= 1")
    ctx = PrecisionContext(q.bits)
    ref_ctx = PrecisionContext(min(q.bits * q.ref_bits_multiplier, PrecisionContext.max_bits))
    a, b = gen_bench_pair(q.m, q.l, q.n, ctx)
    ref = bench_reference(q.m, q.l, q.n, ref_ctx).to_device()
    digits = error_digits(q.bits, q.verbose)
    rows = []
    try:
        for algo in q.algos:
            out = {}
            ops = OpCounter()

            def call():
                if algo == Algorithm.simple:
                    out["c"] = simple_mul(a, b, ctx)
                elif algo == Algorithm.block:
                    out["c"] = block_mul(a, b, q.n_min, ctx)
                else:
                    r = fast_mul(a, b, FastMMConfig(algo, q.n_min), ctx)
                    out["c"] = r.c
                    out["ops"] = r.ops

            sa, sb = a.sub(0, 0, min(q.m, 2 * q.n_min + 2), min(q.l, 2 * q.n_min + 2)), \
                b.sub(0, 0, min(q.l, 2 * q.n_min + 2), min(q.n, 2 * q.n_min + 2))
            _warm(lambda: (simple_mul(sa, sb, ctx) if algo == Algorithm.simple else
                           block_mul(sa, sb, q.n_min, ctx) if algo == Algorithm.block else
                           fast_mul(sa, sb, FastMMConfig(algo, q.n_min), ctx)))
            secs = _time_seconds(call)
            ops = out.get("ops") or ops
            if algo in (Algorithm.simple, Algorithm.block):
                ops = count_simple(q.m, q.l, q.n)
            err = max_rel_error(out["c"], ref)
            rows.append(BenchRecord(
                command="matmul", algorithm=algorithm_name(algo), m=q.m, l=q.l, n=q.n, bits=q.bits,
                n_min=q.n_min, wall_seconds=secs,
                max_rel_error=exact.matrix_scalar_decimal(err.max, 0, digits),
                min_rel_error=exact.matrix_scalar_decimal(err.min, 0, digits),
                mul_count=ops.mul, addsub_count=ops.addsub))
    finally:
        ref.free()
    return rows


@dataclass
class LURequest:
    """bench.hpp:167-176"""
    matrix_kind: str = "random"
    n: int = 128
    bits: int = 256
    kernel: Algorithm = Algorithm.winograd
    n_min: int = 32
    alpha_lo: int = 1
    alpha_hi: int = 10
    seed: int = 1
    verbose: bool = False


@dataclass
class LUOutcome:
    rows: List[BenchRecord]
    any_singular: bool = False


def run_lu(q: LURequest) -> LUOutcome:
    """bench.hpp:187-249"""
    if q.matrix_kind not in ("random", "lotkin"):
        raise DomainError(f"unknown matrix kind '{q.matrix_kind}'")
    if q.alpha_lo < 1 or q.alpha_hi < q.alpha_lo:
        raise DomainError("bad alpha range")
    ctx = PrecisionContext(q.bits)
    a = gen_random(q.n, q.n, q.seed, ctx) if q.matrix_kind == "random" else gen_lotkin(q.n, ctx)
    x_true, b = gen_linear_system(a, ctx)
    digits = error_digits(q.bits, q.verbose)
    out = LUOutcome([])

    def base(name):
        return BenchRecord(command="lu", algorithm=name, m=q.n, l=q.n, n=q.n, bits=q.bits, n_min=q.n_min,
                           seed=q.seed if q.matrix_kind == "random" else None)

    nw = min(q.n, 2 * q.n_min * max(q.alpha_hi, 1) + 2)  # warm-up size
    aw = a.sub(0, 0, nw, nw)
    bw = b.sub(0, 0, nw, 1)
    rec = base("columnwise")
    try:
        res = {}
        _warm(lambda: solve_columnwise(aw, bw))
        rec.wall_seconds = _time_seconds(lambda: res.__setitem__("x", solve_columnwise(a, b)))
        err = max_rel_error_solution(res["x"], x_true)
        rec.max_rel_error = exact.matrix_scalar_decimal(err.max_rel, 0, digits)
    except SingularError:
        rec.max_rel_error = "SINGULAR"
        out.any_singular = True
    out.rows.append(rec)

    for alpha in range(q.alpha_lo, q.alpha_hi + 1):
        cfg = BlockLUConfig.with_alpha(alpha, q.n_min, q.kernel)
        rec = base(algorithm_name(q.kernel))
        rec.k = cfg.block_size
        rec.alpha = alpha
        try:
            schur = OpCounter()
            res = {}

            def call():
                f = lu_blocked(a, cfg, ctx, schur)
                res["x"] = lu_solve(f, b, ctx)

            _warm(lambda: lu_solve(lu_blocked(aw, cfg, ctx), bw, ctx))
            rec.wall_seconds = _time_seconds(call)
            err = max_rel_error_solution(res["x"], x_true)
            rec.max_rel_error = exact.matrix_scalar_decimal(err.max_rel, 0, digits)
            rec.mul_count = schur.mul
            rec.addsub_count = schur.addsub
        except SingularError:
            rec.max_rel_error = "SINGULAR"
            out.any_singular = True
        out.rows.append(rec)
    return out


# ---------------------------------------------------------------------------
# analytic operation-count ratios (opmodel.hpp:46-155; CLI `opcount`)
# ---------------------------------------------------------------------------


def _fixed3(num: int, den: int) -> str:
    """Ratio::fixed3 (opmodel.hpp:59-67): 3 fractional digits, half away from zero."""
    q = (num * 2000 + den) // (den * 2)
    return f"{q // 1000}.{q % 1000:03d}"


def ratio_table(sizes, n_min: int):
    """opmodel.hpp:81-106: per size (m, l, n) the Strassen / Winograd mul and addsub
    counts relative to Simple, as reduced fractions."""
    from math import gcd
    from .mpmm import DimensionError, count_fast
    if not sizes:
        raise DimensionError("ratio_table: empty size list")
    rows = []
    for (m, l, n) in sizes:
        s = count_simple(m, l, n)
        st = count_fast(Algorithm.strassen, m, l, n, n_min)
        wi = count_fast(Algorithm.winograd, m, l, n, n_min)

        def ratio(a, b):
            if b == 0:
                if a == 0:
                    return (1, 1)
                raise DomainError("addsub ratio undefined: simple algorithm performs no additions")
            g = gcd(a, b)
            return (a // g, b // g)
        rows.append(((m, l, n), n_min, ratio(st.mul, s.mul), ratio(st.addsub, s.addsub), ratio(wi.mul, s.mul),
                     ratio(wi.addsub, s.addsub)))
    return rows


def format_ratio_csv(rows) -> str:
    """opmodel.hpp:143-155"""
    out = ["m,l,n,n_min,strassen_mul_ratio,strassen_addsub_ratio,winograd_mul_ratio,winograd_addsub_ratio"]
    for (m, l, n), nm, sm, sa, wm, wa in rows:
        out.append(f"{m},{l},{n},{nm},{_fixed3(*sm)},{_fixed3(*sa)},{_fixed3(*wm)},{_fixed3(*wa)}")
    return "\n".join(out) + "\n"


def format_ratio_table(rows) -> str:
    """opmodel.hpp:123-141 (fixed-width text table)."""
    lw, cw = 18, 10
    nm = rows[0][1] if rows else 0
    lines = [" " * lw + " |" + "Strassen".rjust(2 * cw) + " |" + "Winograd".rjust(2 * cw),
             f"n_min = {nm}".ljust(lw) + " |" + "Add & Sub".rjust(cw) + "Mul".rjust(cw) + " |" +
             "Add & Sub".rjust(cw) + "Mul".rjust(cw),
             "-" * lw + "-+" + "-" * (2 * cw) + "-+" + "-" * (2 * cw)]
    for (m, l, n), _, sm, sa, wm, wa in rows:
        label = f"{m} x {n}" if m == l == n else f"{m} x {l} x {n}"
        lines.append(label.rjust(lw) + " |" + _fixed3(*sa).rjust(cw) + _fixed3(*sm).rjust(cw) + " |" +
                     _fixed3(*wa).rjust(cw) + _fixed3(*wm).rjust(cw))
    return "\n".join(lines) + "\n"


def parse_sizes(tokens) -> list:
    """mpmm_bench.cpp:23-45: integers N (an N x N x N product) and ranges a..b expanding to
    2^k-1, 2^k, 2^k+1 within [a, b]; sorted, unique."""
    sizes = set()
    for tok in tokens:
        if ".." in tok:
            lo, hi = (int(x) for x in tok.split("..", 1))
            if lo == 0 or hi < lo:
                raise DomainError(f"bad size range '{tok}'")
            k = 1
            while (1 << k) <= hi + 1:
                for dd in (-1, 0, 1):
                    v = (1 << k) + dd
                    if lo <= v <= hi:
                        sizes.add(v)
                k += 1
        else:
            sizes.add(int(tok))
    if not sizes:
        raise DomainError("no sizes given")
    return [(s, s, s) for s in sorted(sizes)]
