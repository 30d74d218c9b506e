"""ctypes front-end of the CPU checkers.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this module.  Two checkers:

  orc  -- oracle/_build/libmp_oracle.so: the C restatement (mp_oracle.c) of the
          reference's loops over system MPFR (each function cites the reference);
  ref  -- oracle/_ref/libmpmm_ref.so: the UNMODIFIED reference headers compiled
          from /root/reference by oracle/Makefile (ref_bridge.cpp).

Matrices cross as SoA arrays (include/mpgpu.h); `OMat` mirrors the attributes of
paper_1410_1599_b200.Matrix so the package's comparators accept both.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORC_PATH = HERE / "_build" / "libmp_oracle.so"
REF_PATH = HERE / "_ref" / "libmpmm_ref.so"
EXP_ZERO = -(1 << 31)


def build() -> None:
    """Compile the checkers (make -f oracle/Makefile); the reference bridge only
    when /root/reference is present (the GPU box uses the prebuilt files)."""
    subprocess.run(["make", "-s", "-f", str(HERE / "Makefile")], check=True, capture_output=True)


class OMat:
    def __init__(self, rows, cols, bits, limbs=None, exp=None, sign=None, nlimbs=None):
        self._rows, self._cols, self._bits = int(rows), int(cols), int(bits)
        n = self._rows * self._cols
        L = nlimbs or max(1, (self._bits + 31) // 32)
        self.limbs = np.zeros((L, n), np.uint32) if limbs is None else np.ascontiguousarray(limbs, np.uint32).reshape(-1, n)
        self.exp = np.full(n, EXP_ZERO, np.int32) if exp is None else np.ascontiguousarray(exp, np.int32).reshape(n)
        self.sign = np.zeros(n, np.uint8) if sign is None else np.ascontiguousarray(sign, np.uint8).reshape(n)

    def rows(self):
        return self._rows

    def cols(self):
        return self._cols

    def bits(self):
        return self._bits

    @property
    def nlimbs(self):
        return self.limbs.shape[0]

    @staticmethod
    def of(x) -> "OMat":
        return OMat(x.rows(), x.cols(), x.bits(), x.limbs, x.exp, x.sign)


def _p(a):
    return C.c_void_p(a.ctypes.data)


def _soa(x):
    return _p(x.limbs), _p(x.exp), _p(x.sign)


_orc = None
_ref = None


def orc():
    global _orc
    if _orc is None:
        if not ORC_PATH.exists():
            build()
        _orc = C.CDLL(str(ORC_PATH))
        _orc.orc_log2_max_abs_diff.restype = C.c_double
        _orc.orc_log2_max_abs.restype = C.c_double
    return _orc


def have_ref() -> bool:
    return REF_PATH.exists()


def ref():
    global _ref
    if _ref is None:
        if not REF_PATH.exists():
            build()
        _ref = C.CDLL(str(REF_PATH))
    return _ref


class OracleError(RuntimeError):
    def __init__(self, rc, pivot=0):
        super().__init__(f"oracle rc={rc} pivot={pivot}")
        self.rc, self.pivot = rc, pivot


def _check(rc, pivot=0):
    if rc:
        raise OracleError(rc, pivot)


ALGOS = {"simple": 0, "block": 1, "strassen": 2, "winograd": 3}


def _algo(a):
    return ALGOS[a] if isinstance(a, str) else int(a)


# ---- products ---------------------------------------------------------------

def gemm(algo, param, a, b, bits=None, which="orc", threads=0):
    """C = A*B by the restatement ("orc") or the compiled reference ("ref").
    Returns (OMat C, (mul, addsub))."""
    bits = bits or a.bits()
    L = a.nlimbs
    m, l, n = a.rows(), a.cols(), b.cols()
    c = OMat(m, n, bits, nlimbs=L)
    ops = (C.c_uint64 * 2)()
    if which == "orc":
        rc = orc().orc_gemm(_algo(algo), C.c_int64(param), C.c_long(bits), L, C.c_int64(m), C.c_int64(l),
                            C.c_int64(n), *_soa(a), *_soa(b), *_soa(c), ops)
    elif threads:
        rc = ref().ref_gemm_rows_mt(_algo(algo), C.c_int64(param), C.c_long(bits), L, C.c_int64(m),
                                    C.c_int64(l), C.c_int64(n), *_soa(a), *_soa(b), *_soa(c), threads)
    else:
        rc = ref().ref_gemm(_algo(algo), C.c_int64(param), C.c_long(bits), L, C.c_int64(m), C.c_int64(l),
                            C.c_int64(n), *_soa(a), *_soa(b), *_soa(c), ops)
    _check(rc)
    return c, (int(ops[0]), int(ops[1]))


def gemm_replicas(algo, param, a, b, threads=1):
    """The compiled reference's product run by `threads` threads on copies of the
    same inputs; returns (C, wall seconds of the multiplies)."""
    L = a.nlimbs
    m, l, n = a.rows(), a.cols(), b.cols()
    c = OMat(m, n, a.bits(), nlimbs=L)
    secs = C.c_double(0.0)
    _check(ref().ref_gemm_replicas(_algo(algo), C.c_int64(param), C.c_long(a.bits()), L, C.c_int64(m),
                                   C.c_int64(l), C.c_int64(n), *_soa(a), *_soa(b), *_soa(c), int(threads),
                                   C.byref(secs)))
    return c, secs.value


def fast_mul_trace(algo, n_min, a, b, which="orc"):
    """fast_mul with TopTrace.  Returns (C, sums, products, t, ops)."""
    bits, L = a.bits(), a.nlimbs
    m, l, n = a.rows(), a.cols(), b.cols()
    hm, hl, hn = (m + m % 2) // 2, (l + l % 2) // 2, (n + n % 2) // 2
    total = 4 * hm * hl + 4 * hl * hn + 9 * hm * hn
    c = OMat(m, n, bits, nlimbs=L)
    tl = np.zeros(total * L, np.uint32)
    te = np.zeros(total, np.int32)
    ts = np.zeros(total, np.uint8)
    counts = (C.c_int * 3)()
    ops = (C.c_uint64 * 2)()
    if which == "orc":
        rc = orc().orc_fast_mul_trace(_algo(algo), C.c_int64(n_min), C.c_long(bits), L, C.c_int64(m),
                                      C.c_int64(l), C.c_int64(n), *_soa(a), *_soa(b), *_soa(c), _p(tl), _p(te),
                                      _p(ts), counts)
    else:
        rc = ref().ref_fast_mul_trace(_algo(algo), C.c_int64(n_min), C.c_long(bits), L, C.c_int64(m),
                                      C.c_int64(l), C.c_int64(n), *_soa(a), *_soa(b), *_soa(c), _p(tl),
                                      _p(te), _p(ts), counts, ops)
    _check(rc)
    off = 0

    def take(r, cc):
        nonlocal off
        N = r * cc
        lim = tl[off * L:(off + N) * L].reshape(L, N)
        o = OMat(r, cc, bits, lim.copy(), te[off:off + N].copy(), ts[off:off + N].copy())
        off += N
        return o

    sums = [take(hm, hl) for _ in range(min(4, counts[0]))] + [take(hl, hn) for _ in range(max(0, counts[0] - 4))]
    prods = [take(hm, hn) for _ in range(counts[1])]
    t = [take(hm, hn) for _ in range(counts[2])]
    return c, sums, prods, t, (int(ops[0]), int(ops[1]))


def addsub(is_sub, a, b):
    c = OMat(a.rows(), a.cols(), a.bits(), nlimbs=a.nlimbs)
    _check(orc().orc_addsub(int(is_sub), C.c_long(a.bits()), a.nlimbs, C.c_int64(a.rows()), C.c_int64(a.cols()),
                            *_soa(a), *_soa(b), *_soa(c)))
    return c


def vec_op(op, a, b, bits=None):
    """elementwise 0 add, 1 sub, 2 mul, 3 div at `bits` (MPFR)."""
    bits = bits or a.bits()
    n = a.rows() * a.cols()
    c = OMat(a.rows(), a.cols(), bits, nlimbs=a.nlimbs)
    rc = orc().orc_vec_op(op, C.c_long(bits), a.nlimbs, C.c_int64(n), *_soa(a), *_soa(b), *_soa(c))
    if rc not in (0, 3):
        _check(rc)
    return c


def mat_vec_mul(a, x, which="orc"):
    b = OMat(a.rows(), 1, a.bits(), nlimbs=a.nlimbs)
    f = orc().orc_mat_vec_mul if which == "orc" else ref().ref_mat_vec_mul
    _check(f(C.c_long(a.bits()), a.nlimbs, C.c_int64(a.rows()), C.c_int64(a.cols()), *_soa(a), *_soa(x), *_soa(b)))
    return b


# ---- LU ---------------------------------------------------------------------

def lu_blocked(a, K, kernel, n_min, pivoting=False, which="orc"):
    """Returns (packed OMat, piv or None, (mul, addsub) schur ops).  Raises
    OracleError(3, pivot) on a zero pivot.  which="ref" with K == 0 -> lu_columnwise."""
    n = a.rows()
    p = OMat(n, n, a.bits(), a.limbs.copy(), a.exp.copy(), a.sign.copy())
    zp = C.c_int64(0)
    ops = (C.c_uint64 * 2)()
    if which == "orc":
        piv = np.zeros(n, np.int64)
        rc = orc().orc_lu_blocked(C.c_long(a.bits()), a.nlimbs, C.c_int64(n), *_soa(p), C.c_int64(K), _algo(kernel),
                                  C.c_int64(n_min), 1 if pivoting else 0, _p(piv), C.byref(zp), ops)
    else:
        assert not pivoting, "the reference is pivot-free"
        piv = None
        rc = ref().ref_lu_blocked(C.c_long(a.bits()), a.nlimbs, C.c_int64(n), *_soa(p), C.c_int64(K), _algo(kernel),
                                  C.c_int64(n_min), C.byref(zp), ops)
    _check(rc, zp.value)
    return p, (piv if pivoting else None), (int(ops[0]), int(ops[1]))


def lu_solve(f, b, piv=None, which="orc"):
    n = f.rows()
    x = OMat(n, 1, f.bits(), nlimbs=f.nlimbs)
    zp = C.c_int64(0)
    if which == "orc":
        pv = None if piv is None else np.ascontiguousarray(piv, np.int64)
        rc = orc().orc_lu_solve(C.c_long(f.bits()), f.nlimbs, C.c_int64(n), *_soa(f),
                                None if pv is None else _p(pv), *_soa(b), *_soa(x), C.byref(zp))
    else:
        assert piv is None
        rc = ref().ref_lu_solve(C.c_long(f.bits()), f.nlimbs, C.c_int64(n), *_soa(f), *_soa(b), *_soa(x), C.byref(zp))
    _check(rc, zp.value)
    return x


# ---- generators / model ------------------------------------------------------

def prng_stream(seed, n, which="orc"):
    out = (C.c_uint64 * n)()
    f = orc().orc_prng_stream if which == "orc" else ref().ref_prng_stream
    f.restype = None
    f(C.c_uint64(seed), C.c_int64(n), out)
    return [int(v) for v in out]


def gen_random(rows, cols, seed, bits, which="orc", nlimbs=None):
    x = OMat(rows, cols, bits, nlimbs=nlimbs)
    f = orc().orc_gen_random if which == "orc" else ref().ref_gen_random
    _check(f(C.c_int64(rows), C.c_int64(cols), C.c_uint64(seed), C.c_long(bits), x.nlimbs, *_soa(x)))
    return x


def gen_full(kind, rows, cols, seed, bits, nlimbs=None):
    """kind 0: full-mantissa uniform [-1,1); kind 1: config-3 scaled (see mp_oracle.c)."""
    x = OMat(rows, cols, bits, nlimbs=nlimbs)
    _check(orc().orc_gen_full(kind, C.c_int64(rows * cols), C.c_uint64(seed), C.c_long(bits), x.nlimbs, *_soa(x)))
    return x


def gen_bench_pair(m, l, n, bits):
    a, b = OMat(m, l, bits), OMat(l, n, bits)
    _check(ref().ref_gen_bench_pair(C.c_int64(m), C.c_int64(l), C.c_int64(n), C.c_long(bits), a.nlimbs, *_soa(a),
                                    *_soa(b)))
    return a, b


def bench_reference(m, l, n, bits):
    c = OMat(m, n, bits)
    _check(ref().ref_bench_reference(C.c_int64(m), C.c_int64(l), C.c_int64(n), C.c_long(bits), c.nlimbs, *_soa(c)))
    return c


def to_hex(x):
    n = x.rows() * x.cols()
    buf = C.create_string_buffer(n * (x.bits() // 4 + 32) + 64)
    _check(ref().ref_to_hex(C.c_long(x.bits()), x.nlimbs, C.c_int64(n), *_soa(x), buf, C.c_int64(len(buf))))
    return buf.value.decode().split("\n")


def from_si(values, bits, rows=None, cols=None):
    v = np.ascontiguousarray(np.asarray(values, np.int64).reshape(-1))
    rows = rows or v.size
    cols = cols or 1
    x = OMat(rows, cols, bits)
    orc().orc_from_si(C.c_long(bits), x.nlimbs, C.c_int64(v.size), _p(v), *_soa(x))
    return x


def count_fast(algo, m, l, n, n_min, which="orc"):
    out = (C.c_uint64 * 2)()
    if which == "orc":
        orc().orc_count_fast(_algo(algo), C.c_int64(m), C.c_int64(l), C.c_int64(n), C.c_int64(n_min), out)
    else:
        _check(ref().ref_count_fast(_algo(algo), C.c_int64(m), C.c_int64(l), C.c_int64(n), C.c_int64(n_min), out))
    return int(out[0]), int(out[1])


def recursion_plan(m, l, n, n_min):
    buf = (C.c_int64 * (8 * 64))()
    cnt = C.c_int()
    _check(ref().ref_recursion_plan(C.c_int64(m), C.c_int64(l), C.c_int64(n), C.c_int64(n_min), buf, 64,
                                    C.byref(cnt)))
    return [tuple(buf[8 * i:8 * i + 8]) for i in range(cnt.value)]


def log2_max_abs_diff(x, y):
    n = x.rows() * x.cols()
    return orc().orc_log2_max_abs_diff(C.c_long(x.bits()), x.nlimbs, C.c_int64(n), *_soa(x), *_soa(y))


def log2_max_abs(x):
    n = x.rows() * x.cols()
    return orc().orc_log2_max_abs(C.c_long(x.bits()), x.nlimbs, C.c_int64(n), *_soa(x))


def to_double(x):
    n = x.rows() * x.cols()
    out = np.zeros(n, np.float64)
    orc().orc_to_double(C.c_long(x.bits()), x.nlimbs, C.c_int64(n), *_soa(x), _p(out))
    return out.reshape(x.rows(), x.cols())


# ---- accuracy metrics and benchmark drivers (compiled reference) -------------

def max_rel_error(approx, ref_m):
    """matrix.hpp:260-279 -> (OMat 2x1 {max, min} at ref's precision, skipped)."""
    n = ref_m.rows() * ref_m.cols()
    out = OMat(2, 1, ref_m.bits())
    sk = C.c_int64(0)
    _check(ref().ref_max_rel_error(C.c_long(approx.bits()), approx.nlimbs, C.c_long(ref_m.bits()), ref_m.nlimbs,
                                   C.c_int64(ref_m.rows()), C.c_int64(ref_m.cols()), *_soa(approx), *_soa(ref_m),
                                   *_soa(out), C.byref(sk)))
    return out, int(sk.value)


def solution_error(xhat, xtrue):
    """blocklu.hpp:312-333 -> (OMat 2x1 {max_rel, max_zero_abs}, zero_refs)."""
    n = xtrue.rows() * xtrue.cols()
    out = OMat(2, 1, xtrue.bits())
    zr = C.c_int64(0)
    _check(ref().ref_solution_error(C.c_long(xtrue.bits()), xtrue.nlimbs, C.c_int64(n), *_soa(xhat),
                                    *_soa(xtrue), *_soa(out), C.byref(zr)))
    return out, int(zr.value)


def one_norm(a):
    out = OMat(1, 1, a.bits())
    _check(ref().ref_one_norm(C.c_long(a.bits()), a.nlimbs, C.c_int64(a.rows()), C.c_int64(a.cols()), *_soa(a),
                              *_soa(out)))
    return out


def gen_lotkin(n, bits):
    x = OMat(n, n, bits)
    _check(ref().ref_gen_lotkin(C.c_int64(n), C.c_long(bits), x.nlimbs, *_soa(x)))
    return x


def to_decimal(x, digits):
    n = x.rows() * x.cols()
    buf = C.create_string_buffer(n * (digits + 32) + 64)
    _check(ref().ref_to_decimal(C.c_long(x.bits()), x.nlimbs, C.c_int64(n), *_soa(x), C.c_int(digits), buf,
                                C.c_int64(len(buf))))
    return buf.value.decode().split("\n")


def run_matmul(m, l, n, bits, n_min, algos=("simple", "block", "strassen", "winograd"), ref_mult=2,
               verbose=False):
    """bench.hpp:117-165 -> CSV text (print_csv)."""
    mask = 0
    for a in algos:
        mask |= 1 << _algo(a)
    buf = C.create_string_buffer(1 << 20)
    _check(ref().ref_run_matmul(C.c_int64(m), C.c_int64(l), C.c_int64(n), C.c_long(bits), C.c_int64(n_min), mask,
                                C.c_long(ref_mult), int(verbose), buf, C.c_int64(len(buf))))
    return buf.value.decode()


def run_lu(kind, n, bits, kernel, n_min, alpha_lo, alpha_hi, seed=1, verbose=False):
    """bench.hpp:187-249 -> (CSV text, any_singular)."""
    buf = C.create_string_buffer(1 << 20)
    s = C.c_int(0)
    _check(ref().ref_run_lu(0 if kind == "random" else 1, C.c_int64(n), C.c_long(bits), _algo(kernel),
                            C.c_int64(n_min), C.c_int64(alpha_lo), C.c_int64(alpha_hi), C.c_uint64(seed),
                            int(verbose), buf, C.c_int64(len(buf)), C.byref(s)))
    return buf.value.decode(), bool(s.value)


# ---- text codec / op-count tables (compiled reference) ----------------------

def from_hex(text, bits):
    """-> (OMat 1x1, None) or (None, parse error position)"""
    x = OMat(1, 1, bits)
    pos = C.c_int64(-1)
    rc = ref().ref_from_hex(text.encode(), C.c_long(bits), x.nlimbs, *_soa(x), C.byref(pos))
    if rc == 7:
        return None, int(pos.value)
    _check(rc)
    return x, None


def write_matrix(x):
    n = x.rows() * x.cols()
    buf = C.create_string_buffer(n * (x.bits() // 4 + 32) + 64)
    _check(ref().ref_write_matrix(C.c_long(x.bits()), x.nlimbs, C.c_int64(x.rows()), C.c_int64(x.cols()), *_soa(x),
                                  buf, C.c_int64(len(buf))))
    return buf.value.decode()


def read_matrix(text, cap=1 << 16, max_bits=4096):
    """-> OMat, or raises OracleError (rc 1 DimensionError, 4 IoError, ...)"""
    L = (max_bits + 31) // 32
    lim = np.zeros((L, cap), np.uint32)
    ex = np.zeros(cap, np.int32)
    sg = np.zeros(cap, np.uint8)
    dims = (C.c_int64 * 3)()
    _check(ref().ref_read_matrix(text.encode(), L, C.c_int64(cap), dims, _p(lim), _p(ex), _p(sg)))
    m, n, bits = (int(v) for v in dims)
    N = m * n
    Lb = (bits + 31) // 32
    # stored as L planes of stride N (most significant plane L-1): keep the top Lb planes
    planes = lim.reshape(-1)[:L * N].reshape(L, N)
    return OMat(m, n, bits, planes[L - Lb:].copy(), ex[:N].copy(), sg[:N].copy())


def ratio_table(sizes, n_min, fmt="table"):
    arr = (C.c_int64 * len(sizes))(*sizes)
    buf = C.create_string_buffer(1 << 16)
    _check(ref().ref_ratio_table(0 if fmt == "table" else 1, arr, len(sizes), C.c_int64(n_min), buf,
                                 C.c_int64(len(buf))))
    return buf.value.decode()


def inverse(a, bits):
    n = a.rows()
    x = OMat(n, n, bits)
    piv = C.c_int64(0)
    _check(ref().ref_inverse(C.c_long(a.bits()), a.nlimbs, C.c_int64(n), *_soa(a), C.c_long(bits), x.nlimbs,
                             *_soa(x), C.byref(piv)), piv.value)
    return x


def cond_one(a, hi_bits=0):
    bits = hi_bits or min(2 * a.bits() + 64, 1 << 20)
    out = OMat(1, 1, bits)
    piv = C.c_int64(0)
    _check(ref().ref_cond_one(C.c_long(a.bits()), a.nlimbs, C.c_int64(a.rows()), *_soa(a), C.c_long(hi_bits),
                              out.nlimbs, *_soa(out), C.byref(piv)), piv.value)
    return out
