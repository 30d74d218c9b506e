"""Host-side mirror of the reference's mpmm API (namespace mpmm,
/root/reference/proj/include/mpmm) over the B200 C-ABI (include/mpgpu.h).

Same names, argument meaning and error behaviour as the reference:

    reference (C++)                                   here
    ------------------------------------------------  ---------------------------------
    PrecisionContext(bits)        precision.hpp:18     PrecisionContext(bits)
    Matrix(rows, cols, ctx)       matrix.hpp:20        Matrix.zeros(rows, cols, ctx)
    simple_mul(a, b, ctx[, ops])  matrix.hpp:178-184   simple_mul(a, b, ctx, ops=None)
    block_mul(a, b, n_min, ctx)   matrix.hpp:225-233   block_mul(a, b, n_min, ctx, ops=None)
    add / sub                     matrix.hpp:166-175   add(a, b) / sub(a, b)
    mat_vec_mul(a, x, ctx)        matrix.hpp:282-297   mat_vec_mul(a, x, ctx)
    equal_values(a, b)            matrix.hpp:301-307   equal_values(a, b)
    recursion_plan(m,l,n,cfg)     fastmm.hpp:68-85     recursion_plan(m, l, n, cfg)
    pad_even(a)                   fastmm.hpp:235-237   pad_even(a)
    fast_mul(a, b, cfg, ctx, tr)  fastmm.hpp:244-255   fast_mul(a, b, cfg, ctx, trace=None)
    count_simple / count_fast     opmodel.hpp:17-44    count_simple / count_fast
    lu_columnwise(a)              blocklu.hpp:107-112  lu_columnwise(a)
    lu_blocked(a, cfg, ctx, ops)  blocklu.hpp:121-146  lu_blocked(a, cfg, ctx, schur_ops=None, pivoting=False)
    lu_solve(f, b, ctx)           blocklu.hpp:215-245  lu_solve(f, b, ctx)
    solve / solve_columnwise      blocklu.hpp:248-259  solve / solve_columnwise
    gen_random(r, c, seed, ctx)   matgen.hpp:45-52     gen_random(r, c, seed, ctx)

Every multiply-add runs on the GPU (libmpgpu.so); there is no CPU fallback.
Matrices here are host SoA arrays (see include/mpgpu.h); `DeviceMatrix` keeps
operands resident in HBM between calls.
"""
from __future__ import annotations

import ctypes as C
import enum
import threading
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib as _L

EXP_ZERO = -(1 << 31)

# ---------------------------------------------------------------------------
# errors (errors.hpp:10-48)
# ---------------------------------------------------------------------------


class Error(RuntimeError):
    """mpmm::Error"""


class DimensionError(Error):
    """mpmm::DimensionError"""


class DomainError(Error):
    """mpmm::DomainError"""


class SingularError(Error):
    """mpmm::SingularError; pivot_index is 1-based (0 for scalar division)."""

    def __init__(self, what: str, pivot_index: int = 0):
        super().__init__(what)
        self.pivot_index = pivot_index


class UndefinedMetricError(Error):
    """mpmm::UndefinedMetricError (errors.hpp:41-43)"""


class DeviceError(Error):
    """CUDA / allocation failure (no reference analogue)."""


def _raise(h, rc: int, pivot: int = 0):
    if rc == 0:
        return
    msg = _L.lib.mpgpu_last_error(h).decode() if h else "mpgpu error"
    if rc == 1:
        raise DimensionError(msg)
    if rc == 2:
        raise DomainError(msg)
    if rc == 3:
        raise SingularError(msg, pivot)
    if rc == 6:
        raise UndefinedMetricError(msg)
    raise DeviceError(f"[{rc}] {msg}")


# ---------------------------------------------------------------------------
# precision / algorithms / counters
# ---------------------------------------------------------------------------


class PrecisionContext:
    """precision.hpp:18-36 -- p in [2, 2^20]; RNDN fixed.  The device arithmetic
    supports p <= 9216 (mpgpu.h MPGPU_MAX_PREC: one thread per value up to 1024 bits,
    one warp per value above)."""

    min_bits = 2
    max_bits = 1 << 20

    def __init__(self, bits: int):
        if bits < self.min_bits or bits > self.max_bits:
            raise DomainError(f"precision out of range [2, 2^20]: {bits}")
        self._bits = int(bits)

    def bits(self) -> int:
        return self._bits

    def __eq__(self, o):
        return isinstance(o, PrecisionContext) and o._bits == self._bits

    def __hash__(self):
        return hash(self._bits)

    def __repr__(self):
        return f"PrecisionContext({self._bits})"


class Algorithm(enum.IntEnum):
    """fastmm.hpp:13"""
    simple = 0
    block = 1
    strassen = 2
    winograd = 3


def algorithm_name(a: Algorithm) -> str:
    return Algorithm(a).name


def parse_algorithm(s: str) -> Algorithm:
    try:
        return Algorithm[s]
    except KeyError:
        raise DomainError(f"unknown algorithm '{s}'") from None


@dataclass
class OpCounter:
    """opcounter.hpp:9-20"""
    mul: int = 0
    addsub: int = 0

    def __iadd__(self, o):
        self.mul += o.mul
        self.addsub += o.addsub
        return self

    def __add__(self, o):
        return OpCounter(self.mul + o.mul, self.addsub + o.addsub)


@dataclass
class FastMMConfig:
    """fastmm.hpp:34-37"""
    algorithm: Algorithm = Algorithm.strassen
    n_min: int = 32


@dataclass
class Dims3:
    m: int
    l: int
    n: int


@dataclass
class RecursionLevel:
    level: int
    before: Dims3
    padded: Dims3
    base: bool


@dataclass
class TopTrace:
    """fastmm.hpp:47-51"""
    sums: List["Matrix"] = field(default_factory=list)
    products: List["Matrix"] = field(default_factory=list)
    t: List["Matrix"] = field(default_factory=list)


@dataclass
class BlockLUConfig:
    """blocklu.hpp:26-34"""
    block_size: int = 32
    kernel: Algorithm = Algorithm.winograd
    n_min: int = 32

    @staticmethod
    def with_alpha(alpha: int, n_min: int, kernel: Algorithm) -> "BlockLUConfig":
        return BlockLUConfig(alpha * n_min, kernel, n_min)


@dataclass
class Stats:
    """Per-call device statistics (mpgpu_stats)."""
    mul: int = 0
    addsub: int = 0
    leaf_madds: int = 0
    device_ms: float = 0.0
    leaf_ms: float = 0.0
    preadd_ms: float = 0.0
    postadd_ms: float = 0.0
    launches: int = 0
    depth: int = 0

    @staticmethod
    def of(s: _L.MpgpuStats) -> "Stats":
        return Stats(s.mul, s.addsub, s.leaf_madds, s.device_ms, s.leaf_ms, s.preadd_ms, s.postadd_ms,
                     s.launches, s.depth)


# ---------------------------------------------------------------------------
# handle (one per device, created lazily)
# ---------------------------------------------------------------------------

_handles = {}
_hlock = threading.Lock()
_current_device = 0


def set_device(device: int) -> None:
    global _current_device
    _current_device = int(device)


def handle(device: Optional[int] = None):
    dev = _current_device if device is None else device
    with _hlock:
        h = _handles.get(dev)
        if h is None:
            hp = C.c_void_p()
            rc = _L.lib.mpgpu_init(dev, C.byref(hp))
            if rc != 0:
                raise DeviceError(f"mpgpu_init(device={dev}) failed (rc={rc}): no usable CUDA device?")
            h = hp.value
            _handles[dev] = h
        return h


def set_stream(stream_ptr: Optional[int], device: Optional[int] = None) -> None:
    """Run subsequent device work on an external cudaStream_t (e.g. a torch stream)."""
    h = handle(device)
    _raise(h, _L.lib.mpgpu_set_stream(h, C.c_void_p(stream_ptr or 0)))


def nlimbs_for(bits: int) -> int:
    return int(_L.lib.mpgpu_nlimbs_for(bits))


def record_words(nlimbs: int) -> int:
    return int(_L.lib.mpgpu_record_words(nlimbs))


def _ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


# ---------------------------------------------------------------------------
# host matrices (SoA) and device matrices (records)
# ---------------------------------------------------------------------------


class Matrix:
    """Host MP matrix in the C-ABI's SoA layout (row-major elements):
    limbs (L, rows*cols) uint32 (row L-1 most significant), exp int32 (EXP_ZERO
    for zeros), sign uint8.  All elements carry `bits` bits (matrix.hpp:20-42)."""

    def __init__(self, rows: int, cols: int, ctx: PrecisionContext, limbs=None, exp=None, sign=None):
        if rows < 1 or cols < 1:
            raise DimensionError("matrix dimensions must be at least 1x1")
        self._rows, self._cols = int(rows), int(cols)
        self._bits = ctx.bits()
        n = self._rows * self._cols
        L = max(1, (self._bits + 31) // 32)
        if limbs is None:
            limbs = np.zeros((L, n), np.uint32)
            exp = np.full(n, EXP_ZERO, np.int32)
            sign = np.zeros(n, np.uint8)
        self.limbs = np.ascontiguousarray(limbs, dtype=np.uint32).reshape(-1, n)
        self.exp = np.ascontiguousarray(exp, dtype=np.int32).reshape(n)
        self.sign = np.ascontiguousarray(sign, dtype=np.uint8).reshape(n)

    @staticmethod
    def zeros(rows: int, cols: int, ctx: PrecisionContext) -> "Matrix":
        return Matrix(rows, cols, ctx)

    def rows(self) -> int:
        return self._rows

    def cols(self) -> int:
        return self._cols

    def bits(self) -> int:
        return self._bits

    def ctx(self) -> PrecisionContext:
        return PrecisionContext(self._bits)

    @property
    def nlimbs(self) -> int:
        return self.limbs.shape[0]

    def copy(self) -> "Matrix":
        return Matrix(self._rows, self._cols, self.ctx(), self.limbs.copy(), self.exp.copy(), self.sign.copy())

    def reshaped(self, rows: int, cols: int) -> "Matrix":
        assert rows * cols == self._rows * self._cols
        return Matrix(rows, cols, self.ctx(), self.limbs, self.exp, self.sign)

    def sub(self, i0: int, j0: int, h: int, w: int) -> "Matrix":
        """Exact copy of a window (MatrixView::to_matrix, matrix.hpp:71-77)."""
        if h < 1 or w < 1:
            raise DimensionError("view must be at least 1x1")
        if i0 + h > self._rows or j0 + w > self._cols:
            raise DimensionError("view window exceeds parent matrix")
        idx = (np.arange(i0, i0 + h)[:, None] * self._cols + np.arange(j0, j0 + w)[None, :]).reshape(-1)
        return Matrix(h, w, self.ctx(), self.limbs[:, idx], self.exp[idx], self.sign[idx])

    def to_device(self, device: Optional[int] = None) -> "DeviceMatrix":
        d = DeviceMatrix(self._rows, self._cols, self.ctx(), device)
        d.upload(self)
        return d

    def to_float(self) -> np.ndarray:
        """Nearest-ish float64 of every element (inspection only, not exact)."""
        L = self.nlimbs
        top = self.limbs[L - 1].astype(np.float64)
        if L >= 2:
            top = top + self.limbs[L - 2].astype(np.float64) / 2.0 ** 32
        with np.errstate(over="ignore", under="ignore"):
            v = np.ldexp(top / 2.0 ** 32, np.where(self.exp == EXP_ZERO, 0, self.exp).astype(np.int64))
        v = np.where(self.exp == EXP_ZERO, 0.0, v)
        v = np.where(self.sign != 0, -v, v)
        return v.reshape(self._rows, self._cols)

    def __repr__(self):
        return f"Matrix({self._rows}x{self._cols}, {self._bits} bits)"


def _aligned_limbs(x: Matrix, L: int) -> np.ndarray:
    """x's limbs as L planes, most significant limbs aligned."""
    Lx = x.nlimbs
    if Lx == L:
        return x.limbs
    if Lx > L:
        return x.limbs[Lx - L:]
    out = np.zeros((L, x.limbs.shape[1]), np.uint32)
    out[L - Lx:] = x.limbs
    return out


def equal_values(a: Matrix, b: Matrix) -> bool:
    """matrix.hpp:301-307: same shape, precision and values (+0 == -0)."""
    if a.rows() != b.rows() or a.cols() != b.cols() or a.bits() != b.bits():
        return False
    L = max(a.nlimbs, b.nlimbs)
    la, lb = _aligned_limbs(a, L), _aligned_limbs(b, L)
    za, zb = a.exp == EXP_ZERO, b.exp == EXP_ZERO
    same = (za & zb) | ((~za) & (~zb) & (a.exp == b.exp) & (a.sign == b.sign) & np.all(la == lb, axis=0))
    return bool(np.all(same))


def identical(a: Matrix, b: Matrix) -> bool:
    """Bit-identical including the signs of zeros (stricter than equal_values)."""
    return equal_values(a, b) and bool(np.all(a.sign == b.sign))


class DeviceMatrix:
    """Matrix resident in HBM (mpgpu_mat, AoS records)."""

    def __init__(self, rows: int, cols: int, ctx: PrecisionContext, device: Optional[int] = None):
        self._h = handle(device)
        self.m = _L.MpgpuMat()
        _raise(self._h, _L.lib.mpgpu_alloc_matrix(self._h, rows, cols, ctx.bits(), C.byref(self.m)))

    def rows(self) -> int:
        return self.m.rows

    def cols(self) -> int:
        return self.m.cols

    def bits(self) -> int:
        return self.m.prec

    def ctx(self) -> PrecisionContext:
        return PrecisionContext(self.m.prec)

    @property
    def nbytes(self) -> int:
        return self.m.rows * self.m.cols * 4 * record_words(self.m.nlimbs)

    @property
    def data_ptr(self) -> int:
        return int(self.m.rec or 0)

    def upload(self, x: Matrix) -> None:
        if x.rows() != self.m.rows or x.cols() != self.m.cols:
            raise DimensionError("upload: shape mismatch")
        _raise(self._h, _L.lib.mpgpu_upload(self._h, C.byref(self.m), _ptr(x.limbs), _ptr(x.exp), _ptr(x.sign),
                                             x.nlimbs))

    def download(self) -> Matrix:
        ctx = self.ctx()
        out = Matrix(self.m.rows, self.m.cols, ctx)
        _raise(self._h, _L.lib.mpgpu_download(self._h, C.byref(self.m), _ptr(out.limbs), _ptr(out.exp),
                                               _ptr(out.sign), out.nlimbs))
        return out

    def free(self) -> None:
        if self.m.rec:
            _L.lib.mpgpu_free_matrix(self._h, C.byref(self.m))

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# op model / plan (host-only, no GPU needed)
# ---------------------------------------------------------------------------


def count_simple(m: int, l: int, n: int) -> OpCounter:
    """opmodel.hpp:17-23"""
    if m == 0 or l == 0 or n == 0:
        raise DimensionError("count_simple: dims must be >= 1")
    return OpCounter(m * l * n, m * n * (l - 1))


def count_fast(algo: Algorithm, m: int, l: int, n: int, n_min: int) -> OpCounter:
    """opmodel.hpp:30-44 (computed by the C-ABI's model)."""
    if n_min == 0:
        raise DimensionError("count_fast: n_min must be at least 1")
    if m == 0 or l == 0 or n == 0:
        raise DimensionError("count_simple: dims must be >= 1")
    out = (C.c_uint64 * 2)()
    rc = _L.lib.mpgpu_count_fast(int(algo), m, l, n, n_min, out)
    if rc:
        raise DimensionError("count_fast: bad arguments")
    return OpCounter(int(out[0]), int(out[1]))


def recursion_plan(m: int, l: int, n: int, cfg: FastMMConfig) -> List[RecursionLevel]:
    """fastmm.hpp:68-85"""
    if cfg.n_min == 0:
        raise DimensionError("n_min must be at least 1")
    buf = (C.c_int64 * (8 * 64))()
    cnt = C.c_int()
    _L.lib.mpgpu_recursion_plan(m, l, n, cfg.n_min, buf, 64, C.byref(cnt))
    out = []
    for i in range(cnt.value):
        r = buf[8 * i:8 * i + 8]
        out.append(RecursionLevel(r[0], Dims3(r[1], r[2], r[3]), Dims3(r[4], r[5], r[6]), bool(r[7])))
    return out


def pad_even(a: Matrix) -> Matrix:
    """fastmm.hpp:235-237: zero row/column appended for odd dims; fresh copy."""
    pm, pn = a.rows() + a.rows() % 2, a.cols() + a.cols() % 2
    out = Matrix(pm, pn, a.ctx())
    idx = (np.arange(a.rows())[:, None] * pn + np.arange(a.cols())[None, :]).reshape(-1)
    out.limbs[:, idx] = a.limbs
    out.exp[idx] = a.exp
    out.sign[idx] = a.sign
    return out


# ---------------------------------------------------------------------------
# GEMM entry points
# ---------------------------------------------------------------------------


def _operand(x, ctx: PrecisionContext):
    if isinstance(x, DeviceMatrix):
        return x, False
    if x.bits() != ctx.bits():
        # device path: one precision per call (documented deviation; MPFR would read
        # each operand at its own precision)
        raise DomainError(f"device GEMM requires operands at the context precision "
                          f"({x.bits()} != {ctx.bits()})")
    return x.to_device(), True


def _gemm(algo: Algorithm, param: int, a, b, ctx: PrecisionContext, stats_out: Optional[Stats] = None,
          keep_on_device: bool = False):
    if a.cols() != b.rows():
        raise DimensionError(f"inner dimension mismatch: {a.cols()} vs {b.rows()}")
    if algo in (Algorithm.block, Algorithm.strassen, Algorithm.winograd) and param == 0:
        raise DimensionError("n_min must be at least 1")
    da, ta = _operand(a, ctx)
    db, tb = _operand(b, ctx)
    dc = DeviceMatrix(a.rows(), b.cols(), ctx)
    st = _L.MpgpuStats()
    h = dc._h
    _raise(h, _L.lib.mpgpu_gemm(h, int(algo), int(param), C.byref(da.m), C.byref(db.m), C.byref(dc.m),
                                C.byref(st)))
    if stats_out is not None:
        s = Stats.of(st)
        stats_out.__dict__.update(s.__dict__)
    ops = OpCounter(int(st.mul), int(st.addsub))
    if ta:
        da.free()
    if tb:
        db.free()
    if keep_on_device:
        return dc, ops
    c = dc.download()
    dc.free()
    return c, ops


def gemm_into(algo: Algorithm, param: int, a: "DeviceMatrix", b: "DeviceMatrix", c: "DeviceMatrix") -> Stats:
    """C = A*B on resident device matrices into a preallocated C (no allocation,
    no host traffic) -- the building block of the benchmark's timed region."""
    st = _L.MpgpuStats()
    h = c._h
    _raise(h, _L.lib.mpgpu_gemm(h, int(algo), int(param), C.byref(a.m), C.byref(b.m), C.byref(c.m),
                                C.byref(st)))
    return Stats.of(st)


def gemm_host(algo: Algorithm, param: int, a: Matrix, b: Matrix, c: Matrix, ctx: PrecisionContext) -> Stats:
    """The reference-facing call with HOST buffers: upload A, B, multiply, download C
    (mpgpu_gemm_host).  Pin a/b/c's arrays for full copy bandwidth."""
    st = _L.MpgpuStats()
    h = handle()
    if a.nlimbs != b.nlimbs or a.nlimbs != c.nlimbs:
        raise DomainError("gemm_host: one host limb count for A, B and C")
    _raise(h, _L.lib.mpgpu_gemm_host(h, int(algo), int(param), ctx.bits(), a.rows(), a.cols(), b.cols(),
                                     _ptr(a.limbs), _ptr(a.exp), _ptr(a.sign), _ptr(b.limbs), _ptr(b.exp),
                                     _ptr(b.sign), _ptr(c.limbs), _ptr(c.exp), _ptr(c.sign), a.nlimbs,
                                     C.byref(st)))
    return Stats.of(st)


class DeviceGroup:
    """Several GPUs driven from this one process (mpgpu_group_*, include/mpgpu.h): the C-ABI
    multi-GPU path.  `devices` may repeat a device (shards of one GPU)."""

    def __init__(self, devices):
        devs = (C.c_int * len(devices))(*devices)
        hp = C.c_void_p()
        rc = _L.lib.mpgpu_group_init_devices(len(devices), devs, C.byref(hp))
        if rc:
            raise DeviceError(f"mpgpu_group_init_devices({list(devices)}) failed (rc={rc})")
        self._g = hp.value
        self.devices = list(devices)

    @staticmethod
    def from_mask(mask: int) -> "DeviceGroup":
        return DeviceGroup([d for d in range(32) if mask >> d & 1])

    def size(self) -> int:
        return _L.lib.mpgpu_group_size(self._g)

    def gemm_host(self, algo: Algorithm, param: int, a: Matrix, b: Matrix, c: Matrix, ctx: PrecisionContext) -> Stats:
        """mpgpu_group_gemm_host: the product over every device of the group, host SoA in
        and out; bit-identical to gemm_host on one device."""
        if a.nlimbs != b.nlimbs or a.nlimbs != c.nlimbs:
            raise DomainError("gemm_host: one host limb count for A, B and C")
        st = _L.MpgpuStats()
        rc = _L.lib.mpgpu_group_gemm_host(self._g, int(algo), int(param), ctx.bits(), a.rows(), a.cols(), b.cols(),
                                          _ptr(a.limbs), _ptr(a.exp), _ptr(a.sign), _ptr(b.limbs), _ptr(b.exp),
                                          _ptr(b.sign), _ptr(c.limbs), _ptr(c.exp), _ptr(c.sign), a.nlimbs,
                                          C.byref(st))
        if rc:
            msg = (_L.lib.mpgpu_group_last_error(self._g) or b"").decode()
            raise {1: DimensionError, 2: DomainError}.get(rc, DeviceError)(msg)
        return Stats.of(st)

    def close(self) -> None:
        if getattr(self, "_g", None):
            _L.lib.mpgpu_group_destroy(self._g)
            self._g = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def simple_mul(a, b, ctx: PrecisionContext, ops: Optional[OpCounter] = None, stats: Optional[Stats] = None):
    """matrix.hpp:178-184 -- three-loop inner product, left to right in k."""
    c, o = _gemm(Algorithm.simple, 0, a, b, ctx, stats, isinstance(a, DeviceMatrix))
    if ops is not None:
        ops += o
    return c


def block_mul(a, b, n_min: int, ctx: PrecisionContext, ops: Optional[OpCounter] = None,
              stats: Optional[Stats] = None):
    """matrix.hpp:225-233 -- n_min tiles, k-tiles accumulated left to right."""
    c, o = _gemm(Algorithm.block, n_min, a, b, ctx, stats, isinstance(a, DeviceMatrix))
    if ops is not None:
        ops += o
    return c


@dataclass
class FastMMResult:
    """fastmm.hpp:39-42"""
    c: object
    ops: OpCounter


AUTO_NMIN = -1  # MPGPU_AUTO_NMIN: FastMMConfig(algo, AUTO_NMIN) -> cutoff chosen per precision


def choose_n_min(algo: Algorithm, bits: int, m: int, l: int, n: int):
    """mpgpu_choose_nmin: (n_min, depth, modelled ms) for an m x l x n Strassen / Winograd
    product at `bits` -- the depth whose modelled time (measured leaf-GEMM rate at that leaf
    size + pre/post-addition bytes at the measured bandwidth) is smallest."""
    nm, d, ms = C.c_int64(0), C.c_int32(0), C.c_double(0)
    rc = _L.lib.mpgpu_choose_nmin(int(algo), int(bits), m, l, n, C.byref(nm), C.byref(d), C.byref(ms))
    if rc == 1:
        raise DimensionError("choose_n_min: dimensions must be at least 1")
    if rc:
        raise DomainError("choose_n_min: strassen / winograd at a supported precision")
    return int(nm.value), int(d.value), float(ms.value)


def fast_mul(a, b, cfg: FastMMConfig, ctx: PrecisionContext, trace: Optional[TopTrace] = None,
             stats: Optional[Stats] = None) -> FastMMResult:
    """fastmm.hpp:244-255 -- Strassen / Winograd with cutoff n_min and pad-to-even."""
    if a.cols() != b.rows():
        raise DimensionError(f"inner dimension mismatch: {a.cols()} vs {b.rows()}")
    if cfg.n_min == 0:
        raise DimensionError("n_min must be at least 1")
    if cfg.algorithm not in (Algorithm.strassen, Algorithm.winograd):
        raise DomainError("fast_mul: algorithm must be strassen or winograd")
    if trace is None:
        c, o = _gemm(cfg.algorithm, cfg.n_min, a, b, ctx, stats, isinstance(a, DeviceMatrix))
        return FastMMResult(c, o)
    if cfg.n_min == AUTO_NMIN:
        cfg = FastMMConfig(cfg.algorithm, choose_n_min(cfg.algorithm, ctx.bits(), a.rows(), a.cols(), b.cols())[0])
    return _fast_mul_traced(a, b, cfg, ctx, trace)


def _fast_mul_traced(a, b, cfg, ctx, trace: TopTrace) -> FastMMResult:
    da, ta = _operand(a, ctx)
    db, tb = _operand(b, ctx)
    dc = DeviceMatrix(a.rows(), b.cols(), ctx)
    m, l, n = a.rows(), a.cols(), b.cols()
    hm, hl, hn = (m + m % 2) // 2, (l + l % 2) // 2, (n + n % 2) // 2
    S = record_words(dc.m.nlimbs)
    total = 4 * hm * hl + 4 * hl * hn + 9 * hm * hn
    import torch  # device scratch for the trace (plumbing only)
    buf = torch.empty(total * S, dtype=torch.int32, device=f"cuda:{_current_device}")
    counts = (C.c_int * 3)()
    h = dc._h
    _raise(h, _L.lib.mpgpu_fast_mul_trace(h, int(cfg.algorithm), cfg.n_min, C.byref(da.m), C.byref(db.m),
                                          C.byref(dc.m), C.c_void_p(buf.data_ptr()), counts))
    torch.cuda.synchronize()
    host = buf.cpu().numpy().view(np.uint32).reshape(-1, S)
    off = 0
    L = dc.m.nlimbs

    def take(r, c_):
        nonlocal off
        rec = host[off:off + r * c_]
        off += r * c_
        return _records_to_matrix(rec, r, c_, ctx, L)

    shapes_s = [(hm, hl)] * 4 + [(hl, hn)] * 4
    for i in range(counts[0]):
        trace.sums.append(take(*shapes_s[i]))
    for _ in range(counts[1]):
        trace.products.append(take(hm, hn))
    for _ in range(counts[2]):
        trace.t.append(take(hm, hn))
    c = dc.download()
    dc.free()
    if ta:
        da.free()
    if tb:
        db.free()
    return FastMMResult(c, count_fast(cfg.algorithm, m, l, n, cfg.n_min))


def _records_to_matrix(rec: np.ndarray, rows: int, cols: int, ctx: PrecisionContext, L: int) -> Matrix:
    out = Matrix(rows, cols, ctx)
    Lh = out.nlimbs
    lim = rec[:, :L].T  # (L, N)
    out.limbs[:] = lim[L - Lh:] if L >= Lh else np.vstack([np.zeros((Lh - L, lim.shape[1]), np.uint32), lim])
    out.exp[:] = rec[:, L].view(np.int32)
    out.sign[:] = rec[:, L + 1].astype(np.uint8)
    return out


def _elementwise(op: int, a, b) -> Matrix:
    da, ta = _operand(a, a.ctx())
    db, tb = _operand(b, a.ctx())
    dc = DeviceMatrix(a.rows(), a.cols(), a.ctx())
    _raise(dc._h, _L.lib.mpgpu_vec_op(dc._h, op, C.byref(da.m), C.byref(db.m), C.byref(dc.m)))
    c = dc.download()
    for d, t in ((da, ta), (db, tb), (dc, True)):
        if t:
            d.free()
    return c


def _check_addsub(a, b, name):
    if a.bits() != b.bits():
        raise DomainError(f"mat {name}: mixed precisions")
    if a.rows() != b.rows() or a.cols() != b.cols():
        raise DimensionError(f"shape mismatch: {a.rows()}x{a.cols()} vs {b.rows()}x{b.cols()}")


def add(a: Matrix, b: Matrix) -> Matrix:
    """matrix.hpp:166-169"""
    _check_addsub(a, b, "add")
    return _elementwise(0, a, b)


def sub(a: Matrix, b: Matrix) -> Matrix:
    """matrix.hpp:172-175"""
    _check_addsub(a, b, "sub")
    return _elementwise(1, a, b)


def vec_op(op: int, a: Matrix, b: Matrix) -> Matrix:
    """Elementwise scalar op (0 add, 1 sub, 2 mul, 3 div) -- precision.hpp:127-161."""
    return _elementwise(op, a, b)


def mat_vec_mul(a: Matrix, x: Matrix, ctx: PrecisionContext) -> Matrix:
    """matrix.hpp:282-297: b_i = sum_j a_ij x_j left to right -- the same operation
    sequence as simple_mul(a, x) with x as an n x 1 matrix.  x, b: n x 1."""
    if x.rows() * x.cols() != a.cols():
        raise DimensionError("mat_vec_mul: length mismatch")
    return simple_mul(a, x.reshaped(a.cols(), 1), ctx)


# ---------------------------------------------------------------------------
# LU (blocklu.hpp)
# ---------------------------------------------------------------------------


@dataclass
class LUFactors:
    """blocklu.hpp:16-21 (+ piv: LAPACK-style 0-based row interchanges, or None)."""
    n: int
    packed: Matrix
    piv: Optional[np.ndarray] = None

    def bits(self) -> int:
        return self.packed.bits()


def lu_blocked(a: Matrix, cfg: BlockLUConfig, ctx: PrecisionContext, schur_ops: Optional[OpCounter] = None,
               pivoting: bool = False, stats: Optional[Stats] = None) -> LUFactors:
    """blocklu.hpp:121-146.  pivoting=True adds partial pivoting (extension)."""
    if a.rows() != a.cols():
        raise DimensionError("lu_blocked: matrix must be square")
    if a.bits() != ctx.bits():
        raise DomainError("lu_blocked: working context must match the matrix precision")
    if cfg.block_size == 0:
        raise DimensionError("lu_blocked: block size must be at least 1")
    da = a.to_device()
    n = a.rows()
    piv = np.zeros(n, np.int64)
    zp = C.c_int64(0)
    st = _L.MpgpuStats()
    rc = _L.lib.mpgpu_lu_blocked(da._h, C.byref(da.m), cfg.block_size, int(cfg.kernel), cfg.n_min,
                                 1 if pivoting else 0, _ptr(piv), C.byref(zp), C.byref(st))
    if rc:
        da.free()
        _raise(da._h, rc, zp.value)
    if schur_ops is not None:
        schur_ops += OpCounter(int(st.mul), int(st.addsub))
    if stats is not None:
        stats.__dict__.update(Stats.of(st).__dict__)
    packed = da.download()
    da.free()
    return LUFactors(n, packed, piv if pivoting else None)


def lu_blocked_host(a: Matrix, cfg: BlockLUConfig, ctx: PrecisionContext, pivoting: bool = False,
                    stats: Optional[Stats] = None, out: Optional[Matrix] = None) -> LUFactors:
    """lu_blocked through mpgpu_lu_blocked_host: the factorisation of a host matrix with the
    transfers overlapped (page-locked buffers; `out`, if given, receives the factors and may be
    `a` itself).  Bit-identical to lu_blocked."""
    if a.rows() != a.cols():
        raise DimensionError("lu_blocked: matrix must be square")
    if a.bits() != ctx.bits():
        raise DomainError("lu_blocked: working context must match the matrix precision")
    if cfg.block_size == 0:
        raise DimensionError("lu_blocked: block size must be at least 1")
    n = a.rows()
    if out is None:
        out = Matrix(n, n, a.ctx(), a.limbs.copy(), a.exp.copy(), a.sign.copy())
    elif out is not a:
        out.limbs[:], out.exp[:], out.sign[:] = a.limbs, a.exp, a.sign
    h = handle()
    piv = np.zeros(n, np.int64)
    zp = C.c_int64(0)
    st = _L.MpgpuStats()
    rc = _L.lib.mpgpu_lu_blocked_host(h, a.bits(), n, _ptr(out.limbs), _ptr(out.exp), _ptr(out.sign), out.nlimbs,
                                      cfg.block_size, int(cfg.kernel), cfg.n_min, 1 if pivoting else 0, _ptr(piv),
                                      C.byref(zp), C.byref(st))
    _raise(h, rc, zp.value)
    if stats is not None:
        stats.__dict__.update(Stats.of(st).__dict__)
    return LUFactors(n, out, piv if pivoting else None)


def lu_columnwise(a: Matrix) -> LUFactors:
    """blocklu.hpp:107-112 (== lu_blocked with K >= n)."""
    if a.rows() != a.cols():
        raise DimensionError("lu_columnwise: matrix must be square")
    return lu_blocked(a, BlockLUConfig(a.rows(), Algorithm.simple, 1), a.ctx())


def lu_solve(f: LUFactors, b: Matrix, ctx: PrecisionContext, exact: bool = True) -> Matrix:
    """blocklu.hpp:215-245 (b, x: n x 1); applies f.piv first when present.
    exact=True replays the reference's summation order bit-exactly (serial back
    substitution); exact=False runs it column-oriented (fast, within tolerance)."""
    n = f.n
    if b.rows() * b.cols() != n:
        raise DimensionError("lu_solve: length mismatch")
    df = f.packed.to_device()
    db = b.reshaped(n, 1).to_device()
    dx = DeviceMatrix(n, 1, ctx)
    zp = C.c_int64(0)
    piv = None if f.piv is None else np.ascontiguousarray(f.piv, np.int64)
    rc = _L.lib.mpgpu_lu_solve(df._h, C.byref(df.m), None if piv is None else _ptr(piv), C.byref(db.m),
                               C.byref(dx.m), 1 if exact else 0, C.byref(zp))
    try:
        _raise(df._h, rc, zp.value)
        return dx.download()
    finally:
        df.free()
        db.free()
        dx.free()


def solve(a: Matrix, b: Matrix, cfg: BlockLUConfig, ctx: PrecisionContext, pivoting: bool = False,
          exact: bool = True) -> Matrix:
    """blocklu.hpp:248-252"""
    return lu_solve(lu_blocked(a, cfg, ctx, pivoting=pivoting), b, ctx, exact)


def solve_columnwise(a: Matrix, b: Matrix) -> Matrix:
    """blocklu.hpp:256-259"""
    return lu_solve(lu_columnwise(a), b, a.ctx())


# ---------------------------------------------------------------------------
# accuracy metrics, device-side (matrix.hpp:237-279, blocklu.hpp:306-333)
# ---------------------------------------------------------------------------


@dataclass
class RelErrorStats:
    """matrix.hpp:253-258; max / min are 1x1 Matrices at the reference's precision."""
    max: Matrix
    min: Matrix
    skipped_zero_refs: int = 0


@dataclass
class SolutionError:
    """blocklu.hpp:306-310"""
    max_rel: Matrix
    max_zero_abs: Matrix
    zero_refs: int = 0


def _dev(x, ctx=None):
    if isinstance(x, DeviceMatrix):
        return x, False
    return x.to_device(), True


def _metric_out(ref_bits: int, count: int):
    L = nlimbs_for(ref_bits)
    return (np.zeros((L, count), np.uint32), np.zeros(count, np.int32), np.zeros(count, np.uint8), L)


def _scalars(ol, oe, os_, bits, L):
    out = []
    for e in range(oe.shape[0]):
        m = Matrix(1, 1, PrecisionContext(bits), ol[:, e:e + 1].copy(), oe[e:e + 1].copy(), os_[e:e + 1].copy())
        out.append(m)
    return out


def max_rel_error(approx, ref) -> RelErrorStats:
    """matrix.hpp:260-279 on the device: rel_error = RN(|RN(approx - ref)| / |ref|) at
    ref's precision (precision.hpp:187-193); zero references skipped and counted."""
    if approx.rows() != ref.rows() or approx.cols() != ref.cols():
        raise DimensionError(f"shape mismatch: {approx.rows()}x{approx.cols()} vs {ref.rows()}x{ref.cols()}")
    da, fa = _dev(approx)
    dr, fr = _dev(ref)
    ol, oe, os_, L = _metric_out(ref.bits(), 2)
    skipped = C.c_int64(0)
    try:
        _raise(dr._h, _L.lib.mpgpu_max_rel_error(dr._h, C.byref(da.m), C.byref(dr.m), _ptr(ol), _ptr(oe),
                                                 _ptr(os_), C.byref(skipped)))
    finally:
        if fa:
            da.free()
        if fr:
            dr.free()
    mx, mn = _scalars(ol, oe, os_, ref.bits(), L)
    return RelErrorStats(mx, mn, int(skipped.value))


def max_rel_error_solution(xhat, xtrue) -> SolutionError:
    """blocklu.hpp:312-333 on the device (vectors as n x 1 matrices)."""
    if xhat.rows() * xhat.cols() != xtrue.rows() * xtrue.cols():
        raise DimensionError("solution error: length mismatch")
    dx, fx = _dev(xhat)
    dt, ft = _dev(xtrue)
    ol, oe, os_, L = _metric_out(xtrue.bits(), 2)
    zr = C.c_int64(0)
    try:
        _raise(dt._h, _L.lib.mpgpu_solution_error(dt._h, C.byref(dx.m), C.byref(dt.m), _ptr(ol), _ptr(oe),
                                                  _ptr(os_), C.byref(zr)))
    finally:
        if fx:
            dx.free()
        if ft:
            dt.free()
    mr, mz = _scalars(ol, oe, os_, xtrue.bits(), L)
    return SolutionError(mr, mz, int(zr.value))


def one_norm(a) -> Matrix:
    """matrix.hpp:237-251 on the device: 1x1 Matrix at a's precision."""
    da, fa = _dev(a)
    ol, oe, os_, L = _metric_out(a.bits(), 1)
    try:
        _raise(da._h, _L.lib.mpgpu_one_norm(da._h, C.byref(da.m), _ptr(ol), _ptr(oe), _ptr(os_)))
    finally:
        if fa:
            da.free()
    return _scalars(ol, oe, os_, a.bits(), L)[0]


# ---------------------------------------------------------------------------
# precision conversion, multi-RHS solves, inverse and 1-norm condition number
# (blocklu.hpp:261-301; SURVEY.md §8f rank 3 within the device precision range)
# ---------------------------------------------------------------------------


def convert(a, ctx: PrecisionContext) -> "DeviceMatrix":
    """mpfr_set of every element into ctx (round to nearest), on the device."""
    da, fa = _dev(a)
    out = DeviceMatrix(da.rows(), da.cols(), ctx)
    try:
        _raise(out._h, _L.lib.mpgpu_convert(out._h, C.byref(da.m), C.byref(out.m)))
    except Exception:
        out.free()
        raise
    finally:
        if fa:
            da.free()
    return out


def lu_solve_many(f: LUFactors, bt: Matrix, ctx: PrecisionContext, exact: bool = True) -> Matrix:
    """lu_solve (blocklu.hpp:215-245) for every row of the r x n matrix bt at once."""
    n = f.n
    if bt.cols() != n:
        raise DimensionError("lu_solve_many: right-hand sides must be the rows of an r x n matrix")
    df = f.packed.to_device()
    db = bt.to_device()
    dx = DeviceMatrix(bt.rows(), n, ctx)
    zp = C.c_int64(0)
    piv = None if f.piv is None else np.ascontiguousarray(f.piv, np.int64)
    rc = _L.lib.mpgpu_lu_solve_many(df._h, C.byref(df.m), None if piv is None else _ptr(piv), C.byref(db.m),
                                    C.byref(dx.m), 1 if exact else 0, C.byref(zp))
    try:
        _raise(df._h, rc, zp.value)
        return dx.download()
    finally:
        df.free()
        db.free()
        dx.free()


def _transpose(x: Matrix) -> Matrix:
    r, c = x.rows(), x.cols()
    idx = np.arange(r * c).reshape(r, c).T.reshape(-1)
    return Matrix(c, r, x.ctx(), x.limbs[:, idx], x.exp[idx], x.sign[idx])


def inverse(a: Matrix, ctx: PrecisionContext) -> Matrix:
    """blocklu.hpp:263-281: a copied into ctx, lu_columnwise, one lu_solve per unit
    vector (all n at once on the device), same operation order (bit-exact)."""
    if a.rows() != a.cols():
        raise DimensionError("inverse: matrix must be square")
    n = a.rows()
    dahi = convert(a, ctx)
    ahi = dahi.download()
    dahi.free()
    f = lu_columnwise(ahi)
    from .matgen import from_ints
    eye = from_ints(np.eye(n, dtype=np.int64), ctx, n, n)
    xt = lu_solve_many(f, eye, ctx)  # row j = the solution for e_j = column j of the inverse
    return _transpose(xt)


def cond_one(a: Matrix, ctx_hi: Optional[PrecisionContext] = None) -> Matrix:
    """blocklu.hpp:285-301: ||A||_1 * ||A^-1||_1 with everything at ctx_hi (default
    min(2 bits + 64, max_bits)); 1x1 Matrix.  Device arithmetic: ctx_hi <= 9216 bits."""
    if ctx_hi is None:
        ctx_hi = PrecisionContext(min(2 * a.bits() + 64, PrecisionContext.max_bits))
    dahi = convert(a, ctx_hi)
    try:
        na = one_norm(dahi)
    finally:
        dahi.free()
    ni = one_norm(inverse(a, ctx_hi))
    return vec_op(2, na, ni)
