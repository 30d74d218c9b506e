"""Multi-GPU execution of one MP GEMM (one process per GPU, torch.distributed
plumbing, NCCL for the one exchange step).  DESIGN.md section 6.

Strassen / Winograd (fastmm.hpp:99-229): the recursion tree is split at the bottom.
Every rank runs the pre-additions of the ancestors of its own units only, the leaf
GEMMs of its units, and (when units are whole sibling groups) the first post-addition
level locally; one all-gather of the unit products then gives every rank all of
them, and the remaining post-addition levels (a few percent of the work) run on
each rank.  Elementwise post-additions commute with the split, so the result is
bit-identical to the single-GPU product (and to the reference).  There is no
all-reduce: MP rounded sums are not an NCCL reduction and are order-sensitive.

Default combine: instead of gathering every unit product on every rank, one all-to-all
moves each unit product's row slices to the rank that owns them, and each rank runs
the post-additions for its rows of C only (mpgpu_fast_combine_rows: ownership
propagates through the pad/halve index map), so no post-addition is replicated and
each byte crosses NVLink once.  C stays distributed by rows ('gather' mode keeps the
all-gather + replicated combine when every rank needs all of C).

Simple / Block (matrix.hpp:178-233): C is split by row blocks (row i of C depends on
row i of A and all of B; Block's k-tiles are row-independent), then all-gathered.

The partition arithmetic is pure Python (tested with world_size 2 on gloo).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import List, Tuple

from . import _lib as _L


@dataclass(frozen=True)
class Shard:
    lo: int      # first unit owned by this rank
    hi: int      # one past the last unit owned
    per: int     # units per rank slot (ranks are padded to `per` for all_gather)


def even_ranges(units: int, world: int) -> List[Shard]:
    """Contiguous, padded ranges: rank r owns [r*per, min((r+1)*per, units)), so the
    all-gathered buffer holds unit u at slot u (padding only after the last unit)."""
    per = max(1, math.ceil(units / world))
    return [Shard(min(r * per, units), min((r + 1) * per, units), per) for r in range(world)]


def choose_split(depth: int, world: int) -> int:
    """up_levels in {0, 1}: 0 splits individual leaves (7^d units, leaf products
    exchanged), 1 splits sibling groups (7^(d-1) units, 4/7 of the bytes exchanged
    and the first post-addition level done locally).  Take groups unless that makes
    the busiest rank's leaf work more than 5 % above the leaf split's."""
    if depth < 2:
        return 0
    leaves = 7 ** depth
    busiest_leaf = math.ceil(leaves / world)
    busiest_group = 7 * math.ceil(leaves // 7 / world)
    return 1 if busiest_group <= 1.05 * busiest_leaf else 0


def fast_plan(m: int, l: int, n: int, n_min: int) -> Tuple[int, int, int, int, int]:
    """(depth, leaves, leaf_m, leaf_l, leaf_n) -- mpgpu_fast_plan."""
    out = (C.c_int64 * 5)()
    rc = _L.lib.mpgpu_fast_plan(m, l, n, n_min, out)
    if rc:
        raise ValueError("fast_plan: bad arguments")
    return tuple(int(v) for v in out)


def node_dims(m: int, l: int, n: int, n_min: int, level: int) -> Tuple[int, int]:
    """(rows, cols) of a level-`level` node's product."""
    for _ in range(level):
        m, n = (m + m % 2) // 2, (n + n % 2) // 2
    return m, n


class _Replica:
    """Every rank multiplies its own copy (weak scaling, no exchange)."""
    replicated = True
    mode = "replicas"

    def __init__(self, algo, param, da, db, dc):
        self.algo, self.param, self.da, self.db, self.dc = algo, param, da, db, dc

    def __call__(self):
        from .mpmm import gemm_into
        return gemm_into(self.algo, self.param, self.da, self.db, self.dc)


class _FastSharded:
    replicated = False
    mode = "leaf-shard"

    def __init__(self, algo, n_min, da, db, dc, rank, world, group=None):
        import torch
        from .mpmm import record_words
        self.algo, self.n_min, self.da, self.db, self.dc = int(algo), n_min, da, db, dc
        self.group = group
        m, l, n = da.rows(), da.cols(), db.cols()
        self.l = l
        depth, leaves, *_ = fast_plan(m, l, n, n_min)
        if depth == 0:
            raise ValueError("leaf sharding needs a recursion (depth >= 1)")
        self.up = choose_split(depth, world)
        units = 7 ** (depth - self.up)
        self.shard = even_ranges(units, world)[rank]
        um, un = node_dims(m, l, n, n_min, depth - self.up)
        words = um * un * record_words(dc.m.nlimbs)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.local = torch.zeros(self.shard.per * words, dtype=torch.int32, device=dev)
        self.all = torch.zeros(world * self.shard.per * words, dtype=torch.int32, device=dev)
        self.mode = f"leaf-shard(up={self.up}, units={units}, per_rank={self.shard.per})"

    def __call__(self):
        import torch.distributed as dist
        from .mpmm import Stats, _raise
        st = _L.MpgpuStats()
        h = self.dc._h
        if self.shard.hi > self.shard.lo:
            _raise(h, _L.lib.mpgpu_fast_leaves(h, self.algo, self.n_min, C.byref(self.da.m), C.byref(self.db.m),
                                               self.up, self.shard.lo, self.shard.hi,
                                               C.c_void_p(self.local.data_ptr()), C.byref(st)))
        _streams_join(h)
        all_gather_rows(self.all, self.local, self.group)
        _streams_join(h)
        st2 = _L.MpgpuStats()
        _raise(h, _L.lib.mpgpu_fast_combine(h, self.algo, self.n_min, self.l, self.up,
                                            C.c_void_p(self.all.data_ptr()), C.byref(self.dc.m), C.byref(st2)))
        s = Stats.of(st)
        s.postadd_ms += st2.postadd_ms
        s.launches += st2.launches
        s.mul, s.addsub = _count(self.algo, self.da, self.db, self.n_min)
        return s


# ---------------------------------------------------------------------------
# Row-owned combine: one all-to-all of unit-product row slices, then every rank
# post-adds only the rows of C it owns (no replicated post-additions).
# ---------------------------------------------------------------------------


def level_rows(m: int, depth: int) -> List[int]:
    """rows of a level-t node, t = 0 .. depth (pad odd to even, halve)."""
    out = [m]
    for _ in range(depth):
        m = (m + m % 2) // 2
        out.append(m)
    return out


def owned_c_rows(m: int, depth: int, unit_level: int, lo: int, hi: int) -> List[int]:
    """Rows of C produced from the unit-level rows [lo, hi): a level-t row r comes from
    child row r (top quadrants) or r - m_{t+1} (bottom) -- mpgpu_fast_combine_rows."""
    rows = level_rows(m, depth)
    owned = [r for r in range(lo, min(hi, rows[unit_level]))]
    for t in range(unit_level - 1, -1, -1):
        hm = rows[t + 1]
        mark = set()
        for rc in owned:
            if rc < rows[t]:
                mark.add(rc)
            if rc + hm < rows[t]:
                mark.add(rc + hm)
        owned = sorted(mark)
    return owned


def a2a_pack_plan(my_units: Shard, rows: List[Shard], um: int, un: int, rw: int):
    """2D copies (in 32-bit words) of this rank's unit products into the all-to-all send
    buffer: chunk t holds rows [rows[t].lo, rows[t].hi) of every local unit, padded to
    my_units.per units x rows[t].per rows.  Returns (copies, chunk words)."""
    row_w = un * rw
    unit_w = um * row_w
    chunk = my_units.per * rows[0].per * row_w
    nloc = my_units.hi - my_units.lo
    plan = []
    for t, rr in enumerate(rows):
        h = rr.hi - rr.lo
        if nloc > 0 and h > 0:
            plan.append(dict(dst=t * chunk, dpitch=rows[0].per * row_w, src=rr.lo * row_w, spitch=unit_w,
                             width=h * row_w, height=nloc))
    return plan, chunk


def a2a_unpack_plan(units: List[Shard], my_rows: Shard, rows_per: int, um: int, un: int, rw: int):
    """2D copies from the receive buffer (chunk s = source rank s's units, my rows) into
    the all-units product buffer (unit-major, only my rows filled)."""
    row_w = un * rw
    unit_w = um * row_w
    chunk = units[0].per * rows_per * row_w
    h = my_rows.hi - my_rows.lo
    plan = []
    for s_, us in enumerate(units):
        n = us.hi - us.lo
        if n > 0 and h > 0:
            plan.append(dict(dst=(us.lo * um + my_rows.lo) * row_w, dpitch=unit_w, src=s_ * chunk,
                             spitch=rows_per * row_w, width=h * row_w, height=n))
    return plan


def run_plan_torch(plan, dst, src):
    """Execute a copy plan on flat int32 tensors (CPU or GPU; torch indexing)."""
    for c in plan:
        for r in range(c["height"]):
            d0, s0 = c["dst"] + r * c["dpitch"], c["src"] + r * c["spitch"]
            dst[d0:d0 + c["width"]] = src[s0:s0 + c["width"]]


class _FastRowOwned:
    """Strassen / Winograd over N GPUs with a row-owned combine: leaf products of the
    rank's units (mpgpu_fast_leaves), one all_to_all_single of unit-product row slices,
    then mpgpu_fast_combine_rows for the rank's rows only.  C ends up distributed: rank
    r holds the rows owned_c_rows(..) of C (the rest of its C buffer is not written)."""
    replicated = False

    def __init__(self, algo, n_min, da, db, dc, rank, world, group=None):
        import torch
        from .mpmm import record_words
        self.algo, self.n_min, self.da, self.db, self.dc = int(algo), n_min, da, db, dc
        self.group, self.rank, self.world = group, rank, world
        m, l, n = da.rows(), da.cols(), db.cols()
        self.l = l
        depth, leaves, *_ = fast_plan(m, l, n, n_min)
        if depth == 0:
            raise ValueError("leaf sharding needs a recursion (depth >= 1)")
        self.up = choose_split(depth, world)
        units = 7 ** (depth - self.up)
        self.units = even_ranges(units, world)
        self.shard = self.units[rank]
        um, un = node_dims(m, l, n, n_min, depth - self.up)
        self.rows = even_ranges(um, world)
        self.my_rows = self.rows[rank]
        rw = record_words(dc.m.nlimbs)
        self.rw, self.um, self.un = rw, um, un
        self.pack, chunk = a2a_pack_plan(self.shard, self.rows, um, un, rw)
        self.unpack = a2a_unpack_plan(self.units, self.my_rows, self.rows[0].per, um, un, rw)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.local = torch.zeros(max(1, self.shard.per * um * un * rw), dtype=torch.int32, device=dev)
        self.send = torch.zeros(world * chunk, dtype=torch.int32, device=dev)
        self.recv = torch.zeros_like(self.send)
        self.full = torch.zeros(units * um * un * rw, dtype=torch.int32, device=dev)
        self.c_rows = owned_c_rows(m, depth, depth - self.up, self.my_rows.lo, self.my_rows.hi)
        self.mode = (f"row-owned(up={self.up}, units={units}, per_rank={self.shard.per}, "
                     f"unit_rows_per_rank={self.rows[0].per})")

    def _copies(self, plan, dst, src):
        h = self.dc._h
        for c in plan:
            _raise_rc(h, _L.lib.mpgpu_copy_device_2d(
                h, C.c_void_p(dst.data_ptr() + 4 * c["dst"]), 4 * c["dpitch"],
                C.c_void_p(src.data_ptr() + 4 * c["src"]), 4 * c["spitch"], 4 * c["width"], c["height"]))

    def __call__(self):
        import torch.distributed as dist
        from .mpmm import Stats, _raise
        st = _L.MpgpuStats()
        h = self.dc._h
        if self.shard.hi > self.shard.lo:
            _raise(h, _L.lib.mpgpu_fast_leaves(h, self.algo, self.n_min, C.byref(self.da.m), C.byref(self.db.m),
                                               self.up, self.shard.lo, self.shard.hi,
                                               C.c_void_p(self.local.data_ptr()), C.byref(st)))
        self._copies(self.pack, self.send, self.local)
        _streams_join(h)
        all_to_all_rows(self.recv, self.send, self.group)
        _streams_join(h)
        self._copies(self.unpack, self.full, self.recv)
        st2 = _L.MpgpuStats()
        _raise(h, _L.lib.mpgpu_fast_combine_rows(h, self.algo, self.n_min, self.l, self.up,
                                                 C.c_void_p(self.full.data_ptr()), self.my_rows.lo,
                                                 self.my_rows.hi, C.byref(self.dc.m), C.byref(st2)))
        s = Stats.of(st)
        s.postadd_ms += st2.postadd_ms
        s.launches += st2.launches
        s.mul, s.addsub = _count(self.algo, self.da, self.db, self.n_min)
        return s


class _FastRowOwnedP2P:
    """Strassen / Winograd over N GPUs, one process each, with the exchange FUSED into the
    producing kernels: every rank allocates its unit-product buffer (all units, its own unit
    rows) with cudaMalloc and shares its CUDA IPC handle; each rank maps the others' buffers
    (peer access over NVLink / NVSwitch) and hands mpgpu_fast_leaves_rows a device table of row
    destinations, so the leaf GEMM's (or last local post-addition's) epilogue stores every
    product row straight into the buffer of the rank that owns it.  No all-to-all, no packing,
    no staging: the transfer overlaps the leaf math tile by tile.  Then mpgpu_fast_combine_rows
    for the rank's rows, as _FastRowOwned.  Host barriers order the steps (products landed ->
    combine; combine read -> next step's stores).  Precisions <= 1024 bits."""
    replicated = False

    def __init__(self, algo, n_min, da, db, dc, rank, world, group=None):
        import torch
        import torch.distributed as dist
        from .mpmm import record_words
        self.algo, self.n_min, self.da, self.db, self.dc = int(algo), n_min, da, db, dc
        self.group, self.rank, self.world = group, rank, world
        m, l, n = da.rows(), da.cols(), db.cols()
        self.l = l
        depth, leaves, *_ = fast_plan(m, l, n, n_min)
        if depth == 0:
            raise ValueError("leaf sharding needs a recursion (depth >= 1)")
        self.up = choose_split(depth, world)
        units = 7 ** (depth - self.up)
        self.units = even_ranges(units, world)
        self.shard = self.units[rank]
        um, un = node_dims(m, l, n, n_min, depth - self.up)
        self.rows = even_ranges(um, world)
        self.my_rows = self.rows[rank]
        rw = record_words(dc.m.nlimbs)
        row_w, unit_w = un * rw, um * un * rw
        h = dc._h
        buf = C.c_void_p()
        _raise_rc(h, _L.lib.mpgpu_malloc(h, C.c_size_t(4 * max(1, units * unit_w)), C.byref(buf)))
        self.full_ptr = buf.value
        hb = (C.c_uint8 * 64)()
        _raise_rc(h, _L.lib.mpgpu_ipc_handle(h, C.c_void_p(self.full_ptr), hb))
        handles = [None] * world
        dist.all_gather_object(handles, bytes(hb), group=group)
        self.peers = []
        base = []
        for r_, hnd in enumerate(handles):
            if r_ == rank:
                base.append(self.full_ptr)
                continue
            p = C.c_void_p()
            src = (C.c_uint8 * 64).from_buffer_copy(hnd)
            _raise_rc(h, _L.lib.mpgpu_ipc_open(h, src, C.byref(p)))
            self.peers.append(p.value)
            base.append(p.value)
        tab = [0] * um
        for r_, rr in enumerate(self.rows):
            for row in range(rr.lo, rr.hi):
                tab[row] = base[r_] + 4 * ((self.shard.lo * um + row) * row_w)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.rowtab = torch.tensor(tab, dtype=torch.int64, device=dev)
        self.c_rows = owned_c_rows(m, depth, depth - self.up, self.my_rows.lo, self.my_rows.hi)
        self.mode = (f"row-owned p2p(up={self.up}, units={units}, per_rank={self.shard.per}, "
                     f"unit_rows_per_rank={self.rows[0].per}; exchange fused into the leaf epilogue)")

    def __call__(self):
        import torch
        import torch.distributed as dist
        from .mpmm import Stats, _raise
        st = _L.MpgpuStats()
        h = self.dc._h
        dist.barrier(group=self.group)  # every rank finished reading its buffer (previous step)
        if self.shard.hi > self.shard.lo:
            _raise(h, _L.lib.mpgpu_fast_leaves_rows(h, self.algo, self.n_min, C.byref(self.da.m), C.byref(self.db.m),
                                                    self.up, self.shard.lo, self.shard.hi,
                                                    C.c_void_p(self.rowtab.data_ptr()), C.byref(st)))
        _L.lib.mpgpu_synchronize(h)
        torch.cuda.synchronize()
        dist.barrier(group=self.group)  # every rank's product rows have landed
        torch.cuda.synchronize()
        st2 = _L.MpgpuStats()
        _raise(h, _L.lib.mpgpu_fast_combine_rows(h, self.algo, self.n_min, self.l, self.up,
                                                 C.c_void_p(self.full_ptr), self.my_rows.lo, self.my_rows.hi,
                                                 C.byref(self.dc.m), C.byref(st2)))
        s = Stats.of(st)
        s.postadd_ms += st2.postadd_ms
        s.launches += st2.launches
        s.mul, s.addsub = _count(self.algo, self.da, self.db, self.n_min)
        return s

    def close(self):
        h = self.dc._h
        for p in self.peers:
            _L.lib.mpgpu_ipc_close(h, C.c_void_p(p))
        self.peers = []
        if self.full_ptr:
            _L.lib.mpgpu_free(h, C.c_void_p(self.full_ptr))
            self.full_ptr = None


def _staged(group) -> bool:
    """gloo cannot move CUDA tensors: stage the exchange through host memory (the CPU test of
    the real runners: 2 processes sharing one GPU, gloo over 127.0.0.1)."""
    import torch.distributed as dist
    return dist.get_backend(group) == "gloo"


def all_to_all_rows(recv, send, group):
    import torch.distributed as dist
    if _staged(group):
        r = recv.new_zeros(recv.shape, device="cpu")
        dist.all_to_all_single(r, send.cpu(), group=group)
        recv.copy_(r)
    else:
        dist.all_to_all_single(recv, send, group=group)


def all_gather_rows(out, local, group):
    import torch.distributed as dist
    if _staged(group):
        o = out.new_zeros(out.shape, device="cpu")
        dist.all_gather_into_tensor(o, local.cpu(), group=group)
        out.copy_(o)
    else:
        dist.all_gather_into_tensor(out, local, group=group)


def _streams_join(h):
    """Order the library's stream and torch's current stream (where NCCL collectives are
    enqueued): a no-op when the handle already runs on torch's stream (bench.py sets it)."""
    import torch
    cur = torch.cuda.current_stream()
    if _L.lib.mpgpu_get_stream(h) == cur.cuda_stream:
        return
    _L.lib.mpgpu_synchronize(h)
    cur.synchronize()


def _raise_rc(h, rc):
    from .mpmm import _raise
    _raise(h, rc)


class _RowSharded:
    replicated = False
    mode = "row-shard"

    def __init__(self, algo, param, da, db, dc, rank, world, group=None):
        import torch
        from .mpmm import record_words
        self.algo, self.param, self.da, self.db, self.dc, self.group = int(algo), param, da, db, dc, group
        m, n = da.rows(), db.cols()
        self.shard = even_ranges(m, world)[rank]
        self.words_per_row = n * record_words(dc.m.nlimbs)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.all = torch.zeros(world * self.shard.per * self.words_per_row, dtype=torch.int32, device=dev)
        self.local = self.all.narrow(0, rank * self.shard.per * self.words_per_row,
                                     self.shard.per * self.words_per_row)
        self.mode = f"row-shard(rows_per_rank={self.shard.per})"

    def __call__(self):
        import torch.distributed as dist
        from .mpmm import Stats, _raise
        st = _L.MpgpuStats()
        h = self.dc._h
        rows = self.shard.hi - self.shard.lo
        if rows > 0:
            av, cv = _L.MpgpuMat(), _L.MpgpuMat()
            _L.lib.mpgpu_matrix_view(C.byref(self.da.m), self.shard.lo, 0, rows, self.da.cols(), C.byref(av))
            # C rows land directly in this rank's slot of the gather buffer
            cv.rows, cv.cols, cv.prec, cv.nlimbs = rows, self.db.cols(), self.dc.m.prec, self.dc.m.nlimbs
            cv.rec, cv.ld, cv.owned = self.local.data_ptr(), self.db.cols(), 0
            _raise(h, _L.lib.mpgpu_gemm(h, self.algo, self.param, C.byref(av), C.byref(self.db.m), C.byref(cv),
                                        C.byref(st)))
        _streams_join(h)
        all_gather_rows(self.all, self.local.clone(), self.group)
        _streams_join(h)
        # assemble C (rows beyond m are padding)
        nbytes = self.dc.rows() * self.words_per_row * 4
        _cuda_copy(h, self.dc.data_ptr, self.all.data_ptr(), nbytes)
        s = Stats.of(st)
        s.mul, s.addsub = _count(self.algo, self.da, self.db, self.param)
        return s


def _count(algo, da, db, param):
    out = (C.c_uint64 * 2)()
    _L.lib.mpgpu_count_fast(int(algo), da.rows(), da.cols(), db.cols(), max(1, param), out)
    return int(out[0]), int(out[1])


def _cuda_copy(h, dst: int, src: int, nbytes: int):
    from .mpmm import _raise
    _raise(h, _L.lib.mpgpu_copy_device(h, C.c_void_p(dst), C.c_void_p(src), C.c_size_t(nbytes)))


def make_runner(algo, param, da, db, dc, rank: int, world: int, mode: str = "auto", group=None):
    """mode: 'auto' (fast algorithms: leaf shards whose leaf epilogue stores the product rows
    into their owners' buffers over peer memory (CUDA IPC), then the row-owned combine;
    simple/block: row shards), 'a2a' (the same split with an NCCL all-to-all of the row slices
    instead of the fused stores), 'gather' (leaf shards, all-gather of the unit products and a
    replicated combine -- C complete on every rank), 'replicas' (independent copies, weak)."""
    from .mpmm import Algorithm
    if world <= 1 or mode == "replicas":
        return _Replica(algo, param, da, db, dc)
    if Algorithm(algo) in (Algorithm.strassen, Algorithm.winograd):
        depth, *_ = fast_plan(da.rows(), da.cols(), db.cols(), param)
        if depth >= 1:
            if mode == "gather":
                return _FastSharded(algo, param, da, db, dc, rank, world, group)
            if mode == "a2a" or dc.m.nlimbs > 32:
                return _FastRowOwned(algo, param, da, db, dc, rank, world, group)
            return _FastRowOwnedP2P(algo, param, da, db, dc, rank, world, group)
        return _Replica(algo, param, da, db, dc)
    return _RowSharded(algo, param, da, db, dc, rank, world, group)
