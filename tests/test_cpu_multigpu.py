"""Host-side logic of the multi-GPU split (paper_1410_1599_b200/shard.py) on CPU:
partition coverage / balance, the group-vs-leaf split choice, and the all-gather
slot layout exercised by a real world_size-2 gloo process group."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1410_1599_b200 import shard


@pytest.mark.parametrize("units", [1, 7, 49, 343, 2401, 1000, 16807])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_even_ranges_cover_each_unit_once_in_slot_order(units, world):
    rs = shard.even_ranges(units, world)
    assert len(rs) == world
    seen = []
    for r, s in enumerate(rs):
        assert s.per == rs[0].per
        assert s.lo == min(r * s.per, units)  # unit u sits at gathered slot u
        seen += list(range(s.lo, s.hi))
    assert seen == list(range(units))
    assert max(s.hi - s.lo for s in rs) - min(s.hi - s.lo for s in rs if s.hi > s.lo) <= rs[0].per


def test_choose_split():
    # cfg2 (depth 4): 343 groups spread evenly over 2/4/8 ranks -> exchange groups
    assert all(shard.choose_split(4, w) == 1 for w in (2, 4, 8))
    # cfg4 (depth 3): 49 groups over 8 ranks is 14 % imbalanced -> exchange leaves
    assert shard.choose_split(3, 8) == 0
    assert shard.choose_split(1, 8) == 0


def test_fast_plan_and_node_dims():
    assert shard.fast_plan(1024, 1024, 1024, 64) == (4, 2401, 64, 64, 64)
    assert shard.fast_plan(4096, 4096, 4096, 512) == (3, 343, 512, 512, 512)
    assert shard.fast_plan(1001, 777, 1537, 32) == (5, 16807, 32, 25, 49)
    assert shard.node_dims(1001, 777, 1537, 32, 4) == (63, 97)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, units, words, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s = shard.even_ranges(units, world)[rank]
    local = torch.zeros(s.per * words, dtype=torch.int32)
    for u in range(s.lo, s.hi):  # "unit product" u = its index pattern
        local[(u - s.lo) * words:(u - s.lo + 1) * words] = torch.arange(words, dtype=torch.int32) + 1000 * u
    parts = [torch.zeros_like(local) for _ in range(world)]
    dist.all_gather(parts, local)
    gathered = torch.cat(parts)
    ok = all(torch.equal(gathered[u * words:(u + 1) * words], torch.arange(words, dtype=torch.int32) + 1000 * u)
             for u in range(units))
    q.put((rank, ok))
    dist.destroy_process_group()


@pytest.mark.parametrize("units", [49, 343])
def test_gloo_world2_gather_layout(units):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, units, 5, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = dict(q.get(timeout=10) for _ in range(2))
    assert res == {0: True, 1: True}


@pytest.mark.parametrize("m,l,n,n_min,up", [(1024, 1024, 1024, 64, 1), (1001, 777, 1537, 32, 1), (45, 37, 51, 5, 0),
                                            (33, 29, 40, 4, 1), (100, 100, 100, 1, 0)])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_owned_rows_partition_c(m, l, n, n_min, up, world):
    depth, *_ = shard.fast_plan(m, l, n, n_min)
    if up >= depth:
        pytest.skip("split level above the root")
    um, _ = shard.node_dims(m, l, n, n_min, depth - up)
    seen = []
    for rr in shard.even_ranges(um, world):
        seen += shard.owned_c_rows(m, depth, depth - up, rr.lo, rr.hi)
    assert sorted(seen) == list(range(m))  # every row of C owned by exactly one rank


def _a2a_worker(rank, world, port, units, um, un, rw, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    us = shard.even_ranges(units, world)
    rows = shard.even_ranges(um, world)
    me = us[rank]
    unit_w = um * un * rw
    local = torch.zeros(max(1, me.per * unit_w), dtype=torch.int32)
    for u in range(me.lo, me.hi):  # word w of unit u = 100000 u + w
        local[(u - me.lo) * unit_w:(u - me.lo + 1) * unit_w] = torch.arange(unit_w, dtype=torch.int32) + 100000 * u
    pack, chunk = shard.a2a_pack_plan(me, rows, um, un, rw)
    send = torch.zeros(world * chunk, dtype=torch.int32)
    shard.run_plan_torch(pack, send, local)
    recv = torch.zeros_like(send)
    dist.all_to_all_single(recv, send)
    full = torch.full((units * unit_w,), -1, dtype=torch.int32)
    shard.run_plan_torch(shard.a2a_unpack_plan(us, rows[rank], rows[0].per, um, un, rw), full, recv)
    # my rows of every unit hold the owner's words; the rest is untouched
    ok = True
    mr = rows[rank]
    for u in range(units):
        for r in range(um):
            seg = full[u * unit_w + r * un * rw:u * unit_w + (r + 1) * un * rw]
            want = torch.arange(r * un * rw, (r + 1) * un * rw, dtype=torch.int32) + 100000 * u
            ok &= bool(torch.equal(seg, want)) if mr.lo <= r < mr.hi else bool((seg == -1).all())
    q.put((rank, ok))
    dist.destroy_process_group()


@pytest.mark.parametrize("units,um", [(7, 5), (49, 8), (3, 1)])
def test_gloo_world2_all_to_all_row_slices(units, um):
    world, un, rw = 2, 3, 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_a2a_worker, args=(r, world, port, units, um, un, rw, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}


def test_bench_e2e_owned_row_runs():
    """bench.py's N > 1 e2e leg reads back each rank's own rows of C as contiguous runs."""
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    import bench

    class RowOwned:
        replicated = False
        c_rows = [0, 1, 2, 5, 6, 9]

    class Replica:
        replicated = True

    class Gather:
        replicated = False

    assert bench.owned_row_runs(RowOwned(), 10, 0, 2) == [(0, 3), (5, 7), (9, 10)]
    assert bench.owned_row_runs(Replica(), 10, 1, 2) == [(0, 10)]
    assert bench.owned_row_runs(Gather(), 10, 1, 2) == [(5, 10)]
    assert bench.owned_row_runs(Gather(), 10, 0, 2) == [(0, 5)]
