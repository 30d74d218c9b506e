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
