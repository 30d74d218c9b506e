"""The multi-GPU split on ONE GPU: each rank's share (mpgpu_fast_leaves over its node
range, or a row block of Simple/Block) is computed in turn into the slot an NCCL
all-gather would fill, then combined -- the result must be bit-identical to the
single-call product (no kernels wait on each other; ranks run one after another)."""
import ctypes as C

import numpy as np
import pytest
import torch

from paper_1410_1599_b200 import _lib as L, shard


def _rec_tensor(n_words):
    # torch zero-fills on its own stream while the library writes on the handle's stream:
    # finish the fill (and any pending torch work on a recycled block) before handing it over
    t = torch.zeros(n_words, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    return t


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["strassen", "winograd"])
@pytest.mark.parametrize("m,l,n,bits,n_min", [(64, 64, 64, 256, 8), (45, 37, 51, 128, 5), (33, 29, 40, 512, 4)])
@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("up", [0, 1])
def test_fast_split_bit_exact(P, algo, m, l, n, bits, n_min, world, up):
    ctx = P.PrecisionContext(bits)
    a, b = P.gen_uniform_full(m, l, 3, ctx), P.gen_uniform_full(l, n, 4, ctx)
    want = P.fast_mul(a, b, P.FastMMConfig(P.Algorithm[algo], n_min), ctx).c
    depth, leaves, *_ = shard.fast_plan(m, l, n, n_min)
    if up >= depth:
        pytest.skip("split level above the root")
    da, db = a.to_device(), b.to_device()
    dc = P.DeviceMatrix(m, n, ctx)
    units = 7 ** (depth - up)
    um, un = shard.node_dims(m, l, n, n_min, depth - up)
    words = um * un * P.record_words(dc.m.nlimbs)
    rs = shard.even_ranges(units, world)
    allbuf = _rec_tensor(world * rs[0].per * words)
    h = dc._h
    for r in rs:
        if r.hi > r.lo:
            slot = allbuf.narrow(0, r.lo * words, (r.hi - r.lo) * words)
            assert L.lib.mpgpu_fast_leaves(h, int(P.Algorithm[algo]), n_min, C.byref(da.m), C.byref(db.m), up,
                                           r.lo, r.hi, C.c_void_p(slot.data_ptr()), None) == 0
    assert L.lib.mpgpu_fast_combine(h, int(P.Algorithm[algo]), n_min, l, up, C.c_void_p(allbuf.data_ptr()),
                                    C.byref(dc.m), None) == 0
    assert P.identical(dc.download(), want)


@pytest.mark.gpu
@pytest.mark.parametrize("algo,param", [("simple", 0), ("block", 16)])
def test_row_split_bit_exact(P, algo, param):
    ctx = P.PrecisionContext(256)
    m, l, n = 70, 48, 33
    a, b = P.gen_uniform_full(m, l, 5, ctx), P.gen_uniform_full(l, n, 6, ctx)
    want = P.simple_mul(a, b, ctx) if algo == "simple" else P.block_mul(a, b, param, ctx)
    da, db = a.to_device(), b.to_device()
    dc = P.DeviceMatrix(m, n, ctx)
    h = dc._h
    for r in shard.even_ranges(m, 3):
        rows = r.hi - r.lo
        av, cv = L.MpgpuMat(), L.MpgpuMat()
        assert L.lib.mpgpu_matrix_view(C.byref(da.m), r.lo, 0, rows, l, C.byref(av)) == 0
        assert L.lib.mpgpu_matrix_view(C.byref(dc.m), r.lo, 0, rows, n, C.byref(cv)) == 0
        assert L.lib.mpgpu_gemm(h, int(P.Algorithm[algo]), param, C.byref(av), C.byref(db.m), C.byref(cv), None) == 0
    assert P.identical(dc.download(), want)


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["strassen", "winograd"])
@pytest.mark.parametrize("m,l,n,bits,n_min", [(64, 64, 64, 256, 8), (45, 37, 51, 128, 5), (33, 29, 40, 512, 4)])
@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("up", [0, 1])
def test_row_owned_combine_bit_exact(P, algo, m, l, n, bits, n_min, world, up):
    # every rank's units via mpgpu_fast_leaves, the all-to-all emulated chunk by chunk,
    # mpgpu_fast_combine_rows per rank; the owned rows of all ranks assemble C exactly
    ctx = P.PrecisionContext(bits)
    a, b = P.gen_uniform_full(m, l, 3, ctx), P.gen_uniform_full(l, n, 4, ctx)
    want = P.fast_mul(a, b, P.FastMMConfig(P.Algorithm[algo], n_min), ctx).c
    depth, *_ = shard.fast_plan(m, l, n, n_min)
    if up >= depth:
        pytest.skip("split level above the root")
    da, db = a.to_device(), b.to_device()
    units = 7 ** (depth - up)
    um, un = shard.node_dims(m, l, n, n_min, depth - up)
    L_ = P.nlimbs_for(bits)
    rw = P.record_words(L_)
    us, rows = shard.even_ranges(units, world), shard.even_ranges(um, world)
    h = da._h
    sends = []
    for r in range(world):
        local = _rec_tensor(max(1, us[r].per * um * un * rw))
        if us[r].hi > us[r].lo:
            assert L.lib.mpgpu_fast_leaves(h, int(P.Algorithm[algo]), n_min, C.byref(da.m), C.byref(db.m), up,
                                           us[r].lo, us[r].hi, C.c_void_p(local.data_ptr()), None) == 0
        torch.cuda.synchronize()
        pack, chunk = shard.a2a_pack_plan(us[r], rows, um, un, rw)
        send = _rec_tensor(world * chunk)
        shard.run_plan_torch(pack, send, local)
        sends.append(send)
    out = P.Matrix(m, n, ctx)
    covered = []
    for r in range(world):
        recv = torch.cat([sends[s].narrow(0, r * chunk, chunk) for s in range(world)])
        full = _rec_tensor(units * um * un * rw)
        shard.run_plan_torch(shard.a2a_unpack_plan(us, rows[r], rows[0].per, um, un, rw), full, recv)
        torch.cuda.synchronize()  # torch's stream wrote `full`; the library runs on its own stream
        dc = P.DeviceMatrix(m, n, ctx)
        assert L.lib.mpgpu_fast_combine_rows(h, int(P.Algorithm[algo]), n_min, l, up, C.c_void_p(full.data_ptr()),
                                             rows[r].lo, rows[r].hi, C.byref(dc.m), None) == 0
        part = dc.download()
        own = shard.owned_c_rows(m, depth, depth - up, rows[r].lo, rows[r].hi)
        covered += own
        idx = (np.asarray(own, dtype=np.int64)[:, None] * n + np.arange(n)[None, :]).reshape(-1)
        out.limbs[:, idx] = part.limbs[:, idx]
        out.exp[idx] = part.exp[idx]
        out.sign[idx] = part.sign[idx]
    assert sorted(covered) == list(range(m))
    assert P.identical(out, want)


@pytest.mark.gpu
def test_row_owned_combine_repeat(P):
    # the case that failed once on the driver (Winograd 33x29x40 @512, up=1, world 2), repeated
    for _ in range(50):
        test_row_owned_combine_bit_exact(P, "winograd", 33, 29, 40, 512, 4, 2, 1)
