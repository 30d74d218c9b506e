"""The C-ABI multi-GPU path (mpgpu_group_*, csrc/group.cu): one process driving several
devices.  On a one-GPU host the group repeats device 0 (several shards of one GPU), which
runs the same code -- per-device threads, the peer-copy pull of unit-product row slices,
the row-owned combine, strided host writes -- and must be bit-identical to the one-device
product; with more GPUs present the real devices are used as well."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _host(P, m, n, ctx):
    return P.Matrix(m, n, ctx)


@pytest.mark.parametrize("algo,param", [("simple", 0), ("block", 16), ("strassen", 8), ("winograd", 8),
                                        ("winograd", 5)])
@pytest.mark.parametrize("shards", [1, 2, 3, 8])
@pytest.mark.parametrize("m,l,n,bits", [(64, 64, 64, 256), (45, 37, 51, 128), (33, 29, 40, 512)])
def test_group_gemm_bit_exact(P, algo, param, shards, m, l, n, bits):
    ctx = P.PrecisionContext(bits)
    a, b = P.gen_uniform_full(m, l, 3, ctx), P.gen_uniform_full(l, n, 4, ctx)
    want = P.Matrix(m, n, ctx)
    P.gemm_host(P.Algorithm[algo], param, a, b, want, ctx)
    g = P.DeviceGroup([0] * shards)
    got = P.Matrix(m, n, ctx)
    st = g.gemm_host(P.Algorithm[algo], param, a, b, got, ctx)
    assert P.identical(got, want)
    ops = P.count_fast(P.Algorithm[algo], m, l, n, max(1, param)) if algo in ("strassen", "winograd") else None
    if ops is not None:
        assert (st.mul, st.addsub) == (ops.mul, ops.addsub)
    g.close()


def test_group_real_devices(P):
    ndev = torch.cuda.device_count()
    ctx = P.PrecisionContext(256)
    a, b = P.gen_uniform_full(96, 80, 5, ctx), P.gen_uniform_full(80, 72, 6, ctx)
    want = P.Matrix(96, 72, ctx)
    P.gemm_host(P.Algorithm.winograd, 8, a, b, want, ctx)
    g = P.DeviceGroup.from_mask((1 << ndev) - 1)
    assert g.size() == ndev
    got = P.Matrix(96, 72, ctx)
    g.gemm_host(P.Algorithm.winograd, 8, a, b, got, ctx)
    assert P.identical(got, want)


def test_group_errors(P):
    ctx = P.PrecisionContext(256)
    a, b = P.gen_uniform_full(8, 6, 1, ctx), P.gen_uniform_full(7, 5, 2, ctx)
    g = P.DeviceGroup([0, 0])
    with pytest.raises(P.DimensionError):
        g.gemm_host(P.Algorithm.winograd, 0, a, P.gen_uniform_full(6, 5, 2, ctx), P.Matrix(8, 5, ctx), ctx)
    with pytest.raises(P.DomainError):
        g.gemm_host(9, 4, a, P.gen_uniform_full(6, 5, 2, ctx), P.Matrix(8, 5, ctx), ctx)
    with pytest.raises(P.DeviceError):
        P.DeviceGroup.from_mask(1 << 31)


def test_group_cfg2_shape(P):
    # the bench workload's recursion (depth 4 at n_min 64) on a 4-shard group, bit-exact
    ctx = P.PrecisionContext(256)
    n = 512
    a, b = P.gen_uniform_full(n, n, 1, ctx), P.gen_uniform_full(n, n, 2, ctx)
    want = P.Matrix(n, n, ctx)
    P.gemm_host(P.Algorithm.winograd, 32, a, b, want, ctx)
    got = P.Matrix(n, n, ctx)
    P.DeviceGroup([0, 0, 0, 0]).gemm_host(P.Algorithm.winograd, 32, a, b, got, ctx)
    assert P.identical(got, want)


@pytest.mark.parametrize("pull", ["0", "1"])
def test_group_exchange_variants(P, pull, monkeypatch):
    # fused exchange (epilogue stores rows into their owners' buffers) and the copy-engine pull
    # are the same bits; MPGPU_GROUP_PULL is read once per process, so run each in a subprocess
    import subprocess, sys, textwrap
    code = textwrap.dedent("""
        import sys; sys.path.insert(0, '.')
        import paper_1410_1599_b200 as P
        for bits, (m, l, n), nm in ((256, (96, 80, 72), 8), (1024, (40, 36, 44), 5), (128, (130, 70, 90), 9)):
            ctx = P.PrecisionContext(bits)
            a, b = P.gen_uniform_full(m, l, 3, ctx), P.gen_uniform_full(l, n, 4, ctx)
            for algo in ("strassen", "winograd"):
                want = P.Matrix(m, n, ctx); P.gemm_host(P.Algorithm[algo], nm, a, b, want, ctx)
                for shards in (2, 3, 5):
                    got = P.Matrix(m, n, ctx)
                    P.DeviceGroup([0] * shards).gemm_host(P.Algorithm[algo], nm, a, b, got, ctx)
                    assert P.identical(got, want), (bits, algo, shards)
        print("OK")
    """)
    import os
    env = dict(os.environ, MPGPU_GROUP_PULL=pull)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=600,
                       cwd=str(__import__("pathlib").Path(__file__).resolve().parent.parent))
    assert r.returncode == 0 and "OK" in r.stdout, r.stderr[-3000:]
