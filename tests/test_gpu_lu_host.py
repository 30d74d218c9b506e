"""mpgpu_lu_blocked_host: the blocked LU (blocklu.hpp:121-146) of a host matrix with the
PCIe transfers overlapped -- the first K columns are uploaded first, the rest during the
first panel, each block of K rows is copied back once no later interchange can touch it.
The factors (and pivots) must be bit-identical to the device path's."""
import numpy as np
import pytest

CASES = [
    # (n, K, kernel, n_min, bits, pivoting)
    (256, 64, "winograd", 32, 256, True),
    (256, 64, "winograd", 32, 256, False),
    (200, 48, "strassen", 16, 128, True),
    (130, 32, "block", 16, 512, True),
    (97, 40, "simple", 1, 64, True),
    (50, 64, "winograd", 16, 256, True),    # n < K: one panel
    (192, 64, "winograd", 32, 1024, True),
]


def _pinned(P, a):
    import torch
    lim = torch.empty(a.limbs.shape, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    ex = torch.empty(a.exp.shape, dtype=torch.int32, pin_memory=True).numpy()
    sg = torch.empty(a.sign.shape, dtype=torch.uint8, pin_memory=True).numpy()
    lim[:], ex[:], sg[:] = a.limbs, a.exp, a.sign
    return P.Matrix(a.rows(), a.cols(), a.ctx(), lim, ex, sg)


@pytest.mark.gpu
@pytest.mark.parametrize("n,K,kernel,n_min,bits,pivoting", CASES)
def test_lu_host_matches_device_path(P, n, K, kernel, n_min, bits, pivoting):
    ctx = P.PrecisionContext(bits)
    a = P.gen_uniform_full(n, n, 21, ctx)
    cfg = P.BlockLUConfig(K, P.Algorithm[kernel], n_min)
    want = P.lu_blocked(a, cfg, ctx, pivoting=pivoting)
    for host in (_pinned(P, a), a):  # page-locked (pipelined) and pageable (plain sequence)
        got = P.lu_blocked_host(host, cfg, ctx, pivoting=pivoting)
        assert P.identical(got.packed, want.packed), (n, K, kernel, pivoting)
        if pivoting:
            assert np.array_equal(got.piv, want.piv)


@pytest.mark.gpu
def test_lu_host_in_place_and_singular(P):
    ctx = P.PrecisionContext(256)
    a = P.gen_uniform_full(128, 128, 5, ctx)
    cfg = P.BlockLUConfig(32, P.Algorithm.winograd, 16)
    want = P.lu_blocked(a, cfg, ctx, pivoting=True)
    h = _pinned(P, a)
    got = P.lu_blocked_host(h, cfg, ctx, pivoting=True, out=h)  # factored in place
    assert P.identical(h, want.packed) and got.packed is h
    z = P.Matrix(64, 64, ctx)  # all zeros: zero pivot at index 1 without pivoting
    with pytest.raises(P.SingularError):
        P.lu_blocked_host(_pinned(P, z), P.BlockLUConfig(16, P.Algorithm.winograd, 8), ctx)
