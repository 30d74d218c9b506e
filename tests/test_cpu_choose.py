"""mpgpu_choose_nmin (host-only): the Strassen / Winograd cutoff chosen per precision from the
measured leaf-GEMM throughput table (north star (2)); no GPU needed."""
import pytest


@pytest.mark.parametrize("bits", [64, 128, 256, 512, 1024, 2048, 8192])
@pytest.mark.parametrize("shape", [(128, 128, 128), (1024, 1024, 1024), (1001, 777, 1537), (4096, 4096, 4096),
                                   (3, 5, 7), (1, 9, 9)])
def test_choice_realises_its_depth(P, bits, shape):
    m, l, n = shape
    nm, d, ms = P.choose_n_min(P.Algorithm.winograd, bits, m, l, n)
    assert nm >= 1 and ms >= 0
    plan = P.recursion_plan(m, l, n, P.FastMMConfig(P.Algorithm.winograd, nm))
    assert len(plan) - 1 == d  # the cutoff gives exactly the modelled depth


def test_deeper_at_higher_precision(P):
    # the leaf's cost per madd grows ~L^2 while the additions grow ~L: more bits, more levels
    depths = [P.choose_n_min(P.Algorithm.winograd, b, 1024, 1024, 1024)[1] for b in (128, 256, 1024)]
    assert depths == sorted(depths) and depths[-1] >= 4
    assert P.choose_n_min(P.Algorithm.strassen, 256, 1024, 1024, 1024)[1] >= 3


def test_choice_errors(P):
    with pytest.raises(P.DomainError):
        P.choose_n_min(P.Algorithm.block, 256, 8, 8, 8)
    with pytest.raises(P.DimensionError):
        P.choose_n_min(P.Algorithm.winograd, 256, 0, 8, 8)
