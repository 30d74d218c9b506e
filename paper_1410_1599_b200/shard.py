"""Multi-GPU execution of one MP GEMM step (one process per GPU).

Round-1 state: replicas -- every rank runs the full product on its own copy of the
inputs (weak scaling: per-GPU work fixed as N grows).  The leaf-sharded Winograd
(7^d leaves split over ranks, post-additions after an exchange of level-(d-1)
products) is described in DESIGN.md "Multi-GPU" and lands in a later round.
"""
from __future__ import annotations


class _Replica:
    replicated = True

    def __init__(self, algo, param, da, db, dc):
        self.algo, self.param, self.da, self.db, self.dc = algo, param, da, db, dc

    def __call__(self):
        from .mpmm import gemm_into
        return gemm_into(self.algo, self.param, self.da, self.db, self.dc)


def make_runner(algo, param, da, db, dc, rank: int, world: int):
    return _Replica(algo, param, da, db, dc)
