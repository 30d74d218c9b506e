"""Generate tests/golden/*.npz from the COMPILED REFERENCE (oracle/_ref/libmpmm_ref.so,
the unmodified /root/reference headers over system MPFR).  Run in the build
container (the reference is not present on the GPU box):

    python tests/golden/make_golden.py

Each fixture stores the inputs and the reference's outputs in the C-ABI SoA
layout (limbs / exp / sign), so the oracle restatement (CPU tests) and the GPU
path (gpu tests) are both pinned to frozen reference results on inexact,
full-mantissa inputs -- the case the reference's own tests never freeze
("Gap").
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402


def soa(prefix, x, d):
    d[prefix + "_limbs"] = x.limbs
    d[prefix + "_exp"] = x.exp
    d[prefix + "_sign"] = x.sign
    d[prefix + "_shape"] = np.array([x.rows(), x.cols(), x.bits()], np.int64)


def gemm_case(name, alg, param, m, l, n, bits, kind, seed):
    if kind == "full":
        a = O.gen_full(0, m, l, seed, bits)
        b = O.gen_full(0, l, n, seed + 1, bits)
    elif kind == "scaled":
        a = O.gen_full(1, m, l, seed, bits)
        b = O.gen_full(1, l, n, seed + 1, bits)
    else:
        a = O.gen_random(m, l, seed, bits, "ref")
        b = O.gen_random(l, n, seed + 1, bits, "ref")
    c, ops = O.gemm(alg, param, a, b, which="ref")
    d = {"alg": np.array(alg), "param": np.array(param), "ops": np.array(ops, np.uint64)}
    soa("a", a, d)
    soa("b", b, d)
    soa("c", c, d)
    np.savez_compressed(HERE / f"gemm_{name}.npz", **d)


def lu_case(name, n, K, kernel, n_min, bits, seed):
    a = O.gen_full(0, n, n, seed, bits)
    f, _, ops = O.lu_blocked(a, K, kernel, n_min, which="ref")
    ones = O.from_si(np.ones(n, np.int64), bits, n, 1)
    b = O.mat_vec_mul(a, ones, which="ref")
    x = O.lu_solve(f, b, which="ref")
    d = {"K": np.array(K), "kernel": np.array(kernel), "n_min": np.array(n_min), "ops": np.array(ops, np.uint64)}
    soa("a", a, d)
    soa("f", f, d)
    soa("b", b, d)
    soa("x", x, d)
    np.savez_compressed(HERE / f"lu_{name}.npz", **d)


def main():
    gemm_case("simple_128_full", "simple", 0, 32, 32, 32, 128, "full", 11)
    gemm_case("block_256_full_ragged", "block", 12, 37, 41, 29, 256, "full", 21)
    gemm_case("strassen_256_full_odd", "strassen", 8, 45, 37, 51, 256, "full", 31)
    gemm_case("winograd_256_full_odd", "winograd", 8, 45, 37, 51, 256, "full", 41)
    gemm_case("winograd_512_scaled_odd", "winograd", 4, 33, 25, 39, 512, "scaled", 51)
    gemm_case("winograd_1024_full", "winograd", 8, 24, 20, 28, 1024, "full", 61)
    gemm_case("strassen_128_refgen", "strassen", 4, 24, 24, 24, 128, "ref", 71)
    gemm_case("winograd_100_full", "winograd", 6, 30, 26, 22, 100, "full", 81)
    lu_case("winograd_256", 40, 8, "winograd", 4, 256, 91)
    lu_case("block_128", 33, 8, "block", 4, 128, 92)
    print("wrote", sorted(p.name for p in HERE.glob("*.npz")))


if __name__ == "__main__":
    main()
