"""Full-size parity fixtures: SHA-256 of the COMPILED REFERENCE's outputs (oracle/_ref, the
unmodified /root/reference headers over system MPFR) at BASELINE sizes, for the fast
algorithms whose operation DAG (fastmm.hpp:133-219) is otherwise pinned bit for bit only on
small shapes.  The GPU tests (tests/test_gpu_fullsize_hash.py) regenerate the same inputs
with the product's generators (the same Prng64 streams) and compare hashes.  Run in the build
container (the reference is absent on the GPU box), ~3 minutes on 8 cores:

    python tests/golden/make_fullsize_hashes.py
"""
from __future__ import annotations

import hashlib
import json
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))

# name, algo, n_min, (m, l, n), bits, generator kind (0 full-mantissa uniform, 1 config-3 scaled), seeds
CASES = [
    ("cfg2_winograd", "winograd", 64, (1024, 1024, 1024), 256, 0, (1, 2)),
    ("cfg2_strassen", "strassen", 64, (1024, 1024, 1024), 256, 0, (1, 2)),
    ("cfg3_winograd_nmin32", "winograd", 32, (1001, 777, 1537), 512, 1, (1, 2)),
    ("cfg3_winograd_nmin64", "winograd", 64, (1001, 777, 1537), 512, 1, (1, 2)),
    ("depth3_winograd_1024bit", "winograd", 64, (512, 512, 512), 1024, 0, (1, 2)),
]
LU_CASES = [
    # name, n, K, kernel, n_min, bits, seed  (pivot-free: the reference's lu_blocked)
    ("lu512_winograd_K64", 512, 64, "winograd", 32, 256, 11),
]


def soa_hash(x) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(x.limbs, np.uint32).tobytes())
    h.update(np.ascontiguousarray(x.exp, np.int32).tobytes())
    h.update(np.ascontiguousarray(x.sign, np.uint8).tobytes())
    return h.hexdigest()


def run_gemm(case):
    from oracle import oracle as O
    name, algo, n_min, (m, l, n), bits, kind, (sa, sb) = case
    a = O.gen_full(kind, m, l, sa, bits)
    b = O.gen_full(kind, l, n, sb, bits)
    t0 = time.time()
    c, ops = O.gemm(algo, n_min, a, b, which="ref")
    return {"name": name, "kind": "gemm", "algo": algo, "n_min": n_min, "shape": [m, l, n], "bits": bits,
            "gen": kind, "seeds": [sa, sb], "ops": list(ops), "sha256": soa_hash(c),
            "ref_seconds": time.time() - t0}


def run_lu(case):
    from oracle import oracle as O
    name, n, K, kernel, n_min, bits, seed = case
    a = O.gen_full(0, n, n, seed, bits)
    t0 = time.time()
    f, _, ops = O.lu_blocked(a, K, kernel, n_min, which="ref")
    return {"name": name, "kind": "lu", "n": n, "K": K, "kernel": kernel, "n_min": n_min, "bits": bits,
            "seed": seed, "ops": list(ops), "sha256": soa_hash(f), "ref_seconds": time.time() - t0}


def main():
    with ProcessPoolExecutor(max_workers=len(CASES) + len(LU_CASES)) as ex:
        futs = [ex.submit(run_gemm, c) for c in CASES] + [ex.submit(run_lu, c) for c in LU_CASES]
        out = [f.result() for f in futs]
    (HERE / "fullsize_hashes.json").write_text(json.dumps(out, indent=1) + "\n")
    for r in out:
        print(r["name"], r["sha256"][:16], f"{r['ref_seconds']:.0f}s")


if __name__ == "__main__":
    main()
