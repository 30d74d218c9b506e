"""Measure the leaf-GEMM throughput per precision and leaf size, and the pre/post-addition
cost per record byte, on the B200 -- the table behind mpgpu_choose_nmin (the recursion depth
chosen per precision from measured leaf throughput, BASELINE.json north star (2)).

For each limb count L and leaf edge s, one Winograd product of n = s * 2^d with n_min = s
(7^d leaves of s^3, d chosen so the batch fills the GPU); stats give the leaf kernel time and
the pre / post-addition times.  Prints one JSON line per point and a C table on stdout's end.

    python tools/leaf_table.py > profiles/r02_leaf_table.jsonl
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import paper_1410_1599_b200 as P  # noqa: E402

BITS = [128, 256, 512, 1024]
SIZES = [16, 32, 64, 128, 256, 512]


def main():
    rows = []
    for bits in BITS:
        ctx = P.PrecisionContext(bits)
        L = P.nlimbs_for(bits)
        rw = 4 * P.record_words(L)
        for s in SIZES:
            # enough leaves to fill 148 SMs many times over, bounded device memory / time
            d = 1
            while 7 ** d * max(1, (s // 16) ** 2) < 4000 and d < 4:
                d += 1
            n = s * 2 ** d
            if n * n * rw * 12 > 40e9 or (bits == 1024 and s * 2 ** d > 4096):
                continue
            a = P.gen_uniform_full(n, n, 1, ctx).to_device()
            b = P.gen_uniform_full(n, n, 2, ctx).to_device()
            c = P.DeviceMatrix(n, n, ctx)
            P.gemm_into(P.Algorithm.winograd, s, a, b, c)
            best = None
            for _ in range(3):
                st = P.gemm_into(P.Algorithm.winograd, s, a, b, c)
                if best is None or st.leaf_ms < best.leaf_ms:
                    best = st
            # record bytes moved by the additions: pre-add writes 7/4 of each parent operand
            # and reads it; post-add reads 7 children products and writes the parent
            pre_bytes = post_bytes = 0
            m_ = n
            for t in range(d):
                nodes = 7 ** t
                pre_bytes += nodes * 2 * (m_ * m_) * rw * (1 + 7 / 4)
                post_bytes += nodes * (m_ * m_) * rw * (1 + 7 / 4)
                m_ //= 2
            row = {"bits": bits, "L": L, "leaf": s, "depth": d, "n": n, "leaves": 7 ** d,
                   "leaf_ms": best.leaf_ms, "leaf_madds": best.leaf_madds,
                   "leaf_madd_per_s": best.leaf_madds / (best.leaf_ms * 1e-3),
                   "preadd_ms": best.preadd_ms, "postadd_ms": best.postadd_ms,
                   "preadd_gbs": pre_bytes / (best.preadd_ms * 1e-3) / 1e9,
                   "postadd_gbs": post_bytes / (best.postadd_ms * 1e-3) / 1e9}
            rows.append(row)
            print(json.dumps(row), flush=True)
            for x in (a, b, c):
                x.free()


if __name__ == "__main__":
    main()
