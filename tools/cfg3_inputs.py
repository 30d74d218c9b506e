"""Leaf cost of config 3's scaled inputs vs uniform inputs at the same shape/precision."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1410_1599_b200 as P  # noqa: E402

ctx = P.PrecisionContext(512)
m, l, n = 1001, 777, 1537
for name, gen in (("scaled", P.gen_scaled), ("uniform", P.gen_uniform_full)):
    a, b = gen(m, l, 3, ctx).to_device(), gen(l, n, 4, ctx).to_device()
    c = P.DeviceMatrix(m, n, ctx)
    for _ in range(2):
        st = P.gemm_into(P.Algorithm.winograd, 64, a, b, c)
    print(f"cfg3 {name}: total {st.device_ms:.2f} ms leaf {st.leaf_ms:.2f} ms pre {st.preadd_ms:.2f} post {st.postadd_ms:.2f}")
