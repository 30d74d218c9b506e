"""Repeat a product and print every phase timing (device events) and the host wall time."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_1410_1599_b200 as P

def run(name, m, l, n, bits, nmin, gen, reps=4):
    ctx = P.PrecisionContext(bits)
    a, b = gen(m, l, 3, ctx).to_device(), gen(l, n, 4, ctx).to_device()
    c = P.DeviceMatrix(m, n, ctx)
    for _ in range(reps):
        t0 = time.perf_counter()
        st = P.gemm_into(P.Algorithm.winograd, nmin, a, b, c)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
        print(f"{name}: dev {st.device_ms:.2f} leaf {st.leaf_ms:.2f} pre {st.preadd_ms:.2f} post {st.postadd_ms:.2f} "
              f"gap {st.device_ms - st.leaf_ms - st.preadd_ms - st.postadd_ms:.2f} wall {wall:.2f} ms")

run("cfg2", 1024, 1024, 1024, 256, 64, P.gen_uniform_full)
run("cfg3 scaled", 1001, 777, 1537, 512, 64, P.gen_scaled)
run("cfg3 uniform", 1001, 777, 1537, 512, 64, P.gen_uniform_full)
