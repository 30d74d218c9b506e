"""Worker for tests/test_gpu_shard_procs.py: one rank of a world-size-N run of the REAL
multi-GPU runners (shard.make_runner) on a shared GPU, exchange over gloo (host-staged).
Each rank checks the rows of C it owns against the single-GPU product of the same inputs."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_1410_1599_b200 as P
    from paper_1410_1599_b200 import shard
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    P.set_device(0)
    P.set_stream(torch.cuda.current_stream().cuda_stream)
    out = []
    for algo, param, mode, (m, l, n), bits in [("winograd", 8, "auto", (96, 80, 72), 256),
                                                ("strassen", 5, "auto", (45, 37, 51), 512),
                                                ("winograd", 8, "a2a", (96, 80, 72), 256),
                                                ("strassen", 6, "a2a", (61, 50, 47), 1024),
                                                ("winograd", 8, "gather", (64, 64, 64), 128),
                                                ("block", 16, "auto", (70, 48, 33), 256),
                                                ("simple", 0, "auto", (33, 20, 17), 1024)]:
        ctx = P.PrecisionContext(bits)
        a, b = P.gen_uniform_full(m, l, 3, ctx), P.gen_uniform_full(l, n, 4, ctx)
        da, db = a.to_device(), b.to_device()
        dc, ref = P.DeviceMatrix(m, n, ctx), P.DeviceMatrix(m, n, ctx)
        runner = shard.make_runner(P.Algorithm[algo], param, da, db, dc, rank, world, mode=mode)
        for _ in range(2):  # twice: buffers are reused across steps
            st = runner()
        torch.cuda.synchronize()
        P.gemm_into(P.Algorithm[algo], param, da, db, ref)
        got, want = dc.download(), ref.download()
        own = getattr(runner, "c_rows", None)
        if own is None:
            own = list(range(m))
        idx = (np.asarray(own, dtype=np.int64)[:, None] * n + np.arange(n)[None, :]).reshape(-1)
        bad = int(np.count_nonzero((got.exp[idx] != want.exp[idx]) | (got.sign[idx] != want.sign[idx]) |
                                   np.any(got.limbs[:, idx] != want.limbs[:, idx], axis=0)))
        cnt = P.count_fast(P.Algorithm[algo], m, l, n, max(1, param))
        out.append({"algo": algo, "mode": mode, "runner": runner.__class__.__name__, "rows": len(own), "m": m, "bad": bad,
                    "ops_ok": (st.mul, st.addsub) == (cnt.mul, cnt.addsub)})
        if hasattr(runner, "close"):
            dist.barrier()  # every peer is done with the shared buffers
            runner.close()
        for x in (da, db, dc, ref):
            x.free()
    dist.destroy_process_group()
    print("RESULT " + json.dumps({"rank": rank, "cases": out}), flush=True)


if __name__ == "__main__":
    main()
