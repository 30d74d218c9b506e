"""Full-size single-core timing of the compiled reference (oracle/_ref) on the bench's
config-2 workload, beside the bounded sample bench.py's reference arm uses -- states the
sample's bias.  Runs on the GPU box's host (no GPU needed):

    python tools/ref_fullsize.py [--algo winograd] [--n 1024] [--bits 256] [--n-min 64] > out.json
"""
import argparse
import json
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--algo", default="winograd")
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--bits", type=int, default=256)
    ap.add_argument("--n-min", type=int, default=64)
    a = ap.parse_args()
    A = O.gen_full(0, a.n, a.n, 1, a.bits)
    B = O.gen_full(0, a.n, a.n, 2, a.bits)
    s, nmin_s = a.n // 4, max(1, a.n_min // 4)
    idx = (np.arange(s)[:, None] * a.n + np.arange(s)[None, :]).reshape(-1)
    sa = O.OMat(s, s, a.bits, A.limbs[:, idx], A.exp[idx], A.sign[idx])
    sb = O.OMat(s, s, a.bits, B.limbs[:, idx], B.exp[idx], B.sign[idx])
    _, t_sample = O.gemm_replicas(a.algo, nmin_s, sa, sb, 1)
    _, t_full = O.gemm_replicas(a.algo, a.n_min, A, B, 1)
    lscpu = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
    model = next((ln.split(":", 1)[1].strip() for ln in lscpu.splitlines() if ln.lower().startswith("model name")),
                 None)
    print(json.dumps({
        "what": "compiled reference (oracle/_ref), 1 core, same inputs as bench.py",
        "full": {"n": a.n, "bits": a.bits, "algo": a.algo, "n_min": a.n_min, "seconds": t_full,
                 "madd_per_s": a.n ** 3 / t_full},
        "sample": {"n": s, "n_min": nmin_s, "seconds": t_sample, "madd_per_s": s ** 3 / t_sample},
        "sample_over_full_rate": (s ** 3 / t_sample) / (a.n ** 3 / t_full),
        "cpu_model": model, "nproc": __import__("os").cpu_count(), "unix_time": time.time()}))


if __name__ == "__main__":
    main()
