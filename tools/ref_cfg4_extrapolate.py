"""CPU baseline of BASELINE config 4 (n=4096 @1024 bits, Winograd depth 3) by extrapolation
(SURVEY.md 8(d)): the compiled reference (oracle/_ref) on ONE core at n = 512 and n = 1024 with
the SAME depth (n_min 64 and 128), same input distribution; the n = 4096 time is extrapolated by
the ratio of count_fast operation counts (opmodel.hpp:30-44) from the n = 1024 run (the larger
leaves' cache behaviour is closer to n = 4096's).  Runs on the box host, no GPU:

    python tools/ref_cfg4_extrapolate.py > profiles/r02_ref_cfg4_extrapolated.json
"""
import json
import os
import subprocess
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from oracle import oracle as O  # noqa: E402


def main():
    bits = 1024
    rows = []
    for n, nmin in ((512, 64), (1024, 128)):
        a = O.gen_full(0, n, n, 1, bits)
        b = O.gen_full(0, n, n, 2, bits)
        t0 = time.time()
        _, ops = O.gemm("winograd", nmin, a, b, which="ref")
        dt = time.time() - t0
        rows.append({"n": n, "n_min": nmin, "seconds": dt, "mul": ops[0], "addsub": ops[1],
                     "madd_per_s": n ** 3 / dt})
    full = O.count_fast("winograd", 4096, 4096, 4096, 512)
    base = rows[-1]
    scale = (full[0] + full[1]) / (base["mul"] + base["addsub"])
    model = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
    cpu = next((ln.split(":", 1)[1].strip() for ln in model.splitlines() if ln.lower().startswith("model name")), None)
    print(json.dumps({"what": "compiled reference (oracle/_ref), 1 core, Winograd depth 3 @1024 bits, full-mantissa "
                              "uniform inputs; n=4096 extrapolated from n=1024 by count_fast (mul+addsub) ratio",
                      "measured": rows, "ops_4096": {"mul": full[0], "addsub": full[1]}, "scale_from_1024": scale,
                      "extrapolated_seconds_4096": base["seconds"] * scale,
                      "extrapolated_madd_per_s_4096": 4096 ** 3 / (base["seconds"] * scale),
                      "cpu_model": cpu, "nproc": os.cpu_count()}))


if __name__ == "__main__":
    main()
