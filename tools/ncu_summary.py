"""Summarise ncu evidence into profiles/ (run here, on the .ncu-rep / CSV that gpurun
brought back):

    python tools/ncu_summary.py --rep gpurun_out/prof_leaf_v8.ncu-rep \
        --launches gpurun_out/launches_v8.csv --key winograd_1024_256 --out profiles/r01_leaf

Writes <out>_summary.json (per-launch metrics of the captured leaf kernel: duration,
DRAM bytes, pipe utilisation, issue activity, top stall reasons, registers,
occupancy), <out>_launch_shares.json (share of step time per kernel from the
launch list) and updates profiles/r01_leaf_traffic.json[key] = DRAM bytes per launch
(bench.py's roofline.traffic).
"""
import argparse
import collections
import csv
import io
import json
import subprocess
from pathlib import Path

WANT = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.per_cycle_active",
    "sm__warps_active.avg.per_cycle_active",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "smsp__inst_executed.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "sm__cycles_elapsed.avg.per_second",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, vals = rows[0], rows[1], rows[2:]
    return h, units, vals


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--key", required=True)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    h, units, vals = raw(a.rep)
    v = vals[0]
    summ = {"kernel": v[h.index("Kernel Name")], "report": Path(a.rep).name}
    for k in WANT:
        if k in h:
            i = h.index(k)
            summ[k] = {"value": v[i], "unit": units[i]}
    stalls = {}
    for i, name in enumerate(h):
        if name.startswith("smsp__average_warps_issue_stalled_") and name.endswith("_per_issue_active.ratio"):
            try:
                stalls[name.split("stalled_")[1].replace("_per_issue_active.ratio", "")] = float(v[i])
            except ValueError:
                pass
    summ["stalls_per_issue_top"] = dict(sorted(stalls.items(), key=lambda x: -x[1])[:8])
    rd = float(v[h.index("dram__bytes_read.sum")])
    wr = float(v[h.index("dram__bytes_write.sum")])
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd *= scale.get(units[h.index("dram__bytes_read.sum")], 1)
    wr *= scale.get(units[h.index("dram__bytes_write.sum")], 1)
    summ["dram_bytes_per_launch"] = rd + wr
    try:  # HBM bandwidth of the launch (the leaf is compute-bound: far below the peak)
        t = float(v[h.index("gpu__time_duration.sum")])
        t *= {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0}.get(
            units[h.index("gpu__time_duration.sum")], 1e-3)
        summ["dram_gbs"] = (rd + wr) / t / 1e9
    except (ValueError, IndexError):
        pass
    Path(a.out + "_summary.json").write_text(json.dumps(summ, indent=1))
    tfile = Path(a.out).parent / "r01_leaf_traffic.json"
    t = json.loads(tfile.read_text()) if tfile.exists() else {}
    t[a.key] = rd + wr
    tfile.write_text(json.dumps(t, indent=1))
    if a.launches:
        rows = list(csv.reader(open(a.launches)))
        hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
        hh = rows[hi]
        ki, vi = hh.index("Kernel Name"), hh.index("Metric Value")
        agg = collections.OrderedDict()
        for r in rows[hi + 1:]:
            if len(r) <= vi:
                continue
            name = r[ki].split("(")[0]
            val = float(r[vi].replace(",", ""))
            agg.setdefault(name, [0, 0.0])
            agg[name][0] += 1
            agg[name][1] += val
        tot = sum(x[1] for x in agg.values())
        shares = {k: {"launches": c, "ns": s, "share": s / tot} for k, (c, s) in
                  sorted(agg.items(), key=lambda x: -x[1][1])}
        Path(a.out + "_launch_shares.json").write_text(json.dumps(shares, indent=1))
    print(json.dumps(summ, indent=1)[:1500])


if __name__ == "__main__":
    main()
