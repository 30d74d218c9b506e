"""Dynamic SASS profile from an ncu source-page CSV (ncu -i REP --page source --csv
--print-source sass): per-opcode instruction counts per warp-madd and the hottest
straight-line blocks.

    python tools/sass_hot.py SRC.csv MADDS [--blocks N]
"""
import argparse
import collections
import csv
import re


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("madds", type=float, help="multiply-adds in the captured launch")
    ap.add_argument("--blocks", type=int, default=0)
    ap.add_argument("--dump", default=None, help="write address/count/stall/source lines here")
    a = ap.parse_args()
    rows = list(csv.reader(open(a.csv)))
    hdr = rows[1]
    ix = hdr.index("Instructions Executed")
    isamp = hdr.index("Warp Stall Sampling (All Samples)")
    body = [r for r in rows[2:] if len(r) > ix and r[0].startswith("0x")]
    wm = a.madds / 32.0
    mix = collections.Counter()
    tot = 0
    for r in body:
        n = int(r[ix] or 0)
        op = re.sub(r"^@!?U?P\w+\s+", "", r[1].strip()).split(" ")[0]
        mix[op] += n
        tot += n
    print(f"total warp instr {tot} per warp-madd: {tot / wm:.2f}")
    for op, n in mix.most_common(45):
        print(f"{op:34s} {n:14d} {n / wm:8.2f}")
    if a.dump:
        with open(a.dump, "w") as f:
            for r in body:
                f.write(f"{r[0][-5:]} {int(r[ix] or 0) / wm:8.3f} {r[isamp]:>6s}  {r[1].strip()}\n")


if __name__ == "__main__":
    main()
