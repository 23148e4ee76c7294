#!/usr/bin/env python
"""Per-CUDA-source-line instruction counts and stall samples of one kernel
in an ncu report (--import-source on, -lineinfo builds):

    python tools/ncu_lines.py REPORT.ncu-rep [TOP]
"""
import csv
import io
import subprocess
import sys


def main(path, top=40):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    cur, hdr, agg = None, None, {}
    for r in csv.reader(io.StringIO(raw)):
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name",):
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] == "":
            continue
        try:
            inst, samp = int(r[7] or 0), int(r[6] or 0)
        except ValueError:
            continue
        agg[(cur, int(r[0]))] = (inst, samp, r[1][:90])
    ti = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    print(f"warp instructions {ti}, stall samples {ts}")
    for (f, ln), (i, s_, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{f:20s}{ln:5d} inst {100 * i / ti:5.1f}% samp {100 * s_ / ts:5.1f}%  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
