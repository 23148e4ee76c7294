#!/usr/bin/env python
"""Summarise a warm, back-to-back ncu capture of the hot kernel into
profiles/dram_traffic.json (read by bench.py for roofline.traffic).

The capture (on the GPU box, after the same bench command exited 0 without ncu):

    ncu --cache-control none --clock-control none \
        --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        -k regex:<kernel> -s <skip> -c <count> --csv --log-file <csv> python bench.py ...

--cache-control none keeps L2 across launches (no flush before each kernel),
and three metrics fit one pass, so every launch is profiled once, warm, in the
middle of the timed loop: the dirty residual lines a launch leaves in L2 are
written back during the next one, as in the real back-to-back loop -- unlike
the default cold replay, which flushes L2 before the kernel and never sees its
deferred write-backs (round-1 VERDICT, "What's weak" #3).

    python tools/ncu_traffic.py <csv> <key> [--rho R] [--ranks N]

<key> is "<workload>/n<world>/<accum>/<fused|split>" as bench.py looks it up;
--ranks divides a loopback group kernel's traffic (all ranks of one GPU) by N.
"""
import argparse
import csv
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def parse(path):
    rows = {}
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for rec in csv.DictReader(lines):
        key = (rec["ID"], rec["Kernel Name"])
        val = float(rec["Metric Value"].replace(",", ""))
        unit = rec.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
                 "msecond": 1e6}.get(unit, 1)
        rows.setdefault(key, {})[rec["Metric Name"]] = val * scale
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("key")
    ap.add_argument("--rho", type=float, default=0.01)
    ap.add_argument("--ranks", type=int, default=1)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "dram_traffic.json"))
    a = ap.parse_args()
    rows = parse(a.csv)
    if not rows:
        sys.exit("no kernel rows in " + a.csv)
    rd = [r["dram__bytes_read.sum"] for r in rows.values()]
    wr = [r["dram__bytes_write.sum"] for r in rows.values()]
    ns = [r["gpu__time_duration.sum"] for r in rows.values()]
    names = sorted({k[1] for k in rows})
    tot = [(x + y) / a.ranks for x, y in zip(rd, wr)]
    entry = {"dram_bytes_per_launch": statistics.median(tot),
             "dram_read_per_launch": statistics.median(rd) / a.ranks,
             "dram_write_per_launch": statistics.median(wr) / a.ranks,
             "launches": len(tot), "min": min(tot), "max": max(tot),
             "duration_us_median": statistics.median(ns) / 1e3,
             "kernel": names, "rho_target": a.rho, "ranks_in_kernel": a.ranks,
             "source": f"ncu --cache-control none (warm, back-to-back, one pass) of {len(tot)} launches: "
                       f"{os.path.basename(a.csv)}"}
    data = {}
    if os.path.exists(a.out):
        with open(a.out) as f:
            data = json.load(f)
    data[a.key] = entry
    with open(a.out, "w") as f:
        json.dump(data, f, indent=1, sort_keys=True)
    print(json.dumps({a.key: entry}))


if __name__ == "__main__":
    main()
