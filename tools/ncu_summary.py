#!/usr/bin/env python
"""Summarise ncu outputs for profiles/:
  ncu_summary.py launches <launches.csv>      per-kernel launch count / time share
  ncu_summary.py full <report.ncu-rep>        key metrics of each captured launch
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def launches(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    rows = list(csv.DictReader(lines))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        short = "rs::StepKernel" + name.split("StepKernel")[1][:3] if "StepKernel" in name else name[:70]
        scale = 1e-3 if r["Metric Unit"] == "ns" else (1.0 if r["Metric Unit"] == "us" else 1e3)
        agg[short][0] += 1
        agg[short][1] += float(r["Metric Value"].replace(",", "")) * scale
    total = sum(v[1] for v in agg.values())
    print(f"{'kernel':72s} {'launches':>8s} {'total_us':>12s} {'share':>7s}")
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:72s} {n:8d} {us:12.1f} {100 * us / total:6.1f}%")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    want = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
            "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__occupancy_limit_registers"]
    for r in rows[2:]:
        d = {w: (r[hdr.index(w)], units[hdr.index(w)]) for w in want if w in hdr}
        t_us = float(d["gpu__time_duration.sum"][0]) * (1e-3 if d["gpu__time_duration.sum"][1] == "ns" else 1)
        gb = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            v, u = d[m]
            gb += float(v) * {"Gbyte": 1.0, "Mbyte": 1e-3, "Kbyte": 1e-6, "byte": 1e-9}.get(u, 1.0)
        print("; ".join(f"{k}={v[0]} {v[1]}".strip() for k, v in d.items()),
              f"; traffic={gb:.4f} GB; dram_GBps={gb / (t_us * 1e-6):.1f}")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
