#!/usr/bin/env python
"""Summarise an ncu --set full report (read here, no GPU needed) into profiles/.

usage: python tools/ncu_summary.py <report.ncu-rep> <workload-key> <cells-per-launch> <bytes-per-cell>
Prints the key counters and merges {"<workload>": {...}} into profiles/ncu_summary.json.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
       "smsp__inst_executed.sum", "sm__inst_executed.avg.pct_of_peak_sustained_elapsed",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        res.append({k: (d.get(k), units[h.index(k)] if k in h else "") for k in RAW + ["Kernel Name"]})
    return res


def to_bytes(v, unit):
    v = float(v)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return v * scale


def to_ms(v, unit):
    v = float(v)
    return v * {"ms": 1, "us": 1e-3, "ns": 1e-6, "s": 1e3}.get(unit, 1)


def main():
    rep, key, cells, bpc = sys.argv[1], sys.argv[2], float(sys.argv[3]), float(sys.argv[4])
    rows = raw(rep)
    r = rows[-1]
    rd = to_bytes(*r["dram__bytes_read.sum"])
    wr = to_bytes(*r["dram__bytes_write.sum"])
    ms = to_ms(*r["gpu__time_duration.sum"])
    alg = cells * bpc
    summ = {
        "kernel": r["Kernel Name"][0],
        "report": os.path.basename(rep),
        "duration_ms_ncu": ms,
        "dram_bytes_per_launch": rd + wr,
        "dram_read": rd, "dram_write": wr,
        "algorithmic_bytes_per_launch": alg,
        "traffic_over_algorithmic": (rd + wr) / alg,
        "dram_gbs_ncu": (rd + wr) / ms / 1e6,
        "registers": r["launch__registers_per_thread"][0],
        "warps_active_pct": r["sm__warps_active.avg.pct_of_peak_sustained_active"][0],
        "issue_pct": r["sm__inst_executed.avg.pct_of_peak_sustained_elapsed"][0],
        "dram_pct_of_ncu_peak": r["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"][0],
        "warp_inst_per_cell": float(r["smsp__inst_executed.sum"][0]) / (cells / 32.0)
        if r["smsp__inst_executed.sum"][0] else None,
    }
    print(json.dumps(summ, indent=1))
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    d = {}
    if os.path.exists(p):
        d = json.load(open(p))
    d[key] = summ
    os.makedirs(os.path.dirname(p), exist_ok=True)
    json.dump(d, open(p, "w"), indent=1)


if __name__ == "__main__":
    main()
