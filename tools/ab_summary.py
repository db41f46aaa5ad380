#!/usr/bin/env python
"""Summarise gpurun_out/ab.log (tools/gpu_ab.sh): per library, bench value/map phase and the c3
scenario-A step times.  usage: python tools/ab_summary.py [log]"""
import collections
import json
import re
import sys

cur = None
res = collections.defaultdict(lambda: collections.defaultdict(list))
for line in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ab.log"):
    line = line.strip()
    if line.startswith("=="):
        cur = line[3:]
        continue
    if not line.startswith("{"):
        continue
    try:
        r = json.loads(re.sub(r" \(\d+ s\)$", "", line))
    except ValueError:
        continue
    if "metric" in r:
        res[cur]["f64 MLUPS"].append(r["value"])
        res[cur]["f64 map ms"].append(r["phases_ms"]["map"])
        if "f32" in r:
            res[cur]["f32 MLUPS"].append(r["f32"]["value"])
    elif "op" in r:
        res[cur][f"{r['op']} {r['scen']} {r['var']} {r.get('mapping', 'R1')} ms"].append(r["ms_per_step"])
keys = sorted({k for v in res.values() for k in v})
libs = list(res)
print("| | " + " | ".join(libs) + " |")
print("|---" * (len(libs) + 1) + "|")
for k in keys:
    print(f"| {k} | " + " | ".join(
        "/".join(f"{x:.4g}" for x in res[l].get(k, [])) for l in libs) + " |")
