#!/usr/bin/env python
"""ncu launch list (gpu__time_duration.sum csv) -> per-kernel table with each kernel's share of
the per-step kernels of the timed steps (the last `steps` collide launches and what ran with
them).  usage: python tools/launch_table.py launches.csv "<cmd>" <timed steps>"""
import collections
import csv
import sys

path, cmd, steps = sys.argv[1], sys.argv[2], int(sys.argv[3])
rows = [r for r in csv.reader(open(path)) if r]
h = None
seq = []
for r in rows:
    if "Kernel Name" in r:
        h = r
        continue
    if not h or len(r) != len(h):
        continue
    d = dict(zip(h, r))
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    k = d["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "")
    v = float(d["Metric Value"]) * {"ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(d["Metric Unit"], 1)
    seq.append((k, v))
# the per-step window: from the first kernel after the (steps)-th last k_write_state/setup, i.e.
# everything after the last `steps` collide launches' preceding remap
coll = [i for i, (k, _) in enumerate(seq) if "k_collide" in k]
start = coll[-steps] if len(coll) >= steps else 0
while start > 0 and ("k_remap" in seq[start - 1][0] or "k_map" in seq[start - 1][0]):
    start -= 1
win = seq[start:]
agg = collections.OrderedDict()
for k, v in win:
    agg.setdefault(k, []).append(v)
tot = sum(v for _, v in win)
print("# ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised: "
      "compare shares)")
print(f"# cmd: {cmd}")
print(f"# window: the last {steps} steps' kernels ({len(win)} launches, {tot:.3f} ms)")
print("# kernel | launches | total ms | mean ms | share of the per-step kernels")
for k, l in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k} | {len(l)} | {sum(l):.3f} | {sum(l) / len(l):.4f} | {100 * sum(l) / tot:.1f}%")
