#!/usr/bin/env python
"""Per-source-line instruction/stall summary of an ncu report (needs -lineinfo + --import-source).
usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
lines = []
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] not in ("", "File Path", "Function Name"):
        d = dict(zip(hdr[2:], r[2:]))
        try:
            lines.append((int(r[0]), r[1][:90], float(d.get("Instructions Executed") or 0),
                          float(d.get("Warp Stall Sampling (All Samples)") or 0)))
        except ValueError:
            pass
ti = sum(x[2] for x in lines) or 1
ts = sum(x[3] for x in lines) or 1
print(f"total warp-inst {ti:.3e}  stall samples {ts:.0f}")
for ln, src, ie, st in sorted(lines, key=lambda x: -x[3])[:top]:
    print(f"{ln:5d} {100*ie/ti:5.1f}% inst {100*st/ts:5.1f}% stall  {src}")
