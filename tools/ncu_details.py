#!/usr/bin/env python
"""Flatten an ncu --set full report's details page into 'Section | Metric | Value unit' lines
(read here, no GPU needed), with a header line, for profiles/.

usage: python tools/ncu_details.py <report.ncu-rep> "<header comment>" > profiles/rNN_....txt
"""
import csv
import io
import subprocess
import sys

rep, header = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                     text=True, check=True).stdout
rows = list(csv.DictReader(io.StringIO(out)))
print(f"# {header}")
if rows:
    r0 = rows[0]
    print(f"# kernel: {r0['Kernel Name']}  block {r0['Block Size']}  grid {r0['Grid Size']}")
seen = set()
for r in rows:
    if not r.get("Metric Name"):
        continue
    key = (r["Section Name"], r["Metric Name"])
    if key in seen:
        continue
    seen.add(key)
    print(f"{r['Section Name']} | {r['Metric Name']} | {r['Metric Value']} {r['Metric Unit']}".rstrip())
