#!/usr/bin/env python
"""Stall samples and executed instructions aggregated by CUDA source line (ncu source page,
--print-source cuda,sass). python tools/ncu_lines.py report.ncu-rep kernel_regex [top]"""
import csv
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur_file, agg, hdr = None, {}, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        si = hdr.index("Warp Stall Sampling (All Samples)")
        ei = hdr.index("Instructions Executed")
        s, e = float(r[si] or 0), float(r[ei] or 0)
    except (ValueError, IndexError):
        continue
    k = (cur_file, int(r[0]))
    a = agg.setdefault(k, [0.0, 0.0, r[1].strip()[:70]])
    a[0] += s
    a[1] += e
ts = sum(v[0] for v in agg.values()) or 1
te = sum(v[1] for v in agg.values()) or 1
print(f"total samples {ts:.0f}, warp instructions {te:.0f}")
for (f, l), (s, e, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100 * s / ts:5.1f}% smp {100 * e / te:5.1f}% ins  {f}:{l:<4d} {src}")
