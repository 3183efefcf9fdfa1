#!/usr/bin/env python
"""Top SASS instructions by a given stall reason from an ncu report (source page).
    python tools/ncu_stalls.py report.ncu-rep kernel_regex [reason ...]"""
import csv
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
reasons = sys.argv[3:] or ["stall_long_sb", "stall_wait", "stall_barrier", "stall_short_sb"]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
body = [r for r in rows[2:] if r and r[0].startswith('0x')]
for rs in reasons:
    ci = h.index(rs)
    tot = sum(float(r[ci] or 0) for r in body if len(r) > ci)
    print(f"== {rs}: {tot:.0f} samples")
    top = sorted(((float(r[ci] or 0), i, r[1].strip()) for i, r in enumerate(body) if len(r) > ci), reverse=True)[:12]
    for v, i, ins in top:
        ctx = " | ".join(x[1].strip()[:40] for x in body[max(0, i - 3):i])
        print(f"  {v:6.0f} #{i:5d} {ins[:60]:60s}  <- {ctx}")
