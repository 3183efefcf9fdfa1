"""Text summary of one ncu --set full report (for profiles/): duration, DRAM bytes, throughputs,
occupancy, issue activity, the stall-reason PC samples and the SASS instruction mix.

    python tools/ncu_report.py report.ncu-rep [label] > profiles/rNN/ncu_<label>.txt
"""
import collections
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
label = sys.argv[2] if len(sys.argv) > 2 else rep
raw = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                     text=True).stdout.splitlines()))
h = raw[0]
print(f"ncu --set full summary: {label}")
for r in raw[2:]:
    m = dict(zip(h, r))
    print(f"\n== {m.get('Kernel Name', '?')[:110]}")
    for k in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
              "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
              "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
              "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
              "lts__t_bytes.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active",
              "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum"):
        if k in m:
            print(f"  {k:62s} {m[k]}")
    st = sorted(((float(m[k]), k) for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                 and not k.endswith("_not_issued") and m.get(k, "").replace(".", "").isdigit()), reverse=True)
    tot = sum(v for v, _ in st) or 1
    print("  stall PC samples (share): " + ", ".join(f"{k.split('stalled_')[1]} {v / tot:.2f}" for v, k in st[:10]))
src = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                                     capture_output=True, text=True).stdout.splitlines()))
hi = [i for i, r in enumerate(src) if "Source" in r and any("Instructions Executed" in c for c in r)]
if hi:
    hh = src[hi[0]]
    ci, ie = hh.index("Source"), [i for i, c in enumerate(hh) if c.startswith("Instructions Executed")][0]
    ops, tot = collections.Counter(), 0.0
    for r in src[hi[0] + 1:]:
        try:
            n = float(r[ie] or 0)
        except (ValueError, IndexError):
            continue
        mm = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[ci].strip())
        if mm:
            ops[mm.group(2)] += n
            tot += n
    print(f"\n  SASS instruction mix (first kernel of the report, {tot:,.0f} warp-instructions):")
    print("  " + ", ".join(f"{op} {n / tot * 100:.1f}%" for op, n in ops.most_common(16)))
