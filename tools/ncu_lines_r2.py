"""Per-CUDA-source-line instruction and stall-sample shares of one kernel in an ncu report
(--page source --print-source cuda,sass): where a kernel's instructions and stalls come from.
    python tools/ncu_lines_r2.py report.ncu-rep [top]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
fname, cur, ie, ws = "?", None, None, None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        ie, ws = r.index("Instructions Executed"), r.index("Warp Stall Sampling (All Samples)")
        continue
    if ie is None or len(r) <= ie:
        continue
    if r[0].strip():
        cur = (fname, int(r[0]))
        agg[cur][2] = r[1].strip()[:90]
    elif r[2].strip() and r[2] != "..." and cur is not None:
        try:
            agg[cur][0] += float(r[ie] or 0)
            agg[cur][1] += float(r[ws] or 0)
        except ValueError:
            pass
tot = sum(v[0] for v in agg.values()) or 1
tots = sum(v[1] for v in agg.values()) or 1
print(f"{tot:,.0f} warp-instructions, {tots:,.0f} stall samples")
for (f, l), (n, smp, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{n / tot * 100:5.1f}% inst {smp / tots * 100:5.1f}% stall  {f}:{l:<5d} {src}")
