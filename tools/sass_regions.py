"""Group an ncu SASS source export (--page source --csv --print-source sass) into runs of equal execution count
and print the heaviest runs with their opcode mix (where a kernel's instructions go).
    python tools/sass_regions.py sass.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
h = rows[1]
ie, src, st = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
ins = [(r[src].strip(), int(r[ie]), int(r[st] or 0)) for r in rows[2:] if len(r) > ie and r[ie].isdigit()]
tot = sum(c for _, c, _ in ins) or 1
tots = sum(s for *_, s in ins) or 1


def opn(s):
    t = s.split()
    return t[1] if t[0].startswith('@') else t[0]


op = collections.Counter()
for s, c, _ in ins:
    op[opn(s)] += c
print(f"{len(ins)} SASS lines, {tot:,} warp-instructions")
print("mix:", ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in op.most_common(20)))
reg, cur = [], None
for i, (s, c, sm) in enumerate(ins):
    if cur and cur[1] == c:
        cur[2] += c
        cur[3] += 1
        cur[4] += sm
        cur[5].append(s)
    else:
        cur = [i, c, c, 1, sm, [s]]
        reg.append(cur)
for r in sorted(reg, key=lambda r: -r[2])[:top]:
    mix = collections.Counter(opn(x) for x in r[5])
    print(f"@{r[0]:5d} n={r[3]:4d} exec={r[1]:>9d} share={r[2] / tot * 100:5.2f}% stall={r[4] / tots * 100:5.2f}% "
          f"{dict(mix.most_common(6))}")
