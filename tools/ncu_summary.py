#!/usr/bin/env python
"""Summarise ncu reports for profiles/: per-kernel duration, DRAM bytes, throughputs, occupancy.

    python tools/ncu_summary.py <report.ncu-rep> <workload-name> [--traffic profiles/ncu_traffic.json]

Reads `ncu -i <rep> --page raw --csv` (needs the ncu CLI, no GPU), prints a text table and, with
--traffic, merges {workload: {kernel_short_name: dram_read+write bytes per launch}} into the JSON
that bench.py reports as roofline.traffic.
"""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem_pct"),
    ("sm__inst_executed.sum", "inst"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__shared_mem_per_block_dynamic", "smem_dyn"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__cycles_elapsed.avg.per_second", "sm_hz"),
]


def short(name: str) -> str:
    for k in ("k_p1", "k_p2", "k_fhtshift", "k_range_tables", "k_pass1", "k_pass2"):
        if k in name:
            return k
    return name.split("(")[0][-40:]


def read(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    units = rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        k = {"kernel": d.get("Kernel Name", "?"), "short": short(d.get("Kernel Name", "?"))}
        for m, key in METRICS:
            v = d.get(m)
            if v not in (None, ""):
                try:
                    k[key] = float(v.replace(",", ""))
                except ValueError:
                    k[key] = v
                k[key + "_unit"] = units[hdr.index(m)]
        res.append(k)
    return res


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    return v * scale.get(unit, 1)


def to_ns(v, unit):
    return v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "ns": 1, "us": 1e3, "ms": 1e6}.get(unit, 1)


def main():
    rep, workload = sys.argv[1], sys.argv[2]
    traffic_path = None
    if "--traffic" in sys.argv:
        traffic_path = sys.argv[sys.argv.index("--traffic") + 1]
    ks = read(rep)
    print(f"ncu --set full summary: {os.path.basename(rep)}  workload={workload}")
    print(f"{'kernel':10s} {'us':>9s} {'dramR MB':>9s} {'dramW MB':>9s} {'dram%':>6s} {'L2 MB':>8s} {'sm%':>6s} "
          f"{'smem%':>6s} {'occ%':>6s} {'regs':>5s} {'smemKB':>7s} {'grid':>7s}")
    agg = {}
    for k in ks:
        us = to_ns(k.get("duration", 0), k.get("duration_unit", "ns")) / 1e3
        rd = to_bytes(k.get("dram_read", 0), k.get("dram_read_unit", "byte"))
        wr = to_bytes(k.get("dram_write", 0), k.get("dram_write_unit", "byte"))
        l2 = to_bytes(k.get("l2_bytes", 0), k.get("l2_bytes_unit", "byte"))
        print(f"{k['short']:10s} {us:9.2f} {rd / 1e6:9.2f} {wr / 1e6:9.2f} {k.get('dram_pct', 0):6.1f} {l2 / 1e6:8.2f} "
              f"{k.get('sm_pct', 0):6.1f} {k.get('smem_pct', 0):6.1f} {k.get('occupancy_pct', 0):6.1f} "
              f"{int(k.get('regs', 0)):5d} {k.get('smem_dyn', 0) / 1024:7.1f} {int(k.get('grid', 0)):7d}")
        a = agg.setdefault(k["short"], [])
        a.append(rd + wr)
    if traffic_path:
        data = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
        data.setdefault(workload, {})
        for name, v in agg.items():
            data[workload][name] = sum(v) / len(v)
        json.dump(data, open(traffic_path, "w"), indent=1, sort_keys=True)
        print(f"traffic per launch merged into {traffic_path}")


if __name__ == "__main__":
    main()
