#!/usr/bin/env python
"""Summarise ncu captures for profiles/ (run here, no GPU needed).

  python tools/ncu_summary.py report <file.ncu-rep>      # per-kernel table (markdown)
  python tools/ncu_summary.py launches <launches.csv>    # launch-list shares (markdown)
  python tools/ncu_summary.py traffic <file.ncu-rep> ... # JSON {kernel: dram bytes/launch}
"""
from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs/thread"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC (warp-inst/clk/SM)"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
]


def raw(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def to_bytes(v: str, unit: str) -> float:
    x = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return x * scale.get(unit, 1)


def report(rep: str) -> str:
    h, units, rows = raw(rep)
    lines = []
    for row in rows:
        name = row[h.index("Kernel Name")]
        lines.append(f"### `{name[:110]}`\n")
        lines.append("| metric | value |\n|---|---|")
        for key, label in METRICS:
            if key in h:
                i = h.index(key)
                lines.append(f"| {label} (`{key}`) | {row[i]} {units[i]} |")
        stalls = []
        for i, k in enumerate(h):
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    stalls.append((k.replace("smsp__pcsamp_warps_issue_stalled_", ""),
                                   float(row[i].replace(",", ""))))
                except ValueError:
                    pass
        tot = sum(v for _, v in stalls) or 1.0
        top = sorted(stalls, key=lambda x: -x[1])[:6]
        lines.append("\nWarp-state samples (share): " +
                     ", ".join(f"{k} {v / tot:.1%}" for k, v in top) + "\n")
    return "\n".join(lines)


def traffic(reps: list[str]) -> dict:
    agg = defaultdict(list)
    for rep in reps:
        h, units, rows = raw(rep)
        ir, iw = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
        for row in rows:
            name = row[h.index("Kernel Name")]
            short = name.split("(")[0].split("::")[-1].split("<")[0].strip()
            agg[short].append(to_bytes(row[ir], units[ir]) + to_bytes(row[iw], units[iw]))
    return {k: sum(v) / len(v) for k, v in agg.items()}


def launches(path: str) -> str:
    text = "".join(l for l in open(path) if not l.startswith("=="))
    rows = list(csv.reader(io.StringIO(text)))
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for row in rows[1:]:
        agg[row[ki].split("(")[0][:70]].append(float(row[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    out = ["| kernel | launches | total µs | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        out.append(f"| `{k}` | {len(v)} | {sum(v) / 1e3:.1f} | {sum(v) / tot:.4f} |")
    return "\n".join(out)


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "report":
        print(report(sys.argv[2]))
    elif cmd == "launches":
        print(launches(sys.argv[2]))
    elif cmd == "traffic":
        print(json.dumps(traffic(sys.argv[2:]), indent=1))
