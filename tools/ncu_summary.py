#!/usr/bin/env python
"""Summarise ncu outputs for profiles/: a --set full report (.ncu-rep) and/or
a launch list (--metrics gpu__time_duration.sum --csv log).

  python tools/ncu_summary.py --rep gpurun_out/walk_c2.ncu-rep --launches gpurun_out/launches.csv > profiles/x.md
"""
import argparse
import collections
import csv
import io
import subprocess

KEYS = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg.per_second",
    "launch__grid_size",
    "launch__block_size",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "sm__warps_active.avg.per_cycle_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed.sum.per_cycle_elapsed",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
]


def rep_table(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    lines = []
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        lines.append(f"### {name}\n")
        lines.append("| metric | unit | value |\n|---|---|---|")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                lines.append(f"| {k} | {units[i]} | {r[i]} |")
        lines.append("")
    return "\n".join(lines)


def launches_table(path):
    text = open(path).read()
    rows = list(csv.reader(io.StringIO(text[text.index('"ID"'):] if '"ID"' in text else text)))
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(r[ui], 1.0)
        k = r[ki].split("(")[0]
        tot[k] += float(r[vi].replace(",", "")) * scale
        cnt[k] += 1
    allt = sum(tot.values())
    lines = ["| kernel | launches | total us | avg us | share |", "|---|---|---|---|---|"]
    for k, t in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"| {k} | {cnt[k]} | {t:.1f} | {t / cnt[k]:.1f} | {t / allt:.1%} |")
    return "\n".join(lines)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    a = ap.parse_args()
    if a.launches:
        print("## Launch list (ncu gpu__time_duration.sum, cold-cache, serialised)\n")
        print(launches_table(a.launches))
        print()
    if a.rep:
        print("## ncu --set full\n")
        print(rep_table(a.rep))
