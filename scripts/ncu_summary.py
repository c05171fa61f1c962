#!/usr/bin/env python
"""Summarise an ncu capture of eval_kernel (+ the launch list of the same bench
command) as markdown for profiles/. Usage:
  python scripts/ncu_summary.py gpurun_out/eval_TAG.ncu-rep gpurun_out/launches_TAG.csv
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC (per SM)"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe (IMAD) %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "shared bank conflicts"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2]


def main():
    rep, launches = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None
    h, units, v = raw(rep)
    print("| metric | value |\n|---|---|")
    for key, label in METRICS:
        if key in h:
            i = h.index(key)
            print(f"| {label} (`{key}`) | {v[i]} {units[i]} |")
    stalls = []
    for i, name in enumerate(h):
        if name.startswith("smsp__average_warps_issue_stalled") and \
                name.endswith("per_issue_active.ratio"):
            try:
                stalls.append((float(v[i]), name.split("stalled_")[1].split("_per_issue")[0]))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    print("\nTop stall reasons (warp cycles per issued instruction): " +
          ", ".join(f"{n} {x:.2f}" for x, n in stalls[:8]))
    if launches:
        per = defaultdict(list)
        rows = [r for r in csv.reader(open(launches)) if len(r) > 10]
        hdr = rows[0]
        ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
        for r in rows[1:]:
            if r[mi] == "gpu__time_duration.sum":
                per[r[ki].split("(")[0][:60]].append(float(r[vi].replace(",", "")))
        tot = sum(sum(x) for x in per.values())
        print("\nLaunch list (ncu, serialised, cold): kernel, launches, total, share")
        for k, x in sorted(per.items(), key=lambda kv: -sum(kv[1])):
            print(f"- `{k}`: {len(x)} launches, {sum(x):.1f} (unit as captured), "
                  f"{100 * sum(x) / tot:.1f}%")


if __name__ == "__main__":
    main()
