"""Summarise ncu captures and launch lists into profiles/ (run in the build
container on files brought back in gpurun_out/).

    python tools/ncu_summary.py REPORT.ncu-rep [...]          # --set full captures
    python tools/ncu_summary.py --launches launches.csv       # gpu__time_duration list
"""

from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput (max unit)"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/TEX throughput"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe"),
    ("sm__warps_active.avg.per_cycle_active", "warps active / SM"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def raw(report: str):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True, check=True)
    rows = list(csv.reader(io.StringIO(out.stdout)))
    return rows[0], rows[1], rows[2:]


def summarise(report: str) -> str:
    h, units, rows = raw(report)
    lines = [f"### {report.split('/')[-1]}", ""]
    for r in rows:
        name = r[h.index("Kernel Name")]
        lines.append(f"**{name[:110]}**")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for key, label in METRICS:
            if key in h:
                i = h.index(key)
                lines.append(f"| {label} (`{key}`) | {r[i]} {units[i]} |")
        lines.append("")
    return "\n".join(lines)


def launches(path: str) -> str:
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    data = rows[hi + 1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in data:
        if not r[vi]:
            continue
        name = r[ki].split("(")[0]
        agg[name] += float(r[vi].replace(",", ""))
        cnt[name] += 1
    total = sum(agg.values())
    out = ["| kernel | launches | total us | share |", "|---|---|---|---|"]
    for n, v in sorted(agg.items(), key=lambda x: -x[1]):
        out.append(f"| {n} | {cnt[n]} | {v / 1e3:.1f} | {100 * v / total:.1f}% |")
    return "\n".join(out)


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        print(launches(sys.argv[2]))
    else:
        for rep in sys.argv[1:]:
            print(summarise(rep))
