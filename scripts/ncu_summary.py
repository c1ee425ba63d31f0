"""Summarise one gpu_bench_full.sh capture directory into markdown.

    python scripts/ncu_summary.py gpurun_out/<tag> > profiles/<round>/ncu_summary.md

Reads <dir>/launches.csv (ncu --metrics gpu__time_duration.sum launch list)
and every <dir>/*.ncu-rep (ncu --set full) with `ncu -i ... --page raw --csv`.
"""

import collections
import csv
import glob
import io
import os
import re
import subprocess
import sys

METRICS = [
    ("Duration", "gpu__time_duration.sum"),
    ("Elapsed cycles", "sm__cycles_elapsed.avg"),
    ("Registers / thread", "launch__registers_per_thread"),
    ("Grid size", "launch__grid_size"),
    ("Dynamic smem / block", "launch__shared_mem_per_block_dynamic"),
    ("Blocks / SM limit (smem)", "launch__occupancy_limit_shared_mem"),
    ("Warps active (% of peak)", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("IPC (per SMSP, active)", "smsp__inst_executed.avg.per_cycle_active"),
    ("SM throughput (% peak)", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("ALU pipe (% peak, active)", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
    ("DRAM read", "dram__bytes_read.sum"),
    ("DRAM write", "dram__bytes_write.sum"),
    ("L2 bytes", "lts__t_bytes.sum"),
    ("L2 hit rate", "lts__t_sector_hit_rate.pct"),
    ("L1 hit rate", "l1tex__t_sector_hit_rate.pct"),
    ("Issue slots busy", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
    ("Warp instructions executed", "smsp__inst_executed.sum"),
    ("Achieved occupancy", "sm__warps_active.avg.per_cycle_active"),
]
STALLS = ["wait", "selected", "short_scoreboard", "long_scoreboard", "branch_resolving",
          "no_instructions", "not_selected", "math_pipe_throttle", "mio_throttle", "barrier"]


def kname(n):
    m = re.search(r"(\w+_kernel)(<[^>(]*>)?", n)
    return (m.group(1) + (m.group(2) or "")) if m else n[:60]


def launch_table(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1, "nsecond": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}
    tot, cnt, mx = collections.Counter(), collections.Counter(), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
        k = kname(r[ki])
        tot[k] += v
        cnt[k] += 1
        mx[k] = max(mx[k], v)
    T = sum(tot.values())
    out = ["| kernel | launches | total ms | mean us | max us | share |", "|---|---|---|---|---|---|"]
    for k, v in tot.most_common():
        out.append(f"| `{k}` | {cnt[k]} | {v / 1e6:.1f} | {v / cnt[k] / 1e3:.1f} | "
                   f"{mx[k] / 1e3:.1f} | {100 * v / T:.1f}% |")
    out.append(f"\nTotal device time {T / 1e6:.1f} ms over {sum(cnt.values())} launches.")
    return "\n".join(out)


def report(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        return f"(could not read {path})"
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        out.append(f"### `{kname(name)}` ({os.path.basename(path)})\n")
        out.append("| metric | value |\n|---|---|")
        for label, m in METRICS:
            if m in h:
                i = h.index(m)
                out.append(f"| {label} (`{m}`) | {r[i]} {units[i]} |")
        st = []
        for s in STALLS:
            m = f"smsp__pcsamp_warps_issue_stalled_{s}"
            if m in h and r[h.index(m)]:
                st.append((s, float(r[h.index(m)].replace(",", ""))))
        st.sort(key=lambda x: -x[1])
        out.append("\nTop stall reasons (pc samples): " +
                   ", ".join(f"{s} {int(v)}" for s, v in st[:6]) + "\n")
    return "\n".join(out)


def main():
    d = sys.argv[1]
    print(f"# ncu evidence ({d})\n")
    lp = os.path.join(d, "launches.csv")
    if os.path.exists(lp):
        print("## Launch list (ncu gpu__time_duration.sum, cold-cache, serialised)\n")
        print(launch_table(lp) + "\n")
    for p in sorted(glob.glob(os.path.join(d, "*.ncu-rep"))):
        print("## Full set\n")
        print(report(p))


if __name__ == "__main__":
    main()
