"""Per-source-line hot spots of one ncu report (stall samples, instructions).

    python scripts/ncu_lines.py <report.ncu-rep> [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
lines = []
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] not in ("",) and r[0].isdigit():
        d = dict(zip(hdr, r))
        try:
            samples = int(d["Warp Stall Sampling (All Samples)"])
            inst = int(d["Instructions Executed"])
        except (KeyError, ValueError):
            continue
        lines.append((samples, inst, int(r[0]), r[1].strip()[:90]))
tot_s = sum(x[0] for x in lines) or 1
tot_i = sum(x[1] for x in lines) or 1
print(f"| line | stall samples % | warp instructions % | source |\n|---|---|---|---|")
for s, i, ln, src in sorted(lines, reverse=True)[:top]:
    print(f"| {ln} | {100 * s / tot_s:.1f} | {100 * i / tot_i:.1f} | `{src}` |")
