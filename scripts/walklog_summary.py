"""Critical path of the walk phase from a walk log (scripts/gpu_walklog.sh:
a build with ASIM_WALK_DIAGNOSTICS, search_profile.py --steps with
ASIM_WALK_LOG=<cycles>): per step the longest walk, summed by walker kind
(0 cooperative, 1 scalar, 2 group-lane) and stage count.

    python scripts/walklog_summary.py profiles/r2m/walklog_day.txt.gz [sm_mhz]
"""
import collections
import gzip
import re
import sys

path = sys.argv[1]
mhz = float(sys.argv[2]) if len(sys.argv) > 2 else 1965.0
rx = re.compile(r"walk kind=(\d) S=(\d+) slots=(\d+) ng=(\d+) models=(\d+) chunks=(\d+) cycles=(\d+)")
steps, cur = [], []
with (gzip.open(path, "rt") if path.endswith(".gz") else open(path)) as f:
    for line in f:
        if line.startswith("STEP"):
            steps.append(cur)
            cur = []
            continue
        m = rx.search(line)
        if m:
            cur.append(tuple(map(int, m.groups())))
crit = collections.Counter()
allw = collections.Counter()
for st in steps:
    if st:
        w = max(st, key=lambda x: x[6])
        crit[(w[0], w[1])] += w[6]
    for x in st:
        allw[(x[0], x[1])] += x[6]
names = {0: "cooperative", 1: "scalar", 2: "group-lane"}
print(f"{len(steps)} steps; critical path (sum of each step's longest walk) "
      f"{sum(crit.values()) / mhz / 1e6:.2f} s at {mhz:.0f} MHz")
print("| walker | S | critical path s | all walks (warp-s) |")
print("|---|---|---|---|")
for k, v in crit.most_common():
    print(f"| {names[k[0]]} | {k[1]} | {v / mhz / 1e6:.2f} | {allw[k] / mhz / 1e6:.1f} |")
longest = sorted((max(st, key=lambda x: x[6]) for st in steps if st), key=lambda x: -x[6])[:5]
print("longest walks (kind, S, slots, groups, models, chunks, cycles, cycles/chunk):")
for w in longest:
    print(" ", w, round(w[6] / max(1, w[5])))
