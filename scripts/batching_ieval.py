"""Warp instructions per (request, candidate) evaluation of the batching
kernel, from an ncu launch list of `scripts/bench_batching.py --steps 1
--warmup 0` (metrics smsp__inst_executed.sum, gpu__time_duration.sum) and that
run's JSON line (candidates C, trace requests N):

    ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum -k regex:batching_kernel \\
        --csv --log-file L.csv python scripts/bench_batching.py --steps 1 --warmup 0 \\
        --no-cpu-baseline > B.json
    python scripts/batching_ieval.py L.csv B.json out.json
"""
import csv
import json
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = next(r for r in rows if "Metric Name" in r)
im, iv = hdr.index("Metric Name"), hdr.index("Metric Value")
ik = hdr.index("Kernel Name")
inst = [float(r[iv].replace(",", "")) for r in rows
        if r[im] == "smsp__inst_executed.sum" and "batching_kernel" in r[ik]]
line = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
C, N = line["config"]["feasible"], line["config"]["trace_requests"]
# the timed step is the last launch (warm-up 0, one timed step, then e2e calls)
out = dict(inst_per_eval=inst[0] / (C * N), launches=len(inst), inst_first_launch=inst[0],
           candidates=C, requests=N,
           source="ncu --metrics smsp__inst_executed.sum (first batching_kernel launch of "
                  "scripts/bench_batching.py --steps 1 --warmup 0)")
json.dump(out, open(sys.argv[3], "w"), indent=1)
print(json.dumps(out))
