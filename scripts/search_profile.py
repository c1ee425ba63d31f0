"""Diagnostics (not the benchmark): one full S3 search with profiling on --
phase times of the chunked path (pass 1, pass 2, walk), pass-1 lane
utilisation, walk statistics -- optionally per step.

    python scripts/search_profile.py [hours] [--steps] [--dedup] [--chunk N]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2302_11665_b200 import Simulator  # noqa: E402
from workloads import configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("hours", type=float, nargs="?", default=1.0)
ap.add_argument("--steps", action="store_true")
ap.add_argument("--dedup", action="store_true")
ap.add_argument("--chunk", type=int, default=4096)
ap.add_argument("--reps", type=int, default=2)
args = ap.parse_args()

t0 = time.perf_counter()
prob, tr = configs.s3(duration=args.hours * 3600)
N = len(tr)
print(f"trace {N} requests in {time.perf_counter() - t0:.1f} s", flush=True)
sim = Simulator(0)
sim.set_problem(prob)
sim.set_trace(tr.arrival_ns, tr.model)
sim.set_chunk_size(args.chunk)
buf = torch.zeros(1 << 17, dtype=torch.int64, device="cuda")
for rep in range(args.reps):
    sim.set_profiling(True)
    sim.reset_stats()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rows = []
    with sim.search_handle(dedup=args.dedup, prune=True) as sh:
        while True:
            C = sh.prepare()
            if C < 0:
                break
            if args.steps:
                s0 = sim.stats()
                ts = time.perf_counter()
            if C > 0:
                sh.evaluate(0, C, buf)
                sh.apply(buf)
            else:
                sh.apply(None)
            if args.steps:
                torch.cuda.synchronize()
                s1 = sim.stats()
                print(f"STEP {len(rows)} C={C}", flush=True)  # separates device walk-log lines
                rows.append(dict(C=C, ms=(time.perf_counter() - ts) * 1e3,
                                 **{k: s1[k] - s0[k] for k in ("spec_ms", "pass2_ms", "walk_ms",
                                                               "walk_candidates", "chunk_reruns",
                                                               "spec_stage_updates",
                                                               "spec_live_lanes",
                                                               "spec_lane_slots",
                                                               "walk_critical_chunks")}))
        r = sh.result()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    st = sim.stats()
out = dict(hours=args.hours, N=N, search_ms=dt * 1e3, steps=r.steps, evaluated=r.evaluated,
           best_good=r.best_good, **st,
           lane_util=st["spec_live_lanes"] / max(1, st["spec_lane_slots"]))
print(json.dumps(out), flush=True)
for i, row in enumerate(rows):
    print(i, json.dumps(row))
