"""CPU baseline per SURVEY §8(d): the oracle (event-driven DES + plain Alg. 2,
built -O3 -march=native for this host) timed on the host cores.

* evaluation rate on the GPU's own batch: the S3 step-0 batch (every Alg. 2
  run's additions to the empty placement) on the day trace's 10-min prefix;
* full-search wall times: motivating (all 17 placements brute force, and
  Alg. 2), S4 (day-long trace), S1 on a 5-min trace;
* labelled extrapolations to the S3 10-min and day-long searches: the plain
  search simulates every candidate of every step over the whole trace
  (candidates_per_search x N evaluations at the measured rate).

    python scripts/cpu_baseline.py [out.json]
"""
import json
import os
import platform
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from oracle import search as osearch  # noqa: E402
from workloads import configs  # noqa: E402

import bench  # noqa: E402  (step0_batch: the GPU's step-0 candidates)


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def timed(fn):
    t0 = time.perf_counter()
    r = fn()
    return r, time.perf_counter() - t0


def main():
    oracle.use_timing_build()
    threads = oracle.hardware_threads()
    out = dict(cores=threads, cpu=cpu_model(), build="g++ -O3 -march=native")
    # 1) rate on the S3 step-0 batch x the 10-min prefix of the day trace
    prob, tr = configs.s3(duration=86400.0)
    sub = tr.prefix(int(np.searchsorted(tr.arrival_ns, tr.arrival_ns[0] + 600 * 10**9)))
    cfg, mask = bench.step0_batch(prob)
    n_c = min(len(cfg), 8 * threads)
    sel = np.random.default_rng(0).permutation(len(cfg))[:n_c]
    _, dt = timed(lambda: oracle.evaluate(prob, sub, cfg[sel], mask[sel], threads))
    rate = n_c * len(sub) / dt
    out["s3_step0_rate"] = dict(value=rate, unit="request-placements/s", candidates=int(n_c),
                                of=int(len(cfg)), requests=len(sub), seconds=dt,
                                per_core=rate / threads)
    # 2) full searches
    mp = configs.motivating_problem(slo_scale=5.0)
    mt = configs.motivating_trace(seed=0, n_requests=1000)
    _, out["motivating_bruteforce_s"] = timed(lambda: osearch.bruteforce(mp, mt, threads))
    r, out["motivating_alg2_s"] = timed(lambda: osearch.alg2(mp, mt, threads))
    p4, t4 = configs.s4()
    r4, out["s4_day_alg2_s"] = timed(lambda: osearch.alg2(p4, t4, threads))
    out["s4_day"] = dict(requests=len(t4), best_good=int(r4["good"]))
    p1, t1 = configs.s1(duration=300.0)
    r1, out["s1_5min_alg2_s"] = timed(lambda: osearch.alg2(p1, t1, threads))
    out["s1_5min"] = dict(requests=len(t1), best_good=int(r1["good"]))
    # 3) labelled extrapolations (the plain search: every candidate x the whole trace)
    ext = {}
    for label, dur, cands in (("s3_10min", 600.0, None), ("s3_day", 86400.0, None)):
        n = len(tr.prefix(int(np.searchsorted(tr.arrival_ns, tr.arrival_ns[0] + dur * 10**9))))
        ext[label] = dict(requests=n, note="extrapolation: candidates_per_search x requests / "
                                          "s3_step0_rate; candidates_per_search from the GPU "
                                          "search of the same trace (bench.py config)")
    out["extrapolations"] = ext
    js = json.dumps(out, indent=1)
    print(js)
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            f.write(js + "\n")


if __name__ == "__main__":
    main()
