"""Sweep the chunked path's requests-per-chunk on the S3 1 h search (results
are identical for every chunk size; only the time changes)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2302_11665_b200 import Simulator
from paper_2302_11665_b200 import dist as adist
from workloads import configs

prob, tr = configs.s3(seed=0, duration=3600.0)
stream = torch.cuda.current_stream()
out = {}
with Simulator(0) as sim:
    sim.set_problem(prob)
    sim.set_trace(tr.arrival_ns, tr.model)
    for cs in [int(x) for x in sys.argv[1:]]:
        sim.set_chunk_size(cs)
        ms = []
        for k in range(4):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            with sim.search_handle() as sh:
                adist.run_search(sh, stream=stream)
                r = sh.result()
            e1.record(stream)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        out[cs] = dict(ms=ms[1:], best_good=r.best_good, best_run=r.best_run)
        print(cs, [round(x, 1) for x in ms[1:]], r.best_good, flush=True)
print(json.dumps(out))
