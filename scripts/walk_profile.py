"""Diagnostics (not a benchmark): per-step walk statistics of the S3 search
-- how many candidates walk and the longest single walk (the walk pass's
sequential critical path) -- and the search time per chunk size."""
import os, sys, time
import torch
sys.path.insert(0, ".")
from paper_2302_11665_b200 import Simulator
from workloads import configs

hours = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
sizes = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [4096]
verbose = len(sys.argv) > 3
prob, tr = configs.s3(duration=hours * 3600)
N = len(tr)
sim = Simulator(0); sim.set_problem(prob); sim.set_trace(tr.arrival_ns, tr.model)
buf = torch.zeros(40000, dtype=torch.int64, device="cuda")
for L in sizes:
    sim.set_chunk_size(L)
    J = max(1, min(1024, N // L))
    for rep in range(2):
        sim.set_profiling(True); sim.reset_stats()
        torch.cuda.synchronize(); t0 = time.perf_counter()
        rows = []
        with sim.search_handle(dedup=False, prune=os.environ.get("PRUNE", "1") != "0") as sh:
            step = 0
            while True:
                C = sh.prepare()
                if C < 0:
                    break
                if verbose and rep == 1:
                    s0 = sim.stats(); ts = time.perf_counter()
                if C > 0:
                    sh.evaluate(0, C, buf); sh.apply(buf)
                else:
                    sh.apply(None)
                if verbose and rep == 1:
                    torch.cuda.synchronize(); s1 = sim.stats()
                    rows.append((step, C, s1["walk_candidates"] - s0["walk_candidates"],
                                 s1["chunk_reruns"] - s0["chunk_reruns"],
                                 s1["walk_critical_chunks"] - s0["walk_critical_chunks"],
                                 (time.perf_counter() - ts) * 1e3))
                step += 1
            r = sh.result()
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        st = sim.stats()
    print(f"L={L} J={J} search {dt*1e3:.0f} ms steps {r.steps} sim_ms {st['sim_ms']:.0f} "
          f"walk_cands {st['walk_candidates']} walked_chunks {st['chunk_reruns']} "
          f"critical_chunks {st['walk_critical_chunks']} (= {st['walk_critical_chunks']*N/J/1e6:.2f} M requests) "
          f"best {r.best_good}/{N}", flush=True)
    for row in rows:
        print("  step %3d C=%6d walk_cands=%5d walked=%6d critical=%4d ms=%7.2f" % row)
