"""Experiment: lockstep search vs one context + stream + thread per Alg. 2 run."""
import sys, time, threading
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2302_11665_b200 import Simulator
from paper_2302_11665_b200 import dist as adist
from workloads import configs
hours = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
prob, tr = configs.s3(duration=hours * 3600)
sim = Simulator(0); sim.set_problem(prob); sim.set_trace(tr.arrival_ns, tr.model)
torch.cuda.synchronize(); t0 = time.perf_counter()
res = sim.search(dedup=False); torch.cuda.synchronize(); t_lock = time.perf_counter() - t0
print("lockstep", t_lock, res.best_good, res.best_run, flush=True)
runs = [r["group_cfg"].tolist() for r in res.runs]
sims = []
for r in runs:
    s = Simulator(0); s.set_problem(prob); s.set_trace(tr.arrival_ns, tr.model); sims.append(s)
out = [None] * len(runs); times = [0.0] * len(runs)
def work(i):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        t = time.perf_counter()
        with sims[i].search_handle(runs=[runs[i]], dedup=False) as sh:
            adist.run_search(sh, stream=st)
            out[i] = sh.result()
        torch.cuda.current_stream().synchronize()
        times[i] = time.perf_counter() - t
torch.cuda.synchronize(); t0 = time.perf_counter()
th = [threading.Thread(target=work, args=(i,)) for i in range(len(runs))]
for t in th: t.start()
for t in th: t.join()
torch.cuda.synchronize(); t_conc = time.perf_counter() - t0
print("concurrent", t_conc, "per-run max", max(times), "sum", sum(times))
print("per-run secs", [round(x, 2) for x in times])
goods = [o.best_good for o in out]
print("same per-run goods:", goods == [r["best_good"] for r in res.runs])
