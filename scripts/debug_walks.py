import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2302_11665_b200 import Simulator
from workloads import configs
hours = float(sys.argv[1]) if len(sys.argv) > 1 else 0.25
prob, tr = configs.s3(duration=hours * 3600)
sim = Simulator(0); sim.set_problem(prob); sim.set_trace(tr.arrival_ns, tr.model)
sim.set_profiling(True)
with sim.search_handle(dedup=False) as sh:
    step = 0
    buf = torch.zeros(20000, dtype=torch.int64, device="cuda")
    while True:
        C = sh.prepare()
        if C < 0: break
        sim.reset_stats()
        t0 = time.perf_counter()
        if C > 0:
            sh.evaluate(0, C, buf); sh.apply(buf)
        else:
            sh.apply(None)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        st = sim.stats()
        if step % 5 == 0 or st["chunk_reruns"] > 50:
            print(f"step {step:3d} C={C:6d} walked_chunks={st['chunk_reruns']:6d} sim_ms={st['sim_ms']:8.2f} wall_ms={dt*1e3:8.2f}", flush=True)
        step += 1
    r = sh.result()
print("steps", r.steps, "cands", r.candidates, "sim", r.evaluated, "memo", r.memo_hits, "best", r.best_good, len(tr))
