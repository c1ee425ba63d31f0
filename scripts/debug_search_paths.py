"""Debug: step-by-step comparison of the general and chunked kernels inside
the search; dumps the first mismatching batch for CPU analysis."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2302_11665_b200 import Simulator
from workloads import configs, traces

names = [f"{b}#{i}" for b in ("BERT-1.3B", "MoE-2.4B", "BERT-6.7B") for i in range(2)]
prob = configs.build_problem(names, 8, 13 * 10**9, slo_scale=4.0)
tr = traces.maf2_shaped(9, len(names), 15.0, 600.0)
sim = Simulator(0)
sim.set_problem(prob)
sim.set_trace(tr.arrival_ns, tr.model)
for L in (64, 4096):
    sim.set_chunk_size(L)
    with sim.search_handle(dedup=False) as sh:
        step = 0
        while True:
            C = sh.prepare()
            if C == 0:
                break
            outs = {}
            for path in (1, 2):
                sim.set_path(path)
                buf = torch.zeros(C, dtype=torch.int64, device="cuda")
                sh.evaluate(0, C, buf)
                torch.cuda.synchronize()
                outs[path] = buf.cpu().numpy()
            bad = np.nonzero(outs[1] != outs[2])[0]
            if len(bad):
                print(f"L={L} step {step}: {len(bad)}/{C} mismatches, first {bad[:10]}",
                      outs[1][bad[:10]], outs[2][bad[:10]])
            sim.set_path(1)
            sh.apply(torch.from_numpy(outs[1]).cuda())
            step += 1
        print(f"L={L}: {step} steps done")
