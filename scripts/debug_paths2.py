import sys
import numpy as np
sys.path.insert(0, ".")
import oracle
from paper_2302_11665_b200 import Simulator
from workloads import configs
sim = Simulator(0)
for scale in (1.0, 5.0):
    prob = configs.motivating_problem(slo_scale=scale)
    tr = configs.motivating_trace(seed=2, n_requests=1000)
    sim.set_problem(prob); sim.set_trace(tr.arrival_ns, tr.model)
    # step-0 batch of all three Alg. 2 runs
    bc = np.array([[0, 0], [1, -1], [2, -1]], np.int32)
    bm = np.zeros((3, 2), np.uint64)
    cb = np.array([0, 0, 0, 0, 1, 1, 2, 2], np.int32)
    cm = np.array([0, 0, 1, 1, 0, 1, 0, 1], np.int32)
    cg = np.array([0, 1, 0, 1, 0, 0, 0, 0], np.int32)
    full_cfg = bc[cb]; full_mask = np.zeros((8, 2), np.uint64)
    for c in range(8): full_mask[c, cm[c]] |= np.uint64(1) << np.uint64(cg[c])
    want = oracle.evaluate(prob, tr, full_cfg, full_mask)[0]
    print("scale", scale, "oracle", want)
    for path in (1, 2, 3):
        sim.set_path(path)
        print(" path", path, sim.evaluate_deltas(bc, bm, cb, cm, cg)["good"])
    # single candidate per item
    for path in (2, 3):
        sim.set_path(path)
        got = [int(sim.evaluate_deltas(bc, bm, cb[i:i+1], cm[i:i+1], cg[i:i+1])["good"][0]) for i in range(8)]
        print(" path", path, "one-by-one", got)
