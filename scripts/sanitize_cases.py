"""Small cases for compute-sanitizer (memcheck, racecheck, synccheck,
initcheck): every kernel family of libasim.so on inputs small enough to run
under the sanitizers in seconds.  No torch: the library's own search loop.

    compute-sanitizer --tool memcheck python scripts/sanitize_cases.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2302_11665_b200 import Simulator  # noqa: E402
from workloads import configs, traces  # noqa: E402


def main():
    names = [f"{b}#{i}" for b in ("BERT-1.3B", "BERT-2.7B", "MoE-1.3B", "MoE-5.3B")
             for i in range(2)]
    prob = configs.build_problem(names, 8, 13 * 10**9, slo_scale=4.0)
    tr = traces.maf2_shaped(21, len(names), 20.0, 240.0)
    M = prob.num_models
    rng = np.random.default_rng(0)
    with Simulator(0) as s:
        s.set_problem(prob)
        s.set_trace(tr.arrival_ns, tr.model)
        # general kernel with per-model counts and busy times
        C = 40
        cfg = np.full((C, 8), -1, np.int32)
        mask = np.zeros((C, M), np.uint64)
        for c in range(C):
            p = int(rng.integers(0, prob.num_configs))
            G = 8 // int(prob.cfg_devices[p])
            cfg[c, :G] = p
            for m in range(M):
                if rng.random() < 0.3:
                    mask[c, m] = np.uint64(1) << np.uint64(int(rng.integers(0, G)))
        s.evaluate(cfg, mask, per_model=True, busy=True)
        # chunked path (items, passes 1-3, walkers on side streams), uint32 and int64
        for path in (2, 3):
            s.set_path(path)
            s.set_chunk_size(13)
            bc, bm = cfg[:3], mask[:3]
            cb = np.repeat(np.arange(3, dtype=np.int32), 20)
            cm = rng.integers(0, M, size=60).astype(np.int32)
            cg = np.array([int(rng.integers(0, 8 // int(prob.cfg_devices[cfg[b, 0]])))
                           for b in cb], np.int32)
            s.evaluate_deltas(bc, bm, cb, cm, cg)
        s.set_path(0)
        # the search (component restriction, grouping, every walker), small chunks
        for chunk in (40, 4096):
            s.set_chunk_size(chunk)
            with s.search_handle(dedup=True, prune=True) as h:
                h.run()
        # fast heuristic (statistics rows) and dynamic batching
        with s.search_handle(fast=True) as h:
            h.run()
        inc = configs.batch_increment_ns(prob.stage_ns, 0.9)
        s.evaluate_batching(cfg[:16], mask[:16], inc, 3, per_model=True)
    # the group-lane walker for every uniform component (any stage count) and
    # split steps (two chunked runs on concurrent streams)
    os.environ.update(ASIM_GLANE_WALK="1", ASIM_GLANE_SMAX="16", ASIM_SPLIT="1")
    with Simulator(0) as s:
        s.set_problem(prob)
        s.set_trace(tr.arrival_ns, tr.model)
        for chunk in (40, 4096):
            s.set_chunk_size(chunk)
            with s.search_handle(dedup=False, prune=True) as h:
                h.run()
    print("sanitize cases done")


if __name__ == "__main__":
    main()
