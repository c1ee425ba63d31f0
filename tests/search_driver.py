"""Step-by-step driver of libasim's search for the tests (argument marshalling
and bookkeeping only; every simulation runs in the library)."""

from __future__ import annotations

import numpy as np


def stepwise(sim, **kw):
    """Drive the search through the C ABI (prepare / evaluate / apply) and
    record, after every step, each advancing run's candidate list with its
    goods (asim_search_run_candidates) and the step's pick (history).
    Returns (steps[run] = [(m[], g[], good[], (m*, g*, good*))], result)."""
    import torch

    with sim.search_handle(**kw) as sh:
        R = sh.num_runs()
        steps = [[] for _ in range(R)]
        buf = torch.zeros(1 << 16, dtype=torch.int64, device="cuda")
        while True:
            C = sh.prepare()
            if C < 0:
                break
            if C > 0:
                if buf.numel() < C:
                    buf = torch.zeros(2 * C, dtype=torch.int64, device="cuda")
                sh.evaluate(0, C, buf)
                sh.apply(buf)
            else:
                sh.apply(None)
            for r in range(R):
                hm, hg, hv = sh.history(r)
                if len(hm) > len(steps[r]):
                    m, g, v = sh.candidates(r)
                    steps[r].append((m, g, v, (int(hm[-1]), int(hg[-1]), int(hv[-1]))))
        res = sh.result()
    return steps, res


def placement_after(M, steps_r, i, extra=None):
    """Host mask of a run's selection after its first i picks (+ one more
    (m, g) addition): sel <- sel + (m*, g*) per step (Alg. 1)."""
    mask = np.zeros(M, np.uint64)
    for k in range(i):
        m, g, _ = steps_r[k][3]
        mask[m] |= np.uint64(1) << np.uint64(g)
    if extra is not None:
        m, g = extra
        mask[m] |= np.uint64(1) << np.uint64(g)
    return mask
