"""Verification of the headline search at full size.

The exact bench.py configuration -- S3: 60 mixed BERT/MoE models on 64
devices, the MAF2-shaped trace, the full Alg. 2 (single bucket) ⊃ Alg. 1
search with run pruning -- runs on the GPU step by step, recording every
candidate's good at every step.  The event-driven oracle cannot replay the
whole search, so it re-simulates from scratch, as whole placements:

* every step's winner of the best run and of two other (seeded) runs --
  Alg. 1 picks by simulated attainment at every iteration;
* a seeded 0.1 % sample of all (run, step, candidate) evaluations;
* the final placement.

Every value must match bit-exactly."""

import os

import numpy as np
import pytest

import oracle
from oracle import search as osearch
from tests.search_driver import placement_after, stepwise
from workloads import configs

pytestmark = pytest.mark.gpu


def _verify(prob, tr, steps, res, rng, frac, n_other_runs):
    M = prob.num_models
    runs = [cfg for _, _, cfg in osearch.alg2_runs(prob)]
    G = max(len(c) for c in runs)
    cfgs, masks, want, what = [], [], [], []

    def add(r, mask, good, tag):
        c = np.full(G, -1, np.int32)
        c[:len(runs[r])] = runs[r]
        cfgs.append(c)
        masks.append(mask)
        want.append(good)
        what.append(tag)

    # every step's winner of the best run and of other runs
    others = [r for r in range(len(runs)) if r != res.best_run and steps[r]]
    pick = [res.best_run] + list(rng.choice(others, size=min(n_other_runs, len(others)),
                                            replace=False))
    for r in pick:
        for i, st in enumerate(steps[r]):
            add(r, placement_after(M, steps[r], i + 1), st[3][2], ("winner", r, i))
    # a seeded sample of all candidate evaluations
    flat = [(r, i, k) for r in range(len(runs)) for i, st in enumerate(steps[r])
            for k in range(len(st[0]))]
    n = max(1, int(round(frac * len(flat))))
    for idx in rng.choice(len(flat), size=n, replace=False):
        r, i, k = flat[idx]
        m, g, v, _ = steps[r][i]
        add(r, placement_after(M, steps[r], i, (int(m[k]), int(g[k]))), int(v[k]),
            ("candidate", r, i, k))
    # the final placement
    c = np.full(G, -1, np.int32)
    c[:res.num_groups] = res.group_cfg
    cfgs.append(c)
    masks.append(res.host_mask)
    want.append(res.best_good)
    what.append(("final",))
    got, _, _ = oracle.evaluate(prob, tr, np.stack(cfgs), np.stack(masks),
                                threads=os.cpu_count() or 1)
    bad = [(w, int(a), int(b)) for w, a, b in zip(what, got, want) if a != b]
    assert not bad, bad[:10]
    return len(want), n


def test_s3_headline_search_verified_by_oracle(sim_s3):
    prob, tr, sim = sim_s3
    steps, res = stepwise(sim, dedup=False, prune=True)
    assert res.best_run >= 0 and res.best_good > 0
    total = sum(len(st[0]) for s in steps for st in s)
    assert total == res.candidates
    checked, sampled = _verify(prob, tr, steps, res, np.random.default_rng(0), 1e-3, 2)
    assert sampled >= 100 and checked >= sampled + 100


@pytest.fixture(scope="module")
def sim_s3():
    from paper_2302_11665_b200 import Simulator
    prob, tr = configs.s3(duration=3600.0)
    s = Simulator(0)
    s.set_problem(prob)
    s.set_trace(tr.arrival_ns, tr.model)
    yield prob, tr, s
    s.close()
