"""Determinism and invariance (pin P13): every result is an
integer with index tie-breaks, so it must not depend on how the work is laid
out -- candidate order, time-chunk length, the work-item grouping of the
chunked path, which walker re-simulates a chunk, or repetition."""

import os

import numpy as np
import pytest

from workloads import configs, traces

pytestmark = pytest.mark.gpu


def _sim(prob, tr, env=None):
    from paper_2302_11665_b200 import Simulator
    old = {}
    for k, v in (env or {}).items():  # read once, when the context is created
        old[k] = os.environ.get(k)
        os.environ[k] = v
    try:
        s = Simulator(0)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    s.set_problem(prob)
    s.set_trace(tr.arrival_ns, tr.model)
    return s


def _instance():
    names = [f"{b}#{i}" for b in ("BERT-1.3B", "BERT-2.7B", "MoE-1.3B", "MoE-5.3B")
             for i in range(3)]
    prob = configs.build_problem(names, 8, 13 * 10**9, slo_scale=4.0)
    tr = traces.maf2_shaped(21, len(names), 30.0, 600.0)
    return prob, tr


def _deltas(prob, rng, n_bases=4, per_base=60):
    """Random greedy-step batches: bases with a few models placed, candidates
    = random feasible-looking additions (infeasible ones are data: -1)."""
    M = prob.num_models
    cfgs, masks, cb, cm, cg = [], [], [], [], []
    for b in range(n_bases):
        p = int(rng.integers(0, prob.num_configs))
        G = 8 // int(prob.cfg_devices[p])
        cfg = np.full(8, -1, np.int32)
        cfg[:G] = p
        mask = np.zeros(M, np.uint64)
        for m in rng.choice(M, size=3, replace=False):
            mask[m] |= np.uint64(1) << np.uint64(int(rng.integers(0, G)))
        cfgs.append(cfg)
        masks.append(mask)
        for _ in range(per_base):
            cb.append(b)
            cm.append(int(rng.integers(0, M)))
            cg.append(int(rng.integers(0, G)))
    return (np.stack(cfgs), np.stack(masks), np.array(cb, np.int32), np.array(cm, np.int32),
            np.array(cg, np.int32))


def test_candidate_permutation_invariance():
    prob, tr = _instance()
    rng = np.random.default_rng(3)
    bc, bm, cb, cm, cg = _deltas(prob, rng)
    s = _sim(prob, tr)
    try:
        s.set_chunk_size(97)
        ref = s.evaluate_deltas(bc, bm, cb, cm, cg)
        for seed in range(3):
            perm = np.random.default_rng(seed).permutation(len(cb))
            got = s.evaluate_deltas(bc, bm, cb[perm], cm[perm], cg[perm])
            np.testing.assert_array_equal(got["good"], ref["good"][perm])
            np.testing.assert_array_equal(got["sum_latency_ns"], ref["sum_latency_ns"][perm])
            g = ref["good"][perm]
            assert got["argmax"] == (int(np.argmax(g)) if g.max() >= 0 else -1)
        again = s.evaluate_deltas(bc, bm, cb, cm, cg)  # repetition
        np.testing.assert_array_equal(again["good"], ref["good"])
    finally:
        s.close()


@pytest.mark.parametrize("env", [{"ASIM_GROUP_CANDIDATES": "0"},
                                 {"ASIM_SCALAR_WALK": "0"}, {"ASIM_GLANE_WALK": "0"},
                                 {"ASIM_GLANE_WALK": "1", "ASIM_GLANE_SMAX": "16"},
                                 {"ASIM_SPLIT": "1"},
                                 {"ASIM_SPLIT": "1", "ASIM_GROUP_CANDIDATES": "0"}])
def test_search_layout_invariance(env):
    """The search's step-by-step results with the candidates regrouped or not,
    and whichever walker re-simulates a chunk, at several chunk lengths."""
    from tests.search_driver import stepwise

    prob, tr = _instance()
    out = []
    for e in ({}, env):
        s = _sim(prob, tr, e)
        try:
            for chunk in (4096, 61):
                s.set_chunk_size(chunk)
                steps, res = stepwise(s, dedup=False, prune=False)
                out.append((chunk, steps, res))
        finally:
            s.close()
    _, st0, r0 = out[0]
    for chunk, st, r in out[1:]:  # every layout against the first
        assert (r.best_run, r.best_good) == (r0.best_run, r0.best_good), chunk
        for a, b in zip(st, st0):
            assert len(a) == len(b)
            for x, y in zip(a, b):
                for u, w in zip(x[:3], y[:3]):
                    np.testing.assert_array_equal(u, w)
                assert x[3] == y[3]
