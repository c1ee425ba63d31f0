"""GPU parity of the whole placement search: libasim.so's lockstep Alg. 2 /
Alg. 1 driver (with and without exact de-duplication) must pick the same
placement as the oracle's plain step-by-step search, run by run."""

import numpy as np
import pytest

from oracle import search as osearch
from workloads import configs, traces

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sim():
    from paper_2302_11665_b200 import Simulator
    s = Simulator(0)
    yield s
    s.close()


def _compare(sim, prob, tr, dedup_modes=(False, True)):
    ref = osearch.alg2(prob, tr)
    sim.set_problem(prob)
    sim.set_trace(tr.arrival_ns, tr.model)
    for dedup, prune, bounding in [(d, p, p) for d in dedup_modes for p in (False, True)]:
        res = sim.search(dedup=dedup, prune=prune, bounding=bounding)
        if not bounding:
            assert res.bounded == 0
        assert len(res.runs) == len(ref["runs"])
        for r_gpu, r_ref in zip(res.runs, ref["runs"]):
            if r_gpu["pruned_at"] >= 0:  # stopped early: provably never the best run
                assert prune and r_ref["good"] < ref["good"]
                assert r_gpu["best_good"] <= r_ref["good"]
                continue
            assert r_gpu["best_good"] == r_ref["good"]
            np.testing.assert_array_equal(r_gpu["host_mask"], r_ref["placement"].host_mask)
            np.testing.assert_array_equal(r_gpu["group_cfg"], r_ref["placement"].group_cfg)
        assert res.best_good == ref["good"]
        assert res.best_run == ref["run"]
        if ref["run"] >= 0:
            np.testing.assert_array_equal(res.host_mask, ref["placement"].host_mask)
    return ref


def test_search_motivating(sim):
    for scale in (1.0, 1.5, 3.0, 5.0):
        prob = configs.motivating_problem(slo_scale=scale)
        tr = configs.motivating_trace(seed=2, n_requests=1000)
        _compare(sim, prob, tr)


def test_search_s1_shaped_small(sim):
    names = [f"BERT-1.3B#{i}" for i in range(8)]
    prob = configs.build_problem(names, 8, 13 * 10**9, slo_scale=2.0)
    tr = traces.independent_gamma(3, [3.0] * 8, 4.0, 120.0)
    _compare(sim, prob, tr)


def test_search_s3_shaped_small(sim):
    names = [f"{b}#{i}" for b in ("BERT-1.3B", "BERT-2.7B", "BERT-6.7B", "MoE-1.3B",
                                  "MoE-2.4B", "MoE-5.3B") for i in range(2)]
    prob = configs.build_problem(names, 8, 13 * 10**9, slo_scale=5.0)
    tr = traces.maf2_shaped(4, len(names), 20.0, 300.0)
    _compare(sim, prob, tr)


def test_search_s4_shaped(sim):
    prob, tr = configs.s4(duration=1800.0)
    ref = _compare(sim, prob, tr)
    assert ref["good"] > 0


@pytest.mark.parametrize("chunk", [40, 257])
def test_search_small_chunks_base_speculation(sim, chunk):
    """Many time chunks per step: candidates speculate from the base
    placement's true boundary states (search.cpp); still oracle-exact."""
    names = [f"{b}#{i}" for b in ("BERT-1.3B", "BERT-2.7B", "MoE-5.3B") for i in range(2)]
    prob = configs.build_problem(names, 8, 13 * 10**9, slo_scale=3.0)
    tr = traces.maf2_shaped(11, len(names), 12.0, 900.0)
    sim.set_chunk_size(chunk)
    try:
        _compare(sim, prob, tr)
    finally:
        sim.set_chunk_size(4096)


def test_pruning_stops_hopeless_runs(sim):
    """Exact run pruning (include/asim.h, spec->prune): runs of large
    intra-op-only groups cannot serve the trace (capacity bound below the
    best good another run reaches), are stopped, and the result is that of
    the unpruned search."""
    names = [f"{b}#{i}" for b in ("BERT-1.3B", "BERT-2.7B", "MoE-2.4B") for i in range(3)]
    prob = configs.build_problem(names, 8, 13 * 10**9, slo_scale=5.0)
    tr = traces.maf2_shaped(6, len(names), 60.0, 240.0)
    sim.set_problem(prob)
    sim.set_trace(tr.arrival_ns, tr.model)
    full = sim.search(dedup=False, prune=False)
    pr = sim.search(dedup=False, prune=True)
    assert (pr.best_run, pr.best_good) == (full.best_run, full.best_good)
    np.testing.assert_array_equal(pr.host_mask, full.host_mask)
    pruned = [i for i, r in enumerate(pr.runs) if r["pruned_at"] >= 0]
    assert pruned, "expected at least one hopeless run on this instance"
    for i in pruned:
        assert full.runs[i]["best_good"] < full.best_good
    assert pr.evaluated < full.evaluated


def test_bounding_skips_candidates_exactly(sim):
    """Exact candidate bounding (include/asim.h, spec->cand_bound): a step
    needs only its argmax, so candidates whose component bound cannot beat
    the best value found are never simulated; every run's selections are
    those of the search without it."""
    names = [f"{b}#{i}" for b in ("BERT-1.3B", "BERT-2.7B", "MoE-1.3B") for i in range(3)]
    prob = configs.build_problem(names, 8, 13 * 10**9, slo_scale=5.0)
    tr = traces.maf2_shaped(8, len(names), 10.0, 300.0)
    sim.set_problem(prob)
    sim.set_trace(tr.arrival_ns, tr.model)
    a = sim.search(dedup=False, prune=False, bounding=False)
    b = sim.search(dedup=False, prune=False, bounding=True)
    assert b.bounded > 0 and b.evaluated < a.evaluated
    assert (a.best_run, a.best_good) == (b.best_run, b.best_good)
    for ra, rb in zip(a.runs, b.runs):
        assert ra["best_good"] == rb["best_good"]
        np.testing.assert_array_equal(ra["host_mask"], rb["host_mask"])


# ------------------------------------------------------------------ per step
from tests.search_driver import stepwise  # noqa: E402


def _compare_steps(gpu_steps, ref_runs, prune):
    for r, (gs, rr) in enumerate(zip(gpu_steps, ref_runs)):
        ref_steps = rr["steps"]
        if prune:
            assert len(gs) <= len(ref_steps)
        else:
            assert len(gs) == len(ref_steps), f"run {r}"
        for i, ((m, g, v, chosen), (cands, goods, ci)) in enumerate(zip(gs, ref_steps)):
            np.testing.assert_array_equal(m, [c[0] for c in cands], err_msg=f"run {r} step {i}")
            np.testing.assert_array_equal(g, [c[1] for c in cands], err_msg=f"run {r} step {i}")
            np.testing.assert_array_equal(v, goods, err_msg=f"run {r} step {i} goods")
            assert chosen == (cands[ci][0], cands[ci][1], int(goods[ci])), (r, i)


@pytest.mark.parametrize("dedup,prune", [(False, False), (True, True)])
def test_search_every_step_s3_shaped(sim, dedup, prune):
    """Every greedy step of every Alg. 2 run: the same candidate list
    (m-major, g-minor, memory-feasible), the same good for every
    candidate -- simulated, from the component memo or a duplicate's
    representative -- and the same pick (lowest index on ties)."""
    names = [f"{b}#{i}" for b in ("BERT-1.3B", "BERT-2.7B", "BERT-6.7B", "MoE-1.3B",
                                  "MoE-2.4B", "MoE-5.3B") for i in range(2)]
    prob = configs.build_problem(names, 8, 13 * 10**9, slo_scale=5.0)
    tr = traces.maf2_shaped(4, len(names), 20.0, 300.0)
    ref = osearch.alg2(prob, tr, record=True)
    sim.set_problem(prob)
    sim.set_trace(tr.arrival_ns, tr.model)
    gs, res = stepwise(sim, dedup=dedup, prune=prune)
    _compare_steps(gs, ref["runs"], prune)
    assert res.best_good == ref["good"] and res.best_run == ref["run"]


@pytest.mark.parametrize("chunk", [37, 300])
def test_search_every_step_small_chunks(sim, chunk):
    """As above with many time chunks per step (speculation from the base's
    boundary states, candidate memory mixes, walks): per-step exact."""
    names = [f"{b}#{i}" for b in ("BERT-1.3B", "BERT-2.7B", "MoE-5.3B") for i in range(2)]
    prob = configs.build_problem(names, 8, 13 * 10**9, slo_scale=3.0)
    tr = traces.maf2_shaped(11, len(names), 12.0, 900.0)
    ref = osearch.alg2(prob, tr, record=True)
    sim.set_problem(prob)
    sim.set_trace(tr.arrival_ns, tr.model)
    sim.set_chunk_size(chunk)
    try:
        gs, _ = stepwise(sim, dedup=False, prune=False)
    finally:
        sim.set_chunk_size(4096)
    _compare_steps(gs, ref["runs"], False)


def test_search_more_than_64_models(sim):
    """M > 64: no component restriction (model masks are 64-bit), and late
    steps simulate fewer candidates than there are active runs -- the search
    must still take the chunked path whose boundary states it publishes
    (a general-kernel step left stale chunk buffers)."""
    names = [f"BERT-1.3B#{i}" for i in range(70)]
    prob = configs.build_problem(names, 8, 13 * 10**9, slo_scale=5.0)
    w = np.linspace(1.0, 0.2, 70)
    tr = traces.independent_gamma(5, list(0.05 * w), 2.0, 400.0)
    for chunk in (4096, 23):
        sim.set_problem(prob)
        sim.set_trace(tr.arrival_ns, tr.model)
        sim.set_chunk_size(chunk)
        try:
            _compare(sim, prob, tr, dedup_modes=(False,))
        finally:
            sim.set_chunk_size(4096)


def test_greedy_hand_case_ties_and_strict_best(sim):
    """The GPU search on the hand-worked case of
    test_oracle_pins.test_greedy_ties_and_strict_best_hand_case."""
    from tests.helpers import tiny_problem, trace_of

    prob = tiny_problem([(1, 1)], stage=[[[10]], [[10]]], mem=[[6], [6]], num_devices=2,
                        budget=10)
    for pairs, hist, best, mask in (([(0, 0), (100, 1)], [(0, 0, 1), (1, 1, 2)], 2, [1, 2]),
                                    ([(0, 0)], [(0, 0, 1), (0, 1, 1)], 1, [1, 0])):
        tr = trace_of(pairs)
        sim.set_problem(prob)
        sim.set_trace(tr.arrival_ns, tr.model)
        with sim.search_handle(runs=[[0, 0]], dedup=False, prune=False) as h:
            h.run()
            m, g, v = h.history(0)
            assert list(zip(m.tolist(), g.tolist(), v.tolist())) == hist
            res = h.result()
        assert res.best_good == best and res.host_mask.tolist() == mask


def test_feasibility_hand_cases_gpu(sim):
    """Infeasible placements are data (good = -1), every branch of reading C11
    as in test_oracle_pins.test_feasibility_branches_hand_cases."""
    from tests.helpers import place, tiny_problem, trace_of

    prob = tiny_problem([(1, 1), (2, 1)], stage=[[[5], [2, 3]]] * 3,
                        mem=[[6, 3], [-1, 4], [5, 3]], num_devices=2, budget=10)
    cases = [([0, 0], [[0], [0]], True), ([0, 0], [[0, 2], []], False),
             ([0, 0], [[2], [0]], True), ([0, -1], [[1], []], False),
             ([1, -1], [[0, 1, 2], []], True), ([1, 1], [[0], []], False)]
    tr = trace_of([(0, 0), (1, 1), (2, 2)])
    sim.set_problem(prob)
    sim.set_trace(tr.arrival_ns, tr.model)
    cfg = np.full((len(cases), 3), -1, np.int32)
    mask = np.zeros((len(cases), 3), np.uint64)
    for i, (c, groups, _) in enumerate(cases):
        pl = place([x for x in c if x >= 0], [gm for x, gm in zip(c, groups) if x >= 0], 3)
        cfg[i, :pl.num_groups] = pl.group_cfg
        mask[i] = pl.host_mask
    got = sim.evaluate(cfg, mask)["good"]
    assert [(x >= 0) for x in got] == [w for _, _, w in cases]
    assert all(x == -1 for x, (_, _, w) in zip(got, cases) if not w)
