"""GPU parity of the chunked throughput path (chunk.cu): speculative time
chunks from the idle state + exact fix-up + re-run chains must give the same
integers as the oracle for every chunk size, in both time representations
(uint32 epoch-relative and int64 absolute), for every stage class
(S = 1, 2, 4, 8, 16 and the dynamic path)."""

import numpy as np
import pytest

import oracle
from workloads import Placement, Trace, configs
from tests.helpers import INF, tiny_problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sim():
    from paper_2302_11665_b200 import Simulator
    s = Simulator(0)
    yield s
    s.close()


def _delta_batch(rng, prob, bases, per_base=40):
    """Random greedy-step-like candidates: base + (m, g), sorted like a step."""
    M = prob.num_models
    G = max(b.num_groups for b in bases)
    bc = np.full((len(bases), G), -1, np.int32)
    bm = np.zeros((len(bases), M), np.uint64)
    for i, b in enumerate(bases):
        bc[i, :b.num_groups] = b.group_cfg
        bm[i] = b.host_mask
    cb, cm, cg = [], [], []
    for i, b in enumerate(bases):
        for _ in range(per_base):
            cb.append(i)
            cm.append(int(rng.integers(-1, M)))
            cg.append(int(rng.integers(0, b.num_groups)))
    cb, cm, cg = (np.array(x, np.int32) for x in (cb, cm, cg))
    order = np.lexsort((cg, cm, cb))
    cb, cm, cg = cb[order], cm[order], cg[order]
    full_cfg = bc[cb]
    full_mask = bm[cb].copy()
    for c in range(len(cb)):
        if cm[c] >= 0:
            full_mask[c, cm[c]] |= np.uint64(1) << np.uint64(cg[c])
    return bc, bm, cb, cm, cg, full_cfg, full_mask


def _check(sim, prob, tr, bases, rng, chunk_sizes=(1, 13, 257, 4096), per_base=40):
    bc, bm, cb, cm, cg, fcfg, fmask = _delta_batch(rng, prob, bases, per_base)
    want_g, want_s, _ = oracle.evaluate(prob, tr, fcfg, fmask)
    sim.set_problem(prob)
    sim.set_trace(tr.arrival_ns, tr.model)
    sim.set_path(2)
    try:
        for L in chunk_sizes:
            sim.set_chunk_size(L)
            got = sim.evaluate_deltas(bc, bm, cb, cm, cg)
            np.testing.assert_array_equal(got["good"], want_g, err_msg=f"chunk {L}")
            np.testing.assert_array_equal(got["sum_latency_ns"], want_s, err_msg=f"chunk {L}")
            assert got["argmax"] == (int(np.argmax(want_g)) if want_g.max() >= 0 else -1)
    finally:
        sim.set_path(0)
        sim.set_chunk_size(4096)


def _uniform_bases(rng, prob, p, G, k, p_host):
    out = []
    for _ in range(k):
        groups = [[m for m in range(prob.num_models) if rng.random() < p_host] for _ in range(G)]
        out.append(Placement.from_lists([p] * G, groups, prob.num_models))
    return out


def _bursty_trace(rng, M, n, mean_gap):
    gaps = rng.gamma(1 / 9.0, 9.0 * mean_gap, size=n)  # CV 3
    a = np.floor(np.cumsum(gaps)).astype(np.int64)
    return Trace(a, rng.integers(0, M, size=n).astype(np.int32))


@pytest.mark.parametrize("S", [1, 2, 4, 8, 16, 3])
@pytest.mark.parametrize("u32", [True, False])
def test_stage_classes(sim, S, u32):
    rng = np.random.default_rng(1000 + S + 100 * u32)
    M = 5
    stage = [[list(rng.integers(1, 400 // S + 2, size=S))] for _ in range(M)]
    slo = [int(rng.integers(300, 3000)) for _ in range(M)]
    if not u32:
        slo[0] = INF  # an unbounded SLO forces int64 times
    prob = tiny_problem([(S, 1)], stage, tail=rng.integers(0, 50, size=(M, 1)), slo=slo)
    tr = _bursty_trace(rng, M, 2500, 60.0)
    G = max(1, min(64 // S, 8))
    bases = _uniform_bases(rng, prob, 0, G, 3, 0.4)
    _check(sim, prob, tr, bases, rng)


def test_dynamic_mixed_configs(sim):
    rng = np.random.default_rng(77)
    M = 4
    cfgs = [(1, 1), (3, 1), (2, 1)]
    stage = [[list(rng.integers(1, 60, size=s)) for s, _ in cfgs] for _ in range(M)]
    prob = tiny_problem(cfgs, stage, slo=[int(rng.integers(50, 400)) for _ in range(M)])
    tr = _bursty_trace(rng, M, 3000, 15.0)
    bases = []
    for _ in range(3):
        G = int(rng.integers(2, 9))
        cfg = rng.integers(0, 3, size=G)
        groups = [[m for m in range(M) if rng.random() < 0.4] for _ in range(G)]
        bases.append(Placement.from_lists(cfg, groups, M))
    _check(sim, prob, tr, bases, rng)


def test_overload_rerun_chains(sim):
    """Sustained overload with a loose SLO: queues never drain, so chunk
    starts from idle never meet the true trajectory -> re-run chains; the
    result must still be exact."""
    rng = np.random.default_rng(78)
    prob = tiny_problem([(2, 1)], [[[30, 20]]], slo=[10**7])
    a = np.sort(rng.integers(0, 20 * 3000, size=3000)).astype(np.int64)  # rate 1/20 > 1/30
    tr = Trace(a, np.zeros(3000, np.int32))
    bases = [Placement.from_lists([0, 0], [[0], []], 1)]
    sim.set_profiling(True)
    sim.reset_stats()
    _check(sim, prob, tr, bases, rng, chunk_sizes=(50, 300), per_base=6)
    assert sim.stats()["chunk_reruns"] > 0
    sim.set_profiling(False)


def test_s3_shaped_steps(sim):
    prob, tr = configs.s3(duration=240.0)
    rng = np.random.default_rng(79)
    bases = []
    for size in (1, 2, 4):
        ps = [p for p, (s, n) in enumerate(prob.configs) if s * n == size]
        for p in ps[:2]:
            bases += _uniform_bases(rng, prob, p, 64 // size, 1, 0.06)
    _check(sim, prob, tr, bases, rng, chunk_sizes=(97, 4096), per_base=33)


def test_s4_shaped_int64(sim):
    prob, tr = configs.s4(duration=4 * 3600.0)
    rng = np.random.default_rng(80)
    bases = [Placement.from_lists([4] * 4, [[0], [1], [2], [3]], 4),
             Placement.from_lists([5] * 2, [[0, 1], [2, 3]], 4)]
    _check(sim, prob, tr, bases, rng, chunk_sizes=(500, 4096), per_base=8)


def test_search_same_on_both_paths(sim):
    """The whole search through the general kernel and the chunked kernel."""
    names = [f"{b}#{i}" for b in ("BERT-1.3B", "MoE-2.4B", "BERT-6.7B") for i in range(2)]
    prob = configs.build_problem(names, 8, 13 * 10**9, slo_scale=4.0)
    from workloads import traces
    tr = traces.maf2_shaped(9, len(names), 15.0, 600.0)
    sim.set_problem(prob)
    sim.set_trace(tr.arrival_ns, tr.model)
    res = {}
    for path, L in [(1, 4096), (2, 64), (2, 4096)]:
        sim.set_path(path)
        sim.set_chunk_size(L)
        r = sim.search(dedup=False)
        res[(path, L)] = (r.best_good, r.best_run, r.host_mask.tolist(),
                          [x["best_good"] for x in r.runs])
    sim.set_path(0)
    sim.set_chunk_size(4096)
    vals = list(res.values())
    assert all(v == vals[0] for v in vals)


@pytest.mark.parametrize("scale", [1.0, 2.0, 5.0])
def test_epoch_rebase_long_gaps(sim, scale):
    """uint32 epochs with gaps longer than 2^32 - theta (sparse, bursty
    arrivals): the epoch move must clear every stored free time."""
    prob = configs.motivating_problem(slo_scale=scale)
    rng = np.random.default_rng(int(scale * 10))
    gaps = rng.gamma(1 / 16.0, 16.0 * 1.2e9, size=4000)  # mean 1.2 s, CV 4
    a = np.floor(np.cumsum(gaps)).astype(np.int64)
    tr = Trace(a, rng.integers(0, 2, size=4000).astype(np.int32))
    bases = [Placement.from_lists([0, 0], [[0], [1]], 2), Placement.from_lists([2], [[0]], 2),
             Placement.from_lists([1], [[1]], 2)]
    _check(sim, prob, tr, bases, rng, chunk_sizes=(37, 4096), per_base=12)


def test_uniform_config_with_empty_group_slot(sim):
    """A base whose groups share one config but with an unused group id
    (cfg -1) in between: the uniform kernels address stages at g * S, so such
    a base must take the group-table path -- results stay oracle-exact."""
    rng = np.random.default_rng(79)
    M = 4
    prob = tiny_problem([(2, 1)], [[list(rng.integers(1, 40, size=2))] for _ in range(M)],
                        slo=[int(rng.integers(60, 300)) for _ in range(M)])
    tr = _bursty_trace(rng, M, 3000, 12.0)
    cfg = np.array([0, -1, 0, 0], np.int32)
    mask = np.zeros(M, np.uint64)
    for m in range(M):
        for g in (0, 2, 3):
            if rng.random() < 0.5:
                mask[m] |= np.uint64(1) << np.uint64(g)
    cb, cm, cg = [], [], []
    for m in range(-1, M):
        for g in (0, 2, 3):
            if m >= 0 and (int(mask[m]) >> g) & 1:
                continue
            cb.append(0), cm.append(m), cg.append(g)
    cb, cm, cg = (np.array(x, np.int32) for x in (cb, cm, cg))
    fcfg = np.tile(cfg, (len(cb), 1))
    fmask = np.tile(mask, (len(cb), 1))
    for c in range(len(cb)):
        if cm[c] >= 0:
            fmask[c, cm[c]] |= np.uint64(1) << np.uint64(cg[c])
    want_g, want_s, _ = oracle.evaluate(prob, tr, fcfg, fmask)
    sim.set_problem(prob)
    sim.set_trace(tr.arrival_ns, tr.model)
    for path in (0, 2):
        sim.set_path(path)
        try:
            for L in (64, 4096):
                sim.set_chunk_size(L)
                got = sim.evaluate_deltas(cfg[None, :], mask[None, :], cb, cm, cg)
                np.testing.assert_array_equal(got["good"], want_g)
                np.testing.assert_array_equal(got["sum_latency_ns"], want_s)
        finally:
            sim.set_path(0)
            sim.set_chunk_size(4096)


def _sim_env(env):
    import os
    from paper_2302_11665_b200 import Simulator
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return Simulator(0)
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


@pytest.fixture(scope="module")
def sim_coop():
    """A context whose walk uses only the cooperative walker (the scalar
    register walker switched off), so both walkers stay covered."""
    s = _sim_env({"ASIM_SCALAR_WALK": "0"})
    yield s
    s.close()


@pytest.fixture(scope="module", params=[{"ASIM_GLANE_WALK": "0"},
                                        {"ASIM_GLANE_WALK": "1", "ASIM_GLANE_SMAX": "16"}],
                ids=["glane-off", "glane-all"])
def sim_glane(request):
    """Group-lane walker off (the scalar walker takes every small component)
    and on for every uniform component of <= 32 groups (one group too)."""
    s = _sim_env(request.param)
    yield s
    s.close()


@pytest.mark.parametrize("S", [1, 2, 4, 8, 16])
@pytest.mark.parametrize("u32", [True, False])
def test_stage_classes_group_lane_walker(sim_glane, S, u32):
    test_stage_classes(sim_glane, S, u32)


def test_overload_chains_group_lane_walker(sim_glane):
    test_overload_rerun_chains(sim_glane)
    test_search_same_on_both_paths(sim_glane)
    test_epoch_rebase_long_gaps(sim_glane, 2.0)


@pytest.mark.parametrize("S", [1, 2, 8])
@pytest.mark.parametrize("u32", [True, False])
def test_stage_classes_cooperative_walker(sim_coop, S, u32):
    test_stage_classes(sim_coop, S, u32)


def test_overload_chains_cooperative_walker(sim_coop):
    test_overload_rerun_chains(sim_coop)
    test_search_same_on_both_paths(sim_coop)
