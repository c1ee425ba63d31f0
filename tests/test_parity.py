"""GPU parity: libasim.so (CUDA, sm_100a) vs the CPU oracle, element by
element -- good, sum_latency_ns, good_per_model and argmax must be identical
(integers; SURVEY §8(c) "Parity").  Instance families F1-F6."""

import numpy as np
import pytest

import oracle
from oracle import search as osearch
from workloads import Placement, Trace, configs
from tests.helpers import INF, tiny_problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sim():
    from paper_2302_11665_b200 import Simulator
    s = Simulator(0)
    yield s
    s.close()


def _stack(placements, M):
    G = max([p.num_groups for p in placements] + [1])
    cfg = np.full((len(placements), G), -1, np.int32)
    mask = np.zeros((len(placements), M), np.uint64)
    for i, p in enumerate(placements):
        cfg[i, :p.num_groups] = p.group_cfg
        mask[i] = p.host_mask
    return cfg, mask


def check_full(sim, prob, tr, placements):
    cfg, mask = _stack(placements, prob.num_models)
    sim.set_problem(prob)
    sim.set_trace(tr.arrival_ns, tr.model)
    got = sim.evaluate(cfg, mask, per_model=True)
    g, s, pm = oracle.evaluate(prob, tr, cfg, mask, per_model=True)
    np.testing.assert_array_equal(got["good"], g)
    np.testing.assert_array_equal(got["sum_latency_ns"], s)
    np.testing.assert_array_equal(got["good_per_model"], pm)
    want_arg = int(np.argmax(g)) if len(g) and g.max() >= 0 else -1
    assert got["argmax"] == want_arg
    return g


def _rand_placements(rng, prob, k, G, p_hosted=0.5):
    out = []
    for _ in range(k):
        cfg = rng.integers(0, prob.num_configs, size=G).astype(np.int32)
        slots = np.cumsum([prob.configs[c][0] for c in cfg])
        Gk = int(np.searchsorted(slots, 128, side="right"))
        cfg = cfg[:max(Gk, 1)]
        groups = [[m for m in range(prob.num_models) if rng.random() < p_hosted]
                  for _ in range(len(cfg))]
        out.append(Placement.from_lists(cfg, groups, prob.num_models))
    return out


def _rand_trace(rng, M, n, tmax, dup=True):
    if dup:
        a = np.sort(rng.integers(0, tmax, size=n))
    else:
        a = np.sort(rng.choice(tmax, size=n, replace=False))
    return Trace(a.astype(np.int64), rng.integers(0, M, size=n).astype(np.int32))


# ----------------------------------------------------------------------------- F1
def test_f1_single_group_single_model(sim):
    rng = np.random.default_rng(101)
    for _ in range(40):
        s = int(rng.integers(1, 9))
        d = list(rng.integers(0, 8, size=s))
        slo = int(rng.choice([0, 3, 10, 40, 10**12, INF]))
        prob = tiny_problem([(s, 1)], [[d]], tail=[[int(rng.integers(0, 4))]], slo=[slo])
        tr = _rand_trace(rng, 1, int(rng.integers(1, 300)), 400)
        check_full(sim, prob, tr, [Placement.from_lists([0], [[0]], 1)] * 3)


# ----------------------------------------------------------------------------- F2
def test_f2_replicas_and_bursts(sim):
    rng = np.random.default_rng(102)
    for _ in range(30):
        s = int(rng.integers(1, 4))
        d = [int(rng.integers(1, 5))] * s
        prob = tiny_problem([(s, 1)], [[d]], slo=[int(rng.choice([2, 6, 12, INF]))])
        bursts = np.repeat(np.sort(rng.integers(0, 200, size=20)), rng.integers(1, 8, size=20))
        tr = Trace(bursts.astype(np.int64), np.zeros(len(bursts), np.int32))
        pls = [Placement.from_lists([0] * G, [[0]] * G, 1) for G in range(1, 9)]
        check_full(sim, prob, tr, pls)


# ----------------------------------------------------------------------------- F3
def test_f3_mixed_models_configs(sim):
    rng = np.random.default_rng(103)
    for it in range(30):
        M = int(rng.integers(1, 8))
        P = int(rng.integers(1, 5))
        cfgs = [(int(rng.integers(1, 17)), 1) for _ in range(P)]
        stage = [[list(rng.integers(0, 30, size=s)) for s, _ in cfgs] for _ in range(M)]
        tail = rng.integers(0, 5, size=(M, P))
        slo = [int(rng.choice([0, 20, 60, 200, INF])) for _ in range(M)]
        prob = tiny_problem(cfgs, stage, tail, slo)
        n = int(rng.integers(0, 700))
        tr = _rand_trace(rng, M, n, 3000)
        G = int(rng.integers(1, 65))
        pls = _rand_placements(rng, prob, 40, G, p_hosted=float(rng.uniform(0.05, 0.6)))
        check_full(sim, prob, tr, pls)


# ----------------------------------------------------------------------------- F4
def test_f4_homogeneous_groups(sim):
    rng = np.random.default_rng(104)
    for _ in range(20):
        M = int(rng.integers(1, 5))
        s = int(rng.integers(1, 6))
        d = list(rng.integers(1, 10, size=s))
        prob = tiny_problem([(s, 1)], [[d]] * M, slo=[int(rng.integers(5, 80)) for _ in range(M)])
        tr = _rand_trace(rng, M, 500, 2000)
        pls = _rand_placements(rng, prob, 33, int(rng.integers(1, 20)), 0.4)
        check_full(sim, prob, tr, pls)


# ----------------------------------------------------------------------------- F5
def test_f5_near_bounds(sim):
    rng = np.random.default_rng(105)
    big = 2**40
    prob = tiny_problem([(2, 1), (1, 1)], [[[big, big // 3], [big]], [[7, 3], [5]]],
                        tail=[[big // 7, 0], [1, 2]], slo=[3 * big, INF])
    n = 300
    top = 2**62 - (n + 1) * (2 * big)
    a = np.sort(rng.integers(top - 10**6 * big // 2**20, top, size=n)).astype(np.int64)
    tr = Trace(a, rng.integers(0, 2, size=n).astype(np.int32))
    pls = _rand_placements(rng, prob, 40, 6, 0.5)
    check_full(sim, prob, tr, pls)


# ----------------------------------------------------------------------------- F6
def test_f6_motivating_all_17(sim):
    prob = configs.motivating_problem(slo_scale=1.5)
    tr = configs.motivating_trace(seed=0, n_requests=1000)
    bf = osearch.bruteforce(prob, tr)
    g = check_full(sim, prob, tr, bf["placements"])
    assert len(g) == 17


def test_f6_fig1_burst(sim):
    y = 400_000_000
    prob = tiny_problem([(1, 1), (2, 1)], [[[y], [y // 2, y // 2]]], tail=[[0, y // 10]])
    tr = Trace(np.zeros(4, np.int64), np.zeros(4, np.int32))
    g = check_full(sim, prob, tr, [Placement.from_lists([0], [[0]], 1),
                                   Placement.from_lists([1], [[0]], 1)])
    assert list(g) == [4, 4]


def test_f6_s1_shaped(sim):
    prob, tr = configs.s1(duration=120.0)
    rng = np.random.default_rng(106)
    pls = []
    for G, p in [(16, 0), (8, 1), (8, 2), (4, 5), (2, 9)]:
        groups = [[m for m in range(prob.num_models) if rng.random() < 0.3] for _ in range(G)]
        pls.append(Placement.from_lists([p] * G, groups, prob.num_models))
    check_full(sim, prob, tr, pls)


def test_f6_s3_prefix(sim):
    prob, tr = configs.s3(duration=300.0)
    rng = np.random.default_rng(107)
    pls = []
    for _ in range(6):
        size = int(rng.choice([1, 2, 4, 8]))
        ps = [p for p, (s, n) in enumerate(prob.configs) if s * n == size]
        p = int(rng.choice(ps))
        G = 64 // size
        groups = [[m for m in range(prob.num_models) if rng.random() < 0.1] for _ in range(G)]
        pls.append(Placement.from_lists([p] * G, groups, prob.num_models))
    check_full(sim, prob, tr, pls)


def test_f6_s4_day_prefix(sim):
    prob, tr = configs.s4(duration=6 * 3600.0)
    pls = []
    for p, G in [(4, 4), (5, 2), (6, 1)]:
        groups = [[m for m in range(4) if (m + g) % 2 == 0 or G == 1] for g in range(G)]
        pls.append(Placement.from_lists([p] * G, groups, 4))
    check_full(sim, prob, tr, pls)


# ----------------------------------------------------------------------------- deltas
def test_deltas_match_full(sim):
    rng = np.random.default_rng(108)
    for _ in range(15):
        M = int(rng.integers(1, 6))
        cfgs = [(int(rng.integers(1, 5)), 1) for _ in range(3)]
        stage = [[list(rng.integers(1, 20, size=s)) for s, _ in cfgs] for _ in range(M)]
        mem = rng.integers(1, 6, size=(M, 3))
        prob = tiny_problem(cfgs, stage, slo=[int(rng.integers(10, 100)) for _ in range(M)],
                            mem=mem, budget=9)
        tr = _rand_trace(rng, M, 400, 3000)
        B, G = 3, int(rng.integers(1, 9))
        bases = _rand_placements(rng, prob, B, G, 0.3)
        Gm = max(b.num_groups for b in bases)
        bc, bm = _stack(bases, M)
        cb, cm, cg, full = [], [], [], []
        for b, base in enumerate(bases):
            for m in range(-1, M):
                for g in range(base.num_groups):
                    cb.append(b)
                    cm.append(m)
                    cg.append(g)
                    mask = base.host_mask.copy()
                    if m >= 0:
                        mask[m] |= np.uint64(1) << np.uint64(g)
                    pc = np.full(Gm, -1, np.int32)
                    pc[:base.num_groups] = base.group_cfg
                    full.append(Placement(pc, mask))
        sim.set_problem(prob)
        sim.set_trace(tr.arrival_ns, tr.model)
        got = sim.evaluate_deltas(bc, bm, cb, cm, cg, per_model=True)
        cfg, mask = _stack(full, M)
        g, s, pm = oracle.evaluate(prob, tr, cfg, mask, per_model=True)
        np.testing.assert_array_equal(got["good"], g)
        np.testing.assert_array_equal(got["sum_latency_ns"], s)
        np.testing.assert_array_equal(got["good_per_model"], pm)


def test_empty_trace_and_errors(sim):
    from paper_2302_11665_b200 import AsimError
    prob = tiny_problem([(1, 1)], [[[5]]])
    sim.set_problem(prob)
    sim.set_trace(np.zeros(0, np.int64), np.zeros(0, np.int32))
    got = sim.evaluate(np.zeros((2, 1), np.int32), np.array([[1], [0]], np.uint64))
    assert list(got["good"]) == [0, 0]
    with pytest.raises(AsimError) as e:
        sim.set_trace(np.array([5, 3], np.int64), np.zeros(2, np.int32))
    assert e.value.status == -2
    with pytest.raises(AsimError) as e:
        sim.set_trace(np.array([1], np.int64), np.array([4], np.int32))
    assert e.value.status == -3
    sim.set_trace(np.array([1, 2], np.int64), np.zeros(2, np.int32))
    with pytest.raises(AsimError) as e:  # mask bit on a missing group
        sim.evaluate(np.array([[0, -1]], np.int32), np.array([[2]], np.uint64))
    assert e.value.status == -3
