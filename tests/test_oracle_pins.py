"""Pins: the CPU oracle checked against what the paper and mathematics fix
(SURVEY §8(c) P1-P14).  None of these retypes the oracle's event loop: each
compares it to a printed value, a closed form, an independent recursion, or a
hand-worked case.
"""

import json
import os

import numpy as np
import pytest

import oracle
from workloads import Trace, configs, traces
from tests.helpers import INF, place, random_instance, tiny_problem, trace_of

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ----------------------------------------------------------------------------- P1
def test_p1_fig1_worked_example():
    """(1y+2y+3y+4y)/4 = 2.5y simple; (1.1y+1.6y+2.1y+2.6y)/4 = 1.85y."""
    g = _gold("fig1_worked_example.json")
    y = g["y_ns"]
    prob = tiny_problem([(1, 1), (2, 1)], [[[y], [y // 2, y // 2]]],
                        tail=[[0, y // 10]])
    tr = trace_of([(0, 0)] * 4)
    simple = oracle.simulate(prob, tr, place([0], [[0]], 1), detail=True)
    pipe = oracle.simulate(prob, tr, place([1], [[0]], 1), detail=True)
    assert list(simple["finish_ns"]) == [round(v * y) for v in g["simple_finish_over_y"]]
    assert list(pipe["finish_ns"]) == [round(v * y) for v in g["pipeline_finish_over_y"]]
    assert simple["sum_latency_ns"] / 4 == g["simple_mean_over_y"] * y
    assert pipe["sum_latency_ns"] / 4 == pytest.approx(g["pipeline_mean_over_y"] * y, abs=0)


# ----------------------------------------------------------------------------- P2
@pytest.mark.parametrize("d", [[3, 1], [1, 3], [2, 5, 1], [1, 1, 7, 2], [0, 4, 0]])
@pytest.mark.parametrize("tail", [0, 5])
def test_p2_burst_identity(d, tail):
    """Pipeline throughput = 1 / max stage latency: a burst of n
    simultaneous requests finishes at a + sum(d) + tail + i*max(d)."""
    prob = tiny_problem([(len(d), 1)], [[d]], tail=[[tail]])
    a0 = 100
    tr = trace_of([(a0, 0)] * 6)
    r = oracle.simulate(prob, tr, place([0], [[0]], 1), detail=True)
    want = [a0 + sum(d) + tail + i * max(d) for i in range(6)]
    assert list(r["finish_ns"]) == want


# ----------------------------------------------------------------------------- P3
def _scalar_state_sim(prob, tr, pl):
    """Independent closed form for groups whose hosted models share one stage
    vector d: departure = max(a + sum d, F + max d) (tandem deterministic line
    bottleneck), F = last accepted departure; R2 dispatch, receipt-time SLO."""
    F = {}
    fin = np.full(len(tr), -1, np.int64)
    for i, (a, m) in enumerate(zip(tr.arrival_ns.tolist(), tr.model.tolist())):
        best = None
        for g in pl.hosts(m):
            p = int(pl.group_cfg[g])
            s = prob.configs[p][0]
            d = prob.stage_ns[m, p, :s].tolist()
            dep = max(a + sum(d), F.get(g, 0) + max(d))
            f = dep + int(prob.tail_ns[m, p])
            if best is None or f < best[0]:
                best = (f, g, dep)
        if best is None or best[0] - a > prob.slo_ns[m]:
            continue
        F[best[1]] = best[2]
        fin[i] = best[0]
    return fin


def test_p3_scalar_state_identity():
    rng = np.random.default_rng(3)
    checked = 0
    for _ in range(400):
        s = int(rng.integers(1, 5))
        d = list(rng.integers(0, 6, size=s))
        M = int(rng.integers(1, 3))
        tail = int(rng.integers(0, 3))
        slo = [int(rng.choice([0, 4, 9, 15, INF])) for _ in range(M)]
        prob = tiny_problem([(s, 1)], [[d]] * M, tail=[[tail]] * M, slo=slo)
        G = int(rng.integers(1, 4))
        groups = [[m for m in range(M) if rng.random() < 0.7] for _ in range(G)]
        pl = place([0] * G, groups, M)
        n = int(rng.integers(1, 30))
        a = np.sort(rng.integers(0, 25, size=n)).astype(np.int64)
        tr = Trace(a, rng.integers(0, M, size=n).astype(np.int32))
        r = oracle.simulate(prob, tr, pl, detail=True)
        assert np.array_equal(r["finish_ns"], _scalar_state_sim(prob, tr, pl))
        checked += 1
    assert checked == 400


# ----------------------------------------------------------------------------- P4
def test_p4_lindley_recursion():
    """One (1,1) group, one model, no deadline: fin_i = max(a_i, fin_{i-1}) + D."""
    rng = np.random.default_rng(4)
    for _ in range(50):
        D = int(rng.integers(1, 50))
        a = np.sort(rng.integers(0, 500, size=200)).astype(np.int64)
        prob = tiny_problem([(1, 1)], [[[D]]])
        r = oracle.simulate(prob, Trace(a, np.zeros(200, np.int32)), place([0], [[0]], 1),
                            detail=True)
        fin, prev = [], 0
        for x in a.tolist():
            prev = max(x, prev) + D
            fin.append(prev)
        assert list(r["finish_ns"]) == fin


# ----------------------------------------------------------------------------- P5
@pytest.mark.parametrize("rho", [0.3, 0.6, 0.9])
def test_p5_md1_mean_latency(rho):
    """M/D/1 mean latency W = D + lambda D^2 / (2 (1 - lambda D))."""
    D = 0.4
    lam = rho / D
    n = 400_000 if rho < 0.85 else 1_000_000
    tr = traces.independent_gamma(5, [lam], 1.0, n / lam * 1.02).prefix(n)
    prob = tiny_problem([(1, 1)], [[[int(D * 1e9)]]])
    r = oracle.simulate(prob, tr, place([0], [[0]], 1))
    assert r["good"] == len(tr)
    W = r["sum_latency_ns"] / r["good"] / 1e9
    W_md1 = D + lam * D * D / (2 * (1 - lam * D))
    assert W == pytest.approx(W_md1, rel=0.03)


# ----------------------------------------------------------------------------- P6/P7
def _mean_latency(prob, tr, pl):
    r = oracle.simulate(prob, tr, pl)
    assert r["good"] == len(tr)  # no deadline: everything served
    return r["sum_latency_ns"] / r["good"] / 1e9


def test_p6_motivating_means():
    """simple 0.70 s -> 2-stage model-parallel 0.55 s (Poisson 1.5+1.5,
    D=0.4); the closed forms W_simple, W_pipeline agree."""
    g = _gold("motivating_means.json")
    prob = configs.motivating_problem(slo_scale=1e6)
    tr = configs.motivating_trace(seed=6, n_requests=600_000)
    simple = _mean_latency(prob, tr, place([0, 0], [[0], [1]], 2))
    pipe = _mean_latency(prob, tr, place([2], [[0, 1]], 2))
    assert simple == pytest.approx(g["simple_mean_s"], rel=0.03)
    assert pipe == pytest.approx(g["pipeline_mean_s"], rel=0.03)
    D, lam = 0.4, 3.0
    W_simple = D + lam * D * D / (4 - 2 * lam * D)
    W_pipe = D + lam * D * D / (8 - 4 * lam * D)
    assert simple == pytest.approx(W_simple, rel=0.03)
    assert pipe == pytest.approx(W_pipe, rel=0.03)


@pytest.mark.parametrize("beta", [1.2, 1.5])
def test_p7_uneven_stages_w_pipeline(beta):
    """P:512-514 with D_s = D and D_m = beta D / 2: mean latency of the
    merged Poisson stream on a 2-stage pipeline = D_s + lam D_m^2/(2(1-lam D_m))."""
    D, lam = 0.4, 3.0
    Dm = beta * D / 2
    stages = [int(round(Dm * 1e9)), int(round((D - Dm) * 1e9))]
    prob = tiny_problem([(2, 1)], [[stages], [stages]])
    n = 300_000 if beta < 1.4 else 2_000_000  # rho_m = 0.9 at beta 1.5: slow convergence
    tr = traces.independent_gamma(7, [lam / 2, lam / 2], 1.0, n / lam)
    W = _mean_latency(prob, tr, place([0], [[0, 1]], 2))
    W_pipe = D + lam * Dm * Dm / (2 * (1 - lam * Dm))
    assert W == pytest.approx(W_pipe, rel=0.03)


# ----------------------------------------------------------------------------- P8
def test_p8_infinite_slo_all_good():
    rng = np.random.default_rng(8)
    for _ in range(100):
        prob, tr, pl = random_instance(rng, slo_choices=[INF], allow_unhosted=True)
        r = oracle.simulate(prob, tr, pl)
        hosted = [m for m in range(prob.num_models) if int(pl.host_mask[m])]
        assert r["good"] == int(np.isin(tr.model, hosted).sum())
    prob, tr, pl = random_instance(rng, slo_choices=[INF], allow_unhosted=False)
    assert oracle.simulate(prob, tr, pl)["good"] == len(tr)


# ----------------------------------------------------------------------------- P9
def test_p9_monotone_in_slo_single_model():
    """Attainment non-decreasing in SLO for single-model instances (any groups,
    stages, replicas); reading C18."""
    rng = np.random.default_rng(9)
    for _ in range(300):
        G = int(rng.integers(1, 4))
        P = int(rng.integers(1, 3))
        cfgs = [(int(rng.integers(1, 4)), 1) for _ in range(P)]
        stage = [[list(rng.integers(1, 4, size=s)) for s, _ in cfgs]]
        tail = rng.integers(0, 2, size=(1, P))
        n = int(rng.integers(1, 9))
        tr = Trace(np.sort(rng.integers(0, 6, size=n)).astype(np.int64), np.zeros(n, np.int32))
        cfg = [int(rng.integers(0, P)) for _ in range(G)]
        pl = place(cfg, [[0]] * G, 1)
        prev = -1
        for slo in range(0, 31, 2):
            prob = tiny_problem(cfgs, stage, tail, [slo])
            g = oracle.simulate(prob, tr, pl)["good"]
            assert g >= prev
            prev = g


def test_p9_mixed_model_counterexample():
    """Reading C18: with two models, attainment is NOT monotone in SLO scale.
    One (1,1) group; A (D=10), B (D=100); A@0, B@5, A@20..100 step 10.
    Scale 1.0 -> 10/11 good (B rejected: 105 > 100); scale 1.1 -> 2/11."""
    arr = [(0, 0), (5, 1)] + [(t, 0) for t in range(20, 101, 10)]
    tr = trace_of(arr)
    pl = place([0], [[0, 1]], 2)
    p1 = tiny_problem([(1, 1)], [[[10]], [[100]]], slo=[10, 100])
    p2 = tiny_problem([(1, 1)], [[[10]], [[100]]], slo=[11, 110])
    assert oracle.simulate(p1, tr, pl)["good"] == 10
    assert oracle.simulate(p2, tr, pl)["good"] == 2


# ----------------------------------------------------------------------------- P10
def test_p10a_dispatch_ties_lowest_index():
    """Two (1,1) groups host A (d=10); three requests at t=0 go to g0, g1, g0
    and finish 10, 10, 20; with slo 15 the third is rejected."""
    prob = tiny_problem([(1, 1)], [[[10]]], slo=[INF])
    tr = trace_of([(0, 0)] * 3)
    r = oracle.simulate(prob, tr, place([0, 0], [[0], [0]], 1), detail=True)
    assert list(r["served_by"]) == [0, 1, 0]
    assert list(r["finish_ns"]) == [10, 10, 20]
    prob15 = tiny_problem([(1, 1)], [[[10]]], slo=[15])
    r = oracle.simulate(prob15, tr, place([0, 0], [[0], [0]], 1), detail=True)
    assert r["good"] == 2 and list(r["served_by"]) == [0, 1, -1]


def test_p10b_dispatch_earliest_predicted_finish():
    """g0 (1,1) d=[10]; g1 (2,1) d=[6,6] tail 1; four requests at t=0:
    predictions g0:10 vs g1:13 -> g0; g0:20 vs g1:13 -> g1; g0:20 vs g1:19 -> g1;
    g0:20 vs g1:25 -> g0.  Finishes 10, 13, 19, 20."""
    prob = tiny_problem([(1, 1), (2, 1)], [[[10], [6, 6]]], tail=[[0, 1]])
    tr = trace_of([(0, 0)] * 4)
    r = oracle.simulate(prob, tr, place([0, 1], [[0], [0]], 1), detail=True)
    assert list(r["served_by"]) == [0, 1, 1, 0]
    assert list(r["finish_ns"]) == [10, 13, 19, 20]


def test_p10c_equals_jsq_for_single_stage_equal_d():
    """With single-stage groups of equal d, earliest predicted finish = join
    the group with least remaining work (backlog), lowest index on ties."""
    rng = np.random.default_rng(10)
    for _ in range(100):
        d = int(rng.integers(1, 8))
        G = int(rng.integers(1, 5))
        n = 40
        a = np.sort(rng.integers(0, 60, size=n)).astype(np.int64)
        prob = tiny_problem([(1, 1)], [[[d]]])
        r = oracle.simulate(prob, Trace(a, np.zeros(n, np.int32)), place([0] * G, [[0]] * G, 1),
                            detail=True)
        free = [0] * G  # time each server drains its backlog
        for i, t in enumerate(a.tolist()):
            backlog = [max(f - t, 0) for f in free]
            g = int(np.argmin(backlog))
            free[g] = max(free[g], t) + d
            assert r["served_by"][i] == g and r["finish_ns"][i] == free[g]


# ----------------------------------------------------------------------------- P13/P14
def test_p13_conservation_and_determinism():
    rng = np.random.default_rng(13)
    for _ in range(100):
        prob, tr, pl = random_instance(rng)
        r1 = oracle.simulate(prob, tr, pl, detail=True)
        r2 = oracle.simulate(prob, tr, pl, detail=True)
        assert 0 <= r1["good"] <= len(tr)
        assert int(r1["good_per_model"].sum()) == r1["good"]
        assert r1["good"] == int((r1["finish_ns"] >= 0).sum())
        acc = r1["finish_ns"] >= 0
        assert r1["sum_latency_ns"] == int((r1["finish_ns"][acc] - tr.arrival_ns[acc]).sum())
        lat = r1["finish_ns"][acc] - tr.arrival_ns[acc]
        assert np.all(lat <= prob.slo_ns[tr.model[acc]])
        for k in ("good", "sum_latency_ns"):
            assert r1[k] == r2[k]
        assert np.array_equal(r1["finish_ns"], r2["finish_ns"])


def test_p14_degenerate_cases():
    prob = tiny_problem([(1, 1)], [[[10]], [[5]]])
    empty = Trace(np.zeros(0, np.int64), np.zeros(0, np.int32))
    r = oracle.simulate(prob, empty, place([0], [[0]], 2))
    assert r["good"] == 0 and oracle.attainment(r["good"], 0) == 1.0
    tr = trace_of([(0, 0), (1, 1), (2, 0)])
    r = oracle.simulate(prob, tr, place([0], [[]], 2))  # nothing hosted
    assert r["good"] == 0
    r = oracle.simulate(prob, tr, place([], [], 2))  # no groups at all
    assert r["good"] == 0
    # zero SLO: only requests that finish instantly are good
    p0 = tiny_problem([(1, 1)], [[[0]], [[5]]], slo=[0, 0])
    r = oracle.simulate(p0, tr, place([0], [[0, 1]], 2))
    assert r["good"] == 2


def test_oracle_rejects_bad_input():
    prob = tiny_problem([(1, 1)], [[[10]]])
    with pytest.raises(ValueError):
        oracle.simulate(prob, trace_of([(5, 0), (3, 0)]), place([0], [[0]], 1))
    with pytest.raises(ValueError):
        oracle.simulate(prob, trace_of([(5, 1)]), place([0], [[0]], 1))
    with pytest.raises(ValueError):
        oracle.simulate(prob, trace_of([(-1, 0)]), place([0], [[0]], 1))
    with pytest.raises(ValueError):  # host bit on a missing group
        oracle.simulate(prob, trace_of([(1, 0)]), place([0, -1], [[0], [0]], 1))


# ----------------------------------------------------------------------------- P12
def test_p12a_motivating_slo_sweep_direction():
    """P:121 / Fig. realistic_workloads_results row 4: with tight SLOs AlpaServe
    favours intra-op parallelism; with looser SLOs inter-op (pipeline); simple
    placement is never better than the best model-parallel one."""
    tr = configs.motivating_trace(seed=12, n_requests=100_000)
    pls = dict(simple=place([0, 0], [[0], [1]], 2), intra=place([1], [[0, 1]], 2),
               pipe=place([2], [[0, 1]], 2))
    att = {}
    for scale in (1.0, 1.5, 3.0, 5.0):
        prob = configs.motivating_problem(slo_scale=scale)
        att[scale] = {k: oracle.simulate(prob, tr, v)["good"] for k, v in pls.items()}
    # at scale 1 (SLO = D) pipeline and simple are a near-tie
    assert att[1.0]["intra"] > max(att[1.0]["pipe"], att[1.0]["simple"])
    assert att[1.5]["intra"] > att[1.5]["pipe"] > att[1.5]["simple"]
    for scale in (3.0, 5.0):
        assert att[scale]["pipe"] > att[scale]["intra"] and att[scale]["pipe"] > att[scale]["simple"]


def test_p12bc_burstiness_and_skew_direction():
    """P:323 (CV 3: speedup grows from 1.3x to 1.9x) and P:328 (20/80 split:
    6.6x): model parallelism gains more under burstiness and skew."""
    prob = configs.motivating_problem(slo_scale=1e6)
    simple = place([0, 0], [[0], [1]], 2)
    pipe = place([2], [[0, 1]], 2)

    def ratio(cv, split, seed):
        tr = configs.motivating_trace(seed=seed, n_requests=200_000, cv=cv, split=split)
        return _mean_latency(prob, tr, simple) / _mean_latency(prob, tr, pipe)

    r1 = ratio(1.0, (0.5, 0.5), 21)
    r3 = ratio(3.0, (0.5, 0.5), 22)
    rs = ratio(1.0, (0.2, 0.8), 23)
    assert 1.15 < r1 < 1.45
    assert r3 > r1 + 0.3
    assert rs > 3.0


def test_feasibility_branches_hand_cases():
    """Feasibility (reading C11; Alg. 1 "if sel' is in memory constraint",
    P:711), every branch worked by hand: a 2-device cluster with a 10-byte
    budget per device; config 0 = (1,1) on 1 device, config 1 = (2,1) on 2.
    Per-device bytes: model 0: 6 / 3, model 1: not placeable (-1) / 4,
    model 2: 5 / 3."""
    from oracle import feasible

    prob = tiny_problem([(1, 1), (2, 1)], stage=[[[5], [2, 3]]] * 3,
                        mem=[[6, 3], [-1, 4], [5, 3]], num_devices=2, budget=10)
    M = prob.num_models
    cases = [
        ([0, 0], [[0], [0]], True),       # 2 devices, 6 <= 10 on each
        ([0, 0], [[0, 2], []], False),    # 6 + 5 = 11 > 10: memory
        ([0, 0], [[2], [0]], True),       # 5 and 6
        ([0], [[1]], False),              # (model 1, (1,1)) not placeable
        ([1], [[0, 1, 2]], True),         # 3 + 4 + 3 = 10 <= 10 on both devices
        ([1, 1], [[0], []], False),       # 4 devices > 2 (an empty group still holds its devices)
        ([0, 0, 0], [[0], [], []], False),  # 3 devices > 2
        ([1], [[]], True),                # nothing placed
    ]
    tr = trace_of([(0, 0), (1, 1), (2, 2)])
    for cfg, groups, want in cases:
        pl = place(cfg, groups, M)
        assert feasible(prob, pl) == want, (cfg, groups)
        g, _, _ = oracle.evaluate(prob, tr, np.array([cfg], np.int32),
                                  pl.host_mask[None, :], threads=1)
        assert (g[0] >= 0) == want and (want or g[0] == -1)


def test_greedy_ties_and_strict_best_hand_case():
    """Alg. 1's ties and best updates (reading C12), worked by
    hand.  Two (1,1) groups with memory for one model each; models A = 0 and
    B = 1 identical (10 ns, no deadline).  Trace A@0, B@100: every hosted
    request is good.
      step 1: (A,g0) (A,g1) (B,g0) (B,g1) all give 1 -> the first, (A,g0);
      step 2: g0 is full; (A,g1) gives 1 (a useless replica), (B,g1) gives 2
              -> (B,g1); no feasible addition is left.
    The lowest-index bijection A->g0, B->g1 with best good 2.  Without B's
    request the step-2 tie (A,g1) = (B,g1) = 1 goes to (A,g1) (m-major
    order), and the best stays step 1's selection: 1 is not > 1."""
    from oracle import search as osearch

    prob = tiny_problem([(1, 1)], stage=[[[10]], [[10]]], mem=[[6], [6]], num_devices=2,
                        budget=10)
    res = osearch.greedy(prob, trace_of([(0, 0), (100, 1)]), [0, 0], record=True)
    steps = res["steps"]
    assert [c for c, _, _ in steps] == [[(0, 0), (0, 1), (1, 0), (1, 1)], [(0, 1), (1, 1)]]
    assert [list(g) for _, g, _ in steps] == [[1, 1, 1, 1], [1, 2]]
    assert [i for _, _, i in steps] == [0, 1]
    assert res["good"] == 2 and res["placement"].host_mask.tolist() == [1, 2]

    res = osearch.greedy(prob, trace_of([(0, 0)]), [0, 0], record=True)
    steps = res["steps"]
    assert [list(g) for _, g, _ in steps] == [[1, 1, 0, 0], [1, 1]]
    assert [steps[k][0][i] for k, (_, _, i) in enumerate(steps)] == [(0, 0), (0, 1)]
    assert res["good"] == 1 and res["placement"].host_mask.tolist() == [1, 0]
