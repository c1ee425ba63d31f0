"""Dynamic batching variant (§5.4 "Batching strategy").

Oracle pins (no GPU): each compares the batching DES with something other than
itself -- the independently pinned non-batching simulator (max_batch = 1 with
one hosting group per model), a closed form for a burst, SPEC's form_batch
examples worked by hand, hand-worked head rejection and dispatch
cases, conservation, and SPEC's batching sanity check.
GPU parity (-m gpu): the sm_100a batching kernel against the oracle, bit-exact.
"""

import numpy as np
import pytest

import oracle
from tests.helpers import INF, place, random_instance, tiny_problem, trace_of
from workloads import Placement, Trace, configs

S = 1_000_000_000  # 1 s in ns


def _inc(prob, value=0):
    return np.full(np.shape(prob.stage_ns), value, np.int64)


def _sim(prob, tr, pl, inc, b):
    return oracle.simulate_batching(prob, tr, pl, inc, b, detail=True)


# ------------------------------------------------------------------ equivalence
@pytest.mark.parametrize("seed", range(300))
def test_b1_single_host_equals_fcfs_simulator(seed):
    """max_batch = 1 and every model on at most one group: the central
    per-model queues with earliest-head choice serve each group's requests in
    arrival order and drop a request exactly when FCFS admission at receipt
    would reject it, so the batching DES must reproduce the pinned
    non-batching DES request by request (any increments: batches are size 1)."""
    rng = np.random.default_rng(seed)
    prob, tr, _ = random_instance(rng, n_req=50, dmax=5)
    prob.stage_ns[:, :, 0] = np.maximum(prob.stage_ns[:, :, 0], 1)  # first stage >= 1 ns
    M = prob.num_models
    G = int(rng.integers(1, 4))
    cfg = [int(rng.integers(0, prob.num_configs)) for _ in range(G)]
    groups = [[] for _ in range(G)]
    for m in range(M):
        g = int(rng.integers(-1, G))
        if g >= 0:
            groups[g].append(m)
    pl = place(cfg, groups, M)
    inc = rng.integers(0, 4, size=np.shape(prob.stage_ns))
    a = oracle.simulate(prob, tr, pl, detail=True)
    b = _sim(prob, tr, pl, inc, 1)
    assert a["good"] == b["good"] and a["sum_latency_ns"] == b["sum_latency_ns"]
    assert np.array_equal(a["finish_ns"], b["finish_ns"])
    assert np.array_equal(a["served_by"], b["served_by"])
    assert np.array_equal(a["good_per_model"], b["good_per_model"])


# ------------------------------------------------------------------ closed form
@pytest.mark.parametrize("n,b,d,e", [(1, 4, 7, 3), (10, 3, 100, 0), (10, 3, 100, 40),
                                     (17, 4, 10, 9), (5, 8, 5, 5), (9, 1, 6, 2)])
def test_burst_closed_form(n, b, d, e):
    """n requests at t = 0, one single-stage group, infinite SLO: the first
    runs alone (the group is available on arrival), the rest wait and leave
    in batches of min(b, waiting) when the group frees; a batch of k takes
    d + (k-1) e (P:169 linear latency)."""
    prob = tiny_problem([(1, 1)], [[[d]]])
    tr = trace_of([(0, 0)] * n)
    out = _sim(prob, tr, place([0], [[0]], 1), _inc(prob, e), b)
    expect, t, left = [d], d, n - 1
    while left > 0:
        k = min(b, left)
        t += d + (k - 1) * e
        expect += [t] * k
        left -= k
    assert list(out["finish_ns"]) == expect
    assert out["good"] == n and out["sum_latency_ns"] == sum(expect)


def test_burst_pipeline_closed_form():
    """Two-stage group [d0, d1], tail T, batches of 2: the first stage frees
    after d0 (+e0 per extra member), so batches enter every d0 + e0 while the
    second stage works; with d1 + e1 <= d0 + e0 nothing waits at stage 2."""
    d0, d1, e0, e1, T = 10, 4, 5, 2, 3
    prob = tiny_problem([(2, 1)], [[[d0, d1]]], tail=[[T]])
    inc = _inc(prob)
    inc[0, 0] = [e0, e1]
    tr = trace_of([(0, 0)] * 5)
    out = _sim(prob, tr, place([0], [[0]], 1), inc, 2)
    f0 = d0 + d1 + T                      # alone
    s1 = d0                               # batch {1,2} enters at d0
    f1 = s1 + (d0 + e0) + (d1 + e1) + T
    s2 = s1 + d0 + e0                     # batch {3,4}
    f2 = s2 + (d0 + e0) + (d1 + e1) + T
    assert list(out["finish_ns"]) == [f0, f1, f1, f2, f2]


# ------------------------------------------------------ SPEC form_batch examples
def test_spec_form_batch_two_of_two():
    """two queued requests, delta = 1, D = 0.4 s, both SLOs allow 0.8 s
    of batched latency -> one batch of 2.  A first request keeps the group
    busy over [0, 0.4]; requests at 0.1 and 0.2 wait; at 0.4 the batch of two
    takes 0.8 s and finishes at 1.2 s (latencies 1.1 and 1.0 <= slo 1.1)."""
    D = 4 * S // 10
    prob = tiny_problem([(1, 1)], [[[D]]], slo=[11 * S // 10])
    tr = trace_of([(0, 0), (S // 10, 0), (2 * S // 10, 0)])
    out = _sim(prob, tr, place([0], [[0]], 1), _inc(prob, D), 4)
    assert list(out["finish_ns"]) == [D, 12 * S // 10, 12 * S // 10]


def test_spec_form_batch_prefix_of_one():
    """the longest prefix whose members all meet the SLO.  Same as
    above with slo 1.0 s: a batch of two would give the head 1.1 s > 1.0, so
    the head leaves alone at 0.8 and the second request alone at 1.2 (1.0)."""
    D = 4 * S // 10
    prob = tiny_problem([(1, 1)], [[[D]]], slo=[S])
    tr = trace_of([(0, 0), (S // 10, 0), (2 * S // 10, 0)])
    out = _sim(prob, tr, place([0], [[0]], 1), _inc(prob, D), 4)
    assert list(out["finish_ns"]) == [D, 8 * S // 10, 12 * S // 10]


def test_b1_is_fcfs_spec_example():
    """b = 1 is non-batching FCFS (one group)."""
    prob = tiny_problem([(1, 1)], [[[10]]], slo=[25])
    tr = trace_of([(0, 0), (0, 0), (0, 0), (1, 0)])
    out = _sim(prob, tr, place([0], [[0]], 1), _inc(prob, 3), 1)
    # 1 waits to 10 and ends at 20; 2 and 3 would end at 30: 30 > 25, 29 > 25
    assert list(out["finish_ns"]) == [10, 20, -1, -1]
    assert list(oracle.simulate(prob, tr, place([0], [[0]], 1), detail=True)["finish_ns"]) == \
        [10, 20, -1, -1]


# --------------------------------------------------------------- hand-worked cases
@pytest.mark.parametrize("slo,expect", [(15, [10, -1, 20, -1]), (16, [10, -1, 22, 22])])
def test_head_rejection(slo, expect):
    """d = 10, e = 2.  Request 0 runs alone over [0, 10]; 1 (t=0), 2 (t=6),
    3 (t=7) wait.  At 10 the head (1) would finish at 20 alone, latency
    20 > slo: rejected, and the choice is repeated with 2 as head.
    slo 15: {2,3} would give 22 - 6 = 16 > 15, so 2 leaves alone at 20; at 20
    request 3 alone gives 30 - 7 = 23 > 15: rejected.
    slo 16: {2,3} finish at 22 (latencies 16, 15)."""
    prob = tiny_problem([(1, 1)], [[[10]]], slo=[slo])
    tr = trace_of([(0, 0), (0, 0), (6, 0), (7, 0)])
    out = _sim(prob, tr, place([0], [[0]], 1), _inc(prob, 2), 4)
    assert list(out["finish_ns"]) == expect
    assert out["good"] == sum(f >= 0 for f in expect)


def test_model_choice_earliest_head():
    """One group hosts A (d = 10) and B (d = 4), b = 2, e = 0.  A@0 runs
    alone; B@1, A@2, B@3 wait.  At 10 B's head came first: batch {B@1, B@3}
    finishes at 14; at 14 A@2 runs to 24."""
    prob = tiny_problem([(1, 1)], [[[10]], [[4]]])
    tr = trace_of([(0, 0), (1, 1), (2, 0), (3, 1)])
    out = _sim(prob, tr, place([0], [[0, 1]], 2), _inc(prob), 2)
    assert list(out["finish_ns"]) == [10, 14, 24, 14]


def test_immediate_dispatch_and_idle_pickup():
    """g0 (d = 10) and g1 (d = 6) both host A.  A@0: both available, g1
    finishes first (6).  A@1: only g0 is available -> runs there (11).  A@2:
    nothing available -> waits; g1 becomes available at 6 and takes it (12)."""
    prob = tiny_problem([(1, 1), (1, 1)], [[[10], [6]]])
    tr = trace_of([(0, 0), (1, 0), (2, 0)])
    out = _sim(prob, tr, place([0, 1], [[0], [0]], 1), _inc(prob), 4)
    assert list(out["finish_ns"]) == [6, 11, 12]
    assert list(out["served_by"]) == [1, 0, 1]


def test_equal_time_groups_in_index_order():
    """g0 and g1 (d = 5 each) both free at 5 with two requests waiting and
    b = 1: g0 (lower index) takes the earlier one.  A request arriving at the
    same time 5 finds both busy (completions precede arrivals, C6)."""
    prob = tiny_problem([(1, 1)], [[[5]]])
    tr = trace_of([(0, 0), (0, 0), (1, 0), (2, 0), (5, 0)])
    out = _sim(prob, tr, place([0, 0], [[0], [0]], 1), _inc(prob), 1)
    assert list(out["served_by"]) == [0, 1, 0, 1, 0]
    assert list(out["finish_ns"]) == [5, 5, 10, 10, 15]


def test_degenerate_inputs():
    prob = tiny_problem([(1, 1)], [[[5]], [[5]]])
    empty = Trace(np.zeros(0, np.int64), np.zeros(0, np.int32))
    assert _sim(prob, empty, place([0], [[0]], 2), _inc(prob), 3)["good"] == 0
    tr = trace_of([(0, 1), (1, 1)])
    out = _sim(prob, tr, place([0], [[0]], 2), _inc(prob), 3)  # model 1 hosted nowhere
    assert out["good"] == 0 and list(out["finish_ns"]) == [-1, -1]
    with pytest.raises(ValueError):
        _sim(prob, tr, place([0], [[0]], 2), _inc(prob), 0)  # max_batch < 1
    with pytest.raises(ValueError):
        _sim(prob, tr, place([0], [[0]], 2), _inc(prob, -1), 2)  # negative increment
    z = tiny_problem([(1, 1)], [[[0]]])
    with pytest.raises(ValueError):
        _sim(z, trace_of([(0, 0)]), place([0], [[0]], 1), _inc(z), 2)  # first stage 0 ns


# ------------------------------------------------------------------ invariants
@pytest.mark.parametrize("seed", range(200))
def test_conservation_and_slo(seed):
    """good <= N, per-model counts sum to good, every good request meets its
    SLO, members of a batch share their finish time and group, and max_batch
    above the trace length changes nothing (P13-style)."""
    rng = np.random.default_rng(1000 + seed)
    prob, tr, pl = random_instance(rng, n_req=40, dmax=6)
    prob.stage_ns[:, :, 0] = np.maximum(prob.stage_ns[:, :, 0], 1)
    inc = rng.integers(0, 4, size=np.shape(prob.stage_ns))
    b = int(rng.integers(1, 6))
    out = _sim(prob, tr, pl, inc, b)
    fin, srv = out["finish_ns"], out["served_by"]
    good = fin >= 0
    assert out["good"] == int(good.sum()) == int(out["good_per_model"].sum())
    lat = fin[good] - tr.arrival_ns[good]
    assert np.all(lat <= prob.slo_ns[tr.model[good]])
    assert out["sum_latency_ns"] == int(lat.sum())
    for g in range(pl.num_groups):  # a batch = same group, model and finish: size <= b
        for m in range(prob.num_models):
            f_gm = fin[(srv == g) & good & (tr.model == m)]
            if len(f_gm):
                assert np.unique(f_gm, return_counts=True)[1].max() <= b
    big = _sim(prob, tr, pl, inc, len(tr) + 5)
    bigger = _sim(prob, tr, pl, inc, len(tr) + 50)
    assert np.array_equal(big["finish_ns"], bigger["finish_ns"])


def test_spec_batching_sanity():
    """SPEC S:615 ("when the SLO is tight ... batching is simply
    not a choice" and P:795 "batching is helpful, but the gain is limited") on
    the §5.4 S1 setup (4 req/s per model, CV 4), selective
    replication: at SLO scale 1.5 with delta = 1, mb = 2 changes attainment by
    <= 0.5 %; at SLO scale 8 with delta = 0.9 (reading C35: a batch of 2 runs
    below twice the single latency, else batching cannot gain) mb = 2 and
    mb = 4 are not worse than mb = 1."""
    def run(scale, delta, b):
        prob, tr, inc = configs.s1_batching(seed=0, duration=120.0, slo_scale=scale,
                                            delta=delta)
        M = prob.num_models
        p11 = prob.configs.index((1, 1))
        groups = [[m for m in range(M) if m % 8 == g % 8] for g in range(16)]
        pl = place([p11] * 16, groups, M)
        return _sim(prob, tr, pl, inc, b)["good"] / len(tr)

    assert abs(run(1.5, 1.0, 2) - run(1.5, 1.0, 1)) <= 0.005
    b1 = run(8.0, 0.9, 1)
    assert run(8.0, 0.9, 2) >= b1 and run(8.0, 0.9, 4) >= b1


# ============================================================ GPU parity (-m gpu)
def _stack(placements, M):
    G = max([p.num_groups for p in placements] + [1])
    cfg = np.full((len(placements), G), -1, np.int32)
    mask = np.zeros((len(placements), M), np.uint64)
    for i, p in enumerate(placements):
        cfg[i, :p.num_groups] = p.group_cfg
        mask[i] = p.host_mask
    return cfg, mask


@pytest.fixture(scope="module")
def sim():
    from paper_2302_11665_b200 import Simulator
    s = Simulator(0)
    yield s
    s.close()


def _check(sim, prob, tr, cfg, mask, inc, b):
    sim.set_problem(prob)
    sim.set_trace(tr.arrival_ns, tr.model)
    got = sim.evaluate_batching(cfg, mask, inc, b, per_model=True)
    g, s, pm = oracle.evaluate_batching(prob, tr, cfg, mask, inc, b, per_model=True)
    np.testing.assert_array_equal(got["good"], g)
    np.testing.assert_array_equal(got["sum_latency_ns"], s)
    np.testing.assert_array_equal(got["good_per_model"], pm)
    want = int(np.argmax(g)) if len(g) and g.max() >= 0 else -1
    assert got["argmax"] == want
    return g


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(24))
def test_gpu_parity_random(sim, seed):
    """Random small instances (multi-stage groups, shared hosts, zero-latency
    later stages, duplicate timestamps, unhosted models, finite and infinite
    SLOs), 70 candidates per call = 2 full warps + a ragged tail."""
    rng = np.random.default_rng(5000 + seed)
    prob, tr, _ = random_instance(rng, M=int(rng.integers(1, 5)), P=3, n_req=int(rng.integers(0, 400)),
                                  dmax=6, tmax=200)
    prob.stage_ns[:, :, 0] = np.maximum(prob.stage_ns[:, :, 0], 1)
    inc = rng.integers(0, 4, size=np.shape(prob.stage_ns))
    pls = []
    for _ in range(70):
        G = int(rng.integers(1, 6))
        cfg = [int(rng.integers(0, prob.num_configs)) for _ in range(G)]
        groups = [[m for m in range(prob.num_models) if rng.random() < 0.5] for _ in range(G)]
        pls.append(place(cfg, groups, prob.num_models))
    cfg, mask = _stack(pls, prob.num_models)
    b = int(rng.choice([1, 2, 3, 5, 1000]))
    _check(sim, prob, tr, cfg, mask, inc, b)


@pytest.mark.gpu
def test_gpu_hand_cases(sim):
    """The hand-worked oracle cases, through the C ABI."""
    prob = tiny_problem([(1, 1)], [[[10]]], slo=[16])
    tr = trace_of([(0, 0), (0, 0), (6, 0), (7, 0)])
    cfg, mask = _stack([place([0], [[0]], 1)], 1)
    sim.set_problem(prob)
    sim.set_trace(tr.arrival_ns, tr.model)
    got = sim.evaluate_batching(cfg, mask, _inc(prob, 2), 4)
    assert got["good"][0] == 3 and got["sum_latency_ns"][0] == 10 + 16 + 15
    prob = tiny_problem([(1, 1)], [[[100]]])
    tr = trace_of([(0, 0)] * 10)
    sim.set_problem(prob)
    sim.set_trace(tr.arrival_ns, tr.model)
    got = sim.evaluate_batching(cfg, mask, _inc(prob, 40), 3)
    assert got["sum_latency_ns"][0] == 100 + 3 * 280 + 3 * 460 + 3 * 640


def _s1_placements(prob):
    """Selective replication and model-parallel groups on 16 devices (§5.4:
    AlpaServe vs SR with batching)."""
    M = prob.num_models
    ix = {c: i for i, c in enumerate(prob.configs)}
    out = []
    for size, (s, n) in [(1, (1, 1)), (2, (2, 1)), (2, (1, 2)), (4, (4, 1)), (4, (2, 2)),
                         (8, (8, 1))]:
        G = 16 // size
        groups = [[m for m in range(M) if (m * G // M) % G == g or (m + M // 2) * G // M % G == g]
                  for g in range(G)]
        out.append(place([ix[(s, n)]] * G, groups, M))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("delta,b,scale", [(1.0, 2, 1.5), (0.9, 2, 8.0), (0.9, 4, 8.0),
                                           (0.7, 8, 5.0), (0.9, 1, 5.0)])
def test_gpu_parity_s1_batching(sim, delta, b, scale):
    """§5.4 setup (S1, 4 req/s per model, CV 4; 120 s), SR and pipeline /
    intra-op placements, bit-exact good, latency sums and per-model counts."""
    prob, tr, inc = configs.s1_batching(seed=1, duration=120.0, slo_scale=scale, delta=delta)
    cfg, mask = _stack(_s1_placements(prob), prob.num_models)
    g = _check(sim, prob, tr, cfg, mask, inc, b)
    assert (g >= 0).all()


@pytest.mark.gpu
def test_gpu_parity_s3_shape(sim):
    """S3-shaped (60 models, 64 devices, MAF2-shaped bursts), 10-min prefix,
    random placements of up to 64 groups: bit-exact."""
    prob, tr = configs.s3(seed=0, duration=600.0)
    inc = configs.batch_increment_ns(prob.stage_ns, 0.9)
    rng = np.random.default_rng(7)
    pls = []
    for size in (1, 2, 4, 8):
        for cfg_i, (s, n) in enumerate(prob.configs):
            if s * n != size:
                continue
            G = 64 // size
            groups = [[m for m in range(60) if rng.random() < 0.08 * size] for _ in range(G)]
            pls.append(place([cfg_i] * G, groups, 60))
    cfg, mask = _stack(pls, 60)
    _check(sim, prob, tr, cfg, mask, inc, 4)


@pytest.mark.gpu
def test_gpu_batching_errors(sim):
    from paper_2302_11665_b200 import AsimError
    prob = tiny_problem([(1, 1)], [[[10]]])
    tr = trace_of([(0, 0)])
    sim.set_problem(prob)
    sim.set_trace(tr.arrival_ns, tr.model)
    cfg, mask = _stack([place([0], [[0]], 1)], 1)
    with pytest.raises(AsimError):
        sim.evaluate_batching(cfg, mask, _inc(prob), 0)
    with pytest.raises(AsimError):
        sim.evaluate_batching(cfg, mask, _inc(prob, -1), 2)
    z = tiny_problem([(1, 1)], [[[0]]])
    sim.set_problem(z)
    sim.set_trace(tr.arrival_ns, tr.model)
    with pytest.raises(AsimError):
        sim.evaluate_batching(cfg, mask, _inc(z), 2)
    big = tiny_problem([(1, 1)], [[[5]]] * 65)
    sim.set_problem(big)
    sim.set_trace(tr.arrival_ns, tr.model)
    with pytest.raises(AsimError):
        sim.evaluate_batching(np.zeros((1, 1), np.int32), np.zeros((1, 65), np.uint64),
                              _inc(big), 2)
    empty = Trace(np.zeros(0, np.int64), np.zeros(0, np.int32))
    sim.set_problem(prob)
    sim.set_trace(empty.arrival_ns, empty.model)
    assert sim.evaluate_batching(cfg, mask, _inc(prob), 2)["good"][0] == 0


@pytest.mark.gpu
def test_gpu_batching_bench_config_sampled(sim):
    """The bench configuration (scripts/bench_batching.py: S1 §5.4 setup, 1 h
    trace, 4,736 placements, max_batch 4, delta 0.9) in the launch
    configuration the bench times; 6 sampled candidates re-simulated one by
    one by the oracle must match exactly."""
    import sys
    import os
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(__file__)), "scripts"))
    from bench_batching import placements

    prob, tr, inc = configs.s1_batching(seed=0, duration=3600.0, slo_scale=5.0, delta=0.9)
    cfg, mask = placements(prob, 148 * 32, seed=1)
    sim.set_problem(prob)
    sim.set_trace(tr.arrival_ns, tr.model)
    got = sim.evaluate_batching(cfg, mask, inc, 4, per_model=True)
    rng = np.random.default_rng(3)
    pick = sorted(set(rng.integers(0, len(cfg), size=5).tolist()) | {int(got["argmax"])})
    g, s, pm = oracle.evaluate_batching(prob, tr, cfg[pick], mask[pick], inc, 4, per_model=True)
    np.testing.assert_array_equal(got["good"][pick], g)
    np.testing.assert_array_equal(got["sum_latency_ns"][pick], s)
    np.testing.assert_array_equal(got["good_per_model"][pick], pm)
    assert (got["good"] <= len(tr)).all() and (got["good"] >= 0).all()


@pytest.mark.gpu
def test_gpu_batching_sharded_single_rank(sim):
    """dist.evaluate_batching_sharded at world size 1 (the N>1 logic is
    covered under gloo in tests/test_dist.py)."""
    from paper_2302_11665_b200 import dist as adist
    prob, tr, inc = configs.s1_batching(seed=1, duration=60.0, slo_scale=3.0, delta=0.9)
    cfg, mask = _stack(_s1_placements(prob), prob.num_models)
    sim.set_problem(prob)
    sim.set_trace(tr.arrival_ns, tr.model)
    good, arg = adist.evaluate_batching_sharded(sim, cfg, mask, inc, 2)
    g, _, _ = oracle.evaluate_batching(prob, tr, cfg, mask, inc, 2)
    assert good.cpu().tolist() == g.tolist() and arg == int(np.argmax(g))
