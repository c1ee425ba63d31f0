"""Pins for the shared input generators (workloads/): the §4.1 DP against
exhaustive enumeration, config enumeration, memory
conservation, Gamma-process moments and power-law shares
(S:246-248)."""

import itertools

import numpy as np
import pytest

from workloads import configs, planner, traces


def _exhaustive_min_max(layers, s):
    K = len(layers)
    best = None
    for cuts in itertools.combinations(range(1, K), s - 1):
        edges = (0,) + cuts + (K,)
        v = max(int(sum(layers[a:b])) for a, b in zip(edges, edges[1:]))
        best = v if best is None else min(best, v)
    return best


def test_dp_matches_exhaustive():
    rng = np.random.default_rng(0)
    for _ in range(200):
        K = int(rng.integers(1, 13))
        s = int(rng.integers(1, min(K, 4) + 1))
        layers = rng.integers(0, 20, size=K).astype(np.int64)
        bounds, stage = planner.partition_dp(layers, s)
        assert int(stage.max()) == _exhaustive_min_max(layers.tolist(), s)
        # contiguous, ordered, covering partition
        assert bounds[0][0] == 0 and bounds[-1][1] == K - 1
        for (a, b), (c, d) in zip(bounds, bounds[1:]):
            assert c == b + 1 and a <= b
        assert int(stage.sum()) == int(layers.sum())


def test_dp_spec_examples():
    assert planner.partition_dp(np.array([1, 1, 1, 1]), 2)[0] == [(0, 1), (2, 3)]
    assert planner.partition_dp(np.array([3, 1, 1, 1]), 2)[0] == [(0, 0), (1, 3)]
    assert list(planner.partition_dp(np.array([1, 2, 3]), 3)[1]) == [1, 2, 3]
    with pytest.raises(ValueError):
        planner.partition_dp(np.array([1, 2]), 3)


def test_enumerate_configs():
    assert planner.enumerate_configs(8, 24) == [(1, 8), (2, 4), (4, 2), (8, 1)]
    assert planner.enumerate_configs(1, 24) == [(1, 1)]
    assert planner.enumerate_configs(6, 24) == [(1, 6), (2, 3), (3, 2), (6, 1)]
    assert planner.enumerate_configs(64, 24, pipeline_only=True) == []
    assert planner.enumerate_configs(64, 96, pipeline_only=True) == [(64, 1)]


def test_memory_conservation_and_tables():
    prob, _ = configs.s3(duration=10.0)
    assert prob.num_models == 60 and prob.num_configs == 25
    for m in range(prob.num_models):
        for p, (s, n) in enumerate(prob.configs):
            mem = int(prob.mem_bytes[m, p])
            assert mem * s * n >= 0
            # ceil division: mem*s*n - bytes in [0, s*n)
            from workloads import table1
            nbytes = table1.MODELS[prob.model_names[m].split("#")[0]][0]
            assert 0 <= mem * s * n - nbytes < s * n
    for p, (s, n) in enumerate(prob.configs):
        assert np.all(prob.stage_ns[:, p, s:] == 0)
        assert np.all(prob.stage_ns[:, p, :s] > 0)


def test_motivating_tables():
    p = configs.motivating_problem()
    assert p.configs == [(1, 1), (1, 2), (2, 1)]
    assert list(p.stage_ns[0, 0, :1]) == [400_000_000]
    assert list(p.stage_ns[0, 2, :2]) == [200_000_000, 200_000_000]
    assert list(p.stage_ns[0, 1, :1]) == [230_000_000]  # 0.4*(1/2 + 0.15/2)
    assert list(p.slo_ns) == [2_000_000_000] * 2


def test_gamma_moments():
    rng = np.random.default_rng(1)
    for rate, cv in [(1.5, 1.0), (20.0, 3.0), (8.0, 4.0)]:
        t = traces.gamma_process(rng, rate, cv, 2e5 / rate)
        gaps = np.diff(t)
        assert len(t) / (2e5 / rate) == pytest.approx(rate, rel=0.03)
        assert gaps.std() / gaps.mean() == pytest.approx(cv, rel=0.05)


def test_power_law_split():
    w = traces.power_law_weights(2, 0.5)
    assert w * 8 == pytest.approx([4.686, 3.314], abs=1e-3)
    assert traces.power_law_weights(4, 0.0) == pytest.approx([0.25] * 4)
    assert traces.power_law_weights(1, 0.5) == pytest.approx([1.0])


def test_trace_sorted_deterministic():
    a = traces.maf2_shaped(3, 6, 50.0, 3600.0)
    b = traces.maf2_shaped(3, 6, 50.0, 3600.0)
    assert np.array_equal(a.arrival_ns, b.arrival_ns) and np.array_equal(a.model, b.model)
    assert np.all(np.diff(a.arrival_ns) >= 0)
    assert len(a) == pytest.approx(50 * 3600, rel=0.15)
    m1 = traces.maf1_shaped(4, 8, 40.0, 7200.0)
    assert np.all(np.diff(m1.arrival_ns) >= 0)
    assert len(m1) == pytest.approx(40 * 7200, rel=0.05)
