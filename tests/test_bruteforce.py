"""P11: brute force over every placement of tiny instances bounds the greedy
search (Alg. 1 inside single-bucket Alg. 2) from above; the motivating
example has exactly 17 placements."""

import numpy as np

import oracle
from oracle import search
from workloads import Trace, configs
from tests.helpers import tiny_problem


def test_motivating_has_17_placements():
    p = configs.motivating_problem()
    assert len(search.bruteforce_placements(p)) == 17


def test_optimum_bounds_greedy_random_tiny():
    rng = np.random.default_rng(11)
    for _ in range(25):
        M = int(rng.integers(1, 4))
        D = int(rng.choice([2, 4]))
        cfgs = [(1, 1), (1, 2), (2, 1)] if D == 2 else [(1, 1), (1, 2), (2, 1), (1, 4), (2, 2),
                                                        (4, 1)]
        stage = []
        for m in range(M):
            base = int(rng.integers(4, 12))
            row = []
            for s, n in cfgs:
                tot = int(base * (1 / n + 0.15 * (n - 1) / n)) + 1
                row.append([max(1, tot // s)] * s)
            stage.append(row)
        mem = [[int(rng.integers(3, 9)) * 10 // (s * n) for s, n in cfgs] for _ in range(M)]
        slo = [int(rng.integers(5, 40)) for _ in range(M)]
        prob = tiny_problem(cfgs, stage, slo=slo, mem=mem, num_devices=D, budget=10)
        n = int(rng.integers(5, 60))
        tr = Trace(np.sort(rng.integers(0, 80, size=n)).astype(np.int64),
                   rng.integers(0, M, size=n).astype(np.int32))
        bf = search.bruteforce(prob, tr)
        g = search.alg2(prob, tr)
        assert bf["good"] >= g["good"]
        # the greedy result is itself one of the enumerated placements' values
        assert g["good"] in set(bf["goods"].tolist()) | {0}
        assert oracle.simulate(prob, tr, g["placement"])["good"] == g["good"] if len(
            g["placement"].group_cfg) else True


def test_motivating_search_picks_model_parallel():
    """P:318 direction: at SLO scale 1.5 the best 2-GPU placement is model-parallel."""
    p = configs.motivating_problem(slo_scale=1.5)
    tr = configs.motivating_trace(seed=1, n_requests=3000)
    bf = search.bruteforce(p, tr)
    assert bf["placement"].num_groups == 1  # one 2-GPU group
    g = search.alg2(p, tr)
    assert g["good"] == bf["good"]
