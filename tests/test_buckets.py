"""§8(f2): Alg. 2 with model and device buckets (readings C25-C28
in DESIGN.md).

CPU tests pin the oracle's enumeration rules to SPEC's examples
and hand-worked cases, and check that a bucketed solution's good -- the sum
of its buckets' goods -- equals an independent DES run of the concatenated
placement.  GPU tests require libasim.so's bucketed search to reproduce the
oracle's choice."""

from fractions import Fraction

import numpy as np
import pytest

from oracle import search as osearch
from oracle import simulate
from tests.helpers import tiny_problem, trace_of
from workloads import configs, traces

MS = 10**6


# ------------------------------------------------------------------ CPU pins
def test_homogeneous_models_one_bucket():
    """homogeneous models -> exactly one bucket enumerated."""
    assert osearch.model_buckets([151 * MS] * 6) == [[[0, 1, 2, 3, 4, 5]]]


def test_small_and_104b_two_buckets():
    """0.15 s and 4.6 s models, threshold 4x -> two buckets only."""
    lat = [4600 * MS, 150 * MS, 4600 * MS, 151 * MS]
    assert osearch.model_buckets(lat) == [[[1, 3], [0, 2]]]


def test_s3_is_one_bucket():
    """S3's latencies span 150-395 ms (< 4x): one bucket."""
    prob = configs.table1_problem("S3", 64)
    parts = osearch.model_buckets(prob.meta["latency_ns"])
    assert parts == [[list(range(prob.num_models))]]


def test_chain_enumerates_needed_cuts_only():
    """Latencies 1, 3, 9, 27 with threshold 4: {1,3}{9,27} and {1}{3,9}{27};
    {1}{3}{9,27} is not enumerated ({1} and {3} could form one bucket)."""
    lat = [27, 9, 3, 1]
    assert osearch.model_buckets(lat) == [[[2, 3], [0, 1]], [[3], [1, 2], [0]]]
    assert osearch.model_buckets(lat, max_buckets=2) == [[[2, 3], [0, 1]]]


def test_equal_latencies_never_split():
    lat = [5, 1, 1, 20]
    # 1,1 | 5,20 is valid (20 <= 4*5); 1,1,5 is not (5 > 4*1); never 1 | 1,...
    assert osearch.model_buckets(lat) == [[[1, 2], [0, 3]]]
    assert osearch.model_buckets([4, 1, 1, 16]) == [[[1, 2], [0, 3]], [[0, 1, 2], [3]]]


def test_ratio_boundary_inclusive():
    """max <= ratio * min keeps a bucket: latencies 1 and 4 stay together."""
    assert osearch.model_buckets([1, 4]) == [[[0, 1]]]
    assert osearch.model_buckets([1, 5]) == [[[0], [1]]]


def test_device_buckets():
    assert osearch.device_buckets(4, 1) == [(4,)]
    assert osearch.device_buckets(4, 2) == [(1, 3), (2, 2), (3, 1)]
    assert osearch.device_buckets(5, 3) == [(1, 1, 3), (1, 2, 2), (1, 3, 1), (2, 1, 2),
                                            (2, 2, 1), (3, 1, 1)]
    from math import comb
    assert len(osearch.device_buckets(12, 3)) == comb(11, 2)


def test_discrepancy_pruning():
    lat = [10, 10]
    # equal demand, equal capacity split -> kept
    assert osearch.discrepancy_ok([[0], [1]], (5, 5), lat, [50, 50])
    # 90 % of demand on 10 % of devices, bound 3 -> dropped
    assert not osearch.discrepancy_ok([[0], [1]], (1, 9), lat, [90, 10])
    # a single bucket is always kept
    assert osearch.discrepancy_ok([[0, 1]], (10,), lat, [90, 10])
    # capacity uses the bucket's mean latency: a 4x slower bucket needs 4x devices
    assert osearch.discrepancy_ok([[0], [1]], (2, 8), [10, 40], [50, 50])
    # boundary: r ratio exactly 3 is kept, above is dropped
    assert osearch.discrepancy_ok([[0], [1]], (1, 1), lat, [75, 25])
    assert not osearch.discrepancy_ok([[0], [1]], (1, 1), lat, [76, 24])
    # a bucket without demand next to one with demand: dropped
    assert not osearch.discrepancy_ok([[0], [1]], (1, 1), lat, [10, 0])


def _two_tier():
    """Two fast models (1 ns... 2 ns) and one slow model (20 ns); 4 devices."""
    cfgs = [(1, 1), (2, 1), (1, 2), (4, 1)]
    stage = [[[2], [1, 1], [1], [1, 1, 0, 0]],
             [[2], [1, 1], [1], [1, 1, 0, 0]],
             [[20], [10, 10], [12], [5, 5, 5, 5]]]
    prob = tiny_problem(cfgs, stage, slo=[6, 6, 50], num_devices=4, budget=2,
                        latency=[2, 2, 20])
    rng = np.random.default_rng(5)
    pairs, t = [], 0
    for _ in range(120):
        t += int(rng.integers(0, 4))
        pairs.append((t, int(rng.choice(3, p=[0.45, 0.45, 0.1]))))
    return prob, trace_of(pairs)


def test_bucketed_search_concatenation_is_exact():
    """The bucketed objective (sum over buckets) equals an independent DES
    run of the concatenated placement."""
    prob, tr = _two_tier()
    res = osearch.alg2_buckets(prob, tr)
    assert res["partition"] == [[0, 1], [2]]
    pl = osearch.concat(prob, res["buckets"])
    assert simulate(prob, tr, pl)["good"] == res["good"]
    # one bucket per partition element, devices add up
    assert sum(res["devices"]) == prob.num_devices


def test_single_bucket_reduces_to_alg2():
    prob, tr = _two_tier()
    # a threshold that keeps every model in one bucket gives plain Alg. 2
    res = osearch.alg2_buckets(prob, tr, ratio=Fraction(100))
    assert res["good"] == osearch.alg2(prob, tr)["good"]


# ------------------------------------------------------------------ GPU parity
@pytest.fixture(scope="module")
def sim():
    from paper_2302_11665_b200 import Simulator
    s = Simulator(0)
    yield s
    s.close()


def _compare(sim, prob, tr, **kw):
    ref = osearch.alg2_buckets(prob, tr, **{k: v for k, v in kw.items() if k != "max_buckets"},
                               max_buckets=kw.get("max_buckets", 0))
    sim.set_problem(prob)
    sim.set_trace(tr.arrival_ns, tr.model)
    res = sim.search_buckets(latency=prob.meta["latency_ns"], **kw)
    assert res.best_good == ref["good"]
    assert res.considered == len(ref["considered"])
    if ref["partition"] is not None:
        assert [list(b) for b in res.partition] == ref["partition"]
        assert tuple(res.devices) == tuple(ref["devices"])
        pl = osearch.concat(prob, ref["buckets"])
        np.testing.assert_array_equal(res.placement.group_cfg, pl.group_cfg)
        np.testing.assert_array_equal(res.placement.host_mask, pl.host_mask)
        # and the GPU's own evaluation of the concatenation agrees
        out = sim.evaluate(pl.group_cfg[None, :], pl.host_mask[None, :])
        assert out["good"][0] == ref["good"]
    return res, ref


@pytest.mark.gpu
@pytest.mark.parametrize("fast", [False, True])
def test_buckets_parity_two_tier(sim, fast):
    prob, tr = _two_tier()
    _compare(sim, prob, tr, fast=fast)
    _compare(sim, prob, tr, fast=fast, ratio=Fraction(100))


@pytest.mark.gpu
def test_buckets_parity_bert_mix(sim):
    """S1-sized models next to 6.7B models made 5x slower: two tiers on 8
    devices, discrepancy pruning active."""
    names = [f"BERT-1.3B#{i}" for i in range(4)] + [f"BERT-6.7B#{i}" for i in range(2)]
    per = {n: (int(13.4e9), 800 * MS, None, None) for n in names if n.startswith("BERT-6.7B")}
    prob = configs.build_problem(names, 8, 13 * 10**9, slo_scale=4.0, per_model=per)
    tr = traces.independent_gamma(7, [2.0] * 4 + [0.6] * 2, 2.0, 120.0)
    res, ref = _compare(sim, prob, tr)
    assert len(ref["partition"]) == 2
