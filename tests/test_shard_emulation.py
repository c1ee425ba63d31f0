"""libasim's own sharded search path, emulated on one GPU.

W ranks are W independent contexts (asim_ctx) on cuda:0, each with its own
SearchHandle.  Every step: prepare() on all of them (identical candidate
lists and cost estimates), evaluate() of rank r's contiguous shard only --
asim_search_evaluate with begin > 0, the candidate-memory mix rows of
[begin, end), local-only candidate memory -- then the shards are joined
exactly as dist.gather_all joins them after the all-gather
(dist.concat_shards) and apply() runs on every handle, which re-simulates a
winner another rank simulated (the base pass).  Candidate evaluations within
an iteration are independent, so every rank must end with the
per-run selections of the world-1 search and of the oracle's Alg. 2."""

import numpy as np
import pytest
import torch

from oracle import search as osearch
from workloads import configs, traces

pytestmark = pytest.mark.gpu


def _sims(W, prob, tr, chunk):
    from paper_2302_11665_b200 import Simulator
    sims = []
    for _ in range(W):
        s = Simulator(0)
        s.set_problem(prob)
        s.set_trace(tr.arrival_ns, tr.model)
        s.set_chunk_size(chunk)
        sims.append(s)
    return sims


def emulate(prob, tr, W, chunk=4096, balance="cost", **kw):
    """The dist.run_search loop with W handles on one GPU.  Returns per rank
    (result, per-run histories)."""
    from paper_2302_11665_b200 import dist as adist

    sims = _sims(W, prob, tr, chunk)
    hs = [s.search_handle(**kw) for s in sims]
    locals_ = [torch.zeros(1, dtype=torch.int64, device="cuda") for _ in range(W)]
    begins_nonzero = 0
    try:
        while True:
            Cs = [h.prepare() for h in hs]
            assert len(set(Cs)) == 1, Cs  # identical search state on every rank
            C = Cs[0]
            if C < 0:
                break
            if C == 0:
                for h in hs:
                    h.apply(None)
                continue
            costs = [h.costs(C) for h in hs]
            for c in costs[1:]:
                np.testing.assert_array_equal(c, costs[0])
            assert (costs[0] >= 1).all()
            bounds = (adist.shard_bounds(costs[0], W) if balance == "cost"
                      else [adist.shard(C, r, W)[0] for r in range(W)] + [C])
            pad = max(1, max(bounds[r + 1] - bounds[r] for r in range(W)))
            buf = torch.full((W * pad,), -99, dtype=torch.int64, device="cuda")
            for r, h in enumerate(hs):
                b, e = bounds[r], bounds[r + 1]
                if locals_[r].numel() < pad:
                    locals_[r] = torch.zeros(2 * pad, dtype=torch.int64, device="cuda")
                h.evaluate(b, e, locals_[r])
                begins_nonzero += int(b > 0 and e > b)
                buf[r * pad:r * pad + (e - b)] = locals_[r][:e - b]
            full = adist.concat_shards(buf, pad, bounds)
            assert full.numel() == C
            for h in hs:
                h.apply(full)
        out = []
        for h in hs:
            res = h.result()
            hist = [h.history(r) for r in range(h.num_runs())]
            out.append((res, hist))
        return out, begins_nonzero
    finally:
        for h in hs:
            h.close()
        for s in sims:
            s.close()


def _world1(prob, tr, chunk, **kw):
    from paper_2302_11665_b200 import Simulator
    with Simulator(0) as s:
        s.set_problem(prob)
        s.set_trace(tr.arrival_ns, tr.model)
        s.set_chunk_size(chunk)
        with s.search_handle(**kw) as h:
            from paper_2302_11665_b200 import dist as adist
            adist.run_search(h)
            return h.result(), [h.history(r) for r in range(h.num_runs())]


def _check(prob, tr, W, chunk, balance="cost", **kw):
    ref = osearch.alg2(prob, tr)
    one, one_hist = _world1(prob, tr, chunk, **kw)
    ranks, nz = emulate(prob, tr, W, chunk, balance, **kw)
    assert nz > 0, "no rank evaluated a shard with begin > 0"
    for res, hist in ranks:
        assert (res.best_run, res.best_good) == (one.best_run, one.best_good)
        assert (res.best_run, res.best_good) == (ref["run"], ref["good"])
        np.testing.assert_array_equal(res.host_mask, ref["placement"].host_mask)
        for r, (a, b) in enumerate(zip(hist, one_hist)):
            for x, y in zip(a, b):  # every step's winner and its good, every run
                np.testing.assert_array_equal(x, y, err_msg=f"run {r}")
        for r_gpu, r_one, r_ref in zip(res.runs, one.runs, ref["runs"]):
            assert r_gpu["best_good"] == r_one["best_good"]
            np.testing.assert_array_equal(r_gpu["host_mask"], r_one["host_mask"])
            if r_gpu["pruned_at"] < 0:
                assert r_gpu["best_good"] == r_ref["good"]
                np.testing.assert_array_equal(r_gpu["host_mask"], r_ref["placement"].host_mask)


def _s3_small():
    names = [f"{b}#{i}" for b in ("BERT-1.3B", "BERT-2.7B", "BERT-6.7B", "MoE-1.3B",
                                  "MoE-2.4B", "MoE-5.3B") for i in range(2)]
    prob = configs.build_problem(names, 8, 13 * 10**9, slo_scale=5.0)
    tr = traces.maf2_shaped(4, len(names), 20.0, 300.0)
    return prob, tr


@pytest.mark.parametrize("W", [2, 3, 8])
@pytest.mark.parametrize("chunk", [4096, 40, 257])
def test_sharded_search_emulated(W, chunk):
    prob, tr = _s3_small()
    _check(prob, tr, W, chunk, dedup=False, prune=True)


@pytest.mark.parametrize("W", [2, 3])
def test_sharded_search_emulated_count_split_dedup(W):
    """Equal-count shards (other shard boundaries), de-duplication on."""
    names = [f"{b}#{i}" for b in ("BERT-1.3B", "BERT-2.7B", "MoE-5.3B") for i in range(2)]
    prob = configs.build_problem(names, 8, 13 * 10**9, slo_scale=3.0)
    tr = traces.maf2_shaped(11, len(names), 12.0, 900.0)
    _check(prob, tr, W, 40, balance="count", dedup=True, prune=False)


def test_sharded_search_emulated_int64_times():
    """S4-shaped (23 s SLO: int64 absolute times in the chunked path), W = 3."""
    prob, tr = configs.s4(duration=1800.0)
    _check(prob, tr, 3, 97, dedup=False, prune=True)
