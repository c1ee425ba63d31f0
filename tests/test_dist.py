"""Multi-rank candidate sharding (paper_2302_11665_b200/dist.py) on CPU with
the gloo backend, world size 2 and 3: a CPU engine implementing the stepwise
search protocol (prepare / evaluate shard / apply gathered) drives the same
run_search loop the GPU path uses; every rank must end with the placement the
single-process oracle search finds."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import search as osearch
import oracle
from workloads import Placement, configs, traces


class OracleEngine:
    """Test-only engine: the lockstep Alg. 2 / Alg. 1 protocol on the oracle."""

    def __init__(self, prob, tr):
        self.prob, self.tr = prob, tr
        self.op, self.ot = oracle.OracleProblem(prob), oracle.OracleTrace(tr)
        self.runs = []
        for size, p, cfg in osearch.alg2_runs(prob):
            self.runs.append(dict(cfg=np.array(cfg, np.int32), sel=np.zeros(prob.num_models,
                                                                             np.uint64),
                                  best=np.zeros(prob.num_models, np.uint64), best_good=0,
                                  active=True))
        self.cands = []

    def prepare(self):
        self.cands = []
        for r, run in enumerate(self.runs):
            if not run["active"]:
                continue
            n = 0
            for m in range(self.prob.num_models):
                for g in range(len(run["cfg"])):
                    if (int(run["sel"][m]) >> g) & 1:
                        continue
                    nm = run["sel"].copy()
                    nm[m] |= np.uint64(1) << np.uint64(g)
                    if oracle.feasible(self.op, Placement(run["cfg"], nm)):
                        self.cands.append((r, m, g, nm))
                        n += 1
            if n == 0:
                run["active"] = False
        return len(self.cands) if self.cands else -1

    def evaluate(self, b, e, out, stream=None):
        if e <= b:
            return
        G = max(len(run["cfg"]) for run in self.runs)
        cfg = np.full((e - b, G), -1, np.int32)
        mask = np.zeros((e - b, self.prob.num_models), np.uint64)
        for i, (r, m, g, nm) in enumerate(self.cands[b:e]):
            cfg[i, :len(self.runs[r]["cfg"])] = self.runs[r]["cfg"]
            mask[i] = nm
        good, _, _ = oracle.evaluate(self.op, self.ot, cfg, mask, 1)
        out[:e - b] = torch.from_numpy(good)

    def apply(self, full, stream=None):
        good = full.cpu().numpy()
        best = {}
        for i, (r, m, g, nm) in enumerate(self.cands):
            if r not in best or good[i] > best[r][0]:
                best[r] = (int(good[i]), i)
        for r, (gv, i) in best.items():
            run = self.runs[r]
            run["sel"] = self.cands[i][3]
            if gv > run["best_good"]:
                run["best_good"], run["best"] = gv, run["sel"].copy()


def _problem():
    names = [f"BERT-1.3B#{i}" for i in range(3)] + [f"MoE-2.4B#{i}" for i in range(2)]
    prob = configs.build_problem(names, 4, 13 * 10**9, slo_scale=2.0)
    tr = traces.maf2_shaped(5, len(names), 6.0, 120.0)
    return prob, tr


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2302_11665_b200 import dist as adist
    prob, tr = _problem()
    eng = OracleEngine(prob, tr)
    steps = adist.run_search(eng, device=torch.device("cpu"))
    q.put((rank, steps, [(int(r["best_good"]), r["best"].tolist()) for r in eng.runs]))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_covers_exactly():
    from paper_2302_11665_b200.dist import shard
    for C in (0, 1, 5, 17, 1000):
        for W in (1, 2, 3, 8):
            parts = [shard(C, r, W) for r in range(W)]
            assert parts[0][0] == 0 and parts[-1][1] == C
            for (a, b), (c, d) in zip(parts, parts[1:]):
                assert b == c and a <= b
            assert max(e - b for b, e in parts) <= -(-C // W) if C else True


def test_shard_bounds_balance_cost():
    from paper_2302_11665_b200.dist import shard_bounds
    rng = np.random.default_rng(0)
    for C in (0, 1, 2, 7, 100, 1000):
        for W in (1, 2, 3, 8):
            cost = rng.integers(1, 1000, size=C)
            if C > 3:
                cost[C // 3] = 10**6  # one heavy candidate
            b = shard_bounds(cost, W)
            assert len(b) == W + 1 and b[0] == 0 and b[-1] == C
            assert all(x <= y for x, y in zip(b, b[1:]))
            if C == 0:
                continue
            total = int(cost.sum())
            pref = np.concatenate([[0], np.cumsum(cost)])
            for r in range(W):
                # shard r holds the candidates whose cost prefix ends in
                # (r T / W, (r+1) T / W] (the last shard: up to T)
                for i in range(b[r], b[r + 1]):
                    assert pref[i + 1] * W > r * total
                    if r < W - 1:
                        assert pref[i] * W < (r + 1) * total or i == b[r]
            # equal costs: the count split differs by at most one per shard
            eq = shard_bounds(np.ones(C, np.int64), W)
            sizes = np.diff(eq)
            assert sizes.max() - sizes.min() <= 1


def test_concat_shards_orders_globally():
    from paper_2302_11665_b200.dist import concat_shards, shard_bounds
    for C, W in ((10, 3), (5, 8), (1, 2), (64, 4)):
        bounds = shard_bounds(np.arange(1, C + 1), W)
        pad = max(1, max(np.diff(bounds)))
        buf = torch.full((W * pad,), -7, dtype=torch.int64)
        for r in range(W):
            n = bounds[r + 1] - bounds[r]
            buf[r * pad:r * pad + n] = torch.arange(bounds[r], bounds[r + 1])
        assert concat_shards(buf, pad, bounds).tolist() == list(range(C))


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_search_matches_single_process(world):
    prob, tr = _problem()
    ref = osearch.alg2(prob, tr)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    outs.sort()
    for rank, steps, runs in outs:
        assert runs == outs[0][2]  # identical state on every rank
        for (bg, best), r_ref in zip(runs, ref["runs"]):
            assert bg == r_ref["good"]
            assert best == r_ref["placement"].host_mask.tolist()


def _batching_case():
    from tests.helpers import place
    prob, tr, inc = configs.s1_batching(seed=2, duration=20.0, slo_scale=3.0, delta=0.9)
    M = prob.num_models
    rng = np.random.default_rng(0)
    pls = []
    for p, (s, n) in enumerate(prob.configs):
        G = 16 // (s * n)
        for _ in range(3):
            groups = [[m for m in range(M) if rng.random() < 0.15] for _ in range(G)]
            pls.append(place([p] * G, groups, M))
    cfg = np.full((len(pls), 16), -1, np.int32)
    mask = np.zeros((len(pls), M), np.uint64)
    for i, pl in enumerate(pls):
        cfg[i, :pl.num_groups] = pl.group_cfg
        mask[i] = pl.host_mask
    return prob, tr, inc, cfg, mask


def _batching_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2302_11665_b200 import dist as adist
    prob, tr, inc, cfg, mask = _batching_case()

    def run(b, e):  # CPU engine behind the same sharding logic
        g, _, _ = oracle.evaluate_batching(prob, tr, cfg[b:e], mask[b:e], inc, 3, threads=2)
        return torch.from_numpy(g)

    def first_max(good):  # test-side argmax (the GPU path uses the library kernel)
        g = good.numpy()
        return int(np.argmax(g)) if g.size and g.max() >= 0 else -1

    good, arg = adist.evaluate_sharded(run, first_max, len(cfg), device=torch.device("cpu"))
    q.put((rank, good.tolist(), arg))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_batching_matches_single_process(world):
    prob, tr, inc, cfg, mask = _batching_case()
    ref, _, _ = oracle.evaluate_batching(prob, tr, cfg, mask, inc, 3)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_batching_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = int(np.argmax(ref)) if ref.max() >= 0 else -1
    for rank, good, arg in outs:
        assert good == ref.tolist() and arg == want
