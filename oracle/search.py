"""Oracle placement search -- TEST INFRASTRUCTURE ONLY.

Written step by step in the order and notation of the paper:

Alg. 1 "Simulator-Guided Greedy Model Selection", beam k = 1:
    best_sel <- {} ; beam_sels <- {{}}
    while true:
        new_sels <- {}
        for (m, (g, p)) in M x (G, P):
            sel' <- sel.add_model_to_group(m, g)
            if sel' is in memory constraint: simulate(sel', W); append
        if new_sels = {}: break
        sel* <- pick_highest_slo_attainment(new_sels)
        if sel*.slo_att > best_sel.slo_att: best_sel <- sel*
Readings (C11, C12): (m, g) enumerated m-major, g-minor; a model
is placed at most once per group; ties go to the first candidate; `best`
updates on strict '>'; the empty selection has attainment 0.

Alg. 2 "Enumeration-Based Group Partition and Model-Parallel Configuration
Selection", single bucket: group partitions are D/size equal
groups for every divisor size of the device count, ascending ("all groups
have the same size and the same parallel configurations"); for each,
every config of that size in problem order; the best run (strict '>') wins.

Fast heuristic: "Instead of using the simulator to evaluate all
(model, group) pairs at each iteration, we can run the simulator only once
and place a model with the most unserved requests in an available group with
the lowest utilization."  Readings (C22-C24): unserved(m) = requests
of m not good in the simulation of the current selection; a model qualifies
when unserved > 0 and it has an available group (not hosting it, memory
feasible); utilization(g) = sum over the requests g served of their stage
occupancies / (s_g * horizon) -- the mean stage utilization, horizon common
to all groups; ties -> lowest m, lowest g; the loop ends when no model
qualifies; best selection on strict '>' as in Alg. 1.

Brute force: every placement of a tiny cluster -- every multiset of group
sizes summing to D (non-increasing), every config per group, every
memory-feasible model subset per group.
"""

from __future__ import annotations

import itertools
from fractions import Fraction

import numpy as np

from workloads import Placement

from . import OracleProblem, OracleTrace, evaluate, feasible, simulate


def _add(mask: np.ndarray, m: int, g: int) -> np.ndarray:
    out = mask.copy()
    out[m] |= np.uint64(1) << np.uint64(g)
    return out


def greedy(prob, trace, group_cfg, threads: int = 0, record: bool = False):
    """Alg. 1 with k = 1 on fixed groups `group_cfg`.
    Returns dict(placement, good, steps=[(candidates, goods, chosen)])."""
    op = prob if isinstance(prob, OracleProblem) else OracleProblem(prob)
    ot = trace if isinstance(trace, OracleTrace) else OracleTrace(trace)
    M = op.prob.num_models
    cfg = np.asarray(group_cfg, dtype=np.int32)
    G = len(cfg)
    sel = np.zeros(M, dtype=np.uint64)
    best_sel, best_good = sel.copy(), 0
    steps = []
    while True:
        cands = []
        for m in range(M):
            for g in range(G):
                if (int(sel[m]) >> g) & 1:
                    continue  # already hosted on g
                nm = _add(sel, m, g)
                if feasible(op, Placement(cfg, nm)):
                    cands.append((m, g, nm))
        if not cands:
            break
        masks = np.stack([c[2] for c in cands])
        goods, _, _ = evaluate(op, ot, np.tile(cfg, (len(cands), 1)), masks, threads)
        i = int(np.argmax(goods))  # first maximum = lowest candidate index
        sel = cands[i][2]
        if record:
            steps.append(([(m, g) for m, g, _ in cands], goods.copy(), i))
        if goods[i] > best_good:
            best_sel, best_good = sel.copy(), int(goods[i])
    return dict(placement=Placement(cfg, best_sel), good=best_good, steps=steps)


def utilization_busy(prob, model, group_cfg, served_by):
    """Per group g: sum over the requests it served of sum_k stage_ns[m][cfg_g][k]
    (the numerator of its mean stage utilization, reading C23)."""
    cfg = np.asarray(group_cfg, dtype=np.int64)
    served_by = np.asarray(served_by)
    model = np.asarray(model)
    busy = [0] * len(cfg)
    for g in range(len(cfg)):
        p = int(cfg[g])
        s = int(prob.cfg_stages[p])
        occ = np.asarray(prob.stage_ns)[:, p, :s].sum(axis=1)  # per model, one request
        counts = np.bincount(model[served_by == g], minlength=prob.num_models)
        busy[g] = sum(int(c) * int(o) for c, o in zip(counts, occ))
    return busy


def greedy_fast(prob, trace, group_cfg, record: bool = False):
    """The fast heuristic of P:737 on fixed groups `group_cfg`.
    Returns dict(placement, good, steps=[(good, (m, g) or None)])."""
    op = prob if isinstance(prob, OracleProblem) else OracleProblem(prob)
    ot = trace if isinstance(trace, OracleTrace) else OracleTrace(trace)
    pr = op.prob
    M = pr.num_models
    cfg = np.asarray(group_cfg, dtype=np.int32)
    G = len(cfg)
    n_m = np.bincount(ot.model, minlength=M)
    sel = np.zeros(M, dtype=np.uint64)
    best_sel, best_good = sel.copy(), 0
    steps = []
    while feasible(op, Placement(cfg, sel)):
        # "run the simulator only once"
        r = simulate(op, ot, Placement(cfg, sel), detail=True)
        if r["good"] > best_good:
            best_sel, best_good = sel.copy(), r["good"]
        unserved = [int(n_m[m]) - int(r["good_per_model"][m]) for m in range(M)]
        busy = utilization_busy(pr, ot.model, cfg, r["served_by"])
        pick = None
        for m in sorted(range(M), key=lambda m: (-unserved[m], m)):  # most unserved first
            if unserved[m] <= 0:
                break
            # "an available group with the lowest utilization": busy_g / s_g, lowest g on ties
            avail = [g for g in range(G)
                     if not (int(sel[m]) >> g) & 1 and feasible(op, Placement(cfg, _add(sel, m, g)))]
            if avail:
                g = min(avail, key=lambda g: (Fraction(busy[g], int(pr.cfg_stages[cfg[g]])), g))
                pick = (m, g)
                break
        if record:
            steps.append((r["good"], pick))
        if pick is None:
            break
        sel = _add(sel, *pick)
    return dict(placement=Placement(cfg, best_sel), good=best_good, steps=steps)


def alg2_fast(prob, trace, record: bool = False):
    """Alg. 2 (single bucket) around the fast heuristic; strict '>' across runs."""
    op, ot = OracleProblem(prob), OracleTrace(trace)
    best = dict(placement=Placement(np.zeros(0, np.int32), np.zeros(prob.num_models, np.uint64)),
                good=0, run=-1)
    runs = []
    for r, (size, p, cfg) in enumerate(alg2_runs(prob)):
        res = greedy_fast(op, ot, cfg, record)
        runs.append(res)
        if res["good"] > best["good"]:
            best = dict(res, run=r)
    best["runs"] = runs
    return best


def alg2_runs(prob):
    """Single-bucket Alg. 2 enumeration: [(size, config id, group_cfg list)]."""
    D = prob.num_devices
    devs = prob.cfg_devices
    runs = []
    for size in range(1, D + 1):
        if D % size:
            continue
        for p in range(prob.num_configs):
            if int(devs[p]) == size:
                runs.append((size, p, [p] * (D // size)))
    return runs


def alg2(prob, trace, threads: int = 0, record: bool = False):
    """Alg. 2 (single bucket) around Alg. 1; strict '>' keeps the first best run."""
    op, ot = OracleProblem(prob), OracleTrace(trace)
    best = dict(placement=Placement(np.zeros(0, np.int32), np.zeros(prob.num_models, np.uint64)),
                good=0, run=-1)
    runs = []
    for r, (size, p, cfg) in enumerate(alg2_runs(prob)):
        res = greedy(op, ot, cfg, threads, record)
        runs.append(res)
        if res["good"] > best["good"]:
            best = dict(res, run=r)
    best["runs"] = runs
    return best


def _size_partitions(D, sizes):
    """Multisets of allowed sizes summing to D, non-increasing."""
    sizes = sorted(set(sizes), reverse=True)

    def rec(rem, maxs):
        if rem == 0:
            yield ()
            return
        for s in sizes:
            if s <= rem and s <= maxs:
                for rest in rec(rem - s, s):
                    yield (s,) + rest

    return list(rec(D, D))


def bruteforce_placements(prob):
    """Every placement of the cluster (tiny instances only)."""
    D = prob.num_devices
    M = prob.num_models
    devs = prob.cfg_devices
    by_size = {}
    for p in range(prob.num_configs):
        by_size.setdefault(int(devs[p]), []).append(p)
    out = []
    subsets = [tuple(c) for r in range(M + 1) for c in itertools.combinations(range(M), r)]
    for part in _size_partitions(D, by_size.keys()):
        for cfgs in itertools.product(*[by_size[s] for s in part]):
            G = len(cfgs)
            per_group = []
            for g in range(G):
                ok = []
                for sub in subsets:
                    mem = prob.mem_bytes[list(sub), cfgs[g]] if sub else np.zeros(0, np.int64)
                    if np.all(mem >= 0) and int(mem.sum()) <= prob.budget_bytes:
                        ok.append(sub)
                per_group.append(ok)
            for choice in itertools.product(*per_group):
                out.append(Placement.from_lists(list(cfgs), choice, M))
    return out


def bruteforce(prob, trace, threads: int = 0):
    """Exhaustive optimum: (best placement, best good, all placements, goods)."""
    pls = bruteforce_placements(prob)
    Gmax = max(p.num_groups for p in pls)
    cfg = np.full((len(pls), Gmax), -1, np.int32)
    mask = np.zeros((len(pls), prob.num_models), np.uint64)
    for i, p in enumerate(pls):
        cfg[i, :p.num_groups] = p.group_cfg
        mask[i] = p.host_mask
    goods, _, _ = evaluate(prob, trace, cfg, mask, threads)
    i = int(np.argmax(goods))
    return dict(placement=pls[i], good=int(goods[i]), placements=pls, goods=goods,
                group_cfg=cfg, host_mask=mask)


__all__ = ["greedy", "alg2", "alg2_runs", "bruteforce", "bruteforce_placements", "simulate"]
