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


def greedy(prob, trace, group_cfg, threads: int = 0, record: bool = False, models=None):
    """Alg. 1 with k = 1 on fixed groups `group_cfg`; `models` restricts the
    selectable models (a bucket of Alg. 2: requests of other models
    are simply not served).
    Returns dict(placement, good, steps=[(candidates, goods, chosen)])."""
    op = prob if isinstance(prob, OracleProblem) else OracleProblem(prob)
    ot = trace if isinstance(trace, OracleTrace) else OracleTrace(trace)
    M = op.prob.num_models
    cfg = np.asarray(group_cfg, dtype=np.int32)
    G = len(cfg)
    sel = np.zeros(M, dtype=np.uint64)
    best_sel, best_good = sel.copy(), 0
    steps = []
    allowed = range(M) if models is None else sorted(models)
    while True:
        cands = []
        for m in allowed:
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


def greedy_beam(prob, trace, group_cfg, k: int, threads: int = 0, models=None):
    """Alg. 1 with beam size k (readings C29-C30): every member of
    beam_sels is extended by every feasible (m, g) in (member, m, g) order;
    selections reached twice keep their first occurrence; beam_sels =
    top-k by good (stable: ties keep new_sels order); sel* = the first of them;
    best_sel on strict '>'.  k = 1 is `greedy`."""
    op = prob if isinstance(prob, OracleProblem) else OracleProblem(prob)
    ot = trace if isinstance(trace, OracleTrace) else OracleTrace(trace)
    M = op.prob.num_models
    cfg = np.asarray(group_cfg, dtype=np.int32)
    G = len(cfg)
    allowed = range(M) if models is None else sorted(models)
    beam = [np.zeros(M, dtype=np.uint64)]
    best_sel, best_good = beam[0].copy(), 0
    steps = 0
    while True:
        new_sels, seen = [], set()
        for sel in beam:
            for m in allowed:
                for g in range(G):
                    if (int(sel[m]) >> g) & 1:
                        continue
                    nm = _add(sel, m, g)
                    key = nm.tobytes()
                    if key in seen:
                        continue  # the same selection reached from another member
                    if feasible(op, Placement(cfg, nm)):
                        seen.add(key)
                        new_sels.append(nm)
        if not new_sels:
            break
        goods, _, _ = evaluate(op, ot, np.tile(cfg, (len(new_sels), 1)), np.stack(new_sels),
                               threads)
        order = sorted(range(len(new_sels)), key=lambda i: -int(goods[i]))  # stable
        beam = [new_sels[i] for i in order[:k]]
        steps += 1
        if int(goods[order[0]]) > best_good:  # sel* = pick_highest(beam_sels)
            best_sel, best_good = beam[0].copy(), int(goods[order[0]])
    return dict(placement=Placement(cfg, best_sel), good=best_good, steps=steps)


def alg2_beam(prob, trace, k: int, threads: int = 0):
    """Alg. 2 (single bucket) around Alg. 1 with beam size k."""
    op, ot = OracleProblem(prob), OracleTrace(trace)
    best = dict(placement=Placement(np.zeros(0, np.int32), np.zeros(prob.num_models, np.uint64)),
                good=0, run=-1)
    runs = []
    for r, (size, p, cfg) in enumerate(alg2_runs(prob)):
        res = greedy_beam(op, ot, cfg, k, threads)
        runs.append(res)
        if res["good"] > best["good"]:
            best = dict(res, run=r)
    best["runs"] = runs
    return best


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


def greedy_fast(prob, trace, group_cfg, record: bool = False, models=None):
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
        allowed = range(M) if models is None else models
        for m in sorted(allowed, key=lambda m: (-unserved[m], m)):  # most unserved first
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


def alg2_runs(prob, D=None):
    """Single-bucket Alg. 2 enumeration over D devices (default: the cluster):
    [(size, config id, group_cfg list)]."""
    D = prob.num_devices if D is None else D
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


# ----------------------------------------------------------------- Alg. 2, buckets
# get_potential_model_buckets / get_potential_device_buckets and the
# discrepancy pruning (readings C25-C28 in DESIGN.md).

def model_buckets(latency, ratio=Fraction(4), max_buckets=0):
    """Every model bucket partition (reading C25): models sorted by (latency,
    id) and cut into contiguous buckets, never between equal latencies; in each
    bucket max latency <= ratio * min latency ("separate models whose latency
    difference is larger than a threshold"); cuts only where needed -- no two
    neighbouring buckets could form one valid bucket.  Ordered by bucket count,
    then cut positions; max_buckets > 0 drops partitions with more buckets.
    Returns [[sorted model ids of bucket 1], ...] per partition."""
    M = len(latency)
    order = sorted(range(M), key=lambda m: (latency[m], m))
    lat = [latency[m] for m in order]
    cut_points = [i for i in range(1, M) if lat[i - 1] < lat[i]]

    def ok(a, b):  # order[a:b] forms one bucket
        return lat[b - 1] <= ratio * lat[a]

    out = []
    for k in range(1, M + 1):
        if max_buckets and k > max_buckets:
            break
        for cuts in itertools.combinations(cut_points, k - 1):
            bounds = [0, *cuts, M]
            segs = list(zip(bounds[:-1], bounds[1:]))
            if not all(ok(a, b) for a, b in segs):
                continue
            if any(ok(segs[i][0], segs[i + 1][1]) for i in range(len(segs) - 1)):
                continue  # two neighbours would merge: a cut that is not needed
            out.append([sorted(order[a:b]) for a, b in segs])
    return out


def device_buckets(D, k):
    """get_potential_device_buckets: every (H_1, ..., H_k), H_i >= 1, sum D,
    in lexicographic order (reading C26)."""
    if k == 1:
        return [(D,)]
    out = []
    for h in range(1, D - k + 2):
        out += [(h, *rest) for rest in device_buckets(D - h, k - 1)]
    return out


def discrepancy_ok(buckets, H, latency, demand, bound=Fraction(3)):
    """P:783-785 "eliminate the bucket configurations with high discrepancies in
    the estimated number of requests it can serve per second" (reading C26,
    SPEC S:405): capacity_b = H_b / mean latency of bucket b; r_b = demand
    share / capacity share; kept iff max r <= bound * min r."""
    if len(buckets) == 1:
        return True
    dem = [sum(int(demand[m]) for m in b) for b in buckets]
    if sum(dem) == 0:
        return True
    cap = [Fraction(h) / Fraction(sum(int(latency[m]) for m in b), len(b))
           for b, h in zip(buckets, H)]
    r = [Fraction(d, sum(dem)) / (c / sum(cap)) for d, c in zip(dem, cap)]
    return max(r) <= bound * min(r)


def alg2_buckets(prob, trace, latency=None, ratio=Fraction(4), bound=Fraction(3),
                 max_buckets=0, fast=False, threads: int = 0):
    """Alg. 2 with model and device buckets.  Each bucket is
    solved on its own by Alg. 1 (or the fast heuristic) restricted to its
    models over the whole workload; the bucket's best run wins on
    strict '>' ("plm.slo_att > plm_i*.slo_att"); the concatenation's good is
    the sum over buckets (disjoint models and devices); best_plm on strict '>'.
    Returns dict(good, buckets=[(models, H, run group_cfg, host_mask)], ...)."""
    op, ot = OracleProblem(prob), OracleTrace(trace)
    latency = list(prob.meta["latency_ns"] if latency is None else latency)
    M = prob.num_models
    demand = np.bincount(ot.model, minlength=M)
    cache = {}

    def solve(models, h):  # plm_i*: the best of every (G, P) of the bucket
        key = (tuple(models), h)
        if key not in cache:
            best = None
            for size, p, cfg in alg2_runs(prob, h):
                if fast:
                    res = greedy_fast(op, ot, cfg, models=models)
                else:
                    res = greedy(op, ot, cfg, threads, models=models)
                if res["good"] > (best["good"] if best else 0):
                    best = res
            cache[key] = best
        return cache[key]

    best = dict(good=0, buckets=None, partition=None, devices=None)
    considered = []
    for part in model_buckets(latency, ratio, max_buckets):
        for H in device_buckets(prob.num_devices, len(part)):
            if not discrepancy_ok(part, H, latency, demand, bound):
                continue
            considered.append((part, H))
            sols = [solve(b, h) for b, h in zip(part, H)]
            good = sum(s["good"] for s in sols if s is not None)
            if good > best["good"]:
                best = dict(good=good, partition=part, devices=H,
                            buckets=[(b, h, s["placement"] if s else None)
                                     for b, h, s in zip(part, H, sols)])
    best["considered"] = considered
    return best


def concat(prob, bucket_solutions):
    """plm* = concat(plm_1*, ..., plm_k*) as one Placement (groups of bucket 1
    first)."""
    cfgs, masks = [], np.zeros(prob.num_models, np.uint64)
    for _, _, pl in bucket_solutions:
        if pl is None:
            continue
        off = len(cfgs)
        cfgs += [int(c) for c in pl.group_cfg]
        for m in range(prob.num_models):
            masks[m] |= np.uint64(int(pl.host_mask[m]) << off)
    return Placement(np.array(cfgs, np.int32), masks)
