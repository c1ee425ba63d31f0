"""Small hand-made instances shared by the tests (no method arithmetic)."""

from __future__ import annotations

import numpy as np

from workloads import Placement, Problem, Trace

INF = np.iinfo(np.int64).max


def tiny_problem(configs, stage, tail=None, slo=None, mem=None, num_devices=64,
                 budget=10**15, latency=None):
    """configs: [(s, n)]; stage[m][p] = list of s_p stage ns; tail[m][p]; slo[m]."""
    M, P = len(stage), len(configs)
    S = max(s for s, _ in configs)
    st = np.zeros((M, P, S), np.int64)
    for m in range(M):
        for p, (s, _) in enumerate(configs):
            assert len(stage[m][p]) == s
            st[m, p, :s] = stage[m][p]
    tl = np.zeros((M, P), np.int64) if tail is None else np.asarray(tail, np.int64).reshape(M, P)
    sl = np.full(M, INF, np.int64) if slo is None else np.asarray(slo, np.int64)
    mm = np.ones((M, P), np.int64) if mem is None else np.asarray(mem, np.int64).reshape(M, P)
    lat = latency if latency is not None else [int(st[m, 0].sum()) for m in range(M)]
    p = Problem([f"m{m}" for m in range(M)], list(configs), sl, st, tl, mm, num_devices, budget,
                dict(latency_ns=lat, slo_scale=None))
    p.validate()
    return p


def trace_of(pairs):
    """pairs = [(arrival_ns, model)] (already in order)."""
    a = np.array([x for x, _ in pairs], np.int64)
    m = np.array([y for _, y in pairs], np.int32)
    return Trace(a, m)


def place(group_cfg, groups_models, M):
    return Placement.from_lists(group_cfg, groups_models, M)


def random_instance(rng, M=None, G=None, max_s=4, n_req=40, dmax=5, tmax=30, slo_choices=None,
                    P=None, allow_unhosted=True):
    """Random small instance for parity/determinism tests (family F3-like):
    random configs, stage vectors with zeros and ties, duplicate timestamps."""
    M = M or int(rng.integers(1, 4))
    P = P or int(rng.integers(1, 4))
    configs = [(int(rng.integers(1, max_s + 1)), 1) for _ in range(P)]
    stage = [[list(rng.integers(0, dmax + 1, size=s)) for s, _ in configs] for _ in range(M)]
    tail = rng.integers(0, 3, size=(M, P))
    if slo_choices is None:
        slo_choices = [0, 3, 8, 20, INF]
    slo = [int(rng.choice(slo_choices)) for _ in range(M)]
    prob = tiny_problem(configs, stage, tail, slo)
    G = G or int(rng.integers(1, 5))
    cfg = [int(rng.integers(0, P)) for _ in range(G)]
    groups = []
    for g in range(G):
        groups.append([m for m in range(M) if rng.random() < 0.6])
    if not allow_unhosted:
        for m in range(M):
            if not any(m in gm for gm in groups):
                groups[int(rng.integers(0, G))].append(m)
    pl = place(cfg, groups, M)
    a = np.sort(rng.integers(0, tmax, size=n_req)).astype(np.int64)
    mo = rng.integers(0, M, size=n_req).astype(np.int32)
    return prob, Trace(a, mo), pl
