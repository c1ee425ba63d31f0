"""Concrete inputs for the BASELINE.json configs (SURVEY §8(d) recipe).

motivating  2 x 6.7B-like models (D=0.4 s, 13.4 GB), 2 GPUs of 16 GB,
            independent Poisson 1.5 req/s each
S1          32 x BERT-1.3B, 16 devices, Gamma arrivals, equal split
S2          32 x BERT-6.7B, 64 devices, MAF1-shaped power-law trace
S3          60 mixed BERT/MoE, 64 devices, MAF2-shaped trace (the target)
S4          4 x BERT-104B, 64 devices, pipeline-only configs, Gamma 8 req/s,
            CV 4, power-law 0.5 split

Every constant that the paper does not print (K layers, gamma, per-boundary
communication c_b, trace shape parameters) is an assumption listed in
DESIGN.md ("parity unpinned" inputs).
"""

from __future__ import annotations

import numpy as np

from . import planner, table1, traces
from .problem import Problem

MS = 10**6


def divisors(n: int):
    return [d for d in range(1, n + 1) if n % d == 0]


def all_configs(num_devices: int, max_stages: int, pipeline_only=False):
    """Every (s, n) used by some equal-size group partition of the cluster
    (sizes = divisors of the device count, reading C13)."""
    out = []
    for size in divisors(num_devices):
        out += planner.enumerate_configs(size, max_stages, pipeline_only)
    return out


def build_problem(model_names, num_devices, budget, slo_scale=5.0, num_layers=24,
                  gamma=0.15, comm_ns=500_000, pipeline_only=False, configs=None,
                  per_model=None) -> Problem:
    """per_model[name] = (bytes, latency_ns, K or None, comm_ns or None) overrides Table 1."""
    specs = []
    for name in model_names:
        if per_model and name in per_model:
            specs.append(per_model[name])
        else:
            b, lat = table1.MODELS[name.split("#")[0]]
            specs.append((b, lat, None, None))
    maxK = max((k or num_layers) for _, _, k, _ in specs)
    if configs is None:
        configs = all_configs(num_devices, maxK, pipeline_only)
    stage, tail, mem = planner.config_tables(specs, configs, num_layers, gamma, comm_ns)
    lat = np.array([lt for _, lt, _, _ in specs], dtype=np.int64)
    slo = np.rint(lat.astype(np.float64) * slo_scale).astype(np.int64)
    p = Problem(list(model_names), list(configs), slo, stage, tail, mem, num_devices, budget,
                dict(latency_ns=lat.tolist(), slo_scale=slo_scale, num_layers=num_layers,
                     gamma=gamma, comm_ns=comm_ns))
    p.validate()
    return p


def expand_set(set_name: str):
    names = []
    for base, count in table1.SETS[set_name].items():
        names += [f"{base}#{i}" for i in range(count)]
    return names


def _base(name: str) -> str:
    return name.split("#")[0]


def table1_problem(set_name, num_devices, slo_scale=5.0, pipeline_only=False, **kw) -> Problem:
    names = expand_set(set_name)
    per = {}
    for n in names:
        b, lat = table1.MODELS[_base(n)]
        if _base(n) == "BERT-104B":
            # 96 layers, 2 ms per stage boundary (SURVEY §8(d) assumption)
            per[n] = (b, lat, 96, 2_000_000)
        else:
            per[n] = (b, lat, None, None)
    return build_problem(names, num_devices, table1.DEVICE_BUDGET, slo_scale,
                         pipeline_only=pipeline_only, per_model=per, **kw)


# --------------------------------------------------------------------------- motivating
def motivating_problem(slo_scale=5.0, tail_ns=0) -> Problem:
    """2 models of D = 0.4 s and 13.4 GB on 2 GPUs with 16 GB.
    Configs (1,1) d=[0.4 s]; (2,1) d=[0.2, 0.2] s (zero-overhead pipeline,
    P:517 "D_s = 2 D_m = D"); (1,2) d=[0.23 s] (gamma = 0.15 intra-op model)."""
    per = {n: (int(13.4 * 10**9), 400 * MS, 2, tail_ns) for n in ("A", "B")}
    return build_problem(["A", "B"], 2, table1.V100_MEMORY, slo_scale, num_layers=2,
                         configs=[(1, 1), (1, 2), (2, 1)], per_model=per)


def motivating_trace(seed=0, n_requests=1000, cv=1.0, split=(0.5, 0.5), total_rate=3.0):
    duration = n_requests / total_rate * 1.05
    tr = traces.independent_gamma(seed, [total_rate * split[0], total_rate * split[1]], cv,
                                  duration)
    return tr.prefix(min(n_requests, len(tr)))


# --------------------------------------------------------------------------- S1..S4
def s1(seed=0, rate=64.0, cv=4.0, duration=3600.0, slo_scale=5.0):
    prob = table1_problem("S1", 16, slo_scale)
    M = prob.num_models
    tr = traces.independent_gamma(seed, [rate / M] * M, cv, duration)
    return prob, tr


def s2(seed=0, rate=80.0, duration=3600.0, slo_scale=5.0):
    prob = table1_problem("S2", 64, slo_scale)
    tr = traces.maf1_shaped(seed, prob.num_models, rate, duration)
    return prob, tr


def s3(seed=0, rate=100.0, duration=86400.0, slo_scale=5.0, cv=4.0):
    """The target config; shorter traces are the opening stretch of the day
    (the day's per-model MAF2 window factors, normalised over the day)."""
    prob = table1_problem("S3", 64, slo_scale)
    tr = traces.maf2_shaped(seed, prob.num_models, rate, duration, cv=cv,
                            horizon=max(duration, 86400.0))
    return prob, tr


def s4(seed=0, rate=8.0, cv=4.0, duration=86400.0, slo_scale=5.0):
    prob = table1_problem("S4", 64, slo_scale, pipeline_only=True)
    rng = np.random.default_rng(seed + 1)
    w = traces.power_law_weights(prob.num_models, 0.5, rng)
    tr = traces.split_gamma(seed, rate, cv, duration, w)
    return prob, tr


CONFIGS = {"S1": s1, "S2": s2, "S3": s3, "S4": s4}


# ------------------------------------------------------------- dynamic batching (§5.4)
def batch_increment_ns(stage_ns, delta: float) -> np.ndarray:
    """Per-stage increment of a batched stage: a batch of k occupies stage j for
    stage_ns + (k-1) * round(delta * stage_ns) ns, i.e. "the execution latency
    grows linearly with the batch size" with slope delta (SPEC S:34,
    L(1)(1 + delta (k-1))).  Input generation only (round half even, once)."""
    return np.rint(np.asarray(stage_ns, dtype=np.float64) * delta).astype(np.int64)


def s1_batching(seed=0, rate_per_model=4.0, cv=4.0, duration=600.0, slo_scale=5.0,
                delta=0.9):
    """§5.4 setup: model set S1, "synthetic Gamma Process traffic
    with an average rate of 4 requests/s and a CV of 4 for each model".
    Returns (problem, trace, stage_inc_ns)."""
    prob = table1_problem("S1", 16, slo_scale)
    M = prob.num_models
    tr = traces.independent_gamma(seed, [rate_per_model] * M, cv, duration)
    return prob, tr, batch_increment_ns(prob.stage_ns, delta)
