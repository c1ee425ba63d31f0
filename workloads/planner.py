"""Per-(model, parallel config) stage tables: the inputs Alg. 1's
`parallelize(m, g, p)` produces.

§4.1: the inter-op pass minimises the maximal stage latency,
    F(s, k) = min_{1<=i<=k} max{ F(s-1, i-1), latency(i, k) },
with latency(i, k) the sum of the profiled latencies of layers i..k.  The
intra-op ILP needs Alpa and real operator graphs and is replaced by
SPEC's one-parameter model (reading C16): a layer of latency L run
n-way intra-op takes L*(1/n + gamma*(n-1)/n).

Everything here is integer nanoseconds after one rounding per layer.
"""

from __future__ import annotations

import numpy as np


def enumerate_configs(group_size: int, max_stages: int, pipeline_only: bool = False):
    """All (s, n) with s*n == group_size and s <= max_stages, s ascending
    (`get_potential_parallel_configs`; "drop all configurations that
    use data parallelism")."""
    out = []
    for s in range(1, group_size + 1):
        if group_size % s == 0 and s <= max_stages:
            n = group_size // s
            if pipeline_only and n != 1:
                continue
            out.append((s, n))
    return out


def layer_latencies_ns(latency_ns: int, num_layers: int, n: int, gamma: float) -> np.ndarray:
    """K equal layers each scaled by the intra-op model."""
    per = latency_ns * (1.0 / n + gamma * (n - 1) / n) / num_layers
    return np.full(num_layers, int(np.rint(per)), dtype=np.int64)


def partition_dp(layers: np.ndarray, s: int):
    """The §4.1 DP F(s, k), ties toward the earlier split point
    (S:179).  Returns (boundaries, stage_latencies): boundaries[j] = (i, k)
    0-based inclusive layer range of stage j."""
    K = len(layers)
    if not 1 <= s <= K:
        raise ValueError("need 1 <= s <= K")
    pre = np.concatenate([[0], np.cumsum(layers)]).tolist()

    def lat(i, k):  # layers i..k, 1-based inclusive
        return pre[k] - pre[i - 1]

    INF = float("inf")
    F = [[INF] * (K + 1) for _ in range(s + 1)]
    arg = [[0] * (K + 1) for _ in range(s + 1)]
    F[0][0] = 0
    for t in range(1, s + 1):
        for k in range(t, K + 1):
            best, besti = INF, 0
            for i in range(t, k + 1):  # last stage = layers i..k; >= t-1 layers before
                v = max(F[t - 1][i - 1], lat(i, k))
                if v < best:  # strict: keeps the earliest split on ties
                    best, besti = v, i
            F[t][k] = best
            arg[t][k] = besti
    bounds = []
    k = K
    for t in range(s, 0, -1):
        i = arg[t][k]
        bounds.append((i - 1, k - 1))
        k = i - 1
    bounds.reverse()
    stage = np.array([lat(i + 1, k + 1) for i, k in bounds], dtype=np.int64)
    assert int(stage.max()) == F[s][K]
    return bounds, stage


def config_tables(models, configs, num_layers, gamma=0.15, comm_ns=500_000,
                  max_stages=None):
    """Build (stage_ns[M,P,S], tail_ns[M,P], mem_bytes[M,P]).

    models: list of (weight_bytes, latency_ns, num_layers or None, comm_ns or None)
    tail = (s-1) * comm_ns: inter-stage communication is charged to the
    finish only (reading C4; "most overhead comes from the latency
    imbalance ... instead of the communication").
    mem = ceil(bytes / (s*n)) per device (reading C11).
    """
    M, P = len(models), len(configs)
    S = max_stages or max(s for s, _ in configs)
    stage = np.zeros((M, P, S), dtype=np.int64)
    tail = np.zeros((M, P), dtype=np.int64)
    mem = np.zeros((M, P), dtype=np.int64)
    for mi, (nbytes, lat_ns, K_m, c_m) in enumerate(models):
        K = K_m or num_layers
        c = comm_ns if c_m is None else c_m
        for p, (s, n) in enumerate(configs):
            if s > K:
                mem[mi, p] = -1
                continue
            layers = layer_latencies_ns(lat_ns, K, n, gamma)
            _, st = partition_dp(layers, s)
            stage[mi, p, :s] = st
            tail[mi, p] = (s - 1) * c
            mem[mi, p] = -(-nbytes // (s * n))
    return stage, tail, mem

