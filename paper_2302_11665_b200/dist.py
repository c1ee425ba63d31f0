"""Multi-GPU candidate sharding for the placement search.

Candidate evaluations inside one greedy iteration are independent -- the
paper simulates "all valid selections" of an iteration before taking the top
k (Alg. 1) -- so each lockstep step's global candidate list is
split into contiguous shards, one per rank, balanced by the library's
per-candidate work estimate (asim_search_costs: requests replayed x stages).
The only exchange per step is an all-gather of the int64 good counts (NCCL
over NVLink on B200s); every rank then applies the same per-run argmax
(lowest global index on ties) inside the library, so the search state stays
identical on all ranks without any further broadcast.

`engine` is anything with prepare() -> C (-1 = finished; 0 = nothing to
simulate this step), evaluate(begin, end, out, stream), apply(good_all,
stream) and optionally costs(C) -> int64[C]: api.SearchHandle on the GPU;
tests inject a CPU engine to exercise this logic under gloo, and emulate
several ranks on one GPU with several SearchHandles and `concat_shards`.
"""

from __future__ import annotations

import contextlib

import numpy as np
import torch
import torch.distributed as dist


def shard(C: int, rank: int, world: int):
    """Contiguous shard [begin, end) of C equal-cost candidates for `rank`."""
    return C * rank // world, C * (rank + 1) // world


def shard_bounds(cost, world: int):
    """Contiguous shard bounds [b_0 = 0, b_1, ..., b_world = C] balanced by
    cost: b_r is the first index whose inclusive cost prefix reaches
    r * total / world (exact integer arithmetic, so every rank computes the
    same bounds from the same costs).  Empty shards are allowed."""
    cost = np.asarray(cost, dtype=np.int64)
    C = int(cost.size)
    if C == 0:
        return [0] * (world + 1)
    pref = np.cumsum(cost, dtype=np.int64)
    total = int(pref[-1])
    bounds = [0]
    for r in range(1, world):
        # first i with pref[i] * world >= r * total  ->  shard r starts after it
        i = int(np.searchsorted(pref * world, r * total, side="left"))
        bounds.append(max(bounds[-1], min(C, i + 1)))
    bounds.append(C)
    return bounds


def concat_shards(buf: torch.Tensor, pad: int, bounds) -> torch.Tensor:
    """The gathered buffer (world blocks of `pad` entries, rank r's shard at
    the head of block r) as one vector of the C = bounds[-1] results in
    global candidate order."""
    world = len(bounds) - 1
    parts = [buf[r * pad:r * pad + (bounds[r + 1] - bounds[r])] for r in range(world)]
    return torch.cat(parts)


def gather_all(local: torch.Tensor, bounds, pg=None) -> torch.Tensor:
    """All-gather every rank's shard (padded to the largest) and return the
    concatenated int64 vector of length C, identical on every rank."""
    world = len(bounds) - 1
    pad = max(1, max(bounds[r + 1] - bounds[r] for r in range(world)))
    buf = torch.empty(world * pad, dtype=torch.int64, device=local.device)
    dist.all_gather_into_tensor(buf, local[:pad].contiguous(), group=pg)
    return concat_shards(buf, pad, bounds)


def _on(stream):
    """Run torch ops (the collective, buffer writes) on the stream the library
    kernels use, so NCCL reads each shard after its kernel wrote it and the
    next library call sees the gathered vector."""
    if isinstance(stream, torch.cuda.Stream):
        return torch.cuda.stream(stream)
    return contextlib.nullcontext()


def step_bounds(engine, C: int, world: int):
    costs = engine.costs(C) if hasattr(engine, "costs") else np.ones(C, np.int64)
    return shard_bounds(costs, world)


def run_search(engine, pg=None, stream=None, device=None, on_step=None) -> int:
    """Drive the stepwise search to completion.  Returns the number of steps."""
    world = dist.get_world_size(pg) if (pg is not None or dist.is_initialized()) else 1
    rank = dist.get_rank(pg) if world > 1 else 0
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() \
            else torch.device("cpu")
    steps = 0
    local = torch.empty(0, dtype=torch.int64, device=device)
    while True:
        C = engine.prepare()
        if C < 0:
            return steps
        if C == 0:
            engine.apply(None, stream)
            steps += 1
            continue
        bounds = [0, C] if world == 1 else step_bounds(engine, C, world)
        pad = max(1, max(bounds[r + 1] - bounds[r] for r in range(world)))
        if local.numel() < pad:
            with _on(stream):
                local = torch.zeros(max(pad, 2 * local.numel()), dtype=torch.int64, device=device)
        if world == 1:
            engine.evaluate(0, C, local, stream)
            engine.apply(local, stream)
        else:
            engine.evaluate(bounds[rank], bounds[rank + 1], local, stream)
            with _on(stream):
                full = gather_all(local, bounds, pg)
            engine.apply(full, stream)
        steps += 1
        if on_step is not None:
            on_step(steps, C)


def evaluate_sharded(evaluate_fn, argmax_fn, C: int, pg=None, device=None):
    """Evaluate C independent candidates sharded over the ranks (contiguous
    equal-count split; no data-path collective besides the one all-gather of
    the int64 good counts).

    evaluate_fn(begin, end) -> int64 tensor of the good counts of candidates
    [begin, end) on `device`; argmax_fn(good) -> the global argmax (max good,
    ties -> lowest index, -1 when every candidate is infeasible), e.g. the
    library's argmax kernel (Simulator.argmax).  Returns (good[C], argmax),
    identical on every rank."""
    world = dist.get_world_size(pg) if (pg is not None or dist.is_initialized()) else 1
    rank = dist.get_rank(pg) if world > 1 else 0
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() \
            else torch.device("cpu")
    if C == 0:
        return torch.zeros(0, dtype=torch.int64, device=device), -1
    bounds = [shard(C, r, world)[0] for r in range(world)] + [C]
    b, e = bounds[rank], bounds[rank + 1]
    pad = -(-C // world)
    local = torch.full((pad,), -1, dtype=torch.int64, device=device)
    if e > b:
        local[:e - b] = evaluate_fn(b, e).to(device=device, dtype=torch.int64)
    full = local[:C] if world == 1 else gather_all(local, bounds, pg)
    return full, int(argmax_fn(full))


def evaluate_batching_sharded(sim, group_cfg, host_mask, stage_inc_ns, max_batch: int,
                              pg=None):
    """The dynamic batching evaluator (include/asim.h asim_evaluate_batching)
    over 1-8 GPUs: each rank simulates its contiguous shard of the placements
    on its own device; the global argmax is the library's argmax kernel over
    the gathered counts.  Returns (good[C] on the local device, argmax)."""
    cfg = np.ascontiguousarray(group_cfg, dtype=np.int32)
    mask = np.ascontiguousarray(host_mask, dtype=np.uint64)

    def run(b, e):
        out = sim.evaluate_batching(cfg[b:e], mask[b:e], stage_inc_ns, max_batch,
                                    sum_latency=False, argmax=False)
        return torch.from_numpy(out["good"])

    return evaluate_sharded(run, sim.argmax, len(cfg), pg=pg,
                            device=torch.device("cuda", sim.device))
