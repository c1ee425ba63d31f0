"""Multi-GPU candidate sharding for the placement search.

Candidate evaluations inside one greedy iteration are independent -- the
paper simulates "all valid selections" of an iteration before taking the top
k (Alg. 1) -- so each lockstep step's global candidate list is
split into contiguous shards, one per rank.  The only exchange per step is an
all-gather of the int64 good counts (NCCL over NVLink on B200s); every rank
then applies the same per-run argmax (lowest global index on ties), so the
search state stays identical on all ranks without any further broadcast.

`engine` is anything with prepare() -> C (-1 = finished; 0 = nothing to
simulate this step), evaluate(begin, end, out, stream) and apply(good_all,
stream): api.SearchHandle on the GPU; tests inject a CPU engine to exercise
this logic under gloo.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard(C: int, rank: int, world: int):
    """Contiguous shard [begin, end) of C candidates for `rank`."""
    return C * rank // world, C * (rank + 1) // world


def gather_all(local: torch.Tensor, C: int, world: int, pg=None) -> torch.Tensor:
    """All-gather every rank's shard (padded to ceil(C/world)) and return the
    concatenated int64 vector of length C, identical on every rank."""
    pad = -(-C // world)
    buf = torch.empty(world * pad, dtype=torch.int64, device=local.device)
    dist.all_gather_into_tensor(buf, local[:pad].contiguous(), group=pg)
    parts = []
    for r in range(world):
        b, e = shard(C, r, world)
        parts.append(buf[r * pad:r * pad + (e - b)])
    return torch.cat(parts)


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
        pad = -(-C // world)
        if local.numel() < pad:
            local = torch.zeros(max(pad, 2 * local.numel()), dtype=torch.int64, device=device)
        if world == 1:
            engine.evaluate(0, C, local, stream)
            engine.apply(local, stream)
        else:
            b, e = shard(C, rank, world)
            engine.evaluate(b, e, local, stream)
            full = gather_all(local, C, world, pg)
            engine.apply(full, stream)
        steps += 1
        if on_step is not None:
            on_step(steps, C)


def evaluate_sharded(evaluate_fn, C: int, pg=None, device=None):
    """Evaluate C independent candidates sharded over the ranks (the same
    contiguous split as the search; no data-path collective besides the one
    all-gather of the int64 good counts).

    evaluate_fn(begin, end) -> int64 tensor of the good counts of candidates
    [begin, end) on `device` (e.g. a Simulator.evaluate_batching call on that
    slice).  Returns (good[C], argmax) identical on every rank; argmax = max
    good, ties -> lowest global index, -1 when every candidate is infeasible
    (good < 0)."""
    world = dist.get_world_size(pg) if (pg is not None or dist.is_initialized()) else 1
    rank = dist.get_rank(pg) if world > 1 else 0
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() \
            else torch.device("cpu")
    if C == 0:
        return torch.zeros(0, dtype=torch.int64, device=device), -1
    b, e = shard(C, rank, world)
    pad = -(-C // world)
    local = torch.full((pad,), -1, dtype=torch.int64, device=device)
    if e > b:
        local[:e - b] = evaluate_fn(b, e).to(device=device, dtype=torch.int64)
    full = local[:C] if world == 1 else gather_all(local, C, world, pg)
    best = int(full.max().item())
    arg = int(torch.nonzero(full == best)[0].item()) if best >= 0 else -1
    return full, arg


def evaluate_batching_sharded(sim, group_cfg, host_mask, stage_inc_ns, max_batch: int,
                              pg=None):
    """The dynamic batching evaluator (include/asim.h asim_evaluate_batching)
    over 1-8 GPUs: each rank simulates its contiguous shard of the placements
    on its own device; returns (good[C] on the local device, global argmax)."""
    import numpy as np

    cfg = np.ascontiguousarray(group_cfg, dtype=np.int32)
    mask = np.ascontiguousarray(host_mask, dtype=np.uint64)

    def run(b, e):
        out = sim.evaluate_batching(cfg[b:e], mask[b:e], stage_inc_ns, max_batch,
                                    sum_latency=False, argmax=False)
        return torch.from_numpy(out["good"])

    return evaluate_sharded(run, len(cfg), pg=pg)
