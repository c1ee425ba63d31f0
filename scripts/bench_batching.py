#!/usr/bin/env python
"""Benchmark of the dynamic batching variant.

Workload: the paper's batching experiment setup (§5.4): model set
S1 (32 x BERT-1.3B, 16 devices), Gamma arrivals of 4 req/s per model with
CV 4, here over `--hours` (default 1 h, ~460k requests), batch slope delta
(reading C35, default 0.9), max batch `--max-batch` (default 4).  One STEP =
one asim_evaluate_batching call over C seeded random feasible placements of
every S1 parallel config (inputs resident in HBM), including the argmax.

Prints one JSON line like bench.py: value = C x N / device time, roofline of
the batching kernel against warp-instruction ISSUE (4 per SM per clock: with
one candidate per warp a request step is a sequence of warp-wide
instructions, so issue is the binding roof), with the measured
warp instructions per (request, candidate) evaluation I_eval from ncu
(`--ieval`, or the JSON file written by the ncu launch-list pass:
smsp__inst_executed.sum / (C x N)); e2e through the public API from host
buffers; and the CPU oracle (oracle.evaluate_batching, as it stands) on a
bounded sample.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

METRIC = "simulated request-placements/s (dynamic batching variant, candidate batch)"
UNIT = "request-placements/s"


def placements(prob, C, seed):
    """C seeded random placements: parallel configs round robin over all S1
    configs (equal groups on all devices), each group filled with random
    models up to the memory budget (reading C11)."""
    rng = np.random.default_rng(seed)
    M = prob.num_models
    cfgs = [(p, s * n) for p, (s, n) in enumerate(prob.configs)]
    cfg = np.full((C, 16), -1, np.int32)
    mask = np.zeros((C, M), np.uint64)
    for c in range(C):
        p, size = cfgs[c % len(cfgs)]
        G = prob.num_devices // size
        cfg[c, :G] = p
        for g in range(G):
            used = 0
            for m in rng.permutation(M)[: int(rng.integers(1, M + 1))]:
                mb = int(prob.mem_bytes[m, p])
                if mb >= 0 and used + mb <= prob.budget_bytes:
                    mask[c, m] |= np.uint64(1) << np.uint64(g)
                    used += mb
    return cfg, mask


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--hours", type=float, default=1.0)
    ap.add_argument("--candidates", type=int, default=148 * 32)
    ap.add_argument("--max-batch", type=int, default=4)
    ap.add_argument("--delta", type=float, default=0.9)
    ap.add_argument("--slo-scale", type=float, default=5.0)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ieval", default=os.path.join(ROOT, "profiles", "r2d", "batching_ieval.json"),
                    help="JSON with the ncu-measured warp instructions per evaluation")
    args = ap.parse_args()

    import torch

    from bench import ClockSampler
    from paper_2302_11665_b200 import Simulator
    from workloads import configs

    prob, tr, inc = configs.s1_batching(seed=0, duration=args.hours * 3600.0,
                                        slo_scale=args.slo_scale, delta=args.delta)
    N = len(tr)
    cfg, mask = placements(prob, args.candidates, seed=1)
    C = len(cfg)
    stream = torch.cuda.current_stream()
    sim = Simulator(0)
    sim.set_problem(prob)
    sim.set_trace(tr.arrival_ns, tr.model)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    # inputs resident in HBM: candidates as device tensors
    from paper_2302_11665_b200 import _abi as A
    import ctypes

    d_cfg = torch.from_numpy(cfg).cuda()
    d_mask = torch.from_numpy(mask.view(np.int64)).cuda()
    d_good = torch.empty(C, dtype=torch.int64, device="cuda")
    d_arg = torch.empty(1, dtype=torch.int64, device="cuda")
    inc_h = np.ascontiguousarray(inc, dtype=np.int64)
    cands = A.asim_candidates(C, cfg.shape[1], ctypes.c_void_p(d_cfg.data_ptr()),
                              ctypes.c_void_p(d_mask.data_ptr()), A.ASIM_DEVICE)
    opt = A.asim_batching(args.max_batch, inc_h.ctypes.data)
    res = A.asim_results(ctypes.c_void_p(d_good.data_ptr()), None, None,
                         ctypes.c_void_p(d_arg.data_ptr()), A.ASIM_DEVICE, None)

    def step():
        sim._check(A.asim_evaluate_batching(sim.h, ctypes.byref(cands), ctypes.byref(opt),
                                            ctypes.byref(res),
                                            ctypes.c_void_p(stream.cuda_stream)))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    sim.set_profiling(True)
    sim.reset_stats()
    launches0 = sim.launches
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    with ClockSampler(0) as clk:
        for k in range(args.steps):
            flush.fill_(k & 0xFF)
            torch.cuda.synchronize()
            ev[k][0].record(stream)
            step()
            ev[k][1].record(stream)
            torch.cuda.synchronize()
    total_ms = float(sum(a.elapsed_time(b) for a, b in ev))
    st = sim.stats()
    launches = sim.launches - launches0
    good = d_good.cpu().numpy()
    feasible = int((good >= 0).sum())
    value = feasible * N * args.steps / (total_ms / 1e3)

    # e2e: the public call with host buffers, copies inside the timed region
    cfg_pin = torch.from_numpy(cfg).pin_memory()
    mask_pin = torch.from_numpy(mask.view(np.int64)).pin_memory()
    tot = 0.0
    for k in range(args.steps):
        flush.fill_(k & 0xFF)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = sim.evaluate_batching(cfg_pin.numpy(), mask_pin.numpy().view(np.uint64), inc_h,
                                    args.max_batch, sum_latency=False)
        tot += time.perf_counter() - t0
    assert np.array_equal(out["good"], good)
    e2e = dict(value=feasible * N * args.steps / tot, unit=UNIT,
               h2d_bytes_per_step=int(cfg.nbytes + mask.nbytes + inc_h.nbytes),
               d2h_bytes_per_step=int(C * 8 + 8), ms_per_step=tot / args.steps * 1e3)

    cpu = None
    if not args.no_cpu_baseline:
        import oracle

        threads = oracle.hardware_threads()
        n_c, n_req = min(C, 4 * threads), min(N, 20000)
        while True:
            t0 = time.perf_counter()
            oracle.evaluate_batching(prob, tr.prefix(n_req), cfg[:n_c], mask[:n_c], inc_h,
                                     args.max_batch, threads)
            dt = time.perf_counter() - t0
            if dt >= 0.5 * args.cpu_seconds or n_c >= C:
                break
            n_c = min(C, int(n_c * min(4.0, args.cpu_seconds / max(dt, 1e-3))) + 1)
        cpu = dict(value=n_c * n_req / dt, unit=UNIT, cores=threads, kind="oracle",
                   sample=f"{n_c} of the {C} placements x {n_req}-request trace prefix, "
                          f"{dt:.1f} s wall on {threads} threads")

    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        pass
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    # issue roof: 4 warp instructions per SM per clock
    peak = 4 * sms * sm_max * 1e6 / 1e9  # G warp-instructions/s
    ieval = None
    try:
        ieval = float(json.load(open(args.ieval))["inst_per_eval"])
    except (OSError, KeyError, ValueError):
        pass
    k_evals = feasible * N * args.steps  # (request, candidate) evaluations by the kernel
    achieved = (k_evals * ieval / (st["sim_ms"] / 1e3) / 1e9) if ieval else None
    traffic = None
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))["S1-batching"] / 1e9
    except (OSError, KeyError, ValueError):
        pass
    line = dict(
        metric=METRIC, value=value, unit=UNIT, n_gpus=1, steps=args.steps, warmup=args.warmup,
        ms_per_step=total_ms / args.steps, higher_is_better=True, scaling="weak",
        vs_baseline=None, dtype="int64", data="synthetic",
        config=dict(workload=f"S1 batching (§5.4): 32xBERT-1.3B, 16 devices, Gamma 4 req/s "
                             f"per model CV 4, {args.hours:g} h trace",
                    trace_requests=N, candidates=C, feasible=feasible,
                    max_batch=args.max_batch, delta=args.delta, slo_scale=args.slo_scale,
                    best_attainment=float(good.max()) / max(N, 1),
                    l2="flushed between timed steps (256 MB write)"),
        gpu_launches=int(launches),
        roofline=dict(bound="issue", achieved=achieved, peak=peak, unit="G warp-instructions/s",
                      frac=(achieved / peak) if achieved else None, traffic=traffic,
                      inst_per_eval=ieval, ieval_source=os.path.relpath(args.ieval, ROOT),
                      traffic_unit="GB DRAM per launch (ncu --set full, profiles/traffic.json)",
                      kernel="batching_kernel",
                      kernel_ms=st["sim_ms"], stage_updates=st["stage_updates"],
                      kernel_ms_share=st["sim_ms"] / max(total_ms, 1e-9),
                      stage_updates_per_s=st["stage_updates"] / max(st["sim_ms"], 1e-9) * 1e3,
                      peak_basis=f"{sms} SMs x 4 warp-instructions/clk x {sm_max:.0f} MHz "
                                 "(MEASURED_PEAKS sm_max_mhz)"),
        clocks=clk.summary(), e2e=e2e, cpu_baseline=cpu)
    print(json.dumps(line), flush=True)
    sim.close()


if __name__ == "__main__":
    main()
