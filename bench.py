#!/usr/bin/env python
"""Benchmark: the full placement search (Alg. 2 single bucket ⊃ Alg. 1, k=1)
of AlpaServe (arXiv 2302.11665) with every candidate simulated by libasim.so.

One STEP = one complete search over the workload (every lockstep greedy
iteration of every (group partition, parallel config) run: candidate
encoding, batched simulation, per-run argmax, apply), inputs resident in HBM.

    python bench.py [--gpus N --steps K --warmup W] [--config S3 --hours 1]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --impl reference      # the CPU oracle (test infrastructure)

metric: simulated request-placements/s = sum over simulated candidates of
the trace length, divided by the device time of the search (max over ranks).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "simulated request-placements/s (full greedy placement search)"
UNIT = "request-placements/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="asim", choices=["asim", "reference"])
    ap.add_argument("--config", default="S3", choices=["S1", "S2", "S3", "S4", "motivating"])
    ap.add_argument("--hours", type=float, default=24.0,
                    help="trace length (S1-S4); the north-star target is the day-long S3 trace")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--dedup", action="store_true",
                    help="exact de-duplication of identical candidates (fewer simulations)")
    ap.add_argument("--search", default="greedy", choices=["greedy", "fast"],
                    help="Alg. 1 inside Alg. 2 (the headline) or the fast heuristic of P:737")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-prune", action="store_true",
                    help="disable exact run pruning (capacity bound, include/asim.h)")
    ap.add_argument("--bound", action="store_true",
                    help="exact candidate bounding (include/asim.h; off by default: on S3 the "
                         "component bound rarely excludes a candidate the memo would not)")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--e2e-steps", type=int, default=3,
                    help="searches timed end to end (bounded: a day-long search takes seconds)")
    return ap.parse_args()


def workload(args):
    from workloads import configs

    if args.config == "motivating":
        prob = configs.motivating_problem(slo_scale=5.0)
        tr = configs.motivating_trace(seed=args.seed, n_requests=1000)
        name = "motivating: 2 models, 2 GPUs, 1,000 Poisson requests"
    else:
        prob, tr = configs.CONFIGS[args.config](seed=args.seed, duration=args.hours * 3600.0)
        desc = dict(S1="32xBERT-1.3B, 16 devices, Gamma CV 4, 64 req/s",
                    S2="32xBERT-6.7B, 64 devices, MAF1-shaped 80 req/s",
                    S3="60 mixed BERT/MoE, 64 devices, MAF2-shaped 100 req/s",
                    S4="4xBERT-104B, 64 devices, pipeline-only, Gamma 8 req/s CV 4")[args.config]
        name = f"{args.config}: {desc}, {args.hours:g} h trace"
    return prob, tr, name


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                      f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > i + 2 and r[i + 2].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ----------------------------------------------------------------------------- CPU oracle
def step0_batch(prob):
    """The first greedy step of every Alg. 2 run (reading C13): every
    memory-feasible addition (m, g) to the empty placement, m-major, g-minor
     -- exactly the candidates the GPU evaluates at step 0."""
    from oracle import search as osearch

    M = prob.num_models
    cfgs, masks = [], []
    for size, p, cfg in osearch.alg2_runs(prob):
        mb = [int(prob.mem_bytes[m, p]) for m in range(M)]
        for m in range(M):
            if mb[m] < 0 or mb[m] > prob.budget_bytes:
                continue
            for g in range(len(cfg)):
                c = np.full(64, -1, np.int32)
                c[:len(cfg)] = cfg
                mask = np.zeros(M, np.uint64)
                mask[m] = np.uint64(1) << np.uint64(g)
                cfgs.append(c)
                masks.append(mask)
    return np.stack(cfgs), np.stack(masks)


def cpu_sample(prob, tr, seconds: float, seed: int = 0):
    """Time the CPU oracle (as it stands; built -O3 -march=native for this
    host) on a bounded sample of the GPU's own work: a seeded
    subset of the S3 step-0 batch (every run's additions to the empty
    placement) on the trace's 10-min prefix, sized to ~`seconds` of work."""
    import oracle

    oracle.use_timing_build()
    cfg, mask = step0_batch(prob)
    order = np.random.default_rng(seed).permutation(len(cfg))
    cfg, mask = cfg[order], mask[order]
    sub = tr.prefix(int(np.searchsorted(tr.arrival_ns, tr.arrival_ns[0] + 600 * 10**9)))
    threads = oracle.hardware_threads()
    op, ot = oracle.OracleProblem(prob), oracle.OracleTrace(sub)
    n_c = min(len(cfg), 4 * threads)
    while True:  # calibrate the candidate count to ~seconds of work
        t0 = time.perf_counter()
        oracle.evaluate(op, ot, cfg[:n_c], mask[:n_c], threads)
        dt = time.perf_counter() - t0
        if dt >= 0.2 * seconds or n_c >= len(cfg):
            break
        n_c = min(len(cfg), int(n_c * min(8.0, 0.5 * seconds / max(dt, 1e-3))) + 1)
    n_c = min(len(cfg), max(n_c, int(n_c * seconds / max(dt, 1e-3))))
    t0 = time.perf_counter()
    oracle.evaluate(op, ot, cfg[:n_c], mask[:n_c], threads)
    dt = time.perf_counter() - t0
    return dict(value=n_c * len(sub) / dt, unit=UNIT, cores=threads, kind="oracle",
                sample=f"{n_c} of the {len(cfg)} step-0 candidates (every Alg. 2 run's additions "
                       f"to the empty placement) x the {len(sub)}-request 10-min trace prefix, "
                       f"{dt:.1f} s wall on {threads} threads (oracle built -O3 -march=native)",
                seconds=dt)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    prob, tr, name = workload(args)
    per = max(2.0, min(20.0, 120.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        cpu_sample(prob, tr, per / 4, seed=args.seed)
    vals, secs = [], 0.0
    for k in range(args.steps):
        s = cpu_sample(prob, tr, per, seed=args.seed + k)
        vals.append(s["value"])
        secs += s["seconds"]
    v = float(np.mean(vals))
    line = dict(metric=METRIC, value=v, unit=UNIT, n_gpus=args.gpus, steps=args.steps,
                warmup=args.warmup, ms_per_step=secs / args.steps * 1e3,
                higher_is_better=True, scaling="strong", vs_baseline=None, dtype="int64",
                data="synthetic", impl="reference",
                config={"workload": name, "trace_requests": len(tr)},
                cpu_baseline=dict(kind="oracle", cores=s["cores"], sample=s["sample"], value=v,
                                  unit=UNIT),
                e2e=dict(value=v, unit=UNIT, h2d_bytes_per_step=0, d2h_bytes_per_step=0))
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- GPU arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    pg = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist.group.WORLD

    from paper_2302_11665_b200 import Simulator
    from paper_2302_11665_b200 import dist as adist

    prob, tr, name = workload(args)
    N = len(tr)
    stream = torch.cuda.current_stream()
    sim = Simulator(local)
    sim.set_problem(prob)
    sim.set_trace(tr.arrival_ns, tr.model)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    def one_search(s):
        with s.search_handle(dedup=args.dedup, fast=args.search == "fast",
                             prune=not args.no_prune, bounding=args.bound) as sh:
            if args.search == "fast":
                sh.run(stream=stream)  # every rank computes the whole heuristic
            else:
                adist.run_search(sh, pg=pg, stream=stream)
            return sh.result()

    def barrier():
        if pg is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        res = one_search(sim)
    sim.set_profiling(True)
    sim.reset_stats()
    launches0 = sim.launches
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    evals = 0
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.fill_(k & 0xFF)  # L2 flush between timed steps (outside the events)
            barrier()
            ev[k][0].record(stream)
            res = one_search(sim)
            ev[k][1].record(stream)
            barrier()
            evals += res.evaluated * N
    ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = float(sum(ms))
    st = sim.stats()
    launches = sim.launches - launches0
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if pg is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    value = evals / (total_ms / 1e3)

    # ---- end to end through the public API: every step uploads the problem
    # tables and the trace from host memory (numpy arrays, as a caller holds
    # them; asim_set_trace validates them on the host and copies them to the
    # device), runs the search and reads the placement back.  One long-lived
    # context, warmed up once outside the timed region (a serving process keeps
    # its context).
    e2e = None
    if not args.no_e2e:
        h2d = tr.arrival_ns.nbytes + tr.model.astype(np.int32).nbytes + sum(
            np.asarray(x).nbytes for x in (prob.slo_ns, prob.stage_ns, prob.tail_ns,
                                           prob.mem_bytes, prob.cfg_stages, prob.cfg_devices))
        d2h = 8 * (prob.num_models + 64 + 4)
        tot = 0.0
        e_evals = 0
        ke = max(1, min(args.steps, args.e2e_steps))
        s2 = Simulator(local)
        s2.set_problem(prob)
        s2.set_trace(tr.arrival_ns, tr.model)
        one_search(s2)  # warm-up: first-use allocations
        for k in range(ke):
            flush.fill_(k & 0xFF)
            barrier()
            t0 = time.perf_counter()
            s2.set_problem(prob)
            s2.set_trace(tr.arrival_ns, tr.model)
            r2 = one_search(s2)
            barrier()
            tot += time.perf_counter() - t0
            e_evals += r2.evaluated * N
        s2.close()
        tt = torch.tensor([tot], dtype=torch.float64, device="cuda")
        if pg is not None:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = dict(value=e_evals / float(tt.item()), unit=UNIT, h2d_bytes_per_step=int(h2d),
                   d2h_bytes_per_step=int(d2h), ms_per_step=float(tt.item()) / ke * 1e3,
                   steps=ke, host_buffers="pageable numpy (validated and padded on the host)")

    if rank == 0:
        peaks = {}
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
                peaks = json.load(f)
        except OSError:
            pass
        sm_max = float(peaks.get("sm_max_mhz", 1965.0))
        sms = torch.cuda.get_device_properties(local).multi_processor_count
        # ALU roof: one stage update = 1 integer max + 1 add; the integer
        # min/max pipe issues 16 lanes/clk per SMSP -> 64 updates/clk/SM.
        peak = sms * 64 * sm_max * 1e6 / 1e9  # G stage-updates/s
        # dominant kernel: the chunked path's pass 1 (chunk_kernel SPEC), timed
        # by its own CUDA events on the stream it is launched on; split steps
        # run two chunked runs concurrently, so its time is the union of its
        # launches' [start, end] intervals (busy time), not their sum
        spec = st["spec_ms"] > 0
        k_ms = st["spec_busy_ms"] if spec else st["sim_ms"]
        k_upd = st["spec_stage_updates"] if spec else st["stage_updates"]
        achieved = k_upd / max(k_ms, 1e-9) / 1e6  # G stage-updates/s
        traffic = None
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            try:
                traffic = json.load(open(tp)).get(args.config)
                traffic = float(traffic) / 1e9 if traffic is not None else None  # GB per launch
            except Exception:
                traffic = None
        line = dict(
            metric=METRIC, value=value, unit=UNIT, n_gpus=world, steps=args.steps,
            warmup=args.warmup, ms_per_step=total_ms / args.steps, higher_is_better=True,
            scaling="strong", vs_baseline=None, dtype="int64", data="synthetic",
            config=dict(workload=name, trace_requests=N, models=prob.num_models,
                        devices=prob.num_devices, runs=len(res.runs), search_steps=res.steps,
                        candidates_per_search=res.candidates,
                        simulated_per_search=res.evaluated, memo_hits=res.memo_hits,
                        dedup=bool(args.dedup), search=args.search,
                        best_run=res.best_run, best_attainment=res.best_good / max(N, 1),
                        prune=not args.no_prune,
                        pruned_runs=sum(1 for r in res.runs if r["pruned_at"] >= 0),
                        bounding=bool(args.bound), bounded_candidates=res.bounded,
                        l2="flushed between timed steps (256 MB write)",
                        performed_value=st["spec_live_lanes"] / max(args.steps, 1)
                        / (total_ms / args.steps / 1e3),
                        performed_unit="(request, candidate) pairs replayed per s: each "
                                       "simulated candidate replays only the requests of its "
                                       "own hosting-graph component (component restriction); "
                                       "`value` counts the whole trace per simulated candidate",
                        parallelism=f"candidate-sharded x{world}"),
            gpu_launches=int(launches),
            roofline=dict(bound="alu", achieved=achieved, peak=peak,
                          unit="G stage-updates/s", frac=achieved / peak, traffic=traffic,
                          traffic_unit="GB DRAM per launch of chunk_kernel pass 1, heaviest "
                                       "launch (ncu --set full, profiles/traffic.json)",
                          kernel=("chunk_kernel pass 1 (SPEC: every candidate x time chunk from "
                                  "its speculative start)") if spec else "simulation kernels",
                          kernel_ms_share=k_ms / max(total_ms, 1e-9),
                          kernel_ms=k_ms, kernel_stage_updates=k_upd,
                          all_sim_ms_share=st["sim_ms"] / max(total_ms, 1e-9),
                          kernel_ms_summed=st["spec_ms"],
                          pass2_ms=st["pass2_busy_ms"], walk_ms=st["walk_busy_ms"],
                          pass1_class_share={c: round(x / max(1, sum(st["spec_class_cycles"])), 4)
                                             for c, x in zip(("mixed", "S1", "S2", "S4", "S8",
                                                              "S16"), st["spec_class_cycles"])},
                          walk_critical_chunks=st["walk_critical_chunks"],
                          walk_candidates=st["walk_candidates"],
                          walked_chunks=st["chunk_reruns"],
                          lane_utilization=st["spec_live_lanes"] / max(1, st["spec_lane_slots"]),
                          stage_updates=st["stage_updates"], sim_launches=st["sim_launches"],
                          peak_basis=f"{sms} SMs x 64 int max/clk x {sm_max:.0f} MHz "
                                     "(MEASURED_PEAKS sm_max_mhz)"),
            clocks=clk.summary(),
        )
        if e2e is not None:
            line["e2e"] = e2e
        if world == 1 and not args.no_cpu_baseline:
            cb = cpu_sample(prob, tr, args.cpu_seconds, seed=args.seed)
            cb.pop("seconds", None)
            line["cpu_baseline"] = cb
        print(json.dumps(line), flush=True)
    if pg is not None:
        dist.barrier()
        dist.destroy_process_group()
    sim.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
