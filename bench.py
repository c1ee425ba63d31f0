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
    ap.add_argument("--hours", type=float, default=1.0, help="trace length (S1-S4)")
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
def cpu_sample(prob, tr, seconds: float, seed: int = 0):
    """Time the CPU oracle (as it stands) on a bounded sample of the same
    workload: mid-search placements of every Alg. 2 run (each group filled
    to ~half its memory with seeded random models) plus all their feasible
    additions, on a prefix of the trace sized to ~`seconds` of work."""
    import oracle
    from oracle import search as osearch
    from workloads import Placement

    rng = np.random.default_rng(seed)
    M = prob.num_models
    cands_cfg, cands_mask = [], []
    for size, p, cfg in osearch.alg2_runs(prob):
        G = len(cfg)
        used = np.zeros(G, np.int64)
        mask = np.zeros(M, np.uint64)
        for g in range(G):
            for m in rng.permutation(M):
                mb = int(prob.mem_bytes[m, p])
                if mb >= 0 and used[g] + mb <= prob.budget_bytes // 2:
                    mask[m] |= np.uint64(1) << np.uint64(g)
                    used[g] += mb
        for m in range(M):
            for g in range(G):
                mb = int(prob.mem_bytes[m, p])
                if (int(mask[m]) >> g) & 1 or mb < 0 or used[g] + mb > prob.budget_bytes:
                    continue
                mm = mask.copy()
                mm[m] |= np.uint64(1) << np.uint64(g)
                c = np.full(64, -1, np.int32)
                c[:G] = cfg
                cands_cfg.append(c)
                cands_mask.append(mm)
    order = rng.permutation(len(cands_cfg))
    cfg = np.stack(cands_cfg)[order]
    mask = np.stack(cands_mask)[order]
    threads = oracle.hardware_threads()
    # calibrate: grow (candidates, requests) until ~seconds of CPU work
    n_req, n_c = min(len(tr), 20000), min(len(cfg), 4 * threads)
    op, _ = oracle.OracleProblem(prob), None
    while True:
        sub = tr.prefix(n_req)
        t0 = time.perf_counter()
        oracle.evaluate(op, sub, cfg[:n_c], mask[:n_c], threads)
        dt = time.perf_counter() - t0
        if dt >= 0.25 * seconds or (n_c >= len(cfg) and n_req >= len(tr)):
            break
        grow = min(4.0, 0.5 * seconds / max(dt, 1e-3))
        if n_c < len(cfg):
            n_c = min(len(cfg), int(n_c * grow) + 1)
        else:
            n_req = min(len(tr), int(n_req * grow) + 1)
    scale = max(1.0, seconds / max(dt, 1e-3))
    n_c = min(len(cfg), int(n_c * scale))
    sub = tr.prefix(n_req)
    t0 = time.perf_counter()
    oracle.evaluate(op, sub, cfg[:n_c], mask[:n_c], threads)
    dt = time.perf_counter() - t0
    return dict(value=n_c * n_req / dt, unit=UNIT, cores=threads, kind="oracle",
                sample=f"{n_c} mid-search candidates (of {len(cfg)}, all Alg. 2 runs) x "
                       f"{n_req}-request trace prefix, {dt:.1f} s wall on {threads} threads",
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

    # ---- end to end through the public API from pinned host buffers
    e2e = None
    if not args.no_e2e:
        a_pin = torch.from_numpy(tr.arrival_ns).pin_memory()
        m_pin = torch.from_numpy(tr.model).pin_memory()
        h2d = a_pin.numel() * 8 + m_pin.numel() * 4 + sum(
            np.asarray(x).nbytes for x in (prob.slo_ns, prob.stage_ns, prob.tail_ns,
                                           prob.mem_bytes, prob.cfg_stages, prob.cfg_devices))
        d2h = 0
        tot = 0.0
        e_evals = 0
        # one context per process (created outside the timed region, as a
        # serving process keeps it); every step uploads the problem and the
        # trace from pinned host memory, searches, and reads the result back
        s2 = Simulator(local)
        for k in range(args.steps):
            flush.fill_(k & 0xFF)
            barrier()
            t0 = time.perf_counter()
            s2.set_problem(prob)
            s2.set_trace(a_pin.numpy(), m_pin.numpy())
            r2 = one_search(s2)
            barrier()
            tot += time.perf_counter() - t0
            e_evals += r2.evaluated * N
            d2h = 8 * (prob.num_models + 64 + 4)
        s2.close()
        tt = torch.tensor([tot], dtype=torch.float64, device="cuda")
        if pg is not None:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = dict(value=e_evals / float(tt.item()), unit=UNIT, h2d_bytes_per_step=int(h2d),
                   d2h_bytes_per_step=int(d2h), ms_per_step=float(tt.item()) / args.steps * 1e3)

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
        # by its own CUDA events on the search stream, its own work counter
        spec = st["spec_ms"] > 0
        k_ms = st["spec_ms"] if spec else st["sim_ms"]
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
