"""Python front end of libasim.so: marshals numpy (host) or torch CUDA
(device) arrays into the C ABI of include/asim.h.  No simulation, search or
encoding arithmetic lives here -- every step of the hot path runs in the
library (host runtime in csrc/*.cpp, kernels in csrc/sim.cu).

Problems are duck-typed: any object with num_models, num_configs,
max_stages, slo_ns, cfg_stages, cfg_devices, stage_ns, tail_ns, mem_bytes,
num_devices and budget_bytes (workloads.Problem has them).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _abi as A


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _stream_ptr(stream):
    if stream is None:
        try:
            import torch

            if torch.cuda.is_available():
                return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        except Exception:  # pragma: no cover - torch without CUDA
            pass
        return ctypes.c_void_p(0)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _host(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _ptr(a):
    if a is None:
        return None
    if _is_torch(a):
        return ctypes.c_void_p(a.data_ptr())
    return ctypes.c_void_p(a.ctypes.data)


@dataclass
class SearchResult:
    best_run: int
    best_good: int
    num_groups: int
    group_cfg: np.ndarray
    host_mask: np.ndarray
    steps: int
    candidates: int
    evaluated: int
    request_evals: int
    memo_hits: int
    runs: list
    bounded: int = 0


@dataclass
class BucketResult:
    """Alg. 2 with model / device buckets: the best partition (sorted model ids
    per bucket), its device counts, the run solving each bucket (-1: empty),
    and the concatenated placement (groups of bucket 1 first)."""
    best_good: int
    partition: list
    devices: list
    bucket_runs: list
    group_cfg: np.ndarray
    host_mask: np.ndarray
    partitions: int
    considered: int
    search: SearchResult

    @property
    def placement(self):
        from types import SimpleNamespace
        return SimpleNamespace(group_cfg=self.group_cfg, host_mask=self.host_mask)


class Simulator:
    """One asim context on one CUDA device (one per process and GPU)."""

    def __init__(self, device: int = 0):
        h = ctypes.c_void_p()
        st = A.asim_create(int(device), ctypes.byref(h))
        if st != A.ASIM_OK:
            raise A.AsimError(st, A.asim_last_error(None).decode())
        self.h = h
        self.device = int(device)
        self.M = None
        self.n = 0
        self._keep = []

    # ------------------------------------------------------------- lifetime
    def close(self):
        if getattr(self, "h", None) and A.asim_destroy is not None:  # None at interpreter exit
            A.asim_destroy(self.h)
        self.h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _check(self, st):
        A.check(st, self.h)

    @property
    def launches(self) -> int:
        return int(A.asim_launch_count(self.h))

    def set_profiling(self, on: bool) -> None:
        self._check(A.asim_set_profiling(self.h, int(bool(on))))

    def reset_stats(self) -> None:
        self._check(A.asim_reset_stats(self.h))

    def stats(self) -> dict:
        s = A.asim_stats()
        self._check(A.asim_get_stats(self.h, ctypes.byref(s)))
        return dict(launches=s.launches, sim_launches=s.sim_launches, sim_ms=s.sim_ms,
                    stage_updates=s.stage_updates, request_evals=s.request_evals,
                    chunk_reruns=s.chunk_reruns, walk_candidates=s.walk_candidates,
                    walk_critical_chunks=s.walk_critical_chunks, spec_ms=s.spec_ms,
                    spec_stage_updates=s.spec_stage_updates, pass2_ms=s.pass2_ms,
                    walk_ms=s.walk_ms, spec_lane_slots=s.spec_lane_slots,
                    spec_live_lanes=s.spec_live_lanes, walk_predicted=s.walk_predicted,
                    walk_unpredicted=s.walk_unpredicted, walk_mispredicted=s.walk_mispredicted,
                    spec_class_cycles=list(s.spec_class_cycles),
                    spec_class_updates=list(s.spec_class_updates),
                    spec_class_slots=list(s.spec_class_slots), spec_busy_ms=s.spec_busy_ms,
                    pass2_busy_ms=s.pass2_busy_ms, walk_busy_ms=s.walk_busy_ms)

    def set_chunk_size(self, min_requests: int) -> None:
        self._check(A.asim_set_chunk_size(self.h, int(min_requests)))

    def set_path(self, path: int) -> None:
        """0 auto, 1 general kernel, 2 chunked kernel (identical results)."""
        self._check(A.asim_set_path(self.h, int(path)))

    # ------------------------------------------------------------- inputs
    def set_problem(self, prob) -> None:
        arrs = dict(slo=_host(prob.slo_ns, np.int64), stages=_host(prob.cfg_stages, np.int32),
                    devs=_host(prob.cfg_devices, np.int32), stage=_host(prob.stage_ns, np.int64),
                    tail=_host(prob.tail_ns, np.int64), mem=_host(prob.mem_bytes, np.int64))
        c = A.asim_problem(int(prob.num_models), int(prob.num_configs), int(prob.max_stages),
                           _ptr(arrs["slo"]), _ptr(arrs["stages"]), _ptr(arrs["devs"]),
                           _ptr(arrs["stage"]), _ptr(arrs["tail"]), _ptr(arrs["mem"]),
                           int(prob.num_devices), int(prob.budget_bytes))
        self._check(A.asim_set_problem(self.h, ctypes.byref(c)))
        self.M = int(prob.num_models)

    def set_trace(self, arrival_ns, model, stream=None) -> None:
        """Host numpy arrays or device torch tensors (int64 / int32)."""
        if _is_torch(arrival_ns):
            kind = A.ASIM_DEVICE if arrival_ns.is_cuda else A.ASIM_HOST
            a, m = arrival_ns.contiguous(), model.contiguous()
        else:
            kind = A.ASIM_HOST
            a, m = _host(arrival_ns, np.int64), _host(model, np.int32)
        n = int(a.shape[0])
        self._check(A.asim_set_trace(self.h, n, _ptr(a), _ptr(m), kind, _stream_ptr(stream)))
        self.n = n

    # ------------------------------------------------------------- evaluate
    def evaluate(self, group_cfg, host_mask, per_model=False, sum_latency=True, argmax=True,
                 busy=False, stream=None) -> dict:
        """Full candidates: group_cfg [C, G] int32, host_mask [C, M] uint64 (host)."""
        cfg = _host(group_cfg, np.int32)
        mask = _host(host_mask, np.uint64)
        C, G = cfg.shape
        cands = A.asim_candidates(C, G, _ptr(cfg), _ptr(mask), A.ASIM_HOST)
        return self._run(A.asim_evaluate, cands, C, G, per_model, sum_latency, argmax, busy,
                         stream)

    def evaluate_batching(self, group_cfg, host_mask, stage_inc_ns, max_batch: int,
                          per_model=False, sum_latency=True, argmax=True, stream=None) -> dict:
        """Dynamic batching variant (§5.4, include/asim.h): full
        candidates as in evaluate(); stage_inc_ns [M, P, S] int64 -- a batch of
        k occupies stage j for stage_ns + (k - 1) * stage_inc_ns."""
        cfg = _host(group_cfg, np.int32)
        mask = _host(host_mask, np.uint64)
        inc = _host(stage_inc_ns, np.int64)
        C, G = cfg.shape
        cands = A.asim_candidates(C, G, _ptr(cfg), _ptr(mask), A.ASIM_HOST)
        opt = A.asim_batching(int(max_batch), _ptr(inc))
        good = np.zeros(C, np.int64)
        sl = np.zeros(C, np.int64) if sum_latency else None
        pm = np.zeros((C, self.M), np.int64) if per_model else None
        am = np.zeros(1, np.int64) if argmax else None
        res = A.asim_results(_ptr(good), _ptr(sl), _ptr(pm), _ptr(am), A.ASIM_HOST, None)
        self._check(A.asim_evaluate_batching(self.h, ctypes.byref(cands), ctypes.byref(opt),
                                             ctypes.byref(res), _stream_ptr(stream)))
        return dict(good=good, sum_latency_ns=sl, good_per_model=pm,
                    argmax=int(am[0]) if argmax else None)

    def evaluate_deltas(self, base_cfg, base_mask, cand_base, cand_model, cand_group,
                        per_model=False, sum_latency=True, argmax=True, busy=False,
                        stream=None) -> dict:
        bc = _host(base_cfg, np.int32)
        bm = _host(base_mask, np.uint64)
        cb, cm, cg = (_host(x, np.int32) for x in (cand_base, cand_model, cand_group))
        B, G = bc.shape
        C = int(cb.shape[0])
        d = A.asim_deltas(B, G, _ptr(bc), _ptr(bm), C, _ptr(cb), _ptr(cm), _ptr(cg), A.ASIM_HOST)
        return self._run(A.asim_evaluate_deltas, d, C, G, per_model, sum_latency, argmax, busy,
                         stream)

    def _run(self, fn, cands, C, G, per_model, sum_latency, argmax, busy, stream):
        good = np.zeros(C, np.int64)
        sl = np.zeros(C, np.int64) if sum_latency else None
        pm = np.zeros((C, self.M), np.int64) if per_model else None
        am = np.zeros(1, np.int64) if argmax else None
        bz = np.zeros((C, G), np.int64) if busy else None
        res = A.asim_results(_ptr(good), _ptr(sl), _ptr(pm), _ptr(am), A.ASIM_HOST, _ptr(bz))
        self._check(fn(self.h, ctypes.byref(cands), ctypes.byref(res), _stream_ptr(stream)))
        return dict(good=good, sum_latency_ns=sl, good_per_model=pm,
                    argmax=int(am[0]) if argmax else None, busy_ns=bz)

    def argmax(self, good, stream=None) -> int:
        """Library argmax kernel (max good, lowest index on ties, -1 if none
        is feasible) over a host numpy array or a CUDA torch tensor."""
        if _is_torch(good):
            g = good.contiguous()
            kind = A.ASIM_DEVICE if g.is_cuda else A.ASIM_HOST
        else:
            g, kind = _host(good, np.int64), A.ASIM_HOST
        out = ctypes.c_int64()
        self._check(A.asim_argmax(self.h, _ptr(g), int(g.shape[0]), kind, ctypes.byref(out),
                                  _stream_ptr(stream)))
        return int(out.value)

    # ------------------------------------------------------------- search
    def search_handle(self, runs=None, dedup=True, fast=False, buckets=None,
                      beam=1, prune=True, bounding=False) -> "SearchHandle":
        return SearchHandle(self, runs, dedup, fast, buckets, beam, prune, bounding)

    def search_buckets(self, latency, ratio=4, bound=3, max_buckets=0, fast=False, dedup=True,
                       pg=None, stream=None, beam=1, prune=True,
                       bounding=False) -> BucketResult:
        """Alg. 2 with model and device buckets (include/asim.h).
        latency[m]: single-device latency in ns; ratio / bound: ints or
        fractions.Fraction (threshold 4x and discrepancy bound 3x by default)."""
        from fractions import Fraction

        from . import dist

        b = dict(latency=_host(latency, np.int64), ratio=Fraction(ratio), bound=Fraction(bound),
                 max_buckets=int(max_buckets))
        with self.search_handle(None, dedup, fast, b, beam, prune, bounding) as sh:
            if fast:
                sh.run(stream=stream)
            else:
                dist.run_search(sh, pg=pg, stream=stream)
            res = sh.result()
            M = self.M
            of = np.full(M, -1, np.int32)
            dv = np.zeros(M, np.int32)
            br = np.full(M, -1, np.int32)
            r = A.asim_bucket_result(0, 0, 0, 0, _ptr(of), _ptr(dv), _ptr(br))
            self._check(A.asim_search_buckets_get(sh.h, ctypes.byref(r)))
            k = r.num_buckets
            part = [sorted(int(m) for m in np.nonzero(of == i)[0]) for i in range(k)]
            return BucketResult(r.best_good, part, [int(x) for x in dv[:k]],
                                [int(x) for x in br[:k]], res.group_cfg, res.host_mask,
                                r.partitions, r.considered, res)

    def search(self, runs=None, dedup=True, pg=None, stream=None, fast=False,
               beam=1, prune=True, bounding=False) -> SearchResult:
        """Full Alg. 2 (single bucket) / Alg. 1 search.  With a
        torch.distributed process group the step candidates shard across its
        ranks (dist.run_search).  fast=True runs the fast heuristic of P:737
        instead of Alg. 1 (one simulation per run and step; every rank
        computes it whole -- there is nothing to shard)."""
        from . import dist

        with self.search_handle(runs, dedup, fast, None, beam, prune, bounding) as sh:
            if fast:
                sh.run(stream=stream)
            else:
                dist.run_search(sh, pg=pg, stream=stream)
            return sh.result()


class SearchHandle:
    """Stepwise search protocol of include/asim.h (prepare / evaluate / apply)."""

    def __init__(self, sim: Simulator, runs=None, dedup=True, fast=False, buckets=None,
                 beam=1, prune=True, bounding=False):
        self.sim = sim
        spec = A.asim_search_spec()
        spec.dedup = int(bool(dedup))
        spec.fast = int(bool(fast))
        spec.beam = int(beam)
        spec.prune = int(bool(prune))
        spec.cand_bound = int(bool(bounding))
        self._keep = ()
        if buckets is not None:
            lat = buckets["latency"]
            spec.buckets = 1
            spec.max_buckets = buckets["max_buckets"]
            spec.ratio_num, spec.ratio_den = buckets["ratio"].numerator, buckets["ratio"].denominator
            spec.bound_num, spec.bound_den = buckets["bound"].numerator, buckets["bound"].denominator
            spec.model_latency_ns = _ptr(lat)
            self._keep = (lat,)
        elif runs is not None:
            ng = np.array([len(r) for r in runs], np.int32)
            cfg = np.concatenate([np.asarray(r, np.int32) for r in runs]).astype(np.int32)
            spec.num_runs = len(runs)
            spec.run_num_groups = _ptr(ng)
            spec.run_group_cfg = _ptr(cfg)
            self._keep = (ng, cfg)
        h = ctypes.c_void_p()
        sim._check(A.asim_search_create(sim.h, ctypes.byref(spec), ctypes.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None) and A.asim_search_destroy is not None:
            A.asim_search_destroy(self.h)
        self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        self.close()

    def prepare(self) -> int:
        """Candidates of this step needing simulation (>= 0), or -1 when finished."""
        c = ctypes.c_int64()
        self.sim._check(A.asim_search_prepare(self.h, ctypes.byref(c)))
        return int(c.value)

    def evaluate(self, begin: int, end: int, good_dev, stream=None) -> None:
        """good_dev: torch int64 CUDA tensor with >= end - begin elements."""
        self.sim._check(A.asim_search_evaluate(self.h, int(begin), int(end), _ptr(good_dev),
                                               _stream_ptr(stream)))

    def costs(self, C: int) -> np.ndarray:
        """Per-candidate work estimate of the prepared step (C entries)."""
        out = np.zeros(max(int(C), 0), np.int64)
        self.sim._check(A.asim_search_costs(self.h, out.size, _ptr(out) if out.size else None))
        return out

    def apply(self, good_all_dev, stream=None) -> None:
        self.sim._check(A.asim_search_apply(self.h, _ptr(good_all_dev) if good_all_dev is not None
                                            else None, _stream_ptr(stream)))

    def run(self, stream=None) -> None:
        self.sim._check(A.asim_search_run(self.h, _stream_ptr(stream)))

    def num_runs(self) -> int:
        return int(A.asim_search_num_runs(self.h))

    def _triples(self, fn, run: int):
        n = ctypes.c_int64()
        self.sim._check(fn(self.h, int(run), 0, None, None, None, ctypes.byref(n)))
        k = n.value
        m = np.zeros(k, np.int32)
        g = np.zeros(k, np.int32)
        v = np.zeros(k, np.int64)
        self.sim._check(fn(self.h, int(run), k, _ptr(m), _ptr(g), _ptr(v), ctypes.byref(n)))
        return m, g, v

    def history(self, run: int):
        """(model[i], group[i], good[i]) of every step of `run` so far."""
        return self._triples(A.asim_search_run_history, run)

    def candidates(self, run: int):
        """(model, group, good) of every candidate of `run`'s last step."""
        return self._triples(A.asim_search_run_candidates, run)

    def result(self) -> SearchResult:
        M = self.sim.M
        cfg = np.full(A.ASIM_MAX_GROUPS, -1, np.int32)
        mask = np.zeros(M, np.uint64)
        r = A.asim_search_result(0, 0, 0, _ptr(cfg), _ptr(mask), 0, 0, 0, 0, 0, 0)
        self.sim._check(A.asim_search_result_get(self.h, ctypes.byref(r)))
        runs = []
        for i in range(A.asim_search_num_runs(self.h)):
            ng = ctypes.c_int32()
            bg = ctypes.c_int64()
            stp = ctypes.c_int64()
            rc = np.full(A.ASIM_MAX_GROUPS, -1, np.int32)
            rm = np.zeros(M, np.uint64)
            self.sim._check(A.asim_search_run_info(self.h, i, ctypes.byref(ng), _ptr(rc), _ptr(rm),
                                                   ctypes.byref(bg), ctypes.byref(stp)))
            runs.append(dict(num_groups=ng.value, group_cfg=rc[:ng.value].copy(), host_mask=rm,
                             best_good=bg.value, steps=stp.value,
                             pruned_at=int(A.asim_search_run_pruned(self.h, i))))
        return SearchResult(r.best_run, r.best_good, r.num_groups, cfg[:r.num_groups].copy(),
                            mask, r.steps, r.candidates, r.evaluated, r.request_evals,
                            r.memo_hits, runs, r.bounded)
