"""CPU oracle for AlpaServe's SLO-attainment simulator -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The product
(paper_2302_11665_b200/, include/asim.h) never imports, links or executes it,
and this package imports nothing from the product: the two share only the
seeded input generators in ``workloads/``.

* ``libasim_oracle.so`` (des.cpp): event-driven simulator with explicit FIFO
  queues, an event heap and dry-run dispatch prediction (§4.3, §6
  P:812-813).
* ``simulate_batching`` / ``evaluate_batching`` (des.cpp): the dynamic
  batching variant of §5.4: per-model request queues, batches formed
  by a group when it becomes available, explicit batch events.
* ``oracle.search``: Alg. 1 (k = 1), Alg. 2 single bucket
   and brute force over every placement of tiny instances.

Pins (tests/test_oracle_pins.py) tie this code to the paper's worked example
(P:620), the M/D/1 and pipeline closed forms, the motivating
example's printed means and brute force.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "des.cpp")
_HDR = os.path.join(_HERE, "asim_oracle.h")
_LIB = os.path.join(_HERE, "libasim_oracle.so")
_lock = threading.Lock()
_lib = None
_active = _LIB  # the library lib() loads (the portable build unless use_timing_build())


def build(force: bool = False) -> str:
    """Compile des.cpp (host C++ only; portable -O2, no -march=native so the
    .so also runs on the GPU box's host CPU)."""
    stale = (not os.path.exists(_LIB)
             or os.path.getmtime(_LIB) < max(os.path.getmtime(_SRC), os.path.getmtime(_HDR)))
    if force or stale:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-pthread",
                               "-Wall", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


class _Problem(ctypes.Structure):
    _fields_ = [("num_models", ctypes.c_int32), ("num_configs", ctypes.c_int32),
                ("max_stages", ctypes.c_int32),
                ("slo_ns", ctypes.c_void_p), ("cfg_stages", ctypes.c_void_p),
                ("cfg_devices", ctypes.c_void_p), ("stage_ns", ctypes.c_void_p),
                ("tail_ns", ctypes.c_void_p), ("mem_bytes", ctypes.c_void_p),
                ("num_devices", ctypes.c_int32), ("device_budget_bytes", ctypes.c_int64)]


class _Trace(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("arrival_ns", ctypes.c_void_p),
                ("model", ctypes.c_void_p)]


def use_timing_build() -> str:
    """For the CPU-baseline timings only (bench.py's cpu_baseline / reference
    legs, scripts/cpu_baseline.py): the same des.cpp built -O3 -march=native
    for THIS host, into a temporary directory on it.  The tests
    keep the portable -O2 build.  Switches every later oracle call."""
    import hashlib
    import tempfile

    global _lib, _active
    tag = hashlib.sha1(open(_SRC, "rb").read() + open(_HDR, "rb").read()).hexdigest()[:12]
    path = os.path.join(tempfile.gettempdir(), f"asim_oracle_native_{tag}_{os.getpid()}.so")
    if not os.path.exists(path):
        subprocess.check_call(["g++", "-O3", "-march=native", "-std=c++17", "-shared", "-fPIC",
                               "-pthread", "-o", path, _SRC])
    with _lock:
        _active = path
        _lib = None
    return path


def lib():
    global _lib
    with _lock:
        if _lib is None:
            if _active == _LIB:
                build()
            L = ctypes.CDLL(_active)
            P = ctypes.POINTER(_Problem)
            T = ctypes.POINTER(_Trace)
            vp = ctypes.c_void_p
            L.asim_oracle_simulate.argtypes = [P, T, ctypes.c_int32, vp, vp, vp, vp, vp, vp, vp]
            L.asim_oracle_simulate.restype = ctypes.c_int32
            L.asim_oracle_feasible.argtypes = [P, ctypes.c_int32, vp, vp]
            L.asim_oracle_feasible.restype = ctypes.c_int32
            L.asim_oracle_evaluate.argtypes = [P, T, ctypes.c_int64, ctypes.c_int32, vp, vp,
                                               ctypes.c_int32, vp, vp, vp]
            L.asim_oracle_evaluate.restype = ctypes.c_int32
            L.asim_oracle_simulate_batching.argtypes = [P, T, ctypes.c_int32, vp, vp, vp,
                                                        ctypes.c_int32, vp, vp, vp, vp, vp]
            L.asim_oracle_simulate_batching.restype = ctypes.c_int32
            L.asim_oracle_evaluate_batching.argtypes = [P, T, ctypes.c_int64, ctypes.c_int32, vp,
                                                        vp, vp, ctypes.c_int32, ctypes.c_int32,
                                                        vp, vp, vp]
            L.asim_oracle_evaluate_batching.restype = ctypes.c_int32
            L.asim_oracle_error.restype = ctypes.c_char_p
            L.asim_oracle_hardware_threads.restype = ctypes.c_int32
            _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data if a is not None else None


class OracleProblem:
    """ctypes view of a workloads.Problem (keeps the arrays alive)."""

    def __init__(self, prob):
        self.prob = prob
        self._arrs = dict(
            slo=np.ascontiguousarray(prob.slo_ns, dtype=np.int64),
            stages=np.ascontiguousarray(prob.cfg_stages, dtype=np.int32),
            devs=np.ascontiguousarray(prob.cfg_devices, dtype=np.int32),
            stage=np.ascontiguousarray(prob.stage_ns, dtype=np.int64),
            tail=np.ascontiguousarray(prob.tail_ns, dtype=np.int64),
            mem=np.ascontiguousarray(prob.mem_bytes, dtype=np.int64))
        a = self._arrs
        self.c = _Problem(prob.num_models, prob.num_configs, prob.max_stages,
                          _ptr(a["slo"]), _ptr(a["stages"]), _ptr(a["devs"]), _ptr(a["stage"]),
                          _ptr(a["tail"]), _ptr(a["mem"]), prob.num_devices, prob.budget_bytes)


class OracleTrace:
    def __init__(self, trace):
        self.arrival = np.ascontiguousarray(trace.arrival_ns, dtype=np.int64)
        self.model = np.ascontiguousarray(trace.model, dtype=np.int32)
        self.c = _Trace(len(self.arrival), _ptr(self.arrival), _ptr(self.model))


def _wrap(prob, trace):
    op = prob if isinstance(prob, OracleProblem) else OracleProblem(prob)
    ot = trace if isinstance(trace, OracleTrace) else OracleTrace(trace)
    return op, ot


def _check(rc):
    if rc < 0:
        raise ValueError(lib().asim_oracle_error().decode())
    return rc


def simulate(prob, trace, placement, detail: bool = False) -> dict:
    """Simulate one placement.  Returns good, sum_latency_ns, good_per_model
    and, with detail=True, per-request finish_ns (-1 = rejected) and
    served_by (group, -1 = rejected)."""
    op, ot = _wrap(prob, trace)
    M, N = op.prob.num_models, len(ot.arrival)
    cfg = np.ascontiguousarray(placement.group_cfg, dtype=np.int32)
    mask = np.ascontiguousarray(placement.host_mask, dtype=np.uint64)
    good = np.zeros(1, np.int64)
    sl = np.zeros(1, np.int64)
    pm = np.zeros(M, np.int64)
    fin = np.zeros(N, np.int64) if detail else None
    srv = np.zeros(N, np.int32) if detail else None
    _check(lib().asim_oracle_simulate(ctypes.byref(op.c), ctypes.byref(ot.c), len(cfg),
                                      _ptr(cfg), _ptr(mask), _ptr(good), _ptr(sl), _ptr(pm),
                                      _ptr(fin), _ptr(srv)))
    out = dict(good=int(good[0]), sum_latency_ns=int(sl[0]), good_per_model=pm)
    if detail:
        out.update(finish_ns=fin, served_by=srv)
    return out


def feasible(prob, placement) -> bool:
    op = prob if isinstance(prob, OracleProblem) else OracleProblem(prob)
    cfg = np.ascontiguousarray(placement.group_cfg, dtype=np.int32)
    mask = np.ascontiguousarray(placement.host_mask, dtype=np.uint64)
    return bool(_check(lib().asim_oracle_feasible(ctypes.byref(op.c), len(cfg), _ptr(cfg),
                                                  _ptr(mask))))


def evaluate(prob, trace, group_cfg, host_mask, threads: int = 0, per_model: bool = False):
    """Batch of C placements: group_cfg [C, G] int32, host_mask [C, M] uint64.
    Returns (good[C], sum_latency_ns[C], good_per_model[C, M] or None)."""
    op, ot = _wrap(prob, trace)
    cfg = np.ascontiguousarray(group_cfg, dtype=np.int32)
    mask = np.ascontiguousarray(host_mask, dtype=np.uint64)
    C, G = cfg.shape
    M = op.prob.num_models
    assert mask.shape == (C, M)
    good = np.zeros(C, np.int64)
    sl = np.zeros(C, np.int64)
    pm = np.zeros((C, M), np.int64) if per_model else None
    _check(lib().asim_oracle_evaluate(ctypes.byref(op.c), ctypes.byref(ot.c), C, G, _ptr(cfg),
                                      _ptr(mask), int(threads), _ptr(good), _ptr(sl), _ptr(pm)))
    return good, sl, pm


def simulate_batching(prob, trace, placement, stage_inc_ns, max_batch: int,
                      detail: bool = False) -> dict:
    """Dynamic batching variant (§5.4) of simulate(): a batch of k
    requests occupies stage j for stage_ns + (k-1) * stage_inc_ns[m][p][j]."""
    op, ot = _wrap(prob, trace)
    M, N = op.prob.num_models, len(ot.arrival)
    cfg = np.ascontiguousarray(placement.group_cfg, dtype=np.int32)
    mask = np.ascontiguousarray(placement.host_mask, dtype=np.uint64)
    inc = np.ascontiguousarray(stage_inc_ns, dtype=np.int64)
    assert inc.shape == np.shape(op.prob.stage_ns)
    good = np.zeros(1, np.int64)
    sl = np.zeros(1, np.int64)
    pm = np.zeros(M, np.int64)
    fin = np.zeros(N, np.int64) if detail else None
    srv = np.zeros(N, np.int32) if detail else None
    _check(lib().asim_oracle_simulate_batching(ctypes.byref(op.c), ctypes.byref(ot.c), len(cfg),
                                               _ptr(cfg), _ptr(mask), _ptr(inc), int(max_batch),
                                               _ptr(good), _ptr(sl), _ptr(pm), _ptr(fin),
                                               _ptr(srv)))
    out = dict(good=int(good[0]), sum_latency_ns=int(sl[0]), good_per_model=pm)
    if detail:
        out.update(finish_ns=fin, served_by=srv)
    return out


def evaluate_batching(prob, trace, group_cfg, host_mask, stage_inc_ns, max_batch: int,
                      threads: int = 0, per_model: bool = False):
    """Batch of C placements under dynamic batching; same shapes as evaluate()."""
    op, ot = _wrap(prob, trace)
    cfg = np.ascontiguousarray(group_cfg, dtype=np.int32)
    mask = np.ascontiguousarray(host_mask, dtype=np.uint64)
    inc = np.ascontiguousarray(stage_inc_ns, dtype=np.int64)
    assert inc.shape == np.shape(op.prob.stage_ns)
    C, G = cfg.shape
    M = op.prob.num_models
    assert mask.shape == (C, M)
    good = np.zeros(C, np.int64)
    sl = np.zeros(C, np.int64)
    pm = np.zeros((C, M), np.int64) if per_model else None
    _check(lib().asim_oracle_evaluate_batching(ctypes.byref(op.c), ctypes.byref(ot.c), C, G,
                                               _ptr(cfg), _ptr(mask), _ptr(inc), int(max_batch),
                                               int(threads), _ptr(good), _ptr(sl), _ptr(pm)))
    return good, sl, pm


def hardware_threads() -> int:
    return int(lib().asim_oracle_hardware_threads())


def attainment(good: int, n: int) -> float:
    """SLO attainment = good / N; N = 0 -> 1.0 (reading C9)."""
    if good < 0:
        return -1.0
    return 1.0 if n == 0 else good / n
