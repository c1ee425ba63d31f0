"""ctypes binding of libasim.so (include/asim.h), argument marshalling only.

Every asim_* entry point of the header is bound here under the same name.
There is no fallback: if libasim.so is missing or fails to load, importing
this module raises.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libasim.so")

ASIM_OK, ASIM_EINVAL, ASIM_EUNSORTED, ASIM_ERANGE = 0, -1, -2, -3
ASIM_ENOMEM, ASIM_ECUDA, ASIM_ESTATE = -4, -5, -6
ASIM_HOST, ASIM_DEVICE = 0, 1
ASIM_MAX_GROUPS, ASIM_MAX_STAGES, ASIM_MAX_SLOTS, ASIM_MAX_MODELS = 64, 64, 128, 65535

vp = ctypes.c_void_p
i32 = ctypes.c_int32
i64 = ctypes.c_int64


class asim_problem(ctypes.Structure):
    _fields_ = [("num_models", i32), ("num_configs", i32), ("max_stages", i32),
                ("slo_ns", vp), ("cfg_stages", vp), ("cfg_devices", vp), ("stage_ns", vp),
                ("tail_ns", vp), ("mem_bytes", vp), ("num_devices", i32),
                ("device_budget_bytes", i64)]


class asim_candidates(ctypes.Structure):
    _fields_ = [("num_candidates", i64), ("max_groups", i32), ("group_cfg", vp),
                ("host_mask", vp), ("ptr_kind", i32)]


class asim_deltas(ctypes.Structure):
    _fields_ = [("num_bases", i32), ("max_groups", i32), ("base_group_cfg", vp),
                ("base_host_mask", vp), ("num_candidates", i64), ("cand_base", vp),
                ("cand_model", vp), ("cand_group", vp), ("ptr_kind", i32)]


class asim_results(ctypes.Structure):
    _fields_ = [("good", vp), ("sum_latency_ns", vp), ("good_per_model", vp), ("argmax", vp),
                ("ptr_kind", i32), ("busy_ns", vp)]


class asim_stats(ctypes.Structure):
    _fields_ = [("launches", i64), ("sim_launches", i64), ("sim_ms", ctypes.c_double),
                ("stage_updates", i64), ("request_evals", i64), ("chunk_reruns", i64),
                ("walk_candidates", i64), ("walk_critical_chunks", i64),
                ("spec_ms", ctypes.c_double), ("spec_stage_updates", i64),
                ("pass2_ms", ctypes.c_double), ("walk_ms", ctypes.c_double),
                ("spec_lane_slots", i64), ("spec_live_lanes", i64),
                ("walk_predicted", i64), ("walk_unpredicted", i64), ("walk_mispredicted", i64),
                ("spec_class_cycles", i64 * 6), ("spec_class_updates", i64 * 6),
                ("spec_class_slots", i64 * 6), ("spec_busy_ms", ctypes.c_double),
                ("pass2_busy_ms", ctypes.c_double), ("walk_busy_ms", ctypes.c_double)]


class asim_search_spec(ctypes.Structure):
    _fields_ = [("num_runs", i32), ("run_num_groups", vp), ("run_group_cfg", vp),
                ("dedup", i32), ("fast", i32), ("buckets", i32), ("max_buckets", i32),
                ("ratio_num", i64), ("ratio_den", i64), ("bound_num", i64), ("bound_den", i64),
                ("model_latency_ns", vp), ("beam", i32), ("prune", i32),
                ("cand_bound", i32)]


class asim_bucket_result(ctypes.Structure):
    _fields_ = [("best_good", i64), ("num_buckets", i32), ("partitions", i64),
                ("considered", i64), ("bucket_of_model", vp), ("bucket_devices", vp),
                ("bucket_run", vp)]


class asim_batching(ctypes.Structure):
    _fields_ = [("max_batch", i32), ("stage_inc_ns", vp)]


class asim_search_result(ctypes.Structure):
    _fields_ = [("best_run", i32), ("best_good", i64), ("num_groups", i32), ("group_cfg", vp),
                ("host_mask", vp), ("steps", i64), ("candidates", i64), ("evaluated", i64),
                ("request_evals", i64), ("memo_hits", i64), ("bounded", i64)]


if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -m paper_2302_11665_b200.build` "
        "(there is no CPU fallback)")
_lib = ctypes.CDLL(LIB_PATH)

_P = ctypes.POINTER


def _bind(name, restype, argtypes):
    f = getattr(_lib, name)
    f.restype = restype
    f.argtypes = argtypes
    return f


asim_abi_version = _bind("asim_abi_version", i32, [])
asim_create = _bind("asim_create", i32, [i32, _P(vp)])
asim_destroy = _bind("asim_destroy", None, [vp])
asim_last_error = _bind("asim_last_error", ctypes.c_char_p, [vp])
asim_launch_count = _bind("asim_launch_count", i64, [vp])
asim_set_profiling = _bind("asim_set_profiling", i32, [vp, i32])
asim_get_stats = _bind("asim_get_stats", i32, [vp, _P(asim_stats)])
asim_reset_stats = _bind("asim_reset_stats", i32, [vp])
asim_set_path = _bind("asim_set_path", i32, [vp, i32])
asim_set_chunk_size = _bind("asim_set_chunk_size", i32, [vp, i64])
asim_set_problem = _bind("asim_set_problem", i32, [vp, _P(asim_problem)])
asim_set_trace = _bind("asim_set_trace", i32, [vp, i64, vp, vp, i32, vp])
asim_evaluate = _bind("asim_evaluate", i32, [vp, _P(asim_candidates), _P(asim_results), vp])
asim_evaluate_deltas = _bind("asim_evaluate_deltas", i32,
                             [vp, _P(asim_deltas), _P(asim_results), vp])
asim_evaluate_batching = _bind("asim_evaluate_batching", i32,
                               [vp, _P(asim_candidates), _P(asim_batching), _P(asim_results), vp])
asim_argmax = _bind("asim_argmax", i32, [vp, vp, i64, i32, _P(i64), vp])
asim_attainment = _bind("asim_attainment", ctypes.c_double, [i64, i64])
asim_search_create = _bind("asim_search_create", i32, [vp, _P(asim_search_spec), _P(vp)])
asim_search_destroy = _bind("asim_search_destroy", None, [vp])
asim_search_prepare = _bind("asim_search_prepare", i32, [vp, _P(i64)])
asim_search_evaluate = _bind("asim_search_evaluate", i32, [vp, i64, i64, vp, vp])
asim_search_apply = _bind("asim_search_apply", i32, [vp, vp, vp])
asim_search_costs = _bind("asim_search_costs", i32, [vp, i64, vp])
asim_search_run = _bind("asim_search_run", i32, [vp, vp])
asim_search_result_get = _bind("asim_search_result_get", i32, [vp, _P(asim_search_result)])
asim_search_run_info = _bind("asim_search_run_info", i32,
                             [vp, i32, _P(i32), vp, vp, _P(i64), _P(i64)])
asim_search_num_runs = _bind("asim_search_num_runs", i32, [vp])
asim_search_run_history = _bind("asim_search_run_history", i32,
                                [vp, i32, i64, vp, vp, vp, _P(i64)])
asim_search_run_candidates = _bind("asim_search_run_candidates", i32,
                                   [vp, i32, i64, vp, vp, vp, _P(i64)])
asim_search_run_pruned = _bind("asim_search_run_pruned", i64, [vp, i32])
asim_search_buckets_get = _bind("asim_search_buckets_get", i32, [vp, _P(asim_bucket_result)])

EXPORTED = [n for n in dir() if n.startswith("asim_") and callable(globals()[n])
            and not isinstance(globals()[n], type)]


class AsimError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"asim status {status}: {msg}")
        self.status = status


def check(status: int, ctx=None) -> None:
    if status != ASIM_OK:
        msg = asim_last_error(ctx)
        raise AsimError(status, msg.decode() if msg else "")
