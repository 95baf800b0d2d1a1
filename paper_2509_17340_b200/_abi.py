"""ctypes mirror of include/amppi_b200.h (the C-ABI boundary).

The shared library is built in-tree (paper_2509_17340_b200/libamppi_b200.so,
see __graft_entry__.build()).  Loading fails loudly when it is missing: there
is no CPU fallback for any planning entry point.
"""
from __future__ import annotations

import ctypes
import os

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libamppi_b200.so")

AMPPI_OK = 0
AMPPI_PLANNING_FAILED = 1
AMPPI_INVALID_ARGUMENT = 2
AMPPI_CUDA_ERROR = 3
AMPPI_NCCL_ERROR = 4
AMPPI_NO_SNAPSHOT = 5

c_double_p = ctypes.POINTER(ctypes.c_double)
c_float_p = ctypes.POINTER(ctypes.c_float)
c_int32_p = ctypes.POINTER(ctypes.c_int32)
c_int64_p = ctypes.POINTER(ctypes.c_int64)
c_uint8_p = ctypes.POINTER(ctypes.c_uint8)
c_uint64_p = ctypes.POINTER(ctypes.c_uint64)


class Config(ctypes.Structure):
    """amppi_config == EnsembleConfig (ensemble.hpp:16-23), flattened."""

    _fields_ = [
        ("m_h", ctypes.c_int32), ("m_v", ctypes.c_int32),
        ("lookahead", ctypes.c_double), ("spacing_deg", ctypes.c_double),
        ("terminal_speed", ctypes.c_double), ("min_anchor_distance", ctypes.c_double),
        ("rollouts", ctypes.c_int32), ("horizon", ctypes.c_int32),
        ("lambda_", ctypes.c_double),
        ("sigma", ctypes.c_double * 4),
        ("mppi_dt", ctypes.c_double),
        ("iterations", ctypes.c_int32),
        ("q_track", ctypes.c_double), ("q_vnorm", ctypes.c_double), ("q_c", ctypes.c_double),
        ("q_c_delta", ctypes.c_double), ("q_p", ctypes.c_double), ("q_v", ctypes.c_double),
        ("q_q", ctypes.c_double),
        ("col_scale", ctypes.c_double), ("col_slope", ctypes.c_double),
        ("col_d_min", ctypes.c_double), ("col_d_max", ctypes.c_double),
        ("mass", ctypes.c_double),
        ("gravity", ctypes.c_double * 3),
        ("dyn_dt", ctypes.c_double),
        ("thrust_min", ctypes.c_double), ("thrust_max", ctypes.c_double),
        ("omega_xy_max", ctypes.c_double), ("omega_z_max", ctypes.c_double),
        ("replan_hz", ctypes.c_double), ("r_max", ctypes.c_double),
    ]


class State(ctypes.Structure):
    _fields_ = [("p", ctypes.c_double * 3), ("q", ctypes.c_double * 4), ("v", ctypes.c_double * 3)]


class Control(ctypes.Structure):
    _fields_ = [("thrust", ctypes.c_double), ("omega", ctypes.c_double * 3)]


class Goal(ctypes.Structure):
    _fields_ = [("p_goal", ctypes.c_double * 3), ("v_goal", ctypes.c_double * 3), ("q_goal", ctypes.c_double * 4)]


class Schedule(ctypes.Structure):
    """amppi_schedule: how a call is split over streams / chunks (never its results); 0 = automatic."""

    _fields_ = [
        ("pipeline_chunks", ctypes.c_int32), ("pipeline_ratio", ctypes.c_double),
        ("pipeline_streams", ctypes.c_int32), ("device_chunks", ctypes.c_int32),
        ("chunk_gather", ctypes.c_int32), ("loop_graph", ctypes.c_int32), ("plan_graph", ctypes.c_int32),
        ("trace", ctypes.c_int32),
    ]


class Options(ctypes.Structure):
    _fields_ = [
        ("device", ctypes.c_int32), ("precision", ctypes.c_int32), ("max_scenes", ctypes.c_int32),
        ("max_points", ctypes.c_int64), ("profile", ctypes.c_int32), ("stream", ctypes.c_void_p),
        ("refine_split_cap", ctypes.c_int64), ("schedule", Schedule),
    ]


class PlanResult(ctypes.Structure):
    _fields_ = [
        ("winner", ctypes.c_int32),
        ("control", Control),
        ("breakdown", ctypes.c_double * 5),
        ("stage1", c_double_p), ("stage2", c_double_p), ("ess", c_double_p), ("valid", c_uint8_p),
        ("nominal", c_double_p), ("winner_states", c_double_p), ("winner_controls", c_double_p),
        ("anchor_initial", c_double_p), ("anchor_refined", c_double_p), ("anchor_safe_dir", c_double_p),
        ("anchor_safe_range", c_double_p), ("anchor_ij", c_int32_p), ("guide_coeffs", c_double_p),
        ("sample_costs", c_double_p),
    ]


class SnapshotView(ctypes.Structure):
    _fields_ = [
        ("ranges", c_double_p), ("has_point", c_uint8_p), ("nearest", c_double_p),
        ("safe_range", c_double_p), ("safe_dir", c_double_p), ("safe_point", c_double_p),
        ("filtered", c_double_p), ("n_filtered", ctypes.c_int64),
    ]


class BatchInput(ctypes.Structure):
    _fields_ = [
        ("n_scenes", ctypes.c_int32),
        ("point_offsets", c_int64_p), ("xyz", c_float_p),
        ("poses", ctypes.c_void_p), ("states", ctypes.c_void_p), ("goals", ctypes.c_void_p),
        ("previous", c_double_p), ("previous_len", c_int32_p), ("last_applied", ctypes.c_void_p),
        ("cycles", c_uint64_p), ("seeds", c_uint64_p), ("r_max", ctypes.c_double),
    ]


class BatchOutput(ctypes.Structure):
    _fields_ = [
        ("status", c_int32_p), ("winner", c_int32_p), ("control", c_double_p),
        ("winner_nominal", c_double_p), ("stage2", c_double_p), ("breakdown", c_double_p),
    ]


class LoopRecord(ctypes.Structure):
    _fields_ = [("cycle", ctypes.c_uint64), ("planned", ctypes.c_int32), ("winner", ctypes.c_int32),
                ("x", ctypes.c_double * 10), ("control", ctypes.c_double * 4), ("stage2", ctypes.c_double),
                ("status", ctypes.c_int32), ("n_points", ctypes.c_int32), ("t", ctypes.c_double),
                ("x_after", ctypes.c_double * 10), ("clearance", ctypes.c_double), ("breakdown", ctypes.c_double * 5)]


class EpisodeMetrics(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in
                ("avg_vel", "max_vel", "smoothness", "path_length", "avg_clearance", "min_clearance")]


EXPORTS = {
    "amppi_config_default": (None, [ctypes.POINTER(Config)]),
    "amppi_options_default": (None, [ctypes.POINTER(Options)]),
    "amppi_abi_version": (ctypes.c_int, []),
    "amppi_create": (ctypes.c_int, [ctypes.POINTER(Config), ctypes.POINTER(Options), ctypes.POINTER(ctypes.c_void_p)]),
    "amppi_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "amppi_last_error": (ctypes.c_char_p, [ctypes.c_void_p]),
    "amppi_synchronize": (ctypes.c_int, [ctypes.c_void_p]),
    "amppi_set_config": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(Config)]),
    "amppi_get_config": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(Config)]),
    "amppi_set_schedule": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(Schedule)]),
    "amppi_snapshot": (ctypes.c_int, [ctypes.c_void_p, c_float_p, ctypes.c_int64, ctypes.POINTER(State), ctypes.c_double]),
    "amppi_snapshot_f64": (ctypes.c_int, [ctypes.c_void_p, c_double_p, ctypes.c_int64, ctypes.POINTER(State), ctypes.c_double]),
    "amppi_snapshot_device": (ctypes.c_int, [ctypes.c_void_p, c_float_p, ctypes.c_int64, ctypes.POINTER(State),
                                             ctypes.c_double]),
    "amppi_snapshot_download": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(SnapshotView)]),
    "amppi_plan": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(State), ctypes.POINTER(Goal), c_double_p,
                                  ctypes.c_int32, ctypes.POINTER(Control), ctypes.c_uint64, ctypes.c_uint64,
                                  c_double_p, ctypes.POINTER(PlanResult)]),
    "amppi_cycle_batch": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(BatchInput), ctypes.POINTER(BatchOutput)]),
    "amppi_cycle_batch_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(BatchInput), ctypes.POINTER(BatchOutput)]),
    "amppi_cycle_batch_submit": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(BatchInput), c_int64_p]),
    "amppi_cycle_batch_wait": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(BatchOutput)]),
    "amppi_kernel_times": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_char_p), c_double_p, c_int64_p,
                                          ctypes.c_int32, c_int32_p]),
    "amppi_kernel_times_reset": (ctypes.c_int, [ctypes.c_void_p]),
    "amppi_screen_drift": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(BatchInput), ctypes.c_int32, ctypes.c_int32,
                                          c_double_p]),
    "amppi_set_stream": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "amppi_get_stream": (ctypes.c_void_p, [ctypes.c_void_p]),
    "amppi_nccl_version": (ctypes.c_int, [c_int32_p]),
    "amppi_nccl_unique_id": (ctypes.c_int, [ctypes.c_void_p]),
    "amppi_nccl_comm_init": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int32, ctypes.c_void_p,
                                            ctypes.c_int32, ctypes.c_int32]),
    "amppi_nccl_comm_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "amppi_plan_sharded": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                                          ctypes.POINTER(State), ctypes.POINTER(Goal), c_double_p, ctypes.c_int32,
                                          ctypes.POINTER(Control), ctypes.c_uint64, ctypes.c_uint64,
                                          ctypes.POINTER(PlanResult)]),
    "amppi_sim_scan": (ctypes.c_int, [ctypes.c_int32, c_int32_p, c_uint64_p, ctypes.c_int32, ctypes.c_void_p,
                                      c_uint64_p, ctypes.c_double, ctypes.c_int64, c_float_p, c_int64_p,
                                      ctypes.c_int32]),
    "amppi_sim_scan_host": (ctypes.c_int, [ctypes.c_int32, c_int32_p, c_uint64_p, ctypes.c_int32, ctypes.c_void_p,
                                           c_uint64_p, ctypes.c_double, ctypes.c_int64, c_float_p, c_int64_p]),
    "amppi_probe_fp32_peak": (ctypes.c_int, [ctypes.c_int32, c_double_p, c_double_p]),
    "amppi_shard_begin": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(State), ctypes.POINTER(Goal), c_double_p,
                                         ctypes.c_int32, ctypes.POINTER(Control), ctypes.c_uint64, ctypes.c_uint64,
                                         ctypes.c_int32, ctypes.c_int32]),
    "amppi_shard_screen": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p]),
    "amppi_shard_partials": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p]),
    "amppi_shard_update": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32]),
    "amppi_shard_finish": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(PlanResult)]),
    "amppi_shard_partials_stride": (ctypes.c_int32, [ctypes.c_void_p]),
    "amppi_loop_create": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint64, ctypes.c_uint64,
                                         ctypes.c_int32, ctypes.c_int64, ctypes.POINTER(ctypes.c_void_p)]),
    "amppi_loop_run": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, c_int64_p]),
    "amppi_loop_records": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(LoopRecord), ctypes.c_int64, c_int64_p]),
    "amppi_loop_state": (ctypes.c_int, [ctypes.c_void_p, c_double_p, c_int32_p, c_double_p]),
    "amppi_loop_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "amppi_loop_metrics": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(EpisodeMetrics)]),
    "amppi_cloud_read": (ctypes.c_int, [ctypes.c_char_p, c_double_p, ctypes.c_int64, c_int64_p, c_uint64_p]),
    "amppi_cloud_write": (ctypes.c_int, [ctypes.c_char_p, c_double_p, ctypes.c_int64, ctypes.c_uint64,
                                         ctypes.c_int32]),
    "amppi_partition_csv": (ctypes.c_int, [ctypes.c_char_p, c_double_p]),
    "amppi_anchors_csv": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int32, ctypes.c_int32, c_double_p, c_double_p,
                                         ctypes.c_double, ctypes.c_int32]),
}

_lib = None


def load(path: str | None = None) -> ctypes.CDLL:
    """Load libamppi_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or os.environ.get("AMPPI_LIB_PATH") or LIB_PATH
    if not os.path.exists(p):
        raise RuntimeError(f"{p} not found: run __graft_entry__.build() (no CPU fallback exists)")
    lib = ctypes.CDLL(p)
    lenient = os.environ.get("AMPPI_ABI_LENIENT") == "1"  # tools/ab.py timing older builds
    for name, (res, args) in EXPORTS.items():
        if lenient and not hasattr(lib, name):
            continue
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.amppi_abi_version() != 2:
        raise RuntimeError("libamppi_b200 ABI version mismatch")
    if path is None:
        _lib = lib
    return lib
