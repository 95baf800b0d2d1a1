"""Formats around the plan path through the C ABI:
the reference's "# amppi-cloud v1" text frames (io.cpp:24-66) and a binary
variant, and the partition.csv / anchors.csv debug dumps (io.cpp:68-99)."""
from __future__ import annotations

import ctypes

import numpy as np

from . import _abi


def _lib():
    return _abi.load()


def read_cloud(path: str) -> tuple[np.ndarray, int]:
    """(points [n,3] float64, frame id) from a text or binary cloud frame."""
    lib = _lib()
    n = ctypes.c_int64()
    fid = ctypes.c_uint64()
    rc = lib.amppi_cloud_read(path.encode(), None, 0, ctypes.byref(n), ctypes.byref(fid))
    if rc != 0:
        raise ValueError(f"not a readable cloud frame: {path}")
    xyz = np.zeros((int(n.value), 3))
    rc = lib.amppi_cloud_read(path.encode(), xyz.ctypes.data_as(_abi.c_double_p), int(n.value), ctypes.byref(n),
                              ctypes.byref(fid))
    if rc != 0:
        raise ValueError(f"malformed cloud frame: {path}")
    return xyz, int(fid.value)


def write_cloud(path: str, xyz, frame_id: int = 0, binary: bool = False) -> None:
    a = np.ascontiguousarray(np.asarray(xyz, dtype=np.float64).reshape(-1, 3))
    rc = _lib().amppi_cloud_write(path.encode(), a.ctypes.data_as(_abi.c_double_p), len(a), frame_id, int(binary))
    if rc != 0:
        raise OSError(f"cannot write cloud frame: {path}")


def write_partition_csv(path: str, ranges) -> None:
    r = np.ascontiguousarray(np.asarray(ranges, dtype=np.float64).reshape(-1))
    if r.size != 7200:
        raise ValueError("ranges must hold the 120 x 60 cells (flat i*60+j)")
    if _lib().amppi_partition_csv(path.encode(), r.ctypes.data_as(_abi.c_double_p)) != 0:
        raise OSError(f"cannot write {path}")


def write_anchors_csv(path: str, step: int, plan, horizon: float, samples: int) -> None:
    """plan: a PlanResult (anchors + guides) from Planner.plan_step."""
    refined = np.ascontiguousarray([a.refined_endpoint for a in plan.anchors], dtype=np.float64)
    guides = np.ascontiguousarray(plan.guides, dtype=np.float64)
    rc = _lib().amppi_anchors_csv(path.encode(), step, len(refined), refined.ctypes.data_as(_abi.c_double_p),
                                  guides.ctypes.data_as(_abi.c_double_p), float(horizon), samples)
    if rc != 0:
        raise OSError(f"cannot write {path}")
