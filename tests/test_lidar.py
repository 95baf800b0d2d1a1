"""Synthetic input generator: the FP32 LiDAR of
amppi_sim_scan (GPU) / amppi_sim_scan_host (CPU) against the oracle's FP64
restatement of lidar_scan (sim_world.cpp:248-328), and the GPU scan against
its host twin.

* CPU: per frame the FP32 scan and the oracle return the same number of hits
  (same rays hit), and, aligned ray by ray, the points agree to FP32 accuracy
  (<= 1e-3 m for >= 99.9% of them; the rest are rays grazing a silhouette,
  where FP32 and FP64 pick different surfaces).
* GPU: the device scan equals the host scan bit for bit (shared sim_ray.h
  arithmetic, no FMA contraction on either side), so the CPU baseline plans
  exactly the scenes the device planned.
"""
import math

import numpy as np
import pytest


def _frames():
    out = []
    for s in range(6):
        kind = 1 + s % 3
        for f in range(4):
            yaw = 0.15 * f - 0.2 * s
            pose = np.array([4.0 + 2.5 * f, -3.0 + 1.2 * s, 1.5 + 0.2 * f, math.cos(yaw / 2), 0.0, 0.0,
                             math.sin(yaw / 2), 3.0, 0.0, 0.0])
            out.append((kind, s + 1, pose, 1000 * s + 31 * f + 7))
    return out


def test_host_scan_matches_oracle_lidar(oracle, product_lib):
    from paper_2509_17340_b200.workloads import scan_scenes_host

    n_pts, n_close, worst_count = 0, 0, 0
    for kind, seed, pose, fseed in _frames():
        ref = oracle.scene(kind, seed).lidar(pose, fseed)
        xyz, off = scan_scenes_host([kind], [seed], 1, pose[None], np.array([fseed], dtype=np.uint64), 10.0, 8000)
        worst_count = max(worst_count, abs(len(ref) - len(xyz)))
        if len(ref) == len(xyz) and len(ref):
            d = np.linalg.norm(xyz.astype(np.float64) - ref, axis=1)
            n_pts += len(d)
            n_close += int((d <= 1e-3).sum())
    assert worst_count <= 1, worst_count
    assert n_pts > 20000
    assert n_close >= 0.999 * n_pts, (n_close, n_pts)


@pytest.mark.gpu
def test_device_scan_equals_host_scan():
    from paper_2509_17340_b200.workloads import scenes

    dev = scenes(96, points=20000, frames=20, first=300)
    host = scenes(96, points=20000, frames=20, first=300, host=True)
    assert np.array_equal(dev["offsets"], host["offsets"])
    assert np.array_equal(dev["xyz"].view(np.uint32), host["xyz"].view(np.uint32))
    for k in ("poses", "states", "goals", "last", "cycles", "seeds"):
        assert np.array_equal(dev[k], host[k]), k


@pytest.mark.gpu
def test_device_scan_1m_point_accumulation_equals_host():
    """C3-sized accumulations (verticals / inclines, ~300-420 frames)."""
    from paper_2509_17340_b200.workloads import scenes

    for kind in (2, 3):
        dev = scenes(1, points=1_000_000, frames=600, first=7, kinds=kind, frame_step=0.004)
        host = scenes(1, points=1_000_000, frames=600, first=7, kinds=kind, host=True, frame_step=0.004)
        assert dev["offsets"][-1] == 1_000_000
        assert np.array_equal(dev["xyz"].view(np.uint32), host["xyz"].view(np.uint32))
