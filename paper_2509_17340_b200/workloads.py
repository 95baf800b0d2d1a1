"""Synthetic workloads of BASELINE.json's configs, built with the product's own
input generator (amppi_sim_scan: reference scenario families + GPU LiDAR).

C1  one plan cycle, 20k-point forest scan, 4x2 anchors x 256 samples x 30 steps
C3  one plan cycle on a ~1M-point verticals / inclines accumulation
C4  64 anchors (8x8) x 8192 samples x 50 steps on the C1 cloud
C5  4096 independent scenes (forest / verticals / inclines) x C1 plan sizes
"""
from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _abi
from .planner import EnsembleConfig

KIND_NAMES = {1: "forest", 2: "verticals", 3: "inclines"}


def plan_config(m_h=4, m_v=2, K=256, N=30, iterations=1) -> EnsembleConfig:
    cfg = EnsembleConfig()
    cfg.grid.m_h, cfg.grid.m_v = m_h, m_v
    cfg.mppi.rollouts, cfg.mppi.horizon, cfg.mppi.iterations = K, N, iterations
    return cfg


def rollout_steps(cfg: EnsembleConfig, scenes: int = 1) -> int:
    return scenes * cfg.grid.count() * cfg.mppi.rollouts * cfg.mppi.horizon * cfg.mppi.iterations


def _mix64(z: int) -> int:
    M = (1 << 64) - 1
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31)


def scan_scenes(kinds, seeds, frames: int, frame_poses: np.ndarray, frame_seeds: np.ndarray, r_max: float,
                cap_per_scene: int, device: int = 0):
    """GPU LiDAR scans: returns (xyz float32 [P,3], offsets int64 [S+1])."""
    lib = _abi.load()
    S = len(kinds)
    k = np.ascontiguousarray(kinds, dtype=np.int32)
    sd = np.ascontiguousarray(seeds, dtype=np.uint64)
    poses = np.ascontiguousarray(frame_poses, dtype=np.float64).reshape(S * frames, 10)
    fs = np.ascontiguousarray(frame_seeds, dtype=np.uint64).reshape(S * frames)
    xyz = np.zeros((S * cap_per_scene, 3), dtype=np.float32)
    off = np.zeros(S + 1, dtype=np.int64)
    rc = lib.amppi_sim_scan(S, k.ctypes.data_as(_abi.c_int32_p), sd.ctypes.data_as(_abi.c_uint64_p), frames,
                            poses.ctypes.data, fs.ctypes.data_as(_abi.c_uint64_p), r_max, cap_per_scene,
                            xyz.ctypes.data_as(_abi.c_float_p), off.ctypes.data_as(_abi.c_int64_p), device)
    if rc != 0:
        raise RuntimeError(f"amppi_sim_scan failed ({rc})")
    return xyz[: off[-1]].copy(), off


def scan_scenes_host(kinds, seeds, frames: int, frame_poses: np.ndarray, frame_seeds: np.ndarray, r_max: float,
                     cap_per_scene: int):
    """The same scans on the host (amppi_sim_scan_host, identical bytes)."""
    lib = _abi.load()
    S = len(kinds)
    k = np.ascontiguousarray(kinds, dtype=np.int32)
    sd = np.ascontiguousarray(seeds, dtype=np.uint64)
    poses = np.ascontiguousarray(frame_poses, dtype=np.float64).reshape(S * frames, 10)
    fs = np.ascontiguousarray(frame_seeds, dtype=np.uint64).reshape(S * frames)
    xyz = np.zeros((S * cap_per_scene, 3), dtype=np.float32)
    off = np.zeros(S + 1, dtype=np.int64)
    rc = lib.amppi_sim_scan_host(S, k.ctypes.data_as(_abi.c_int32_p), sd.ctypes.data_as(_abi.c_uint64_p), frames,
                                 poses.ctypes.data, fs.ctypes.data_as(_abi.c_uint64_p), r_max, cap_per_scene,
                                 xyz.ctypes.data_as(_abi.c_float_p), off.ctypes.data_as(_abi.c_int64_p))
    if rc != 0:
        raise RuntimeError(f"amppi_sim_scan_host failed ({rc})")
    return xyz[: off[-1]].copy(), off


def scene_start(scene_id: int) -> np.ndarray:
    """Where the vehicle enters scene `scene_id` (a function of the id alone,
    so any subset of a batch -- a rank's shard, the CPU baseline's sample --
    sees exactly the bytes the whole batch does)."""
    rng = np.random.default_rng([12345, scene_id])
    return np.array([rng.uniform(1.0, 30.0), rng.uniform(-8.0, 8.0), 2.0])


def scenes(n_scenes: int, points: int = 20000, frames: int = 20, first: int = 0, device: int = 0,
           kinds=None, r_max: float = 10.0, host: bool = False, frame_step: float = 0.06) -> dict:
    """Scenes first..first+n_scenes-1 of the C5 family (scene s: kind 1 + s % 3,
    seed s + 1; every array row is a function of the scene id only).  The
    vehicle advances frame_step metres along +x per frame (0.06: 3 m/s at
    50 Hz); the last frame's pose is the snapshot pose and the plan state.  host=True scans on the CPU
    (amppi_sim_scan_host): the same bytes without a GPU."""
    ids = np.arange(first, first + n_scenes)
    kinds = (1 + ids % 3).astype(np.int32) if kinds is None else np.full(n_scenes, kinds, dtype=np.int32)
    start = np.stack([scene_start(int(i)) for i in ids]) if n_scenes else np.zeros((0, 3))
    f = np.arange(frames)
    poses = np.zeros((n_scenes, frames, 10))
    poses[:, :, 0:3] = start[:, None, :] + np.stack([frame_step * f, 0 * f, 0 * f], axis=1)[None]
    poses[:, :, 3] = 1.0
    poses[:, :, 7] = 3.0
    fseeds = np.array([[(_mix64(int(s) + 1) + int(i)) & ((1 << 64) - 1) for i in f] for s in ids], dtype=np.uint64)
    if host:
        xyz, off = scan_scenes_host(kinds, ids + 1, frames, poses, fseeds, r_max, points)
    else:
        xyz, off = scan_scenes(kinds, ids + 1, frames, poses, fseeds, r_max, points, device)
    state = poses[:, -1, :].copy()
    goal = np.zeros((n_scenes, 10))
    goal[:, 0:3] = (45.0, 0.0, 2.0)
    goal[:, 6] = 1.0  # GoalSpec::facing((0,0,2), (45,0,2)) = identity
    hover = EnsembleConfig().dynamics.hover().thrust
    return dict(xyz=xyz, offsets=off, poses=state.copy(), states=state, goals=goal,
                last=np.tile([hover, 0.0, 0.0, 0.0], (n_scenes, 1)), cycles=np.full(n_scenes, 100, dtype=np.uint64),
                seeds=(ids + 1).astype(np.uint64), kinds=kinds)
