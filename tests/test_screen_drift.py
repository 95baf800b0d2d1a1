"""The FP32 screening's soundness argument, measured (DESIGN.md §2 "The d_max
jump"; round-1 VERDICT weak item 3).

The screening integrates every rollout in FP32 and only selects the softmin
support; it is sound while, at every step, the FP32 clearance d32 is on the
same side of d_max as the FP64 clearance d64 whenever |d32 - d_max| is at
least the band 1e-4 d_max + 1e-4 (inside the band the step is flagged and the
FP64 refine decides).  amppi_screen_drift integrates sampled rollouts of a
planned batch both ways (the screening's FP32 draws, clamp and RK4 with the
FP32 grid query; the refine's FP64 path with the exact FP64 query) and
reports the largest position and clearance differences and the number of
steps that violate the band.  Asserted here on C5 scenes of every kind
(forest, verticals, inclines) and on C4-sized instances; the whole-batch
numbers are in profiles/r02_screen_drift.md (tools/screen_drift.py).
"""
import numpy as np
import pytest
import torch

BAND = 1e-4 * 1.0 + 1e-4  # amb_band(d_max = 1.0)


def _device_batch(d):
    dev = torch.device("cuda", 0)
    t = {k: torch.from_numpy(np.ascontiguousarray(d[k])).to(dev)
         for k in ("xyz", "offsets", "poses", "states", "goals", "last")}
    t["cycles"] = torch.from_numpy(d["cycles"].view(np.int64)).to(dev)
    t["seeds"] = torch.from_numpy(d["seeds"].view(np.int64)).to(dev)
    return t, {k: v.data_ptr() for k, v in t.items()}


def _drift(cfg, n_scenes, first, stride, kinds=None, iterations_checked=(0,), offset=None):
    from paper_2509_17340_b200 import Planner
    from paper_2509_17340_b200.workloads import scenes

    d = scenes(n_scenes, points=20000, frames=20, first=first, kinds=kinds)
    if offset is not None:  # the whole scene translated (points, pose, state, goal)
        d["xyz"] = (d["xyz"].astype(np.float64) + np.asarray(offset)).astype(np.float32)
        for k in ("poses", "states", "goals"):
            d[k][:, :3] += offset
    t, ptr = _device_batch(d)
    status = torch.zeros(n_scenes, dtype=torch.int32, device="cuda:0")
    with Planner(cfg, max_scenes=n_scenes, max_points=int(d["offsets"][-1])) as p:
        p.cycle_batch_device(ptr, {"status": status.data_ptr()}, n_scenes)
        p.synchronize()
        return [p.screen_drift(ptr, n_scenes, it, stride) for it in iterations_checked]


def _check(r):
    assert r["rollouts"] > 0
    assert r["validity_mismatches"] == 0
    assert r["dmax_side_violations"] == 0
    # the band is 2e-4 m: the FP32 clearance must sit far inside it (whole C5
    # batch: 3.8e-6 m; C4 instances: 6.1e-6 m; profiles/r02_screen_drift.md)
    assert r["max_clearance_diff"] < BAND / 10, r
    assert r["max_pos_diff"] < BAND / 4, r
    # k_support's window allows 1e-4 |rho| of FP32 error between a sample and
    # the minimum: each cost must be within half of that
    assert r["max_rel_cost_diff"] < 5e-5, r


@pytest.mark.gpu
@pytest.mark.parametrize("kind", [1, 2, 3])
def test_screen_drift_c5_scenes(kind):
    from paper_2509_17340_b200.workloads import plan_config

    (r,) = _drift(plan_config(), 96, first=500 + kind, stride=1, kinds=kind)
    _check(r)
    assert r["rollouts"] >= 96 * 8 * 256 * 0.9
    assert r["steps_compared"] > 0


@pytest.mark.gpu
def test_screen_drift_far_from_world_origin():
    """Scenes 8 km / 4 km from the world origin: the screening's local frame
    keeps the drift where it is near the origin (in world coordinates an FP32
    ulp there is 1e-3 m, five times the band)."""
    from paper_2509_17340_b200.workloads import plan_config

    (r,) = _drift(plan_config(), 48, first=900, stride=1, offset=(8192.0, -4096.0, 0.0))
    _check(r)


@pytest.mark.gpu
def test_screen_drift_c4_instances():
    """C4's 50-step horizon: the longest FP32 integration of any config."""
    from paper_2509_17340_b200.workloads import plan_config

    (r,) = _drift(plan_config(8, 8, K=8192, N=50), 2, first=40, stride=8)
    _check(r)


@pytest.mark.gpu
def test_screen_drift_later_iteration():
    """Two MPPI iterations: the perturbation stream of iteration 1."""
    from paper_2509_17340_b200.workloads import plan_config

    r0, r1 = _drift(plan_config(iterations=2), 32, first=7, stride=2, iterations_checked=(0, 1))
    _check(r0)
    _check(r1)


@pytest.mark.gpu
def test_screen_drift_rejects_bad_arguments():
    from paper_2509_17340_b200 import Planner
    from paper_2509_17340_b200.workloads import plan_config, scenes

    d = scenes(4, points=20000, frames=20, first=0)
    t, ptr = _device_batch(d)
    with Planner(plan_config(), max_scenes=4, max_points=int(d["offsets"][-1])) as p:
        p.cycle_batch_device(ptr, {}, 4)
        with pytest.raises(ValueError):
            p.screen_drift(ptr, 4, 0, 0)
        with pytest.raises(ValueError):
            p.screen_drift(ptr, 4, 1, 1)  # one iteration only
