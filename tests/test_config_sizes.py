"""Parity at BASELINE.json's full config sizes
against the CPU oracle on identical inputs.

* C4: one forest scene (C1's 20k-point cloud), 8x8 anchors x 8192 samples x
  50 steps -- unsharded, and sample-sharded over 2 and 4 shards (one context
  per shard on one GPU, the all-reduce / all-gather done as tensor ops
  between the phases of the multi-GPU protocol, sharding.plan_step_sharded_local).
* C3: one full plan cycle (snapshot + plan, C1 plan sizes) on ~1M-point
  accumulated scans of the verticals and the inclines scenes.

The contract is the one of tests/test_plan_parity.py (bit-exact integers,
FP64 results <= 1e-9).  SURVEY.md §8c allows an instance whose oracle top-2
stage-I gap is below tau = 1e-5 |S_min| + 1e-3 to count as a near-tie rather
than a failure; the FP64 refine of the screened support makes that allowance
unnecessary here, so near-ties are counted and printed, not excused."""
import math

import numpy as np
import pytest

from test_plan_parity import forest_cycle_inputs, make_cfg, rel, run_case

pytestmark = pytest.mark.gpu


def near_ties(o):
    """(stage-I near-tie instances, stage-II winner near-tie) of an oracle plan."""
    n1 = 0
    for row in o["sample_costs"]:
        f = np.sort(row[np.isfinite(row)])
        if f.size >= 2 and f[1] - f[0] < 1e-5 * abs(f[0]) + 1e-3:
            n1 += 1
    s2 = np.sort(o["stage2"][np.isfinite(o["stage2"])])
    tie2 = bool(s2.size >= 2 and s2[1] - s2[0] < 1e-5 * abs(s2[0]) + 1e-3)
    return n1, tie2


@pytest.fixture(scope="module")
def c4_inputs(oracle):
    from paper_2509_17340_b200 import ControlInput, GoalSpec, State

    cloud, pose = forest_cycle_inputs(oracle, frames=20)
    cloud = cloud.astype(np.float32).astype(np.float64)
    x = State.from_array(pose)
    goal = GoalSpec.facing(tuple(pose[:3]), (45, 0, 2))
    prev = np.tile(np.array([9.81, 0.1, -0.05, 0.02]), (50, 1))
    la = ControlInput(10.2, (0.0, 0.1, 0.0))
    cfg = make_cfg(8, 8, K=8192, N=50)
    osnap = oracle.snapshot(cloud, pose, cfg.r_max)
    o = oracle.plan(osnap, oracle.config(cfg), pose, goal.p_goal, goal.v_goal, goal.q_goal, prev, la.vec(), 4, 9)
    assert o["rc"] == 0
    return cfg, cloud, pose, x, goal, prev, la, o


def _check_plan(r, o):
    valid = np.array([p.valid for p in r.per_instance])
    assert np.array_equal(valid, o["valid"].astype(bool))
    assert r.winner == o["winner"]
    assert rel(r.control.vec(), o["control"]) <= 1e-9
    st1 = np.array([p.stage1 for p in r.per_instance])
    st2 = np.array([p.stage2 for p in r.per_instance])
    assert rel(st1[valid], o["stage1"][valid]) <= 1e-9
    assert rel(st2[valid], o["stage2"][valid]) <= 1e-9
    assert rel([p.ess for p in r.per_instance], o["ess"]) <= 1e-7
    for m in np.flatnonzero(valid):
        assert rel(r.per_instance[m].nominal, o["nominal"][m]) <= 1e-9, m
    ij = np.array([[a.coarse_i, a.coarse_j] for a in r.anchors])
    assert np.array_equal(ij, o["anchor_ij"])


def test_c4_full_size_unsharded(c4_inputs, oracle):
    """64 x 8192 x 50 on one context: the bounded, lane-compacted FP32
    screening of 26.2 M rollout-steps, FP64 support refine, stage II."""
    from paper_2509_17340_b200 import Planner

    cfg, cloud, pose, x, goal, prev, la, o = c4_inputs
    with Planner(cfg, precision=32, max_points=1 << 16) as p:
        snap = p.build_snapshot(cloud, x, cfg.r_max)
        r = p.plan_step(x, goal, snap, prev, la, 4, 9, want_sample_costs=True)
    _check_plan(r, o)
    # every sample the oracle weights is screened within the FP32 tolerance or
    # provably outside the support (aborted / flagged lower bound)
    sc, osc = r.sample_costs, o["sample_costs"]
    aborted = sc >= 3.0e38
    rho = np.min(np.where(np.isfinite(osc), osc, np.inf), axis=1, keepdims=True)
    assert np.all((osc > rho + 64 * cfg.mppi.lambda_)[aborted])
    ok = np.isfinite(osc) & ~aborted & (o["sample_margin"] > 1e-3)
    assert rel(sc[ok], osc[ok]) <= 1e-4
    n1, tie2 = near_ties(o)
    print(f"C4 unsharded: {ok.sum()} samples checked, {aborted.sum()} aborted, near-ties: stage I {n1}/64 "
          f"instances, stage II {tie2}")


@pytest.mark.parametrize("G", [2, 4])
def test_c4_full_size_sharded(c4_inputs, oracle, G):
    """The same plan with the 8192 samples of every instance split over G
    shards (global sample index in the RNG key; all-reduce MIN of the FP32
    minimum, all-gather of the FP64 softmin partials, fixed-order merge)."""
    from paper_2509_17340_b200 import Planner
    from paper_2509_17340_b200.sharding import plan_step_sharded_local

    cfg, cloud, pose, x, goal, prev, la, o = c4_inputs
    planners = [Planner(cfg, precision=32, max_points=1 << 16) for _ in range(G)]
    try:
        snaps = [p.build_snapshot(cloud, x, cfg.r_max) for p in planners]
        outs = plan_step_sharded_local(planners, snaps, x, goal, prev, la, 4, 9)
    finally:
        for p in planners:
            p.close()
    for r in outs:
        _check_plan(r, o)


def _scan_1m(oracle, kind, seed, pose):
    sc = oracle.scene(kind, seed)
    frames, n, f = [], 0, 0
    while n < 1_000_000:
        fr = sc.lidar(pose, 5000 + f)
        frames.append(fr)
        n += fr.shape[0]
        f += 1
        assert f < 2000
    return np.concatenate(frames)[:1_000_000], f


@pytest.mark.parametrize("kind,seed,p", [(2, 7, (12.0, -2.0, 2.0)), (3, 5, (9.0, 1.0, 2.0))],
                         ids=["verticals", "inclines"])
def test_c3_full_plan_cycle_1m_points(oracle, kind, seed, p):
    """C3: snapshot of an accumulated ~1M-point scan (float32 coordinates)
    followed by a full plan cycle at C1 plan sizes (4x2 x 256 x 30)."""
    pose = np.array([*p, 1.0, 0.0, 0.0, 0.0, 2.5, 0.3, 0.0])
    cloud, frames = _scan_1m(oracle, kind, seed, pose)
    assert cloud.shape[0] == 1_000_000
    cfg = make_cfg(4, 2, K=256, N=30)
    prev = np.tile(np.array([9.81, 0.1, -0.05, 0.02]), (30, 1))
    r, o = run_case(oracle, cfg, cloud, pose, pose, goal_target=(45, 0, 2), previous=prev,
                    last_applied=np.array([10.2, 0.0, 0.1, 0.0]), cycle=100, seed=1, f64=False)
    from test_plan_parity import get_planner
    from test_snapshot_parity import check

    check(get_planner(cfg, 32), oracle, cloud, pose, f64=False)  # the 1M-point snapshot itself, bit-exact
    n1, tie2 = near_ties(o)
    print(f"C3 kind {kind}: {frames} frames, winner {r.winner}, near-ties: stage I {n1}/8, stage II {tie2}")
