"""GPU parity of plan_step (anchors, guides, stage-I MPPI updates, stage II,
selection) against the CPU oracle on identical inputs.

Contract:
  * bit-exact: anchor coarse cells (I, J), validity flags, the winner index;
  * FP64 values (anchors, guides): <= 1e-12 relative;
  * returned plan values (stage1/stage2/ess/nominal/control/breakdown) come
    from FP64 kernels in both precision modes: <= 1e-9 relative/absolute.
    They differ from the oracle only through libm last-ulp differences of
    exp/log/sin/cos in the perturbation and collision terms;
  * FP32 screening costs (per sample): <= 1e-4 relative, except samples whose
    clearance passes within 1e-4 m of a collision-branch boundary.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def wall_cloud():  # test_ensemble.cpp:15-21
    pts = []
    y = -3.0
    while y <= 0.5:
        z = 0.5
        while z <= 3.5:
            pts.append((4.0, y, z))
            z += 0.12
        y += 0.08
    return np.array(pts)


def make_cfg(m_h=5, m_v=3, K=128, N=25, iterations=1, cap=None):
    from paper_2509_17340_b200 import EnsembleConfig, apply_velocity_cap

    cfg = EnsembleConfig()
    cfg.grid.m_h, cfg.grid.m_v = m_h, m_v
    cfg.mppi.rollouts, cfg.mppi.horizon, cfg.mppi.iterations = K, N, iterations
    if cap:
        cfg = apply_velocity_cap(cfg, cap)
    return cfg


_planners = {}


def get_planner(cfg, precision):
    from paper_2509_17340_b200 import Planner

    key = (repr(cfg), precision)
    if key not in _planners:
        _planners[key] = Planner(cfg, precision=precision, max_points=1 << 20)
    return _planners[key]


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return np.max(np.abs(a - b) / np.maximum(1.0, np.abs(b))) if a.size else 0.0


def run_case(oracle, cfg, pts, pose, x, goal_target=None, goal=None, previous=None, last_applied=None, cycle=0,
             seed=0, precision=32, injected=None, f64=True, expect_fail=False):
    from paper_2509_17340_b200 import ControlInput, GoalSpec, PlanningFailed, State

    pts = np.asarray(pts, dtype=np.float64).reshape(-1, 3)
    if not f64:
        pts = pts.astype(np.float32).astype(np.float64)
    if goal is None:
        goal = GoalSpec.facing(tuple(x[:3]), goal_target)
    la = last_applied if last_applied is not None else cfg.dynamics.hover().vec()
    planner = get_planner(cfg, precision)
    snap = planner.build_snapshot(pts, State.from_array(pose), cfg.r_max, f64=f64)
    osnap = oracle.snapshot(pts, pose, cfg.r_max)
    ocfg = oracle.config(cfg)
    o = oracle.plan(osnap, ocfg, x, goal.p_goal, goal.v_goal, goal.q_goal, previous, la, cycle, seed, injected)
    if expect_fail:
        assert o["rc"] == 1
        with pytest.raises(PlanningFailed):
            planner.plan_step(State.from_array(x), goal, snap, previous, ControlInput(la[0], tuple(la[1:])), cycle,
                              seed, injected_delta=injected)
        return None, o
    assert o["rc"] == 0
    r = planner.plan_step(State.from_array(x), goal, snap, previous, ControlInput(la[0], tuple(la[1:])), cycle, seed,
                          injected_delta=injected, want_sample_costs=True)
    M = cfg.grid.count()
    # anchors / guides
    ij = np.array([[a.coarse_i, a.coarse_j] for a in r.anchors])
    assert np.array_equal(ij, o["anchor_ij"]), "anchor coarse cells"
    assert rel([a.initial_endpoint for a in r.anchors], o["anchor_initial"]) <= 1e-12
    assert rel([a.refined_endpoint for a in r.anchors], o["anchor_refined"]) <= 1e-12
    assert rel([a.safe_dir for a in r.anchors], o["anchor_safe_dir"]) <= 1e-12
    assert rel([a.safe_range for a in r.anchors], o["anchor_safe_range"]) == 0.0
    assert rel(r.guides, o["guide_coeffs"]) <= 1e-11
    # per instance
    valid = np.array([p.valid for p in r.per_instance])
    assert np.array_equal(valid, o["valid"].astype(bool)), "valid flags"
    st1 = np.array([p.stage1 for p in r.per_instance])
    st2 = np.array([p.stage2 for p in r.per_instance])
    ess = np.array([p.ess for p in r.per_instance])
    assert rel(st1, o["stage1"]) <= 1e-9, (st1, o["stage1"])
    fin = np.isfinite(o["stage2"])
    assert np.array_equal(np.isfinite(st2), fin)
    assert rel(st2[fin], o["stage2"][fin]) <= 1e-9
    assert rel(ess, o["ess"]) <= 1e-7
    for m in range(M):
        if valid[m]:
            assert rel(r.per_instance[m].nominal, o["nominal"][m]) <= 1e-9, m
    assert r.winner == o["winner"], "winner"
    assert rel(r.control.vec(), o["control"]) <= 1e-9
    bd = [r.breakdown.track, r.breakdown.vnorm, r.breakdown.ctrl, r.breakdown.goal, r.breakdown.collision]
    assert rel(bd, o["breakdown"]) <= 1e-9
    assert rel(r.winner_states, o["winner_states"]) <= 1e-9
    # screening costs; FP32 screening may stop a sample early (reported as
    # FLT_MAX) only when it provably lies outside the softmin support
    sc, osc, margin = r.sample_costs, o["sample_costs"], o["sample_margin"]
    aborted = sc >= 3.0e38
    if aborted.any():
        assert precision == 32
        rho = np.min(np.where(np.isfinite(osc), osc, np.inf), axis=1, keepdims=True)
        assert np.all((osc > rho + 64 * cfg.mppi.lambda_)[aborted]), "an aborted sample was in the support"
    fin = np.isfinite(osc) & ~aborted
    assert np.array_equal(np.isfinite(sc) & ~aborted, fin)
    # samples whose clearance comes within the d_max band are flagged by the
    # screening and report a lower bound (device_math.cuh screen_collision)
    ok = fin & (margin > 1e-3)
    assert np.all(sc[fin] <= osc[fin] * (1 + 1e-4) + 1e-2)
    tol = 1e-4 if precision == 32 else 1e-11
    assert rel(sc[ok], osc[ok]) <= tol
    return r, o


IDENT = np.array([0, 0, 0, 1, 0, 0, 0, 0, 0, 0], dtype=np.float64)


def state(p, v=(0, 0, 0), q=(1, 0, 0, 0)):
    return np.array(list(p) + list(q) + list(v), dtype=np.float64)


@pytest.mark.parametrize("precision", [32, 64])
def test_single_instance_equals_plain_mppi(oracle, precision):
    """test_ensemble.cpp:32-76 configuration (M=1, K=32, seed 77, cycle 5)."""
    cfg = make_cfg(1, 1, K=32)
    x = state((0, 0, 2))
    r, o = run_case(oracle, cfg, np.zeros((0, 3)), x, x, goal_target=(20, 0, 2), cycle=5, seed=77,
                    precision=precision)
    assert r.winner == 0


@pytest.mark.parametrize("precision", [32, 64])
def test_blocked_corridor_winner(oracle, precision):
    """test_ensemble.cpp:78-98: the free-side instance (1) must win."""
    cfg = make_cfg(2, 1, K=64)
    x = state((0, 0, 2), v=(2.0, 0, 0))
    r, o = run_case(oracle, cfg, wall_cloud(), x, x, goal_target=(20, 0, 2), cycle=0, seed=3, precision=precision)
    assert r.winner == 1
    assert r.per_instance[0].stage2 > r.per_instance[1].stage2


@pytest.mark.parametrize("precision", [32, 64])
def test_stage2_chain_over_cycles(oracle, precision):
    """test_ensemble.cpp:127-153: 5 cycles feeding the winner nominal back."""
    cfg = make_cfg(5, 3, K=32)
    x = state((0, 0, 2))
    prev = None
    for cycle in range(5):
        r, o = run_case(oracle, cfg, wall_cloud(), x, x, goal_target=(25, -3, 2), previous=prev, cycle=cycle,
                        seed=31, precision=precision)
        prev = o["nominal"][o["winner"]]


def test_paper_default_grid_on_cell_boundaries(oracle):
    """5x3 anchors straight at the goal sit exactly on
    18-degree boundaries; (I, J) must be 8..12 x 4..6 like the oracle."""
    cfg = make_cfg(5, 3, K=32)
    x = state((0, 0, 2))
    r, o = run_case(oracle, cfg, np.zeros((0, 3)), x, x, goal_target=(45, 0, 2))
    ij = sorted({(a.coarse_i, a.coarse_j) for a in r.anchors})
    assert ij == sorted((i, j) for i in range(8, 13) for j in range(4, 7))


@pytest.mark.parametrize("precision", [32, 64])
def test_injected_perturbations(oracle, precision):
    cfg = make_cfg(4, 2, K=64, N=30)
    rs = np.random.default_rng(123)
    inj = rs.normal(size=(1, 8, 64, 30, 4)) * np.array([1.0, 1.0, 1.0, 0.5])
    x = state((1.0, 0.5, 2.0), v=(1.5, 0.2, 0.0))
    run_case(oracle, cfg, wall_cloud() + np.array([1.0, 0.0, 0.0]), x, x, goal_target=(30, 2, 2), cycle=9,
             seed=5, precision=precision, injected=inj)


@pytest.mark.parametrize("precision", [32, 64])
def test_two_iterations(oracle, precision):
    cfg = make_cfg(3, 2, K=64, N=20, iterations=2)
    x = state((0, 0, 2), v=(1.0, 0, 0))
    run_case(oracle, cfg, wall_cloud(), x, x, goal_target=(20, 4, 3), cycle=3, seed=11, precision=precision)


def test_near_goal_hold_branch(oracle):
    cfg = make_cfg(4, 2, K=64)
    x = state((5.0, 1.0, 2.0), v=(0.3, 0, 0))
    r, o = run_case(oracle, cfg, wall_cloud(), x, x, goal_target=(5.2, 1.1, 2.1), cycle=1, seed=2)
    assert all(np.allclose(a.refined_endpoint, (5.2, 1.1, 2.1)) for a in r.anchors)


def test_planning_failed_raises(oracle):
    cfg = make_cfg(2, 1, K=16)
    x = state((0, 0, 2))
    x[7] = float("nan")  # non-finite velocity: every rollout invalid
    run_case(oracle, cfg, wall_cloud(), IDENT, x, goal_target=(20, 0, 2), expect_fail=True)


def forest_cycle_inputs(oracle, frames=24):
    """C1: forest seed 1 scan accumulated into exactly 20k float32 points."""
    pose = state((10.0, 1.5, 2.0), v=(3.0, 0.2, 0.0))
    sc = oracle.scene(1, 1)
    cloud = np.concatenate([sc.lidar(pose, 1000 + f) for f in range(frames)])[:20000]
    return cloud, pose


@pytest.mark.parametrize("precision", [32, 64])
def test_c1_forest_cycle(oracle, precision):
    """BASELINE config 1: 8 anchors (4x2) x 256 samples x 30 steps on a 20k forest scan."""
    cfg = make_cfg(4, 2, K=256, N=30)
    cloud, pose = forest_cycle_inputs(oracle)
    prev = np.tile(np.array([9.81, 0.1, -0.05, 0.02]), (30, 1))
    run_case(oracle, cfg, cloud, pose, pose, goal_target=(45, 0, 2), previous=prev,
             last_applied=np.array([10.2, 0.0, 0.1, 0.0]), cycle=100, seed=1, precision=precision, f64=False)


@pytest.mark.parametrize("path", ["latency", "throughput"])
def test_far_from_world_origin(oracle, path):
    """The same forest cycle translated 8 km / 4 km from the world origin,
    where an FP32 world coordinate's ulp (1e-3 m) is five times the d_max band:
    the FP32 screening runs in the snapshot pose's local frame (to_local_f),
    so its costs keep their accuracy and the plan still matches the oracle."""
    off = np.array([8192.0, -4096.0, 0.0])
    cloud, pose = forest_cycle_inputs(oracle)
    cloud = np.asarray(cloud, dtype=np.float32).astype(np.float64) + off  # exact in FP64
    pose = pose.copy()
    pose[:3] += off
    prev = np.tile(np.array([9.81, 0.1, -0.05, 0.02]), (30, 1))
    cfg = make_cfg(4, 2, K=256, N=30) if path == "latency" else make_cfg(8, 8, K=2048, N=30)
    run_case(oracle, cfg, cloud, pose, pose, goal_target=tuple(np.array([45.0, 0.0, 2.0]) + off), previous=prev,
             last_applied=np.array([10.2, 0.0, 0.1, 0.0]), cycle=100, seed=1, f64=True)


def test_large_ensemble_shape(oracle):
    """C4 shape (8x8 anchors, N=50) at a reduced K the oracle finishes quickly."""
    cfg = make_cfg(8, 8, K=512, N=50)
    cloud, pose = forest_cycle_inputs(oracle, frames=20)
    run_case(oracle, cfg, cloud, pose, pose, goal_target=(45, 0, 2), cycle=4, seed=9, f64=False)


def test_throughput_screening_path(oracle):
    """S*M*K >= 148*128*4 with K > 64 selects the bounded, lane-compacted FP32
    screening (k_stage1_f32_bound + k_stage1_f32c); per-sample costs checked."""
    cfg = make_cfg(8, 8, K=2048, N=30)
    cloud, pose = forest_cycle_inputs(oracle, frames=20)
    prev = np.tile(np.array([9.81, 0.1, -0.05, 0.02]), (30, 1))
    run_case(oracle, cfg, cloud, pose, pose, goal_target=(45, 0, 2), previous=prev, cycle=7, seed=3, f64=False)


def test_refine_overflow_path(oracle, monkeypatch):
    """Support pairs beyond the split-refine scratch take the fused FP64
    re-rollout (k_refine); forced here with a 5-pair split capacity."""
    from paper_2509_17340_b200 import Planner

    cfg = make_cfg(4, 2, K=256, N=30)
    planner = Planner(cfg, precision=32, max_points=1 << 20, refine_split_cap=5)
    key = (repr(cfg), 32)
    saved = _planners.get(key)
    _planners[key] = planner
    try:
        cloud, pose = forest_cycle_inputs(oracle)
        run_case(oracle, cfg, cloud, pose, pose, goal_target=(45, 0, 2), cycle=11, seed=2, f64=False)
    finally:
        planner.close()
        if saved is not None:
            _planners[key] = saved
        else:
            _planners.pop(key)


def test_screening_is_deterministic(oracle):
    """Race evidence without compute-sanitizer (closed on this pool): the
    lane-compacted main pass repacks live samples through shared memory
    under block barriers every 10 steps, and the bound pass, the support and
    the refine use atomics; repeated plans of the same inputs must give the
    same bits for every per-sample screening cost and every returned value."""
    from paper_2509_17340_b200 import ControlInput, GoalSpec, Planner, State

    cfg = make_cfg(8, 8, K=2048, N=30)
    cloud, pose = forest_cycle_inputs(oracle, frames=20)
    x = State.from_array(pose)
    goal = GoalSpec.facing(tuple(pose[:3]), (45, 0, 2))
    prev = np.tile(np.array([9.81, 0.1, -0.05, 0.02]), (30, 1))
    runs = []
    with Planner(cfg, precision=32, max_points=1 << 16) as p:
        for _ in range(4):
            snap = p.build_snapshot(cloud, x, cfg.r_max)
            r = p.plan_step(x, goal, snap, prev, ControlInput(10.2, (0.0, 0.1, 0.0)), 7, 3, want_sample_costs=True)
            runs.append(r)
    for r in runs[1:]:
        assert np.array_equal(r.sample_costs.view(np.uint64), runs[0].sample_costs.view(np.uint64))
        assert r.winner == runs[0].winner
        assert np.array_equal(r.control.vec(), runs[0].control.vec())
        for a, b in zip(r.per_instance, runs[0].per_instance):
            assert a.stage1 == b.stage1 and a.ess == b.ess
