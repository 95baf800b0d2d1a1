"""Sample-sharded plan_step (config C4; amppi_shard_*, sharding.py) against
the unsharded device plan and the CPU oracle.

The shards run in one process on one GPU (plan_step_sharded_local: one
context per shard, the all-reduce / all-gather as tensor ops between phases),
which exercises every kernel of the multi-GPU protocol; results must not
depend on the shard count beyond FP64 summation order (<= 1e-12)."""
import numpy as np
import pytest

from test_plan_parity import forest_cycle_inputs, make_cfg, rel, run_case

pytestmark = pytest.mark.gpu


def _inputs(oracle):
    from paper_2509_17340_b200 import ControlInput, GoalSpec, State

    cloud, pose = forest_cycle_inputs(oracle, frames=20)
    x = State.from_array(pose)
    goal = GoalSpec.facing(tuple(pose[:3]), (45, 0, 2))
    prev = np.tile(np.array([9.81, 0.1, -0.05, 0.02]), (30, 1))
    return cloud, pose, x, goal, prev, ControlInput(10.2, (0.0, 0.1, 0.0))


def _sharded(cfg, cloud, x, goal, prev, la, G, cycle, seed):
    from paper_2509_17340_b200 import Planner
    from paper_2509_17340_b200.sharding import plan_step_sharded_local

    planners = [Planner(cfg, precision=32, max_points=1 << 16) for _ in range(G)]
    try:
        snaps = [p.build_snapshot(cloud, x, cfg.r_max) for p in planners]
        return plan_step_sharded_local(planners, snaps, x, goal, prev, la, cycle, seed)
    finally:
        for p in planners:
            p.close()


def _same(a, b, tol):
    assert a.winner == b.winner
    assert rel(a.control.vec(), b.control.vec()) <= tol
    for pa, pb in zip(a.per_instance, b.per_instance):
        assert pa.valid == pb.valid
        if pa.valid:
            assert rel(pa.stage1, pb.stage1) <= tol
            assert rel(pa.stage2, pb.stage2) <= tol
            assert rel(pa.ess, pb.ess) <= 1e-9
            assert rel(pa.nominal, pb.nominal) <= tol


@pytest.mark.parametrize("G,iterations", [(1, 1), (2, 1), (3, 2), (4, 1)])
def test_shards_equal_unsharded(oracle, G, iterations):
    """Small instances: each shard screens in the single-pass mode."""
    from paper_2509_17340_b200 import Planner

    cfg = make_cfg(4, 4, K=512, N=30, iterations=iterations)
    cloud, pose, x, goal, prev, la = _inputs(oracle)
    ref_planner = Planner(cfg, precision=32, max_points=1 << 16)
    try:
        snap = ref_planner.build_snapshot(cloud, x, cfg.r_max)
        ref = ref_planner.plan_step(x, goal, snap, prev, la, 21, 5)
    finally:
        ref_planner.close()
    outs = _sharded(cfg, cloud, x, goal, prev, la, G, 21, 5)
    for o in outs:
        _same(o, ref, 1e-12)


def test_c4_shape_two_shards_vs_oracle(oracle):
    """C4 shape (8x8 anchors) at K = 4096: each of 2 shards runs the bounded,
    lane-compacted screening on its 2048 samples; the merged plan matches the
    oracle's unsharded plan_step."""
    cfg = make_cfg(8, 8, K=4096, N=30)
    cloud, pose, x, goal, prev, la = _inputs(oracle)
    outs = _sharded(cfg, cloud, x, goal, prev, la, 2, 4, 9)
    osnap = oracle.snapshot(cloud.astype(np.float32).astype(np.float64), pose, cfg.r_max)
    o = oracle.plan(osnap, oracle.config(cfg), pose, goal.p_goal, goal.v_goal, goal.q_goal, prev, la.vec(), 4, 9)
    for r in outs:
        assert r.winner == o["winner"]
        assert rel(r.control.vec(), o["control"]) <= 1e-9
        st1 = np.array([p.stage1 for p in r.per_instance])
        valid = np.array([p.valid for p in r.per_instance])
        assert np.array_equal(valid, o["valid"].astype(bool))
        assert rel(st1[valid], o["stage1"][valid]) <= 1e-9
        for m in np.flatnonzero(valid):
            assert rel(r.per_instance[m].nominal, o["nominal"][m]) <= 1e-9


def test_native_nccl_single_rank_equals_unsharded(oracle):
    """amppi_plan_sharded through a 1-rank NCCL communicator made by the C ABI
    (amppi_nccl_unique_id / amppi_nccl_comm_init): the NCCL all-reduce and
    all-gather run on the context stream and the result equals plan_step."""
    from paper_2509_17340_b200 import Planner
    from paper_2509_17340_b200.sharding import NcclComm, plan_step_sharded_native

    cfg = make_cfg(8, 8, K=1024, N=30, iterations=2)
    cloud, pose, x, goal, prev, la = _inputs(oracle)
    comm = NcclComm(NcclComm.unique_id(), 0, 1, 0)
    try:
        with Planner(cfg, precision=32, max_points=1 << 16) as p:
            snap = p.build_snapshot(cloud, x, cfg.r_max)
            ref = p.plan_step(x, goal, snap, prev, la, 21, 5)
            nat = plan_step_sharded_native(p, comm, x, goal, snap, prev, la, 21, 5)
    finally:
        comm.close()
    _same(nat, ref, 1e-12)
