"""World-size-2 (gloo, CPU) tests of the multi-rank decomposition
(paper_2509_17340_b200/sharding.py):

* scene sharding: the rank ranges partition the batch; each rank plans its
  scenes (CPU oracle standing in for the device planner on this GPU-less
  host) and an all-gather reassembles exactly the single-process results;
* sample sharding: per-rank softmin partials over disjoint sample ranges,
  all-gathered and merged in rank order, reproduce the single-process
  compute_weights + update_nominal result of the oracle (mppi.cpp:70-101).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_17340_b200.sharding import merge_softmin, shard_ranges, softmin_partials


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def test_shard_ranges_partition():
    for total in (0, 1, 7, 4096, 4097):
        for world in (1, 2, 3, 8):
            r = shard_ranges(total, world)
            assert len(r) == world
            assert sum(n for _, n in r) == total
            assert all(r[i][0] + r[i][1] == r[i + 1][0] for i in range(world - 1))
            assert max(n for _, n in r) - min(n for _, n in r) <= 1


def _scene_worker(rank, world, port, out):
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__))))
    from oracle_py import Oracle
    from test_plan_parity import make_cfg, wall_cloud

    _init(rank, world, port)
    orc = Oracle()
    orc.set_workers(1)
    cfg = make_cfg(2, 2, K=16, N=10)
    ocfg = orc.config(cfg)
    S = 6
    first, n = shard_ranges(S, world)[rank]
    local = torch.zeros(S, 5, dtype=torch.float64)  # winner, control(4)
    for s in range(first, first + n):
        x = np.array([0, 0.3 * s, 2, 1, 0, 0, 0, 1.0, 0, 0], dtype=np.float64)
        snap = orc.snapshot(wall_cloud(), x, 10.0)
        o = orc.plan(snap, ocfg, x, [20, 0, 2], [0, 0, 0], [1, 0, 0, 0], None, [9.81, 0, 0, 0], 3, 100 + s)
        local[s, 0] = o["winner"]
        local[s, 1:] = torch.from_numpy(o["control"])
    dist.all_reduce(local)  # disjoint scene rows: the sum is the gather
    if rank == 0:
        out.put(local.numpy())
    dist.destroy_process_group()


def test_scene_sharding_gloo(oracle):
    from test_plan_parity import make_cfg, wall_cloud

    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_scene_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = make_cfg(2, 2, K=16, N=10)
    ocfg = oracle.config(cfg)
    for s in range(6):
        x = np.array([0, 0.3 * s, 2, 1, 0, 0, 0, 1.0, 0, 0], dtype=np.float64)
        snap = oracle.snapshot(wall_cloud(), x, 10.0)
        o = oracle.plan(snap, ocfg, x, [20, 0, 2], [0, 0, 0], [1, 0, 0, 0], None, [9.81, 0, 0, 0], 3, 100 + s)
        assert got[s, 0] == o["winner"]
        assert np.array_equal(got[s, 1:], o["control"])


def _sample_worker(rank, world, port, costs, deltas, lam, out):
    _init(rank, world, port)
    first, n = shard_ranges(costs.shape[0], world)[rank]
    m, eta, w2, ed = softmin_partials(costs[first:first + n], deltas[first:first + n], lam)
    N = deltas.shape[1]
    mine = torch.tensor([m, eta, w2] + list(np.asarray(ed).ravel()), dtype=torch.float64)
    gathered = [torch.zeros(3 + N * 4, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gathered, mine)
    parts = [(float(t[0]), float(t[1]), float(t[2]), t[3:].numpy().reshape(N, 4)) for t in gathered]
    rho, du, ess = merge_softmin(parts, lam)
    if rank == 0:
        out.put((rho, du, ess))
    dist.destroy_process_group()


@pytest.mark.parametrize("spread", [30.0, 0.3])
def test_sample_sharding_merge_gloo(oracle, spread):
    """Costs with a realistic (one-hot) and a flat (many-sample) softmin."""
    rs = np.random.default_rng(7)
    K, N, lam = 64, 12, 0.1
    costs = 5000.0 + spread * rs.random(K)
    costs[5] = np.inf  # an invalid rollout
    deltas = rs.normal(size=(K, N, 4))
    # single-process reference: compute_weights + weighted sum (mppi.cpp:70-101)
    fin = np.isfinite(costs)
    rho = costs[fin].min()
    w = np.where(fin, np.exp(-(np.where(fin, costs, rho) - rho) / lam), 0.0)
    w = w / w.sum()
    du_ref = np.tensordot(w, deltas, axes=(0, 0))
    ess_ref = 1.0 / (w * w).sum()
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_sample_worker, args=(r, world, port, costs, deltas, lam, q)) for r in range(world)]
    for p in procs:
        p.start()
    rho_m, du_m, ess_m = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert rho_m == rho
    assert np.max(np.abs(du_m - du_ref)) <= 1e-12
    assert abs(ess_m - ess_ref) <= 1e-9 * ess_ref


def test_merge_raises_when_every_rank_is_empty():
    e = (np.inf, 0.0, 0.0, np.zeros((3, 4)))
    with pytest.raises(RuntimeError, match="no valid rollout"):
        merge_softmin([e, e], 0.1)


# ---------------------------------------------------------------------------
# the same decompositions with the device planner: two processes on cuda:0,
# host-side gloo collectives (on CUDA tensors for the sample-sharded plan);
# no kernel waits on another process, so sharing one GPU is safe
# ---------------------------------------------------------------------------
def _device_sample_worker(rank, world, port, out):
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__))))
    from test_sample_sharding import _inputs

    from oracle_py import Oracle
    from paper_2509_17340_b200 import Planner
    from paper_2509_17340_b200.sharding import TorchComm, plan_step_sharded
    from test_plan_parity import make_cfg

    _init(rank, world, port)
    torch.cuda.set_device(0)
    cfg = make_cfg(8, 8, K=2048, N=30, iterations=2)
    cloud, pose, x, goal, prev, la = _inputs(Oracle())
    with Planner(cfg, precision=32, max_points=1 << 16) as p:
        snap = p.build_snapshot(cloud, x, cfg.r_max)
        r = plan_step_sharded(p, x, goal, snap, prev, la, 13, 4, TorchComm())
    out.put((rank, r.winner, r.control.vec(), [pi.stage1 for pi in r.per_instance],
             [pi.nominal if pi.valid else None for pi in r.per_instance]))
    dist.destroy_process_group()


@pytest.mark.gpu
def test_sample_sharded_plan_two_ranks_gloo_device(oracle):
    """plan_step_sharded through a real torch.distributed communicator
    (TorchComm over gloo, CUDA tensors), 2 ranks x 1024 samples per instance:
    both ranks return the unsharded plan."""
    from paper_2509_17340_b200 import Planner
    from test_plan_parity import make_cfg, rel
    from test_sample_sharding import _inputs

    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_device_sample_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    cfg = make_cfg(8, 8, K=2048, N=30, iterations=2)
    cloud, pose, x, goal, prev, la = _inputs(oracle)
    with Planner(cfg, precision=32, max_points=1 << 16) as p:
        snap = p.build_snapshot(cloud, x, cfg.r_max)
        ref = p.plan_step(x, goal, snap, prev, la, 13, 4)
    for rank, winner, control, st1, nominal in got:
        assert winner == ref.winner
        assert rel(control, ref.control.vec()) <= 1e-12
        assert rel(st1, [pi.stage1 for pi in ref.per_instance]) <= 1e-12
        for m, pi in enumerate(ref.per_instance):
            if pi.valid:
                assert rel(nominal[m], pi.nominal) <= 1e-12


def _device_scene_worker(rank, world, port, out):
    _init(rank, world, port)
    from paper_2509_17340_b200 import Planner
    from paper_2509_17340_b200.workloads import plan_config, scenes

    S = 300
    first, n = shard_ranges(S, world)[rank]
    d = scenes(n, points=20000, frames=20, first=first)
    cfg = plan_config()
    with Planner(cfg, max_scenes=n, max_points=int(d["offsets"][-1])) as p:
        r = p.cycle_batch(d["offsets"], d["xyz"], d["poses"], d["states"], d["goals"], d["last"], d["cycles"],
                          d["seeds"])
    local = torch.zeros(S, 5, dtype=torch.float64)
    local[first:first + n, 0] = torch.from_numpy(r["winner"].astype(np.float64))
    local[first:first + n, 1:] = torch.from_numpy(r["control"])
    dist.all_reduce(local)  # disjoint rows
    if rank == 0:
        out.put(local.numpy())
    dist.destroy_process_group()


@pytest.mark.gpu
def test_scene_sharded_batch_two_ranks_gloo_device():
    """C5 scene sharding with the device planner: 2 ranks plan halves of a
    300-scene batch; the gathered results equal one process planning it all
    (scenes are a function of their id, so a rank's shard is the batch's)."""
    from paper_2509_17340_b200 import Planner
    from paper_2509_17340_b200.workloads import plan_config, scenes

    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_device_scene_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    d = scenes(300, points=20000, frames=20, first=0)
    with Planner(plan_config(), max_scenes=300, max_points=int(d["offsets"][-1])) as p:
        r = p.cycle_batch(d["offsets"], d["xyz"], d["poses"], d["states"], d["goals"], d["last"], d["cycles"],
                          d["seeds"])
    assert np.array_equal(got[:, 0].astype(np.int32), r["winner"])
    assert np.array_equal(got[:, 1:], r["control"])
