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
