"""Multi-GPU decomposition of the plan cycle.

Scene sharding (config C5): independent scenes are split into contiguous,
balanced ranges, one per rank; every rank runs the whole cycle for its scenes
and no collective touches the data path.

Sample sharding (config C4): each rank owns a contiguous range of the K
samples of every instance and keeps the *global* sample index in the RNG key
(stream (seed, m, cycle*iters+iter, k), mppi.cpp:16-22), so its draws equal
the single-GPU run.  The MPPI update (compute_weights + update_nominal,
mppi.cpp:70-101) is decomposable with a log-sum-exp style rescaling: rank g
reports, per instance,

    m_g   = min_k S_k                               (its samples, +inf if none)
    eta_g = sum_k exp(-(S_k - m_g) / lambda)
    w2_g  = sum_k exp(-2 (S_k - m_g) / lambda)
    ed_g  = sum_k exp(-(S_k - m_g) / lambda) * delta_k     ([N, 4])

and after one all-gather every rank merges them in rank order:

    rho = min_g m_g,  a_g = exp(-(m_g - rho) / lambda)
    eta = sum_g a_g eta_g,  du = sum_g a_g ed_g / eta,  ess = eta^2 / sum_g a_g^2 w2_g

which equals the single-process result up to floating-point summation order.
"""
from __future__ import annotations

import math

import numpy as np


def shard_ranges(total: int, world: int) -> list[tuple[int, int]]:
    """Balanced contiguous [first, first+count) ranges, one per rank."""
    if world < 1:
        raise ValueError("world size must be positive")
    base, extra = divmod(total, world)
    out, first = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append((first, n))
        first += n
    return out


def softmin_partials(costs: np.ndarray, deltas: np.ndarray, lam: float):
    """Per-rank partials for one instance: costs [k], applied deltas [k, N, 4]."""
    fin = np.isfinite(costs)
    if not fin.any():
        return math.inf, 0.0, 0.0, np.zeros(deltas.shape[1:])
    m = float(np.min(costs[fin]))
    e = np.where(fin, np.exp(-(np.where(fin, costs, m) - m) / lam), 0.0)
    return m, float(e.sum()), float((e * e).sum()), np.tensordot(e, deltas, axes=(0, 0))


def merge_softmin(partials, lam: float):
    """Merge rank partials (in rank order) -> (rho, du [N,4], ess); raises
    RuntimeError("no valid rollout") like compute_weights when every rank is
    empty (mppi.cpp:75)."""
    rho = min(p[0] for p in partials)
    if not math.isfinite(rho):
        raise RuntimeError("no valid rollout")
    eta, w2 = 0.0, 0.0
    ed = np.zeros_like(partials[0][3])
    for m, eta_g, w2_g, ed_g in partials:
        if not math.isfinite(m):
            continue
        a = math.exp(-(m - rho) / lam)
        eta += a * eta_g
        w2 += a * a * w2_g
        ed = ed + a * ed_g
    return rho, ed / eta, eta * eta / w2


# ---------------------------------------------------------------------------
# Device path (amppi_shard_*): one planner per GPU, collectives on torch
# CUDA tensors.  The partial math above is what k_partials / k_merge compute.
# ---------------------------------------------------------------------------
class TorchComm:
    """torch.distributed collectives (NCCL on GPUs) for plan_step_sharded."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def allreduce_min(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)

    def allgather(self, out, t):
        try:
            self.dist.all_gather_into_tensor(out, t, group=self.group)
        except (RuntimeError, NotImplementedError):  # backends without the fused form (gloo on some builds)
            parts = list(out.chunk(self.world))
            self.dist.all_gather(parts, t, group=self.group)
            out.copy_(__import__("torch").cat(parts))


def plan_step_sharded(planner, x, goal, snap, previous, last_applied, cycle: int, seed: int, comm,
                      want_rollout: bool = True):
    """plan_step with this rank's share of the samples (config C4).

    Every rank calls it with the same inputs; each screens and refines samples
    shard_ranges(K, world)[rank] of every instance, and all ranks return the
    same PlanResult.  planner must launch on torch's current CUDA stream (the
    collectives are ordered on it)."""
    import torch

    cfg = planner.cfg
    M, K = cfg.grid.count(), cfg.mppi.rollouts
    k0, n = shard_ranges(K, comm.world)[comm.rank]
    if n == 0:
        raise ValueError("more shards than samples")
    stream = torch.cuda.current_stream()
    planner.set_stream(stream.cuda_stream)
    dev = stream.device
    stride = planner.shard_partials_stride()
    local_min = torch.empty(M, dtype=torch.float32, device=dev)
    partials = torch.empty(M * stride, dtype=torch.float64, device=dev)
    gathered = torch.empty(comm.world * M * stride, dtype=torch.float64, device=dev)
    planner.shard_begin(x, goal, snap, previous, last_applied, cycle, seed, k0, k0 + n)
    for it in range(cfg.mppi.iterations):
        planner.shard_screen(it, local_min.data_ptr())
        comm.allreduce_min(local_min)
        planner.shard_partials(it, local_min.data_ptr(), partials.data_ptr())
        comm.allgather(gathered, partials)
        planner.shard_update(it, gathered.data_ptr(), comm.world)
    return planner.shard_finish(want_rollout)


def plan_step_sharded_local(planners, snaps, x, goal, previous, last_applied, cycle: int, seed: int,
                            want_rollout: bool = True):
    """The same protocol run in one process over len(planners) contexts (one
    shard each, any devices): the collectives are plain tensor ops between
    phases.  Used to check the sharded path against the unsharded plan."""
    import torch

    G = len(planners)
    cfg = planners[0].cfg
    M, K = cfg.grid.count(), cfg.mppi.rollouts
    ranges = shard_ranges(K, G)
    stride = planners[0].shard_partials_stride()
    dev = torch.device("cuda", planners[0].device)
    mins = [torch.empty(M, dtype=torch.float32, device=dev) for _ in range(G)]
    parts = [torch.empty(M * stride, dtype=torch.float64, device=dev) for _ in range(G)]
    for p, sn, (k0, n) in zip(planners, snaps, ranges):
        p.shard_begin(x, goal, sn, previous, last_applied, cycle, seed, k0, k0 + n)
    for it in range(cfg.mppi.iterations):
        for p, lm in zip(planners, mins):
            p.shard_screen(it, lm.data_ptr())
            p.synchronize()
        gmin = torch.stack(mins).amin(dim=0).contiguous()
        torch.cuda.synchronize(dev)
        for p, pt in zip(planners, parts):
            p.shard_partials(it, gmin.data_ptr(), pt.data_ptr())
            p.synchronize()
        allp = torch.cat(parts).contiguous()
        torch.cuda.synchronize(dev)
        for p in planners:
            p.shard_update(it, allp.data_ptr(), G)
            p.synchronize()
    return [p.shard_finish(want_rollout) for p in planners]


# ---------------------------------------------------------------------------
# Native NCCL path (amppi_plan_sharded): the same protocol driven from C++,
# with a communicator created through the C ABI (amppi_nccl_*).
# ---------------------------------------------------------------------------
class NcclComm:
    """An NCCL communicator made by the library's own NCCL entry points.

    Rank 0 calls ``NcclComm.unique_id()`` and ships the 128 bytes to every
    rank (e.g. torch.distributed.broadcast_object_list); each rank then
    builds ``NcclComm(uid, rank, world, device)``."""

    def __init__(self, uid: bytes, rank: int, world: int, device: int):
        import ctypes

        from . import _abi

        self.lib = _abi.load()
        self.rank, self.world = rank, world
        buf = ctypes.create_string_buffer(bytes(uid), 128)
        h = ctypes.c_void_p()
        rc = self.lib.amppi_nccl_comm_init(ctypes.byref(h), world, buf, rank, device)
        if rc != _abi.AMPPI_OK:
            raise RuntimeError(f"amppi_nccl_comm_init failed ({rc})")
        self.h = h

    @staticmethod
    def unique_id() -> bytes:
        import ctypes

        from . import _abi

        buf = ctypes.create_string_buffer(128)
        rc = _abi.load().amppi_nccl_unique_id(buf)
        if rc != _abi.AMPPI_OK:
            raise RuntimeError(f"amppi_nccl_unique_id failed ({rc}): NCCL not loadable")
        return buf.raw

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.amppi_nccl_comm_destroy(self.h)
            self.h = None


def plan_step_sharded_native(planner, comm: NcclComm, x, goal, snap, previous, last_applied, cycle: int,
                             seed: int, want_rollout: bool = True):
    """plan_step_sharded with the collectives issued by the library itself
    (ncclAllReduce / ncclAllGather on the planner's stream)."""
    import ctypes

    if snap.planner is not planner or snap.generation != planner._gen:
        raise ValueError("snapshot does not belong to this planner's current device state")
    prev, prev_len = planner._prev(previous)
    bufs, r = planner._result_buffers(want_rollout, False)
    xs, gs, lc = x.to_c(), goal.to_c(), last_applied.to_c()
    from .planner import _ptr

    planner._check(planner.lib.amppi_plan_sharded(
        planner._h, comm.h, comm.rank, comm.world, ctypes.byref(xs), ctypes.byref(gs),
        None if prev is None else _ptr(prev, ctypes.c_double), prev_len, ctypes.byref(lc), ctypes.c_uint64(cycle),
        ctypes.c_uint64(seed), ctypes.byref(r)))
    return planner._make_result(r, bufs)
