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
