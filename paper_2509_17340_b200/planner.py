"""Host-side mirror of the reference planner interface over the C-ABI.

Names, argument meaning and error behaviour follow the reference C++ API:

* ``EnsembleConfig`` and its nested ``AnchorGrid`` / ``MppiConfig`` /
  ``CostWeights`` / ``DynamicsParams``  (proj/include/amppi/ensemble.hpp:16-23,
  guidance.hpp:10-19, mppi.hpp:14-21, costs.hpp:13-29, types.hpp:40-53)
* ``State``, ``ControlInput``, ``GoalSpec.facing`` (types.hpp:18-38,
  costs.hpp:42-56)
* ``PointCloudBuffer`` (perception.hpp:39-55)
* ``Planner.build_snapshot`` == ``build_snapshot`` (perception.cpp:237-246)
* ``Planner.plan_step`` == ``plan_step`` (ensemble.cpp:29-179); raises
  ``PlanningFailed`` (a ``RuntimeError("planning failed")``) exactly where the
  reference throws (ensemble.cpp:158).

Every computation runs in the CUDA kernels behind libamppi_b200.so; this
module only marshals arguments.
"""
from __future__ import annotations

import ctypes
import math
from collections import deque
from collections.abc import Sequence as _SeqABC
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _abi

M_CELLS = 7200
M_COARSE = 200


# ---------------------------------------------------------------------------
# configuration (reference defaults = Table I)
# ---------------------------------------------------------------------------
@dataclass
class AnchorGrid:
    m_h: int = 5
    m_v: int = 3
    lookahead: float = 5.0
    spacing_deg: float = 18.0
    terminal_speed: float = 3.0
    min_anchor_distance: float = 0.5

    def count(self) -> int:
        return self.m_h * self.m_v


@dataclass
class MppiConfig:
    rollouts: int = 128
    horizon: int = 25
    lambda_: float = 0.1
    sigma: tuple = (1.0, 1.0, 1.0, 0.5)
    dt: float = 0.05
    iterations: int = 1


@dataclass
class CollisionParams:
    scale: float = 1.0e6
    slope: float = 5.0
    d_min: float = 0.4
    d_max: float = 1.0


@dataclass
class CostWeights:
    q_track: float = 15.0
    q_vnorm: float = 0.15
    q_c: float = 0.5
    q_c_delta: float = 0.5
    q_p: float = 3.0
    q_v: float = 0.25
    q_q: float = 1.0
    collision: CollisionParams = field(default_factory=CollisionParams)


@dataclass
class DynamicsParams:
    mass: float = 1.0
    gravity: tuple = (0.0, 0.0, -9.81)
    dt: float = 0.05
    thrust_min: float = 0.3
    thrust_max: float = 16.35
    omega_xy_max: float = 3.0
    omega_z_max: float = 2.0

    def hover(self) -> "ControlInput":
        g = self.gravity
        return ControlInput(self.mass * math.sqrt((g[0] * g[0] + g[1] * g[1]) + g[2] * g[2]), (0.0, 0.0, 0.0))


@dataclass
class EnsembleConfig:
    grid: AnchorGrid = field(default_factory=AnchorGrid)
    mppi: MppiConfig = field(default_factory=MppiConfig)
    weights: CostWeights = field(default_factory=CostWeights)
    dynamics: DynamicsParams = field(default_factory=DynamicsParams)
    replan_hz: float = 50.0
    r_max: float = 10.0

    def to_c(self) -> _abi.Config:
        c = _abi.Config()
        g, m, w, d = self.grid, self.mppi, self.weights, self.dynamics
        c.m_h, c.m_v = g.m_h, g.m_v
        c.lookahead, c.spacing_deg = g.lookahead, g.spacing_deg
        c.terminal_speed, c.min_anchor_distance = g.terminal_speed, g.min_anchor_distance
        c.rollouts, c.horizon, c.lambda_ = m.rollouts, m.horizon, m.lambda_
        for i in range(4):
            c.sigma[i] = m.sigma[i]
        c.mppi_dt, c.iterations = m.dt, m.iterations
        c.q_track, c.q_vnorm, c.q_c, c.q_c_delta = w.q_track, w.q_vnorm, w.q_c, w.q_c_delta
        c.q_p, c.q_v, c.q_q = w.q_p, w.q_v, w.q_q
        c.col_scale, c.col_slope = w.collision.scale, w.collision.slope
        c.col_d_min, c.col_d_max = w.collision.d_min, w.collision.d_max
        c.mass = d.mass
        for i in range(3):
            c.gravity[i] = d.gravity[i]
        c.dyn_dt = d.dt
        c.thrust_min, c.thrust_max = d.thrust_min, d.thrust_max
        c.omega_xy_max, c.omega_z_max = d.omega_xy_max, d.omega_z_max
        c.replan_hz, c.r_max = self.replan_hz, self.r_max
        return c


def apply_velocity_cap(cfg: EnsembleConfig, cap: float) -> EnsembleConfig:
    """metrics.cpp:74-81: rescale Q_vnorm by (ref/cap)^2, retarget terminal speed."""
    import copy

    if not cap > 0.0:
        return cfg
    out = copy.deepcopy(cfg)
    ref = cfg.grid.terminal_speed
    out.weights.q_vnorm = cfg.weights.q_vnorm * (ref / cap) * (ref / cap)
    out.grid.terminal_speed = cap
    return out


# ---------------------------------------------------------------------------
# value types
# ---------------------------------------------------------------------------
@dataclass
class State:
    p: tuple = (0.0, 0.0, 0.0)
    q: tuple = (1.0, 0.0, 0.0, 0.0)  # w, x, y, z
    v: tuple = (0.0, 0.0, 0.0)

    def to_c(self) -> _abi.State:
        s = _abi.State()
        s.p[:] = [float(x) for x in self.p]
        s.q[:] = [float(x) for x in self.q]
        s.v[:] = [float(x) for x in self.v]
        return s

    def as_array(self) -> np.ndarray:
        return np.array(list(self.p) + list(self.q) + list(self.v), dtype=np.float64)

    @staticmethod
    def from_array(a) -> "State":
        a = [float(x) for x in a]
        return State(tuple(a[0:3]), tuple(a[3:7]), tuple(a[7:10]))


@dataclass
class ControlInput:
    thrust: float = 0.0
    omega: tuple = (0.0, 0.0, 0.0)

    def to_c(self) -> _abi.Control:
        c = _abi.Control()
        c.thrust = float(self.thrust)
        c.omega[:] = [float(x) for x in self.omega]
        return c

    def vec(self) -> np.ndarray:
        return np.array([self.thrust, *self.omega], dtype=np.float64)


@dataclass
class GoalSpec:
    p_goal: tuple = (0.0, 0.0, 0.0)
    v_goal: tuple = (0.0, 0.0, 0.0)
    q_goal: tuple = (1.0, 0.0, 0.0, 0.0)

    @staticmethod
    def facing(frm, target) -> "GoalSpec":
        """Level attitude yawed toward the target (costs.hpp:47-55)."""
        d = [target[i] - frm[i] for i in range(3)]
        q = (1.0, 0.0, 0.0, 0.0)
        if d[0] * d[0] + d[1] * d[1] > 1e-12:
            ha = 0.5 * math.atan2(d[1], d[0])
            s = math.sin(ha)
            q = (math.cos(ha), s * 0.0, s * 0.0, s * 1.0)
        return GoalSpec(tuple(float(t) for t in target), (0.0, 0.0, 0.0), q)

    def to_c(self) -> _abi.Goal:
        g = _abi.Goal()
        g.p_goal[:] = [float(x) for x in self.p_goal]
        g.v_goal[:] = [float(x) for x in self.v_goal]
        g.q_goal[:] = [float(x) for x in self.q_goal]
        return g


class PointCloudBuffer:
    """Ring of world-frame frames, oldest evicted first (perception.cpp:44-62)."""

    def __init__(self, capacity: int = 10):
        self._frames: deque = deque()
        self._capacity = capacity

    def push(self, world_frame_points) -> None:
        self._frames.append(np.ascontiguousarray(np.asarray(world_frame_points, dtype=np.float64).reshape(-1, 3)))
        while len(self._frames) > self._capacity:
            self._frames.popleft()

    def frames(self) -> int:
        return len(self._frames)

    def capacity(self) -> int:
        return self._capacity

    def total_points(self) -> int:
        return sum(len(f) for f in self._frames)

    def points(self) -> np.ndarray:
        if not self._frames:
            return np.zeros((0, 3), dtype=np.float64)
        return np.concatenate(list(self._frames), axis=0)


class PlanningFailed(RuntimeError):
    def __init__(self):
        super().__init__("planning failed")


class AmppiError(RuntimeError):
    pass


@dataclass
class InstanceRecord:
    stage1: float
    stage2: float
    ess: float
    valid: bool
    nominal: Optional[np.ndarray]


@dataclass
class Anchor:
    initial_endpoint: np.ndarray
    refined_endpoint: np.ndarray
    safe_dir: np.ndarray
    safe_range: float
    coarse_i: int
    coarse_j: int


@dataclass
class CostBreakdown:
    track: float
    vnorm: float
    ctrl: float
    goal: float
    collision: float

    def stage2(self) -> float:
        return self.goal + self.collision

    def stage1(self) -> float:
        return self.track + self.vnorm + self.ctrl + self.stage2()


@dataclass
class PlanResult:
    winner: int
    control: ControlInput
    per_instance: Sequence  # [M] InstanceRecord (built on access)
    anchors: Sequence       # [M] Anchor (built on access)
    guides: np.ndarray  # [M, 3, 6]
    breakdown: CostBreakdown
    winner_states: Optional[np.ndarray] = None   # [N+1, 10]
    winner_controls: Optional[np.ndarray] = None  # [N, 4]
    sample_costs: Optional[np.ndarray] = None     # [M, K]


@dataclass
class PerceptionSnapshot:
    """Device-resident snapshot handle; ``download()`` copies it out."""

    planner: "Planner"
    pose: State
    r_max: float
    generation: int

    def download(self) -> dict:
        return self.planner.download_snapshot(self)


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(ctypes.POINTER(ctype))


class _Records(_SeqABC):
    """Read-only list of per-instance records built on first access: a plan
    with 64 instances otherwise spends ~0.3 ms of Python building records the
    caller mostly never reads (bench C4's closed loop reads one)."""

    def __init__(self, n: int, make):
        self._n, self._make, self._cache = n, make, {}

    def __len__(self) -> int:
        return self._n

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(self._n))]
        if i < 0:
            i += self._n
        if not 0 <= i < self._n:
            raise IndexError(i)
        r = self._cache.get(i)
        if r is None:
            r = self._cache[i] = self._make(i)
        return r

    def __repr__(self) -> str:
        return repr(list(self))


class Planner:
    """One amppi_ctx: device arenas + stream for one host thread."""

    def __init__(self, cfg: EnsembleConfig | None = None, *, device: int = 0, precision: int = 32,
                 max_points: int = 1 << 20, max_scenes: int = 1, profile: bool = False, stream: int | None = None,
                 refine_split_cap: int = -1, **schedule):
        """``schedule``: amppi_schedule fields (pipeline_chunks, pipeline_ratio,
        pipeline_streams, device_chunks, chunk_gather, loop_graph, trace);
        they change how calls are split over streams and chunks, never their
        results."""
        self.cfg = cfg or EnsembleConfig()
        self.lib = _abi.load()
        opt = _abi.Options()
        self.lib.amppi_options_default(ctypes.byref(opt))
        opt.device, opt.precision, opt.max_scenes = device, precision, max_scenes
        opt.max_points, opt.profile = max_points, 1 if profile else 0
        opt.stream = stream
        opt.refine_split_cap = refine_split_cap
        self._schedule = {}
        for k, v in schedule.items():
            if k not in dict(_abi.Schedule._fields_):
                raise TypeError(f"unknown schedule field {k!r}")
            setattr(opt.schedule, k, v)
            self._schedule[k] = v
        self._ccfg = self.cfg.to_c()
        h = ctypes.c_void_p()
        rc = self.lib.amppi_create(ctypes.byref(self._ccfg), ctypes.byref(opt), ctypes.byref(h))
        if rc != _abi.AMPPI_OK:
            raise AmppiError(f"amppi_create failed with status {rc}")
        self._h = h
        self._gen = 0
        self.precision = precision
        self.max_scenes = max_scenes
        self.device = device

    # -- lifecycle -------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "_h", None):
            self.lib.amppi_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _check(self, rc: int) -> None:
        if rc == _abi.AMPPI_OK:
            return
        if rc == _abi.AMPPI_PLANNING_FAILED:
            raise PlanningFailed()
        msg = self.lib.amppi_last_error(self._h).decode()
        if rc == _abi.AMPPI_INVALID_ARGUMENT:
            raise ValueError(msg)
        raise AmppiError(f"status {rc}: {msg}")

    # -- build_snapshot --------------------------------------------------
    def build_snapshot(self, buffer, pose: State, r_max: float = 10.0, *, f64: bool = False) -> PerceptionSnapshot:
        pts = buffer.points() if isinstance(buffer, PointCloudBuffer) else np.asarray(buffer)
        pts = pts.reshape(-1, 3)
        n = int(pts.shape[0])
        ps = pose.to_c()
        if f64:
            a = np.ascontiguousarray(pts, dtype=np.float64)
            rc = self.lib.amppi_snapshot_f64(self._h, _ptr(a, ctypes.c_double), n, ctypes.byref(ps), float(r_max))
        else:
            a = np.ascontiguousarray(pts, dtype=np.float32)
            rc = self.lib.amppi_snapshot(self._h, _ptr(a, ctypes.c_float), n, ctypes.byref(ps), float(r_max))
        self._check(rc)
        self._gen += 1
        return PerceptionSnapshot(self, pose, float(r_max), self._gen)

    def download_snapshot(self, snap: PerceptionSnapshot) -> dict:
        if snap.generation != self._gen:
            raise ValueError("stale snapshot: a newer build_snapshot replaced it on the device")
        out = {
            "ranges": np.zeros(M_CELLS), "has_point": np.zeros(M_CELLS, dtype=np.uint8),
            "nearest": np.zeros((M_CELLS, 3)), "safe_range": np.zeros(M_COARSE),
            "safe_dir": np.zeros((M_COARSE, 3)), "safe_point": np.zeros((M_COARSE, 3)),
            "filtered": np.zeros((M_CELLS, 3)),
        }
        v = _abi.SnapshotView()
        v.ranges = _ptr(out["ranges"], ctypes.c_double)
        v.has_point = _ptr(out["has_point"], ctypes.c_uint8)
        v.nearest = _ptr(out["nearest"], ctypes.c_double)
        v.safe_range = _ptr(out["safe_range"], ctypes.c_double)
        v.safe_dir = _ptr(out["safe_dir"], ctypes.c_double)
        v.safe_point = _ptr(out["safe_point"], ctypes.c_double)
        v.filtered = _ptr(out["filtered"], ctypes.c_double)
        self._check(self.lib.amppi_snapshot_download(self._h, ctypes.byref(v)))
        out["filtered"] = out["filtered"][: v.n_filtered].copy()
        return out

    # -- plan_step -------------------------------------------------------
    def plan_step(self, x: State, goal: GoalSpec, snap: PerceptionSnapshot, previous=None,
                  last_applied: ControlInput | None = None, cycle: int = 0, seed: int = 0, *,
                  injected_delta: np.ndarray | None = None, want_rollout: bool = True,
                  want_sample_costs: bool = False) -> PlanResult:
        if snap.planner is not self or snap.generation != self._gen:
            raise ValueError("snapshot does not belong to this planner's current device state")
        cfg = self.cfg
        M, N, K = cfg.grid.count(), cfg.mppi.horizon, cfg.mppi.rollouts
        la = last_applied if last_applied is not None else cfg.dynamics.hover()
        prev, prev_len = self._prev(previous)
        bufs, r = self._result_buffers(want_rollout, want_sample_costs)
        inj = None
        if injected_delta is not None:
            inj = np.ascontiguousarray(injected_delta, dtype=np.float64)
            expect = cfg.mppi.iterations * M * K * N * 4
            if inj.size != expect:
                raise ValueError(f"injected_delta must hold {expect} values")
        xs, gs, lc = x.to_c(), goal.to_c(), la.to_c()
        rc = self.lib.amppi_plan(self._h, ctypes.byref(xs), ctypes.byref(gs),
                                 None if prev is None else _ptr(prev, ctypes.c_double), prev_len,
                                 ctypes.byref(lc), ctypes.c_uint64(cycle), ctypes.c_uint64(seed),
                                 None if inj is None else _ptr(inj, ctypes.c_double), ctypes.byref(r))
        self._check(rc)
        return self._make_result(r, bufs)

    @staticmethod
    def _prev(previous):
        prev = None if previous is None else np.ascontiguousarray(np.asarray(previous, dtype=np.float64).reshape(-1, 4))
        return prev, (0 if prev is None else int(prev.shape[0]))

    def _result_buffers(self, want_rollout: bool, want_sample_costs: bool):
        cfg = self.cfg
        M, N, K = cfg.grid.count(), cfg.mppi.horizon, cfg.mppi.rollouts
        bufs = {
            "stage1": np.zeros(M), "stage2": np.zeros(M), "ess": np.zeros(M), "valid": np.zeros(M, dtype=np.uint8),
            "nominal": np.zeros((M, N, 4)), "anchor_initial": np.zeros((M, 3)), "anchor_refined": np.zeros((M, 3)),
            "anchor_safe_dir": np.zeros((M, 3)), "anchor_safe_range": np.zeros(M),
            "anchor_ij": np.zeros((M, 2), dtype=np.int32), "guide_coeffs": np.zeros((M, 3, 6)),
        }
        r = _abi.PlanResult()
        for k, arr in bufs.items():
            ct = {np.uint8: ctypes.c_uint8, np.int32: ctypes.c_int32}.get(arr.dtype.type, ctypes.c_double)
            setattr(r, k, _ptr(arr, ct))
        if want_rollout:
            bufs["winner_states"] = np.zeros((N + 1, 10))
            bufs["winner_controls"] = np.zeros((N, 4))
            r.winner_states = _ptr(bufs["winner_states"], ctypes.c_double)
            r.winner_controls = _ptr(bufs["winner_controls"], ctypes.c_double)
        if want_sample_costs:
            bufs["sample_costs"] = np.zeros((M, K))
            r.sample_costs = _ptr(bufs["sample_costs"], ctypes.c_double)
        return bufs, r

    def _make_result(self, r, bufs) -> PlanResult:
        M = self.cfg.grid.count()
        # bufs are this call's own arrays, so records may view them
        per = _Records(M, lambda m: InstanceRecord(float(bufs["stage1"][m]), float(bufs["stage2"][m]),
                                                   float(bufs["ess"][m]), bool(bufs["valid"][m]),
                                                   bufs["nominal"][m] if bufs["valid"][m] else None))
        anchors = _Records(M, lambda m: Anchor(bufs["anchor_initial"][m], bufs["anchor_refined"][m],
                                               bufs["anchor_safe_dir"][m], float(bufs["anchor_safe_range"][m]),
                                               int(bufs["anchor_ij"][m, 0]), int(bufs["anchor_ij"][m, 1])))
        return PlanResult(
            winner=int(r.winner),
            control=ControlInput(r.control.thrust, tuple(r.control.omega)),
            per_instance=per, anchors=anchors, guides=bufs["guide_coeffs"],
            breakdown=CostBreakdown(*[float(v) for v in r.breakdown]),
            winner_states=bufs.get("winner_states"), winner_controls=bufs.get("winner_controls"),
            sample_costs=bufs.get("sample_costs"),
        )

    # -- sample-sharded plan_step (C4) -------------------------------------
    # Phase calls of amppi_shard_* (include/amppi_b200.h); device buffers are
    # raw CUDA pointers (e.g. torch tensor .data_ptr()) used on the planner's
    # stream.  sharding.plan_step_sharded drives them.
    def shard_begin(self, x: State, goal: GoalSpec, snap: PerceptionSnapshot, previous, last_applied: ControlInput,
                    cycle: int, seed: int, k_begin: int, k_end: int) -> None:
        if snap.planner is not self or snap.generation != self._gen:
            raise ValueError("snapshot does not belong to this planner's current device state")
        prev, prev_len = self._prev(previous)
        xs, gs, lc = x.to_c(), goal.to_c(), last_applied.to_c()
        self._check(self.lib.amppi_shard_begin(self._h, ctypes.byref(xs), ctypes.byref(gs),
                                               None if prev is None else _ptr(prev, ctypes.c_double), prev_len,
                                               ctypes.byref(lc), ctypes.c_uint64(cycle), ctypes.c_uint64(seed),
                                               int(k_begin), int(k_end)))

    def shard_screen(self, it: int, local_min_ptr: int) -> None:
        self._check(self.lib.amppi_shard_screen(self._h, it, ctypes.c_void_p(local_min_ptr)))

    def shard_partials(self, it: int, global_min_ptr: int, partials_ptr: int) -> None:
        self._check(self.lib.amppi_shard_partials(self._h, it, ctypes.c_void_p(global_min_ptr),
                                                  ctypes.c_void_p(partials_ptr)))

    def shard_update(self, it: int, all_partials_ptr: int, n_shards: int) -> None:
        self._check(self.lib.amppi_shard_update(self._h, it, ctypes.c_void_p(all_partials_ptr), n_shards))

    def shard_finish(self, want_rollout: bool = True) -> PlanResult:
        bufs, r = self._result_buffers(want_rollout, False)
        self._check(self.lib.amppi_shard_finish(self._h, ctypes.byref(r)))
        return self._make_result(r, bufs)

    def shard_partials_stride(self) -> int:
        return int(self.lib.amppi_shard_partials_stride(self._h))

    # -- batched scenes (C5) ---------------------------------------------
    def cycle_batch(self, offsets: np.ndarray, xyz: np.ndarray, poses: np.ndarray, states: np.ndarray,
                    goals: np.ndarray, last_applied: np.ndarray, cycles: np.ndarray, seeds: np.ndarray,
                    previous: np.ndarray | None = None, r_max: float = 10.0) -> dict:
        """Snapshot + plan for S independent scenes from host arrays.

        poses/states: [S,10]; goals: [S,10] (p, v, q); last_applied: [S,4];
        previous: [S,N,4] or None (hover warm start)."""
        bi, arrs, out, bo = self._batch_structs(offsets, xyz, poses, states, goals, last_applied, cycles, seeds,
                                                previous, r_max)
        self._gen += 1  # the batch overwrites the single-scene snapshot slot
        self._check(self.lib.amppi_cycle_batch(self._h, ctypes.byref(bi), ctypes.byref(bo)))
        return out

    def cycle_batch_submit(self, offsets: np.ndarray, xyz: np.ndarray, poses: np.ndarray, states: np.ndarray,
                           goals: np.ndarray, last_applied: np.ndarray, cycles: np.ndarray, seeds: np.ndarray,
                           previous: np.ndarray | None = None, r_max: float = 10.0) -> int:
        """Streaming form (amppi_cycle_batch_submit): queue the batch and return
        a ticket; up to three batches in flight, so the next batch's upload
        overlaps this one's planning.  xyz should be pinned memory (e.g. a
        torch pin_memory() tensor's numpy view) for the copy to be asynchronous."""
        bi, arrs, out, bo = self._batch_structs(offsets, xyz, poses, states, goals, last_applied, cycles, seeds,
                                                previous, r_max)
        t = ctypes.c_int64()
        self._gen += 1
        self._check(self.lib.amppi_cycle_batch_submit(self._h, ctypes.byref(bi), ctypes.byref(t)))
        self._inflight = getattr(self, "_inflight", {})
        self._inflight[int(t.value)] = (arrs, out, bo)  # the host arrays must outlive the upload
        return int(t.value)

    def cycle_batch_wait(self, ticket: int) -> dict:
        arrs, out, bo = self._inflight.pop(ticket)
        self._check(self.lib.amppi_cycle_batch_wait(self._h, ticket, ctypes.byref(bo)))
        return out

    def _batch_structs(self, offsets, xyz, poses, states, goals, last_applied, cycles, seeds, previous, r_max):
        S = int(len(offsets) - 1)
        N, M = self.cfg.mppi.horizon, self.cfg.grid.count()
        off = np.asarray(offsets)
        if S < 1 or off[0] != 0 or np.any(np.diff(off) < 0):
            raise ValueError("offsets must start at 0 and be non-decreasing, with at least one scene")
        if np.asarray(xyz).reshape(-1, 3).shape[0] != int(off[-1]):
            raise ValueError(f"xyz holds {np.asarray(xyz).reshape(-1, 3).shape[0]} points, offsets[-1] = {off[-1]}")
        for name, a, w in (("poses", poses, 10), ("states", states, 10), ("goals", goals, 10),
                           ("last_applied", last_applied, 4)):
            if np.asarray(a).shape != (S, w):
                raise ValueError(f"{name} must have shape ({S}, {w})")
        for name, a in (("cycles", cycles), ("seeds", seeds)):
            if np.asarray(a).shape != (S,):
                raise ValueError(f"{name} must have shape ({S},)")
        if previous is not None and np.asarray(previous).shape != (S, N, 4):
            raise ValueError(f"previous must have shape ({S}, {N}, 4)")
        arrs = dict(
            offsets=np.ascontiguousarray(offsets, dtype=np.int64), xyz=np.ascontiguousarray(xyz, dtype=np.float32),
            poses=np.ascontiguousarray(poses, dtype=np.float64), states=np.ascontiguousarray(states, dtype=np.float64),
            goals=np.ascontiguousarray(goals, dtype=np.float64),
            last=np.ascontiguousarray(last_applied, dtype=np.float64),
            cycles=np.ascontiguousarray(cycles, dtype=np.uint64), seeds=np.ascontiguousarray(seeds, dtype=np.uint64))
        bi = _abi.BatchInput()
        bi.n_scenes = S
        bi.point_offsets = _ptr(arrs["offsets"], ctypes.c_int64)
        bi.xyz = _ptr(arrs["xyz"], ctypes.c_float)
        bi.poses = arrs["poses"].ctypes.data
        bi.states = arrs["states"].ctypes.data
        bi.goals = arrs["goals"].ctypes.data
        bi.last_applied = arrs["last"].ctypes.data
        bi.cycles = _ptr(arrs["cycles"], ctypes.c_uint64)
        bi.seeds = _ptr(arrs["seeds"], ctypes.c_uint64)
        if previous is not None:
            arrs["prev"] = np.ascontiguousarray(previous, dtype=np.float64)
            bi.previous = _ptr(arrs["prev"], ctypes.c_double)
        bi.r_max = float(r_max)
        out = dict(status=np.zeros(S, dtype=np.int32), winner=np.zeros(S, dtype=np.int32),
                   control=np.zeros((S, 4)), winner_nominal=np.zeros((S, N, 4)), stage2=np.zeros((S, M)),
                   breakdown=np.zeros((S, 5)))
        bo = _abi.BatchOutput()
        bo.status = _ptr(out["status"], ctypes.c_int32)
        bo.winner = _ptr(out["winner"], ctypes.c_int32)
        bo.control = _ptr(out["control"], ctypes.c_double)
        bo.winner_nominal = _ptr(out["winner_nominal"], ctypes.c_double)
        bo.stage2 = _ptr(out["stage2"], ctypes.c_double)
        bo.breakdown = _ptr(out["breakdown"], ctypes.c_double)
        return bi, arrs, out, bo

    def cycle_batch_device(self, dev: dict, out: dict, n_scenes: int, r_max: float = 10.0) -> None:
        """Same cycle on device-resident inputs (dict of raw device pointers,
        e.g. torch tensors' data_ptr()); enqueued on the planner's stream."""
        bi = self._device_batch_input(dev, n_scenes, r_max)
        bo = _abi.BatchOutput()
        for k, ct in (("status", ctypes.c_int32), ("winner", ctypes.c_int32), ("control", ctypes.c_double),
                      ("winner_nominal", ctypes.c_double), ("stage2", ctypes.c_double),
                      ("breakdown", ctypes.c_double)):
            if out.get(k):
                setattr(bo, k, ctypes.cast(ctypes.c_void_p(out[k]), ctypes.POINTER(ct)))
        self._gen += 1  # the batch overwrites the single-scene snapshot slot
        self._check(self.lib.amppi_cycle_batch_device(self._h, ctypes.byref(bi), ctypes.byref(bo)))

    DRIFT_KEYS = ("rollouts", "max_pos_diff", "max_clearance_diff", "steps_compared", "dmax_side_violations",
                  "flagged_steps", "max_rel_cost_diff", "validity_mismatches")

    def screen_drift(self, dev: dict, n_scenes: int, iteration: int = 0, sample_stride: int = 1) -> dict:
        """FP32-screening vs FP64 drift of the batch cycle_batch_device just
        planned on `dev` (amppi_screen_drift; verification only)."""
        bi = self._device_batch_input(dev, n_scenes, 10.0)
        st = np.zeros(8)
        self._check(self.lib.amppi_screen_drift(self._h, ctypes.byref(bi), int(iteration), int(sample_stride),
                                                _ptr(st, ctypes.c_double)))
        return {k: (float(v) if k.startswith("max") else int(v)) for k, v in zip(self.DRIFT_KEYS, st)}

    @staticmethod
    def _device_batch_input(dev: dict, n_scenes: int, r_max: float):
        bi = _abi.BatchInput()
        bi.n_scenes = n_scenes
        bi.point_offsets = ctypes.cast(ctypes.c_void_p(dev["offsets"]), _abi.c_int64_p)
        bi.xyz = ctypes.cast(ctypes.c_void_p(dev["xyz"]), _abi.c_float_p)
        bi.poses = dev["poses"]
        bi.states = dev["states"]
        bi.goals = dev["goals"]
        bi.last_applied = dev["last"]
        bi.cycles = ctypes.cast(ctypes.c_void_p(dev["cycles"]), _abi.c_uint64_p)
        bi.seeds = ctypes.cast(ctypes.c_void_p(dev["seeds"]), _abi.c_uint64_p)
        if dev.get("prev"):
            bi.previous = ctypes.cast(ctypes.c_void_p(dev["prev"]), _abi.c_double_p)
        bi.r_max = float(r_max)
        return bi

    def synchronize(self) -> None:
        self._check(self.lib.amppi_synchronize(self._h))

    def set_schedule(self, **fields) -> None:
        """Replace schedule fields (unnamed ones keep their current value)."""
        for k in fields:
            if k not in dict(_abi.Schedule._fields_):
                raise TypeError(f"unknown schedule field {k!r}")
        self._schedule.update(fields)
        sch = _abi.Schedule()
        for k, v in self._schedule.items():
            setattr(sch, k, v)
        self._check(self.lib.amppi_set_schedule(self._h, ctypes.byref(sch)))

    def set_config(self, cfg: EnsembleConfig) -> None:
        """plan_step takes cfg per call (ensemble.hpp:59-63): weights, dynamics
        and sampling parameters may change between calls; sizes may not."""
        c = cfg.to_c()
        self._check(self.lib.amppi_set_config(self._h, ctypes.byref(c)))
        if cfg.weights.collision.d_max != self.cfg.weights.collision.d_max:
            self._gen += 1  # the snapshot's collision grid was sized for the old d_max
        self.cfg, self._ccfg = cfg, c

    def set_stream(self, stream: int) -> None:
        self._check(self.lib.amppi_set_stream(self._h, ctypes.c_void_p(stream)))

    def kernel_times(self) -> dict:
        cap = 64
        names = (ctypes.c_char_p * cap)()
        ms = np.zeros(cap)
        launches = np.zeros(cap, dtype=np.int64)
        count = ctypes.c_int32()
        self._check(self.lib.amppi_kernel_times(self._h, names, _ptr(ms, ctypes.c_double),
                                                _ptr(launches, ctypes.c_int64), cap, ctypes.byref(count)))
        return {names[i].decode(): (float(ms[i]), int(launches[i])) for i in range(min(count.value, cap))}

    def kernel_times_reset(self) -> None:
        self._check(self.lib.amppi_kernel_times_reset(self._h))


class ClosedLoop:
    """GPU-resident closed loop (amppi_loop_*): execute_cycle
    (ensemble.cpp:245-305) with the LiDAR, the point-cloud ring and the vehicle
    on the device.  Uses the planner's configuration and stream."""

    STATUS = {0: "running", 1: "success", 2: "collision", 3: "timeout", 4: "planner_failure"}

    def __init__(self, planner: Planner, scene_kind: int, scene_seed: int, seed: int, buffer_capacity: int = 10,
                 max_cycles: int = 4096):
        self.planner = planner
        self.lib = planner.lib
        h = ctypes.c_void_p()
        planner._check(self.lib.amppi_loop_create(planner._h, scene_kind, ctypes.c_uint64(scene_seed),
                                                  ctypes.c_uint64(seed), buffer_capacity, max_cycles,
                                                  ctypes.byref(h)))
        self._h = h

    def run(self, cycles: int) -> int:
        self.planner._gen += 1  # the loop overwrites the single-scene snapshot slot
        ran = ctypes.c_int64()
        self.planner._check(self.lib.amppi_loop_run(self._h, cycles, ctypes.byref(ran)))
        return int(ran.value)

    def records(self) -> list:
        n = ctypes.c_int64()
        self.planner._check(self.lib.amppi_loop_records(self._h, None, 0, ctypes.byref(n)))
        buf = (_abi.LoopRecord * max(int(n.value), 1))()
        self.planner._check(self.lib.amppi_loop_records(self._h, buf, int(n.value), ctypes.byref(n)))
        return [dict(cycle=int(r.cycle), planned=bool(r.planned), winner=int(r.winner), x=np.array(r.x[:]),
                     control=np.array(r.control[:]), stage2=float(r.stage2), status=int(r.status),
                     n_points=int(r.n_points), t=float(r.t), x_after=np.array(r.x_after[:]),
                     clearance=float(r.clearance), breakdown=np.array(r.breakdown[:]))
                for r in buf[: int(n.value)]]

    def metrics(self) -> dict:
        """EpisodeMetrics (metrics.hpp:11-18) computed on the device log."""
        m = _abi.EpisodeMetrics()
        self.planner._check(self.lib.amppi_loop_metrics(self._h, ctypes.byref(m)))
        return {k: float(getattr(m, k)) for k, _ in _abi.EpisodeMetrics._fields_}

    def trajectory_csv(self) -> str:
        """The episode as the reference's TrajectoryLog CSV (# amppi-trajectory v1,
        %.17g; ensemble.cpp:192-230)."""
        lines = ["# amppi-trajectory v1",
                 "t,px,py,pz,vx,vy,vz,qw,qx,qy,qz,thrust,wx,wy,wz,winner,stage2,"
                 "clearance,j_track,j_vnorm,j_ctrl,j_goal,j_col"]
        for r in self.records():
            x = r["x_after"]
            vals = [r["t"], x[0], x[1], x[2], x[7], x[8], x[9], x[3], x[4], x[5], x[6], *r["control"]]
            row = ",".join("%.17g" % v for v in vals) + ",%d," % r["winner"]
            row += ",".join("%.17g" % v for v in [r["stage2"], r["clearance"], *r["breakdown"]])
            lines.append(row)
        return "\n".join(lines) + "\n"

    def state(self):
        x = np.zeros(10)
        st = ctypes.c_int32()
        t = ctypes.c_double()
        self.planner._check(self.lib.amppi_loop_state(self._h, _ptr(x, ctypes.c_double), ctypes.byref(st),
                                                      ctypes.byref(t)))
        return x, self.STATUS.get(int(st.value), str(st.value)), float(t.value)

    def close(self) -> None:
        if self._h:
            self.lib.amppi_loop_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
