"""ctypes wrapper of the CPU oracle (oracle/oracle_capi.h) — TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import
this module, and only as the checker / the timed CPU baseline.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_LIB = os.path.join(ROOT, "oracle", "_build", "liboracle.so")
KAT_RUNNER = os.path.join(ROOT, "oracle", "_build", "kat_runner")

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int32)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_u64p = ctypes.POINTER(ctypes.c_uint64)


class OracleConfig(ctypes.Structure):
    """Mirrors amppi_config field for field (oracle_capi.h)."""

    _fields_ = [
        ("m_h", ctypes.c_int32), ("m_v", ctypes.c_int32),
        ("lookahead", ctypes.c_double), ("spacing_deg", ctypes.c_double),
        ("terminal_speed", ctypes.c_double), ("min_anchor_distance", ctypes.c_double),
        ("rollouts", ctypes.c_int32), ("horizon", ctypes.c_int32),
        ("lambda_", ctypes.c_double), ("sigma", ctypes.c_double * 4), ("mppi_dt", ctypes.c_double),
        ("iterations", ctypes.c_int32),
        ("q_track", ctypes.c_double), ("q_vnorm", ctypes.c_double), ("q_c", ctypes.c_double),
        ("q_c_delta", ctypes.c_double), ("q_p", ctypes.c_double), ("q_v", ctypes.c_double),
        ("q_q", ctypes.c_double),
        ("col_scale", ctypes.c_double), ("col_slope", ctypes.c_double),
        ("col_d_min", ctypes.c_double), ("col_d_max", ctypes.c_double),
        ("mass", ctypes.c_double), ("gravity", ctypes.c_double * 3), ("dyn_dt", ctypes.c_double),
        ("thrust_min", ctypes.c_double), ("thrust_max", ctypes.c_double),
        ("omega_xy_max", ctypes.c_double), ("omega_z_max", ctypes.c_double),
        ("replan_hz", ctypes.c_double), ("r_max", ctypes.c_double),
    ]


class OraclePlanOut(ctypes.Structure):
    _fields_ = [
        ("winner", _ip), ("control", _dp), ("stage1", _dp), ("stage2", _dp), ("ess", _dp), ("valid", _u8p),
        ("nominal", _dp), ("anchor_initial", _dp), ("anchor_refined", _dp), ("anchor_safe_dir", _dp),
        ("anchor_safe_range", _dp), ("anchor_ij", _ip), ("guide_coeffs", _dp), ("breakdown", _dp),
        ("winner_states", _dp), ("sample_costs", _dp), ("sample_margin", _dp),
    ]


def _p(a: np.ndarray, ct=ctypes.c_double):
    return a.ctypes.data_as(ctypes.POINTER(ct))


class Oracle:
    def __init__(self, path: str = ORACLE_LIB):
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make -C oracle`")
        L = ctypes.CDLL(path)
        vp = ctypes.c_void_p
        sig = {
            "oracle_config_default": (None, [ctypes.POINTER(OracleConfig)]),
            "oracle_set_workers": (None, [ctypes.c_uint]),
            "oracle_workers": (ctypes.c_uint, []),
            "oracle_snapshot_new": (vp, [_dp, ctypes.c_int64, _dp, ctypes.c_double]),
            "oracle_snapshot_free": (None, [vp]),
            "oracle_snapshot_filtered_count": (ctypes.c_int64, [vp]),
            "oracle_snapshot_get": (None, [vp, _dp, _u8p, _dp, _dp, _dp, _dp, _dp]),
            "oracle_snapshot_nearest": (ctypes.c_double, [vp, _dp]),
            "oracle_plan": (ctypes.c_int, [vp, ctypes.POINTER(OracleConfig), _dp, _dp, _dp, _dp, _dp, ctypes.c_int32,
                                           _dp, ctypes.c_uint64, ctypes.c_uint64, _dp, ctypes.POINTER(OraclePlanOut)]),
            "oracle_perturbations": (None, [ctypes.POINTER(OracleConfig), ctypes.c_uint64, ctypes.c_uint64,
                                            ctypes.c_uint64, ctypes.c_int32, _dp]),
            "oracle_goal_facing": (None, [_dp, _dp, _dp]),
            "oracle_scene_new": (vp, [ctypes.c_int32, ctypes.c_uint64]),
            "oracle_scene_free": (None, [vp]),
            "oracle_scene_obstacle_count": (ctypes.c_int64, [vp]),
            "oracle_lidar_scan": (ctypes.c_int64, [vp, _dp, ctypes.c_uint64, ctypes.c_double, _dp, ctypes.c_int64]),
            "oracle_true_clearance": (ctypes.c_double, [vp, _dp]),
            "oracle_loop_new": (vp, [ctypes.c_int32, ctypes.c_uint64, ctypes.POINTER(OracleConfig), ctypes.c_uint64,
                                     ctypes.c_int32]),
            "oracle_loop_run": (ctypes.c_int64, [vp, ctypes.c_int64]),
            "oracle_loop_status": (ctypes.c_int32, [vp]),
            "oracle_loop_records": (ctypes.c_int64, [vp]),
            "oracle_loop_cloud_size": (ctypes.c_int64, [vp, ctypes.c_int64]),
            "oracle_loop_get": (None, [vp, ctypes.c_int64, _dp, _dp, _dp, _ip, _dp, _u64p, _ip, _ip, _dp, _dp, _dp]),
            "oracle_loop_goal": (None, [vp, _dp, _dp, _dp]),
            "oracle_loop_state": (None, [vp, _dp]),
            "oracle_loop_free": (None, [vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        self.L = L

    # -- config --------------------------------------------------------------
    def config(self, base=None) -> OracleConfig:
        """OracleConfig from a planner.EnsembleConfig (or the defaults)."""
        c = OracleConfig()
        if base is None:
            self.L.oracle_config_default(ctypes.byref(c))
            return c
        ac = base.to_c()
        ctypes.memmove(ctypes.byref(c), ctypes.byref(ac), ctypes.sizeof(c))
        return c

    def set_workers(self, n: int) -> None:
        self.L.oracle_set_workers(n)

    # -- snapshot ------------------------------------------------------------
    def snapshot(self, pts: np.ndarray, pose: np.ndarray, r_max: float = 10.0) -> "OracleSnapshot":
        a = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        ps = np.ascontiguousarray(pose, dtype=np.float64)
        h = self.L.oracle_snapshot_new(_p(a), a.shape[0], _p(ps), r_max)
        return OracleSnapshot(self, h)

    # -- plan ----------------------------------------------------------------
    def plan(self, snap: "OracleSnapshot", cfg: OracleConfig, x, goal_p, goal_v, goal_q, previous=None,
             last_applied=None, cycle=0, seed=0, injected=None) -> dict:
        M, N, K = cfg.m_h * cfg.m_v, cfg.horizon, cfg.rollouts
        out = {
            "winner": np.zeros(1, dtype=np.int32), "control": np.zeros(4), "stage1": np.zeros(M),
            "stage2": np.zeros(M), "ess": np.zeros(M), "valid": np.zeros(M, dtype=np.uint8),
            "nominal": np.zeros((M, N, 4)), "anchor_initial": np.zeros((M, 3)), "anchor_refined": np.zeros((M, 3)),
            "anchor_safe_dir": np.zeros((M, 3)), "anchor_safe_range": np.zeros(M),
            "anchor_ij": np.zeros((M, 2), dtype=np.int32), "guide_coeffs": np.zeros((M, 3, 6)),
            "breakdown": np.zeros(5), "winner_states": np.zeros((N + 1, 10)), "sample_costs": np.zeros((M, K)),
            "sample_margin": np.zeros((M, K)),
        }
        o = OraclePlanOut()
        for k, arr in out.items():
            ct = {np.uint8: ctypes.c_uint8, np.int32: ctypes.c_int32}.get(arr.dtype.type, ctypes.c_double)
            setattr(o, k, _p(arr, ct))
        xs = np.ascontiguousarray(x, dtype=np.float64)
        gp = np.ascontiguousarray(goal_p, dtype=np.float64)
        gv = np.ascontiguousarray(goal_v, dtype=np.float64)
        gq = np.ascontiguousarray(goal_q, dtype=np.float64)
        la = np.ascontiguousarray(last_applied if last_applied is not None else [cfg.mass * 9.81, 0, 0, 0],
                                  dtype=np.float64)
        prev = None if previous is None else np.ascontiguousarray(previous, dtype=np.float64).reshape(-1, 4)
        inj = None if injected is None else np.ascontiguousarray(injected, dtype=np.float64)
        rc = self.L.oracle_plan(snap.h, ctypes.byref(cfg), _p(xs), _p(gp), _p(gv), _p(gq),
                                None if prev is None else _p(prev), 0 if prev is None else prev.shape[0],
                                _p(la), cycle, seed, None if inj is None else _p(inj), ctypes.byref(o))
        out["rc"] = rc
        out["winner"] = int(out["winner"][0]) if rc == 0 else -1
        return out

    def perturbations(self, cfg: OracleConfig, seed, instance, cycle, k) -> np.ndarray:
        out = np.zeros((cfg.horizon, 4))
        self.L.oracle_perturbations(ctypes.byref(cfg), seed, instance, cycle, k, _p(out))
        return out

    def goal_facing(self, frm, target) -> np.ndarray:
        q = np.zeros(4)
        self.L.oracle_goal_facing(_p(np.asarray(frm, dtype=np.float64)), _p(np.asarray(target, dtype=np.float64)),
                                  _p(q))
        return q

    # -- sim -----------------------------------------------------------------
    def scene(self, kind: int, seed: int) -> "OracleScene":
        return OracleScene(self, self.L.oracle_scene_new(kind, seed))

    def loop(self, kind: int, scene_seed: int, cfg: OracleConfig, seed: int, capacity: int = 10) -> "OracleLoop":
        return OracleLoop(self, self.L.oracle_loop_new(kind, scene_seed, ctypes.byref(cfg), seed, capacity), cfg)


class OracleSnapshot:
    def __init__(self, o: Oracle, h):
        self.o, self.h = o, h

    def __del__(self):
        try:
            self.o.L.oracle_snapshot_free(self.h)
        except Exception:
            pass

    def get(self) -> dict:
        n = self.o.L.oracle_snapshot_filtered_count(self.h)
        out = {"ranges": np.zeros(7200), "has_point": np.zeros(7200, dtype=np.uint8), "nearest": np.zeros((7200, 3)),
               "safe_range": np.zeros(200), "safe_dir": np.zeros((200, 3)), "safe_point": np.zeros((200, 3)),
               "filtered": np.zeros((max(n, 1), 3))}
        self.o.L.oracle_snapshot_get(self.h, _p(out["ranges"]), _p(out["has_point"], ctypes.c_uint8),
                                     _p(out["nearest"]), _p(out["safe_range"]), _p(out["safe_dir"]),
                                     _p(out["safe_point"]), _p(out["filtered"]))
        out["filtered"] = out["filtered"][:n]
        return out

    def nearest(self, p) -> float:
        return self.o.L.oracle_snapshot_nearest(self.h, _p(np.asarray(p, dtype=np.float64)))


class OracleScene:
    def __init__(self, o: Oracle, h):
        self.o, self.h = o, h

    def __del__(self):
        try:
            self.o.L.oracle_scene_free(self.h)
        except Exception:
            pass

    def lidar(self, pose: np.ndarray, frame_seed: int, r_max: float = 10.0) -> np.ndarray:
        cap = 7200
        out = np.zeros((cap, 3))
        n = self.o.L.oracle_lidar_scan(self.h, _p(np.asarray(pose, dtype=np.float64)), frame_seed, r_max, _p(out), cap)
        return out[:n].copy()

    def true_clearance(self, p) -> float:
        return self.o.L.oracle_true_clearance(self.h, _p(np.asarray(p, dtype=np.float64)))


class OracleLoop:
    def __init__(self, o: Oracle, h, cfg: OracleConfig):
        self.o, self.h, self.cfg = o, h, cfg

    def __del__(self):
        try:
            self.o.L.oracle_loop_free(self.h)
        except Exception:
            pass

    def run(self, cycles: int) -> int:
        return self.o.L.oracle_loop_run(self.h, cycles)

    def status(self) -> int:
        return self.o.L.oracle_loop_status(self.h)

    def state(self) -> np.ndarray:
        x = np.zeros(10)
        self.o.L.oracle_loop_state(self.h, _p(x))
        return x

    def goal(self):
        gp, gv, gq = np.zeros(3), np.zeros(3), np.zeros(4)
        self.o.L.oracle_loop_goal(self.h, _p(gp), _p(gv), _p(gq))
        return gp, gv, gq

    def records(self) -> list:
        N = self.cfg.horizon
        out = []
        for i in range(self.o.L.oracle_loop_records(self.h)):
            n = self.o.L.oracle_loop_cloud_size(self.h, i)
            r = {"cloud": np.zeros((max(n, 1), 3)), "x": np.zeros(10), "prev": np.zeros((N, 4)),
                 "prev_len": np.zeros(1, dtype=np.int32), "last_applied": np.zeros(4),
                 "cycle": np.zeros(1, dtype=np.uint64), "planned": np.zeros(1, dtype=np.int32),
                 "winner": np.zeros(1, dtype=np.int32), "control": np.zeros(4), "stage2": np.zeros(1),
                 "winner_nominal": np.zeros((N, 4))}
            self.o.L.oracle_loop_get(self.h, i, _p(r["cloud"]), _p(r["x"]), _p(r["prev"]),
                                     _p(r["prev_len"], ctypes.c_int32), _p(r["last_applied"]),
                                     _p(r["cycle"], ctypes.c_uint64), _p(r["planned"], ctypes.c_int32),
                                     _p(r["winner"], ctypes.c_int32), _p(r["control"]), _p(r["stage2"]),
                                     _p(r["winner_nominal"]))
            r["cloud"] = r["cloud"][:n]
            r["prev_len"] = int(r["prev_len"][0])
            r["cycle"] = int(r["cycle"][0])
            r["planned"] = bool(r["planned"][0])
            r["winner"] = int(r["winner"][0])
            r["stage2"] = float(r["stage2"][0])
            out.append(r)
        return out


# ---------------------------------------------------------------------------
# reference RNG (rng.hpp) vectorised, for regenerating the reference tests'
# seeded inputs (e.g. RandomStream(777) clouds of acceptance.cpp:155-161)
# ---------------------------------------------------------------------------
_G = np.uint64(0x9E3779B97F4A7C15)


def mix64(z: np.ndarray) -> np.ndarray:
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


class RandomStream:
    """RandomStream(key) with uniform draws only (counter-based, vectorised)."""

    def __init__(self, key: int):
        self.key = mix64(np.uint64(key) ^ _G)
        self.counter = 0

    def uniforms(self, n: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
        ctr = np.arange(self.counter + 1, self.counter + n + 1, dtype=np.uint64)
        self.counter += n
        with np.errstate(over="ignore"):
            u = mix64(self.key + ctr * _G)
        unit = (u >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
        return lo + (hi - lo) * unit


def random_cloud(rs: RandomStream, n: int, spread: float) -> np.ndarray:
    """random_cloud(rs, n, spread) of test_perception.cpp:46-53 (x, y, z drawn in order)."""
    return rs.uniforms(3 * n, -spread, spread).reshape(n, 3)
