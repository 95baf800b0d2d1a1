"""Probe of the d_max discontinuity: best sample grazing an obstacle point at
d_max (1 + eps); reports FP32 vs FP64 side and whether the plan still matches."""
import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from conftest import _ensure_oracle
_ensure_oracle()
from oracle_py import Oracle
from test_plan_parity import make_cfg, run_case, state
from test_dmax_boundary import _scenario
oracle = Oracle()
cfg, inj, x, far, traj = _scenario(oracle)
dmax = cfg.weights.collision.d_max
n = np.array([0.31, 0.83, 0.47]); n /= np.linalg.norm(n)
flips = fails = 0
for step in (6, 13, 22):
    p = traj[step, 0:3]
    for eps in np.linspace(-4e-7, 4e-7, 41):
        q = p + n * dmax * (1.0 + eps)
        d = np.linalg.norm(traj[:, 0:3] - q, axis=1)
        if not np.all(np.delete(d, step) > dmax * (1 + 1e-6)):
            continue
        try:
            r, o = run_case(oracle, cfg, np.vstack([q, far]), x, x, goal_target=(20, 0, 2), cycle=0, seed=1, injected=inj)
            ok = True
        except AssertionError as e:
            ok = False
            fails += 1
        if ok:
            s32, s64 = r.sample_costs[0][0] > 4e4, o["sample_costs"][0][0] > 4e4
            if s32 != s64:
                flips += 1
                print("flip", step, eps, r.sample_costs[0][0], o["sample_costs"][0][0])
        else:
            print("FAIL", step, eps)
print("flips", flips, "fails", fails)
