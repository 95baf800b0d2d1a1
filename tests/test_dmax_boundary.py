"""The collision term jumps at d_max (C exp(-a (d_max - d_min)) -> 0), so an
FP32 screening distance on the wrong side of d_max would change a sample's
FP32 cost by ~5e4 while its FP64 cost does not move.  The screening flags
steps within a band of d_max and keeps a lower-bound cost for the sample,
which k_support admits by that bound.  Here the best sample (zero
perturbation, every other sample far worse) passes a single obstacle point
at d_max (1 + eps), |eps| from 3e-8 to 1e-3 (in and past the band): the FP64 result must
equal the oracle's for every eps (contract of test_plan_parity), and the
flagged screening cost must bound the FP64 one from below."""
import numpy as np
import pytest

from test_plan_parity import make_cfg, run_case, state

pytestmark = pytest.mark.gpu


def _scenario(oracle):
    cfg = make_cfg(1, 1, K=64, N=30)
    rs = np.random.default_rng(4)
    inj = rs.normal(size=(1, 1, 64, 30, 4)) * np.array([1.0, 1.0, 1.0, 0.5]) * 2.0
    inj[0, 0, 0] = 0.0  # sample 0 flies the nominal exactly
    x = state((0.0, 0.0, 2.0), v=(2.0, 0.0, 0.0))
    far = np.array([[60.0, 40.0, 2.0]])
    _, o = run_case(oracle, cfg, far, x, x, goal_target=(20, 0, 2), cycle=0, seed=1, injected=inj)
    assert o["ess"][0] < 1.001  # sample 0 carries the whole softmin weight
    return cfg, inj, x, far, o["winner_states"]


@pytest.mark.parametrize("step", [8, 17])
def test_best_sample_grazes_d_max(oracle, step):
    cfg, inj, x, far, traj = _scenario(oracle)
    dmax = cfg.weights.collision.d_max
    p = traj[step, 0:3]
    for eps in (-1e-3, -3e-7, -1e-7, -3e-8, 0.0, 3e-8, 1e-7, 2e-7, 3e-7, 1e-3):
        q = p + np.array([0.0, 1.0, 0.0]) * dmax * (1.0 + eps)
        # every other step of sample 0 stays clear of the point
        d = np.linalg.norm(traj[:, 0:3] - q, axis=1)
        assert np.all(np.delete(d, step) > dmax * (1 + 1e-6))
        r, o = run_case(oracle, cfg, np.vstack([q, far]), x, x, goal_target=(20, 0, 2), cycle=0, seed=1,
                        injected=inj)
        assert r.sample_costs[0][0] <= o["sample_costs"][0][0] * (1 + 1e-4)


def test_every_sample_flagged(oracle):
    """All samples fly the same (zero-perturbation) trajectory past a point at
    d_max (1 + 1e-7): every screening cost is flagged, so k_support has no
    unflagged minimum and admits every finite sample; the FP64 refine then
    decides, as in the oracle."""
    cfg, inj, x, far, traj = _scenario(oracle)
    zero = np.zeros_like(inj)
    dmax = cfg.weights.collision.d_max
    q = traj[12, 0:3] + np.array([0.0, 1.0, 0.0]) * dmax * (1.0 + 1e-7)
    r, o = run_case(oracle, cfg, np.vstack([q, far]), x, x, goal_target=(20, 0, 2), cycle=0, seed=1, injected=zero)
    assert np.all(r.sample_costs[0] <= o["sample_costs"][0] * (1 + 1e-4))
