"""BASELINE config 2 (C2): a 200-cycle synthetic forest flight at 7 m/s goal
speed with 4x2 anchors x 256 samples x 30 steps.  The oracle drives the loop
(execute_cycle, ensemble.cpp:245-305) and records every cycle's exact inputs;
the GPU path re-plans each recorded cycle through the C-ABI (snapshot from the
recorded buffer, same state / previous nominal / last control / cycle / seed)
and must select the same instance with the same control (SURVEY.md §8d
replay protocol)."""
import numpy as np
import pytest

from test_plan_parity import make_cfg, rel

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("precision", [32])
def test_forest_flight_replay(oracle, precision):
    from paper_2509_17340_b200 import ControlInput, GoalSpec, Planner, PlanningFailed, State

    cfg = make_cfg(4, 2, K=256, N=30, cap=7.0)
    loop = oracle.loop(1, 1, oracle.config(cfg), seed=1, capacity=10)
    ran = loop.run(200)
    recs = loop.records()
    assert ran == len(recs) and ran >= 100
    gp, gv, gq = loop.goal()
    goal = GoalSpec(tuple(gp), tuple(gv), tuple(gq))
    planner = Planner(cfg, precision=precision, max_points=1 << 16)
    mismatches = []
    for r in recs:
        snap = planner.build_snapshot(r["cloud"], State.from_array(r["x"]), cfg.r_max, f64=True)
        prev = r["prev"] if r["prev_len"] == cfg.mppi.horizon else None
        la = ControlInput(r["last_applied"][0], tuple(r["last_applied"][1:]))
        try:
            res = planner.plan_step(State.from_array(r["x"]), goal, snap, prev, la, r["cycle"], 1,
                                    want_rollout=False)
        except PlanningFailed:
            assert not r["planned"], r["cycle"]
            continue
        assert r["planned"]
        if res.winner != r["winner"] or rel(res.control.vec(), r["control"]) > 1e-9:
            mismatches.append((r["cycle"], res.winner, r["winner"], res.control.vec(), r["control"]))
            continue
        assert rel(res.per_instance[res.winner].stage2, r["stage2"]) <= 1e-9
        assert rel(res.per_instance[res.winner].nominal, r["winner_nominal"]) <= 1e-9
    planner.close()
    assert not mismatches, mismatches[:5]
