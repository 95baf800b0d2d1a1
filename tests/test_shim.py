"""The C++ shim (include/amppi_b200.hpp) compiles against the C ABI and, on a
B200, reproduces the oracle through the reference-signature calls:

* examples/shim_plan.cpp: the test_ensemble.cpp:127-153 scenario (5 cycles,
  plan_step with a reused PlanScratch);
* tests/native/shim_loop.cpp: execute_cycle (ensemble.cpp:245-305) written
  against the shim -- build_snapshot(buffer, pose, r_max), plan_step(...,
  scratch), rk4_step -- run for two back-to-back episodes with
  apply_velocity_cap configs (the run_batch pattern, metrics.cpp:141-147) and
  compared cycle by cycle with the oracle's execute_cycle loop; plus the
  value semantics of PerceptionSnapshot (perception.hpp:132-133): a snapshot
  planned on after a newer one was built gives the same plan."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2509_17340_b200")
ORACLE_DIR = os.path.join(ROOT, "oracle", "_build")
FLAGS = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-Wall", "-Wextra", "-Werror"]


def build(tmp_path):
    exe = str(tmp_path / "shim_plan")
    subprocess.run(FLAGS + ["-o", exe, os.path.join(ROOT, "examples", "shim_plan.cpp"), f"-L{LIBDIR}", "-lamppi_b200",
                            f"-Wl,-rpath,{LIBDIR}"], check=True)
    return exe


def build_loop(tmp_path):
    exe = str(tmp_path / "shim_loop")
    subprocess.run(FLAGS + ["-o", exe, os.path.join(ROOT, "tests", "native", "shim_loop.cpp"), f"-L{LIBDIR}",
                            "-lamppi_b200", f"-Wl,-rpath,{LIBDIR}", f"-L{ORACLE_DIR}", "-loracle",
                            f"-Wl,-rpath,{ORACLE_DIR}"], check=True)
    return exe


def test_shim_compiles_and_links(tmp_path, product_lib, oracle):
    assert os.path.exists(build(tmp_path))
    assert os.path.exists(build_loop(tmp_path))


@pytest.mark.gpu
def test_shim_matches_oracle(tmp_path, oracle):
    exe = build(tmp_path)
    lines = [json.loads(ln) for ln in subprocess.run([exe], capture_output=True, text=True, check=True).stdout.splitlines()]
    assert len(lines) == 5
    from test_plan_parity import make_cfg, wall_cloud

    cfg = make_cfg(5, 3, K=32)
    ocfg = oracle.config(cfg)
    x = np.array([0, 0, 2, 1, 0, 0, 0, 0, 0, 0], dtype=np.float64)
    snap = oracle.snapshot(wall_cloud(), x, 10.0)
    q = oracle.goal_facing(x[:3], [25, -3, 2])
    prev = None
    for cyc, ln in enumerate(lines):
        o = oracle.plan(snap, ocfg, x, [25, -3, 2], [0, 0, 0], q, prev, [9.81, 0, 0, 0], cyc, 31)
        assert ln["winner"] == o["winner"]
        assert np.max(np.abs(np.array(ln["control"]) - o["control"])) <= 1e-9
        prev = o["nominal"][o["winner"]]


@pytest.mark.gpu
def test_shim_execute_cycle_two_caps_vs_oracle_loop(tmp_path, oracle):
    from paper_2509_17340_b200 import apply_velocity_cap
    from test_plan_parity import make_cfg

    exe = build_loop(tmp_path)
    cycles, caps, seed = 40, (5.0, 7.0), 7
    out = subprocess.run([exe, "1", "1", str(seed), str(cycles)] + [str(c) for c in caps], capture_output=True,
                         text=True, check=True).stdout
    lines = [json.loads(ln) for ln in out.splitlines()]
    snap = {ln["tag"]: ln for ln in lines if ln["tag"].startswith("snap_")}
    # an older snapshot, planned on after a newer one was built, plans identically
    assert snap["snap_again"]["winner"] == snap["snap_first"]["winner"]
    assert snap["snap_again"]["control"] == snap["snap_first"]["control"]
    assert snap["snap_again"]["stage2"] == snap["snap_first"]["stage2"]
    for cap in caps:
        got = [ln for ln in lines if ln["tag"] == "loop" and ln["cap"] == cap]
        assert len(got) == cycles
        cfg = apply_velocity_cap(make_cfg(4, 2, K=256, N=30), cap)
        lo = oracle.loop(1, 1, oracle.config(cfg), seed, capacity=10)
        n = lo.run(cycles)
        recs = lo.records()
        assert n >= 20, n
        for g, o in zip(got[:n], recs[:n]):
            assert g["cycle"] == o["cycle"]
            assert np.max(np.abs(np.array(g["x"]) - o["x"])) <= 1e-9, (cap, g["cycle"])
            assert g["winner"] == (o["winner"] if o["planned"] else -1), (cap, g["cycle"])
            assert np.max(np.abs(np.array(g["control"]) - o["control"])) <= 1e-8, (cap, g["cycle"])
