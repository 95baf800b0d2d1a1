"""The C++ shim (include/amppi_b200.hpp) compiles against the C ABI and, on a
B200, reproduces the oracle's results for the test_ensemble.cpp:127-153
scenario through the reference-style build_snapshot / plan_step calls."""
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2509_17340_b200")


def build(tmp_path):
    exe = str(tmp_path / "shim_plan")
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-o", exe,
                    os.path.join(ROOT, "examples", "shim_plan.cpp"), f"-L{LIBDIR}", "-lamppi_b200",
                    f"-Wl,-rpath,{LIBDIR}"], check=True)
    return exe


def test_shim_compiles_and_links(tmp_path, product_lib):
    assert os.path.exists(build(tmp_path))


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
