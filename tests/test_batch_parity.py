"""GPU parity of the batched plan cycle (config C5's path: amppi_cycle_batch /
amppi_cycle_batch_device) against the CPU oracle, scene by scene.

160 scenes select the throughput schedules bench.py measures: the fused
one-CTA-per-scene snapshot (S >= 148) and bounded, lane-compacted FP32
screening (S*M*K >= 148*128*4).  Contract as in test_plan_parity.py: winner
and status bit-exact, returned FP64 values <= 1e-9.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

S = 160


@pytest.fixture(scope="module")
def batch():
    from paper_2509_17340_b200 import Planner
    from paper_2509_17340_b200.workloads import plan_config, scenes

    cfg = plan_config()
    data = scenes(S, points=20000, frames=20, first=0)
    planner = Planner(cfg, precision=32, max_scenes=S, max_points=int(data["offsets"][-1]))
    yield cfg, data, planner
    planner.close()


def _rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.abs(b)))) if a.size else 0.0


def _check_against_oracle(oracle, cfg, data, out, previous=None, cycle_shift=0):
    ocfg = oracle.config(cfg)
    off = data["offsets"]
    n_pass = 0
    for s in range(S):
        pts = data["xyz"][off[s]:off[s + 1]].astype(np.float64)
        snap = oracle.snapshot(pts, data["poses"][s], cfg.r_max)
        g = data["goals"][s]
        prev = None if previous is None else previous[s]
        o = oracle.plan(snap, ocfg, data["states"][s], g[0:3], g[3:6], g[6:10], prev, data["last"][s],
                        int(data["cycles"][s]) + cycle_shift, int(data["seeds"][s]))
        assert out["status"][s] == o["rc"], s
        if o["rc"] != 0:
            continue
        assert out["winner"][s] == o["winner"], s
        assert _rel(out["control"][s], o["control"]) <= 1e-9, s
        fin = np.isfinite(o["stage2"])
        assert np.array_equal(np.isfinite(out["stage2"][s]), fin), s
        assert _rel(out["stage2"][s][fin], o["stage2"][fin]) <= 1e-9, s
        assert _rel(out["breakdown"][s], o["breakdown"]) <= 1e-9, s
        assert _rel(out["winner_nominal"][s], o["nominal"][o["winner"]]) <= 1e-9, s
        n_pass += 1
    return n_pass


def _host_call(planner, data, previous=None, cycle_shift=0):
    return planner.cycle_batch(data["offsets"], data["xyz"], data["poses"], data["states"], data["goals"],
                               data["last"], data["cycles"] + np.uint64(cycle_shift), data["seeds"],
                               previous=previous)


def test_batch_cycle_matches_oracle(oracle, batch):
    cfg, data, planner = batch
    out = _host_call(planner, data)
    assert _check_against_oracle(oracle, cfg, data, out) > S // 2


def test_batch_warm_start_matches_oracle(oracle, batch):
    """Second cycle fed with each scene's winner nominal (shift_nominal path)."""
    cfg, data, planner = batch
    first = _host_call(planner, data)
    out = _host_call(planner, data, previous=first["winner_nominal"], cycle_shift=1)
    assert _check_against_oracle(oracle, cfg, data, out, previous=first["winner_nominal"], cycle_shift=1) > S // 2


def test_batch_two_iterations_paper_grid(oracle):
    """The paper's default ensemble (5x3 anchors x 256 samples x 25 steps)
    with two MPPI iterations per cycle, on the throughput schedules: the
    nominal update between iterations, the second iteration's perturbation
    stream and its bound / main passes, scene by scene against the oracle."""
    from paper_2509_17340_b200 import Planner
    from paper_2509_17340_b200.workloads import plan_config, scenes

    cfg = plan_config(m_h=5, m_v=3, K=256, N=25, iterations=2)
    data = scenes(S, points=20000, frames=20, first=3000)
    with Planner(cfg, precision=32, max_scenes=S, max_points=int(data["offsets"][-1])) as planner:
        out = _host_call(planner, data)
    assert _check_against_oracle(oracle, cfg, data, out) > S // 2


def test_batch_precision64_matches_oracle(oracle):
    """The FP64 screening (precision 64: every sample rolled out in FP64,
    k_stage1_f64) on the batch path, scene by scene against the oracle."""
    from paper_2509_17340_b200 import Planner
    from paper_2509_17340_b200.workloads import plan_config, scenes

    cfg = plan_config()
    data = scenes(S, points=20000, frames=20, first=4000)
    with Planner(cfg, precision=64, max_scenes=S, max_points=int(data["offsets"][-1])) as planner:
        out = _host_call(planner, data)
    assert _check_against_oracle(oracle, cfg, data, out) > S // 2


@pytest.fixture(scope="module")
def big_batch():
    from paper_2509_17340_b200 import Planner
    from paper_2509_17340_b200.workloads import plan_config, scenes

    cfg = plan_config()
    data = scenes(2 * 148 + 5, points=20000, frames=20, first=1000)
    planner = Planner(cfg, precision=32, max_scenes=len(data["states"]), max_points=int(data["offsets"][-1]))
    yield cfg, data, planner
    planner.close()


def test_chunked_batches_equal_single_chunk(big_batch, monkeypatch):
    """amppi_cycle_batch overlaps chunk c+1's point upload with chunk c's
    planning, and chunks alternate between two compute streams (host and
    device entry points); results must not depend on the chunking."""
    import torch

    cfg, data, planner = big_batch
    one = _host_call(planner, data)
    planner.set_schedule(pipeline_chunks=2)
    two = _host_call(planner, data)
    for k in one:
        assert np.array_equal(one[k], two[k]), k
    # other chunk schedules (growth ratio) give the same results too
    for ratio in (1.0, 1.6):
        planner.set_schedule(pipeline_ratio=ratio)
        again = _host_call(planner, data)
        for k in one:
            assert np.array_equal(one[k], again[k]), (ratio, k)
    planner.set_schedule(pipeline_ratio=0.0, pipeline_chunks=0)
    S = len(data["states"])
    dev = torch.device("cuda", 0)
    keep = {k: torch.from_numpy(np.ascontiguousarray(data[k])).to(dev)
            for k in ("xyz", "offsets", "poses", "states", "goals", "last")}
    keep["cycles"] = torch.from_numpy(data["cycles"].view(np.int64)).to(dev)
    keep["seeds"] = torch.from_numpy(data["seeds"].view(np.int64)).to(dev)
    N, M = cfg.mppi.horizon, cfg.grid.count()
    for chunks in (2, 3):
        planner.set_schedule(device_chunks=chunks)
        dout = {"status": torch.zeros(S, dtype=torch.int32, device=dev),
                "winner": torch.zeros(S, dtype=torch.int32, device=dev),
                "control": torch.zeros(S, 4, dtype=torch.float64, device=dev),
                "winner_nominal": torch.zeros(S, N, 4, dtype=torch.float64, device=dev),
                "stage2": torch.zeros(S, M, dtype=torch.float64, device=dev),
                "breakdown": torch.zeros(S, 5, dtype=torch.float64, device=dev)}
        planner.cycle_batch_device({k: v.data_ptr() for k, v in keep.items()},
                                   {k: v.data_ptr() for k, v in dout.items()}, S, cfg.r_max)
        planner.synchronize()
        for k in dout:
            assert np.array_equal(dout[k].cpu().numpy(), one[k]), (chunks, k)


def test_device_entry_point_equals_host(batch):
    import torch

    cfg, data, planner = batch
    host = _host_call(planner, data)
    dev = torch.device("cuda", 0)
    keep = {k: torch.from_numpy(np.ascontiguousarray(data[k])).to(dev)
            for k in ("xyz", "offsets", "poses", "states", "goals", "last")}
    keep["cycles"] = torch.from_numpy(data["cycles"].view(np.int64)).to(dev)
    keep["seeds"] = torch.from_numpy(data["seeds"].view(np.int64)).to(dev)
    N, M = cfg.mppi.horizon, cfg.grid.count()
    dout = {"status": torch.zeros(S, dtype=torch.int32, device=dev), "winner": torch.zeros(S, dtype=torch.int32, device=dev),
            "control": torch.zeros(S, 4, dtype=torch.float64, device=dev),
            "winner_nominal": torch.zeros(S, N, 4, dtype=torch.float64, device=dev),
            "stage2": torch.zeros(S, M, dtype=torch.float64, device=dev),
            "breakdown": torch.zeros(S, 5, dtype=torch.float64, device=dev)}
    planner.cycle_batch_device({k: v.data_ptr() for k, v in keep.items()}, {k: v.data_ptr() for k, v in dout.items()},
                               S, cfg.r_max)
    planner.synchronize()
    for k in dout:
        a, b = dout[k].cpu().numpy(), host[k]
        assert np.array_equal(a, b) or np.allclose(a, b, rtol=0, atol=0, equal_nan=True), k


def test_streaming_batches_equal_blocking(big_batch):
    """amppi_cycle_batch_submit / _wait with two and three batches in flight
    (the next batch's upload overlapping the current one's planning) return
    exactly what the blocking call returns for each batch."""
    import torch

    cfg, data, planner = big_batch
    pinned = torch.from_numpy(data["xyz"]).pin_memory()
    args = [data["offsets"], pinned.numpy(), data["poses"], data["states"], data["goals"], data["last"]]
    cyc = [data["cycles"] + np.uint64(d) for d in (11, 12, 13)]
    ref = [planner.cycle_batch(*args, c, data["seeds"]) for c in cyc]
    t0 = planner.cycle_batch_submit(*args, cyc[0], data["seeds"])
    t1 = planner.cycle_batch_submit(*args, cyc[1], data["seeds"])
    got0 = planner.cycle_batch_wait(t0)
    t2 = planner.cycle_batch_submit(*args, cyc[2], data["seeds"])
    got1 = planner.cycle_batch_wait(t1)
    got2 = planner.cycle_batch_wait(t2)
    for got, r in zip((got0, got1, got2), ref):
        for k in r:
            assert np.array_equal(got[k], r[k]), k
    assert not np.array_equal(ref[0]["control"], ref[1]["control"])  # the batches really differ
    # three in flight (the bench's e2e pattern), then a fourth refused until one is collected
    ts = [planner.cycle_batch_submit(*args, c, data["seeds"]) for c in cyc]
    with pytest.raises(ValueError, match="in flight"):
        planner.cycle_batch_submit(*args, cyc[0], data["seeds"])
    for t, r in zip(ts, ref):
        got = planner.cycle_batch_wait(t)
        for k in r:
            assert np.array_equal(got[k], r[k]), k
