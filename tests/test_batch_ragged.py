"""Ragged batches through the batched plan cycle (C5's path) against the CPU
oracle: empty scenes, single-point and tiny scenes, random scene sizes in one
batch, and a scene past 65536 points -- which the host entry point routes to
the many-CTA keying schedule and the device entry point (per-scene counts
not visible to the host) handles inside the fused per-scene snapshot by
re-keying.  Contract as test_batch_parity.py: status and winner bit-exact,
returned FP64 values <= 1e-9."""
import numpy as np
import pytest

from test_batch_parity import _rel

pytestmark = pytest.mark.gpu

S = 150  # >= 148: the fused per-scene snapshot and the throughput screening


def _ragged(data, sizes):
    off = data["offsets"]
    pts = [data["xyz"][off[s]:off[s] + n] for s, n in enumerate(sizes)]
    xyz = np.concatenate(pts).astype(np.float32) if pts else np.zeros((0, 3), np.float32)
    offsets = np.zeros(len(sizes) + 1, dtype=np.int64)
    offsets[1:] = np.cumsum([len(p) for p in pts])
    out = dict(data)
    out["xyz"], out["offsets"] = xyz, offsets
    return out


@pytest.fixture(scope="module")
def ragged():
    from paper_2509_17340_b200 import Planner
    from paper_2509_17340_b200.workloads import plan_config, scenes

    cfg = plan_config()
    data = scenes(S, points=20000, frames=20, first=3000)
    off = data["offsets"]
    full = np.diff(off)
    rs = np.random.default_rng(9)
    sizes = [int(rs.integers(0, n + 1)) for n in full]
    sizes[0], sizes[1], sizes[2], sizes[3] = 0, 1, 7, 100
    sizes[5] = int(full[5])
    rag = _ragged(data, sizes)
    # scene 4 with > 65536 points: its own scan plus the scans of scenes 6..9
    big = np.concatenate([data["xyz"][off[4]:off[5]]] + [data["xyz"][off[s]:off[s + 1]] for s in range(6, 10)])
    parts = [rag["xyz"][rag["offsets"][s]:rag["offsets"][s + 1]] for s in range(S)]
    parts[4] = big.astype(np.float32)
    huge = dict(rag)
    huge["xyz"] = np.concatenate(parts)
    huge["offsets"] = np.concatenate([[0], np.cumsum([len(p) for p in parts])]).astype(np.int64)
    assert huge["offsets"][5] - huge["offsets"][4] > 65536
    planner = Planner(cfg, precision=32, max_scenes=S, max_points=int(huge["offsets"][-1]))
    yield cfg, rag, huge, planner
    planner.close()


def _host(planner, d):
    return planner.cycle_batch(d["offsets"], d["xyz"], d["poses"], d["states"], d["goals"], d["last"], d["cycles"],
                               d["seeds"])


def _check(oracle, cfg, d, out, which):
    ocfg = oracle.config(cfg)
    off = d["offsets"]
    checked = 0
    for s in which:
        pts = d["xyz"][off[s]:off[s + 1]].astype(np.float64)
        snap = oracle.snapshot(pts, d["poses"][s], cfg.r_max)
        g = d["goals"][s]
        o = oracle.plan(snap, ocfg, d["states"][s], g[0:3], g[3:6], g[6:10], None, d["last"][s], int(d["cycles"][s]),
                        int(d["seeds"][s]))
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
        checked += 1
    return checked


def test_ragged_batch_matches_oracle(oracle, ragged):
    """Empty, 1-, 7- and 100-point scenes and random sizes, fused snapshot."""
    cfg, rag, _, planner = ragged
    out = _host(planner, rag)
    assert _check(oracle, cfg, rag, out, range(S)) > S // 2


def test_scene_past_65536_points_host_entry(oracle, ragged):
    """max points per scene > 65536: the host entry point keys with many
    CTAs per scene (k_key_points / k_resolve_ties / k_finalize_scene)."""
    cfg, _, huge, planner = ragged
    out = _host(planner, huge)
    _check(oracle, cfg, huge, out, range(12))


def test_scene_past_65536_points_device_entry(oracle, ragged):
    """The device entry point keeps the fused per-scene snapshot; the scene
    past the 16-bit candidate log re-keys its points in pass B."""
    import torch

    cfg, _, huge, planner = ragged
    dev = torch.device("cuda", 0)
    keep = {k: torch.from_numpy(np.ascontiguousarray(huge[k])).to(dev)
            for k in ("xyz", "offsets", "poses", "states", "goals", "last")}
    keep["cycles"] = torch.from_numpy(huge["cycles"].view(np.int64)).to(dev)
    keep["seeds"] = torch.from_numpy(huge["seeds"].view(np.int64)).to(dev)
    N, M = cfg.mppi.horizon, cfg.grid.count()
    dout = {"status": torch.zeros(S, dtype=torch.int32, device=dev), "winner": torch.zeros(S, dtype=torch.int32, device=dev),
            "control": torch.zeros(S, 4, dtype=torch.float64, device=dev),
            "winner_nominal": torch.zeros(S, N, 4, dtype=torch.float64, device=dev),
            "stage2": torch.zeros(S, M, dtype=torch.float64, device=dev),
            "breakdown": torch.zeros(S, 5, dtype=torch.float64, device=dev)}
    planner.cycle_batch_device({k: v.data_ptr() for k, v in keep.items()}, {k: v.data_ptr() for k, v in dout.items()},
                               S, cfg.r_max)
    planner.synchronize()
    out = {k: v.cpu().numpy() for k, v in dout.items()}
    _check(oracle, cfg, huge, out, range(12))
    host = _host(planner, huge)
    for k in out:
        assert np.array_equal(out[k], host[k]), k


def test_chunked_batches_with_a_scene_past_65536_points(oracle):
    """A batch large enough to be split into concurrent chunks that contains a
    scene past the fused snapshot's limit: that scene takes the many-CTA
    keying, whose candidate log is shared per launch, so the batch must run
    as one chunk (host entry, forced pipeline chunks; device entry with a
    capacity that selects the many-CTA keying) -- results equal the plain run."""
    import torch

    from paper_2509_17340_b200 import Planner
    from paper_2509_17340_b200.workloads import plan_config, scenes

    cfg = plan_config()
    S2 = 320
    data = scenes(S2, points=20000, frames=20, first=5000)
    off = data["offsets"]
    parts = [data["xyz"][off[s]:off[s + 1]] for s in range(S2)]
    parts[200] = np.concatenate(parts[200:205])  # > 65536 points
    big = dict(data)
    big["xyz"] = np.concatenate(parts).astype(np.float32)
    big["offsets"] = np.concatenate([[0], np.cumsum([len(p) for p in parts])]).astype(np.int64)
    assert big["offsets"][201] - big["offsets"][200] > 65536
    with Planner(cfg, precision=32, max_scenes=S2, max_points=int(big["offsets"][-1])) as p:
        ref = _host(p, big)
        p.set_schedule(pipeline_chunks=4)
        chunked = _host(p, big)
    for k in ref:
        assert np.array_equal(ref[k], chunked[k]), k
    _check(oracle, cfg, big, ref, [199, 200, 201])
    # device entry: capacity / scenes > 65536 selects the many-CTA keying
    with Planner(cfg, precision=32, max_scenes=S2, max_points=S2 * 70000, device_chunks=3) as p:
        dev = torch.device("cuda", 0)
        keep = {k: torch.from_numpy(np.ascontiguousarray(big[k])).to(dev)
                for k in ("xyz", "offsets", "poses", "states", "goals", "last")}
        keep["cycles"] = torch.from_numpy(big["cycles"].view(np.int64)).to(dev)
        keep["seeds"] = torch.from_numpy(big["seeds"].view(np.int64)).to(dev)
        N, M = cfg.mppi.horizon, cfg.grid.count()
        dout = {"status": torch.zeros(S2, dtype=torch.int32, device=dev),
                "winner": torch.zeros(S2, dtype=torch.int32, device=dev),
                "control": torch.zeros(S2, 4, dtype=torch.float64, device=dev),
                "winner_nominal": torch.zeros(S2, N, 4, dtype=torch.float64, device=dev),
                "stage2": torch.zeros(S2, M, dtype=torch.float64, device=dev),
                "breakdown": torch.zeros(S2, 5, dtype=torch.float64, device=dev)}
        p.cycle_batch_device({k: v.data_ptr() for k, v in keep.items()}, {k: v.data_ptr() for k, v in dout.items()},
                             S2, cfg.r_max)
        p.synchronize()
        for k in dout:
            assert np.array_equal(dout[k].cpu().numpy(), ref[k]), k


def test_batch_invalidates_the_single_scene_snapshot(ragged):
    """cycle_batch overwrites the single-scene perception slot: planning on a
    snapshot built before it is refused (the Python generation check, and the
    C ABI's AMPPI_NO_SNAPSHOT underneath), not silently planned on another
    scene's perception."""
    import ctypes

    from paper_2509_17340_b200 import ControlInput, GoalSpec, State, _abi

    cfg, rag, _, planner = ragged
    pts = rag["xyz"][rag["offsets"][10]:rag["offsets"][11]]
    x = State.from_array(rag["states"][10])
    snap = planner.build_snapshot(pts, x, cfg.r_max)
    _host(planner, rag)
    with pytest.raises(ValueError):
        planner.plan_step(x, GoalSpec((45, 0, 2)), snap, None, ControlInput(9.81), 1, 1)
    xs, gs, lc = x.to_c(), GoalSpec((45, 0, 2)).to_c(), ControlInput(9.81).to_c()
    rc = planner.lib.amppi_plan(planner._h, ctypes.byref(xs), ctypes.byref(gs), None, 0, ctypes.byref(lc),
                                ctypes.c_uint64(1), ctypes.c_uint64(1), None, None)
    assert rc == _abi.AMPPI_NO_SNAPSHOT
