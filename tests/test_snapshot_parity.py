"""GPU parity of build_snapshot (K1 keying, K1b tie-break, K2 partition /
pooling / filtered cloud) against the CPU oracle: bit-exact per-cell ranges,
occupancy, nearest points, pooled safe ranges/directions/points and the
flat-order world-frame filtered cloud.

Inputs: the reference tests' own seeded clouds (test_perception.cpp:102-253,
acceptance.cpp:152-226), edge cases (empty, single point, axis / boundary
points, exact range ties, out-of-range points), rotated poses and synthetic
LiDAR scans from the oracle's restated simulator (forest 20k, verticals 1M).
"""
import math

import numpy as np
import pytest

from oracle_py import RandomStream, random_cloud

pytestmark = pytest.mark.gpu

IDENT = np.array([0, 0, 0, 1, 0, 0, 0, 0, 0, 0], dtype=np.float64)


@pytest.fixture(scope="module")
def planner():
    from paper_2509_17340_b200 import EnsembleConfig, Planner

    p = Planner(EnsembleConfig(), max_points=1 << 21)
    yield p
    p.close()


def check(planner, oracle, pts, pose=IDENT, r_max=10.0, f64=True):
    from paper_2509_17340_b200 import State

    pts = np.asarray(pts, dtype=np.float64).reshape(-1, 3)
    if not f64:
        pts = pts.astype(np.float32).astype(np.float64)  # the oracle sees the device's float values
    snap = planner.build_snapshot(pts, State.from_array(pose), r_max, f64=f64)
    d = snap.download()
    o = oracle.snapshot(pts, pose, r_max).get()
    assert np.array_equal(d["has_point"], o["has_point"]), "occupancy"
    assert np.array_equal(d["ranges"], o["ranges"]), "ranges"
    assert np.array_equal(d["nearest"], o["nearest"]), "nearest (argmin point) per cell"
    assert np.array_equal(d["safe_range"], o["safe_range"]), "pooled safe range"
    assert np.array_equal(d["safe_dir"], o["safe_dir"]), "pooled argmax direction"
    assert np.array_equal(d["safe_point"], o["safe_point"]), "safe point"
    assert d["filtered"].shape == o["filtered"].shape
    assert np.array_equal(d["filtered"], o["filtered"]), "filtered cloud (world, flat order)"
    return d


def test_empty_cloud(planner, oracle):
    d = check(planner, oracle, np.zeros((0, 3)))
    assert (d["ranges"] == 10.0).all() and d["filtered"].shape[0] == 0


def test_single_point(planner, oracle):
    p = 4.0 * np.array([math.cos(0.01) * math.cos(0.01), math.cos(0.01) * math.sin(0.01), math.sin(0.01)])
    d = check(planner, oracle, p[None])
    assert d["has_point"].sum() == 1


@pytest.mark.parametrize("trial", range(5))
def test_reference_random_clouds_seed101(planner, oracle, trial):
    rs = RandomStream(101)
    for _ in range(trial):
        random_cloud(rs, 10000, 12.0)
    check(planner, oracle, random_cloud(rs, 10000, 12.0))


def test_reference_random_cloud_seed202_and_float_path(planner, oracle):
    cloud = random_cloud(RandomStream(202), 20000, 12.0)
    check(planner, oracle, cloud, f64=True)
    check(planner, oracle, cloud, f64=False)


def test_acceptance_partition_oracle_100_clouds(planner, oracle):
    """acceptance.cpp:152-226: 100 x 10k clouds from RandomStream(777)."""
    rs = RandomStream(777)
    for _ in range(100):
        cloud = random_cloud(rs, 10000, 12.0)
        rs.uniforms(300)  # the 100 clearance queries drawn between clouds
        check(planner, oracle, cloud)


def test_axis_and_boundary_points(planner, oracle):
    """atan2 at +/-0, pi/2, the +pi wrap, exact cell boundaries, r_max."""
    pts = []
    for r in (0.5, 3.0, 9.999, 10.0):
        for a in np.arange(-180, 181, 3.0):  # exact 3-degree lattice directions
            ar = math.radians(a)
            pts.append((r * math.cos(ar), r * math.sin(ar), 0.0))
        for e in np.arange(-90, 91, 3.0):
            er = math.radians(e)
            pts.append((r * math.cos(er), 0.0, r * math.sin(er)))
            pts.append((-r * math.cos(er), -0.0, r * math.sin(er)))
    pts += [(0.0, 0.0, 5.0), (0.0, 0.0, -5.0), (-4.0, 0.0, 0.0), (-4.0, -0.0, 0.0), (0.0, -3.0, 0.0),
            (0.03, 0.0, 0.0), (0.05, 0.0, 0.0), (10.0000001, 0.0, 0.0), (0.0, 10.0, 0.0)]
    check(planner, oracle, np.array(pts))


def test_exact_range_ties_first_point_wins(planner, oracle):
    a = (5.0, 0.125, 0.0625)
    b = (5.0, 0.0625, 0.125)  # same cell, identical range bits, different point
    for order in ([a, b], [b, a], [b, a, b, a, a]):
        d = check(planner, oracle, np.array(order))
        f = np.nonzero(d["has_point"])[0]
        assert len(f) == 1 and tuple(d["nearest"][f[0]]) == order[0]
    # many duplicates across "frames" with interleaved closer points
    rs = np.random.default_rng(5)
    base = rs.uniform(-8, 8, size=(500, 3))
    cloud = np.concatenate([base, base[::-1], base[:100], base * 0.5])
    check(planner, oracle, cloud)


def test_rotated_translated_pose(planner, oracle):
    cloud = random_cloud(RandomStream(606), 8000, 11.0)
    for yaw, tilt, t in ((0.5 * math.pi, 0.0, (1.0, 1.0, 2.0)), (0.3, 0.2, (-2.5, 4.0, 1.0)), (2.9, -0.4, (0, 0, 0))):
        q = np.array([math.cos(yaw / 2) * math.cos(tilt / 2), -math.sin(yaw / 2) * math.sin(tilt / 2),
                      math.cos(yaw / 2) * math.sin(tilt / 2), math.sin(yaw / 2) * math.cos(tilt / 2)])
        q /= np.linalg.norm(q)
        pose = np.concatenate([t, q, [0.0, 0.0, 0.0]])
        check(planner, oracle, cloud + np.array(t), pose)
        check(planner, oracle, cloud + np.array(t), pose, f64=False)


def test_r_max_variants(planner, oracle):
    cloud = random_cloud(RandomStream(11), 20000, 14.0)
    for r_max in (5.0, 10.0, 12.5):
        check(planner, oracle, cloud, r_max=r_max)


def _scan(oracle, kind, seed, frames, pose, start_seed=0):
    sc = oracle.scene(kind, seed)
    out = [sc.lidar(pose, start_seed + f) for f in range(frames)]
    return np.concatenate(out, axis=0)


def test_forest_scan_20k(planner, oracle):
    pose = np.array([8.0, 1.0, 2.0, 1, 0, 0, 0, 0, 0, 0], dtype=np.float64)
    cloud = _scan(oracle, 1, 1, 24, pose)[:20000]
    assert cloud.shape[0] >= 15000
    check(planner, oracle, cloud, pose, f64=False)
    check(planner, oracle, cloud, pose, f64=True)


def test_dense_1m_point_scan(planner, oracle):
    """C3: ~1M accumulated points on a verticals scene."""
    pose = np.array([12.0, -2.0, 2.0, 1, 0, 0, 0, 0, 0, 0], dtype=np.float64)
    frame = _scan(oracle, 2, 7, 1, pose)
    reps = int(math.ceil(1_000_000 / frame.shape[0]))
    cloud = _scan(oracle, 2, 7, reps, pose)[:1_000_000]
    check(planner, oracle, cloud, pose, f64=False)
