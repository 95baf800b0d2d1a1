"""Formats around the plan path (amppi_cloud_* and the
debug dumps): byte-for-byte against restatements of the reference writers
(io.cpp:24-99) and exact round trips; the last test runs them through the
device path (frames -> files -> buffer -> device snapshot + plan -> dumps)."""
import numpy as np
import pytest

from paper_2509_17340_b200 import io as aio


def _ref_cloud_text(xyz, frame_id):  # write_cloud_frame (io.cpp:24-35)
    out = ["# amppi-cloud v1", f"frame {frame_id}"]
    out += ["%.17g %.17g %.17g" % tuple(p) for p in xyz]
    return "\n".join(out) + "\n"


@pytest.fixture()
def cloud():
    rs = np.random.default_rng(11)
    xyz = rs.normal(scale=7.0, size=(3000, 3))
    xyz[0] = [0.1, -0.0, 1e-300]
    xyz[1] = [np.pi, np.e, -1e15]
    return xyz


def test_text_frame_matches_reference_writer_and_round_trips(cloud, tmp_path):
    p = tmp_path / "f.cloud"
    aio.write_cloud(str(p), cloud, frame_id=42)
    assert p.read_text() == _ref_cloud_text(cloud, 42)
    back, fid = aio.read_cloud(str(p))
    assert fid == 42
    assert np.array_equal(back.view(np.uint64), cloud.view(np.uint64))  # %.17g: bit-exact


def test_binary_frame_round_trips(cloud, tmp_path):
    p = tmp_path / "f.bin"
    aio.write_cloud(str(p), cloud, frame_id=7, binary=True)
    back, fid = aio.read_cloud(str(p))
    assert fid == 7 and np.array_equal(back, cloud)
    assert p.stat().st_size == len(b"# amppi-cloud-bin v1\n") + 16 + cloud.nbytes


def test_reader_accepts_reference_files_and_rejects_malformed(tmp_path):
    p = tmp_path / "r.cloud"
    p.write_text("# amppi-cloud v1\nframe 3\n1 2 3\n\n4.5e-1 -6 7\n")  # blank lines are skipped (io.cpp:47)
    xyz, fid = aio.read_cloud(str(p))
    assert fid == 3 and np.array_equal(xyz, [[1, 2, 3], [0.45, -6, 7]])
    for bad in ("# amppi-cloud v1\nframe 1\n1 2\n", "frame 1\n1 2 3\n", "# amppi-cloud v1\n1 2 3\n"):
        p.write_text(bad)
        with pytest.raises(ValueError):
            aio.read_cloud(str(p))


def test_partition_csv_matches_reference_writer(oracle, tmp_path):
    rs = np.random.default_rng(5)
    pts = rs.normal(scale=4.0, size=(5000, 3))
    snap = oracle.snapshot(pts, np.array([0, 0, 0, 1.0, 0, 0, 0, 0, 0, 0]), 10.0).get()
    ranges = snap["ranges"]
    p = tmp_path / "partition.csv"
    aio.write_partition_csv(str(p), ranges)
    ref = ["i,j,range"] + ["%d,%d,%.17g" % (i, j, ranges[i * 60 + j]) for i in range(120) for j in range(60)]
    assert p.read_text() == "\n".join(ref) + "\n"  # write_partition_csv (io.cpp:68-76)


def test_anchors_csv_matches_reference_writer(oracle, tmp_path):
    from test_plan_parity import make_cfg, wall_cloud

    cfg = make_cfg(4, 2, K=32, N=25)
    x = np.array([0, 0, 2, 1, 0, 0, 0, 2.0, 0, 0])
    snap = oracle.snapshot(wall_cloud(), x, 10.0)
    o = oracle.plan(snap, oracle.config(cfg), x, [20, 0, 2], [0, 0, 0], [1, 0, 0, 0], None, [9.81, 0, 0, 0], 3, 7)

    class Anchor:
        def __init__(self, r):
            self.refined_endpoint = r

    class Plan:
        anchors = [Anchor(r) for r in o["anchor_refined"]]
        guides = o["guide_coeffs"].reshape(-1, 3, 6)

    T = cfg.mppi.horizon * cfg.mppi.dt
    p = tmp_path / "anchors.csv"
    aio.write_anchors_csv(str(p), 5, Plan, T, 10)
    ref = ["step,anchor,x,y,z"]
    for a, r in enumerate(o["anchor_refined"]):
        ref.append("5,%d,%.17g,%.17g,%.17g" % (a, *r))
        c = Plan.guides[a]
        for s in range(1, 11):
            t = min(max(T * s / 10, 0.0), T)
            pt = []
            for ax in range(3):
                v = c[ax, 5]
                for k in range(4, -1, -1):
                    v = v * t + c[ax, k]
                pt.append(v)
            ref.append("5,%d,%.17g,%.17g,%.17g" % (a, *pt))
    assert p.read_text() == "\n".join(ref) + "\n"  # write_anchors_csv (io.cpp:78-99)


@pytest.mark.gpu
def test_cloud_files_through_the_device_path(oracle, tmp_path):
    """The formats in the device job: LiDAR frames written as text and binary
    cloud files, read back into a PointCloudBuffer, planned on the device; the
    device snapshot's partition.csv is byte-equal to the one written from the
    oracle's snapshot of the same frames, and the anchors.csv dump of the
    device plan matches the oracle plan's dump to 1e-12."""
    from paper_2509_17340_b200 import ControlInput, GoalSpec, Planner, PointCloudBuffer, State
    from test_plan_parity import make_cfg

    sc = oracle.scene(1, 3)
    pose = np.array([6.0, 0.5, 2.0, 1, 0, 0, 0, 2.0, 0, 0], dtype=np.float64)
    buf = PointCloudBuffer(8)
    for f in range(8):
        pts = sc.lidar(pose, 900 + f)
        p = tmp_path / f"frame{f}.{'bin' if f % 2 else 'cloud'}"
        aio.write_cloud(str(p), pts, frame_id=f, binary=bool(f % 2))
        back, fid = aio.read_cloud(str(p))
        assert fid == f and np.array_equal(back, pts)
        buf.push(back)
    cloud = buf.points()
    cfg = make_cfg(4, 2, K=128, N=25)
    x = State.from_array(pose)
    goal = GoalSpec.facing(tuple(pose[:3]), (40.0, 0.0, 2.0))
    with Planner(cfg, max_points=1 << 16) as planner:
        snap = planner.build_snapshot(buf, x, cfg.r_max, f64=True)
        dev = snap.download()
        plan = planner.plan_step(x, goal, snap, None, ControlInput(9.81), 7, 3)
    osnap = oracle.snapshot(cloud, pose, cfg.r_max)
    orng = osnap.get()["ranges"]
    aio.write_partition_csv(str(tmp_path / "dev.csv"), dev["ranges"])
    aio.write_partition_csv(str(tmp_path / "ora.csv"), orng)
    assert (tmp_path / "dev.csv").read_bytes() == (tmp_path / "ora.csv").read_bytes()
    o = oracle.plan(osnap, oracle.config(cfg), pose, goal.p_goal, goal.v_goal, goal.q_goal, None,
                    [9.81, 0, 0, 0], 7, 3)

    class OPlan:
        anchors = [type("A", (), {"refined_endpoint": r}) for r in o["anchor_refined"]]
        guides = o["guide_coeffs"].reshape(-1, 3, 6)

    T = cfg.mppi.horizon * cfg.mppi.dt
    aio.write_anchors_csv(str(tmp_path / "dev_a.csv"), 7, plan, T, 10)
    aio.write_anchors_csv(str(tmp_path / "ora_a.csv"), 7, OPlan, T, 10)
    dl = (tmp_path / "dev_a.csv").read_text().splitlines()
    ol = (tmp_path / "ora_a.csv").read_text().splitlines()
    assert dl[0] == ol[0] and len(dl) == len(ol)
    dv = np.array([[float(v) for v in ln.split(",")] for ln in dl[1:]])
    ov = np.array([[float(v) for v in ln.split(",")] for ln in ol[1:]])
    assert np.array_equal(dv[:, :2], ov[:, :2])
    assert np.max(np.abs(dv[:, 2:] - ov[:, 2:]) / np.maximum(1.0, np.abs(ov[:, 2:]))) <= 1e-12
