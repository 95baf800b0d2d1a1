"""Formats around the plan path (amppi_cloud_* and the
debug dumps): byte-for-byte against restatements of the reference writers
(io.cpp:24-99) and exact round trips.  CPU only (no device needed)."""
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
