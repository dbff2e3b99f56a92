"""On-disk formats (dataset.hpp) through the C-ABI,
checked against the reference's own test cases (proj/tests/test_dataset.cpp)
and an independent numpy/zlib PNG codec (oracle/orc_dataset.py).  Host file
I/O: runs without a GPU."""
import numpy as np
import pytest

import paper_2405_02187_b200 as csf
from oracle import orc_dataset as od


def _rand_depth(seed, w=37, h=23):
    rng = np.random.default_rng(seed)
    r = rng.uniform(-0.5, 6.0, (h, w))
    return np.where(r > 0, r, 0.0)


def test_png_round_trip_exact_at_storage_resolution(tmp_path):
    # test_dataset.cpp:28-44
    d = _rand_depth(101)
    p = tmp_path / "depth.png"
    csf.write_depth_png16(p, d, 5000.0)
    back = csf.read_depth_png16(p, 5000.0)
    assert back.shape == d.shape
    assert np.array_equal(back, od.quantize_depth(d, 5000.0))
    # the oracle decodes the product's file to the same integers
    u = od.decode_u16(p.read_bytes())
    assert np.array_equal(u.astype(np.float64) / 5000.0, back)


@pytest.mark.parametrize("filters,split", [((0,), 0), ((1,), 0), ((2,), 7), ((3,), 0), ((4,), 0), ((0, 1, 2, 3, 4), 50)])
def test_png_reader_every_filter_and_idat_split(tmp_path, filters, split):
    rng = np.random.default_rng(7)
    u = rng.integers(0, 65536, size=(19, 33), dtype=np.uint16)
    u[rng.random(u.shape) < 0.2] = 0
    p = tmp_path / "f.png"
    p.write_bytes(od.encode_u16(u, filters, split))
    back = csf.read_depth_png16(p, 1000.0)
    assert np.array_equal(back, np.where(u > 0, u.astype(np.float64) / 1000.0, 0.0))


def test_png_edges_out_of_range_and_corrupt(tmp_path):
    d = np.array([[0.0, -1.0, 1e-5, 13.107], [13.1072, 1.0 / 5000.0 * 0.5, 2.5, np.nan]])
    p = tmp_path / "e.png"
    csf.write_depth_png16(p, d, 5000.0)
    back = csf.read_depth_png16(p, 5000.0)
    assert np.array_equal(back, od.quantize_depth(np.nan_to_num(d, nan=0.0), 5000.0))
    # test_dataset.cpp:46-53: corrupt / missing files throw runtime_error
    bad = tmp_path / "bad.png"
    bad.write_text("this is not a png")
    with pytest.raises(RuntimeError):
        csf.read_depth_png16(bad, 5000.0)
    with pytest.raises(RuntimeError):
        csf.read_depth_png16(tmp_path / "missing.png", 5000.0)
    # an 8-bit PNG is refused
    rgb = od.SIG + od._chunk(b"IHDR", bytes.fromhex("00000002000000020800000000")) + od._chunk(b"IEND", b"")
    p8 = tmp_path / "p8.png"
    p8.write_bytes(rgb)
    with pytest.raises(RuntimeError, match="16-bit"):
        csf.read_depth_png16(p8, 5000.0)
    # a flipped byte in IDAT fails the CRC
    good = bytearray((tmp_path / "e.png").read_bytes())
    good[45] ^= 0xff
    flip = tmp_path / "flip.png"
    flip.write_bytes(bytes(good))
    with pytest.raises(RuntimeError):
        csf.read_depth_png16(flip, 5000.0)


def test_intrinsics_round_trip_and_validation(tmp_path):
    # test_dataset.cpp:55-84
    k = csf.intrinsics(517.3, 516.5, 318.6, 255.3, 640, 480, 5000.0)
    p = tmp_path / "intrinsics.txt"
    csf.write_intrinsics(p, k)
    r = csf.read_intrinsics(p)
    assert (r.fx, r.fy, r.cx, r.cy, r.width, r.height, r.depth_scale) == (517.3, 516.5, 318.6, 255.3, 640, 480, 5000.0)
    p.write_text("1 2 3 4 5 6\n")
    with pytest.raises(RuntimeError):
        csf.read_intrinsics(p)
    p.write_text("-1 2 3 4 5 6 7\n")
    with pytest.raises(RuntimeError):
        csf.read_intrinsics(p)
    with pytest.raises(RuntimeError):
        csf.read_intrinsics(tmp_path / "nope.txt")
    p.write_text("# comment\n10 11 # trailing\n 5 6\n64 48 1000\n")
    r = csf.read_intrinsics(p)
    assert (r.fx, r.fy, r.cx, r.cy, r.width, r.height, r.depth_scale) == (10, 11, 5, 6, 64, 48, 1000)


def _exp_rot(phi):
    th = np.linalg.norm(phi)
    K = np.array([[0, -phi[2], phi[1]], [phi[2], 0, -phi[0]], [-phi[1], phi[0], 0]]) / th
    return np.eye(3) + np.sin(th) * K + (1 - np.cos(th)) * K @ K


def test_trajectory_round_trip(tmp_path):
    # test_dataset.cpp:86-103
    rng = np.random.default_rng(107)
    traj = []
    for i in range(10):
        xi = rng.uniform(-1, 1, 6)
        pose = np.concatenate([_exp_rot(xi[3:]).reshape(9), xi[:3]])
        traj.append(csf.TrajectoryEntry(0.25 * i + 1300000000.0, pose))
    # cover every branch of the matrix -> quaternion conversion (trace <= 0, each axis)
    for ax in range(3):
        phi = np.zeros(3)
        phi[ax] = 3.0
        traj.append(csf.TrajectoryEntry(1.0 + ax, np.concatenate([_exp_rot(phi).reshape(9), [ax, 0, 0]])))
    p = tmp_path / "traj.txt"
    csf.write_trajectory(p, traj)
    back = csf.read_trajectory(p)
    assert len(back) == len(traj)
    for a, b in zip(back, traj):
        assert a.timestamp == b.timestamp
        assert np.array_equal(a.pose[9:], b.pose[9:])
        assert np.linalg.norm(a.pose[:9] - b.pose[:9]) < 1e-12
    # the reader's rotation is Eigen's normalized().toRotationMatrix() (restated)
    line = "5.0 1 2 3 0.1 0.2 0.3 0.9\n"
    p.write_text("# header\n" + line + "garbage line\n")
    (e,) = csf.read_trajectory(p)
    assert np.array_equal(e.pose[:9], od.quat_to_rot(0.9, 0.1, 0.2, 0.3).reshape(9))


def test_sequence_directory_round_trip(tmp_path):
    # test_dataset.cpp:105-137 (frames from the oracle's renderer)
    from oracle import orc
    d, gt, _ = orc.workload(1, 3, 64, 48)
    k = csf.intrinsics(70.0, 70.0, 31.5, 23.5, 64, 48, 5000.0)
    traj = [csf.TrajectoryEntry(10.0 + 0.1 * i, gt[i]) for i in range(3)]
    csf.write_sequence(tmp_path, k, [x.astype(np.float64) for x in d], traj)
    seq = csf.open_sequence(tmp_path)
    assert len(seq.frames) == 3 and len(seq.groundtruth) == 3
    assert seq.intrinsics.fx == k.fx and seq.frames[1].timestamp == 10.1
    assert np.array_equal(seq.load_depth(1), od.quantize_depth(d[1].astype(np.float64), 5000.0))
    assert np.array_equal(seq.groundtruth[2].pose[9:], gt[2][9:])
    with pytest.raises(RuntimeError):
        csf.open_sequence(tmp_path / "nothere")
