"""save_volume / load_volume (tsdf.cpp:61-153) on device volumes, restating the
reference's checkpoint test (test_tsdf.cpp:513-570): the dense single-channel
file is the reference's "CSFVOL 1" format (float32 planes), the derivative
plane is written only when in use, corrupt/truncated/missing files raise
std::runtime_error.  The hashed/multi-channel extension round-trips the block
table (bit-exact) and every channel."""
import os

import numpy as np
import pytest

import paper_2405_02187_b200 as csf
from paper_2405_02187_b200 import capi

pytestmark = pytest.mark.gpu


def _dense(ctx, channels=1):
    # VolumeParams::cube(10, 0.04, (0.5, -0.25, 1.0)), weight_cap 64
    return csf.TsdfVolume((10, 10, 10), 0.04, (0.5, -0.25, 1.0), 5 * 0.04, 64.0, channels=channels, ctx=ctx)


def test_checkpoint_roundtrip_reference_cases(gpu_ctx, tmp_path):
    rng = np.random.default_rng(123)
    vol = _dense(gpu_ctx)
    n = 1000
    field = np.zeros((n, 2))
    field[:, 0] = rng.uniform(-1.0, 1.0, n)
    weight = np.floor(rng.uniform(0.0, 5.0, n))
    vol.upload(field, weight)
    path = tmp_path / "vol.csfvol"
    csf.save_volume(path, vol)
    head = path.read_bytes().split(b"\ndata\n", 1)[0].decode().splitlines()
    assert head[0] == "CSFVOL 1" and head[1] == "dims 10 10 10" and head[-1] == "channels field weight"
    plain = os.path.getsize(path)
    back = csf.load_volume(path, channels=1, ctx=gpu_ctx)  # a Complex volume, im = 0 (tsdf.cpp:139-147)
    f2, w2 = back.download()
    assert np.array_equal(f2[:, 0], field[:, 0].astype(np.float32).astype(np.float64))
    assert np.array_equal(w2, weight.astype(np.float32).astype(np.float64))
    assert np.all(f2[:, 1] == 0.0)
    p = back.params
    assert tuple(p.dims) == (10, 10, 10) and p.voxel_size == 0.04 and tuple(p.origin) == (0.5, -0.25, 1.0)
    assert p.mu == 5 * 0.04 and p.weight_cap == 64.0

    # derivative channel kept only when in use
    field[17, 1] = 3.25e-9
    vol.upload(field, weight)
    csf.save_volume(path, vol)
    assert os.path.getsize(path) > plain + 3 * n
    f3, _ = csf.load_volume(path, ctx=gpu_ctx).download()
    assert f3[17, 1] == float(np.float32(3.25e-9)) and f3[16, 1] == 0.0

    # corrupt, truncated and missing checkpoints raise std::runtime_error
    bad = tmp_path / "bad.csfvol"
    bad.write_bytes(b"NOTAVOL 1\n")
    with pytest.raises(RuntimeError):
        csf.load_volume(bad, ctx=gpu_ctx)
    data = path.read_bytes()
    bad.write_bytes(data[: len(data) // 2])
    with pytest.raises(RuntimeError):
        csf.load_volume(bad, ctx=gpu_ctx)
    with pytest.raises(RuntimeError):
        csf.load_volume(tmp_path / "missing.csfvol", ctx=gpu_ctx)


def test_checkpoint_hashed_multichannel(gpu_ctx, oracle_built, tmp_path):
    from oracle import orc
    d, gt, k = orc.workload(2, 3, 160, 120)
    D = 3
    vol = csf.HashedVolume(0.02, (0.0, 0.0, 0.0), 0.1, 128.0, 16, 1 << 14, channels=D, ctx=gpu_ctx)
    rng = np.random.default_rng(5)
    intr = np.zeros((4, 1 + D))
    intr[:, 0] = [k.fx, k.fy, k.cx, k.cy]
    for i in range(3):
        pose = np.zeros((12, 1 + D))
        pose[:, 0] = gt[i]
        pose[:, 1:] = rng.uniform(-1, 1, (12, D)) * 1e-8
        vol.surface_update(d[i].astype(np.float64), pose, intr)
    path = tmp_path / "hashed.csfvol"
    vol.save(path)
    back = csf.load_volume(path, ctx=gpu_ctx)
    assert isinstance(back, csf.HashedVolume) and back.channels == D
    for a, b in zip(vol.hash_tables(), back.hash_tables()):
        assert np.array_equal(a, b)
    f1, w1 = vol.download()
    f2, w2 = back.download()
    assert np.array_equal(f2, f1.astype(np.float32).astype(np.float64))
    assert np.array_equal(w2, w1.astype(np.float32).astype(np.float64))
    # the reloaded volume raycasts like the original (float32 field)
    pose = gt[1]
    V1, N1 = vol.raycast(pose, intr[:, :1].repeat(1 + D, 1) * np.r_[1, [0] * D], 80, 60)
    V2, N2 = back.raycast(pose, intr[:, :1].repeat(1 + D, 1) * np.r_[1, [0] * D], 80, 60)
    hit = (N1[..., 0] ** 2).sum(-1) > 0.5
    assert hit.sum() > 100 and np.abs(V1[..., 0] - V2[..., 0])[hit].max() < 1e-3
