"""Depth images that carry perturbation channels (the reference's
Image<Complex> depth of measured_tsdf / surface_update, tsdf.hpp:96-102 and
144-145): the channels enter psi through the bilinear depth sample.

  * the reference's pin (test_tsdf.cpp:194-231): seeding one depth pixel
    with im = h gives d psi / d D = (bilinear weight of that corner) / mu;
  * csf_measured_tsdf_lifted and csf_surface_update_lifted against the oracle
    (real parts bit-identical, channels within 1e-9), dense and hashed,
    depth-seeded and pose-seeded channels together.
"""
import ctypes as C

import numpy as np
import pytest

import paper_2405_02187_b200 as csf
from paper_2405_02187_b200 import capi

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def orc(oracle_built):
    from oracle import orc as o
    return o


def test_dpsi_ddepth_is_bilinear_weight_over_mu(gpu_ctx, orc):
    """test_tsdf.cpp:194-231: a voxel straight ahead of an identity camera over
    a flat 2 m depth image; corner (x0, y0) seeded with h: Im(psi)/h equals
    its bilinear weight / mu on the device and in the oracle."""
    w, h = 64, 48
    k = csf.intrinsics(60.0, 60.0, 31.3, 23.6, w, h)
    mu = 0.1
    hstep = 1e-8
    depth = np.zeros((h, w, 2))
    depth[..., 0] = 2.0
    w2c = np.zeros((12, 2))
    w2c[[0, 4, 8], 0] = 1.0
    pt = np.array([[0.013, -0.021, 1.97]])  # projects inside the cell (31, 22)
    lx = k.fx * pt[0, 0] / pt[0, 2] + k.cx
    ly = k.fy * pt[0, 1] / pt[0, 2] + k.cy
    x0, y0 = int(np.floor(lx)), int(np.floor(ly))
    fx, fy = lx - x0, ly - y0
    weights = {(x0, y0): (1 - fx) * (1 - fy), (x0 + 1, y0): fx * (1 - fy), (x0, y0 + 1): (1 - fx) * fy,
               (x0 + 1, y0 + 1): fx * fy}
    center = np.zeros((3, 2))
    for (cx_, cy_), wt in weights.items():
        dd = depth.copy()
        dd[cy_, cx_, 1] = hstep
        psi_g, ok_g = csf.measured_tsdf(dd, w2c, k, mu, pt, center, ctx=gpu_ctx)
        intr = np.array([[k.fx, 0.0], [k.fy, 0.0], [k.cx, 0.0], [k.cy, 0.0]])
        psi_o, ok_o = orc.measured_tsdf(dd, w2c, intr, mu, pt, center)
        assert ok_g[0] and ok_o[0]
        assert psi_g[0, 0] == psi_o[0, 0]
        assert abs(psi_g[0, 1] / hstep - wt / mu) <= 1e-9 * (wt / mu)
        assert abs(psi_g[0, 1] - psi_o[0, 1]) <= 1e-12 * abs(psi_o[0, 1])


@pytest.mark.parametrize("hashed", [False, True])
def test_surface_update_lifted_depth_parity(gpu_ctx, orc, hashed):
    """Three frames fused with depth channels seeded on a patch of pixels (one
    direction each) and a pose channel: fields, weights and hash tables
    against the oracle's surface_update over Image<Lifted<3>>."""
    d, gt, k = orc.workload(1, 3, 80, 60)
    D = 3
    rng = np.random.default_rng(5)
    if hashed:
        params = capi.HashParams(0.04, (C.c_double * 3)(0.0, 0.0, 0.0), 0.12, 128.0, 16, 1 << 14)
        vol_g = csf.HashedVolume(0.04, (0.0, 0.0, 0.0), 0.12, 128.0, 16, 1 << 14, channels=D, ctx=gpu_ctx)
    else:
        params = capi.VolumeParams((C.c_int * 3)(64, 64, 64), 0.04, (C.c_double * 3)(-2.1, -1.28, -0.1), 0.12, 128.0)
        vol_g = csf.TsdfVolume((64, 64, 64), 0.04, (-2.1, -1.28, -0.1), 0.12, 128.0, channels=D, ctx=gpu_ctx)
    vol_o = orc.Volume(params, D, hashed)
    intr = np.zeros((4, 1 + D))
    intr[:, 0] = [k.fx, k.fy, k.cx, k.cy]
    for f in range(3):
        depth = np.zeros((60, 80, 1 + D))
        depth[..., 0] = d[f]
        depth[20:40, 30:50, 1] = 1e-8                      # depth patch (direction 0)
        depth[..., 2] = 1e-8 * rng.uniform(-1, 1, (60, 80)) * (d[f] > 0)  # per-pixel depth noise (direction 1)
        pose = np.zeros((12, 1 + D))
        pose[:, 0] = gt[f]
        pose[9, 3] = 1e-8                                  # camera x (direction 2)
        assert vol_g.surface_update(depth, pose, intr) == vol_o.surface_update(depth, pose, intr)
    if hashed:
        for a, b in zip(vol_g.hash_tables(), vol_o.hash_tables()):
            assert np.array_equal(a, b)
    f_g, w_g = vol_g.download()
    f_o, w_o = vol_o.download()
    assert np.array_equal(w_g, w_o) and np.array_equal(f_g[:, 0], f_o[:, 0])
    s = np.maximum(np.maximum(np.abs(f_g[:, 1:]), np.abs(f_o[:, 1:])), 1e-8)
    assert (np.abs(f_g[:, 1:] - f_o[:, 1:]) <= 1e-9 * s).all()
    assert np.abs(f_g[:, 1]).max() > 1e-10 and np.abs(f_g[:, 2]).max() > 1e-10
