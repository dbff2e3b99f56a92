"""Point queries of the stage API on the device against the oracle:
sample_tsdf / sample_gradient (tsdf.hpp:148-196) at lifted world points of a
fused volume (dense and hashed) and measured_tsdf (tsdf.hpp:97-140) at voxel
positions.  Real parts and validity bit-identical; channels within 1e-9
relative (the first-order trilinear/lifted paths round differently by ~1 ulp).
Reference pins restated: a point in free space far from any observation has
no sample (test_tsdf.cpp:343), a sample needs all 8 corners observed."""
import numpy as np
import pytest

import paper_2405_02187_b200 as csf
from paper_2405_02187_b200 import capi

pytestmark = pytest.mark.gpu


def close(a, b, scale):
    s = np.maximum(np.maximum(np.abs(a), np.abs(b)), scale)
    return bool((np.abs(a - b) <= 1e-9 * s).all())


@pytest.mark.parametrize("hashed", [False, True])
def test_sample_points_parity(gpu_ctx, oracle_built, hashed):
    from oracle import orc
    d, gt, k = orc.workload(1, 3, 80, 60)
    D = 2
    rng = np.random.default_rng(7)
    if hashed:
        params = capi.HashParams(0.04, (capi.C.c_double * 3)(0.0, 0.0, 0.0), 0.12, 128.0, 16, 1 << 14)
        vg = csf.HashedVolume(0.04, (0.0, 0.0, 0.0), 0.12, 128.0, 16, 1 << 14, channels=D, ctx=gpu_ctx)
    else:
        params = capi.VolumeParams((capi.C.c_int * 3)(64, 64, 64), 0.04, (capi.C.c_double * 3)(-2.1, -1.28, -0.1),
                                   0.12, 128.0)
        vg = csf.TsdfVolume((64, 64, 64), 0.04, (-2.1, -1.28, -0.1), 0.12, 128.0, channels=D, ctx=gpu_ctx)
    vo = orc.Volume(params, D, hashed)
    intr = np.zeros((4, 1 + D))
    intr[:, 0] = [k.fx, k.fy, k.cx, k.cy]
    for i in range(3):
        pose = np.zeros((12, 1 + D))
        pose[:, 0] = gt[i]
        pose[:, 1:] = rng.uniform(-1, 1, (12, D)) * 1e-8
        vg.surface_update(d[i].astype(np.float64), pose, intr)
        vo.surface_update(d[i].astype(np.float64), pose, intr)
    # points near the observed surfaces (raycast hits) and random ones
    V, _ = vg.raycast(gt[1], intr, 80, 60)
    hits = V[..., 0].reshape(-1, 3)
    hits = hits[np.abs(hits).sum(1) > 0][:400]
    pts = np.zeros((hits.shape[0] + 200, 3, 1 + D))
    pts[: hits.shape[0], :, 0] = hits + rng.normal(scale=0.01, size=hits.shape)
    pts[hits.shape[0]:, :, 0] = rng.uniform([-2, -2, 0], [2, 2, 3], size=(200, 3))
    pts[..., 1:] = rng.uniform(-1, 1, pts[..., 1:].shape) * 1e-8
    for grad in (False, True):
        if grad:
            g, okg = vg.sample_gradient(pts)
        else:
            g, okg = vg.sample_tsdf(pts)
        o, oko = vo.sample_points(pts, grad=grad)
        assert np.array_equal(okg, oko) and okg.sum() > 100 and (~okg).sum() > 10
        assert np.array_equal(g[okg][..., 0], o[oko][..., 0])
        assert close(g[okg][..., 1:], o[oko][..., 1:], 1e-8)


def test_measured_tsdf_points(gpu_ctx, oracle_built):
    from oracle import orc
    d, gt, k = orc.workload(1, 1, 80, 60)
    D = 2
    rng = np.random.default_rng(3)
    c2w = gt[0]
    R = c2w[:9].reshape(3, 3)
    t = c2w[9:]
    w2c = np.zeros((12, 1 + D))
    w2c[:9, 0] = R.T.reshape(9)
    w2c[9:, 0] = -R.T @ t
    w2c[:, 1:] = rng.uniform(-1, 1, (12, D)) * 1e-8
    intr = np.zeros((4, 1 + D))
    intr[:, 0] = [k.fx, k.fy, k.cx, k.cy]
    intr[0, 1] = 1e-8
    center = np.zeros((3, 1 + D))
    center[:, 0] = t
    pts = t + rng.uniform(-1.5, 1.5, size=(2000, 3)) + R[:, 2] * 1.5
    psi_g, ok_g = csf.measured_tsdf(d[0].astype(np.float64), w2c, intr, 0.12, pts, center, ctx=gpu_ctx)
    psi_o, ok_o = orc.measured_tsdf(d[0].astype(np.float64), w2c, intr, 0.12, pts, center)
    assert np.array_equal(ok_g, ok_o) and ok_g.sum() > 50
    assert np.array_equal(psi_g[ok_g, 0], psi_o[ok_o, 0])
    assert close(psi_g[ok_g, 1:], psi_o[ok_o, 1:], 1e-8)
