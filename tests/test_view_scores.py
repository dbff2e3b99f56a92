"""BASELINE config 5: active-scanning view scoring (builder-defined objective;
DESIGN.md §3.7).  Each candidate view is raycast through the fused hashed TSDF
with its pose lifted on the 6 twist channels; the score is the pairwise_sum
(diff.hpp:16-37) of sigma(beta (w0 - W~(p))) over the view's raycast hits.
The device is compared with the CPU oracle (one Lifted<6> pass per view):
scores bit-identical (every real operation in the oracle's order), gradients
within 1e-9 relative."""
import numpy as np
import pytest

import paper_2405_02187_b200 as csf
from paper_2405_02187_b200 import capi


def test_config5_views_are_valid_poses():
    v = csf.config5_views(16, seed=4)
    assert v.shape == (16, 12)
    R = v[:, :9].reshape(-1, 3, 3)
    assert np.allclose(R @ R.transpose(0, 2, 1), np.eye(3), atol=1e-12)
    assert np.allclose(np.linalg.det(R), 1.0)
    assert np.array_equal(v, csf.config5_views(16, seed=4))


@pytest.mark.gpu
def test_view_scores_parity(gpu_ctx, oracle_built):
    from oracle import orc
    n = 6
    d, gt, k = orc.workload(2, n, 160, 120)
    hp = capi.HashParams(0.02, (capi.C.c_double * 3)(0.0, 0.0, 0.0), 0.1, 128.0, 20, 1 << 16)
    vol_g = csf.HashedVolume(0.02, (0.0, 0.0, 0.0), 0.1, 128.0, 20, 1 << 16, channels=6, ctx=gpu_ctx)
    vol_o = orc.Volume(hp, 6, True)
    intr = np.zeros((4, 7))
    intr[:, 0] = [k.fx, k.fy, k.cx, k.cy]
    for i in range(n):
        pose = np.zeros((12, 7))
        pose[:, 0] = gt[i]
        vol_g.surface_update(d[i].astype(np.float64), pose, intr)
        vol_o.surface_update(d[i].astype(np.float64), pose, intr)
    kv = csf.intrinsics(k.fx / 2, k.fy / 2, k.cx / 2, k.cy / 2, 80, 60)
    views = np.concatenate([gt[[1, 3]], csf.config5_views(4, seed=4)])
    s_g, g_g = vol_g.view_scores(views, kv, w0=10.0, beta=0.5)
    s_o, g_o = vol_o.view_scores(views, kv, w0=10.0, beta=0.5)
    assert np.array_equal(s_g, s_o)
    scale = np.maximum(np.abs(g_o), 1e-6 * np.abs(s_o)[:, None] + 1e-12)
    assert (np.abs(g_g - g_o) <= 1e-9 * scale).all(), np.abs(g_g - g_o).max()
    assert (s_g[:2] > 0).all() and np.abs(g_g[:2]).max() > 0
