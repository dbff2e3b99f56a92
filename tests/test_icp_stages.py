"""The reference's remaining hot-path stage functions through the C-ABI on
the device: associate (icp.cpp:89-126), linearized_step (icp.cpp:146-153),
pairwise_sum (diff.hpp:16-37); plus the host-side depth lifts complex_depth /
perturb_depth (frames.cpp:77-102) with the reference's error behaviour
(test_frames.cpp perturb_depth cases).  Results are bit-identical to the CPU
oracle."""
import numpy as np
import pytest

import paper_2405_02187_b200 as csf
from paper_2405_02187_b200 import capi


def test_perturb_depth_rules():
    d = np.full((6, 8), 2.0)
    out = csf.perturb_depth(d, 3, 2, h=1e-8)
    assert out.shape == (6, 8, 2) and out[2, 3, 1] == 1e-8 and np.count_nonzero(out[..., 1]) == 1
    assert np.array_equal(out[..., 0], d)
    with pytest.raises(csf.InvalidArgument):
        csf.perturb_depth(d, 8, 0)            # out of bounds
    z = d.copy()
    z[2, 3] = 0.0
    with pytest.raises(csf.InvalidArgument):
        csf.perturb_depth(z, 3, 2)            # no depth
    e = d.copy()
    e[2, 4] = 2.2
    with pytest.raises(csf.InvalidArgument):
        csf.perturb_depth(e, 3, 2)            # discontinuity beyond delta_edge
    csf.perturb_depth(e, 3, 2, delta_edge=0.25)
    csf.perturb_depth(d, 0, 0)                # border pixel: out-of-bounds neighbours are skipped
    with pytest.raises(csf.InvalidArgument):
        csf.perturb_depth(d, 1, 1, h=0.0)     # StepSize


def test_oracle_pairwise_sum_shape(oracle_built):
    from oracle import orc
    rng = np.random.default_rng(0)
    t = rng.normal(size=37)
    assert abs(orc.pairwise_sum(t) - t.sum()) < 1e-12
    assert orc.pairwise_sum([]) == 0.0


@pytest.mark.gpu
@pytest.mark.parametrize("n", [0, 1, 8, 9, 31, 1000, 100003])
def test_pairwise_sum_bit_exact(gpu_ctx, oracle_built, n):
    from oracle import orc
    rng = np.random.default_rng(n)
    t = rng.normal(size=n) * np.exp(rng.normal(size=n) * 5)
    assert csf.pairwise_sum(t, ctx=gpu_ctx) == orc.pairwise_sum(t)
    lanes = rng.normal(size=(n, 3))
    out = csf.pairwise_sum(lanes, ctx=gpu_ctx)
    for c in range(3):
        assert out[c] == orc.pairwise_sum(lanes[:, c])


@pytest.mark.gpu
def test_associate_and_linearized_step(gpu_ctx, oracle_built):
    from oracle import orc
    d, gt, k = orc.workload(1, 5, 160, 120)
    vol = csf.TsdfVolume((128, 128, 128), 0.02, (-2.1, -1.28, -0.1), 0.06, 128.0, channels=0, ctx=gpu_ctx)
    intr = np.array([[k.fx], [k.fy], [k.cx], [k.cy]])
    for i in range(4):
        vol.surface_update(d[i].astype(np.float64), gt[i].reshape(12, 1), intr)
    V, N = vol.raycast(gt[3], intr, 160, 120)
    pv, pn = V[..., 0], N[..., 0]
    dm = np.zeros((120, 160, 2))
    dm[..., 0] = csf.bilateral_filter(d[4].astype(np.float64), ctx=gpu_ctx)
    mv, mn = csf.measure_surface(dm, np.c_[intr, np.zeros((4, 1))], ctx=gpu_ctx)
    mv, mn = mv[..., 0], mn[..., 0]
    cfg = csf.default_icp_cfg()
    for stride in (1, 2):
        c_g = csf.associate((mv, mn), (pv, pn), gt[4], gt[3], k, cfg, stride, ctx=gpu_ctx)
        c_o = orc.associate(mv, mn, pv, pn, gt[4], gt[3], k, cfg, stride)
        assert c_g.shape[0] > 1000 and np.array_equal(c_g, c_o)
    d_g = csf.linearized_step(c_g, gt[4], ctx=gpu_ctx)
    assert np.array_equal(d_g, orc.linearized_step(c_o, gt[4]))
    seq = orc.linearized_step(c_o, gt[4], sequential=True)   # the reference's literal sequential sum
    assert np.allclose(d_g, seq, rtol=1e-9, atol=1e-14)
    assert np.array_equal(csf.linearized_step(np.zeros((0, 9)), gt[4], ctx=gpu_ctx), np.zeros(6))
