"""The deterministic elementary functions on the device path
(include/csf_detmath.h: exp for the bilateral weights, frames.cpp:28-29;
sin/cos for exp_map, se3.hpp:84-96, and the association gate cos(30 deg),
icp.cpp:97) against glibc 2.39's exp/sin/cos — what the reference links —
over the argument ranges the path feeds them.  The device and the oracle use
the same header, so every real channel is bit-identical between them; this
pins how far that shared arithmetic is from the reference's libm: at most
2 ulp everywhere tested, and exactly equal on most arguments."""
import math

import numpy as np
import pytest


@pytest.fixture(scope="module")
def orc(oracle_built):
    from oracle import orc as o
    return o


def _pin(orc, fn, x, max_ulp=2.0):
    u, d, g = orc.detmath_ulp(fn, x)
    assert np.all(np.isfinite(d) == np.isfinite(g))
    worst = float(u.max()) if u.size else 0.0
    assert worst <= max_ulp, (fn, worst, x[np.argmax(u)])
    return u


def test_exp_bilateral_ranges(orc):
    rng = np.random.default_rng(0)
    # spatial weights: -(dx^2 + dy^2) / (2 sigma_s^2), |dx|, |dy| <= 3, sigma_s = 4.5
    spatial = np.array([-(dx * dx + dy * dy) / (2.0 * 4.5 * 4.5) for dy in range(-3, 4) for dx in range(-3, 4)])
    _pin(orc, "exp", spatial)
    # range weights: -(q - c)^2 / (2 sigma_r^2), sigma_r = 0.03, depth steps up to 20 m; into underflow
    dq = np.concatenate([rng.uniform(0.0, 0.1, 200000), rng.uniform(0.0, 20.0, 100000)])
    u = _pin(orc, "exp", -(dq * dq) / (2.0 * 0.03 * 0.03))
    assert (u == 0).mean() > 0.5
    _pin(orc, "exp", rng.uniform(-745.0, 0.0, 100000))
    _pin(orc, "exp", np.array([0.0, -0.0, -1e-300, -708.0, -745.1, -800.0]))


def test_sin_cos_exp_map_ranges(orc):
    rng = np.random.default_rng(1)
    for x in (rng.uniform(-1e-3, 1e-3, 100000),           # ICP increments (theta, theta / 2)
              rng.uniform(-math.pi, math.pi, 200000),      # seeded / keyframe twists, view poses
              rng.uniform(0.0, 400.0, 100000),             # config-4 terrain waves k . (x, y) + phase
              np.array([0.0, 1e-300, math.pi / 6, math.pi / 2, math.pi])):
        for fn in ("sin", "cos"):
            _pin(orc, fn, x)


def test_association_gate_constant(orc):
    """cos(30 deg) of the association angle gate (icp.cpp:97) is the correctly
    rounded value on both sides."""
    u, d, g = orc.detmath_ulp("cos", np.array([30.0 * math.pi / 180.0]))
    assert d[0] == g[0] and u[0] == 0.0


def _runs(orc, cfg, d, gt):
    det = orc.pipeline_run(cfg, d, gt)
    orc.use_libm(True)
    try:
        libm = orc.pipeline_run(cfg, d, gt)
    finally:
        orc.use_libm(False)
    return det, libm


@pytest.mark.parametrize("config", [1, 2])
def test_libm_oracle_agrees(orc, config):
    """The whole pipeline with glibc's exp/sin/cos (-DORC_LIBM, the
    reference's libm) against the default csf_detmath build on the same
    inputs: identical discrete decisions (ICP iterations, correspondences,
    allocated / visible / new blocks, fused voxels) and real poses, objective
    and gradient within 1e-9 relative.  (config 1 at its stated size, 5
    frames; config 2 at 320x240, 4 frames, 5 mm hashed.)"""
    import bench
    import paper_2405_02187_b200 as csf
    from paper_2405_02187_b200 import capi
    if config == 1:
        d, gt, k = orc.workload(1, 5)
        cfg = bench.pipeline_cfg1(csf, capi, k, list(range(6)), 5)
    else:
        d, gt, k = orc.workload(2, 4, 320, 240)
        cfg = bench.pipeline_cfg(csf, capi, k, bench.DIRS, 4)
    (g0, o0, p0, s0, _), (g1, o1, p1, s1, _) = _runs(orc, cfg, d, gt)
    assert np.array_equal(s0[:, :7], s1[:, :7])
    assert abs(o0 - o1) <= 1e-9 * abs(o0)
    assert np.abs(p0[..., 0] - p1[..., 0]).max() <= 1e-9
    sc = np.maximum(np.abs(g0), 1e-12)
    assert (np.abs(g0 - g1) <= 1e-9 * sc).all(), (g0, g1)
