"""Second-order CSFD (BASELINE config 3): the frame loop carried in reference
Bicomplex arithmetic (csfd.hpp:83-140), one parameter pair per Bicomplex, the
csfd_hessian pattern (diff.hpp:58-72) applied to the whole pipeline.

CPU tests pin the oracle's second-order path with the reference's own
bicomplex pin (im1 of a Bicomplex pass is bit-identical to the Complex pass,
test_csfd.cpp:193-204), symmetry of mirrored pairs (to rounding: swapping the
seeds reorders the two cross terms of the im12 product, csfd.hpp:103-108) and
a finite-difference check of a diagonal entry.  GPU tests compare the
packed device run (pairs as channel slots of one evaluation) with the oracle's
one-pass-per-pair run: real channels bit-identical, Hessian entries within
1e-9 relative (mixed scale).
"""
import ctypes as C

import numpy as np
import pytest

import paper_2405_02187_b200 as csf
from paper_2405_02187_b200 import capi

RTOL = 1e-9


def close(a, b, rtol=RTOL, scale=0.0):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    s = np.maximum(np.maximum(np.abs(a), np.abs(b)), scale)
    err = np.abs(a - b) / np.where(s > 0, s, 1.0)
    return bool((np.abs(a - b) <= rtol * s).all()), float(err.max()) if a.size else 0.0


def dense_params(n=64, vs=0.04):
    return capi.VolumeParams((C.c_int * 3)(n, n, n), vs, (C.c_double * 3)(-2.1, -1.28, -0.1), 3 * vs, 128.0)


def cfg_dense(k, n, pairs=None, dirs=(), h=1e-8):
    return csf.make_pipeline_cfg(hashed=False, k=k, dirs=list(dirs), h=h, objective=capi.OBJECTIVE_TRAJECTORY_ERROR,
                                 max_frames=n, dense=dense_params(), pairs=pairs)


def cfg_hashed(k, n, pairs=None, dirs=(), h=1e-8):
    hp = capi.HashParams(0.02, (C.c_double * 3)(0.0, 0.0, 0.0), 0.1, 128.0, 20, 1 << 16)
    return csf.make_pipeline_cfg(hashed=True, k=k, dirs=list(dirs), h=h, objective=capi.OBJECTIVE_TRAJECTORY_ERROR,
                                 max_frames=n, hash_params=hp, pairs=pairs)


@pytest.fixture(scope="module")
def orc(oracle_built):
    from oracle import orc as o
    return o


# ----------------------------------------------------------------------------- oracle (CPU)
def test_oracle_bicomplex_pins(orc):
    """im1/im2 of every pair equal the Complex (first-order) pass bit for bit;
    mirrored pairs agree to rounding."""
    n = 3
    d, gt, k = orc.workload(1, n, 80, 60)
    pairs = [(0, 3), (3, 0), (2, 8), (8, 2), (6, 6)]
    H, g1, g2, obj, poses, _, _ = orc.pipeline_hessian(cfg_dense(k, n, pairs=pairs), d, gt)
    g, obj1, poses1, _, _ = orc.pipeline_run(cfg_dense(k, n, dirs=[0, 3, 2, 8, 6]), d, gt)
    first = dict(zip([0, 3, 2, 8, 6], g))
    assert obj == obj1
    assert np.array_equal(poses[..., 0], poses1[..., 0])
    for p, (i, j) in enumerate(pairs):
        assert g1[p] == first[i] and g2[p] == first[j]
    assert close(H[0], H[1], rtol=1e-12)[0] and close(H[2], H[3], rtol=1e-12)[0]
    assert np.all(np.isfinite(H)) and np.abs(H).max() > 0


def test_oracle_hessian_diagonal_fd(orc):
    """H[rho_x, rho_x] against a central difference of the first-order
    gradient.  Left-multiplying the first pose by exp(eps e0) moves along the
    same one-parameter subgroup as the seed, so the difference quotient
    approximates the same second derivative; shifting gt[0] also shifts frame
    0's own objective term (||rho e0||^2), whose curvature 2 is added back."""
    n = 3
    d, gt, k = orc.workload(1, n, 80, 60)
    H, *_ = orc.pipeline_hessian(cfg_dense(k, n, pairs=[(0, 0)]), d, gt)
    eps = 1e-6  # the tracked frames make the third derivative large: 1e-5 leaves a 6e-4 truncation error

    def g0(shift):
        g = gt.copy()
        g[0, 9] += shift
        return orc.pipeline_run(cfg_dense(k, n, dirs=[0]), d, g)[0][0]

    fd = (g0(eps) - g0(-eps)) / (2 * eps) + 2.0
    assert abs(fd - H[0]) < 1e-4 * abs(H[0]), (fd, H[0])


# ----------------------------------------------------------------------------- device parity (B200)
def _device(gpu_ctx, cfg, d, gt):
    pipe = csf.Pipeline(cfg, ctx=gpu_ctx)
    pipe.upload(d, gt)
    pipe.run()
    return pipe.hessian(poses=True, stats=True)


@pytest.mark.gpu
@pytest.mark.parametrize("hashed", [False, True])
def test_pipeline_hessian_parity(gpu_ctx, orc, hashed):
    n = 4
    if hashed:
        d, gt, k = orc.workload(2, n, 160, 120)
        pairs = [(0, 0), (0, 4), (4, 0), (3, 9), (6, 8), (9, 9), (2, 5)]
        cfg = cfg_hashed(k, n, pairs=pairs)
    else:
        d, gt, k = orc.workload(1, n, 80, 60)
        pairs = [(0, 0), (1, 5), (5, 1), (2, 7), (6, 9), (4, 4)]
        cfg = cfg_dense(k, n, pairs=pairs)
    r = _device(gpu_ctx, cfg, d, gt)
    H, g1, g2, obj, poses, stats, _ = orc.pipeline_hessian(cfg, d, gt)
    assert r.objective == obj
    assert np.array_equal(r.poses[..., 0], poses[..., 0])          # real channel bit-identical
    assert np.array_equal(r.stats[:, :2], stats[:, :2])            # iterations, correspondences
    if hashed:
        assert np.array_equal(r.stats[:, 3:5], stats[:, 3:5])      # allocated / visible blocks
    ok, err = close(r.poses[..., 1:], poses[..., 1:], scale=cfg.h * cfg.h)
    assert ok, err
    ok, err = close(r.hessian, H, scale=1e-12)
    assert ok, (err, r.hessian, H)
    ok, err = close(r.grad1, g1, scale=1e-12)
    assert ok, err
    ok, err = close(r.grad2, g2, scale=1e-12)
    assert ok, err
    assert np.all(np.isfinite(r.hessian)) and np.abs(r.hessian).max() > 0


@pytest.mark.gpu
def test_pipeline_hessian_properties(gpu_ctx, orc):
    """Device-only properties at a larger size: mirrored pairs agree (to
    rounding) and each pair's im1/im2 derivatives equal the first-order packed
    run."""
    n = 6
    d, gt, k = csf.synth_workload(2, n, 320, 240, ctx=gpu_ctx)
    pairs = [(0, 6), (6, 0), (1, 1), (7, 3), (3, 7)]
    r = _device(gpu_ctx, cfg_hashed(k, n, pairs=pairs), d, gt)
    assert close(r.hessian[0], r.hessian[1], rtol=1e-10)[0] and close(r.hessian[3], r.hessian[4], rtol=1e-10)[0]
    pipe = csf.Pipeline(cfg_hashed(k, n, dirs=[0, 6, 1, 7, 3]), ctx=gpu_ctx)
    pipe.upload(d, gt)
    pipe.run()
    g = dict(zip([0, 6, 1, 7, 3], pipe.result().gradient))
    for p, (i, j) in enumerate(pairs):
        assert close(r.grad1[p], g[i], scale=1e-12)[0] and close(r.grad2[p], g[j], scale=1e-12)[0]


@pytest.mark.gpu
def test_pipeline_hessian_all_pairs_launches(gpu_ctx, orc):
    """BASELINE config 3's width — all 55 pairs of the 10 directions (165
    bicomplex slots) — on a small hashed run: every kernel launches at that
    channel count (an integrate launch once failed there on the 48 KB
    shared-memory threshold), the real channel matches the first-order run
    bit for bit and mirrored pairs agree."""
    n = 3
    d, gt, k = orc.workload(2, n, 160, 120)
    pairs = [(i, j) for i in range(10) for j in range(i, 10)]
    r = _device(gpu_ctx, cfg_hashed(k, n, pairs=pairs), d, gt)
    p1 = csf.Pipeline(cfg_hashed(k, n, dirs=list(range(10))), ctx=gpu_ctx)
    p1.upload(d, gt)
    p1.run()
    first = p1.result()
    assert r.objective == first.objective
    assert np.array_equal(r.poses[..., 0], first.poses[..., 0])
    assert np.all(np.isfinite(r.hessian)) and np.abs(r.hessian).max() > 0
    for p, (i, j) in enumerate(pairs):
        s = max(abs(first.gradient[i]), abs(first.gradient[j]), 1e-12)
        assert abs(r.grad1[p] - first.gradient[i]) <= 1e-9 * s and abs(r.grad2[p] - first.gradient[j]) <= 1e-9 * s
