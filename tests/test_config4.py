"""BASELINE config 4 pieces (builder-defined): the terrain
heightfield scene (sum of plane waves, Lipschitz-safe distance bound) rendered
identically by the device harness and the oracle, and keyframe perturbation
directions (codes 10 + 6 (kf - 1) + c: exp(xi) applied to the tracked pose of
keyframe kf before fusion) — real channel bit-identical to the oracle,
derivatives within 1e-9."""
import ctypes as C

import numpy as np
import pytest

import paper_2405_02187_b200 as csf
from paper_2405_02187_b200 import capi


@pytest.fixture(scope="module")
def orc(oracle_built):
    from oracle import orc as o
    return o


def test_config4_oracle_scene(orc):
    d, gt, k = orc.workload(4, 2, 80, 60)
    assert (d > 0).mean() > 0.7
    v = d[d > 0]
    assert v.min() >= 0.3 and v.max() < 21.0
    step = np.linalg.norm(gt[1, 9:] - gt[0, 9:])
    assert 0.05 < step < 0.08


def _cfg(k, n, dirs):
    hp = capi.HashParams(0.02, (C.c_double * 3)(0.0, 0.0, 0.0), 0.1, 128.0, 20, 1 << 17)
    return csf.make_pipeline_cfg(hashed=True, k=k, dirs=dirs, h=1e-8, objective=capi.OBJECTIVE_TRAJECTORY_ERROR,
                                 max_frames=n, hash_params=hp, keyframe_interval=2)


def test_keyframe_directions_oracle(orc):
    """Keyframe seeds on the CPU oracle: packing is exact per channel and a
    keyframe direction only moves the trajectory from its keyframe on."""
    n = 5
    d, gt, k = orc.workload(4, n, 80, 60)
    dirs = [0, 10, 16, 21]
    g, obj, poses, _, _ = orc.pipeline_run(_cfg(k, n, dirs), d, gt)
    g1, _, poses1, _, _ = orc.pipeline_run(_cfg(k, n, [16]), d, gt)
    assert np.array_equal(poses[..., 0], poses1[..., 0])
    assert g[2] == g1[0]
    assert np.all(poses[:2, :, 2] == 0.0) and np.all(poses[:4, :, 3] == 0.0)   # kf1 = frame 2, kf2 = frame 4
    assert np.abs(poses[2:, :, 2]).max() > 0 and np.abs(poses[4:, :, 3]).max() > 0


@pytest.mark.gpu
def test_config4_synth_bit_exact(gpu_ctx, orc):
    d_g, gt_g, _ = csf.synth_workload(4, 2, 160, 120, ctx=gpu_ctx)
    d_o, gt_o, _ = orc.workload(4, 2, 160, 120)
    assert np.array_equal(gt_g, gt_o)
    assert np.array_equal(d_g, d_o)


@pytest.mark.gpu
def test_keyframe_pipeline_parity(gpu_ctx, orc):
    n = 5
    d, gt, k = orc.workload(4, n, 160, 120)
    cfg = _cfg(k, n, [0, 3, 6, 10, 15, 16, 21])
    pipe = csf.Pipeline(cfg, ctx=gpu_ctx)
    pipe.upload(d, gt)
    pipe.run()
    r = pipe.result()
    g_o, obj_o, poses_o, stats_o, _ = orc.pipeline_run(cfg, d, gt)
    assert r.objective == obj_o
    assert np.array_equal(r.poses[..., 0], poses_o[..., 0])
    assert np.array_equal(r.stats[:, :2], stats_o[:, :2])
    assert np.array_equal(r.stats[:, 3:5], stats_o[:, 3:5])
    s = np.maximum(np.maximum(np.abs(r.poses[..., 1:]), np.abs(poses_o[..., 1:])), 1e-8)
    assert (np.abs(r.poses[..., 1:] - poses_o[..., 1:]) <= 1e-9 * s).all()
    s = np.maximum(np.maximum(np.abs(r.gradient), np.abs(g_o)), 1e-12)
    assert (np.abs(r.gradient - g_o) <= 1e-9 * s).all(), (r.gradient, g_o)
