"""Edge cases through the C-ABI on the device, against the oracle where a
value is produced: empty (all-invalid) and ragged (odd-sized, tiny) frames,
holes, the hashed pool at capacity, the zero-real-part divisor, argument
validation (SURVEY §8(b) error convention)."""
import numpy as np
import pytest

import paper_2405_02187_b200 as csf
from paper_2405_02187_b200 import capi

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("w,h", [(1, 1), (2, 3), (7, 5), (33, 17), (161, 121)])
def test_ragged_frames_bit_exact(gpu_ctx, oracle_built, w, h):
    from oracle import orc
    rng = np.random.default_rng(w * 1000 + h)
    d = rng.uniform(0.5, 4.0, (h, w))
    d[rng.random((h, w)) < 0.2] = 0.0  # holes
    assert np.array_equal(csf.bilateral_filter(d, ctx=gpu_ctx), orc.bilateral_filter(d))
    if w >= 2 and h >= 2:
        assert np.array_equal(csf.downsample_depth(d, ctx=gpu_ctx), orc.downsample_depth(d))
    intr = np.array([[20.0], [21.0], [w / 2.0], [h / 2.0]])
    vg, ng = csf.measure_surface(d, intr, ctx=gpu_ctx)
    vo, no = orc.measure_surface(d.reshape(h, w, 1), intr)
    assert np.array_equal(vg.reshape(-1), vo.reshape(-1)) and np.array_equal(ng.reshape(-1), no.reshape(-1))


def test_all_invalid_frame(gpu_ctx, oracle_built):
    """A frame with no valid pixel: filters return zeros, fusion observes
    nothing, the raycast misses everywhere, tracking stops on < 12
    correspondences (icp.cpp:199) and returns the initial pose."""
    w, h = 80, 60
    k = csf.intrinsics(60.0, 60.0, 39.5, 29.5, w, h)
    zero = np.zeros((h, w))
    assert not csf.bilateral_filter(zero, ctx=gpu_ctx).any()
    vol = csf.TsdfVolume((32, 32, 32), 0.05, (-0.8, -0.8, 0.2), 0.15, 128.0, channels=0, ctx=gpu_ctx)
    eye = np.array([1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0], dtype=np.float64)
    vol.surface_update(zero, eye, k)
    f, wts = vol.download()
    assert not wts.any() and np.all(f.reshape(-1) == 1.0)
    V, N = vol.raycast(eye, k, w, h)
    assert not V.any() and not N.any()
    r = csf.track_frame(vol, zero, eye, k)
    assert np.array_equal(r.pose, eye) and r.iterations == 0 and not r.converged
    hv = csf.HashedVolume(0.01, (0.0, 0.0, 0.0), 0.05, 128.0, 12, 1 << 10, channels=0, ctx=gpu_ctx)
    assert hv.surface_update(zero, eye, k) == 0 and hv.block_count() == 0


def test_hashed_pool_exhaustion_raises(gpu_ctx, oracle_built):
    """More band blocks than the pool holds: the capacity error surfaces as a
    RuntimeError (std::runtime_error), never as silent truncation."""
    from oracle import orc
    d, gt, k = orc.workload(2, 1, 160, 120)
    hv = csf.HashedVolume(0.005, (0.0, 0.0, 0.0), 0.025, 128.0, 12, 16, channels=0, ctx=gpu_ctx)
    with pytest.raises(RuntimeError):
        hv.surface_update(d[0].astype(np.float64), gt[0], k)


def test_zero_real_divisor_is_a_domain_error(gpu_ctx):
    """Complex division by a zero real part throws std::domain_error
    (csfd.hpp:52-58); a lifted intrinsic fx = 0 divides by it."""
    d = np.full((8, 8), 1.0)
    intr = np.array([[0.0, 1e-8], [10.0, 0.0], [4.0, 0.0], [4.0, 0.0]])
    with pytest.raises(csf.DomainError):
        csf.measure_surface(np.stack([d, np.zeros_like(d)], -1), intr, ctx=gpu_ctx)
    vol = csf.TsdfVolume((16, 16, 16), 0.05, (0.0, 0.0, 0.0), 0.15, 128.0, channels=1, ctx=gpu_ctx)
    eye = np.zeros((12, 2))
    eye[[0, 4, 8], 0] = 1.0
    with pytest.raises(csf.DomainError):
        vol.surface_update(d, eye, intr)
    with pytest.raises(csf.DomainError):
        vol.raycast(eye, intr, 8, 8)


def test_argument_validation(gpu_ctx):
    """Bad inputs are std::invalid_argument (InvalidArgument) at the boundary."""
    k = csf.intrinsics(60.0, 60.0, 39.5, 29.5, 80, 60)
    with pytest.raises(csf.InvalidArgument):
        csf.bilateral_filter(np.ones((16, 16)), radius=9, ctx=gpu_ctx)
    vol = csf.TsdfVolume((16, 16, 16), 0.05, (0.0, 0.0, 0.0), 0.15, 128.0, channels=0, ctx=gpu_ctx)
    with pytest.raises(csf.InvalidArgument):
        csf.track_frame(vol, np.ones((60, 80)), np.eye(4), k, cfg=csf.default_icp_cfg(solver=capi.SOLVER_NEWTON, h=1e-3))
    with pytest.raises(csf.InvalidArgument):
        csf.lift_pose(np.zeros(7))
    with pytest.raises(csf.InvalidArgument):
        csf.perturb_depth(np.ones((4, 4)), 1, 1, h=1e-3)


def test_run_host_rejects_more_frames_than_configured(gpu_ctx, oracle_built):
    """csf_pipeline_run_host validates the frame count against max_frames
    before any upload (std::invalid_argument at the boundary), and the
    pipeline stays usable afterwards."""
    from oracle import orc
    n = 3
    d, gt, k = orc.workload(2, n + 1, 160, 120)
    hp = capi.HashParams(0.02, (capi.C.c_double * 3)(0.0, 0.0, 0.0), 0.1, 128.0, 16, 1 << 14)
    cfg = csf.make_pipeline_cfg(hashed=True, k=k, dirs=[0, 1], h=1e-8, objective=1, max_frames=n, hash_params=hp)
    pipe = csf.Pipeline(cfg, ctx=gpu_ctx)
    with pytest.raises(csf.InvalidArgument):
        pipe.run_host(d, gt)
    r = pipe.run_host(d[:n], gt[:n])
    pipe.upload(d[:n], gt[:n])
    pipe.run()
    s = pipe.result()
    assert r.objective == s.objective and np.array_equal(r.gradient, s.gradient)
