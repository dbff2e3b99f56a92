"""The C-ABI's threading and host-buffer contract (include/csf_b200.h):

  * different contexts (one per GPU or host thread) may run concurrently —
    here two contexts on one device, each driven from its own host thread,
    give exactly the serial results (function attributes and device
    properties are cached per device, launch errors per host thread);
  * host buffers are only borrowed for the duration of a call — a pinned
    destination handed to csf_pipeline_result holds the final values when
    the call returns;
  * an empty frame is rejected up front (CSF_EINVAL -> ValueError), and
    frames above VGA (multi-segment ICP tiles) track exactly like the oracle.
"""
import ctypes as C
import threading

import numpy as np
import pytest

import paper_2405_02187_b200 as csf
from paper_2405_02187_b200 import capi

pytestmark = pytest.mark.gpu


def _cfg(k, n, dirs):
    hp = capi.HashParams(0.02, (C.c_double * 3)(0.0, 0.0, 0.0), 0.1, 128.0, 20, 1 << 16)
    return csf.make_pipeline_cfg(hashed=True, k=k, dirs=dirs, h=1e-8, objective=capi.OBJECTIVE_TRAJECTORY_ERROR,
                                 max_frames=n, hash_params=hp)


def _run(ctx, cfg, d, gt, reps=1):
    p = csf.Pipeline(cfg, ctx=ctx)
    p.upload(d, gt)
    out = None
    for _ in range(reps):
        p.run()
        out = p.result()
    p.close()
    return out


def test_two_contexts_concurrently(oracle_built):
    from oracle import orc
    n = 5
    d, gt, k = orc.workload(2, n, 160, 120)
    cfg_a = _cfg(k, n, list(range(10)))
    cfg_b = _cfg(k, n, [0, 3, 7])
    ctx_a, ctx_b = csf.Context(0), csf.Context(0)
    serial_a = _run(ctx_a, cfg_a, d, gt)
    serial_b = _run(ctx_b, cfg_b, d, gt)
    results = {}
    errors = []

    def worker(name, ctx, cfg):
        try:
            results[name] = _run(ctx, cfg, d, gt, reps=3)
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    ts = [threading.Thread(target=worker, args=("a", ctx_a, cfg_a)),
          threading.Thread(target=worker, args=("b", ctx_b, cfg_b))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    for name, ref in (("a", serial_a), ("b", serial_b)):
        r = results[name]
        assert r.objective == ref.objective
        assert np.array_equal(r.gradient, ref.gradient)
        assert np.array_equal(r.poses, ref.poses) and np.array_equal(r.stats, ref.stats)
    # packing is exact: the 3-direction context's columns are the 10-direction run's
    assert np.array_equal(serial_b.gradient, serial_a.gradient[[0, 3, 7]])


def test_pinned_result_buffers(gpu_ctx, oracle_built):
    import torch
    from oracle import orc
    n = 4
    d, gt, k = orc.workload(2, n, 160, 120)
    cfg = _cfg(k, n, list(range(10)))
    p = csf.Pipeline(cfg, ctx=gpu_ctx)
    p.upload(d, gt)
    p.run()
    ref = p.result()
    grad = torch.zeros(10, dtype=torch.float64).pin_memory()
    poses = torch.zeros((n, 12, 11), dtype=torch.float64).pin_memory()
    stats = torch.zeros((n, 8), dtype=torch.int32).pin_memory()
    obj = C.c_double()
    for _ in range(3):
        p.run()  # queued work ahead of the read-back
        gpu_ctx.check(gpu_ctx.lib.csf_pipeline_result(
            p.h, C.cast(grad.data_ptr(), C.POINTER(C.c_double)), C.byref(obj),
            C.cast(poses.data_ptr(), C.POINTER(C.c_double)), C.cast(stats.data_ptr(), C.POINTER(C.c_int32))))
        # read immediately: the call must have completed the copies
        assert np.array_equal(grad.numpy(), ref.gradient)
        assert np.array_equal(poses.numpy(), ref.poses) and np.array_equal(stats.numpy(), ref.stats)
        assert obj.value == ref.objective
        grad.zero_()
        poses.zero_()
        stats.zero_()


def test_empty_frame_rejected(gpu_ctx):
    """A frame with no pixels is rejected up front (CSF_EINVAL -> ValueError)."""
    k = csf.intrinsics(100.0, 100.0, 0.0, 0.0, 0, 0)
    hp = capi.HashParams(0.02, (C.c_double * 3)(0.0, 0.0, 0.0), 0.1, 128.0, 16, 1 << 10)
    cfg = csf.make_pipeline_cfg(hashed=True, k=k, dirs=[0], h=1e-8, objective=capi.OBJECTIVE_TRAJECTORY_ERROR,
                                max_frames=1, hash_params=hp)
    with pytest.raises(ValueError):
        csf.Pipeline(cfg, ctx=gpu_ctx)


def test_multi_segment_tiles_1280x960(gpu_ctx, oracle_built):
    """Frames above VGA make the ICP tiles longer than one shared-memory
    segment (1280x960: 307200 slots at levels 0 and 1, 2080-slot tiles, four
    segments), and 20 directions (the 10 of config 2 plus the keyframe twists
    of frames 1 and 2) need two channel passes of the 16 warps: the level
    kernel re-measures and re-associates per segment and pass.  Real channel,
    stats and hash tables bit-identical to the oracle, derivatives within 1e-9."""
    from oracle import orc
    n = 3
    d, gt, k = orc.workload(2, n, 1280, 960)
    hp = capi.HashParams(0.01, (C.c_double * 3)(0.0, 0.0, 0.0), 0.05, 128.0, 20, 1 << 17)
    cfg = csf.make_pipeline_cfg(hashed=True, k=k, dirs=list(range(20)), h=1e-8,
                                objective=capi.OBJECTIVE_TRAJECTORY_ERROR, max_frames=n, hash_params=hp,
                                keyframe_interval=1)
    p = csf.Pipeline(cfg, ctx=gpu_ctx)
    p.upload(d, gt)
    p.run()
    r = p.result()
    g_o, obj_o, poses_o, stats_o, vol_o = orc.pipeline_run_keep(cfg, d, gt)
    assert r.objective == obj_o
    assert np.array_equal(r.poses[..., 0], poses_o[..., 0])
    assert np.array_equal(r.stats[:, :7], stats_o[:, :7])
    for x, y in zip(p.volume().hash_tables(), vol_o.hash_tables()):
        assert np.array_equal(x, y)
    s = np.maximum(np.maximum(np.abs(r.gradient), np.abs(g_o)), 1e-12)
    assert (np.abs(r.gradient - g_o) <= 1e-9 * s).all(), (r.gradient, g_o)
    assert r.stats[1:, 1].min() > 100
