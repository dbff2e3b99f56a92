"""The committed golden fixtures (tests/golden/*.npz, made by
tests/golden/make_golden.py from the CPU oracle): the oracle must reproduce
them bit for bit (drift guard, CPU), and the device pipeline must match them
under the parity rule of tests/test_bench_configs.py (GPU): objective, real
pose channel and every decision column bit-identical, channels and the
derivatives within 1e-9 relative.

Cases: BASELINE config 1 at its stated size (10 frames, 160x120, dense 128^3
at 2 cm, h = 1e-20, 6 twist directions) and the config-2 scene at 160x120
(hashed 2 cm, 3 frames, all 10 directions)."""
import ctypes as C
import hashlib
from pathlib import Path

import numpy as np
import pytest

import bench
import paper_2405_02187_b200 as csf
from paper_2405_02187_b200 import capi

GOLDEN = Path(__file__).resolve().parent / "golden"
RTOL = 1e-9


def _case(name, orc, icp):
    if name == "config1_full":
        d, g, k = orc.workload(1, 10)
        return d, g, bench.pipeline_cfg1(csf, capi, k, bench.DIRS1, 10, icp=icp)
    d, g, k = orc.workload(2, 3, 160, 120)
    hp = capi.HashParams(0.02, (C.c_double * 3)(0.0, 0.0, 0.0), 0.1, 128.0, 16, 1 << 14)
    cfg = csf.make_pipeline_cfg(hashed=True, k=k, dirs=bench.DIRS, h=1e-8, objective=capi.OBJECTIVE_TRAJECTORY_ERROR,
                                max_frames=3, hash_params=hp, icp=icp)
    return d, g, cfg


def _load(name):
    z = np.load(GOLDEN / f"{name}.npz")
    return {k: z[k] for k in z.files}


def _rel_ok(a, b, scale):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    s = np.maximum(np.maximum(np.abs(a), np.abs(b)), scale)
    return bool((np.abs(a - b) <= RTOL * s).all())


@pytest.fixture(scope="module")
def orc(oracle_built):
    from oracle import orc as o
    return o


@pytest.mark.parametrize("name", ["config1_full", "config2_small"])
def test_oracle_reproduces_golden(orc, name):
    gold = _load(name)
    d, g, cfg = _case(name, orc, bench.reference_icp())
    assert hashlib.sha256(d.tobytes()).digest() == gold["depth_sha256"].tobytes(), "synthetic input drifted"
    grad, obj, poses, stats, _ = orc.pipeline_run(cfg, d, g)
    assert obj == gold["objective"][0]
    assert np.array_equal(stats, gold["stats"])
    assert np.array_equal(poses, gold["poses"])
    assert np.array_equal(grad, gold["gradient"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["config1_full", "config2_small"])
def test_device_matches_golden(gpu_ctx, orc, name):
    gold = _load(name)
    d, g, cfg = _case(name, orc, None)
    pipe = csf.Pipeline(cfg, ctx=gpu_ctx)
    pipe.upload(d, g)
    pipe.run()
    r = pipe.result()
    assert r.objective == gold["objective"][0]
    assert np.array_equal(r.stats[:, :7], gold["stats"][:, :7])
    assert np.array_equal(r.poses[..., 0], gold["poses"][..., 0])
    assert _rel_ok(r.poses[..., 1:], gold["poses"][..., 1:], cfg.h)
    assert _rel_ok(r.gradient, gold["gradient"], 1e-12)
