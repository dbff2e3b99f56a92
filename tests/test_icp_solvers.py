"""ICP energy, its CSFD derivatives and every tracker solver on the device.

icp_energy (icp.hpp:70-85) sums r^2 with the reference's pairwise_sum tree
(diff.hpp:16-37); icp_gradient / icp_hessian (icp.cpp:132-144) are the 6
Complex / 21 Bicomplex passes of csfd_gradient / csfd_hessian, evaluated on
the device as one packed pass.  track_frame (icp.cpp:169-244) runs the
reference's solver families: linearized, Newton (Levenberg damping + -g line
search, descent.hpp:109-144), gradient descent and Polak-Ribiere NCG
(descent.hpp:58-101).  The energy and the real track are compared bit for bit
with the CPU oracle; derivative channels within 1e-12 relative.
"""
import numpy as np
import pytest

import paper_2405_02187_b200 as csf
from paper_2405_02187_b200 import capi

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def orc(oracle_built):
    from oracle import orc as o
    return o


def _rot(rng):
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def _corrs(rng, n):
    v = rng.uniform(-1, 1, size=(n, 3)) + np.array([0, 0, 2.0])
    mv = v + rng.normal(scale=0.01, size=(n, 3))
    mn = rng.normal(size=(n, 3))
    mn /= np.linalg.norm(mn, axis=1, keepdims=True)
    return np.concatenate([v, mv, mn], axis=1)


@pytest.mark.parametrize("n", [0, 1, 8, 9, 17, 300, 4099, 76800])
def test_icp_energy_derivs_parity(gpu_ctx, orc, n):
    rng = np.random.default_rng(n)
    corrs = _corrs(rng, n)
    base = np.concatenate([_rot(rng).reshape(9), rng.uniform(-1, 1, 3)])
    for xi in (None, rng.normal(scale=1e-3, size=6)):
        E, g, H = csf.icp_energy_derivs(corrs, base, xi, ctx=gpu_ctx)
        Eo, go, Ho = orc.icp_energy_derivs(corrs, base, xi)
        assert E == Eo                                   # pairwise_sum tree, bit for bit
        assert np.array_equal(g, go)                     # Complex passes
        assert np.array_equal(H, Ho) and np.array_equal(H, H.T)
    if n:
        assert csf.icp_loss(corrs, base, ctx=gpu_ctx) == orc.icp_energy_derivs(corrs, base)[0]


@pytest.mark.parametrize("solver", [capi.SOLVER_LINEARIZED, capi.SOLVER_NEWTON, capi.SOLVER_GRADIENT_DESCENT,
                                    capi.SOLVER_CONJUGATE_GRADIENT])
def test_track_frame_solvers(gpu_ctx, orc, solver):
    d, gt, k = orc.workload(1, 6, 160, 120)
    params = capi.VolumeParams((capi.C.c_int * 3)(128, 128, 128), 0.02, (capi.C.c_double * 3)(-2.1, -1.28, -0.1),
                               0.06, 128.0)
    vol_g = csf.TsdfVolume((128, 128, 128), 0.02, (-2.1, -1.28, -0.1), 0.06, 128.0, channels=0, ctx=gpu_ctx)
    vol_o = orc.Volume(params, 0, False)
    intr = np.array([[k.fx], [k.fy], [k.cx], [k.cy]])
    for i in range(4):
        p = gt[i].reshape(12, 1)
        vol_g.surface_update(d[i].astype(np.float64), p, intr)
        vol_o.surface_update(d[i].astype(np.float64), p, intr)
    cfg = csf.default_icp_cfg(solver=solver)
    init = gt[4]
    r_g = csf.track_frame(vol_g, d[4].astype(np.float64), init, k, cfg)
    p_o, r_o = vol_o.track_frame(d[4].astype(np.float64), init, k, cfg, canonical=True)
    assert np.array_equal(r_g.pose, p_o)
    assert r_g.iterations == r_o.iterations and r_g.correspondences == r_o.correspondences
    assert bool(r_g.converged) == bool(r_o.converged)
    assert r_g.final_loss == r_o.final_loss and np.isfinite(r_g.final_loss)
    assert np.linalg.norm(r_g.pose[9:] - gt[4][9:]) < 0.02
    # track_frame(..., TrackTrace*) (icp.cpp:213-228): the rows are bit-identical too
    tr = csf.TrackTrace(ground_truth=gt[4])
    r_t = csf.track_frame(vol_g, d[4].astype(np.float64), init, k, cfg, trace=tr)
    _, _, rows_o = vol_o.track_frame_traced(d[4].astype(np.float64), init, k, cfg)
    assert np.array_equal(r_t.pose, p_o) and len(tr.rows) == len(rows_o) == r_o.iterations
    for row, ro in zip(tr.rows, rows_o):
        assert (row.iteration, row.loss, row.gradient_norm) == (int(ro[0]), ro[1], ro[2])
        assert np.isfinite(row.translation_error) and np.isfinite(row.rotation_error)
    assert tr.rows[-1].loss == r_g.final_loss
