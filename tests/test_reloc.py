"""Relocalization (reloc.hpp).

CPU (oracle): the reference's own reloc_energy restated (reloc.hpp:48-69) and
the builder-defined bodies checked against the SPEC.md:556-596 properties —
E = 0 for the query frame at its true pose after a one-frame fusion, the CSFD
gradient against central finite differences, a symmetric Hessian, a
non-increasing loss trace, Newton recovering a (3 deg, 5 cm) perturbation,
nearest-neighbour error pins.

GPU: the device RelocProblem / reloc_energy / gradient / Hessian /
relocalize / depth_cloud / eval_nn_error against the oracle on the same
seeded inputs: flattened voxels, energies and overlaps bit-identical;
derivatives within 1e-9 relative (bit-identical in practice: per-channel
exact division); relocalize trajectories identical.
"""
import numpy as np
import pytest

from paper_2405_02187_b200 import capi

W, H = 80, 60


def _scene(n=4):
    from oracle import orc
    d, gt, k = orc.workload(1, n, W, H)
    return d.astype(np.float64), gt, k


def _dense_params():
    return capi.VolumeParams((capi.C.c_int * 3)(64, 64, 64), 0.04, (capi.C.c_double * 3)(-2.1, -1.28, -0.1), 0.12,
                             128.0)


def _hash_params():
    return capi.HashParams(0.04, (capi.C.c_double * 3)(0.0, 0.0, 0.0), 0.12, 128.0, 14, 1 << 14)


def _intr(k):
    a = np.zeros((4, 1))
    a[:, 0] = [k.fx, k.fy, k.cx, k.cy]
    return a


def _perturb(pose12, deg=3.0, cm=5.0, seed=0):
    """exp([rho; phi]) * pose with |phi| = deg, |rho| = cm (se3.hpp:77-105 via Rodrigues, host)."""
    rng = np.random.default_rng(seed)
    a = rng.normal(size=3)
    a *= np.deg2rad(deg) / np.linalg.norm(a)
    t = rng.normal(size=3)
    t *= cm / 100.0 / np.linalg.norm(t)
    th = np.linalg.norm(a)
    K = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]]) / th
    R = np.eye(3) + np.sin(th) * K + (1 - np.cos(th)) * K @ K
    R0 = pose12[:9].reshape(3, 3)
    out = np.empty(12)
    out[:9] = (R @ R0).reshape(9)
    out[9:] = R @ pose12[9:] + t
    return out


def _oracle_ref(frames, hashed=False):
    from oracle import orc
    d, gt, k = _scene()
    vo = orc.Volume(_hash_params() if hashed else _dense_params(), 0, hashed)
    for i in frames:
        vo.surface_update(d[i], gt[i].reshape(12, 1), _intr(k))
    return vo, d, gt, k


# ----------------------------------------------------------------------------- CPU: oracle properties
def test_oracle_energy_zero_at_true_pose(oracle_built):
    from oracle import orc
    vo, d, gt, k = _oracle_ref([1])
    r = orc.Reloc(vo, d[1], k)
    E, _, _, ov = r.energy(gt[1])
    assert ov > 1000 and E == 0.0


def test_oracle_gradient_vs_fd_and_hessian_symmetric(oracle_built):
    from oracle import orc
    vo, d, gt, k = _oracle_ref([0, 1, 2])
    r = orc.Reloc(vo, d[3], k)
    p = _perturb(gt[3], 1.0, 1.0, seed=3)
    E, g, Hm, ov = r.energy(p, order=2)
    assert ov > 1000 and E > 0
    eps = 1e-6
    for i in range(6):
        xi = np.zeros(6)
        xi[i] = eps
        fd = (r.energy(_exp_step(p, xi))[0] - r.energy(_exp_step(p, -xi))[0]) / (2 * eps)
        assert abs(fd - g[i]) <= 1e-4 * max(abs(g).max(), 1e-12), (i, fd, g[i])
    assert np.array_equal(Hm, Hm.T)
    # the Hessian pass's diagonal-pair im1 is the gradient (csfd.hpp im1 == Complex)
    _, g1, _, _ = r.energy(p, order=1)
    assert np.array_equal(g1, g)


def _exp_step(pose12, xi):
    """apply_increment on the host: exp(xi) * pose (se3.hpp:77-119), numpy."""
    rho, phi = xi[:3], xi[3:]
    th = np.linalg.norm(phi)
    S = np.array([[0, -phi[2], phi[1]], [phi[2], 0, -phi[0]], [-phi[1], phi[0], 0]])
    if th < 1e-7:
        R = np.eye(3) + S
        V = np.eye(3) + 0.5 * S
    else:
        A = np.sin(th) / th
        B = (1 - np.cos(th)) / th ** 2
        Cc = (th - np.sin(th)) / th ** 3
        R = np.eye(3) + A * S + B * S @ S
        V = np.eye(3) + B * S + Cc * S @ S
    t = V @ rho
    R0 = pose12[:9].reshape(3, 3)
    out = np.empty(12)
    out[:9] = (R @ R0).reshape(9)
    out[9:] = R @ pose12[9:] + t
    return out


def _cfg(**kw):
    c = capi.RelocCfg(0.5, -1.0, 50, 25, 1e-6, 1.0, 0.5, 1e-4, 1e-8, 0.05, 0.9)
    for a, v in kw.items():
        setattr(c, a, v)
    return c


def test_oracle_relocalize_newton_recovers(oracle_built):
    from oracle import orc
    vo, d, gt, k = _oracle_ref([0, 1, 2, 3])
    r = orc.Reloc(vo, d[2], k)
    init = _perturb(gt[2], 3.0, 5.0, seed=1)
    res = {}
    for m in (capi.RELOC_GRADIENT_DESCENT, capi.RELOC_NEWTON):
        pose, it, conv, loss, losses, gn = r.relocalize(init, m, _cfg(max_iterations=30))
        assert it > 0 and np.all(np.diff(losses) <= 1e-12)
        assert losses[-1] == loss and loss < r.energy(init)[0]
        res[m] = (pose, it, loss)
    pose_n = res[capi.RELOC_NEWTON][0]
    terr = np.linalg.norm(pose_n[9:] - gt[2][9:])
    R = pose_n[:9].reshape(3, 3) @ gt[2][:9].reshape(3, 3).T
    rerr = np.degrees(np.arccos(np.clip((np.trace(R) - 1) / 2, -1, 1)))
    assert terr < 0.01 and rerr < 0.5, (terr, rerr)
    assert res[capi.RELOC_NEWTON][2] <= res[capi.RELOC_GRADIENT_DESCENT][2]


def test_oracle_nn_error_pins(oracle_built):
    from oracle import orc
    rng = np.random.default_rng(2)
    q = rng.uniform(-1, 1, (500, 3))
    eye = np.array([1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0], dtype=np.float64)
    assert orc.nn_error(eye, q, q) == (0.0, False)
    T = eye.copy()
    T[9] = 0.001
    m, out = orc.nn_error(T, q, q + np.array([0.001, 0, 0]))
    assert m < 1e-15 and not out
    T[9] = 0.5
    assert orc.nn_error(T, q, q)[1]


# ----------------------------------------------------------------------------- GPU: device vs oracle
@pytest.mark.gpu
@pytest.mark.parametrize("hashed", [False, True])
def test_reloc_problem_and_energy_parity(gpu_ctx, oracle_built, hashed):
    import paper_2405_02187_b200 as csf
    from oracle import orc
    vo, d, gt, k = _oracle_ref([0, 1, 2], hashed)
    if hashed:
        vg = csf.HashedVolume(0.04, (0.0, 0.0, 0.0), 0.12, 128.0, 14, 1 << 14, channels=0, ctx=gpu_ctx)
    else:
        vg = csf.TsdfVolume((64, 64, 64), 0.04, (-2.1, -1.28, -0.1), 0.12, 128.0, channels=0, ctx=gpu_ctx)
    for i in (0, 1, 2):
        vg.surface_update(d[i], gt[i], k)
    ro = orc.Reloc(vo, d[3], k)
    rg = csf.RelocProblem(vg, d[3], k)
    co, vals = ro.arrays()
    assert rg.n_voxels == ro.n_voxels > 1000 and rg.mu == ro.mu
    assert np.array_equal(rg.voxel_centers, co) and np.array_equal(rg.reference_values, vals)
    for s in range(3):
        p = _perturb(gt[3], 2.0, 3.0, seed=s)
        Eo, go, Ho, ovo = ro.energy(p, order=2)
        Eg, gg, Hg, ovg = rg.energy_derivs(p, order=2)
        assert Eg == Eo and ovg == ovo
        scale = np.abs(Ho).max()
        assert np.abs(gg - go).max() <= 1e-9 * np.abs(go).max()
        assert np.abs(Hg - Ho).max() <= 1e-9 * scale
        g1 = csf.reloc_gradient(rg, p)
        assert np.abs(g1 - go).max() <= 1e-9 * np.abs(go).max()
        assert csf.reloc_loss(rg, p) == Eo


@pytest.mark.gpu
def test_relocalize_parity(gpu_ctx, oracle_built):
    import paper_2405_02187_b200 as csf
    from oracle import orc
    vo, d, gt, k = _oracle_ref([0, 1, 2, 3])
    vg = csf.TsdfVolume((64, 64, 64), 0.04, (-2.1, -1.28, -0.1), 0.12, 128.0, channels=0, ctx=gpu_ctx)
    for i in range(4):
        vg.surface_update(d[i], gt[i], k)
    ro = orc.Reloc(vo, d[2], k)
    rg = csf.RelocProblem(vg, d[2], k)
    init = _perturb(gt[2], 3.0, 5.0, seed=1)
    for m in (csf.RelocMethod.GRADIENT_DESCENT, csf.RelocMethod.NEWTON):
        cfg = _cfg(max_iterations=20)
        po, ito, convo, losso, lo, gno = ro.relocalize(init, int(m), cfg)
        rr = csf.relocalize(rg, init, m, cfg)
        assert rr.iterations == ito and rr.converged == convo
        np.testing.assert_allclose(rr.pose, po, rtol=0, atol=1e-12)
        np.testing.assert_allclose(rr.losses, lo, rtol=1e-9, atol=0)
        assert np.all(np.diff(rr.losses) <= 1e-12)


@pytest.mark.gpu
def test_reloc_errors(gpu_ctx, oracle_built):
    import paper_2405_02187_b200 as csf
    d, gt, k = _scene()
    empty = csf.TsdfVolume((32, 32, 32), 0.04, (-2.1, -1.28, -0.1), 0.12, 128.0, channels=0, ctx=gpu_ctx)
    with pytest.raises(csf.InvalidArgument):
        csf.RelocProblem(empty, d[0], k)
    vg = csf.TsdfVolume((64, 64, 64), 0.04, (-2.1, -1.28, -0.1), 0.12, 128.0, channels=0, ctx=gpu_ctx)
    vg.surface_update(d[0], gt[0], k)
    rg = csf.RelocProblem(vg, d[0], k)
    away = gt[0].copy()
    away[9:] += 100.0  # camera far outside the volume: nothing overlaps
    with pytest.raises(RuntimeError):
        csf.reloc_loss(rg, away)
    with pytest.raises(csf.InvalidArgument):
        csf.build_reference([], k, _dense_params(), ctx=gpu_ctx)
    with pytest.raises(csf.InvalidArgument):
        csf.eval_nn_error(gt[0], np.zeros((0, 3)), np.zeros((4, 3)), ctx=gpu_ctx)


@pytest.mark.gpu
def test_build_reference_select_cloud_nn(gpu_ctx, oracle_built):
    import paper_2405_02187_b200 as csf
    from oracle import orc
    d, gt, k = _scene()
    idx = csf.select_reference_frames(list(gt), gt[2], count=3)
    assert idx[0] == 2 and len(idx) == 3
    vol = csf.build_reference([(d[i], gt[i]) for i in idx], k, _dense_params(), ctx=gpu_ctx)
    vo = orc.Volume(_dense_params(), 0, False)
    for i in idx:
        vo.surface_update(d[i], gt[i].reshape(12, 1), _intr(k))
    fg, wg = vol.download()
    fo, wo = vo.download()
    assert np.array_equal(wg, wo) and np.array_equal(fg[..., 0] if fg.ndim > 1 else fg, fo[..., 0] if fo.ndim > 1 else fo)
    for stride in (1, 3):
        cg = csf.depth_cloud(d[1], k, gt[1], stride, ctx=gpu_ctx)
        co = orc.depth_cloud(d[1], k, gt[1], stride)
        assert cg.shape == co.shape and np.array_equal(cg, co)
    q = csf.depth_cloud(d[1], k, gt[1], 2, ctx=gpu_ctx)
    r = csf.depth_cloud(d[2], k, gt[2], 1, ctx=gpu_ctx)
    T = _perturb(np.array([1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0], dtype=np.float64), 0.5, 1.0, seed=5)
    e = csf.eval_nn_error(T, q, r, ctx=gpu_ctx)
    mo, oo = orc.nn_error(T, q, r)
    assert e.mean == mo and e.outlier == oo
