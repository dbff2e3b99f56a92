"""Surfel (X-EF) front end (surfel.hpp).

CPU: the oracle restatement (oracle/orc_surfel.hpp) against the reference's
own test cases (proj/tests/test_surfel.cpp): single-pixel create / merge /
confidence, index-map registration and order, determinism, one-to-many
coverage.

GPU: the device map (csrc/surfel.cu) against the oracle on the same seeded
frames: index map offsets/entries identical, association lists (indices and
lifted weights) identical, and a 3-frame fusion with lifted pose channels —
every position / normal / confidence channel, radius and timestamp of every
surfel bit-identical; predict_maps identical."""
import numpy as np
import pytest

from paper_2405_02187_b200 import capi


def _cfg(**kw):
    c = capi.SurfelCfg(0.05, 30.0, 0.05, 0.025, 1)
    for a, v in kw.items():
        setattr(c, a, v)
    return c


def _tiny():
    return capi.Intrinsics(10.0, 10.0, 4.0, 4.0, 9, 9, 5000.0)


def _center_patch(z, D):
    d = np.zeros((9, 9, 1 + D))
    for (x, y) in ((4, 4), (5, 4), (4, 5)):
        d[y, x, 0] = z
    return d


def _pose(D, p12=None):
    p = np.zeros((12, 1 + D))
    p[:, 0] = p12 if p12 is not None else [1, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0]
    return p


def _frames(n=3, D=2, h=1e-8, seed=5):
    """config-1 room frames at 80x60 (oracle renderer), poses lifted on D twist-like channels."""
    from oracle import orc
    d, gt, k = orc.workload(1, n, 80, 60)
    rng = np.random.default_rng(seed)
    depth = np.zeros(d.shape + (1 + D,))
    depth[..., 0] = d
    poses = []
    for i in range(n):
        p = _pose(D, gt[i])
        p[:, 1:] = rng.uniform(-1, 1, (12, D)) * h
        poses.append(p)
    return depth, poses, gt, k


# ----------------------------------------------------------------------------- CPU: oracle vs reference cases
def test_oracle_create_merge_confidence(oracle_built):
    # test_surfel.cpp:243-280
    from oracle import orc
    k = _tiny()
    assert orc.sample_confidence(k, 4, 4) == 1.0 and orc.sample_confidence(k, 0, 0) < 1.0
    m = orc.Surfels(1)
    assert m.update(_center_patch(1.0, 1), _pose(1), k, 0, _cfg()) == (0, 1)
    s = m.download()
    assert np.array_equal(s["position"][0, :, 0], [0.0, 0.0, 1.0])
    assert s["confidence"][0, 0] == 1.0 and s["timestamp"][0] == 0
    assert abs(s["radius"][0] - np.sqrt(2.0) / k.fx) <= 1e-12 * s["radius"][0]
    assert m.update(_center_patch(1.0, 1), _pose(1), k, 1, _cfg()) == (1, 0)
    t = m.download()
    assert np.linalg.norm(t["position"][0, :, 0] - s["position"][0, :, 0]) <= 1e-9
    assert t["confidence"][0, 0] == 2.0 and t["timestamp"][0] == 1


def test_oracle_map_fusion_properties(oracle_built):
    # test_surfel.cpp:87-160, 282-319, 399-427
    from oracle import orc
    depth, poses, gt, k = _frames(2, D=1)
    base = orc.Surfels(1)
    base.update(depth[0], _pose(1, gt[0]), k, 0, _cfg())  # unseeded first view (pose_cast<Complex>)
    b = base.download()
    n0 = len(b["radius"])
    assert n0 > 1000 and np.all(b["radius"] > 0) and np.all(b["confidence"][:, 0] > 0)
    assert np.all(np.abs(np.linalg.norm(b["normal"][:, :, 0], axis=1) - 1.0) < 1e-6)
    # index map: every visible surfel exactly once, nearest-first per cell
    offs, ent = base.index_map(gt[1], k)
    assert len(ent) == len(set(ent.tolist())) and offs[-1] == len(ent) and len(ent) > 1000
    runs = []
    for t in range(2):
        m = orc.Surfels(1)
        m.upload(b)
        st = m.update(depth[1], poses[1], k, 1, _cfg())
        runs.append((st, m.download()))
    (st, a), (_, a2) = runs
    assert st[0] > 500 and st[1] > 0
    assert np.all(a["confidence"][:n0, 0] >= b["confidence"][:, 0])
    for key in a:
        assert np.array_equal(a[key], a2[key])  # deterministic
    # one-to-many reaches more stored surfels than one-to-one
    cover = {}
    for otm in (1, 0):
        m = orc.Surfels(1)
        m.upload(b)
        p = poses[1].copy()
        p[:, 1] = 0.0
        p[10, 1] = 1e-8  # seed ty
        m.update(depth[1], p, k, 1, _cfg(one_to_many=otm))
        pos = m.download()["position"][:n0, :, 1]
        cover[otm] = int(np.count_nonzero(np.any(pos != 0.0, axis=1)))
    assert 0 < cover[0] < cover[1]


# ----------------------------------------------------------------------------- GPU: device vs oracle
@pytest.mark.gpu
def test_surfel_tiny_cases_on_device(gpu_ctx):
    import paper_2405_02187_b200 as csf
    from oracle import orc
    k = _tiny()
    for x, y in ((4, 4), (0, 0), (8, 3)):
        assert csf.sample_confidence(k, x, y) == orc.sample_confidence(k, x, y)
    m = csf.SurfelMap(1, ctx=gpu_ctx)
    st = csf.update_surfels(m, _center_patch(1.0, 1), _pose(1), k, 0)
    assert (st.merged_pixels, st.created) == (0, 1)
    st = csf.update_surfels(m, _center_patch(1.0, 1), _pose(1), k, 1)
    assert (st.merged_pixels, st.created) == (1, 0)
    s = m.download()
    assert s["confidence"][0, 0] == 2.0 and s["timestamp"][0] == 1


@pytest.mark.gpu
@pytest.mark.parametrize("D,otm", [(2, 1), (1, 0), (0, 1)])
def test_surfel_fusion_parity(gpu_ctx, oracle_built, D, otm):
    import paper_2405_02187_b200 as csf
    from oracle import orc
    depth, poses, gt, k = _frames(3, D=max(D, 1))
    if D == 0:
        depth = depth[..., :1]
        poses = [p[:, :1] for p in poses]
    cfg = _cfg(one_to_many=otm)
    mo = orc.Surfels(D)
    mg = csf.SurfelMap(D, ctx=gpu_ctx)
    for f in range(3):
        if f == 2:
            # the index map and the association lists of the third frame
            oo, eo = mo.index_map(gt[f], k)
            im = csf.render_index_map(mg, gt[f], k)
            assert np.array_equal(im.offsets, oo) and np.array_equal(im.entries, eo)
            co, io, wo = mo.associate(depth[f], poses[f], k, cfg)
            cg, ig, wg = csf.associate_all(mg, depth[f], poses[f], k, cfg)
            assert np.array_equal(cg, co) and np.array_equal(ig, io)
            assert np.array_equal(wg, wo)
        so = mo.update(depth[f], poses[f], k, f, cfg)
        sg = csf.update_surfels(mg, depth[f], poses[f], k, f, cfg)
        assert (sg.merged_pixels, sg.created) == so
        a, b = mg.download(), mo.download()
        for key in a:
            assert np.array_equal(a[key], b[key]), (f, key)
    Vg, Ng = csf.predict_maps(mg, gt[1], k)
    Vo, No = mo.predict(gt[1], k)
    assert np.array_equal(Vg, Vo) and np.array_equal(Ng, No) and np.count_nonzero(Vg[..., 2]) > 1000


@pytest.mark.gpu
def test_surfel_ply_export(gpu_ctx, tmp_path):
    # test_surfel.cpp:486-530
    import paper_2405_02187_b200 as csf
    depth, poses, gt, k = _frames(1, D=1)
    m = csf.SurfelMap(1, ctx=gpu_ctx)
    csf.update_surfels(m, depth[0], poses[0], k, 0)
    p = tmp_path / "s.ply"
    csf.write_surfel_ply(p, m)
    lines = p.read_text().splitlines()
    n = m.size()
    assert lines[0] == "ply" and lines[2] == f"element vertex {n}" and lines[12] == "end_header"
    assert len(lines) == 13 + n and len(lines[13].split()) == 9


@pytest.mark.gpu
def test_surfel_real_depth_path(gpu_ctx):
    """An unperturbed (h, w) depth is lifted on the device: the same map as
    the explicit zero-channel lifted depth, bit for bit."""
    import paper_2405_02187_b200 as csf
    depth, poses, gt, k = _frames(2, D=2)
    a = csf.SurfelMap(2, ctx=gpu_ctx)
    b = csf.SurfelMap(2, ctx=gpu_ctx)
    for f in range(2):
        sa = csf.update_surfels(a, depth[f], poses[f], k, f)
        sb = csf.update_surfels(b, np.ascontiguousarray(depth[f][..., 0]), poses[f], k, f)
        assert (sa.merged_pixels, sa.created) == (sb.merged_pixels, sb.created)
    da, db = a.download(), b.download()
    for key in da:
        assert np.array_equal(da[key], db[key])
