"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes wrapper of oracle/_build/liborc.so (the CPU restatement of the
reference hot path).  Imported only by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline / --impl reference legs — never by the product.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from paper_2405_02187_b200 import capi as _capi  # struct layouts only (no product calls)

LIB_PATH = Path(__file__).resolve().parent / "_build" / "liborc.so"
LIBM_PATH = Path(__file__).resolve().parent / "_build" / "liborc_libm.so"
_LIB = None
_LIBS = {}


def use_libm(enable: bool) -> None:
    """Switch every wrapper below to the -DORC_LIBM build (glibc exp/sin/cos)
    or back to the default (csf_detmath.h) build."""
    global _LIB, LIB_PATH
    _LIBS[str(LIB_PATH)] = _LIB
    LIB_PATH = LIBM_PATH if enable else LIBM_PATH.parent / "liborc.so"
    _LIB = _LIBS.get(str(LIB_PATH))


def lib() -> C.CDLL:
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"oracle library {LIB_PATH} missing: run make -C oracle")
        L = C.CDLL(str(LIB_PATH))
        dp, ip, vp = C.POINTER(C.c_double), C.c_int, C.c_void_p
        i32p, u64p, fp = C.POINTER(C.c_int32), C.POINTER(C.c_uint64), C.POINTER(C.c_float)
        sig = {
            "orc_last_error": (C.c_char_p, []),
            "orc_bilateral": (ip, [dp, ip, ip, C.c_double, C.c_double, ip, dp]),
            "orc_downsample": (ip, [dp, ip, ip, C.c_double, dp]),
            "orc_measure": (ip, [dp, ip, ip, dp, ip, dp, dp]),
            "orc_volume_create_dense": (ip, [C.POINTER(_capi.VolumeParams), ip, C.POINTER(vp)]),
            "orc_volume_create_hashed": (ip, [C.POINTER(_capi.HashParams), ip, C.POINTER(vp)]),
            "orc_volume_destroy": (None, [vp]),
            "orc_surface_update": (ip, [vp, dp, ip, ip, dp, dp, C.POINTER(C.c_int)]),
            "orc_raycast": (ip, [vp, dp, dp, ip, ip, C.POINTER(_capi.RaycastCfg), dp, dp]),
            "orc_volume_voxels": (C.c_longlong, [vp]),
            "orc_volume_download": (ip, [vp, dp, dp]),
            "orc_volume_upload": (ip, [vp, dp, dp]),
            "orc_volume_block_count": (ip, [vp]),
            "orc_volume_hash": (ip, [vp, i32p, u64p, i32p, i32p]),
            "orc_track_frame": (ip, [vp, dp, ip, ip, dp, C.POINTER(_capi.Intrinsics), C.POINTER(_capi.IcpCfg), ip,
                                     dp, C.POINTER(_capi.TrackResult)]),
            "orc_track_frame_traced": (ip, [vp, dp, ip, ip, dp, C.POINTER(_capi.Intrinsics), C.POINTER(_capi.IcpCfg),
                                            dp, C.POINTER(_capi.TrackResult), dp, ip, C.POINTER(C.c_int)]),
            "orc_workload": (ip, [ip, ip, ip, ip, fp, dp, C.POINTER(_capi.Intrinsics)]),
            "orc_pipeline_run": (ip, [C.POINTER(_capi.PipelineCfg), fp, dp, ip, dp, dp, dp, i32p, dp]),
            "orc_pipeline_run_keep": (ip, [C.POINTER(_capi.PipelineCfg), fp, dp, ip, dp, dp, dp, i32p,
                                           C.POINTER(vp)]),
            "orc_associate": (ip, [dp, dp, dp, dp, ip, ip, dp, dp, C.POINTER(_capi.Intrinsics), C.POINTER(_capi.IcpCfg),
                                   ip, dp, C.POINTER(C.c_int)]),
            "orc_linearized_step": (ip, [dp, ip, dp, ip, dp]),
            "orc_sample_points": (ip, [vp, dp, ip, ip, dp, i32p]),
            "orc_measured_points": (ip, [dp, ip, ip, dp, dp, C.c_double, dp, dp, ip, ip, dp, i32p, ip]),
            "orc_surface_update_lifted": (ip, [vp, dp, ip, ip, dp, dp, C.POINTER(C.c_int)]),
            "orc_view_scores": (ip, [vp, dp, ip, C.POINTER(_capi.Intrinsics), C.c_double, C.c_double, C.c_double,
                                     dp, dp]),
            "orc_icp_energy_derivs": (ip, [dp, ip, dp, dp, C.c_double, dp, dp, dp]),
            "orc_reloc_create": (ip, [vp, dp, ip, ip, C.POINTER(_capi.Intrinsics), C.POINTER(vp)]),
            "orc_reloc_destroy": (None, [vp]),
            "orc_reloc_info": (ip, [vp, C.POINTER(C.c_int), dp, dp, dp]),
            "orc_reloc_energy": (ip, [vp, dp, ip, C.c_double, dp, dp, dp, C.POINTER(C.c_long)]),
            "orc_relocalize": (ip, [vp, dp, ip, C.POINTER(_capi.RelocCfg), dp, C.POINTER(_capi.RelocResult), dp, dp]),
            "orc_depth_cloud": (ip, [dp, ip, ip, C.POINTER(_capi.Intrinsics), dp, ip, dp, C.POINTER(C.c_int)]),
            "orc_nn_error": (ip, [dp, dp, ip, dp, ip, dp, C.POINTER(C.c_int)]),
            "orc_surfels_create": (ip, [ip, C.POINTER(vp)]),
            "orc_surfels_destroy": (None, [vp]),
            "orc_surfels_count": (ip, [vp]),
            "orc_surfels_download": (ip, [vp, dp, dp, dp, dp, i32p]),
            "orc_surfels_upload": (ip, [vp, ip, dp, dp, dp, dp, i32p]),
            "orc_update_surfels": (ip, [vp, dp, ip, ip, dp, C.POINTER(_capi.Intrinsics), ip,
                                        C.POINTER(_capi.SurfelCfg), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
            "orc_render_index_map": (ip, [vp, dp, C.POINTER(_capi.Intrinsics), C.POINTER(C.c_uint32), i32p,
                                          C.POINTER(C.c_int)]),
            "orc_associate_surfels": (ip, [vp, dp, ip, ip, dp, C.POINTER(_capi.Intrinsics), C.POINTER(_capi.SurfelCfg),
                                           i32p, i32p, dp, ip, C.POINTER(C.c_int)]),
            "orc_predict_maps": (ip, [vp, dp, C.POINTER(_capi.Intrinsics), dp, dp]),
            "orc_sample_confidence": (C.c_double, [C.POINTER(_capi.Intrinsics), ip, ip]),
            "orc_pipeline_hessian": (ip, [C.POINTER(_capi.PipelineCfg), fp, dp, ip, dp, dp, dp, dp, dp, i32p, dp]),
            "orc_detmath_ulp": (ip, [ip, dp, ip, dp, dp, dp]),
            "orc_default_icp_cfg": (None, [C.POINTER(_capi.IcpCfg)]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _LIB = L
    return _LIB


def _check(rc: int) -> None:
    if rc != 0:
        msg = lib().orc_last_error()
        raise RuntimeError(f"oracle error {rc}: {msg.decode() if msg else ''}")


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def bilateral_filter(depth, sigma_s=4.5, sigma_r=0.03, radius=3):
    d = np.ascontiguousarray(depth, dtype=np.float64)
    h, w = d.shape
    out = np.empty_like(d)
    _check(lib().orc_bilateral(_dp(d), w, h, sigma_s, sigma_r, radius, _dp(out)))
    return out


def downsample_depth(depth, sigma_r=0.03):
    d = np.ascontiguousarray(depth, dtype=np.float64)
    h, w = d.shape
    out = np.empty((h // 2, w // 2))
    _check(lib().orc_downsample(_dp(d), w, h, sigma_r, _dp(out)))
    return out


def measure_surface(depth_lifted, intr_lifted):
    d = np.ascontiguousarray(depth_lifted, dtype=np.float64)
    h, w, cc = d.shape
    k = np.ascontiguousarray(intr_lifted, dtype=np.float64)
    V = np.empty((h, w, 3, cc))
    N = np.empty_like(V)
    _check(lib().orc_measure(_dp(d), w, h, _dp(k), cc - 1, _dp(V), _dp(N)))
    return V, N


class Volume:
    def __init__(self, params, channels: int, hashed: bool, handle=None):
        self.h = C.c_void_p()
        self.channels = channels
        self.hashed = hashed
        self.params = params
        if handle is not None:  # adopt an oracle volume handle (orc_pipeline_run_keep)
            self.h = handle
        elif hashed:
            _check(lib().orc_volume_create_hashed(C.byref(params), channels, C.byref(self.h)))
        else:
            _check(lib().orc_volume_create_dense(C.byref(params), channels, C.byref(self.h)))

    def __del__(self):
        try:
            if self.h:
                lib().orc_volume_destroy(self.h)
        except Exception:
            pass

    def surface_update(self, depth, pose, intr) -> int:
        """depth (h, w) real or (h, w, 1+D) lifted."""
        d = np.ascontiguousarray(depth, dtype=np.float64)
        h, w = d.shape[:2]
        p = np.ascontiguousarray(pose, dtype=np.float64)
        k = np.ascontiguousarray(intr, dtype=np.float64)
        nv = C.c_int()
        fn = lib().orc_surface_update_lifted if d.ndim == 3 else lib().orc_surface_update
        _check(fn(self.h, _dp(d), w, h, _dp(p), _dp(k), C.byref(nv)))
        return nv.value

    def raycast(self, pose, intr, w, h, cfg=None):
        p = np.ascontiguousarray(pose, dtype=np.float64)
        k = np.ascontiguousarray(intr, dtype=np.float64)
        V = np.empty((h, w, 3, 1 + self.channels))
        N = np.empty_like(V)
        _check(lib().orc_raycast(self.h, _dp(p), _dp(k), w, h, C.byref(cfg) if cfg is not None else None, _dp(V),
                                 _dp(N)))
        return V, N

    def download(self):
        n = lib().orc_volume_voxels(self.h)
        f = np.empty((n, 1 + self.channels))
        wt = np.empty(n)
        _check(lib().orc_volume_download(self.h, _dp(f), _dp(wt)))
        return f, wt

    def upload(self, field, weight):
        f = np.ascontiguousarray(field, dtype=np.float64)
        w = np.ascontiguousarray(weight, dtype=np.float64)
        _check(lib().orc_volume_upload(self.h, _dp(f), _dp(w)))

    def block_count(self) -> int:
        return lib().orc_volume_block_count(self.h)

    def hash_tables(self):
        nb = self.block_count()
        heads = np.empty(1 << self.params.bucket_bits, dtype=np.int32)
        keys = np.empty(nb, dtype=np.uint64)
        nxt = np.empty(nb, dtype=np.int32)
        coords = np.empty((nb, 3), dtype=np.int32)
        _check(lib().orc_volume_hash(self.h, heads.ctypes.data_as(C.POINTER(C.c_int32)),
                                     keys.ctypes.data_as(C.POINTER(C.c_uint64)),
                                     nxt.ctypes.data_as(C.POINTER(C.c_int32)),
                                     coords.ctypes.data_as(C.POINTER(C.c_int32))))
        return heads, keys, nxt, coords

    def sample_points(self, pts, grad=False):
        P = np.ascontiguousarray(pts, dtype=np.float64)
        n = P.shape[0]
        out = np.zeros((n, 3, 1 + self.channels) if grad else (n, 1 + self.channels))
        ok = np.zeros(n, dtype=np.int32)
        _check(lib().orc_sample_points(self.h, _dp(P), n, int(grad), _dp(out), ok.ctypes.data_as(C.POINTER(C.c_int32))))
        return out, ok.astype(bool)

    def view_scores(self, poses, k, w0=10.0, beta=0.5, h=1e-8):
        """BASELINE config 5 objective and its view-twist gradient (builder-defined)."""
        p = np.ascontiguousarray(poses, dtype=np.float64).reshape(-1, 12)
        sc = np.empty(p.shape[0])
        g = np.empty((p.shape[0], 6))
        _check(lib().orc_view_scores(self.h, _dp(p), p.shape[0], C.byref(k), w0, beta, h, _dp(sc), _dp(g)))
        return sc, g

    def track_frame(self, depth, init_pose12, k, cfg, canonical=True):
        d = np.ascontiguousarray(depth, dtype=np.float64)
        h, w = d.shape
        init = np.ascontiguousarray(init_pose12, dtype=np.float64)
        out = np.empty(12)
        res = _capi.TrackResult()
        _check(lib().orc_track_frame(self.h, _dp(d), w, h, _dp(init), C.byref(k), C.byref(cfg), int(canonical),
                                     _dp(out), C.byref(res)))
        return out, res

    def track_frame_traced(self, depth, init_pose12, k, cfg):
        d = np.ascontiguousarray(depth, dtype=np.float64)
        h, w = d.shape
        init = np.ascontiguousarray(init_pose12, dtype=np.float64)
        out = np.empty(12)
        res = _capi.TrackResult()
        cap = 64
        rows = np.zeros((cap, 3))
        n = C.c_int()
        _check(lib().orc_track_frame_traced(self.h, _dp(d), w, h, _dp(init), C.byref(k), C.byref(cfg), _dp(out),
                                            C.byref(res), _dp(rows), cap, C.byref(n)))
        return out, res, rows[:n.value].copy()


def workload(config: int, n_frames: int, width: int = 0, height: int = 0):
    if width == 0:
        w, h = (160, 120) if config == 1 else (640, 480)
    else:
        w, h = width, height
    depth = np.empty((n_frames, h, w), dtype=np.float32)
    gt = np.empty((n_frames, 12))
    k = _capi.Intrinsics()
    _check(lib().orc_workload(config, n_frames, width, height, depth.ctypes.data_as(C.POINTER(C.c_float)), _dp(gt),
                              C.byref(k)))
    return depth, gt, k


def pipeline_run(cfg, depth, gt):
    d = np.ascontiguousarray(depth, dtype=np.float32)
    g = np.ascontiguousarray(gt, dtype=np.float64).reshape(-1, 12)
    n = d.shape[0]
    D = cfg.n_dirs
    grad = np.empty(D)
    obj = C.c_double()
    poses = np.empty((n, 12, 1 + D))
    stats = np.empty((n, 8), dtype=np.int32)
    secs = C.c_double()
    _check(lib().orc_pipeline_run(C.byref(cfg), d.ctypes.data_as(C.POINTER(C.c_float)), _dp(g), n, _dp(grad),
                                  C.byref(obj), _dp(poses), stats.ctypes.data_as(C.POINTER(C.c_int32)),
                                  C.byref(secs)))
    return grad, obj.value, poses, stats, secs.value


def pipeline_run_keep(cfg, depth, gt):
    """pipeline_run that also returns the run's final volume (a Volume)."""
    d = np.ascontiguousarray(depth, dtype=np.float32)
    g = np.ascontiguousarray(gt, dtype=np.float64).reshape(-1, 12)
    n = d.shape[0]
    D = cfg.n_dirs
    grad = np.empty(D)
    obj = C.c_double()
    poses = np.empty((n, 12, 1 + D))
    stats = np.empty((n, 8), dtype=np.int32)
    h = C.c_void_p()
    _check(lib().orc_pipeline_run_keep(C.byref(cfg), d.ctypes.data_as(C.POINTER(C.c_float)), _dp(g), n, _dp(grad),
                                       C.byref(obj), _dp(poses), stats.ctypes.data_as(C.POINTER(C.c_int32)),
                                       C.byref(h)))
    vol = Volume(cfg.hash if cfg.hashed else cfg.dense, D, bool(cfg.hashed), handle=h)
    return grad, obj.value, poses, stats, vol


def pipeline_hessian(cfg, depth, gt):
    """Second-order run, one Bicomplex pass per pair (the reference's
    csfd_hessian pattern).  Returns (hessian[P], grad1[P], grad2[P], objective,
    poses[n][12][1+3P], stats, seconds)."""
    d = np.ascontiguousarray(depth, dtype=np.float32)
    g = np.ascontiguousarray(gt, dtype=np.float64).reshape(-1, 12)
    n = d.shape[0]
    P = cfg.n_pairs
    hess, g1, g2 = np.empty(P), np.empty(P), np.empty(P)
    obj = C.c_double()
    poses = np.empty((n, 12, 1 + 3 * P))
    stats = np.empty((n, 8), dtype=np.int32)
    secs = C.c_double()
    _check(lib().orc_pipeline_hessian(C.byref(cfg), d.ctypes.data_as(C.POINTER(C.c_float)), _dp(g), n, _dp(hess),
                                      _dp(g1), _dp(g2), C.byref(obj), _dp(poses),
                                      stats.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(secs)))
    return hess, g1, g2, obj.value, poses, stats, secs.value


def icp_energy_derivs(corrs, base12, xi=None, h=1e-8):
    """icp_energy / icp_gradient / icp_hessian of the reference restatement."""
    c = np.ascontiguousarray(corrs, dtype=np.float64).reshape(-1, 9)
    b = np.ascontiguousarray(base12, dtype=np.float64)
    x = None if xi is None else np.ascontiguousarray(xi, dtype=np.float64)
    E = C.c_double()
    g = np.empty(6)
    H = np.empty((6, 6))
    _check(lib().orc_icp_energy_derivs(_dp(c) if c.size else None, c.shape[0], _dp(b), _dp(x) if x is not None else None,
                                       h, C.byref(E), _dp(g), _dp(H)))
    return E.value, g, H


def associate(mv, mn, pv, pn, c2w, pc2w, k, cfg, stride=1):
    mv, mn, pv, pn = (np.ascontiguousarray(a, dtype=np.float64) for a in (mv, mn, pv, pn))
    h, w = mv.shape[:2]
    out = np.empty((w * h, 9))
    n = C.c_int()
    _check(lib().orc_associate(_dp(mv), _dp(mn), _dp(pv), _dp(pn), w, h, _dp(np.ascontiguousarray(c2w, dtype=float)),
                               _dp(np.ascontiguousarray(pc2w, dtype=float)), C.byref(k), C.byref(cfg), stride, _dp(out),
                               C.byref(n)))
    return out[: n.value].copy()


def linearized_step(corrs, base12, sequential=False):
    c = np.ascontiguousarray(corrs, dtype=np.float64).reshape(-1, 9)
    d = np.empty(6)
    _check(lib().orc_linearized_step(_dp(c) if c.size else None, c.shape[0],
                                     _dp(np.ascontiguousarray(base12, dtype=np.float64)), int(sequential), _dp(d)))
    return d


def pairwise_sum(terms):
    """diff.hpp:16-37 restated in Python (test reference for the device tree)."""
    def block(x):
        if len(x) <= 8:
            acc = x[0]
            for v in x[1:]:
                acc = acc + v
            return acc
        half = len(x) // 2
        return block(x[:half]) + block(x[half:])
    t = [float(v) for v in terms]
    return 0.0 if not t else 0.0 + block(t)


def measured_tsdf(depth, w2c, intr, mu, pts, center):
    """depth (h, w) real or (h, w, 1+D) lifted (the reference's Image<S> depth)."""
    d = np.ascontiguousarray(depth, dtype=np.float64)
    h, w = d.shape[:2]
    pose = np.ascontiguousarray(w2c, dtype=np.float64)
    D = pose.shape[1] - 1
    P = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
    out = np.zeros((P.shape[0], 1 + D))
    ok = np.zeros(P.shape[0], dtype=np.int32)
    _check(lib().orc_measured_points(_dp(d), w, h, _dp(pose), _dp(np.ascontiguousarray(intr, dtype=np.float64)), mu,
                                     _dp(P), _dp(np.ascontiguousarray(center, dtype=np.float64)), P.shape[0], D,
                                     _dp(out), ok.ctypes.data_as(C.POINTER(C.c_int32)), int(d.ndim == 3)))
    return out, ok.astype(bool)


class Reloc:
    """RelocProblem (orc_reloc.hpp) over an oracle Volume."""

    def __init__(self, vol: "Volume", depth, k):
        d = np.ascontiguousarray(depth, dtype=np.float64)
        h, w = d.shape
        self.h = C.c_void_p()
        _check(lib().orc_reloc_create(vol.h, _dp(d), w, h, C.byref(k), C.byref(self.h)))
        n = C.c_int()
        mu = C.c_double()
        _check(lib().orc_reloc_info(self.h, C.byref(n), C.byref(mu), None, None))
        self.n_voxels, self.mu = n.value, mu.value

    def __del__(self):
        try:
            if self.h:
                lib().orc_reloc_destroy(self.h)
        except Exception:
            pass

    def arrays(self):
        c = np.empty((self.n_voxels, 3))
        v = np.empty(self.n_voxels)
        n = C.c_int()
        mu = C.c_double()
        _check(lib().orc_reloc_info(self.h, C.byref(n), C.byref(mu), _dp(c), _dp(v)))
        return c, v

    def energy(self, pose, order=0, h=1e-8):
        p = np.ascontiguousarray(pose, dtype=np.float64).reshape(12)
        E = C.c_double()
        g = np.zeros(6)
        H = np.zeros((6, 6))
        ov = C.c_long()
        _check(lib().orc_reloc_energy(self.h, _dp(p), order, h, C.byref(E), _dp(g), _dp(H), C.byref(ov)))
        return E.value, g, H, ov.value

    def relocalize(self, init, method, cfg):
        p = np.ascontiguousarray(init, dtype=np.float64).reshape(12)
        out = np.empty(12)
        res = _capi.RelocResult()
        n = max(cfg.max_iterations, 1)
        losses = np.zeros(n)
        gn = np.zeros(n)
        _check(lib().orc_relocalize(self.h, _dp(p), method, C.byref(cfg), _dp(out), C.byref(res), _dp(losses), _dp(gn)))
        it = res.iterations
        return out, it, bool(res.converged), res.final_loss, losses[:it].copy(), gn[:it].copy()


def depth_cloud(depth, k, pose, stride=1):
    d = np.ascontiguousarray(depth, dtype=np.float64)
    h, w = d.shape
    out = np.empty((max(w * h, 1), 3))
    n = C.c_int()
    _check(lib().orc_depth_cloud(_dp(d), w, h, C.byref(k), _dp(np.ascontiguousarray(pose, dtype=np.float64)), stride,
                                 _dp(out), C.byref(n)))
    return out[:n.value].copy()


def nn_error(T, q, r):
    q = np.ascontiguousarray(q, dtype=np.float64).reshape(-1, 3)
    r = np.ascontiguousarray(r, dtype=np.float64).reshape(-1, 3)
    mean = C.c_double()
    out = C.c_int()
    _check(lib().orc_nn_error(_dp(np.ascontiguousarray(T, dtype=np.float64)), _dp(q), q.shape[0], _dp(r), r.shape[0],
                              C.byref(mean), C.byref(out)))
    return mean.value, bool(out.value)


def _i32(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


class Surfels:
    """SurfelMapT<FT<D>> (orc_surfel.hpp)."""

    def __init__(self, D: int):
        self.D = D
        self.h = C.c_void_p()
        _check(lib().orc_surfels_create(D, C.byref(self.h)))

    def __del__(self):
        try:
            if self.h:
                lib().orc_surfels_destroy(self.h)
        except Exception:
            pass

    def size(self):
        return lib().orc_surfels_count(self.h)

    def download(self):
        n, Cc = self.size(), 1 + self.D
        out = {"position": np.zeros((n, 3, Cc)), "normal": np.zeros((n, 3, Cc)), "radius": np.zeros(n),
               "confidence": np.zeros((n, Cc)), "timestamp": np.zeros(n, dtype=np.int32)}
        if n:
            _check(lib().orc_surfels_download(self.h, _dp(out["position"]), _dp(out["normal"]), _dp(out["radius"]),
                                              _dp(out["confidence"]), _i32(out["timestamp"])))
        return out

    def upload(self, d):
        arr = {k: np.ascontiguousarray(d[k], dtype=np.int32 if k == "timestamp" else np.float64) for k in d}
        _check(lib().orc_surfels_upload(self.h, len(arr["radius"]), _dp(arr["position"]), _dp(arr["normal"]),
                                        _dp(arr["radius"]), _dp(arr["confidence"]), _i32(arr["timestamp"])))

    def update(self, depth, pose, k, frame, cfg):
        d = np.ascontiguousarray(depth, dtype=np.float64)
        h, w = d.shape[:2]
        mp, cr = C.c_int(), C.c_int()
        _check(lib().orc_update_surfels(self.h, _dp(d), w, h, _dp(np.ascontiguousarray(pose, dtype=np.float64)),
                                        C.byref(k), frame, C.byref(cfg), C.byref(mp), C.byref(cr)))
        return mp.value, cr.value

    def index_map(self, pose12, k):
        offs = np.zeros(16 * k.width * k.height + 1, dtype=np.uint32)
        ent = np.zeros(max(self.size(), 1), dtype=np.int32)
        m = C.c_int()
        _check(lib().orc_render_index_map(self.h, _dp(np.ascontiguousarray(pose12, dtype=np.float64)), C.byref(k),
                                          offs.ctypes.data_as(C.POINTER(C.c_uint32)), _i32(ent), C.byref(m)))
        return offs, ent[:m.value].copy()

    def associate(self, depth, pose, k, cfg, cap=1 << 22):
        d = np.ascontiguousarray(depth, dtype=np.float64)
        h, w = d.shape[:2]
        counts = np.zeros((h, w), dtype=np.int32)
        idx = np.zeros(cap, dtype=np.int32)
        wts = np.zeros((cap, 1 + self.D))
        T = C.c_int()
        _check(lib().orc_associate_surfels(self.h, _dp(d), w, h, _dp(np.ascontiguousarray(pose, dtype=np.float64)),
                                           C.byref(k), C.byref(cfg), _i32(counts), _i32(idx), _dp(wts), cap,
                                           C.byref(T)))
        return counts, idx[:T.value].copy(), wts[:T.value].copy()

    def predict(self, pose12, k):
        V = np.zeros((k.height, k.width, 3))
        N = np.zeros_like(V)
        _check(lib().orc_predict_maps(self.h, _dp(np.ascontiguousarray(pose12, dtype=np.float64)), C.byref(k), _dp(V),
                                      _dp(N)))
        return V, N


def sample_confidence(k, x, y):
    return lib().orc_sample_confidence(C.byref(k), x, y)


def detmath_ulp(fn: str, x):
    """csf_detmath.h exp/sin/cos vs glibc on the same arguments: (ulp errors,
    deterministic values, glibc values)."""
    a = np.ascontiguousarray(x, dtype=np.float64)
    u, d, g = np.empty_like(a), np.empty_like(a), np.empty_like(a)
    code = {"exp": 0, "sin": 1, "cos": 2}[fn]
    _check(lib().orc_detmath_ulp(code, _dp(a), a.size, _dp(u), _dp(d), _dp(g)))
    return u, d, g


def default_icp_cfg(**kw):
    """The reference's IcpConfig defaults (icp.hpp:33-53) from the oracle
    (no product library involved); keyword overrides as the product's."""
    c = _capi.IcpCfg()
    lib().orc_default_icp_cfg(C.byref(c))
    for k, v in kw.items():
        if k in ("level_iterations", "level_pixel_stride"):
            getattr(c, k)[:] = list(v)
        else:
            setattr(c, k, v)
    return c
