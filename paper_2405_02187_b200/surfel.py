"""Surfel (X-EF) front end — host mirror of proj/include/csf/surfel.hpp over
the C-ABI.  The SurfelMap lives in HBM; position,
normal and confidence carry D derivative channels (the reference's Complex
is D = 1) as a trailing axis of size 1+D.  Every call runs on the sm_100a
kernels (csrc/surfel.cu)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import capi as _capi
from . import Context, _ctx, _dp, _f64, lift_pose


def default_surfel_cfg(**kw) -> _capi.SurfelCfg:
    """AssociationThresholds + SurfelFusionConfig defaults (surfel.hpp:55-60, 84-91)."""
    from . import library
    c = _capi.SurfelCfg()
    library().csf_default_surfel_cfg(C.byref(c))
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def _i32(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


class SurfelMap:
    """surfel.hpp:24-31 — append-only surfel set resident on the device."""

    def __init__(self, channels: int = 1, ctx: Optional[Context] = None):
        self.ctx = _ctx(ctx)
        self.channels = channels
        self.h = C.c_void_p()
        self.ctx.check(self.ctx.lib.csf_surfels_create(self.ctx.h, channels, C.byref(self.h)))

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            self.ctx.lib.csf_surfels_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def clear(self) -> None:
        """An empty map that keeps its device capacity (no re-allocation)."""
        self.ctx.check(self.ctx.lib.csf_surfels_clear(self.h))

    def size(self) -> int:
        n = C.c_int()
        self.ctx.check(self.ctx.lib.csf_surfels_count(self.h, C.byref(n)))
        return n.value

    def __len__(self):
        return self.size()

    def download(self) -> dict:
        n, Cc = self.size(), 1 + self.channels
        out = {"position": np.zeros((n, 3, Cc)), "normal": np.zeros((n, 3, Cc)), "radius": np.zeros(n),
               "confidence": np.zeros((n, Cc)), "timestamp": np.zeros(n, dtype=np.int32)}
        if n:
            self.ctx.check(self.ctx.lib.csf_surfels_download(self.h, _dp(out["position"]), _dp(out["normal"]),
                                                             _dp(out["radius"]), _dp(out["confidence"]),
                                                             _i32(out["timestamp"])))
        return out

    def upload(self, d: dict) -> None:
        n = len(d["radius"])
        arr = {k: np.ascontiguousarray(d[k], dtype=np.int32 if k == "timestamp" else np.float64) for k in d}
        self.ctx.check(self.ctx.lib.csf_surfels_upload(self.h, n, _dp(arr["position"]), _dp(arr["normal"]),
                                                       _dp(arr["radius"]), _dp(arr["confidence"]),
                                                       _i32(arr["timestamp"])))


def _lifted_depth(depth, D):
    d = _f64(depth)
    if d.ndim == 2:
        q = np.zeros(d.shape + (1 + D,))
        q[..., 0] = d
        d = q
    if d.ndim != 3 or d.shape[2] != 1 + D:
        raise ValueError(f"depth must be (h, w) or (h, w, {1 + D})")
    return np.ascontiguousarray(d)


@dataclass
class IndexMap:
    """surfel.hpp:36-49"""
    width: int
    height: int
    offsets: np.ndarray
    entries: np.ndarray

    def at(self, x: int, y: int) -> np.ndarray:
        c = y * self.width + x
        return self.entries[self.offsets[c]:self.offsets[c + 1]]


def render_index_map(map: SurfelMap, camera_to_world, k: _capi.Intrinsics) -> IndexMap:
    """surfel.cpp:30-64"""
    ctx = map.ctx
    offs = np.zeros(16 * k.width * k.height + 1, dtype=np.uint32)
    ent = np.zeros(max(map.size(), 1), dtype=np.int32)
    m = C.c_int()
    ctx.check(ctx.lib.csf_render_index_map(map.h, _dp(lift_pose(camera_to_world, 0)[:, 0].copy()), C.byref(k),
                                           offs.ctypes.data_as(C.POINTER(C.c_uint32)), _i32(ent), C.byref(m)))
    return IndexMap(4 * k.width, 4 * k.height, offs, ent[:m.value].copy())


def associate_all(map: SurfelMap, depth, camera_to_world, k: _capi.Intrinsics, cfg=None):
    """surfel.cpp:66-108 for every pixel at once: (counts (h, w), indices (T,),
    weights (T, 1+D)) in pixel scan order, candidate order within a pixel."""
    ctx = map.ctx
    D = map.channels
    d = _lifted_depth(depth, D)
    h, w = d.shape[:2]
    pose = np.ascontiguousarray(lift_pose(camera_to_world, D))
    cfg = cfg if cfg is not None else default_surfel_cfg()
    counts = np.zeros((h, w), dtype=np.int32)
    T = C.c_int()
    ctx.check(ctx.lib.csf_associate_surfels(map.h, _dp(d), w, h, _dp(pose), C.byref(k), C.byref(cfg), _i32(counts),
                                            None, None, 0, C.byref(T)))
    idx = np.zeros(max(T.value, 1), dtype=np.int32)
    wts = np.zeros((max(T.value, 1), 1 + D))
    ctx.check(ctx.lib.csf_associate_surfels(map.h, _dp(d), w, h, _dp(pose), C.byref(k), C.byref(cfg), _i32(counts),
                                            _i32(idx), _dp(wts), T.value, C.byref(T)))
    return counts, idx[:T.value].copy(), wts[:T.value].copy()


def associate_one_to_many(x: int, y: int, map: SurfelMap, depth, camera_to_world, k, cfg=None):
    """surfel.hpp:71-74 for one pixel: [(index, weight (1+D,))] in candidate order."""
    counts, idx, wts = associate_all(map, depth, camera_to_world, k, cfg)
    flat = counts.reshape(-1)
    p = y * counts.shape[1] + x
    s = int(flat[:p].sum())
    return [(int(idx[s + j]), wts[s + j]) for j in range(int(flat[p]))]


def sample_confidence(k: _capi.Intrinsics, x: int, y: int) -> float:
    """surfel.cpp:110-119"""
    from . import library
    return float(library().csf_sample_confidence(C.byref(k), x, y))


@dataclass
class SurfelUpdateStats:
    """surfel.hpp:93-96"""
    merged_pixels: int
    created: int


def update_surfels(map: SurfelMap, depth, camera_to_world, k: _capi.Intrinsics, frame_index: int,
                   cfg=None) -> SurfelUpdateStats:
    """surfel.cpp:121-236: lifted depth (h, w[, 1+D]) at a lifted camera->world pose (12, 1+D)."""
    ctx = map.ctx
    D = map.channels
    pose = np.ascontiguousarray(lift_pose(camera_to_world, D))
    cfg = cfg if cfg is not None else default_surfel_cfg()
    mp, cr = C.c_int(), C.c_int()
    raw = np.asarray(depth)
    if raw.ndim == 2:  # unperturbed depth: lifted on the device
        d = np.ascontiguousarray(raw, dtype=np.float64)
        h, w = d.shape
        ctx.check(ctx.lib.csf_update_surfels_real(map.h, _dp(d), w, h, _dp(pose), C.byref(k), frame_index,
                                                  C.byref(cfg), C.byref(mp), C.byref(cr)))
    else:
        d = _lifted_depth(depth, D)
        h, w = d.shape[:2]
        ctx.check(ctx.lib.csf_update_surfels(map.h, _dp(d), w, h, _dp(pose), C.byref(k), frame_index, C.byref(cfg),
                                             C.byref(mp), C.byref(cr)))
    return SurfelUpdateStats(mp.value, cr.value)


def predict_maps(map: SurfelMap, camera_to_world, k: _capi.Intrinsics):
    """surfel.cpp:238-263: world-frame (vertices, normals) of shape (h, w, 3)."""
    ctx = map.ctx
    V = np.zeros((k.height, k.width, 3))
    N = np.zeros_like(V)
    ctx.check(ctx.lib.csf_predict_maps(map.h, _dp(lift_pose(camera_to_world, 0)[:, 0].copy()), C.byref(k), _dp(V),
                                       _dp(N)))
    return V, N


def write_surfel_ply(path, map: SurfelMap) -> None:
    """surfel.cpp:265-295: ASCII PLY (position, normal, radius, confidence, timestamp)."""
    d = map.download()
    n = len(d["radius"])
    lines = ["ply", "format ascii 1.0", f"element vertex {n}", "property float x", "property float y",
             "property float z", "property float nx", "property float ny", "property float nz", "property float radius",
             "property float confidence", "property int timestamp", "end_header"]
    g = lambda v: format(float(v), ".9g")  # std::setprecision(9)
    for i in range(n):
        p, q = d["position"][i, :, 0], d["normal"][i, :, 0]
        lines.append(" ".join([g(p[0]), g(p[1]), g(p[2]), g(q[0]), g(q[1]), g(q[2]), g(d["radius"][i]),
                               g(d["confidence"][i, 0]), str(int(d["timestamp"][i]))]))
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")
