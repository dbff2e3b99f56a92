"""Camera relocalization — host mirror of proj/include/csf/reloc.hpp over the
C-ABI.

The reference implements reloc_energy<S> (reloc.hpp:48-69) and declares the
rest without bodies; the builder-defined bodies run on the
device: RelocProblem is resident in HBM, reloc_energy / reloc_gradient /
reloc_hessian are one packed device pass each, relocalize keeps only the
6-vector step logic on the host, depth_cloud and eval_nn_error are device
kernels.  build_reference and select_reference_frames compose existing
calls.  Errors follow the reference: InvalidArgument (std::invalid_argument)
for bad inputs or an unobserved reference, RuntimeError (std::runtime_error)
when no voxel overlaps.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Optional, Sequence

import numpy as np

from . import capi as _capi
from . import (Context, InvalidArgument, TsdfVolume, _ctx, _dp, _f64, _Volume, lift_pose)


class RelocMethod(IntEnum):
    """reloc.hpp:82-85"""
    GRADIENT_DESCENT = _capi.RELOC_GRADIENT_DESCENT
    NEWTON = _capi.RELOC_NEWTON


def default_reloc_cfg(**kw) -> _capi.RelocCfg:
    """RelocConfig (reloc.hpp:86-98) with the reference defaults; keyword overrides."""
    c = _capi.RelocCfg()
    _capi_lib().csf_default_reloc_cfg(C.byref(c))
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def _capi_lib():
    from . import library
    return library()


def _pose12(p) -> np.ndarray:
    return np.ascontiguousarray(lift_pose(p, 0)[:, 0])


class RelocProblem:
    """reloc.hpp:35-46: the reference volume flattened to its observed voxels
    (W > 0, storage order) plus the query depth, intrinsics and mu (the
    volume's).  Device-resident; `voxel_centers` / `reference_values` download
    on access."""

    def __init__(self, reference: _Volume, query_depth, k: _capi.Intrinsics):
        self.ctx = reference.ctx
        d = _f64(query_depth)
        if d.ndim != 2:
            raise InvalidArgument("query depth must be (h, w)")
        h, w = d.shape
        self.width, self.height = w, h
        self.intrinsics = k
        self.h = C.c_void_p()
        self.ctx.check(self.ctx.lib.csf_reloc_create(reference.h, _dp(np.ascontiguousarray(d)), w, h, C.byref(k),
                                                     C.byref(self.h)))
        n = C.c_int()
        mu = C.c_double()
        self.ctx.check(self.ctx.lib.csf_reloc_info(self.h, C.byref(n), C.byref(mu), None, None))
        self.n_voxels = n.value
        self.mu = mu.value

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            self.ctx.lib.csf_reloc_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def voxel_centers(self) -> np.ndarray:
        c = np.empty((self.n_voxels, 3))
        self.ctx.check(self.ctx.lib.csf_reloc_info(self.h, None, None, _dp(c), None))
        return c

    @property
    def reference_values(self) -> np.ndarray:
        v = np.empty(self.n_voxels)
        self.ctx.check(self.ctx.lib.csf_reloc_info(self.h, None, None, None, _dp(v)))
        return v

    def energy_derivs(self, pose, order: int = 2, h: float = 1e-8):
        """(E, g[6], H[6,6], overlap) at the camera->world pose in one device pass."""
        p = _pose12(pose)
        E = C.c_double()
        g = np.zeros(6)
        H = np.zeros((6, 6))
        ov = C.c_longlong()
        self.ctx.check(self.ctx.lib.csf_reloc_energy(self.h, _dp(p), order, h, C.byref(E),
                                                     _dp(g) if order >= 1 else None, _dp(H) if order >= 2 else None,
                                                     C.byref(ov)))
        return E.value, g, H, ov.value


def reloc_energy(problem: RelocProblem, query_pose) -> float:
    """reloc.hpp:48-69 at a real camera->world pose."""
    return problem.energy_derivs(query_pose, 0)[0]


def reloc_loss(problem: RelocProblem, pose) -> float:
    """reloc.hpp:71 — reloc_energy at the pose."""
    return problem.energy_derivs(pose, 0)[0]


def reloc_gradient(problem: RelocProblem, pose, h: float = 1e-8) -> np.ndarray:
    """reloc.hpp:75-77: d/dxi of reloc_energy(exp(xi) pose) at 0 (6 Complex passes, packed)."""
    return problem.energy_derivs(pose, 1, h)[1]


def reloc_hessian(problem: RelocProblem, pose, h: float = 1e-8) -> np.ndarray:
    """reloc.hpp:78-80: the symmetric Hessian (21 Bicomplex passes, packed)."""
    return problem.energy_derivs(pose, 2, h)[2]


@dataclass
class RelocResult:
    """reloc.hpp:100-106 plus the trace rows (loss, gradient norm per iteration)."""
    pose: np.ndarray
    iterations: int
    converged: bool
    final_loss: float
    method: RelocMethod
    losses: np.ndarray = field(default_factory=lambda: np.zeros(0))
    gradient_norms: np.ndarray = field(default_factory=lambda: np.zeros(0))


def relocalize(problem: RelocProblem, initial, method: RelocMethod = RelocMethod.NEWTON,
               cfg: Optional[_capi.RelocCfg] = None) -> RelocResult:
    """reloc.hpp:116-124: gradient descent, or steepest descent switching to the
    Newton direction once the loss is below the switch threshold; both with
    the backtracking line search of descent.hpp:34-52."""
    cfg = cfg if cfg is not None else default_reloc_cfg()
    init = _pose12(initial)
    out = np.empty(12)
    res = _capi.RelocResult()
    n = max(int(cfg.max_iterations), 0)
    losses = np.zeros(max(n, 1))
    gn = np.zeros(max(n, 1))
    ctx = problem.ctx
    ctx.check(ctx.lib.csf_relocalize(problem.h, _dp(init), int(method), C.byref(cfg), _dp(out), C.byref(res),
                                     _dp(losses), _dp(gn)))
    it = res.iterations
    return RelocResult(out.reshape(12), it, bool(res.converged), res.final_loss, RelocMethod(int(method)),
                       losses[:it].copy(), gn[:it].copy())


def build_reference(frames: Sequence, k: _capi.Intrinsics, params: _capi.VolumeParams,
                    ctx: Optional[Context] = None) -> TsdfVolume:
    """reloc.hpp:16-20: fuse (depth, camera->world) frames into a fresh dense
    volume at their poses (real scalar).  InvalidArgument on no frames."""
    if len(frames) == 0:
        raise InvalidArgument("build_reference: no frames")
    vol = TsdfVolume(tuple(params.dims), params.voxel_size, tuple(params.origin), params.mu, params.weight_cap,
                     channels=0, ctx=ctx)
    for depth, pose in frames:
        vol.surface_update(_f64(depth), pose, k)
    return vol


def select_reference_frames(poses: Sequence, initial, count: int = 10) -> list:
    """reloc.hpp:22-26: indices of the `count` poses whose camera centres are
    nearest the initial estimate, nearest first, ties by index."""
    t0 = _pose12(initial)[9:]
    d = []
    for i, p in enumerate(poses):
        t = _pose12(p)[9:]
        e = t - t0
        d.append((e[0] * e[0] + (e[1] * e[1] + e[2] * e[2]), i))
    d.sort()
    return [i for _, i in d[:max(count, 0)]]


def depth_cloud(depth, k: _capi.Intrinsics, camera_to_world, stride: int = 1,
                ctx: Optional[Context] = None) -> np.ndarray:
    """reloc.hpp:126-129: world points (n, 3) of the valid pixels at the stride, row-major."""
    c = _ctx(ctx)
    d = np.ascontiguousarray(_f64(depth))
    h, w = d.shape
    s = max(int(stride), 1)
    cap = ((w + s - 1) // s) * ((h + s - 1) // s)
    out = np.empty((max(cap, 1), 3))
    n = C.c_int()
    c.check(c.lib.csf_depth_cloud(c.h, _dp(d), w, h, C.byref(k), _dp(_pose12(camera_to_world)), int(stride),
                                  _dp(out), C.byref(n)))
    return out[:n.value].copy()


@dataclass
class NnError:
    """reloc.hpp:131-134"""
    mean: float
    outlier: bool


def eval_nn_error(transform, query, reference, ctx: Optional[Context] = None) -> NnError:
    """reloc.hpp:136-138: mean nearest-neighbour distance from transform * query to reference."""
    c = _ctx(ctx)
    q = np.ascontiguousarray(_f64(query).reshape(-1, 3))
    r = np.ascontiguousarray(_f64(reference).reshape(-1, 3))
    mean = C.c_double()
    out = C.c_int32()
    c.check(c.lib.csf_eval_nn_error(c.h, _dp(_pose12(transform)), _dp(q) if q.size else None, q.shape[0],
                                    _dp(r) if r.size else None, r.shape[0], C.byref(mean), C.byref(out)))
    return NnError(mean.value, bool(out.value))
