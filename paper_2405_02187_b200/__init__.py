"""B200-native CSFD dense-SLAM hot path (X-SLAM, arXiv 2405.02187).

Python host mirror of the reference's C++ API (proj/include/csf/*.hpp) over
the C-ABI in include/csf_b200.h.  Names, argument meaning and error types
follow the reference:

    bilateral_filter, downsample_depth, build_depth_pyramid  (frames.hpp:56-65)
    measure_surface                                            (frames.hpp:86-114)
    TsdfVolume / HashedVolume, surface_update, raycast         (tsdf.hpp:38-284)
    track_frame                                                (icp.hpp:130-133)
    Pipeline (the CSFD frame-derivative run)
    RelocProblem, reloc_energy/gradient/hessian, relocalize   (reloc.hpp:35-138)

Errors: CSF_EINVAL -> InvalidArgument (ValueError, std::invalid_argument),
CSF_EDOMAIN -> DomainError (ArithmeticError, std::domain_error), everything
else -> RuntimeError (std::runtime_error).

Lifted values carry D perturbation channels as a trailing axis of size 1+D
(index 0 = real part).  Poses are camera->world (12, 1+D): rotation
row-major then translation.  Every compute call runs on the sm_100a kernels;
importing works without a GPU but creating a Context requires one.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence, Tuple

import numpy as np

from . import capi as _capi

__all__ = [
    "InvalidArgument", "DomainError", "Context", "bilateral_filter", "downsample_depth", "build_depth_pyramid",
    "measure_surface", "TsdfVolume", "HashedVolume", "surface_update", "raycast", "track_frame", "TrackResult",
    "TrackTrace", "TraceRow", "write_trace_csv",
    "icp_energy", "icp_loss", "icp_gradient", "icp_hessian", "icp_energy_derivs", "associate", "linearized_step",
    "pairwise_sum", "complex_depth", "perturb_depth",
    "Pipeline", "PipelineResult", "HessianResult", "synth_workload", "look_at", "config5_views", "save_volume", "load_volume", "measured_tsdf", "default_icp_cfg", "default_raycast_cfg", "intrinsics",
    "lift_pose", "lift_intrinsics", "library",
]


class InvalidArgument(ValueError):
    """std::invalid_argument"""


class DomainError(ArithmeticError):
    """std::domain_error"""


_LIB: Optional[C.CDLL] = None


def library() -> C.CDLL:
    global _LIB
    if _LIB is None:
        _LIB = _capi.load_library()
    return _LIB


def _raise(rc: int, msg: str) -> None:
    if rc == _capi.CSF_OK:
        return
    if rc == _capi.CSF_EINVAL:
        raise InvalidArgument(msg)
    if rc == _capi.CSF_EDOMAIN:
        raise DomainError(msg)
    raise RuntimeError(f"csf_b200 error {rc}: {msg}")


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _fp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


class Context:
    """One device context: a CUDA stream and an error flag (csf_ctx_create)."""

    _default: Optional["Context"] = None

    def __init__(self, device: int = 0):
        self.lib = library()
        h = C.c_void_p()
        rc = self.lib.csf_ctx_create(device, C.byref(h))
        if rc != _capi.CSF_OK:
            raise RuntimeError(f"csf_ctx_create(device={device}) failed with {rc}: no usable CUDA device "
                               "(the sm_100a path has no CPU fallback)")
        self.h = h
        self.device = device

    @classmethod
    def default(cls) -> "Context":
        if cls._default is None:
            cls._default = Context(0)
        return cls._default

    def check(self, rc: int) -> None:
        if rc != _capi.CSF_OK:
            msg = self.lib.csf_last_error(self.h)
            _raise(rc, msg.decode() if msg else "")

    def synchronize(self) -> None:
        self.check(self.lib.csf_ctx_synchronize(self.h))

    def attach_comm(self, n_ranks: int, rank: int, unique_id: bytes) -> None:
        """The context's NCCL communicator for csf_gather_columns (rank 0's
        comm_unique_id(), shared with every rank)."""
        if len(unique_id) != 128:
            raise InvalidArgument("unique_id must be 128 bytes")
        self.check(self.lib.csf_ctx_attach_comm(self.h, n_ranks, rank, unique_id))

    def gather_columns(self, local, counts) -> np.ndarray:
        """csf_gather_columns: counts[r] columns from every rank r, in rank
        order, on every rank (SURVEY §8(e) collective C2)."""
        loc = _f64(np.asarray(local, dtype=np.float64).reshape(-1))
        cnt = (C.c_int * len(counts))(*[int(c) for c in counts])
        out = np.zeros(int(sum(counts)))
        self.check(self.lib.csf_gather_columns(self.h, _dp(loc), cnt, _dp(out)))
        return out

    @property
    def launch_count(self) -> int:
        n = C.c_ulonglong()
        self.check(self.lib.csf_ctx_launch_count(self.h, C.byref(n)))
        return int(n.value)

    def profile(self, enable: bool = True) -> None:
        """Per-kernel-category CUDA-event timing on this context's stream."""
        self.check(self.lib.csf_ctx_profile(self.h, int(enable)))

    def profile_read(self) -> dict:
        """{category: (total_ms, launches)} since the last read."""
        names = C.create_string_buffer(32 * 16)
        ms = np.zeros(16)
        cnt = np.zeros(16, dtype=np.int64)
        n = C.c_int()
        self.check(self.lib.csf_ctx_profile_read(self.h, 16, names, _dp(ms),
                                                 cnt.ctypes.data_as(C.POINTER(C.c_longlong)), C.byref(n)))
        out = {}
        for i in range(n.value):
            nm = names.raw[32 * i: 32 * i + 32].split(b"\0", 1)[0].decode()
            out[nm] = (float(ms[i]), int(cnt[i]))
        return out

    @property
    def stream(self) -> int:
        return int(self.lib.csf_ctx_stream(self.h) or 0)

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.csf_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _ctx(ctx: Optional[Context]) -> Context:
    return ctx if ctx is not None else Context.default()


# ----------------------------------------------------------------------------- config helpers
def intrinsics(fx=525.0, fy=525.0, cx=319.5, cy=239.5, width=640, height=480, depth_scale=5000.0):
    """frames.hpp:15-22 defaults."""
    return _capi.Intrinsics(fx, fy, cx, cy, width, height, depth_scale)


def default_icp_cfg(**kw) -> _capi.IcpCfg:
    c = _capi.IcpCfg()
    library().csf_default_icp_cfg(C.byref(c))
    for k, v in kw.items():
        if k in ("level_iterations", "level_pixel_stride"):
            getattr(c, k)[:] = list(v)
        else:
            setattr(c, k, v)
    return c


def default_raycast_cfg(**kw) -> _capi.RaycastCfg:
    c = _capi.RaycastCfg(0.0, 10.0, 0.5)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def lift_pose(pose, channels: int = 0) -> np.ndarray:
    """(12,) / (3,4) / (4,4) real pose -> (12, 1+D) with zero channels."""
    p = np.asarray(pose, dtype=np.float64)
    if p.shape == (4, 4):
        p = np.concatenate([p[:3, :3].reshape(9), p[:3, 3]])
    elif p.shape == (3, 4):
        p = np.concatenate([p[:, :3].reshape(9), p[:, 3]])
    if p.shape == (12,):
        out = np.zeros((12, 1 + channels))
        out[:, 0] = p
        return out
    if p.shape == (12, 1 + channels):
        return _f64(p)
    raise InvalidArgument(f"pose must be (12,), (3,4), (4,4) or (12,{1 + channels}); got {p.shape}")


def lift_intrinsics(k, channels: int = 0) -> np.ndarray:
    if isinstance(k, _capi.Intrinsics):
        out = np.zeros((4, 1 + channels))
        out[:, 0] = [k.fx, k.fy, k.cx, k.cy]
        return out
    a = np.asarray(k, dtype=np.float64)
    if a.shape == (4,):
        out = np.zeros((4, 1 + channels))
        out[:, 0] = a
        return out
    if a.shape == (4, 1 + channels):
        return _f64(a)
    raise InvalidArgument(f"intrinsics must be csf Intrinsics, (4,) or (4,{1 + channels}); got {a.shape}")


# ----------------------------------------------------------------------------- frames
def bilateral_filter(depth, sigma_s: float = 4.5, sigma_r: float = 0.03, radius: int = 3,
                     ctx: Optional[Context] = None) -> np.ndarray:
    """frames.cpp:7-38 on the device."""
    c = _ctx(ctx)
    d = _f64(depth)
    h, w = d.shape
    out = np.empty_like(d)
    c.check(c.lib.csf_bilateral_filter(c.h, _dp(d), w, h, sigma_s, sigma_r, radius, _dp(out)))
    return out


def downsample_depth(depth, sigma_r: float = 0.03, ctx: Optional[Context] = None) -> np.ndarray:
    """frames.cpp:40-66 on the device."""
    c = _ctx(ctx)
    d = _f64(depth)
    h, w = d.shape
    out = np.empty((h // 2, w // 2))
    c.check(c.lib.csf_downsample_depth(c.h, _dp(d), w, h, sigma_r, _dp(out)))
    return out


def build_depth_pyramid(depth, levels: int = 3, sigma_r: float = 0.03, ctx: Optional[Context] = None):
    """frames.cpp:68-75."""
    pyr = [_f64(depth)]
    for _ in range(1, levels):
        pyr.append(downsample_depth(pyr[-1], sigma_r, ctx))
    return pyr


def measure_surface(depth, k, channels: int = 0, ctx: Optional[Context] = None):
    """frames.hpp:86-114.  depth (h, w) or (h, w, 1+D); returns (V, N) of shape (h, w, 3, 1+D)."""
    c = _ctx(ctx)
    d = _f64(depth)
    if d.ndim == 2:
        d = np.ascontiguousarray(np.stack([d] + [np.zeros_like(d)] * channels, axis=-1))
    h, w, cc = d.shape
    D = cc - 1
    kk = lift_intrinsics(k, D)
    V = np.empty((h, w, 3, 1 + D))
    N = np.empty((h, w, 3, 1 + D))
    c.check(c.lib.csf_measure_surface(c.h, _dp(d), w, h, _dp(kk), D, _dp(V), _dp(N)))
    return V, N


# ----------------------------------------------------------------------------- volumes
class _Volume:
    hashed = False

    def __init__(self, ctx: Optional[Context], channels: int):
        self.ctx = _ctx(ctx)
        self.channels = channels
        self.h = C.c_void_p()

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            self.ctx.lib.csf_volume_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def surface_update(self, depth, pose, k) -> int:
        """tsdf.cpp:11-40; returns the visible block count (hashed) or 0.
        depth (h, w) real, or (h, w, 1+D) lifted: the reference's
        Image<Complex> depth, whose channels enter psi (tsdf.hpp:144-145)."""
        d = _f64(depth)
        p = lift_pose(pose, self.channels)
        kk = lift_intrinsics(k, self.channels)
        nv = C.c_int(0)
        if d.ndim == 3:
            h, w, cc = d.shape
            if cc != 1 + self.channels:
                raise InvalidArgument(f"lifted depth must have 1 + {self.channels} channels")
            self.ctx.check(self.ctx.lib.csf_surface_update_lifted(self.h, _dp(d), w, h, _dp(p), _dp(kk),
                                                                  C.byref(nv)))
        else:
            h, w = d.shape
            self.ctx.check(self.ctx.lib.csf_surface_update(self.h, _dp(d), w, h, _dp(p), _dp(kk), C.byref(nv)))
        return nv.value

    def raycast(self, pose, k, width: int, height: int, cfg: Optional[_capi.RaycastCfg] = None):
        """tsdf.hpp:209-284; returns (V, N) of shape (h, w, 3, 1+D)."""
        p = lift_pose(pose, self.channels)
        kk = lift_intrinsics(k, self.channels)
        V = np.empty((height, width, 3, 1 + self.channels))
        N = np.empty_like(V)
        cfgp = C.byref(cfg) if cfg is not None else None
        self.ctx.check(self.ctx.lib.csf_raycast(self.h, _dp(p), _dp(kk), width, height, cfgp, _dp(V), _dp(N)))
        return V, N

    def voxel_count(self) -> int:
        raise NotImplementedError

    def download(self):
        n = self.voxel_count()
        field = np.empty((n, 1 + self.channels))
        weight = np.empty(n)
        self.ctx.check(self.ctx.lib.csf_volume_download(self.h, _dp(field), _dp(weight)))
        return field, weight

    def upload(self, field, weight):
        f = _f64(field)
        wt = _f64(weight)
        self.ctx.check(self.ctx.lib.csf_volume_upload(self.h, _dp(f), _dp(wt)))

    def _points(self, points):
        P = _f64(points)
        if P.ndim == 2 and P.shape[1] == 3:
            Q = np.zeros((P.shape[0], 3, 1 + self.channels))
            Q[..., 0] = P
            P = Q
        if P.ndim != 3 or P.shape[1:] != (3, 1 + self.channels):
            raise InvalidArgument(f"points must be (n, 3) or (n, 3, {1 + self.channels})")
        return np.ascontiguousarray(P)

    def sample_tsdf(self, points):
        """tsdf.hpp:148-177 at lifted world points: (values (n, 1+D), valid (n,) bool)."""
        P = self._points(points)
        out = np.zeros((P.shape[0], 1 + self.channels))
        ok = np.zeros(P.shape[0], dtype=np.int32)
        self.ctx.check(self.ctx.lib.csf_sample_tsdf(self.h, _dp(P), P.shape[0], _dp(out),
                                                    ok.ctypes.data_as(C.POINTER(C.c_int32))))
        return out, ok.astype(bool)

    def sample_gradient(self, points):
        """tsdf.hpp:181-196: (gradients (n, 3, 1+D), valid (n,) bool)."""
        P = self._points(points)
        out = np.zeros((P.shape[0], 3, 1 + self.channels))
        ok = np.zeros(P.shape[0], dtype=np.int32)
        self.ctx.check(self.ctx.lib.csf_sample_gradient(self.h, _dp(P), P.shape[0], _dp(out),
                                                        ok.ctypes.data_as(C.POINTER(C.c_int32))))
        return out, ok.astype(bool)

    def save(self, path) -> None:
        """save_volume (tsdf.cpp:61-97): the "CSFVOL 1" checkpoint."""
        self.ctx.check(self.ctx.lib.csf_volume_save(self.h, str(path).encode()))


class TsdfVolume(_Volume):
    """Dense lattice volume (tsdf.hpp:38-78), F carries `channels` perturbation channels."""

    def __init__(self, dims=(128, 128, 128), voxel_size=0.02, origin=(0.0, 0.0, 0.0), mu=0.1, weight_cap=128.0,
                 channels: int = 0, ctx: Optional[Context] = None):
        super().__init__(ctx, channels)
        self.params = _capi.VolumeParams((C.c_int * 3)(*dims), voxel_size, (C.c_double * 3)(*origin), mu, weight_cap)
        self.ctx.check(self.ctx.lib.csf_volume_create_dense(self.ctx.h, C.byref(self.params), channels,
                                                            C.byref(self.h)))

    @classmethod
    def cube(cls, n: int, voxel: float, origin, channels: int = 0, ctx: Optional[Context] = None):
        """VolumeParams::cube (tsdf.hpp:28-35): mu = 5 voxels."""
        return cls((n, n, n), voxel, origin, 5.0 * voxel, 128.0, channels, ctx)

    def voxel_count(self) -> int:
        d = self.params.dims
        return d[0] * d[1] * d[2]


class HashedVolume(_Volume):
    """Hashed 8^3-block volume (builder-defined)."""
    hashed = True

    def __init__(self, voxel_size=0.005, origin=(0.0, 0.0, 0.0), mu=0.025, weight_cap=128.0, bucket_bits=20,
                 max_blocks=1 << 18, channels: int = 0, ctx: Optional[Context] = None):
        super().__init__(ctx, channels)
        self.params = _capi.HashParams(voxel_size, (C.c_double * 3)(*origin), mu, weight_cap, bucket_bits, max_blocks)
        self.ctx.check(self.ctx.lib.csf_volume_create_hashed(self.ctx.h, C.byref(self.params), channels,
                                                             C.byref(self.h)))

    def block_count(self) -> int:
        n = C.c_int()
        self.ctx.check(self.ctx.lib.csf_volume_block_count(self.h, C.byref(n)))
        return n.value

    def voxel_count(self) -> int:
        return self.block_count() * 512

    def hash_tables(self):
        nb = self.block_count()
        heads = np.empty(1 << self.params.bucket_bits, dtype=np.int32)
        keys = np.empty(nb, dtype=np.uint64)
        nxt = np.empty(nb, dtype=np.int32)
        coords = np.empty((nb, 3), dtype=np.int32)
        self.ctx.check(self.ctx.lib.csf_volume_download_hash(
            self.h, heads.ctypes.data_as(C.POINTER(C.c_int32)), keys.ctypes.data_as(C.POINTER(C.c_uint64)),
            nxt.ctypes.data_as(C.POINTER(C.c_int32)), coords.ctypes.data_as(C.POINTER(C.c_int32))))
        return heads, keys, nxt, coords

    def view_scores(self, poses, k: _capi.Intrinsics, w0: float = 10.0, beta: float = 0.5, h: float = 1e-8):
        """BASELINE config 5 (builder-defined objective, csf_view_scores): per candidate
        camera->world view (n, 12) the soft count of weakly observed surface it would see
        and its CSFD gradient w.r.t. the view's twist.  Needs channels == 6."""
        P = _f64(poses).reshape(-1, 12)
        sc = np.empty(P.shape[0])
        g = np.empty((P.shape[0], 6))
        self.ctx.check(self.ctx.lib.csf_view_scores(self.h, _dp(P), P.shape[0], C.byref(k), w0, beta, h, _dp(sc),
                                                    _dp(g)))
        return sc, g


def look_at(eye, target, up=(0.0, 0.0, 1.0)) -> np.ndarray:
    """camera->world pose (12,) of a camera at `eye` looking at `target` (z forward, y down)."""
    eye, target, up = (np.asarray(a, dtype=np.float64) for a in (eye, target, up))
    z = target - eye
    z /= np.linalg.norm(z)
    x = np.cross(z, up)
    if np.linalg.norm(x) < 1e-9:
        x = np.cross(z, np.array([1.0, 0.0, 0.0]))
    x /= np.linalg.norm(x)
    y = np.cross(z, x)
    R = np.stack([x, y, z], axis=1)
    return np.concatenate([R.reshape(9), eye])


def comm_unique_id() -> bytes:
    """A fresh NCCL unique id (csf_comm_unique_id), created on rank 0."""
    buf = C.create_string_buffer(128)
    rc = library().csf_comm_unique_id(buf)
    if rc != _capi.CSF_OK:
        raise RuntimeError("csf_comm_unique_id failed (libnccl.so.2 unavailable?)")
    return buf.raw


def config5_views(n: int = 256, seed: int = 4) -> np.ndarray:
    """BASELINE config 5 candidate views (builder-defined, synthetic): n camera->world
    poses (n, 12) with eyes uniform in the free annulus kept clear around the config-2
    camera orbit (radius 0.9-1.5 m, height 0.9-1.7 m) looking at targets uniform in the
    room interior, drawn from a seeded generator."""
    rng = np.random.default_rng(seed)
    out = np.empty((n, 12))
    for i in range(n):
        r, th, z = rng.uniform(0.9, 1.5), rng.uniform(0.0, 2 * np.pi), rng.uniform(0.9, 1.7)
        eye = np.array([r * np.cos(th), r * np.sin(th), z])
        target = np.array([rng.uniform(-1.6, 1.6), rng.uniform(-1.6, 1.6), rng.uniform(0.3, 2.5)])
        out[i] = look_at(eye, target)
    return out


def measured_tsdf(depth, world_to_camera, k, mu: float, points, center, ctx: Optional[Context] = None):
    """tsdf.hpp:97-140 at real voxel positions (n, 3): (psi (n, 1+D), valid (n,) bool); the
    pose (12, 1+D), intrinsics (4, 1+D) and camera centre (3, 1+D) carry D channels."""
    c = _ctx(ctx)
    d = _f64(depth)
    pose = _f64(world_to_camera)
    D = pose.shape[1] - 1 if pose.ndim == 2 else 0
    lifted = d.ndim == 3
    if lifted:  # (h, w, 1+D): the depth carries its own channels (tsdf.hpp:97-102)
        h, w, cc = d.shape
        D = max(D, cc - 1)
        if cc != 1 + D:
            raise InvalidArgument("lifted depth and pose channel counts differ")
    else:
        h, w = d.shape
    pose = lift_pose(pose, D)
    kk = lift_intrinsics(k, D)
    cen = _f64(center).reshape(3, -1)
    if cen.shape[1] != 1 + D:
        cen = np.concatenate([cen[:, :1], np.zeros((3, D))], axis=1)
    P = np.ascontiguousarray(_f64(points).reshape(-1, 3))
    out = np.zeros((P.shape[0], 1 + D))
    ok = np.zeros(P.shape[0], dtype=np.int32)
    fn = c.lib.csf_measured_tsdf_lifted if lifted else c.lib.csf_measured_tsdf
    c.check(fn(c.h, _dp(d), w, h, _dp(pose), _dp(kk), mu, _dp(P), _dp(np.ascontiguousarray(cen)), P.shape[0], D,
               _dp(out), ok.ctypes.data_as(C.POINTER(C.c_int32))))
    return out, ok.astype(bool)


def save_volume(path, volume: _Volume) -> None:
    """tsdf.hpp:288 save_volume(path, volume)."""
    volume.save(path)


def load_volume(path, channels: int = -1, ctx: Optional[Context] = None) -> _Volume:
    """tsdf.hpp:289 load_volume(path): a dense TsdfVolume (or, for the hashed
    extension of the format, a HashedVolume) on the device; channels = -1 keeps
    the file's derivative channels.  Errors: RuntimeError (std::runtime_error)."""
    c = _ctx(ctx)
    h = C.c_void_p()
    c.check(c.lib.csf_volume_load(c.h, str(path).encode(), channels, C.byref(h)))
    with open(path, "rb") as f:
        head = f.read(4096).split(b"\ndata\n", 1)[0].decode(errors="replace").splitlines()
    fields = {ln.split()[0]: ln.split()[1:] for ln in head[1:] if ln.strip()}
    n_im = fields.get("channels", []).count("derivative")
    ch = channels if channels >= 0 else n_im
    vs, org = float(fields["voxel_size"][0]), tuple(float(x) for x in fields["origin"])
    mu, cap = float(fields["mu"][0]), float(fields["weight_cap"][0])
    if "hashed" in fields:
        vol = HashedVolume.__new__(HashedVolume)
        _Volume.__init__(vol, c, ch)
        bits, mb = int(fields["hashed"][0]), int(fields["hashed"][1])
        vol.params = _capi.HashParams(vs, (C.c_double * 3)(*org), mu, cap, bits, mb)
    else:
        vol = TsdfVolume.__new__(TsdfVolume)
        _Volume.__init__(vol, c, ch)
        dims = tuple(int(x) for x in fields["dims"])
        vol.params = _capi.VolumeParams((C.c_int * 3)(*dims), vs, (C.c_double * 3)(*org), mu, cap)
    vol.h = h
    return vol


def surface_update(volume: _Volume, depth, camera_to_world, k) -> int:
    return volume.surface_update(depth, camera_to_world, k)


def raycast(volume: _Volume, camera_to_world, k, width=None, height=None, cfg=None):
    if width is None:
        width, height = k.width, k.height
    return volume.raycast(camera_to_world, k, width, height, cfg)


@dataclass
class TrackResult:
    """icp.hpp:119-125"""
    pose: np.ndarray
    iterations: int
    converged: bool
    final_loss: float
    correspondences: int


@dataclass
class TraceRow:
    """icp.hpp:103-109"""
    iteration: int
    loss: float
    gradient_norm: float
    translation_error: float
    rotation_error: float  # degrees


@dataclass
class TrackTrace:
    """icp.hpp:111-114: optional ground truth (12,) and the per-iteration rows."""
    ground_truth: Optional[np.ndarray] = None
    rows: list = None

    def __post_init__(self):
        if self.rows is None:
            self.rows = []


def track_frame(volume: _Volume, depth, init_camera_to_world, k, cfg: Optional[_capi.IcpCfg] = None,
                trace: Optional[TrackTrace] = None) -> TrackResult:
    """icp.cpp:169-244 on the device, every solver family (cfg.solver:
    linearized, Newton — the reference default — gradient descent, NCG).
    With `trace`, one TraceRow per iteration is appended (icp.cpp:213-228)."""
    ctx = volume.ctx
    d = _f64(depth)
    h, w = d.shape
    init = lift_pose(init_camera_to_world, 0)[:, 0].copy()
    out = np.empty(12)
    res = _capi.TrackResult()
    cfg = cfg if cfg is not None else default_icp_cfg()
    if trace is None:
        ctx.check(ctx.lib.csf_track_frame(volume.h, _dp(d), w, h, _dp(init), C.byref(k), C.byref(cfg), _dp(out),
                                          C.byref(res)))
    else:
        cap = max(int(sum(cfg.level_iterations)), 1)
        rows = np.zeros((cap, 15))
        n = C.c_int()
        ctx.check(ctx.lib.csf_track_frame_traced(volume.h, _dp(d), w, h, _dp(init), C.byref(k), C.byref(cfg),
                                                 _dp(out), C.byref(res), _dp(rows), cap, C.byref(n)))
        gt = None if trace.ground_truth is None else lift_pose(trace.ground_truth, 0)[:, 0]
        for r in rows[:min(n.value, cap)]:
            te = re_ = float("nan")
            if gt is not None:
                dt = r[12:15] - gt[9:]
                te = float(np.sqrt(dt[0] * dt[0] + (dt[1] * dt[1] + dt[2] * dt[2])))
                rel = gt[:9].reshape(3, 3).T @ r[3:12].reshape(3, 3)
                re_ = float(np.degrees(np.arccos(np.clip((np.trace(rel) - 1.0) / 2.0, -1.0, 1.0))))  # se3.hpp:109-113
            trace.rows.append(TraceRow(int(r[0]), float(r[1]), float(r[2]), te, re_))
    return TrackResult(out, res.iterations, bool(res.converged), res.final_loss, res.correspondences)


def write_trace_csv(path, trace: TrackTrace) -> None:
    """icp.cpp:155-167"""
    lines = ["iteration,loss,gradient norm,translation error,rotation error"]
    g = lambda v: format(v, ".17g") if v == v else "nan"
    for r in trace.rows:
        lines.append(f"{r.iteration},{g(r.loss)},{g(r.gradient_norm)},{g(r.translation_error)},{g(r.rotation_error)}")
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")


# ----------------------------------------------------------------------------- icp: associate / linearized step
def associate(measured, predicted, camera_to_world, predicted_camera_to_world, k, cfg=None, pixel_stride: int = 1,
              ctx: Optional[Context] = None) -> np.ndarray:
    """icp.cpp:89-126: correspondences (n, 9) in scan order from measured (V camera, N) and
    predicted (V, N world) maps of shape (h, w, 3) each."""
    c = _ctx(ctx)
    mv, mn = (_f64(a)[..., :3] if _f64(a).ndim == 3 else _f64(a)[..., :, 0] for a in measured)
    pv, pn = (_f64(a)[..., :3] if _f64(a).ndim == 3 else _f64(a)[..., :, 0] for a in predicted)
    mv, mn, pv, pn = (np.ascontiguousarray(a) for a in (mv, mn, pv, pn))
    h, w = mv.shape[:2]
    cw = lift_pose(camera_to_world, 0)[:, 0].copy()
    pw = lift_pose(predicted_camera_to_world, 0)[:, 0].copy()
    cfg = cfg if cfg is not None else default_icp_cfg()
    stride = max(1, pixel_stride)
    out = np.empty((((w + stride - 1) // stride) * ((h + stride - 1) // stride), 9))
    n = C.c_int()
    c.check(c.lib.csf_associate(c.h, _dp(mv), _dp(mn), _dp(pv), _dp(pn), w, h, _dp(cw), _dp(pw), C.byref(k),
                                C.byref(cfg), stride, _dp(out), C.byref(n)))
    return out[: n.value].copy()


def linearized_step(corrs, base, ctx: Optional[Context] = None) -> np.ndarray:
    """icp.cpp:146-153: the small-angle Gauss-Newton step (canonical tiled normal equations)."""
    c = _ctx(ctx)
    cc = _corrs(corrs)
    b = lift_pose(base, 0)[:, 0].copy()
    d = np.empty(6)
    c.check(c.lib.csf_linearized_step(c.h, _dp(cc) if cc.size else None, cc.shape[0], _dp(b), _dp(d)))
    return d


def pairwise_sum(terms, ctx: Optional[Context] = None):
    """diff.hpp:16-37: the reference's fixed summation tree (per lane of (n, C) terms)."""
    c = _ctx(ctx)
    t = _f64(terms)
    scalar = t.ndim == 1
    t = np.ascontiguousarray(t.reshape(-1, 1) if scalar else t.reshape(t.shape[0], int(np.prod(t.shape[1:]))))
    out = np.empty(t.shape[1])
    c.check(c.lib.csf_pairwise_sum(c.h, _dp(t) if t.size else None, t.shape[0], t.shape[1], _dp(out)))
    return float(out[0]) if scalar else out


# ----------------------------------------------------------------------------- frames: depth lifts
def complex_depth(depth) -> np.ndarray:
    """frames.cpp:77-81: depth lifted with a zero channel, shape (h, w, 2)."""
    d = _f64(depth)
    out = np.zeros(d.shape + (2,))
    out[..., 0] = d
    return out


def perturb_depth(depth, x: int, y: int, h: float = 1e-8, delta_edge: float = 0.1) -> np.ndarray:
    """frames.cpp:83-102: seed pixel (x, y) with im = h; refuses (InvalidArgument) out-of-bounds
    pixels, pixels without depth and pixels on a depth discontinuity (an in-bounds 4-neighbour
    invalid or more than delta_edge away)."""
    if not (0.0 < h <= 1e-6):
        raise InvalidArgument("StepSize: step must satisfy 0 < h <= 1e-6")
    d = _f64(depth)
    H, W = d.shape
    if not (0 <= x < W and 0 <= y < H):
        raise InvalidArgument("perturb_depth: pixel out of bounds")
    center = d[y, x]
    if not center > 0.0:
        raise InvalidArgument("perturb_depth: pixel has no depth")
    for nx, ny in ((x - 1, y), (x + 1, y), (x, y - 1), (x, y + 1)):
        if not (0 <= nx < W and 0 <= ny < H):
            continue
        v = d[ny, nx]
        if not v > 0.0 or abs(v - center) > delta_edge:
            raise InvalidArgument("perturb_depth: pixel sits on a depth discontinuity")
    out = complex_depth(d)
    out[y, x, 1] = h
    return out


# ----------------------------------------------------------------------------- icp energy
def _corrs(corrs) -> np.ndarray:
    """Correspondences as (n, 9): vertex (camera), model vertex, model normal (world) — icp.hpp:27-31."""
    c = np.ascontiguousarray(corrs, dtype=np.float64)
    if c.ndim == 3 and c.shape[1:] == (3, 3):
        c = c.reshape(-1, 9)
    if c.ndim != 2 or c.shape[1] != 9:
        raise InvalidArgument(f"correspondences must be (n, 9) or (n, 3, 3); got {c.shape}")
    return np.ascontiguousarray(c)


def _energy(corrs, base, xi, h, want_g, want_h, ctx):
    c = _ctx(ctx)
    cc = _corrs(corrs)
    b = lift_pose(base, 0)[:, 0].copy()
    x = np.zeros(6) if xi is None else _f64(xi).reshape(6)
    E = C.c_double()
    g = np.zeros(6)
    H = np.zeros((6, 6))
    c.check(c.lib.csf_icp_energy_derivs(c.h, _dp(cc) if cc.size else None, cc.shape[0], _dp(b), _dp(x), h,
                                        C.byref(E), _dp(g) if want_g else None, _dp(H) if want_h else None))
    return E.value, g, H


def icp_energy(corrs, xi, base, ctx: Optional[Context] = None) -> float:
    """icp.hpp:70-85: sum over correspondences of ((exp(xi) base v - mv) . mn)^2, pairwise_sum tree."""
    return _energy(corrs, base, xi, 1e-8, False, False, ctx)[0]


def icp_loss(corrs, base, ctx: Optional[Context] = None) -> float:
    """icp.cpp:128-130: icp_energy at xi = 0."""
    return _energy(corrs, base, None, 1e-8, False, False, ctx)[0]


def icp_gradient(corrs, base, h: float = 1e-8, ctx: Optional[Context] = None) -> np.ndarray:
    """icp.cpp:132-137: CSFD gradient (6 Complex passes, one packed device pass)."""
    return _energy(corrs, base, None, h, True, False, ctx)[1]


def icp_hessian(corrs, base, h: float = 1e-8, ctx: Optional[Context] = None) -> np.ndarray:
    """icp.cpp:139-144: CSFD Hessian (21 Bicomplex passes, mirrored; one packed device pass)."""
    return _energy(corrs, base, None, h, False, True, ctx)[2]


def icp_energy_derivs(corrs, base, xi=None, h: float = 1e-8, ctx: Optional[Context] = None):
    """(energy, gradient[6], hessian[6,6]) at xi in one device call (csf_icp_energy_derivs)."""
    return _energy(corrs, base, xi, h, True, True, ctx)


# ----------------------------------------------------------------------------- pipeline
@dataclass
class PipelineResult:
    gradient: np.ndarray
    objective: float
    poses: Optional[np.ndarray] = None
    stats: Optional[np.ndarray] = None


class Pipeline:
    """The CSFD frame-derivative run on the device (csf_pipeline_*)."""

    def __init__(self, cfg: _capi.PipelineCfg, ctx: Optional[Context] = None):
        self.ctx = _ctx(ctx)
        self.cfg = cfg
        self.order = 2 if cfg.order == 2 else 1
        self.n_pairs = cfg.n_pairs if self.order == 2 else 0
        # outputs per run: D first-order derivatives, or one Hessian entry per pair
        self.D = self.n_pairs if self.order == 2 else cfg.n_dirs
        self.slots = 3 * self.n_pairs if self.order == 2 else cfg.n_dirs
        self.h = C.c_void_p()
        self.ctx.check(self.ctx.lib.csf_pipeline_create(self.ctx.h, C.byref(cfg), C.byref(self.h)))
        self.n_frames = 0

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            self.ctx.lib.csf_pipeline_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def upload(self, depth: np.ndarray, gt: np.ndarray) -> None:
        d = np.ascontiguousarray(depth, dtype=np.float32)
        g = _f64(gt).reshape(-1, 12)
        self.n_frames = self.n_run = d.shape[0]
        self.ctx.check(self.ctx.lib.csf_pipeline_upload(self.h, _fp(d), _dp(g), self.n_frames))

    def run(self, n_frames: Optional[int] = None) -> None:
        self.n_run = n_frames or self.n_frames
        self.ctx.check(self.ctx.lib.csf_pipeline_run(self.h, self.n_run))

    def set_graph(self, enable: bool = True) -> None:
        """Replay runs as one captured CUDA graph (csf_pipeline_set_graph)."""
        self.ctx.check(self.ctx.lib.csf_pipeline_set_graph(self.h, int(enable)))

    def result(self, poses: bool = True, stats: bool = True) -> PipelineResult:
        n = getattr(self, "n_run", self.n_frames)
        g = np.zeros(max(self.D, 1))
        obj = C.c_double()
        P = np.empty((n, 12, 1 + self.slots)) if poses else None
        S = np.empty((n, 8), dtype=np.int32) if stats else None
        self.ctx.check(self.ctx.lib.csf_pipeline_result(
            self.h, _dp(g), C.byref(obj), _dp(P) if P is not None else None,
            S.ctypes.data_as(C.POINTER(C.c_int32)) if S is not None else None))
        return PipelineResult(g[: self.D].copy(), obj.value, P, S)

    def volume(self) -> "_Volume":
        """The pipeline's volume after the last run (csf_pipeline_volume):
        borrowed from the pipeline, which it keeps alive; read-only use
        (download, hash_tables, block_count, sample_*)."""
        h = C.c_void_p()
        self.ctx.check(self.ctx.lib.csf_pipeline_volume(self.h, C.byref(h)))
        cls = HashedVolume if self.cfg.hashed else TsdfVolume
        v = cls.__new__(cls)
        _Volume.__init__(v, self.ctx, self.slots)
        v.h = h
        v.params = self.cfg.hash if self.cfg.hashed else self.cfg.dense
        v._owner = self
        v.close = lambda: None  # the pipeline owns the handle
        return v

    def run_host(self, depth: np.ndarray, gt: np.ndarray, rgb: np.ndarray | None = None) -> PipelineResult:
        """End-to-end call from host buffers (upload + run + read back).
        rgb: optional uint8 colour frames [n][h][w][3] (csf_pipeline_run_host_rgbd:
        ingested beside the depth, unused by the path, as the reference)."""
        d = np.ascontiguousarray(depth, dtype=np.float32)
        g = _f64(gt).reshape(-1, 12)
        self.n_frames = self.n_run = d.shape[0]
        grad = np.zeros(max(self.D, 1))
        obj = C.c_double()
        if rgb is None:
            self.ctx.check(self.ctx.lib.csf_pipeline_run_host(self.h, _fp(d), _dp(g), self.n_frames, _dp(grad),
                                                              C.byref(obj)))
        else:
            c = np.ascontiguousarray(rgb, dtype=np.uint8)
            if c.shape != d.shape + (3,):
                raise ValueError(f"rgb must be {d.shape + (3,)} uint8, got {c.shape}")
            self.ctx.check(self.ctx.lib.csf_pipeline_run_host_rgbd(
                self.h, _fp(d), c.ctypes.data_as(C.POINTER(C.c_ubyte)), _dp(g), self.n_frames, _dp(grad),
                C.byref(obj)))
        return PipelineResult(grad[: self.D].copy(), obj.value)

    def rgb_frame(self, frame: int) -> np.ndarray:
        """Colour frame `frame` as ingested by the last run_host(rgb=...)."""
        out = np.empty((self.cfg.k.height, self.cfg.k.width, 3), np.uint8)
        self.ctx.check(self.ctx.lib.csf_pipeline_download_rgb(self.h, frame, out.ctypes.data_as(C.POINTER(C.c_ubyte))))
        return out

    def hessian(self, poses: bool = False, stats: bool = False) -> "HessianResult":
        """Order-2 result: H_{i_p j_p} per pair and the pair's first-order
        derivatives d obj / d param i_p, j_p (csf_pipeline_hessian)."""
        P_ = self.n_pairs
        H, g1, g2 = np.empty(P_), np.empty(P_), np.empty(P_)
        obj = C.c_double()
        n = getattr(self, "n_run", self.n_frames)
        P = np.empty((n, 12, 1 + self.slots)) if poses else None
        S = np.empty((n, 8), dtype=np.int32) if stats else None
        self.ctx.check(self.ctx.lib.csf_pipeline_hessian(
            self.h, _dp(H), _dp(g1), _dp(g2), C.byref(obj), _dp(P) if P is not None else None,
            S.ctypes.data_as(C.POINTER(C.c_int32)) if S is not None else None))
        return HessianResult(H, g1, g2, obj.value, P, S)


@dataclass
class HessianResult:
    hessian: np.ndarray
    grad1: np.ndarray
    grad2: np.ndarray
    objective: float
    poses: Optional[np.ndarray] = None
    stats: Optional[np.ndarray] = None


def make_pipeline_cfg(*, hashed: bool, k: _capi.Intrinsics, dirs: Sequence[int], h: float, objective: int,
                      max_frames: int, dense: Optional[_capi.VolumeParams] = None,
                      hash_params: Optional[_capi.HashParams] = None, icp: Optional[_capi.IcpCfg] = None,
                      rc: Optional[_capi.RaycastCfg] = None,
                      pairs: Optional[Sequence[Tuple[int, int]]] = None,
                      keyframe_interval: int = 0) -> _capi.PipelineCfg:
    """Pipeline descriptor.  `dirs` = first-order parameters (0..5 twist, 6..9
    fx, fy, cx, cy); `pairs` (instead of dirs) = second-order parameter pairs
    (i, j), order 2 (BASELINE config 3).  keyframe_interval K > 0 enables the
    keyframe codes 10 + 6 (kf - 1) + c (BASELINE config 4)."""
    cfg = _capi.PipelineCfg()
    cfg.hashed = int(hashed)
    if dense is not None:
        cfg.dense = dense
    if hash_params is not None:
        cfg.hash = hash_params
    cfg.k = k
    cfg.icp = icp if icp is not None else default_icp_cfg(solver=_capi.SOLVER_LINEARIZED)
    cfg.rc = rc if rc is not None else default_raycast_cfg()
    cfg.h = h
    cfg.n_dirs = len(dirs)
    for i, d in enumerate(dirs):
        cfg.dirs[i] = d
    cfg.objective = objective
    cfg.max_frames = max_frames
    cfg.keyframe_interval = keyframe_interval
    cfg.order = 1
    if pairs is not None:
        if len(dirs):
            raise ValueError("make_pipeline_cfg: give dirs (order 1) or pairs (order 2), not both")
        if not 0 < len(pairs) <= _capi.CSF_MAX_PAIRS:
            raise ValueError("make_pipeline_cfg: 1..CSF_MAX_PAIRS pairs")
        cfg.order = 2
        cfg.n_pairs = len(pairs)
        for p, (i, j) in enumerate(pairs):
            cfg.pair_i[p] = i
            cfg.pair_j[p] = j
    return cfg


def synth_workload(config: int, n_frames: int, width: int = 0, height: int = 0, ctx: Optional[Context] = None):
    """BASELINE config 1/2 inputs rendered on the device: (depth float32 (n,h,w), gt (n,12), Intrinsics)."""
    c = _ctx(ctx)
    k = _capi.Intrinsics()
    if width == 0:
        w, h = (160, 120) if config == 1 else (640, 480)
    else:
        w, h = width, height
    depth = np.empty((n_frames, h, w), dtype=np.float32)
    gt = np.empty((n_frames, 12))
    c.check(c.lib.csf_synth_workload(c.h, config, n_frames, width, height, _fp(depth), _dp(gt), C.byref(k)))
    return depth, gt, k


# ----------------------------------------------------------------------------- relocalization (reloc.hpp)
from .reloc import (NnError, RelocMethod, RelocProblem, RelocResult, build_reference, default_reloc_cfg,  # noqa: E402
                    depth_cloud, eval_nn_error, relocalize, reloc_energy, reloc_gradient, reloc_hessian, reloc_loss,
                    select_reference_frames)

__all__ += ["NnError", "RelocMethod", "RelocProblem", "RelocResult", "build_reference", "default_reloc_cfg",
            "depth_cloud", "eval_nn_error", "relocalize", "reloc_energy", "reloc_gradient", "reloc_hessian",
            "reloc_loss", "select_reference_frames"]

# ----------------------------------------------------------------------------- on-disk formats (dataset.hpp)
from .dataset import (Sequence, SequenceFrame, TrajectoryEntry, open_sequence, read_depth_png16,  # noqa: E402
                      read_intrinsics, read_trajectory, write_depth_png16, write_intrinsics, write_sequence,
                      write_trajectory)

__all__ += ["Sequence", "SequenceFrame", "TrajectoryEntry", "open_sequence", "read_depth_png16", "read_intrinsics",
            "read_trajectory", "write_depth_png16", "write_intrinsics", "write_sequence", "write_trajectory"]

# ----------------------------------------------------------------------------- surfel front end (surfel.hpp)
from .surfel import (IndexMap, SurfelMap, SurfelUpdateStats, associate_all, associate_one_to_many,  # noqa: E402
                     default_surfel_cfg, predict_maps, render_index_map, sample_confidence, update_surfels,
                     write_surfel_ply)

__all__ += ["IndexMap", "SurfelMap", "SurfelUpdateStats", "associate_all", "associate_one_to_many",
            "default_surfel_cfg", "predict_maps", "render_index_map", "sample_confidence", "update_surfels",
            "write_surfel_ply"]
