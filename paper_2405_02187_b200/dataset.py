"""On-disk formats — host mirror of proj/include/csf/dataset.hpp over the
C-ABI: 16-bit depth PNGs, the intrinsics text file,
TUM-style trajectories, and sequence directories (depth/ + associations.txt
+ groundtruth.txt + intrinsics.txt).  File I/O runs on the host, as in the
reference (dataset.cpp); the decoded frames feed the device pipeline.
Errors: RuntimeError (std::runtime_error) with the reference's messages."""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from pathlib import Path
from typing import List, Sequence as Seq

import numpy as np

from . import capi as _capi


def _lib():
    from . import library
    return library()


def _check(rc: int) -> None:
    if rc == _capi.CSF_OK:
        return
    msg = (_lib().csf_io_last_error() or b"").decode()
    if rc == _capi.CSF_EINVAL:
        from . import InvalidArgument
        raise InvalidArgument(msg or "invalid argument")
    raise RuntimeError(msg)


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def write_depth_png16(path, depth, scale: float) -> None:
    """dataset.hpp:19-20: depth in metres -> 16-bit PNG at `scale` units per metre (0 = no measurement)."""
    d = np.ascontiguousarray(depth, dtype=np.float64)
    h, w = d.shape
    _check(_lib().csf_write_depth_png16(os.fsencode(str(path)), _dp(d), w, h, float(scale)))


def read_depth_png16(path, scale: float) -> np.ndarray:
    """dataset.hpp:21: 16-bit grayscale PNG -> depth (h, w) in metres."""
    w, h = C.c_int(), C.c_int()
    p = os.fsencode(str(path))
    _check(_lib().csf_read_depth_png16(p, float(scale), None, C.byref(w), C.byref(h)))
    out = np.empty((h.value, w.value))
    _check(_lib().csf_read_depth_png16(p, float(scale), _dp(out), C.byref(w), C.byref(h)))
    return out


def read_intrinsics(path) -> _capi.Intrinsics:
    """dataset.hpp:23-27: seven numbers fx fy cx cy width height depth_scale ('#' comments)."""
    k = _capi.Intrinsics()
    _check(_lib().csf_read_intrinsics(os.fsencode(str(path)), C.byref(k)))
    return k


def write_intrinsics(path, k: _capi.Intrinsics) -> None:
    _check(_lib().csf_write_intrinsics(os.fsencode(str(path)), C.byref(k)))


@dataclass
class TrajectoryEntry:
    """dataset.hpp:30-33 (pose camera->world as 12 numbers)."""
    timestamp: float
    pose: np.ndarray


def read_trajectory(path) -> List[TrajectoryEntry]:
    """dataset.hpp:35-36: lines 't tx ty tz qx qy qz qw'."""
    p = os.fsencode(str(path))
    n = C.c_int()
    _check(_lib().csf_read_trajectory(p, None, None, 0, C.byref(n)))
    ts = np.empty(max(n.value, 1))
    poses = np.empty((max(n.value, 1), 12))
    _check(_lib().csf_read_trajectory(p, _dp(ts), _dp(poses), n.value, C.byref(n)))
    return [TrajectoryEntry(float(ts[i]), poses[i].copy()) for i in range(n.value)]


def write_trajectory(path, traj: Seq[TrajectoryEntry]) -> None:
    ts = np.ascontiguousarray([e.timestamp for e in traj], dtype=np.float64)
    poses = np.ascontiguousarray([np.asarray(e.pose, dtype=np.float64).reshape(12) for e in traj]).reshape(-1, 12)
    _check(_lib().csf_write_trajectory(os.fsencode(str(path)), _dp(ts) if len(traj) else None,
                                       _dp(poses) if len(traj) else None, len(traj)))


@dataclass
class SequenceFrame:
    """dataset.hpp:38-41"""
    timestamp: float
    depth_path: str


@dataclass
class Sequence:
    """dataset.hpp:43-51"""
    directory: str
    intrinsics: _capi.Intrinsics
    frames: List[SequenceFrame] = field(default_factory=list)
    groundtruth: List[TrajectoryEntry] = field(default_factory=list)

    def load_depth(self, i: int) -> np.ndarray:
        """Depth of frame i, resolved against `directory` (dataset.cpp:179-184)."""
        p = Path(self.frames[i].depth_path)
        full = p if p.is_absolute() else Path(self.directory) / p
        return read_depth_png16(full, self.intrinsics.depth_scale)


def _strip(line: str) -> str:
    h = line.find("#")
    return line if h < 0 else line[:h]


def open_sequence(directory) -> Sequence:
    """dataset.hpp:53-55 (dataset.cpp:186-209)."""
    d = Path(directory)
    seq = Sequence(str(directory), read_intrinsics(d / "intrinsics.txt"))
    assoc = d / "associations.txt"
    if not assoc.exists():
        raise RuntimeError(f"cannot open associations: {assoc}")
    for line in assoc.read_text().splitlines():
        parts = _strip(line).split()
        if len(parts) < 2:
            continue
        try:
            t = float(parts[0])
        except ValueError:
            continue
        seq.frames.append(SequenceFrame(t, parts[1]))
    if not seq.frames:
        raise RuntimeError(f"sequence has no frames: {directory}")
    gt = d / "groundtruth.txt"
    if gt.exists():
        seq.groundtruth = read_trajectory(gt)
    return seq


def write_sequence(directory, k: _capi.Intrinsics, depths, groundtruth: Seq[TrajectoryEntry] = ()) -> None:
    """dataset.hpp:57-62 (dataset.cpp:211-238): depth/NNNNNN.png + associations.txt
    (+ groundtruth.txt) + intrinsics.txt."""
    d = Path(directory)
    (d / "depth").mkdir(parents=True, exist_ok=True)
    write_intrinsics(d / "intrinsics.txt", k)
    lines = ["# timestamp depth_file"]
    for i, depth in enumerate(depths):
        name = f"depth/{i:06d}.png"
        write_depth_png16(d / name, depth, k.depth_scale)
        t = groundtruth[i].timestamp if i < len(groundtruth) else float(i)
        lines.append(f"{t!r} {name}")
    (d / "associations.txt").write_text("\n".join(lines) + "\n")
    if len(groundtruth):
        write_trajectory(d / "groundtruth.txt", groundtruth)
