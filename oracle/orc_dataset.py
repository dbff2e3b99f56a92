"""ORACLE — TEST INFRASTRUCTURE ONLY.

Independent numpy/zlib restatement of the on-disk formats of
proj/src/dataset.cpp (the reference links libpng, absent here): a PNG codec
for 16-bit grayscale images that can write every row filter (0-4) and split
IDAT chunks, so the product's reader is checked against files it did not
write, and decodes the product's files on its own; quantize_depth
(synth.cpp:147-158); Eigen's quaternion <-> rotation formulas.
"""
from __future__ import annotations

import struct
import zlib

import numpy as np

SIG = b"\x89PNG\r\n\x1a\n"


def quantize_depth(d, scale=5000.0):
    """synth.cpp:147-158"""
    d = np.asarray(d, dtype=np.float64)
    q = np.round(d * scale)  # numpy rounds half to even; std::round half away — fix below
    q = np.where(np.abs(d * scale - np.trunc(d * scale)) == 0.5, np.trunc(d * scale) + np.sign(d), q)
    ok = (d > 0) & (q >= 1.0) & (q <= 65535.0)
    return np.where(ok, q / scale, 0.0)


def _chunk(t: bytes, data: bytes) -> bytes:
    return struct.pack(">I", len(data)) + t + data + struct.pack(">I", zlib.crc32(t + data) & 0xffffffff)


def _paeth(a, b, c):
    p = a + b - c
    pa, pb, pc = abs(p - a), abs(p - b), abs(p - c)
    if pa <= pb and pa <= pc:
        return a
    return b if pb <= pc else c


def encode_u16(img: np.ndarray, filters=None, idat_split: int = 0) -> bytes:
    """16-bit grayscale PNG of uint16 img (h, w); filters: per-row filter types."""
    h, w = img.shape
    raw = img.astype(">u2").tobytes()
    stride = 2 * w
    prev = bytearray(stride)
    out = bytearray()
    for y in range(h):
        row = raw[y * stride:(y + 1) * stride]
        f = 0 if filters is None else int(filters[y % len(filters)])
        enc = bytearray(stride)
        for i in range(stride):
            a = row[i - 2] if i >= 2 else 0
            b = prev[i]
            c = prev[i - 2] if i >= 2 else 0
            pred = [0, a, b, (a + b) // 2, _paeth(a, b, c)][f]
            enc[i] = (row[i] - pred) & 0xff
        out += bytes([f]) + enc
        prev = bytearray(row)
    z = zlib.compress(bytes(out))
    parts = [z] if idat_split <= 0 else [z[i:i + idat_split] for i in range(0, len(z), idat_split)]
    ihdr = struct.pack(">IIBBBBB", w, h, 16, 0, 0, 0, 0)
    return SIG + _chunk(b"IHDR", ihdr) + b"".join(_chunk(b"IDAT", p) for p in parts) + _chunk(b"IEND", b"")


def decode_u16(data: bytes) -> np.ndarray:
    assert data[:8] == SIG
    pos, idat, w = 8, b"", None
    while pos < len(data):
        n = struct.unpack(">I", data[pos:pos + 4])[0]
        t = data[pos + 4:pos + 8]
        body = data[pos + 8:pos + 8 + n]
        if t == b"IHDR":
            w, h, bd, ct, _, _, il = struct.unpack(">IIBBBBB", body)
            assert bd == 16 and ct == 0 and il == 0
        elif t == b"IDAT":
            idat += body
        elif t == b"IEND":
            break
        pos += 12 + n
    raw = zlib.decompress(idat)
    stride = 2 * w
    prev = bytearray(stride)
    rows = []
    for y in range(h):
        f = raw[y * (stride + 1)]
        enc = raw[y * (stride + 1) + 1:(y + 1) * (stride + 1)]
        cur = bytearray(stride)
        for i in range(stride):
            a = cur[i - 2] if i >= 2 else 0
            b = prev[i]
            c = prev[i - 2] if i >= 2 else 0
            pred = [0, a, b, (a + b) // 2, _paeth(a, b, c)][f]
            cur[i] = (enc[i] + pred) & 0xff
        rows.append(bytes(cur))
        prev = cur
    return np.frombuffer(b"".join(rows), dtype=">u2").reshape(h, w).astype(np.uint16)


def quat_to_rot(qw, qx, qy, qz):
    """Eigen Quaterniond(w, x, y, z).normalized().toRotationMatrix()"""
    n = np.sqrt(qx * qx + qy * qy + qz * qz + qw * qw)
    w, x, y, z = qw / n, qx / n, qy / n, qz / n
    tx, ty, tz = 2 * x, 2 * y, 2 * z
    twx, twy, twz = tx * w, ty * w, tz * w
    txx, txy, txz = tx * x, ty * x, tz * x
    tyy, tyz, tzz = ty * y, tz * y, tz * z
    return np.array([[1 - (tyy + tzz), txy - twz, txz + twy], [txy + twz, 1 - (txx + tzz), tyz - twx],
                     [txz - twy, tyz + twx, 1 - (txx + tyy)]])
