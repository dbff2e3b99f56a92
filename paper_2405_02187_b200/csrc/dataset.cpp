// On-disk formats either side of the hot path:
// proj/include/csf/dataset.hpp / proj/src/dataset.cpp — 16-bit depth PNGs,
// the plain-text intrinsics file and TUM-style timestamped trajectories.
//
// Host code (file I/O and parsing, as in the reference).  The reference links
// libpng, which this image lacks; the PNG container is written and read here
// directly over zlib (deflate) with the same observable behaviour:
//   write_depth_png16 (dataset.cpp:30-68): 16-bit grayscale, big-endian
//     samples, q = round(d * scale) kept when 1 <= q <= 65535, else 0;
//     rows written with filter type 0.
//   read_depth_png16  (dataset.cpp:70-107): any valid non-interlaced 16-bit
//     grayscale PNG (all five row filters, any IDAT split); v > 0 -> v/scale;
//     anything else -> "expected 16-bit grayscale PNG" (std::runtime_error).
//   read/write_intrinsics (dataset.cpp:109-141), read/write_trajectory
//     (dataset.cpp:143-177) with the quaternion <-> rotation conversions of
//     Eigen::Quaterniond (normalized().toRotationMatrix(), and the
//     trace-branch construction from a rotation matrix), restated.
#include <zlib.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/csf_b200.h"

namespace {

thread_local std::string g_io_err;

int io_fail(const std::string& what, const std::string& path) {
  g_io_err = what + ": " + path;
  return CSF_ERUNTIME;
}

void put32(std::vector<uint8_t>& o, uint32_t v) {
  o.push_back(static_cast<uint8_t>(v >> 24));
  o.push_back(static_cast<uint8_t>(v >> 16));
  o.push_back(static_cast<uint8_t>(v >> 8));
  o.push_back(static_cast<uint8_t>(v));
}
uint32_t get32(const uint8_t* p) {
  return (uint32_t(p[0]) << 24) | (uint32_t(p[1]) << 16) | (uint32_t(p[2]) << 8) | uint32_t(p[3]);
}

void chunk(std::vector<uint8_t>& o, const char* type, const uint8_t* data, size_t n) {
  put32(o, static_cast<uint32_t>(n));
  const size_t start = o.size();
  o.insert(o.end(), type, type + 4);
  if (n) o.insert(o.end(), data, data + n);
  put32(o, static_cast<uint32_t>(crc32(0L, o.data() + start, static_cast<uInt>(n + 4))));
}

const uint8_t kSig[8] = {137, 80, 78, 71, 13, 10, 26, 10};

int paeth(int a, int b, int c) {
  const int p = a + b - c;
  const int pa = std::abs(p - a), pb = std::abs(p - b), pc = std::abs(p - c);
  if (pa <= pb && pa <= pc) return a;
  if (pb <= pc) return b;
  return c;
}

// Eigen::Quaterniond(w, x, y, z).normalized().toRotationMatrix()
void quat_to_rot(double qw, double qx, double qy, double qz, double* R) {
  const double n = std::sqrt(qx * qx + qy * qy + qz * qz + qw * qw);  // coeffs() order x, y, z, w
  const double w = qw / n, x = qx / n, y = qy / n, z = qz / n;
  const double tx = 2 * x, ty = 2 * y, tz = 2 * z;
  const double twx = tx * w, twy = ty * w, twz = tz * w;
  const double txx = tx * x, txy = ty * x, txz = tz * x;
  const double tyy = ty * y, tyz = tz * y, tzz = tz * z;
  R[0] = 1 - (tyy + tzz); R[1] = txy - twz;       R[2] = txz + twy;
  R[3] = txy + twz;       R[4] = 1 - (txx + tzz); R[5] = tyz - twx;
  R[6] = txz - twy;       R[7] = tyz + twx;       R[8] = 1 - (txx + tyy);
}

// Eigen::Quaterniond(const Matrix3d&) (quaternion_assign_impl: trace branch,
// else the largest diagonal), returned as (x, y, z, w).
void rot_to_quat(const double* m, double* q) {
  auto M = [&](int r, int c) { return m[3 * r + c]; };
  const double t = M(0, 0) + M(1, 1) + M(2, 2);
  if (t > 0) {
    double s = std::sqrt(t + 1.0);
    q[3] = 0.5 * s;
    s = 0.5 / s;
    q[0] = (M(2, 1) - M(1, 2)) * s;
    q[1] = (M(0, 2) - M(2, 0)) * s;
    q[2] = (M(1, 0) - M(0, 1)) * s;
  } else {
    int i = 0;
    if (M(1, 1) > M(0, 0)) i = 1;
    if (M(2, 2) > M(i, i)) i = 2;
    const int j = (i + 1) % 3, k = (j + 1) % 3;
    double s = std::sqrt(M(i, i) - M(j, j) - M(k, k) + 1.0);
    q[i] = 0.5 * s;
    s = 0.5 / s;
    q[3] = (M(k, j) - M(j, k)) * s;
    q[j] = (M(j, i) + M(i, j)) * s;
    q[k] = (M(k, i) + M(i, k)) * s;
  }
}

void strip_comment(std::string& line) {
  const auto hash = line.find('#');
  if (hash != std::string::npos) line.erase(hash);
}

}  // namespace

extern "C" const char* csf_io_last_error(void) { return g_io_err.c_str(); }

extern "C" int csf_write_depth_png16(const char* path, const double* depth, int w, int h, double scale) {
  if (!path || !depth || w <= 0 || h <= 0) return CSF_EINVAL;
  const size_t stride = 1 + 2 * static_cast<size_t>(w);
  std::vector<uint8_t> raw(stride * h);
  for (int y = 0; y < h; ++y) {
    uint8_t* row = raw.data() + stride * y;
    row[0] = 0;  // filter: None
    for (int x = 0; x < w; ++x) {
      const double d = depth[static_cast<size_t>(y) * w + x];
      uint16_t v = 0;
      if (d > 0.0) {
        const double q = std::round(d * scale);
        if (q >= 1.0 && q <= 65535.0) v = static_cast<uint16_t>(q);
      }
      row[1 + 2 * x] = static_cast<uint8_t>(v >> 8);  // PNG is big-endian
      row[2 + 2 * x] = static_cast<uint8_t>(v & 0xff);
    }
  }
  uLongf zlen = compressBound(static_cast<uLong>(raw.size()));
  std::vector<uint8_t> z(zlen);
  if (compress2(z.data(), &zlen, raw.data(), static_cast<uLong>(raw.size()), Z_DEFAULT_COMPRESSION) != Z_OK)
    return io_fail("deflate failed", path);
  std::vector<uint8_t> out(kSig, kSig + 8);
  uint8_t ihdr[13];
  const uint32_t ww = static_cast<uint32_t>(w), hh = static_cast<uint32_t>(h);
  for (int i = 0; i < 4; ++i) {
    ihdr[i] = static_cast<uint8_t>(ww >> (24 - 8 * i));
    ihdr[4 + i] = static_cast<uint8_t>(hh >> (24 - 8 * i));
  }
  ihdr[8] = 16;  // bit depth
  ihdr[9] = 0;   // grayscale
  ihdr[10] = ihdr[11] = ihdr[12] = 0;
  chunk(out, "IHDR", ihdr, 13);
  chunk(out, "IDAT", z.data(), zlen);
  chunk(out, "IEND", nullptr, 0);
  std::FILE* f = std::fopen(path, "wb");
  if (!f) return io_fail("cannot open for writing", path);
  const bool ok = std::fwrite(out.data(), 1, out.size(), f) == out.size();
  std::fclose(f);
  return ok ? CSF_OK : io_fail("write failed", path);
}

// depth == NULL: report the size only.
extern "C" int csf_read_depth_png16(const char* path, double scale, double* depth, int* w_out, int* h_out) {
  if (!path || !w_out || !h_out) return CSF_EINVAL;
  std::FILE* f = std::fopen(path, "rb");
  if (!f) return io_fail("cannot open for reading", path);
  std::vector<uint8_t> buf;
  uint8_t tmp[1 << 16];
  size_t got;
  while ((got = std::fread(tmp, 1, sizeof(tmp), f)) > 0) buf.insert(buf.end(), tmp, tmp + got);
  std::fclose(f);
  if (buf.size() < 8 || std::memcmp(buf.data(), kSig, 8) != 0) return io_fail("libpng read failed", path);
  size_t pos = 8;
  uint32_t w = 0, h = 0;
  int bit_depth = -1, color = -1, interlace = 0;
  std::vector<uint8_t> idat;
  bool seen_end = false;
  while (pos + 12 <= buf.size()) {
    const uint32_t len = get32(buf.data() + pos);
    if (pos + 12 + static_cast<size_t>(len) > buf.size()) return io_fail("libpng read failed", path);
    const uint8_t* type = buf.data() + pos + 4;
    const uint8_t* data = type + 4;
    const uint32_t crc = get32(data + len);
    if (crc != static_cast<uint32_t>(crc32(0L, type, len + 4))) return io_fail("libpng read failed", path);
    if (!std::memcmp(type, "IHDR", 4)) {
      if (len != 13) return io_fail("libpng read failed", path);
      w = get32(data);
      h = get32(data + 4);
      bit_depth = data[8];
      color = data[9];
      interlace = data[12];
    } else if (!std::memcmp(type, "IDAT", 4)) {
      idat.insert(idat.end(), data, data + len);
    } else if (!std::memcmp(type, "IEND", 4)) {
      seen_end = true;
      break;
    }
    pos += 12 + len;
  }
  if (!seen_end || w == 0 || h == 0) return io_fail("libpng read failed", path);
  if (bit_depth != 16 || color != 0 || interlace != 0) return io_fail("expected 16-bit grayscale PNG", path);
  if (w > 1u << 15 || h > 1u << 15) return io_fail("libpng read failed", path);
  *w_out = static_cast<int>(w);
  *h_out = static_cast<int>(h);
  if (!depth) return CSF_OK;
  const size_t stride = 1 + 2 * static_cast<size_t>(w);
  std::vector<uint8_t> raw(stride * h);
  uLongf rlen = static_cast<uLongf>(raw.size());
  if (uncompress(raw.data(), &rlen, idat.data(), static_cast<uLong>(idat.size())) != Z_OK || rlen != raw.size())
    return io_fail("libpng read failed", path);
  const int bpp = 2;
  std::vector<uint8_t> prev(stride - 1, 0), cur(stride - 1);
  for (uint32_t y = 0; y < h; ++y) {
    const uint8_t* row = raw.data() + stride * y;
    const int filter = row[0];
    for (size_t i = 0; i + 1 < stride; ++i) {
      const int a = i >= bpp ? cur[i - bpp] : 0, b = prev[i], c = i >= bpp ? prev[i - bpp] : 0;
      int v = row[1 + i];
      switch (filter) {
        case 0: break;
        case 1: v += a; break;
        case 2: v += b; break;
        case 3: v += (a + b) / 2; break;
        case 4: v += paeth(a, b, c); break;
        default: return io_fail("libpng read failed", path);
      }
      cur[i] = static_cast<uint8_t>(v);
    }
    for (uint32_t x = 0; x < w; ++x) {
      const uint16_t v = static_cast<uint16_t>((cur[2 * x] << 8) | cur[2 * x + 1]);
      depth[static_cast<size_t>(y) * w + x] = v > 0 ? static_cast<double>(v) / scale : 0.0;
    }
    std::swap(prev, cur);
  }
  return CSF_OK;
}

extern "C" int csf_read_intrinsics(const char* path, csf_intrinsics* k) {
  if (!path || !k) return CSF_EINVAL;
  std::ifstream in(path);
  if (!in) return io_fail("cannot open intrinsics", path);
  std::vector<double> nums;
  std::string line;
  while (std::getline(in, line)) {
    strip_comment(line);
    std::istringstream ls(line);
    double v;
    while (ls >> v) nums.push_back(v);
  }
  if (nums.size() != 7) return io_fail("intrinsics file must contain exactly 7 numbers", path);
  csf_intrinsics o;
  o.fx = nums[0];
  o.fy = nums[1];
  o.cx = nums[2];
  o.cy = nums[3];
  o.width = static_cast<int>(nums[4]);
  o.height = static_cast<int>(nums[5]);
  o.depth_scale = nums[6];
  if (o.fx <= 0 || o.fy <= 0 || o.width <= 0 || o.height <= 0 || o.depth_scale <= 0)
    return io_fail("intrinsics values out of range", path);
  *k = o;
  return CSF_OK;
}

extern "C" int csf_write_intrinsics(const char* path, const csf_intrinsics* k) {
  if (!path || !k) return CSF_EINVAL;
  std::ofstream out(path);
  if (!out) return io_fail("cannot write intrinsics", path);
  out << "# fx fy cx cy width height depth_scale\n";
  out.precision(17);
  out << k->fx << " " << k->fy << " " << k->cx << " " << k->cy << " " << k->width << " " << k->height << " "
      << k->depth_scale << "\n";
  return out ? CSF_OK : io_fail("cannot write intrinsics", path);
}

// timestamps [cap], poses [cap][12] camera->world (rotation row-major,
// translation); both NULL: count only.
extern "C" int csf_read_trajectory(const char* path, double* timestamps, double* poses, int cap, int* n_out) {
  if (!path || !n_out) return CSF_EINVAL;
  std::ifstream in(path);
  if (!in) return io_fail("cannot open trajectory", path);
  std::string line;
  int n = 0;
  while (std::getline(in, line)) {
    strip_comment(line);
    std::istringstream ls(line);
    double t, tx, ty, tz, qx, qy, qz, qw;
    if (!(ls >> t >> tx >> ty >> tz >> qx >> qy >> qz >> qw)) continue;
    if ((timestamps || poses) && n < cap) {
      if (timestamps) timestamps[n] = t;
      if (poses) {
        quat_to_rot(qw, qx, qy, qz, poses + 12 * n);
        poses[12 * n + 9] = tx;
        poses[12 * n + 10] = ty;
        poses[12 * n + 11] = tz;
      }
    }
    ++n;
  }
  *n_out = n;
  return CSF_OK;
}

extern "C" int csf_write_trajectory(const char* path, const double* timestamps, const double* poses, int n) {
  if (!path || n < 0 || (n > 0 && (!timestamps || !poses))) return CSF_EINVAL;
  std::ofstream out(path);
  if (!out) return io_fail("cannot write trajectory", path);
  out << "# timestamp tx ty tz qx qy qz qw\n";
  out.precision(17);
  for (int i = 0; i < n; ++i) {
    const double* p = poses + 12 * i;
    double q[4];
    rot_to_quat(p, q);
    out << timestamps[i] << " " << p[9] << " " << p[10] << " " << p[11] << " " << q[0] << " " << q[1] << " " << q[2]
        << " " << q[3] << "\n";
  }
  return out ? CSF_OK : io_fail("cannot write trajectory", path);
}
