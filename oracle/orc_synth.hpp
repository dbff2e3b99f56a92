// ORACLE — TEST INFRASTRUCTURE ONLY (see orc_core.hpp header).
//
// Synthetic inputs: restates proj/include/csf/synth.hpp:17-73 and
// proj/src/synth.cpp:11-158 (SDF primitives, sphere-trace renderer storing
// camera-z depth, orbit poses, the platform-pinned GaussianSource, additive
// noise, 16-bit quantisation).  BUILDER-DEFINED additions (no reference):
// depth-dependent noise sigma = a*z^2, i.i.d. pixel dropout, and the seeded
// scene/trajectory generators of BASELINE configs 1 and 2 (DESIGN.md
// "Synthetic inputs").  Uniform draws use the top 53 bits of mt19937_64, the
// same construction GaussianSource uses (synth.cpp:121-127), so inputs are
// identical on every host.
#pragma once

#include <random>

#include "orc_core.hpp"
#include "orc_frames.hpp"

namespace orc {

struct SdfSphere { Vec3d center; double radius = 0.5; };
struct SdfBox { Vec3d center; Vec3d half_extents{0.25, 0.25, 0.25}; };
struct SdfPlane { Vec3d normal{0.0, 0.0, 1.0}; double offset = 0.0; };
// BUILDER-DEFINED (BASELINE config 4): a heightfield terrain as a sum of plane
// waves, z = sum_i a_i sin(kx_i x + ky_i y + phase_i).  Its distance bound
// (z - height) / sqrt(1 + L^2), L = sum_i |a_i| |k_i| >= |grad height|, keeps
// sphere tracing Lipschitz-safe (SURVEY §8(d) "needs a Lipschitz-safe step").
struct TerrainWave { double a = 0.0, kx = 0.0, ky = 0.0, phase = 0.0; };

inline double vmax3(const Vec3d& q) { return std::max(q[0], std::max(q[1], q[2])); }

// synth.cpp:11-34
struct Scene {
  std::vector<SdfSphere> spheres;
  std::vector<SdfBox> boxes;
  std::vector<SdfPlane> planes;
  std::vector<TerrainWave> terrain;
  double terrain_inv_lip = 1.0;
  double height(double x, double y) const {
    double hgt = 0.0;
    for (const auto& w : terrain) hgt = hgt + w.a * m_sin((w.kx * x + w.ky * y) + w.phase);
    return hgt;
  }
  double signed_distance(const Vec3d& p) const {
    double d = std::numeric_limits<double>::max();
    for (const auto& s : spheres) d = std::min(d, norm(p - s.center) - s.radius);
    for (const auto& b : boxes) {
      const Vec3d r = p - b.center;
      const Vec3d q(std::fabs(r[0]) - b.half_extents[0], std::fabs(r[1]) - b.half_extents[1],
                    std::fabs(r[2]) - b.half_extents[2]);
      const Vec3d outside(std::max(q[0], 0.0), std::max(q[1], 0.0), std::max(q[2], 0.0));
      const double inside = std::min(vmax3(q), 0.0);
      d = std::min(d, norm(outside) + inside);
    }
    for (const auto& pl : planes) d = std::min(d, dot(pl.normal, p) - pl.offset);
    if (!terrain.empty()) d = std::min(d, (p[2] - height(p[0], p[1])) * terrain_inv_lip);
    return d;
  }
  // synth.cpp:36-45
  Vec3d normal(const Vec3d& p, double eps = 1e-5) const {
    Vec3d n;
    for (int i = 0; i < 3; ++i) {
      Vec3d lo = p, hi = p;
      lo[i] -= eps;
      hi[i] += eps;
      n[i] = signed_distance(hi) - signed_distance(lo);
    }
    return normalized(n);
  }
};

// synth.cpp:55-90
inline Image<double> render_depth(const Scene& scene, const Pose& c2w, const Intrinsics& k, double far = 20.0,
                                  double hit_eps = 1e-6) {
  Image<double> depth(k.width, k.height, 0.0);
  const Vec3d origin = c2w.translation;
#pragma omp parallel for schedule(static)
  for (int y = 0; y < k.height; ++y)
    for (int x = 0; x < k.width; ++x) {
      Vec3d dir_cam((x - k.cx) / k.fx, (y - k.cy) / k.fy, 1.0);
      const double zfac = 1.0 / norm(dir_cam);
      dir_cam = Vec3d(dir_cam[0] * zfac, dir_cam[1] * zfac, dir_cam[2] * zfac);
      const Vec3d dir = c2w.rotation * dir_cam;
      double s = 0.0;
      for (int it = 0; it < 512 && s < far; ++it) {
        const double phi = scene.signed_distance(origin + s * dir);
        if (phi < hit_eps) {
          for (int r = 0; r < 3; ++r) {
            const Vec3d p = origin + s * dir;
            const double res = scene.signed_distance(p);
            const double slope = dot(dir, scene.normal(p));
            s -= res / std::min(slope, -0.05);
          }
          depth.at(x, y) = s * zfac;
          break;
        }
        s += phi;
      }
    }
  return depth;
}

// synth.cpp:92-105 (cos/sin through the deterministic kernels)
inline Pose orbit_pose(const Vec3d& target, double radius, double height, double angle) {
  const Vec3d eye = target + Vec3d(radius * m_cos(angle), radius * m_sin(angle), height);
  const Vec3d zc = normalized(target - eye);
  const Vec3d xc = normalized(cross(zc, Vec3d(0.0, 0.0, 1.0)));
  const Vec3d yc = cross(zc, xc);
  Pose p;
  for (int r = 0; r < 3; ++r) {
    p.rotation(r, 0) = xc[r];
    p.rotation(r, 1) = yc[r];
    p.rotation(r, 2) = zc[r];
  }
  p.translation = eye;
  return p;
}

// Camera at `eye` looking at `target` with the orbit_pose construction.
inline Pose look_at_pose(const Vec3d& eye, const Vec3d& target) {
  const Vec3d zc = normalized(target - eye);
  const Vec3d xc = normalized(cross(zc, Vec3d(0.0, 0.0, 1.0)));
  const Vec3d yc = cross(zc, xc);
  Pose p;
  for (int r = 0; r < 3; ++r) {
    p.rotation(r, 0) = xc[r];
    p.rotation(r, 1) = yc[r];
    p.rotation(r, 2) = zc[r];
  }
  p.translation = eye;
  return p;
}

// synth.cpp:116-133
class GaussianSource {
 public:
  explicit GaussianSource(uint64_t seed) : state_(seed) {}
  double next() {
    if (have_spare_) {
      have_spare_ = false;
      return spare_;
    }
    constexpr double kScale = 1.0 / 9007199254740992.0;
    double u1;
    do {
      u1 = static_cast<double>(state_() >> 11) * kScale;
    } while (u1 <= 0.0);
    const double u2 = static_cast<double>(state_() >> 11) * kScale;
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 2.0 * M_PI * u2;
    spare_ = r * std::sin(a);
    have_spare_ = true;
    return r * std::cos(a);
  }

 private:
  std::mt19937_64 state_;
  bool have_spare_ = false;
  double spare_ = 0.0;
};

// Top-53-bit uniform in [lo, hi) (builder-defined; same construction as above).
struct Uniform53 {
  std::mt19937_64 g;
  explicit Uniform53(uint64_t seed) : g(seed) {}
  double next01() { return static_cast<double>(g() >> 11) * (1.0 / 9007199254740992.0); }
  double next(double lo, double hi) { return lo + (hi - lo) * next01(); }
};

// synth.cpp:135-145
inline Image<double> add_depth_noise(const Image<double>& depth, double sigma, uint64_t seed) {
  GaussianSource gauss(seed);
  Image<double> out = depth;
  for (auto& d : out.data) {
    if (!(d > 0.0)) continue;
    const double noisy = d + sigma * gauss.next();
    d = noisy > 0.0 ? noisy : 0.0;
  }
  return out;
}

// Builder-defined sensor model for configs 2-4: sigma(z) = a*z^2 additive
// Gaussian on valid pixels, then i.i.d. dropout with probability p from an
// independent stream.
inline Image<double> add_depth_noise_quadratic(const Image<double>& depth, double a, double dropout,
                                               uint64_t seed) {
  GaussianSource gauss(seed);
  Uniform53 drop(seed ^ 0x9e3779b97f4a7c15ULL);
  Image<double> out = depth;
  for (auto& d : out.data) {
    if (!(d > 0.0)) continue;
    const double sigma = a * d * d;
    const double noisy = d + sigma * gauss.next();
    d = noisy > 0.0 ? noisy : 0.0;
    if (dropout > 0.0 && drop.next01() < dropout) d = 0.0;
  }
  return out;
}

// synth.cpp:147-158
inline Image<double> quantize_depth(const Image<double>& depth, double scale = 5000.0) {
  Image<double> out = depth;
  for (auto& d : out.data) {
    if (!(d > 0.0)) {
      d = 0.0;
      continue;
    }
    const double q = std::round(d * scale);
    d = (q >= 1.0 && q <= 65535.0) ? q / scale : 0.0;
  }
  return out;
}

// Round-trip through float32 (BASELINE: frames are float32 metres).
inline Image<double> to_float32(const Image<double>& depth) {
  Image<double> out = depth;
  for (auto& d : out.data) d = static_cast<double>(static_cast<float>(d));
  return out;
}

// Inward-facing room: six half-spaces whose union leaves the box interior
// free (SdfBox is solid inside, synth.hpp:22-31, so it cannot model a room).
inline void add_room(Scene& s, double x0, double x1, double y0, double y1, double z0, double z1) {
  s.planes.push_back({Vec3d(0.0, 0.0, 1.0), z0});
  s.planes.push_back({Vec3d(0.0, 0.0, -1.0), -z1});
  s.planes.push_back({Vec3d(1.0, 0.0, 0.0), x0});
  s.planes.push_back({Vec3d(-1.0, 0.0, 0.0), -x1});
  s.planes.push_back({Vec3d(0.0, 1.0, 0.0), y0});
  s.planes.push_back({Vec3d(0.0, -1.0, 0.0), -y1});
}

}  // namespace orc
