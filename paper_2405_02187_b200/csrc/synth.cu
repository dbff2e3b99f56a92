// Synthetic-input harness (not on the timed path): the reference's SDF scene
// model and sphere-trace renderer (proj/src/synth.cpp:11-90) as a device
// kernel, plus the builder-defined BASELINE config-1/2 scene, trajectory and
// sensor-noise generators (host).  The renderer uses the oracle's operation
// order with -fmad=false, so a frame rendered here is bit-identical to
// oracle/orc_synth.hpp render_depth on the same scene and pose.
#include <cmath>
#include <cstdio>
#include <random>
#include <thread>
#include <vector>

#include "../../include/csf_b200.h"
#include "csf_internal.h"
#include "lifted.cuh"

namespace csfd {

struct SynthScene {
  int n_spheres, n_boxes, n_planes, n_waves;
  double sph[64][4];   // cx cy cz r
  double box[256][6];  // cx cy cz hx hy hz
  double pln[16][4];   // nx ny nz offset
  double wave[8][4];   // terrain plane waves: a kx ky phase (config 4)
  double inv_lip;      // 1 / sqrt(1 + L^2)
};

// config-4 terrain height (oracle Scene::height): sum of plane waves
CSF_HD double terrain_height(const SynthScene& s, double x, double y) {
  double hgt = 0.0;
  for (int i = 0; i < s.n_waves; ++i)
    hgt = hgt + s.wave[i][0] * csf_det::sin((s.wave[i][1] * x + s.wave[i][2] * y) + s.wave[i][3]);
  return hgt;
}

__constant__ SynthScene c_scene;

CSF_DEV double vnorm(double a, double b, double c) { return sqrt(a * a + (b * b + c * c)); }
CSF_DEV double dmin(double d, double x) { return x < d ? x : d; }  // std::min(d, x)
CSF_DEV double dmax(double a, double b) { return a < b ? b : a; }  // std::max(a, b)

CSF_DEV double scene_sdf(double px, double py, double pz) {
  double d = 1.7976931348623157e308;
  for (int i = 0; i < c_scene.n_spheres; ++i) {
    const double* s = c_scene.sph[i];
    d = dmin(d, vnorm(px - s[0], py - s[1], pz - s[2]) - s[3]);
  }
  for (int i = 0; i < c_scene.n_boxes; ++i) {
    const double* b = c_scene.box[i];
    const double q0 = fabs(px - b[0]) - b[3], q1 = fabs(py - b[1]) - b[4], q2 = fabs(pz - b[2]) - b[5];
    const double inside = dmin(dmax(q0, dmax(q1, q2)), 0.0);
    d = dmin(d, vnorm(dmax(q0, 0.0), dmax(q1, 0.0), dmax(q2, 0.0)) + inside);
  }
  for (int i = 0; i < c_scene.n_planes; ++i) {
    const double* p = c_scene.pln[i];
    d = dmin(d, (p[0] * px + (p[1] * py + p[2] * pz)) - p[3]);
  }
  if (c_scene.n_waves > 0) d = dmin(d, (pz - terrain_height(c_scene, px, py)) * c_scene.inv_lip);
  return d;
}

__global__ void k_render(const double* __restrict__ poses, int n_frames, double fx, double fy, double cx, double cy,
                         int w, int h, double far_clip, double hit_eps, double* __restrict__ out) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y * blockDim.y + threadIdx.y;
  const int f = blockIdx.z;
  if (x >= w || y >= h || f >= n_frames) return;
  const double* P = poses + 12 * f;
  double dc0 = (static_cast<double>(x) - cx) / fx, dc1 = (static_cast<double>(y) - cy) / fy, dc2 = 1.0;
  const double zfac = 1.0 / vnorm(dc0, dc1, dc2);
  dc0 = dc0 * zfac;
  dc1 = dc1 * zfac;
  dc2 = dc2 * zfac;
  double dir[3];
  for (int r = 0; r < 3; ++r) dir[r] = P[3 * r] * dc0 + (P[3 * r + 1] * dc1 + P[3 * r + 2] * dc2);
  const double ox = P[9], oy = P[10], oz = P[11];
  double s = 0.0, depth = 0.0;
  for (int it = 0; it < 512 && s < far_clip; ++it) {
    const double phi = scene_sdf(ox + s * dir[0], oy + s * dir[1], oz + s * dir[2]);
    if (phi < hit_eps) {
      for (int r = 0; r < 3; ++r) {
        const double px = ox + s * dir[0], py = oy + s * dir[1], pz = oz + s * dir[2];
        const double res = scene_sdf(px, py, pz);
        double n[3];
        const double eps = 1e-5;
        n[0] = scene_sdf(px + eps, py, pz) - scene_sdf(px - eps, py, pz);
        n[1] = scene_sdf(px, py + eps, pz) - scene_sdf(px, py - eps, pz);
        n[2] = scene_sdf(px, py, pz + eps) - scene_sdf(px, py, pz - eps);
        const double z2 = n[0] * n[0] + (n[1] * n[1] + n[2] * n[2]);
        if (z2 > 0.0) {
          const double l = sqrt(z2);
          n[0] = n[0] / l;
          n[1] = n[1] / l;
          n[2] = n[2] / l;
        }
        const double slope = dir[0] * n[0] + (dir[1] * n[1] + dir[2] * n[2]);
        s -= res / (-0.05 < slope ? -0.05 : slope);
      }
      depth = s * zfac;
      break;
    }
    s += phi;
  }
  out[(static_cast<long long>(f) * h + y) * w + x] = depth;
}

}  // namespace csfd

namespace csfi {

struct Uniform53 {
  std::mt19937_64 g;
  explicit Uniform53(uint64_t seed) : g(seed) {}
  double next01() { return static_cast<double>(g() >> 11) * (1.0 / 9007199254740992.0); }
  double next(double lo, double hi) { return lo + (hi - lo) * next01(); }
};

// Box-Muller over the top 53 bits of mt19937_64 (synth.cpp:116-133).
struct Gaussian {
  std::mt19937_64 st;
  bool have = false;
  double spare = 0.0;
  explicit Gaussian(uint64_t seed) : st(seed) {}
  double next() {
    if (have) {
      have = false;
      return spare;
    }
    const double k = 1.0 / 9007199254740992.0;
    double u1;
    do {
      u1 = static_cast<double>(st() >> 11) * k;
    } while (u1 <= 0.0);
    const double u2 = static_cast<double>(st() >> 11) * k;
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 2.0 * M_PI * u2;
    spare = r * std::sin(a);
    have = true;
    return r * std::cos(a);
  }
};

static void add_room(csfd::SynthScene& s) {
  const double pl[6][4] = {{0, 0, 1, 0.0}, {0, 0, -1, -3.0}, {1, 0, 0, -2.0},
                           {-1, 0, 0, -2.0}, {0, 1, 0, -2.0}, {0, -1, 0, -2.0}};
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 4; ++j) s.pln[s.n_planes + i][j] = pl[i][j];
  s.n_planes += 6;
}

// The oracle's config1_scene / config2_scene / config4_scene (oracle/orc_pipeline.hpp).
static csfd::SynthScene config_scene(int config) {
  csfd::SynthScene s{};
  s.inv_lip = 1.0;
  if (config == 4) {
    Uniform53 u(3);
    double lip = 0.0;
    for (int i = 0; i < 6; ++i) {
      const double amp = u.next(0.1, 0.4);
      const double lambda = u.next(2.5, 20.0);
      const double ang = u.next(0.0, 2.0 * M_PI);
      const double phase = u.next(0.0, 2.0 * M_PI);
      const double k = (2.0 * M_PI) / lambda;
      double* w = s.wave[s.n_waves++];
      w[0] = amp;
      w[1] = k * csf_det::cos(ang);
      w[2] = k * csf_det::sin(ang);
      w[3] = phase;
      lip = lip + amp * k;
    }
    s.inv_lip = 1.0 / std::sqrt(1.0 + lip * lip);
    int placed = 0;
    while (placed < 200) {
      const double x = u.next(-30.0, 30.0);
      const double y = u.next(-30.0, 30.0);
      const double hx = u.next(0.3, 1.5), hy = u.next(0.3, 1.5), hz = u.next(0.3, 2.0);
      const double r = std::sqrt(x * x + y * y);
      if (std::fabs(r - 10.0) < 1.2 + std::sqrt(hx * hx + hy * hy)) continue;  // keep the flight path clear
      double* d = s.box[s.n_boxes++];
      d[0] = x; d[1] = y; d[2] = csfd::terrain_height(s, x, y) + hz - 0.3; d[3] = hx; d[4] = hy; d[5] = hz;
      ++placed;
    }
    return s;
  }
  add_room(s);
  if (config == 1) {
    Uniform53 u(0);
    for (int i = 0; i < 3; ++i) {
      const double r = u.next(0.3, 0.6);
      const double cx = u.next(-1.6, -0.6), cy = u.next(-1.0, 1.0), cz = u.next(0.3, 1.2);
      double* d = s.sph[s.n_spheres++];
      d[0] = cx; d[1] = cy; d[2] = cz; d[3] = r;
    }
  } else {
    Uniform53 u(1);
    int placed = 0;
    while (placed < 20) {
      const bool sphere = (placed % 2) == 0;
      const double r = sphere ? u.next(0.1, 0.35) : u.next(0.08, 0.3);
      const double c0 = u.next(-1.8, 1.8), c1 = u.next(-1.8, 1.8), c2 = u.next(0.2, 2.5);
      const double radial = std::sqrt(c0 * c0 + c1 * c1);
      const double bound = sphere ? r : r * 1.7320508075688772;
      if (std::fabs(radial - 1.2) < bound + 0.35 && std::fabs(c2 - 1.3) < bound + 0.45) continue;
      if (sphere) {
        double* d = s.sph[s.n_spheres++];
        d[0] = c0; d[1] = c1; d[2] = c2; d[3] = r;
      } else {
        const double hy = u.next(0.08, 0.3), hz = u.next(0.08, 0.3);
        double* d = s.box[s.n_boxes++];
        d[0] = c0; d[1] = c1; d[2] = c2; d[3] = r; d[4] = hy; d[5] = hz;
      }
      ++placed;
    }
  }
  return s;
}

static void normalize3(double* v) {
  const double z = v[0] * v[0] + (v[1] * v[1] + v[2] * v[2]);
  if (z > 0.0) {
    const double l = std::sqrt(z);
    v[0] /= l; v[1] /= l; v[2] /= l;
  }
}

// synth.cpp:92-105 with the deterministic cos/sin
static void orbit_pose(const double* target, double radius, double height, double angle, double* P) {
  const double eye[3] = {target[0] + radius * csf_det::cos(angle), target[1] + radius * csf_det::sin(angle),
                         target[2] + height};
  double zc[3] = {target[0] - eye[0], target[1] - eye[1], target[2] - eye[2]};
  normalize3(zc);
  double xc[3] = {zc[1] * 1.0 - zc[2] * 0.0, zc[2] * 0.0 - zc[0] * 1.0, zc[0] * 0.0 - zc[1] * 0.0};
  normalize3(xc);
  const double yc[3] = {zc[1] * xc[2] - zc[2] * xc[1], zc[2] * xc[0] - zc[0] * xc[2], zc[0] * xc[1] - zc[1] * xc[0]};
  for (int r = 0; r < 3; ++r) {
    P[3 * r] = xc[r];
    P[3 * r + 1] = yc[r];
    P[3 * r + 2] = zc[r];
  }
  P[9] = eye[0]; P[10] = eye[1]; P[11] = eye[2];
}

// oracle look_at_pose: the orbit_pose construction toward an explicit target
static void look_at_pose(const double* eye, const double* target, double* P) {
  double zc[3] = {target[0] - eye[0], target[1] - eye[1], target[2] - eye[2]};
  normalize3(zc);
  double xc[3] = {zc[1] * 1.0 - zc[2] * 0.0, zc[2] * 0.0 - zc[0] * 1.0, zc[0] * 0.0 - zc[1] * 0.0};
  normalize3(xc);
  const double yc[3] = {zc[1] * xc[2] - zc[2] * xc[1], zc[2] * xc[0] - zc[0] * xc[2], zc[0] * xc[1] - zc[1] * xc[0]};
  for (int r = 0; r < 3; ++r) {
    P[3 * r] = xc[r];
    P[3 * r + 1] = yc[r];
    P[3 * r + 2] = zc[r];
  }
  P[9] = eye[0]; P[10] = eye[1]; P[11] = eye[2];
}

int synth_workload(cudaStream_t stream, int config, int n_frames, int width, int height, float* depth_out,
                   double* gt_out, csf_intrinsics* k_out, std::string* err) {
  if (config != 1 && config != 2 && config != 4) {
    *err = "csf_synth_workload: config must be 1, 2 or 4";
    return CSF_EINVAL;
  }
  csf_intrinsics k;
  if (config == 1) {
    k.fx = 120.0; k.fy = 120.0; k.cx = 80.0; k.cy = 60.0; k.width = 160; k.height = 120;
  } else {
    k.fx = 525.0; k.fy = 525.0; k.cx = 319.5; k.cy = 239.5; k.width = 640; k.height = 480;
  }
  k.depth_scale = 5000.0;
  if (width > 0) {
    const double s = static_cast<double>(width) / k.width;
    k.fx *= s; k.fy *= s; k.cx *= s; k.cy *= s;
    k.width = width;
    k.height = height;
  }
  if (k_out) *k_out = k;
  const csfd::SynthScene scene = config_scene(config);
  const double target[3] = {0.0, 0.0, 1.0};
  for (int f = 0; f < n_frames; ++f) {
    if (config == 1) {
      orbit_pose(target, 1.0, 0.4, static_cast<double>(f) * (3.0 * M_PI / 180.0), gt_out + 12 * f);
    } else if (config == 4) {
      const double th = static_cast<double>(f) * (0.36 * M_PI / 180.0);
      const double ex = 10.0 * csf_det::cos(th), ey = 10.0 * csf_det::sin(th);
      const double tt = th + 0.6;
      const double tx = 10.0 * csf_det::cos(tt), ty = 10.0 * csf_det::sin(tt);
      const double eye[3] = {ex, ey, csfd::terrain_height(scene, ex, ey) + 2.0};
      const double tgt[3] = {tx, ty, csfd::terrain_height(scene, tx, ty) + 0.5};
      look_at_pose(eye, tgt, gt_out + 12 * f);
    } else {
      orbit_pose(target, 1.2, 0.3, static_cast<double>(f) * (1.5 * M_PI / 180.0), gt_out + 12 * f);
    }
  }
  const size_t P = static_cast<size_t>(k.width) * k.height;
  double* d_poses = nullptr;
  double* d_depth = nullptr;
  if (cudaMalloc(&d_poses, sizeof(double) * 12 * n_frames) != cudaSuccess ||
      cudaMalloc(&d_depth, sizeof(double) * P * n_frames) != cudaSuccess) {
    *err = "csf_synth_workload: device allocation failed";
    cudaFree(d_poses);
    return CSF_ENOMEM;
  }
  cudaMemcpyToSymbolAsync(csfd::c_scene, &scene, sizeof(scene), 0, cudaMemcpyHostToDevice, stream);
  cudaMemcpyAsync(d_poses, gt_out, sizeof(double) * 12 * n_frames, cudaMemcpyHostToDevice, stream);
  const dim3 block(16, 16), grid((k.width + 15) / 16, (k.height + 15) / 16, n_frames);
  csfd::k_render<<<grid, block, 0, stream>>>(d_poses, n_frames, k.fx, k.fy, k.cx, k.cy, k.width, k.height, 20.0, 1e-6,
                                             d_depth);
  std::vector<double> host(P * n_frames);
  cudaMemcpyAsync(host.data(), d_depth, sizeof(double) * P * n_frames, cudaMemcpyDeviceToHost, stream);
  const cudaError_t e = cudaStreamSynchronize(stream);
  cudaFree(d_poses);
  cudaFree(d_depth);
  if (e != cudaSuccess) {
    *err = std::string("csf_synth_workload: ") + cudaGetErrorString(e);
    return CSF_ECUDA;
  }
  // sensor model per frame (independent seeds -> frames in parallel)
  auto noise = [&](int f) {
    double* d = host.data() + P * f;
    if (config == 1) {
      Gaussian g(1000 + f);
      for (size_t i = 0; i < P; ++i) {
        if (!(d[i] > 0.0)) continue;
        const double n = d[i] + 0.001 * g.next();
        d[i] = n > 0.0 ? n : 0.0;
      }
    } else if (config == 4) {
      Gaussian g(4000 + f);
      for (size_t i = 0; i < P; ++i) {
        if (!(d[i] > 0.0)) continue;
        const double sigma = 0.0012 * d[i] * d[i];
        const double n = d[i] + sigma * g.next();
        d[i] = n > 0.0 ? n : 0.0;
      }
      for (size_t i = 0; i < P; ++i)
        if (d[i] < 0.3) d[i] = 0.0;  // depth range 0.3-20 m
    } else {
      const uint64_t seed = 2000 + f;
      Gaussian g(seed);
      Uniform53 drop(seed ^ 0x9e3779b97f4a7c15ULL);
      for (size_t i = 0; i < P; ++i) {
        if (!(d[i] > 0.0)) continue;
        const double sigma = 0.0012 * d[i] * d[i];
        const double n = d[i] + sigma * g.next();
        d[i] = n > 0.0 ? n : 0.0;
        if (drop.next01() < 0.05) d[i] = 0.0;
      }
    }
    float* o = depth_out + P * f;
    for (size_t i = 0; i < P; ++i) o[i] = static_cast<float>(d[i]);
  };
  const int nthreads = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  std::vector<std::thread> pool;
  for (int t = 0; t < nthreads; ++t)
    pool.emplace_back([&, t] {
      for (int f = t; f < n_frames; f += nthreads) noise(f);
    });
  for (auto& th : pool) th.join();
  return CSF_OK;
}

}  // namespace csfi
