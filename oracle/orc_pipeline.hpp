// ORACLE — TEST INFRASTRUCTURE ONLY (see orc_core.hpp header).
//
// BUILDER-DEFINED (no reference): the lifted tracker
// and the CSFD frame-derivative driver.  The reference's track_frame
// (icp.cpp:169-244) is double-only; this lifts its kLinearized solver to the
// packed scalar S = Lifted<D>:
//   - preprocessing (bilateral, pyramid) and every gate read real parts only;
//   - measured vertices/normals, the raycast prediction, J, r, the 6x6 normal
//     equations and their LDLT solve carry all D channels;
//   - the normal equations use the canonical slot-tiled reduction order.
// The driver seeds D directions (first-frame twist components and/or the
// four intrinsics), fuses frame 0 at exp(xi0*) * T0_gt, then tracks and fuses
// frames 1..N-1, and differentiates an objective of the lifted trajectory.
#pragma once

#include "orc_icp.hpp"
#include "orc_synth.hpp"

namespace orc {

template <typename S>
struct LiftedTrackResult {
  PoseT<S> pose;
  int iterations = 0;
  bool converged = false;
  int correspondences = 0;
};

template <typename S>
SurfaceMaps<double> real_maps(const SurfaceMaps<S>& m) {
  SurfaceMaps<double> o;
  o.vertices = Image<Vec3d>(m.vertices.width, m.vertices.height, Vec3d());
  o.normals = Image<Vec3d>(m.normals.width, m.normals.height, Vec3d());
  for (std::size_t i = 0; i < m.vertices.data.size(); ++i)
    for (int c = 0; c < 3; ++c) {
      o.vertices.data[i][c] = real_part(m.vertices.data[i][c]);
      o.normals.data[i][c] = real_part(m.normals.data[i][c]);
    }
  return o;
}

template <typename S, typename V, typename K>
LiftedTrackResult<S> track_frame_lifted(const V& volume, const Image<double>& depth, const PoseT<S>& init,
                                        const IntrinsicsT<K>& k, const IcpConfig& cfg, const RaycastConfig& rc = {}) {
  LiftedTrackResult<S> out;
  const int levels = std::clamp(cfg.levels, 1, 3);
  const auto pyramid = build_depth_pyramid(bilateral_filter(depth), levels);
  PoseT<S> pose = init;
  int iteration = 0;
  for (int li = 0; li < levels; ++li) {
    const int level = levels - 1 - li;
    const IntrinsicsT<K> kl = k.at_level(level);
    const Intrinsics klr = real_intrinsics(kl);
    const SurfaceMaps<S> measured = measure_surface<S>(pyramid[level], kl);
    const SurfaceMaps<double> measured_re = real_maps(measured);
    const PoseT<S> prediction_pose = pose;
    const SurfaceMaps<S> predicted = raycast<S>(volume, prediction_pose, kl, rc);
    const SurfaceMaps<double> predicted_re = real_maps(predicted);
    const int stride = std::max(1, cfg.level_pixel_stride[li]);
    for (int it = 0; it < cfg.level_iterations[li]; ++it) {
      std::vector<CorrIndex> idx;
      associate(measured_re, predicted_re, real_pose(pose), real_pose(prediction_pose), klr, cfg, stride, &idx);
      out.correspondences = static_cast<int>(idx.size());
      if (idx.size() < 12) break;
      const NormalEq<S> ne = tiled_normal_equations(idx, klr.width, klr.height, stride, measured, predicted, pose);
      S nb[6];
      for (int i = 0; i < 6; ++i) nb[i] = -ne.b[i];
      const Ldlt6<S> ldlt(ne.a);
      S d[6];
      ldlt.solve(nb, d);
      bool finite = true;
      for (int i = 0; i < 6; ++i) finite = finite && isfinite_s(d[i]);
      Vec6<S> delta;
      for (int i = 0; i < 6; ++i) delta[i] = finite ? d[i] : S(0.0);
      pose = apply_increment(delta, pose);
      ++iteration;
      Vec6<double> dre;
      for (int i = 0; i < 6; ++i) dre[i] = real_part(delta[i]);
      if (norm6(dre) < cfg.step_tolerance) {
        if (level == 0) out.converged = true;
        break;
      }
    }
  }
  out.pose = pose;
  out.iterations = iteration;
  return out;
}

// ---------------------------------------------------------------------------
// Driver
// ---------------------------------------------------------------------------
enum class Objective { kFinalTranslationError = 0, kTrajectoryError = 1 };

struct PipelineConfig {
  bool hashed = false;
  VolumeParams dense;
  HashParams hash;
  Intrinsics k;
  IcpConfig icp;
  RaycastConfig rc;
  double h = 1e-8;
  std::vector<int> directions;  // parameter per channel: 0..5 twist (rho, phi), 6..9 fx, fy, cx, cy,
                                // 10 + 6 (kf - 1) + c: keyframe kf's twist component c
  Objective objective = Objective::kFinalTranslationError;
  int keyframe_interval = 0;    // BUILDER-DEFINED (config 4): keyframes at frames kf * K
};

struct PipelineResult {
  std::vector<double> gradient;        // [D]
  double objective = 0.0;
  std::vector<double> poses;           // [N][12][1+D]  (R row-major, t)
  std::vector<int> iterations;         // [N]
  std::vector<int> correspondences;    // [N]
  std::vector<int> blocks;             // [N] allocated blocks after frame (hashed)
  std::vector<int> visible;            // [N] visible blocks of frame (hashed)
  std::vector<int> converged;          // [N] track_frame converged at level 0
  std::vector<int> fresh;              // [N] blocks newly allocated by the frame (hashed)
  std::vector<int> fused;              // [N] voxels fused by the frame
};

template <int D>
void store_pose(const PoseT<Lifted<D>>& p, double* out) {
  for (int e = 0; e < 12; ++e) {
    const Lifted<D>& s = e < 9 ? p.rotation(e / 3, e % 3) : p.translation[e - 9];
    out[e * (1 + D)] = s.re;
    for (int d = 0; d < D; ++d) out[e * (1 + D) + 1 + d] = s.im[d];
  }
}

// One lifted run of the frame loop for any CSFD scalar S (Lifted<D> packs D
// first-order directions; Bicomplex carries one second-order pair): seed
// pose exp(xi) * T0_gt with lifted intrinsics ks, fuse frame 0, then track and
// fuse frames 1..N-1; the objective is evaluated in S.
template <typename S>
struct LiftedRun {
  std::vector<PoseT<S>> poses;
  S objective = S(0.0);
  std::vector<int> iterations, correspondences, blocks, visible, converged, fresh, fused;
};

// Keyframe perturbation seeds of keyframe kf (first order only): exp(xi) *
// pose with xi[c].im[d] = h for the channels coded 10 + 6 (kf - 1) + c.
template <typename S>
Vec6<S> keyframe_xi(const PipelineConfig& cfg, int kf) {
  Vec6<S> xi;
  for (int i = 0; i < 6; ++i) xi[i] = S(0.0);
  if constexpr (!std::is_same_v<S, Bicomplex> && !std::is_same_v<S, double>) {
    for (std::size_t d = 0; d < cfg.directions.size(); ++d) {
      const int c = cfg.directions[d] - (10 + 6 * (kf - 1));
      if (c >= 0 && c < 6) xi[c].im[d] = cfg.h;
    }
  }
  return xi;
}

template <typename S, typename V>
LiftedRun<S> run_lifted(V& vol, const PipelineConfig& cfg, const std::vector<Image<double>>& frames,
                        const std::vector<Pose>& gt, const Vec6<S>& xi, const IntrinsicsT<S>& ks) {
  const int n = static_cast<int>(frames.size());
  LiftedRun<S> res;
  res.poses.resize(n);
  res.iterations.assign(n, 0);
  res.correspondences.assign(n, 0);
  res.blocks.assign(n, 0);
  res.visible.assign(n, 0);
  res.converged.assign(n, 0);
  res.fresh.assign(n, 0);
  res.fused.assign(n, 0);
  const Intrinsics kr = cfg.k;
  auto integrate = [&](int f) {
    if constexpr (V::kHashed) {
      AllocStats st;
      const std::vector<int> visible = allocate_band(vol, frames[f], kr, real_pose(res.poses[f]), &st);
      res.fused[f] = static_cast<int>(surface_update_blocks(vol, visible, frames[f], res.poses[f], ks));
      res.blocks[f] = vol.n_blocks();
      res.visible[f] = st.touched;
      res.fresh[f] = st.fresh;
    } else {
      res.fused[f] = static_cast<int>(surface_update(vol, frames[f], res.poses[f], ks));
    }
  };
  res.poses[0] = exp_map(xi) * pose_cast<S>(gt[0]);
  integrate(0);
  for (int f = 1; f < n; ++f) {
    const LiftedTrackResult<S> tr = track_frame_lifted<S>(vol, frames[f], res.poses[f - 1], ks, cfg.icp, cfg.rc);
    res.poses[f] = tr.pose;
    res.iterations[f] = tr.iterations;
    res.correspondences[f] = tr.correspondences;
    res.converged[f] = tr.converged ? 1 : 0;
    if constexpr (!std::is_same_v<S, Bicomplex>) {
      if (cfg.keyframe_interval > 0 && f % cfg.keyframe_interval == 0)
        res.poses[f] = exp_map(keyframe_xi<S>(cfg, f / cfg.keyframe_interval)) * res.poses[f];
    }
    integrate(f);
  }
  S obj(0.0);
  if (cfg.objective == Objective::kFinalTranslationError) {
    const Vec3<S> diff = res.poses[n - 1].translation -
                         Vec3<S>(S(gt[n - 1].translation[0]), S(gt[n - 1].translation[1]), S(gt[n - 1].translation[2]));
    obj = sqrt(dot(diff, diff));
  } else {
    for (int f = 0; f < n; ++f) {
      const Vec3<S> diff = res.poses[f].translation -
                           Vec3<S>(S(gt[f].translation[0]), S(gt[f].translation[1]), S(gt[f].translation[2]));
      obj = obj + dot(diff, diff);
    }
  }
  res.objective = obj;
  return res;
}

// Seed parameter `prm` of a lifted scalar set: 0..5 twist (rho, phi), 6..9
// fx, fy, cx, cy.  `set` writes the perturbation into the scalar.
template <typename S, typename Fn>
void seed_parameter(int prm, Vec6<S>& xi, IntrinsicsT<S>& ks, Fn&& set) {
  if (prm >= 0 && prm < 6) set(xi[prm]);
  else if (prm == 6) set(ks.fx);
  else if (prm == 7) set(ks.fy);
  else if (prm == 8) set(ks.cx);
  else if (prm == 9) set(ks.cy);
  else throw std::invalid_argument("unknown direction parameter");
}

template <typename S>
IntrinsicsT<S> lift_intrinsics(const Intrinsics& k) {
  IntrinsicsT<S> ks;
  ks.fx = S(k.fx); ks.fy = S(k.fy); ks.cx = S(k.cx); ks.cy = S(k.cy);
  ks.width = k.width; ks.height = k.height; ks.depth_scale = k.depth_scale;
  return ks;
}

template <int D, typename V>
PipelineResult run_pipeline_on(V& vol, const PipelineConfig& cfg, const std::vector<Image<double>>& frames,
                               const std::vector<Pose>& gt) {
  using S = Lifted<D>;
  if (static_cast<int>(cfg.directions.size()) != D) throw std::invalid_argument("direction count != D");
  const int n = static_cast<int>(frames.size());
  Vec6<S> xi;
  for (int i = 0; i < 6; ++i) xi[i] = S(0.0);
  IntrinsicsT<S> ks = lift_intrinsics<S>(cfg.k);
  for (int d = 0; d < D; ++d)
    if (cfg.directions[d] < 10) seed_parameter(cfg.directions[d], xi, ks, [&](S& s) { s.im[d] = cfg.h; });
  const LiftedRun<S> run = run_lifted<S>(vol, cfg, frames, gt, xi, ks);
  PipelineResult res;
  res.poses.assign(static_cast<std::size_t>(n) * 12 * (1 + D), 0.0);
  res.iterations = run.iterations;
  res.correspondences = run.correspondences;
  res.blocks = run.blocks;
  res.visible = run.visible;
  res.converged = run.converged;
  res.fresh = run.fresh;
  res.fused = run.fused;
  res.objective = run.objective.re;
  res.gradient.resize(D);
  for (int d = 0; d < D; ++d) res.gradient[d] = run.objective.im[d] / cfg.h;
  for (int f = 0; f < n; ++f) store_pose(run.poses[f], &res.poses[static_cast<std::size_t>(f) * 12 * (1 + D)]);
  return res;
}

// ---------------------------------------------------------------------------
// Second order (BASELINE config 3): one Bicomplex pass per parameter pair
// (i, j) — the reference's csfd_hessian pattern (diff.hpp:58-72), applied to
// the whole frame loop.  im1 is seeded on parameter i, im2 on parameter j;
// H_ij = im12 / h^2 (csfd.hpp:319), g_i = im1 / h, g_j = im2 / h.  The volume
// stores Bicomplex fields (builder-defined; see Measure<Bicomplex>).
// ---------------------------------------------------------------------------
struct HessianResult {
  std::vector<double> hessian;   // [P]  H_{i_p j_p}
  std::vector<double> grad1;     // [P]  d obj / d param i_p
  std::vector<double> grad2;     // [P]  d obj / d param j_p
  double objective = 0.0;
  std::vector<double> poses;     // [N][12][1 + 3P]: re, then (im1, im2, im12) per pair
  std::vector<int> iterations, correspondences, blocks, visible, converged, fresh, fused;
};

template <typename V>
LiftedRun<Bicomplex> run_pair(V& vol, const PipelineConfig& cfg, const std::vector<Image<double>>& frames,
                              const std::vector<Pose>& gt, int pi, int pj) {
  using S = Bicomplex;
  Vec6<S> xi;
  for (int i = 0; i < 6; ++i) xi[i] = S(0.0);
  IntrinsicsT<S> ks = lift_intrinsics<S>(cfg.k);
  seed_parameter(pi, xi, ks, [&](S& s) { s.im1 = cfg.h; });
  seed_parameter(pj, xi, ks, [&](S& s) { s.im2 = cfg.h; });
  return run_lifted<S>(vol, cfg, frames, gt, xi, ks);
}

inline HessianResult run_pipeline_hessian(const PipelineConfig& cfg, const std::vector<std::pair<int, int>>& pairs,
                                          const std::vector<Image<double>>& frames, const std::vector<Pose>& gt) {
  const int n = static_cast<int>(frames.size());
  const int P = static_cast<int>(pairs.size());
  const int C = 1 + 3 * P;
  HessianResult res;
  res.hessian.resize(P);
  res.grad1.resize(P);
  res.grad2.resize(P);
  res.poses.assign(static_cast<std::size_t>(n) * 12 * C, 0.0);
  for (int p = 0; p < P; ++p) {
    LiftedRun<Bicomplex> run;
    if (cfg.hashed) {
      HashedVolumeT<Bicomplex> vol(cfg.hash);
      run = run_pair(vol, cfg, frames, gt, pairs[p].first, pairs[p].second);
    } else {
      TsdfVolumeT<Bicomplex> vol(cfg.dense);
      run = run_pair(vol, cfg, frames, gt, pairs[p].first, pairs[p].second);
    }
    const Bicomplex& o = run.objective;
    res.hessian[p] = o.im12 / (cfg.h * cfg.h);
    res.grad1[p] = o.im1 / cfg.h;
    res.grad2[p] = o.im2 / cfg.h;
    if (p == 0) {
      res.objective = o.re;
      res.iterations = run.iterations;
      res.correspondences = run.correspondences;
      res.blocks = run.blocks;
      res.visible = run.visible;
      res.converged = run.converged;
      res.fresh = run.fresh;
      res.fused = run.fused;
    }
    for (int f = 0; f < n; ++f)
      for (int e = 0; e < 12; ++e) {
        const Bicomplex& s = e < 9 ? run.poses[f].rotation(e / 3, e % 3) : run.poses[f].translation[e - 9];
        double* dst = &res.poses[(static_cast<std::size_t>(f) * 12 + e) * C];
        dst[0] = s.re;
        dst[1 + 3 * p] = s.im1;
        dst[2 + 3 * p] = s.im2;
        dst[3 + 3 * p] = s.im12;
      }
  }
  return res;
}

template <int D>
PipelineResult run_pipeline(const PipelineConfig& cfg, const std::vector<Image<double>>& frames,
                            const std::vector<Pose>& gt) {
  if (cfg.hashed) {
    HashedVolumeT<Lifted<D>> vol(cfg.hash);
    return run_pipeline_on<D>(vol, cfg, frames, gt);
  }
  TsdfVolumeT<Lifted<D>> vol(cfg.dense);
  return run_pipeline_on<D>(vol, cfg, frames, gt);
}

inline PipelineResult run_pipeline_dyn(const PipelineConfig& cfg, const std::vector<Image<double>>& frames,
                                       const std::vector<Pose>& gt) {
  switch (cfg.directions.size()) {
    case 1: return run_pipeline<1>(cfg, frames, gt);
    case 2: return run_pipeline<2>(cfg, frames, gt);
    case 3: return run_pipeline<3>(cfg, frames, gt);
    case 4: return run_pipeline<4>(cfg, frames, gt);
    case 5: return run_pipeline<5>(cfg, frames, gt);
    case 6: return run_pipeline<6>(cfg, frames, gt);
    case 7: return run_pipeline<7>(cfg, frames, gt);
    case 8: return run_pipeline<8>(cfg, frames, gt);
    case 10: return run_pipeline<10>(cfg, frames, gt);
    case 12: return run_pipeline<12>(cfg, frames, gt);
    case 20: return run_pipeline<20>(cfg, frames, gt);
    default: throw std::invalid_argument("oracle pipeline: unsupported direction count");
  }
}

// ---------------------------------------------------------------------------
// BASELINE configs 1 and 2 inputs (builder-defined geometry)
// ---------------------------------------------------------------------------
struct Workload {
  Scene scene;
  Intrinsics k;
  std::vector<Pose> gt;
  std::vector<Image<double>> frames;
};

// Config 1: 4x4x3 m room + 3 spheres (seed 0), 10 frames 160x120,
// fx=fy=120 cx=80 cy=60, orbit radius 1 m, 3 deg step, sigma = 1 mm.
inline Scene config1_scene(uint64_t seed = 0) {
  Scene s;
  add_room(s, -2.0, 2.0, -2.0, 2.0, 0.0, 3.0);
  Uniform53 u(seed);
  for (int i = 0; i < 3; ++i) {
    SdfSphere sp;
    sp.radius = u.next(0.3, 0.6);
    // draws in statement order (constructor-argument order is unspecified)
    const double cx = u.next(-1.6, -0.6);
    const double cy = u.next(-1.0, 1.0);
    const double cz = u.next(0.3, 1.2);
    sp.center = Vec3d(cx, cy, cz);
    s.spheres.push_back(sp);
  }
  return s;
}
inline Intrinsics config1_intrinsics() {
  Intrinsics k;
  k.fx = 120.0; k.fy = 120.0; k.cx = 80.0; k.cy = 60.0; k.width = 160; k.height = 120;
  return k;
}
inline Pose config1_pose(int f) {
  return orbit_pose(Vec3d(0.0, 0.0, 1.0), 1.0, 0.4, static_cast<double>(f) * (3.0 * M_PI / 180.0));
}
inline VolumeParams config1_volume() {
  VolumeParams vp = VolumeParams::cube(128, 0.02, Vec3d(-2.1, -1.28, -0.1));
  vp.mu = 0.06;
  return vp;
}

// Config 2: room + 20 random spheres/boxes (seed 1), VGA, K = 525/525/319.5/239.5,
// sigma = 0.0012 z^2, 5% dropout; hashed 5 mm voxels, mu = 5 voxels.
inline Scene config2_scene(uint64_t seed = 1) {
  Scene s;
  add_room(s, -2.0, 2.0, -2.0, 2.0, 0.0, 3.0);
  Uniform53 u(seed);
  int placed = 0;
  while (placed < 20) {
    const bool sphere = (placed % 2) == 0;
    const double r = sphere ? u.next(0.1, 0.35) : u.next(0.08, 0.3);
    const double c0 = u.next(-1.8, 1.8);
    const double c1 = u.next(-1.8, 1.8);
    const double c2 = u.next(0.2, 2.5);
    const Vec3d c(c0, c1, c2);
    const double radial = std::sqrt(c[0] * c[0] + c[1] * c[1]);
    const double bound = sphere ? r : r * 1.7320508075688772;
    if (std::fabs(radial - 1.2) < bound + 0.35 && std::fabs(c[2] - 1.3) < bound + 0.45) continue;  // keep the orbit free
    if (sphere) {
      s.spheres.push_back({c, r});
    } else {
      const double hy = u.next(0.08, 0.3), hz = u.next(0.08, 0.3);
      s.boxes.push_back({c, Vec3d(r, hy, hz)});
    }
    ++placed;
  }
  return s;
}
inline Pose config2_pose(int f) {
  return orbit_pose(Vec3d(0.0, 0.0, 1.0), 1.2, 0.3, static_cast<double>(f) * (1.5 * M_PI / 180.0));
}
inline HashParams config2_hash() {
  HashParams hp;
  hp.voxel_size = 0.005;
  hp.mu = 5.0 * hp.voxel_size;
  hp.bucket_bits = 20;
  hp.max_blocks = 1 << 19;
  return hp;
}

// Config 4: 60x60 m procedural terrain (6 plane waves) + 200 boxes (seed 3),
// VGA, depth range 0.3-20 m, sigma = 0.0012 z^2; the camera flies a half
// circle of radius 10 m, 2 m above the ground, looking ~6 m ahead
// (0.36 deg / 6.3 cm per frame over 500 frames); boxes keep clear of the
// flight path (|r - 10| > 1.2 m + their footprint radius).  Hashed 2 cm voxels.
inline Scene config4_scene(uint64_t seed = 3) {
  Scene s;
  Uniform53 u(seed);
  double lip = 0.0;
  for (int i = 0; i < 6; ++i) {
    TerrainWave w;
    const double amp = u.next(0.1, 0.4);
    const double lambda = u.next(2.5, 20.0);
    const double ang = u.next(0.0, 2.0 * M_PI);
    const double phase = u.next(0.0, 2.0 * M_PI);
    const double k = (2.0 * M_PI) / lambda;
    w.a = amp;
    w.kx = k * m_cos(ang);
    w.ky = k * m_sin(ang);
    w.phase = phase;
    s.terrain.push_back(w);
    lip = lip + amp * k;
  }
  s.terrain_inv_lip = 1.0 / std::sqrt(1.0 + lip * lip);
  int placed = 0;
  while (placed < 200) {
    const double x = u.next(-30.0, 30.0);
    const double y = u.next(-30.0, 30.0);
    const double hx = u.next(0.3, 1.5), hy = u.next(0.3, 1.5), hz = u.next(0.3, 2.0);
    const double r = std::sqrt(x * x + y * y);
    if (std::fabs(r - 10.0) < 1.2 + std::sqrt(hx * hx + hy * hy)) continue;  // keep the flight path clear
    s.boxes.push_back({Vec3d(x, y, s.height(x, y) + hz - 0.3), Vec3d(hx, hy, hz)});
    ++placed;
  }
  return s;
}
inline Pose config4_pose(const Scene& s, int f) {
  const double th = static_cast<double>(f) * (0.36 * M_PI / 180.0);
  const double ex = 10.0 * m_cos(th), ey = 10.0 * m_sin(th);
  const double tt = th + 0.6;
  const double tx = 10.0 * m_cos(tt), ty = 10.0 * m_sin(tt);
  return look_at_pose(Vec3d(ex, ey, s.height(ex, ey) + 2.0), Vec3d(tx, ty, s.height(tx, ty) + 0.5));
}
inline HashParams config4_hash() {
  HashParams hp;
  hp.voxel_size = 0.02;
  hp.mu = 5.0 * hp.voxel_size;
  hp.bucket_bits = 20;
  hp.max_blocks = 1 << 21;
  return hp;
}

inline Workload make_workload(int config, int n_frames, int width = 0, int height = 0) {
  Workload w;
  if (config == 1) {
    w.scene = config1_scene(0);
    w.k = config1_intrinsics();
  } else if (config == 4) {
    w.scene = config4_scene(3);
    w.k = Intrinsics();
  } else {
    w.scene = config2_scene(1);
    w.k = Intrinsics();
  }
  if (width > 0) {  // reduced-resolution variant of the same geometry (tests)
    const double s = static_cast<double>(width) / w.k.width;
    w.k.fx *= s; w.k.fy *= s; w.k.cx *= s; w.k.cy *= s;
    w.k.width = width;
    w.k.height = height;
  }
  for (int f = 0; f < n_frames; ++f) {
    const Pose p = config == 1 ? config1_pose(f) : config == 4 ? config4_pose(w.scene, f) : config2_pose(f);
    w.gt.push_back(p);
    Image<double> d = render_depth(w.scene, p, w.k);
    if (config == 1) {
      d = add_depth_noise(d, 0.001, 1000 + f);
    } else if (config == 4) {
      d = add_depth_noise_quadratic(d, 0.0012, 0.0, 4000 + f);
      for (auto& z : d.data)
        if (z < 0.3) z = 0.0;  // depth range 0.3-20 m (the renderer stops at 20 m)
    } else {
      d = add_depth_noise_quadratic(d, 0.0012, 0.05, 2000 + f);
    }
    w.frames.push_back(to_float32(d));
  }
  return w;
}

}  // namespace orc
