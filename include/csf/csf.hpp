// csf/csf.hpp — the reference's own signatures (proj/include/csf/*.hpp) in
// namespace csf, over the device implementation of csf/b200.hpp.
//
// Same names, argument order and defaults as frames.hpp, tsdf.hpp, icp.hpp and
// diff.hpp; no context argument: every call runs on the calling thread's
// default device context (device 0, or csf::set_device before the first
// call).  Poses are csf::Pose (se3.hpp:21-45 without Eigen: rotation(r, c)
// and translation[i]); the dense / hashed volume, images and maps are the
// b200 types.  Errors are the reference's exception types.
#pragma once

#include "b200.hpp"

namespace csf {

using b200::Correspondence;
using b200::Image;
using b200::Lifted;
using b200::SurfaceMaps;
using b200::TrackResult;
using b200::TrackTrace;
using b200::Volume;
using b200::Complex;
using b200::Bicomplex;
using b200::csfd_gradient;
using b200::csfd_hessian;
using Intrinsics = csf_intrinsics;
using IcpConfig = csf_icp_cfg;
using RaycastConfig = csf_raycast_cfg;

namespace detail {
inline int& device_slot() {
  static thread_local int dev = 0;
  return dev;
}
}  // namespace detail
// The device of the calling thread's default context (before its first use).
inline void set_device(int device) { detail::device_slot() = device; }
inline b200::Context& default_context() {
  static thread_local b200::Context ctx(detail::device_slot());
  return ctx;
}

// se3.hpp:21-45 PoseT<double>: R (row-major) and t
struct Pose {
  struct Rotation {
    std::array<double, 9> m{1, 0, 0, 0, 1, 0, 0, 0, 1};
    double& operator()(int r, int c) { return m[3 * r + c]; }
    double operator()(int r, int c) const { return m[3 * r + c]; }
  } rotation;
  std::array<double, 3> translation{};
  std::array<double, 12> packed() const {
    std::array<double, 12> a{};
    for (int e = 0; e < 9; ++e) a[e] = rotation.m[e];
    for (int e = 0; e < 3; ++e) a[9 + e] = translation[e];
    return a;
  }
  static Pose from(const std::array<double, 12>& a) {
    Pose p;
    for (int e = 0; e < 9; ++e) p.rotation.m[e] = a[e];
    for (int e = 0; e < 3; ++e) p.translation[e] = a[9 + e];
    return p;
  }
};

// frames.hpp:56-65 / frames.cpp:7-75
inline Image<double> bilateral_filter(const Image<double>& depth, double sigma_s = 4.5, double sigma_r = 0.03,
                                      int radius = 3) {
  return b200::bilateral_filter(default_context(), depth, sigma_s, sigma_r, radius);
}
inline std::vector<Image<double>> build_depth_pyramid(const Image<double>& depth, int levels = 3,
                                                      double sigma_r = 0.03) {
  return b200::build_depth_pyramid(default_context(), depth, levels, sigma_r);
}
// frames.hpp:86-87 (real depth)
inline SurfaceMaps measure_surface(const Image<double>& depth, const Intrinsics& k) {
  return b200::measure_surface(default_context(), depth, k);
}

// tsdf.hpp:144-145 surface_update(volume, depth, camera_to_world, k): real
// depth [h][w], or the lifted (Image<Complex>) depth [h][w][1+D]
inline int surface_update(Volume& volume, const Image<double>& depth, const Pose& camera_to_world,
                          const Intrinsics& k) {
  return b200::surface_update(default_context(), volume, depth,
                              b200::LiftedPose::real(camera_to_world.packed(), volume.channels()),
                              b200::LiftedIntrinsics(k, volume.channels()));
}
inline int surface_update(Volume& volume, const std::vector<double>& lifted_depth, const b200::LiftedPose& c2w,
                          const Intrinsics& k) {
  return b200::surface_update(default_context(), volume, lifted_depth, k.width, k.height, c2w,
                              b200::LiftedIntrinsics(k, volume.channels()));
}
// tsdf.hpp:209-211 raycast(volume, camera_to_world, k, cfg = {})
inline SurfaceMaps raycast(const Volume& volume, const Pose& camera_to_world, const Intrinsics& k,
                           const RaycastConfig* cfg = nullptr) {
  return b200::raycast(default_context(), volume, b200::LiftedPose::real(camera_to_world.packed(), volume.channels()),
                       b200::LiftedIntrinsics(k, volume.channels()), k.width, k.height, cfg);
}
// tsdf.hpp:148-149, 181-183 at a real world point
inline std::optional<double> sample_tsdf(const Volume& volume, const std::array<double, 3>& p_world) {
  std::vector<double> pt(3 * (1 + volume.channels()), 0.0);
  for (int a = 0; a < 3; ++a) pt[a * (1 + volume.channels())] = p_world[a];
  const auto r = b200::sample_tsdf(volume, pt);
  if (!r) return std::nullopt;
  return (*r)[0];
}
inline std::optional<std::array<double, 3>> sample_gradient(const Volume& volume, const std::array<double, 3>& p) {
  std::vector<double> pt(3 * (1 + volume.channels()), 0.0);
  for (int a = 0; a < 3; ++a) pt[a * (1 + volume.channels())] = p[a];
  const auto r = b200::sample_gradient(volume, pt);
  if (!r) return std::nullopt;
  return std::array<double, 3>{(*r)[0][0], (*r)[1][0], (*r)[2][0]};
}
// tsdf.hpp:97-102 measured_tsdf(depth, world_to_camera, k, mu, p_world, camera_center)
inline std::optional<double> measured_tsdf(const Image<double>& depth, const Pose& world_to_camera,
                                           const Intrinsics& k, double mu, const std::array<double, 3>& p_world,
                                           const std::array<double, 3>& camera_center) {
  const auto r = b200::measured_tsdf(default_context(), depth.data, depth.width, depth.height,
                                     b200::LiftedPose::real(world_to_camera.packed()), b200::LiftedIntrinsics(k, 0),
                                     mu, p_world, std::vector<double>(camera_center.begin(), camera_center.end()));
  if (!r) return std::nullopt;
  return (*r)[0];
}
// tsdf.hpp:288-289
inline void save_volume(const std::string& path, const Volume& volume) { b200::save_volume(path, volume); }
inline std::unique_ptr<Volume> load_volume(const std::string& path) {
  return b200::load_volume(default_context(), path);
}

// icp.hpp:59-65 associate(measured, predicted, camera_to_world, prediction_pose, k, cfg, stride)
inline std::vector<Correspondence> associate(const SurfaceMaps& measured, const SurfaceMaps& predicted,
                                             const Pose& camera_to_world, const Pose& prediction_camera_to_world,
                                             const Intrinsics& k, const IcpConfig& cfg, int pixel_stride = 1) {
  return b200::associate(default_context(), measured, predicted, camera_to_world.packed(),
                         prediction_camera_to_world.packed(), k, cfg, pixel_stride);
}
// icp.hpp:96-97
inline std::array<double, 6> linearized_step(const std::vector<Correspondence>& corrs, const Pose& base) {
  return b200::linearized_step(default_context(), corrs, base.packed());
}
// icp.hpp:70-91
inline double icp_loss(const std::vector<Correspondence>& corrs, const Pose& base) {
  return b200::icp_loss(default_context(), corrs, base.packed());
}
inline std::array<double, 6> icp_gradient(const std::vector<Correspondence>& corrs, const Pose& base) {
  return b200::icp_gradient(default_context(), corrs, base.packed());
}
// icp.hpp:130-133 track_frame(volume, depth, initial, k, cfg = {}, trace = nullptr)
inline TrackResult track_frame(const Volume& volume, const Image<double>& depth, const Pose& initial,
                               const Intrinsics& k, const IcpConfig* cfg = nullptr, TrackTrace* trace = nullptr) {
  return b200::track_frame(default_context(), volume, depth, initial.packed(), k, cfg, trace);
}
// diff.hpp:33-37
inline double pairwise_sum(const std::vector<double>& terms, double init = 0.0) {
  return b200::pairwise_sum(default_context(), terms, init);
}

}  // namespace csf
