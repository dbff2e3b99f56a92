// csf/b200.hpp — C++ mirror of the reference API (proj/include/csf/*.hpp)
// over the C-ABI in include/csf_b200.h.  Header-only; link libcsf_b200.so.
//
// Names, argument meaning and error behaviour follow the reference:
//   bilateral_filter / build_depth_pyramid   frames.hpp:56-65, frames.cpp:7-75
//   measure_surface                          frames.hpp:86-114
//   TsdfVolume (+ HashedVolume), surface_update, raycast   tsdf.hpp:38-284
//   track_frame (every solver family)        icp.hpp:130-133
//   icp_energy / icp_loss / icp_gradient / icp_hessian   icp.hpp:70-91
//   Pipeline: csfd_pipeline_gradient / csfd_pipeline_hessian (the CSFD
//   frame-derivative run; first order or bicomplex pairs)
// Errors are thrown as std::invalid_argument / std::domain_error /
// std::runtime_error exactly where the reference throws them.  Scalars are
// plain structs (no Eigen): Complex{re, im}, lifted values as (1+D) doubles.
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "../csf_b200.h"

namespace csf {
namespace b200 {

inline void check(csf_ctx ctx, int rc) {
  if (rc == CSF_OK) return;
  const std::string msg = ctx ? csf_last_error(ctx) : "csf_b200 error";
  if (rc == CSF_EINVAL) throw std::invalid_argument(msg);
  if (rc == CSF_EDOMAIN) throw std::domain_error(msg);
  throw std::runtime_error(msg);
}

// image.hpp:12-35
template <typename T>
struct Image {
  int width = 0, height = 0;
  std::vector<T> data;
  Image() = default;
  Image(int w, int h, T fill = T{}) : width(w), height(h), data(static_cast<size_t>(w) * h, fill) {}
  bool in_bounds(int x, int y) const { return x >= 0 && x < width && y >= 0 && y < height; }
  T& at(int x, int y) { return data[static_cast<size_t>(y) * width + x]; }
  const T& at(int x, int y) const { return data[static_cast<size_t>(y) * width + x]; }
};

// A pose with D perturbation channels: 12 scalars x (1+D), rotation
// row-major then translation (se3.hpp:21-45 with the channels unpacked).
struct LiftedPose {
  int channels = 0;
  std::vector<double> v;  // [12][1+D]
  explicit LiftedPose(int D = 0) : channels(D), v(12 * (1 + D), 0.0) {
    for (int i = 0; i < 3; ++i) at(4 * i, 0) = 1.0;
  }
  double& at(int e, int c) { return v[e * (1 + channels) + c]; }
  double at(int e, int c) const { return v[e * (1 + channels) + c]; }
  static LiftedPose real(const std::array<double, 12>& p, int D = 0) {
    LiftedPose o(D);
    for (int e = 0; e < 12; ++e) o.at(e, 0) = p[e];
    return o;
  }
};

struct LiftedIntrinsics {
  int channels = 0;
  std::vector<double> v;  // [4][1+D]: fx, fy, cx, cy
  LiftedIntrinsics(const csf_intrinsics& k, int D = 0) : channels(D), v(4 * (1 + D), 0.0) {
    v[0] = k.fx;
    v[1 + D] = k.fy;
    v[2 * (1 + D)] = k.cx;
    v[3 * (1 + D)] = k.cy;
  }
};

class Context {
 public:
  explicit Context(int device = 0) {
    if (csf_ctx_create(device, &ctx_) != CSF_OK)
      throw std::runtime_error("csf_b200: no usable CUDA device (no CPU fallback)");
  }
  ~Context() { csf_ctx_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  csf_ctx get() const { return ctx_; }

 private:
  csf_ctx ctx_ = nullptr;
};

// frames.cpp:7-38
inline Image<double> bilateral_filter(Context& c, const Image<double>& depth, double sigma_s = 4.5,
                                      double sigma_r = 0.03, int radius = 3) {
  Image<double> out(depth.width, depth.height);
  check(c.get(), csf_bilateral_filter(c.get(), depth.data.data(), depth.width, depth.height, sigma_s, sigma_r, radius,
                                      out.data.data()));
  return out;
}

// frames.cpp:40-75
inline Image<double> downsample_depth(Context& c, const Image<double>& depth, double sigma_r = 0.03) {
  Image<double> out(depth.width / 2, depth.height / 2);
  check(c.get(), csf_downsample_depth(c.get(), depth.data.data(), depth.width, depth.height, sigma_r, out.data.data()));
  return out;
}
inline std::vector<Image<double>> build_depth_pyramid(Context& c, const Image<double>& depth, int levels = 3,
                                                      double sigma_r = 0.03) {
  std::vector<Image<double>> pyr{depth};
  for (int l = 1; l < levels; ++l) pyr.push_back(downsample_depth(c, pyr.back(), sigma_r));
  return pyr;
}

// tsdf.hpp:38-78 — a device-resident volume whose field carries D channels.
class Volume {
 public:
  Volume(Context& c, const csf_volume_params& p, int channels) : ctx_(c.get()), channels_(channels), n_(1) {
    check(ctx_, csf_volume_create_dense(ctx_, &p, channels, &vol_));
    n_ = static_cast<size_t>(p.dims[0]) * p.dims[1] * p.dims[2];
  }
  Volume(Context& c, const csf_hash_params& p, int channels) : ctx_(c.get()), channels_(channels), hashed_(true) {
    check(ctx_, csf_volume_create_hashed(ctx_, &p, channels, &vol_));
  }
  // adopts a handle from csf_volume_load
  Volume(Context& c, csf_volume v) : ctx_(c.get()), vol_(v) {
    int hashed = 0;
    long long n = 0;
    check(ctx_, csf_volume_info(vol_, &channels_, &hashed, &n));
    hashed_ = hashed != 0;
    n_ = static_cast<size_t>(n);
  }
  ~Volume() { csf_volume_destroy(vol_); }
  Volume(const Volume&) = delete;
  Volume& operator=(const Volume&) = delete;
  csf_volume get() const { return vol_; }
  csf_ctx ctx() const { return ctx_; }
  int channels() const { return channels_; }
  size_t voxel_count() const {
    if (!hashed_) return n_;
    int nb = 0;
    check(ctx_, csf_volume_block_count(vol_, &nb));
    return static_cast<size_t>(nb) * 512;
  }
  // host copies: field [n][1+D], weight [n]
  void download(std::vector<double>& field, std::vector<double>& weight) const {
    const size_t n = voxel_count();
    field.resize(n * (1 + channels_));
    weight.resize(n);
    check(ctx_, csf_volume_download(vol_, field.data(), weight.data()));
  }
  void upload(const std::vector<double>& field, const std::vector<double>& weight) {
    check(ctx_, csf_volume_upload(vol_, field.data(), weight.data()));
  }

 private:
  csf_ctx ctx_;
  csf_volume vol_ = nullptr;
  int channels_ = 0;
  bool hashed_ = false;
  size_t n_ = 0;
};

// tsdf.cpp:11-40 — surface_update(volume, depth, camera_to_world, k)
inline int surface_update(Context& c, Volume& vol, const Image<double>& depth, const LiftedPose& camera_to_world,
                          const LiftedIntrinsics& k) {
  if (camera_to_world.channels != vol.channels() || k.channels != vol.channels())
    throw std::invalid_argument("surface_update: channel count mismatch");
  int n_visible = 0;
  check(c.get(), csf_surface_update(vol.get(), depth.data.data(), depth.width, depth.height, camera_to_world.v.data(),
                                    k.v.data(), &n_visible));
  return n_visible;
}

// frames.hpp:67-71 SurfaceMaps with channels unpacked: [h][w][3][1+D]
struct SurfaceMaps {
  int width = 0, height = 0, channels = 0;
  std::vector<double> vertices, normals;
};

// tsdf.hpp:209-284
inline SurfaceMaps raycast(Context& c, const Volume& vol, const LiftedPose& camera_to_world,
                           const LiftedIntrinsics& k, int width, int height, const csf_raycast_cfg* cfg = nullptr) {
  SurfaceMaps m;
  m.width = width;
  m.height = height;
  m.channels = vol.channels();
  m.vertices.resize(static_cast<size_t>(width) * height * 3 * (1 + m.channels));
  m.normals.resize(m.vertices.size());
  check(c.get(), csf_raycast(vol.get(), camera_to_world.v.data(), k.v.data(), width, height, cfg, m.vertices.data(),
                             m.normals.data()));
  return m;
}

// icp.hpp:119-133
struct TrackResult {
  std::array<double, 12> pose{};
  int iterations = 0;
  bool converged = false;
  double final_loss = 0.0;
  int correspondences = 0;
};
// icp.hpp:103-114
struct TraceRow {
  int iteration = 0;
  double loss = 0.0, gradient_norm = 0.0, translation_error = 0.0, rotation_error = 0.0;
};
struct TrackTrace {
  bool has_ground_truth = false;
  std::array<double, 12> ground_truth{};
  std::vector<TraceRow> rows;
};
inline TrackResult track_frame(Context& c, const Volume& vol, const Image<double>& depth,
                               const std::array<double, 12>& init_camera_to_world, const csf_intrinsics& k,
                               const csf_icp_cfg* cfg = nullptr, TrackTrace* trace = nullptr) {
  csf_icp_cfg def;
  csf_default_icp_cfg(&def);
  const csf_icp_cfg& cf = cfg ? *cfg : def;
  TrackResult r;
  csf_track_result tr{};
  if (!trace) {
    check(c.get(), csf_track_frame(vol.get(), depth.data.data(), depth.width, depth.height,
                                   init_camera_to_world.data(), &k, &cf, r.pose.data(), &tr));
  } else {
    const int cap = std::max(1, cf.level_iterations[0] + cf.level_iterations[1] + cf.level_iterations[2]);
    std::vector<double> rows(15 * static_cast<size_t>(cap));
    int n = 0;
    check(c.get(), csf_track_frame_traced(vol.get(), depth.data.data(), depth.width, depth.height,
                                          init_camera_to_world.data(), &k, &cf, r.pose.data(), &tr, rows.data(), cap,
                                          &n));
    for (int i = 0; i < n && i < cap; ++i) {
      const double* w = rows.data() + 15 * i;
      TraceRow row;
      row.iteration = static_cast<int>(w[0]);
      row.loss = w[1];
      row.gradient_norm = w[2];
      row.translation_error = row.rotation_error = std::nan("");
      if (trace->has_ground_truth) {  // icp.cpp:220-226 (host arithmetic on the returned pose)
        const auto& g = trace->ground_truth;
        const double dx = w[12] - g[9], dy = w[13] - g[10], dz = w[14] - g[11];
        row.translation_error = std::sqrt(dx * dx + (dy * dy + dz * dz));
        double tr3 = 0.0;  // trace(g_R^T R)
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b) tr3 += g[3 * b + a] * w[3 + 3 * b + a];
        row.rotation_error = std::acos(std::max(-1.0, std::min(1.0, (tr3 - 1.0) / 2.0))) * 180.0 / M_PI;
      }
      trace->rows.push_back(row);
    }
  }
  r.iterations = tr.iterations;
  r.converged = tr.converged != 0;
  r.final_loss = tr.final_loss;
  r.correspondences = tr.correspondences;
  return r;
}

// icp.hpp:27-31
struct Correspondence {
  std::array<double, 3> vertex{}, model_vertex{}, model_normal{};
};
namespace detail {
inline std::vector<double> pack(const std::vector<Correspondence>& corrs) {
  std::vector<double> out(corrs.size() * 9);
  for (size_t i = 0; i < corrs.size(); ++i)
    for (int k = 0; k < 3; ++k) {
      out[9 * i + k] = corrs[i].vertex[k];
      out[9 * i + 3 + k] = corrs[i].model_vertex[k];
      out[9 * i + 6 + k] = corrs[i].model_normal[k];
    }
  return out;
}
}  // namespace detail

// icp.hpp:70-85 (real xi; pairwise_sum tree on the device)
inline double icp_energy(Context& c, const std::vector<Correspondence>& corrs, const std::array<double, 6>& xi,
                         const std::array<double, 12>& base) {
  const std::vector<double> p = detail::pack(corrs);
  double e = 0.0;
  check(c.get(), csf_icp_energy_derivs(c.get(), p.data(), static_cast<int>(corrs.size()), base.data(), xi.data(),
                                       1e-8, &e, nullptr, nullptr));
  return e;
}
// icp.cpp:128-144
inline double icp_loss(Context& c, const std::vector<Correspondence>& corrs, const std::array<double, 12>& base) {
  return icp_energy(c, corrs, std::array<double, 6>{}, base);
}
inline std::array<double, 6> icp_gradient(Context& c, const std::vector<Correspondence>& corrs,
                                          const std::array<double, 12>& base, double h = 1e-8) {
  const std::vector<double> p = detail::pack(corrs);
  std::array<double, 6> g{};
  double e = 0.0;
  check(c.get(), csf_icp_energy_derivs(c.get(), p.data(), static_cast<int>(corrs.size()), base.data(), nullptr, h, &e,
                                       g.data(), nullptr));
  return g;
}
inline std::array<std::array<double, 6>, 6> icp_hessian(Context& c, const std::vector<Correspondence>& corrs,
                                                        const std::array<double, 12>& base, double h = 1e-8) {
  const std::vector<double> p = detail::pack(corrs);
  double hh[36];
  double e = 0.0;
  check(c.get(), csf_icp_energy_derivs(c.get(), p.data(), static_cast<int>(corrs.size()), base.data(), nullptr, h, &e,
                                       nullptr, hh));
  std::array<std::array<double, 6>, 6> out{};
  for (int r = 0; r < 6; ++r)
    for (int col = 0; col < 6; ++col) out[r][col] = hh[6 * r + col];
  return out;
}

// ---------------------------------------------------------------------------
// reloc.hpp:35-138 — relocalization.  RelocProblem is device-resident; the
// energy and its CSFD derivatives are one packed device pass each.
// ---------------------------------------------------------------------------
class RelocProblem {
 public:
  // reloc.hpp:44-45: throws std::invalid_argument if the reference has no
  // observed voxels.
  RelocProblem(const Volume& reference, const Image<double>& query, const csf_intrinsics& k)
      : ctx_(reference.ctx()) {
    check(ctx_, csf_reloc_create(reference.get(), query.data.data(), query.width, query.height, &k, &r_));
    check(ctx_, csf_reloc_info(r_, &n_, &mu_, nullptr, nullptr));
  }
  ~RelocProblem() { csf_reloc_destroy(r_); }
  RelocProblem(const RelocProblem&) = delete;
  RelocProblem& operator=(const RelocProblem&) = delete;
  csf_reloc get() const { return r_; }
  csf_ctx ctx() const { return ctx_; }
  int voxel_count() const { return n_; }
  double mu() const { return mu_; }
  // E (+ gradient, + Hessian [36]) at a camera->world pose; order 0/1/2
  double energy(const std::array<double, 12>& pose, int order = 0, double h = 1e-8, double* g = nullptr,
                double* hess = nullptr, long long* overlap = nullptr) const {
    double e = 0.0, gg[6], hh[36];
    check(ctx_, csf_reloc_energy(r_, pose.data(), order, h, &e, order >= 1 ? (g ? g : gg) : nullptr,
                                 order == 2 ? (hess ? hess : hh) : nullptr, overlap));
    return e;
  }

 private:
  csf_ctx ctx_;
  csf_reloc r_ = nullptr;
  int n_ = 0;
  double mu_ = 0.1;
};

// reloc.hpp:48-80
inline double reloc_energy(const RelocProblem& p, const std::array<double, 12>& query_pose) {
  return p.energy(query_pose);
}
inline double reloc_loss(const RelocProblem& p, const std::array<double, 12>& pose) { return p.energy(pose); }
inline std::array<double, 6> reloc_gradient(const RelocProblem& p, const std::array<double, 12>& pose,
                                            double h = 1e-8) {
  std::array<double, 6> g{};
  p.energy(pose, 1, h, g.data());
  return g;
}
inline std::array<std::array<double, 6>, 6> reloc_hessian(const RelocProblem& p, const std::array<double, 12>& pose,
                                                          double h = 1e-8) {
  double hh[36], g[6];
  p.energy(pose, 2, h, g, hh);
  std::array<std::array<double, 6>, 6> out{};
  for (int r = 0; r < 6; ++r)
    for (int col = 0; col < 6; ++col) out[r][col] = hh[6 * r + col];
  return out;
}

// reloc.hpp:82-124
enum class RelocMethod { kGradientDescent = CSF_RELOC_GRADIENT_DESCENT, kNewton = CSF_RELOC_NEWTON };
struct RelocResult {
  std::array<double, 12> pose{};
  int iterations = 0;
  bool converged = false;
  double final_loss = 0.0;
  RelocMethod method = RelocMethod::kNewton;
  std::vector<double> losses, gradient_norms;  // trace rows
};
inline csf_reloc_cfg default_reloc_config() {
  csf_reloc_cfg c;
  csf_default_reloc_cfg(&c);
  return c;
}
inline RelocResult relocalize(const RelocProblem& p, const std::array<double, 12>& initial, RelocMethod method,
                              const csf_reloc_cfg& cfg = default_reloc_config()) {
  RelocResult r;
  r.method = method;
  const size_t n = static_cast<size_t>(cfg.max_iterations > 0 ? cfg.max_iterations : 1);
  r.losses.resize(n);
  r.gradient_norms.resize(n);
  csf_reloc_result res{};
  check(p.ctx(), csf_relocalize(p.get(), initial.data(), static_cast<int>(method), &cfg,
                                                 r.pose.data(), &res, r.losses.data(), r.gradient_norms.data()));
  r.iterations = res.iterations;
  r.converged = res.converged != 0;
  r.final_loss = res.final_loss;
  r.losses.resize(res.iterations);
  r.gradient_norms.resize(res.iterations);
  return r;
}

// reloc.hpp:126-129
inline std::vector<std::array<double, 3>> depth_cloud(Context& c, const Image<double>& depth, const csf_intrinsics& k,
                                                      const std::array<double, 12>& camera_to_world, int stride = 1) {
  const int s = stride > 0 ? stride : 1;
  std::vector<double> buf(3 * static_cast<size_t>((depth.width + s - 1) / s) * ((depth.height + s - 1) / s) + 3);
  int n = 0;
  check(c.get(), csf_depth_cloud(c.get(), depth.data.data(), depth.width, depth.height, &k, camera_to_world.data(),
                                 stride, buf.data(), &n));
  std::vector<std::array<double, 3>> out(n);
  for (int i = 0; i < n; ++i) out[i] = {buf[3 * i], buf[3 * i + 1], buf[3 * i + 2]};
  return out;
}

// reloc.hpp:131-138
struct NnError {
  double mean = 0.0;
  bool outlier = false;
};
inline NnError eval_nn_error(Context& c, const std::array<double, 12>& transform,
                             const std::vector<std::array<double, 3>>& query,
                             const std::vector<std::array<double, 3>>& reference) {
  NnError e;
  int32_t out = 0;
  check(c.get(), csf_eval_nn_error(c.get(), transform.data(), query.empty() ? nullptr : query[0].data(),
                                   static_cast<int>(query.size()), reference.empty() ? nullptr : reference[0].data(),
                                   static_cast<int>(reference.size()), &e.mean, &out));
  e.outlier = out != 0;
  return e;
}

// ---------------------------------------------------------------------------
// surfel.hpp — the surfel (X-EF) front end; the map lives on the device with
// D derivative channels (the reference's Complex is D = 1).
// ---------------------------------------------------------------------------
struct SurfelHost {  // surfel.hpp:16-22, channels unpacked
  std::vector<double> position, normal;  // [3][1+D]
  double radius = 0.0;
  std::vector<double> confidence;  // [1+D]
  int timestamp = 0;
};
inline csf_surfel_cfg default_surfel_config() {
  csf_surfel_cfg c;
  csf_default_surfel_cfg(&c);
  return c;
}
struct SurfelUpdateStats {  // surfel.hpp:93-96
  int merged_pixels = 0;
  int created = 0;
};
class SurfelMap {
 public:
  SurfelMap(Context& c, int channels = 1) : ctx_(c.get()), channels_(channels) {
    check(ctx_, csf_surfels_create(ctx_, channels, &m_));
  }
  ~SurfelMap() { csf_surfels_destroy(m_); }
  SurfelMap(const SurfelMap&) = delete;
  SurfelMap& operator=(const SurfelMap&) = delete;
  csf_surfels get() const { return m_; }
  csf_ctx ctx() const { return ctx_; }
  int channels() const { return channels_; }
  std::size_t size() const {
    int n = 0;
    check(ctx_, csf_surfels_count(m_, &n));
    return static_cast<std::size_t>(n);
  }
  std::vector<SurfelHost> download() const {
    const std::size_t n = size(), C = 1 + channels_;
    std::vector<double> p(3 * n * C), q(3 * n * C), r(n), c(n * C);
    std::vector<int32_t> t(n);
    if (n) check(ctx_, csf_surfels_download(m_, p.data(), q.data(), r.data(), c.data(), t.data()));
    std::vector<SurfelHost> out(n);
    for (std::size_t i = 0; i < n; ++i) {
      out[i].position.assign(p.begin() + 3 * i * C, p.begin() + 3 * (i + 1) * C);
      out[i].normal.assign(q.begin() + 3 * i * C, q.begin() + 3 * (i + 1) * C);
      out[i].radius = r[i];
      out[i].confidence.assign(c.begin() + i * C, c.begin() + (i + 1) * C);
      out[i].timestamp = t[i];
    }
    return out;
  }

 private:
  csf_ctx ctx_;
  csf_surfels m_ = nullptr;
  int channels_ = 1;
};
// surfel.cpp:121-236: depth [h][w][1+D] lifted, pose lifted (channels = map's)
inline SurfelUpdateStats update_surfels(SurfelMap& map, const std::vector<double>& lifted_depth, int w, int h,
                                        const LiftedPose& camera_to_world, const csf_intrinsics& k, int frame_index,
                                        const csf_surfel_cfg& cfg = default_surfel_config()) {
  if (camera_to_world.channels != map.channels())
    throw std::invalid_argument("update_surfels: channel count mismatch");
  SurfelUpdateStats s;
  check(map.ctx(), csf_update_surfels(map.get(), lifted_depth.data(), w, h, camera_to_world.v.data(), &k, frame_index,
                                      &cfg, &s.merged_pixels, &s.created));
  return s;
}
// surfel.cpp:238-263
inline SurfaceMaps predict_maps(const SurfelMap& map, const std::array<double, 12>& camera_to_world,
                                const csf_intrinsics& k) {
  SurfaceMaps m;
  m.width = k.width;
  m.height = k.height;
  m.vertices.resize(3 * static_cast<std::size_t>(k.width) * k.height);
  m.normals.resize(m.vertices.size());
  check(map.ctx(), csf_predict_maps(map.get(), camera_to_world.data(), &k, m.vertices.data(), m.normals.data()));
  return m;
}
// surfel.cpp:110-119
inline double sample_confidence(const csf_intrinsics& k, int x, int y) { return csf_sample_confidence(&k, x, y); }


// ---------------------------------------------------------------------------
// frames.hpp:86-114 measure_surface: depth [h][w] real (or [h][w][1+D] lifted
// with the intrinsics' D channels); maps [h][w][3][1+D]
// ---------------------------------------------------------------------------
inline SurfaceMaps measure_surface(Context& c, const Image<double>& depth, const csf_intrinsics& k) {
  SurfaceMaps m;
  m.width = depth.width;
  m.height = depth.height;
  m.vertices.resize(static_cast<size_t>(depth.width) * depth.height * 3);
  m.normals.resize(m.vertices.size());
  const LiftedIntrinsics kk(k, 0);
  check(c.get(), csf_measure_surface(c.get(), depth.data.data(), depth.width, depth.height, kk.v.data(), 0,
                                     m.vertices.data(), m.normals.data()));
  return m;
}
inline SurfaceMaps measure_surface(Context& c, const std::vector<double>& lifted_depth, int w, int h,
                                   const LiftedIntrinsics& k) {
  if (lifted_depth.size() != static_cast<size_t>(w) * h * (1 + k.channels))
    throw std::invalid_argument("measure_surface: lifted depth size");
  SurfaceMaps m;
  m.width = w;
  m.height = h;
  m.channels = k.channels;
  m.vertices.resize(static_cast<size_t>(w) * h * 3 * (1 + k.channels));
  m.normals.resize(m.vertices.size());
  check(c.get(), csf_measure_surface(c.get(), lifted_depth.data(), w, h, k.v.data(), k.channels, m.vertices.data(),
                                     m.normals.data()));
  return m;
}

// tsdf.cpp:11-40 with the reference's Image<Complex> depth (tsdf.hpp:144-145):
// lifted depth [h][w][1+D], D = the volume's channels
inline int surface_update(Context& c, Volume& vol, const std::vector<double>& lifted_depth, int w, int h,
                          const LiftedPose& camera_to_world, const LiftedIntrinsics& k) {
  if (camera_to_world.channels != vol.channels() || k.channels != vol.channels() ||
      lifted_depth.size() != static_cast<size_t>(w) * h * (1 + vol.channels()))
    throw std::invalid_argument("surface_update: channel count mismatch");
  int n_visible = 0;
  check(c.get(), csf_surface_update_lifted(vol.get(), lifted_depth.data(), w, h, camera_to_world.v.data(),
                                           k.v.data(), &n_visible));
  return n_visible;
}

// tsdf.hpp:148-196 sample_tsdf / sample_gradient at a lifted world point
// [3][1+D] (D = the volume's channels): std::nullopt where the reference
// returns no value.
using Lifted = std::vector<double>;  // [1+D]
inline std::optional<Lifted> sample_tsdf(const Volume& vol, const std::vector<double>& point) {
  const int C = 1 + vol.channels();
  if (point.size() != static_cast<size_t>(3 * C)) throw std::invalid_argument("sample_tsdf: point is [3][1+D]");
  Lifted out(C);
  int32_t ok = 0;
  check(vol.ctx(), csf_sample_tsdf(vol.get(), point.data(), 1, out.data(), &ok));
  if (!ok) return std::nullopt;
  return out;
}
inline std::optional<std::array<Lifted, 3>> sample_gradient(const Volume& vol, const std::vector<double>& point) {
  const int C = 1 + vol.channels();
  if (point.size() != static_cast<size_t>(3 * C)) throw std::invalid_argument("sample_gradient: point is [3][1+D]");
  std::vector<double> out(3 * C);
  int32_t ok = 0;
  check(vol.ctx(), csf_sample_gradient(vol.get(), point.data(), 1, out.data(), &ok));
  if (!ok) return std::nullopt;
  std::array<Lifted, 3> g;
  for (int a = 0; a < 3; ++a) g[a].assign(out.begin() + a * C, out.begin() + (a + 1) * C);
  return g;
}

// tsdf.hpp:97-140 measured_tsdf(depth, world_to_camera, k, mu, p_world,
// camera_center): depth real [h][w] or lifted [h][w][1+D]; psi [1+D]
inline std::optional<Lifted> measured_tsdf(Context& c, const std::vector<double>& depth, int w, int h,
                                           const LiftedPose& world_to_camera, const LiftedIntrinsics& k, double mu,
                                           const std::array<double, 3>& p_world,
                                           const std::vector<double>& camera_center) {
  const int D = world_to_camera.channels, C = 1 + D;
  if (k.channels != D || camera_center.size() != static_cast<size_t>(3 * C))
    throw std::invalid_argument("measured_tsdf: channel count mismatch");
  const size_t P = static_cast<size_t>(w) * h;
  const bool lifted = depth.size() == P * C && D > 0;
  if (!lifted && depth.size() != P) throw std::invalid_argument("measured_tsdf: depth size");
  Lifted psi(C);
  int32_t ok = 0;
  check(c.get(), (lifted ? csf_measured_tsdf_lifted : csf_measured_tsdf)(
                     c.get(), depth.data(), w, h, world_to_camera.v.data(), k.v.data(), mu, p_world.data(),
                     camera_center.data(), 1, D, psi.data(), &ok));
  if (!ok) return std::nullopt;
  return psi;
}

// tsdf.hpp:288-289 / tsdf.cpp:61-153 — the "CSFVOL 1" checkpoint
inline void save_volume(const std::string& path, const Volume& vol) {
  check(vol.ctx(), csf_volume_save(vol.get(), path.c_str()));
}
inline std::unique_ptr<Volume> load_volume(Context& c, const std::string& path, int channels = -1) {
  csf_volume v = nullptr;
  check(c.get(), csf_volume_load(c.get(), path.c_str(), channels, &v));
  return std::unique_ptr<Volume>(new Volume(c, v));
}

// icp.cpp:89-126 associate(measured, predicted, camera_to_world,
// prediction_camera_to_world, k, cfg, stride): real maps [h][w][3]
inline std::vector<Correspondence> associate(Context& c, const SurfaceMaps& measured, const SurfaceMaps& predicted,
                                             const std::array<double, 12>& camera_to_world,
                                             const std::array<double, 12>& prediction_camera_to_world,
                                             const csf_intrinsics& k, const csf_icp_cfg& cfg, int pixel_stride = 1) {
  if (measured.channels != 0 || predicted.channels != 0) throw std::invalid_argument("associate: real maps");
  const size_t P = static_cast<size_t>(measured.width) * measured.height;
  std::vector<double> flat(P * 9);
  int n = 0;
  check(c.get(), csf_associate(c.get(), measured.vertices.data(), measured.normals.data(), predicted.vertices.data(),
                               predicted.normals.data(), measured.width, measured.height, camera_to_world.data(),
                               prediction_camera_to_world.data(), &k, &cfg, pixel_stride, flat.data(), &n));
  std::vector<Correspondence> out(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i)
    for (int q = 0; q < 3; ++q) {
      out[i].vertex[q] = flat[9 * i + q];
      out[i].model_vertex[q] = flat[9 * i + 3 + q];
      out[i].model_normal[q] = flat[9 * i + 6 + q];
    }
  return out;
}
// icp.cpp:146-153 linearized_step(corrs, base)
inline std::array<double, 6> linearized_step(Context& c, const std::vector<Correspondence>& corrs,
                                             const std::array<double, 12>& base) {
  const std::vector<double> flat = detail::pack(corrs);
  std::array<double, 6> d{};
  check(c.get(), csf_linearized_step(c.get(), flat.data(), static_cast<int>(corrs.size()), base.data(), d.data()));
  return d;
}

// diff.hpp:16-37 pairwise_sum(terms, init = 0) — the reference's fixed tree
inline double pairwise_sum(Context& c, const std::vector<double>& terms, double init = 0.0) {
  double out = 0.0;
  check(c.get(), csf_pairwise_sum(c.get(), terms.data(), static_cast<int>(terms.size()), 1, &out));
  return init + out;
}

// ---------------------------------------------------------------------------
// csfd.hpp:33-140 truncated first- and second-order CSFD scalars and
// diff.hpp:46-72 csfd_gradient / csfd_hessian of a user function f(x) with x
// a 6-vector of those scalars.  Host arithmetic (f is user code); the
// concrete functions of the hot path (icp_gradient / icp_hessian,
// reloc_gradient / reloc_hessian, the pipeline) run as packed device passes.
// ---------------------------------------------------------------------------
struct Complex {
  double re = 0.0, im = 0.0;
  Complex() = default;
  Complex(double r, double i = 0.0) : re(r), im(i) {}
};
inline Complex operator+(Complex a, Complex b) { return {a.re + b.re, a.im + b.im}; }
inline Complex operator-(Complex a, Complex b) { return {a.re - b.re, a.im - b.im}; }
inline Complex operator-(Complex a) { return {-a.re, -a.im}; }
inline Complex operator*(Complex a, Complex b) { return {a.re * b.re, a.re * b.im + a.im * b.re}; }
inline Complex operator/(Complex a, Complex b) {
  if (b.re == 0.0) throw std::domain_error("Complex division by zero real part");
  return {a.re / b.re, (a.im * b.re - a.re * b.im) / (b.re * b.re)};
}
inline Complex sqrt(Complex a) {
  const double r = std::sqrt(a.re);
  return {r, a.im * (0.5 / r)};
}
inline Complex sin(Complex a) { return {std::sin(a.re), std::cos(a.re) * a.im}; }
inline Complex cos(Complex a) { return {std::cos(a.re), -std::sin(a.re) * a.im}; }
inline Complex exp(Complex a) {
  const double e = std::exp(a.re);
  return {e, e * a.im};
}
struct Bicomplex {
  double re = 0.0, im1 = 0.0, im2 = 0.0, im12 = 0.0;
  Bicomplex() = default;
  Bicomplex(double r, double a = 0.0, double b = 0.0, double ab = 0.0) : re(r), im1(a), im2(b), im12(ab) {}
};
inline Bicomplex operator+(Bicomplex a, Bicomplex b) {
  return {a.re + b.re, a.im1 + b.im1, a.im2 + b.im2, a.im12 + b.im12};
}
inline Bicomplex operator-(Bicomplex a, Bicomplex b) {
  return {a.re - b.re, a.im1 - b.im1, a.im2 - b.im2, a.im12 - b.im12};
}
inline Bicomplex operator-(Bicomplex a) { return {-a.re, -a.im1, -a.im2, -a.im12}; }
inline Bicomplex operator*(Bicomplex a, Bicomplex b) {
  return {a.re * b.re, a.re * b.im1 + a.im1 * b.re, a.re * b.im2 + a.im2 * b.re,
          a.re * b.im12 + a.im12 * b.re + a.im1 * b.im2 + a.im2 * b.im1};
}
inline Bicomplex operator/(Bicomplex a, Bicomplex b) {
  if (b.re == 0.0) throw std::domain_error("Bicomplex division by zero real part");
  const double inv = 1.0 / b.re, inv2 = inv * inv;
  const double q1 = (a.im1 * b.re - a.re * b.im1) * inv2;
  const double q2 = (a.im2 * b.re - a.re * b.im2) * inv2;
  const double q12 = (a.im12 - (a.re * inv) * b.im12 - q1 * b.im2 - q2 * b.im1) * inv;
  return {a.re * inv, q1, q2, q12};
}
template <typename F>
std::array<double, 6> csfd_gradient(F&& f, const std::array<double, 6>& x, double h = 1e-8) {
  if (!(h > 0.0) || h > 1e-6) throw std::invalid_argument("StepSize: step must satisfy 0 < h <= 1e-6");
  std::array<double, 6> g{};
  for (int i = 0; i < 6; ++i) {
    std::array<Complex, 6> xc;
    for (int j = 0; j < 6; ++j) xc[j] = Complex(x[j], i == j ? h : 0.0);
    g[i] = f(xc).im / h;
  }
  return g;
}
template <typename F>
std::array<std::array<double, 6>, 6> csfd_hessian(F&& f, const std::array<double, 6>& x, double h = 1e-8) {
  if (!(h > 0.0) || h > 1e-6) throw std::invalid_argument("StepSize: step must satisfy 0 < h <= 1e-6");
  std::array<std::array<double, 6>, 6> H{};
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j <= i; ++j) {
      std::array<Bicomplex, 6> xb;
      for (int k = 0; k < 6; ++k) xb[k] = Bicomplex(x[k], k == i ? h : 0.0, k == j ? h : 0.0, 0.0);
      H[i][j] = H[j][i] = f(xb).im12 / (h * h);
    }
  return H;
}

// ---------------------------------------------------------------------------
// dataset.hpp:17-36 — on-disk formats (host file I/O; std::runtime_error)
// ---------------------------------------------------------------------------
namespace detail {
inline void io_check(int rc) {
  if (rc == CSF_OK) return;
  if (rc == CSF_EINVAL) throw std::invalid_argument("csf_b200: invalid argument");
  throw std::runtime_error(csf_io_last_error());
}
}  // namespace detail
inline void write_depth_png16(const std::string& path, const Image<double>& depth, double scale) {
  detail::io_check(csf_write_depth_png16(path.c_str(), depth.data.data(), depth.width, depth.height, scale));
}
inline Image<double> read_depth_png16(const std::string& path, double scale) {
  int w = 0, h = 0;
  detail::io_check(csf_read_depth_png16(path.c_str(), scale, nullptr, &w, &h));
  Image<double> out(w, h);
  detail::io_check(csf_read_depth_png16(path.c_str(), scale, out.data.data(), &w, &h));
  return out;
}
inline csf_intrinsics read_intrinsics(const std::string& path) {
  csf_intrinsics k{};
  detail::io_check(csf_read_intrinsics(path.c_str(), &k));
  return k;
}
inline void write_intrinsics(const std::string& path, const csf_intrinsics& k) {
  detail::io_check(csf_write_intrinsics(path.c_str(), &k));
}
struct TrajectoryEntry {
  double timestamp = 0.0;
  std::array<double, 12> pose{};
};
inline std::vector<TrajectoryEntry> read_trajectory(const std::string& path) {
  int n = 0;
  detail::io_check(csf_read_trajectory(path.c_str(), nullptr, nullptr, 0, &n));
  std::vector<double> ts(n), ps(12 * static_cast<size_t>(n));
  detail::io_check(csf_read_trajectory(path.c_str(), ts.data(), ps.data(), n, &n));
  std::vector<TrajectoryEntry> out(n);
  for (int i = 0; i < n; ++i) {
    out[i].timestamp = ts[i];
    for (int e = 0; e < 12; ++e) out[i].pose[e] = ps[12 * i + e];
  }
  return out;
}
inline void write_trajectory(const std::string& path, const std::vector<TrajectoryEntry>& traj) {
  std::vector<double> ts, ps;
  for (const auto& e : traj) {
    ts.push_back(e.timestamp);
    ps.insert(ps.end(), e.pose.begin(), e.pose.end());
  }
  detail::io_check(csf_write_trajectory(path.c_str(), ts.data(), ps.data(), static_cast<int>(traj.size())));
}

// The CSFD frame-derivative run; extension of the reference
// API: gradient over first-order directions, or Hessian entries over
// bicomplex pairs (csfd_hessian's pattern applied to the whole frame loop).
class Pipeline {
 public:
  Pipeline(Context& c, const csf_pipeline_cfg& cfg) : ctx_(c.get()), cfg_(cfg) {
    check(ctx_, csf_pipeline_create(ctx_, &cfg_, &p_));
  }
  ~Pipeline() { csf_pipeline_destroy(p_); }
  Pipeline(const Pipeline&) = delete;
  Pipeline& operator=(const Pipeline&) = delete;
  // depth [n][h][w] float32 metres, gt [n][12]
  std::vector<double> csfd_pipeline_gradient(const std::vector<float>& depth, const std::vector<double>& gt, int n,
                                             double* objective = nullptr) {
    if (cfg_.order == 2) throw std::invalid_argument("csfd_pipeline_gradient: pipeline has order 2");
    std::vector<double> g(static_cast<size_t>(cfg_.n_dirs));
    double obj = 0.0;
    check(ctx_, csf_pipeline_run_host(p_, depth.data(), gt.data(), n, g.data(), &obj));
    if (objective) *objective = obj;
    return g;
  }
  // RGB-D ingest (BASELINE config 2): rgb [n][h][w][3] uint8 beside the depth;
  // colour is uploaded, unused (the reference has no colour term)
  std::vector<double> csfd_pipeline_gradient_rgbd(const std::vector<float>& depth,
                                                  const std::vector<unsigned char>& rgb,
                                                  const std::vector<double>& gt, int n, double* objective = nullptr) {
    if (cfg_.order == 2) throw std::invalid_argument("csfd_pipeline_gradient_rgbd: pipeline has order 2");
    if (rgb.size() != depth.size() * 3) throw std::invalid_argument("csfd_pipeline_gradient_rgbd: rgb size");
    std::vector<double> g(static_cast<size_t>(cfg_.n_dirs));
    double obj = 0.0;
    check(ctx_, csf_pipeline_run_host_rgbd(p_, depth.data(), rgb.data(), gt.data(), n, g.data(), &obj));
    if (objective) *objective = obj;
    return g;
  }
  // H_{pair_i[p], pair_j[p]} per pair
  std::vector<double> csfd_pipeline_hessian(const std::vector<float>& depth, const std::vector<double>& gt, int n,
                                            double* objective = nullptr) {
    if (cfg_.order != 2) throw std::invalid_argument("csfd_pipeline_hessian: pipeline has order 1");
    check(ctx_, csf_pipeline_upload(p_, depth.data(), gt.data(), n));
    check(ctx_, csf_pipeline_run(p_, n));
    std::vector<double> hs(static_cast<size_t>(cfg_.n_pairs));
    check(ctx_, csf_pipeline_hessian(p_, hs.data(), nullptr, nullptr, objective, nullptr, nullptr));
    return hs;
  }

 private:
  csf_ctx ctx_;
  csf_pipeline_cfg cfg_;
  csf_pipeline p_ = nullptr;
};

}  // namespace b200
}  // namespace csf
