// ORACLE — TEST INFRASTRUCTURE ONLY (see orc_core.hpp header).
//
// Camera relocalization.  The reference implements one
// function of its reloc module, the template reloc_energy<S>
// (proj/include/csf/reloc.hpp:48-69); everything else in reloc.hpp is
// declared without a body (there is no src/reloc.cpp).  reloc_energy is
// restated literally below; the declared-only pieces get BUILDER-DEFINED
// bodies that follow the header's own comments (reloc.hpp:16-46, 71-131) and
// SPEC.md:533-600, with the rules stated in DESIGN.md §3.9:
//   * RelocProblem flattens the observed voxels (W > 0) in storage order —
//     dense: linear index (k*ny + j)*nx + i; hashed: block pool order, then
//     the block-local index — with centre origin + vs*(i, j, k) and the real
//     field value; mu = the reference volume's mu.
//   * relocalize: steepest descent, or the eta-switched Newton direction
//     (once loss < switch threshold; -H^-1 g when the LDLT succeeds, is
//     finite and descends), both through backtracking_search
//     (descent.hpp:34-52); a trial pose with no overlapping voxel counts as
//     +inf; stop when |step| < step_tolerance (converged), when the line
//     search fails, or when the slope is not negative (converged iff the
//     gradient is exactly zero).
//   * depth_cloud: valid pixels at the stride in row-major order,
//     camera_to_world * backproject(k, x, y, d).
//   * eval_nn_error: mean over query points (pairwise_sum order) of the
//     distance from transform * q to its nearest reference point.
#pragma once

#include <cmath>
#include <limits>
#include <stdexcept>

#include "orc_icp.hpp"

namespace orc {

// reloc.hpp:35-46
struct RelocProblem {
  std::vector<Vec3d> voxel_centers;
  std::vector<double> reference_values;
  Image<Complex> query_depth;
  Intrinsics intrinsics;
  double mu = 0.1;
};

template <typename F>
void observed_voxels(const TsdfVolumeT<F>& v, std::vector<Vec3d>* centers, std::vector<double>* values) {
  const int nx = v.params.dims[0], ny = v.params.dims[1], nz = v.params.dims[2];
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        const std::size_t idx = v.index(i, j, k);
        if (!(v.weight[idx] > 0.0)) continue;
        centers->push_back(v.voxel_position(i, j, k));
        values->push_back(real_part(v.tsdf[idx]));
      }
}

template <typename F>
void observed_voxels(const HashedVolumeT<F>& v, std::vector<Vec3d>* centers, std::vector<double>* values) {
  for (int b = 0; b < v.n_blocks(); ++b)
    for (int l = 0; l < kBlockVoxels; ++l) {
      const std::size_t idx = static_cast<std::size_t>(b) * kBlockVoxels + l;
      if (!(v.weight[idx] > 0.0)) continue;
      const int i = v.coords[3 * b] * 8 + (l & 7);
      const int j = v.coords[3 * b + 1] * 8 + ((l >> 3) & 7);
      const int k = v.coords[3 * b + 2] * 8 + (l >> 6);
      centers->push_back(v.voxel_position(i, j, k));
      values->push_back(real_part(v.tsdf[idx]));
    }
}

// RelocProblem(reference, query, k) (reloc.hpp:44-45; builder-defined body)
template <typename V>
RelocProblem make_reloc_problem(const V& reference, const Image<double>& query, const Intrinsics& k) {
  RelocProblem p;
  observed_voxels(reference, &p.voxel_centers, &p.reference_values);
  if (p.voxel_centers.empty()) throw std::invalid_argument("RelocProblem: reference has no observed voxels");
  p.query_depth = complex_depth(query);
  p.intrinsics = k;
  p.mu = vol_mu(reference);
  return p;
}

// reloc.hpp:48-69 (the reference's own body).  `overlap` (optional) receives
// the number of mutually observed voxels.
template <typename S>
S reloc_energy(const RelocProblem& problem, const PoseT<S>& query_pose, long* overlap_out = nullptr) {
  const PoseT<S> world_to_camera = query_pose.inverse();
  const Vec3<S> camera_center = query_pose.translation;
  std::vector<S> terms(problem.voxel_centers.size(), S(0.0));
  long overlap = 0;
#pragma omp parallel for schedule(static) reduction(+ : overlap)
  for (std::ptrdiff_t i = 0; i < static_cast<std::ptrdiff_t>(problem.voxel_centers.size()); ++i) {
    const Vec3d& c = problem.voxel_centers[i];
    const Vec3<S> p{S(c[0]), S(c[1]), S(c[2])};
    const std::optional<S> measured =
        measured_tsdf(problem.query_depth, world_to_camera, problem.intrinsics, problem.mu, p, camera_center);
    if (!measured) continue;
    const S diff = *measured - S(problem.reference_values[i]);
    terms[i] = diff * diff;
    ++overlap;
  }
  if (overlap_out) *overlap_out = overlap;
  if (overlap == 0) throw std::runtime_error("relocalization energy: no overlapping voxels");
  return pairwise_sum(terms);
}

// reloc.hpp:71-80 — derivatives in the twist applied on top of `pose`
// (left increment, se3.hpp:116-119), evaluated at zero: 6 Complex passes /
// 21 Bicomplex passes (diff.hpp:46-72).
inline double reloc_loss(const RelocProblem& problem, const Pose& pose) { return reloc_energy<double>(problem, pose); }
inline Vec6<double> reloc_gradient(const RelocProblem& problem, const Pose& pose, const StepSize& step = {}) {
  return csfd_gradient(
      [&](const auto& xi) {
        using S = typename std::decay_t<decltype(xi)>::value_type;
        return reloc_energy<S>(problem, apply_increment(xi, pose_cast<S>(pose)));
      },
      Vec6<double>{}, step);
}
inline Mat6d reloc_hessian(const RelocProblem& problem, const Pose& pose, const StepSize& step = {}) {
  return csfd_hessian(
      [&](const auto& xi) {
        using S = typename std::decay_t<decltype(xi)>::value_type;
        return reloc_energy<S>(problem, apply_increment(xi, pose_cast<S>(pose)));
      },
      Vec6<double>{}, step);
}

// reloc.hpp:82-114
enum class RelocMethod { kGradientDescent, kNewton };
struct RelocConfig {
  double switch_relative = 0.5;
  double switch_absolute = -1.0;
  int max_iterations = 50;
  double step_tolerance = 1e-6;
  LineSearchConfig line_search;
  StepSize step;
  // builder-defined safeguards
  double max_step = 0.05;
  double min_overlap_ratio = 0.9;
};
struct RelocResult {
  Pose pose;
  int iterations = 0;
  bool converged = false;
  double final_loss = 0.0;
  RelocMethod method = RelocMethod::kNewton;
  std::vector<double> losses;  // trace: loss after each iteration (TraceRow::loss)
  std::vector<double> gradient_norms;
};

inline Pose step_pose(const Pose& pose, const Vec6<double>& d) { return apply_increment(d, pose); }

// relocalize (reloc.hpp:116-124; builder-defined body).
// The overlap-restricted sum also decreases when the view slides off the
// model, so a trial keeping fewer than min_overlap_ratio x the current
// overlap counts as +inf, and directions are scaled to twist length
// max_step (steepest descent: exactly; Newton: at most).
inline RelocResult relocalize(const RelocProblem& problem, const Pose& initial, RelocMethod method,
                              const RelocConfig& cfg = {}) {
  RelocResult out;
  out.method = method;
  Pose pose = initial;
  long cur_ov = 0, trial_ov = 0;
  double loss = reloc_energy<double>(problem, pose, &cur_ov);
  const double threshold = cfg.switch_absolute >= 0.0 ? cfg.switch_absolute : cfg.switch_relative * loss;
  auto trial_loss = [&](const Vec6<double>& d) {
    long ov = 0;
    double e;
    try {
      e = reloc_energy<double>(problem, step_pose(pose, d), &ov);
    } catch (const std::runtime_error&) {
      return std::numeric_limits<double>::infinity();
    }
    trial_ov = ov;
    if (static_cast<double>(ov) < cfg.min_overlap_ratio * static_cast<double>(cur_ov))
      return std::numeric_limits<double>::infinity();
    return e;
  };
  for (int it = 0; it < cfg.max_iterations; ++it) {
    const Vec6<double> g = reloc_gradient(problem, pose, cfg.step);
    const double gn = norm6(g);
    Vec6<double> dir;
    const double sg = gn > 0.0 ? cfg.max_step / gn : 0.0;
    for (int i = 0; i < 6; ++i) dir[i] = -g[i] * sg;
    if (method == RelocMethod::kNewton && loss < threshold) {
      const Mat6d hm = reloc_hessian(problem, pose, cfg.step);
      double a[kNA];
      for (int r = 0; r < 6; ++r)
        for (int c = 0; c <= r; ++c) a[tri(r, c)] = hm[r][c];
      const Ldlt6<double> ldlt(a);
      if (ldlt.ok) {
        double ng[6], d[6];
        for (int i = 0; i < 6; ++i) ng[i] = -g[i];
        ldlt.solve(ng, d);
        bool finite = true;
        Vec6<double> nd;
        for (int i = 0; i < 6; ++i) {
          finite = finite && std::isfinite(d[i]);
          nd[i] = d[i];
        }
        if (finite && dot6(g, nd) < 0.0) {
          const double nn = norm6(nd);
          if (nn > cfg.max_step) {
            const double sn = cfg.max_step / nn;
            for (int i = 0; i < 6; ++i) nd[i] = nd[i] * sn;
          }
          dir = nd;
        }
      }
    }
    const double slope = dot6(g, dir);
    if (!(slope < 0.0)) {
      out.converged = gn == 0.0;
      break;
    }
    const LineSearchResult r = backtracking_search(
        [&](double alpha) {
          Vec6<double> d;
          for (int i = 0; i < 6; ++i) d[i] = alpha * dir[i];
          return trial_loss(d);
        },
        loss, slope, cfg.line_search);
    if (!r.ok) break;
    Vec6<double> step;
    for (int i = 0; i < 6; ++i) step[i] = r.alpha * dir[i];
    pose = step_pose(pose, step);
    loss = r.loss;
    cur_ov = trial_ov;
    ++out.iterations;
    out.losses.push_back(loss);
    out.gradient_norms.push_back(gn);
    if (norm6(step) < cfg.step_tolerance) {
      out.converged = true;
      break;
    }
  }
  out.pose = pose;
  out.final_loss = loss;
  return out;
}

// select_reference_frames (reloc.hpp:22-26; builder-defined body)
inline std::vector<std::size_t> select_reference_frames(const std::vector<Pose>& poses, const Pose& initial,
                                                        int count = 10) {
  std::vector<std::pair<double, std::size_t>> d;
  for (std::size_t i = 0; i < poses.size(); ++i) {
    const Vec3d diff = poses[i].translation - initial.translation;
    d.push_back({squared_norm(diff), i});
  }
  std::sort(d.begin(), d.end());
  std::vector<std::size_t> out;
  for (std::size_t i = 0; i < d.size() && static_cast<int>(i) < count; ++i) out.push_back(d[i].second);
  return out;
}

// depth_cloud (reloc.hpp:126-129; builder-defined body)
inline std::vector<Vec3d> depth_cloud(const Image<double>& depth, const Intrinsics& k, const Pose& camera_to_world,
                                      int stride = 1) {
  if (stride < 1) throw std::invalid_argument("depth_cloud: stride must be >= 1");
  std::vector<Vec3d> out;
  for (int y = 0; y < depth.height; y += stride)
    for (int x = 0; x < depth.width; x += stride) {
      const double d = depth.at(x, y);
      if (!depth_valid(d)) continue;
      out.push_back(camera_to_world * backproject(k, double(x), double(y), d));
    }
  return out;
}

// eval_nn_error (reloc.hpp:131-138; builder-defined body)
struct NnError {
  double mean = 0.0;
  bool outlier = false;
};
inline NnError eval_nn_error(const Pose& transform, const std::vector<Vec3d>& query,
                             const std::vector<Vec3d>& reference) {
  if (query.empty() || reference.empty()) throw std::invalid_argument("eval_nn_error: empty cloud");
  std::vector<double> dist(query.size());
#pragma omp parallel for schedule(static)
  for (std::ptrdiff_t i = 0; i < static_cast<std::ptrdiff_t>(query.size()); ++i) {
    const Vec3d q = transform * query[i];
    double best = std::numeric_limits<double>::infinity();
    for (const Vec3d& r : reference) {
      const Vec3d dd = q - r;
      const double s = squared_norm(dd);
      if (s < best) best = s;
    }
    dist[i] = std::sqrt(best);
  }
  NnError e;
  e.mean = pairwise_sum(dist) / static_cast<double>(query.size());
  e.outlier = e.mean > 0.1;
  return e;
}

}  // namespace orc
