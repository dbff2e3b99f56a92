// ORACLE — TEST INFRASTRUCTURE ONLY (see orc_core.hpp header).
//
// Restates proj/include/csf/icp.hpp:27-133, proj/src/icp.cpp:15-244 and
// proj/include/csf/descent.hpp:16-144.  Eigen::LDLT<Mat6d> is restated as
// Ldlt6 (diagonal pivoting, unit-lower L, D on the diagonal) with a fixed,
// stated operation order — Eigen's internal order cannot be verified here
// (SURVEY F3 / H1), so this order IS the contract the sm_100a solver copies.
//
// Reduction order of the normal equations: the reference sums sequentially
// (icp.cpp:19-27).  The canonical order used by the tracker (and by the GPU)
// is "slot-tiled" (tiled_normal_equations below: tiles of the strided slot
// grid, 32 correspondence streams per tile combined by a fixed butterfly,
// tiles summed in groups of kGroup).  The correspondence-list form
// (normal_equations, csf_linearized_step) cuts the list into tiles of kTile
// entries summed sequentially, the tiles in groups of kGroup.
// normal_equations(..., sequential=true) keeps the reference's literal order
// for the KAT pins.
#pragma once

#include <functional>

#include "orc_tsdf.hpp"

namespace orc {

constexpr int kTile = 256;
constexpr int kGroup = 16;

// icp.hpp:27-31
struct Correspondence {
  Vec3d vertex, model_vertex, model_normal;
};

// icp.hpp:33-53, descent.hpp:16-21
enum class IcpSolver { kLinearized = 0, kNewton = 1, kGradientDescent = 2, kConjugateGradient = 3 };
struct LineSearchConfig {
  double initial_step = 1.0, shrink = 0.5, sufficient_decrease = 1e-4;
  int max_backtracks = 25;
};
struct IcpConfig {
  IcpSolver solver = IcpSolver::kNewton;
  double d_max = 0.1;
  double theta_max_deg = 30.0;
  int levels = 3;
  std::array<int, 3> level_iterations = {10, 5, 4};
  std::array<int, 3> level_pixel_stride = {1, 1, 2};
  double step_tolerance = 1e-6;
  double levenberg_lambda0 = 1e-6;
  int ncg_restart = 6;
  LineSearchConfig line_search;
  StepSize step;
};

// cos of the normal gate, evaluated with the deterministic cosine so host
// and device agree (icp.cpp:97).
inline double gate_cos(double theta_max_deg) { return m_cos(theta_max_deg * M_PI / 180.0); }

// One association with its pixel bookkeeping (x, y measured; u, v model).
struct CorrIndex {
  int x, y, u, v;
};

// icp.cpp:89-126
inline std::vector<Correspondence> associate(const SurfaceMaps<double>& measured,
                                             const SurfaceMaps<double>& predicted, const Pose& camera_to_world,
                                             const Pose& predicted_camera_to_world, const Intrinsics& k,
                                             const IcpConfig& cfg, int pixel_stride = 1,
                                             std::vector<CorrIndex>* index = nullptr) {
  std::vector<Correspondence> corrs;
  const Pose world_to_predicted = predicted_camera_to_world.inverse();
  const double cos_max = gate_cos(cfg.theta_max_deg);
  const int stride = std::max(1, pixel_stride);
  for (int y = 0; y < measured.vertices.height; y += stride)
    for (int x = 0; x < measured.vertices.width; x += stride) {
      const Vec3d& vertex = measured.vertices.at(x, y);
      const Vec3d& normal = measured.normals.at(x, y);
      if (!vertex_valid(vertex) || !normal_valid(normal)) continue;
      const Vec3d world = camera_to_world * vertex;
      const Vec3d in_predicted = world_to_predicted * world;
      if (in_predicted.z() <= 0.0) continue;
      const auto uv = project(k, in_predicted);
      const int u = static_cast<int>(std::lround(uv[0]));
      const int v = static_cast<int>(std::lround(uv[1]));
      if (!predicted.vertices.in_bounds(u, v)) continue;
      const Vec3d& model_normal = predicted.normals.at(u, v);
      if (!normal_valid(model_normal)) continue;
      const Vec3d& model_vertex = predicted.vertices.at(u, v);
      if (norm(world - model_vertex) > cfg.d_max) continue;
      const Vec3d world_normal = camera_to_world.rotation * normal;
      if (dot(world_normal, model_normal) < cos_max) continue;
      corrs.push_back({vertex, model_vertex, model_normal});
      if (index) index->push_back({x, y, u, v});
    }
  return corrs;
}

// icp.hpp:70-85
template <typename S>
S icp_energy(const std::vector<Correspondence>& corrs, const Vec6<S>& xi, const Pose& base) {
  const PoseT<S> pose = exp_map(xi) * pose_cast<S>(base);
  std::vector<S> terms(corrs.size(), S(0.0));
#pragma omp parallel for schedule(static)
  for (std::ptrdiff_t i = 0; i < static_cast<std::ptrdiff_t>(corrs.size()); ++i) {
    const Correspondence& c = corrs[i];
    const Vec3<S> v(S(c.vertex[0]), S(c.vertex[1]), S(c.vertex[2]));
    const Vec3<S> mv(S(c.model_vertex[0]), S(c.model_vertex[1]), S(c.model_vertex[2]));
    const Vec3<S> mn(S(c.model_normal[0]), S(c.model_normal[1]), S(c.model_normal[2]));
    const Vec3<S> moved = pose * v;
    const Vec3<S> offset = moved - mv;
    const S r = dot(offset, mn);
    terms[i] = r * r;
  }
  return pairwise_sum(terms);
}

// icp.cpp:128-144
inline double icp_loss(const std::vector<Correspondence>& corrs, const Pose& base) {
  Vec6<double> z{};
  return icp_energy(corrs, z, base);
}
inline Vec6<double> icp_gradient(const std::vector<Correspondence>& corrs, const Pose& base, const StepSize& step = {}) {
  return csfd_gradient([&](const auto& xi) { return icp_energy(corrs, xi, base); }, Vec6<double>{}, step);
}
inline Mat6d icp_hessian(const std::vector<Correspondence>& corrs, const Pose& base, const StepSize& step = {}) {
  return csfd_hessian([&](const auto& xi) { return icp_energy(corrs, xi, base); }, Vec6<double>{}, step);
}

// ---------------------------------------------------------------------------
// Normal equations.  28 accumulators per scalar: A lower triangle row-major
// (r >= c, index r*(r+1)/2 + c), then b[0..5], then the real term count.
// ---------------------------------------------------------------------------
constexpr int kNA = 21;
inline int tri(int r, int c) { return r * (r + 1) / 2 + c; }

template <typename S>
struct NormalEq {
  S a[kNA];
  S b[6];
  NormalEq() {
    for (auto& x : a) x = S(0.0);
    for (auto& x : b) x = S(0.0);
  }
};

// Per-correspondence Jacobian row and residual — icp.cpp:20-24.
template <typename S>
void jacobian_row(const Vec3<S>& vertex, const Vec3<S>& mv, const Vec3<S>& mn, const PoseT<S>& base, S j[6], S* r) {
  const Vec3<S> p = base * vertex;
  *r = dot(p - mv, mn);
  const Vec3<S> pn = cross(p, mn);
  j[0] = mn[0]; j[1] = mn[1]; j[2] = mn[2];
  j[3] = pn[0]; j[4] = pn[1]; j[5] = pn[2];
}

template <typename S>
void accumulate_row(NormalEq<S>& ne, const S j[6], const S& r) {
  for (int rr = 0; rr < 6; ++rr)
    for (int c = 0; c <= rr; ++c) ne.a[tri(rr, c)] = ne.a[tri(rr, c)] + j[rr] * j[c];
  for (int i = 0; i < 6; ++i) ne.b[i] = ne.b[i] + j[i] * r;
}

template <typename S>
void add_into(NormalEq<S>& dst, const NormalEq<S>& src) {
  for (int q = 0; q < kNA; ++q) dst.a[q] = dst.a[q] + src.a[q];
  for (int i = 0; i < 6; ++i) dst.b[i] = dst.b[i] + src.b[i];
}

// Reference order (sequential) or canonical slot-tiled order over the
// correspondence list (every correspondence is one slot).
inline NormalEq<double> normal_equations(const std::vector<Correspondence>& corrs, const Pose& base,
                                         bool sequential) {
  NormalEq<double> total;
  NormalEq<double> tile, group;
  const std::size_t n_tiles = (corrs.size() + kTile - 1) / kTile;
  for (std::size_t i = 0; i < corrs.size(); ++i) {
    double j[6], r;
    const Correspondence& c = corrs[i];
    jacobian_row<double>(c.vertex, c.model_vertex, c.model_normal, base, j, &r);
    accumulate_row(sequential ? total : tile, j, r);
    if (!sequential && ((i + 1) % kTile == 0 || i + 1 == corrs.size())) {
      const std::size_t t = i / kTile;
      add_into(group, tile);
      tile = NormalEq<double>();
      if ((t + 1) % kGroup == 0 || t + 1 == n_tiles) {
        add_into(total, group);
        group = NormalEq<double>();
      }
    }
  }
  return total;
}

// ---------------------------------------------------------------------------
// Ldlt6 — restates Eigen::LDLT<Mat6d> (diagonal pivoting) with fixed order.
// ---------------------------------------------------------------------------
template <typename S>
struct Ldlt6 {
  S m[6][6];
  int transp[6];
  bool ok = true;

  explicit Ldlt6(const S a_lower[kNA]) {
    for (int r = 0; r < 6; ++r)
      for (int c = 0; c < 6; ++c) m[r][c] = r >= c ? a_lower[tri(r, c)] : a_lower[tri(c, r)];
    factor();
  }

  static double absre(const S& x) { return std::fabs(real_part(x)); }

  void factor() {
    S temp[6];
    for (int k = 0; k < 6; ++k) {
      int piv = k;
      double best = absre(m[k][k]);
      for (int i = k + 1; i < 6; ++i)
        if (absre(m[i][i]) > best) {
          best = absre(m[i][i]);
          piv = i;
        }
      transp[k] = piv;
      if (piv != k) {
        for (int j = 0; j < k; ++j) std::swap(m[k][j], m[piv][j]);
        for (int i = piv + 1; i < 6; ++i) std::swap(m[i][k], m[i][piv]);
        std::swap(m[k][k], m[piv][piv]);
        for (int i = k + 1; i < piv; ++i) {
          const S tmp = m[i][k];
          m[i][k] = m[piv][i];
          m[piv][i] = tmp;
        }
      }
      if (k > 0) {
        for (int j = 0; j < k; ++j) temp[j] = m[j][j] * m[k][j];
        S s = m[k][0] * temp[0];
        for (int j = 1; j < k; ++j) s = s + m[k][j] * temp[j];
        m[k][k] = m[k][k] - s;
        for (int i = k + 1; i < 6; ++i) {
          S si = m[i][0] * temp[0];
          for (int j = 1; j < k; ++j) si = si + m[i][j] * temp[j];
          m[i][k] = m[i][k] - si;
        }
      }
      const S akk = m[k][k];
      const bool pivot_valid = absre(akk) > 0.0;
      if (k == 0 && !pivot_valid) {
        ok = false;
        for (int j = 0; j < 6; ++j) transp[j] = j;
        break;
      }
      if (k < 5) {
        if (pivot_valid) {
          for (int i = k + 1; i < 6; ++i) m[i][k] = m[i][k] / akk;
        } else {
          for (int i = k + 1; i < 6; ++i) ok = ok && real_part(m[i][k]) == 0.0;
        }
      }
    }
  }

  void solve(const S rhs[6], S dst[6]) const {
    for (int i = 0; i < 6; ++i) dst[i] = rhs[i];
    for (int k = 0; k < 6; ++k) std::swap(dst[k], dst[transp[k]]);
    for (int i = 0; i < 6; ++i)
      for (int j = i + 1; j < 6; ++j) dst[j] = dst[j] - dst[i] * m[j][i];
    const double tol = std::numeric_limits<double>::min();
    for (int i = 0; i < 6; ++i) {
      if (absre(m[i][i]) > tol)
        dst[i] = dst[i] / m[i][i];
      else
        dst[i] = S(0.0);
    }
    for (int i = 5; i >= 0; --i) {
      if (i < 5) {
        S s = m[i + 1][i] * dst[i + 1];
        for (int j = i + 2; j < 6; ++j) s = s + m[j][i] * dst[j];
        dst[i] = dst[i] - s;
      }
    }
    for (int k = 5; k >= 0; --k) std::swap(dst[k], dst[transp[k]]);
  }
};

// Canonical tiling of the tracker's normal equations (builder-defined,
// SURVEY H3; the device's k_icp_level / k_icp_reduce2, icp.cu):
//   * the strided slot grid (row-major) is cut into at most kLevelMaxTiles
//     tiles of T = 32 * ceil(n_slots / (32 * kLevelMaxTiles)) slots;
//   * inside a tile the correspondences, in slot order, are dealt to 32
//     streams (entry e of the tile to stream e mod 32), each summed
//     sequentially from 0;
//   * the 32 streams are combined by the fixed halving tree
//     s[l] = s[l] + s[l + off] for off = 16, 8, 4, 2, 1 (l < off), i.e. lane
//     0 of an xor butterfly;
//   * tile partials are summed from 0 in tile order within groups of kGroup
//     tiles, group totals from 0 in group order.
constexpr int kLevelMaxTiles = 148;
inline int icp_tile_slots(long long n_slots) {
  const long long u = (n_slots + 32LL * kLevelMaxTiles - 1) / (32LL * kLevelMaxTiles);
  return static_cast<int>(32 * (u > 0 ? u : 1));
}

template <typename S>
NormalEq<S> tiled_normal_equations(const std::vector<CorrIndex>& idx, int width, int height, int stride,
                                   const SurfaceMaps<S>& measured, const SurfaceMaps<S>& predicted,
                                   const PoseT<S>& base) {
  const int nxs = (width + stride - 1) / stride;
  const int nys = (height + stride - 1) / stride;
  const long long n_slots = static_cast<long long>(nxs) * nys;
  const int T = icp_tile_slots(n_slots);
  const int n_tiles = static_cast<int>((n_slots + T - 1) / T);
  std::vector<NormalEq<S>> partial(n_tiles);
  std::vector<NormalEq<S>> streams(32);
  int cur = -1, entries = 0;
  auto finish = [&]() {
    if (cur < 0) return;
    for (int off = 16; off > 0; off >>= 1)
      for (int l = 0; l < off; ++l) add_into(streams[l], streams[l + off]);
    partial[cur] = streams[0];
    for (auto& st : streams) st = NormalEq<S>();
  };
  for (const CorrIndex& c : idx) {  // scan order == slot order
    const long long slot = static_cast<long long>(c.y / stride) * nxs + c.x / stride;
    const int t = static_cast<int>(slot / T);
    if (t != cur) {
      finish();
      cur = t;
      entries = 0;
    }
    S j[6], r;
    jacobian_row<S>(measured.vertices.at(c.x, c.y), predicted.vertices.at(c.u, c.v), predicted.normals.at(c.u, c.v),
                    base, j, &r);
    accumulate_row(streams[entries % 32], j, r);
    ++entries;
  }
  finish();
  NormalEq<S> total, group;
  for (int t = 0; t < n_tiles; ++t) {
    add_into(group, partial[t]);
    if ((t + 1) % kGroup == 0 || t + 1 == n_tiles) {
      add_into(total, group);
      group = NormalEq<S>();
    }
  }
  return total;
}

// icp.cpp:146-153 (with the reduction order selectable)
inline Vec6<double> linearized_step(const std::vector<Correspondence>& corrs, const Pose& base,
                                    bool sequential = false) {
  const NormalEq<double> ne = normal_equations(corrs, base, sequential);
  double nb[6];
  for (int i = 0; i < 6; ++i) nb[i] = -ne.b[i];
  const Ldlt6<double> ldlt(ne.a);
  double d[6];
  ldlt.solve(nb, d);
  Vec6<double> out{};
  bool finite = true;
  for (int i = 0; i < 6; ++i) finite = finite && std::isfinite(d[i]);
  if (finite)
    for (int i = 0; i < 6; ++i) out[i] = d[i];
  return out;
}

// descent.hpp:23-52
struct LineSearchResult {
  double alpha = 0.0, loss = 0.0;
  int evaluations = 0;
  bool ok = false;
};
template <typename F>
LineSearchResult backtracking_search(F&& loss_at_step, double loss0, double slope, const LineSearchConfig& cfg) {
  LineSearchResult out;
  double alpha = cfg.initial_step;
  for (int k = 0; k < cfg.max_backtracks; ++k) {
    const double trial = loss_at_step(alpha);
    ++out.evaluations;
    if (trial <= loss0 + cfg.sufficient_decrease * alpha * slope) {
      out.alpha = alpha;
      out.loss = trial;
      out.ok = true;
      return out;
    }
    alpha *= cfg.shrink;
  }
  return out;
}

inline double dot6(const Vec6<double>& a, const Vec6<double>& b) {
  Vec6<double> p;
  for (int i = 0; i < 6; ++i) p[i] = a[i] * b[i];
  return sum6(p);
}

// descent.hpp:58-101
class GradientStepper {
 public:
  enum class Kind { kGradientDescent, kConjugateGradient };
  explicit GradientStepper(Kind kind, int restart_every = 6) : kind_(kind), restart_every_(restart_every) {}
  void reset() {
    have_previous_ = false;
    since_restart_ = 0;
  }
  Vec6<double> propose(const Vec6<double>& g) {
    Vec6<double> neg;
    for (int i = 0; i < 6; ++i) neg[i] = -g[i];
    if (kind_ == Kind::kGradientDescent) return neg;
    bool restart = !have_previous_ || since_restart_ >= restart_every_ || dot6(prev_g_, prev_g_) == 0.0;
    Vec6<double> direction = neg;
    if (!restart) {
      Vec6<double> diff;
      for (int i = 0; i < 6; ++i) diff[i] = g[i] - prev_g_[i];
      const double beta = std::max(0.0, dot6(g, diff) / dot6(prev_g_, prev_g_));
      for (int i = 0; i < 6; ++i) direction[i] = neg[i] + beta * prev_d_[i];
      if (dot6(g, direction) >= 0.0) {
        direction = neg;
        restart = true;
      }
    }
    if (restart) since_restart_ = 0;
    ++since_restart_;
    prev_g_ = g;
    prev_d_ = direction;
    have_previous_ = true;
    return direction;
  }

 private:
  Kind kind_;
  int restart_every_;
  int since_restart_ = 0;
  bool have_previous_ = false;
  Vec6<double> prev_g_{}, prev_d_{};
};

// descent.hpp:109-144
template <typename TrialLoss>
Vec6<double> levenberg_newton_step(const Vec6<double>& gradient, const Mat6d& hessian, double loss0,
                                   TrialLoss&& trial_loss, double& lambda, const LineSearchConfig& search,
                                   double* loss_after = nullptr, int max_attempts = 8) {
  for (int attempt = 0; attempt < max_attempts; ++attempt) {
    double a[kNA];
    for (int r = 0; r < 6; ++r)
      for (int c = 0; c <= r; ++c) a[tri(r, c)] = hessian[r][c] + lambda * (r == c ? 1.0 : 0.0);
    const Ldlt6<double> ldlt(a);
    if (ldlt.ok) {
      double ng[6], d[6];
      for (int i = 0; i < 6; ++i) ng[i] = -gradient[i];
      ldlt.solve(ng, d);
      bool finite = true;
      for (int i = 0; i < 6; ++i) finite = finite && std::isfinite(d[i]);
      if (finite) {
        Vec6<double> delta;
        for (int i = 0; i < 6; ++i) delta[i] = d[i];
        const double trial = trial_loss(delta);
        if (trial < loss0) {
          lambda = std::max(lambda * 0.1, 1e-12);
          if (loss_after) *loss_after = trial;
          return delta;
        }
      }
    }
    lambda *= 10.0;
  }
  const double slope = -dot6(gradient, gradient);
  if (slope < 0.0) {
    const LineSearchResult r = backtracking_search(
        [&](double a) {
          Vec6<double> d;
          for (int i = 0; i < 6; ++i) d[i] = -a * gradient[i];
          return trial_loss(d);
        },
        loss0, slope, search);
    if (r.ok) {
      if (loss_after) *loss_after = r.loss;
      Vec6<double> d;
      for (int i = 0; i < 6; ++i) d[i] = -r.alpha * gradient[i];
      return d;
    }
  }
  if (loss_after) *loss_after = loss0;
  return Vec6<double>{};
}

// icp.hpp:103-125
struct TraceRow {
  int iteration = 0;
  double loss = 0.0, gradient_norm = 0.0, translation_error = 0.0, rotation_error = 0.0;
};
struct TrackResult {
  Pose pose;
  int iterations = 0;
  bool converged = false;
  double final_loss = 0.0;
  int correspondences = 0;
};

struct StepOutcome {
  Vec6<double> delta{};
  double loss_after = 0.0;
  Vec6<double> gradient{};
};

// icp.cpp:169-244 — the reference's real tracker, every solver family.
// `canonical_order` switches the linearized solver's normal equations to the
// slot-tiled order (the GPU's); false keeps the literal sequential sum.
template <typename V>
TrackResult track_frame(const V& volume, const Image<double>& depth, const Pose& init, const Intrinsics& k,
                        const IcpConfig& cfg, std::vector<TraceRow>* trace = nullptr,
                        bool canonical_order = true) {
  TrackResult out;
  out.pose = init;
  const int levels = std::clamp(cfg.levels, 1, 3);
  const auto pyramid = build_depth_pyramid(bilateral_filter(depth), levels);
  Pose pose = init;
  double lambda = cfg.levenberg_lambda0;
  GradientStepper stepper(cfg.solver == IcpSolver::kConjugateGradient ? GradientStepper::Kind::kConjugateGradient
                                                                      : GradientStepper::Kind::kGradientDescent,
                          cfg.ncg_restart);
  int iteration = 0;
  for (int li = 0; li < levels; ++li) {
    const int level = levels - 1 - li;
    const Intrinsics kl = k.at_level(level);
    const SurfaceMaps<double> measured = measure_surface<double>(pyramid[level], kl);
    const Pose prediction_pose = pose;
    const SurfaceMaps<double> predicted = raycast<double>(volume, prediction_pose, kl);
    stepper.reset();
    for (int it = 0; it < cfg.level_iterations[li]; ++it) {
      std::vector<CorrIndex> idx;
      const int stride = std::max(1, cfg.level_pixel_stride[li]);
      const auto corrs = associate(measured, predicted, pose, prediction_pose, kl, cfg, stride, &idx);
      out.correspondences = static_cast<int>(corrs.size());
      if (corrs.size() < 12) break;
      StepOutcome s;
      if (cfg.solver == IcpSolver::kLinearized) {
        // canonical: slot-tiled over the strided pixel grid (the device order);
        // otherwise the reference's literal sequential sum (icp.cpp:19-27)
        const NormalEq<double> ne = canonical_order
                                        ? tiled_normal_equations<double>(idx, kl.width, kl.height, stride, measured,
                                                                         predicted, pose)
                                        : normal_equations(corrs, pose, true);
        for (int i = 0; i < 6; ++i) s.gradient[i] = 2.0 * ne.b[i];
        double nb[6], d[6];
        for (int i = 0; i < 6; ++i) nb[i] = -ne.b[i];
        const Ldlt6<double> ldlt(ne.a);
        ldlt.solve(nb, d);
        bool finite = true;
        for (int i = 0; i < 6; ++i) finite = finite && std::isfinite(d[i]);
        for (int i = 0; i < 6; ++i) s.delta[i] = finite ? d[i] : 0.0;
        s.loss_after = icp_energy(corrs, s.delta, pose);
      } else if (cfg.solver == IcpSolver::kNewton) {
        const double loss0 = icp_loss(corrs, pose);
        s.gradient = icp_gradient(corrs, pose, cfg.step);
        const Mat6d hess = icp_hessian(corrs, pose, cfg.step);
        s.loss_after = loss0;
        s.delta = levenberg_newton_step(
            s.gradient, hess, loss0, [&](const Vec6<double>& d) { return icp_energy(corrs, d, pose); }, lambda,
            cfg.line_search, &s.loss_after);
      } else {
        const double loss0 = icp_loss(corrs, pose);
        s.gradient = icp_gradient(corrs, pose, cfg.step);
        s.loss_after = loss0;
        const Vec6<double> dir = stepper.propose(s.gradient);
        const double slope = dot6(s.gradient, dir);
        if (slope < 0.0) {
          const LineSearchResult r = backtracking_search(
              [&](double alpha) {
                Vec6<double> d;
                for (int i = 0; i < 6; ++i) d[i] = alpha * dir[i];
                return icp_energy(corrs, d, pose);
              },
              loss0, slope, cfg.line_search);
          if (r.ok) {
            for (int i = 0; i < 6; ++i) s.delta[i] = r.alpha * dir[i];
            s.loss_after = r.loss;
          }
        }
      }
      pose = apply_increment(s.delta, pose);
      ++iteration;
      const double mean_loss = s.loss_after / static_cast<double>(corrs.size());
      out.final_loss = mean_loss;
      if (trace) {
        TraceRow row;
        row.iteration = iteration;
        row.loss = mean_loss;
        row.gradient_norm = norm6(s.gradient);
        row.translation_error = std::nan("");
        row.rotation_error = std::nan("");
        trace->push_back(row);
      }
      if (norm6(s.delta) < cfg.step_tolerance) {
        if (level == 0) out.converged = true;
        break;
      }
    }
  }
  out.pose = pose;
  out.iterations = iteration;
  return out;
}

}  // namespace orc
