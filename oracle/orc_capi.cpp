// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points of the CPU oracle for tests/ (ctypes), the smoke
// check and bench.py's CPU-baseline leg.  The POD structs are the product's
// (include/csf_b200.h) so both sides are driven with the same descriptors;
// nothing here links the product library.
#include <chrono>
#include <cmath>
#include <limits>
#include <cstring>
#include <memory>
#include <string>

#include "../include/csf_b200.h"
#include "orc_pipeline.hpp"
#include "orc_reloc.hpp"
#include "orc_surfel.hpp"

using namespace orc;

namespace {

thread_local std::string g_err;

int guard(const std::function<void()>& fn) {
  try {
    fn();
    return CSF_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return CSF_EINVAL;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return CSF_EDOMAIN;
  } catch (const std::exception& e) {
    g_err = e.what();
    return CSF_ERUNTIME;
  }
}

Intrinsics to_intr(const csf_intrinsics& k) {
  Intrinsics o;
  o.fx = k.fx; o.fy = k.fy; o.cx = k.cx; o.cy = k.cy;
  o.width = k.width; o.height = k.height; o.depth_scale = k.depth_scale;
  return o;
}
IcpConfig to_icp(const csf_icp_cfg& c) {
  IcpConfig o;
  o.solver = static_cast<IcpSolver>(c.solver);
  o.d_max = c.d_max;
  o.theta_max_deg = c.theta_max_deg;
  o.levels = c.levels;
  for (int i = 0; i < 3; ++i) {
    o.level_iterations[i] = c.level_iterations[i];
    o.level_pixel_stride[i] = c.level_pixel_stride[i];
  }
  o.step_tolerance = c.step_tolerance;
  o.levenberg_lambda0 = c.levenberg_lambda0;
  o.ncg_restart = c.ncg_restart;
  o.step = StepSize(c.h);
  return o;
}
VolumeParams to_vp(const csf_volume_params& p) {
  VolumeParams o;
  for (int i = 0; i < 3; ++i) o.dims[i] = p.dims[i];
  o.voxel_size = p.voxel_size;
  o.origin = Vec3d(p.origin[0], p.origin[1], p.origin[2]);
  o.mu = p.mu;
  o.weight_cap = p.weight_cap;
  return o;
}
HashParams to_hp(const csf_hash_params& p) {
  HashParams o;
  o.voxel_size = p.voxel_size;
  o.origin = Vec3d(p.origin[0], p.origin[1], p.origin[2]);
  o.mu = p.mu;
  o.weight_cap = p.weight_cap;
  o.bucket_bits = p.bucket_bits;
  o.max_blocks = p.max_blocks;
  return o;
}
RaycastConfig to_rc(const csf_raycast_cfg* c) {
  RaycastConfig o;
  if (c) {
    o.near_clip = c->near_clip;
    o.far_clip = c->far_clip;
    o.step_fraction = c->step_fraction;
  }
  return o;
}

template <int D> using FT = std::conditional_t<D == 0, double, Lifted<D>>;

template <int D> FT<D> load_s(const double* p) {
  if constexpr (D == 0) {
    return p[0];
  } else {
    Lifted<D> o(p[0]);
    for (int d = 0; d < D; ++d) o.im[d] = p[1 + d];
    return o;
  }
}
template <int D> void store_s(double* p, const FT<D>& v) {
  if constexpr (D == 0) {
    p[0] = v;
  } else {
    p[0] = v.re;
    for (int d = 0; d < D; ++d) p[1 + d] = v.im[d];
  }
}
template <int D> PoseT<FT<D>> load_pose(const double* p) {
  PoseT<FT<D>> o;
  for (int e = 0; e < 9; ++e) o.rotation(e / 3, e % 3) = load_s<D>(p + e * (1 + D));
  for (int e = 0; e < 3; ++e) o.translation[e] = load_s<D>(p + (9 + e) * (1 + D));
  return o;
}
template <int D> IntrinsicsT<FT<D>> load_intr(const double* p, int w, int h) {
  IntrinsicsT<FT<D>> k;
  k.fx = load_s<D>(p);
  k.fy = load_s<D>(p + (1 + D));
  k.cx = load_s<D>(p + 2 * (1 + D));
  k.cy = load_s<D>(p + 3 * (1 + D));
  k.width = w;
  k.height = h;
  return k;
}

struct VolBase {
  virtual ~VolBase() = default;
  virtual int channels() const = 0;
  virtual void fuse(const Image<double>& depth, const double* pose, const double* intr, int* n_visible) = 0;
  // lifted depth [h][w][1+D]: the reference's Image<Complex> depth (tsdf.hpp:144-145)
  virtual void fuse_lifted(const double* depth, int w, int h, const double* pose, const double* intr,
                           int* n_visible) = 0;
  virtual void raycast(const double* pose, const double* intr, int w, int h, const RaycastConfig& rc, double* vert,
                       double* norm) = 0;
  virtual long long voxels() const = 0;
  virtual void download(double* field, double* weight) const = 0;
  virtual void upload(const double* field, const double* weight) = 0;
  virtual int blocks() const = 0;
  virtual void hash_tables(int32_t* heads, uint64_t* keys, int32_t* next, int32_t* coords) const = 0;
  virtual TrackResult track(const Image<double>& depth, const Pose& init, const Intrinsics& k, const IcpConfig& cfg,
                            bool canonical, std::vector<TraceRow>* trace = nullptr) const = 0;
  virtual void view_scores(const double* poses, int n, const Intrinsics& k, double w0, double beta, double h,
                           double* scores, double* grads) const = 0;
  virtual void sample_points(const double* pts, int n, int grad, double* out, int32_t* valid) const = 0;
  virtual RelocProblem reloc_problem(const Image<double>& query, const Intrinsics& k) const = 0;
};

template <int D, bool H>
struct Vol : VolBase {
  using F = FT<D>;
  using V = std::conditional_t<H, HashedVolumeT<F>, TsdfVolumeT<F>>;
  V vol;
  template <typename P> explicit Vol(const P& p) : vol(p) {}
  int channels() const override { return D; }
  void fuse(const Image<double>& depth, const double* pose, const double* intr, int* n_visible) override {
    const PoseT<F> c2w = load_pose<D>(pose);
    const IntrinsicsT<F> k = load_intr<D>(intr, depth.width, depth.height);
    if constexpr (H) {
      Intrinsics kr = real_intrinsics(k);
      AllocStats st;
      const auto vis = allocate_band(vol, depth, kr, real_pose(c2w), &st);
      surface_update_blocks(vol, vis, depth, c2w, k);
      if (n_visible) *n_visible = st.touched;
    } else {
      surface_update(vol, depth, c2w, k);
      if (n_visible) *n_visible = 0;
    }
  }
  void fuse_lifted(const double* depth, int w, int h, const double* pose, const double* intr, int* n_visible) override {
    Image<F> dl(w, h, F(0.0));
    Image<double> dr(w, h, 0.0);
    for (int i = 0; i < w * h; ++i) {
      dl.data[i] = load_s<D>(depth + static_cast<std::size_t>(i) * (1 + D));
      dr.data[i] = depth[static_cast<std::size_t>(i) * (1 + D)];
    }
    const PoseT<F> c2w = load_pose<D>(pose);
    const IntrinsicsT<F> k = load_intr<D>(intr, w, h);
    if constexpr (H) {
      Intrinsics kr = real_intrinsics(k);
      AllocStats st;
      const auto vis = allocate_band(vol, dr, kr, real_pose(c2w), &st);
      surface_update_blocks(vol, vis, dl, c2w, k);
      if (n_visible) *n_visible = st.touched;
    } else {
      surface_update(vol, dl, c2w, k);
      if (n_visible) *n_visible = 0;
    }
  }
  void raycast(const double* pose, const double* intr, int w, int h, const RaycastConfig& rc, double* vert,
               double* norm) override {
    const PoseT<F> c2w = load_pose<D>(pose);
    const IntrinsicsT<F> k = load_intr<D>(intr, w, h);
    const SurfaceMaps<F> m = orc::raycast<F>(vol, c2w, k, rc);
    for (std::size_t i = 0; i < m.vertices.data.size(); ++i)
      for (int c = 0; c < 3; ++c) {
        store_s<D>(vert + (i * 3 + c) * (1 + D), m.vertices.data[i][c]);
        store_s<D>(norm + (i * 3 + c) * (1 + D), m.normals.data[i][c]);
      }
  }
  long long voxels() const override { return static_cast<long long>(vol.tsdf.size()); }
  void download(double* field, double* weight) const override {
    for (std::size_t i = 0; i < vol.tsdf.size(); ++i) {
      store_s<D>(field + i * (1 + D), vol.tsdf[i]);
      weight[i] = vol.weight[i];
    }
  }
  void upload(const double* field, const double* weight) override {
    for (std::size_t i = 0; i < vol.tsdf.size(); ++i) {
      vol.tsdf[i] = load_s<D>(field + i * (1 + D));
      vol.weight[i] = weight[i];
    }
  }
  int blocks() const override {
    if constexpr (H) return vol.n_blocks();
    return 0;
  }
  void hash_tables(int32_t* heads, uint64_t* keys, int32_t* next, int32_t* coords) const override {
    if constexpr (H) {
      if (heads) std::memcpy(heads, vol.heads.data(), sizeof(int32_t) * vol.heads.size());
      if (keys) std::memcpy(keys, vol.keys.data(), sizeof(uint64_t) * vol.keys.size());
      if (next) std::memcpy(next, vol.next.data(), sizeof(int32_t) * vol.next.size());
      if (coords) std::memcpy(coords, vol.coords.data(), sizeof(int32_t) * vol.coords.size());
    }
  }
  TrackResult track(const Image<double>& depth, const Pose& init, const Intrinsics& k, const IcpConfig& cfg,
                    bool canonical, std::vector<TraceRow>* trace = nullptr) const override {
    return track_frame(vol, depth, init, k, cfg, trace, canonical);
  }
  RelocProblem reloc_problem(const Image<double>& query, const Intrinsics& k) const override {
    return make_reloc_problem(vol, query, k);
  }
  void sample_points(const double* pts, int n, int grad, double* out, int32_t* valid) const override {
    for (int i = 0; i < n; ++i) {
      Vec3<F> p;
      for (int c = 0; c < 3; ++c) p[c] = load_s<D>(pts + (3 * i + c) * (1 + D));
      if (!grad) {
        const auto f = sample_tsdf<F>(vol, p);
        valid[i] = f.has_value();
        if (f) store_s<D>(out + i * (1 + D), *f);
      } else {
        const auto g = sample_gradient<F>(vol, p);
        valid[i] = g.has_value();
        if (g)
          for (int c = 0; c < 3; ++c) store_s<D>(out + (3 * i + c) * (1 + D), (*g)[c]);
      }
    }
  }
  // config 5: one Lifted<6> pass per view over the volume's real field
  void view_scores(const double* poses, int n, const Intrinsics& k, double w0, double beta, double h, double* scores,
                   double* grads) const override {
    if constexpr (H && D == 6) {
      using S = Lifted<6>;
      for (int v = 0; v < n; ++v) {
        Vec6<S> xi;
        for (int i = 0; i < 6; ++i) {
          xi[i] = S(0.0);
          xi[i].im[i] = h;
        }
        Pose base;
        for (int e = 0; e < 9; ++e) base.rotation(e / 3, e % 3) = poses[12 * v + e];
        for (int e = 0; e < 3; ++e) base.translation[e] = poses[12 * v + 9 + e];
        const PoseT<S> view = exp_map(xi) * pose_cast<S>(base);
        const S sc = view_coverage_score<S>(vol, view, k, w0, beta);
        scores[v] = sc.re;
        if (grads)
          for (int d = 0; d < 6; ++d) grads[6 * v + d] = sc.im[d] / h;
      }
    } else {
      throw std::invalid_argument("view_scores: needs a hashed volume with 6 channels");
    }
  }
};

template <bool H, typename P> VolBase* make_vol(int D, const P& p) {
  switch (D) {
    case 0: return new Vol<0, H>(p);
    case 1: return new Vol<1, H>(p);
    case 2: return new Vol<2, H>(p);
    case 3: return new Vol<3, H>(p);
    case 4: return new Vol<4, H>(p);
    case 5: return new Vol<5, H>(p);
    case 6: return new Vol<6, H>(p);
    case 8: return new Vol<8, H>(p);
    case 10: return new Vol<10, H>(p);
    default: throw std::invalid_argument("oracle: unsupported channel count");
  }
}

Image<double> image_of(const double* d, int w, int h) {
  Image<double> im(w, h, 0.0);
  std::memcpy(im.data.data(), d, sizeof(double) * w * h);
  return im;
}

template <int D>
void measure_impl(const double* depth, int w, int h, const double* intr, double* vert, double* norm) {
  using S = FT<D>;
  Image<S> dimg(w, h, S(0.0));
  for (int i = 0; i < w * h; ++i) dimg.data[i] = load_s<D>(depth + i * (1 + D));
  const IntrinsicsT<S> k = load_intr<D>(intr, w, h);
  const auto m = measure_surface<S>(dimg, k);
  for (int i = 0; i < w * h; ++i)
    for (int c = 0; c < 3; ++c) {
      store_s<D>(vert + (i * 3 + c) * (1 + D), m.vertices.data[i][c]);
      store_s<D>(norm + (i * 3 + c) * (1 + D), m.normals.data[i][c]);
    }
}

}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

int orc_bilateral(const double* depth, int w, int h, double ss, double sr, int r, double* out) {
  return guard([&] {
    const auto o = bilateral_filter(image_of(depth, w, h), ss, sr, r);
    std::memcpy(out, o.data.data(), sizeof(double) * w * h);
  });
}

int orc_downsample(const double* depth, int w, int h, double sr, double* out) {
  return guard([&] {
    const auto o = downsample_depth(image_of(depth, w, h), sr);
    std::memcpy(out, o.data.data(), sizeof(double) * o.data.size());
  });
}

int orc_measure(const double* depth, int w, int h, const double* intr, int D, double* vert, double* norm) {
  return guard([&] {
    switch (D) {
      case 0: measure_impl<0>(depth, w, h, intr, vert, norm); break;
      case 1: measure_impl<1>(depth, w, h, intr, vert, norm); break;
      case 2: measure_impl<2>(depth, w, h, intr, vert, norm); break;
      case 3: measure_impl<3>(depth, w, h, intr, vert, norm); break;
      case 4: measure_impl<4>(depth, w, h, intr, vert, norm); break;
      default: throw std::invalid_argument("orc_measure: unsupported channel count");
    }
  });
}

int orc_volume_create_dense(const csf_volume_params* p, int D, void** out) {
  return guard([&] { *out = make_vol<false>(D, to_vp(*p)); });
}
int orc_volume_create_hashed(const csf_hash_params* p, int D, void** out) {
  return guard([&] { *out = make_vol<true>(D, to_hp(*p)); });
}
void orc_volume_destroy(void* v) { delete static_cast<VolBase*>(v); }
int orc_surface_update(void* v, const double* depth, int w, int h, const double* pose, const double* intr,
                       int* n_visible) {
  return guard([&] { static_cast<VolBase*>(v)->fuse(image_of(depth, w, h), pose, intr, n_visible); });
}
int orc_surface_update_lifted(void* v, const double* depth, int w, int h, const double* pose, const double* intr,
                              int* n_visible) {
  return guard([&] { static_cast<VolBase*>(v)->fuse_lifted(depth, w, h, pose, intr, n_visible); });
}
int orc_raycast(void* v, const double* pose, const double* intr, int w, int h, const csf_raycast_cfg* rc, double* vert,
                double* norm) {
  return guard([&] { static_cast<VolBase*>(v)->raycast(pose, intr, w, h, to_rc(rc), vert, norm); });
}
long long orc_volume_voxels(void* v) { return static_cast<VolBase*>(v)->voxels(); }
int orc_volume_download(void* v, double* field, double* weight) {
  return guard([&] { static_cast<VolBase*>(v)->download(field, weight); });
}
int orc_volume_upload(void* v, const double* field, const double* weight) {
  return guard([&] { static_cast<VolBase*>(v)->upload(field, weight); });
}
int orc_volume_block_count(void* v) { return static_cast<VolBase*>(v)->blocks(); }
int orc_volume_hash(void* v, int32_t* heads, uint64_t* keys, int32_t* next, int32_t* coords) {
  return guard([&] { static_cast<VolBase*>(v)->hash_tables(heads, keys, next, coords); });
}
int orc_track_frame(void* v, const double* depth, int w, int h, const double* init_pose, const csf_intrinsics* k,
                    const csf_icp_cfg* cfg, int canonical, double* out_pose, csf_track_result* res) {
  return guard([&] {
    Pose init;
    for (int e = 0; e < 9; ++e) init.rotation(e / 3, e % 3) = init_pose[e];
    for (int e = 0; e < 3; ++e) init.translation[e] = init_pose[9 + e];
    const TrackResult r =
        static_cast<VolBase*>(v)->track(image_of(depth, w, h), init, to_intr(*k), to_icp(*cfg), canonical != 0);
    for (int e = 0; e < 9; ++e) out_pose[e] = r.pose.rotation(e / 3, e % 3);
    for (int e = 0; e < 3; ++e) out_pose[9 + e] = r.pose.translation[e];
    if (res) {
      res->iterations = r.iterations;
      res->converged = r.converged;
      res->correspondences = r.correspondences;
      res->final_loss = r.final_loss;
    }
  });
}

// track_frame with the trace rows [cap][3] (iteration, loss, gradient norm).
int orc_track_frame_traced(void* v, const double* depth, int w, int h, const double* init_pose,
                           const csf_intrinsics* k, const csf_icp_cfg* cfg, double* out_pose, csf_track_result* res,
                           double* rows, int cap, int* n_rows) {
  return guard([&] {
    Pose init;
    for (int e = 0; e < 9; ++e) init.rotation(e / 3, e % 3) = init_pose[e];
    for (int e = 0; e < 3; ++e) init.translation[e] = init_pose[9 + e];
    std::vector<TraceRow> tr;
    const TrackResult r =
        static_cast<VolBase*>(v)->track(image_of(depth, w, h), init, to_intr(*k), to_icp(*cfg), true, &tr);
    for (int e = 0; e < 9; ++e) out_pose[e] = r.pose.rotation(e / 3, e % 3);
    for (int e = 0; e < 3; ++e) out_pose[9 + e] = r.pose.translation[e];
    if (res) {
      res->iterations = r.iterations;
      res->converged = r.converged;
      res->correspondences = r.correspondences;
      res->final_loss = r.final_loss;
    }
    *n_rows = static_cast<int>(tr.size());
    for (int i = 0; i < static_cast<int>(tr.size()) && i < cap; ++i) {
      rows[3 * i] = tr[i].iteration;
      rows[3 * i + 1] = tr[i].loss;
      rows[3 * i + 2] = tr[i].gradient_norm;
    }
  });
}

// Oracle synthetic workload (configs 1/2): depth [n][h][w] float32, gt [n][12].
int orc_workload(int config, int n_frames, int width, int height, float* depth, double* gt, csf_intrinsics* k) {
  return guard([&] {
    const Workload w = make_workload(config, n_frames, width, height);
    const std::size_t P = static_cast<std::size_t>(w.k.width) * w.k.height;
    for (int f = 0; f < n_frames; ++f) {
      for (std::size_t i = 0; i < P; ++i) depth[f * P + i] = static_cast<float>(w.frames[f].data[i]);
      for (int e = 0; e < 9; ++e) gt[12 * f + e] = w.gt[f].rotation(e / 3, e % 3);
      for (int e = 0; e < 3; ++e) gt[12 * f + 9 + e] = w.gt[f].translation[e];
    }
    if (k) {
      k->fx = w.k.fx; k->fy = w.k.fy; k->cx = w.k.cx; k->cy = w.k.cy;
      k->width = w.k.width; k->height = w.k.height; k->depth_scale = w.k.depth_scale;
    }
  });
}

// The CSFD frame-derivative run.  poses [n][12][1+D], stats [n][8]
// (iterations, correspondences, 0, blocks, visible, ...).  Returns wall
// seconds through *seconds (the CPU baseline's timed region).
}  // extern "C"

namespace {
PipelineConfig to_pipeline(const csf_pipeline_cfg* c) {
  PipelineConfig cfg;
  cfg.hashed = c->hashed != 0;
  cfg.dense = to_vp(c->dense);
  cfg.hash = to_hp(c->hash);
  cfg.k = to_intr(c->k);
  cfg.icp = to_icp(c->icp);
  cfg.rc = to_rc(&c->rc);
  cfg.h = StepSize(c->h).h;
  cfg.directions.assign(c->dirs, c->dirs + c->n_dirs);
  cfg.objective = static_cast<Objective>(c->objective);
  cfg.keyframe_interval = c->keyframe_interval;
  return cfg;
}
void to_frames(const PipelineConfig& cfg, const float* depth, const double* gt_in, int n_frames,
               std::vector<Image<double>>* frames, std::vector<Pose>* gt) {
  const std::size_t P = static_cast<std::size_t>(cfg.k.width) * cfg.k.height;
  for (int f = 0; f < n_frames; ++f) {
    Image<double> im(cfg.k.width, cfg.k.height, 0.0);
    for (std::size_t i = 0; i < P; ++i) im.data[i] = static_cast<double>(depth[f * P + i]);
    frames->push_back(std::move(im));
    Pose p;
    for (int e = 0; e < 9; ++e) p.rotation(e / 3, e % 3) = gt_in[12 * f + e];
    for (int e = 0; e < 3; ++e) p.translation[e] = gt_in[12 * f + 9 + e];
    gt->push_back(p);
  }
}
// The device's per-frame stats row (csf_b200.h csf_pipeline_result):
// iterations, correspondences, converged, blocks, visible, new blocks, fused voxels, 0.
template <typename R>
void write_stats(int n_frames, const R& r, int32_t* stats) {
  for (int f = 0; f < n_frames; ++f) {
    stats[8 * f] = r.iterations[f];
    stats[8 * f + 1] = r.correspondences[f];
    stats[8 * f + 2] = r.converged[f];
    stats[8 * f + 3] = r.blocks[f];
    stats[8 * f + 4] = r.visible[f];
    stats[8 * f + 5] = r.fresh[f];
    stats[8 * f + 6] = r.fused[f];
    stats[8 * f + 7] = 0;
  }
}

Pose pose12(const double* p) {
  Pose o;
  for (int e = 0; e < 9; ++e) o.rotation(e / 3, e % 3) = p[e];
  for (int e = 0; e < 3; ++e) o.translation[e] = p[9 + e];
  return o;
}
void store_pose12(const Pose& o, double* p) {
  for (int e = 0; e < 9; ++e) p[e] = o.rotation(e / 3, e % 3);
  for (int e = 0; e < 3; ++e) p[9 + e] = o.translation[e];
}
std::vector<Vec3d> cloud_of(const double* p, int n) {
  std::vector<Vec3d> o(n);
  for (int i = 0; i < n; ++i) o[i] = Vec3d(p[3 * i], p[3 * i + 1], p[3 * i + 2]);
  return o;
}
}  // namespace

// ---- surfels (orc_surfel.hpp) over F = FT<D>
struct SurfBase {
  virtual ~SurfBase() = default;
  virtual int channels() const = 0;
  virtual int count() const = 0;
  virtual void download(double* pos, double* nrm, double* rad, double* conf, int32_t* ts) const = 0;
  virtual void upload(int n, const double* pos, const double* nrm, const double* rad, const double* conf,
                      const int32_t* ts) = 0;
  virtual void update(const double* depth, int w, int h, const double* c2w, const Intrinsics& k, int frame,
                      const SurfelFusionConfig& cfg, int* merged, int* created) = 0;
  virtual void index_map(const double* c2w12, const Intrinsics& k, uint32_t* offsets, int32_t* entries,
                         int* n) const = 0;
  virtual void associate(const double* depth, int w, int h, const double* c2w, const Intrinsics& k,
                         const SurfelFusionConfig& cfg, int32_t* counts, int32_t* idx, double* wts, int cap,
                         int* total) const = 0;
  virtual void predict(const double* c2w12, const Intrinsics& k, double* V, double* N) const = 0;
};

template <int D>
struct Surf : SurfBase {
  using F = FT<D>;
  SurfelMapT<F> map;
  int channels() const override { return D; }
  int count() const override { return static_cast<int>(map.size()); }
  void download(double* pos, double* nrm, double* rad, double* conf, int32_t* ts) const override {
    for (std::size_t i = 0; i < map.size(); ++i) {
      const auto& s = map.surfels[i];
      for (int c = 0; c < 3; ++c) {
        if (pos) store_s<D>(pos + (3 * i + c) * (1 + D), s.position[c]);
        if (nrm) store_s<D>(nrm + (3 * i + c) * (1 + D), s.normal[c]);
      }
      if (rad) rad[i] = s.radius;
      if (conf) store_s<D>(conf + i * (1 + D), s.confidence);
      if (ts) ts[i] = s.timestamp;
    }
  }
  void upload(int n, const double* pos, const double* nrm, const double* rad, const double* conf,
              const int32_t* ts) override {
    map.surfels.assign(n, SurfelT<F>{});
    for (int i = 0; i < n; ++i) {
      auto& s = map.surfels[i];
      for (int c = 0; c < 3; ++c) {
        s.position[c] = load_s<D>(pos + (3 * i + c) * (1 + D));
        s.normal[c] = load_s<D>(nrm + (3 * i + c) * (1 + D));
      }
      s.radius = rad[i];
      s.confidence = load_s<D>(conf + i * (1 + D));
      s.timestamp = ts[i];
    }
  }
  Image<F> lifted_depth(const double* depth, int w, int h) const {
    Image<F> d(w, h, F(0.0));
    for (int i = 0; i < w * h; ++i) d.data[i] = load_s<D>(depth + static_cast<std::size_t>(i) * (1 + D));
    return d;
  }
  void update(const double* depth, int w, int h, const double* c2w, const Intrinsics& k, int frame,
              const SurfelFusionConfig& cfg, int* merged, int* created) override {
    Intrinsics kk = k;
    kk.width = w;
    kk.height = h;
    const auto st = update_surfels(map, lifted_depth(depth, w, h), load_pose<D>(c2w), kk, frame, cfg);
    *merged = st.merged_pixels;
    *created = st.created;
  }
  void index_map(const double* c2w12, const Intrinsics& k, uint32_t* offsets, int32_t* entries,
                 int* n) const override {
    Pose p;
    for (int e = 0; e < 9; ++e) p.rotation(e / 3, e % 3) = c2w12[e];
    for (int e = 0; e < 3; ++e) p.translation[e] = c2w12[9 + e];
    const IndexMap im = render_index_map(map, p, k);
    std::copy(im.offsets.begin(), im.offsets.end(), offsets);
    if (entries) std::copy(im.entries.begin(), im.entries.end(), entries);
    *n = static_cast<int>(im.entries.size());
  }
  void associate(const double* depth, int w, int h, const double* c2w, const Intrinsics& k,
                 const SurfelFusionConfig& cfg, int32_t* counts, int32_t* idx, double* wts, int cap,
                 int* total) const override {
    Intrinsics kk = k;
    kk.width = w;
    kk.height = h;
    const PoseT<F> pose = load_pose<D>(c2w);
    const SurfaceMaps<F> frame = measure_surface<F>(lifted_depth(depth, w, h), kk);
    const IndexMap im = render_index_map(map, real_pose(pose), kk);
    int t = 0;
    for (int y = 0; y < h; ++y)
      for (int x = 0; x < w; ++x) {
        auto slot = associate_one_to_many(x, y, frame, im, map, pose, cfg.thresholds);
        if (!cfg.one_to_many && slot.size() > 1) {
          std::size_t best = 0;
          for (std::size_t j = 1; j < slot.size(); ++j)
            if (real_part(slot[j].weight) > real_part(slot[best].weight)) best = j;
          slot = {slot[best]};
        }
        counts[y * w + x] = static_cast<int32_t>(slot.size());
        for (const auto& a : slot) {
          if (idx && t < cap) {
            idx[t] = a.index;
            store_s<D>(wts + static_cast<std::size_t>(t) * (1 + D), a.weight);
          }
          ++t;
        }
      }
    *total = t;
  }
  void predict(const double* c2w12, const Intrinsics& k, double* V, double* N) const override {
    Pose p;
    for (int e = 0; e < 9; ++e) p.rotation(e / 3, e % 3) = c2w12[e];
    for (int e = 0; e < 3; ++e) p.translation[e] = c2w12[9 + e];
    const SurfaceMaps<double> m = predict_maps(map, p, k);
    for (int i = 0; i < k.width * k.height; ++i)
      for (int c = 0; c < 3; ++c) {
        V[3 * i + c] = m.vertices.data[i][c];
        N[3 * i + c] = m.normals.data[i][c];
      }
  }
};

SurfelFusionConfig to_sfc(const csf_surfel_cfg* c) {
  SurfelFusionConfig o;
  if (c) {
    o.thresholds.depth = c->depth;
    o.thresholds.normal_deg = c->normal_deg;
    o.thresholds.distance = c->distance;
    o.thresholds.sigma = c->sigma;
    o.one_to_many = c->one_to_many != 0;
  }
  return o;
}

extern "C" {

int orc_surfels_create(int D, void** out) {
  return guard([&] {
    switch (D) {
      case 0: *out = static_cast<SurfBase*>(new Surf<0>()); break;
      case 1: *out = static_cast<SurfBase*>(new Surf<1>()); break;
      case 2: *out = static_cast<SurfBase*>(new Surf<2>()); break;
      case 6: *out = static_cast<SurfBase*>(new Surf<6>()); break;
      default: throw std::invalid_argument("orc_surfels_create: channels must be 0, 1, 2 or 6");
    }
  });
}
void orc_surfels_destroy(void* m) { delete static_cast<SurfBase*>(m); }
int orc_surfels_count(void* m) { return static_cast<SurfBase*>(m)->count(); }
int orc_surfels_download(void* m, double* pos, double* nrm, double* rad, double* conf, int32_t* ts) {
  return guard([&] { static_cast<SurfBase*>(m)->download(pos, nrm, rad, conf, ts); });
}
int orc_surfels_upload(void* m, int n, const double* pos, const double* nrm, const double* rad, const double* conf,
                       const int32_t* ts) {
  return guard([&] { static_cast<SurfBase*>(m)->upload(n, pos, nrm, rad, conf, ts); });
}
int orc_update_surfels(void* m, const double* depth, int w, int h, const double* c2w, const csf_intrinsics* k,
                       int frame, const csf_surfel_cfg* cfg, int* merged, int* created) {
  return guard([&] { static_cast<SurfBase*>(m)->update(depth, w, h, c2w, to_intr(*k), frame, to_sfc(cfg), merged,
                                                       created); });
}
int orc_render_index_map(void* m, const double* c2w12, const csf_intrinsics* k, uint32_t* offsets, int32_t* entries,
                         int* n) {
  return guard([&] { static_cast<SurfBase*>(m)->index_map(c2w12, to_intr(*k), offsets, entries, n); });
}
int orc_associate_surfels(void* m, const double* depth, int w, int h, const double* c2w, const csf_intrinsics* k,
                          const csf_surfel_cfg* cfg, int32_t* counts, int32_t* idx, double* wts, int cap, int* total) {
  return guard([&] { static_cast<SurfBase*>(m)->associate(depth, w, h, c2w, to_intr(*k), to_sfc(cfg), counts, idx,
                                                          wts, cap, total); });
}
int orc_predict_maps(void* m, const double* c2w12, const csf_intrinsics* k, double* V, double* N) {
  return guard([&] { static_cast<SurfBase*>(m)->predict(c2w12, to_intr(*k), V, N); });
}
double orc_sample_confidence(const csf_intrinsics* k, int x, int y) { return sample_confidence(to_intr(*k), x, y); }

// ---- relocalization (orc_reloc.hpp)
int orc_reloc_create(void* v, const double* depth, int w, int h, const csf_intrinsics* k, void** out) {
  return guard([&] {
    Intrinsics kk = to_intr(*k);
    kk.width = w;
    kk.height = h;
    *out = new RelocProblem(static_cast<VolBase*>(v)->reloc_problem(image_of(depth, w, h), kk));
  });
}
void orc_reloc_destroy(void* p) { delete static_cast<RelocProblem*>(p); }
int orc_reloc_info(void* p, int* n, double* mu, double* centers, double* values) {
  return guard([&] {
    const auto* r = static_cast<RelocProblem*>(p);
    *n = static_cast<int>(r->voxel_centers.size());
    *mu = r->mu;
    if (centers)
      for (int i = 0; i < *n; ++i)
        for (int c = 0; c < 3; ++c) centers[3 * i + c] = r->voxel_centers[i][c];
    if (values) std::memcpy(values, r->reference_values.data(), sizeof(double) * *n);
  });
}
// order 0: E; 1: + g (6 Complex passes); 2: + H (21 Bicomplex passes)
int orc_reloc_energy(void* p, const double* pose, int order, double h, double* E, double* g, double* H, long* overlap) {
  return guard([&] {
    const auto& r = *static_cast<RelocProblem*>(p);
    const Pose ps = pose12(pose);
    *E = reloc_energy<double>(r, ps, overlap);
    if (order >= 1) {
      const auto gg = reloc_gradient(r, ps, StepSize(h));
      for (int i = 0; i < 6; ++i) g[i] = gg[i];
    }
    if (order >= 2) {
      const auto hh = reloc_hessian(r, ps, StepSize(h));
      for (int i = 0; i < 6; ++i)
        for (int j = 0; j < 6; ++j) H[6 * i + j] = hh[i][j];
    }
  });
}
int orc_relocalize(void* p, const double* init, int method, const csf_reloc_cfg* cfg, double* out_pose,
                   csf_reloc_result* res, double* losses, double* gnorms) {
  return guard([&] {
    RelocConfig c;
    c.switch_relative = cfg->switch_relative;
    c.switch_absolute = cfg->switch_absolute;
    c.max_iterations = cfg->max_iterations;
    c.step_tolerance = cfg->step_tolerance;
    c.step = StepSize(cfg->h);
    c.line_search.initial_step = cfg->ls_initial_step;
    c.line_search.shrink = cfg->ls_shrink;
    c.line_search.sufficient_decrease = cfg->ls_sufficient_decrease;
    c.line_search.max_backtracks = cfg->ls_max_backtracks;
    c.max_step = cfg->max_step;
    c.min_overlap_ratio = cfg->min_overlap_ratio;
    const RelocResult r = relocalize(*static_cast<RelocProblem*>(p), pose12(init),
                                     method == CSF_RELOC_NEWTON ? RelocMethod::kNewton : RelocMethod::kGradientDescent, c);
    store_pose12(r.pose, out_pose);
    res->iterations = r.iterations;
    res->converged = r.converged;
    res->final_loss = r.final_loss;
    for (int i = 0; i < r.iterations; ++i) {
      if (losses) losses[i] = r.losses[i];
      if (gnorms) gnorms[i] = r.gradient_norms[i];
    }
  });
}
int orc_depth_cloud(const double* depth, int w, int h, const csf_intrinsics* k, const double* pose, int stride,
                    double* out, int* n) {
  return guard([&] {
    const auto c = depth_cloud(image_of(depth, w, h), to_intr(*k), pose12(pose), stride);
    *n = static_cast<int>(c.size());
    if (out)
      for (std::size_t i = 0; i < c.size(); ++i)
        for (int e = 0; e < 3; ++e) out[3 * i + e] = c[i][e];
  });
}
int orc_nn_error(const double* transform, const double* query, int nq, const double* ref, int nr, double* mean,
                 int* outlier) {
  return guard([&] {
    const NnError e = eval_nn_error(pose12(transform), cloud_of(query, nq), cloud_of(ref, nr));
    *mean = e.mean;
    *outlier = e.outlier;
  });
}

int orc_sample_points(void* v, const double* pts, int n, int grad, double* out, int32_t* valid) {
  return guard([&] { static_cast<VolBase*>(v)->sample_points(pts, n, grad, out, valid); });
}

// lifted != 0: depth is [h][w][1+D] (tsdf.hpp:97-102 takes Image<S> depth)
int orc_measured_points(const double* depth, int w, int h, const double* w2c, const double* intr, double mu,
                        const double* pts, const double* center, int n, int D, double* out, int32_t* valid,
                        int lifted) {
  return guard([&] {
    auto run = [&](auto tag) {
      constexpr int DD = decltype(tag)::value;
      using S = FT<DD>;
      const PoseT<S> pose = load_pose<DD>(w2c);
      const IntrinsicsT<S> k = load_intr<DD>(intr, w, h);
      Vec3<S> c;
      for (int e = 0; e < 3; ++e) c[e] = load_s<DD>(center + e * (1 + DD));
      auto eval = [&](const auto& dimg) {
        for (int i = 0; i < n; ++i) {
          const Vec3<S> p(S(pts[3 * i]), S(pts[3 * i + 1]), S(pts[3 * i + 2]));
          const auto m = measured_tsdf<S>(dimg, pose, k, mu, p, c);
          valid[i] = m.has_value();
          if (m) store_s<DD>(out + i * (1 + DD), *m);
        }
      };
      if (lifted) {
        Image<S> dl(w, h, S(0.0));
        for (int i = 0; i < w * h; ++i) dl.data[i] = load_s<DD>(depth + static_cast<std::size_t>(i) * (1 + DD));
        eval(dl);
      } else {
        eval(image_of(depth, w, h));
      }
    };
    switch (D) {
      case 0: run(std::integral_constant<int, 0>{}); break;
      case 1: run(std::integral_constant<int, 1>{}); break;
      case 2: run(std::integral_constant<int, 2>{}); break;
      case 3: run(std::integral_constant<int, 3>{}); break;
      default: throw std::invalid_argument("orc_measured_points: unsupported channel count");
    }
  });
}

int orc_view_scores(void* v, const double* poses, int n, const csf_intrinsics* k, double w0, double beta, double h,
                    double* scores, double* grads) {
  return guard([&] { static_cast<VolBase*>(v)->view_scores(poses, n, to_intr(*k), w0, beta, h, scores, grads); });
}

// associate (icp.cpp:89-126) over maps [h][w][3]; corrs [n][9]
int orc_associate(const double* mv, const double* mn, const double* pv, const double* pn, int w, int h,
                  const double* c2w, const double* pc2w, const csf_intrinsics* k, const csf_icp_cfg* cfg, int stride,
                  double* corrs, int* n) {
  return guard([&] {
    SurfaceMaps<double> meas, pred;
    meas.vertices = Image<Vec3d>(w, h, Vec3d());
    meas.normals = Image<Vec3d>(w, h, Vec3d());
    pred.vertices = Image<Vec3d>(w, h, Vec3d());
    pred.normals = Image<Vec3d>(w, h, Vec3d());
    for (int i = 0; i < w * h; ++i) {
      meas.vertices.data[i] = Vec3d(mv[3 * i], mv[3 * i + 1], mv[3 * i + 2]);
      meas.normals.data[i] = Vec3d(mn[3 * i], mn[3 * i + 1], mn[3 * i + 2]);
      pred.vertices.data[i] = Vec3d(pv[3 * i], pv[3 * i + 1], pv[3 * i + 2]);
      pred.normals.data[i] = Vec3d(pn[3 * i], pn[3 * i + 1], pn[3 * i + 2]);
    }
    Pose a, b;
    for (int e = 0; e < 9; ++e) {
      a.rotation(e / 3, e % 3) = c2w[e];
      b.rotation(e / 3, e % 3) = pc2w[e];
    }
    for (int e = 0; e < 3; ++e) {
      a.translation[e] = c2w[9 + e];
      b.translation[e] = pc2w[9 + e];
    }
    Intrinsics kk = to_intr(*k);
    kk.width = w;
    kk.height = h;
    const auto cs = associate(meas, pred, a, b, kk, to_icp(*cfg), stride);
    for (std::size_t i = 0; i < cs.size(); ++i)
      for (int c = 0; c < 3; ++c) {
        corrs[9 * i + c] = cs[i].vertex[c];
        corrs[9 * i + 3 + c] = cs[i].model_vertex[c];
        corrs[9 * i + 6 + c] = cs[i].model_normal[c];
      }
    *n = static_cast<int>(cs.size());
  });
}

// linearized_step (icp.cpp:146-153), canonical tiled or literal sequential order
int orc_linearized_step(const double* corrs, int n, const double* base, int sequential, double* delta) {
  return guard([&] {
    std::vector<Correspondence> cs(n);
    for (int i = 0; i < n; ++i) {
      const double* c = corrs + 9 * i;
      cs[i].vertex = Vec3d(c[0], c[1], c[2]);
      cs[i].model_vertex = Vec3d(c[3], c[4], c[5]);
      cs[i].model_normal = Vec3d(c[6], c[7], c[8]);
    }
    Pose b;
    for (int e = 0; e < 9; ++e) b.rotation(e / 3, e % 3) = base[e];
    for (int e = 0; e < 3; ++e) b.translation[e] = base[9 + e];
    const Vec6<double> d = linearized_step(cs, b, sequential != 0);
    for (int i = 0; i < 6; ++i) delta[i] = d[i];
  });
}

// icp_energy / icp_gradient / icp_hessian (icp.hpp:70-91) at xi (NULL = 0).
int orc_icp_energy_derivs(const double* corrs, int n, const double* base, const double* xi, double h, double* E,
                          double* g, double* H) {
  return guard([&] {
    std::vector<Correspondence> cs(n);
    for (int i = 0; i < n; ++i) {
      const double* c = corrs + 9 * i;
      cs[i].vertex = Vec3d(c[0], c[1], c[2]);
      cs[i].model_vertex = Vec3d(c[3], c[4], c[5]);
      cs[i].model_normal = Vec3d(c[6], c[7], c[8]);
    }
    Pose b;
    for (int e = 0; e < 9; ++e) b.rotation(e / 3, e % 3) = base[e];
    for (int e = 0; e < 3; ++e) b.translation[e] = base[9 + e];
    Vec6<double> x{};
    if (xi)
      for (int k = 0; k < 6; ++k) x[k] = xi[k];
    const StepSize step(h);
    auto f = [&](const auto& v) { return icp_energy(cs, v, b); };
    if (E) *E = icp_energy(cs, x, b);
    if (g) {
      const Vec6<double> gr = csfd_gradient(f, x, step);
      for (int k = 0; k < 6; ++k) g[k] = gr[k];
    }
    if (H) {
      const Mat6d hs = csfd_hessian(f, x, step);
      for (int r = 0; r < 6; ++r)
        for (int c = 0; c < 6; ++c) H[6 * r + c] = hs[r][c];
    }
  });
}

// Second-order run: one Bicomplex pass per pair (csfd_hessian pattern).
int orc_pipeline_hessian(const csf_pipeline_cfg* c, const float* depth, const double* gt_in, int n_frames,
                         double* hessian, double* grad1, double* grad2, double* objective, double* poses,
                         int32_t* stats, double* seconds) {
  return guard([&] {
    const PipelineConfig cfg = to_pipeline(c);
    if (c->n_pairs <= 0 || c->n_pairs > CSF_MAX_PAIRS) throw std::invalid_argument("orc_pipeline_hessian: n_pairs");
    std::vector<std::pair<int, int>> pairs;
    for (int p = 0; p < c->n_pairs; ++p) pairs.emplace_back(c->pair_i[p], c->pair_j[p]);
    std::vector<Image<double>> frames;
    std::vector<Pose> gt;
    to_frames(cfg, depth, gt_in, n_frames, &frames, &gt);
    const auto t0 = std::chrono::steady_clock::now();
    const HessianResult r = run_pipeline_hessian(cfg, pairs, frames, gt);
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    if (objective) *objective = r.objective;
    for (int p = 0; p < c->n_pairs; ++p) {
      if (hessian) hessian[p] = r.hessian[p];
      if (grad1) grad1[p] = r.grad1[p];
      if (grad2) grad2[p] = r.grad2[p];
    }
    if (poses) std::memcpy(poses, r.poses.data(), sizeof(double) * r.poses.size());
    if (stats) write_stats(n_frames, r, stats);
  });
}

// orc_pipeline_run that also hands back the run's final volume (an orc
// volume handle: orc_volume_download / orc_volume_hash / orc_volume_destroy).
int orc_pipeline_run_keep(const csf_pipeline_cfg* c, const float* depth, const double* gt_in, int n_frames,
                          double* gradient, double* objective, double* poses, int32_t* stats, void** vol_out) {
  return guard([&] {
    const PipelineConfig cfg = to_pipeline(c);
    std::vector<Image<double>> frames;
    std::vector<Pose> gt;
    to_frames(cfg, depth, gt_in, n_frames, &frames, &gt);
    PipelineResult r;
    VolBase* keep = nullptr;
    auto run = [&](auto dtag) {
      constexpr int D = decltype(dtag)::value;
      if (cfg.hashed) {
        auto* v = new Vol<D, true>(cfg.hash);
        keep = v;
        r = run_pipeline_on<D>(v->vol, cfg, frames, gt);
      } else {
        auto* v = new Vol<D, false>(cfg.dense);
        keep = v;
        r = run_pipeline_on<D>(v->vol, cfg, frames, gt);
      }
    };
    switch (cfg.directions.size()) {
      case 1: run(std::integral_constant<int, 1>{}); break;
      case 2: run(std::integral_constant<int, 2>{}); break;
      case 3: run(std::integral_constant<int, 3>{}); break;
      case 4: run(std::integral_constant<int, 4>{}); break;
      case 5: run(std::integral_constant<int, 5>{}); break;
      case 6: run(std::integral_constant<int, 6>{}); break;
      case 8: run(std::integral_constant<int, 8>{}); break;
      case 10: run(std::integral_constant<int, 10>{}); break;
      case 20: run(std::integral_constant<int, 20>{}); break;
      default: throw std::invalid_argument("orc_pipeline_run_keep: unsupported direction count");
    }
    if (objective) *objective = r.objective;
    if (gradient)
      for (int d = 0; d < c->n_dirs; ++d) gradient[d] = r.gradient[d];
    if (poses) std::memcpy(poses, r.poses.data(), sizeof(double) * r.poses.size());
    if (stats) write_stats(n_frames, r, stats);
    *vol_out = keep;
  });
}

int orc_pipeline_run(const csf_pipeline_cfg* c, const float* depth, const double* gt_in, int n_frames,
                     double* gradient, double* objective, double* poses, int32_t* stats, double* seconds) {
  return guard([&] {
    const PipelineConfig cfg = to_pipeline(c);
    std::vector<Image<double>> frames;
    std::vector<Pose> gt;
    to_frames(cfg, depth, gt_in, n_frames, &frames, &gt);
    const auto t0 = std::chrono::steady_clock::now();
    const PipelineResult r = run_pipeline_dyn(cfg, frames, gt);
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    if (objective) *objective = r.objective;
    if (gradient)
      for (int d = 0; d < c->n_dirs; ++d) gradient[d] = r.gradient[d];
    if (poses) std::memcpy(poses, r.poses.data(), sizeof(double) * r.poses.size());
    if (stats) write_stats(n_frames, r, stats);
  });
}

// The reference's IcpConfig defaults (icp.hpp:33-53, restated in
// orc_icp.hpp) in the shared descriptor: bench.py's --impl reference builds
// its configuration from these, so that arm never loads the product library.
void orc_default_icp_cfg(csf_icp_cfg* c) {
  const IcpConfig d;
  c->solver = static_cast<int>(d.solver);
  c->d_max = d.d_max;
  c->theta_max_deg = d.theta_max_deg;
  c->levels = d.levels;
  for (int i = 0; i < 3; ++i) {
    c->level_iterations[i] = d.level_iterations[i];
    c->level_pixel_stride[i] = d.level_pixel_stride[i];
  }
  c->step_tolerance = d.step_tolerance;
  c->levenberg_lambda0 = d.levenberg_lambda0;
  c->ncg_restart = d.ncg_restart;
  c->h = d.step.h;
}

// tests/test_detmath.py: the deterministic elementary functions used on the
// device path (include/csf_detmath.h) against glibc, in ulps of the glibc
// result.  fn: 0 exp, 1 sin, 2 cos.  out_ulp[i] per argument.
int orc_detmath_ulp(int fn, const double* x, int n, double* out_ulp, double* det_out, double* libm_out) {
  return guard([&] {
    for (int i = 0; i < n; ++i) {
      const double d = fn == 0 ? csf_det::exp(x[i]) : fn == 1 ? csf_det::sin(x[i]) : csf_det::cos(x[i]);
      const double g = fn == 0 ? std::exp(x[i]) : fn == 1 ? std::sin(x[i]) : std::cos(x[i]);
      double ulp;
      if (d == g) {
        ulp = 0.0;
      } else {
        const double a = std::fabs(g);
        const double step = std::nextafter(a, INFINITY) - a;  // ulp of the glibc value
        ulp = std::fabs(d - g) / (step > 0.0 ? step : std::numeric_limits<double>::denorm_min());
      }
      out_ulp[i] = ulp;
      if (det_out) det_out[i] = d;
      if (libm_out) libm_out[i] = g;
    }
  });
}

}  // extern "C"
