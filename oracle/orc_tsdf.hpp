// ORACLE — TEST INFRASTRUCTURE ONLY (see orc_core.hpp header).
//
// Dense TSDF: restates proj/include/csf/tsdf.hpp:21-284 and
// proj/src/tsdf.cpp:11-40.  The stored field type F generalises the
// reference's Complex to Lifted<D> (packed directions) or double.
//
// Hashed TSDF (BUILDER-DEFINED — the reference has no voxel hashing,
// SPEC.md:345): 8^3 voxel blocks addressed by a chained hash over 2^B buckets
// whose chains are kept sorted by block key, so the table layout depends only
// on the set of keys; blocks are allocated in first-touch order of the
// per-pixel truncation-band samples (pixel row-major, sample index ascending).
// DESIGN.md "Hashed TSDF" states the exact rules; the sm_100a path implements
// the same rules and the tests compare the tables bit for bit.
#pragma once

#include <algorithm>
#include <optional>
#include <unordered_set>

#include "orc_frames.hpp"

namespace orc {

// tsdf.hpp:21-36
struct VolumeParams {
  int dims[3] = {128, 128, 128};
  double voxel_size = 0.02;
  Vec3d origin;
  double mu = 0.1;
  double weight_cap = 128.0;
  static VolumeParams cube(int n, double voxel, const Vec3d& o) {
    VolumeParams p;
    p.dims[0] = p.dims[1] = p.dims[2] = n;
    p.voxel_size = voxel;
    p.origin = o;
    p.mu = 5.0 * voxel;
    return p;
  }
};

// tsdf.hpp:38-78 (field type generalised)
template <typename F>
struct TsdfVolumeT {
  using field_type = F;
  static constexpr bool kHashed = false;
  VolumeParams params;
  std::vector<F> tsdf;
  std::vector<double> weight;
  explicit TsdfVolumeT(const VolumeParams& p)
      : params(p), tsdf(static_cast<std::size_t>(p.dims[0]) * p.dims[1] * p.dims[2], F(1.0)),
        weight(tsdf.size(), 0.0) {}
  std::size_t index(int i, int j, int k) const {
    return (static_cast<std::size_t>(k) * params.dims[1] + j) * params.dims[0] + i;
  }
  Vec3d voxel_position(int i, int j, int k) const {
    const double vs = params.voxel_size;
    return params.origin + Vec3d(vs * double(i), vs * double(j), vs * double(k));
  }
  // corner lookup used by sample_tsdf
  bool corner(int i, int j, int k, const F** f, double* w) const {
    const std::size_t idx = index(i, j, k);
    *f = &tsdf[idx];
    *w = weight[idx];
    return true;
  }
  bool cell_in_grid(int i0, int j0, int k0) const {
    return !(i0 < 0 || j0 < 0 || k0 < 0 || i0 + 1 >= params.dims[0] || j0 + 1 >= params.dims[1] ||
             k0 + 1 >= params.dims[2]);
  }
};

// ---------------------------------------------------------------------------
// Hashed volume (builder-defined)
// ---------------------------------------------------------------------------
struct HashParams {
  double voxel_size = 0.005;
  Vec3d origin;
  double mu = 0.025;
  double weight_cap = 128.0;
  int bucket_bits = 20;
  int max_blocks = 1 << 18;
};

constexpr int kBlockSide = 8;
constexpr int kBlockVoxels = 512;
constexpr int kCoordBias = 1 << 20;

inline uint64_t block_key(int bx, int by, int bz) {
  return (static_cast<uint64_t>(static_cast<uint32_t>(bx + kCoordBias)) << 42) |
         (static_cast<uint64_t>(static_cast<uint32_t>(by + kCoordBias)) << 21) |
         static_cast<uint64_t>(static_cast<uint32_t>(bz + kCoordBias));
}
inline uint32_t block_hash(int bx, int by, int bz, int bits) {
  const uint32_t h = (static_cast<uint32_t>(bx) * 73856093u) ^ (static_cast<uint32_t>(by) * 19349669u) ^
                     (static_cast<uint32_t>(bz) * 83492791u);
  return h & ((1u << bits) - 1u);
}
inline int floor_div8(int i) { return i >> 3; }  // arithmetic shift == floor for int32

template <typename F>
struct HashedVolumeT {
  using field_type = F;
  static constexpr bool kHashed = true;
  HashParams params;
  std::vector<int32_t> heads;        // [2^bits], -1 = empty
  std::vector<uint64_t> keys;        // [n_blocks]
  std::vector<int32_t> next;         // [n_blocks], -1 = end of chain
  std::vector<int32_t> coords;       // [n_blocks][3]
  std::vector<F> tsdf;               // [n_blocks * 512]
  std::vector<double> weight;        // [n_blocks * 512]
  explicit HashedVolumeT(const HashParams& p) : params(p), heads(std::size_t(1) << p.bucket_bits, -1) {}
  int n_blocks() const { return static_cast<int>(keys.size()); }

  int find(int bx, int by, int bz) const {
    const uint64_t key = block_key(bx, by, bz);
    int32_t e = heads[block_hash(bx, by, bz, params.bucket_bits)];
    while (e >= 0) {
      if (keys[e] == key) return e;
      if (keys[e] > key) return -1;  // chains are sorted ascending
      e = next[e];
    }
    return -1;
  }
  // Insert a new block (caller guarantees absence); returns its pool id.
  int insert(int bx, int by, int bz) {
    if (n_blocks() >= params.max_blocks) throw std::runtime_error("hashed volume: block pool exhausted");
    const uint64_t key = block_key(bx, by, bz);
    const int id = n_blocks();
    keys.push_back(key);
    next.push_back(-1);
    coords.push_back(bx);
    coords.push_back(by);
    coords.push_back(bz);
    tsdf.resize(tsdf.size() + kBlockVoxels, F(1.0));
    weight.resize(weight.size() + kBlockVoxels, 0.0);
    int32_t* link = &heads[block_hash(bx, by, bz, params.bucket_bits)];
    while (*link >= 0 && keys[*link] < key) link = &next[*link];
    next[id] = *link;
    *link = id;
    return id;
  }
  Vec3d voxel_position(int i, int j, int k) const {
    const double vs = params.voxel_size;
    return params.origin + Vec3d(vs * double(i), vs * double(j), vs * double(k));
  }
  static int local_index(int i, int j, int k) { return ((k & 7) * 8 + (j & 7)) * 8 + (i & 7); }
  bool corner(int i, int j, int k, const F** f, double* w) const {
    const int b = find(floor_div8(i), floor_div8(j), floor_div8(k));
    if (b < 0) return false;
    const std::size_t idx = static_cast<std::size_t>(b) * kBlockVoxels + local_index(i, j, k);
    *f = &tsdf[idx];
    *w = weight[idx];
    return true;
  }
  bool cell_in_grid(int, int, int) const { return true; }
};

template <typename V> const VolumeParams* dense_params(const V&) { return nullptr; }

// Common accessors over both volume kinds.
template <typename F> double vol_voxel_size(const TsdfVolumeT<F>& v) { return v.params.voxel_size; }
template <typename F> double vol_voxel_size(const HashedVolumeT<F>& v) { return v.params.voxel_size; }
template <typename F> const Vec3d& vol_origin(const TsdfVolumeT<F>& v) { return v.params.origin; }
template <typename F> const Vec3d& vol_origin(const HashedVolumeT<F>& v) { return v.params.origin; }
template <typename F> double vol_mu(const TsdfVolumeT<F>& v) { return v.params.mu; }
template <typename F> double vol_mu(const HashedVolumeT<F>& v) { return v.params.mu; }

// tsdf.hpp:86
inline constexpr double kDepthEdgeLimit = 0.1;

// tsdf.hpp:97-140 — depth element type DS (Complex in the reference; double
// for unperturbed frames), evaluation scalar S, intrinsics scalar K.
template <typename S, typename DS, typename K>
std::optional<S> measured_tsdf(const Image<DS>& depth, const PoseT<S>& world_to_camera,
                               const IntrinsicsT<K>& k, double mu, const Vec3<S>& p_world,
                               const Vec3<S>& camera_center) {
  const Vec3<S> pc = world_to_camera * p_world;
  if (!(real_part(pc.z()) > 0.0)) return std::nullopt;
  const std::array<S, 2> px = project(k, pc);
  const S lx = px[0], ly = px[1];
  const int x0 = ifloor_s(lx), y0 = ifloor_s(ly);
  if (x0 < 0 || y0 < 0 || x0 + 1 >= depth.width || y0 + 1 >= depth.height) return std::nullopt;
  const DS& d00 = depth.at(x0, y0);
  const DS& d10 = depth.at(x0 + 1, y0);
  const DS& d01 = depth.at(x0, y0 + 1);
  const DS& d11 = depth.at(x0 + 1, y0 + 1);
  if (!depth_valid(d00) || !depth_valid(d10) || !depth_valid(d01) || !depth_valid(d11)) return std::nullopt;
  const double near = std::min(std::min(real_part(d00), real_part(d10)), std::min(real_part(d01), real_part(d11)));
  const double far = std::max(std::max(real_part(d00), real_part(d10)), std::max(real_part(d01), real_part(d11)));
  if (far - near > kDepthEdgeLimit) return std::nullopt;
  const S fx = lx - S(double(x0));
  const S fy = ly - S(double(y0));
  const S top = Measure<S>::in(d00) + fx * (Measure<S>::in(d10) - Measure<S>::in(d00));
  const S bot = Measure<S>::in(d01) + fx * (Measure<S>::in(d11) - Measure<S>::in(d01));
  const S sampled = top + fy * (bot - top);
  const Vec3<S> ray((lx - kval<S>(k.cx)) / kval<S>(k.fx), (ly - kval<S>(k.cy)) / kval<S>(k.fy), S(1.0));
  const S lambda = sqrt(dot(ray, ray));
  const Vec3<S> diff = camera_center - p_world;
  const S eta = sampled - sqrt(dot(diff, diff)) / lambda;
  if (real_part(eta) < -mu) return std::nullopt;
  return clamp(eta / S(mu), -1.0, 1.0);
}

// tsdf.cpp:11-40 — dense fusion over every voxel (OpenMP over z slices).
// Returns the number of voxels fused (the device's stats column 6).
template <typename F, typename DS, typename K>
long long surface_update(TsdfVolumeT<F>& volume, const Image<DS>& depth, const PoseT<F>& camera_to_world,
                         const IntrinsicsT<K>& k) {
  const PoseT<F> world_to_camera = camera_to_world.inverse();
  const Vec3<F>& center = camera_to_world.translation;
  const VolumeParams& vp = volume.params;
  const double cap = vp.weight_cap;
  const int nx = vp.dims[0], ny = vp.dims[1], nz = vp.dims[2];
  long long fused = 0;
#pragma omp parallel for schedule(static) reduction(+ : fused)
  for (int kk = 0; kk < nz; ++kk)
    for (int jj = 0; jj < ny; ++jj)
      for (int ii = 0; ii < nx; ++ii) {
        const Vec3d p = volume.voxel_position(ii, jj, kk);
        const Vec3<F> pw(F(p.x()), F(p.y()), F(p.z()));
        const auto sample = measured_tsdf<F>(depth, world_to_camera, k, vp.mu, pw, center);
        if (!sample) continue;
        const std::size_t idx = volume.index(ii, jj, kk);
        const double w = volume.weight[idx];
        F& f = volume.tsdf[idx];
        f = (F(w) * f + *sample) / F(w + 1.0);
        volume.weight[idx] = std::min(w + 1.0, cap);
        ++fused;
      }
  return fused;
}

// ---------------------------------------------------------------------------
// Hashed allocation + fusion (builder-defined)
// ---------------------------------------------------------------------------
// Number of truncation-band samples per pixel: spacing <= one voxel.
inline int band_samples(double mu, double voxel_size) {
  return std::max(2, static_cast<int>(std::ceil((2.0 * mu) / voxel_size)) + 1);
}

// Voxel-cell coordinate of a world point along one axis: ifloor((p - o)/vs),
// the same expression sample_tsdf uses (tsdf.hpp:151-154).
inline int cell_of(double p, double o, double vs) { return ifloor((p - o) / vs); }

// Candidate block keys of one pixel's band [d - mu, d + mu] (z in camera
// frame), consecutive duplicates removed.  Writes up to K (bx,by,bz) triples.
inline int pixel_band_blocks(double d, int x, int y, const Intrinsics& k, const Pose& c2w, const HashParams& hp,
                             int K, int* out) {
  int n = 0;
  if (!(d > 0.0)) return 0;
  const double mu = hp.mu, vs = hp.voxel_size;
  const double lo = d - mu;
  const double step = (2.0 * mu) / static_cast<double>(K - 1);
  const double rx = (static_cast<double>(x) - k.cx) / k.fx;
  const double ry = (static_cast<double>(y) - k.cy) / k.fy;
  int pbx = 0, pby = 0, pbz = 0;
  bool have = false;
  for (int s = 0; s < K; ++s) {
    const double z = lo + static_cast<double>(s) * step;
    if (!(z > 0.0)) continue;
    const Vec3d q(z * rx, z * ry, z);
    const Vec3d w = c2w * q;
    const int bx = floor_div8(cell_of(w.x(), hp.origin.x(), vs));
    const int by = floor_div8(cell_of(w.y(), hp.origin.y(), vs));
    const int bz = floor_div8(cell_of(w.z(), hp.origin.z(), vs));
    if (have && bx == pbx && by == pby && bz == pbz) continue;
    out[3 * n] = bx; out[3 * n + 1] = by; out[3 * n + 2] = bz;
    ++n;
    pbx = bx; pby = by; pbz = bz;
    have = true;
  }
  return n;
}

struct AllocStats {
  int touched = 0;  // distinct blocks touched this frame (visible list size)
  int fresh = 0;    // newly allocated blocks
};

// Allocate the band blocks of `depth` at the real pose; returns the visible
// list (pool ids, first-touch order).
template <typename F>
std::vector<int> allocate_band(HashedVolumeT<F>& vol, const Image<double>& depth, const Intrinsics& k,
                               const Pose& c2w, AllocStats* stats = nullptr) {
  const int K = band_samples(vol.params.mu, vol.params.voxel_size);
  std::vector<int> buf(3 * K);
  std::vector<int> visible;
  std::unordered_set<uint64_t> touched;
  int fresh = 0;
  for (int y = 0; y < depth.height; ++y)
    for (int x = 0; x < depth.width; ++x) {
      const int n = pixel_band_blocks(depth.at(x, y), x, y, k, c2w, vol.params, K, buf.data());
      for (int c = 0; c < n; ++c) {
        const int bx = buf[3 * c], by = buf[3 * c + 1], bz = buf[3 * c + 2];
        const uint64_t key = block_key(bx, by, bz);
        if (!touched.insert(key).second) continue;
        int id = vol.find(bx, by, bz);
        if (id < 0) {
          id = vol.insert(bx, by, bz);
          ++fresh;
        }
        visible.push_back(id);
      }
    }
  if (stats) {
    stats->touched = static_cast<int>(visible.size());
    stats->fresh = fresh;
  }
  return visible;
}

// Fusion over the visible blocks with the reference's per-voxel rule
// (tsdf.cpp:25-37).
template <typename F, typename DS, typename K>
long long surface_update_blocks(HashedVolumeT<F>& vol, const std::vector<int>& visible, const Image<DS>& depth,
                                const PoseT<F>& camera_to_world, const IntrinsicsT<K>& k) {
  const PoseT<F> world_to_camera = camera_to_world.inverse();
  const Vec3<F>& center = camera_to_world.translation;
  const double cap = vol.params.weight_cap, mu = vol.params.mu;
  long long fused = 0;
#pragma omp parallel for schedule(static) reduction(+ : fused)
  for (std::ptrdiff_t vb = 0; vb < static_cast<std::ptrdiff_t>(visible.size()); ++vb) {
    const int b = visible[vb];
    const int bx = vol.coords[3 * b], by = vol.coords[3 * b + 1], bz = vol.coords[3 * b + 2];
    for (int lz = 0; lz < 8; ++lz)
      for (int ly = 0; ly < 8; ++ly)
        for (int lx = 0; lx < 8; ++lx) {
          const Vec3d p = vol.voxel_position(8 * bx + lx, 8 * by + ly, 8 * bz + lz);
          const Vec3<F> pw(F(p.x()), F(p.y()), F(p.z()));
          const auto sample = measured_tsdf<F>(depth, world_to_camera, k, mu, pw, center);
          if (!sample) continue;
          const std::size_t idx = static_cast<std::size_t>(b) * kBlockVoxels + (lz * 8 + ly) * 8 + lx;
          const double w = vol.weight[idx];
          F& f = vol.tsdf[idx];
          f = (F(w) * f + *sample) / F(w + 1.0);
          vol.weight[idx] = std::min(w + 1.0, cap);
          ++fused;
        }
  }
  return fused;
}

// ---------------------------------------------------------------------------
// Sampling and raycast — tsdf.hpp:148-284 (generic over volume kind)
// ---------------------------------------------------------------------------
template <typename S, typename V>
std::optional<S> sample_tsdf(const V& vol, const Vec3<S>& p_world) {
  const double vs = vol_voxel_size(vol);
  const Vec3d& o = vol_origin(vol);
  const S gx = (p_world.x() - S(o.x())) / S(vs);
  const S gy = (p_world.y() - S(o.y())) / S(vs);
  const S gz = (p_world.z() - S(o.z())) / S(vs);
  const int i0 = ifloor_s(gx), j0 = ifloor_s(gy), k0 = ifloor_s(gz);
  if (!vol.cell_in_grid(i0, j0, k0)) return std::nullopt;
  const S fx = gx - S(double(i0));
  const S fy = gy - S(double(j0));
  const S fz = gz - S(double(k0));
  S accum = S(0.0);
  for (int dk = 0; dk < 2; ++dk)
    for (int dj = 0; dj < 2; ++dj)
      for (int di = 0; di < 2; ++di) {
        const typename V::field_type* f = nullptr;
        double w = 0.0;
        if (!vol.corner(i0 + di, j0 + dj, k0 + dk, &f, &w)) return std::nullopt;
        if (!(w > 0.0)) return std::nullopt;
        const S wx = di ? fx : S(1.0) - fx;
        const S wy = dj ? fy : S(1.0) - fy;
        const S wz = dk ? fz : S(1.0) - fz;
        accum += wx * wy * wz * Measure<S>::in(*f);
      }
  return accum;
}

// Real-channel-only sample (identical to the real part of sample_tsdf<S>).
template <typename V>
std::optional<double> sample_tsdf_real(const V& vol, const Vec3d& p) {
  return sample_tsdf<double>(vol, p);
}

// tsdf.hpp:181-196
template <typename S, typename V>
std::optional<Vec3<S>> sample_gradient(const V& vol, const Vec3<S>& p_world) {
  const double h = vol_voxel_size(vol);
  Vec3<S> g;
  for (int axis = 0; axis < 3; ++axis) {
    Vec3<S> lo = p_world, hi = p_world;
    lo[axis] -= S(h);
    hi[axis] += S(h);
    const auto flo = sample_tsdf<S>(vol, lo);
    const auto fhi = sample_tsdf<S>(vol, hi);
    if (!flo || !fhi) return std::nullopt;
    g[axis] = (*fhi - *flo) / S(2.0 * h);
  }
  return g;
}

// tsdf.hpp:198-204
struct RaycastConfig {
  double near_clip = 0.0;
  double far_clip = 10.0;
  double step_fraction = 0.5;
};

// Camera-frame ray direction of pixel (x, y): the reference lifts the double
// expression (tsdf.hpp:228); with lifted intrinsics the same expression is
// evaluated in S (identical real part).
template <typename S> Vec3<S> ray_dir_cam(int x, int y, const IntrinsicsT<double>& k) {
  return {S((x - k.cx) / k.fx), S((y - k.cy) / k.fy), S(1.0)};
}
template <typename S, typename K, typename = std::enable_if_t<!std::is_same_v<K, double>>>
Vec3<S> ray_dir_cam(int x, int y, const IntrinsicsT<K>& k) {
  return {(S(double(x)) - k.cx) / k.fx, (S(double(y)) - k.cy) / k.fy, S(1.0)};
}

// tsdf.hpp:209-284.  Hashed volumes have no bounding box: the march runs over
// [near_clip, far_clip] (builder-defined).  The march itself only needs real
// parts (every branch reads real parts); the lifted samples at the crossing
// are re-evaluated at the same alpha values, which reproduces the
// reference's lifted f_prev/f bit for bit.
template <typename S, typename V, typename K>
SurfaceMaps<S> raycast(const V& vol, const PoseT<S>& camera_to_world, const IntrinsicsT<K>& k,
                       const RaycastConfig& cfg = {}) {
  SurfaceMaps<S> maps;
  maps.vertices = Image<Vec3<S>>(k.width, k.height, Vec3<S>());
  maps.normals = Image<Vec3<S>>(k.width, k.height, Vec3<S>());
  const double step = cfg.step_fraction * vol_mu(vol);
  Vec3d box_lo, box_hi;
  bool use_box = false;
  if constexpr (!V::kHashed) {
    const VolumeParams& vp = vol.params;
    use_box = true;
    box_lo = vp.origin;
    box_hi = vp.origin + Vec3d(vp.voxel_size * (double(vp.dims[0]) - 1.0), vp.voxel_size * (double(vp.dims[1]) - 1.0),
                               vp.voxel_size * (double(vp.dims[2]) - 1.0));
  }
  const Pose real_c2w = real_pose(camera_to_world);
#pragma omp parallel for schedule(dynamic, 8)
  for (int y = 0; y < k.height; ++y) {
    for (int x = 0; x < k.width; ++x) {
      const Vec3<S> dir_cam = ray_dir_cam<S>(x, y, k);
      const S ray_norm = sqrt(dot(dir_cam, dir_cam));
      const Vec3<S> dir = camera_to_world.rotation * (dir_cam / ray_norm);
      const Vec3<S>& o = camera_to_world.translation;
      double t0 = cfg.near_clip, t1 = cfg.far_clip;
      bool hit_box = true;
      if (use_box) {
        for (int axis = 0; axis < 3; ++axis) {
          const double od = real_part(o[axis]);
          const double dd = real_part(dir[axis]);
          if (std::fabs(dd) < 1e-12) {
            if (od < box_lo[axis] || od > box_hi[axis]) hit_box = false;
            continue;
          }
          double ta = (box_lo[axis] - od) / dd;
          double tb = (box_hi[axis] - od) / dd;
          if (ta > tb) std::swap(ta, tb);
          t0 = std::max(t0, ta);
          t1 = std::min(t1, tb);
        }
      }
      if (!hit_box || t0 >= t1) continue;
      const Vec3d ore(real_part(o[0]), real_part(o[1]), real_part(o[2]));
      const Vec3d dre(real_part(dir[0]), real_part(dir[1]), real_part(dir[2]));
      bool have_prev = false;
      double alpha_prev = 0.0, f_prev = 0.0;
      (void)real_c2w;
      for (double alpha = t0; alpha <= t1; alpha += step) {
        // real part of o + S(alpha) * dir
        const Vec3d p(ore[0] + alpha * dre[0], ore[1] + alpha * dre[1], ore[2] + alpha * dre[2]);
        const auto f = sample_tsdf<double>(vol, p);
        if (!f) {
          have_prev = false;
          continue;
        }
        if (have_prev && f_prev > 0.0 && *f < 0.0) {
          const auto sample_at = [&](double a) {
            const Vec3<S> q = o + S(a) * dir;
            return *sample_tsdf<S>(vol, q);
          };
          const S fl_prev = sample_at(alpha_prev);
          const S fl = sample_at(alpha);
          const S span = S(alpha - alpha_prev);
          const S alpha_star = S(alpha_prev) - span * fl_prev / (fl - fl_prev);
          const Vec3<S> v = o + alpha_star * dir;
          const auto grad = sample_gradient<S>(vol, v);
          if (grad) {
            const S len2 = dot(*grad, *grad);
            if (real_part(len2) > 0.0) {
              maps.vertices.at(x, y) = v;
              maps.normals.at(x, y) = *grad / sqrt(len2);
            }
          }
          break;
        }
        have_prev = true;
        alpha_prev = alpha;
        f_prev = *f;
      }
    }
  }
  return maps;
}

// ---------------------------------------------------------------------------
// BUILDER-DEFINED (BASELINE config 5; the spec's unimplemented "smooth
// visibility score"): soft count of weakly observed surface
// seen from a view.  W~ = trilinear interpolation of the integral fusion
// weights (sample_tsdf's cell and dk, dj, di order, tsdf.hpp:148-177;
// unallocated corners count 0); score = pairwise_sum over all pixels
// (row-major) of sigma(beta (w0 - W~(p))) at raycast hits (valid normal,
// frames.hpp:73-81), 0 elsewhere.
// ---------------------------------------------------------------------------
template <typename S, typename V>
S interpolated_weight(const V& vol, const Vec3<S>& p_world) {
  const double vs = vol_voxel_size(vol);
  const Vec3d& o = vol_origin(vol);
  const S gx = (p_world.x() - S(o.x())) / S(vs);
  const S gy = (p_world.y() - S(o.y())) / S(vs);
  const S gz = (p_world.z() - S(o.z())) / S(vs);
  const int i0 = ifloor_s(gx), j0 = ifloor_s(gy), k0 = ifloor_s(gz);
  const S fx = gx - S(double(i0));
  const S fy = gy - S(double(j0));
  const S fz = gz - S(double(k0));
  S accum = S(0.0);
  for (int dk = 0; dk < 2; ++dk)
    for (int dj = 0; dj < 2; ++dj)
      for (int di = 0; di < 2; ++di) {
        const typename V::field_type* f = nullptr;
        double w = 0.0;
        if (!vol.corner(i0 + di, j0 + dj, k0 + dk, &f, &w)) w = 0.0;
        const S wx = di ? fx : S(1.0) - fx;
        const S wy = dj ? fy : S(1.0) - fy;
        const S wz = dk ? fz : S(1.0) - fz;
        accum += wx * wy * wz * S(w);
      }
  return accum;
}

template <typename S, typename V, typename K>
S view_coverage_score(const V& vol, const PoseT<S>& view, const IntrinsicsT<K>& k, double w0, double beta,
                      const RaycastConfig& rc = {}) {
  const SurfaceMaps<S> maps = raycast<S>(vol, view, k, rc);
  std::vector<S> terms(maps.vertices.data.size(), S(0.0));
  for (std::size_t i = 0; i < terms.size(); ++i) {
    const Vec3<S>& n = maps.normals.data[i];
    const double n0 = real_part(n[0]), n1 = real_part(n[1]), n2 = real_part(n[2]);
    if (!(n0 * n0 + (n1 * n1 + n2 * n2) > 0.5)) continue;
    const S wt = interpolated_weight<S>(vol, maps.vertices.data[i]);
    const S z = S(beta) * (S(w0) - wt);
    terms[i] = S(1.0) / (S(1.0) + exp(-z));
  }
  return pairwise_sum(terms);
}

}  // namespace orc
