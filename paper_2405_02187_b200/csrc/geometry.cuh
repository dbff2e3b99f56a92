// Device TSDF geometry: volume views (dense / hashed voxel blocks), projective
// measurement, trilinear sampling, and the 6x6 LDLT — generic over the scalar
// S (double or a channel group L<G>).  Each function names the reference
// function it re-implements; the evaluation order is the oracle's
// (oracle/orc_tsdf.hpp, oracle/orc_icp.hpp).
#pragma once

#include "lifted.cuh"

namespace csfd {

constexpr int kBlockVoxels = 512;
constexpr int kCoordBias = 1 << 20;
constexpr unsigned long long kEmptyKey = ~0ULL;

CSF_DEV unsigned long long block_key(int bx, int by, int bz) {
  return (static_cast<unsigned long long>(static_cast<unsigned>(bx + kCoordBias)) << 42) |
         (static_cast<unsigned long long>(static_cast<unsigned>(by + kCoordBias)) << 21) |
         static_cast<unsigned long long>(static_cast<unsigned>(bz + kCoordBias));
}
CSF_DEV unsigned block_hash(int bx, int by, int bz, unsigned mask) {
  return ((static_cast<unsigned>(bx) * 73856093u) ^ (static_cast<unsigned>(by) * 19349669u) ^
          (static_cast<unsigned>(bz) * 83492791u)) & mask;
}

// Voxel storage shared by both volume kinds: rw[v] = (F.re, W) and the
// perturbation channels fim[v*Dp + d] (voxel-major, channel-minor).
struct VoxelStore {
  double2* rw;
  double* fim;
  int Dp;
};

// Lookup-cache hook of the sampling functions (no state is needed: hashed
// volumes resolve in-window blocks through a dense block-id grid).
struct NoCache {
  CSF_DEV void reset() {}
};

// Dense lattice (tsdf.hpp:38-78): index (k*ny + j)*nx + i.
struct DenseView {
  using Cache = NoCache;
  VoxelStore vox;
  int nx, ny, nz;
  double vs, ox, oy, oz, mu, cap;
  static constexpr bool kHashed = false;
  CSF_DEV bool cell_in_grid(int i0, int j0, int k0) const {
    return !(i0 < 0 || j0 < 0 || k0 < 0 || i0 + 1 >= nx || j0 + 1 >= ny || k0 + 1 >= nz);
  }
  // returns the voxel index or -1
  CSF_DEV long long voxel(int i, int j, int k) const {
    return (static_cast<long long>(k) * ny + j) * nx + i;
  }
  CSF_DEV long long voxel(int i, int j, int k, NoCache&) const { return voxel(i, j, k); }
};

// Hashed 8^3 blocks: chained buckets, chains sorted by key (builder-defined;
// oracle/orc_tsdf.hpp HashedVolumeT).
// Hashed 8^3 blocks: chained buckets, chains sorted by key (builder-defined;
// oracle/orc_tsdf.hpp HashedVolumeT).  The hash table is the canonical
// structure; `grid` is a derived dense block-id index over a window of
// 2^gbits blocks per axis (centred on block 0) so in-window lookups are one
// load instead of a chain walk.  Blocks outside the window use the chains.
struct HashView {
  using Cache = NoCache;
  VoxelStore vox;
  const int* heads;
  const unsigned long long* keys;
  const int* next;
  const int* grid;
  const unsigned* occ;  // one bit per 8^3-block super-block of the window
  const unsigned char* sdist;  // Chebyshev distance to the nearest occupied super-block (0: occupied)
  unsigned mask;
  int gbits;
  double vs, ox, oy, oz, mu, cap;
  static constexpr bool kHashed = true;
  CSF_DEV bool cell_in_grid(int, int, int) const { return true; }
  CSF_DEV int find(int bx, int by, int bz) const {
    const unsigned long long key = block_key(bx, by, bz);
    int e = __ldg(heads + block_hash(bx, by, bz, mask));
    while (e >= 0) {
      const unsigned long long k = __ldg(keys + e);
      if (k == key) return e;
      if (k > key) return -1;
      e = __ldg(next + e);
    }
    return -1;
  }
  CSF_DEV int block(int bx, int by, int bz) const {
    const int half = 1 << (gbits - 1);
    const unsigned ux = static_cast<unsigned>(bx + half), uy = static_cast<unsigned>(by + half),
                   uz = static_cast<unsigned>(bz + half);
    const unsigned side = 1u << gbits;
    if (ux < side && uy < side && uz < side)
      return __ldg(grid + ((static_cast<size_t>(uz) << gbits | uy) << gbits | ux));
    return find(bx, by, bz);
  }
  // -1: super-block outside the window (unknown), 0: no allocated block in
  // it, 1: at least one.
  CSF_DEV int super_occupied(int bx, int by, int bz) const {
    const int half = 1 << (gbits - 1);
    const unsigned ux = static_cast<unsigned>(bx + half), uy = static_cast<unsigned>(by + half),
                   uz = static_cast<unsigned>(bz + half);
    const unsigned side = 1u << gbits;
    if (!(ux < side && uy < side && uz < side)) return -1;
    const int sb = gbits - 3;
    const unsigned bit = ((uz >> 3) << sb | (uy >> 3)) << sb | (ux >> 3);
    return (__ldg(occ + (bit >> 5)) >> (bit & 31)) & 1u;
  }
  // Block-occupancy pyramid below the super-block level: bitmaps at 4^3- and
  // 2^3-block granularity stored after the super-block bits in `occ`.
  // Returns the span (in blocks, 4 or 2) of the largest known-empty aligned
  // cell containing block (bx, by, bz), or 0 (occupied / outside the window).
  CSF_DEV int empty_span(int bx, int by, int bz) const {
    const int half = 1 << (gbits - 1);
    const unsigned ux = static_cast<unsigned>(bx + half), uy = static_cast<unsigned>(by + half),
                   uz = static_cast<unsigned>(bz + half);
    const unsigned side = 1u << gbits;
    if (!(ux < side && uy < side && uz < side)) return 0;
    const unsigned* occ4 = occ + ((1u << (3 * (gbits - 3))) >> 5);
    const unsigned* occ2 = occ4 + ((1u << (3 * (gbits - 2))) >> 5);
    const int s4 = gbits - 2, s2 = gbits - 1;
    const unsigned b4 = ((uz >> 2) << s4 | (uy >> 2)) << s4 | (ux >> 2);
    if (!((__ldg(occ4 + (b4 >> 5)) >> (b4 & 31)) & 1u)) return 4;
    const unsigned b2 = ((uz >> 1) << s2 | (uy >> 1)) << s2 | (ux >> 1);
    if (!((__ldg(occ2 + (b2 >> 5)) >> (b2 & 31)) & 1u)) return 2;
    return 0;
  }
  // All empty-space information of block (bx, by, bz): the super-block
  // distance, then (inside an occupied super-block) the 4^3- and 2^3-cell
  // bits and the block id issued together, so a march trip pays at most two
  // memory latencies instead of a chain of four.
  // sd: super_dist; es: empty_span; blk: block id (-1 unallocated).
  CSF_DEV void probe(int bx, int by, int bz, int* sd, int* es, int* blk) const {
    const int half = 1 << (gbits - 1);
    const unsigned ux = static_cast<unsigned>(bx + half), uy = static_cast<unsigned>(by + half),
                   uz = static_cast<unsigned>(bz + half);
    const unsigned side = 1u << gbits;
    if (!(ux < side && uy < side && uz < side)) {
      *sd = 0;
      *es = 0;
      *blk = find(bx, by, bz);
      return;
    }
    const int sb = gbits - 3, s4 = gbits - 2, s2 = gbits - 1;
    const unsigned* occ4 = occ + ((1u << (3 * sb)) >> 5);
    const unsigned* occ2 = occ4 + ((1u << (3 * s4)) >> 5);
    const unsigned bsb = ((uz >> 3) << sb | (uy >> 3)) << sb | (ux >> 3);
    const unsigned b4 = ((uz >> 2) << s4 | (uy >> 2)) << s4 | (ux >> 2);
    const unsigned b2 = ((uz >> 1) << s2 | (uy >> 1)) << s2 | (ux >> 1);
    const int d = __ldg(sdist + bsb);
    *sd = d;
    if (d > 0) {  // empty super-block neighbourhood: nothing finer needed
      *es = 0;
      *blk = -1;
      return;
    }
    const unsigned w4 = __ldg(occ4 + (b4 >> 5));
    const unsigned w2 = __ldg(occ2 + (b2 >> 5));
    const int id = __ldg(grid + ((static_cast<size_t>(uz) << gbits | uy) << gbits | ux));
    *es = !((w4 >> (b4 & 31)) & 1u) ? 4 : (!((w2 >> (b2 & 31)) & 1u) ? 2 : 0);
    *blk = id;
  }
  // probe() of the block of cell (i0, j0, k0) and the voxel ids of the cell's
  // 8 corners (-1: unallocated), every load issued in one round trip (the
  // march's in-band trips otherwise chain distance -> block id -> corner ids
  // -> voxels).  sd, es, blk: as probe().
  CSF_DEV void probe_cell(int i0, int j0, int k0, int* sd, int* es, int* blk, long long* v) const {
    const int half = 1 << (gbits - 1);
    const unsigned side = 1u << gbits;
    const unsigned ux = static_cast<unsigned>((i0 >> 3) + half), uy = static_cast<unsigned>((j0 >> 3) + half),
                   uz = static_cast<unsigned>((k0 >> 3) + half);
    const unsigned ux1 = static_cast<unsigned>(((i0 + 1) >> 3) + half), uy1 = static_cast<unsigned>(((j0 + 1) >> 3) + half),
                   uz1 = static_cast<unsigned>(((k0 + 1) >> 3) + half);
    if (!(ux < side && uy < side && uz < side && ux1 < side && uy1 < side && uz1 < side)) {
      probe(i0 >> 3, j0 >> 3, k0 >> 3, sd, es, blk);
#pragma unroll
      for (int c = 0; c < 8; ++c) v[c] = voxel(i0 + (c & 1), j0 + ((c >> 1) & 1), k0 + (c >> 2));
      return;
    }
    const int sb = gbits - 3, s4 = gbits - 2, s2 = gbits - 1;
    const unsigned* occ4 = occ + ((1u << (3 * sb)) >> 5);
    const unsigned* occ2 = occ4 + ((1u << (3 * s4)) >> 5);
    const unsigned bsb = ((uz >> 3) << sb | (uy >> 3)) << sb | (ux >> 3);
    const unsigned b4 = ((uz >> 2) << s4 | (uy >> 2)) << s4 | (ux >> 2);
    const unsigned b2 = ((uz >> 1) << s2 | (uy >> 1)) << s2 | (ux >> 1);
    const int d = __ldg(sdist + bsb);
    const unsigned w4 = __ldg(occ4 + (b4 >> 5));
    const unsigned w2 = __ldg(occ2 + (b2 >> 5));
    int g[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const unsigned cx = (c & 1) ? ux1 : ux, cy = ((c >> 1) & 1) ? uy1 : uy, cz = (c >> 2) ? uz1 : uz;
      g[c] = __ldg(grid + ((static_cast<size_t>(cz) << gbits | cy) << gbits | cx));
    }
    *sd = d;
    *es = d > 0 ? 0 : (!((w4 >> (b4 & 31)) & 1u) ? 4 : (!((w2 >> (b2 & 31)) & 1u) ? 2 : 0));
    *blk = d > 0 ? -1 : g[0];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int i = i0 + (c & 1), j = j0 + ((c >> 1) & 1), k = k0 + (c >> 2);
      v[c] = g[c] < 0 ? -1 : static_cast<long long>(g[c]) * kBlockVoxels + (((k & 7) * 8 + (j & 7)) * 8 + (i & 7));
    }
  }
  // d > 0: every super-block within Chebyshev distance d - 1 of this one is
  // inside the window and empty; 0: occupied or outside the window.
  CSF_DEV int super_dist(int bx, int by, int bz) const {
    const int half = 1 << (gbits - 1);
    const unsigned ux = static_cast<unsigned>(bx + half), uy = static_cast<unsigned>(by + half),
                   uz = static_cast<unsigned>(bz + half);
    const unsigned side = 1u << gbits;
    if (!(ux < side && uy < side && uz < side)) return 0;
    const int sb = gbits - 3;
    return __ldg(sdist + ((((uz >> 3) << sb | (uy >> 3)) << sb) | (ux >> 3)));
  }
  CSF_DEV long long voxel(int i, int j, int k) const {
    const int b = block(i >> 3, j >> 3, k >> 3);
    if (b < 0) return -1;
    return static_cast<long long>(b) * kBlockVoxels + (((k & 7) * 8 + (j & 7)) * 8 + (i & 7));
  }
  CSF_DEV long long voxel(int i, int j, int k, NoCache&) const { return voxel(i, j, k); }
};

// Stored field value of voxel v as S (channel group g0).
template <typename S> CSF_DEV S field_at(const VoxelStore& vs, long long v, double fre, int g0);
template <> CSF_DEV double field_at<double>(const VoxelStore&, long long, double fre, int) { return fre; }
template <typename S> CSF_DEV S field_at(const VoxelStore& vs, long long v, double fre, int g0) {
  S o;
  o.re = fre;
  const double* p = vs.fim + v * vs.Dp + g0;
#pragma unroll
  for (int g = 0; g < Traits<S>::G; ++g) o.im[g] = p[g];
  return o;
}

// sample_tsdf (tsdf.hpp:148-177): all 8 corners must exist with W > 0.
template <typename S, typename V>
CSF_DEV bool sample_tsdf(const V& vol, const V3<S>& p, int g0, S* out, typename V::Cache& cache) {
  const S gx = (p.v[0] - vol.ox) / vol.vs;
  const S gy = (p.v[1] - vol.oy) / vol.vs;
  const S gz = (p.v[2] - vol.oz) / vol.vs;
  const int i0 = ifloor(re(gx)), j0 = ifloor(re(gy)), k0 = ifloor(re(gz));
  if (!vol.cell_in_grid(i0, j0, k0)) return false;
  const S fx = gx - static_cast<double>(i0);
  const S fy = gy - static_cast<double>(j0);
  const S fz = gz - static_cast<double>(k0);
  // all eight corner lookups and loads are issued before any test; the
  // accumulation keeps the reference's dk, dj, di order (tsdf.hpp:163-176)
  long long v[8];
  bool ok = true;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    v[c] = vol.voxel(i0 + (c & 1), j0 + ((c >> 1) & 1), k0 + (c >> 2), cache);
    ok = ok && v[c] >= 0;
  }
  if (!ok) return false;
  double2 rw[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) rw[c] = vol.vox.rw[v[c]];
#pragma unroll
  for (int c = 0; c < 8; ++c) ok = ok && rw[c].y > 0.0;
  if (!ok) return false;
  if constexpr (Traits<S>::G == 0) {
    S accum = 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const double wx = (c & 1) ? fx : 1.0 - fx;
      const double wy = ((c >> 1) & 1) ? fy : 1.0 - fy;
      const double wz = (c >> 2) ? fz : 1.0 - fz;
      accum = accum + ((wx * wy) * wz) * rw[c].x;
    }
    *out = accum;
  } else if constexpr (Traits<S>::kOrder == 2) {
    // Second order: the reference's lifted accumulation, operation for
    // operation in Bicomplex arithmetic (no tangent shortcut at order 2).
    S accum = lit<S>(0.0);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const S wx = (c & 1) ? fx : 1.0 - fx;
      const S wy = ((c >> 1) & 1) ? fy : 1.0 - fy;
      const S wz = (c >> 2) ? fz : 1.0 - fz;
      accum = accum + ((wx * wy) * wz) * field_at<S>(vol.vox, v[c], rw[c].x, g0);
    }
    *out = accum;
  } else {
    // Real channel: the reference's accumulation (bit-identical).  Channels:
    // the interpolant is linear in the corner values and trilinear in the
    // cell fractions, so  im = sum_c w_c * F_c.im + (ds/dfx, ds/dfy, ds/dfz) . (fx, fy, fz).im
    // — the same first-order quantity with 11 instead of ~64 operations per
    // channel (rounding differs from the per-operation rule by ~1 ulp).
    const double fxr = fx.re, fyr = fy.re, fzr = fz.re;
    double acc = 0.0, dsx = 0.0, dsy = 0.0, dsz = 0.0;
    double wgt[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const double wx = (c & 1) ? fxr : 1.0 - fxr;
      const double wy = ((c >> 1) & 1) ? fyr : 1.0 - fyr;
      const double wz = (c >> 2) ? fzr : 1.0 - fzr;
      wgt[c] = (wx * wy) * wz;
      acc = acc + wgt[c] * rw[c].x;
      const double F = rw[c].x;
      dsx += ((c & 1) ? 1.0 : -1.0) * (wy * wz) * F;
      dsy += (((c >> 1) & 1) ? 1.0 : -1.0) * (wx * wz) * F;
      dsz += ((c >> 2) ? 1.0 : -1.0) * (wx * wy) * F;
    }
    S accum;
    accum.re = acc;
#pragma unroll
    for (int g = 0; g < Traits<S>::G; ++g) {
      double t = dsx * fx.im[g] + dsy * fy.im[g] + dsz * fz.im[g];
#pragma unroll
      for (int c = 0; c < 8; ++c) t += wgt[c] * vol.vox.fim[v[c] * vol.vox.Dp + g0 + g];
      accum.im[g] = t;
    }
    *out = accum;
  }
  return true;
}
template <typename S, typename V>
CSF_DEV bool sample_tsdf(const V& vol, const V3<S>& p, int g0, S* out) {
  NoCache c;
  return sample_tsdf<S>(vol, p, g0, out, c);
}

// sample_gradient (tsdf.hpp:181-196)
template <typename S, typename V>
CSF_DEV bool sample_gradient(const V& vol, const V3<S>& p, int g0, V3<S>* g, typename V::Cache& cache) {
  const double h = vol.vs;
#pragma unroll
  for (int axis = 0; axis < 3; ++axis) {
    V3<S> lo = p, hi = p;
    lo.v[axis] = lo.v[axis] - h;
    hi.v[axis] = hi.v[axis] + h;
    S flo, fhi;
    if (!sample_tsdf<S>(vol, lo, g0, &flo, cache)) return false;
    if (!sample_tsdf<S>(vol, hi, g0, &fhi, cache)) return false;
    g->v[axis] = (fhi - flo) / (2.0 * h);
  }
  return true;
}

// Lifted intrinsics of one pyramid level.
template <typename S> struct Intr {
  S fx, fy, cx, cy;
  int w, h;
};

// measured_tsdf (tsdf.hpp:97-140).  depth: the real depth image; dch
// (nullable): its perturbation channels [h*w][dstride] (a lifted depth image,
// "the depth image carries its own channels", tsdf.hpp:96-102 / 144-145),
// channel g of this channel group at dch[pixel * dstride + g0 + g].  Validity
// and the edge test read real corner depths; the bilinear sample carries the
// corners' channels (bilinear_depth<S>, frames.hpp:127-145).
template <typename S>
CSF_DEV bool measured_tsdf(const double* depth, int w, int h, const Pose<S>& w2c, const Intr<S>& k, double mu,
                           double px, double py, double pz, const V3<S>& center, S* psi,
                           const double* __restrict__ dch = nullptr, int dstride = 0, int g0 = 0) {
  V3<S> pc;
#pragma unroll
  for (int r = 0; r < 3; ++r)
    pc.v[r] = sum3(w2c.R.m[3 * r] * px, w2c.R.m[3 * r + 1] * py, w2c.R.m[3 * r + 2] * pz) + w2c.t.v[r];
  if (!(re(pc.v[2]) > 0.0)) return false;
  const S lx = (k.fx * pc.v[0]) / pc.v[2] + k.cx;
  const S ly = (k.fy * pc.v[1]) / pc.v[2] + k.cy;
  const int x0 = ifloor(re(lx)), y0 = ifloor(re(ly));
  if (x0 < 0 || y0 < 0 || x0 + 1 >= w || y0 + 1 >= h) return false;
  const double d00 = depth[y0 * w + x0];
  const double d10 = depth[y0 * w + x0 + 1];
  const double d01 = depth[(y0 + 1) * w + x0];
  const double d11 = depth[(y0 + 1) * w + x0 + 1];
  if (!(d00 > 0.0) || !(d10 > 0.0) || !(d01 > 0.0) || !(d11 > 0.0)) return false;
  const double nearv = fmin(fmin(d00, d10), fmin(d01, d11));
  const double farv = fmax(fmax(d00, d10), fmax(d01, d11));
  if (farv - nearv > 0.1) return false;
  const S fx = lx - static_cast<double>(x0);
  const S fy = ly - static_cast<double>(y0);
  S sampled;
  if constexpr (Traits<S>::G > 0) {
    if (dch) {
      auto corner = [&](int cx_, int cy_, double re_) {
        S c = lit<S>(re_);
        const double* src = dch + static_cast<long long>(cy_ * w + cx_) * dstride + g0;
#pragma unroll
        for (int g = 0; g < Traits<S>::G; ++g) c.im[g] = src[g];
        return c;
      };
      const S c00 = corner(x0, y0, d00), c10 = corner(x0 + 1, y0, d10);
      const S c01 = corner(x0, y0 + 1, d01), c11 = corner(x0 + 1, y0 + 1, d11);
      const S top = c00 + fx * (c10 - c00);
      const S bot = c01 + fx * (c11 - c01);
      sampled = top + fy * (bot - top);
    } else {
      const S top = d00 + fx * (d10 - d00);
      const S bot = d01 + fx * (d11 - d01);
      sampled = top + fy * (bot - top);
    }
  } else {
    const S top = d00 + fx * (d10 - d00);
    const S bot = d01 + fx * (d11 - d01);
    sampled = top + fy * (bot - top);
  }
  const S rx = (lx - k.cx) / k.fx;
  const S ry = (ly - k.cy) / k.fy;
  const S one = lit<S>(1.0);
  const S lambda = sqrt_s(sum3(rx * rx, ry * ry, one * one));
  const S dx = center.v[0] - px, dy = center.v[1] - py, dz = center.v[2] - pz;
  const S eta = sampled - sqrt_s(sum3(dx * dx, dy * dy, dz * dz)) / lambda;
  if (re(eta) < -mu) return false;
  *psi = clamp_s(eta / mu, -1.0, 1.0);
  return true;
}

// ----------------------------------------------------------------------------
// Ldlt6 — the oracle's restatement of Eigen::LDLT<Mat6d> (oracle/orc_icp.hpp)
// ----------------------------------------------------------------------------
CSF_HD int tri(int r, int c) { return r * (r + 1) / 2 + c; }

template <typename S> CSF_HD void swap_s(S& a, S& b) {
  const S t = a;
  a = b;
  b = t;
}
template <typename S> CSF_HD double absre(const S& x) { return fabs(re(x)); }

// Factor the symmetric matrix given by its lower triangle and solve A x = rhs.
// Returns false when Eigen would report info() != Success.  The pivoted
// (data-dependent) indexing runs on `ws`, a 48-scalar workspace the caller
// places in shared memory: m[36] (row-major), temp[6], x[6].
template <typename S>
CSF_DEV bool ldlt6_solve(const S* a_lower, const S* rhs, S* dst, S* ws) {
  S* m = ws;
  S* temp = ws + 36;
  S* x = ws + 42;
  int transp[6];
  bool ok = true;
#pragma unroll
  for (int r = 0; r < 6; ++r)
#pragma unroll
    for (int c = 0; c < 6; ++c) m[6 * r + c] = r >= c ? a_lower[tri(r, c)] : a_lower[tri(c, r)];
  for (int k = 0; k < 6; ++k) {
    int piv = k;
    double best = absre(m[7 * k]);
    for (int i = k + 1; i < 6; ++i)
      if (absre(m[7 * i]) > best) {
        best = absre(m[7 * i]);
        piv = i;
      }
    transp[k] = piv;
    if (piv != k) {
      for (int j = 0; j < k; ++j) swap_s(m[6 * k + j], m[6 * piv + j]);
      for (int i = piv + 1; i < 6; ++i) swap_s(m[6 * i + k], m[6 * i + piv]);
      swap_s(m[7 * k], m[7 * piv]);
      for (int i = k + 1; i < piv; ++i) {
        const S tmp = m[6 * i + k];
        m[6 * i + k] = m[6 * piv + i];
        m[6 * piv + i] = tmp;
      }
    }
    if (k > 0) {
      for (int j = 0; j < k; ++j) temp[j] = m[7 * j] * m[6 * k + j];
      S s = m[6 * k] * temp[0];
      for (int j = 1; j < k; ++j) s = s + m[6 * k + j] * temp[j];
      m[7 * k] = m[7 * k] - s;
      for (int i = k + 1; i < 6; ++i) {
        S si = m[6 * i] * temp[0];
        for (int j = 1; j < k; ++j) si = si + m[6 * i + j] * temp[j];
        m[6 * i + k] = m[6 * i + k] - si;
      }
    }
    const S akk = m[7 * k];
    const bool pivot_valid = absre(akk) > 0.0;
    if (k == 0 && !pivot_valid) {
      ok = false;
      for (int j = 0; j < 6; ++j) transp[j] = j;
      break;
    }
    if (k < 5) {
      if (pivot_valid) {
        for (int i = k + 1; i < 6; ++i) m[6 * i + k] = m[6 * i + k] / akk;
      } else {
        for (int i = k + 1; i < 6; ++i) ok = ok && re(m[6 * i + k]) == 0.0;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 6; ++i) x[i] = rhs[i];
  for (int k = 0; k < 6; ++k) swap_s(x[k], x[transp[k]]);
  for (int i = 0; i < 6; ++i)
    for (int j = i + 1; j < 6; ++j) x[j] = x[j] - x[i] * m[6 * j + i];
  const double tol = 2.2250738585072014e-308;  // numeric_limits<double>::min()
  for (int i = 0; i < 6; ++i) {
    if (absre(m[7 * i]) > tol)
      x[i] = x[i] / m[7 * i];
    else
      x[i] = lit<S>(0.0);
  }
  for (int i = 4; i >= 0; --i) {
    S s = m[6 * (i + 1) + i] * x[i + 1];
    for (int j = i + 2; j < 6; ++j) s = s + m[6 * j + i] * x[j];
    x[i] = x[i] - s;
  }
  for (int k = 5; k >= 0; --k) swap_s(x[k], x[transp[k]]);
#pragma unroll
  for (int i = 0; i < 6; ++i) dst[i] = x[i];
  return ok;
}

// Register-resident variant of ldlt6_solve: the same operations in the same
// order, with every loop fully unrolled and the pivot swaps expressed as
// predicated swaps over compile-time indices (no dynamic indexing, so the
// matrix never leaves registers).  Split into the factorization and the
// solve phase so the ICP solve can factor the real matrix once and apply
// the real factors to every channel's tangent right-hand side.
// `degenerate` (optional) reports a zero pivot or a pivot below the solve's
// tolerance — the cases where the solve is not the linear operator A^-1.
template <typename S>
CSF_HD bool ldlt6_factor_reg(const S* a_lower, S (&m)[6][6], int (&transp)[6], bool* degenerate = nullptr) {
  bool ok = true, stop = false, degen = false;
#pragma unroll
  for (int r = 0; r < 6; ++r)
#pragma unroll
    for (int c = 0; c < 6; ++c) m[r][c] = r >= c ? a_lower[tri(r, c)] : a_lower[tri(c, r)];
  S temp[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    if (stop) continue;
    int piv = k;
    double best = absre(m[k][k]);
#pragma unroll
    for (int i = k + 1; i < 6; ++i)
      if (absre(m[i][i]) > best) {
        best = absre(m[i][i]);
        piv = i;
      }
    transp[k] = piv;
#pragma unroll
    for (int i = k + 1; i < 6; ++i) {
      if (piv == i) {
#pragma unroll
        for (int j = 0; j < k; ++j) swap_s(m[k][j], m[i][j]);
#pragma unroll
        for (int r = i + 1; r < 6; ++r) swap_s(m[r][k], m[r][i]);
        swap_s(m[k][k], m[i][i]);
#pragma unroll
        for (int r = k + 1; r < i; ++r) {
          const S tmp = m[r][k];
          m[r][k] = m[i][r];
          m[i][r] = tmp;
        }
      }
    }
    if (k > 0) {
#pragma unroll
      for (int j = 0; j < k; ++j) temp[j] = m[j][j] * m[k][j];
      S sacc = m[k][0] * temp[0];
#pragma unroll
      for (int j = 1; j < k; ++j) sacc = sacc + m[k][j] * temp[j];
      m[k][k] = m[k][k] - sacc;
#pragma unroll
      for (int i = k + 1; i < 6; ++i) {
        S si = m[i][0] * temp[0];
#pragma unroll
        for (int j = 1; j < k; ++j) si = si + m[i][j] * temp[j];
        m[i][k] = m[i][k] - si;
      }
    }
    const S akk = m[k][k];
    const bool pivot_valid = absre(akk) > 0.0;
    if (!pivot_valid) degen = true;
    if (k == 0 && !pivot_valid) {
      ok = false;
#pragma unroll
      for (int j = 0; j < 6; ++j) transp[j] = j;
      stop = true;
      continue;
    }
    if (k < 5) {
      if (pivot_valid) {
#pragma unroll
        for (int i = k + 1; i < 6; ++i) m[i][k] = m[i][k] / akk;
      } else {
#pragma unroll
        for (int i = k + 1; i < 6; ++i) ok = ok && re(m[i][k]) == 0.0;
      }
    }
  }
  const double tol = 2.2250738585072014e-308;  // numeric_limits<double>::min()
#pragma unroll
  for (int i = 0; i < 6; ++i)
    if (!(absre(m[i][i]) > tol)) degen = true;
  if (degenerate) *degenerate = degen || stop;
  return ok;
}

// The solve phase of ldlt6_solve (transpositions, unit-lower forward
// substitution, diagonal, backward substitution, inverse transpositions).
// M may be the factor of the same scalar type or, for the tangent solve,
// plain double factors applied to a double right-hand side.
template <typename S, typename M>
CSF_HD void ldlt6_apply_reg(const M (&m)[6][6], const int (&transp)[6], const S* rhs, S* dst) {
  S x[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) x[i] = rhs[i];
#pragma unroll
  for (int k = 0; k < 6; ++k)
#pragma unroll
    for (int i = k + 1; i < 6; ++i)
      if (transp[k] == i) swap_s(x[k], x[i]);
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int j = i + 1; j < 6; ++j) x[j] = x[j] - x[i] * m[j][i];
  const double tol = 2.2250738585072014e-308;
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    if (absre(m[i][i]) > tol)
      x[i] = x[i] / m[i][i];
    else
      x[i] = lit<S>(0.0);
  }
#pragma unroll
  for (int i = 4; i >= 0; --i) {
    S sacc = m[i + 1][i] * x[i + 1];
#pragma unroll
    for (int j = i + 2; j < 6; ++j) sacc = sacc + m[j][i] * x[j];
    x[i] = x[i] - sacc;
  }
#pragma unroll
  for (int k = 5; k >= 0; --k)
#pragma unroll
    for (int i = k + 1; i < 6; ++i)
      if (transp[k] == i) swap_s(x[k], x[i]);
#pragma unroll
  for (int i = 0; i < 6; ++i) dst[i] = x[i];
}

template <typename S>
CSF_HD bool ldlt6_solve_reg(const S* a_lower, const S* rhs, S* dst) {
  S m[6][6];
  int transp[6];
  const bool ok = ldlt6_factor_reg<S>(a_lower, m, transp);
  ldlt6_apply_reg<S>(m, transp, rhs, dst);
  return ok;
}

// Real measured vertex at (x, y) (frames.hpp:38-41 via measure_surface).
CSF_DEV bool vertex_at(const double* depth, int w, int x, int y, double fx, double fy, double cx, double cy,
                       V3<double>* v) {
  const double d = depth[y * w + x];
  if (!(d > 0.0)) return false;
  *v = mk3<double>(d * (static_cast<double>(x) - cx) / fx, d * (static_cast<double>(y) - cy) / fy, d);
  return true;
}

// associate (icp.cpp:89-126) for one strided slot (x, y): the measured
// vertex/normal recomputed from the pyramid depth (measure_surface), the
// real-part gates in the reference's order (z > 0, bounds, model normal
// valid, distance, angle) and the lround pixel pick.  Returns true for a
// correspondence with model pixel (u, v).
CSF_DEV bool associate_slot(const double* __restrict__ depth, int w, int h, int x, int y, double fx, double fy,
                            double cx, double cy, const Pose<double>& c2w, const Pose<double>& w2p,
                            const double* __restrict__ vre, const double* __restrict__ nre, double d_max,
                            double cos_max, int* u_out, int* v_out, double* mv_out = nullptr,
                            double* mn_out = nullptr) {
  // the three depths are fetched together (one memory round trip), then the
  // validity tests run in the reference's order
  const double d0 = depth[y * w + x];
  const double d1 = x + 1 < w ? depth[y * w + x + 1] : 0.0;
  const double d2 = y + 1 < h ? depth[(y + 1) * w + x] : 0.0;
  if (!(d0 > 0.0 && x + 1 < w && y + 1 < h && d1 > 0.0 && d2 > 0.0)) return false;
  const double tx0 = static_cast<double>(x) - cx, tx1 = static_cast<double>(x + 1) - cx;
  const double ty0 = static_cast<double>(y) - cy, ty1 = static_cast<double>(y + 1) - cy;
  const V3<double> vert = mk3<double>(d0 * tx0 / fx, d0 * ty0 / fy, d0);
  const V3<double> vx = mk3<double>(d1 * tx1 / fx, d1 * ty0 / fy, d1);
  const V3<double> vy = mk3<double>(d2 * tx0 / fx, d2 * ty1 / fy, d2);
  V3<double> n = cross3(sub3(vx, vert), sub3(vy, vert));
  const double len2 = dot3(n, n);
  if (!(len2 > 0.0)) return false;
  const double l = sqrt(len2);
  n = mk3<double>(n.v[0] / l, n.v[1] / l, n.v[2] / l);
  if (dot3(n, vert) > 0.0) n = mk3<double>(-n.v[0], -n.v[1], -n.v[2]);
  if (!(dot3(n, n) > 0.5)) return false;
  const V3<double> world = apply(c2w, vert);
  const V3<double> inp = apply(w2p, world);
  if (!(inp.v[2] > 0.0)) return false;
  const double uvx = (fx * inp.v[0]) / inp.v[2] + cx;
  const double uvy = (fy * inp.v[1]) / inp.v[2] + cy;
  const int u = static_cast<int>(lround(uvx));
  const int v = static_cast<int>(lround(uvy));
  if (!(u >= 0 && u < w && v >= 0 && v < h)) return false;
  const long long m = static_cast<long long>(v) * w + u;
  // both model values are loaded together (one memory round trip); the
  // tests keep the reference's order (normal valid, then distance)
  const V3<double> mn = mk3<double>(nre[3 * m], nre[3 * m + 1], nre[3 * m + 2]);
  const V3<double> mv = mk3<double>(vre[3 * m], vre[3 * m + 1], vre[3 * m + 2]);
  if (!(dot3(mn, mn) > 0.5)) return false;
  const V3<double> dd = sub3(world, mv);
  if (sqrt(dot3(dd, dd)) > d_max) return false;
  const V3<double> wn = matvec(c2w.R, n);
  if (dot3(wn, mn) < cos_max) return false;
  *u_out = u;
  *v_out = v;
  if (mv_out)
#pragma unroll
    for (int k = 0; k < 3; ++k) mv_out[k] = mv.v[k];
  if (mn_out)
#pragma unroll
    for (int k = 0; k < 3; ++k) mn_out[k] = mn.v[k];
  return true;
}

}  // namespace csfd
