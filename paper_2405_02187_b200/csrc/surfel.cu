// Surfel (X-EF) front end on sm_100a (reference
// proj/include/csf/surfel.hpp, proj/src/surfel.cpp).
//
//   render_index_map  surfel.cpp:30-64  — project every surfel, key
//       (cell, depth, index); two stable CUB radix sorts (depth bits, then
//       cell) give the reference's std::sort order exactly; per-cell counts +
//       exclusive scan give the offsets.
//   associate_one_to_many  surfel.cpp:66-108 — one thread per pixel walks
//       the 16 cells of its 4x4 block in the reference's order; real-part
//       gates; count pass, exclusive scan, fill pass -> the (surfel, pixel,
//       lifted weight) list in pixel scan order, candidate order within.
//   update_surfels    surfel.cpp:121-236 — the list is stably radix-sorted
//       by surfel index, so each surfel's contributions form one segment in
//       the reference's accumulation order (pixel scan order); one thread
//       per touched surfel accumulates and commits once (the reference's
//       "accumulate in scan order, commit once per surfel"); unmatched
//       pixels are appended in scan order (flag / scan / scatter).
//   predict_maps      surfel.cpp:238-263 — nearest surfel per pixel by
//       atomicMin on the depth bits, then atomicMin on the index among the
//       surfels at that depth (the reference keeps the first minimum).
//
// Derivative channels: every lifted quantity is evaluated one channel per
// pass (S = L<1>, the reference's Complex), the real part shared; channel
// divisions are the reference's per-channel quotient (CSF_EXACT_CHANNELS),
// so every channel is bit-identical to a Complex pass of the reference.
#define CSF_EXACT_CHANNELS 1
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <vector>

#include "csf_internal.h"
#include "geometry.cuh"

namespace csfd {

template <int G> CSF_DEV L<G> exp_s(const L<G>& z) {
  const double f = csf_det::exp(z.re);
  return lift(z, f, f);
}
CSF_DEV double exp_s(double x) { return csf_det::exp(x); }

// surfel.cpp:110-119
CSF_DEV double sample_confidence_dev(double fx_unused, double cx, double cy, int w, int h, int x, int y) {
  (void)fx_unused;
  const double dx = static_cast<double>(x) - cx;
  const double dy = static_cast<double>(y) - cy;
  const double half_diagonal = 0.5 * sqrt(static_cast<double>(w) * w + static_cast<double>(h) * h);
  double g = sqrt(dx * dx + dy * dy) / half_diagonal;
  g = g < 0.0 ? 0.0 : (1.0 < g ? 1.0 : g);  // std::clamp(g, 0, 1)
  return csf_det::exp(-g * g / 0.72);
}

struct SurfCam {
  double R[9], t[3];  // real world->camera (index map / gates / prediction)
  double fx, fy, cx, cy;
  int w, h;
};

CSF_DEV V3<double> w2c_apply(const SurfCam& c, const V3<double>& p) {
  Pose<double> T;
#pragma unroll
  for (int e = 0; e < 9; ++e) T.R.m[e] = c.R[e];
#pragma unroll
  for (int e = 0; e < 3; ++e) T.t.v[e] = c.t[e];
  return apply(T, p);
}

CSF_DEV V3<double> real3(const double* a, long long i, int C) {
  return mk3<double>(a[(3 * i) * C], a[(3 * i + 1) * C], a[(3 * i + 2) * C]);
}

// ---------------------------------------------------------------------------
// render_index_map
// ---------------------------------------------------------------------------
__global__ void k_si_project(const double* __restrict__ pos, int n, int C, SurfCam cam,
                             unsigned* __restrict__ cellk, unsigned long long* __restrict__ depthk,
                             int* __restrict__ flag) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int W4 = 4 * cam.w, H4 = 4 * cam.h;
  unsigned cell = 0xffffffffu;
  unsigned long long dk = ~0ull;
  const V3<double> p = w2c_apply(cam, real3(pos, i, C));
  if (p.v[2] > 0.0) {
    const double px = (cam.fx * p.v[0]) / p.v[2] + cam.cx;  // project (frames.hpp:44-47)
    const double py = (cam.fy * p.v[1]) / p.v[2] + cam.cy;
    const int cx = static_cast<int>(floor((px + 0.5) * 4.0));  // supersample_cell (surfel.cpp:24-26)
    const int cy = static_cast<int>(floor((py + 0.5) * 4.0));
    if (!(cx < 0 || cy < 0 || cx >= W4 || cy >= H4)) {
      cell = static_cast<unsigned>(cy) * static_cast<unsigned>(W4) + static_cast<unsigned>(cx);
      dk = static_cast<unsigned long long>(__double_as_longlong(p.v[2]));  // z > 0: bits order as values
    }
  }
  cellk[i] = cell;
  depthk[i] = dk;
  flag[i] = cell != 0xffffffffu ? 1 : 0;
}

// visible surfels compacted in index order (the sorts then see only them)
__global__ void k_si_compact(const unsigned long long* __restrict__ depthk, const int* __restrict__ flag,
                             const int* __restrict__ fpos, int n, unsigned long long* __restrict__ dk_out,
                             int* __restrict__ idx_out) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !flag[i]) return;
  const int j = fpos[i];
  dk_out[j] = depthk[i];
  idx_out[j] = i;
}

__global__ void k_si_gather_cell(const unsigned* __restrict__ cellk, const int* __restrict__ idx, int n,
                                 unsigned* __restrict__ out, unsigned* __restrict__ counts) {
  pdl_wait();
  pdl_trigger();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const unsigned c = cellk[idx[j]];
  out[j] = c;
  if (c != 0xffffffffu) atomicAdd(&counts[c], 1u);
}

// ---------------------------------------------------------------------------
// association
// ---------------------------------------------------------------------------
// world-frame lifted vertex / normal per pixel (camera_to_world * v, R * n)
template <typename S>
__global__ void k_sf_world(const double* __restrict__ V, const double* __restrict__ N, int P, int D,
                           const double* __restrict__ c2w /*[12][C]*/, double* __restrict__ VW,
                           double* __restrict__ NW, int* __restrict__ valid) {
  pdl_wait();
  pdl_trigger();
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const int C = 1 + D;
  constexpr int G = Traits<S>::G;
  const double vz = V[(3LL * p + 2) * C];
  const V3<double> nre = real3(N, p, C);
  const bool ok = vz > 0.0 && dot3(nre, nre) > 0.5;  // vertex_valid / normal_valid (frames.hpp:73-81)
  valid[p] = ok ? 1 : 0;
  if (!ok) return;
  const int passes = G > 0 ? D : 1;
  for (int ch = 0; ch < passes; ++ch) {
    Pose<S> T;
#pragma unroll
    for (int e = 0; e < 9; ++e) T.R.m[e] = load_ch<S>(c2w + e * C, ch, G);
#pragma unroll
    for (int e = 0; e < 3; ++e) T.t.v[e] = load_ch<S>(c2w + (9 + e) * C, ch, G);
    V3<S> v, nn;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      v.v[c] = load_ch<S>(V + (3LL * p + c) * C, ch, G);
      nn.v[c] = load_ch<S>(N + (3LL * p + c) * C, ch, G);
    }
    const V3<S> vw = apply(T, v);
    const V3<S> nw = matvec(T.R, nn);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      store_ch<S>(VW + (3LL * p + c) * C, vw.v[c], ch, G, ch == 0);
      store_ch<S>(NW + (3LL * p + c) * C, nw.v[c], ch, G, ch == 0);
    }
  }
}

struct AssocGates {
  double depth, cos_gate, distance, kernel_scale;
  int one_to_many;
};

// fill == 0: counts[p] (+ merged); fill == 1: the lists at offs[p].
template <typename S>
__global__ void k_sf_assoc(const double* __restrict__ V, const double* __restrict__ VW, const double* __restrict__ NW,
                           const int* __restrict__ valid, int D, SurfCam cam, const unsigned* __restrict__ offsets,
                           const int* __restrict__ entries, const double* __restrict__ spos,
                           const double* __restrict__ snrm, AssocGates g, int fill, int* __restrict__ counts,
                           const int* __restrict__ offs, int* __restrict__ pidx, int* __restrict__ ppix,
                           double* __restrict__ pw, int* __restrict__ merged, int* __restrict__ cflag) {
  pdl_wait();
  pdl_trigger();
  const int P = cam.w * cam.h;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  bool merged_px = false;
  if (p < P) {
    const int C = 1 + D;
    constexpr int G = Traits<S>::G;
    int cnt = 0;
    if (valid[p]) {
      const int x = p % cam.w, y = p / cam.w;
      const V3<double> vre = real3(V, p, C);
      const double ray_depth = sqrt(dot3(vre, vre));
      const V3<double> ray_dir = mk3<double>(vre.v[0] / ray_depth, vre.v[1] / ray_depth, vre.v[2] / ray_depth);
      const V3<double> vwre = real3(VW, p, C), nwre = real3(NW, p, C);
      const int W4 = 4 * cam.w;
      int best = -1;
      double best_w = 0.0;
      int out = fill ? offs[p] : 0;
      for (int cy = 4 * y; cy < 4 * y + 4; ++cy)
        for (int cx = 4 * x; cx < 4 * x + 4; ++cx) {
          const unsigned cell = static_cast<unsigned>(cy) * W4 + cx;
          for (unsigned e = offsets[cell]; e < offsets[cell + 1]; ++e) {
            const int i = entries[e];
            const V3<double> s_pos = real3(spos, i, C);
            const V3<double> s_cam = w2c_apply(cam, s_pos);
            if (fabs(dot3(s_cam, ray_dir) - ray_depth) > g.depth) continue;
            if (dot3(real3(snrm, i, C), nwre) < g.cos_gate) continue;
            const V3<double> dd = sub3(s_pos, vwre);
            if (sqrt(dot3(dd, dd)) > g.distance) continue;
            if (!g.one_to_many) {
              // real weight of the candidate (the real channel of the lifted exp)
              const double wre = csf_det::exp(dot3(dd, dd) * g.kernel_scale);
              if (best < 0 || wre > best_w) {
                best = i;
                best_w = wre;
              }
              continue;
            }
            if (fill) {
              pidx[out] = i;
              ppix[out] = p;
              const int passes = G > 0 ? D : 1;
              for (int ch = 0; ch < passes; ++ch) {
                V3<S> off;
#pragma unroll
                for (int c = 0; c < 3; ++c)
                  off.v[c] = load_ch<S>(spos + (3LL * i + c) * C, ch, G) - load_ch<S>(VW + (3LL * p + c) * C, ch, G);
                const S w = exp_s(dot3(off, off) * g.kernel_scale);
                store_ch<S>(pw + static_cast<long long>(out) * C, w, ch, G, ch == 0);
              }
              ++out;
            }
            ++cnt;
          }
        }
      if (!g.one_to_many && best >= 0) {
        cnt = 1;
        if (fill) {
          const int i = best;
          pidx[out] = i;
          ppix[out] = p;
          const int passes = G > 0 ? D : 1;
          for (int ch = 0; ch < passes; ++ch) {
            V3<S> off;
#pragma unroll
            for (int c = 0; c < 3; ++c)
              off.v[c] = load_ch<S>(spos + (3LL * i + c) * C, ch, G) - load_ch<S>(VW + (3LL * p + c) * C, ch, G);
            const S w = exp_s(dot3(off, off) * g.kernel_scale);
            store_ch<S>(pw + static_cast<long long>(out) * C, w, ch, G, ch == 0);
          }
        }
      }
      merged_px = cnt > 0;
    }
    if (!fill) {
      counts[p] = cnt;
      cflag[p] = (valid[p] && cnt == 0) ? 1 : 0;
    }
  }
  if (!fill && merged) {
    const unsigned b = __ballot_sync(0xffffffffu, merged_px);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(merged, __popc(b));
  }
}

__global__ void k_sf_seg_count(const int* __restrict__ pidx, int T, int* __restrict__ seg) {
  pdl_wait();
  pdl_trigger();
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < T) atomicAdd(&seg[pidx[q]], 1);
}

struct CommitArgs {
  double radius_scale;
  int frame;
};

// One thread per surfel: accumulate its segment (pixel scan order) and
// commit once (surfel.cpp:170-224).  Channel passes run from the last to the
// first so the real parts (written by pass 0) are read before they change.
template <typename S>
__global__ void k_sf_commit(int n, int D, SurfCam cam, const int* __restrict__ seg_off, const int* __restrict__ order,
                            const int* __restrict__ ppix, const double* __restrict__ pw, const double* __restrict__ V,
                            const double* __restrict__ VW, const double* __restrict__ NW, CommitArgs a,
                            double* __restrict__ spos, double* __restrict__ snrm, double* __restrict__ sconf,
                            double* __restrict__ srad, int* __restrict__ sts) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int b = seg_off[i], e = seg_off[i + 1];
  if (b == e) return;
  const int C = 1 + D;
  constexpr int G = Traits<S>::G;
  const int passes = G > 0 ? D : 1;
  for (int ch = passes - 1; ch >= 0; --ch) {
    V3<S> ps = mk3<S>(lit<S>(0.0), lit<S>(0.0), lit<S>(0.0)), ns = ps;
    S wsum = lit<S>(0.0);
    double wre = 0.0, rsum = 0.0;
    for (int j = b; j < e; ++j) {
      const int q = order[j];
      const int p = ppix[q];
      const int x = p % cam.w, y = p / cam.w;
      const double conf = sample_confidence_dev(cam.fx, cam.cx, cam.cy, cam.w, cam.h, x, y);
      const double radius = a.radius_scale * V[(3LL * p + 2) * C];
      const S m = load_ch<S>(pw + static_cast<long long>(q) * C, ch, G) * conf;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        ps.v[c] = ps.v[c] + load_ch<S>(VW + (3LL * p + c) * C, ch, G) * m;
        ns.v[c] = ns.v[c] + load_ch<S>(NW + (3LL * p + c) * C, ch, G) * m;
      }
      wsum = wsum + m;
      wre += re(m);
      rsum += re(m) * radius;
    }
    const S c_old = load_ch<S>(sconf + static_cast<long long>(i) * C, ch, G);
    const S denom = c_old + wsum;
    V3<S> np, bl;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      np.v[c] = (load_ch<S>(spos + (3LL * i + c) * C, ch, G) * c_old + ps.v[c]) / denom;
      bl.v[c] = (load_ch<S>(snrm + (3LL * i + c) * C, ch, G) * c_old + ns.v[c]) / denom;
    }
    const S len2 = dot3(bl, bl);
    const bool renorm = re(len2) > 0.0;
    V3<S> nn = bl;
    if (renorm) {
      const S l = sqrt_s(len2);
#pragma unroll
      for (int c = 0; c < 3; ++c) nn.v[c] = bl.v[c] / l;
    }
    const bool last = ch == 0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      store_ch<S>(spos + (3LL * i + c) * C, np.v[c], ch, G, last);
      if (renorm) store_ch<S>(snrm + (3LL * i + c) * C, nn.v[c], ch, G, last);
    }
    store_ch<S>(sconf + static_cast<long long>(i) * C, denom, ch, G, last);
    if (last) {
      sts[i] = a.frame;
      const double r_old = srad[i];
      const double averaged = (re(c_old) * r_old + rsum) / (re(c_old) + wre);
      srad[i] = averaged < r_old ? averaged : r_old;  // std::min(radius, averaged)
    }
  }
}

// segments of the surfel-sorted pair list: flag[j] = first pair of a surfel
__global__ void k_sf_seg_flags(const int* __restrict__ key, int T, int* __restrict__ flag) {
  pdl_wait();
  pdl_trigger();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < T) flag[j] = (j == 0 || key[j] != key[j - 1]) ? 1 : 0;
}
__global__ void k_sf_seg_write(const int* __restrict__ key, const int* __restrict__ flag, const int* __restrict__ rank,
                               int T, int* __restrict__ ustart, int* __restrict__ usurf) {
  pdl_wait();
  pdl_trigger();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= T) return;
  if (flag[j]) {
    ustart[rank[j]] = j;
    usurf[rank[j]] = key[j];
  }
  if (j == T - 1) ustart[rank[j] + flag[j]] = T;
}

// lifted value from a cached real part and the channel ch read from memory
template <typename S> CSF_DEV S with_re(const double* base, double r, int ch);
template <> CSF_DEV double with_re<double>(const double*, double r, int) { return r; }
template <> CSF_DEV L<1> with_re<L<1>>(const double* base, double r, int ch) {
  L<1> o;
  o.re = r;
  o.im[0] = base[1 + ch];
  return o;
}

// Commit over the touched surfels only: kLanes lanes per surfel, lane g
// evaluating channels g, g + kLanes, ... (one Complex pass each).  Every lane
// caches the surfel's old real state, the warp synchronises, then lane 0
// writes the new real parts while each lane writes only its own channels.
constexpr int kLanes = 8;
template <typename S>
__global__ void k_sf_commit_u(int U, int D, SurfCam cam, const int* __restrict__ ustart, const int* __restrict__ usurf,
                              const int* __restrict__ order, const int* __restrict__ ppix,
                              const double* __restrict__ pw, const double* __restrict__ V,
                              const double* __restrict__ VW, const double* __restrict__ NW, CommitArgs a,
                              double* __restrict__ spos, double* __restrict__ snrm, double* __restrict__ sconf,
                              double* __restrict__ srad, int* __restrict__ sts) {
  pdl_wait();
  pdl_trigger();
  const long long t = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const int u = static_cast<int>(t / kLanes), g = static_cast<int>(t % kLanes);
  const bool active = u < U;
  const int C = 1 + D;
  constexpr int G = Traits<S>::G;
  const int passes = G > 0 ? D : 1;
  int i = 0, b = 0, e = 0;
  double p_re[3] = {0, 0, 0}, n_re[3] = {0, 0, 0}, c_re = 0.0, r_old = 0.0;
  if (active) {
    i = usurf[u];
    b = ustart[u];
    e = ustart[u + 1];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      p_re[c] = spos[(3LL * i + c) * C];
      n_re[c] = snrm[(3LL * i + c) * C];
    }
    c_re = sconf[static_cast<long long>(i) * C];
    r_old = srad[i];
  }
  __syncwarp();
  if (!active) return;
  for (int ch = g; ch < passes; ch += kLanes) {
    V3<S> ps = mk3<S>(lit<S>(0.0), lit<S>(0.0), lit<S>(0.0)), ns = ps;
    S wsum = lit<S>(0.0);
    double wre = 0.0, rsum = 0.0;
    for (int j = b; j < e; ++j) {
      const int q = order[j];
      const int p = ppix[q];
      const int x = p % cam.w, y = p / cam.w;
      const double conf = sample_confidence_dev(cam.fx, cam.cx, cam.cy, cam.w, cam.h, x, y);
      const S m = load_ch<S>(pw + static_cast<long long>(q) * C, ch, G) * conf;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        ps.v[c] = ps.v[c] + load_ch<S>(VW + (3LL * p + c) * C, ch, G) * m;
        ns.v[c] = ns.v[c] + load_ch<S>(NW + (3LL * p + c) * C, ch, G) * m;
      }
      wsum = wsum + m;
      if (ch == 0) {
        const double radius = a.radius_scale * V[(3LL * p + 2) * C];
        wre += re(m);
        rsum += re(m) * radius;
      }
    }
    const S c_old = with_re<S>(sconf + static_cast<long long>(i) * C, c_re, ch);
    const S denom = c_old + wsum;
    V3<S> np, bl;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      np.v[c] = (with_re<S>(spos + (3LL * i + c) * C, p_re[c], ch) * c_old + ps.v[c]) / denom;
      bl.v[c] = (with_re<S>(snrm + (3LL * i + c) * C, n_re[c], ch) * c_old + ns.v[c]) / denom;
    }
    const S len2 = dot3(bl, bl);
    const bool renorm = re(len2) > 0.0;
    V3<S> nn = bl;
    if (renorm) {
      const S l = sqrt_s(len2);
#pragma unroll
      for (int c = 0; c < 3; ++c) nn.v[c] = bl.v[c] / l;
    }
    const bool first = ch == 0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      store_ch<S>(spos + (3LL * i + c) * C, np.v[c], ch, G, first);
      if (renorm) store_ch<S>(snrm + (3LL * i + c) * C, nn.v[c], ch, G, first);
    }
    store_ch<S>(sconf + static_cast<long long>(i) * C, denom, ch, G, first);
    if (first) {
      sts[i] = a.frame;
      const double averaged = (c_re * r_old + rsum) / (c_re + wre);
      srad[i] = averaged < r_old ? averaged : r_old;  // std::min(radius, averaged)
    }
  }
}

// unmatched valid pixels appended in scan order (surfel.cpp:226-235)
__global__ void k_sf_create(const int* __restrict__ cflag, const int* __restrict__ crank, int P, int n0, int D,
                            SurfCam cam, CommitArgs a, const double* __restrict__ V, const double* __restrict__ VW,
                            const double* __restrict__ NW, double* __restrict__ spos, double* __restrict__ snrm,
                            double* __restrict__ sconf, double* __restrict__ srad, int* __restrict__ sts) {
  pdl_wait();
  pdl_trigger();
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P || !cflag[p]) return;
  const int C = 1 + D;
  const long long i = n0 + crank[p];
  for (int k = 0; k < 3 * C; ++k) {
    spos[3 * i * C + k] = VW[3LL * p * C + k];
    snrm[3 * i * C + k] = NW[3LL * p * C + k];
  }
  const int x = p % cam.w, y = p / cam.w;
  sconf[i * C] = sample_confidence_dev(cam.fx, cam.cx, cam.cy, cam.w, cam.h, x, y);
  for (int c = 1; c < C; ++c) sconf[i * C + c] = 0.0;
  srad[i] = a.radius_scale * V[(3LL * p + 2) * C];
  sts[i] = a.frame;
}

// ---------------------------------------------------------------------------
// predict_maps
// ---------------------------------------------------------------------------
CSF_DEV bool pred_pixel(const SurfCam& cam, const double* pos, int i, int C, int* pix, double* z) {
  const V3<double> c = w2c_apply(cam, real3(pos, i, C));
  if (!(c.v[2] > 0.0)) return false;
  const double px = (cam.fx * c.v[0]) / c.v[2] + cam.cx;
  const double py = (cam.fy * c.v[1]) / c.v[2] + cam.cy;
  const int x = static_cast<int>(lround(px)), y = static_cast<int>(lround(py));
  if (x < 0 || y < 0 || x >= cam.w || y >= cam.h) return false;
  *pix = y * cam.w + x;
  *z = c.v[2];
  return true;
}

__global__ void k_pred_z(const double* __restrict__ pos, int n, int C, SurfCam cam,
                         unsigned long long* __restrict__ zbest) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  int pix;
  double z;
  if (i < n && pred_pixel(cam, pos, i, C, &pix, &z))
    atomicMin(&zbest[pix], static_cast<unsigned long long>(__double_as_longlong(z)));
}

__global__ void k_pred_idx(const double* __restrict__ pos, int n, int C, SurfCam cam,
                           const unsigned long long* __restrict__ zbest, int* __restrict__ ibest) {
  pdl_wait();
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  int pix;
  double z;
  if (i < n && pred_pixel(cam, pos, i, C, &pix, &z) &&
      static_cast<unsigned long long>(__double_as_longlong(z)) == zbest[pix])
    atomicMin(&ibest[pix], i);
}

__global__ void k_pred_write(const int* __restrict__ ibest, int P, int C, const double* __restrict__ pos,
                             const double* __restrict__ nrm, double* __restrict__ Vo, double* __restrict__ No) {
  pdl_wait();
  pdl_trigger();
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const int i = ibest[p];
  const bool hit = i != 0x7fffffff;
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    Vo[3LL * p + c] = hit ? pos[(3LL * i + c) * C] : 0.0;
    No[3LL * p + c] = hit ? nrm[(3LL * i + c) * C] : 0.0;
  }
}

__global__ void k_fill_u64(unsigned long long* a, int n, unsigned long long v) {
  pdl_wait();  // PDL-launched: order against the previous kernel on the stream
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = v;
}
// real depth [P] -> lifted depth [P][C] with zero channels
__global__ void k_expand_depth(const double* __restrict__ real, long long P, int C, double* __restrict__ lifted) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= P * C) return;
  const long long p = i / C;
  lifted[i] = (i % C) == 0 ? real[p] : 0.0;
}

__global__ void k_fill_iota(int* a, int n) {
  pdl_wait();  // PDL-launched: order against the previous kernel on the stream
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = i;
}
__global__ void k_fill_i32(int* a, int n, int v) {
  pdl_wait();  // PDL-launched: order against the previous kernel on the stream
  pdl_trigger();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = v;
}

}  // namespace csfd

// ============================================================================
namespace csfi {

using namespace csfd;

static void chk(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) note_launch_error(what, e);
}

template <typename T>
static cudaError_t grow(T*& p, size_t& cap, size_t need) {
  if (need <= cap && p) return cudaSuccess;
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
  // headroom: the map grows every frame; re-allocating (and the implicit
  // device synchronisation of cudaFree) per frame would dominate
  const size_t want = need + need / 2 + 1024;
  const cudaError_t e = cudaMalloc(&p, sizeof(T) * want);
  if (e == cudaSuccess) cap = want;
  return e;
}

static SurfCam make_cam(const double* c2w12, const double* k4, int w, int h) {
  // real_pose(camera_to_world).inverse() = (R^T, -(R^T t)) (se3.hpp; oracle PoseT::inverse)
  SurfCam c;
  Pose<double> T;
  for (int e = 0; e < 9; ++e) T.R.m[e] = c2w12[e];
  for (int e = 0; e < 3; ++e) T.t.v[e] = c2w12[9 + e];
  const Pose<double> inv = inverse(T);
  for (int e = 0; e < 9; ++e) c.R[e] = inv.R.m[e];
  for (int e = 0; e < 3; ++e) c.t[e] = inv.t.v[e];
  c.fx = k4[0];
  c.fy = k4[1];
  c.cx = k4[2];
  c.cy = k4[3];
  c.w = w;
  c.h = h;
  return c;
}

static int grid1(long long n, int b = 256) { return static_cast<int>(std::max<long long>(1, (n + b - 1) / b)); }

// Builds the index map of the first n surfels into ws.offsets [16 w h + 1] /
// ws.entries [m] (device).  Returns 0/4/5; *m_out = entries.
int surfel_index_map(cudaStream_t s, SurfelScratch& ws, const double* pos, int n, int D, const double* c2w12,
                     const double* k4, int w, int h, int* m_out) {
  const int C = 1 + D;
  const SurfCam cam = make_cam(c2w12, k4, w, h);
  const size_t cells = static_cast<size_t>(16) * w * h;
  const size_t nn = static_cast<size_t>(std::max(n, 1));
  if (grow(ws.offsets, ws.offsets_cap, cells + 1) || grow(ws.cellk, ws.cellk_cap, 2 * nn) ||
      grow(ws.depthk, ws.depthk_cap, 3 * nn) || grow(ws.sidx, ws.sidx_cap, 4 * nn))
    return 5;
  unsigned* cellA = ws.cellk;       // per surfel
  unsigned* cellB = ws.cellk + nn;  // compacted, depth order / then sorted by cell
  unsigned long long* d0 = ws.depthk;
  unsigned long long* d1 = ws.depthk + nn;
  unsigned long long* d2 = ws.depthk + 2 * nn;
  int* iA = ws.sidx;
  int* iB = ws.sidx + nn;
  int* flag = ws.sidx + 2 * nn;
  int* fpos = ws.sidx + 3 * nn;
  size_t t0 = 0, t3 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t0, flag, fpos, static_cast<int>(nn), s);
  cub::DeviceScan::ExclusiveSum(nullptr, t3, ws.offsets, ws.offsets, static_cast<int>(cells + 1), s);
  if (grow(ws.cub, ws.cub_cap, std::max(t0, t3))) return 5;
  cudaMemsetAsync(ws.offsets, 0, sizeof(unsigned) * (cells + 1), s);
  int m = 0;
  if (n > 0) {
    launch_pdl(k_si_project, dim3(grid1(n)), dim3(256), 0, s, pos, n, C, cam, cellA, d0, flag);
    size_t b0 = ws.cub_cap;
    cub::DeviceScan::ExclusiveSum(ws.cub, b0, flag, fpos, n, s);
    launch_pdl(k_si_compact, dim3(grid1(n)), dim3(256), 0, s, static_cast<const unsigned long long*>(d0),
               static_cast<const int*>(flag), static_cast<const int*>(fpos), n, d1, iA);
    int hv[2];
    cudaMemcpyAsync(&hv[0], fpos + n - 1, sizeof(int), cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(&hv[1], flag + n - 1, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) return 4;
    m = hv[0] + hv[1];
  }
  if (m > 0) {
    size_t t1 = 0, t2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, t1, d1, d2, iA, iB, m, 0, 64, s);
    cub::DeviceRadixSort::SortPairs(nullptr, t2, cellB, cellB, iB, iA, m, 0, 32, s);
    if (grow(ws.cub, ws.cub_cap, std::max(t1, t2))) return 5;
    int bits = 1;  // cell keys < 16 w h
    while (bits < 32 && (static_cast<size_t>(1) << bits) < cells) ++bits;
    size_t b1 = ws.cub_cap;
    cub::DeviceRadixSort::SortPairs(ws.cub, b1, d1, d2, iA, iB, m, 0, 64, s);  // by depth (stable: index order)
    launch_pdl(k_si_gather_cell, dim3(grid1(m)), dim3(256), 0, s, static_cast<const unsigned*>(cellA),
               static_cast<const int*>(iB), m, cellB, ws.offsets);
    unsigned* cellC = reinterpret_cast<unsigned*>(d0);  // d0 is free after the compaction
    size_t b2 = ws.cub_cap;
    cub::DeviceRadixSort::SortPairs(ws.cub, b2, cellB, cellC, iB, iA, m, 0, bits, s);  // then by cell (stable)
  }
  size_t b3 = ws.cub_cap;
  cub::DeviceScan::ExclusiveSum(ws.cub, b3, ws.offsets, ws.offsets, static_cast<int>(cells + 1), s);
  ws.entries = iA;  // the m sorted surfel indices
  chk("surfel_index_map");
  *m_out = m;
  return 0;
}

// Association over all pixels (surfel.cpp:66-108 batched): after
// surfel_index_map.  depth [P][C], c2w [12][C] (device); fills ws.V/N/VW/NW,
// ws.counts/offs/cflag and (fill) the pair lists.  *total pairs, *merged.
int surfel_associate(cudaStream_t s, SurfelScratch& ws, const double* spos, const double* snrm, int D,
                     const double* depth, const double* c2w, const double* intr_lifted, const double* c2w12,
                     const double* k4, int w, int h, const AssocParams& ap, int* total, int* merged) {
  const int C = 1 + D;
  const int P = w * h;
  const SurfCam cam = make_cam(c2w12, k4, w, h);
  if (grow(ws.V, ws.V_cap, 3 * static_cast<size_t>(P) * C) || grow(ws.N, ws.N_cap, 3 * static_cast<size_t>(P) * C) ||
      grow(ws.VW, ws.VW_cap, 3 * static_cast<size_t>(P) * C) ||
      grow(ws.NW, ws.NW_cap, 3 * static_cast<size_t>(P) * C) || grow(ws.pint, ws.pint_cap, 5 * static_cast<size_t>(P) + 8))
    return 5;
  int* valid = ws.pint;
  int* counts = valid + P;
  int* offs = counts + P;
  int* cflag = offs + P;
  int* crank = cflag + P;
  int* d_merged = crank + P;
  size_t t1 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t1, counts, offs, P, s);
  if (grow(ws.cub, ws.cub_cap, t1)) return 5;
  const Launch lch{s, nullptr, &ws.launches};
  launch_measure(lch, depth, w, h, intr_lifted, D, ws.V, ws.N);
  if (D > 0)
    launch_pdl(k_sf_world<L<1>>, dim3(grid1(P)), dim3(256), 0, s, static_cast<const double*>(ws.V),
               static_cast<const double*>(ws.N), P, D, c2w, ws.VW, ws.NW, valid);
  else
    launch_pdl(k_sf_world<double>, dim3(grid1(P)), dim3(256), 0, s, static_cast<const double*>(ws.V),
               static_cast<const double*>(ws.N), P, D, c2w, ws.VW, ws.NW, valid);
  cudaMemsetAsync(d_merged, 0, sizeof(int), s);
  AssocGates g{ap.depth, ap.cos_gate, ap.distance, ap.kernel_scale, ap.one_to_many};
  auto assoc = [&](int fill) {
    if (D > 0)
      launch_pdl(k_sf_assoc<L<1>>, dim3(grid1(P)), dim3(256), 0, s, static_cast<const double*>(ws.V),
                 static_cast<const double*>(ws.VW), static_cast<const double*>(ws.NW),
                 static_cast<const int*>(valid), D, cam, static_cast<const unsigned*>(ws.offsets),
                 static_cast<const int*>(ws.entries), spos, snrm, g, fill, counts, static_cast<const int*>(offs),
                 ws.pidx, ws.ppix, ws.pw, d_merged, cflag);
    else
      launch_pdl(k_sf_assoc<double>, dim3(grid1(P)), dim3(256), 0, s, static_cast<const double*>(ws.V),
                 static_cast<const double*>(ws.VW), static_cast<const double*>(ws.NW),
                 static_cast<const int*>(valid), D, cam, static_cast<const unsigned*>(ws.offsets),
                 static_cast<const int*>(ws.entries), spos, snrm, g, fill, counts, static_cast<const int*>(offs),
                 ws.pidx, ws.ppix, ws.pw, d_merged, cflag);
  };
  assoc(0);
  size_t b = ws.cub_cap;
  cub::DeviceScan::ExclusiveSum(ws.cub, b, counts, offs, P, s);
  b = ws.cub_cap;
  cub::DeviceScan::ExclusiveSum(ws.cub, b, cflag, crank, P, s);
  int hv[4];
  cudaMemcpyAsync(&hv[0], offs + P - 1, sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&hv[1], counts + P - 1, sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&hv[2], d_merged, sizeof(int), cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return 4;
  const int T = hv[0] + hv[1];
  if (grow(ws.pidx, ws.pidx_cap, 2 * static_cast<size_t>(T) + 2) || grow(ws.ppix, ws.ppix_cap, static_cast<size_t>(T) + 1) ||
      grow(ws.pw, ws.pw_cap, static_cast<size_t>(T) * C + 1))
    return 5;
  if (T > 0) assoc(1);
  chk("surfel_associate");
  *total = T;
  *merged = hv[2];
  return 0;
}

int surfel_created_count(cudaStream_t s, SurfelScratch& ws, int P, int* created) {
  const int* cflag = ws.pint + 3 * P;
  const int* crank = ws.pint + 4 * P;
  int hv[2];
  cudaMemcpyAsync(&hv[0], crank + P - 1, sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&hv[1], cflag + P - 1, sizeof(int), cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return 4;
  *created = hv[0] + hv[1];
  return 0;
}

// Commit the association of the last surfel_associate into the first n
// surfels and append the created ones at n (capacity checked by the caller).
int surfel_commit(cudaStream_t s, SurfelScratch& ws, SurfelArrays m, int n, int D, int T, const double* c2w12,
                  const double* k4, int w, int h, int frame, double radius_scale) {
  const int C = 1 + D;
  const int P = w * h;
  const SurfCam cam = make_cam(c2w12, k4, w, h);
  const size_t TT = static_cast<size_t>(std::max(T, 1));
  if (grow(ws.seg, ws.seg_cap, 4 * TT + 2)) return 5;
  int* sorted_idx = ws.pidx + T;  // second half of pidx
  if (grow(ws.order, ws.order_cap, 2 * TT + 2)) return 5;
  int* qin = ws.order;
  int* qout = ws.order + T;
  int* flag = ws.seg;
  int* rank = ws.seg + TT;
  int* ustart = ws.seg + 2 * TT;
  int* usurf = ws.seg + 3 * TT + 1;
  size_t t1 = 0, t2 = 0;
  int bits = 1;
  while (bits < 31 && (1 << bits) < n) ++bits;
  cub::DeviceRadixSort::SortPairs(nullptr, t1, ws.pidx, sorted_idx, qin, qout, static_cast<int>(TT), 0, bits, s);
  cub::DeviceScan::ExclusiveSum(nullptr, t2, flag, rank, static_cast<int>(TT), s);
  if (grow(ws.cub, ws.cub_cap, std::max(t1, t2))) return 5;
  const CommitArgs a{radius_scale, frame};
  if (T > 0) {
    launch_pdl(k_fill_iota, dim3(grid1(T)), dim3(256), 0, s, qin, T);
    size_t b = ws.cub_cap;
    cub::DeviceRadixSort::SortPairs(ws.cub, b, ws.pidx, sorted_idx, qin, qout, T, 0, bits, s);  // stable by surfel
    launch_pdl(k_sf_seg_flags, dim3(grid1(T)), dim3(256), 0, s, static_cast<const int*>(sorted_idx), T, flag);
    b = ws.cub_cap;
    cub::DeviceScan::ExclusiveSum(ws.cub, b, flag, rank, T, s);
    launch_pdl(k_sf_seg_write, dim3(grid1(T)), dim3(256), 0, s, static_cast<const int*>(sorted_idx),
               static_cast<const int*>(flag), static_cast<const int*>(rank), T, ustart, usurf);
    int hv[2];
    cudaMemcpyAsync(&hv[0], rank + T - 1, sizeof(int), cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(&hv[1], flag + T - 1, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) return 4;
    const int U = hv[0] + hv[1];
    const long long threads = static_cast<long long>(U) * kLanes;
    if (D > 0)
      launch_pdl(k_sf_commit_u<L<1>>, dim3(grid1(threads, 128)), dim3(128), 0, s, U, D, cam,
                 static_cast<const int*>(ustart), static_cast<const int*>(usurf), static_cast<const int*>(qout),
                 static_cast<const int*>(ws.ppix), static_cast<const double*>(ws.pw), static_cast<const double*>(ws.V),
                 static_cast<const double*>(ws.VW), static_cast<const double*>(ws.NW), a, m.pos, m.nrm, m.conf, m.rad,
                 m.ts);
    else
      launch_pdl(k_sf_commit_u<double>, dim3(grid1(threads, 128)), dim3(128), 0, s, U, D, cam,
                 static_cast<const int*>(ustart), static_cast<const int*>(usurf), static_cast<const int*>(qout),
                 static_cast<const int*>(ws.ppix), static_cast<const double*>(ws.pw), static_cast<const double*>(ws.V),
                 static_cast<const double*>(ws.VW), static_cast<const double*>(ws.NW), a, m.pos, m.nrm, m.conf, m.rad,
                 m.ts);
  }
  launch_pdl(k_sf_create, dim3(grid1(P)), dim3(256), 0, s, static_cast<const int*>(ws.pint + 3 * P),
             static_cast<const int*>(ws.pint + 4 * P), P, n, D, cam, a, static_cast<const double*>(ws.V),
             static_cast<const double*>(ws.VW), static_cast<const double*>(ws.NW), m.pos, m.nrm, m.conf, m.rad, m.ts);
  chk("surfel_commit");
  (void)C;
  return 0;
}

int surfel_predict(cudaStream_t s, SurfelScratch& ws, const double* pos, const double* nrm, int n, int D,
                   const double* c2w12, const double* k4, int w, int h, double* Vo, double* No) {
  const int C = 1 + D;
  const int P = w * h;
  const SurfCam cam = make_cam(c2w12, k4, w, h);
  if (grow(ws.zbest, ws.zbest_cap, static_cast<size_t>(P)) || grow(ws.ibest, ws.ibest_cap, static_cast<size_t>(P)))
    return 5;
  launch_pdl(k_fill_u64, dim3(grid1(P)), dim3(256), 0, s, ws.zbest, P, ~0ull);
  launch_pdl(k_fill_i32, dim3(grid1(P)), dim3(256), 0, s, ws.ibest, P, 0x7fffffff);
  if (n > 0) {
    launch_pdl(k_pred_z, dim3(grid1(n)), dim3(256), 0, s, pos, n, C, cam, ws.zbest);
    launch_pdl(k_pred_idx, dim3(grid1(n)), dim3(256), 0, s, pos, n, C, cam,
               static_cast<const unsigned long long*>(ws.zbest), ws.ibest);
  }
  launch_pdl(k_pred_write, dim3(grid1(P)), dim3(256), 0, s, static_cast<const int*>(ws.ibest), P, C, pos, nrm, Vo, No);
  chk("surfel_predict");
  return 0;
}

void launch_expand_depth(cudaStream_t s, const double* real, long long P, int C, double* lifted) {
  const long long n = P * C;
  if (n > 0) k_expand_depth<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(real, P, C, lifted);
  chk("expand_depth");
}

void surfel_scratch_release(SurfelScratch& ws) {
  cudaFree(ws.offsets);
  cudaFree(ws.cellk);
  cudaFree(ws.depthk);
  cudaFree(ws.sidx);
  cudaFree(ws.cub);
  cudaFree(ws.V);
  cudaFree(ws.N);
  cudaFree(ws.VW);
  cudaFree(ws.NW);
  cudaFree(ws.pint);
  cudaFree(ws.pidx);
  cudaFree(ws.ppix);
  cudaFree(ws.pw);
  cudaFree(ws.seg);
  cudaFree(ws.order);
  cudaFree(ws.zbest);
  cudaFree(ws.ibest);
  ws = SurfelScratch{};
}

}  // namespace csfi
