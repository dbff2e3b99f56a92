// TSDF kernels for sm_100a: fusion (dense lattice and hashed 8^3 blocks),
// hashed-block allocation, and raycast surface prediction.
//
//   surface_update / measured_tsdf — proj/src/tsdf.cpp:11-40, tsdf.hpp:97-140
//   sample_tsdf / sample_gradient  — proj/include/csf/tsdf.hpp:148-196
//   raycast                        — proj/include/csf/tsdf.hpp:209-284
//   hashed allocation              — builder-defined (oracle/orc_tsdf.hpp)
//
// Layout: rw[v] = (F.re, W) as one 16 B load, perturbation channels
// fim[v*Dp + d] voxel-major / channel-minor so a fused voxel's channel group
// is one contiguous run.  The raycast march reads only rw (the real channel
// decides every branch); channels are gathered once per hit pixel.
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "csf_internal.h"
#include "geometry.cuh"

namespace csfd {

// ----------------------------------------------------------------------------
// block prologue: the frame's pose (c2w) -> w2c per channel group in smem
// layout in smem: w2c[12][1+Dp], center[3][1+Dp], intr[4][1+Dp]
// ----------------------------------------------------------------------------
template <typename S>
__device__ void stage_pose_w2c(const double* __restrict__ pose, const double* __restrict__ intr, int Dp, double* sm) {
  constexpr int G = Traits<S>::G;
  const int C = 1 + Dp;
  const int ngroups = G == 0 ? 1 : Dp / G;
  double* w2c = sm;
  double* center = sm + 12 * C;
  double* kk = sm + 15 * C;
  for (int i = threadIdx.x; i < 4 * C; i += blockDim.x) kk[i] = intr[i];
  for (int i = threadIdx.x; i < 3 * C; i += blockDim.x) center[i] = pose[9 * C + i];
  for (int gi = threadIdx.x; gi < ngroups; gi += blockDim.x) {
    const int g0 = gi * G;
    Pose<S> c2w;
#pragma unroll
    for (int e = 0; e < 9; ++e) c2w.R.m[e] = load_ch<S>(pose + e * C, g0, G);
#pragma unroll
    for (int e = 0; e < 3; ++e) c2w.t.v[e] = load_ch<S>(pose + (9 + e) * C, g0, G);
    const Pose<S> inv = inverse(c2w);
#pragma unroll
    for (int e = 0; e < 9; ++e) store_ch<S>(w2c + e * C, inv.R.m[e], g0, G, gi == 0);
#pragma unroll
    for (int e = 0; e < 3; ++e) store_ch<S>(w2c + (9 + e) * C, inv.t.v[e], g0, G, gi == 0);
  }
  __syncthreads();
}

// The 19 x NDP channel block of the staged inputs, restaged contiguous and
// 16-byte aligned after them, so the fusion contraction reads two channels
// per shared-memory load (double2) instead of one.
__host__ __device__ constexpr int jac_offset(int C) { return (19 * C + 1) & ~1; }
template <int NDP>
CSF_DEV void stage_jacobian(double* sm) {
  if constexpr (NDP > 0 && NDP % 2 == 0) {
    constexpr int C = 1 + NDP;
    double* sj = sm + jac_offset(C);
    for (int i = threadIdx.x; i < 19 * NDP; i += blockDim.x) sj[i] = sm[(i / NDP) * C + 1 + i % NDP];
    __syncthreads();
  }
}
// staged inputs, plus the aligned channel block when the kernel restages it
// (first order, fixed even channel count)
static size_t integrate_smem(int Dp, bool jac) {
  return sizeof(double) * (jac ? jac_offset(1 + Dp) + 19 * Dp : 19 * (1 + Dp));
}

template <typename S>
__device__ void load_pose_intr(const double* sm, int Dp, int g0, Pose<S>* w2c, V3<S>* center, Intr<S>* k) {
  const int C = 1 + Dp;
  constexpr int G = Traits<S>::G;
#pragma unroll
  for (int e = 0; e < 9; ++e) w2c->R.m[e] = load_ch<S>(sm + e * C, g0, G);
#pragma unroll
  for (int e = 0; e < 3; ++e) w2c->t.v[e] = load_ch<S>(sm + (9 + e) * C, g0, G);
#pragma unroll
  for (int e = 0; e < 3; ++e) center->v[e] = load_ch<S>(sm + (12 + e) * C, g0, G);
  k->fx = load_ch<S>(sm + 15 * C, g0, G);
  k->fy = load_ch<S>(sm + 16 * C, g0, G);
  k->cx = load_ch<S>(sm + 17 * C, g0, G);
  k->cy = load_ch<S>(sm + 18 * C, g0, G);
}

// Fuse one voxel: the real pass decides validity, then every channel group
// re-evaluates psi (bit-identical real part) and updates its channels.
template <typename S>
__device__ bool fuse_voxel(const VoxelStore& vox, long long v, double px, double py, double pz,
                           const double* __restrict__ depth, int w, int h, double mu, double cap, int Dp,
                           const double* sm, const double* __restrict__ dch = nullptr) {
  constexpr int G = Traits<S>::G;
  const int passes = G == 0 ? 1 : Dp / G;
  double2 rw = make_double2(0.0, 0.0);
  double fre = 0.0;
  for (int gi = 0; gi < passes; ++gi) {
    const int g0 = gi * G;
    Pose<S> w2c;
    V3<S> c;
    Intr<S> k;
    load_pose_intr<S>(sm, Dp, g0, &w2c, &c, &k);
    S psi;
    // validity depends on real parts only: the first pass decides for all
    if (!measured_tsdf<S>(depth, w, h, w2c, k, mu, px, py, pz, c, &psi, dch, Dp, g0)) return false;
    if (gi == 0) rw = vox.rw[v];
    const S f = field_at<S>(vox, v, rw.x, g0);
    const S fn = (rw.y * f + psi) / (rw.y + 1.0);
    fre = re(fn);
    if constexpr (G > 0) {
      double* dst = vox.fim + v * vox.Dp + g0;
#pragma unroll
      for (int g = 0; g < G; ++g) dst[g] = fn.im[g];
    }
  }
  const double wn = rw.y + 1.0;
  vox.rw[v] = make_double2(fre, cap < wn ? cap : wn);
  return true;
}

#ifdef CSF_EXACT_CHANNELS
constexpr bool kAdjointFusion = false;
#else
constexpr bool kAdjointFusion = true;
#endif

// Count of fused voxels (bench's algorithmic-byte model): per-thread in a
// register, one warp-reduced atomic per warp at kernel end (a per-voxel-warp
// atomic on one address serialises ~3.4e5 atomics per frame in one L2 slice).
// (The generic lifted fusion keeps the in-loop warp-aggregated atomic: an
// extra live counter across its loop raised the order-2 kernel's spills from
// 124 to 332 bytes.)
CSF_DEV void count_updates(int* upd, bool fused) {
  if (!upd) return;
  const unsigned m = __activemask();
  const unsigned b = __ballot_sync(m, fused);
  if ((threadIdx.x & 31) == __ffs(m) - 1 && b) atomicAdd(upd, __popc(b));
}
CSF_DEV void flush_updates(int* upd, int count) {
  if (!upd) return;
  const int total = __reduce_add_sync(0xffffffffu, count);
  if ((threadIdx.x & 31) == 0 && total) atomicAdd(upd, total);
}

// Fusion with adjoint-form channels.  The real channel is the reference's
// chain (bit-identical to measured_tsdf<double> and the running average).
// Every perturbation channel of psi is a linear function of the channels of
// the frame's 19 lifted inputs (world->camera R, t; camera centre; fx, fy,
// cx, cy), so one reverse sweep through the real chain gives the 19 partials
// and each channel costs one 19-term contraction instead of a full lifted
// re-evaluation (rounding differs from the per-operation rule by a few ulp).
// Shared-memory layout as stage_pose_w2c: w2c[12][C], centre[3][C], intr[4][C].
// NDP > 0: the channel count is a compile-time constant, so the voxel's
// (F.re, W) and all channel loads are issued together as soon as the voxel is
// known to fuse (one DRAM round trip instead of one per channel); NDP == 0
// keeps the runtime channel loop.
template <int NDP>
CSF_DEV bool fuse_voxel_adjoint(const VoxelStore& vox, long long v, double px, double py, double pz,
                                const double* __restrict__ depth, int w, int h, double mu, double cap, int Dp,
                                const double* sm) {
  if constexpr (NDP > 0) Dp = NDP;
  const int C = 1 + Dp;
  double R[9], t[3], c[3];
#pragma unroll
  for (int e = 0; e < 9; ++e) R[e] = sm[e * C];
#pragma unroll
  for (int e = 0; e < 3; ++e) {
    t[e] = sm[(9 + e) * C];
    c[e] = sm[(12 + e) * C];
  }
  const double kfx = sm[15 * C], kfy = sm[16 * C], kcx = sm[17 * C], kcy = sm[18 * C];
  double pc[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) pc[r] = (R[3 * r] * px + (R[3 * r + 1] * py + R[3 * r + 2] * pz)) + t[r];
  if (!(pc[2] > 0.0)) return false;
  const double lx = (kfx * pc[0]) / pc[2] + kcx;
  const double ly = (kfy * pc[1]) / pc[2] + kcy;
  const int x0 = ifloor(lx), y0 = ifloor(ly);
  if (x0 < 0 || y0 < 0 || x0 + 1 >= w || y0 + 1 >= h) return false;
  const double d00 = depth[y0 * w + x0];
  const double d10 = depth[y0 * w + x0 + 1];
  const double d01 = depth[(y0 + 1) * w + x0];
  const double d11 = depth[(y0 + 1) * w + x0 + 1];
  if (!(d00 > 0.0) || !(d10 > 0.0) || !(d01 > 0.0) || !(d11 > 0.0)) return false;
  const double nearv = fmin(fmin(d00, d10), fmin(d01, d11));
  const double farv = fmax(fmax(d00, d10), fmax(d01, d11));
  if (farv - nearv > 0.1) return false;
  const double fxf = lx - static_cast<double>(x0);
  const double fyf = ly - static_cast<double>(y0);
  const double top = d00 + fxf * (d10 - d00);
  const double bot = d01 + fxf * (d11 - d01);
  const double sampled = top + fyf * (bot - top);
  const double rx = (lx - kcx) / kfx;
  const double ry = (ly - kcy) / kfy;
  const double lam = sqrt(rx * rx + (ry * ry + 1.0 * 1.0));
  const double dx = c[0] - px, dy = c[1] - py, dz = c[2] - pz;
  const double dist = sqrt(dx * dx + (dy * dy + dz * dz));
  const double eta = sampled - dist / lam;
  if (eta < -mu) return false;
  const double q = eta / mu;
  double psi = 1.0 < q ? 1.0 : q;
  psi = -1.0 > psi ? -1.0 : psi;
  const bool sat = 1.0 < q || -1.0 > q;
  // issue the voxel's loads before the reverse sweep
  double chan[NDP > 0 ? NDP : 1];
  if constexpr (NDP > 0) {
    const double* src = vox.fim + v * NDP;
    if constexpr (NDP % 2 == 0) {
#pragma unroll
      for (int d = 0; d < NDP; d += 2) {
        const double2 t = __ldcs(reinterpret_cast<const double2*>(src + d));
        chan[d] = t.x;
        chan[d + 1] = t.y;
      }
    } else {
#pragma unroll
      for (int d = 0; d < NDP; ++d) chan[d] = __ldcs(src + d);
    }
  }
  const double2 rw = vox.rw[v];
  const double wt = rw.y;
  const double fre = (wt * rw.x + psi) / (wt + 1.0);
  if (Dp > 0) {
    // reverse sweep: partials of psi with respect to the 19 lifted inputs
    double g[19];
#pragma unroll
    for (int k = 0; k < 19; ++k) g[k] = 0.0;
    if (!sat) {
      // derivative-only quantities: reciprocals instead of divisions (the
      // real chain above keeps every division)
      const double eb = 1.0 / mu, ilam = 1.0 / lam;
      const double sb = eb, distb = -eb * ilam, lamb = eb * dist * (ilam * ilam);
      const double Sb = lamb * (0.5 * ilam);
      const double rxb = 2.0 * rx * Sb, ryb = 2.0 * ry * Sb;
      const double ikfx = 1.0 / kfx, ikfy = 1.0 / kfy;
      double lxb = rxb * ikfx, lyb = ryb * ikfy;
      double cxb = -lxb, cyb = -lyb;
      double fxb = -lxb * rx, fyb = -lyb * ry;
      const double topb = sb * (1.0 - fyf), botb = sb * fyf, fyfb = sb * (bot - top);
      const double fxfb = topb * (d10 - d00) + botb * (d11 - d01);
      lxb += fxfb;
      lyb += fyfb;
      const double iz = 1.0 / pc[2];
      fxb += lxb * pc[0] * iz;
      fyb += lyb * pc[1] * iz;
      cxb += lxb;
      cyb += lyb;
      const double pcb[3] = {lxb * kfx * iz, lyb * kfy * iz,
                             -(lxb * kfx * pc[0] + lyb * kfy * pc[1]) * iz * iz};
      const double pp[3] = {px, py, pz};
#pragma unroll
      for (int r = 0; r < 3; ++r) {
#pragma unroll
        for (int j = 0; j < 3; ++j) g[3 * r + j] = pcb[r] * pp[j];
        g[9 + r] = pcb[r];
      }
      const double cd = distb / dist;
      g[12] = cd * dx;
      g[13] = cd * dy;
      g[14] = cd * dz;
      g[15] = fxb;
      g[16] = fyb;
      g[17] = cxb;
      g[18] = cyb;
    }
    const double inv_w1 = 1.0 / (wt + 1.0);
    double* fim = vox.fim + v * vox.Dp;
    if constexpr (NDP > 0) {
      if constexpr (NDP % 2 == 0) {
        const double* sj = sm + jac_offset(C);
#pragma unroll
        for (int d = 0; d < NDP; d += 2) {
          double pim0 = 0.0, pim1 = 0.0;
#pragma unroll
          for (int k = 0; k < 19; ++k) {
            const double2 j = *reinterpret_cast<const double2*>(sj + k * NDP + d);
            pim0 = fma(g[k], j.x, pim0);
            pim1 = fma(g[k], j.y, pim1);
          }
          chan[d] = (wt * chan[d] + pim0) * inv_w1;
          chan[d + 1] = (wt * chan[d + 1] + pim1) * inv_w1;
        }
      } else {
#pragma unroll
        for (int d = 0; d < NDP; ++d) {
          double pim = 0.0;
#pragma unroll
          for (int k = 0; k < 19; ++k) pim = fma(g[k], sm[k * C + 1 + d], pim);
          chan[d] = (wt * chan[d] + pim) * inv_w1;
        }
      }
      if constexpr (NDP % 2 == 0) {
#pragma unroll
        for (int d = 0; d < NDP; d += 2)
          __stcs(reinterpret_cast<double2*>(fim + d), make_double2(chan[d], chan[d + 1]));
      } else {
#pragma unroll
        for (int d = 0; d < NDP; ++d) __stcs(fim + d, chan[d]);
      }
    } else {
      for (int d = 0; d < Dp; ++d) {
        double pim = 0.0;
#pragma unroll
        for (int k = 0; k < 19; ++k) pim = fma(g[k], sm[k * C + 1 + d], pim);
        fim[d] = (wt * fim[d] + pim) * inv_w1;
      }
    }
  }
  const double wn = wt + 1.0;
  vox.rw[v] = make_double2(fre, cap < wn ? cap : wn);
  return true;
}

// Second-order fusion in tangent form.  Every Bicomplex operation of
// measured_tsdf<B<1>> (csfd.hpp:103-140 rules, the truncated product: im12 =
// a.re b12 + a12 b.re + a1 b2 + a2 b1) is evaluated on the channel slots only,
// with the real intermediates of the one real chain (bit-identical to the
// reference's double chain) shared by all pairs: the generic path re-runs the
// real chain, its IEEE divisions and square roots once per pair.  Quotients
// and square roots use the real pass's reciprocals (a few ulp per channel, as
// the first-order adjoint form).  Per pair: the 19 inputs' (im1, im2, im12)
// from shared memory, the voxel's three field slots read and written.
struct Ch3 {
  double a, b, ab;  // im1, im2, im12
};
// kF: contract the slot arithmetic with explicit fused multiply-adds (the
// library builds with -fmad=false so that real chains stay bit-identical;
// slots are held to the 1e-9 tolerance, not to the per-operation rounding).
// The fusion measured faster with them (order-2 fusion 274 -> 257 ms per
// config-3 step), the lift slower (138 -> 142 ms), so each picks its form.
// x * y (both lifted), real parts xr, yr
template <bool kF = false>
CSF_DEV Ch3 ch_mul(double xr, const Ch3& x, double yr, const Ch3& y) {
  if constexpr (kF)
    return {fma(xr, y.a, x.a * yr), fma(xr, y.b, x.b * yr), fma(x.b, y.a, fma(x.a, y.b, fma(xr, y.ab, x.ab * yr)))};
  return {xr * y.a + x.a * yr, xr * y.b + x.b * yr, ((xr * y.ab + x.ab * yr) + x.a * y.b) + x.b * y.a};
}
// x / y with real parts xr, yr; inv = 1 / yr, inv2 = inv * inv
template <bool kF = false>
CSF_DEV Ch3 ch_div(double xr, const Ch3& x, double yr, const Ch3& y, double inv, double inv2) {
  if constexpr (kF) {
    const double k = ((2.0 * xr) * inv2) * inv;
    double ab = fma(-fma(x.a, y.b, x.b * y.a), inv2, x.ab * inv);
    ab = fma(-(xr * y.ab), inv2, ab);
    return {fma(x.a, yr, -(xr * y.a)) * inv2, fma(x.b, yr, -(xr * y.b)) * inv2, fma(k * y.a, y.b, ab)};
  }
  return {(x.a * yr - xr * y.a) * inv2, (x.b * yr - xr * y.b) * inv2,
          ((x.ab * inv - (x.a * y.b + x.b * y.a) * inv2) - (xr * y.ab) * inv2) + ((((2.0 * xr) * y.a) * y.b) * inv2) * inv};
}
// lift2 (csfd.hpp:212-263): d1 = f'(x), d2 = f''(x)
template <bool kF = false>
CSF_DEV Ch3 ch_lift(const Ch3& z, double d1, double d2) {
  if constexpr (kF) return {d1 * z.a, d1 * z.b, fma(d2 * z.a, z.b, d1 * z.ab)};
  return {d1 * z.a, d1 * z.b, d1 * z.ab + (d2 * z.a) * z.b};
}
// x * c + y
CSF_DEV Ch3 ch_fma(const Ch3& x, double c, const Ch3& y) { return {fma(x.a, c, y.a), fma(x.b, c, y.b), fma(x.ab, c, y.ab)}; }
CSF_DEV Ch3 ch_add(const Ch3& x, const Ch3& y) { return {x.a + y.a, x.b + y.b, x.ab + y.ab}; }
CSF_DEV Ch3 ch_sub(const Ch3& x, const Ch3& y) { return {x.a - y.a, x.b - y.b, x.ab - y.ab}; }
CSF_DEV Ch3 ch_scale(const Ch3& x, double c) { return {x.a * c, x.b * c, x.ab * c}; }
CSF_DEV Ch3 ch_at(const double* row, int o) { return {row[o], row[o + 1], row[o + 2]}; }

CSF_DEV bool fuse_voxel_pairs(const VoxelStore& vox, long long v, double px, double py, double pz,
                              const double* __restrict__ depth, int w, int h, double mu, double cap, int Dp,
                              const double* sm) {
  const int C = 1 + Dp;
  double R[9], t[3], c[3];
#pragma unroll
  for (int e = 0; e < 9; ++e) R[e] = sm[e * C];
#pragma unroll
  for (int e = 0; e < 3; ++e) {
    t[e] = sm[(9 + e) * C];
    c[e] = sm[(12 + e) * C];
  }
  const double kfx = sm[15 * C], kfy = sm[16 * C], kcx = sm[17 * C], kcy = sm[18 * C];
  // ---- the real chain (fuse_voxel_adjoint's, measured_tsdf<double>)
  double pc[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) pc[r] = (R[3 * r] * px + (R[3 * r + 1] * py + R[3 * r + 2] * pz)) + t[r];
  if (!(pc[2] > 0.0)) return false;
  const double ax = kfx * pc[0], ay = kfy * pc[1];
  const double lx = ax / pc[2] + kcx;
  const double ly = ay / pc[2] + kcy;
  const int x0 = ifloor(lx), y0 = ifloor(ly);
  if (x0 < 0 || y0 < 0 || x0 + 1 >= w || y0 + 1 >= h) return false;
  const double d00 = depth[y0 * w + x0];
  const double d10 = depth[y0 * w + x0 + 1];
  const double d01 = depth[(y0 + 1) * w + x0];
  const double d11 = depth[(y0 + 1) * w + x0 + 1];
  if (!(d00 > 0.0) || !(d10 > 0.0) || !(d01 > 0.0) || !(d11 > 0.0)) return false;
  const double nearv = fmin(fmin(d00, d10), fmin(d01, d11));
  const double farv = fmax(fmax(d00, d10), fmax(d01, d11));
  if (farv - nearv > 0.1) return false;
  const double fxf = lx - static_cast<double>(x0);
  const double fyf = ly - static_cast<double>(y0);
  const double top = d00 + fxf * (d10 - d00);
  const double bot = d01 + fxf * (d11 - d01);
  const double sampled = top + fyf * (bot - top);
  const double nx = lx - kcx, ny = ly - kcy;
  const double rx = nx / kfx;
  const double ry = ny / kfy;
  const double lam2 = rx * rx + (ry * ry + 1.0 * 1.0);
  const double lam = sqrt(lam2);
  const double dx = c[0] - px, dy = c[1] - py, dz = c[2] - pz;
  const double dist2 = dx * dx + (dy * dy + dz * dz);
  const double dist = sqrt(dist2);
  const double eta = sampled - dist / lam;
  if (eta < -mu) return false;
  const double q = eta / mu;
  double psi = 1.0 < q ? 1.0 : q;
  psi = -1.0 > psi ? -1.0 : psi;
  const bool sat = 1.0 < q || -1.0 > q;
  const double2 rw = vox.rw[v];
  const double wt = rw.y;
  const double fre = (wt * rw.x + psi) / (wt + 1.0);
  const double inv_w1 = 1.0 / (wt + 1.0);
  double* fim = vox.fim + v * vox.Dp;
  const int NP = Dp / 3;
  if (sat) {
    // psi is the literal +-1 (clamp_s): its channels are zero
    for (int pr = 0; pr < NP; ++pr) {
      double* f3 = fim + 3 * pr;
#pragma unroll
      for (int k = 0; k < 3; ++k) f3[k] = (wt * f3[k]) * inv_w1;
    }
  } else {
    // reciprocals of the chain's divisors and the sqrt derivatives
    const double iz = 1.0 / pc[2], iz2 = iz * iz;
    const double ifx = 1.0 / kfx, ifx2 = ifx * ifx, ify = 1.0 / kfy, ify2 = ify * ify;
    const double ilam = 1.0 / lam, ilam2 = ilam * ilam;
    const double l1 = 0.5 / lam, l2 = (-0.5 * l1) / lam2;
    const double s1 = 0.5 / dist, s2 = (-0.5 * s1) / dist2;
    const double dd0 = d10 - d00, dd1 = d11 - d01, bt = bot - top;
    const double imu = 1.0 / mu;
    for (int pr = 0; pr < NP; ++pr) {
      const int o = 1 + 3 * pr;
      Ch3 pcc[3];
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const Ch3 r0 = ch_at(sm + (3 * r) * C, o), r1 = ch_at(sm + (3 * r + 1) * C, o);
        const Ch3 r2 = ch_at(sm + (3 * r + 2) * C, o), tr = ch_at(sm + (9 + r) * C, o);
        pcc[r] = ch_fma(r0, px, ch_fma(r1, py, ch_fma(r2, pz, tr)));
      }
      const Ch3 cfx = ch_at(sm + 15 * C, o), cfy = ch_at(sm + 16 * C, o);
      const Ch3 ccx = ch_at(sm + 17 * C, o), ccy = ch_at(sm + 18 * C, o);
      // lx = (fx pc0) / pc2 + cx, ly likewise
      const Ch3 lxc = ch_add(ch_div<true>(ax, ch_mul<true>(kfx, cfx, pc[0], pcc[0]), pc[2], pcc[2], iz, iz2), ccx);
      const Ch3 lyc = ch_add(ch_div<true>(ay, ch_mul<true>(kfy, cfy, pc[1], pcc[1]), pc[2], pcc[2], iz, iz2), ccy);
      // bilinear depth: top + fy (bot - top), top/bot linear in fx
      const Ch3 btc = ch_sub(ch_scale(lxc, dd1), ch_scale(lxc, dd0));
      const Ch3 smp = ch_add(ch_scale(lxc, dd0), ch_mul<true>(fyf, lyc, bt, btc));
      // lambda = sqrt(rx^2 + ry^2 + 1)
      const Ch3 rxc = ch_div<true>(nx, ch_sub(lxc, ccx), kfx, cfx, ifx, ifx2);
      const Ch3 ryc = ch_div<true>(ny, ch_sub(lyc, ccy), kfy, cfy, ify, ify2);
      const Ch3 lamc = ch_lift<true>(ch_add(ch_mul<true>(rx, rxc, rx, rxc), ch_mul<true>(ry, ryc, ry, ryc)), l1, l2);
      // dist = |center - p|
      const Ch3 c0 = ch_at(sm + 12 * C, o), c1 = ch_at(sm + 13 * C, o), c2 = ch_at(sm + 14 * C, o);
      const Ch3 distc =
          ch_lift<true>(ch_add(ch_mul<true>(dx, c0, dx, c0), ch_add(ch_mul<true>(dy, c1, dy, c1), ch_mul<true>(dz, c2, dz, c2))), s1, s2);
      const Ch3 psic = ch_scale(ch_sub(smp, ch_div<true>(dist, distc, lam, lamc, ilam, ilam2)), imu);
      double* f3 = fim + 3 * pr;
      f3[0] = fma(wt, f3[0], psic.a) * inv_w1;
      f3[1] = fma(wt, f3[1], psic.b) * inv_w1;
      f3[2] = fma(wt, f3[2], psic.ab) * inv_w1;
    }
  }
  const double wn = wt + 1.0;
  vox.rw[v] = make_double2(fre, cap < wn ? cap : wn);
  return true;
}

// LD: the depth image carries perturbation channels (dch [P][Dp]): the
// generic lifted evaluation (the adjoint form's 19 partials omit the depth
// corners' channels).
template <typename S, int NDP = 0, bool LD = false>
__global__ void __launch_bounds__(256, 2) k_integrate_dense(DenseView vol, const double* __restrict__ depth, int w,
                                                         int h, const double* __restrict__ pose,
                                                         const double* __restrict__ intr, int Dp, int* upd,
                                                         const double* __restrict__ dch) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ double sm[];
  constexpr bool kAdj = kAdjointFusion && Traits<S>::kOrder == 1 && !LD;
  constexpr bool kPairs = kAdjointFusion && Traits<S>::kOrder == 2 && !LD;
  stage_pose_w2c<S>(pose, intr, Dp, sm);
  if constexpr (kAdj) stage_jacobian<NDP>(sm);
  const long long n = static_cast<long long>(vol.nx) * vol.ny * vol.nz;
  int fused = 0;
  for (long long v = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; v < n;
       v += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(v % vol.nx);
    const int j = static_cast<int>((v / vol.nx) % vol.ny);
    const int k = static_cast<int>(v / (static_cast<long long>(vol.nx) * vol.ny));
    const double px = vol.ox + vol.vs * static_cast<double>(i);
    const double py = vol.oy + vol.vs * static_cast<double>(j);
    const double pz = vol.oz + vol.vs * static_cast<double>(k);
    if constexpr (kAdj)
      fused += fuse_voxel_adjoint<NDP>(vol.vox, v, px, py, pz, depth, w, h, vol.mu, vol.cap, Dp, sm);
    else if constexpr (kPairs)
      count_updates(upd, fuse_voxel_pairs(vol.vox, v, px, py, pz, depth, w, h, vol.mu, vol.cap, Dp, sm));
    else
      count_updates(upd, fuse_voxel<S>(vol.vox, v, px, py, pz, depth, w, h, vol.mu, vol.cap, Dp, sm,
                                       LD ? dch : nullptr));
  }
  flush_updates(upd, fused);
}

// resident CTAs per SM the fusion kernel is compiled for (register budget)
#ifndef CSF_INT_MINB
#define CSF_INT_MINB 2
#endif
template <typename S, int NDP = 0, bool LD = false>
__global__ void __launch_bounds__(256, CSF_INT_MINB) k_integrate_hashed(HashView vol, const int* __restrict__ coords,
                                                          const int* __restrict__ visible,
                                                          const int* __restrict__ counters,
                                                          const double* __restrict__ depth, int w, int h,
                                                          const double* __restrict__ pose,
                                                          const double* __restrict__ intr, int Dp, int* upd,
                                                          const double* __restrict__ dch) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ double sm[];
  constexpr bool kAdj = kAdjointFusion && Traits<S>::kOrder == 1 && !LD;
  constexpr bool kPairs = kAdjointFusion && Traits<S>::kOrder == 2 && !LD;
  stage_pose_w2c<S>(pose, intr, Dp, sm);
  if constexpr (kAdj) stage_jacobian<NDP>(sm);
  const int n_vis = counters[0];
  int fused = 0;
  for (int vb = blockIdx.x; vb < n_vis; vb += gridDim.x) {
    const int b = visible[vb];
    if (b < 0) continue;
    const int bx = coords[3 * b], by = coords[3 * b + 1], bz = coords[3 * b + 2];
    for (int l = threadIdx.x; l < kBlockVoxels; l += blockDim.x) {
      const int lx = l & 7, ly = (l >> 3) & 7, lz = l >> 6;
      const double px = vol.ox + vol.vs * static_cast<double>(8 * bx + lx);
      const double py = vol.oy + vol.vs * static_cast<double>(8 * by + ly);
      const double pz = vol.oz + vol.vs * static_cast<double>(8 * bz + lz);
      const long long vv = static_cast<long long>(b) * kBlockVoxels + l;
      if constexpr (kAdj)
        fused += fuse_voxel_adjoint<NDP>(vol.vox, vv, px, py, pz, depth, w, h, vol.mu, vol.cap, Dp, sm);
      else if constexpr (kPairs)
        count_updates(upd, fuse_voxel_pairs(vol.vox, vv, px, py, pz, depth, w, h, vol.mu, vol.cap, Dp, sm));
      else
        count_updates(upd, fuse_voxel<S>(vol.vox, vv, px, py, pz, depth, w, h, vol.mu, vol.cap, Dp, sm,
                                         LD ? dch : nullptr));
    }
  }
  flush_updates(upd, fused);
}

__global__ void k_init_volume(double2* rw, double* fim, long long n, int Dp) {
  pdl_wait();
  pdl_trigger();
  const long long t0 = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long v = t0; v < n; v += stride) rw[v] = make_double2(1.0, 0.0);
  const long long nf = n * Dp;  // the channels, coalesced 16-byte stores
  double2* f2 = reinterpret_cast<double2*>(fim);
  for (long long i = t0; i < nf / 2; i += stride) f2[i] = make_double2(0.0, 0.0);
  if ((nf & 1) && t0 == 0) fim[nf - 1] = 0.0;
}

// Graph-safe reset of a hashed volume (every bound read on the device, no
// host round trip): voxels of the allocated blocks back to F = 1, W = 0, and
// the hash chains, block-id window and occupancy bits of those blocks
// cleared.  n_blocks itself is zeroed by the caller afterwards.
__global__ void k_reset_hashed(const int* n_blocks, double2* rw, double* fim, int Dp, int* heads, unsigned mask,
                               int* next, const int* coords, int* grid, unsigned* occ, int gbits) {
  pdl_wait();
  pdl_trigger();
  const long long nb = *n_blocks;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  const long long t0 = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  for (long long v = t0; v < nb * 512; v += stride) rw[v] = make_double2(1.0, 0.0);
  // the allocated blocks' channels are one prefix of the pool: zeroed
  // coalesced, 16 bytes per store (a per-voxel channel loop strides by Dp)
  {
    const long long n = nb * 512 * Dp;
    double2* f2 = reinterpret_cast<double2*>(fim);
    for (long long i = t0; i < n / 2; i += stride) f2[i] = make_double2(0.0, 0.0);
    if ((n & 1) && t0 == 0) fim[n - 1] = 0.0;
  }
  const int half = 1 << (gbits - 1);
  const unsigned side = 1u << gbits;
  for (long long b = t0; b < nb; b += stride) {
    const int bx = coords[3 * b], by = coords[3 * b + 1], bz = coords[3 * b + 2];
    heads[block_hash(bx, by, bz, mask)] = -1;
    next[b] = -1;
    const unsigned ux = static_cast<unsigned>(bx + half), uy = static_cast<unsigned>(by + half),
                   uz = static_cast<unsigned>(bz + half);
    if (ux < side && uy < side && uz < side) {
      grid[(static_cast<size_t>(uz) << gbits | uy) << gbits | ux] = -1;
      // the words holding this block's occupancy bits (any other block
      // sharing a word is cleared as well: every block is)
      const int sb = gbits - 3, s4 = gbits - 2, s2 = gbits - 1;
      const unsigned bit = ((uz >> 3) << sb | (uy >> 3)) << sb | (ux >> 3);
      occ[bit >> 5] = 0u;
      unsigned* occ4 = occ + ((1u << (3 * sb)) >> 5);
      const unsigned b4 = ((uz >> 2) << s4 | (uy >> 2)) << s4 | (ux >> 2);
      occ4[b4 >> 5] = 0u;
      unsigned* occ2 = occ4 + ((1u << (3 * s4)) >> 5);
      const unsigned b2 = ((uz >> 1) << s2 | (uy >> 1)) << s2 | (ux >> 1);
      occ2[b2 >> 5] = 0u;
    }
  }
}

// ----------------------------------------------------------------------------
// Hashed allocation (builder-defined; oracle/orc_tsdf.hpp allocate_band)
// ----------------------------------------------------------------------------
__global__ void k_band(const double* __restrict__ depth, int w, int h, const double* __restrict__ pose,
                       const double* __restrict__ intr, int C, double mu, double vs, double ox, double oy, double oz,
                       int K, unsigned long long* __restrict__ cand) {
  pdl_wait();
  pdl_trigger();
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= w || y >= h) return;
  const long long pix = static_cast<long long>(y) * w + x;
  unsigned long long* out = cand + pix * K;
  const double d = depth[pix];
  if (!(d > 0.0)) {
    for (int s = 0; s < K; ++s) out[s] = kEmptyKey;
    return;
  }
  Pose<double> c2w;
#pragma unroll
  for (int e = 0; e < 9; ++e) c2w.R.m[e] = pose[e * C];
#pragma unroll
  for (int e = 0; e < 3; ++e) c2w.t.v[e] = pose[(9 + e) * C];
  const double fx = intr[0], fy = intr[C], cx = intr[2 * C], cy = intr[3 * C];
  const double lo = d - mu;
  const double step = (2.0 * mu) / static_cast<double>(K - 1);
  const double rx = (static_cast<double>(x) - cx) / fx;
  const double ry = (static_cast<double>(y) - cy) / fy;
  int pbx = 0, pby = 0, pbz = 0;
  bool have = false;
  for (int s = 0; s < K; ++s) {
    out[s] = kEmptyKey;
    const double z = lo + static_cast<double>(s) * step;
    if (!(z > 0.0)) continue;
    const V3<double> wp = apply(c2w, mk3<double>(z * rx, z * ry, z));
    const int bx = ifloor((wp.v[0] - ox) / vs) >> 3;
    const int by = ifloor((wp.v[1] - oy) / vs) >> 3;
    const int bz = ifloor((wp.v[2] - oz) / vs) >> 3;
    if (have && bx == pbx && by == pby && bz == pbz) continue;
    out[s] = block_key(bx, by, bz);
    pbx = bx; pby = by; pbz = bz;
    have = true;
  }
}

CSF_DEV unsigned set_hash(unsigned long long key, int bits) {
  return static_cast<unsigned>((key * 0x9E3779B97F4A7C15ULL) >> (64 - bits));
}

__global__ void k_touch(const unsigned long long* __restrict__ cand, int n, unsigned long long* set_keys,
                        int* set_first, int* set_slot, int bits, int* err, int* counters) {
  pdl_wait();
  pdl_trigger();
  // grid-stride (a few waves of resident CTAs instead of one CTA per 256
  // slots: the kernel is CTA-launch-bound otherwise)
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x) {
    const unsigned long long key = cand[s];
    if (key == kEmptyKey) {
      set_slot[s] = -1;
      continue;
    }
    const unsigned mask = (1u << bits) - 1u;
    unsigned hsh = set_hash(key, bits);
    bool placed = false;
    for (unsigned probe = 0; probe <= mask; ++probe) {
      const unsigned long long prev = atomicCAS(set_keys + hsh, kEmptyKey, key);
      if (prev == kEmptyKey || prev == key) {
        atomicMin(set_first + hsh, s);
        set_slot[s] = static_cast<int>(hsh);
        placed = true;
        break;
      }
      hsh = (hsh + 1u) & mask;
    }
    if (!placed) {
      set_slot[s] = -1;
      atomicExch(counters + 2, 1);
      raise(err, kErrNoMem);
    }
  }
}

__global__ void k_flags(HashView vol, const unsigned long long* __restrict__ cand, int n,
                        const int* __restrict__ set_first, const int* __restrict__ set_slot, int* first_flag,
                        int* new_flag, int* cand_block) {
  pdl_wait();
  pdl_trigger();
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x) {
    const int hs = set_slot[s];
    const bool first = hs >= 0 && set_first[hs] == s;
    int nf = 0;
    if (first) {
      const unsigned long long key = cand[s];
      const int bx = static_cast<int>((key >> 42) & 0x1FFFFF) - kCoordBias;
      const int by = static_cast<int>((key >> 21) & 0x1FFFFF) - kCoordBias;
      const int bz = static_cast<int>(key & 0x1FFFFF) - kCoordBias;
      const int id = vol.block(bx, by, bz);  // the dense index (one load) or the chain
      cand_block[s] = id;
      nf = id < 0;
    }
    first_flag[s] = first;
    new_flag[s] = nf;
  }
}

// Lock-free insertion into a chain kept sorted by key: the resulting chains
// depend only on the key set, never on thread order.
__device__ void chain_insert(int* heads, const unsigned long long* keys, int* next, unsigned bucket, int id,
                             unsigned long long key) {
  while (true) {
    int* link = heads + bucket;
    int cur = *reinterpret_cast<volatile int*>(link);
    while (cur >= 0 && *reinterpret_cast<const volatile unsigned long long*>(keys + cur) < key) {
      link = next + cur;
      cur = *reinterpret_cast<volatile int*>(link);
    }
    *reinterpret_cast<volatile int*>(next + id) = cur;
    __threadfence();
    if (atomicCAS(link, cur, id) == cur) return;
  }
}

// Mark block (ux, uy, uz) (window coordinates) in every occupancy level.
CSF_DEV void occ_mark(unsigned* occ, int gbits, unsigned ux, unsigned uy, unsigned uz) {
  const int sb = gbits - 3, s4 = gbits - 2, s2 = gbits - 1;
  const unsigned bit = ((uz >> 3) << sb | (uy >> 3)) << sb | (ux >> 3);
  atomicOr(occ + (bit >> 5), 1u << (bit & 31));
  unsigned* occ4 = occ + ((1u << (3 * sb)) >> 5);
  const unsigned b4 = ((uz >> 2) << s4 | (uy >> 2)) << s4 | (ux >> 2);
  atomicOr(occ4 + (b4 >> 5), 1u << (b4 & 31));
  unsigned* occ2 = occ4 + ((1u << (3 * s4)) >> 5);
  const unsigned b2 = ((uz >> 1) << s2 | (uy >> 1)) << s2 | (ux >> 1);
  atomicOr(occ2 + (b2 >> 5), 1u << (b2 & 31));
}

CSF_DEV void insert_slot(HashView vol, int* heads, unsigned long long* keys, int* next, int* coords,
                         const int* n_blocks, int max_blocks, const unsigned long long* __restrict__ cand,
                         const int* __restrict__ first_flag, const int* __restrict__ new_flag,
                         const int* __restrict__ first_rank, const int* __restrict__ new_rank,
                         const int* __restrict__ cand_block, int* visible, int* err, int s);
__global__ void k_insert(HashView vol, int* heads, unsigned long long* keys, int* next, int* coords, const int* n_blocks,
                         int max_blocks, const unsigned long long* __restrict__ cand, int n,
                         const int* __restrict__ first_flag, const int* __restrict__ new_flag,
                         const int* __restrict__ first_rank, const int* __restrict__ new_rank,
                         const int* __restrict__ cand_block, int* visible, int* err) {
  pdl_wait();
  pdl_trigger();
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n; s += gridDim.x * blockDim.x)
    insert_slot(vol, heads, keys, next, coords, n_blocks, max_blocks, cand, first_flag, new_flag, first_rank,
                new_rank, cand_block, visible, err, s);
}

CSF_DEV void insert_slot(HashView vol, int* heads, unsigned long long* keys, int* next, int* coords,
                         const int* n_blocks, int max_blocks, const unsigned long long* __restrict__ cand,
                         const int* __restrict__ first_flag, const int* __restrict__ new_flag,
                         const int* __restrict__ first_rank, const int* __restrict__ new_rank,
                         const int* __restrict__ cand_block, int* visible, int* err, int s) {
  if (!first_flag[s]) return;
  int id = cand_block[s];
  if (new_flag[s]) {
    id = *n_blocks + new_rank[s];
    if (id >= max_blocks) {
      raise(err, kErrNoMem);
      visible[first_rank[s]] = -1;
      return;
    }
    const unsigned long long key = cand[s];
    const int bx = static_cast<int>((key >> 42) & 0x1FFFFF) - kCoordBias;
    const int by = static_cast<int>((key >> 21) & 0x1FFFFF) - kCoordBias;
    const int bz = static_cast<int>(key & 0x1FFFFF) - kCoordBias;
    keys[id] = key;
    coords[3 * id] = bx;
    coords[3 * id + 1] = by;
    coords[3 * id + 2] = bz;
    __threadfence();
    chain_insert(heads, keys, next, block_hash(bx, by, bz, vol.mask), id, key);
    const int half = 1 << (vol.gbits - 1);
    const unsigned ux = static_cast<unsigned>(bx + half), uy = static_cast<unsigned>(by + half),
                   uz = static_cast<unsigned>(bz + half);
    const unsigned side = 1u << vol.gbits;
    if (ux < side && uy < side && uz < side) {
      const_cast<int*>(vol.grid)[(static_cast<size_t>(uz) << vol.gbits | uy) << vol.gbits | ux] = id;
      occ_mark(const_cast<unsigned*>(vol.occ), vol.gbits, ux, uy, uz);
    }
  }
  visible[first_rank[s]] = id;
}

__global__ void k_alloc_finalize(int* n_blocks, int max_blocks, const int* first_flag, const int* new_flag,
                                 const int* first_rank, const int* new_rank, int n, int* counters) {
  pdl_wait();
  pdl_trigger();
  const int n_vis = n > 0 ? first_rank[n - 1] + first_flag[n - 1] : 0;
  const int n_new = n > 0 ? new_rank[n - 1] + new_flag[n - 1] : 0;
  const int old = *n_blocks;
  const int nb = old + n_new > max_blocks ? max_blocks : old + n_new;
  *n_blocks = nb;
  counters[0] = n_vis;
  counters[1] = n_new;
  counters[3] = old;
}

// ----------------------------------------------------------------------------
// Raycast (tsdf.hpp:209-284) as two kernels:
//   k_raycast_march — one thread per pixel, real channel only: the slab clip,
//     the fixed-step march and the zero-crossing test (every branch of the
//     reference reads real parts).  Hashed volumes skip the samples whose
//     base corner lies in an unallocated block: those samples are invalid by
//     definition, alpha still advances by the same repeated addition, and the
//     skip stops 1e-6 m before the block's analytic exit so the exact
//     per-sample test decides every boundary case.  Output: the crossing's
//     (alpha_prev, alpha) or a miss.
//   k_raycast_lift_coop / k_raycast_lift2_coop — the lifted epilogue: a
//     real pass per hit pixel (8 lanes: the two samples at the recorded
//     alphas, bit-identical, and the 6 central differences), then the
//     channels per (pixel, channel pair) in tangent form (first order) or per
//     (pixel, parameter pair) in Bicomplex arithmetic (second order).
// ----------------------------------------------------------------------------
// Pixel order of the raycast kernels: 8x4-pixel warp tiles in row-major
// tile order (lin = 32 * tile + lane).  The rays of a warp are a compact
// patch, so their march trip counts and their lift gathers (shared voxels)
// are more alike than along a 32-pixel row.  lin < tiled_count(w, h).
CSF_HD long long tiled_count(int w, int h) { return 32LL * ((w + 7) / 8) * ((h + 3) / 4); }
CSF_DEV bool tile_pixel(long long lin, int w, int h, int* x, int* y) {
  const int tiles_x = (w + 7) >> 3;
  const long long t = lin >> 5;
  const int l = static_cast<int>(lin & 31);
  *x = 8 * static_cast<int>(t % tiles_x) + (l & 7);
  *y = 4 * static_cast<int>(t / tiles_x) + (l >> 3);
  return *x < w && *y < h;
}

struct Box {
  bool use;
  double lo[3], hi[3];
};

// Real trilinear sample with all eight corner loads issued before any test.
template <typename V>
CSF_DEV bool sample_real(const V& vol, double px, double py, double pz, typename V::Cache& cache, double* out) {
  const double gx = (px - vol.ox) / vol.vs;
  const double gy = (py - vol.oy) / vol.vs;
  const double gz = (pz - vol.oz) / vol.vs;
  const int i0 = ifloor(gx), j0 = ifloor(gy), k0 = ifloor(gz);
  if (!vol.cell_in_grid(i0, j0, k0)) return false;
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
  const double fx = gx - static_cast<double>(i0);
  const double fy = gy - static_cast<double>(j0);
  const double fz = gz - static_cast<double>(k0);
  double accum = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const double wx = (c & 1) ? fx : 1.0 - fx;
    const double wy = ((c >> 1) & 1) ? fy : 1.0 - fy;
    const double wz = (c >> 2) ? fz : 1.0 - fz;
    accum = accum + ((wx * wy) * wz) * rw[c].x;
  }
  *out = accum;
  return true;
}

// sample_real with the corner voxel ids already known (HashView::probe_cell):
// the same arithmetic, the corner loads in one round trip.
template <typename V>
CSF_DEV bool sample_real_at(const V& vol, double px, double py, double pz, const long long* v, double* out) {
  const double gx = (px - vol.ox) / vol.vs;
  const double gy = (py - vol.oy) / vol.vs;
  const double gz = (pz - vol.oz) / vol.vs;
  const int i0 = ifloor(gx), j0 = ifloor(gy), k0 = ifloor(gz);
  bool ok = true;
#pragma unroll
  for (int c = 0; c < 8; ++c) ok = ok && v[c] >= 0;
  if (!ok) return false;
  double2 rw[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) rw[c] = vol.vox.rw[v[c]];
#pragma unroll
  for (int c = 0; c < 8; ++c) ok = ok && rw[c].y > 0.0;
  if (!ok) return false;
  const double fx = gx - static_cast<double>(i0);
  const double fy = gy - static_cast<double>(j0);
  const double fz = gz - static_cast<double>(k0);
  double accum = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const double wx = (c & 1) ? fx : 1.0 - fx;
    const double wy = ((c >> 1) & 1) ? fy : 1.0 - fy;
    const double wz = (c >> 2) ? fz : 1.0 - fz;
    accum = accum + ((wx * wy) * wz) * rw[c].x;
  }
  *out = accum;
  return true;
}

// Exit distance of the ray from the axis-aligned box of `span` blocks whose
// lowest block is (bx, by, bz) (inverse direction precomputed; used only to
// bound skipped alphas, with a margin, so ~1 ulp error is immaterial).
CSF_DEV double box_exit(const HashView& vol, int bx, int by, int bz, int span, const V3<double>& o,
                        const V3<double>& invd) {
  const int b[3] = {bx, by, bz};
  const double org[3] = {vol.ox, vol.oy, vol.oz};
  const double side = vol.vs * static_cast<double>(8 * span);
  double t = 1e300;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double lo = org[a] + vol.vs * static_cast<double>(8 * b[a]);
    if (invd.v[a] > 0.0) t = fmin(t, ((lo + side) - o.v[a]) * invd.v[a]);
    else if (invd.v[a] < 0.0) t = fmin(t, (lo - o.v[a]) * invd.v[a]);
  }
  return t;
}

// Debug statistics of the table march (tools/march_stats.py; null = off):
// [0] rays, [1] loop trips, [2] super-block skips, [3] block skips,
// [4] samples, [5] valid samples, [6] hits, [7] sum over warps of max trips.
__device__ unsigned long long* g_march_stats = nullptr;
#ifdef CSF_MARCH_STATS
#define CSF_MSTAT(x) x
#else
#define CSF_MSTAT(x)
#endif

template <typename V>
__global__ void __launch_bounds__(128) k_raycast_march(V vol, const double* __restrict__ pose,
                                                       const double* __restrict__ intr, int w, int h, int Dp,
                                                       double near_clip, double far_clip, double step, Box box,
                                                       double2* __restrict__ hits, double* __restrict__ vre,
                                                       double* __restrict__ nre, const double* __restrict__ atab,
                                                       int n_tab) {
  pdl_wait();
  pdl_trigger();
  __shared__ double s_pose[16];
  const int C = 1 + Dp;
  if (threadIdx.x < 12) s_pose[threadIdx.x] = pose[threadIdx.x * C];
  else if (threadIdx.x < 16) s_pose[threadIdx.x] = intr[(threadIdx.x - 12) * C];
  __syncthreads();
  int x, y;
  if (!tile_pixel(blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x, w, h, &x, &y)) return;
  const int pix = y * w + x;
  Pose<double> c2w;
#pragma unroll
  for (int e = 0; e < 9; ++e) c2w.R.m[e] = s_pose[e];
#pragma unroll
  for (int e = 0; e < 3; ++e) c2w.t.v[e] = s_pose[9 + e];
  const double fxk = s_pose[12], fyk = s_pose[13], cxk = s_pose[14], cyk = s_pose[15];
  const V3<double> dc = mk3<double>((static_cast<double>(x) - cxk) / fxk, (static_cast<double>(y) - cyk) / fyk, 1.0);
  const double rn = sqrt(dot3(dc, dc));
  const V3<double> dir = matvec(c2w.R, mk3<double>(dc.v[0] / rn, dc.v[1] / rn, dc.v[2] / rn));
  const V3<double> o = c2w.t;
#pragma unroll
  for (int c = 0; c < 3; ++c) vre[3LL * pix + c] = nre[3LL * pix + c] = 0.0;
  hits[pix] = make_double2(0.0, -1.0);  // y < 0: no crossing

  double t0 = near_clip, t1 = far_clip;
  if (box.use) {
    bool hit_box = true;
#pragma unroll
    for (int axis = 0; axis < 3; ++axis) {
      const double od = o.v[axis], dd = dir.v[axis];
      if (fabs(dd) < 1e-12) {
        if (od < box.lo[axis] || od > box.hi[axis]) hit_box = false;
        continue;
      }
      double ta = (box.lo[axis] - od) / dd;
      double tb = (box.hi[axis] - od) / dd;
      if (ta > tb) {
        const double t = ta;
        ta = tb;
        tb = t;
      }
      t0 = t0 < ta ? ta : t0;  // std::max(t0, ta)
      t1 = tb < t1 ? tb : t1;  // std::min(t1, tb)
    }
    if (!hit_box) return;
  }
  if (t0 >= t1) return;

  typename V::Cache cache;
  cache.reset();
  V3<double> invd;
#pragma unroll
  for (int a = 0; a < 3; ++a) invd.v[a] = dir.v[a] != 0.0 ? 1.0 / dir.v[a] : 0.0;
  bool have_prev = false;
  double alpha_prev = 0.0, f_prev = 0.0;
  if constexpr (V::kHashed) {
    if (atab) {
      // Every ray of a hashed volume marches the same alpha sequence (t0 =
      // near, no slab clip): index it from the table instead of re-adding.
      // Semantics are the loop below, sample for sample.
      const int nmax = n_tab - 1;  // atab[nmax] > t1 (sentinel)
      const double inv_step = 1.0 / step;
#ifdef CSF_MARCH_STATS
      unsigned long long* const dbg = g_march_stats;
      unsigned trips = 0, sskip = 0, bskip = 0, nsamp = 0, nvalid = 0;
      auto flush = [&](bool hit) {
        if (!dbg) return;
        atomicAdd(dbg + 0, 1ULL);
        atomicAdd(dbg + 1, trips);
        atomicAdd(dbg + 2, sskip);
        atomicAdd(dbg + 3, bskip);
        atomicAdd(dbg + 4, nsamp);
        atomicAdd(dbg + 5, nvalid);
        if (hit) atomicAdd(dbg + 6, 1ULL);
        unsigned mx = trips;
        for (int o2 = 16; o2 > 0; o2 >>= 1) mx = max(mx, __shfl_xor_sync(__activemask(), mx, o2));
        if ((threadIdx.x & 31) == __ffs(__activemask()) - 1) atomicAdd(dbg + 7, mx);
      };
#endif
      int n = 0;
      while (n < nmax) {
        CSF_MSTAT(++trips);
        const double alpha = atab[n];
        const double px = o.v[0] + alpha * dir.v[0], py = o.v[1] + alpha * dir.v[1],
                     pz = o.v[2] + alpha * dir.v[2];
        const int i0 = ifloor((px - vol.ox) / vol.vs), j0 = ifloor((py - vol.oy) / vol.vs),
                  k0 = ifloor((pz - vol.oz) / vol.vs);
        const int bx = i0 >> 3, by = j0 >> 3, bz = k0 >> 3;
        // empty space: the cube of (2d - 1)^3 empty super-blocks around this
        // one (distance field), else this unallocated block
        int sd, es, blk;
        long long cv[8];
        vol.probe_cell(i0, j0, k0, &sd, &es, &blk, cv);
        int span = 0, lx = bx, ly = by, lz = bz;
        if (sd > 0) {
          span = 8 * (2 * sd - 1);
          lx = ((bx >> 3) - (sd - 1)) << 3;
          ly = ((by >> 3) - (sd - 1)) << 3;
          lz = ((bz >> 3) - (sd - 1)) << 3;
        } else if (es) {
          span = es;  // an empty aligned 4^3- or 2^3-block cell
          const int m2 = ~(es - 1);
          lx = bx & m2;
          ly = by & m2;
          lz = bz & m2;
        } else if (blk < 0) {
          span = 1;
        }
        if (span > 0) {
          have_prev = false;
          CSF_MSTAT(if (span >= 8) ++sskip; else ++bskip;)
          const double lim = box_exit(vol, lx, ly, lz, span, o, invd) - 1e-6;
          // first index > n whose alpha reaches lim (or the sentinel)
          int g = static_cast<int>(fmin(fmax((lim - atab[0]) * inv_step, 0.0), static_cast<double>(nmax)));
          g = g < n + 1 ? n + 1 : g;
          while (g > n + 1 && __ldg(atab + g - 1) >= lim) --g;
          while (g < nmax && __ldg(atab + g) < lim) ++g;
          n = g;
          continue;
        }
        double f;
        CSF_MSTAT(++nsamp);
        if (!sample_real_at(vol, px, py, pz, cv, &f)) {
          have_prev = false;
          ++n;
          continue;
        }
        CSF_MSTAT(++nvalid);
        if (have_prev && f_prev > 0.0 && f < 0.0) {
          hits[pix] = make_double2(alpha_prev, alpha);
          hits[w * h + pix] = make_double2(f_prev, f);
          CSF_MSTAT(flush(true));
          return;
        }
        have_prev = true;
        alpha_prev = alpha;
        f_prev = f;
        ++n;
      }
      CSF_MSTAT(flush(false));
      return;
    }
  }
  double alpha = t0;
  while (alpha <= t1) {
    const double px = o.v[0] + alpha * dir.v[0], py = o.v[1] + alpha * dir.v[1], pz = o.v[2] + alpha * dir.v[2];
    if constexpr (V::kHashed) {
      // unallocated base block: every sample until the block exit is invalid
      const int i0 = ifloor((px - vol.ox) / vol.vs), j0 = ifloor((py - vol.oy) / vol.vs),
                k0 = ifloor((pz - vol.oz) / vol.vs);
      const int bx = i0 >> 3, by = j0 >> 3, bz = k0 >> 3;
      const int occ = vol.super_occupied(bx, by, bz);
      int span = 0;
      if (occ == 0) span = 8;                      // empty 8^3-block super-block
      else if (vol.block(bx, by, bz) < 0) span = 1;  // unallocated block
      if (span > 0) {
        have_prev = false;
        const int m = span == 8 ? ~7 : ~0;
        const double lim = box_exit(vol, bx & m, by & m, bz & m, span, o, invd) - 1e-6;
        alpha += step;
        while (alpha < lim && alpha <= t1) alpha += step;
        continue;
      }
    }
    double f;
    if (!sample_real(vol, px, py, pz, cache, &f)) {
      have_prev = false;
      alpha += step;
      continue;
    }
    if (have_prev && f_prev > 0.0 && f < 0.0) {
      hits[pix] = make_double2(alpha_prev, alpha);
      hits[w * h + pix] = make_double2(f_prev, f);
      return;
    }
    have_prev = true;
    alpha_prev = alpha;
    f_prev = f;
    alpha += step;
  }
}

// Segmented march (hashed volumes, alpha table): the small pyramid levels
// have few rays, so the level's time is the longest ray's sequential chain.
// A ray's table indices are cut into S segments marched by S threads.  The
// reference's crossing rule only carries the previous sample across a step
// (have_prev resets on an invalid sample), so "crossing at index n" is a
// pure predicate of samples n-1 and n: each segment evaluates the sample
// before its first index to seed that state, marches its range with the
// exact per-sample semantics, and the smallest crossing index over the
// segments (atomicMin) is the sequential loop's first crossing.
CSF_DEV bool table_sample(const HashView& vol, const V3<double>& o, const V3<double>& dir, double alpha, double* f) {
  const double px = o.v[0] + alpha * dir.v[0], py = o.v[1] + alpha * dir.v[1], pz = o.v[2] + alpha * dir.v[2];
  const int i0 = ifloor((px - vol.ox) / vol.vs), j0 = ifloor((py - vol.oy) / vol.vs),
            k0 = ifloor((pz - vol.oz) / vol.vs);
  // one round trip for the occupancy test and the corner ids (probe_cell)
  int sd, es, blk;
  long long cv[8];
  vol.probe_cell(i0, j0, k0, &sd, &es, &blk, cv);
  if (sd > 0 || blk < 0) return false;
  return sample_real_at(vol, px, py, pz, cv, f);
}

CSF_DEV void ray_of(const double* s_pose, int x, int y, V3<double>* o, V3<double>* dir) {
  Pose<double> c2w;
#pragma unroll
  for (int e = 0; e < 9; ++e) c2w.R.m[e] = s_pose[e];
#pragma unroll
  for (int e = 0; e < 3; ++e) c2w.t.v[e] = s_pose[9 + e];
  const double fxk = s_pose[12], fyk = s_pose[13], cxk = s_pose[14], cyk = s_pose[15];
  const V3<double> dc = mk3<double>((static_cast<double>(x) - cxk) / fxk, (static_cast<double>(y) - cyk) / fyk, 1.0);
  const double rn = sqrt(dot3(dc, dc));
  *dir = matvec(c2w.R, mk3<double>(dc.v[0] / rn, dc.v[1] / rn, dc.v[2] / rn));
  *o = c2w.t;
}

__global__ void __launch_bounds__(128) k_raycast_march_seg(HashView vol, const double* __restrict__ pose,
                                                           const double* __restrict__ intr, int w, int h, int Dp,
                                                           int S, const double* __restrict__ atab, int n_tab,
                                                           double step, unsigned* __restrict__ first) {
  pdl_wait();
  pdl_trigger();
  __shared__ double s_pose[16];
  const int C = 1 + Dp;
  if (threadIdx.x < 12) s_pose[threadIdx.x] = pose[threadIdx.x * C];
  else if (threadIdx.x < 16) s_pose[threadIdx.x] = intr[(threadIdx.x - 12) * C];
  __syncthreads();
  const long long T = tiled_count(w, h);
  const long long item = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (item >= T * S) return;
  const int seg = static_cast<int>(item / T);
  int px_, py_;
  if (!tile_pixel(item % T, w, h, &px_, &py_)) return;
  const int pix = py_ * w + px_;
  V3<double> o, dir;
  ray_of(s_pose, px_, py_, &o, &dir);
  V3<double> invd;
#pragma unroll
  for (int a = 0; a < 3; ++a) invd.v[a] = dir.v[a] != 0.0 ? 1.0 / dir.v[a] : 0.0;
  const int nmax = n_tab - 1;
  const int n0 = static_cast<int>(static_cast<long long>(nmax) * seg / S);
  const int n1 = static_cast<int>(static_cast<long long>(nmax) * (seg + 1) / S);
  double f_prev = 0.0;
  bool have_prev = n0 > 0 && table_sample(vol, o, dir, atab[n0 - 1], &f_prev);
  const double inv_step = 1.0 / step;
  int n = n0;
  while (n < n1) {
    const double alpha = atab[n];
    const double px = o.v[0] + alpha * dir.v[0], py = o.v[1] + alpha * dir.v[1], pz = o.v[2] + alpha * dir.v[2];
    const int i0 = ifloor((px - vol.ox) / vol.vs), j0 = ifloor((py - vol.oy) / vol.vs),
              k0 = ifloor((pz - vol.oz) / vol.vs);
    const int bx = i0 >> 3, by = j0 >> 3, bz = k0 >> 3;
    int sd, es, blk;
    long long cv[8];
    vol.probe_cell(i0, j0, k0, &sd, &es, &blk, cv);
    int span = 0, lx = bx, ly = by, lz = bz;
    if (sd > 0) {
      span = 8 * (2 * sd - 1);
      lx = ((bx >> 3) - (sd - 1)) << 3;
      ly = ((by >> 3) - (sd - 1)) << 3;
      lz = ((bz >> 3) - (sd - 1)) << 3;
    } else if (es) {
      span = es;
      const int m2 = ~(es - 1);
      lx = bx & m2;
      ly = by & m2;
      lz = bz & m2;
    } else if (blk < 0) {
      span = 1;
    }
    if (span > 0) {
      have_prev = false;
      const double lim = box_exit(vol, lx, ly, lz, span, o, invd) - 1e-6;
      int g = static_cast<int>(fmin(fmax((lim - atab[0]) * inv_step, 0.0), static_cast<double>(nmax)));
      g = g < n + 1 ? n + 1 : g;
      while (g > n + 1 && __ldg(atab + g - 1) >= lim) --g;
      while (g < nmax && __ldg(atab + g) < lim) ++g;
      n = g;
      continue;
    }
    double f;
    if (!sample_real_at(vol, px, py, pz, cv, &f)) {
      have_prev = false;
      ++n;
      continue;
    }
    if (have_prev && f_prev > 0.0 && f < 0.0) {
      atomicMin(first + pix, static_cast<unsigned>(n));
      return;
    }
    have_prev = true;
    f_prev = f;
    ++n;
  }
}

// Crossing of each pixel from the smallest segment index: the hit alphas and
// the two sample values (re-evaluated, bit-identical), real maps cleared.
__global__ void __launch_bounds__(128) k_raycast_march_fin(HashView vol, const double* __restrict__ pose,
                                                           const double* __restrict__ intr, int w, int h, int Dp,
                                                           const double* __restrict__ atab,
                                                           const unsigned* __restrict__ first, double2* __restrict__ hits,
                                                           double* __restrict__ vre, double* __restrict__ nre) {
  pdl_wait();
  pdl_trigger();
  __shared__ double s_pose[16];
  const int C = 1 + Dp;
  if (threadIdx.x < 12) s_pose[threadIdx.x] = pose[threadIdx.x * C];
  else if (threadIdx.x < 16) s_pose[threadIdx.x] = intr[(threadIdx.x - 12) * C];
  __syncthreads();
  const int pix = blockIdx.x * blockDim.x + threadIdx.x;
  if (pix >= w * h) return;
#pragma unroll
  for (int c = 0; c < 3; ++c) vre[3LL * pix + c] = nre[3LL * pix + c] = 0.0;
  const unsigned n = first[pix];
  if (n == 0xFFFFFFFFu) {
    hits[pix] = make_double2(0.0, -1.0);
    return;
  }
  V3<double> o, dir;
  ray_of(s_pose, pix % w, pix / w, &o, &dir);
  double f_prev = 0.0, f = 0.0;
  table_sample(vol, o, dir, atab[n - 1], &f_prev);
  table_sample(vol, o, dir, atab[n], &f);
  hits[pix] = make_double2(atab[n - 1], atab[n]);
  hits[w * h + pix] = make_double2(f_prev, f);
}

// Real trilinear sample that also returns what the channel pass needs: the
// corner voxel ids, the corner weights and the derivative of the sample with
// respect to the cell fractions (real parts of sample_tsdf<S>, bit-identical).
template <typename V>
CSF_DEV bool sample_real_ex(const V& vol, double px, double py, double pz, double* out, int* vid, double* wgt,
                            double* ds, double* Fout = nullptr, double* frac = nullptr) {
  const double gx = (px - vol.ox) / vol.vs;
  const double gy = (py - vol.oy) / vol.vs;
  const double gz = (pz - vol.oz) / vol.vs;
  const int i0 = ifloor(gx), j0 = ifloor(gy), k0 = ifloor(gz);
  if (!vol.cell_in_grid(i0, j0, k0)) return false;
  long long v[8];
  bool ok = true;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    v[c] = vol.voxel(i0 + (c & 1), j0 + ((c >> 1) & 1), k0 + (c >> 2));
    ok = ok && v[c] >= 0;
  }
  if (!ok) return false;
  double2 rw[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) rw[c] = vol.vox.rw[v[c]];
#pragma unroll
  for (int c = 0; c < 8; ++c) ok = ok && rw[c].y > 0.0;
  if (!ok) return false;
  const double fx = gx - static_cast<double>(i0);
  const double fy = gy - static_cast<double>(j0);
  const double fz = gz - static_cast<double>(k0);
  double acc = 0.0, dsx = 0.0, dsy = 0.0, dsz = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const double wx = (c & 1) ? fx : 1.0 - fx;
    const double wy = ((c >> 1) & 1) ? fy : 1.0 - fy;
    const double wz = (c >> 2) ? fz : 1.0 - fz;
    wgt[c] = (wx * wy) * wz;
    acc = acc + wgt[c] * rw[c].x;
    const double F = rw[c].x;
    dsx += ((c & 1) ? 1.0 : -1.0) * (wy * wz) * F;
    dsy += (((c >> 1) & 1) ? 1.0 : -1.0) * (wx * wz) * F;
    dsz += ((c >> 2) ? 1.0 : -1.0) * (wx * wy) * F;
    vid[c] = static_cast<int>(v[c]);
    if (Fout) Fout[c] = rw[c].x;
  }
  ds[0] = dsx;
  ds[1] = dsy;
  ds[2] = dsz;
  if (frac) {
    frac[0] = fx;
    frac[1] = fy;
    frac[2] = fz;
  }
  *out = acc;
  return true;
}

// Channels d .. d + CH - 1 of a sample at positions with channels pim[k]
// (CH = 2: one 16-byte load per corner; needs Dp and d even).
template <int CH>
CSF_DEV void sample_channels(const VoxelStore& vox, const int* vid, const double* wgt, const double* ds,
                             const double (*pim)[3], double vs, double inv_vs2, int d, double* out) {
  double fv[8][CH];
  if constexpr (CH == 2) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const double2 v2 = __ldg(reinterpret_cast<const double2*>(vox.fim + static_cast<long long>(vid[c]) * vox.Dp + d));
      fv[c][0] = v2.x;
      fv[c][1] = v2.y;
    }
  } else {
#pragma unroll
    for (int c = 0; c < 8; ++c) fv[c][0] = __ldg(vox.fim + static_cast<long long>(vid[c]) * vox.Dp + d);
  }
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    double t = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a) t += ds[a] * CSF_CH_DIV(pim[k][a] * vs, vs * vs, inv_vs2);
#pragma unroll
    for (int c = 0; c < 8; ++c) t += wgt[c] * fv[c][k];
    out[k] = t;
  }
}

// Cooperative lift: the per-pixel real chain (2 crossing samples, 6
// gradient samples) is split over 8 lanes per pixel and its intermediates go
// to shared memory; then one thread per (pixel, channel) evaluates the
// tangent-form channel from them.  Real parts are bit-identical to the L<G>
// evaluation (same sample_real_ex arithmetic); each channel follows the
// truncated-Complex rule of every operation (csfd.hpp:44-58) applied to the
// saved real intermediates.  Many light threads keep far more voxel-channel gathers
// in flight than one heavy thread per (pixel, group).
// Per-sample rows of 9 (the real pass's 4 pixels x 8 samples per warp store
// one field offset together: rows of 8 gave 4-way bank conflicts) and an odd
// record size in doubles (161: the channel pass's lanes read ~6 pixels'
// records at one field offset; an even size put pixels p, p + 4 on one bank pair).
struct LiftRec {
  double wgt[8][9];
  double ds[8][3];
  double f[8];
  double dc[3], dn[3], dir[3], grad[3];
  double rn, a0, a1, astar, num, den, ln;
  int vid[8][9];
  int ok;
  int pad_[3];
};
static_assert(sizeof(LiftRec) % 16 == 8, "LiftRec: odd size in doubles");
constexpr int kLiftPix = 32;  // max pixels per block (8 lanes each in the real pass)
// pixels per block: as many as keep the channel pass to one round of items
// (items = channel-pass items per pixel)
inline int lift_pixels(int items) { return items <= 8 ? kLiftPix : (items >= 256 ? 1 : 256 / items); }
// Pixel p of a lift CTA: one 8x4 warp tile (tile_pixel) when the CTA takes
// 32 pixels, else npix consecutive pixels.  -1: outside the image.
CSF_DEV int lift_pixel(int npix, int p, int w, int h) {
  if (npix == kLiftPix) {
    int x, y;
    return tile_pixel(static_cast<long long>(blockIdx.x) * kLiftPix + p, w, h, &x, &y) ? y * w + x : -1;
  }
  const long long pix = static_cast<long long>(blockIdx.x) * npix + p;
  return pix < static_cast<long long>(w) * h ? static_cast<int>(pix) : -1;
}
inline unsigned lift_grid(int npix, int w, int h) {
  return static_cast<unsigned>(npix == kLiftPix ? tiled_count(w, h) / kLiftPix
                                                : (static_cast<long long>(w) * h + npix - 1) / npix);
}

#ifndef CSF_LIFT_MINB
#define CSF_LIFT_MINB 2
#endif
template <typename V, int CH>
__global__ void __launch_bounds__(256, CSF_LIFT_MINB) k_raycast_lift_coop(V vol, const double* __restrict__ pose,
                                                           const double* __restrict__ intr, int w, int h, int Dp,
                                                           const double2* __restrict__ hits, double* __restrict__ vre,
                                                           double* __restrict__ nre, double* __restrict__ vim,
                                                           double* __restrict__ nim, int npix) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ double sm[];
  const int C = 1 + Dp;
  LiftRec* recs = reinterpret_cast<LiftRec*>(sm + 16 * C);
  for (int i = threadIdx.x; i < 12 * C; i += blockDim.x) sm[i] = pose[i];
  for (int i = threadIdx.x; i < 4 * C; i += blockDim.x) sm[12 * C + i] = intr[i];
  __syncthreads();
  const double* kk = sm + 12 * C;
  const int P = w * h;
  const double hv = vol.vs;
  // ---- real pass: lane s of pixel p
  {
    const int p = threadIdx.x >> 3, s = threadIdx.x & 7;
    const int pix = p < npix ? lift_pixel(npix, p, w, h) : -1;
    LiftRec& r = recs[p < npix ? p : 0];
    // the crossing alphas and the march's two samples, loaded together
    double2 hit = make_double2(0.0, -1.0), fpair = make_double2(0.0, 0.0);
    if (pix >= 0) {
      hit = hits[pix];
      fpair = hits[P + pix];
    }
    const bool active = hit.y >= 0.0;
    const int x = pix >= 0 ? pix % w : 0, y = pix >= 0 ? pix / w : 0;
    double R[9], T[3];
#pragma unroll
    for (int e = 0; e < 9; ++e) R[e] = sm[e * C];
#pragma unroll
    for (int e = 0; e < 3; ++e) T[e] = sm[(9 + e) * C];
    const double fxk = kk[0], fyk = kk[C], cxk = kk[2 * C], cyk = kk[3 * C];
    const double tx = static_cast<double>(x) - cxk, ty = static_cast<double>(y) - cyk;
    const double dc[3] = {tx / fxk, ty / fyk, 1.0};
    const double rn = sqrt(dc[0] * dc[0] + (dc[1] * dc[1] + 1.0 * 1.0));
    const double dn[3] = {dc[0] / rn, dc[1] / rn, dc[2] / rn};
    double dir[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) dir[q] = R[3 * q] * dn[0] + (R[3 * q + 1] * dn[1] + R[3 * q + 2] * dn[2]);
    const double a0 = hit.x, a1 = hit.y;
    // f0, f1: the march's samples at a0, a1 (same arithmetic as sample_real_ex)
    const double f0 = active ? fpair.x : 0.0, f1 = active ? fpair.y : 0.0;
    const double span = a1 - a0;
    const double num = span * f0, den = f1 - f0;
    const double astar = a0 - num / den;
    const double vv[3] = {T[0] + astar * dir[0], T[1] + astar * dir[1], T[2] + astar * dir[2]};
    // all eight samples at once: lanes 0, 1 the crossing pair (corner data
    // for the channels), lanes 2..7 the central differences
    bool ok = true;
    double g = 0.0;
    if (active) {
      double q[3];
      if (s < 2) {
        const double a = s == 0 ? a0 : a1;
        q[0] = T[0] + a * dir[0];
        q[1] = T[1] + a * dir[1];
        q[2] = T[2] + a * dir[2];
      } else {
        const int axis = (s - 2) >> 1;
        q[0] = vv[0];
        q[1] = vv[1];
        q[2] = vv[2];
        q[axis] = (s & 1) ? q[axis] + hv : q[axis] - hv;
      }
      ok = sample_real_ex(vol, q[0], q[1], q[2], &g, r.vid[s], r.wgt[s], r.ds[s]) || s < 2;
    }
    const unsigned lane0 = (threadIdx.x & 31) & ~7u;
    const unsigned all_ok = __ballot_sync(0xffffffffu, ok);
    const bool group_ok = ((all_ok >> lane0) & 0xffu) == 0xffu;
    double fs[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) fs[k] = __shfl_sync(0xffffffffu, g, lane0 + 2 + k);
    if (s == 0 && p < npix) {
      bool good = active && group_ok;
      double grad[3], ln = 0.0;
#pragma unroll
      for (int a = 0; a < 3; ++a) grad[a] = (fs[2 * a + 1] - fs[2 * a]) / (2.0 * hv);
      const double len2 = grad[0] * grad[0] + (grad[1] * grad[1] + grad[2] * grad[2]);
      good = good && len2 > 0.0;
      if (good) {
        ln = sqrt(len2);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          vre[3LL * pix + c] = vv[c];
          nre[3LL * pix + c] = grad[c] / ln;
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          r.dc[c] = dc[c];
          r.dn[c] = dn[c];
          r.dir[c] = dir[c];
          r.grad[c] = grad[c];
        }
        r.f[0] = f0;
        r.f[1] = f1;
        r.rn = rn;
        r.a0 = a0;
        r.a1 = a1;
        r.astar = astar;
        r.num = num;
        r.den = den;
        r.ln = ln;
      }
      r.ok = good ? 1 : 0;
    }
  }
  __syncthreads();
  if (Dp == 0) return;
  // ---- channel pass: one thread per (pixel, CH channels); CH = 2 gathers
  // each corner's two channels with one 16-byte load (twice the pixels per
  // warp-wide gather, so adjacent pixels' shared voxels cost one L1 line)
  const double fxk = kk[0], fyk = kk[C];
  const double inv_fx2 = 1.0 / (fxk * fxk), inv_fy2 = 1.0 / (fyk * fyk), inv_vs2 = 1.0 / (hv * hv);
  const double inv_2h2 = 1.0 / ((2.0 * hv) * (2.0 * hv));
  (void)inv_fx2; (void)inv_fy2; (void)inv_vs2; (void)inv_2h2;
  const int Dh = Dp / CH;
  for (int it = threadIdx.x; it < npix * Dh; it += blockDim.x) {
    const int p = it / Dh, d = (it - p * Dh) * CH;
    const LiftRec& r = recs[p];
    const int pix = lift_pixel(npix, p, w, h);
    if (pix < 0) continue;
    if (!r.ok) {  // no surface: zero channels (no separate memset of the maps)
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int k = 0; k < CH; ++k) {
          vim[(3LL * pix + c) * Dp + d + k] = 0.0;
          nim[(3LL * pix + c) * Dp + d + k] = 0.0;
        }
      continue;
    }
    const int x = pix % w, y = pix / w;
    const double tx = static_cast<double>(x) - kk[2 * C], ty = static_cast<double>(y) - kk[3 * C];
    const double rn = r.rn, den = r.den, num = r.num, ln = r.ln;
    const double inv_rn2 = 1.0 / (rn * rn), inv_den2 = 1.0 / (den * den), inv_ln2 = 1.0 / (ln * ln);
    (void)inv_rn2; (void)inv_den2; (void)inv_ln2;
    double diri[CH][3], Ti[CH][3];
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      const int ch = 1 + d + k;
      const double dci[3] = {CSF_CH_DIV(-kk[2 * C + ch] * fxk - tx * kk[ch], fxk * fxk, inv_fx2),
                             CSF_CH_DIV(-kk[3 * C + ch] * fyk - ty * kk[C + ch], fyk * fyk, inv_fy2), 0.0};
      const double doti = (r.dc[0] * dci[0] + dci[0] * r.dc[0]) + ((r.dc[1] * dci[1] + dci[1] * r.dc[1]) + 0.0);
      const double rni = (0.5 / rn) * doti;
      double dni[3];
#pragma unroll
      for (int a2 = 0; a2 < 3; ++a2) dni[a2] = CSF_CH_DIV(dci[a2] * rn - r.dc[a2] * rni, rn * rn, inv_rn2);
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const double t0 = sm[(3 * q) * C] * dni[0] + sm[(3 * q) * C + ch] * r.dn[0];
        const double t1 = sm[(3 * q + 1) * C] * dni[1] + sm[(3 * q + 1) * C + ch] * r.dn[1];
        const double t2 = sm[(3 * q + 2) * C] * dni[2] + sm[(3 * q + 2) * C + ch] * r.dn[2];
        diri[k][q] = t0 + (t1 + t2);
        Ti[k][q] = sm[(9 + q) * C + ch];
      }
    }
    double f0i[CH], f1i[CH];
    {
      double q0i[CH][3], q1i[CH][3];
#pragma unroll
      for (int k = 0; k < CH; ++k)
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          q0i[k][q] = Ti[k][q] + r.a0 * diri[k][q];
          q1i[k][q] = Ti[k][q] + r.a1 * diri[k][q];
        }
      sample_channels<CH>(vol.vox, r.vid[0], r.wgt[0], r.ds[0], q0i, hv, inv_vs2, d, f0i);
      sample_channels<CH>(vol.vox, r.vid[1], r.wgt[1], r.ds[1], q1i, hv, inv_vs2, d, f1i);
    }
    double vvi[CH][3];
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      const double numi = (r.a1 - r.a0) * f0i[k], deni = f1i[k] - f0i[k];
      const double asti = -CSF_CH_DIV(numi * den - num * deni, den * den, inv_den2);
#pragma unroll
      for (int a2 = 0; a2 < 3; ++a2) vvi[k][a2] = Ti[k][a2] + (r.astar * diri[k][a2] + asti * r.dir[a2]);
    }
    double gi[CH][3];
#pragma unroll
    for (int axis = 0; axis < 3; ++axis) {
      double lo[CH], hi[CH];
      sample_channels<CH>(vol.vox, r.vid[2 + 2 * axis], r.wgt[2 + 2 * axis], r.ds[2 + 2 * axis], vvi, hv, inv_vs2, d,
                          lo);
      sample_channels<CH>(vol.vox, r.vid[3 + 2 * axis], r.wgt[3 + 2 * axis], r.ds[3 + 2 * axis], vvi, hv, inv_vs2, d,
                          hi);
#pragma unroll
      for (int k = 0; k < CH; ++k)
        gi[k][axis] = CSF_CH_DIV((hi[k] - lo[k]) * (2.0 * hv), (2.0 * hv) * (2.0 * hv), inv_2h2);
    }
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      const double l2i = (r.grad[0] * gi[k][0] + gi[k][0] * r.grad[0]) +
                         ((r.grad[1] * gi[k][1] + gi[k][1] * r.grad[1]) + (r.grad[2] * gi[k][2] + gi[k][2] * r.grad[2]));
      const double lni = (0.5 / ln) * l2i;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        vim[(3LL * pix + c) * Dp + d + k] = vvi[k][c];
        nim[(3LL * pix + c) * Dp + d + k] = CSF_CH_DIV(gi[k][c] * ln - r.grad[c] * lni, ln * ln, inv_ln2);
      }
    }
  }
}

// ---- second order, cooperative: the per-pixel real pass of the first-order
// lift (8 lanes per pixel: the crossing pair and the 6 central differences)
// records each sample's corner voxels and their real fields; then one thread
// per (pixel, pair) evaluates the lifted epilogue of raycast<S> (tsdf.hpp:
// 255-284) in Bicomplex arithmetic with those corners (no block lookups, no
// (F, W) loads): sample_tsdf<S> / sample_gradient<S>'s operations.
// Per-sample rows at odd strides (9, 3, 13) and a record size of 8 mod 16
// doubles: the real pass's 32 lanes (4 pixels x 8 samples) store one field
// offset together, and these strides put each half-warp on distinct bank
// pairs (the 8-double rows gave 8-way conflicts).
struct LiftRec2 {
  double F[8][9];  // corner real fields per sample
  int vid[8][9];   // corner voxel ids per sample
  int ok;
  int pad_;
#ifndef CSF_EXACT_CHANNELS
  // tangent form: per sample the trilinear weights, dS/df (ds), the mixed
  // second derivatives d2S/df_a df_b (E: xy, xz, yz) and the weight products
  // of the edge differences (wp: 4 x wy wz, 4 x wx wz, 4 x wx wy); per pixel
  // the real intermediates of the epilogue
  double wgt[8][9];
  double ds[8][3];
  double E[8][3];
  double wp[8][13];
  double dc[2], rn, a0, a1, f0, f1, num, den, astar, ln;
  double dn[3], dir[3], grad[3];
  double pad2_[7];
#endif
};
#ifndef CSF_EXACT_CHANNELS
static_assert(sizeof(LiftRec2) % 128 == 64, "LiftRec2: 8 mod 16 doubles");
#endif

// sample_tsdf<S> (order-2 branch) with the corners known and valid.
template <typename S, typename V>
CSF_DEV S sample_tsdf_at(const V& vol, const V3<S>& p, const int* vid, const double* F, int g0) {
  const S gx = (p.v[0] - vol.ox) / vol.vs;
  const S gy = (p.v[1] - vol.oy) / vol.vs;
  const S gz = (p.v[2] - vol.oz) / vol.vs;
  const int i0 = ifloor(re(gx)), j0 = ifloor(re(gy)), k0 = ifloor(re(gz));
  const S fx = gx - static_cast<double>(i0);
  const S fy = gy - static_cast<double>(j0);
  const S fz = gz - static_cast<double>(k0);
  S accum = lit<S>(0.0);
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const S wx = (c & 1) ? fx : 1.0 - fx;
    const S wy = ((c >> 1) & 1) ? fy : 1.0 - fy;
    const S wz = (c >> 2) ? fz : 1.0 - fz;
    accum = accum + ((wx * wy) * wz) * field_at<S>(vol.vox, vid[c], F[c], g0);
  }
  return accum;
}

template <typename V>
__global__ void __launch_bounds__(256) k_raycast_lift2_coop(V vol, const double* __restrict__ pose,
                                                            const double* __restrict__ intr, int w, int h, int Dp,
                                                            const double2* __restrict__ hits, double* __restrict__ vre,
                                                            double* __restrict__ nre, double* __restrict__ vim,
                                                            double* __restrict__ nim) {
  pdl_wait();
  pdl_trigger();
  using S = B<1>;
  constexpr int G = Traits<S>::G;
  extern __shared__ double sm[];
  const int C = 1 + Dp;
  LiftRec2* recs = reinterpret_cast<LiftRec2*>(sm + 16 * C);
  for (int i = threadIdx.x; i < 12 * C; i += blockDim.x) sm[i] = pose[i];
  for (int i = threadIdx.x; i < 4 * C; i += blockDim.x) sm[12 * C + i] = intr[i];
  __syncthreads();
  const double* kk = sm + 12 * C;
  const int P = w * h;
  const double hv = vol.vs;
  // ---- real pass: lane s of pixel p (k_raycast_lift_coop's arithmetic)
  {
    const int p = threadIdx.x >> 3, s = threadIdx.x & 7;
    const int pix = lift_pixel(kLiftPix, p, w, h);
    LiftRec2& r = recs[p];
    double2 hit = make_double2(0.0, -1.0), fpair = make_double2(0.0, 0.0);
    if (pix >= 0) {
      hit = hits[pix];
      fpair = hits[P + pix];
    }
    const bool active = hit.y >= 0.0;
    const int x = pix >= 0 ? pix % w : 0, y = pix >= 0 ? pix / w : 0;
    double R[9], T[3];
#pragma unroll
    for (int e = 0; e < 9; ++e) R[e] = sm[e * C];
#pragma unroll
    for (int e = 0; e < 3; ++e) T[e] = sm[(9 + e) * C];
    const double fxk = kk[0], fyk = kk[C], cxk = kk[2 * C], cyk = kk[3 * C];
    const double tx = static_cast<double>(x) - cxk, ty = static_cast<double>(y) - cyk;
    const double dc[3] = {tx / fxk, ty / fyk, 1.0};
    const double rn = sqrt(dc[0] * dc[0] + (dc[1] * dc[1] + 1.0 * 1.0));
    const double dn[3] = {dc[0] / rn, dc[1] / rn, dc[2] / rn};
    double dir[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) dir[q] = R[3 * q] * dn[0] + (R[3 * q + 1] * dn[1] + R[3 * q + 2] * dn[2]);
    const double a0 = hit.x, a1 = hit.y;
    const double f0 = active ? fpair.x : 0.0, f1 = active ? fpair.y : 0.0;
    const double astar = a0 - ((a1 - a0) * f0) / (f1 - f0);
    const double vv[3] = {T[0] + astar * dir[0], T[1] + astar * dir[1], T[2] + astar * dir[2]};
    bool ok = true;
    double g = 0.0;
    if (active) {
      double q[3];
      if (s < 2) {
        const double a = s == 0 ? a0 : a1;
        q[0] = T[0] + a * dir[0];
        q[1] = T[1] + a * dir[1];
        q[2] = T[2] + a * dir[2];
      } else {
        const int axis = (s - 2) >> 1;
        q[0] = vv[0];
        q[1] = vv[1];
        q[2] = vv[2];
        q[axis] = (s & 1) ? q[axis] + hv : q[axis] - hv;
      }
#ifndef CSF_EXACT_CHANNELS
      double fr[3];
      ok = sample_real_ex(vol, q[0], q[1], q[2], &g, r.vid[s], r.wgt[s], r.ds[s], r.F[s], fr);
      if (ok) {
        const double wx[2] = {1.0 - fr[0], fr[0]}, wy[2] = {1.0 - fr[1], fr[1]}, wz[2] = {1.0 - fr[2], fr[2]};
        double exy = 0.0, exz = 0.0, eyz = 0.0;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int cx = c & 1, cy = (c >> 1) & 1, cz = c >> 2;
          const double sgx = cx ? 1.0 : -1.0, sgy = cy ? 1.0 : -1.0, sgz = cz ? 1.0 : -1.0;
          exy += (sgx * sgy) * wz[cz] * r.F[s][c];
          exz += (sgx * sgz) * wy[cy] * r.F[s][c];
          eyz += (sgy * sgz) * wx[cx] * r.F[s][c];
        }
        r.E[s][0] = exy;
        r.E[s][1] = exz;
        r.E[s][2] = eyz;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          r.wp[s][m] = wy[m & 1] * wz[m >> 1];
          r.wp[s][4 + m] = wx[m & 1] * wz[m >> 1];
          r.wp[s][8 + m] = wx[m & 1] * wy[m >> 1];
        }
      }
#else
      double wgt[8], ds[3];
      ok = sample_real_ex(vol, q[0], q[1], q[2], &g, r.vid[s], wgt, ds, r.F[s]);
#endif
    }
    const unsigned lane0 = (threadIdx.x & 31) & ~7u;
    const unsigned all_ok = __ballot_sync(0xffffffffu, ok);
    const bool group_ok = ((all_ok >> lane0) & 0xffu) == 0xffu;
    double fs[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) fs[k] = __shfl_sync(0xffffffffu, g, lane0 + 2 + k);
    if (s == 0) {
      bool good = active && group_ok;
      double grad[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) grad[a] = (fs[2 * a + 1] - fs[2 * a]) / (2.0 * hv);
      const double len2 = grad[0] * grad[0] + (grad[1] * grad[1] + grad[2] * grad[2]);
      good = good && len2 > 0.0;
      r.ok = good ? 1 : 0;
#ifndef CSF_EXACT_CHANNELS
      if (good) {
        // the real outputs (bit-identical to the Bicomplex chain's real parts)
        const double ln = sqrt(len2);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          vre[3LL * pix + c] = vv[c];
          nre[3LL * pix + c] = grad[c] / ln;
          r.dn[c] = dn[c];
          r.dir[c] = dir[c];
          r.grad[c] = grad[c];
        }
        r.dc[0] = dc[0];
        r.dc[1] = dc[1];
        r.rn = rn;
        r.a0 = a0;
        r.a1 = a1;
        r.f0 = f0;
        r.f1 = f1;
        r.num = (a1 - a0) * f0;
        r.den = f1 - f0;
        r.astar = astar;
        r.ln = ln;
      }
#endif
    }
  }
  __syncthreads();
#ifndef CSF_EXACT_CHANNELS
  // ---- one thread per (pixel, pair): the Bicomplex epilogue in tangent form
  // (Ch3 slots over the recorded reals; the trilinear samples through their
  // weights, first and mixed second derivatives in the cell fractions)
  {
    const int passes = Dp / G;
    const double ivs = 1.0 / hv, i2h = 1.0 / (2.0 * hv);
    for (int it = threadIdx.x; it < kLiftPix * passes; it += blockDim.x) {
      const int p = it / passes, gi = it - p * passes;
      const LiftRec2& r = recs[p];
      const int pix = lift_pixel(kLiftPix, p, w, h);
      if (pix < 0 || !r.ok) continue;
      const int x = pix % w, y = pix / w;
      const int o = 1 + gi * G;
      const double fxk = kk[0], fyk = kk[C], cxk = kk[2 * C], cyk = kk[3 * C];
      const Ch3 cfx = ch_at(kk, o), cfy = ch_at(kk + C, o), ccx = ch_at(kk + 2 * C, o), ccy = ch_at(kk + 3 * C, o);
      // dcs = ((x - cx) / fx, (y - cy) / fy, 1)
      const double ifx = 1.0 / fxk, ify = 1.0 / fyk;
      const Ch3 zero = {0.0, 0.0, 0.0};
      const Ch3 dc0 = ch_div(static_cast<double>(x) - cxk, ch_scale(ccx, -1.0), fxk, cfx, ifx, ifx * ifx);
      const Ch3 dc1 = ch_div(static_cast<double>(y) - cyk, ch_scale(ccy, -1.0), fyk, cfy, ify, ify * ify);
      // rns = sqrt(dot(dcs, dcs)); dn = dcs / rns
      const double rn2 = r.dc[0] * r.dc[0] + (r.dc[1] * r.dc[1] + 1.0 * 1.0);
      const double l1 = 0.5 / r.rn, l2 = (-0.5 * l1) / rn2;
      const Ch3 rnc = ch_lift(ch_add(ch_mul(r.dc[0], dc0, r.dc[0], dc0), ch_mul(r.dc[1], dc1, r.dc[1], dc1)), l1, l2);
      const double irn = 1.0 / r.rn, irn2 = irn * irn;
      const Ch3 dnc[3] = {ch_div(r.dc[0], dc0, r.rn, rnc, irn, irn2), ch_div(r.dc[1], dc1, r.rn, rnc, irn, irn2),
                          ch_div(1.0, zero, r.rn, rnc, irn, irn2)};
      // dirs = R dn; T = t
      Ch3 dirc[3], Tc[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const Ch3 m0 = ch_mul(sm[(3 * q) * C], ch_at(sm + (3 * q) * C, o), r.dn[0], dnc[0]);
        const Ch3 m1 = ch_mul(sm[(3 * q + 1) * C], ch_at(sm + (3 * q + 1) * C, o), r.dn[1], dnc[1]);
        const Ch3 m2 = ch_mul(sm[(3 * q + 2) * C], ch_at(sm + (3 * q + 2) * C, o), r.dn[2], dnc[2]);
        dirc[q] = ch_add(m0, ch_add(m1, m2));
        Tc[q] = ch_at(sm + (9 + q) * C, o);
      }
      // a trilinear sample of recorded sample s at a position with channels pc
      auto sample = [&](int sidx, const Ch3* pc) {
        const int* vid = r.vid[sidx];
        Ch3 Gc[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const double* src = vol.vox.fim + static_cast<long long>(vid[c]) * vol.vox.Dp + (o - 1);
          Gc[c] = {__ldg(src), __ldg(src + 1), __ldg(src + 2)};
        }
        Ch3 fr[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) fr[a] = ch_scale(pc[a], ivs);
        Ch3 acc = zero;
#pragma unroll
        for (int c = 0; c < 8; ++c) acc = ch_add(acc, ch_scale(Gc[c], r.wgt[sidx][c]));
        // dS/df of the im1 and im2 fields (edge differences)
        double d1[3], d2[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const int st = 1 << a;
          double s1 = 0.0, s2 = 0.0;
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            // the four edges along axis a: low corner index with bit a clear
            const int lo = a == 0 ? 2 * m : a == 1 ? (m & 1) + 4 * (m >> 1) : m;
            s1 += r.wp[sidx][4 * a + m] * (Gc[lo + st].a - Gc[lo].a);
            s2 += r.wp[sidx][4 * a + m] * (Gc[lo + st].b - Gc[lo].b);
          }
          d1[a] = s1;
          d2[a] = s2;
        }
        const double* D = r.ds[sidx];
        const double* E = r.E[sidx];
        Ch3 out;
        out.a = acc.a + ((D[0] * fr[0].a + D[1] * fr[1].a) + D[2] * fr[2].a);
        out.b = acc.b + ((D[0] * fr[0].b + D[1] * fr[1].b) + D[2] * fr[2].b);
        out.ab = acc.ab + ((D[0] * fr[0].ab + D[1] * fr[1].ab) + D[2] * fr[2].ab) +
                 (((d1[0] * fr[0].b + d1[1] * fr[1].b) + d1[2] * fr[2].b) +
                  ((d2[0] * fr[0].a + d2[1] * fr[1].a) + d2[2] * fr[2].a)) +
                 ((E[0] * (fr[0].a * fr[1].b + fr[1].a * fr[0].b) + E[1] * (fr[0].a * fr[2].b + fr[2].a * fr[0].b)) +
                  E[2] * (fr[1].a * fr[2].b + fr[2].a * fr[1].b));
        return out;
      };
      Ch3 q0[3], q1[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        q0[a] = ch_add(Tc[a], ch_scale(dirc[a], r.a0));
        q1[a] = ch_add(Tc[a], ch_scale(dirc[a], r.a1));
      }
      const Ch3 flp = sample(0, q0), flh = sample(1, q1);
      // astar = a0 - (span f0) / (f1 - f0)
      const double iden = 1.0 / r.den;
      const Ch3 qa = ch_div(r.num, ch_scale(flp, r.a1 - r.a0), r.den, ch_sub(flh, flp), iden, iden * iden);
      const Ch3 ast = ch_scale(qa, -1.0);
      Ch3 vc[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) vc[a] = ch_add(Tc[a], ch_mul(r.astar, ast, r.dir[a], dirc[a]));
      Ch3 gc[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) gc[a] = ch_scale(ch_sub(sample(3 + 2 * a, vc), sample(2 + 2 * a, vc)), i2h);
      // n = grad / |grad|
      const double len2 = r.grad[0] * r.grad[0] + (r.grad[1] * r.grad[1] + r.grad[2] * r.grad[2]);
      const double n1 = 0.5 / r.ln, n2 = (-0.5 * n1) / len2;
      const Ch3 lnc = ch_lift(ch_add(ch_mul(r.grad[0], gc[0], r.grad[0], gc[0]),
                                     ch_add(ch_mul(r.grad[1], gc[1], r.grad[1], gc[1]),
                                            ch_mul(r.grad[2], gc[2], r.grad[2], gc[2]))),
                              n1, n2);
      const double iln = 1.0 / r.ln, iln2 = iln * iln;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const Ch3 nc = ch_div(r.grad[c], gc[c], r.ln, lnc, iln, iln2);
        double* vi = vim + (3LL * pix + c) * Dp + (o - 1);
        double* ni = nim + (3LL * pix + c) * Dp + (o - 1);
        vi[0] = vc[c].a;
        vi[1] = vc[c].b;
        vi[2] = vc[c].ab;
        ni[0] = nc.a;
        ni[1] = nc.b;
        ni[2] = nc.ab;
      }
    }
    return;
  }
#endif
  // ---- one thread per (pixel, pair): the Bicomplex chain
  const int passes = Dp / G;
  for (int it = threadIdx.x; it < kLiftPix * passes; it += blockDim.x) {
    const int p = it / passes, gi = it - p * passes;
    const LiftRec2& r = recs[p];
    const int pix = lift_pixel(kLiftPix, p, w, h);
    if (pix < 0 || !r.ok) continue;
    const double2 hit = hits[pix];
    const double alpha_prev = hit.x, alpha_hit = hit.y;
    const int x = pix % w, y = pix / w;
    const int g0 = gi * G;
    Pose<S> Ps;
#pragma unroll
    for (int e = 0; e < 9; ++e) Ps.R.m[e] = load_ch<S>(sm + e * C, g0, G);
#pragma unroll
    for (int e = 0; e < 3; ++e) Ps.t.v[e] = load_ch<S>(sm + (9 + e) * C, g0, G);
    const S fx = load_ch<S>(kk, g0, G), fy = load_ch<S>(kk + C, g0, G);
    const S cx = load_ch<S>(kk + 2 * C, g0, G), cy = load_ch<S>(kk + 3 * C, g0, G);
    const S one = lit<S>(1.0);
    const V3<S> dcs = mk3<S>((static_cast<double>(x) - cx) / fx, (static_cast<double>(y) - cy) / fy, one);
    const S rns = sqrt_s(dot3(dcs, dcs));
    const V3<S> dirs = matvec(Ps.R, mk3<S>(dcs.v[0] / rns, dcs.v[1] / rns, dcs.v[2] / rns));
    const V3<S>& os = Ps.t;
    auto at = [&](double a) {
      return mk3<S>(os.v[0] + a * dirs.v[0], os.v[1] + a * dirs.v[1], os.v[2] + a * dirs.v[2]);
    };
    const S fl_prev = sample_tsdf_at<S>(vol, at(alpha_prev), r.vid[0], r.F[0], g0);
    const S fl = sample_tsdf_at<S>(vol, at(alpha_hit), r.vid[1], r.F[1], g0);
    const double span = alpha_hit - alpha_prev;
    const S astar = alpha_prev - (span * fl_prev) / (fl - fl_prev);
    const V3<S> v = mk3<S>(os.v[0] + astar * dirs.v[0], os.v[1] + astar * dirs.v[1], os.v[2] + astar * dirs.v[2]);
    V3<S> grad;
#pragma unroll
    for (int axis = 0; axis < 3; ++axis) {  // sample_gradient<S> (tsdf.hpp:181-196)
      V3<S> lo = v, hi = v;
      lo.v[axis] = lo.v[axis] - hv;
      hi.v[axis] = hi.v[axis] + hv;
      const S flo = sample_tsdf_at<S>(vol, lo, r.vid[2 + 2 * axis], r.F[2 + 2 * axis], g0);
      const S fhi = sample_tsdf_at<S>(vol, hi, r.vid[3 + 2 * axis], r.F[3 + 2 * axis], g0);
      grad.v[axis] = (fhi - flo) / (2.0 * hv);
    }
    const S len2 = dot3(grad, grad);
    const S ln = sqrt_s(len2);
    const V3<S> n = mk3<S>(grad.v[0] / ln, grad.v[1] / ln, grad.v[2] / ln);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      if (gi == 0) {
        vre[3LL * pix + c] = re(v.v[c]);
        nre[3LL * pix + c] = re(n.v[c]);
      }
      double* vi = vim + (3LL * pix + c) * Dp + g0;
      double* ni = nim + (3LL * pix + c) * Dp + g0;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        vi[g] = v.v[c].im[g];
        ni[g] = n.v[c].im[g];
      }
    }
  }
}

}  // namespace csfd

// ============================================================================
namespace csfi {

using namespace csfd;

static void chk(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) note_launch_error(what, e);
}

int pick_group(int D) {
  if (D <= 0) return 0;
  if (D <= 6) return D;
  int best = 4, best_dp = padded_channels(D, 4);
  for (int g : {5, 6}) {
    const int dp = padded_channels(D, g);
    if (dp <= best_dp) {
      best = g;
      best_dp = dp;
    }
  }
  return best;
}

#define CSF_DISPATCH_G(G, BODY)                       \
  switch (G) {                                        \
    case 0: { constexpr int kG = 0; BODY; } break;    \
    case 1: { constexpr int kG = 1; BODY; } break;    \
    case 2: { constexpr int kG = 2; BODY; } break;    \
    case 3: { constexpr int kG = 3; BODY; } break;    \
    case 4: { constexpr int kG = 4; BODY; } break;    \
    case 5: { constexpr int kG = 5; BODY; } break;    \
    case 6: { constexpr int kG = 6; BODY; } break;    \
    default: note_error("csf_b200: no kernel for group width " + std::to_string(G)); \
  }

// Compile-time channel counts of the adjoint fusion kernels (all channel
// loads of a voxel issued together); other counts use the runtime loop.
static bool fixed_channels(int Dp) { return (Dp >= 1 && Dp <= 12) || Dp == 16 || Dp == 20 || Dp == 24; }
#define CSF_DISPATCH_NDP(Dp, BODY)                                                       \
  switch (Dp) {                                                                         \
    case 1: { constexpr int kN = 1; BODY; } break;    case 2: { constexpr int kN = 2; BODY; } break;   \
    case 3: { constexpr int kN = 3; BODY; } break;    case 4: { constexpr int kN = 4; BODY; } break;   \
    case 5: { constexpr int kN = 5; BODY; } break;    case 6: { constexpr int kN = 6; BODY; } break;   \
    case 7: { constexpr int kN = 7; BODY; } break;    case 8: { constexpr int kN = 8; BODY; } break;   \
    case 9: { constexpr int kN = 9; BODY; } break;    case 10: { constexpr int kN = 10; BODY; } break; \
    case 11: { constexpr int kN = 11; BODY; } break;  case 12: { constexpr int kN = 12; BODY; } break; \
    case 16: { constexpr int kN = 16; BODY; } break;  case 20: { constexpr int kN = 20; BODY; } break; \
    case 24: { constexpr int kN = 24; BODY; } break;                                               \
    default: note_error("csf_b200: no fusion kernel for " + std::to_string(Dp) + " channels");     \
  }

static DenseView dense_view(const DenseDev& v, int Dp) {
  DenseView d;
  d.vox = {v.rw, v.fim, Dp};
  d.nx = v.nx; d.ny = v.ny; d.nz = v.nz;
  d.vs = v.vs; d.ox = v.ox; d.oy = v.oy; d.oz = v.oz; d.mu = v.mu; d.cap = v.cap;
  return d;
}
static HashView hash_view(const HashDev& v, int Dp) {
  HashView d;
  d.vox = {v.rw, v.fim, Dp};
  d.heads = v.heads; d.keys = v.keys; d.next = v.next;
  d.grid = v.grid;
  d.occ = v.occ;
  d.sdist = v.sdist;
  d.gbits = v.gbits;
  d.mask = (1u << v.bits) - 1u;
  d.vs = v.vs; d.ox = v.ox; d.oy = v.oy; d.oz = v.oz; d.mu = v.mu; d.cap = v.cap;
  return d;
}

}  // namespace csfi

namespace csfd {
// ----------------------------------------------------------------------------
// Point queries of the stage API (tsdf.hpp:97-196): one thread per (point,
// channel) in L<1> (or double without channels); the real part is the
// reference's and bit-identical in every channel thread.
// ----------------------------------------------------------------------------
template <typename S>
CSF_DEV V3<S> load_point(const double* pts, int i, int C, int ch) {
  V3<S> p;
#pragma unroll
  for (int c = 0; c < 3; ++c) p.v[c] = load_ch<S>(pts + (3LL * i + c) * C, ch, 1);
  return p;
}

template <typename V, typename S>
__global__ void k_sample_points(V vol, const double* __restrict__ pts, int n, int Dp, int grad,
                                double* __restrict__ out, int* __restrict__ valid) {
  pdl_wait();
  pdl_trigger();
  const int lanes = Dp > 0 ? Dp : 1;
  const long long item = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (item >= static_cast<long long>(n) * lanes) return;
  const int i = static_cast<int>(item / lanes), ch = static_cast<int>(item % lanes);
  const int C = 1 + Dp;
  const V3<S> p = load_point<S>(pts, i, C, ch);
  NoCache cache;
  bool ok;
  if (!grad) {
    S f;
    ok = sample_tsdf<S>(vol, p, ch, &f, cache);
    if (ok) store_ch<S>(out + static_cast<long long>(i) * C, f, ch, Dp > 0 ? 1 : 0, ch == 0);
  } else {
    V3<S> g;
    ok = sample_gradient<S>(vol, p, ch, &g, cache);
    if (ok)
#pragma unroll
      for (int c = 0; c < 3; ++c) store_ch<S>(out + (3LL * i + c) * C, g.v[c], ch, Dp > 0 ? 1 : 0, ch == 0);
  }
  if (ch == 0) valid[i] = ok ? 1 : 0;
}

// measured_tsdf at real voxel positions pts [n][3] for a lifted world->camera
// pose, lifted intrinsics and lifted camera centre.
template <typename S>
__global__ void k_measured_points(const double* __restrict__ depth, int w, int h, const double* __restrict__ w2c,
                                  const double* __restrict__ intr, double mu, const double* __restrict__ pts,
                                  const double* __restrict__ center, int n, int Dp, double* __restrict__ out,
                                  int* __restrict__ valid, const double* __restrict__ dch) {
  pdl_wait();
  pdl_trigger();
  const int lanes = Dp > 0 ? Dp : 1;
  const long long item = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (item >= static_cast<long long>(n) * lanes) return;
  const int i = static_cast<int>(item / lanes), ch = static_cast<int>(item % lanes);
  const int C = 1 + Dp, G = Dp > 0 ? 1 : 0;
  Pose<S> pose;
#pragma unroll
  for (int e = 0; e < 9; ++e) pose.R.m[e] = load_ch<S>(w2c + e * C, ch, G);
#pragma unroll
  for (int e = 0; e < 3; ++e) pose.t.v[e] = load_ch<S>(w2c + (9 + e) * C, ch, G);
  Intr<S> k;
  k.fx = load_ch<S>(intr, ch, G);
  k.fy = load_ch<S>(intr + C, ch, G);
  k.cx = load_ch<S>(intr + 2 * C, ch, G);
  k.cy = load_ch<S>(intr + 3 * C, ch, G);
  k.w = w;
  k.h = h;
  V3<S> c;
#pragma unroll
  for (int e = 0; e < 3; ++e) c.v[e] = load_ch<S>(center + e * C, ch, G);
  S psi;
  const bool ok = measured_tsdf<S>(depth, w, h, pose, k, mu, pts[3LL * i], pts[3LL * i + 1], pts[3LL * i + 2], c, &psi,
                                   dch, Dp, ch);
  if (ok) store_ch<S>(out + static_cast<long long>(i) * C, psi, ch, G, ch == 0);
  if (ch == 0) valid[i] = ok ? 1 : 0;
}
}  // namespace csfd

namespace csfi {

void launch_sample_points(const Launch& L, bool hashed, const DenseDev& dd, const HashDev& hd, int Dp,
                          const double* pts, int n, int grad, double* out, int* valid) {
  const long long items = static_cast<long long>(n) * (Dp > 0 ? Dp : 1);
  const dim3 grid(static_cast<unsigned>((items + 127) / 128)), block(128);
  if (items == 0) return;
  if (hashed) {
    const HashView v = hash_view(hd, Dp);
    if (Dp > 0) launch_pdl(k_sample_points<HashView, csfd::L<1>>, grid, block, 0, L.stream, v, pts, n, Dp, grad, out, valid);
    else launch_pdl(k_sample_points<HashView, double>, grid, block, 0, L.stream, v, pts, n, Dp, grad, out, valid);
  } else {
    const DenseView v = dense_view(dd, Dp);
    if (Dp > 0) launch_pdl(k_sample_points<DenseView, csfd::L<1>>, grid, block, 0, L.stream, v, pts, n, Dp, grad, out, valid);
    else launch_pdl(k_sample_points<DenseView, double>, grid, block, 0, L.stream, v, pts, n, Dp, grad, out, valid);
  }
  ++*L.launches;
  chk("sample_points");
}

void launch_measured_points(const Launch& L, const double* depth, int w, int h, const double* w2c, const double* intr,
                            double mu, const double* pts, const double* center, int n, int Dp, double* out,
                            int* valid, const double* dch) {
  const long long items = static_cast<long long>(n) * (Dp > 0 ? Dp : 1);
  if (items == 0) return;
  const dim3 grid(static_cast<unsigned>((items + 127) / 128)), block(128);
  if (Dp > 0)
    launch_pdl(k_measured_points<csfd::L<1>>, grid, block, 0, L.stream, depth, w, h, w2c, intr, mu, pts, center, n, Dp, out,
               valid, dch);
  else
    launch_pdl(k_measured_points<double>, grid, block, 0, L.stream, depth, w, h, w2c, intr, mu, pts, center, n, Dp,
               out, valid, static_cast<const double*>(nullptr));
  ++*L.launches;
  chk("measured_points");
}

// Super-block distance field: separable L-infinity distance transform of the
// occupancy bitmap over the 2^(gbits-3) cube of super-blocks, capped at 8;
// cells outside the window count as occupied (unknown).
__global__ void k_sdist_axis(const unsigned* __restrict__ occ, const unsigned char* __restrict__ in, int sb, int axis,
                             unsigned char* __restrict__ out) {
  const int n = 1 << sb;
  const long long cell = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (cell >= (1LL << (3 * sb))) return;
  const int x = static_cast<int>(cell & (n - 1)), y = static_cast<int>((cell >> sb) & (n - 1)),
            z = static_cast<int>(cell >> (2 * sb));
  const int c[3] = {x, y, z};
  int best = 8;
  for (int d = -7; d <= 7; ++d) {
    int q[3] = {c[0], c[1], c[2]};
    q[axis] += d;
    const int ad = d < 0 ? -d : d;
    int v;
    if (q[axis] < 0 || q[axis] >= n) {
      v = 0;  // outside the window: treated as occupied
    } else {
      const long long qc = (static_cast<long long>(q[2]) << (2 * sb)) | (static_cast<long long>(q[1]) << sb) | q[0];
      v = in ? in[qc] : static_cast<int>(!((occ[qc >> 5] >> (qc & 31)) & 1u)) * 8;  // 0 occupied, 8 empty
    }
    const int m = ad > v ? ad : v;
    best = m < best ? m : best;
  }
  out[cell] = static_cast<unsigned char>(best);
}

void launch_super_dist(cudaStream_t stream, const HashDev& v) {
  if (!v.sdist || !v.sdist_tmp) return;
  const int sb = v.gbits - 3;
  const long long cells = 1LL << (3 * sb);
  const int grid = static_cast<int>((cells + 255) / 256);
  k_sdist_axis<<<grid, 256, 0, stream>>>(v.occ, nullptr, sb, 0, v.sdist_tmp);
  k_sdist_axis<<<grid, 256, 0, stream>>>(v.occ, v.sdist_tmp, sb, 1, v.sdist);
  k_sdist_axis<<<grid, 256, 0, stream>>>(v.occ, v.sdist, sb, 2, v.sdist_tmp);
  cudaMemcpyAsync(v.sdist, v.sdist_tmp, static_cast<size_t>(cells), cudaMemcpyDeviceToDevice, stream);
  chk("super_dist");
}

void launch_reset_hashed(const Launch& L, const HashDev& v, int Dp) {
  launch_pdl(k_reset_hashed, dim3(sm_count() * 8), dim3(256), 0, L.stream, static_cast<const int*>(v.n_blocks),
             v.rw, v.fim, Dp, v.heads, (1u << v.bits) - 1u, v.next, static_cast<const int*>(v.coords), v.grid, v.occ,
             v.gbits);
  ++*L.launches;
  chk("reset_hashed");
}

void launch_init_volume(const Launch& L, double2* rw, double* fim, long long n, int Dp) {
  launch_pdl(k_init_volume, dim3(sm_count() * 8), dim3(256), 0, L.stream, rw, fim, n, Dp);
  ++*L.launches;
  chk("init_volume");
}

void launch_integrate_dense(const Launch& L, const DenseDev& v, int G, int Dp, const double* depth, int w, int h,
                            const double* pose, const double* intr, int* upd, const double* dch) {
  const DenseView view = dense_view(v, Dp);
  const bool jac = v.order != 2 && !dch && Dp % 2 == 0 && Dp <= 24;
  const size_t smem = integrate_smem(Dp, jac);
  const long long n = static_cast<long long>(v.nx) * v.ny * v.nz;
  const int grid = static_cast<int>(std::min<long long>((n + 255) / 256, sm_count() * 16LL));
  const double* nd = nullptr;
  if (v.order == 2)
    launch_pdl(k_integrate_dense<B<1>>, dim3(grid), dim3(256), smem, L.stream, view, depth, w, h, pose, intr, Dp, upd,
               nd);
  else if (dch && G > 0) {
    CSF_DISPATCH_G(G, (launch_pdl(k_integrate_dense<Scal<kG>, 0, true>, dim3(grid), dim3(256), smem, L.stream, view,
                                  depth, w, h, pose, intr, Dp, upd, dch)));
  } else if (kAdjointFusion && G > 0 && fixed_channels(Dp)) {
    CSF_DISPATCH_NDP(Dp, (launch_pdl(k_integrate_dense<csfd::L<1>, kN>, dim3(grid), dim3(256), smem, L.stream, view,
                                     depth, w, h, pose, intr, Dp, upd, nd)));
  } else
    CSF_DISPATCH_G(G, (launch_pdl(k_integrate_dense<Scal<kG>>, dim3(grid), dim3(256), smem, L.stream, view, depth, w,
                                  h, pose, intr, Dp, upd, nd)));
  ++*L.launches;
  chk("integrate_dense");
}

void launch_integrate_hashed(const Launch& L, const HashDev& v, int G, int Dp, const AllocScratch& a,
                             const double* depth, int w, int h, const double* pose, const double* intr, int* upd,
                             const double* dch) {
  const HashView view = hash_view(v, Dp);
  const bool jac = v.order != 2 && !dch && Dp % 2 == 0 && Dp <= 24;
  const size_t smem = integrate_smem(Dp, jac);
  const int grid = sm_count() * 8;
  const double* nd = nullptr;
  if (v.order == 2)
    launch_pdl(k_integrate_hashed<B<1>>, dim3(grid), dim3(256), smem, L.stream, view, v.coords, a.visible,
               a.counters, depth, w, h, pose, intr, Dp, upd, nd);
  else if (dch && G > 0) {
    CSF_DISPATCH_G(G, (launch_pdl(k_integrate_hashed<Scal<kG>, 0, true>, dim3(grid), dim3(256), smem, L.stream,
                                  view, v.coords, a.visible, a.counters, depth, w, h, pose, intr, Dp, upd, dch)));
  } else if (kAdjointFusion && G > 0 && fixed_channels(Dp)) {
    CSF_DISPATCH_NDP(Dp, (launch_pdl(k_integrate_hashed<csfd::L<1>, kN>, dim3(grid), dim3(256), smem, L.stream, view,
                                     v.coords, a.visible, a.counters, depth, w, h, pose, intr, Dp, upd, nd)));
  } else
    CSF_DISPATCH_G(G, (launch_pdl(k_integrate_hashed<Scal<kG>>, dim3(grid), dim3(256), smem, L.stream, view,
                                  v.coords, a.visible, a.counters, depth, w, h, pose, intr, Dp, upd, nd)));
  ++*L.launches;
  chk("integrate_hashed");
}

// Derived lookup indices of a hashed volume whose table was loaded from a
// checkpoint: the block-id window grid and the super-block occupancy bits.
__global__ void k_rebuild_index(const int* __restrict__ coords, int n_blocks, int* grid, unsigned* occ, int gbits) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n_blocks) return;
  const int half = 1 << (gbits - 1);
  const unsigned ux = static_cast<unsigned>(coords[3 * b] + half), uy = static_cast<unsigned>(coords[3 * b + 1] + half),
                 uz = static_cast<unsigned>(coords[3 * b + 2] + half);
  const unsigned side = 1u << gbits;
  if (ux < side && uy < side && uz < side) {
    grid[(static_cast<size_t>(uz) << gbits | uy) << gbits | ux] = b;
    occ_mark(occ, gbits, ux, uy, uz);
  }
}

void launch_rebuild_index(cudaStream_t stream, const int* coords, int n_blocks, int* grid, unsigned* occ, int gbits) {
  if (n_blocks > 0) k_rebuild_index<<<(n_blocks + 255) / 256, 256, 0, stream>>>(coords, n_blocks, grid, occ, gbits);
}

void march_stats_enable(unsigned long long* buf) { cudaMemcpyToSymbol(g_march_stats, &buf, sizeof(buf)); }

int band_samples(double mu, double vs) {
  const int k = static_cast<int>(std::ceil((2.0 * mu) / vs)) + 1;
  return k < 2 ? 2 : k;
}

void launch_allocate(const Launch& L, const HashDev& v, int Dp, AllocScratch& a, const double* depth, int w, int h,
                     const double* pose, const double* intr) {
  const HashView view = hash_view(v, Dp);
  const int K = band_samples(v.mu, v.vs);
  const int n = w * h * K;
  const int C = 1 + Dp;
  cudaMemsetAsync(a.set_keys, 0xFF, sizeof(unsigned long long) << a.set_bits, L.stream);
  cudaMemsetAsync(a.set_first, 0x7F, sizeof(int) << a.set_bits, L.stream);
  const dim3 b2(32, 8), g2((w + 31) / 32, (h + 7) / 8);
  launch_pdl(k_band, dim3(g2), dim3(b2), 0, L.stream, depth, w, h, pose, intr, C, v.mu, v.vs, v.ox, v.oy, v.oz, K, a.cand);
  const int tb = 256, gb = std::min((n + tb - 1) / tb, 8 * csfi::sm_count());  // grid-stride kernels
  launch_pdl(k_touch, dim3(gb), dim3(tb), 0, L.stream, a.cand, n, a.set_keys, a.set_first, a.set_slot, a.set_bits, L.err, a.counters);
  launch_pdl(k_flags, dim3(gb), dim3(tb), 0, L.stream, view, a.cand, n, a.set_first, a.set_slot, a.first_flag, a.new_flag, a.cand_block);
  size_t bytes = a.cub_tmp_bytes;
  cub::DeviceScan::ExclusiveSum(a.cub_tmp, bytes, a.first_flag, a.first_rank, n, L.stream);
  bytes = a.cub_tmp_bytes;
  cub::DeviceScan::ExclusiveSum(a.cub_tmp, bytes, a.new_flag, a.new_rank, n, L.stream);
  launch_pdl(k_insert, dim3(gb), dim3(tb), 0, L.stream, view, v.heads, v.keys, v.next, v.coords, v.n_blocks, v.max_blocks, a.cand, n,
                                    a.first_flag, a.new_flag, a.first_rank, a.new_rank, a.cand_block, a.visible, L.err);
  launch_pdl(k_alloc_finalize, dim3(1), dim3(1), 0, L.stream, v.n_blocks, v.max_blocks, a.first_flag, a.new_flag, a.first_rank,
                                          a.new_rank, n, a.counters);
  launch_super_dist(L.stream, v);
  *L.launches += 10;
  chk("allocate");
}

size_t alloc_scan_bytes(int n) {
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, static_cast<int*>(nullptr), static_cast<int*>(nullptr), n);
  return bytes;
}

template <typename V>
static void raycast_impl(const Launch& L, const V& view, Box box, int order, int Dp, const double* pose,
                         const double* intr, int w, int h, double near_clip, double far_clip, double step,
                         double2* hits, double* vre, double* nre, double* vim, double* nim,
                         const double* atab = nullptr, int n_tab = 0, unsigned* seg_first = nullptr) {
  const int P = w * h;
  if (L.phase != 2) {
    // Segments per ray (hashed volumes): enough threads to fill the GPU at
    // the small levels, where the longest ray sets the kernel time.
    int S = 1;
    if constexpr (V::kHashed) {
      // (measured: 640k / 1.3M / 160k targets and S = 2 at level 0 are slower)
      constexpr int kSegMax = 16;
      constexpr long long kTargetThreads = 320000;
      while (S < kSegMax && static_cast<long long>(P) * S * 2 <= kTargetThreads) S *= 2;
      if (!atab || !seg_first) S = 1;
    }
    if (S > 1) {
      if constexpr (V::kHashed) {
        cudaMemsetAsync(seg_first, 0xFF, sizeof(unsigned) * P, L.stream);
        const long long items = tiled_count(w, h) * S;
        launch_pdl(k_raycast_march_seg, dim3(static_cast<unsigned>((items + 127) / 128)), dim3(128), 0, L.stream, view,
                   pose, intr, w, h, Dp, S, atab, n_tab, step, seg_first);
        launch_pdl(k_raycast_march_fin, dim3((P + 127) / 128), dim3(128), 0, L.stream, view, pose, intr, w, h, Dp, atab,
                   static_cast<const unsigned*>(seg_first), hits, vre, nre);
        *L.launches += 1;
      }
    } else {
      const unsigned march_grid = static_cast<unsigned>((tiled_count(w, h) + 127) / 128);
      launch_pdl(k_raycast_march<V>, dim3(march_grid), dim3(128), 0, L.stream, view, pose, intr, w, h, Dp,
                 near_clip, far_clip, step, box, hits, vre, nre, atab, n_tab);
    }
    if (Dp > 0 && vim && order == 2) {  // the first-order lift writes every pixel
      cudaMemsetAsync(vim, 0, sizeof(double) * 3 * Dp * static_cast<size_t>(P), L.stream);
      cudaMemsetAsync(nim, 0, sizeof(double) * 3 * Dp * static_cast<size_t>(P), L.stream);
    }
    *L.launches += 1;
  }
  if (L.phase == 1) return;
  const size_t smem = sizeof(double) * 16 * (1 + Dp);
  if (order == 2) {
    // second order: the cooperative real pass, then one thread per (hit
    // pixel, pair) in Bicomplex arithmetic over the recorded corners
    launch_pdl(k_raycast_lift2_coop<V>, dim3(lift_grid(kLiftPix, w, h)), dim3(8 * kLiftPix),
               smem + sizeof(LiftRec2) * kLiftPix, L.stream, view, pose, intr, w, h, Dp, hits, vre, nre, vim, nim);
    *L.launches += 1;
    return;
  }
  // first order: the cooperative lift (8 lanes per pixel for the real chain,
  // then one thread per (pixel, channel))
  const bool pair = Dp % 2 == 0;
  const int npix = lift_pixels(pair ? Dp / 2 : Dp);
  const size_t smem_c = smem + sizeof(LiftRec) * npix;
  if (pair)
    launch_pdl(k_raycast_lift_coop<V, 2>, dim3(lift_grid(npix, w, h)), dim3(8 * kLiftPix), smem_c, L.stream, view,
               pose, intr, w, h, Dp, hits, vre, nre, vim, nim, npix);
  else
    launch_pdl(k_raycast_lift_coop<V, 1>, dim3(lift_grid(npix, w, h)), dim3(8 * kLiftPix), smem_c, L.stream, view,
               pose, intr, w, h, Dp, hits, vre, nre, vim, nim, npix);
  *L.launches += 1;
}

void launch_raycast_dense(const Launch& L, const DenseDev& v, int G, int Dp, const double* pose, const double* intr,
                          int w, int h, double near_clip, double far_clip, double step, double2* hits, double* vre,
                          double* nre, double* vim, double* nim) {
  const DenseView view = dense_view(v, Dp);
  Box box;
  box.use = true;
  box.lo[0] = v.ox; box.lo[1] = v.oy; box.lo[2] = v.oz;
  box.hi[0] = v.ox + v.vs * (static_cast<double>(v.nx) - 1.0);
  box.hi[1] = v.oy + v.vs * (static_cast<double>(v.ny) - 1.0);
  box.hi[2] = v.oz + v.vs * (static_cast<double>(v.nz) - 1.0);
  raycast_impl(L, view, box, v.order, Dp, pose, intr, w, h, near_clip, far_clip, step, hits, vre, nre, vim, nim);
  chk("raycast_dense");
}

void launch_raycast_hashed(const Launch& L, const HashDev& v, int G, int Dp, const double* pose, const double* intr,
                           int w, int h, double near_clip, double far_clip, double step, double2* hits, double* vre,
                           double* nre, double* vim, double* nim) {
  const HashView view = hash_view(v, Dp);
  Box box;
  box.use = false;
  raycast_impl(L, view, box, v.order, Dp, pose, intr, w, h, near_clip, far_clip, step, hits, vre, nre, vim, nim,
               v.alpha_tab, v.alpha_n, v.seg_first);
  chk("raycast_hashed");
}

}  // namespace csfi
