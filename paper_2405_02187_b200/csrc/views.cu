// BASELINE config 5 on sm_100a: active-scanning view scoring.
//
// Builder-defined objective (no reference: the spec's task-gradient module
// with its "smooth visibility score" is unimplemented): the
// soft count of weakly observed surface a candidate view would see,
//   S(T) = pairwise_sum over the view's pixels (row-major) of
//          sigma(beta * (w0 - W~(p)))   for raycast hits p, 0 elsewhere,
// where W~ is the trilinear interpolation of the integral fusion weights at
// the hit point (unallocated corners count 0) and sigma the logistic
// function.  Each view is raycast with its pose lifted on the 6 twist
// channels (exp(xi) T, se3.hpp:77-119), so one evaluation gives S and
// dS/dxi.  Real parts follow the oracle's operation order
// (oracle/orc_tsdf.hpp view_coverage_score); hits are the raycast's valid
// normals (frames.hpp:73-81).
#include <cstdio>

#include "csf_internal.h"
#include "geometry.cuh"

namespace csfd {

constexpr int kViewD = 6;

__global__ void k_view_seed(const double* __restrict__ view, const double* __restrict__ k4, double hstep,
                            double* pose, double* intr) {
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x != 0) return;
  using S = L<kViewD>;
  constexpr int C = 1 + kViewD;
  S xi[6];
  for (int i = 0; i < 6; ++i) {
    xi[i] = lit<S>(0.0);
    xi[i].im[i] = hstep;
  }
  Pose<S> base;
  for (int e = 0; e < 9; ++e) base.R.m[e] = lit<S>(view[e]);
  for (int e = 0; e < 3; ++e) base.t.v[e] = lit<S>(view[9 + e]);
  const Pose<S> p = compose(exp_map<S>(xi), base);
  for (int e = 0; e < 9; ++e) store_ch<S>(pose + e * C, p.R.m[e], 0, kViewD, true);
  for (int e = 0; e < 3; ++e) store_ch<S>(pose + (9 + e) * C, p.t.v[e], 0, kViewD, true);
  for (int i = 0; i < 4; ++i) {
    intr[i * C] = k4[i];
    for (int d = 0; d < kViewD; ++d) intr[i * C + 1 + d] = 0.0;
  }
}

// Trilinear interpolation of the weights at a lifted point (the
// sample_tsdf cell and dk, dj, di order, tsdf.hpp:148-177; W has no channels).
template <typename S>
CSF_DEV S interpolated_weight(const HashView& vol, const V3<S>& p) {
  const S gx = (p.v[0] - vol.ox) / vol.vs;
  const S gy = (p.v[1] - vol.oy) / vol.vs;
  const S gz = (p.v[2] - vol.oz) / vol.vs;
  const int i0 = ifloor(re(gx)), j0 = ifloor(re(gy)), k0 = ifloor(re(gz));
  const S fx = gx - static_cast<double>(i0);
  const S fy = gy - static_cast<double>(j0);
  const S fz = gz - static_cast<double>(k0);
  double wc[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const long long v = vol.voxel(i0 + (c & 1), j0 + ((c >> 1) & 1), k0 + (c >> 2));
    wc[c] = v >= 0 ? vol.vox.rw[v].y : 0.0;
  }
  S accum = lit<S>(0.0);
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const S wx = (c & 1) ? fx : 1.0 - fx;
    const S wy = ((c >> 1) & 1) ? fy : 1.0 - fy;
    const S wz = (c >> 2) ? fz : 1.0 - fz;
    accum = accum + ((wx * wy) * wz) * wc[c];
  }
  return accum;
}

template <typename S>
CSF_DEV S exp_s(const S& z) {
  const double f = csf_det::exp(z.re);
  return lift(z, f, f);  // csfd.hpp:174-176
}

__global__ void __launch_bounds__(128) k_view_terms(HashView vol, const double* __restrict__ vre,
                                                    const double* __restrict__ nre, const double* __restrict__ vim,
                                                    int P, double w0, double beta, double* __restrict__ terms) {
  pdl_wait();
  pdl_trigger();
  using S = L<kViewD>;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P) return;
  const double n0 = nre[3LL * i], n1 = nre[3LL * i + 1], n2 = nre[3LL * i + 2];
  S term = lit<S>(0.0);
  if (n0 * n0 + (n1 * n1 + n2 * n2) > 0.5) {
    V3<S> p;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      p.v[c].re = vre[3LL * i + c];
#pragma unroll
      for (int d = 0; d < kViewD; ++d) p.v[c].im[d] = vim[(3LL * i + c) * kViewD + d];
    }
    const S wt = interpolated_weight<S>(vol, p);
    const S z = beta * (w0 - wt);
    term = 1.0 / (1.0 + exp_s(-z));
  }
  terms[i] = term.re;
#pragma unroll
  for (int d = 0; d < kViewD; ++d) terms[static_cast<long long>(1 + d) * P + i] = term.im[d];
}

}  // namespace csfd

namespace csfi {

using namespace csfd;

void launch_view_seed(const Launch& L, const double* view12, const double* k4, double h, double* pose_out,
                      double* intr_out) {
  launch_pdl(k_view_seed, dim3(1), dim3(32), 0, L.stream, view12, k4, h, pose_out, intr_out);
  ++*L.launches;
}

void launch_view_terms(const Launch& L, const HashDev& v, const double* vre, const double* nre, const double* vim,
                       int w, int h, double w0, double beta, double* terms) {
  HashView view;
  view.vox = {v.rw, v.fim, kViewD};
  view.heads = v.heads;
  view.keys = v.keys;
  view.next = v.next;
  view.grid = v.grid;
  view.occ = v.occ;
  view.sdist = v.sdist;
  view.gbits = v.gbits;
  view.mask = (1u << v.bits) - 1u;
  view.vs = v.vs; view.ox = v.ox; view.oy = v.oy; view.oz = v.oz; view.mu = v.mu; view.cap = v.cap;
  const int P = w * h;
  launch_pdl(k_view_terms, dim3((P + 127) / 128), dim3(128), 0, L.stream, view, vre, nre, vim, P, w0, beta, terms);
  ++*L.launches;
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) note_launch_error("view_terms", e);
}

}  // namespace csfi
