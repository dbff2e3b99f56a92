// Frame preprocessing kernels for sm_100a: bilateral filter, depth-aware
// pyramid downsampling, and vertex/normal measurement.
//
//   bilateral_filter  — proj/src/frames.cpp:7-38
//   downsample_depth  — proj/src/frames.cpp:40-66
//   measure_surface   — proj/include/csf/frames.hpp:86-114
//
// These run on the real channel only and are shared by every CSFD direction
// of a run.  The bilateral weights use the deterministic exp of
// include/csf_detmath.h (the oracle's function).
#include <cstdio>

#include "csf_internal.h"
#include "lifted.cuh"

namespace csfd {

constexpr int kMaxRadius = 7;

constexpr int kBX = 32, kBY = 8;

// One 32x8 output tile per CTA; the (32+2r)x(8+2r) input window is staged in
// shared memory once and reused by all 49 taps of every pixel.  The spatial
// weights exp(-(dx^2+dy^2)/(2 sigma_s^2)) are computed per CTA into shared
// memory (deterministic exp, the oracle's values): the kernel reads nothing
// from the host at launch time, so a run captured in a CUDA graph replays
// exactly (a constant-memory upload from a host stack array did not).
__global__ void __launch_bounds__(kBX* kBY) k_bilateral(const float* __restrict__ in_f32,
                                                         const double* __restrict__ in_f64,
                                                         double* __restrict__ raw_out, double* __restrict__ out,
                                                         int w, int h, int radius, double inv2ss, double inv2sr) {
  pdl_wait();
  pdl_trigger();
  __shared__ double c_spatial[(2 * kMaxRadius + 1) * (2 * kMaxRadius + 1)];
  extern __shared__ double tile[];
  const int tw = kBX + 2 * radius, th = kBY + 2 * radius;
  {
    const int sd = 2 * radius + 1;
    const int i = threadIdx.y * kBX + threadIdx.x;
    if (i < sd * sd) {
      const int dy = i / sd - radius, dx = i % sd - radius;
      c_spatial[i] = csf_det::exp(static_cast<double>(-(dx * dx + dy * dy)) * inv2ss);
    }
  }
  const int x0 = blockIdx.x * kBX - radius, y0 = blockIdx.y * kBY - radius;
  for (int i = threadIdx.y * kBX + threadIdx.x; i < tw * th; i += kBX * kBY) {
    const int tx = x0 + i % tw, ty = y0 + i / tw;
    double v = 0.0;
    if (tx >= 0 && tx < w && ty >= 0 && ty < h) {
      const long long idx = static_cast<long long>(ty) * w + tx;
      v = in_f32 ? static_cast<double>(in_f32[idx]) : in_f64[idx];
    }
    tile[i] = v;
  }
  __syncthreads();
  const int x = blockIdx.x * kBX + threadIdx.x, y = blockIdx.y * kBY + threadIdx.y;
  if (x >= w || y >= h) return;
  const double center = tile[(threadIdx.y + radius) * tw + threadIdx.x + radius];
  const long long o = static_cast<long long>(y) * w + x;
  if (raw_out) raw_out[o] = center;
  if (!(center > 0.0)) {
    out[o] = 0.0;
    return;
  }
  const int side = 2 * radius + 1;
  double wsum = 0.0, vsum = 0.0;
  for (int dy = -radius; dy <= radius; ++dy) {
    const int qy = y + dy;
    if (qy < 0 || qy >= h) continue;
    for (int dx = -radius; dx <= radius; ++dx) {
      const int qx = x + dx;
      if (qx < 0 || qx >= w) continue;
      const double q = tile[(threadIdx.y + radius + dy) * tw + threadIdx.x + radius + dx];
      if (!(q > 0.0)) continue;
      const double dd = q - center;
      const double wt = c_spatial[(dy + radius) * side + dx + radius] * csf_det::exp(-dd * dd * inv2sr);
      wsum += wt;
      vsum += wt * q;
    }
  }
  out[o] = vsum / wsum;
}

// frames.cpp:40-66 — output pixel (x, y) centred on input (2x, 2y).
__global__ void k_downsample(const double* __restrict__ in, double* __restrict__ out, int w, int h, int wo, int ho,
                             double reject) {
  pdl_wait();
  pdl_trigger();
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= wo || y >= ho) return;
  const double tap[5] = {1.0 / 16, 4.0 / 16, 6.0 / 16, 4.0 / 16, 1.0 / 16};
  const int cx = 2 * x, cy = 2 * y;
  const double center = in[static_cast<long long>(cy) * w + cx];
  const long long o = static_cast<long long>(y) * wo + x;
  if (!(center > 0.0)) {
    out[o] = 0.0;
    return;
  }
  double wsum = 0.0, vsum = 0.0;
#pragma unroll
  for (int dy = -2; dy <= 2; ++dy) {
#pragma unroll
    for (int dx = -2; dx <= 2; ++dx) {
      const int qx = cx + dx, qy = cy + dy;
      if (qx < 0 || qx >= w || qy < 0 || qy >= h) continue;
      const double q = in[static_cast<long long>(qy) * w + qx];
      if (!(q > 0.0) || fabs(q - center) > reject) continue;
      const double wt = tap[dx + 2] * tap[dy + 2];
      wsum += wt;
      vsum += wt * q;
    }
  }
  out[o] = vsum / wsum;
}

// frames.hpp:86-114 — lifted depth [P][1+D] and lifted intrinsics [4][1+D];
// one channel per pass (S = L<1>), channel c of the outputs written by pass c.
template <typename S>
__device__ V3<S> backproject_px(const S& d, int x, int y, const S& fx, const S& fy, const S& cx, const S& cy) {
  return mk3<S>(d * (static_cast<double>(x) - cx) / fx, d * (static_cast<double>(y) - cy) / fy, d);
}

__global__ void k_measure(const double* __restrict__ depth, int w, int h, const double* __restrict__ intr, int D,
                          double* __restrict__ vert, double* __restrict__ norm) {
  pdl_wait();
  pdl_trigger();
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= w || y >= h) return;
  using S = L<1>;
  const int C = 1 + D;
  const long long p = static_cast<long long>(y) * w + x;
  const int passes = D > 0 ? D : 1;
  for (int c = 0; c < passes; ++c) {
    auto ld = [&](const double* b) {
      S s;
      s.re = b[0];
      s.im[0] = D > 0 ? b[1 + c] : 0.0;
      return s;
    };
    const S fx = ld(intr), fy = ld(intr + C), cx = ld(intr + 2 * C), cy = ld(intr + 3 * C);
    auto vtx = [&](int xx, int yy, bool* valid) {
      const S d = ld(depth + (static_cast<long long>(yy) * w + xx) * C);
      *valid = d.re > 0.0;
      if (!*valid) return mk3<S>(lit<S>(0.0), lit<S>(0.0), lit<S>(0.0));
      return backproject_px<S>(d, xx, yy, fx, fy, cx, cy);
    };
    bool v0, vx = false, vy = false;
    const V3<S> v = vtx(x, y, &v0);
    V3<S> n = mk3<S>(lit<S>(0.0), lit<S>(0.0), lit<S>(0.0));
    if (v0 && x + 1 < w && y + 1 < h) {
      const V3<S> a = vtx(x + 1, y, &vx);
      const V3<S> b = vtx(x, y + 1, &vy);
      if (vx && vy) {
        V3<S> nn = cross3(sub3(a, v), sub3(b, v));
        const S len2 = dot3(nn, nn);
        if (len2.re > 0.0) {
          const S l = sqrt_s(len2);
          nn = mk3<S>(nn.v[0] / l, nn.v[1] / l, nn.v[2] / l);
          if (dot3(nn, v).re > 0.0) nn = mk3<S>(-nn.v[0], -nn.v[1], -nn.v[2]);
          n = nn;
        }
      }
    }
    for (int k = 0; k < 3; ++k) {
      double* vb = vert + (p * 3 + k) * C;
      double* nb = norm + (p * 3 + k) * C;
      if (c == 0) {
        vb[0] = v.v[k].re;
        nb[0] = n.v[k].re;
      }
      if (D > 0) {
        vb[1 + c] = v.v[k].im[0];
        nb[1 + c] = n.v[k].im[0];
      }
    }
  }
}

}  // namespace csfd

namespace csfi {

static void check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) note_launch_error(what, e);
}

void launch_bilateral(const Launch& L, const float* in_f32, const double* in_f64, double* raw_out, double* out, int w,
                      int h, double sigma_s, double sigma_r, int radius) {
  if (radius > csfd::kMaxRadius) radius = csfd::kMaxRadius;
  const double inv2ss = 1.0 / (2.0 * sigma_s * sigma_s);
  const double inv2sr = 1.0 / (2.0 * sigma_r * sigma_r);
  const dim3 block(csfd::kBX, csfd::kBY);
  const dim3 grid((w + csfd::kBX - 1) / csfd::kBX, (h + csfd::kBY - 1) / csfd::kBY);
  const size_t smem = sizeof(double) * (csfd::kBX + 2 * radius) * (csfd::kBY + 2 * radius);
  csfd::launch_pdl(csfd::k_bilateral, dim3(grid), dim3(block), smem, L.stream, in_f32, in_f64, raw_out, out, w, h,
                   radius, inv2ss, inv2sr);
  ++*L.launches;
  check_launch("bilateral");
}

void launch_downsample(const Launch& L, const double* in, double* out, int w, int h, double sigma_r) {
  const int wo = w / 2, ho = h / 2;
  const dim3 block(32, 8), grid((wo + 31) / 32, (ho + 7) / 8);
  csfd::launch_pdl(csfd::k_downsample, dim3(grid), dim3(block), 0, L.stream, in, out, w, h, wo, ho, 3.0 * sigma_r);
  ++*L.launches;
  check_launch("downsample");
}

void launch_measure(const Launch& L, const double* depth, int w, int h, const double* intr, int D, double* vert,
                    double* norm) {
  const dim3 block(32, 8), grid((w + 31) / 32, (h + 7) / 8);
  csfd::launch_pdl(csfd::k_measure, dim3(grid), dim3(block), 0, L.stream, depth, w, h, intr, D, vert, norm);
  ++*L.launches;
  check_launch("measure");
}

}  // namespace csfi
