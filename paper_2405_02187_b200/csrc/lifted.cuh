// Device CSFD scalar and fixed-size geometry for sm_100a.
//
// L<G> carries the real channel plus G perturbation channels of one channel
// group.  A kernel evaluates the D packed directions of a run as ceil(D/G)
// passes of L<G> (the real channel is recomputed bit-identically in every
// pass), which bounds register pressure independently of D.  Channel
// arithmetic follows the truncated Complex rules of the reference
// (proj/include/csf/csfd.hpp:44-58, 148-155, 267-292) operation for
// operation; the whole library is compiled with -fmad=false so every real
// channel is bit-identical to the CPU oracle (oracle/orc_core.hpp).
//
// S = double instantiates the same templates as the plain real path (the
// reference's double pipeline).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/csf_detmath.h"

#define CSF_DEV __device__ __forceinline__

namespace csfd {

// ----------------------------------------------------------------------------
// Programmatic dependent launch (sm_90+).  Every kernel of the library is
// launched with programmatic stream serialization (launch_pdl) and begins
// with pdl_wait() — it waits for the previous kernel on the stream to
// complete and its memory to be visible before touching anything — then
// pdl_trigger() lets the next kernel be scheduled as soon as every CTA of
// this one is resident.  The chain of dependent launches (~40 per frame)
// then no longer pays the full launch gap between kernels.
// ----------------------------------------------------------------------------
CSF_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
CSF_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }

}  // namespace csfd
namespace csfi {
// Opt `fn` into `bytes` of dynamic shared memory on the current device
// (cudaFuncSetAttribute is per device); thread-safe, cached per (device, fn).
void ensure_dyn_smem(const void* fn, size_t bytes);
// SM count of the current device (cached per device).
int sm_count();
}  // namespace csfi
namespace csfd {

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                       Args... args) {
  if (smem > 48 * 1024) csfi::ensure_dyn_smem(reinterpret_cast<const void*>(kern), smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// ----------------------------------------------------------------------------
// error flag: first error code wins (0 = ok)
// ----------------------------------------------------------------------------
enum DevErr : int { kErrNone = 0, kErrDomain = 2, kErrNoMem = 5 };

CSF_DEV void raise(int* err, int code) {
  if (err) atomicCAS(err, 0, code);
}

// ----------------------------------------------------------------------------
// L<G>
// ----------------------------------------------------------------------------
template <int G>
struct L {
  double re;
  double im[G > 0 ? G : 1];
};
template <int G> struct ScalarOf { using type = L<G>; };
template <> struct ScalarOf<0> { using type = double; };
template <int G> using Scal = typename ScalarOf<G>::type;

// ----------------------------------------------------------------------------
// B<NP>: NP second-order direction pairs sharing one real channel.  Pair p
// occupies three channel slots (im1, im2, im12) — exactly one reference
// Bicomplex per pair (csfd.hpp:83-140), so slot 3p+2 of a packed run equals
// the im12 of a standalone Bicomplex pass seeded on that pair.  Storage
// follows the first-order layout (element-major, slot-minor), so the voxel
// store, poses and maps address second-order runs unchanged.
// ----------------------------------------------------------------------------
template <int NP>
struct B {
  double re;
  double im[3 * NP];
};

// G = channel slots per value; kOrder = CSFD order (0 = plain real path).
template <typename S> struct Traits;
template <> struct Traits<double> {
  static constexpr int G = 0;
  static constexpr int kOrder = 0;
};
template <int G_> struct Traits<L<G_>> {
  static constexpr int G = G_;
  static constexpr int kOrder = 1;
};
template <int NP> struct Traits<B<NP>> {
  static constexpr int G = 3 * NP;
  static constexpr int kOrder = 2;
};

template <typename S> CSF_HD S lit(double x);
template <> CSF_HD double lit<double>(double x) { return x; }
template <typename S> CSF_HD S lit(double x) {
  S o;
  o.re = x;
#pragma unroll
  for (int g = 0; g < Traits<S>::G; ++g) o.im[g] = 0.0;
  return o;
}

CSF_HD double re(double x) { return x; }
template <int G> CSF_DEV double re(const L<G>& x) { return x.re; }

// -- lifted (x) lifted -------------------------------------------------------
template <int G> CSF_DEV L<G> operator+(const L<G>& a, const L<G>& b) {
  L<G> o;
  o.re = a.re + b.re;
#pragma unroll
  for (int g = 0; g < G; ++g) o.im[g] = a.im[g] + b.im[g];
  return o;
}
template <int G> CSF_DEV L<G> operator-(const L<G>& a, const L<G>& b) {
  L<G> o;
  o.re = a.re - b.re;
#pragma unroll
  for (int g = 0; g < G; ++g) o.im[g] = a.im[g] - b.im[g];
  return o;
}
template <int G> CSF_DEV L<G> operator-(const L<G>& a) {
  L<G> o;
  o.re = -a.re;
#pragma unroll
  for (int g = 0; g < G; ++g) o.im[g] = -a.im[g];
  return o;
}
template <int G> CSF_DEV L<G> operator*(const L<G>& a, const L<G>& b) {
  L<G> o;
  o.re = a.re * b.re;
#pragma unroll
  for (int g = 0; g < G; ++g) o.im[g] = a.re * b.im[g] + a.im[g] * b.re;
  return o;
}
// Channel division.  The real part is always the IEEE quotient (it drives
// control flow and must match the oracle bit for bit).  By default the
// perturbation channels share one reciprocal of the divisor term
// (im = num * (1/den)): within ~1 ulp of the reference's per-channel
// quotient (csfd.hpp:57), i.e. far inside the 1e-9 derivative tolerance, at
// one division per operation instead of one per channel.  Define
// CSF_EXACT_CHANNELS to evaluate the reference's per-channel quotient.
#ifdef CSF_EXACT_CHANNELS
#define CSF_CH_DIV(num, den, inv) ((num) / (den))
#else
#define CSF_CH_DIV(num, den, inv) ((num) * (inv))
#endif

// Division without the zero-real check (callers that can meet b.re == 0 use
// div_checked).
template <int G> CSF_DEV L<G> operator/(const L<G>& a, const L<G>& b) {
  L<G> o;
  o.re = a.re / b.re;
  const double den = b.re * b.re;
  const double inv = 1.0 / den;
  (void)inv;
#pragma unroll
  for (int g = 0; g < G; ++g) o.im[g] = CSF_CH_DIV(a.im[g] * b.re - a.re * b.im[g], den, inv);
  return o;
}

// -- lifted (x) real constant, i.e. lifted (x) S(c) with zero channels --------
// (a.re*0 terms contribute only signed zeros and are dropped)
template <int G> CSF_DEV L<G> operator+(const L<G>& a, double c) {
  L<G> o = a;
  o.re = a.re + c;
  return o;
}
template <int G> CSF_DEV L<G> operator+(double c, const L<G>& a) {
  L<G> o = a;
  o.re = c + a.re;
  return o;
}
template <int G> CSF_DEV L<G> operator-(const L<G>& a, double c) {
  L<G> o = a;
  o.re = a.re - c;
  return o;
}
template <int G> CSF_DEV L<G> operator-(double c, const L<G>& a) {
  L<G> o;
  o.re = c - a.re;
#pragma unroll
  for (int g = 0; g < G; ++g) o.im[g] = -a.im[g];
  return o;
}
template <int G> CSF_DEV L<G> operator*(const L<G>& a, double c) {
  L<G> o;
  o.re = a.re * c;
#pragma unroll
  for (int g = 0; g < G; ++g) o.im[g] = a.im[g] * c;
  return o;
}
template <int G> CSF_DEV L<G> operator*(double c, const L<G>& a) {
  L<G> o;
  o.re = c * a.re;
#pragma unroll
  for (int g = 0; g < G; ++g) o.im[g] = c * a.im[g];
  return o;
}
// a / S(c): im = (a.im*c - a.re*0)/(c*c)  (csfd.hpp:57 with b.im = 0)
template <int G> CSF_DEV L<G> operator/(const L<G>& a, double c) {
  L<G> o;
  o.re = a.re / c;
  const double den = c * c;
  const double inv = 1.0 / den;
  (void)inv;
#pragma unroll
  for (int g = 0; g < G; ++g) o.im[g] = CSF_CH_DIV(a.im[g] * c, den, inv);
  return o;
}
// S(c) / b: im = (0*b.re - c*b.im)/(b.re*b.re)
template <int G> CSF_DEV L<G> operator/(double c, const L<G>& b) {
  L<G> o;
  o.re = c / b.re;
  const double den = b.re * b.re;
  const double inv = 1.0 / den;
  (void)inv;
#pragma unroll
  for (int g = 0; g < G; ++g) o.im[g] = CSF_CH_DIV(-(c * b.im[g]), den, inv);
  return o;
}

// -- B<NP> arithmetic: the reference Bicomplex rules (csfd.hpp:103-121) per
// pair, in the oracle's evaluation order (oracle/orc_core.hpp Bicomplex).
// Constants enter as Bicomplex(c) with zero slots; the exact-zero terms of the
// general formulas are dropped.
template <int NP> CSF_DEV double re(const B<NP>& x) { return x.re; }
template <int NP> CSF_DEV B<NP> operator+(const B<NP>& a, const B<NP>& b) {
  B<NP> o;
  o.re = a.re + b.re;
#pragma unroll
  for (int g = 0; g < 3 * NP; ++g) o.im[g] = a.im[g] + b.im[g];
  return o;
}
template <int NP> CSF_DEV B<NP> operator-(const B<NP>& a, const B<NP>& b) {
  B<NP> o;
  o.re = a.re - b.re;
#pragma unroll
  for (int g = 0; g < 3 * NP; ++g) o.im[g] = a.im[g] - b.im[g];
  return o;
}
template <int NP> CSF_DEV B<NP> operator-(const B<NP>& a) {
  B<NP> o;
  o.re = -a.re;
#pragma unroll
  for (int g = 0; g < 3 * NP; ++g) o.im[g] = -a.im[g];
  return o;
}
template <int NP> CSF_DEV B<NP> operator*(const B<NP>& a, const B<NP>& b) {
  B<NP> o;
  o.re = a.re * b.re;
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const double a1 = a.im[3 * p], a2 = a.im[3 * p + 1], a12 = a.im[3 * p + 2];
    const double b1 = b.im[3 * p], b2 = b.im[3 * p + 1], b12 = b.im[3 * p + 2];
    o.im[3 * p] = a.re * b1 + a1 * b.re;
    o.im[3 * p + 1] = a.re * b2 + a2 * b.re;
    o.im[3 * p + 2] = ((a.re * b12 + a12 * b.re) + a1 * b2) + a2 * b1;
  }
  return o;
}
template <int NP> CSF_DEV B<NP> operator/(const B<NP>& a, const B<NP>& b) {
  B<NP> o;
  o.re = a.re / b.re;
  const double den = b.re * b.re;
  // the channel slots' reciprocals: 1/b.re squared for 1/b.re^2 (one IEEE
  // division fewer per Bicomplex quotient; the real quotient above keeps its
  // division).  CSF_B_DEN_DIV keeps the separate division (the order-2 ICP
  // kernels, measured faster with it).
  const double inv = 1.0 / b.re;
  const double inv2 = inv * inv;
#ifdef CSF_B_DEN_DIV
  const double inv_den = 1.0 / den;
#else
  const double inv_den = inv2;
#endif
  (void)inv_den;
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const double a1 = a.im[3 * p], a2 = a.im[3 * p + 1], a12 = a.im[3 * p + 2];
    const double b1 = b.im[3 * p], b2 = b.im[3 * p + 1], b12 = b.im[3 * p + 2];
    o.im[3 * p] = CSF_CH_DIV(a1 * b.re - a.re * b1, den, inv_den);
    o.im[3 * p + 1] = CSF_CH_DIV(a2 * b.re - a.re * b2, den, inv_den);
    o.im[3 * p + 2] = ((a12 * inv - (a1 * b2 + a2 * b1) * inv2) - (a.re * b12) * inv2) +
                      ((((2.0 * a.re) * b1) * b2) * inv2) * inv;
  }
  return o;
}
template <int NP> CSF_DEV B<NP> operator+(const B<NP>& a, double c) {
  B<NP> o = a;
  o.re = a.re + c;
  return o;
}
template <int NP> CSF_DEV B<NP> operator+(double c, const B<NP>& a) {
  B<NP> o = a;
  o.re = c + a.re;
  return o;
}
template <int NP> CSF_DEV B<NP> operator-(const B<NP>& a, double c) {
  B<NP> o = a;
  o.re = a.re - c;
  return o;
}
template <int NP> CSF_DEV B<NP> operator-(double c, const B<NP>& a) {
  B<NP> o;
  o.re = c - a.re;
#pragma unroll
  for (int g = 0; g < 3 * NP; ++g) o.im[g] = -a.im[g];
  return o;
}
template <int NP> CSF_DEV B<NP> operator*(const B<NP>& a, double c) {
  B<NP> o;
  o.re = a.re * c;
#pragma unroll
  for (int g = 0; g < 3 * NP; ++g) o.im[g] = a.im[g] * c;
  return o;
}
template <int NP> CSF_DEV B<NP> operator*(double c, const B<NP>& a) {
  B<NP> o;
  o.re = c * a.re;
#pragma unroll
  for (int g = 0; g < 3 * NP; ++g) o.im[g] = c * a.im[g];
  return o;
}
// a / Bicomplex(c): im1,2 = (a.im*c)/(c*c), im12 = a.im12 * (1/c)
template <int NP> CSF_DEV B<NP> operator/(const B<NP>& a, double c) {
  B<NP> o;
  o.re = a.re / c;
  const double den = c * c;
  const double inv = 1.0 / c;
#ifdef CSF_B_DEN_DIV
  const double inv_den = 1.0 / den;
#else
  const double inv_den = inv * inv;
#endif
  (void)inv_den;
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    o.im[3 * p] = CSF_CH_DIV(a.im[3 * p] * c, den, inv_den);
    o.im[3 * p + 1] = CSF_CH_DIV(a.im[3 * p + 1] * c, den, inv_den);
    o.im[3 * p + 2] = a.im[3 * p + 2] * inv;
  }
  return o;
}
// Bicomplex(c) / b
template <int NP> CSF_DEV B<NP> operator/(double c, const B<NP>& b) {
  B<NP> o;
  o.re = c / b.re;
  const double den = b.re * b.re;
  const double inv = 1.0 / b.re;
  const double inv2 = inv * inv;
#ifdef CSF_B_DEN_DIV
  const double inv_den = 1.0 / den;
#else
  const double inv_den = inv2;
#endif
  (void)inv_den;
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const double b1 = b.im[3 * p], b2 = b.im[3 * p + 1], b12 = b.im[3 * p + 2];
    o.im[3 * p] = CSF_CH_DIV(-(c * b1), den, inv_den);
    o.im[3 * p + 1] = CSF_CH_DIV(-(c * b2), den, inv_den);
    o.im[3 * p + 2] = -((c * b12) * inv2) + ((((2.0 * c) * b1) * b2) * inv2) * inv;
  }
  return o;
}
// lift2 (csfd.hpp:212-263): (f, d1*im1, d1*im2, d1*im12 + d2*im1*im2)
template <int NP> CSF_DEV B<NP> lift2(const B<NP>& z, double f, double d1, double d2) {
  B<NP> o;
  o.re = f;
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    o.im[3 * p] = d1 * z.im[3 * p];
    o.im[3 * p + 1] = d1 * z.im[3 * p + 1];
    o.im[3 * p + 2] = d1 * z.im[3 * p + 2] + (d2 * z.im[3 * p]) * z.im[3 * p + 1];
  }
  return o;
}
template <int NP> CSF_DEV bool finite_s(const B<NP>& x) {
  bool ok = isfinite(x.re);
#pragma unroll
  for (int g = 0; g < 3 * NP; ++g) ok = ok && isfinite(x.im[g]);
  return ok;
}

template <typename S> CSF_DEV S div_checked(const S& a, const S& b, int* err) {
  if (re(b) == 0.0) raise(err, kErrDomain);
  return a / b;
}

// -- elementary lifts (csfd.hpp:174-205) --------------------------------------
CSF_DEV double dsqrt(double x) { return ::sqrt(x); }
template <int G> CSF_DEV L<G> lift(const L<G>& z, double f, double d1) {
  L<G> o;
  o.re = f;
#pragma unroll
  for (int g = 0; g < G; ++g) o.im[g] = d1 * z.im[g];
  return o;
}
CSF_HD double sqrt_s(double x) { return ::sqrt(x); }
template <int G> CSF_DEV L<G> sqrt_s(const L<G>& z) {
  const double f = ::sqrt(z.re);
  return lift(z, f, 0.5 / f);
}
CSF_HD double sin_s(double x) { return csf_det::sin(x); }
template <int G> CSF_DEV L<G> sin_s(const L<G>& z) { return lift(z, csf_det::sin(z.re), csf_det::cos(z.re)); }
CSF_HD double cos_s(double x) { return csf_det::cos(x); }
template <int G> CSF_DEV L<G> cos_s(const L<G>& z) { return lift(z, csf_det::cos(z.re), -csf_det::sin(z.re)); }
// Bicomplex lifts (csfd.hpp:230-245)
template <int NP> CSF_DEV B<NP> sqrt_s(const B<NP>& z) {
  const double f = ::sqrt(z.re);
  const double d1 = 0.5 / f;
  return lift2(z, f, d1, (-0.5 * d1) / z.re);
}
template <int NP> CSF_DEV B<NP> sin_s(const B<NP>& z) {
  const double s = csf_det::sin(z.re), c = csf_det::cos(z.re);
  return lift2(z, s, c, -s);
}
template <int NP> CSF_DEV B<NP> cos_s(const B<NP>& z) {
  const double s = csf_det::sin(z.re), c = csf_det::cos(z.re);
  return lift2(z, c, -s, -c);
}

// min/max/clamp keep the winning operand whole; ties keep the first
// (csfd.hpp:281-288)
template <typename S> CSF_DEV S smin(const S& a, const S& b) { return re(b) < re(a) ? b : a; }
template <typename S> CSF_DEV S smax(const S& a, const S& b) { return re(b) > re(a) ? b : a; }
template <typename S> CSF_DEV S clamp_s(const S& x, double lo, double hi) {
  return smax(smin(x, lit<S>(hi)), lit<S>(lo));
}
CSF_DEV int ifloor(double x) { return static_cast<int>(::floor(x)); }

CSF_HD bool finite_s(double x) { return isfinite(x); }
template <int G> CSF_DEV bool finite_s(const L<G>& x) {
  bool ok = isfinite(x.re);
#pragma unroll
  for (int g = 0; g < G; ++g) ok = ok && isfinite(x.im[g]);
  return ok;
}

// ----------------------------------------------------------------------------
// fixed-size vectors with Eigen's small-size order (a0 + (a1 + a2))
// ----------------------------------------------------------------------------
template <typename S> struct V3 {
  S v[3];
};
template <typename S> struct M3 {
  S m[9];  // row-major
};

template <typename S> CSF_HD V3<S> mk3(const S& a, const S& b, const S& c) {
  V3<S> o;
  o.v[0] = a; o.v[1] = b; o.v[2] = c;
  return o;
}
template <typename S> CSF_HD S sum3(const S& a0, const S& a1, const S& a2) { return a0 + (a1 + a2); }
template <typename S> CSF_HD S dot3(const V3<S>& a, const V3<S>& b) {
  return sum3(a.v[0] * b.v[0], a.v[1] * b.v[1], a.v[2] * b.v[2]);
}
template <typename S> CSF_HD V3<S> add3(const V3<S>& a, const V3<S>& b) {
  return mk3(a.v[0] + b.v[0], a.v[1] + b.v[1], a.v[2] + b.v[2]);
}
template <typename S> CSF_HD V3<S> sub3(const V3<S>& a, const V3<S>& b) {
  return mk3(a.v[0] - b.v[0], a.v[1] - b.v[1], a.v[2] - b.v[2]);
}
template <typename S> CSF_HD V3<S> cross3(const V3<S>& a, const V3<S>& b) {
  return mk3(a.v[1] * b.v[2] - a.v[2] * b.v[1], a.v[2] * b.v[0] - a.v[0] * b.v[2], a.v[0] * b.v[1] - a.v[1] * b.v[0]);
}
template <typename S> CSF_HD V3<S> matvec(const M3<S>& m, const V3<S>& p) {
  V3<S> o;
#pragma unroll
  for (int r = 0; r < 3; ++r) o.v[r] = sum3(m.m[3 * r] * p.v[0], m.m[3 * r + 1] * p.v[1], m.m[3 * r + 2] * p.v[2]);
  return o;
}
template <typename S> CSF_HD M3<S> matmul(const M3<S>& a, const M3<S>& b) {
  M3<S> o;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      o.m[3 * r + c] = sum3(a.m[3 * r] * b.m[c], a.m[3 * r + 1] * b.m[3 + c], a.m[3 * r + 2] * b.m[6 + c]);
  return o;
}
template <typename S> CSF_HD M3<S> transpose3(const M3<S>& a) {
  M3<S> o;
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int c = 0; c < 3; ++c) o.m[3 * r + c] = a.m[3 * c + r];
  return o;
}

// Pose (se3.hpp:21-45): rotation row-major + translation.
template <typename S> struct Pose {
  M3<S> R;
  V3<S> t;
};
template <typename S> CSF_HD V3<S> apply(const Pose<S>& p, const V3<S>& x) { return add3(matvec(p.R, x), p.t); }
template <typename S> CSF_HD Pose<S> compose(const Pose<S>& a, const Pose<S>& b) {
  Pose<S> o;
  o.R = matmul(a.R, b.R);
  o.t = add3(matvec(a.R, b.t), a.t);
  return o;
}
template <typename S> CSF_HD Pose<S> inverse(const Pose<S>& p) {
  Pose<S> o;
  o.R = transpose3(p.R);
  const V3<S> rt = matvec(o.R, p.t);
  o.t = mk3(-rt.v[0], -rt.v[1], -rt.v[2]);
  return o;
}

// exp of a twist (rho, phi) — se3.hpp:77-105, same branch and order.
template <typename S> CSF_HD Pose<S> exp_map(const S xi[6]) {
  const V3<S> rho = mk3(xi[0], xi[1], xi[2]);
  const V3<S> phi = mk3(xi[3], xi[4], xi[5]);
  const S t2 = dot3(phi, phi);
  S a, b, c;
  if (re(t2) < 1e-14) {
    a = lit<S>(1.0) - t2 / lit<S>(6.0);
    b = lit<S>(0.5) - t2 / lit<S>(24.0);
    c = lit<S>(1.0 / 6.0) - t2 / lit<S>(120.0);
  } else {
    const S t = sqrt_s(t2);
    a = sin_s(t) / t;
    const S sh = sin_s(t / lit<S>(2.0));
    b = lit<S>(2.0) * sh * sh / t2;
    c = (t - sin_s(t)) / (t2 * t);
  }
  const S z = lit<S>(0.0);
  M3<S> px;
  px.m[0] = z;         px.m[1] = -phi.v[2]; px.m[2] = phi.v[1];
  px.m[3] = phi.v[2];  px.m[4] = z;         px.m[5] = -phi.v[0];
  px.m[6] = -phi.v[1]; px.m[7] = phi.v[0];  px.m[8] = z;
  const M3<S> px2 = matmul(px, px);
  Pose<S> out;
  M3<S> v;
#pragma unroll
  for (int e = 0; e < 9; ++e) {
    const S id = lit<S>((e == 0 || e == 4 || e == 8) ? 1.0 : 0.0);
    out.R.m[e] = (id + a * px.m[e]) + b * px2.m[e];
    v.m[e] = (id + b * px.m[e]) + c * px2.m[e];
  }
  out.t = matvec(v, rho);
  return out;
}

// ----------------------------------------------------------------------------
// channel-group load/store helpers.  Packed arrays are element-major,
// channel-minor: value e occupies [e*(1+Dp) .. e*(1+Dp)+Dp].
// ----------------------------------------------------------------------------
template <typename S> CSF_DEV S load_ch(const double* base, int g0, int n_valid);
template <> CSF_DEV double load_ch<double>(const double* base, int, int) { return base[0]; }
template <typename S> CSF_DEV S load_ch(const double* base, int g0, int n_valid) {
  S o;
  o.re = base[0];
#pragma unroll
  for (int g = 0; g < Traits<S>::G; ++g) o.im[g] = (g < n_valid) ? base[1 + g0 + g] : 0.0;
  return o;
}
template <typename S> CSF_DEV void store_ch(double* base, const S& v, int g0, int n_valid, bool write_re);
template <> CSF_DEV void store_ch<double>(double* base, const double& v, int, int, bool write_re) {
  if (write_re) base[0] = v;
}
template <typename S> CSF_DEV void store_ch(double* base, const S& v, int g0, int n_valid, bool write_re) {
  if (write_re) base[0] = v.re;
#pragma unroll
  for (int g = 0; g < Traits<S>::G; ++g)
    if (g < n_valid) base[1 + g0 + g] = v.im[g];
}

}  // namespace csfd
