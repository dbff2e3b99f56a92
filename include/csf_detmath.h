/*
 * csf_detmath.h — deterministic elementary functions shared by host and device.
 *
 * Why this exists: the CSFD pipeline's real channel must be bit-identical on
 * the CPU (g++ -ffp-contract=off) and on sm_100a (nvcc -fmad=false), because
 * every discrete decision of the reference path (pixel picks via ifloor/lround,
 * validity and edge gates, zero crossings, |delta| < tol, LDLT pivots) reads
 * real parts.  glibc and libdevice exp/sin/cos differ in the last ulp, so the
 * few transcendental calls that sit on the device path use these
 * implementations on BOTH sides:
 *   - exp : bilateral spatial/range weights   (reference frames.cpp:28-29)
 *   - sin/cos : exp_map closed form            (reference se3.hpp:89-95)
 *   - cos : association angle gate cos(30 deg) (reference icp.cpp:97)
 * Only IEEE-exact operations (+ - * / and integer/bit manipulation) are used,
 * with an explicit evaluation order and no fused multiply-add, so any
 * IEEE-754 binary64 implementation yields the same bits.  Pinned against
 * glibc 2.39 in tests/test_detmath.py over the path's argument ranges: exp and
 * cos within 1 ulp, sin within 2 ulp (equal on 74-100% of arguments); the
 * whole oracle pipeline built with glibc instead (-DORC_LIBM) takes the same
 * discrete decisions and real poses within 2e-15 on configs 1 and 2.
 *
 * Algorithms (published, restated): Cody–Waite argument reduction with a
 * two-constant ln2 split (exp) and a three-constant pi/2 split (sin/cos, as in
 * fdlibm's medium-argument path), followed by Horner evaluation of the Taylor
 * series on the reduced interval.
 */
#ifndef CSF_DETMATH_H
#define CSF_DETMATH_H

#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define CSF_HD __host__ __device__ __forceinline__
#else
#define CSF_HD static inline
#endif

#ifdef __cplusplus
extern "C++" {
namespace csf_det {

CSF_HD double bits_to_double(uint64_t u) {
  double d;
  memcpy(&d, &u, sizeof d);
  return d;
}

CSF_HD double dfloor(double x) {
#if defined(__CUDA_ARCH__)
  return ::floor(x);
#else
  return __builtin_floor(x);
#endif
}

/* 2^k for k in [-1022, 1023], exact. */
CSF_HD double pow2i(int k) {
  return bits_to_double((uint64_t)(k + 1023) << 52);
}

/* exp(x): |error| <~ 1 ulp, deterministic. */
CSF_HD double exp(double x) {
  if (x != x) return x;
  if (x > 709.782712893384) return bits_to_double(0x7ff0000000000000ULL);
  if (x < -745.1332191019412) return 0.0;
  const double kInvLn2 = 1.4426950408889634074;
  /* ln2 split: hi has 32 significant bits so kd*hi is exact for |k| < 2^21. */
  const double kLn2Hi = 6.93147180369123816490e-01;
  const double kLn2Lo = 1.90821492927058770002e-10;
  const double kd = dfloor(x * kInvLn2 + 0.5);
  const int k = (int)kd;
  const double r = (x - kd * kLn2Hi) - kd * kLn2Lo;
  /* exp(r) = 1 + r*P(r), P Horner over 1/n!, n = 1..13, |r| <= 0.347. */
  double p = 1.0 / 6227020800.0;            /* 1/13! */
  p = p * r + 1.0 / 479001600.0;            /* 1/12! */
  p = p * r + 1.0 / 39916800.0;             /* 1/11! */
  p = p * r + 1.0 / 3628800.0;              /* 1/10! */
  p = p * r + 1.0 / 362880.0;               /* 1/9!  */
  p = p * r + 1.0 / 40320.0;                /* 1/8!  */
  p = p * r + 1.0 / 5040.0;                 /* 1/7!  */
  p = p * r + 1.0 / 720.0;                  /* 1/6!  */
  p = p * r + 1.0 / 120.0;                  /* 1/5!  */
  p = p * r + 1.0 / 24.0;                   /* 1/4!  */
  p = p * r + 1.0 / 6.0;                    /* 1/3!  */
  p = p * r + 0.5;                          /* 1/2!  */
  p = p * r + 1.0;                          /* 1/1!  */
  const double e = 1.0 + p * r;
  if (k >= -1022 && k <= 1023) return e * pow2i(k);
  if (k > 1023) return (e * pow2i(1023)) * pow2i(k - 1023);
  /* subnormal range: two exact-ish scalings, same order on every platform */
  return (e * pow2i(k + 600)) * pow2i(-600);
}

/* Reduced-argument kernels on |r| <= pi/4. */
CSF_HD double sin_kernel(double r) {
  const double r2 = r * r;
  double p = -1.0 / 1307674368000.0;        /* -1/15! */
  p = p * r2 + 1.0 / 6227020800.0;          /* +1/13! */
  p = p * r2 - 1.0 / 39916800.0;            /* -1/11! */
  p = p * r2 + 1.0 / 362880.0;              /* +1/9!  */
  p = p * r2 - 1.0 / 5040.0;                /* -1/7!  */
  p = p * r2 + 1.0 / 120.0;                 /* +1/5!  */
  p = p * r2 - 1.0 / 6.0;                   /* -1/3!  */
  return r + (r * r2) * p;
}

CSF_HD double cos_kernel(double r) {
  const double r2 = r * r;
  double p = 1.0 / 20922789888000.0;        /* +1/16! */
  p = p * r2 - 1.0 / 87178291200.0;         /* -1/14! */
  p = p * r2 + 1.0 / 479001600.0;           /* +1/12! */
  p = p * r2 - 1.0 / 3628800.0;             /* -1/10! */
  p = p * r2 + 1.0 / 40320.0;               /* +1/8!  */
  p = p * r2 - 1.0 / 720.0;                 /* -1/6!  */
  p = p * r2 + 1.0 / 24.0;                  /* +1/4!  */
  return (1.0 - 0.5 * r2) + (r2 * r2) * p;
}

/* x = n*(pi/2) + r, |n| < 2^20 keeps every n*c product exact. */
CSF_HD double reduce_pio2(double x, int* quadrant) {
  const double kTwoOverPi = 6.36619772367581382433e-01;
  const double kPio2_1 = 1.57079632673412561417e+00;  /* first 33 bits */
  const double kPio2_2 = 6.07710050630396597660e-11;  /* next 33 bits  */
  const double kPio2_3 = 2.02226624879595063154e-21;  /* tail          */
  const double nd = dfloor(x * kTwoOverPi + 0.5);
  double r = x - nd * kPio2_1;
  r = r - nd * kPio2_2;
  r = r - nd * kPio2_3;
  *quadrant = ((int)nd) & 3;
  return r;
}

CSF_HD double sin(double x) {
  if (x != x) return x;
  if (x > 1.6e6 || x < -1.6e6) return bits_to_double(0x7ff8000000000000ULL); /* outside |x| < 1.6e6: NaN */
  int q;
  const double r = reduce_pio2(x, &q);
  switch (q) {
    case 0: return sin_kernel(r);
    case 1: return cos_kernel(r);
    case 2: return -sin_kernel(r);
    default: return -cos_kernel(r);
  }
}

CSF_HD double cos(double x) {
  if (x != x) return x;
  if (x > 1.6e6 || x < -1.6e6) return bits_to_double(0x7ff8000000000000ULL);
  int q;
  const double r = reduce_pio2(x, &q);
  switch (q) {
    case 0: return cos_kernel(r);
    case 1: return -sin_kernel(r);
    case 2: return -cos_kernel(r);
    default: return sin_kernel(r);
  }
}

}  // namespace csf_det
}  // extern "C++"
#endif /* __cplusplus */

#endif /* CSF_DETMATH_H */
