// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the reference's CSFD numerics (proj/include/csf/csfd.hpp,
// se3.hpp, diff.hpp, image.hpp).  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load anything under
// oracle/.  The product (paper_2405_02187_b200/) never links this code.
//
// The reference itself cannot be compiled here (Eigen3, libpng and doctest
// are absent), so every function below cites the
// reference file:line it restates.  Eigen's fixed-size expression order is
// fixed explicitly (3-term sums a0 + (a1 + a2), 6-term sums split 3|3) —
// Eigen's own unrolling cannot be checked without its source.
//
// Transcendentals: by default exp/sin/cos come from include/csf_detmath.h so
// the oracle's real channel is bit-identical to the sm_100a path; define
// ORC_LIBM to use glibc instead (the reference's literal choice).
#pragma once

#include <cmath>
#include <cstddef>
#include <array>
#include <cstdint>
#include <limits>
#include <stdexcept>
#include <vector>

#include "../include/csf_detmath.h"

namespace orc {

// ---------------------------------------------------------------------------
// elementary real functions on the device path
// ---------------------------------------------------------------------------
inline double m_exp(double x) {
#ifdef ORC_LIBM
  return std::exp(x);
#else
  return csf_det::exp(x);
#endif
}
inline double m_sin(double x) {
#ifdef ORC_LIBM
  return std::sin(x);
#else
  return csf_det::sin(x);
#endif
}
inline double m_cos(double x) {
#ifdef ORC_LIBM
  return std::cos(x);
#else
  return csf_det::cos(x);
#endif
}

// csfd.hpp:16-28
inline constexpr double kDefaultStep = 1e-8;
struct StepSize {
  double h = kDefaultStep;
  constexpr StepSize() = default;
  explicit StepSize(double step) : h(step) {
    if (!(step > 0.0) || step > 1e-6)
      throw std::invalid_argument("StepSize: step must satisfy 0 < h <= 1e-6");
  }
};

// ---------------------------------------------------------------------------
// Complex — csfd.hpp:33-76 (truncated first order)
// ---------------------------------------------------------------------------
struct Complex {
  double re = 0.0, im = 0.0;
  constexpr Complex() = default;
  constexpr Complex(double r) : re(r) {}
  constexpr Complex(double r, double i) : re(r), im(i) {}
  Complex operator-() const { return {-re, -im}; }
  friend Complex operator+(const Complex& a, const Complex& b) { return {a.re + b.re, a.im + b.im}; }
  friend Complex operator-(const Complex& a, const Complex& b) { return {a.re - b.re, a.im - b.im}; }
  friend Complex operator*(const Complex& a, const Complex& b) {
    return {a.re * b.re, a.re * b.im + a.im * b.re};
  }
  friend Complex operator/(const Complex& a, const Complex& b) {
    if (b.re == 0.0) throw std::domain_error("Complex division by zero real part");
    return {a.re / b.re, (a.im * b.re - a.re * b.im) / (b.re * b.re)};
  }
  Complex& operator+=(const Complex& o) { return *this = *this + o; }
  Complex& operator-=(const Complex& o) { return *this = *this - o; }
  Complex& operator*=(const Complex& o) { return *this = *this * o; }
  Complex& operator/=(const Complex& o) { return *this = *this / o; }
  friend bool operator<(const Complex& a, const Complex& b) { return a.re < b.re; }
  friend bool operator>(const Complex& a, const Complex& b) { return a.re > b.re; }
};

// ---------------------------------------------------------------------------
// Bicomplex — csfd.hpp:83-140 (truncated second order, one pair)
// ---------------------------------------------------------------------------
struct Bicomplex {
  double re = 0.0, im1 = 0.0, im2 = 0.0, im12 = 0.0;
  constexpr Bicomplex() = default;
  constexpr Bicomplex(double r) : re(r) {}
  constexpr Bicomplex(double r, double a, double b, double c) : re(r), im1(a), im2(b), im12(c) {}
  Bicomplex operator-() const { return {-re, -im1, -im2, -im12}; }
  friend Bicomplex operator+(const Bicomplex& a, const Bicomplex& b) {
    return {a.re + b.re, a.im1 + b.im1, a.im2 + b.im2, a.im12 + b.im12};
  }
  friend Bicomplex operator-(const Bicomplex& a, const Bicomplex& b) {
    return {a.re - b.re, a.im1 - b.im1, a.im2 - b.im2, a.im12 - b.im12};
  }
  friend Bicomplex operator*(const Bicomplex& a, const Bicomplex& b) {
    return {a.re * b.re, a.re * b.im1 + a.im1 * b.re, a.re * b.im2 + a.im2 * b.re,
            a.re * b.im12 + a.im12 * b.re + a.im1 * b.im2 + a.im2 * b.im1};
  }
  friend Bicomplex operator/(const Bicomplex& a, const Bicomplex& b) {
    if (b.re == 0.0) throw std::domain_error("Bicomplex division by zero real part");
    const double den = b.re * b.re;
    const double inv = 1.0 / b.re;
    const double inv2 = inv * inv;
    return {a.re / b.re, (a.im1 * b.re - a.re * b.im1) / den, (a.im2 * b.re - a.re * b.im2) / den,
            a.im12 * inv - (a.im1 * b.im2 + a.im2 * b.im1) * inv2 - a.re * b.im12 * inv2 +
                2.0 * a.re * b.im1 * b.im2 * inv2 * inv};
  }
  Bicomplex& operator+=(const Bicomplex& o) { return *this = *this + o; }
  Bicomplex& operator-=(const Bicomplex& o) { return *this = *this - o; }
  Bicomplex& operator*=(const Bicomplex& o) { return *this = *this * o; }
  Bicomplex& operator/=(const Bicomplex& o) { return *this = *this / o; }
  friend bool operator<(const Bicomplex& a, const Bicomplex& b) { return a.re < b.re; }
  friend bool operator>(const Bicomplex& a, const Bicomplex& b) { return a.re > b.re; }
};

// ---------------------------------------------------------------------------
// Lifted<D> — D independent first-order directions packed as channels of one
// evaluation.  Channel d follows the Complex formula exactly, so
// Lifted<1> == Complex and channel d of Lifted<D> is bit-identical to a
// Complex pass seeded in direction d alone.
// ---------------------------------------------------------------------------
template <int D>
struct Lifted {
  double re = 0.0;
  double im[D] = {};
  Lifted() = default;
  Lifted(double r) : re(r) {}
  Lifted operator-() const {
    Lifted o;
    o.re = -re;
    for (int d = 0; d < D; ++d) o.im[d] = -im[d];
    return o;
  }
  friend Lifted operator+(const Lifted& a, const Lifted& b) {
    Lifted o;
    o.re = a.re + b.re;
    for (int d = 0; d < D; ++d) o.im[d] = a.im[d] + b.im[d];
    return o;
  }
  friend Lifted operator-(const Lifted& a, const Lifted& b) {
    Lifted o;
    o.re = a.re - b.re;
    for (int d = 0; d < D; ++d) o.im[d] = a.im[d] - b.im[d];
    return o;
  }
  friend Lifted operator*(const Lifted& a, const Lifted& b) {
    Lifted o;
    o.re = a.re * b.re;
    for (int d = 0; d < D; ++d) o.im[d] = a.re * b.im[d] + a.im[d] * b.re;
    return o;
  }
  friend Lifted operator/(const Lifted& a, const Lifted& b) {
    if (b.re == 0.0) throw std::domain_error("Complex division by zero real part");
    Lifted o;
    o.re = a.re / b.re;
    const double den = b.re * b.re;
    for (int d = 0; d < D; ++d) o.im[d] = (a.im[d] * b.re - a.re * b.im[d]) / den;
    return o;
  }
  Lifted& operator+=(const Lifted& o) { return *this = *this + o; }
  Lifted& operator-=(const Lifted& o) { return *this = *this - o; }
  Lifted& operator*=(const Lifted& o) { return *this = *this * o; }
  Lifted& operator/=(const Lifted& o) { return *this = *this / o; }
  friend bool operator<(const Lifted& a, const Lifted& b) { return a.re < b.re; }
  friend bool operator>(const Lifted& a, const Lifted& b) { return a.re > b.re; }
};

// ---------------------------------------------------------------------------
// real_part / channel traits
// ---------------------------------------------------------------------------
inline double real_part(double x) { return x; }
inline double real_part(const Complex& z) { return z.re; }
inline double real_part(const Bicomplex& z) { return z.re; }
template <int D>
double real_part(const Lifted<D>& z) { return z.re; }

inline bool isfinite_s(double x) { return std::isfinite(x); }
inline bool isfinite_s(const Complex& z) { return std::isfinite(z.re) && std::isfinite(z.im); }
inline bool isfinite_s(const Bicomplex& z) {
  return std::isfinite(z.re) && std::isfinite(z.im1) && std::isfinite(z.im2) && std::isfinite(z.im12);
}
template <int D>
bool isfinite_s(const Lifted<D>& z) {
  if (!std::isfinite(z.re)) return false;
  for (int d = 0; d < D; ++d)
    if (!std::isfinite(z.im[d])) return false;
  return true;
}

// ---------------------------------------------------------------------------
// Elementary lifts — csfd.hpp:148-263
// ---------------------------------------------------------------------------
inline Complex lift1(const Complex& z, double f, double d1) { return {f, d1 * z.im}; }
inline Bicomplex lift2(const Bicomplex& z, double f, double d1, double d2) {
  return {f, d1 * z.im1, d1 * z.im2, d1 * z.im12 + d2 * z.im1 * z.im2};
}
template <int D>
Lifted<D> liftd(const Lifted<D>& z, double f, double d1) {
  Lifted<D> o;
  o.re = f;
  for (int d = 0; d < D; ++d) o.im[d] = d1 * z.im[d];
  return o;
}

// double overloads (csfd.hpp:158-172)
inline double exp(double x) { return m_exp(x); }
inline double sqrt(double x) { return std::sqrt(x); }
inline double sin(double x) { return m_sin(x); }
inline double cos(double x) { return m_cos(x); }
inline double acos(double x) { return std::acos(x); }
inline double log(double x) { return std::log(x); }
inline double abs(double x) { return std::fabs(x); }

// Complex (csfd.hpp:174-205)
inline Complex exp(const Complex& z) { const double f = m_exp(z.re); return lift1(z, f, f); }
inline Complex log(const Complex& z) {
  if (!(z.re > 0.0)) throw std::domain_error("log of non-positive real part");
  return lift1(z, std::log(z.re), 1.0 / z.re);
}
inline Complex sqrt(const Complex& z) {
  if (z.re < 0.0) throw std::domain_error("sqrt of negative real part");
  const double f = std::sqrt(z.re);
  return lift1(z, f, 0.5 / f);
}
inline Complex sin(const Complex& z) { return lift1(z, m_sin(z.re), m_cos(z.re)); }
inline Complex cos(const Complex& z) { return lift1(z, m_cos(z.re), -m_sin(z.re)); }
inline Complex acos(const Complex& z) {
  if (z.re < -1.0 || z.re > 1.0) throw std::domain_error("acos argument outside [-1, 1]");
  return lift1(z, std::acos(z.re), -1.0 / std::sqrt(1.0 - z.re * z.re));
}

// Bicomplex (csfd.hpp:212-253)
inline Bicomplex exp(const Bicomplex& z) { const double f = m_exp(z.re); return lift2(z, f, f, f); }
inline Bicomplex log(const Bicomplex& z) {
  if (!(z.re > 0.0)) throw std::domain_error("log of non-positive real part");
  const double inv = 1.0 / z.re;
  return lift2(z, std::log(z.re), inv, -inv * inv);
}
inline Bicomplex sqrt(const Bicomplex& z) {
  if (z.re < 0.0) throw std::domain_error("sqrt of negative real part");
  const double f = std::sqrt(z.re);
  const double d1 = 0.5 / f;
  return lift2(z, f, d1, -0.5 * d1 / z.re);
}
inline Bicomplex sin(const Bicomplex& z) {
  const double s = m_sin(z.re), c = m_cos(z.re);
  return lift2(z, s, c, -s);
}
inline Bicomplex cos(const Bicomplex& z) {
  const double s = m_sin(z.re), c = m_cos(z.re);
  return lift2(z, c, -s, -c);
}
inline Bicomplex acos(const Bicomplex& z) {
  if (z.re < -1.0 || z.re > 1.0) throw std::domain_error("acos argument outside [-1, 1]");
  const double u = 1.0 - z.re * z.re;
  const double d1 = -1.0 / std::sqrt(u);
  return lift2(z, std::acos(z.re), d1, d1 * z.re / u);
}

// Lifted<D>: the Complex lifts per channel
template <int D> Lifted<D> exp(const Lifted<D>& z) { const double f = m_exp(z.re); return liftd(z, f, f); }
template <int D> Lifted<D> sqrt(const Lifted<D>& z) {
  if (z.re < 0.0) throw std::domain_error("sqrt of negative real part");
  const double f = std::sqrt(z.re);
  return liftd(z, f, 0.5 / f);
}
template <int D> Lifted<D> sin(const Lifted<D>& z) { return liftd(z, m_sin(z.re), m_cos(z.re)); }
template <int D> Lifted<D> cos(const Lifted<D>& z) { return liftd(z, m_cos(z.re), -m_sin(z.re)); }
template <int D> Lifted<D> acos(const Lifted<D>& z) {
  if (z.re < -1.0 || z.re > 1.0) throw std::domain_error("acos argument outside [-1, 1]");
  return liftd(z, std::acos(z.re), -1.0 / std::sqrt(1.0 - z.re * z.re));
}

// abs / min / max / clamp / ifloor — csfd.hpp:267-292
inline Complex abs(const Complex& z) { return z.re < 0.0 ? -z : z; }
inline Bicomplex abs(const Bicomplex& z) { return z.re < 0.0 ? -z : z; }
template <int D> Lifted<D> abs(const Lifted<D>& z) { return z.re < 0.0 ? -z : z; }

template <typename S> S smin(const S& a, const S& b) { return b < a ? b : a; }
template <typename S> S smax(const S& a, const S& b) { return b > a ? b : a; }
template <typename S> S clamp(const S& x, double lo, double hi) { return smax(smin(x, S(hi)), S(lo)); }

inline int ifloor(double x) { return static_cast<int>(std::floor(x)); }
template <typename S> int ifloor_s(const S& z) { return ifloor(real_part(z)); }

// promote / extract — csfd.hpp:297-320
inline Complex promote(double x, const StepSize& s) {
  if (!std::isfinite(x)) throw std::invalid_argument("promote: non-finite real value");
  return {x, s.h};
}
inline Bicomplex promote2(double x, const StepSize& s, bool seed1, bool seed2) {
  if (!std::isfinite(x)) throw std::invalid_argument("promote2: non-finite real value");
  return {x, seed1 ? s.h : 0.0, seed2 ? s.h : 0.0, 0.0};
}
inline double extract_derivative(const Complex& z, const StepSize& s) { return z.im / s.h; }
inline double extract_hessian(const Bicomplex& z, const StepSize& s) { return z.im12 / (s.h * s.h); }

// lift_measurement — csfd.hpp:324-333.  A stored/measured value with `Dm`
// channels enters an S evaluation: double drops channels, Complex/Lifted keep
// them (channel count must agree), Bicomplex drops them.
inline double lift_measurement_d(const Complex& m) { return m.re; }
template <typename S> struct Measure;
template <> struct Measure<double> {
  template <typename M> static double in(const M& m) { return real_part(m); }
};
template <> struct Measure<Complex> {
  static Complex in(const Complex& m) { return m; }
  static Complex in(const Lifted<1>& m) { return {m.re, m.im[0]}; }
  static Complex in(double m) { return Complex(m); }
};
template <> struct Measure<Bicomplex> {
  template <typename M> static Bicomplex in(const M& m) { return Bicomplex(real_part(m)); }
  // BUILDER-DEFINED extension: a Bicomplex-stored volume (second-order CSFD
  // of the whole pipeline, BASELINE config 3) keeps its own channels; the
  // reference only ever stores Complex fields and drops them (csfd.hpp:331).
  static Bicomplex in(const Bicomplex& m) { return m; }
};
template <int D> struct Measure<Lifted<D>> {
  static Lifted<D> in(const Lifted<D>& m) { return m; }
  static Lifted<D> in(double m) { return Lifted<D>(m); }
  static Lifted<D> in(const Complex& m) {
    static_assert(D == 1, "Complex measurement into Lifted<D != 1>");
    Lifted<D> o(m.re);
    o.im[0] = m.im;
    return o;
  }
};

// ---------------------------------------------------------------------------
// Fixed-size linear algebra with Eigen's small-size evaluation order.
// ---------------------------------------------------------------------------
template <typename S>
struct Vec3 {
  S v[3];
  Vec3() : v{S(0.0), S(0.0), S(0.0)} {}
  Vec3(const S& a, const S& b, const S& c) : v{a, b, c} {}
  S& operator[](int i) { return v[i]; }
  const S& operator[](int i) const { return v[i]; }
  S& x() { return v[0]; }
  S& y() { return v[1]; }
  S& z() { return v[2]; }
  const S& x() const { return v[0]; }
  const S& y() const { return v[1]; }
  const S& z() const { return v[2]; }
};

template <typename S>
struct Mat3 {
  S m[3][3];
  Mat3() {
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) m[r][c] = S(0.0);
  }
  static Mat3 identity() {
    Mat3 o;
    for (int i = 0; i < 3; ++i) o.m[i][i] = S(1.0);
    return o;
  }
  S& operator()(int r, int c) { return m[r][c]; }
  const S& operator()(int r, int c) const { return m[r][c]; }
};

template <typename S> using Vec6 = std::array<S, 6>;

using Vec3d = Vec3<double>;
using Mat3d = Mat3<double>;

template <typename S> Vec3<S> operator+(const Vec3<S>& a, const Vec3<S>& b) { return {a[0] + b[0], a[1] + b[1], a[2] + b[2]}; }
template <typename S> Vec3<S> operator-(const Vec3<S>& a, const Vec3<S>& b) { return {a[0] - b[0], a[1] - b[1], a[2] - b[2]}; }
template <typename S> Vec3<S> operator-(const Vec3<S>& a) { return {-a[0], -a[1], -a[2]}; }
// scalar * vector: functor(scalar, coeff) (Eigen scalar_product_op(lhs, rhs))
template <typename S> Vec3<S> operator*(const S& s, const Vec3<S>& a) { return {s * a[0], s * a[1], s * a[2]}; }
template <typename S> Vec3<S> operator/(const Vec3<S>& a, const S& s) { return {a[0] / s, a[1] / s, a[2] / s}; }
// vector * scalar: functor(coeff, scalar)
template <typename S> Vec3<S> operator*(const Vec3<S>& a, const S& s) { return {a[0] * s, a[1] * s, a[2] * s}; }

// 3-term redux: a0 + (a1 + a2)
template <typename S> S sum3(const S& a0, const S& a1, const S& a2) { return a0 + (a1 + a2); }
template <typename S> S dot(const Vec3<S>& a, const Vec3<S>& b) { return sum3(a[0] * b[0], a[1] * b[1], a[2] * b[2]); }
template <typename S> S squared_norm(const Vec3<S>& a) { return dot(a, a); }
template <typename S> S norm(const Vec3<S>& a) { return sqrt(squared_norm(a)); }
template <typename S> Vec3<S> cross(const Vec3<S>& a, const Vec3<S>& b) {
  return {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
}
template <typename S> Vec3<S> operator*(const Mat3<S>& m, const Vec3<S>& p) {
  Vec3<S> o;
  for (int r = 0; r < 3; ++r) o[r] = sum3(m(r, 0) * p[0], m(r, 1) * p[1], m(r, 2) * p[2]);
  return o;
}
template <typename S> Mat3<S> operator*(const Mat3<S>& a, const Mat3<S>& b) {
  Mat3<S> o;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) o(r, c) = sum3(a(r, 0) * b(0, c), a(r, 1) * b(1, c), a(r, 2) * b(2, c));
  return o;
}
template <typename S> Mat3<S> operator+(const Mat3<S>& a, const Mat3<S>& b) {
  Mat3<S> o;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) o(r, c) = a(r, c) + b(r, c);
  return o;
}
template <typename S> Mat3<S> operator*(const S& s, const Mat3<S>& a) {
  Mat3<S> o;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) o(r, c) = s * a(r, c);
  return o;
}
template <typename S> Mat3<S> transpose(const Mat3<S>& a) {
  Mat3<S> o;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) o(r, c) = a(c, r);
  return o;
}
inline Vec3d normalized(const Vec3d& a) {
  const double z = squared_norm(a);
  if (z > 0.0) return a / std::sqrt(z);
  return a;
}

// 6-term redux: (a0 + (a1 + a2)) + (a3 + (a4 + a5))
template <typename S> S sum6(const Vec6<S>& a) { return sum3(a[0], a[1], a[2]) + sum3(a[3], a[4], a[5]); }
inline double norm6(const Vec6<double>& a) {
  Vec6<double> sq;
  for (int i = 0; i < 6; ++i) sq[i] = a[i] * a[i];
  return std::sqrt(sum6(sq));
}

// ---------------------------------------------------------------------------
// se3 — se3.hpp:11-119
// ---------------------------------------------------------------------------
template <typename S> Mat3<S> skew(const Vec3<S>& v) {
  Mat3<S> m;
  m(0, 0) = S(0.0); m(0, 1) = -v.z(); m(0, 2) = v.y();
  m(1, 0) = v.z();  m(1, 1) = S(0.0); m(1, 2) = -v.x();
  m(2, 0) = -v.y(); m(2, 1) = v.x();  m(2, 2) = S(0.0);
  return m;
}

template <typename S>
struct PoseT {
  Mat3<S> rotation = Mat3<S>::identity();
  Vec3<S> translation;
  static PoseT identity() { return {}; }
  Vec3<S> operator*(const Vec3<S>& p) const { return rotation * p + translation; }
  PoseT operator*(const PoseT& o) const { return {rotation * o.rotation, rotation * o.translation + translation}; }
  PoseT inverse() const {
    const Mat3<S> rt = transpose(rotation);
    return {rt, -(rt * translation)};
  }
};
using Pose = PoseT<double>;

template <typename S> PoseT<S> pose_cast(const Pose& p) {
  PoseT<S> o;
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) o.rotation(r, c) = S(p.rotation(r, c));
    o.translation[r] = S(p.translation[r]);
  }
  return o;
}
template <typename S> Pose real_pose(const PoseT<S>& p) {
  Pose o;
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) o.rotation(r, c) = real_part(p.rotation(r, c));
    o.translation[r] = real_part(p.translation[r]);
  }
  return o;
}

// se3.hpp:77-105
template <typename S> PoseT<S> exp_map(const Vec6<S>& xi) {
  const Vec3<S> rho(xi[0], xi[1], xi[2]);
  const Vec3<S> phi(xi[3], xi[4], xi[5]);
  const S t2 = dot(phi, phi);
  S a, b, c;
  if (real_part(t2) < 1e-14) {
    a = S(1.0) - t2 / S(6.0);
    b = S(0.5) - t2 / S(24.0);
    c = S(1.0 / 6.0) - t2 / S(120.0);
  } else {
    const S t = sqrt(t2);
    a = sin(t) / t;
    const S sh = sin(t / S(2.0));
    b = S(2.0) * sh * sh / t2;
    c = (t - sin(t)) / (t2 * t);
  }
  const Mat3<S> px = skew(phi);
  const Mat3<S> px2 = px * px;
  PoseT<S> out;
  out.rotation = (Mat3<S>::identity() + a * px) + b * px2;
  const Mat3<S> v = (Mat3<S>::identity() + b * px) + c * px2;
  out.translation = v * rho;
  return out;
}

// se3.hpp:109-113
template <typename S> S log_angle(const PoseT<S>& p) {
  const S tr = sum3(p.rotation(0, 0), p.rotation(1, 1), p.rotation(2, 2));
  const S arg = (tr - S(1.0)) / S(2.0);
  return acos(clamp(arg, -1.0, 1.0));
}

// se3.hpp:116-119
template <typename S> PoseT<S> apply_increment(const Vec6<S>& delta, const PoseT<S>& pose) {
  return exp_map(delta) * pose;
}

// ---------------------------------------------------------------------------
// diff.hpp:16-72
// ---------------------------------------------------------------------------
template <typename T> T pairwise_block(const T* first, std::size_t n) {
  if (n <= 8) {
    T acc = first[0];
    for (std::size_t k = 1; k < n; ++k) acc = acc + first[k];
    return acc;
  }
  const std::size_t half = n / 2;
  return pairwise_block(first, half) + pairwise_block(first + half, n - half);
}
template <typename T> T pairwise_sum(const std::vector<T>& terms, T init = T{}) {
  if (terms.empty()) return init;
  return init + pairwise_block(terms.data(), terms.size());
}

template <typename F> Vec6<double> csfd_gradient(F&& f, const Vec6<double>& x, const StepSize& step = {}) {
  Vec6<double> g;
  for (int i = 0; i < 6; ++i) {
    Vec6<Complex> xs;
    for (int k = 0; k < 6; ++k) xs[k] = Complex(x[k], k == i ? step.h : 0.0);
    g[i] = extract_derivative(f(xs), step);
  }
  return g;
}
using Mat6d = std::array<std::array<double, 6>, 6>;
template <typename F> Mat6d csfd_hessian(F&& f, const Vec6<double>& x, const StepSize& step = {}) {
  Mat6d h{};
  for (int i = 0; i < 6; ++i)
    for (int j = i; j < 6; ++j) {
      Vec6<Bicomplex> xs;
      for (int k = 0; k < 6; ++k) xs[k] = Bicomplex(x[k], k == i ? step.h : 0.0, k == j ? step.h : 0.0, 0.0);
      const double hij = extract_hessian(f(xs), step);
      h[i][j] = hij;
      h[j][i] = hij;
    }
  return h;
}

// image.hpp:12-35
template <typename T>
struct Image {
  int width = 0, height = 0;
  std::vector<T> data;
  Image() = default;
  Image(int w, int h, T fill = T{}) : width(w), height(h), data(static_cast<std::size_t>(w) * h, fill) {}
  bool in_bounds(int x, int y) const { return x >= 0 && x < width && y >= 0 && y < height; }
  T& at(int x, int y) { return data[static_cast<std::size_t>(y) * width + x]; }
  const T& at(int x, int y) const { return data[static_cast<std::size_t>(y) * width + x]; }
};

}  // namespace orc
