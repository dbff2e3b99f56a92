// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// Pins the CPU restatement against the reference's own known-answer and
// property tests.  Each TEST names the reference test it restates
// (proj/tests/<file>:<lines>); the expected values and tolerances are the
// reference's.  The reference ships no stored golden vectors, so
// these analytic/property pins are the oracle's anchor.  Run by
// tests/test_oracle_kats.py (CPU, no GPU).
#include <cstdio>
#include <cstring>
#include <functional>
#include <random>
#include <string>

#include "orc_pipeline.hpp"

namespace orc {
namespace {

struct Case {
  const char* name;
  std::function<void()> fn;
};
std::vector<Case>& registry() {
  static std::vector<Case> r;
  return r;
}
struct Reg {
  Reg(const char* n, std::function<void()> f) { registry().push_back({n, std::move(f)}); }
};
int g_fail = 0, g_checks = 0;
const char* g_case = "";

#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)
#define TEST(name) static void CAT(t_, __LINE__)(); static Reg CAT(r_, __LINE__)(name, CAT(t_, __LINE__)); static void CAT(t_, __LINE__)()
#define CHECK(c)                                                                       \
  do {                                                                                 \
    ++g_checks;                                                                        \
    if (!(c)) {                                                                        \
      ++g_fail;                                                                        \
      std::printf("  FAIL [%s] %s:%d: %s\n", g_case, __FILE__, __LINE__, #c);          \
    }                                                                                  \
  } while (0)
#define CHECK_THROWS(expr, T)            \
  do {                                   \
    bool thrown = false;                 \
    try {                                \
      (void)(expr);                      \
    } catch (const T&) {                 \
      thrown = true;                     \
    }                                    \
    CHECK(thrown);                       \
  } while (0)

// oracles.hpp:11-32
double rel_err(double got, double want) {
  const double denom = std::fabs(want) > 1e-300 ? std::fabs(want) : 1.0;
  return std::fabs(got - want) / denom;
}
template <typename F> double fd1(F&& f, double x, double delta) { return (f(x + delta) - f(x - delta)) / (2.0 * delta); }
double approx(double a, double b, double eps) {  // doctest::Approx semantics
  return std::fabs(a - b) <= eps * (1.0 + std::max(std::fabs(a), std::fabs(b)));
}
std::mt19937_64 rng(unsigned s) { return std::mt19937_64(s); }
double uni(std::mt19937_64& g, double lo, double hi) { return std::uniform_real_distribution<double>(lo, hi)(g); }

// ---------------------------------------------------------------- csfd ----
template <typename S> S messy(S x) {  // test_csfd.cpp:19-25
  S a = exp(sin(x) * S(0.5)) + x * x / (S(1.0) + abs(x));
  S b = sqrt(a + S(2.0));
  S c = smin(b, a) + smax(b * S(0.25), a * a);
  S d = clamp(c, -0.75, 3.5);
  return d / (S(1.0) + c * c) + cos(a) * b;
}
template <typename S> S g1l(S x) { return exp(sin(x) * cos(x)); }
double g1(double x) { return std::exp(std::sin(x) * std::cos(x)); }
double g1p(double x) { return g1(x) * std::cos(2.0 * x); }
double g1pp(double x) { return g1p(x) * std::cos(2.0 * x) - 2.0 * g1(x) * std::sin(2.0 * x); }
template <typename S> S g2l(S x) { return sqrt(S(1.0) + x * x) / (S(2.0) + cos(x)); }
double g2p(double x) {
  const double r = std::sqrt(1.0 + x * x), d = 2.0 + std::cos(x);
  return (x / r) / d + r * std::sin(x) / (d * d);
}

TEST("csfd: step size validation (test_csfd.cpp:56-65)") {
  CHECK_THROWS(StepSize(0.0), std::invalid_argument);
  CHECK_THROWS(StepSize(-1e-8), std::invalid_argument);
  CHECK_THROWS(StepSize(2e-6), std::invalid_argument);
  CHECK_THROWS(StepSize(std::nan("")), std::invalid_argument);
  CHECK(StepSize().h == 1e-8);
  CHECK(StepSize(1e-20).h == 1e-20);
}
TEST("csfd: truncated product / z/z / zero-real division (test_csfd.cpp:67-86)") {
  const Complex p = Complex(1.0, 1e-8) * Complex(2.0, 3e-8);
  CHECK(p.re == 2.0 && p.im == 5e-8);
  const Complex q = Complex(3.7, 1e-8) / Complex(3.7, 1e-8);
  CHECK(q.re == 1.0 && q.im == 0.0);
  CHECK_THROWS(Complex(1.0, 0.0) / Complex(0.0, 1e-8), std::domain_error);
  CHECK_THROWS(Bicomplex(1.0) / Bicomplex(0.0, 1e-8, 0.0, 0.0), std::domain_error);
  CHECK_THROWS(Lifted<3>(1.0) / Lifted<3>(0.0), std::domain_error);
}
TEST("csfd: elementary lifts (test_csfd.cpp:88-105)") {
  const double h = 1e-8;
  const Complex e = exp(Complex(0.0, h));
  CHECK(e.re == 1.0 && e.im == h);
  const Complex s = sqrt(Complex(4.0, h));
  CHECK(s.re == 2.0 && s.im == h / 4.0);
  const Complex a = acos(Complex(0.5, h));
  CHECK(approx(a.re, M_PI / 3.0, 1e-15));
  CHECK(approx(a.im, -h / std::sqrt(0.75), 1e-15));
  CHECK_THROWS(log(Complex(-1.0, 1e-8)), std::domain_error);
  CHECK_THROWS(sqrt(Complex(-4.0, 1e-8)), std::domain_error);
  CHECK_THROWS(acos(Complex(1.5, 1e-8)), std::domain_error);
  CHECK_THROWS(acos(Bicomplex(-1.0001)), std::domain_error);
  CHECK_THROWS(promote(std::nan(""), StepSize()), std::invalid_argument);
  CHECK(promote(2.5, StepSize()).im == 1e-8);
}
TEST("csfd: first derivatives vs analytic 1e-12 (test_csfd.cpp:124-135)") {
  auto g = rng(17);
  const StepSize s;
  for (int k = 0; k < 100; ++k) {
    const double x = uni(g, -2.0, 2.0);
    CHECK(rel_err(extract_derivative(g1l(Complex(x, s.h)), s), g1p(x)) < 1e-12);
    CHECK(rel_err(extract_derivative(g2l(Complex(x, s.h)), s), g2p(x)) < 1e-12);
  }
}
TEST("csfd: h plateau 1e-7..1e-9 (test_csfd.cpp:137-147)") {
  for (double x : {-1.3, 0.2, 0.9, 1.7}) {
    const double d7 = extract_derivative(g1l(Complex(x, 1e-7)), StepSize(1e-7));
    const double d8 = extract_derivative(g1l(Complex(x, 1e-8)), StepSize(1e-8));
    const double d9 = extract_derivative(g1l(Complex(x, 1e-9)), StepSize(1e-9));
    CHECK(rel_err(d7, d8) < 1e-9);
    CHECK(rel_err(d9, d8) < 1e-9);
  }
}
TEST("csfd: real channel bit-identical to double (test_csfd.cpp:180-191)") {
  auto g = rng(31);
  for (int k = 0; k < 200; ++k) {
    const double x = uni(g, -2.5, 2.5);
    const double plain = messy<double>(x);
    CHECK(messy<Complex>(Complex(x, 1e-8)).re == plain);
    CHECK(messy<Bicomplex>(Bicomplex(x, 1e-8, 1e-8, 0.0)).re == plain);
    Lifted<4> l(x);
    l.im[2] = 1e-8;
    CHECK(messy<Lifted<4>>(l).re == plain);
  }
}
TEST("csfd: bicomplex im1 == complex im; Lifted<D> channel d == Complex pass d") {
  auto g = rng(37);
  for (int k = 0; k < 100; ++k) {
    const double x = uni(g, -2.5, 2.5);
    const Complex c = messy<Complex>(Complex(x, 1e-8));
    const Bicomplex b = messy<Bicomplex>(Bicomplex(x, 1e-8, 0.0, 0.0));
    CHECK(b.im1 == c.im);
    CHECK(b.im2 == 0.0 && b.im12 == 0.0);
    Lifted<5> l(x);
    for (int d = 0; d < 5; ++d) l.im[d] = d == 3 ? 1e-8 : 1e-9 * d;
    const Lifted<5> r = messy<Lifted<5>>(l);
    CHECK(r.im[3] == c.im);
    const Complex c1 = messy<Complex>(Complex(x, 1e-9));
    CHECK(r.im[1] == c1.im);
  }
}
TEST("csfd: x^2 y hessian, 2nd derivatives, symmetry (test_csfd.cpp:206-261)") {
  const StepSize s;
  auto f = [](Bicomplex x, Bicomplex y) { return x * x * y; };
  CHECK(approx(extract_hessian(f(promote2(1.0, s, true, true), Bicomplex(2.0)), s), 4.0, 1e-12));
  CHECK(approx(extract_hessian(f(promote2(1.0, s, true, false), promote2(2.0, s, false, true)), s), 2.0, 1e-12));
  CHECK(extract_hessian(f(Bicomplex(1.0), promote2(2.0, s, true, true)), s) == 0.0);
  auto g = rng(41);
  for (int k = 0; k < 60; ++k) {
    const double x = uni(g, -2.0, 2.0);
    CHECK(rel_err(extract_hessian(g1l(Bicomplex(x, s.h, s.h, 0.0)), s), g1pp(x)) < 1e-10);
  }
  auto h2 = [](Bicomplex x, Bicomplex y) {
    return exp(x * y) / (Bicomplex(2.0) + sin(x)) + sqrt(y * y + Bicomplex(1.0));
  };
  auto g3 = rng(43);
  for (int k = 0; k < 50; ++k) {
    const double x = uni(g3, -1.5, 1.5), y = uni(g3, -1.5, 1.5);
    const double hxy = extract_hessian(h2(promote2(x, s, true, false), promote2(y, s, false, true)), s);
    const double hyx = extract_hessian(h2(promote2(x, s, false, true), promote2(y, s, true, false)), s);
    CHECK(rel_err(hxy, hyx) < 1e-13);
  }
}
TEST("csfd: min/max ties, abs, clamp channels (test_csfd.cpp:263-294)") {
  const Complex a(2.0, 5e-8), b(2.0, 9e-8);
  CHECK(smin(a, b).im == 5e-8 && smax(a, b).im == 5e-8);
  CHECK(abs(Complex(-3.0, 7e-8)).im == -7e-8 && abs(Complex(0.0, 7e-8)).im == 7e-8);
  CHECK(abs(Bicomplex(-1.0, 2e-8, 3e-8, 4e-16)).im12 == -4e-16);
  CHECK(clamp(Complex(0.5, 3e-8), -1.0, 1.0).im == 3e-8);
  CHECK(clamp(Complex(1.5, 3e-8), -1.0, 1.0).re == 1.0 && clamp(Complex(1.5, 3e-8), -1.0, 1.0).im == 0.0);
  CHECK(clamp(Complex(-1.5, 3e-8), -1.0, 1.0).im == 0.0);
  CHECK(clamp(Complex(1.0, 3e-8), -1.0, 1.0).im == 3e-8);
}
TEST("csfd: bicomplex (a/b)*b (test_csfd.cpp:308-321)") {
  auto g = rng(53);
  for (int k = 0; k < 100; ++k) {
    const Bicomplex a(uni(g, -4, 4), uni(g, -1e-6, 1e-6), uni(g, -1e-6, 1e-6), uni(g, -1e-12, 1e-12));
    const Bicomplex b(uni(g, 0.5, 4), uni(g, -1e-6, 1e-6), uni(g, -1e-6, 1e-6), uni(g, -1e-12, 1e-12));
    const Bicomplex r = (a / b) * b;
    CHECK(rel_err(r.re, a.re) < 1e-14);
    CHECK(std::fabs(r.im1 - a.im1) < 1e-18 + 1e-12 * std::fabs(a.im1));
    CHECK(std::fabs(r.im12 - a.im12) < 1e-22 + 1e-10 * std::fabs(a.im12));
  }
}
TEST("csfd: gradient/hessian drivers (test_csfd.cpp:323-350)") {
  auto f = [](const auto& xi) {
    using S = std::decay_t<decltype(xi[0])>;
    return xi[0] * xi[0] * xi[1] + exp(xi[2]) + sin(xi[3]) * xi[4] + xi[5] * xi[5] * S(0.5);
  };
  const Vec6<double> x{1.0, 2.0, 0.3, -0.7, 1.4, 2.2};
  const auto g = csfd_gradient(f, x);
  CHECK(approx(g[0], 2.0 * x[0] * x[1], 1e-12));
  CHECK(approx(g[2], std::exp(x[2]), 1e-12));
  CHECK(approx(g[3], std::cos(x[3]) * x[4], 1e-12));
  const auto h = csfd_hessian(f, x);
  CHECK(approx(h[0][0], 2.0 * x[1], 1e-12));
  CHECK(approx(h[3][4], std::cos(x[3]), 1e-12));
  CHECK(approx(h[3][3], -std::sin(x[3]) * x[4], 1e-12));
  CHECK(h[0][2] == 0.0);
  bool sym = true;
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) sym = sym && h[i][j] == h[j][i];
  CHECK(sym);
}
TEST("csfd: pairwise_sum determinism (test_csfd.cpp:352-364)") {
  auto g = rng(59);
  std::vector<double> t(10001);
  for (auto& v : t) v = uni(g, -1.0, 1.0);
  const double s1 = pairwise_sum(t), s2 = pairwise_sum(t);
  CHECK(s1 == s2);
  long double ref = 0.0L;
  for (double v : t) ref += v;
  CHECK(rel_err(s1, static_cast<double>(ref)) < 1e-12);
  CHECK(pairwise_sum(std::vector<double>{}) == 0.0);
  CHECK(pairwise_sum(std::vector<double>{4.25}) == 4.25);
}
TEST("csfd: lifted vector norm/dot/matvec (test_csfd.cpp:366-388)") {
  const StepSize s;
  Vec3<Complex> v(Complex(3.0, s.h), Complex(4.0, 0.0), Complex(0.0, 0.0));
  const Complex n = norm(v);
  CHECK(approx(n.re, 5.0, 1e-15) && approx(extract_derivative(n, s), 0.6, 1e-12));
  CHECK(approx(extract_derivative(dot(v, v), s), 6.0, 1e-12));
  Mat3<Complex> m = Mat3<Complex>::identity();
  m(0, 1) = Complex(1.0, 0.0);
  const Vec3<Complex> mv = m * v;
  CHECK(mv.x().re == 7.0 && mv.x().im == s.h);
}

// ---------------------------------------------------------------- se3 -----
Vec6<double> random_twist(std::mt19937_64& g, double tmax, double rmax) {
  Vec6<double> xi;
  for (int i = 0; i < 3; ++i) xi[i] = uni(g, -tmax, tmax);
  for (int i = 3; i < 6; ++i) xi[i] = uni(g, -rmax, rmax);
  return xi;
}
double mat_diff(const Mat3d& a, const Mat3d& b) {
  double s = 0;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) s += (a(r, c) - b(r, c)) * (a(r, c) - b(r, c));
  return std::sqrt(s);
}
// Rodrigues oracle (independent closed form via libm)
Mat3d angle_axis(const Vec3d& phi) {
  const double t = std::sqrt(dot(phi, phi));
  const Vec3d a = phi / t;
  const double c = std::cos(t), s = std::sin(t);
  Mat3d m;
  for (int r = 0; r < 3; ++r)
    for (int cc = 0; cc < 3; ++cc) m(r, cc) = (r == cc ? c : 0.0) + (1 - c) * a[r] * a[cc];
  m(0, 1) -= s * a[2]; m(0, 2) += s * a[1];
  m(1, 0) += s * a[2]; m(1, 2) -= s * a[0];
  m(2, 0) -= s * a[1]; m(2, 1) += s * a[0];
  return m;
}
TEST("se3: exp(0)=I, translation, quarter turn, angle-axis (test_se3.cpp:39-86)") {
  const Pose p = exp_map<double>(Vec6<double>{});
  CHECK(mat_diff(p.rotation, Mat3d::identity()) == 0.0 && squared_norm(p.translation) == 0.0);
  const Pose t = exp_map<double>(Vec6<double>{1.0, -2.0, 3.0, 0, 0, 0});
  CHECK(t.translation.x() == 1.0 && t.translation.y() == -2.0 && t.translation.z() == 3.0);
  const Pose q = exp_map<double>(Vec6<double>{0, 0, 0, 0, 0, M_PI / 2.0});
  Mat3d want;
  want(0, 1) = -1; want(1, 0) = 1; want(2, 2) = 1;
  CHECK(mat_diff(q.rotation, want) < 1e-15);
  auto g = rng(67);
  for (int k = 0; k < 50; ++k) {
    const Vec3d phi(uni(g, -2, 2), uni(g, -2, 2), uni(g, -2, 2));
    CHECK(mat_diff(exp_map<double>(Vec6<double>{0, 0, 0, phi[0], phi[1], phi[2]}).rotation, angle_axis(phi)) < 1e-13);
  }
}
TEST("se3: compose/inverse (test_se3.cpp:104-126)") {
  auto g = rng(71);
  for (int k = 0; k < 20; ++k) {
    const Pose a = exp_map<double>(random_twist(g, 1.0, 2.0));
    const Pose b = exp_map<double>(random_twist(g, 1.0, 2.0));
    const Pose id = a * a.inverse();
    CHECK(mat_diff(id.rotation, Mat3d::identity()) < 1e-14 && norm(id.translation) < 1e-14);
    const Pose lhs = (a * b).inverse(), rhs = b.inverse() * a.inverse();
    CHECK(mat_diff(lhs.rotation, rhs.rotation) < 1e-13 && norm(lhs.translation - rhs.translation) < 1e-13);
  }
}
TEST("se3: log_angle round trip (test_se3.cpp:128-140)") {
  auto g = rng(73);
  for (int k = 0; k < 40; ++k) {
    const double theta = uni(g, 1e-3, M_PI - 1e-3);
    const Vec3d axis = normalized(Vec3d(uni(g, -1, 1), uni(g, -1, 1), uni(g, -1, 1)));
    const Pose p = exp_map<double>(Vec6<double>{0, 0, 0, theta * axis[0], theta * axis[1], theta * axis[2]});
    CHECK(approx(log_angle(p), theta, 1e-10));
  }
  CHECK(log_angle(Pose::identity()) == 0.0);
}
TEST("se3: point jacobian [I | -skew(p)] (test_se3.cpp:142-159)") {
  const Vec3d p(0.4, -1.2, 2.0);
  const Mat3d sk = skew(p);
  for (int row = 0; row < 3; ++row) {
    auto f = [&](const auto& xi) {
      using S = std::decay_t<decltype(xi[0])>;
      const Vec3<S> ps{S(p[0]), S(p[1]), S(p[2])};
      return (exp_map(xi) * ps)[row];
    };
    const auto gr = csfd_gradient(f, Vec6<double>{});
    for (int i = 0; i < 6; ++i) {
      const double want = i < 3 ? (i == row ? 1.0 : 0.0) : -sk(row, i - 3);
      CHECK(approx(gr[i], want, 1e-10));
    }
  }
}
TEST("se3: lifted exp real channel bit-identical (test_se3.cpp:187-200)") {
  auto g = rng(83);
  for (int k = 0; k < 20; ++k) {
    const Vec6<double> xi = random_twist(g, 1.0, 2.0);
    const Pose pd = exp_map<double>(xi);
    Vec6<Lifted<3>> xl;
    for (int i = 0; i < 6; ++i) {
      xl[i] = Lifted<3>(xi[i]);
      xl[i].im[k % 3] = i == (k % 6) ? 1e-8 : 0.0;
    }
    const PoseT<Lifted<3>> pl = exp_map(xl);
    bool same = true;
    for (int r = 0; r < 3; ++r) {
      for (int c = 0; c < 3; ++c) same = same && pl.rotation(r, c).re == pd.rotation(r, c);
      same = same && pl.translation[r].re == pd.translation[r];
    }
    CHECK(same);
  }
}
TEST("se3: twist derivatives vs FD (test_se3.cpp:161-185)") {
  auto g = rng(79);
  const Vec3d p(1.0, 0.5, -0.7);
  for (int k = 0; k < 10; ++k) {
    const Vec6<double> xi0 = random_twist(g, 0.8, 1.2);
    auto f = [&](const auto& xi) {
      using S = std::decay_t<decltype(xi[0])>;
      const auto q = exp_map(xi) * Vec3<S>(S(p[0]), S(p[1]), S(p[2]));
      return q[0] + S(2.0) * q[1] - q[2];
    };
    const auto gr = csfd_gradient(f, xi0);
    for (int i = 0; i < 6; ++i) {
      auto fi = [&](double v) {
        Vec6<double> x = xi0;
        x[i] = v;
        return f(x);
      };
      CHECK(approx(gr[i], fd1(fi, xi0[i], 1e-6), 1e-6));
    }
  }
}

// ------------------------------------------------------------- frames -----
Intrinsics test_camera() {
  Intrinsics k;
  k.fx = 80; k.fy = 80; k.cx = 31.5; k.cy = 23.5; k.width = 64; k.height = 48;
  return k;
}
Image<double> plane_depth(const Intrinsics& k, const Vec3d& n, double rho) {
  Image<double> d(k.width, k.height, 0.0);
  for (int y = 0; y < k.height; ++y)
    for (int x = 0; x < k.width; ++x) {
      const Vec3d dir((x - k.cx) / k.fx, (y - k.cy) / k.fy, 1.0);
      const double den = dot(n, dir);
      if (den > 1e-6 && rho / den > 0.0) d.at(x, y) = rho / den;
    }
  return d;
}
TEST("frames: project/backproject, at_level (test_frames.cpp:44-71)") {
  const Intrinsics k = test_camera();
  auto g = rng(89);
  for (int i = 0; i < 50; ++i) {
    const Vec3d p(uni(g, -1, 1), uni(g, -1, 1), uni(g, 0.5, 4.0));
    const auto px = project(k, p);
    CHECK(norm(backproject(k, px[0], px[1], p.z()) - p) < 1e-12);
  }
  const auto c = project(k, Vec3d(0, 0, 2));
  CHECK(c[0] == k.cx && c[1] == k.cy);
  const Intrinsics k1 = k.at_level(1);
  CHECK(k1.fx == k.fx / 2.0 && k1.cy == k.cy / 2.0 && k1.width == 32 && k1.height == 24);
  CHECK(k.at_level(2).fx == k.fx / 4.0 && k.at_level(2).width == 16);
}
TEST("frames: bilateral constant/holes/step/noise (test_frames.cpp:73-123)") {
  const Image<double> f = bilateral_filter(Image<double>(32, 24, 2.0));
  bool all = true;
  for (double v : f.data) all = all && v == 2.0;
  CHECK(all);
  Image<double> h(16, 16, 0.0);
  h.at(8, 8) = 1.5;
  const auto fh = bilateral_filter(h);
  CHECK(fh.at(8, 8) == 1.5 && fh.at(7, 8) == 0.0 && fh.at(0, 0) == 0.0);
  Image<double> s(32, 16, 0.0);
  for (int y = 0; y < 16; ++y)
    for (int x = 0; x < 32; ++x) s.at(x, y) = x < 16 ? 1.0 : 2.0;
  const auto fs = bilateral_filter(s);
  bool step_ok = true;
  for (int i = 0; i < 32 * 16; ++i) step_ok = step_ok && approx(fs.data[i], s.data[i], 1e-12);
  CHECK(step_ok);
  auto g = rng(97);
  std::normal_distribution<double> noise(0.0, 0.01);
  Image<double> d(48, 48, 0.0);
  for (auto& v : d.data) v = 2.0 + noise(g);
  const auto fd = bilateral_filter(d);
  auto var = [](const Image<double>& im) {
    double m = 0;
    int n = 0;
    for (int y = 8; y < im.height - 8; ++y)
      for (int x = 8; x < im.width - 8; ++x) m += im.at(x, y), ++n;
    m /= n;
    double v = 0;
    for (int y = 8; y < im.height - 8; ++y)
      for (int x = 8; x < im.width - 8; ++x) v += (im.at(x, y) - m) * (im.at(x, y) - m);
    return v / n;
  };
  CHECK(var(fd) < 0.4 * var(d));
}
TEST("frames: pyramid (test_frames.cpp:125-164)") {
  const auto c = downsample_depth(Image<double>(32, 24, 1.7));
  CHECK(c.width == 16 && c.height == 12);
  bool ok = true;
  for (double v : c.data) ok = ok && approx(v, 1.7, 1e-14);
  CHECK(ok);
  Image<double> d(32, 32, 0.0);
  for (int y = 0; y < 32; ++y)
    for (int x = 0; x < 32; ++x) d.at(x, y) = x < 16 ? 1.0 : 2.0;
  const auto pyr = build_depth_pyramid(d, 3);
  CHECK(pyr.size() == 3 && pyr[2].width == 8);
  ok = true;
  for (int y = 0; y < pyr[1].height; ++y)
    for (int x = 0; x < pyr[1].width; ++x) ok = ok && approx(pyr[1].at(x, y), (2 * x) < 16 ? 1.0 : 2.0, 1e-12);
  CHECK(ok);
  const Intrinsics k = test_camera();
  const Image<double> ramp = plane_depth(k, normalized(Vec3d(0.15, -0.1, 1.0)), 2.0);
  const auto p2 = build_depth_pyramid(ramp, 2);
  ok = true;
  for (int y = 2; y < p2[1].height - 2; ++y)
    for (int x = 2; x < p2[1].width - 2; ++x) ok = ok && approx(p2[1].at(x, y), ramp.at(2 * x, 2 * y), 2e-4);
  CHECK(ok);
}
TEST("frames: measure_surface flat/tilted/holes (test_frames.cpp:166-216)") {
  const Intrinsics k = test_camera();
  const auto maps = measure_surface<double>(Image<double>(k.width, k.height, 1.5), k);
  const Vec3d v = maps.vertices.at(10, 7);
  CHECK(v.x() == 1.5 * (10 - k.cx) / k.fx && v.y() == 1.5 * (7 - k.cy) / k.fy && v.z() == 1.5);
  bool ok = true;
  for (int y = 1; y < k.height - 1; ++y)
    for (int x = 1; x < k.width - 1; ++x) ok = ok && approx(maps.normals.at(x, y).z(), -1.0, 1e-12);
  CHECK(ok);
  CHECK(norm(maps.normals.at(k.width - 1, 5)) == 0.0 && norm(maps.normals.at(5, k.height - 1)) == 0.0);
  const Vec3d n = normalized(Vec3d(0.2, -0.3, 1.0));
  const auto tm = measure_surface<double>(plane_depth(k, n, 2.0), k);
  int checked = 0;
  ok = true;
  for (int y = 4; y < k.height - 4; y += 3)
    for (int x = 4; x < k.width - 4; x += 3) {
      const Vec3d got = tm.normals.at(x, y);
      if (norm(got) == 0.0) continue;
      ok = ok && norm(got + n) < 1e-9;
      ++checked;
    }
  CHECK(ok && checked > 50);
  Image<double> d(k.width, k.height, 1.0);
  d.at(5, 5) = 0.0;
  const auto hm = measure_surface<double>(d, k);
  CHECK(!vertex_valid(hm.vertices.at(5, 5)) && vertex_valid(hm.vertices.at(6, 5)));
  CHECK(!normal_valid(hm.normals.at(5, 5)) && !normal_valid(hm.normals.at(4, 5)) &&
        !normal_valid(hm.normals.at(5, 4)) && normal_valid(hm.normals.at(7, 7)));
}
TEST("frames: depth seed gain and normal derivative vs FD (test_frames.cpp:218-266)") {
  const Intrinsics k = test_camera();
  const Image<double> d = plane_depth(k, normalized(Vec3d(0.1, 0.05, 1.0)), 2.0);
  const StepSize s;
  const auto maps = measure_surface<Complex>(perturb_depth(d, 20, 15, s), k);
  const auto& v = maps.vertices.at(20, 15);
  CHECK(approx(extract_derivative(v.z(), s), 1.0, 1e-12));
  CHECK(approx(extract_derivative(v.x(), s), (20 - k.cx) / k.fx, 1e-12));
  CHECK(maps.vertices.at(40, 30).z().im == 0.0);
  const int sx = 21, sy = 16;
  const auto lifted = measure_surface<Complex>(perturb_depth(d, sx, sy, s), k);
  for (auto [nx, ny] : {std::pair{sx, sy}, {sx - 1, sy}, {sx, sy - 1}})
    for (int comp = 0; comp < 3; ++comp) {
      Image<double> dp = d, dm = d;
      dp.at(sx, sy) += 1e-6;
      dm.at(sx, sy) -= 1e-6;
      const double want = (measure_surface<double>(dp, k).normals.at(nx, ny)[comp] -
                           measure_surface<double>(dm, k).normals.at(nx, ny)[comp]) / 2e-6;
      CHECK(std::fabs(extract_derivative(lifted.normals.at(nx, ny)[comp], s) - want) < 1e-5);
    }
}
TEST("frames: perturb guard and bilinear (test_frames.cpp:268-318)") {
  Image<double> d(16, 16, 1.0);
  const StepSize s;
  CHECK_THROWS(perturb_depth(d, 20, 20, s), std::invalid_argument);
  d.at(4, 4) = 0.0;
  CHECK_THROWS(perturb_depth(d, 4, 4, s), std::invalid_argument);
  CHECK_THROWS(perturb_depth(d, 5, 4, s), std::invalid_argument);
  d.at(4, 4) = 1.0;
  d.at(10, 10) = 1.5;
  CHECK_THROWS(perturb_depth(d, 10, 10, s), std::invalid_argument);
  CHECK_THROWS(perturb_depth(d, 9, 10, s), std::invalid_argument);
  Image<double> b(8, 8, 0.0);
  for (int y = 0; y < 8; ++y)
    for (int x = 0; x < 8; ++x) b.at(x, y) = 1.0 + 0.1 * x + 0.2 * y;
  CHECK(bilinear_depth(b, 3.0, 4.0) == b.at(3, 4));
  CHECK(approx(bilinear_depth(b, 2.25, 5.5), 1.0 + 0.1 * 2.25 + 0.2 * 5.5, 1e-14));
  Image<Complex> bc(8, 8, Complex(0.0));
  for (int i = 0; i < 64; ++i) bc.data[i] = Complex(b.data[i]);
  bc.at(2, 5).im = s.h;
  CHECK(approx(extract_derivative(bilinear_depth(bc, Complex(2.25), Complex(5.5)), s), 0.75 * 0.5, 1e-12));
  b.at(3, 3) = 0.0;
  CHECK(bilinear_depth(b, 2.5, 2.5) == 0.0 && bilinear_depth(b, -0.5, 2.0) == 0.0 && bilinear_depth(b, 7.5, 2.0) == 0.0);
}

// --------------------------------------------------------------- tsdf -----
Intrinsics small_camera() {
  Intrinsics k;
  k.fx = 120; k.fy = 120; k.cx = 79.5; k.cy = 59.5; k.width = 160; k.height = 120;
  return k;
}
struct SphereFixture {
  Scene scene;
  Intrinsics k = small_camera();
  TsdfVolumeT<Complex> volume{VolumeParams::cube(64, 0.02, Vec3d(-0.63, -0.63, -0.63))};
  std::vector<Pose> poses;
  SphereFixture() {
    scene.spheres.push_back({Vec3d(), 0.5});
    for (int i = 0; i < 8; ++i) poses.push_back(orbit_pose(Vec3d(), 1.6, 0.8, 2.0 * M_PI * i / 8));
    for (const Pose& p : poses)
      surface_update(volume, complex_depth(render_depth(scene, p, k)), pose_cast<Complex>(p), k);
  }
};
const SphereFixture& sphere_fixture() {
  static SphereFixture f;
  return f;
}
TEST("tsdf: fresh volume lattice (test_tsdf.cpp:70-88)") {
  const VolumeParams p = VolumeParams::cube(8, 0.1, Vec3d(1, 2, 3));
  CHECK(approx(p.mu, 0.5, 1e-12));
  TsdfVolumeT<Complex> vol(p);
  bool ok = vol.tsdf.size() == 512;
  for (std::size_t i = 0; i < vol.tsdf.size(); ++i) ok = ok && vol.tsdf[i].re == 1.0 && vol.tsdf[i].im == 0.0 && vol.weight[i] == 0.0;
  CHECK(ok);
  CHECK(norm(vol.voxel_position(1, 2, 3) - Vec3d(1.1, 2.2, 3.3)) < 1e-15);
  CHECK(vol.index(1, 0, 0) == 1 && vol.index(0, 1, 0) == 8 && vol.index(0, 0, 1) == 64);
}
TEST("tsdf: projective measurement KATs (test_tsdf.cpp:90-147)") {
  const Intrinsics k = small_camera();
  const double d = 2.0, mu = 0.1;
  const Image<Complex> depth(k.width, k.height, Complex(d));
  const Pose id = Pose::identity();
  const Vec3d c;
  auto psi = [&](const Vec3d& p) { return measured_tsdf<double>(depth, id, k, mu, p, c); };
  CHECK(psi(Vec3d(0, 0, d)).has_value() && std::fabs(*psi(Vec3d(0, 0, d))) < 1e-12);
  CHECK(approx(*psi(Vec3d(0, 0, d - 0.5 * mu)), 0.5, 1e-9));
  CHECK(*psi(Vec3d(0, 0, 0.5)) == 1.0);
  CHECK(approx(*psi(Vec3d(0, 0, d + 0.5 * mu)), -0.5, 1e-9));
  CHECK(!psi(Vec3d(0, 0, d + 1.5 * mu)).has_value());
  CHECK(!psi(Vec3d(0, 0, -1.0)).has_value());
  CHECK(!psi(Vec3d(5.0, 0, 2.0)).has_value());
  Image<Complex> holey = depth;
  holey.at(79, 59) = Complex(0.0);
  CHECK(!measured_tsdf<double>(holey, id, k, mu, Vec3d(0, 0, d), c).has_value());
  for (auto px : {std::pair{20.0, 15.0}, {130.5, 100.5}, {3.0, 110.0}}) {
    const Vec3d dir((px.first - k.cx) / k.fx, (px.second - k.cy) / k.fy, 1.0);
    const auto v = psi(d * dir);
    CHECK(v.has_value() && std::fabs(*v) < 1e-9);
  }
}
TEST("tsdf: d psi / d xi vs FD, d psi / d D, saturation (test_tsdf.cpp:149-246)") {
  const Intrinsics k = small_camera();
  const double mu = 0.1;
  Scene scene;
  const Vec3d pn = normalized(Vec3d(-0.2, 0.1, -1.0));
  scene.planes.push_back({pn, dot(pn, Vec3d(0, 0, 2))});
  const Pose base = Pose::identity();
  const Image<Complex> depth = complex_depth(render_depth(scene, base, k));
  const Vec3d probe(0.15, -0.1, 1.93);
  auto value = [&](const Vec6<double>& xi) {
    const Pose c2w = apply_increment(xi, base);
    return *measured_tsdf<double>(depth, c2w.inverse(), k, mu, probe, c2w.translation);
  };
  auto lifted = [&](const Vec6<Complex>& xi) {
    const PoseT<Complex> c2w = exp_map(xi) * pose_cast<Complex>(base);
    return *measured_tsdf<Complex>(depth, c2w.inverse(), k, mu, Vec3<Complex>(probe[0], probe[1], probe[2]),
                                   c2w.translation);
  };
  const auto g = csfd_gradient(lifted, Vec6<double>{});
  double gn = 0;
  for (int i = 0; i < 6; ++i) {
    const double fd = fd1([&](double t) { Vec6<double> xi{}; xi[i] = t; return value(xi); }, 0.0, 1e-6);
    CHECK(approx(g[i], fd, 1e-5));
    gn += g[i] * g[i];
  }
  CHECK(std::sqrt(gn) > 0.1);
  // depth pixel derivative
  Image<double> plain(k.width, k.height, 2.0);
  const double px = 83.25, py = 61.5;
  const Vec3d pr = (2.0 - 0.02) * Vec3d((px - k.cx) / k.fx, (py - k.cy) / k.fy, 1.0);
  const StepSize h;
  const auto v = measured_tsdf<Complex>(perturb_depth(plain, 83, 61, h), pose_cast<Complex>(Pose::identity()), k, mu,
                                        Vec3<Complex>(pr[0], pr[1], pr[2]), Vec3<Complex>());
  CHECK(approx(extract_derivative(*v, h), (1.0 - 0.25) * (1.0 - 0.5) / mu, 1e-9));
  // saturation
  Vec6<Complex> xi;
  for (auto& x : xi) x = Complex(0.0);
  xi[2].im = 1e-8;
  const PoseT<Complex> c2w = exp_map(xi);
  const auto sat = measured_tsdf<Complex>(Image<Complex>(k.width, k.height, Complex(2.0)), c2w.inverse(), k, 0.1,
                                          Vec3<Complex>(0.0, 0.0, 0.5), c2w.translation);
  CHECK(sat->re == 1.0 && sat->im == 0.0);
}
TEST("tsdf: single-frame fusion stores psi bit for bit (test_tsdf.cpp:248-276)") {
  const SphereFixture& fx = sphere_fixture();
  TsdfVolumeT<Complex> vol(VolumeParams::cube(24, 0.02, Vec3d(-0.24, -0.24, 0.1)));
  const Pose pose = fx.poses[0];
  const Image<Complex> depth = complex_depth(render_depth(fx.scene, pose, fx.k));
  surface_update(vol, depth, pose_cast<Complex>(pose), fx.k);
  const Pose w2c = pose.inverse();
  int observed = 0;
  bool ok = true;
  for (int kk = 0; kk < 24; ++kk)
    for (int j = 0; j < 24; ++j)
      for (int i = 0; i < 24; ++i) {
        const std::size_t idx = vol.index(i, j, kk);
        const auto m = measured_tsdf<double>(depth, w2c, fx.k, vol.params.mu, vol.voxel_position(i, j, kk), pose.translation);
        if (m) {
          ++observed;
          ok = ok && vol.weight[idx] == 1.0 && vol.tsdf[idx].re == *m;
        } else {
          ok = ok && vol.weight[idx] == 0.0 && vol.tsdf[idx].re == 1.0;
        }
      }
  CHECK(ok && observed > 500);
}
TEST("tsdf: capped running average (test_tsdf.cpp:278-309)") {
  const Intrinsics k = small_camera();
  VolumeParams p = VolumeParams::cube(4, 0.02, Vec3d(-0.03, -0.03, 1.9));
  p.weight_cap = 4.0;
  TsdfVolumeT<Complex> vol(p);
  const PoseT<Complex> id = PoseT<Complex>::identity();
  auto flat = [&](double d) { return Image<Complex>(k.width, k.height, Complex(d)); };
  surface_update(vol, flat(2.00), id, k);
  surface_update(vol, flat(2.01), id, k);
  const std::size_t idx = vol.index(1, 1, 1);
  const auto m1 = measured_tsdf<double>(flat(2.00), Pose(), k, p.mu, vol.voxel_position(1, 1, 1), Vec3d());
  const auto m2 = measured_tsdf<double>(flat(2.01), Pose(), k, p.mu, vol.voxel_position(1, 1, 1), Vec3d());
  CHECK(vol.weight[idx] == 2.0 && approx(vol.tsdf[idx].re, 0.5 * (*m1 + *m2), 1e-15));
  for (int i = 0; i < 10; ++i) surface_update(vol, flat(2.00), id, k);
  CHECK(vol.weight[idx] == 4.0);
  const double late = vol.tsdf[idx].re;
  surface_update(vol, flat(2.00), id, k);
  CHECK(vol.weight[idx] == 4.0 && std::fabs(vol.tsdf[idx].re - *m1) < std::fabs(late - *m1));
}
TEST("tsdf: fused sphere accuracy (test_tsdf.cpp:311-345)") {
  const SphereFixture& fx = sphere_fixture();
  const double mu = fx.volume.params.mu;
  double max_err = 0, sum_err = 0;
  int n_band = 0, inside_unseen = 0;
  for (int kk = 0; kk < 64; ++kk)
    for (int j = 0; j < 64; ++j)
      for (int i = 0; i < 64; ++i) {
        const Vec3d p = fx.volume.voxel_position(i, j, kk);
        const double sdf = norm(p) - 0.5;
        const std::size_t idx = fx.volume.index(i, j, kk);
        const double w = fx.volume.weight[idx];
        if (std::fabs(sdf) < 0.5 * mu && w >= 3.0) {
          const double err = std::fabs(mu * fx.volume.tsdf[idx].re - sdf);
          max_err = std::max(max_err, err);
          sum_err += err;
          ++n_band;
        }
        if (sdf < -2.0 * mu && w > 0.0) ++inside_unseen;
      }
  CHECK(n_band > 2000 && sum_err / n_band < 0.025 && max_err < 0.1 && inside_unseen == 0);
}
TEST("tsdf: affine field trilinear exact (test_tsdf.cpp:347-390)") {
  VolumeParams p = VolumeParams::cube(12, 0.05, Vec3d(-0.2, -0.1, 0.0));
  TsdfVolumeT<Complex> vol(p);
  const Vec3d g(0.21, -0.34, 0.05);
  const double c = 0.1;
  for (int kk = 0; kk < 12; ++kk)
    for (int j = 0; j < 12; ++j)
      for (int i = 0; i < 12; ++i) {
        vol.tsdf[vol.index(i, j, kk)] = Complex(c + dot(g, vol.voxel_position(i, j, kk)));
        vol.weight[vol.index(i, j, kk)] = 1.0;
      }
  auto r = rng(77);
  for (int t = 0; t < 30; ++t) {
    const Vec3d q(uni(r, -0.15, 0.3), uni(r, -0.05, 0.4), uni(r, 0.05, 0.5));
    const auto f = sample_tsdf<double>(vol, q);
    CHECK(f.has_value() && approx(*f, c + dot(g, q), 1e-13));
    const auto fg = sample_gradient<double>(vol, q);
    if (fg) CHECK(norm(*fg - g) < 1e-12);
  }
  CHECK(!sample_tsdf<double>(vol, Vec3d(-0.21, 0, 0.1)).has_value());
  CHECK(!sample_tsdf<double>(vol, Vec3d(0, 0, 0.56)).has_value());
  const StepSize h;
  const auto fq = sample_tsdf<Complex>(vol, Vec3<Complex>(Complex(0.05, h.h), Complex(0.12), Complex(0.3)));
  CHECK(approx(extract_derivative(*fq, h), g.x(), 1e-12));
  vol.weight[vol.index(4, 4, 4)] = 0.0;
  CHECK(!sample_tsdf<double>(vol, Vec3d(-0.01, 0.09, 0.19)).has_value());
}
TEST("tsdf: raycast recovers the fused sphere (test_tsdf.cpp:392-441)") {
  const SphereFixture& fx = sphere_fixture();
  const Pose view = orbit_pose(Vec3d(), 1.5, 0.7, 0.39);
  const auto maps = raycast<double>(fx.volume, view, fx.k);
  int hits = 0, misses_ok = 0;
  double max_e = 0, sum_e = 0, worst_n = 1.0;
  bool phantom_ok = true, required = true;
  for (int y = 0; y < fx.k.height; ++y)
    for (int x = 0; x < fx.k.width; ++x) {
      const Vec3d dir = normalized(view.rotation * Vec3d((x - fx.k.cx) / fx.k.fx, (y - fx.k.cy) / fx.k.fy, 1.0));
      const Vec3d o = view.translation;
      const double tca = -dot(o, dir);
      const double b2 = squared_norm(o + tca * dir);
      const bool valid = normal_valid(maps.normals.at(x, y));
      const double tic = b2 < 0.25 ? tca - std::sqrt(0.25 - b2) : 0.0;
      const double hz = (o + tic * dir).z();
      if (b2 < 0.46 * 0.46 && tca > 0.0 && hz > -0.1) {
        required = required && valid;
        if (!valid) continue;
        const Vec3d v = maps.vertices.at(x, y);
        const double e = std::fabs(norm(v) - 0.5);
        max_e = std::max(max_e, e);
        sum_e += e;
        worst_n = std::min(worst_n, dot(maps.normals.at(x, y), normalized(v)));
        ++hits;
      } else if (b2 > 0.54 * 0.54) {
        if (!valid) ++misses_ok;
        else phantom_ok = phantom_ok && std::fabs(norm(maps.vertices.at(x, y)) - 0.5) < 0.06;
      }
    }
  CHECK(required && hits > 1000 && misses_ok > 1000 && sum_e / hits < 0.005 && max_e < 0.03 && worst_n > 0.95 &&
        phantom_ok);
}
TEST("tsdf: lifted raycast real channel bit-identical (test_tsdf.cpp:443-460)") {
  const SphereFixture& fx = sphere_fixture();
  const Pose view = orbit_pose(Vec3d(), 1.5, 0.7, 0.39);
  const auto plain = raycast<double>(fx.volume, view, fx.k);
  const auto lifted = raycast<Complex>(fx.volume, pose_cast<Complex>(view), fx.k);
  bool ok = true;
  for (int y = 0; y < fx.k.height; y += 7)
    for (int x = 0; x < fx.k.width; x += 7)
      for (int c = 0; c < 3; ++c)
        ok = ok && lifted.vertices.at(x, y)[c].re == plain.vertices.at(x, y)[c] &&
             lifted.vertices.at(x, y)[c].im == 0.0 && lifted.normals.at(x, y)[c].re == plain.normals.at(x, y)[c];
  CHECK(ok);
}
TEST("tsdf: raycast d(hit distance)/d xi vs FD (test_tsdf.cpp:462-511)") {
  const SphereFixture& fx = sphere_fixture();
  const Pose base = orbit_pose(Vec3d(), 1.5, 0.7, 0.39);
  RaycastConfig cfg;
  cfg.near_clip = 0.95;
  const Vec3d ob = base.translation;
  auto hit = [&](const Vec6<double>& xi) {
    const auto m = raycast<double>(fx.volume, apply_increment(xi, base), fx.k, cfg);
    return norm(m.vertices.at(80, 60) - ob);
  };
  const StepSize h;
  double gn = 0;
  for (int comp = 0; comp < 6; ++comp) {
    Vec6<Complex> xi;
    for (auto& x : xi) x = Complex(0.0);
    xi[comp].im = h.h;
    const auto m = raycast<Complex>(fx.volume, exp_map(xi) * pose_cast<Complex>(base), fx.k, cfg);
    CHECK(normal_valid(m.normals.at(80, 60)));
    const Vec3<Complex> diff = m.vertices.at(80, 60) - Vec3<Complex>(ob[0], ob[1], ob[2]);
    const double deriv = extract_derivative(sqrt(dot(diff, diff)), h);
    const double fd = fd1([&](double t) { Vec6<double> s{}; s[comp] = t; return hit(s); }, 0.0, 1e-5);
    CHECK(approx(deriv, fd, 1e-5));
    gn += deriv * deriv;
  }
  CHECK(std::sqrt(gn) > 0.2);
}

// ---------------------------------------------------------------- icp -----
std::vector<Correspondence> synthetic_corrs(unsigned seed, int n, const Pose& base, const Vec6<double>& xi_true) {
  auto g = rng(seed);
  const Pose target = apply_increment(xi_true, base);
  std::vector<Correspondence> c;
  for (int i = 0; i < n; ++i) {
    const Vec3d v(uni(g, -0.8, 0.8), uni(g, -0.6, 0.6), uni(g, 1.2, 3.0));
    Vec3d nrm(uni(g, -1, 1), uni(g, -1, 1), uni(g, -1, 1));
    if (norm(nrm) < 1e-3) nrm = Vec3d(0, 0, 1);
    c.push_back({v, target * v, normalized(nrm)});
  }
  return c;
}
Pose reference_pose(double a) { return orbit_pose(Vec3d(0.2, 0.1, 0.4), 1.9, 1.4, a); }
double terr(const Pose& a, const Pose& b) { return norm(a.translation - b.translation); }
double rerr_deg(const Pose& a, const Pose& b) {
  Pose rel;
  rel.rotation = transpose(b.rotation) * a.rotation;
  return log_angle(rel) * 180.0 / M_PI;
}
Scene default_scene() {  // synth.cpp:47-53
  Scene s;
  s.planes.push_back({Vec3d(0, 0, 1), 0.0});
  s.spheres.push_back({Vec3d(0.0, 0.0, 0.6), 0.5});
  s.boxes.push_back({Vec3d(0.75, 0.45, 0.25), Vec3d(0.25, 0.2, 0.25)});
  return s;
}
TEST("icp: association counts and gates (test_icp.cpp:100-159)") {
  const Intrinsics k = small_camera();
  const Scene scene = default_scene();
  const Pose ref = reference_pose(0.0);
  const auto rc = measure_surface<double>(render_depth(scene, ref, k), k);
  SurfaceMaps<double> pred;
  pred.vertices = Image<Vec3d>(k.width, k.height, Vec3d());
  pred.normals = Image<Vec3d>(k.width, k.height, Vec3d());
  for (int y = 0; y < k.height; ++y)
    for (int x = 0; x < k.width; ++x) {
      if (!vertex_valid(rc.vertices.at(x, y)) || !normal_valid(rc.normals.at(x, y))) continue;
      pred.vertices.at(x, y) = ref * rc.vertices.at(x, y);
      pred.normals.at(x, y) = ref.rotation * rc.normals.at(x, y);
    }
  const Pose query = reference_pose(0.12);
  const auto meas = measure_surface<double>(render_depth(scene, query, k), k);
  IcpConfig cfg;
  const auto aligned = associate(meas, pred, query, ref, k, cfg);
  CHECK(aligned.size() > 8000);
  double mr = 0;
  for (const auto& c : aligned) mr += std::fabs(dot(query * c.vertex - c.model_vertex, c.model_normal));
  CHECK(mr / aligned.size() < 0.003);
  Pose off = query;
  off.translation[2] += 0.25;
  const auto shifted = associate(meas, pred, off, ref, k, cfg);
  CHECK(shifted.size() < aligned.size() / 10);
  IcpConfig tight = cfg;
  tight.theta_max_deg = 5.0;
  CHECK(associate(meas, pred, off, ref, k, tight).size() <= shifted.size());
  const auto strided = associate(meas, pred, query, ref, k, cfg, 2);
  CHECK(strided.size() > aligned.size() / 6 && strided.size() < aligned.size() / 3);
}
TEST("icp: energy zero at truth, lifted channels pure (test_icp.cpp:161-188)") {
  const Pose base = reference_pose(0.3);
  const Vec6<double> xt{0.02, -0.015, 0.01, 0.015, -0.01, 0.02};
  const auto corrs = synthetic_corrs(7, 300, base, xt);
  CHECK(icp_energy(corrs, xt, base) == 0.0);
  CHECK(icp_loss(corrs, base) > 1e-4);
  const double plain = icp_loss(corrs, base);
  Vec6<Complex> zc;
  for (auto& z : zc) z = Complex(0.0);
  CHECK(icp_energy(corrs, zc, base).re == plain && icp_energy(corrs, zc, base).im == 0.0);
  Vec6<Bicomplex> zb;
  for (auto& z : zb) z = Bicomplex(0.0);
  CHECK(icp_energy(corrs, zb, base).re == plain);
  Vec6<Complex> sc = zc;
  sc[3].im = 1e-8;
  Vec6<Bicomplex> sb = zb;
  sb[3].im1 = 1e-8;
  CHECK(icp_energy(corrs, sb, base).im1 == icp_energy(corrs, sc, base).im);
}
TEST("icp: CSFD gradient/Hessian vs FD, zero gradient at truth (test_icp.cpp:190-230)") {
  const Pose base = reference_pose(0.3);
  const Vec6<double> xt{0.03, -0.02, 0.025, 0.02, -0.015, 0.01};
  const auto corrs = synthetic_corrs(11, 250, base, xt);
  const auto grad = icp_gradient(corrs, base);
  for (int c = 0; c < 6; ++c) {
    const double fd = fd1([&](double t) { Vec6<double> xi{}; xi[c] = t; return icp_energy(corrs, xi, base); }, 0.0, 1e-6);
    CHECK(rel_err(grad[c], fd) < 5e-7);
  }
  const auto hess = icp_hessian(corrs, base);
  bool sym = true;
  for (int i = 0; i < 6; ++i)
    for (int j = 0; j < 6; ++j) sym = sym && hess[i][j] == hess[j][i];
  CHECK(sym);
  auto energy = [&](const auto& xi) { return icp_energy(corrs, xi, base); };
  for (int c = 0; c < 6; ++c) {
    Vec6<double> p{}, m{};
    p[c] = 1e-6;
    m[c] = -1e-6;
    const auto gp = csfd_gradient(energy, p), gm = csfd_gradient(energy, m);
    for (int r = 0; r < 6; ++r) CHECK(rel_err(hess[r][c], (gp[r] - gm[r]) / 2e-6) < 2e-5);
  }
  const auto g0 = icp_gradient(corrs, apply_increment(xt, base));
  CHECK(norm6(g0) == 0.0);
}
TEST("icp: linearized one-shot and damped Newton (test_icp.cpp:232-266)") {
  const Pose base = reference_pose(1.1);
  const Vec6<double> xs{1.2e-3, -0.8e-3, 0.9e-3, 0.7e-3, -1.1e-3, 0.6e-3};
  const auto small_set = synthetic_corrs(21, 400, base, xs);
  for (bool seq : {true, false}) {
    const auto one = linearized_step(small_set, base, seq);
    Vec6<double> d;
    for (int i = 0; i < 6; ++i) d[i] = one[i] - xs[i];
    CHECK(norm6(d) < 5e-6);
  }
  const Vec6<double> xt{0.05, -0.04, 0.03, 0.04, -0.03, 0.05};
  const auto corrs = synthetic_corrs(23, 400, base, xt);
  const Pose target = apply_increment(xt, base);
  Pose pose = base;
  double lambda = 1e-6;
  for (int it = 0; it < 10; ++it) {
    const double l0 = icp_loss(corrs, pose);
    const auto g = icp_gradient(corrs, pose);
    const auto h = icp_hessian(corrs, pose);
    const auto delta = levenberg_newton_step(g, h, l0, [&](const Vec6<double>& d) { return icp_energy(corrs, d, pose); },
                                             lambda, LineSearchConfig());
    pose = apply_increment(delta, pose);
    if (norm6(delta) < 1e-12) break;
  }
  CHECK(icp_loss(corrs, pose) < 1e-18 && terr(pose, target) < 1e-8 && rerr_deg(pose, target) < 1e-7);
}
TEST("icp: first-order steppers deterministic (test_icp.cpp:268-321)") {
  const Pose base = reference_pose(2.0);
  const Vec6<double> xt{0.02, -0.015, 0.02, 0.015, -0.01, 0.015};
  const auto corrs = synthetic_corrs(31, 300, base, xt);
  auto run = [&](GradientStepper::Kind kind, int iters, std::vector<Pose>* trail) {
    GradientStepper st(kind, 6);
    Pose pose = base;
    double last = icp_loss(corrs, pose);
    for (int it = 0; it < iters; ++it) {
      const auto g = icp_gradient(corrs, pose);
      const auto dir = st.propose(g);
      const double slope = dot6(g, dir);
      if (!(slope < 0.0)) return -1.0;
      const auto r = backtracking_search(
          [&](double a) { Vec6<double> d; for (int i = 0; i < 6; ++i) d[i] = a * dir[i]; return icp_energy(corrs, d, pose); },
          last, slope, LineSearchConfig());
      if (!r.ok || !(r.loss < last)) return -1.0;
      Vec6<double> step;
      for (int i = 0; i < 6; ++i) step[i] = r.alpha * dir[i];
      pose = apply_increment(step, pose);
      last = r.loss;
      if (trail) trail->push_back(pose);
    }
    return last;
  };
  const double initial = icp_loss(corrs, base);
  const double gd = run(GradientStepper::Kind::kGradientDescent, 60, nullptr);
  const double ncg = run(GradientStepper::Kind::kConjugateGradient, 60, nullptr);
  CHECK(gd >= 0 && gd < initial / 100.0);
  CHECK(ncg >= 0 && ncg < initial / 100.0 && ncg <= gd);
  std::vector<Pose> a, b;
  run(GradientStepper::Kind::kGradientDescent, 20, &a);
  run(GradientStepper::Kind::kGradientDescent, 20, &b);
  bool same = a.size() == b.size();
  for (std::size_t i = 0; same && i < a.size(); ++i)
    same = mat_diff(a[i].rotation, b[i].rotation) == 0.0 && norm(a[i].translation - b[i].translation) == 0.0;
  CHECK(same);
}
struct TrackFixture {
  Scene scene;
  Intrinsics k = small_camera();
  TsdfVolumeT<Complex> volume{VolumeParams::cube(72, 0.026, Vec3d(-0.7, -0.8, -0.33))};
  Pose frame_pose;
  Image<double> frame_depth;
  TrackFixture() {
    scene.planes.push_back({Vec3d(0, 0, 1), 0.0});
    scene.spheres.push_back({Vec3d(0.0, 0.1, 0.55), 0.5});
    scene.spheres.push_back({Vec3d(0.85, 0.55, 0.3), 0.3});
    const Vec3d target(0.25, 0.15, 0.35);
    for (int i = 0; i < 8; ++i) {
      const Pose p = orbit_pose(target, 1.9, 1.4, 2.0 * M_PI * i / 8);
      surface_update(volume, complex_depth(render_depth(scene, p, k)), pose_cast<Complex>(p), k);
    }
    frame_pose = orbit_pose(target, 1.9, 1.4, 0.39);
    frame_depth = render_depth(scene, frame_pose, k);
  }
};
const TrackFixture& track_fixture() {
  static TrackFixture f;
  return f;
}
TEST("icp: track_frame refines a perturbed pose, bit-identical rerun (test_icp.cpp:323-370)") {
  const TrackFixture& fx = track_fixture();
  const Pose init = apply_increment(Vec6<double>{0.03, -0.02, 0.02, 0.02, -0.015, 0.015}, fx.frame_pose);
  CHECK(terr(init, fx.frame_pose) > 0.02);
  IcpConfig cfg;
  std::vector<TraceRow> trace;
  const TrackResult res = track_frame(fx.volume, fx.frame_depth, init, fx.k, cfg, &trace);
  CHECK(res.iterations > 0 && res.converged && res.correspondences > 500);
  CHECK(terr(res.pose, fx.frame_pose) < 0.008 && rerr_deg(res.pose, fx.frame_pose) < 0.15 && res.final_loss < 2e-5);
  CHECK(trace.size() == std::size_t(res.iterations) && trace.back().loss < trace.front().loss);
  const TrackResult again = track_frame(fx.volume, fx.frame_depth, init, fx.k, cfg);
  CHECK(mat_diff(again.pose.rotation, res.pose.rotation) == 0.0 && norm(again.pose.translation - res.pose.translation) == 0.0);
}
TEST("icp: every solver family improves the pose (test_icp.cpp:372-405)") {
  const TrackFixture& fx = track_fixture();
  const Pose init = apply_increment(Vec6<double>{0.03, -0.02, 0.02, 0.02, -0.015, 0.015}, fx.frame_pose);
  const double t0 = terr(init, fx.frame_pose);
  IcpConfig cfg;
  cfg.solver = IcpSolver::kLinearized;
  for (bool canon : {true, false}) {
    const auto lin = track_frame(fx.volume, fx.frame_depth, init, fx.k, cfg, nullptr, canon);
    CHECK(terr(lin.pose, fx.frame_pose) < 0.008 && rerr_deg(lin.pose, fx.frame_pose) < 0.15);
  }
  cfg.solver = IcpSolver::kGradientDescent;
  CHECK(terr(track_frame(fx.volume, fx.frame_depth, init, fx.k, cfg).pose, fx.frame_pose) < t0 / 2.0);
  cfg.solver = IcpSolver::kConjugateGradient;
  CHECK(terr(track_frame(fx.volume, fx.frame_depth, init, fx.k, cfg).pose, fx.frame_pose) < t0 / 2.0);
  cfg.level_iterations = {30, 20, 15};
  CHECK(terr(track_frame(fx.volume, fx.frame_depth, init, fx.k, cfg).pose, fx.frame_pose) < 0.008);
}

// -------------------------------------------------------------- synth -----
TEST("synth: primitives, normals, orbit, gaussian (test_synth.cpp:30-181)") {
  Scene s;
  s.spheres.push_back({Vec3d(), 0.5});
  CHECK(approx(s.signed_distance(Vec3d(1, 0, 0)), 0.5, 1e-12) && approx(s.signed_distance(Vec3d()), -0.5, 1e-12));
  Scene b;
  b.boxes.push_back({Vec3d(), Vec3d(1, 1, 1)});
  CHECK(approx(b.signed_distance(Vec3d(2, 2, 0)), std::sqrt(2.0), 1e-12) && approx(b.signed_distance(Vec3d(0.5, 0, 0)), -0.5, 1e-12));
  Scene u;
  u.spheres.push_back({Vec3d(0, 0, 1), 0.5});
  u.planes.push_back({Vec3d(0, 0, 1), 0.0});
  CHECK(approx(u.signed_distance(Vec3d(0, 0, 0.4)), 0.1, 1e-12) && approx(u.signed_distance(Vec3d(3, 0, 0.4)), 0.4, 1e-12));
  CHECK(norm(u.normal(Vec3d(0.7, 0, 1)) - Vec3d(1, 0, 0)) < 1e-6);
  const Vec3d target(0.2, -0.1, 0.5);
  for (double a : {0.0, 1.1, 3.0, 5.5}) {
    const Pose p = orbit_pose(target, 2.0, 1.2, a);
    const Mat3d rrt = p.rotation * transpose(p.rotation);
    CHECK(mat_diff(rrt, Mat3d::identity()) < 1e-12);
    const Vec3d fwd = normalized(target - p.translation);
    CHECK(norm(Vec3d(p.rotation(0, 2), p.rotation(1, 2), p.rotation(2, 2)) - fwd) < 1e-12);
  }
  GaussianSource g1(5), g2(5);
  bool same = true;
  double m = 0, v = 0;
  for (int i = 0; i < 20000; ++i) {
    const double a = g1.next();
    same = same && a == g2.next();
    m += a;
    v += a * a;
  }
  m /= 20000;
  v = v / 20000 - m * m;
  CHECK(same && std::fabs(m) < 0.03 && std::fabs(v - 1.0) < 0.05);
  // rendered sphere vs analytic (test_synth.cpp:81-115)
  const Intrinsics k = small_camera();
  Scene sp;
  sp.spheres.push_back({Vec3d(0, 0, 3), 1.0});
  const auto d = render_depth(sp, Pose::identity(), k);
  const double dz = d.at(80, 60);
  CHECK(dz > 0.0);
  const Vec3d ray((80 - k.cx) / k.fx, (60 - k.cy) / k.fy, 1.0);
  const Vec3d hitp = dz * ray;
  CHECK(std::fabs(norm(hitp - Vec3d(0, 0, 3)) - 1.0) < 1e-5);
}

// ------------------------------------------- builder-defined pieces -----
TEST("hashed: chains sorted, find/insert consistent, occupancy order-free") {
  HashParams hp;
  hp.bucket_bits = 4;  // force long chains
  HashedVolumeT<double> a(hp), b(hp);
  std::vector<std::array<int, 3>> keys;
  auto g = rng(5);
  for (int i = 0; i < 300; ++i) keys.push_back({int(uni(g, -50, 50)), int(uni(g, -50, 50)), int(uni(g, -50, 50))});
  for (auto& kk : keys)
    if (a.find(kk[0], kk[1], kk[2]) < 0) a.insert(kk[0], kk[1], kk[2]);
  bool ok = true;
  for (auto& kk : keys) ok = ok && a.find(kk[0], kk[1], kk[2]) >= 0;
  CHECK(ok);
  for (std::size_t h = 0; h < a.heads.size(); ++h)
    for (int e = a.heads[h]; e >= 0 && a.next[e] >= 0; e = a.next[e]) ok = ok && a.keys[e] < a.keys[a.next[e]];
  CHECK(ok);
  CHECK(a.find(1000, 0, 0) < 0);
  // same key set in another order gives the same chains (as key sequences)
  for (auto it = keys.rbegin(); it != keys.rend(); ++it)
    if (b.find((*it)[0], (*it)[1], (*it)[2]) < 0) b.insert((*it)[0], (*it)[1], (*it)[2]);
  for (std::size_t h = 0; h < a.heads.size(); ++h) {
    std::vector<uint64_t> ca, cb;
    for (int e = a.heads[h]; e >= 0; e = a.next[e]) ca.push_back(a.keys[e]);
    for (int e = b.heads[h]; e >= 0; e = b.next[e]) cb.push_back(b.keys[e]);
    ok = ok && ca == cb;
  }
  CHECK(ok);
}
TEST("hashed: fusion equals dense fusion on allocated voxels") {
  const Intrinsics k = small_camera();
  Scene scene;
  scene.spheres.push_back({Vec3d(0, 0, 0), 0.5});
  const Pose p = orbit_pose(Vec3d(), 1.6, 0.8, 0.3);
  const Image<double> depth = render_depth(scene, p, k);
  HashParams hp;
  hp.voxel_size = 0.02;
  hp.mu = 0.1;
  hp.origin = Vec3d(-0.64, -0.64, -0.64);
  HashedVolumeT<Complex> hv(hp);
  AllocStats st;
  const auto vis = allocate_band(hv, depth, k, p, &st);
  surface_update_blocks(hv, vis, depth, pose_cast<Complex>(p), k);
  VolumeParams vp = VolumeParams::cube(64, 0.02, hp.origin);
  vp.mu = 0.1;
  TsdfVolumeT<Complex> dv(vp);
  surface_update(dv, depth, pose_cast<Complex>(p), k);
  CHECK(st.fresh > 50 && st.touched == st.fresh);
  bool ok = true;
  int compared = 0;
  for (int b = 0; b < hv.n_blocks(); ++b)
    for (int l = 0; l < 512; ++l) {
      const int i = 8 * hv.coords[3 * b] + (l & 7), j = 8 * hv.coords[3 * b + 1] + ((l >> 3) & 7),
                kk = 8 * hv.coords[3 * b + 2] + (l >> 6);
      if (i < 0 || j < 0 || kk < 0 || i >= 64 || j >= 64 || kk >= 64) continue;
      const std::size_t di = dv.index(i, j, kk), hi = std::size_t(b) * 512 + l;
      ok = ok && dv.tsdf[di].re == hv.tsdf[hi].re && dv.weight[di] == hv.weight[hi];
      ++compared;
    }
  CHECK(ok && compared > 10000);
  // raycast of the hashed volume sees the sphere
  const auto maps = raycast<double>(hv, p, k);
  int hits = 0;
  double worst = 0;
  for (std::size_t i = 0; i < maps.vertices.data.size(); ++i)
    if (normal_valid(maps.normals.data[i])) {
      ++hits;
      worst = std::max(worst, std::fabs(norm(maps.vertices.data[i]) - 0.5));
    }
  CHECK(hits > 1000 && worst < 0.03);
}
TEST("pipeline: packed channels == single-direction passes") {
  // reduced config-1 style run: 4 frames at 80x60, 64^3 volume
  Workload w = make_workload(1, 4, 80, 60);
  PipelineConfig cfg;
  cfg.hashed = false;
  cfg.dense = VolumeParams::cube(64, 0.04, Vec3d(-2.1, -1.28, -0.1));
  cfg.dense.mu = 0.12;
  cfg.k = w.k;
  cfg.icp.solver = IcpSolver::kLinearized;
  cfg.h = 1e-20;
  cfg.directions = {0, 4, 6};
  const PipelineResult packed = run_pipeline<3>(cfg, w.frames, w.gt);
  bool same = true;
  for (int d = 0; d < 3; ++d) {
    PipelineConfig c1 = cfg;
    c1.directions = {cfg.directions[d]};
    const PipelineResult one = run_pipeline<1>(c1, w.frames, w.gt);
    same = same && one.gradient[0] == packed.gradient[d] && one.objective == packed.objective;
  }
  CHECK(same);
}

// CSFD of the whole frame loop against a central finite difference of real
// reruns with the seed moved by +-eps (the objective keeps the unshifted
// ground truth), wherever the +-eps runs take every discrete decision of the
// unperturbed run (iterations, correspondences, blocks, visible, converged,
// fused voxels per frame).  Dense volumes: the camera sits inside the volume
// box, so the raycast starts at near_clip for every pose (tsdf.hpp:234-254):
// the reference's alpha is a double, so CSFD differentiates with the sample
// positions along each ray held fixed, and a slab entry that moves with the
// pose (camera outside the box) would shift every sample and make FD and
// CSFD differ by that (non-differentiable) resampling term.  Hashed volumes
// have no slab (alpha starts at near_clip).
template <typename VL, typename VR>
void csfd_vs_fd(const char* what, VL make_vol, VR make_vol_real, const PipelineConfig& cfg, const Workload& w,
                double tol) {
  using S = Lifted<6>;
  auto vol = make_vol();
  // a generic base point: the synthetic first pose is exactly on the orbit,
  // where voxel centres / pixel centres can tie with a threshold (ifloor at an
  // integer, a zero crossing exactly on a sample) and any perturbation flips
  // a decision; a small fixed twist moves the seed off those ties
  const double base[6] = {0.0031, -0.0017, 0.0023, 0.0011, -0.0029, 0.0007};
  Vec6<S> xi;
  for (int i = 0; i < 6; ++i) {
    xi[i] = S(base[i]);
    xi[i].im[i] = cfg.h;
  }
  const LiftedRun<S> lifted = run_lifted<S>(vol, cfg, w.frames, w.gt, xi, lift_intrinsics<S>(cfg.k));
  const double eps = 1e-9;  // larger steps cross kinks of the piecewise-smooth loop (C0 trilinear cells)
  auto same_decisions = [&](const LiftedRun<double>& r) {
    return r.iterations == lifted.iterations && r.correspondences == lifted.correspondences &&
           r.blocks == lifted.blocks && r.visible == lifted.visible && r.converged == lifted.converged &&
           r.fused == lifted.fused;
  };
  double worst = 0.0;
  int compared = 0;
  for (int d = 0; d < 6; ++d) {
    double f[2];
    bool ok = true;
    for (int sgn = 0; sgn < 2; ++sgn) {
      auto v = make_vol_real();
      Vec6<double> x{};
      for (int i = 0; i < 6; ++i) x[i] = base[i];
      x[d] = x[d] + (sgn ? -eps : eps);
      const LiftedRun<double> r = run_lifted<double>(v, cfg, w.frames, w.gt, x, lift_intrinsics<double>(cfg.k));
      if (!same_decisions(r))
        for (std::size_t fr = 0; fr < r.iterations.size(); ++fr)
          if (r.iterations[fr] != lifted.iterations[fr] || r.correspondences[fr] != lifted.correspondences[fr] ||
              r.fused[fr] != lifted.fused[fr] || r.visible[fr] != lifted.visible[fr])
            std::printf("      frame %zu: it %d/%d corr %d/%d fused %d/%d visible %d/%d\n", fr, r.iterations[fr],
                        lifted.iterations[fr], r.correspondences[fr], lifted.correspondences[fr], r.fused[fr],
                        lifted.fused[fr], r.visible[fr], lifted.visible[fr]);
      ok = ok && same_decisions(r);
      f[sgn] = r.objective;
    }
    const double fd = (f[0] - f[1]) / (2.0 * eps);
    const double cs = lifted.objective.im[d] / cfg.h;
    const double rel = std::fabs(fd - cs) / std::max(std::fabs(cs), 1e-3 * std::fabs(lifted.objective.re) + 1e-12);
    std::printf("    %s d%d: CSFD %.10g FD %.10g rel %.2e%s\n", what, d, cs, fd, rel, ok ? "" : " (decisions moved)");
    if (ok) {
      worst = std::max(worst, rel);
      ++compared;
    }
  }
  CHECK(compared == 6);
  CHECK(worst <= tol);
}

TEST("pipeline: CSFD gradient vs central FD, hashed (config-2 scene, 160x120, 3 frames)") {
  const Workload w = make_workload(2, 3, 160, 120);
  PipelineConfig cfg;
  cfg.hashed = true;
  cfg.hash = config2_hash();
  cfg.hash.voxel_size = 0.02;
  cfg.hash.mu = 0.1;
  cfg.hash.max_blocks = 1 << 16;
  cfg.k = w.k;
  cfg.h = 1e-8;
  cfg.objective = Objective::kTrajectoryError;
  csfd_vs_fd("hashed", [&] { return HashedVolumeT<Lifted<6>>(cfg.hash); },
             [&] { return HashedVolumeT<double>(cfg.hash); }, cfg, w, 1e-5);
}

TEST("pipeline: CSFD gradient vs central FD, dense with the camera inside the box (config-1 scene, 80x60)") {
  const Workload w = make_workload(1, 3, 80, 60);
  PipelineConfig cfg;
  cfg.hashed = false;
  cfg.dense = VolumeParams::cube(64, 0.04, Vec3d(-1.28, -1.28, -0.1));  // contains the 1 m orbit at z = 1.4
  cfg.dense.mu = 0.12;
  cfg.k = w.k;
  cfg.h = 1e-20;
  cfg.objective = Objective::kFinalTranslationError;
  csfd_vs_fd("dense", [&] { return TsdfVolumeT<Lifted<6>>(cfg.dense); },
             [&] { return TsdfVolumeT<double>(cfg.dense); }, cfg, w, 1e-5);
}

}  // namespace
}  // namespace orc

using orc::registry;
using orc::g_case;
using orc::g_fail;
using orc::g_checks;
using orc::Case;

int main(int argc, char** argv) {
  const char* filter = argc > 1 ? argv[1] : nullptr;
  int ran = 0;
  for (const Case& c : registry()) {
    if (filter && !std::strstr(c.name, filter)) continue;
    g_case = c.name;
    const int before = g_fail;
    try {
      c.fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::printf("  EXCEPTION [%s]: %s\n", c.name, e.what());
    }
    std::printf("%s %s\n", g_fail == before ? "ok  " : "FAIL", c.name);
    ++ran;
  }
  std::printf("KAT summary: cases=%d checks=%d failures=%d\n", ran, g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
