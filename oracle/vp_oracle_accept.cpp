// vp_oracle_accept.cpp -- independent high-accuracy quadrature for the
// SPEC's acceptance checks of the near-field model.
//
// TEST INFRASTRUCTURE ONLY (see vp_oracle.h).  The near-field soundness
// sweep (PAPER.md Figs. nf0/nf1/nf2) compares, at points
// the model classifies "far", the far rule's value of
//     I_T(x) = int_T log|x - y| f(y) dA_y
// (the quantity whose error the model bounds by eps)
// with this adaptive oracle: recursive 4-way midpoint subdivision of T with
// a fixed order-30 collapsed Gauss-Jacobi rule (256 nodes, exact to degree
// 30) in long double, refined where the four children disagree with their
// parent.  "oracle = recursive subdivision quadrature to 1e-15".
#include <omp.h>

#include <cmath>
#include <cstdint>
#include <vector>

#include "vp_oracle.h"

namespace {

struct Rule {
  std::vector<long double> x, y, w;
};

const Rule& rule30() {
  static Rule R = [] {
    Rule r;
    int len = 0;
    vpo_simplex_rule(30, &len, nullptr, nullptr, nullptr);
    std::vector<double> x(len), y(len), w(len);
    vpo_simplex_rule(30, &len, x.data(), y.data(), w.data());
    r.x.assign(x.begin(), x.end());
    r.y.assign(y.begin(), y.end());
    r.w.assign(w.begin(), w.end());
    return r;
  }();
  return R;
}

// f at the physical point y, or (kind 3) the Koornwinder expansion at the
// reference coordinates of the element
struct Density {
  int kind;
  int p;
  const double* coeffs;
  long double x0, y0, e1x, e1y, e2x, e2y, det;
  long double operator()(long double x, long double y) const {
    switch (kind) {
      case 0: return 1.0L;
      case 1: return std::sin(x + 2.0L * y);
      case 2: return std::exp(-x * x - y * y);
      default: {
        // inverse affine map, then the expansion (double basis evaluation)
        const long double dx = x - x0, dy = y - y0;
        const long double xi = (e2y * dx - e2x * dy) / det, eta = (-e1y * dx + e1x * dy) / det;
        double k[(32 + 1) * (32 + 2) / 2];
        vpo_koornwinder(p, (double)xi, (double)eta, k);
        long double s = 0.0L;
        for (int j = 0; j < (p + 1) * (p + 2) / 2; ++j) s += (long double)coeffs[j] * k[j];
        return s;
      }
    }
  }
};

long double tri_rule(const long double a[2], const long double b[2], const long double c[2], long double tx,
                     long double ty, const Density& f) {
  const Rule& R = rule30();
  const long double e1x = b[0] - a[0], e1y = b[1] - a[1], e2x = c[0] - a[0], e2y = c[1] - a[1];
  const long double det = std::fabs(e1x * e2y - e2x * e1y);
  long double s = 0.0L;
  for (size_t i = 0; i < R.w.size(); ++i) {
    const long double x = a[0] + R.x[i] * e1x + R.y[i] * e2x, y = a[1] + R.x[i] * e1y + R.y[i] * e2y;
    const long double dx = tx - x, dy = ty - y;
    s += R.w[i] * f(x, y) * 0.5L * std::log(dx * dx + dy * dy);
  }
  return s * det;
}

long double adapt(const long double a[2], const long double b[2], const long double c[2], long double tx,
                  long double ty, const Density& f, long double whole, long double tol, int depth) {
  long double mab[2] = {(a[0] + b[0]) * 0.5L, (a[1] + b[1]) * 0.5L};
  long double mbc[2] = {(b[0] + c[0]) * 0.5L, (b[1] + c[1]) * 0.5L};
  long double mca[2] = {(c[0] + a[0]) * 0.5L, (c[1] + a[1]) * 0.5L};
  const long double* ch[4][3] = {{a, mab, mca}, {mab, b, mbc}, {mca, mbc, c}, {mbc, mca, mab}};
  long double part[4], sum = 0.0L;
  for (int k = 0; k < 4; ++k) {
    part[k] = tri_rule(ch[k][0], ch[k][1], ch[k][2], tx, ty, f);
    sum += part[k];
  }
  if (depth >= 40 || std::fabs(sum - whole) <= tol) return sum;
  long double s = 0.0L;
  for (int k = 0; k < 4; ++k) s += adapt(ch[k][0], ch[k][1], ch[k][2], tx, ty, f, part[k], tol * 0.5L, depth + 1);
  return s;
}

}  // namespace

extern "C" {

// Adaptive I_T(x) = int_T log|x - y| f(y) dA for points x outside T.
// tri = (ax, ay, bx, by, cx, cy); fkind 0: 1, 1: sin(x + 2y), 2: exp(-x^2 -
// y^2), 3: sum_j coeffs[j] K_j(xi, eta) (order p, reference coordinates of
// T).  tol: absolute tolerance of the subdivision (1e-17 scale).
int vpo_adaptive_log_integral(const double* tri, int fkind, int p, const double* coeffs, int64_t n,
                              const double* pts, double tol, int nthreads, double* out) {
  if (!tri || !pts || !out || n < 0 || fkind < 0 || fkind > 3 || (fkind == 3 && (!coeffs || p < 0 || p > 32)))
    return 1;
  rule30();  // build once before the parallel region
  Density f{fkind, p, coeffs, tri[0], tri[1], tri[2] - tri[0], tri[3] - tri[1], tri[4] - tri[0], tri[5] - tri[1], 0};
  f.det = f.e1x * f.e2y - f.e2x * f.e1y;
  const long double a[2] = {tri[0], tri[1]}, b[2] = {tri[2], tri[3]}, c[2] = {tri[4], tri[5]};
#pragma omp parallel for schedule(dynamic, 4) num_threads(nthreads > 0 ? nthreads : omp_get_max_threads())
  for (int64_t i = 0; i < n; ++i) {
    const long double tx = pts[2 * i], ty = pts[2 * i + 1];
    const long double whole = tri_rule(a, b, c, tx, ty, f);
    out[i] = (double)adapt(a, b, c, tx, ty, f, whole, (long double)tol, 0);
  }
  return 0;
}

}  // extern "C"
