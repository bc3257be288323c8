// vp_setup.cpp -- host setup: rules, synthetic configurations, density
// coefficients (see include/vp_setup.h for the contract and anchors).
#include "vp_setup.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "koorn.cuh"

namespace {

constexpr double kPi = 3.14159265358979323846;

std::mutex g_mu;
std::string g_err;
int fail(int code, const std::string& m) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_err = m;
  return code;
}

template <class F>
void parallel_for(int64_t n, F&& f) {
  unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  if (n < 4096 || nt == 1) {
    for (int64_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::vector<std::thread> th;
  const int64_t chunk = (n + nt - 1) / nt;
  for (unsigned k = 0; k < nt; ++k) {
    const int64_t lo = k * chunk, hi = std::min(n, lo + chunk);
    if (lo >= hi) break;
    th.emplace_back([lo, hi, &f] {
      for (int64_t i = lo; i < hi; ++i) f(i);
    });
  }
  for (auto& t : th) t.join();
}

double legendre(int n, double x) {
  if (n == 0) return 1.0;
  double p0 = 1.0, p1 = x;
  for (int k = 1; k < n; ++k) {
    const double p2 = ((2 * k + 1) * x * p1 - k * p0) / (k + 1);
    p0 = p1;
    p1 = p2;
  }
  return p1;
}
double dlegendre(int n, double x) {
  if (n == 0) return 0.0;
  return n * (legendre(n - 1, x) - x * legendre(n, x)) / (1.0 - x * x);
}

// Gauss-Legendre by Newton on the three-term recurrence (gauss.hpp:17-46).
void gl_rule(int n, double* x, double* w) {
  for (int i = 0; i < (n + 1) / 2; ++i) {
    double z = std::cos(kPi * (i + 0.75) / (n + 0.5));
    double dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = z;
      for (int k = 1; k < n; ++k) {
        const double p2 = ((2 * k + 1) * z * p1 - k * p0) / (k + 1);
        p0 = p1;
        p1 = p2;
      }
      dp = n * (z * p1 - p0) / (z * z - 1.0);
      const double dz = p1 / dp;
      z -= dz;
      if (std::abs(dz) < 1e-15) break;
    }
    x[i] = -z;
    x[n - 1 - i] = z;
    const double ww = 2.0 / ((1.0 - z * z) * dp * dp);
    w[i] = ww;
    w[n - 1 - i] = ww;
  }
  if (n % 2 == 1) x[n / 2] = 0.0;
}

// Jacobi P_n^{(1,0)} and derivative on [-1,1].
void jacobi10(int n, double x, double& p, double& dp) {
  const double al = 1.0, be = 0.0;
  double p0 = 1.0, p1 = (al + 1.0) + (al + be + 2.0) * (x - 1.0) * 0.5;
  if (n == 0) {
    p = 1.0;
    dp = 0.0;
    return;
  }
  for (int k = 2; k <= n; ++k) {
    const double s = 2.0 * k + al + be;
    const double a1 = 2.0 * k * (k + al + be) * (s - 2.0);
    const double a2 = (s - 1.0) * (s * (s - 2.0) * x + al * al - be * be);
    const double a3 = 2.0 * (k + al - 1.0) * (k + be - 1.0) * s;
    const double p2 = (a2 * p1 - a3 * p0) / a1;
    p0 = p1;
    p1 = p2;
  }
  p = p1;
  const double s = 2.0 * n + al + be;
  dp = (n * ((al - be) - s * x) * p1 + 2.0 * (n + al) * (n + be) * p0) / (s * (1.0 - x * x));
}

// Gauss-Jacobi (alpha=1, beta=0): eigenvalues of the Jacobi matrix by Sturm
// bisection, Newton polish, weights 4/((1-x^2) P_n'(x)^2) on [-1,1].
void gj10_rule(int n, double* x01, double* w01) {
  const double al = 1.0, be = 0.0;
  std::vector<double> a(n), b2(n, 0.0);
  for (int k = 0; k < n; ++k) {
    const double s = 2.0 * k + al + be;
    a[k] = (be * be - al * al) / (s * (s + 2.0));
    if (k >= 1) b2[k] = 4.0 * k * (k + al) * (k + be) * (k + al + be) / (s * s * (s + 1.0) * (s - 1.0));
  }
  auto count_below = [&](double lam) {
    int c = 0;
    double d = a[0] - lam;
    if (d < 0) ++c;
    for (int k = 1; k < n; ++k) {
      if (d == 0.0) d = 1e-300;
      d = (a[k] - lam) - b2[k] / d;
      if (d < 0) ++c;
    }
    return c;
  };
  for (int i = 0; i < n; ++i) {
    double lo = -1.0, hi = 1.0;
    for (int it = 0; it < 200 && hi - lo > 1e-17; ++it) {
      const double mid = 0.5 * (lo + hi);
      if (count_below(mid) > i) hi = mid; else lo = mid;
    }
    double z = 0.5 * (lo + hi), p, dp;
    for (int it = 0; it < 5; ++it) {
      jacobi10(n, z, p, dp);
      const double dz = p / dp;
      z -= dz;
      if (std::abs(dz) < 1e-16) break;
    }
    jacobi10(n, z, p, dp);
    const double w = 4.0 / ((1.0 - z * z) * dp * dp);
    x01[i] = 0.5 * (1.0 + z);
    w01[i] = 0.25 * w;  // int_0^1 (1-u) g(u) du
  }
}

// small dense solve with partial pivoting, A row-major n x n, overwrites b
bool dense_solve(int n, std::vector<double> A, std::vector<double>& b) {
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r)
      if (std::abs(A[r * n + c]) > std::abs(A[piv * n + c])) piv = r;
    if (A[piv * n + c] == 0.0) return false;
    if (piv != c) {
      for (int k = 0; k < n; ++k) std::swap(A[c * n + k], A[piv * n + k]);
      std::swap(b[c], b[piv]);
    }
    for (int r = c + 1; r < n; ++r) {
      const double f = A[r * n + c] / A[c * n + c];
      if (f == 0.0) continue;
      for (int k = c; k < n; ++k) A[r * n + k] -= f * A[c * n + k];
      b[r] -= f * b[c];
    }
  }
  for (int c = n - 1; c >= 0; --c) {
    double s = b[c];
    for (int k = c + 1; k < n; ++k) s -= A[c * n + k] * b[k];
    b[c] = s / A[c * n + c];
  }
  return true;
}

}  // namespace

extern "C" {

const char* vps_last_error(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  return g_err.c_str();
}

int vps_koorn_size(int p) { return vp::koorn_size(p); }

int vps_gauss_legendre(int n, double* x, double* w) {
  if (n < 1 || !x || !w) return fail(1, "gauss_legendre: order must be >= 1");
  gl_rule(n, x, w);
  return 0;
}

int vps_gauss_jacobi10(int n, double* x, double* w) {
  if (n < 1 || !x || !w) return fail(1, "gauss_jacobi: order must be >= 1");
  gj10_rule(n, x, w);
  return 0;
}

int vps_simplex_rule(int order, int* len, double* x, double* y, double* w) {
  if (order < 0 || order > 200 || !len) return fail(1, "simplex_rule: order out of range");
  const int n = order / 2 + 1;  // 2n-1 >= order in each collapsed direction
  *len = n * n;
  if (!x) return 0;
  std::vector<double> gx(n), gw(n), lx(n), lw(n);
  gj10_rule(n, gx.data(), gw.data());
  gl_rule(n, lx.data(), lw.data());
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      const double u = gx[i], v = 0.5 * (1.0 + lx[j]);
      x[i * n + j] = u;
      y[i * n + j] = v * (1.0 - u);
      w[i * n + j] = gw[i] * (0.5 * lw[j]);
    }
  return 0;
}

// Fully symmetric rules computed by this repository's own moment-fitting solver
// (tools/make_sym_rules.py -> sym_rules.inc): positive weights, interior
// points, exact to the stated degree with about two thirds of the points of
// the collapsed Gauss-Jacobi rule (degree 12: 33 against 49), i.e. the point
// counts of the Xiao-Gimbutas tables the SPEC names (rules.hpp:121-125),
// which are third-party data and absent.
namespace {
struct SymRule {
  int degree, n1, n21, n111, points;
  double p[64];
};
const SymRule kSymRules[] = {
#include "sym_rules.inc"
};
const SymRule* sym_rule_for(int order) {
  for (const SymRule& r : kSymRules)
    if (r.degree == order) return &r;
  return nullptr;
}
}  // namespace

// The evaluation's far / near rule of a given order (load_far_rule, rules.hpp:
// 121-125): the symmetric rule of that degree where one is tabulated, the
// collapsed Gauss-Jacobi rule otherwise.
int vps_quad_rule(int order, int* len, double* x, double* y, double* w) {
  const SymRule* r = sym_rule_for(order);
  if (!r) return vps_simplex_rule(order, len, x, y, w);
  if (!len) return fail(1, "quad_rule: len is null");
  *len = r->points;
  if (!x) return 0;
  if (!y || !w) return fail(1, "quad_rule: null output array");
  int n = 0, k = 0;
  if (r->n1) {
    x[n] = 1.0 / 3.0; y[n] = 1.0 / 3.0; w[n] = r->p[k++]; ++n;
  }
  for (int i = 0; i < r->n21; ++i) {
    const double wi = r->p[k], a = r->p[k + 1], c = 1.0 - 2.0 * a;
    k += 2;
    const double px[3] = {a, a, c}, py[3] = {a, c, a};
    for (int j = 0; j < 3; ++j, ++n) { x[n] = px[j]; y[n] = py[j]; w[n] = wi; }
  }
  for (int i = 0; i < r->n111; ++i) {
    const double wi = r->p[k], a = r->p[k + 1], b = r->p[k + 2], c = 1.0 - a - b;
    k += 3;
    const double px[6] = {a, b, a, c, b, c}, py[6] = {b, a, c, a, c, b};
    for (int j = 0; j < 6; ++j, ++n) { x[n] = px[j]; y[n] = py[j]; w[n] = wi; }
  }
  return 0;
}

// Radial GGQ by moment fitting (restating ggq.hpp:33-182): unknowns r_j and
// log w_j; Levenberg-Marquardt from GL^alpha guesses, then damped Newton.
int vps_ggq(int ng, double* rout, double* wout, double* max_residual) {
  if (ng < 0 || ng > 20 || !rout || !wout) return fail(1, "ggq: order must be in [0, 20]");
  const int nq = ng + 1, ne = 2 * nq;
  std::vector<double> b(nq, 0.0), c(nq, 0.0);
  {
    const int ngl = ng + 4;
    std::vector<double> gx(ngl), gw(ngl);
    gl_rule(ngl, gx.data(), gw.data());
    for (int n = 0; n <= ng; ++n)
      for (int i = 0; i < ngl; ++i) {
        const double r = 0.5 * (1.0 + gx[i]);
        b[n] += 0.5 * gw[i] * r * legendre(n, 2 * r - 1);
      }
    std::vector<double> hx(24), hw(24);
    gl_rule(24, hx.data(), hw.data());
    for (int k = 0; k < 80; ++k) {
      const double hi = std::ldexp(1.0, -k), lo = 0.5 * hi;
      for (int i = 0; i < 24; ++i) {
        const double r = 0.5 * (lo + hi) + 0.5 * (hi - lo) * hx[i];
        const double ww = 0.5 * (hi - lo) * hw[i];
        for (int n = 0; n <= ng; ++n) c[n] += ww * r * std::log(r) * legendre(n, 2 * r - 1);
      }
    }
  }
  auto residual = [&](const std::vector<double>& r, const std::vector<double>& lw,
                      std::vector<double>& res) {
    res.assign(ne, 0.0);
    for (int n = 0; n <= ng; ++n) {
      double s0 = 0.0, s1 = 0.0;
      for (int j = 0; j < nq; ++j) {
        const double w = std::exp(lw[j]), p = legendre(n, 2 * r[j] - 1);
        s0 += w * r[j] * p;
        s1 += w * r[j] * std::log(r[j]) * p;
      }
      res[2 * n] = s0 - b[n];
      res[2 * n + 1] = s1 - c[n];
    }
  };
  auto jacobian = [&](const std::vector<double>& r, const std::vector<double>& lw,
                      std::vector<double>& J) {
    J.assign(ne * ne, 0.0);
    for (int n = 0; n <= ng; ++n)
      for (int j = 0; j < nq; ++j) {
        const double w = std::exp(lw[j]), rr = r[j], lr = std::log(rr);
        const double p = legendre(n, 2 * rr - 1), dp = 2 * dlegendre(n, 2 * rr - 1);
        J[(2 * n) * ne + j] = w * (p + rr * dp);
        J[(2 * n) * ne + nq + j] = w * rr * p;
        J[(2 * n + 1) * ne + j] = w * (lr * p + p + rr * lr * dp);
        J[(2 * n + 1) * ne + nq + j] = w * rr * lr * p;
      }
  };
  auto norm = [](const std::vector<double>& v) {
    double s = 0;
    for (double x : v) s += x * x;
    return std::sqrt(s);
  };
  auto maxabs = [](const std::vector<double>& v) {
    double s = 0;
    for (double x : v) s = std::max(s, std::abs(x));
    return s;
  };
  std::vector<double> glx(nq), glw(nq);
  gl_rule(nq, glx.data(), glw.data());
  auto newton = [&](std::vector<double>& r, std::vector<double>& lw, std::vector<double>& res,
                    double& cost, int iters) {
    std::vector<double> J, tr(nq), tl(nq), tres;
    for (int it = 0; it < iters; ++it) {
      if (maxabs(res) <= 1e-14) break;
      jacobian(r, lw, J);
      std::vector<double> st(ne);
      for (int i = 0; i < ne; ++i) st[i] = -res[i];
      if (!dense_solve(ne, J, st)) break;
      double sigma = 1.0;
      bool stepped = false;
      for (int tries = 0; tries < 40; ++tries, sigma *= 0.5) {
        bool ok = true;
        for (int j = 0; j < nq; ++j) {
          tr[j] = r[j] + sigma * st[j];
          tl[j] = lw[j] + sigma * st[nq + j];
          if (!(tr[j] > 0.0 && tr[j] < 1.0)) ok = false;
        }
        if (!ok) continue;
        residual(tr, tl, tres);
        if (norm(tres) < cost) {
          r = tr;
          lw = tl;
          res = tres;
          cost = norm(tres);
          stepped = true;
          break;
        }
      }
      if (!stepped) break;
    }
  };
  auto accept = [&](const std::vector<double>& r, const std::vector<double>& lw,
                    const std::vector<double>& res) {
    if (!(maxabs(res) <= 1e-13)) return false;
    std::vector<int> idx(nq);
    for (int j = 0; j < nq; ++j) idx[j] = j;
    std::sort(idx.begin(), idx.end(), [&](int a, int bb) { return r[a] < r[bb]; });
    for (int j = 0; j < nq; ++j) {
      rout[j] = r[idx[j]];
      wout[j] = std::exp(lw[idx[j]]);
    }
    if (max_residual) *max_residual = maxabs(res);
    return true;
  };
  for (int pass = 0; pass < 2; ++pass) {
    for (double alpha : {1.0, 1.5, 2.0}) {
      std::vector<double> r(nq), lw(nq), res, J, tr(nq), tl(nq), tres;
      for (int j = 0; j < nq; ++j) {
        r[j] = std::pow(0.5 * (1.0 + glx[j]), alpha);
        lw[j] = std::log(0.5 / nq);
      }
      residual(r, lw, res);
      double cost = norm(res), lam = 1e-3;
      if (pass == 1) {
        // Levenberg-Marquardt globalisation (ggq.hpp:112-139) before Newton
        for (int it = 0; it < 400; ++it) {
          if (maxabs(res) <= 1e-14) break;
          jacobian(r, lw, J);
          std::vector<double> JtJ(ne * ne, 0.0), g(ne, 0.0);
          for (int i = 0; i < ne; ++i)
            for (int k = 0; k < ne; ++k) {
              double s = 0;
              for (int e = 0; e < ne; ++e) s += J[e * ne + i] * J[e * ne + k];
              JtJ[i * ne + k] = s;
            }
          for (int i = 0; i < ne; ++i) {
            double s = 0;
            for (int e = 0; e < ne; ++e) s += J[e * ne + i] * res[e];
            g[i] = -s;
          }
          bool stepped = false;
          for (int tries = 0; tries < 60; ++tries) {
            std::vector<double> A = JtJ, st = g;
            for (int d = 0; d < ne; ++d) A[d * ne + d] += lam * std::max(JtJ[d * ne + d], 1e-12);
            if (dense_solve(ne, A, st)) {
              bool ok = true;
              for (int j = 0; j < nq; ++j) {
                tr[j] = r[j] + st[j];
                tl[j] = lw[j] + st[nq + j];
                if (!(tr[j] > 0.0 && tr[j] < 1.0)) ok = false;
              }
              if (ok) {
                residual(tr, tl, tres);
                if (norm(tres) < cost) {
                  r = tr;
                  lw = tl;
                  res = tres;
                  cost = norm(tres);
                  lam = std::max(lam * 0.2, 1e-15);
                  stepped = true;
                  break;
                }
              }
            }
            lam *= 8;
          }
          if (!stepped) break;
        }
        if (!(maxabs(res) < 1e-3)) continue;
      }
      // damped Newton on the square system (ggq.hpp:141-164)
      newton(r, lw, res, cost, 200);
      if (accept(r, lw, res)) return 0;
    }
  }
  return fail(2, "ggq: moment fitting failed to converge");
}

// Arc-length parametrised circular arc as a Legendre series on tau in [0,1]:
// G(tau) = (cx, cy) + R (cos th(tau), sin th(tau)), th = th0 + tau (th1 - th0);
// coefficients by Gauss-Legendre projection (exact to rounding for deg >= 16
// on arcs of a mesh-sized angle).  *len = R |th1 - th0|.
int vps_circle_arc(double cx, double cy, double R, double th0, double th1, int deg, double* gx, double* gy,
                   double* len) {
  if (deg < 1 || deg > 40 || !gx || !gy || !(R > 0.0)) return fail(1, "circle_arc: deg in [1,40], R > 0");
  // Gauss-Legendre in long double: a double rule leaves ~1e-14 noise in the
  // tail coefficients, which the curved-element tests resolve.
  const int nq = deg + 12;
  std::vector<long double> x(nq), w(nq);
  for (int i = 0; i < nq; ++i) {
    long double z = cosl(3.14159265358979323846264338L * (i + 0.75L) / (nq + 0.5L)), dp = 0.0L;
    for (int it = 0; it < 100; ++it) {
      long double p0 = 1.0L, p1 = z;
      for (int k = 1; k < nq; ++k) {
        const long double p2 = ((2 * k + 1) * z * p1 - k * p0) / (k + 1);
        p0 = p1;
        p1 = p2;
      }
      dp = nq * (p0 - z * p1) / (1.0L - z * z);
      const long double dz = p1 / dp;
      z -= dz;
      if (fabsl(dz) < 1e-19L) break;
    }
    x[i] = z;
    w[i] = 2.0L / ((1.0L - z * z) * dp * dp);
  }
  for (int n = 0; n <= deg; ++n) {
    long double ax = 0.0L, ay = 0.0L;
    for (int i = 0; i < nq; ++i) {
      const long double tau = 0.5L * (1.0L + x[i]);
      const long double th = th0 + tau * ((long double)th1 - th0);
      long double p0 = 1.0L, pn = x[i];
      if (n == 0) pn = 1.0L;
      for (int k = 1; k < n; ++k) {
        const long double p2 = ((2 * k + 1) * x[i] * pn - k * p0) / (k + 1);
        p0 = pn;
        pn = p2;
      }
      ax += w[i] * (cx + R * cosl(th)) * pn;
      ay += w[i] * (cy + R * sinl(th)) * pn;
    }
    gx[n] = (double)(ax * (2 * n + 1) / 2.0L);
    gy[n] = (double)(ay * (2 * n + 1) / 2.0L);
  }
  if (len) *len = R * std::abs(th1 - th0);
  return 0;
}

int vps_lattice_nodes(int p, double* x, double* y) {
  if (p < 0 || p > vp::kMaxP || !x || !y) return fail(1, "lattice: order out of range");
  int k = 0;
  const double d = p + 3;
  for (int j = 0; j <= p; ++j)
    for (int i = 0; i + j <= p; ++i) {
      x[k] = (i + 1) / d;
      y[k] = (j + 1) / d;
      ++k;
    }
  return 0;
}

double vps_density_eval(int kind, const double* prm, int np, double x, double y) {
  switch (kind) {
    case VPS_F_CONST:
      return np > 0 ? prm[0] : 1.0;
    case VPS_F_SQUARE:
      return std::sin(3 * x) * std::cos(2 * y) + x * x;
    case VPS_F_GAUSS: {
      const double dx = x - prm[0], dy = y - prm[1];
      return std::exp(-prm[2] * (dx * dx + dy * dy));
    }
    case VPS_F_BUMPS: {
      double s = 0.0;
      for (int k = 0; 4 * k + 3 < np; ++k) {
        const double dx = x - prm[4 * k], dy = y - prm[4 * k + 1], sg = prm[4 * k + 2];
        s += prm[4 * k + 3] * std::exp(-(dx * dx + dy * dy) / (sg * sg));
      }
      return s;
    }
    case VPS_F_COSSIN:
      return std::cos(4 * kPi * x) * std::sin(2 * kPi * y);
    case VPS_F_LINEAR:
      return prm[0] + prm[1] * x + prm[2] * y;
  }
  return 0.0;
}

int vps_project_density(int64_t n_vert, const double* vxy, int64_t n_tri, const int32_t* tri,
                        int p, int kind, const double* params, int n_params, double* coeffs) {
  if (p < 0 || p > vp::kMaxP) return fail(1, "project_density: order out of range");
  if (n_tri <= 0 || n_vert <= 0 || !vxy || !tri || !coeffs) return fail(1, "project_density: empty mesh");
  const int M = vp::koorn_size(p);
  int len = 0;
  const int ord = 2 * p + 16;
  vps_simplex_rule(ord, &len, nullptr, nullptr, nullptr);
  std::vector<double> rx(len), ry(len), rw(len), V((size_t)len * M);
  vps_simplex_rule(ord, &len, rx.data(), ry.data(), rw.data());
  for (int i = 0; i < len; ++i) vp::koorn_eval(p, rx[i], ry[i], &V[(size_t)i * M]);
  parallel_for(n_tri, [&](int64_t e) {
    const int32_t a = tri[3 * e], b = tri[3 * e + 1], c = tri[3 * e + 2];
    const double x0 = vxy[2 * a], y0 = vxy[2 * a + 1];
    const double e1x = vxy[2 * b] - x0, e1y = vxy[2 * b + 1] - y0;
    const double e2x = vxy[2 * c] - x0, e2y = vxy[2 * c + 1] - y0;
    double* out = coeffs + e * M;
    for (int j = 0; j < M; ++j) out[j] = 0.0;
    for (int i = 0; i < len; ++i) {
      const double X = x0 + rx[i] * e1x + ry[i] * e2x, Y = y0 + rx[i] * e1y + ry[i] * e2y;
      const double f = rw[i] * vps_density_eval(kind, params, n_params, X, Y);
      const double* Vi = &V[(size_t)i * M];
      for (int j = 0; j < M; ++j) out[j] += f * Vi[j];
    }
  });
  return 0;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Synthetic configurations (BASELINE.json:configs).
namespace {

struct Rng {
  std::mt19937_64 g;
  explicit Rng(uint64_t s) : g(s) {}
  double u() { return (double)(g() >> 11) * 0x1.0p-53; }
};

struct Mesh {
  std::vector<double> v;
  std::vector<int32_t> t;
};

// structured grid [x0,x0+nx*hx] x [y0,y0+ny*hy], 2 triangles per cell
// (diagonal v00-v11), interior vertices optionally jittered by U[-j h, j h]
Mesh grid_mesh(int nx, int ny, double x0, double y0, double hx, double hy, double jit, Rng* rng) {
  Mesh m;
  m.v.resize(2 * (size_t)(nx + 1) * (ny + 1));
  for (int j = 0; j <= ny; ++j)
    for (int i = 0; i <= nx; ++i) {
      double x = x0 + i * hx, y = y0 + j * hy;
      if (rng && i > 0 && i < nx && j > 0 && j < ny) {
        x += (2.0 * rng->u() - 1.0) * jit * hx;
        y += (2.0 * rng->u() - 1.0) * jit * hy;
      }
      const size_t k = (size_t)j * (nx + 1) + i;
      m.v[2 * k] = x;
      m.v[2 * k + 1] = y;
    }
  m.t.reserve(6 * (size_t)nx * ny);
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      const int32_t v00 = j * (nx + 1) + i, v10 = v00 + 1, v01 = v00 + nx + 1, v11 = v01 + 1;
      m.t.insert(m.t.end(), {v00, v10, v11, v00, v11, v01});
    }
  return m;
}

// Ring mesh: centre vertex plus rings k=1..K with n[k] vertices at normalised
// radius rad[k] and angle 2 pi (i + off[k]) / n[k]; ring pairs are merged by
// angle with exact rational comparisons.  `shape(rho, theta, x, y)` maps to
// the plane.
template <class Shape>
Mesh ring_mesh(const std::vector<int>& n, const std::vector<double>& rad, const std::vector<double>& off2,
               Shape shape) {
  // off2[k] is twice the angular offset in cells (0 or 1), so angles compare as
  // (2 i + off2) / (2 n) exactly in integers
  Mesh m;
  const int K = (int)n.size() - 1;
  std::vector<int32_t> base(K + 1);
  m.v.push_back(0.0);
  m.v.push_back(0.0);
  base[0] = 0;
  int32_t nv = 1;
  for (int k = 1; k <= K; ++k) {
    base[k] = nv;
    for (int i = 0; i < n[k]; ++i) {
      const double th = 2.0 * kPi * (i + 0.5 * off2[k]) / n[k];
      double x, y;
      shape(rad[k], th, x, y);
      m.v.push_back(x);
      m.v.push_back(y);
      ++nv;
    }
  }
  for (int i = 0; i < n[1]; ++i)
    m.t.insert(m.t.end(), {0, base[1] + i, base[1] + (i + 1) % n[1]});
  for (int k = 2; k <= K; ++k) {
    const int64_t ni = n[k - 1], no = n[k];
    const int64_t oi = (int64_t)off2[k - 1], oo = (int64_t)off2[k];
    int64_t i = 0, o = 0;
    while (i < ni || o < no) {
      // angle of the next inner / outer vertex, as (2*idx + off) / (2 n)
      bool adv_inner;
      if (i >= ni) adv_inner = false;
      else if (o >= no) adv_inner = true;
      else adv_inner = (2 * (i + 1) + oi) * no <= (2 * (o + 1) + oo) * ni;
      const int32_t vi = base[k - 1] + (int32_t)(i % ni), vo = base[k] + (int32_t)(o % no);
      if (adv_inner) {
        m.t.insert(m.t.end(), {vi, vo, base[k - 1] + (int32_t)((i + 1) % ni)});
        ++i;
      } else {
        m.t.insert(m.t.end(), {vi, vo, base[k] + (int32_t)((o + 1) % no)});
        ++o;
      }
    }
  }
  return m;
}

double star_rb(double th) { return 1.0 + 0.3 * std::cos(5.0 * th); }

// star mesh with grading h(r) = h0 (0.25 + 0.75 (1 - r/r_b)) (BASELINE config 3/5)
Mesh star_mesh(int K, double* h0_out = nullptr) {
  // perimeter factor of the star boundary relative to the unit circle
  double per = 0.0;
  const int NS = 20000;
  for (int i = 0; i < NS; ++i) {
    const double th = 2 * kPi * (i + 0.5) / NS, rb = star_rb(th), drb = -1.5 * std::sin(5 * th);
    per += std::sqrt(rb * rb + drb * drb) * (2 * kPi / NS);
  }
  const double lfac = per / (2 * kPi);
  const double c = std::log(4.0) / 0.75;  // rho(tau) = (1 - e^{-0.75 c tau})/0.75, rho(1) = 1
  std::vector<int> n(K + 1);
  std::vector<double> rad(K + 1), off(K + 1, 0.0);
  n[0] = 1;
  rad[0] = 0.0;
  for (int k = 1; k <= K; ++k) {
    const double tau = (double)k / K;
    rad[k] = (k == K) ? 1.0 : (1.0 - std::exp(-0.75 * c * tau)) / 0.75;
    const double drho = c * (1.0 - 0.75 * rad[k]) / K;
    n[k] = std::max(6, (int)std::lround(2 * kPi * rad[k] * lfac / drho));
  }
  if (h0_out) *h0_out = c / K;
  return ring_mesh(n, rad, off, [](double rho, double th, double& x, double& y) {
    const double r = rho * star_rb(th);
    x = r * std::cos(th);
    y = r * std::sin(th);
  });
}

int star_K_for(int64_t target_tris) {
  int bestK = 4;
  int64_t bestd = INT64_MAX;
  for (int K = 4; K < 2000; ++K) {
    // triangle count depends only on ring counts; cheap to recompute
    const double c = std::log(4.0) / 0.75;
    double per = 0.0;
    const int NS = 2000;
    for (int i = 0; i < NS; ++i) {
      const double th = 2 * kPi * (i + 0.5) / NS, rb = star_rb(th), drb = -1.5 * std::sin(5 * th);
      per += std::sqrt(rb * rb + drb * drb) * (2 * kPi / NS);
    }
    const double lfac = per / (2 * kPi);
    int64_t tot = 0;
    int prev = 1;
    for (int k = 1; k <= K; ++k) {
      const double tau = (double)k / K;
      const double rad = (k == K) ? 1.0 : (1.0 - std::exp(-0.75 * c * tau)) / 0.75;
      const double drho = c * (1.0 - 0.75 * rad) / K;
      const int nk = std::max(6, (int)std::lround(2 * kPi * rad * lfac / drho));
      tot += (k == 1) ? nk : (prev + nk);
      prev = nk;
    }
    const int64_t d = std::llabs(tot - target_tris);
    if (d < bestd) {
      bestd = d;
      bestK = K;
    }
    if (tot > 2 * target_tris) break;
  }
  return bestK;
}

void lattice_targets(const Mesh& m, int p, std::vector<double>& txy) {
  const int M = vp::koorn_size(p);
  std::vector<double> lx(M), ly(M);
  vps_lattice_nodes(p, lx.data(), ly.data());
  const int64_t E = (int64_t)m.t.size() / 3;
  txy.resize(2 * (size_t)E * M);
  for (int64_t e = 0; e < E; ++e) {
    const int32_t a = m.t[3 * e], b = m.t[3 * e + 1], c = m.t[3 * e + 2];
    const double x0 = m.v[2 * a], y0 = m.v[2 * a + 1];
    const double e1x = m.v[2 * b] - x0, e1y = m.v[2 * b + 1] - y0;
    const double e2x = m.v[2 * c] - x0, e2y = m.v[2 * c + 1] - y0;
    for (int k = 0; k < M; ++k) {
      txy[2 * (e * M + k)] = x0 + lx[k] * e1x + ly[k] * e2x;
      txy[2 * (e * M + k) + 1] = y0 + lx[k] * e1y + ly[k] * e2y;
    }
  }
}

struct Built {
  Mesh mesh;
  std::vector<double> txy;
  vps_config_info info;
};

int build_config(int config, int q_override, uint64_t seed, Built& B, bool want_arrays) {
  vps_config_info& I = B.info;
  std::memset(&I, 0, sizeof(I));
  I.seed = seed;
  I.eps = 1e-12;
  Rng rng(seed);
  switch (config) {
    case 1: {  // unit square 16x16, jitter 0.1h, p=4, q=p+2, same-mesh targets
      I.p = 4;
      I.q = 6;
      I.density_kind = VPS_F_SQUARE;
      I.n_params = 0;
      B.mesh = grid_mesh(16, 16, 0.0, 0.0, 1.0 / 16, 1.0 / 16, 0.1, &rng);
      if (want_arrays) lattice_targets(B.mesh, I.p, B.txy);
      I.n_tgt = (int64_t)B.mesh.t.size() / 3 * vp::koorn_size(I.p);
      break;
    }
    case 2: {  // unit disk polar rings 16k, p=8, q=2p, staggered targets
      I.p = 8;
      I.q = 16;
      I.density_kind = VPS_F_GAUSS;
      const double r = std::sqrt(rng.u()), th = 2 * kPi * rng.u();
      I.n_params = 3;
      I.params[0] = r * std::cos(th);
      I.params[1] = r * std::sin(th);
      I.params[2] = 8.0;
      const int K = 16;
      std::vector<int> n(K + 1);
      std::vector<double> rad(K + 1), off(K + 1, 0.0), rad2(K + 1), off2(K + 1, 1.0);
      n[0] = 1;
      for (int k = 1; k <= K; ++k) {
        n[k] = 16 * k;
        rad[k] = (double)k / K;
        rad2[k] = (k - 0.5) / K;
      }
      auto disk = [](double rho, double th2, double& x, double& y) {
        x = rho * std::cos(th2);
        y = rho * std::sin(th2);
      };
      B.mesh = ring_mesh(n, rad, off, disk);
      I.staggered = 1;
      if (want_arrays) {
        Mesh tm = ring_mesh(n, rad2, off2, disk);
        lattice_targets(tm, I.p, B.txy);
      }
      I.n_tgt = (int64_t)B.mesh.t.size() / 3 * vp::koorn_size(I.p);
      break;
    }
    case 3:
    case 5: {  // star, graded, p=8, q=2p (config 5: sweep), same-mesh targets
      I.p = 8;
      I.q = 16;
      I.density_kind = VPS_F_BUMPS;
      I.n_params = 40;
      for (int k = 0; k < 10; ++k) {
        double cx, cy;
        for (;;) {
          cx = (2.0 * rng.u() - 1.0) * 1.3;
          cy = (2.0 * rng.u() - 1.0) * 1.3;
          const double rr = std::sqrt(cx * cx + cy * cy), th = std::atan2(cy, cx);
          if (rr < star_rb(th)) break;
        }
        const double sg = 0.05 + 0.15 * rng.u();
        const double A = 2.0 * rng.u() - 1.0;
        I.params[4 * k] = cx;
        I.params[4 * k + 1] = cy;
        I.params[4 * k + 2] = sg;
        I.params[4 * k + 3] = A;
      }
      const int64_t target = config == 3 ? 65536 : 262144;
      static int cachedK[2] = {0, 0};
      int& K = cachedK[config == 3 ? 0 : 1];
      if (K == 0) K = star_K_for(target);
      B.mesh = star_mesh(K);
      if (want_arrays) lattice_targets(B.mesh, I.p, B.txy);
      I.n_tgt = (int64_t)B.mesh.t.size() / 3 * vp::koorn_size(I.p);
      break;
    }
    case 4: {  // unit square 512x1024, jitter 0.1h, p=6, q=2p, staggered targets
      I.p = 6;
      I.q = 12;
      I.density_kind = VPS_F_COSSIN;
      I.n_params = 0;
      const int nx = 512, ny = 1024;
      const double hx = 1.0 / nx, hy = 1.0 / ny;
      B.mesh = grid_mesh(nx, ny, 0.0, 0.0, hx, hy, 0.1, &rng);
      I.staggered = 1;
      if (want_arrays) {
        Mesh tm = grid_mesh(nx, ny, 0.5 * hx, 0.5 * hy, hx, hy, 0.0, nullptr);
        lattice_targets(tm, I.p, B.txy);
      }
      I.n_tgt = (int64_t)B.mesh.t.size() / 3 * vp::koorn_size(I.p);
      break;
    }
    default:
      return fail(1, "config: id must be in 1..5");
  }
  if (q_override > 0) I.q = q_override;
  I.n_vert = (int64_t)B.mesh.v.size() / 2;
  I.n_tri = (int64_t)B.mesh.t.size() / 3;
  return 0;
}

}  // namespace

extern "C" {

int vps_config_info_get(int config, int q_override, uint64_t seed, vps_config_info* info) {
  if (!info) return fail(1, "config: null info");
  Built B;
  if (int rc = build_config(config, q_override, seed, B, false)) return rc;
  *info = B.info;
  return 0;
}

int vps_config_fill(int config, int q_override, uint64_t seed, double* vxy, int32_t* tri,
                    double* txy, double* coeffs) {
  Built B;
  if (int rc = build_config(config, q_override, seed, B, true)) return rc;
  const vps_config_info& I = B.info;
  if (vxy) std::memcpy(vxy, B.mesh.v.data(), B.mesh.v.size() * sizeof(double));
  if (tri) std::memcpy(tri, B.mesh.t.data(), B.mesh.t.size() * sizeof(int32_t));
  if (txy) std::memcpy(txy, B.txy.data(), B.txy.size() * sizeof(double));
  if (coeffs)
    return vps_project_density(I.n_vert, B.mesh.v.data(), I.n_tri, B.mesh.t.data(), I.p,
                               I.density_kind, I.params, I.n_params, coeffs);
  return 0;
}

}  // extern "C"
