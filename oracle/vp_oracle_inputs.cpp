// vp_oracle_inputs.cpp -- the oracle's own inputs: rules, seeded synthetic
// configurations and density coefficients.
//
// TEST INFRASTRUCTURE ONLY (see vp_oracle.h).  This file lets liboracle.so
// stand alone: the reference arm of bench.py and the oracle side of the
// parity tests build their problems here, without loading the product
// library.  tests/test_oracle_inputs.py checks that these inputs agree with
// the product's host generators (vp_setup.cpp): meshes and targets byte for
// byte, rules and coefficients to rounding.
//
// Anchors:
//   Gauss-Jacobi rule ........ Golub-Welsch on the Jacobi matrix of P^{(1,0)}
//                              (own algorithm: implicit-shift QL + Newton polish)
//   simplex rule ............. collapsed Duffy map; contract of
//                              validate_rule, rules.hpp:60-85
//   far / near rule .......... load_far_rule, rules.hpp:121-125: fully symmetric
//                              rules of orders 6, 10, 12 expanded from the
//                              moment-fitted orbit table sym_rules.inc
//                              (tools/make_sym_rules.py), else the simplex rule
//   GGQ ...................... build_ggq, ggq.hpp:33-182 (moments :33-50,
//                              Levenberg-Marquardt :110-139, Newton :141-164)
//   density projection ....... L2 projection onto koornwinder_eval,
//                              koornwinder.hpp:77-113 (north_star: order-p
//                              coefficients per triangle)
//   configurations ........... BASELINE.json configs 1-5 as fixed in SURVEY.md
//                              §8(d) and DESIGN.md §2.11 (seed, PRNG mapping,
//                              ring/star/grid recipes, stagger)
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "vp_oracle.h"

namespace {

constexpr double kPi = 3.14159265358979323846;

std::string g_in_err;
int in_fail(int code, const char* m) {
  g_in_err = m;
  return code;
}

inline int nmodes(int p) { return (p + 1) * (p + 2) / 2; }

// ---------------------------------------------------------------------------
// 1-D rules

// P_n^{(1,0)}(x) and its derivative, three-term recurrence (alpha=1, beta=0)
void jac10(int n, double x, double& p, double& dp) {
  double pm = 1.0, pc = 0.5 * (3.0 * x + 1.0);  // P_0, P_1 = ((a+b+2)x + (a-b))/2
  if (n == 0) {
    p = 1.0;
    dp = 0.0;
    return;
  }
  for (int k = 2; k <= n; ++k) {
    const double s = 2.0 * k + 1.0;  // 2k + a + b
    const double A = 2.0 * k * (k + 1.0) * (s - 2.0);
    const double B = (s - 1.0) * (s * (s - 2.0) * x + 1.0);
    const double C = 2.0 * k * (k - 1.0) * s;
    const double pn = (B * pc - C * pm) / A;
    pm = pc;
    pc = pn;
  }
  p = pc;
  const double s = 2.0 * n + 1.0;
  dp = (n * (1.0 - s * x) * pc + 2.0 * (n + 1.0) * n * pm) / (s * (1.0 - x * x));
}

// eigenvalues of a symmetric tridiagonal matrix (diag d, off-diagonal e[1..])
// by the implicit-shift QL iteration; returns ascending
void tridiag_eigs(std::vector<double> d, std::vector<double> e, std::vector<double>& out) {
  const int n = (int)d.size();
  for (int i = 1; i < n; ++i) e[i - 1] = e[i];
  e[n - 1] = 0.0;
  for (int l = 0; l < n; ++l) {
    for (int iter = 0; iter < 60; ++iter) {
      int m = l;
      for (; m < n - 1; ++m) {
        const double dd = std::abs(d[m]) + std::abs(d[m + 1]);
        if (std::abs(e[m]) <= 1e-17 * dd) break;
      }
      if (m == l) break;
      double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
      double r = std::hypot(g, 1.0);
      g = d[m] - d[l] + e[l] / (g + (g >= 0 ? r : -r));
      double s = 1.0, c = 1.0, p = 0.0;
      int i = m - 1;
      for (; i >= l; --i) {
        double f = s * e[i];
        const double b = c * e[i];
        r = std::hypot(f, g);
        e[i + 1] = r;
        if (r == 0.0) {
          d[i + 1] -= p;
          e[m] = 0.0;
          break;
        }
        s = f / r;
        c = g / r;
        g = d[i + 1] - p;
        r = (d[i] - g) * s + 2.0 * c * b;
        p = s * r;
        d[i + 1] = g + p;
        g = c * r - b;
      }
      if (r == 0.0 && i >= l) continue;
      d[l] -= p;
      e[l] = g;
      e[m] = 0.0;
    }
  }
  std::sort(d.begin(), d.end());
  out = d;
}

// Gauss-Jacobi rule for the weight (1-u) on [0,1]: Golub-Welsch eigenvalues
// of the Jacobi matrix, Newton-polished on P_n^{(1,0)}, Christoffel weights
void gj10(int n, double* x01, double* w01) {
  std::vector<double> a(n), b(n, 0.0), z;
  for (int k = 0; k < n; ++k) {
    const double s = 2.0 * k + 1.0;
    a[k] = -1.0 / (s * (s + 2.0));
    if (k >= 1) b[k] = std::sqrt(4.0 * k * (k + 1.0) * k * (k + 1.0) / (s * s * (s + 1.0) * (s - 1.0)));
  }
  tridiag_eigs(a, b, z);
  for (int i = 0; i < n; ++i) {
    double t = z[i], p, dp;
    for (int it = 0; it < 8; ++it) {
      jac10(n, t, p, dp);
      const double dt = p / dp;
      t -= dt;
      if (std::abs(dt) < 1e-16) break;
    }
    jac10(n, t, p, dp);
    x01[i] = 0.5 * (1.0 + t);
    w01[i] = 0.25 * (4.0 / ((1.0 - t * t) * dp * dp));
  }
}

double leg(int n, double x) {
  double p0 = 1.0, p1 = x;
  if (n == 0) return 1.0;
  for (int k = 1; k < n; ++k) {
    const double p2 = ((2 * k + 1) * x * p1 - k * p0) / (k + 1);
    p0 = p1;
    p1 = p2;
  }
  return p1;
}
double dleg(int n, double x) { return n == 0 ? 0.0 : n * (leg(n - 1, x) - x * leg(n, x)) / (1.0 - x * x); }

// Gaussian elimination with partial pivoting on a dense row-major n x n copy
bool solve_dense(int n, std::vector<double> A, std::vector<double>& x) {
  for (int c = 0; c < n; ++c) {
    int pr = c;
    double best = std::abs(A[c * n + c]);
    for (int r = c + 1; r < n; ++r)
      if (std::abs(A[r * n + c]) > best) {
        best = std::abs(A[r * n + c]);
        pr = r;
      }
    if (best == 0.0) return false;
    if (pr != c) {
      for (int k = 0; k < n; ++k) std::swap(A[c * n + k], A[pr * n + k]);
      std::swap(x[c], x[pr]);
    }
    for (int r = c + 1; r < n; ++r) {
      const double f = A[r * n + c] / A[c * n + c];
      if (f == 0.0) continue;
      for (int k = c; k < n; ++k) A[r * n + k] -= f * A[c * n + k];
      x[r] -= f * x[c];
    }
  }
  for (int c = n - 1; c >= 0; --c) {
    double s = x[c];
    for (int k = c + 1; k < n; ++k) s -= A[c * n + k] * x[k];
    x[c] = s / A[c * n + c];
  }
  return true;
}

// ---------------------------------------------------------------------------
// GGQ by moment fitting (ggq.hpp:96-182).  Unknowns: nodes r_j in (0,1) and
// log-weights; targets b_n = int r P_n(2r-1), c_n = int r log r P_n(2r-1).
struct Ggq {
  int ng, nq, ne;
  std::vector<double> b, c;
  explicit Ggq(int g) : ng(g), nq(g + 1), ne(2 * (g + 1)), b(g + 1, 0.0), c(g + 1, 0.0) {
    // b_n: Gauss-Legendre with ng+4 points on [0,1]; c_n: 80 dyadic panels
    // toward r = 0, 24 Gauss-Legendre points each (ggq.hpp:33-50)
    std::vector<double> x(ng + 4), w(ng + 4);
    vpo_gauss_legendre(ng + 4, x.data(), w.data());
    for (int n = 0; n <= ng; ++n)
      for (int i = 0; i < ng + 4; ++i) {
        const double r = 0.5 * (1.0 + x[i]);
        b[n] += 0.5 * w[i] * r * leg(n, 2 * r - 1);
      }
    std::vector<double> hx(24), hw(24);
    vpo_gauss_legendre(24, hx.data(), hw.data());
    for (int k = 0; k < 80; ++k) {
      const double hi = std::ldexp(1.0, -k), lo = 0.5 * hi;
      for (int i = 0; i < 24; ++i) {
        const double r = 0.5 * (lo + hi) + 0.5 * (hi - lo) * hx[i];
        const double ww = 0.5 * (hi - lo) * hw[i];
        for (int n = 0; n <= ng; ++n) c[n] += ww * r * std::log(r) * leg(n, 2 * r - 1);
      }
    }
  }
  void resid(const std::vector<double>& z, std::vector<double>& f) const {
    f.assign(ne, 0.0);
    for (int n = 0; n <= ng; ++n) {
      double s0 = 0.0, s1 = 0.0;
      for (int j = 0; j < nq; ++j) {
        const double r = z[j], w = std::exp(z[nq + j]), p = leg(n, 2 * r - 1);
        s0 += w * r * p;
        s1 += w * r * std::log(r) * p;
      }
      f[2 * n] = s0 - b[n];
      f[2 * n + 1] = s1 - c[n];
    }
  }
  void jac(const std::vector<double>& z, std::vector<double>& J) const {
    J.assign(ne * ne, 0.0);
    for (int n = 0; n <= ng; ++n)
      for (int j = 0; j < nq; ++j) {
        const double r = z[j], w = std::exp(z[nq + j]), lr = std::log(r);
        const double p = leg(n, 2 * r - 1), dp = 2 * dleg(n, 2 * r - 1);
        J[(2 * n) * ne + j] = w * (p + r * dp);
        J[(2 * n) * ne + nq + j] = w * r * p;
        J[(2 * n + 1) * ne + j] = w * (lr * p + p + r * lr * dp);
        J[(2 * n + 1) * ne + nq + j] = w * r * lr * p;
      }
  }
  static double l2(const std::vector<double>& v) {
    double s = 0;
    for (double x : v) s += x * x;
    return std::sqrt(s);
  }
  static double linf(const std::vector<double>& v) {
    double s = 0;
    for (double x : v) s = std::max(s, std::abs(x));
    return s;
  }
  bool feasible(const std::vector<double>& z) const {
    for (int j = 0; j < nq; ++j)
      if (!(z[j] > 0.0 && z[j] < 1.0)) return false;
    return true;
  }
  // one accepted step of Levenberg-Marquardt (Marquardt-scaled damping)
  bool lm_step(std::vector<double>& z, std::vector<double>& f, double& cost, double& lam) const {
    std::vector<double> J, JtJ(ne * ne, 0.0), g(ne, 0.0), t(ne), ft;
    jac(z, J);
    for (int i = 0; i < ne; ++i) {
      for (int k = 0; k < ne; ++k) {
        double s = 0;
        for (int e = 0; e < ne; ++e) s += J[e * ne + i] * J[e * ne + k];
        JtJ[i * ne + k] = s;
      }
      double s = 0;
      for (int e = 0; e < ne; ++e) s += J[e * ne + i] * f[e];
      g[i] = -s;
    }
    for (int tries = 0; tries < 60; ++tries, lam *= 8) {
      std::vector<double> A = JtJ, st = g;
      for (int d = 0; d < ne; ++d) A[d * ne + d] += lam * std::max(JtJ[d * ne + d], 1e-12);
      if (!solve_dense(ne, A, st)) continue;
      for (int i = 0; i < ne; ++i) t[i] = z[i] + st[i];
      if (!feasible(t)) continue;
      resid(t, ft);
      if (l2(ft) < cost) {
        z = t;
        f = ft;
        cost = l2(ft);
        lam = std::max(lam * 0.2, 1e-15);
        return true;
      }
    }
    return false;
  }
  // one accepted step of damped Newton on the square system
  bool newton_step(std::vector<double>& z, std::vector<double>& f, double& cost) const {
    std::vector<double> J, st(ne), t(ne), ft;
    jac(z, J);
    for (int i = 0; i < ne; ++i) st[i] = -f[i];
    if (!solve_dense(ne, J, st)) return false;
    double sig = 1.0;
    for (int tries = 0; tries < 40; ++tries, sig *= 0.5) {
      for (int i = 0; i < ne; ++i) t[i] = z[i] + sig * st[i];
      if (!feasible(t)) continue;
      resid(t, ft);
      if (l2(ft) < cost) {
        z = t;
        f = ft;
        cost = l2(ft);
        return true;
      }
    }
    return false;
  }
  bool solve(double* rout, double* wout, double* res_out) const {
    std::vector<double> gx(nq), gw(nq);
    vpo_gauss_legendre(nq, gx.data(), gw.data());
    // pass 0: damped Newton alone from the warped Gauss-Legendre guesses;
    // pass 1: the reference's order (ggq.hpp:110-164), Levenberg-Marquardt
    // first, then Newton once in the basin
    for (int pass = 0; pass < 2; ++pass)
      for (double alpha : {1.0, 1.5, 2.0}) {
        std::vector<double> z(ne), f;
        for (int j = 0; j < nq; ++j) {
          z[j] = std::pow(0.5 * (1.0 + gx[j]), alpha);
          z[nq + j] = std::log(0.5 / nq);
        }
        resid(z, f);
        double cost = l2(f), lam = 1e-3;
        if (pass == 1) {
          for (int it = 0; it < 400 && linf(f) > 1e-14; ++it)
            if (!lm_step(z, f, cost, lam)) break;
          if (!(linf(f) < 1e-3)) continue;
        }
        for (int it = 0; it < 200 && linf(f) > 1e-14; ++it)
          if (!newton_step(z, f, cost)) break;
        if (!(linf(f) <= 1e-13)) continue;
        std::vector<int> idx(nq);
        for (int j = 0; j < nq; ++j) idx[j] = j;
        std::sort(idx.begin(), idx.end(), [&](int a, int bb) { return z[a] < z[bb]; });
        for (int j = 0; j < nq; ++j) {
          rout[j] = z[idx[j]];
          wout[j] = std::exp(z[nq + idx[j]]);
        }
        if (res_out) *res_out = linf(f);
        return true;
      }
    return false;
  }
};

// ---------------------------------------------------------------------------
// densities
double f_eval(int kind, const double* prm, int np, double x, double y) {
  switch (kind) {
    case 0: return np > 0 ? prm[0] : 1.0;
    case 1: return std::sin(3 * x) * std::cos(2 * y) + x * x;
    case 2: {
      const double dx = x - prm[0], dy = y - prm[1];
      return std::exp(-prm[2] * (dx * dx + dy * dy));
    }
    case 3: {
      double s = 0.0;
      for (int k = 0; 4 * k + 3 < np; ++k) {
        const double dx = x - prm[4 * k], dy = y - prm[4 * k + 1], sg = prm[4 * k + 2];
        s += prm[4 * k + 3] * std::exp(-(dx * dx + dy * dy) / (sg * sg));
      }
      return s;
    }
    case 4: return std::cos(4 * kPi * x) * std::sin(2 * kPi * y);
    case 5: return prm[0] + prm[1] * x + prm[2] * y;
  }
  return 0.0;
}

// ---------------------------------------------------------------------------
// synthetic meshes
struct Rng53 {  // mt19937_64, u = (x >> 11) 2^-53
  std::mt19937_64 g;
  explicit Rng53(uint64_t s) : g(s) {}
  double next() { return (double)(g() >> 11) * 0x1.0p-53; }
};

struct TriMesh {
  std::vector<double> v;   // [nv * 2]
  std::vector<int32_t> t;  // [nt * 3]
  int64_t nv() const { return (int64_t)v.size() / 2; }
  int64_t nt() const { return (int64_t)t.size() / 3; }
};

// nx x ny cells over [x0, x0 + nx hx] x [y0, y0 + ny hy], split along the
// (i,j)-(i+1,j+1) diagonal; interior vertices jittered by U[-jit h, jit h]
TriMesh cell_grid(int nx, int ny, double x0, double y0, double hx, double hy, double jit, Rng53* rng) {
  TriMesh m;
  const int64_t W = nx + 1;
  m.v.resize(2 * (size_t)W * (ny + 1));
  for (int j = 0; j <= ny; ++j)
    for (int i = 0; i <= nx; ++i) {
      double x = x0 + i * hx, y = y0 + j * hy;
      const bool interior = i > 0 && i < nx && j > 0 && j < ny;
      if (rng && interior) {
        x += (2.0 * rng->next() - 1.0) * jit * hx;  // x draw first, then y
        y += (2.0 * rng->next() - 1.0) * jit * hy;
      }
      m.v[2 * (j * W + i)] = x;
      m.v[2 * (j * W + i) + 1] = y;
    }
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      const int32_t a = (int32_t)(j * W + i), b = a + 1, d = (int32_t)(a + W), c = d + 1;
      const int32_t tr[6] = {a, b, c, a, c, d};
      m.t.insert(m.t.end(), tr, tr + 6);
    }
  return m;
}

// centre + rings k = 1..K: ring k has cnt[k] vertices at normalised radius
// rad[k], angle 2 pi (i + half[k]/2) / cnt[k]; neighbouring rings are zipped
// by comparing angles as exact integer fractions
template <class Map>
TriMesh rings(const std::vector<int>& cnt, const std::vector<double>& rad, const std::vector<double>& half, Map map) {
  TriMesh m;
  const int K = (int)cnt.size() - 1;
  std::vector<int32_t> first(K + 1, 0);
  m.v = {0.0, 0.0};
  for (int k = 1; k <= K; ++k) {
    first[k] = (int32_t)m.nv();
    for (int i = 0; i < cnt[k]; ++i) {
      double x, y;
      map(rad[k], 2.0 * kPi * (i + 0.5 * half[k]) / cnt[k], x, y);
      m.v.push_back(x);
      m.v.push_back(y);
    }
  }
  for (int i = 0; i < cnt[1]; ++i) {
    const int32_t tr[3] = {0, first[1] + i, first[1] + (i + 1) % cnt[1]};
    m.t.insert(m.t.end(), tr, tr + 3);
  }
  for (int k = 2; k <= K; ++k) {
    const int64_t a = cnt[k - 1], b = cnt[k], ha = (int64_t)half[k - 1], hb = (int64_t)half[k];
    for (int64_t i = 0, o = 0; i < a || o < b;) {
      const bool inner = i < a && (o >= b || (2 * (i + 1) + ha) * b <= (2 * (o + 1) + hb) * a);
      const int32_t vi = first[k - 1] + (int32_t)(i % a), vo = first[k] + (int32_t)(o % b);
      const int32_t third = inner ? first[k - 1] + (int32_t)((i + 1) % a) : first[k] + (int32_t)((o + 1) % b);
      const int32_t tr[3] = {vi, vo, third};
      m.t.insert(m.t.end(), tr, tr + 3);
      if (inner) ++i; else ++o;
    }
  }
  return m;
}

double star_r(double th) { return 1.0 + 0.3 * std::cos(5.0 * th); }

// boundary length of the star over 2 pi (midpoint rule with ns samples)
double star_len_factor(int ns) {
  double per = 0.0;
  for (int i = 0; i < ns; ++i) {
    const double th = 2 * kPi * (i + 0.5) / ns, rb = star_r(th), drb = -1.5 * std::sin(5 * th);
    per += std::sqrt(rb * rb + drb * drb) * (2 * kPi / ns);
  }
  return per / (2 * kPi);
}

// graded rings: rho(tau) = (1 - e^{-0.75 c tau}) / 0.75 with c = log 4 / 0.75,
// so h(rho) = h0 (1 - 0.75 rho) and the boundary is 4x finer than the centre;
// ring k holds max(6, round(2 pi rho lfac / drho)) vertices
void star_rings(int K, double lfac, std::vector<int>& cnt, std::vector<double>& rad) {
  const double c = std::log(4.0) / 0.75;
  cnt.assign(K + 1, 1);
  rad.assign(K + 1, 0.0);
  for (int k = 1; k <= K; ++k) {
    const double tau = (double)k / K;
    rad[k] = (k == K) ? 1.0 : (1.0 - std::exp(-0.75 * c * tau)) / 0.75;
    const double drho = c * (1.0 - 0.75 * rad[k]) / K;
    cnt[k] = std::max(6, (int)std::lround(2 * kPi * rad[k] * lfac / drho));
  }
}

int star_rings_for(int64_t want) {
  const double lfac = star_len_factor(2000);
  int best = 4;
  int64_t bestd = INT64_MAX;
  for (int K = 4; K < 2000; ++K) {
    std::vector<int> cnt;
    std::vector<double> rad;
    star_rings(K, lfac, cnt, rad);
    int64_t tris = cnt[1];
    for (int k = 2; k <= K; ++k) tris += cnt[k - 1] + cnt[k];
    if (std::llabs(tris - want) < bestd) {
      bestd = std::llabs(tris - want);
      best = K;
    }
    if (tris > 2 * want) break;
  }
  return best;
}

TriMesh star(int K) {
  std::vector<int> cnt;
  std::vector<double> rad;
  star_rings(K, star_len_factor(20000), cnt, rad);
  return rings(cnt, rad, std::vector<double>(K + 1, 0.0), [](double rho, double th, double& x, double& y) {
    const double r = rho * star_r(th);
    x = r * std::cos(th);
    y = r * std::sin(th);
  });
}

// targets: the shifted principal lattice ((i+1)/(p+3), (j+1)/(p+3)) mapped
// into every triangle of `m`, element-major
void lattice_into(const TriMesh& m, int p, std::vector<double>& txy) {
  const int M = nmodes(p);
  std::vector<double> lx(M), ly(M);
  vpo_lattice_nodes(p, lx.data(), ly.data());
  txy.resize(2 * (size_t)m.nt() * M);
  for (int64_t e = 0; e < m.nt(); ++e) {
    const int32_t* id = &m.t[3 * e];
    const double ax = m.v[2 * id[0]], ay = m.v[2 * id[0] + 1];
    const double ux = m.v[2 * id[1]] - ax, uy = m.v[2 * id[1] + 1] - ay;
    const double wx = m.v[2 * id[2]] - ax, wy = m.v[2 * id[2] + 1] - ay;
    for (int k = 0; k < M; ++k) {
      txy[2 * (e * M + k)] = ax + lx[k] * ux + ly[k] * wx;
      txy[2 * (e * M + k) + 1] = ay + lx[k] * uy + ly[k] * wy;
    }
  }
}

struct Cfg {
  TriMesh mesh;
  std::vector<double> txy;
  vpo_config_info info;
};

int make_config(int id, int q_override, uint64_t seed, bool arrays, Cfg& C) {
  vpo_config_info& I = C.info;
  std::memset(&I, 0, sizeof(I));
  I.seed = seed;
  I.eps = 1e-12;
  Rng53 rng(seed);
  auto disk = [](double rho, double th, double& x, double& y) {
    x = rho * std::cos(th);
    y = rho * std::sin(th);
  };
  if (id == 1) {  // [0,1]^2, 16 x 16 cells, jitter 0.1 h, p = 4, q = p + 2
    I.p = 4;
    I.q = 6;
    I.density_kind = 1;
    C.mesh = cell_grid(16, 16, 0.0, 0.0, 1.0 / 16, 1.0 / 16, 0.1, &rng);
    if (arrays) lattice_into(C.mesh, I.p, C.txy);
  } else if (id == 2) {  // unit disk, rings of 16 k vertices, staggered targets
    I.p = 8;
    I.q = 16;
    I.density_kind = 2;
    const double r = std::sqrt(rng.next()), th = 2 * kPi * rng.next();
    I.n_params = 3;
    I.params[0] = r * std::cos(th);
    I.params[1] = r * std::sin(th);
    I.params[2] = 8.0;
    const int K = 16;
    std::vector<int> cnt(K + 1, 1);
    std::vector<double> rad(K + 1, 0.0), rad_t(K + 1, 0.0);
    for (int k = 1; k <= K; ++k) {
      cnt[k] = 16 * k;
      rad[k] = (double)k / K;
      rad_t[k] = (k - 0.5) / K;  // target rings half a ring inward
    }
    C.mesh = rings(cnt, rad, std::vector<double>(K + 1, 0.0), disk);
    I.staggered = 1;
    if (arrays)  // target mesh rotated by half an angular cell per ring
      lattice_into(rings(cnt, rad_t, std::vector<double>(K + 1, 1.0), disk), I.p, C.txy);
  } else if (id == 3 || id == 5) {  // graded star, 10 Gaussian bumps
    I.p = 8;
    I.q = 16;
    I.density_kind = 3;
    I.n_params = 40;
    for (int k = 0; k < 10; ++k) {
      double cx, cy;
      do {  // rejection sampling in the star
        cx = (2.0 * rng.next() - 1.0) * 1.3;
        cy = (2.0 * rng.next() - 1.0) * 1.3;
      } while (!(std::sqrt(cx * cx + cy * cy) < star_r(std::atan2(cy, cx))));
      const double sg = 0.05 + 0.15 * rng.next();
      const double A = 2.0 * rng.next() - 1.0;
      I.params[4 * k] = cx;
      I.params[4 * k + 1] = cy;
      I.params[4 * k + 2] = sg;
      I.params[4 * k + 3] = A;
    }
    static int Kc[2] = {0, 0};
    int& K = Kc[id == 3 ? 0 : 1];
    if (K == 0) K = star_rings_for(id == 3 ? 65536 : 262144);
    C.mesh = star(K);
    if (arrays) lattice_into(C.mesh, I.p, C.txy);
  } else if (id == 4) {  // [0,1]^2, 512 x 1024 cells, staggered by (h/2, h/2)
    I.p = 6;
    I.q = 12;
    I.density_kind = 4;
    const int nx = 512, ny = 1024;
    const double hx = 1.0 / nx, hy = 1.0 / ny;
    C.mesh = cell_grid(nx, ny, 0.0, 0.0, hx, hy, 0.1, &rng);
    I.staggered = 1;
    if (arrays) lattice_into(cell_grid(nx, ny, 0.5 * hx, 0.5 * hy, hx, hy, 0.0, nullptr), I.p, C.txy);
  } else {
    return in_fail(1, "config: id must be in 1..5");
  }
  if (q_override > 0) I.q = q_override;
  I.n_vert = C.mesh.nv();
  I.n_tri = C.mesh.nt();
  I.n_tgt = I.n_tri * nmodes(I.p);
  return 0;
}

}  // namespace

extern "C" {

const char* vpo_inputs_last_error(void) { return g_in_err.c_str(); }

int vpo_lattice_nodes(int p, double* x, double* y) {
  if (p < 0 || p > 32 || !x || !y) return in_fail(1, "lattice: order out of range");
  const double d = p + 3;
  int k = 0;
  for (int j = 0; j <= p; ++j)
    for (int i = 0; i + j <= p; ++i, ++k) {
      x[k] = (i + 1) / d;
      y[k] = (j + 1) / d;
    }
  return 0;
}

int vpo_gauss_jacobi10(int n, double* x, double* w) {
  if (n < 1 || !x || !w) return in_fail(1, "gauss_jacobi: order must be >= 1");
  gj10(n, x, w);
  return 0;
}

int vpo_simplex_rule(int order, int* len, double* x, double* y, double* w) {
  if (order < 0 || order > 200 || !len) return in_fail(1, "simplex_rule: order out of range");
  const int n = order / 2 + 1;  // 2n - 1 >= order per collapsed direction
  *len = n * n;
  if (!x) return 0;
  std::vector<double> ux(n), uw(n), vx(n), vw(n);
  gj10(n, ux.data(), uw.data());
  vpo_gauss_legendre(n, vx.data(), vw.data());
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      const double u = ux[i], v = 0.5 * (1.0 + vx[j]);
      x[i * n + j] = u;
      y[i * n + j] = v * (1.0 - u);
      w[i * n + j] = uw[i] * (0.5 * vw[j]);
    }
  return 0;
}

// The evaluation's far / near rule (load_far_rule, rules.hpp:121-125): the
// fully symmetric rule of that degree from the oracle's own copy of the
// moment-fitted orbit table (tools/make_sym_rules.py), expanded orbit by
// orbit; the collapsed Gauss-Jacobi rule for every other order.
namespace {
struct SymOrbits {
  int degree, n1, n21, n111, points;
  double p[64];
};
const SymOrbits kSymOrbits[] = {
#include "sym_rules.inc"
};
}  // namespace

int vpo_quad_rule(int order, int* len, double* x, double* y, double* w) {
  const SymOrbits* r = nullptr;
  for (const SymOrbits& t : kSymOrbits)
    if (t.degree == order) r = &t;
  if (!r) return vpo_simplex_rule(order, len, x, y, w);
  if (!len) return in_fail(1, "quad_rule: len is null");
  *len = r->points;
  if (!x) return 0;
  if (!y || !w) return in_fail(1, "quad_rule: null output array");
  int n = 0;
  const double* q = r->p;
  if (r->n1) {
    x[n] = 1.0 / 3.0;
    y[n] = 1.0 / 3.0;
    w[n++] = *q++;
  }
  for (int i = 0; i < r->n21; ++i, q += 2) {  // (a, a, c), c = 1 - 2a: (x, y) = (l2, l3)
    const double a = q[1], c = 1.0 - 2.0 * a;
    const double pts[3][2] = {{a, a}, {a, c}, {c, a}};
    for (const auto& pt : pts) {
      x[n] = pt[0];
      y[n] = pt[1];
      w[n++] = q[0];
    }
  }
  for (int i = 0; i < r->n111; ++i, q += 3) {  // the six permutations of (a, b, c)
    const double a = q[1], b = q[2], c = 1.0 - a - b;
    const double pts[6][2] = {{a, b}, {b, a}, {a, c}, {c, a}, {b, c}, {c, b}};
    for (const auto& pt : pts) {
      x[n] = pt[0];
      y[n] = pt[1];
      w[n++] = q[0];
    }
  }
  return 0;
}

int vpo_ggq(int ng, double* r, double* w, double* max_residual) {
  if (ng < 0 || ng > 20 || !r || !w) return in_fail(1, "ggq: order must be in [0, 20]");
  if (!Ggq(ng).solve(r, w, max_residual)) return in_fail(2, "ggq: moment fitting failed to converge");
  return 0;
}

double vpo_density_eval(int kind, const double* params, int n_params, double x, double y) {
  return f_eval(kind, params, n_params, x, y);
}

int vpo_project_density(int64_t n_vert, const double* vxy, int64_t n_tri, const int32_t* tri, int p, int kind,
                        const double* params, int n_params, double* coeffs) {
  if (p < 0 || p > 12) return in_fail(1, "project_density: order out of range");
  if (n_tri <= 0 || n_vert <= 0 || !vxy || !tri || !coeffs) return in_fail(1, "project_density: empty mesh");
  const int M = nmodes(p), ord = 2 * p + 16;
  int len = 0;
  vpo_simplex_rule(ord, &len, nullptr, nullptr, nullptr);
  std::vector<double> rx(len), ry(len), rw(len), K((size_t)len * M);
  vpo_simplex_rule(ord, &len, rx.data(), ry.data(), rw.data());
  for (int i = 0; i < len; ++i) vpo_koornwinder(p, rx[i], ry[i], &K[(size_t)i * M]);
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < n_tri; ++e) {
    const int32_t* id = tri + 3 * e;
    const double ax = vxy[2 * id[0]], ay = vxy[2 * id[0] + 1];
    const double ux = vxy[2 * id[1]] - ax, uy = vxy[2 * id[1] + 1] - ay;
    const double wx = vxy[2 * id[2]] - ax, wy = vxy[2 * id[2] + 1] - ay;
    double* c = coeffs + e * M;
    std::fill(c, c + M, 0.0);
    for (int i = 0; i < len; ++i) {  // c_j = sum_i w_i f(rho(xi_i)) K_j(xi_i)
      const double X = ax + rx[i] * ux + ry[i] * wx, Y = ay + rx[i] * uy + ry[i] * wy;
      const double fw = rw[i] * f_eval(kind, params, n_params, X, Y);
      for (int j = 0; j < M; ++j) c[j] += fw * K[(size_t)i * M + j];
    }
  }
  return 0;
}

int vpo_config_info_get(int config, int q_override, uint64_t seed, vpo_config_info* info) {
  if (!info) return in_fail(1, "config: null info");
  Cfg C;
  if (int rc = make_config(config, q_override, seed, false, C)) return rc;
  *info = C.info;
  return 0;
}

int vpo_config_fill(int config, int q_override, uint64_t seed, double* vxy, int32_t* tri, double* txy,
                    double* coeffs) {
  Cfg C;
  if (int rc = make_config(config, q_override, seed, true, C)) return rc;
  const vpo_config_info& I = C.info;
  if (vxy) std::memcpy(vxy, C.mesh.v.data(), C.mesh.v.size() * sizeof(double));
  if (tri) std::memcpy(tri, C.mesh.t.data(), C.mesh.t.size() * sizeof(int32_t));
  if (txy) std::memcpy(txy, C.txy.data(), C.txy.size() * sizeof(double));
  if (coeffs)
    return vpo_project_density(I.n_vert, C.mesh.v.data(), I.n_tri, C.mesh.t.data(), I.p, I.density_kind, I.params,
                               I.n_params, coeffs);
  return 0;
}

}  // extern "C"
