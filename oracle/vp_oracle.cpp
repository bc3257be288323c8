// vp_oracle.cpp -- CPU restatement of the volume-potential hot path.
//
// TEST INFRASTRUCTURE ONLY (see vp_oracle.h).  Plain C++20, OpenMP over
// targets, compiled with -O2 -ffp-contract=off and no fast-math so every
// floating-point operation is a single IEEE round-to-nearest operation in
// source order.  The GPU product reproduces the list predicates with the
// same operation order using explicitly rounded intrinsics; everything
// else is compared against this file with a tolerance.
//
// Anchors (reference file:line):
//   Koornwinder basis ........ koornwinder.hpp:77-113, :117-120
//   rules / w_edge ........... rules.hpp:44-54, :60-85
//   Gauss-Legendre ........... gauss.hpp:17-46
//   quadtree ................. quadtree.hpp:24-126
//   C_N table ................ SPEC.md:424-438
//   near-field model ......... SPEC.md:416-458
//   locate / nearby .......... SPEC.md:368-386
//   far (direct) ............. SPEC.md:497-505, :572-580, :618
//   near_eval ................ SPEC.md:507-515, :535-536
//   self_eval ................ SPEC.md:517-526, :537-539
//   subtract-and-add ......... SPEC.md:582-590

#include "vp_oracle.h"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

constexpr int kMaxOrder = 32;
constexpr double kPi = 3.14159265358979323846;
constexpr double kInv4Pi = 1.0 / (4.0 * kPi);
constexpr double kInv2Pi = 1.0 / (2.0 * kPi);
constexpr double kBaryTol = 1e-12;
constexpr int kMaxNearDepth = 40;

std::mutex g_err_mu;
std::string g_err;

int fail(int code, const std::string& msg) {
  std::lock_guard<std::mutex> lk(g_err_mu);
  g_err = msg;
  return code;
}

inline int ksize(int p) { return (p + 1) * (p + 2) / 2; }

// ---------------------------------------------------------------------------
// Koornwinder basis, graded order n outer / m inner (koornwinder.hpp:12-21).
// Same recurrences as koorn_eval_impl<double> (koornwinder.hpp:77-113):
// homogenised Legendre in (u, v) = (2y-(1-x), 1-x) and Jacobi P^{(2m+1,0)}.
void koorn(int N, double x, double y, double* out) {
  double Lm[kMaxOrder + 2];
  const double v = 1.0 - x;
  const double u = 2.0 * y - v;
  const double v2 = v * v;
  Lm[0] = 1.0;
  if (N >= 1) Lm[1] = u;
  for (int m = 1; m + 1 <= N; ++m)
    Lm[m + 1] = ((2 * m + 1) * (u * Lm[m]) - double(m) * (v2 * Lm[m - 1])) / double(m + 1);
  const double t = 2.0 * x - 1.0;
  for (int m = 0; m <= N; ++m) {
    const double a = 2 * m + 1;
    double pprev = 1.0;                          // P_0
    double pcur = 0.5 * (a + (a + 2.0) * t);     // P_1
    for (int k = 0; m + k <= N; ++k) {
      const double pk = (k == 0) ? pprev : pcur;
      const int n = m + k;
      const double c = std::sqrt((double)((2 * m + 1) * (2 * n + 2)));
      out[n * (n + 1) / 2 + m] = c * (pk * Lm[m]);
      if (k >= 1 && m + k + 1 <= N) {
        const double kk = k;
        const double c1 = 2 * (kk + 1) * (kk + a + 1) * (2 * kk + a);
        const double c2 = (2 * kk + a + 1) * (a * a);
        const double c3 = (2 * kk + a) * (2 * kk + a + 1) * (2 * kk + a + 2);
        const double c4 = 2 * (kk + a) * kk * (2 * kk + a + 2);
        const double pn = ((c2 * pcur + c3 * (t * pcur)) - c4 * pprev) / c1;
        pprev = pcur;
        pcur = pn;
      }
    }
  }
}

// f_T(x, y) = sum_j c_j K_j(x, y)
inline double density(int p, const double* c, double x, double y) {
  double k[(kMaxOrder + 1) * (kMaxOrder + 2) / 2];
  koorn(p, x, y, k);
  double s = 0.0;
  const int M = ksize(p);
  for (int j = 0; j < M; ++j) s += c[j] * k[j];
  return s;
}

// C_N calibration.  Orders below 12
// are uncalibrated in the paper; policy: clamp to C_12.
double cn_lookup(int n) {
  static const int kn[6] = {12, 20, 25, 30, 40, 50};
  static const double kc[6] = {12.0, 6.8, 3.0, 2.5, 2.0, 1.0};
  if (n <= 12) return 12.0;
  if (n >= 50) return 1.0;
  for (int i = 0; i + 1 < 6; ++i) {
    if (n == kn[i]) return kc[i];
    if (n > kn[i] && n < kn[i + 1]) {
      const double f = double(n - kn[i]) / double(kn[i + 1] - kn[i]);
      return kc[i] + (kc[i + 1] - kc[i]) * f;
    }
  }
  return 1.0;
}

// w_edge (rules.hpp:44-54): max weight among nodes whose edge distance is
// strictly below the median (element size/2 after nth_element).
double w_edge(int len, const double* x, const double* y, const double* w) {
  std::vector<double> d(len);
  for (int i = 0; i < len; ++i)
    d[i] = std::min({x[i], y[i], (1.0 - x[i] - y[i]) / std::sqrt(2.0)});
  std::vector<double> s = d;
  std::nth_element(s.begin(), s.begin() + s.size() / 2, s.end());
  const double med = s[s.size() / 2];
  double best = 0.0;
  for (int i = 0; i < len; ++i)
    if (d[i] < med) best = std::max(best, w[i]);
  return best;
}

// Ball near-field model: circumscribed circle scaled by
// `factor`, centre stored relative to vertex a; exact operation order shared
// with the GPU (vp_device.cuh rn_ball).
struct Ball {
  double ux, uy, rr;  // centre - a, factor^2 * R^2
};
Ball ball_of(double ax, double ay, double bx, double by, double cx, double cy, double factor) {
  const double bxr = bx - ax, byr = by - ay, cxr = cx - ax, cyr = cy - ay;
  const double t1 = bxr * cyr, t2 = byr * cxr;
  const double d = 2.0 * (t1 - t2);
  const double b2 = bxr * bxr + byr * byr, c2 = cxr * cxr + cyr * cyr;
  const double u1 = cyr * b2, u2 = byr * c2;
  const double v1 = bxr * c2, v2 = cxr * b2;
  Ball B;
  B.ux = (u1 - u2) / d;
  B.uy = (v1 - v2) / d;
  const double R2 = B.ux * B.ux + B.uy * B.uy;
  B.rr = (factor * factor) * R2;
  return B;
}
bool in_ball(const Ball& B, double ax, double ay, double tx, double ty) {
  const double dx = (tx - ax) - B.ux, dy = (ty - ay) - B.uy;
  return dx * dx + dy * dy < B.rr;
}
constexpr int kBallMaxDepth = 20;  // ball model: accept at this depth (no rho_d cut-off exists)

// ---------------------------------------------------------------------------
// Quadtree over points (quadtree.hpp:24-126): closed rectangles, quadrant by
// >= against the centre, leaf capacity m, minimum box diameter 1e-12 * root.
struct QTree {
  struct Node {
    double lox, loy, hix, hiy;
    int child0 = -1;
    std::vector<int> items;
  };
  const double* pts = nullptr;
  std::vector<Node> nodes;
  int cap = 32;
  double min_diam = 0.0;

  static double diam(const Node& n) {
    const double w = n.hix - n.lox, h = n.hiy - n.loy;
    return std::sqrt(w * w + h * h);
  }
  void build(int64_t n, const double* p, int m) {
    pts = p;
    cap = m;
    double lox = 1e300, loy = 1e300, hix = -1e300, hiy = -1e300;
    for (int64_t i = 0; i < n; ++i) {
      lox = std::min(lox, p[2 * i]);
      loy = std::min(loy, p[2 * i + 1]);
      hix = std::max(hix, p[2 * i]);
      hiy = std::max(hiy, p[2 * i + 1]);
    }
    const double margin = 1e-9 * std::max({std::abs(lox), std::abs(loy), std::abs(hix),
                                           std::abs(hiy), hix - lox, hiy - loy, 1e-30});
    Node root;
    root.lox = lox - margin;
    root.loy = loy - margin;
    root.hix = hix + margin;
    root.hiy = hiy + margin;
    nodes.clear();
    nodes.push_back(root);
    min_diam = 1e-12 * diam(nodes[0]);
    std::vector<int> all(n);
    for (int64_t i = 0; i < n; ++i) all[i] = (int)i;
    split(0, std::move(all));
  }
  void split(size_t ni, std::vector<int> items) {
    const Node box = nodes[ni];
    const double cx = (box.lox + box.hix) * 0.5, cy = (box.loy + box.hiy) * 0.5;
    // Deviation (documented in DESIGN.md): also stop when the box can no
    // longer be halved in floating point.  With every point coincident the
    // root box is degenerate, min_diam falls below the fp spacing and the
    // reference's subdivide (quadtree.hpp:79-109) recurses without end.
    const bool unsplittable = !(cx > box.lox && cx < box.hix) && !(cy > box.loy && cy < box.hiy);
    if ((int)items.size() <= cap || diam(box) < min_diam || unsplittable) {
      nodes[ni].items = std::move(items);
      return;
    }
    std::vector<int> b[4];
    for (int idx : items) {
      const int qd = (pts[2 * idx] >= cx ? 1 : 0) + (pts[2 * idx + 1] >= cy ? 2 : 0);
      b[qd].push_back(idx);
    }
    const size_t c0 = nodes.size();
    nodes[ni].child0 = (int)c0;
    const double qx0[4] = {box.lox, cx, box.lox, cx}, qx1[4] = {cx, box.hix, cx, box.hix};
    const double qy0[4] = {box.loy, box.loy, cy, cy}, qy1[4] = {cy, cy, box.hiy, box.hiy};
    for (int k = 0; k < 4; ++k) {
      Node c;
      c.lox = qx0[k];
      c.hix = qx1[k];
      c.loy = qy0[k];
      c.hiy = qy1[k];
      nodes.push_back(c);
    }
    for (int k = 0; k < 4; ++k) split(c0 + k, std::move(b[k]));
  }
  void query(size_t ni, double lox, double loy, double hix, double hiy, std::vector<int>& out,
             int64_t& visited) const {
    const Node& n = nodes[ni];
    ++visited;
    if (!(lox <= n.hix && n.lox <= hix && loy <= n.hiy && n.loy <= hiy)) return;
    if (n.child0 < 0) {
      const bool all_in = lox <= n.lox && n.hix <= hix && loy <= n.loy && n.hiy <= hiy;
      for (int idx : n.items) {
        const double px = pts[2 * idx], py = pts[2 * idx + 1];
        if (all_in || (px >= lox && px <= hix && py >= loy && py <= hiy)) out.push_back(idx);
      }
      return;
    }
    for (int k = 0; k < 4; ++k) query(n.child0 + k, lox, loy, hix, hiy, out, visited);
  }
};

// ---------------------------------------------------------------------------
// Curved elements (PAPER.md:1023-1044 blending map,
// SPEC.md:339-376).  The curved side is gamma(tau L) = G(tau) = sum_n c_n
// P_n(2 tau - 1); vertices (v0, v1, v2) = (gamma(L), gamma(0), O) so that
// rho(0,0) = gamma(L), rho(1,0) = gamma(0), rho(0,1) = O.
// Every operation below has a fixed order that the GPU reproduces with
// explicitly rounded intrinsics (predicates that decide lists and counts).
struct CurveC {
  const double* cx;
  const double* cy;
  int D;
  double L;
};

void curve_eval(const CurveC& C, double tau, double& gx, double& gy) {
  const double x = 2.0 * tau - 1.0;
  double p0 = 1.0, p1 = x;
  gx = C.cx[0];
  gy = C.cy[0];
  if (C.D >= 1) {
    gx = gx + C.cx[1] * x;
    gy = gy + C.cy[1] * x;
  }
  for (int n = 1; n < C.D; ++n) {
    const double a = (double)(2 * n + 1) * x;
    const double b = a * p1;
    const double c = (double)n * p0;
    const double p2 = (b - c) / (double)(n + 1);
    gx = gx + C.cx[n + 1] * p2;
    gy = gy + C.cy[n + 1] * p2;
    p0 = p1;
    p1 = p2;
  }
}

// G, dG/dtau and d2G/dtau2 (P'_{n+1} = P'_{n-1} + (2n+1) P_n, same for P'')
void curve_eval_d(const CurveC& C, double tau, double g[2], double g1[2], double g2[2]) {
  const double x = 2.0 * tau - 1.0;
  double p0 = 1.0, p1 = x, d0 = 0.0, d1 = 1.0, e0 = 0.0, e1 = 0.0;
  g[0] = C.cx[0]; g[1] = C.cy[0];
  g1[0] = 0.0; g1[1] = 0.0;
  g2[0] = 0.0; g2[1] = 0.0;
  if (C.D >= 1) {
    g[0] = g[0] + C.cx[1] * x; g[1] = g[1] + C.cy[1] * x;
    g1[0] = g1[0] + C.cx[1] * d1; g1[1] = g1[1] + C.cy[1] * d1;
  }
  for (int n = 1; n < C.D; ++n) {
    const double a = (double)(2 * n + 1) * x;
    const double p2 = (a * p1 - (double)n * p0) / (double)(n + 1);
    const double d2 = d0 + (double)(2 * n + 1) * p1;
    const double e2 = e0 + (double)(2 * n + 1) * d1;
    g[0] = g[0] + C.cx[n + 1] * p2; g[1] = g[1] + C.cy[n + 1] * p2;
    g1[0] = g1[0] + C.cx[n + 1] * d2; g1[1] = g1[1] + C.cy[n + 1] * d2;
    g2[0] = g2[0] + C.cx[n + 1] * e2; g2[1] = g2[1] + C.cy[n + 1] * e2;
    p0 = p1; p1 = p2; d0 = d1; d1 = d2; e0 = e1; e1 = e2;
  }
  g1[0] = 2.0 * g1[0]; g1[1] = 2.0 * g1[1];
  g2[0] = 4.0 * g2[0]; g2[1] = 4.0 * g2[1];
}

struct BlendGeom {
  double PLx, PLy, P0x, P0y, Ox, Oy;
};

// rho(xi, eta) of PAPER.md eq. for:blend
void blend(const BlendGeom& B, const CurveC& C, double xi, double eta, double& x, double& y) {
  const double om = 1.0 - xi;
  const double lam = om - eta;
  const double bx = (lam * B.PLx + xi * B.P0x) + eta * B.Ox;
  const double by = (lam * B.PLy + xi * B.P0y) + eta * B.Oy;
  if (!(om > 1e-13)) {  // xi -> 1 limit: the bracket vanishes
    x = bx;
    y = by;
    return;
  }
  double gx, gy;
  curve_eval(C, om, gx, gy);
  const double Dx = (gx - om * B.PLx) - xi * B.P0x;
  const double Dy = (gy - om * B.PLy) - xi * B.P0y;
  const double r = lam / om;
  x = bx + r * Dx;
  y = by + r * Dy;
}

// rho and its Jacobian [dx/dxi dx/deta; dy/dxi dy/deta]
void blend_jac(const BlendGeom& B, const CurveC& C, double xi, double eta, double& x, double& y,
               double J[4]) {
  const double om0 = 1.0 - xi;
  const double om = om0 > 1e-13 ? om0 : 1e-13;
  const double lam = om0 - eta;
  double g[2], g1[2], g2[2];
  curve_eval_d(C, om, g, g1, g2);
  const double bx = (lam * B.PLx + xi * B.P0x) + eta * B.Ox;
  const double by = (lam * B.PLy + xi * B.P0y) + eta * B.Oy;
  const double Dx = (g[0] - om * B.PLx) - xi * B.P0x;
  const double Dy = (g[1] - om * B.PLy) - xi * B.P0y;
  const double r = lam / om;
  x = bx + r * Dx;
  y = by + r * Dy;
  const double drx = -eta / (om * om), dre = -1.0 / om;
  const double dDx = (B.PLx - g1[0]) - B.P0x, dDy = (B.PLy - g1[1]) - B.P0y;
  J[0] = ((B.P0x - B.PLx) + drx * Dx) + r * dDx;
  J[1] = (B.Ox - B.PLx) + dre * Dx;
  J[2] = ((B.P0y - B.PLy) + drx * Dy) + r * dDy;
  J[3] = (B.Oy - B.PLy) + dre * Dy;
}

constexpr int kBlendNewton = 12;  // fixed count: identical iterates on CPU and GPU

// Newton inverse of the blending map seeded by (xi, eta)
void blend_inverse(const BlendGeom& B, const CurveC& C, double tx, double ty, double& xi, double& eta) {
  for (int it = 0; it < kBlendNewton; ++it) {
    double x, y, J[4];
    blend_jac(B, C, xi, eta, x, y, J);
    const double rx = tx - x, ry = ty - y;
    const double dj = J[0] * J[3] - J[1] * J[2];
    const double dxi = (J[3] * rx - J[1] * ry) / dj;
    const double deta = (J[0] * ry - J[2] * rx) / dj;
    xi = xi + dxi;
    eta = eta + deta;
  }
}

// Newton inverse to convergence (quadrature points; values, not predicates)
void blend_inverse_tol(const BlendGeom& B, const CurveC& C, double tx, double ty, double& xi, double& eta) {
  for (int it = 0; it < 40; ++it) {
    double x, y, J[4];
    blend_jac(B, C, xi, eta, x, y, J);
    const double rx = tx - x, ry = ty - y;
    const double dj = J[0] * J[3] - J[1] * J[2];
    const double dxi = (J[3] * rx - J[1] * ry) / dj;
    const double deta = (J[0] * ry - J[2] * rx) / dj;
    xi = xi + dxi;
    eta = eta + deta;
    if (std::abs(dxi) + std::abs(deta) < 1e-15) break;
  }
}

// s~ = argmin_s |v - gamma(s)| on the curved side gamma(s) = G(1 - s/L):
// best of 33 samples, then 10 Newton steps on (gamma - v).gamma' = 0,
// clamped to [0, L] (SPEC.md:537 asks golden section + Newton; any exact
// minimiser gives the same panels).
double curved_argmin(const CurveC& C, double vx, double vy) {
  const double L = C.L;
  int best = 0;
  double bd = 1e300;
  for (int i = 0; i <= 32; ++i) {
    double gx, gy;
    curve_eval(C, 1.0 - (double)i / 32.0, gx, gy);
    const double dx = gx - vx, dy = gy - vy;
    const double d2 = dx * dx + dy * dy;
    if (d2 < bd) {
      bd = d2;
      best = i;
    }
  }
  double s = L * ((double)best / 32.0);
  for (int it = 0; it < 10; ++it) {
    double g[2], g1[2], g2[2];
    curve_eval_d(C, 1.0 - s / L, g, g1, g2);
    const double tx = -g1[0] / L, ty = -g1[1] / L;       // gamma'(s)
    const double ax = g2[0] / (L * L), ay = g2[1] / (L * L);  // gamma''(s)
    const double dx = g[0] - vx, dy = g[1] - vy;
    const double phi = dx * tx + dy * ty;
    const double dphi = (tx * tx + ty * ty) + (dx * ax + dy * ay);
    if (!(dphi > 0.0)) break;
    s = s - phi / dphi;
    s = std::min(std::max(s, 0.0), L);
  }
  return s;
}

// ---------------------------------------------------------------------------
// Per-problem setup: element geometry, near-field models, sources.
struct Setup {
  const vpo_problem* pr = nullptr;
  int64_t E = 0;
  int M = 0;
  // element geometry, SoA
  std::vector<double> x0, y0, e1x, e1y, e2x, e2y, det;
  std::vector<double> rho0, rho0n, two_a;  // two_a[3E]
  std::vector<double> bb;                  // near-field bbox [4E] lox loy hix hiy
  std::vector<char> all_near;
  std::vector<int32_t> all_near_ids;
  double query_half = 0.0;
  double kd[kMaxNearDepth + 2];
  QTree qt;
  std::vector<double> corners;
  // sources
  std::vector<double> sx, sy, sq;

  bool curved(int64_t e) const { return pr->curve_id && pr->curve_id[e] >= 0; }
  CurveC curve(int64_t e) const {
    const int c = pr->curve_id[e], D = pr->curve_deg;
    return CurveC{pr->curve_cx + (int64_t)c * (D + 1), pr->curve_cy + (int64_t)c * (D + 1), D, pr->curve_len[c]};
  }
  BlendGeom bgeom(int64_t e) const {
    const int32_t* id = pr->tri + 3 * e;
    return BlendGeom{pr->vxy[2 * id[0]], pr->vxy[2 * id[0] + 1], pr->vxy[2 * id[1]], pr->vxy[2 * id[1] + 1],
                     pr->vxy[2 * id[2]], pr->vxy[2 * id[2] + 1]};
  }
  // element map (affine or blending) at a reference point, and |J| there
  void map_point(int64_t e, double xi, double eta, double& x, double& y) const {
    if (curved(e)) {
      blend(bgeom(e), curve(e), xi, eta, x, y);
      return;
    }
    x = x0[e] + (xi * e1x[e] + eta * e2x[e]);
    y = y0[e] + (xi * e1y[e] + eta * e2y[e]);
  }
  double jac_at(int64_t e, double xi, double eta) const {
    if (!curved(e)) return det[e];
    double x, y, J[4];
    blend_jac(bgeom(e), curve(e), xi, eta, x, y, J);
    return std::abs(J[0] * J[3] - J[1] * J[2]);
  }

  int init(const vpo_problem* p, bool want_lists, bool want_sources) {
    pr = p;
    if (!p || p->n_tri <= 0 || p->n_vert <= 0 || !p->vxy || !p->tri)
      return fail(1, "oracle: empty mesh (invariant: n_tri > 0, n_vert > 0)");
    if (p->p < 0 || p->p > kMaxOrder) return fail(1, "oracle: density order out of range");
    if (p->eps <= 0.0) return fail(1, "oracle: eps must be > 0");
    E = p->n_tri;
    M = ksize(p->p);
    x0.resize(E); y0.resize(E); e1x.resize(E); e1y.resize(E); e2x.resize(E); e2y.resize(E);
    det.resize(E);
    for (int64_t e = 0; e < E; ++e) {
      const int32_t a = p->tri[3 * e], b = p->tri[3 * e + 1], c = p->tri[3 * e + 2];
      if (a < 0 || b < 0 || c < 0 || a >= p->n_vert || b >= p->n_vert || c >= p->n_vert)
        return fail(1, "oracle: triangle vertex index out of range");
      const double ax = p->vxy[2 * a], ay = p->vxy[2 * a + 1];
      x0[e] = ax;
      y0[e] = ay;
      e1x[e] = p->vxy[2 * b] - ax;
      e1y[e] = p->vxy[2 * b + 1] - ay;
      e2x[e] = p->vxy[2 * c] - ax;
      e2y[e] = p->vxy[2 * c + 1] - ay;
      const double t1 = e1x[e] * e2y[e];
      const double t2 = e2x[e] * e1y[e];
      det[e] = t1 - t2;  // |J_T| = 2 area(T)
      if (!(det[e] > 0.0)) return fail(1, "oracle: triangle not counter-clockwise (det <= 0)");
    }
    if (want_lists) {
      if (p->len_q <= 0 || p->len_n <= 0) return fail(1, "oracle: empty rule");
      const double we = w_edge(p->len_q, p->far_x, p->far_y, p->far_w);
      const double wn = w_edge(p->len_n, p->near_x, p->near_y, p->near_w);
      const double cq = cn_lookup(p->q), cn = cn_lookup(p->n_n);
      rho0.resize(E); rho0n.resize(E); two_a.resize(3 * E); bb.resize(4 * E);
      all_near.assign(E, 0);
      all_near_ids.clear();
      for (int d = 0; d <= kMaxNearDepth + 1; ++d) kd[d] = std::pow(4.0, -(double)d / (double)p->n_n);
      for (int64_t e = 0; e < E; ++e) {
        // w scaled by area(T)/area(Delta^1) = det
        const double w = we * det[e];
        const double den = p->eps * cq;
        rho0[e] = std::pow(w / den, 1.0 / (double)p->q);
        const double wnn = wn * det[e];
        const double denn = p->eps * cn;
        rho0n[e] = std::pow(wnn / denn, 1.0 / (double)p->n_n);
        // the list model uses the stored vertices themselves
        const int32_t id[3] = {p->tri[3 * e], p->tri[3 * e + 1], p->tri[3 * e + 2]};
        double px[3], py[3];
        for (int k = 0; k < 3; ++k) { px[k] = p->vxy[2 * id[k]]; py[k] = p->vxy[2 * id[k] + 1]; }
        if (p->near_model == 1) {  // ball model: ta = (ux, uy, factor^2 R^2)
          const Ball B = ball_of(px[0], py[0], px[1], py[1], px[2], py[2], p->ball_factor);
          two_a[3 * e] = B.ux;
          two_a[3 * e + 1] = B.uy;
          two_a[3 * e + 2] = B.rr;
          const double r = std::sqrt(B.rr) * (1.0 + 1e-9) + 1e-300;
          const double cxm = px[0] + B.ux, cym = py[0] + B.uy;
          bb[4 * e] = cxm - r; bb[4 * e + 1] = cym - r; bb[4 * e + 2] = cxm + r; bb[4 * e + 3] = cym + r;
          continue;
        }
        if (!(rho0[e] > 1.0)) {  // model undefined -> element all-near
          all_near[e] = 1;
          all_near_ids.push_back((int32_t)e);
          for (int k = 0; k < 3; ++k) two_a[3 * e + k] = 0.0;
          bb[4 * e] = bb[4 * e + 1] = bb[4 * e + 2] = bb[4 * e + 3] = 0.0;
          continue;
        }
        const double g = (rho0[e] + 1.0 / rho0[e]) * 0.5;
        double lox = 1e300, loy = 1e300, hix = -1e300, hiy = -1e300;
        for (int k = 0; k < 3; ++k) {
          const int k1 = (k + 1) % 3;
          const double dx = px[k1] - px[k], dy = py[k1] - py[k];
          const double len = std::sqrt(dx * dx + dy * dy);
          two_a[3 * e + k] = g * len;  // 2a = (rho0 + 1/rho0)/2 * len
          // the ellipse lies in the disc of radius a about the side midpoint
          const double mx = (px[k] + px[k1]) * 0.5, my = (py[k] + py[k1]) * 0.5;
          const double r = two_a[3 * e + k] * 0.5 * (1.0 + 1e-9) + 1e-300;
          lox = std::min(lox, mx - r); hix = std::max(hix, mx + r);
          loy = std::min(loy, my - r); hiy = std::max(hiy, my + r);
        }
        if (curved(e)) {  // the element itself (for locate) bulges past its chord
          const CurveC C = curve(e);
          for (int k = 0; k <= 32; ++k) {
            double gx, gy;
            curve_eval(C, k / 32.0, gx, gy);
            const double pad = 1e-9 * C.L + 1e-300;
            lox = std::min(lox, gx - 0.05 * C.L - pad); hix = std::max(hix, gx + 0.05 * C.L + pad);
            loy = std::min(loy, gy - 0.05 * C.L - pad); hiy = std::max(hiy, gy + 0.05 * C.L + pad);
          }
        }
        bb[4 * e] = lox; bb[4 * e + 1] = loy; bb[4 * e + 2] = hix; bb[4 * e + 3] = hiy;
      }
      // quadtree over the four corners of every near-field bbox
      corners.assign(8 * E, 0.0);
      query_half = 0.0;
      for (int64_t e = 0; e < E; ++e) {
        const double* b = &bb[4 * e];
        corners[8 * e + 0] = b[0]; corners[8 * e + 1] = b[1];
        corners[8 * e + 2] = b[2]; corners[8 * e + 3] = b[1];
        corners[8 * e + 4] = b[0]; corners[8 * e + 5] = b[3];
        corners[8 * e + 6] = b[2]; corners[8 * e + 7] = b[3];
        if (!all_near[e]) query_half = std::max({query_half, b[2] - b[0], b[3] - b[1]});
      }
      qt.build(4 * E, corners.data(), 32);
    }
    if (want_sources) {
      if (p->len_q <= 0) return fail(1, "oracle: empty far rule");
      const int L = p->len_q;
      sx.resize(E * L); sy.resize(E * L); sq.resize(E * L);
#pragma omp parallel for schedule(static)
      for (int64_t e = 0; e < E; ++e) {
        const double* c = p->coeffs + e * M;
        for (int i = 0; i < L; ++i) {
          const double xi = p->far_x[i], eta = p->far_y[i];
          map_point(e, xi, eta, sx[e * L + i], sy[e * L + i]);
          const double f = density(p->p, c, xi, eta);
          // q_i = w_i |J_T| f(y_i) / (4 pi): sum q log r^2 = (1/2pi) sum w|J|f log r
          sq[e * L + i] = (p->far_w[i] * jac_at(e, xi, eta)) * f * kInv4Pi;
        }
      }
    }
    return 0;
  }

  // Reference coordinates of t in element e (inverse affine map) and the
  // barycentric containment test with tolerance 1e-12.
  bool ref_coords(int64_t e, double tx, double ty, double& xi, double& eta) const {
    const double i00 = e2y[e] / det[e], i01 = -e2x[e] / det[e];
    const double i10 = -e1y[e] / det[e], i11 = e1x[e] / det[e];
    const double dx = tx - x0[e], dy = ty - y0[e];
    const double a0 = i00 * dx, a1 = i01 * dy;
    xi = a0 + a1;
    const double b0 = i10 * dx, b1 = i11 * dy;
    eta = b0 + b1;
    if (curved(e)) {
      // blending-map inverse seeded by the chord's affine inverse, with a
      // residual check so a non-converged iterate never counts as inside
      const BlendGeom B = bgeom(e);
      const CurveC C = curve(e);
      blend_inverse(B, C, tx, ty, xi, eta);
      double x, y;
      blend(B, C, xi, eta, x, y);
      const double rx = tx - x, ry = ty - y;
      const double tolr = 1e-9 * C.L;
      if (!(rx * rx + ry * ry <= tolr * tolr)) return false;
    }
    const double l0 = (1.0 - xi) - eta;
    return xi >= -kBaryTol && eta >= -kBaryTol && l0 >= -kBaryTol;
  }

  // t strictly inside the union of the three open ellipses of e
  // (SPEC.md:450-458): |t-P| + |t-Q| < 2a for side PQ.
  bool in_near(int64_t e, double tx, double ty) const {
    if (pr->near_model == 1) {
      const Ball B{two_a[3 * e], two_a[3 * e + 1], two_a[3 * e + 2]};
      return in_ball(B, pr->vxy[2 * pr->tri[3 * e]], pr->vxy[2 * pr->tri[3 * e] + 1], tx, ty);
    }
    if (all_near[e]) return true;
    const int32_t* id = pr->tri + 3 * e;
    double d[3];
    for (int k = 0; k < 3; ++k) {
      const double dx = tx - pr->vxy[2 * id[k]], dy = ty - pr->vxy[2 * id[k] + 1];
      d[k] = std::sqrt(dx * dx + dy * dy);
    }
    const double* ta = &two_a[3 * e];
    return (d[0] + d[1] < ta[0]) || (d[1] + d[2] < ta[1]) || (d[2] + d[0] < ta[2]);
  }

  // S(t) and the sorted N(t) for one target.
  void lists(double tx, double ty, int32_t& self, std::vector<int32_t>& near,
             std::vector<int>& scratch, double& sxi, double& seta) const {
    scratch.clear();
    int64_t visited = 0;
    qt.query(0, tx - query_half, ty - query_half, tx + query_half, ty + query_half, scratch,
             visited);
    std::vector<int32_t> cand;
    cand.reserve(scratch.size() / 2 + all_near_ids.size());
    for (int pt : scratch) cand.push_back(pt / 4);
    for (int32_t e : all_near_ids) cand.push_back(e);
    std::sort(cand.begin(), cand.end());
    cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
    self = -1;
    sxi = seta = 0.0;
    for (int32_t e : cand) {
      const double* b = &bb[4 * e];
      if (!all_near[e] && !(tx >= b[0] && tx <= b[2] && ty >= b[1] && ty <= b[3])) continue;
      double xi, eta;
      if (self < 0 && ref_coords(e, tx, ty, xi, eta)) {  // ties -> lowest id
        self = e;
        sxi = xi;
        seta = eta;
      }
    }
    near.clear();
    for (int32_t e : cand) {
      if (e == self) continue;
      const double* b = &bb[4 * e];
      if (!all_near[e] && !(tx >= b[0] && tx <= b[2] && ty >= b[1] && ty <= b[3])) continue;
      if (in_near(e, tx, ty)) near.push_back(e);
    }
  }

  // sum_{i in T} q_i log r^2: the far-sum contribution of element e's sources
  double subtract(int64_t e, double tx, double ty) const {
    const int L = pr->len_q;
    double s = 0.0;
    for (int i = 0; i < L; ++i) {
      const double dx = tx - sx[e * L + i], dy = ty - sy[e * L + i];
      const double r2 = dx * dx + dy * dy;
      if (r2 > 0.0) s += sq[e * L + i] * std::log(r2);
    }
    return s;
  }

  // near_eval: recursive 4-way midpoint
  // split of the reference simplex; a sub-simplex at depth d is accepted when
  // t lies outside its three-ellipse model built with the N_n rule and w
  // scaled by its area, rho_d = rho0n(T) 4^{-d/N_n}; rho_d <= 1 accepts
  // (collapsed ellipses).
  struct NearAcc {
    double sum = 0.0;
    int64_t leaves = 0, rho_le1 = 0;
    int32_t max_depth = 0;
    int err = 0;
  };
  // side lengths of the depth-0 image of the reference simplex (vertices
  // x0 + (xi e1 + eta e2), the sub-simplex vertex formula at depth 0)
  void side_lengths0(int64_t e, double l[3]) const {
    const double rx[3] = {0.0, 1.0, 0.0}, ry[3] = {0.0, 0.0, 1.0};
    double px[3], py[3];
    for (int k = 0; k < 3; ++k) {
      const double s0 = rx[k] * e1x[e], s1 = ry[k] * e2x[e];
      px[k] = x0[e] + (s0 + s1);
      const double t0 = rx[k] * e1y[e], t1 = ry[k] * e2y[e];
      py[k] = y0[e] + (t0 + t1);
    }
    for (int k = 0; k < 3; ++k) {
      const int k1 = (k + 1) % 3;
      const double dx = px[k1] - px[k], dy = py[k1] - py[k];
      l[k] = std::sqrt(dx * dx + dy * dy);
    }
  }

  void near_rec(int64_t e, double tx, double ty, const double a[2], const double b[2],
                const double c[2], int d, NearAcc& acc) const {
    if (d > kMaxNearDepth) {
      acc.err = 2;
      return;
    }
    const double X0 = x0[e], Y0 = y0[e];
    const double E1x = e1x[e], E1y = e1y[e], E2x = e2x[e], E2y = e2y[e];
    const double* vv[3] = {a, b, c};
    const bool cv = curved(e);
    double px[3], py[3];
    for (int k = 0; k < 3; ++k) {
      if (cv) {
        blend(bgeom(e), curve(e), vv[k][0], vv[k][1], px[k], py[k]);
        continue;
      }
      const double s0 = vv[k][0] * E1x, s1 = vv[k][1] * E2x;
      px[k] = X0 + (s0 + s1);
      const double t0 = vv[k][0] * E1y, t1 = vv[k][1] * E2y;
      py[k] = Y0 + (t0 + t1);
    }
    const double rd = rho0n[e] * kd[d];
    bool accept;
    if (pr->near_model == 1) {
      const Ball B = ball_of(px[0], py[0], px[1], py[1], px[2], py[2], pr->ball_factor);
      accept = d >= kBallMaxDepth || !in_ball(B, px[0], py[0], tx, ty);
    } else if (!(rd > 1.0)) {
      accept = true;
      acc.rho_le1++;
    } else {
      const double g = (rd + 1.0 / rd) * 0.5;
      double dist[3];
      for (int k = 0; k < 3; ++k) {
        const double dx = tx - px[k], dy = ty - py[k];
        dist[k] = std::sqrt(dx * dx + dy * dy);
      }
      // the midpoint split makes every depth-d sub-simplex congruent to the
      // element scaled by 2^-d with the same side order, so its side k has
      // length l_k 2^-d exactly (l_k of the depth-0 reference image)
      double l0[3];
      side_lengths0(e, l0);
      const double sc = std::ldexp(1.0, -d);
      bool nearp = false;
      for (int k = 0; k < 3 && !nearp; ++k) {
        const int k1 = (k + 1) % 3;
        double len;
        if (cv) {  // curved map: sub-simplices are not congruent; use their mapped chords
          const double sxk = px[k1] - px[k], syk = py[k1] - py[k];
          len = std::sqrt(sxk * sxk + syk * syk);
        } else {
          len = l0[k] * sc;
        }
        const double ta = g * len;
        if (dist[k] + dist[k1] < ta) nearp = true;
      }
      accept = !nearp;
    }
    if (accept) {
      acc.leaves++;
      acc.max_depth = std::max(acc.max_depth, d);
      const int Ln = pr->len_n;
      const double* cf = pr->coeffs + e * M;
      double s = 0.0;
      for (int i = 0; i < Ln; ++i) {
        const double u = pr->near_x[i], v = pr->near_y[i];
        const double xi = a[0] + (u * (b[0] - a[0]) + v * (c[0] - a[0]));
        const double eta = a[1] + (u * (b[1] - a[1]) + v * (c[1] - a[1]));
        double yx, yy;
        map_point(e, xi, eta, yx, yy);
        const double f = density(pr->p, cf, xi, eta);
        const double dx = tx - yx, dy = ty - yy;
        const double jw = cv ? jac_at(e, xi, eta) : 1.0;
        s += pr->near_w[i] * jw * f * std::log(dx * dx + dy * dy);
      }
      acc.sum += s * ((cv ? 1.0 : det[e]) * std::ldexp(1.0, -2 * d)) * kInv4Pi;
      return;
    }
    const double mab[2] = {(a[0] + b[0]) * 0.5, (a[1] + b[1]) * 0.5};
    const double mbc[2] = {(b[0] + c[0]) * 0.5, (b[1] + c[1]) * 0.5};
    const double mca[2] = {(c[0] + a[0]) * 0.5, (c[1] + a[1]) * 0.5};
    near_rec(e, tx, ty, a, mab, mca, d + 1, acc);
    near_rec(e, tx, ty, mab, b, mbc, d + 1, acc);
    near_rec(e, tx, ty, mca, mbc, c, d + 1, acc);
    near_rec(e, tx, ty, mbc, mca, mab, d + 1, acc);
  }

  int near_eval(int64_t e, double tx, double ty, NearAcc& acc) const {
    const double a[2] = {0.0, 0.0}, b[2] = {1.0, 0.0}, c[2] = {0.0, 1.0};
    near_rec(e, tx, ty, a, b, c, 0, acc);
    return acc.err;
  }

  // self_eval for straight triangles:
  // three sub-triangles (t, A, B); radius-arc-length coordinates with the
  // GGQ radial rule and composite Gauss-Legendre over dyadic panels refined
  // toward s~ = argmin |t - gamma(s)|; Jacobian |(gamma - t) x gamma'| = h.
  struct SelfAcc {
    double sum = 0.0;
    int64_t panels = 0, degenerate = 0;
  };
  // panel boundaries of [0, L] refined toward st
  static void panels_of(double st, double L, double dmin, std::vector<double>& bnd) {
    int N = 0;
    for (double x = st; !(x < dmin); x *= 0.5) ++N;
    int Mm = 0;
    for (double x = L - st; !(x < dmin); x *= 0.5) ++Mm;
    bnd.clear();
    bnd.push_back(0.0);
    for (int i = 1; i <= N; ++i) bnd.push_back(st - std::ldexp(st, -i));
    bnd.push_back(st);
    for (int i = Mm; i >= 1; --i) bnd.push_back(st + std::ldexp(L - st, -i));
    bnd.push_back(L);
  }

  // self_eval on a curved element: sub-element (t, gamma)
  // with Jacobian |(gamma(s) - t) x gamma'(s)| and r0(s) = |gamma(s) - t|;
  // the two straight sub-triangles as for triangles; the density at every
  // quadrature point through the Newton inverse of the blending map seeded
  // on the (r, s) line in reference coordinates.
  void self_eval_curved(int64_t e, double tx, double ty, double txi, double teta, SelfAcc& acc) const {
    const BlendGeom B = bgeom(e);
    const CurveC C = curve(e);
    const double* cf = pr->coeffs + e * M;
    const double vx[3] = {B.PLx, B.P0x, B.Ox}, vy[3] = {B.PLy, B.P0y, B.Oy};
    const double refx[3] = {0.0, 1.0, 0.0}, refy[3] = {0.0, 0.0, 1.0};
    double total = 0.0;
    std::vector<double> bnd;
    for (int k = 0; k < 3; ++k) {
      const int k1 = (k + 1) % 3;
      double L, st, dmin, hconst = 0.0;
      const bool arc = (k == 0);
      if (arc) {
        L = C.L;
        st = curved_argmin(C, tx, ty);
        double gx, gy;
        curve_eval(C, 1.0 - st / L, gx, gy);
        dmin = std::sqrt((tx - gx) * (tx - gx) + (ty - gy) * (ty - gy));
        // t on the arc: unlike a straight side, the sub-element (t, gamma)
        // keeps its area (the lens between the arc and the chords from t),
        // so it is not skipped; its integrand vanishes like
        // (s - s~)^2 log|s - s~| at s~, and the panels refine to 1e-9 L
        if (!(dmin > 1e-13 * L)) dmin = 1e-9 * L;
      } else {
        const double ABx = vx[k1] - vx[k], ABy = vy[k1] - vy[k];
        L = std::sqrt(ABx * ABx + ABy * ABy);
        const double vAx = tx - vx[k], vAy = ty - vy[k];
        const double cr = ABx * vAy - ABy * vAx;
        hconst = std::abs(cr) / L;
        if (!(hconst > 1e-13 * L)) {
          acc.degenerate++;
          continue;
        }
        const double sp = (vAx * ABx + vAy * ABy) / L;
        st = std::min(std::max(sp, 0.0), L);
        const double gx = vx[k] + (st / L) * ABx, gy = vy[k] + (st / L) * ABy;
        dmin = std::sqrt((tx - gx) * (tx - gx) + (ty - gy) * (ty - gy));
      }
      panels_of(st, L, dmin, bnd);
      double sub = 0.0;
      for (size_t pi = 0; pi + 1 < bnd.size(); ++pi) {
        const double s0 = bnd[pi], s1 = bnd[pi + 1];
        if (!(s1 > s0)) continue;
        acc.panels++;
        const double mid = 0.5 * (s0 + s1), half = 0.5 * (s1 - s0);
        for (int gq = 0; gq < pr->n_l; ++gq) {
          const double s = mid + half * pr->gl_x[gq];
          const double ws = half * pr->gl_w[gq];
          const double sl = s / L;
          double px, py, jf, grx, gry;
          if (arc) {
            double g[2], g1[2], g2[2];
            curve_eval_d(C, 1.0 - sl, g, g1, g2);
            px = g[0];
            py = g[1];
            const double tgx = -g1[0] / L, tgy = -g1[1] / L;
            jf = std::abs((px - tx) * tgy - (py - ty) * tgx);
            grx = sl;  // rho(xi, 0) = G(1 - xi) = gamma(xi L)
            gry = 0.0;
          } else {
            px = vx[k] + sl * (vx[k1] - vx[k]);
            py = vy[k] + sl * (vy[k1] - vy[k]);
            jf = hconst;
            grx = refx[k] + sl * (refx[k1] - refx[k]);
            gry = refy[k] + sl * (refy[k1] - refy[k]);
          }
          const double r0 = std::sqrt((px - tx) * (px - tx) + (py - ty) * (py - ty));
          const double lr0 = std::log(r0);
          double inner = 0.0;
          for (int j = 0; j <= pr->n_g; ++j) {
            const double rj = pr->ggq_r[j];
            const double yx = tx + rj * (px - tx), yy = ty + rj * (py - ty);
            double xi = txi + rj * (grx - txi), eta = teta + rj * (gry - teta);
            blend_inverse_tol(B, C, yx, yy, xi, eta);
            const double f = density(pr->p, cf, std::min(std::max(xi, 0.0), 1.0),
                                     std::min(std::max(eta, 0.0), 1.0 - std::min(std::max(xi, 0.0), 1.0)));
            inner += pr->ggq_w[j] * rj * (lr0 + std::log(rj)) * f;
          }
          sub += ws * jf * inner;
        }
      }
      total += sub;
    }
    acc.sum += total * kInv2Pi;
  }

  void self_eval(int64_t e, double tx, double ty, double txi, double teta, SelfAcc& acc) const {
    if (curved(e)) {
      self_eval_curved(e, tx, ty, txi, teta, acc);
      return;
    }
    const int32_t* id = pr->tri + 3 * e;
    const double refx[3] = {0.0, 1.0, 0.0}, refy[3] = {0.0, 0.0, 1.0};
    const double* cf = pr->coeffs + e * M;
    double total = 0.0;
    for (int k = 0; k < 3; ++k) {
      const int k1 = (k + 1) % 3;
      const double Ax = pr->vxy[2 * id[k]], Ay = pr->vxy[2 * id[k] + 1];
      const double Bx = pr->vxy[2 * id[k1]], By = pr->vxy[2 * id[k1] + 1];
      const double ABx = Bx - Ax, ABy = By - Ay;
      const double L = std::sqrt(ABx * ABx + ABy * ABy);
      const double vAx = tx - Ax, vAy = ty - Ay;
      const double cr = ABx * vAy - ABy * vAx;
      const double h = std::abs(cr) / L;
      if (!(h > 1e-13 * L)) {  // target on the side line: zero-area sub-triangle
        acc.degenerate++;
        continue;
      }
      const double sp = (vAx * ABx + vAy * ABy) / L;
      const double st = std::min(std::max(sp, 0.0), L);
      const double gx = Ax + (st / L) * ABx, gy = Ay + (st / L) * ABy;
      const double dmin = std::sqrt((tx - gx) * (tx - gx) + (ty - gy) * (ty - gy));
      // dyadic panel boundaries
      std::vector<double> bnd;
      int N = 0;
      for (double x = st; !(x < dmin); x *= 0.5) ++N;
      int Mm = 0;
      for (double x = L - st; !(x < dmin); x *= 0.5) ++Mm;
      bnd.push_back(0.0);
      for (int i = 1; i <= N; ++i) bnd.push_back(st - std::ldexp(st, -i));
      bnd.push_back(st);
      for (int i = Mm; i >= 1; --i) bnd.push_back(st + std::ldexp(L - st, -i));
      bnd.push_back(L);
      const double Arx = refx[k], Ary = refy[k];
      const double BRx = refx[k1] - refx[k], BRy = refy[k1] - refy[k];
      double sub = 0.0;
      for (size_t pi = 0; pi + 1 < bnd.size(); ++pi) {
        const double s0 = bnd[pi], s1 = bnd[pi + 1];
        if (!(s1 > s0)) continue;
        acc.panels++;
        const double mid = 0.5 * (s0 + s1), half = 0.5 * (s1 - s0);
        for (int gq = 0; gq < pr->n_l; ++gq) {
          const double s = mid + half * pr->gl_x[gq];
          const double ws = half * pr->gl_w[gq];
          const double sl = s / L;
          const double px = Ax + sl * ABx, py = Ay + sl * ABy;
          const double r0 = std::sqrt((px - tx) * (px - tx) + (py - ty) * (py - ty));
          const double lr0 = std::log(r0);
          const double grx = Arx + sl * BRx, gry = Ary + sl * BRy;
          double inner = 0.0;
          for (int j = 0; j <= pr->n_g; ++j) {
            const double rj = pr->ggq_r[j];
            const double yx = txi + rj * (grx - txi), yy = teta + rj * (gry - teta);
            const double f = density(pr->p, cf, yx, yy);
            inner += pr->ggq_w[j] * rj * (lr0 + std::log(rj)) * f;
          }
          sub += ws * inner;
        }
      }
      total += sub * h;
    }
    acc.sum += total * kInv2Pi;
  }
};

}  // namespace

extern "C" {

const char* vpo_last_error(void) {
  std::lock_guard<std::mutex> lk(g_err_mu);
  return g_err.c_str();
}

int vpo_koornwinder(int order, double x, double y, double* out) {
  if (order < 0 || order > kMaxOrder || !out) return fail(1, "koornwinder: order out of range");
  // koornwinder.hpp:117-120
  if (x < -1e-9 || y < -1e-9 || x + y > 1 + 1e-9)
    return fail(2, "koornwinder: point outside the reference simplex");
  koorn(order, x, y, out);
  return 0;
}

double vpo_cn_lookup(int n) { return cn_lookup(n); }

double vpo_w_edge(int len, const double* x, const double* y, const double* w) {
  if (len <= 0) return 0.0;
  return w_edge(len, x, y, w);
}

// rules.hpp:60-85
int vpo_validate_rule(int order, int len, const double* x, const double* y, const double* w) {
  if (len <= 0) return fail(2, "rule table: empty rule");
  if (order < 0 || order > kMaxOrder) return fail(1, "rule table: order out of range (invariant: 0 <= order <= 32)");
  double ws = 0.0;
  for (int i = 0; i < len; ++i) {
    if (w[i] <= 0.0) return fail(2, "rule table: non-positive weight (invariant: weights > 0)");
    if (x[i] < 0 || y[i] < 0 || x[i] + y[i] > 1) return fail(2, "rule table: node outside the simplex");
    ws += w[i];
  }
  if (std::abs(ws - 0.5) > 1e-13) return fail(2, "rule table: weights do not sum to the simplex area");
  const int d = ksize(order);
  std::vector<double> acc(d, 0.0), v(d);
  for (int i = 0; i < len; ++i) {
    koorn(order, x[i], y[i], v.data());
    for (int j = 0; j < d; ++j) acc[j] += w[i] * v[j];
  }
  acc[0] -= std::sqrt(2.0) * 0.5;
  for (int j = 0; j < d; ++j)
    if (std::abs(acc[j]) > 1e-12) return fail(2, "rule table: exactness check failed at declared order");
  return 0;
}

// gauss.hpp:17-46: Newton on the three-term recurrence from cos guesses
int vpo_gauss_legendre(int n, double* x, double* w) {
  if (n < 1) return fail(1, "gauss_legendre: order must be >= 1");
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
  return 0;
}

int vpo_quadtree_query(int64_t n_pts, const double* pts, int leaf_cap, double lox, double loy,
                       double hix, double hiy, int32_t* out, int64_t cap, int64_t* n_out,
                       int64_t* visited) {
  if (n_pts <= 0) return fail(1, "quadtree: empty input");
  if (leaf_cap < 1) return fail(1, "quadtree: leaf capacity must be >= 1");
  if (!(lox <= hix && loy <= hiy)) return fail(1, "quadtree: malformed rectangle");
  QTree t;
  t.build(n_pts, pts, leaf_cap);
  std::vector<int> res;
  int64_t vis = 0;
  t.query(0, lox, loy, hix, hiy, res, vis);
  std::sort(res.begin(), res.end());
  if (n_out) *n_out = (int64_t)res.size();
  if (visited) *visited = vis;
  if (out) {
    if ((int64_t)res.size() > cap) return fail(1, "quadtree: output capacity too small");
    for (size_t i = 0; i < res.size(); ++i) out[i] = res[i];
  }
  return 0;
}

int vpo_element_models(const vpo_problem* pr, double* rho0, double* rho0n, double* two_a) {
  Setup s;
  if (int rc = s.init(pr, true, false)) return rc;
  for (int64_t e = 0; e < s.E; ++e) {
    if (rho0) rho0[e] = s.rho0[e];
    if (rho0n) rho0n[e] = s.rho0n[e];
    if (two_a)
      for (int k = 0; k < 3; ++k) two_a[3 * e + k] = s.two_a[3 * e + k];
  }
  return 0;
}

int vpo_nearlist(const vpo_problem* pr, int64_t n_tgt, const double* txy, int32_t* self_out,
                 int64_t* offsets, int32_t* ids, int64_t ids_cap, int64_t* n_ids) {
  if (n_tgt < 0 || (n_tgt > 0 && !txy)) return fail(1, "nearlist: bad target array");
  Setup s;
  if (int rc = s.init(pr, true, false)) return rc;
  std::vector<std::vector<int32_t>> lists(n_tgt);
  std::vector<int32_t> selfv(n_tgt);
#pragma omp parallel
  {
    std::vector<int> scratch;
    std::vector<int32_t> nl;
#pragma omp for schedule(dynamic, 64)
    for (int64_t t = 0; t < n_tgt; ++t) {
      double a, b;
      s.lists(txy[2 * t], txy[2 * t + 1], selfv[t], nl, scratch, a, b);
      lists[t] = nl;
    }
  }
  int64_t tot = 0;
  for (int64_t t = 0; t < n_tgt; ++t) tot += (int64_t)lists[t].size();
  if (n_ids) *n_ids = tot;
  if (self_out)
    for (int64_t t = 0; t < n_tgt; ++t) self_out[t] = selfv[t];
  if (offsets) {
    offsets[0] = 0;
    for (int64_t t = 0; t < n_tgt; ++t) offsets[t + 1] = offsets[t] + (int64_t)lists[t].size();
  }
  if (ids) {
    if (tot > ids_cap) return fail(1, "nearlist: ids capacity too small");
    int64_t o = 0;
    for (int64_t t = 0; t < n_tgt; ++t)
      for (int32_t e : lists[t]) ids[o++] = e;
  }
  return 0;
}

int vpo_sources(const vpo_problem* pr, double* sx, double* sy, double* q) {
  Setup s;
  if (int rc = s.init(pr, false, true)) return rc;
  const size_t n = s.sx.size();
  std::memcpy(sx, s.sx.data(), n * sizeof(double));
  std::memcpy(sy, s.sy.data(), n * sizeof(double));
  std::memcpy(q, s.sq.data(), n * sizeof(double));
  return 0;
}

// Neumaier-compensated direct sum (fmm_eval direct path, SPEC.md:572-580,
// :618).  Targets go four at a time through one sweep of the sources (each
// target keeps its own sum in source order, so the bits are those of the
// one-target loop); the sweep is what costs memory bandwidth on the host.
static inline void neumaier(double& sum, double& comp, double term) {
  const double tt = sum + term;
  if (std::abs(sum) >= std::abs(term))
    comp += (sum - tt) + term;
  else
    comp += (term - tt) + sum;
  sum = tt;
}

static void far_sum_impl(const Setup& s, int64_t n_tgt, const double* txy, double* u_far) {
  const int64_t S = (int64_t)s.sx.size();
  const double* sx = s.sx.data();
  const double* sy = s.sy.data();
  const double* sq = s.sq.data();
  constexpr int B = 4;
  const int64_t nb = (n_tgt + B - 1) / B;
#pragma omp for schedule(dynamic, 1)
  for (int64_t blk = 0; blk < nb; ++blk) {
    const int64_t t0 = blk * B;
    const int nt = (int)std::min<int64_t>(B, n_tgt - t0);
    double tx[B], ty[B], sum[B], comp[B];
    for (int k = 0; k < B; ++k) {
      const int64_t t = t0 + std::min(k, nt - 1);
      tx[k] = txy[2 * t];
      ty[k] = txy[2 * t + 1];
      sum[k] = comp[k] = 0.0;
    }
    for (int64_t j = 0; j < S; ++j) {
      const double xj = sx[j], yj = sy[j], qj = sq[j];
      for (int k = 0; k < B; ++k) {
        const double dx = tx[k] - xj, dy = ty[k] - yj;
        const double r2 = dx * dx + dy * dy;
        if (!(r2 > 0.0)) continue;  // coincident pair contributes 0
        neumaier(sum[k], comp[k], qj * std::log(r2));
      }
    }
    for (int k = 0; k < nt; ++k) u_far[t0 + k] = sum[k] + comp[k];
  }
}

int vpo_far_sum(const vpo_problem* pr, int64_t n_tgt, const double* txy, int nthreads,
                double* u_far) {
  Setup s;
  if (int rc = s.init(pr, false, true)) return rc;
#ifdef _OPENMP
  const int nt = nthreads > 0 ? nthreads : omp_get_max_threads();
#pragma omp parallel num_threads(nt)
#endif
  far_sum_impl(s, n_tgt, txy, u_far);
  return 0;
}

int vpo_near_pair(const vpo_problem* pr, double tx, double ty, int32_t elem, double* val,
                  double* sub, int64_t* leaves, int32_t* depth) {
  Setup s;
  if (int rc = s.init(pr, true, true)) return rc;
  if (elem < 0 || elem >= s.E) return fail(1, "near_pair: element out of range");
  Setup::NearAcc acc;
  if (s.near_eval(elem, tx, ty, acc))
    return fail(2, "near_eval: recursion depth > 40 (target effectively on element boundary)");
  if (val) *val = acc.sum;
  if (sub) *sub = s.subtract(elem, tx, ty);
  if (leaves) *leaves = acc.leaves;
  if (depth) *depth = acc.max_depth;
  return 0;
}

int vpo_self(const vpo_problem* pr, double tx, double ty, int32_t elem, double* val, double* sub,
             int64_t* panels) {
  Setup s;
  if (int rc = s.init(pr, false, true)) return rc;
  if (elem < 0 || elem >= s.E) return fail(1, "self: element out of range");
  // reference coordinates via the inverse element map
  double xi, eta;
  s.ref_coords(elem, tx, ty, xi, eta);
  Setup::SelfAcc acc;
  s.self_eval(elem, tx, ty, xi, eta, acc);
  if (val) *val = acc.sum;
  if (sub) *sub = s.subtract(elem, tx, ty);
  if (panels) *panels = acc.panels;
  return 0;
}

static int evaluate_setup(const Setup& s, int64_t n_tgt, const double* txy, int nthreads, double* u,
                          double* u_far, vpo_stats* st) {
  const vpo_problem* pr = s.pr;
  if (n_tgt < 0 || (n_tgt > 0 && (!txy || !u))) return fail(1, "evaluate: bad target array");
  if (pr->n_l <= 0 || pr->n_g < 0 || !pr->gl_x || !pr->ggq_r) return fail(1, "evaluate: missing self rules");
  std::vector<double> uf(n_tgt);
  int64_t outside = 0, npairs = 0, nself = 0, leaves = 0, panels = 0, rle1 = 0, degen = 0;
  int32_t maxd = 0;
  std::atomic<int> err{0};
#ifdef _OPENMP
  const int nt = nthreads > 0 ? nthreads : omp_get_max_threads();
#pragma omp parallel num_threads(nt)
#endif
  {
    far_sum_impl(s, n_tgt, txy, uf.data());
    std::vector<int> scratch;
    std::vector<int32_t> nl;
#pragma omp for schedule(dynamic, 16) reduction(+ : outside, npairs, nself, leaves, panels, rle1, degen) reduction(max : maxd)
    for (int64_t t = 0; t < n_tgt; ++t) {
      const double tx = txy[2 * t], ty = txy[2 * t + 1];
      int32_t self;
      double xi, eta;
      s.lists(tx, ty, self, nl, scratch, xi, eta);
      // subtract-and-add
      double corr = 0.0;
      for (int32_t e : nl) {
        Setup::NearAcc acc;
        if (s.near_eval(e, tx, ty, acc)) err = 2;
        corr += acc.sum - s.subtract(e, tx, ty);
        leaves += acc.leaves;
        rle1 += acc.rho_le1;
        maxd = std::max(maxd, acc.max_depth);
      }
      npairs += (int64_t)nl.size();
      if (self >= 0) {
        Setup::SelfAcc sa;
        s.self_eval(self, tx, ty, xi, eta, sa);
        corr += sa.sum - s.subtract(self, tx, ty);
        panels += sa.panels;
        degen += sa.degenerate;
        nself++;
      } else {
        outside++;
      }
      u[t] = uf[t] + corr;
    }
  }
  if (err) return fail(2, "near_eval: recursion depth > 40 (target effectively on element boundary)");
  if (u_far) std::memcpy(u_far, uf.data(), n_tgt * sizeof(double));
  if (st) {
    st->n_targets = n_tgt;
    st->n_outside = outside;
    st->n_near_pairs = npairs;
    st->n_self = nself;
    st->n_leaves = leaves;
    st->n_panels = panels;
    st->n_rho_le1 = rle1;
    st->n_degenerate = degen;
    st->max_depth = maxd;
    st->pad = 0;
  }
  return 0;
}

int vpo_evaluate(const vpo_problem* pr, int64_t n_tgt, const double* txy, int nthreads,
                 double* u, double* u_far, vpo_stats* st) {
  Setup s;
  if (int rc = s.init(pr, true, true)) return rc;
  return evaluate_setup(s, n_tgt, txy, nthreads, u, u_far, st);
}

}  // extern "C"

struct vpo_ctx {
  Setup s;
};

extern "C" {

int vpo_open(const vpo_problem* pr, vpo_ctx** out) {
  if (!out) return fail(1, "open: null output");
  *out = nullptr;
  vpo_ctx* c = new vpo_ctx;
  if (int rc = c->s.init(pr, true, true)) {
    delete c;
    return rc;
  }
  *out = c;
  return 0;
}

int vpo_ctx_evaluate(vpo_ctx* c, int64_t n_tgt, const double* txy, int nthreads, double* u, double* u_far,
                     vpo_stats* st) {
  if (!c) return fail(1, "evaluate: null context");
  return evaluate_setup(c->s, n_tgt, txy, nthreads, u, u_far, st);
}

void vpo_close(vpo_ctx* c) { delete c; }

}  // extern "C"
