// vp_curves.cpp -- arc-length boundary curves for curved elements
// (the reference's curve layer, curve.hpp:16-332, and the
// mesher's annotate_boundary).  Host-only setup code: it
// turns a closed parametric curve into per-element Legendre series of the
// arc-length parametrisation that vp_set_curves consumes.
//
// Design (not a translation of curve.hpp): lengths by composite
// Gauss-Legendre in long double over panels that split at every
// non-smooth point of the curve (Hermite knots), s -> t by a bracketed
// Newton iteration on the exact partial integral (no interpolant, so
// positions are accurate to rounding), closest points by sampling plus
// Newton on (Gamma(s) - v) . Gamma'(s) = 0.
#include <algorithm>
#include <cmath>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "vp_setup.h"

namespace {

typedef long double ld;
constexpr ld kPiL = 3.141592653589793238462643383279502884L;

std::mutex g_mu;
std::string g_err;
int fail(int code, const std::string& m) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_err = m;
  return code;
}

// Gauss-Legendre on [-1, 1] in long double
void gl_ld(int n, std::vector<ld>& x, std::vector<ld>& w) {
  x.resize(n);
  w.resize(n);
  for (int i = 0; i < n; ++i) {
    ld z = cosl(kPiL * (i + 0.75L) / (n + 0.5L)), dp = 0.0L;
    for (int it = 0; it < 100; ++it) {
      ld p0 = 1.0L, p1 = z;
      for (int k = 1; k < n; ++k) {
        const ld p2 = ((2 * k + 1) * z * p1 - k * p0) / (k + 1);
        p0 = p1;
        p1 = p2;
      }
      dp = n * (p0 - z * p1) / (1.0L - z * z);
      const ld dz = p1 / dp;
      z -= dz;
      if (fabsl(dz) < 1e-19L) break;
    }
    x[i] = z;
    w[i] = 2.0L / ((1.0L - z * z) * dp * dp);
  }
}

constexpr int kGL = 24;        // nodes per length panel
constexpr int kUniform = 1024; // uniform panels in t (plus knots)

}  // namespace

struct vps_curve {
  int kind = 0;
  std::vector<ld> prm;
  std::vector<ld> ht, hx, hy, hdx, hdy;  // Hermite samples
  std::vector<ld> brk;                   // panel breakpoints in t, brk[0] = 0, back = 1
  std::vector<ld> pre;                   // arc length at brk
  std::vector<ld> gx, gw;                // GL rule
  ld L = 0.0L;
  bool ccw = true;

  // position p, derivative d, second derivative dd at parameter t
  void eval(ld t, ld p[2], ld d[2], ld dd[2]) const {
    switch (kind) {
      case VPS_CURVE_CIRCLE: {
        const ld a = 2 * kPiL * t, r = prm[2], k = 2 * kPiL * r, k2 = 4 * kPiL * kPiL * r;
        p[0] = prm[0] + r * cosl(a); p[1] = prm[1] + r * sinl(a);
        d[0] = -k * sinl(a); d[1] = k * cosl(a);
        dd[0] = -k2 * cosl(a); dd[1] = -k2 * sinl(a);
        return;
      }
      case VPS_CURVE_ELLIPSE: {
        const ld u = 2 * kPiL * t, a = prm[0], b = prm[1], k = 2 * kPiL, k2 = k * k;
        p[0] = a * cosl(u); p[1] = b * sinl(u);
        d[0] = -k * a * sinl(u); d[1] = k * b * cosl(u);
        dd[0] = -k2 * a * cosl(u); dd[1] = -k2 * b * sinl(u);
        return;
      }
      case VPS_CURVE_WOBBLY: {  // r(theta) = a + b cos(k theta)
        const ld u = 2 * kPiL * t, a = prm[0], b = prm[1], kk = prm[2];
        const ld r = a + b * cosl(kk * u), rp = -b * kk * sinl(kk * u), rpp = -b * kk * kk * cosl(kk * u);
        const ld c = cosl(u), s = sinl(u), k = 2 * kPiL, k2 = k * k;
        p[0] = r * c; p[1] = r * s;
        d[0] = k * (rp * c - r * s); d[1] = k * (rp * s + r * c);
        dd[0] = k2 * ((rpp - r) * c - 2 * rp * s); dd[1] = k2 * ((rpp - r) * s + 2 * rp * c);
        return;
      }
      case VPS_CURVE_ARC: {  // (cx, cy, r, th0, th1): theta = th0 + t (th1 - th0)
        const ld w = prm[4] - prm[3], a = prm[3] + t * w, r = prm[2];
        p[0] = prm[0] + r * cosl(a); p[1] = prm[1] + r * sinl(a);
        d[0] = -r * w * sinl(a); d[1] = r * w * cosl(a);
        dd[0] = -r * w * w * cosl(a); dd[1] = -r * w * w * sinl(a);
        return;
      }
      default: {  // periodic cubic Hermite
        const size_t n = ht.size();
        t -= floorl(t);
        size_t i = std::upper_bound(ht.begin(), ht.end(), t) - ht.begin();
        i = i == 0 ? n - 1 : i - 1;
        const ld ta = ht[i], tb = i + 1 < n ? ht[i + 1] : ht[0] + 1.0L;
        if (i == n - 1 && t < ta) t += 1.0L;
        const size_t j = (i + 1) % n;
        const ld h = tb - ta, u = (t - ta) / h;
        // basis h00 = 2u^3-3u^2+1, h10 = u^3-2u^2+u, h01 = -2u^3+3u^2, h11 = u^3-u^2
        const ld b0 = (2 * u - 3) * u * u + 1, b1 = ((u - 2) * u + 1) * u, b2 = (3 - 2 * u) * u * u, b3 = (u - 1) * u * u;
        const ld d0 = 6 * u * (u - 1), d1 = (3 * u - 4) * u + 1, d2 = 6 * u * (1 - u), d3 = (3 * u - 2) * u;
        const ld e0 = 12 * u - 6, e1 = 6 * u - 4, e2 = 6 - 12 * u, e3 = 6 * u - 2;
        const ld ma[2] = {hdx[i] * h, hdy[i] * h}, mb[2] = {hdx[j] * h, hdy[j] * h};
        const ld pa[2] = {hx[i], hy[i]}, pb[2] = {hx[j], hy[j]};
        for (int c = 0; c < 2; ++c) {
          p[c] = pa[c] * b0 + ma[c] * b1 + pb[c] * b2 + mb[c] * b3;
          d[c] = (pa[c] * d0 + ma[c] * d1 + pb[c] * d2 + mb[c] * d3) / h;
          dd[c] = (pa[c] * e0 + ma[c] * e1 + pb[c] * e2 + mb[c] * e3) / (h * h);
        }
        return;
      }
    }
  }
  ld speed(ld t) const {
    ld p[2], d[2], dd[2];
    eval(t, p, d, dd);
    return sqrtl(d[0] * d[0] + d[1] * d[1]);
  }
  // arc length over [a, b] inside one panel
  ld seglen(ld a, ld b) const {
    ld s = 0.0L;
    for (int k = 0; k < kGL; ++k) s += gw[k] * speed(0.5L * (a + b) + 0.5L * (b - a) * gx[k]);
    return 0.5L * (b - a) * s;
  }
  // s in [0, L] -> t in [0, 1]
  ld param(ld s) const {
    if (s <= 0.0L) return 0.0L;
    if (s >= L) return 1.0L;
    size_t k = std::upper_bound(pre.begin(), pre.end(), s) - pre.begin();
    k = k == 0 ? 0 : std::min(k - 1, brk.size() - 2);
    const ld a = brk[k], b = brk[k + 1];
    ld lo = a, hi = b;
    ld t = a + (s - pre[k]) / (pre[k + 1] - pre[k]) * (b - a);
    for (int it = 0; it < 60; ++it) {
      const ld f = pre[k] + seglen(a, t) - s;
      if (f > 0) hi = t; else lo = t;
      const ld sp = speed(t);
      ld tn = sp > 0 ? t - f / sp : 0.5L * (lo + hi);
      if (!(tn > lo && tn < hi)) tn = 0.5L * (lo + hi);  // safeguard: stay in the bracket
      const ld dt = tn - t;
      t = tn;
      if (fabsl(dt) < 1e-19L * (1.0L + fabsl(t))) break;
    }
    return t;
  }
  ld wrap(ld s) const {
    s -= L * floorl(s / L);
    if (s >= L) s -= L;
    return s;
  }
  // position and unit tangent at arc length s
  void point(ld s, ld p[2], ld tan[2], ld curv[2]) const {
    ld d[2], dd[2];
    eval(param(wrap(s)), p, d, dd);
    const ld n2 = d[0] * d[0] + d[1] * d[1], n = sqrtl(n2);
    tan[0] = d[0] / n;
    tan[1] = d[1] / n;
    const ld dot = d[0] * dd[0] + d[1] * dd[1];
    curv[0] = (dd[0] - d[0] * dot / n2) / n2;  // d2 Gamma / ds2
    curv[1] = (dd[1] - d[1] * dot / n2) / n2;
  }
};

extern "C" {

int vps_curve_create(int kind, const double* params, int n_params, vps_curve** out) {
  if (!out) return fail(1, "curve: null output");
  *out = nullptr;
  auto c = std::make_unique<vps_curve>();
  c->kind = kind;
  gl_ld(kGL, c->gx, c->gw);
  std::vector<ld> knots;
  switch (kind) {
    case VPS_CURVE_CIRCLE:
      if (n_params != 3 || !(params[2] > 0)) return fail(1, "curve: circle needs (cx, cy, r > 0)");
      break;
    case VPS_CURVE_ELLIPSE:
      if (n_params != 2 || !(params[0] > 0) || !(params[1] > 0)) return fail(1, "curve: ellipse needs (a > 0, b > 0)");
      break;
    case VPS_CURVE_WOBBLY:
      if (n_params != 3) return fail(1, "curve: wobbly ellipse needs (a, b, k)");
      if (!(params[0] > std::abs(params[1]))) return fail(1, "wobbly: need a > |b|");
      break;
    case VPS_CURVE_ARC:
      if (n_params != 5 || !(params[2] > 0)) return fail(1, "curve: arc needs (cx, cy, r > 0, th0, th1)");
      break;
    case VPS_CURVE_HERMITE: {
      if (n_params < 15 || n_params % 5 != 0) return fail(1, "hermite curve: need >= 3 consistent samples");
      const int n = n_params / 5;
      for (int i = 0; i < n; ++i) {
        c->ht.push_back(params[5 * i]);
        c->hx.push_back(params[5 * i + 1]);
        c->hy.push_back(params[5 * i + 2]);
        c->hdx.push_back(params[5 * i + 3]);
        c->hdy.push_back(params[5 * i + 4]);
      }
      for (int i = 1; i < n; ++i)
        if (!(c->ht[i] > c->ht[i - 1])) return fail(1, "hermite curve: parameters must increase");
      if (c->ht.front() < 0 || c->ht.back() >= 1.0L) return fail(1, "hermite curve: parameters must lie in [0,1)");
      knots = c->ht;
      break;
    }
    default:
      return fail(1, "curve: unknown kind");
  }
  for (int i = 0; i < n_params; ++i)
    if (!std::isfinite(params[i])) return fail(1, "curve: non-finite parameter");
  if (kind != VPS_CURVE_HERMITE) c->prm.assign(params, params + n_params);
  // panels: uniform grid plus the curve's non-smooth points
  for (int i = 0; i <= kUniform; ++i) c->brk.push_back((ld)i / kUniform);
  for (ld k : knots) c->brk.push_back(k);
  std::sort(c->brk.begin(), c->brk.end());
  c->brk.erase(std::unique(c->brk.begin(), c->brk.end(), [](ld a, ld b) { return fabsl(a - b) < 1e-15L; }),
               c->brk.end());
  c->pre.assign(c->brk.size(), 0.0L);
  ld area2 = 0.0L;
  for (size_t i = 0; i + 1 < c->brk.size(); ++i) {
    const ld a = c->brk[i], b = c->brk[i + 1];
    ld len = 0.0L;
    for (int k = 0; k < kGL; ++k) {
      const ld t = 0.5L * (a + b) + 0.5L * (b - a) * c->gx[k];
      ld p[2], d[2], dd[2];
      c->eval(t, p, d, dd);
      len += c->gw[k] * sqrtl(d[0] * d[0] + d[1] * d[1]);
      area2 += 0.5L * (b - a) * c->gw[k] * (p[0] * d[1] - p[1] * d[0]);
    }
    c->pre[i + 1] = c->pre[i] + 0.5L * (b - a) * len;
  }
  c->L = c->pre.back();
  c->ccw = area2 > 0.0L;
  if (!(c->L > 0.0L)) return fail(2, "curve: zero length");
  ld p0[2], p1[2], d[2], dd[2];
  c->eval(0.0L, p0, d, dd);
  c->eval(1.0L, p1, d, dd);
  if (kind != VPS_CURVE_HERMITE && hypotl(p0[0] - p1[0], p0[1] - p1[1]) > 1e-8L * c->L)
    return fail(1, "reparametrize: curve is not closed");
  *out = c.release();
  return 0;
}

void vps_curve_destroy(vps_curve* c) { delete c; }

double vps_curve_length(const vps_curve* c) { return c ? (double)c->L : 0.0; }

int vps_curve_ccw(const vps_curve* c) { return c && c->ccw ? 1 : 0; }

int vps_curve_param(const vps_curve* c, double s, double* t) {
  if (!c || !t) return fail(1, "curve: null argument");
  *t = (double)c->param(c->wrap(s));
  return 0;
}

int vps_curve_points(const vps_curve* c, int64_t n, const double* s, double* xy, double* tangent, double* dd) {
  if (!c || !s || !xy) return fail(1, "curve: null argument");
  for (int64_t i = 0; i < n; ++i) {
    ld p[2], tn[2], cv[2];
    c->point(s[i], p, tn, cv);
    xy[2 * i] = (double)p[0];
    xy[2 * i + 1] = (double)p[1];
    if (tangent) {
      tangent[2 * i] = (double)tn[0];
      tangent[2 * i + 1] = (double)tn[1];
    }
    if (dd) {
      dd[2 * i] = (double)cv[0];
      dd[2 * i + 1] = (double)cv[1];
    }
  }
  return 0;
}

int vps_curve_closest(const vps_curve* c, int64_t n, const double* xy, double* s_out, double* dist_out) {
  if (!c || !xy || !s_out) return fail(1, "curve: null argument");
  constexpr int kSamples = 2048;
  std::vector<ld> sp(2 * kSamples);
  for (int i = 0; i < kSamples; ++i) {
    ld p[2], tn[2], cv[2];
    c->point(c->L * i / kSamples, p, tn, cv);
    sp[2 * i] = p[0];
    sp[2 * i + 1] = p[1];
  }
  for (int64_t q = 0; q < n; ++q) {
    const ld vx = xy[2 * q], vy = xy[2 * q + 1];
    int best = 0;
    ld bd = 1e300L;
    for (int i = 0; i < kSamples; ++i) {
      const ld d2 = (sp[2 * i] - vx) * (sp[2 * i] - vx) + (sp[2 * i + 1] - vy) * (sp[2 * i + 1] - vy);
      if (d2 < bd) {
        bd = d2;
        best = i;
      }
    }
    ld s = c->L * best / kSamples;
    const ld h = c->L / kSamples;
    for (int it = 0; it < 40; ++it) {
      ld p[2], tn[2], cv[2];
      c->point(s, p, tn, cv);
      const ld dx = p[0] - vx, dy = p[1] - vy;
      const ld phi = dx * tn[0] + dy * tn[1];
      const ld dphi = 1.0L + dx * cv[0] + dy * cv[1];
      ld step = dphi > 0 ? phi / dphi : phi;
      step = std::max(-h, std::min(h, step));  // stay near the sampled basin
      s -= step;
      if (fabsl(step) < 1e-17L * c->L) break;
    }
    s = c->wrap(s);
    ld p[2], tn[2], cv[2];
    c->point(s, p, tn, cv);
    s_out[q] = (double)s;
    if (dist_out) dist_out[q] = (double)hypotl(p[0] - vx, p[1] - vy);
  }
  return 0;
}

// G(tau) = Gamma(s_from + tau (s_to - s_from)) as a degree-deg Legendre series
int vps_curve_segment(const vps_curve* c, double s_from, double s_to, int deg, double* gx, double* gy,
                      double* len) {
  if (!c || !gx || !gy) return fail(1, "curve: null argument");
  if (deg < 1 || deg > 64) return fail(1, "curve_segment: deg in [1, 64]");
  if (!(s_to != s_from)) return fail(1, "curve_segment: empty segment");
  const int nq = deg + 12;
  std::vector<ld> x, w;
  gl_ld(nq, x, w);
  std::vector<ld> px(nq), py(nq), P(nq);
  for (int i = 0; i < nq; ++i) {
    const ld tau = 0.5L * (1.0L + x[i]);
    ld p[2], tn[2], cv[2];
    c->point((ld)s_from + tau * ((ld)s_to - (ld)s_from), p, tn, cv);
    px[i] = p[0];
    py[i] = p[1];
  }
  std::vector<ld> p0(nq, 1.0L), p1(x);
  for (int n = 0; n <= deg; ++n) {
    const std::vector<ld>& pn = n == 0 ? p0 : p1;
    ld ax = 0.0L, ay = 0.0L;
    for (int i = 0; i < nq; ++i) {
      ax += w[i] * px[i] * pn[i];
      ay += w[i] * py[i] * pn[i];
    }
    gx[n] = (double)(ax * (2 * n + 1) / 2.0L);
    gy[n] = (double)(ay * (2 * n + 1) / 2.0L);
    if (n >= 1) {  // advance P_{n-1}, P_n -> P_n, P_{n+1}
      for (int i = 0; i < nq; ++i) {
        const ld p2 = ((2 * n + 1) * x[i] * p1[i] - n * p0[i]) / (n + 1);
        p0[i] = p1[i];
        p1[i] = p2;
      }
    }
  }
  if (len) *len = std::abs(s_to - s_from);
  return 0;
}

const char* vps_curve_last_error(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  return g_err.c_str();
}

}  // extern "C"
