// vp_curve.cuh -- curved (blending-map) elements, SURVEY.md §8(f3).
//
// A curved element stores its vertices as (gamma(L), gamma(0), O) and its
// curved side as a Legendre series gamma(tau L) = G(tau) = sum_n c_n
// P_n(2 tau - 1), tau in [0, 1].  The
// blending map rho(xi, eta) sends (0,0) -> gamma(L), (1,0) -> gamma(0),
// (0,1) -> O and the reference side eta = 0 onto gamma.
//
// Every function is templated on X: X = true rounds each operation
// separately (__dadd_rn & co. on the device, plain operations on the host
// built with -ffp-contract=off) in the operation order of the oracle
// (oracle/vp_oracle.cpp curve_eval .. curved_argmin), so the predicates that
// decide lists, leaf counts and panel counts are bit-identical; X = false
// lets the compiler contract to FMA for the quadrature values.
#pragma once
#include <cstdint>

namespace vp {

struct CurvesDev {
  const int32_t* ecurve;  // [E] curve id, -1 straight; nullptr: no curved elements
  const double* cx;       // [n_curves * (D+1)]
  const double* cy;
  const double* len;      // [n_curves] arc length L
  int D;
  int pad;
};

struct CurveRef {
  const double* cx;
  const double* cy;
  int D;
  double L;
};

template <bool X>
__host__ __device__ __forceinline__ double c_add(double a, double b) {
#ifdef __CUDA_ARCH__
  if constexpr (X) return __dadd_rn(a, b);
#endif
  return a + b;
}
template <bool X>
__host__ __device__ __forceinline__ double c_sub(double a, double b) {
#ifdef __CUDA_ARCH__
  if constexpr (X) return __dsub_rn(a, b);
#endif
  return a - b;
}
template <bool X>
__host__ __device__ __forceinline__ double c_mul(double a, double b) {
#ifdef __CUDA_ARCH__
  if constexpr (X) return __dmul_rn(a, b);
#endif
  return a * b;
}
__host__ __device__ __forceinline__ double c_div(double a, double b) { return a / b; }  // IEEE on both sides
__host__ __device__ __forceinline__ double c_sqrt(double a) {
#ifdef __CUDA_ARCH__
  return __dsqrt_rn(a);
#else
  return std::sqrt(a);
#endif
}

// Legendre recurrence P_{n+1} = la_n x P_n - lb_n P_{n-1}, la_n = (2n+1)/(n+1),
// lb_n = n/(n+1): the X = false paths multiply instead of dividing
constexpr int kMaxCurveDeg = 64;
__host__ __device__ __forceinline__ double leg_la(int n) { return (double)(2 * n + 1) / (double)(n + 1); }
__host__ __device__ __forceinline__ double leg_lb(int n) { return (double)n / (double)(n + 1); }
#ifdef __CUDACC__
__constant__ double c_leg_la[kMaxCurveDeg + 1], c_leg_lb[kMaxCurveDeg + 1];
#endif
__host__ __device__ __forceinline__ double p_next(int n, double x, double p1, double p0) {
#ifdef __CUDA_ARCH__
  return fma(c_leg_la[n] * x, p1, -c_leg_lb[n] * p0);
#else
  return leg_la(n) * x * p1 - leg_lb(n) * p0;
#endif
}

template <bool X>
__host__ __device__ inline void curve_eval(const CurveRef& C, double tau, double& gx, double& gy) {
  const double x = c_sub<X>(c_mul<X>(2.0, tau), 1.0);
  double p0 = 1.0, p1 = x;
  gx = C.cx[0];
  gy = C.cy[0];
  if (C.D >= 1) {
    gx = c_add<X>(gx, c_mul<X>(C.cx[1], x));
    gy = c_add<X>(gy, c_mul<X>(C.cy[1], x));
  }
  for (int n = 1; n < C.D; ++n) {
    double p2;
    if constexpr (X) {
      const double a = c_mul<X>((double)(2 * n + 1), x);
      const double b = c_mul<X>(a, p1);
      const double c = c_mul<X>((double)n, p0);
      p2 = c_div(c_sub<X>(b, c), (double)(n + 1));
    } else {
      p2 = p_next(n, x, p1, p0);
    }
    gx = c_add<X>(gx, c_mul<X>(C.cx[n + 1], p2));
    gy = c_add<X>(gy, c_mul<X>(C.cy[n + 1], p2));
    p0 = p1;
    p1 = p2;
  }
}

// G, dG/dtau, d2G/dtau2
template <bool X>
__host__ __device__ inline void curve_eval_d(const CurveRef& C, double tau, double g[2], double g1[2],
                                             double g2[2]) {
  const double x = c_sub<X>(c_mul<X>(2.0, tau), 1.0);
  double p0 = 1.0, p1 = x, d0 = 0.0, d1 = 1.0, e0 = 0.0, e1 = 0.0;
  g[0] = C.cx[0];
  g[1] = C.cy[0];
  g1[0] = g1[1] = g2[0] = g2[1] = 0.0;
  if (C.D >= 1) {
    g[0] = c_add<X>(g[0], c_mul<X>(C.cx[1], x));
    g[1] = c_add<X>(g[1], c_mul<X>(C.cy[1], x));
    g1[0] = c_add<X>(g1[0], c_mul<X>(C.cx[1], d1));
    g1[1] = c_add<X>(g1[1], c_mul<X>(C.cy[1], d1));
  }
  for (int n = 1; n < C.D; ++n) {
    const double k2 = (double)(2 * n + 1);
    double p2;
    if constexpr (X) {
      const double a = c_mul<X>(k2, x);
      p2 = c_div(c_sub<X>(c_mul<X>(a, p1), c_mul<X>((double)n, p0)), (double)(n + 1));
    } else {
      p2 = p_next(n, x, p1, p0);
    }
    const double d2 = c_add<X>(d0, c_mul<X>(k2, p1));
    const double e2 = c_add<X>(e0, c_mul<X>(k2, d1));
    const double cxn = C.cx[n + 1], cyn = C.cy[n + 1];
    g[0] = c_add<X>(g[0], c_mul<X>(cxn, p2));
    g[1] = c_add<X>(g[1], c_mul<X>(cyn, p2));
    g1[0] = c_add<X>(g1[0], c_mul<X>(cxn, d2));
    g1[1] = c_add<X>(g1[1], c_mul<X>(cyn, d2));
    g2[0] = c_add<X>(g2[0], c_mul<X>(cxn, e2));
    g2[1] = c_add<X>(g2[1], c_mul<X>(cyn, e2));
    p0 = p1; p1 = p2; d0 = d1; d1 = d2; e0 = e1; e1 = e2;
  }
  g1[0] = c_mul<X>(2.0, g1[0]);
  g1[1] = c_mul<X>(2.0, g1[1]);
  g2[0] = c_mul<X>(4.0, g2[0]);
  g2[1] = c_mul<X>(4.0, g2[1]);
}

// G and dG/dtau only (the Newton steps never need G''); same operations as
// curve_eval_d for the two outputs
template <bool X>
__host__ __device__ inline void curve_eval_d1(const CurveRef& C, double tau, double g[2], double g1[2]) {
  const double x = c_sub<X>(c_mul<X>(2.0, tau), 1.0);
  double p0 = 1.0, p1 = x, d0 = 0.0, d1 = 1.0;
  g[0] = C.cx[0];
  g[1] = C.cy[0];
  g1[0] = g1[1] = 0.0;
  if (C.D >= 1) {
    g[0] = c_add<X>(g[0], c_mul<X>(C.cx[1], x));
    g[1] = c_add<X>(g[1], c_mul<X>(C.cy[1], x));
    g1[0] = c_add<X>(g1[0], c_mul<X>(C.cx[1], d1));
    g1[1] = c_add<X>(g1[1], c_mul<X>(C.cy[1], d1));
  }
  for (int n = 1; n < C.D; ++n) {
    const double k2 = (double)(2 * n + 1);
    double p2;
    if constexpr (X) {
      const double a = c_mul<X>(k2, x);
      p2 = c_div(c_sub<X>(c_mul<X>(a, p1), c_mul<X>((double)n, p0)), (double)(n + 1));
    } else {
      p2 = p_next(n, x, p1, p0);
    }
    const double d2 = c_add<X>(d0, c_mul<X>(k2, p1));
    const double cxn = C.cx[n + 1], cyn = C.cy[n + 1];
    g[0] = c_add<X>(g[0], c_mul<X>(cxn, p2));
    g[1] = c_add<X>(g[1], c_mul<X>(cyn, p2));
    g1[0] = c_add<X>(g1[0], c_mul<X>(cxn, d2));
    g1[1] = c_add<X>(g1[1], c_mul<X>(cyn, d2));
    p0 = p1; p1 = p2; d0 = d1; d1 = d2;
  }
  g1[0] = c_mul<X>(2.0, g1[0]);
  g1[1] = c_mul<X>(2.0, g1[1]);
}

struct BlendGeom {
  double PLx, PLy, P0x, P0y, Ox, Oy;
};

// rho(xi, eta) (PAPER.md eq. for:blend); xi -> 1 limit per SPEC.md:395
template <bool X>
__host__ __device__ inline void blend(const BlendGeom& B, const CurveRef& C, double xi, double eta, double& x,
                                      double& y) {
  const double om = c_sub<X>(1.0, xi);
  const double lam = c_sub<X>(om, eta);
  const double bx = c_add<X>(c_add<X>(c_mul<X>(lam, B.PLx), c_mul<X>(xi, B.P0x)), c_mul<X>(eta, B.Ox));
  const double by = c_add<X>(c_add<X>(c_mul<X>(lam, B.PLy), c_mul<X>(xi, B.P0y)), c_mul<X>(eta, B.Oy));
  if (!(om > 1e-13)) {
    x = bx;
    y = by;
    return;
  }
  double gx, gy;
  curve_eval<X>(C, om, gx, gy);
  const double Dx = c_sub<X>(c_sub<X>(gx, c_mul<X>(om, B.PLx)), c_mul<X>(xi, B.P0x));
  const double Dy = c_sub<X>(c_sub<X>(gy, c_mul<X>(om, B.PLy)), c_mul<X>(xi, B.P0y));
  const double r = c_div(lam, om);
  x = c_add<X>(bx, c_mul<X>(r, Dx));
  y = c_add<X>(by, c_mul<X>(r, Dy));
}

// rho and its Jacobian [dx/dxi dx/deta; dy/dxi dy/deta]
template <bool X>
__host__ __device__ inline void blend_jac(const BlendGeom& B, const CurveRef& C, double xi, double eta, double& x,
                                          double& y, double J[4]) {
  const double om0 = c_sub<X>(1.0, xi);
  const double om = om0 > 1e-13 ? om0 : 1e-13;
  const double lam = c_sub<X>(om0, eta);
  double g[2], g1[2];
  curve_eval_d1<X>(C, om, g, g1);
  const double bx = c_add<X>(c_add<X>(c_mul<X>(lam, B.PLx), c_mul<X>(xi, B.P0x)), c_mul<X>(eta, B.Ox));
  const double by = c_add<X>(c_add<X>(c_mul<X>(lam, B.PLy), c_mul<X>(xi, B.P0y)), c_mul<X>(eta, B.Oy));
  const double Dx = c_sub<X>(c_sub<X>(g[0], c_mul<X>(om, B.PLx)), c_mul<X>(xi, B.P0x));
  const double Dy = c_sub<X>(c_sub<X>(g[1], c_mul<X>(om, B.PLy)), c_mul<X>(xi, B.P0y));
  double r, drx, dre;
  if constexpr (X) {
    r = c_div(lam, om);
    drx = c_div(-eta, c_mul<X>(om, om));
    dre = c_div(-1.0, om);
  } else {
    const double inv = 1.0 / om;
    r = lam * inv;
    dre = -inv;
    drx = -eta * inv * inv;
  }
  x = c_add<X>(bx, c_mul<X>(r, Dx));
  y = c_add<X>(by, c_mul<X>(r, Dy));
  const double dDx = c_sub<X>(c_sub<X>(B.PLx, g1[0]), B.P0x), dDy = c_sub<X>(c_sub<X>(B.PLy, g1[1]), B.P0y);
  J[0] = c_add<X>(c_add<X>(c_sub<X>(B.P0x, B.PLx), c_mul<X>(drx, Dx)), c_mul<X>(r, dDx));
  J[1] = c_add<X>(c_sub<X>(B.Ox, B.PLx), c_mul<X>(dre, Dx));
  J[2] = c_add<X>(c_add<X>(c_sub<X>(B.P0y, B.PLy), c_mul<X>(drx, Dy)), c_mul<X>(r, dDy));
  J[3] = c_add<X>(c_sub<X>(B.Oy, B.PLy), c_mul<X>(dre, Dy));
}

constexpr int kBlendNewton = 12;  // fixed iteration count: identical iterates on CPU and GPU

template <bool X>
__host__ __device__ inline void newton_step(const BlendGeom& B, const CurveRef& C, double tx, double ty,
                                            double& xi, double& eta, double& dxi, double& deta) {
  double x, y, J[4];
  blend_jac<X>(B, C, xi, eta, x, y, J);
  const double rx = c_sub<X>(tx, x), ry = c_sub<X>(ty, y);
  const double dj = c_sub<X>(c_mul<X>(J[0], J[3]), c_mul<X>(J[1], J[2]));
  if constexpr (X) {
    dxi = c_div(c_sub<X>(c_mul<X>(J[3], rx), c_mul<X>(J[1], ry)), dj);
    deta = c_div(c_sub<X>(c_mul<X>(J[0], ry), c_mul<X>(J[2], rx)), dj);
  } else {
    const double inv = 1.0 / dj;
    dxi = (J[3] * rx - J[1] * ry) * inv;
    deta = (J[0] * ry - J[2] * rx) * inv;
  }
  xi = c_add<X>(xi, dxi);
  eta = c_add<X>(eta, deta);
}

// Newton inverse of the blending map, fixed 12 steps
template <bool X>
__host__ __device__ inline void blend_inverse(const BlendGeom& B, const CurveRef& C, double tx, double ty,
                                              double& xi, double& eta) {
  for (int it = 0; it < kBlendNewton; ++it) {
    double dxi, deta;
    newton_step<X>(B, C, tx, ty, xi, eta, dxi, deta);
  }
}

// Newton inverse to convergence (quadrature points: values, not predicates).
// Quadratic convergence: after a step of size delta the error is O(delta^2),
// so stopping at delta < tol leaves ~tol^2.
__host__ __device__ inline void blend_inverse_tol(const BlendGeom& B, const CurveRef& C, double tx, double ty,
                                                  double& xi, double& eta, double tol = 1e-15) {
  for (int it = 0; it < 40; ++it) {
    double dxi, deta;
    newton_step<false>(B, C, tx, ty, xi, eta, dxi, deta);
    if (fabs(dxi) + fabs(deta) < tol) break;
  }
}

// s~ = argmin_s |v - gamma(s)|, gamma(s) = G(1 - s/L): best of 33 samples,
// then 10 clamped Newton steps on (gamma - v).gamma' = 0
template <bool X>
__host__ __device__ inline double curved_argmin(const CurveRef& C, double vx, double vy) {
  const double L = C.L;
  int best = 0;
  double bd = 1e300;
  for (int i = 0; i <= 32; ++i) {
    double gx, gy;
    curve_eval<X>(C, c_sub<X>(1.0, c_div((double)i, 32.0)), gx, gy);
    const double dx = c_sub<X>(gx, vx), dy = c_sub<X>(gy, vy);
    const double d2 = c_add<X>(c_mul<X>(dx, dx), c_mul<X>(dy, dy));
    if (d2 < bd) {
      bd = d2;
      best = i;
    }
  }
  double s = c_mul<X>(L, c_div((double)best, 32.0));
  for (int it = 0; it < 10; ++it) {
    double g[2], g1[2], g2[2];
    curve_eval_d<X>(C, c_sub<X>(1.0, c_div(s, L)), g, g1, g2);
    const double tx = c_div(-g1[0], L), ty = c_div(-g1[1], L);
    const double LL = c_mul<X>(L, L);
    const double ax = c_div(g2[0], LL), ay = c_div(g2[1], LL);
    const double dx = c_sub<X>(g[0], vx), dy = c_sub<X>(g[1], vy);
    const double phi = c_add<X>(c_mul<X>(dx, tx), c_mul<X>(dy, ty));
    const double dphi = c_add<X>(c_add<X>(c_mul<X>(tx, tx), c_mul<X>(ty, ty)),
                                 c_add<X>(c_mul<X>(dx, ax), c_mul<X>(dy, ay)));
    if (!(dphi > 0.0)) break;
    s = c_sub<X>(s, c_div(phi, dphi));
    s = s < 0.0 ? 0.0 : s;
    s = s > L ? L : s;
  }
  return s;
}

}  // namespace vp
