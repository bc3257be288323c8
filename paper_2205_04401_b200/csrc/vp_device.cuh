// vp_device.cuh -- device-side building blocks of the evaluator.
//
//  * ElemRec: per-element record in HBM (192 B, one contiguous gather per
//    element): the stored vertices, the near-field model 2a per side, the
//    affine map and its inverse, rho0 of the N_n model and the near-field
//    bbox.  Built on the host in vp_api.cu with the same operation order as
//    the oracle so list predicates are bit-reproducible.
//  * exact-rounding predicates (no FMA contraction) shared by the list build
//    (K3), the near sub-simplex acceptance (K4) and the self panel counts (K5).
//  * density<P>: Koornwinder expansion with compile-time recurrence
//    coefficients (koornwinder.hpp:77-113 recurrences, division-free).
#pragma once
#include <cstdint>

#include "koorn.cuh"

namespace vp {

struct alignas(64) ElemRec {
  double x0, y0, x1, y1, x2, y2;  // stored vertices (CCW)
  double ta0, ta1, ta2;           // 2a of the sides v0v1, v1v2, v2v0; ta0 < 0: all-near
  double i00, i01, i10, i11;      // inverse affine map
  double e1x, e1y, e2x, e2y, det; // affine map, det = |J| = 2 area
  double rho0n;                   // rho0 of the N_n (near-rule) model
  double bx0, by0, bx1, by1;      // near-field bbox (conservative)
  double pad;
};
static_assert(sizeof(ElemRec) == 192, "ElemRec layout");

constexpr double kInv4Pi = 0.079577471545947667884;  // 1/(4 pi)
constexpr double kInv2Pi = 0.15915494309189533577;   // 1/(2 pi)
constexpr double kBaryTol = 1e-12;
constexpr int kMaxNearDepth = 40;

#ifdef __CUDACC__

__device__ __forceinline__ double rn_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double rn_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double rn_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double rn_div(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double rn_sqrt(double a) { return __dsqrt_rn(a); }

// |t - P| with separately rounded operations
__device__ __forceinline__ double rn_dist(double tx, double ty, double px, double py) {
  const double dx = rn_sub(tx, px), dy = rn_sub(ty, py);
  return rn_sqrt(rn_add(rn_mul(dx, dx), rn_mul(dy, dy)));
}

// barycentric containment with tolerance; also returns
// the reference coordinates of t
__device__ __forceinline__ bool rn_locate(const ElemRec& E, double tx, double ty, double& xi,
                                          double& eta) {
  const double dx = rn_sub(tx, E.x0), dy = rn_sub(ty, E.y0);
  xi = rn_add(rn_mul(E.i00, dx), rn_mul(E.i01, dy));
  eta = rn_add(rn_mul(E.i10, dx), rn_mul(E.i11, dy));
  const double l0 = rn_sub(rn_sub(1.0, xi), eta);
  return xi >= -kBaryTol && eta >= -kBaryTol && l0 >= -kBaryTol;
}

// t inside the union of the element's three open ellipses
__device__ __forceinline__ bool rn_in_near(const ElemRec& E, double tx, double ty) {
  if (E.ta0 < 0.0) return true;  // all-near model
  const double d0 = rn_dist(tx, ty, E.x0, E.y0);
  const double d1 = rn_dist(tx, ty, E.x1, E.y1);
  const double d2 = rn_dist(tx, ty, E.x2, E.y2);
  return (rn_add(d0, d1) < E.ta0) || (rn_add(d1, d2) < E.ta1) || (rn_add(d2, d0) < E.ta2);
}

// ---------------------------------------------------------------------------
// compile-time Koornwinder recurrence coefficients
__host__ __device__ constexpr double kc_la(int m) { return double(2 * m + 1) / double(m + 1); }
__host__ __device__ constexpr double kc_lb(int m) { return double(m) / double(m + 1); }
__host__ __device__ constexpr double kc_c1(int m, int k) {
  return 2.0 * (k + 1) * (k + (2 * m + 1) + 1) * (2.0 * k + (2 * m + 1));
}
__host__ __device__ constexpr double kc_ja(int m, int k) {
  return (2.0 * k + (2 * m + 1)) * (2.0 * k + (2 * m + 1) + 1) * (2.0 * k + (2 * m + 1) + 2) /
         kc_c1(m, k);
}
__host__ __device__ constexpr double kc_jb(int m, int k) {
  return (2.0 * k + (2 * m + 1) + 1) * (double(2 * m + 1) * double(2 * m + 1)) / kc_c1(m, k);
}
__host__ __device__ constexpr double kc_jc(int m, int k) {
  return 2.0 * (k + (2 * m + 1)) * k * (2.0 * k + (2 * m + 1) + 2) / kc_c1(m, k);
}

// f(x, y) = sum_j cc_j K_j(x, y) where cc_j already includes the
// normalisation c_mn (pre-scaled per element).  ~4 FP64 ops per mode.
template <int P>
__device__ __forceinline__ double density(const double* __restrict__ cc, double x, double y) {
  const double v = 1.0 - x;
  const double u = fma(2.0, y, -v);
  const double v2 = v * v;
  const double t = fma(2.0, x, -1.0);
  double Lm = 1.0, Lprev = 0.0, f = 0.0;
#pragma unroll
  for (int m = 0; m <= P; ++m) {
    double s = cc[koorn_index(m, m)];
    if (m + 1 <= P) {
      const double a = 2 * m + 1;
      double p0 = 1.0;
      double p1 = fma(0.5 * (a + 2.0), t, 0.5 * a);
      s = fma(cc[koorn_index(m, m + 1)], p1, s);
#pragma unroll
      for (int k = 1; m + k + 1 <= P; ++k) {
        const double al = fma(kc_ja(m, k), t, kc_jb(m, k));
        const double p2 = fma(al, p1, -kc_jc(m, k) * p0);
        s = fma(cc[koorn_index(m, m + k + 1)], p2, s);
        p0 = p1;
        p1 = p2;
      }
    }
    f = fma(s, Lm, f);
    if (m < P) {
      const double Ln = (m == 0) ? u : fma(kc_la(m) * u, Lm, -kc_lb(m) * v2 * Lprev);
      Lprev = Lm;
      Lm = Ln;
    }
  }
  return f;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

#endif  // __CUDACC__

}  // namespace vp
